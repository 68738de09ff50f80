set -x; mkdir -p gpurun_out/tmp
for cfg in "tn_sgd:8192 8192 512 1 0 3,6" "tn_plain:8192 8192 512 1 0 -"; do
  name=${cfg%%:*}; shape=${cfg#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 3 -c 1 -f -o gpurun_out/tmp/r2_ncu_$name python tools/gemm_check.py --one $shape > gpurun_out/r2_ncu_$name.log 2>&1
  ncu -i gpurun_out/tmp/r2_ncu_$name.ncu-rep --page raw --csv > gpurun_out/r2_ncu_${name}_raw.csv 2>&1
  ncu -i gpurun_out/tmp/r2_ncu_$name.ncu-rep --page details --csv > gpurun_out/r2_ncu_${name}_details.csv 2>&1
  python tools/ncu_stalls.py gpurun_out/tmp/r2_ncu_$name.ncu-rep 60 > gpurun_out/r2_ncu_${name}_stalls.txt 2>&1
  ncu -i gpurun_out/tmp/r2_ncu_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/tmp/src.csv 2>&1; gzip -c gpurun_out/tmp/src.csv > gpurun_out/r2_ncu_${name}_source.csv.gz
done
rm -rf gpurun_out/tmp
