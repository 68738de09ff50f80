set -x; mkdir -p gpurun_out
for cfg in "tn_sgd:8192 8192 512 1 0 3,6" "tn_plain:8192 8192 512 1 0 -" "nn_sgd:8192 8192 512 0 0 3,6" "nt_sgd:8192 8192 512 0 1 3,6"; do
  name=${cfg%%:*}; shape=${cfg#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 3 -c 1 -f -o gpurun_out/r2_ncu_$name python tools/gemm_check.py --one $shape > gpurun_out/r2_ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  python tools/gemm_check.py --one $shape 2>&1 | tail -1
done
