mkdir -p gpurun_out/probe
python tools/gemm_probe_both.py || exit 1
timeout 600 ncu --set full --clock-control none -k regex:"^(?!.*(elementwise|distribution|fill|uniform|copy)).*" -f -o gpurun_out/probe/both python tools/gemm_probe_both.py > gpurun_out/probe/both.log 2>&1; echo "ncu $?"
ls -la gpurun_out/probe
ncu -i gpurun_out/probe/both.ncu-rep --page raw --csv > gpurun_out/probe/both_raw.csv 2>&1
ncu -i gpurun_out/probe/both.ncu-rep --page details --csv > gpurun_out/probe/both_details.csv 2>&1
rm -f gpurun_out/probe/both.ncu-rep; gzip gpurun_out/probe/*.csv; ls -la gpurun_out/probe
