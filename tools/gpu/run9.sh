set -x; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2_pytest_gpu_3.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/r2_pytest_gpu_3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/r2_smoke.log
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.opt 3 > gpurun_out/r2_pull_steps.txt 2>&1; cat gpurun_out/r2_pull_steps.txt | head -40
timeout 300 python tools/pull_profile.py alexconv_b128.data 2 > gpurun_out/r2_pull_steps_conv.txt 2>&1; head -20 gpurun_out/r2_pull_steps_conv.txt
timeout 600 ncu --set full --clock-control none -k regex:nary -c 12 -f -o gpurun_out/pull python tools/pull_profile.py cfg2_mlp5x8192_b512.opt 3 > /dev/null 2>&1; echo "ncu pull rc=$?"
ncu -i gpurun_out/pull.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size > gpurun_out/r2_ncu_pull_raw.csv 2>&1; rm -f gpurun_out/pull.ncu-rep
timeout 900 python bench.py > gpurun_out/r2_bench_2.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/r2_bench_2.log | cut -c1-600
