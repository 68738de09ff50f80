set -x; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2_pytest_gpu_4.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_pytest_gpu_4.log
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.opt 3 > gpurun_out/r2_pull_steps.txt 2>&1; head -8 gpurun_out/r2_pull_steps.txt
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.loop 3 > gpurun_out/r2_pull_steps_loop.txt 2>&1; head -16 gpurun_out/r2_pull_steps_loop.txt
timeout 300 python tools/pull_profile.py alexconv_b128.data 2 > gpurun_out/r2_pull_steps_conv.txt 2>&1; head -12 gpurun_out/r2_pull_steps_conv.txt
TPX_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/r2_bench_share2.log 2>&1; echo "share2 exit $?"; grep -v "^\[" gpurun_out/r2_bench_share2.log | tail -2 | cut -c1-400; grep "peer arenas" gpurun_out/r2_bench_share2.log | head -2
timeout 900 python bench.py > gpurun_out/r2_bench_3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/r2_bench_3.log | cut -c1-300
