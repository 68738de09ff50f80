set -x; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "numeric" > gpurun_out/r2_pytest_k7.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_pytest_k7.log
timeout 1200 python -m pytest tests/test_gpu_peer.py -x -q --timeout 900 -k "bench_two" > gpurun_out/r2_pytest_bench2.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_pytest_bench2.log
TPX_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/r2_bench_share2.log 2>&1; echo "share2 exit $?"; grep -v "^\[" gpurun_out/r2_bench_share2.log | tail -1 | cut -c1-300
