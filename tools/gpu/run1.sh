set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/r2_pytest_gpu_1.log 2>&1; echo "pytest exit $?"
tail -30 gpurun_out/r2_pytest_gpu_1.log
timeout 600 python bench.py > gpurun_out/r2_bench_1.log 2>&1; echo "bench exit $?"
tail -5 gpurun_out/r2_bench_1.log
