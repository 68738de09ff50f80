mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/s3_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s3_pytest_gpu.log
timeout 600 python bench.py --no-variants > gpurun_out/s3_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/s3_bench.log | cut -c1-400
