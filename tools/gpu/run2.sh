set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q --timeout 850 > gpurun_out/r2_pytest_peer.log 2>&1; echo "peer exit $?"
tail -30 gpurun_out/r2_pytest_peer.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 --deselect tests/test_gpu_peer.py > gpurun_out/r2_pytest_gpu_2.log 2>&1; echo "pytest exit $?"
tail -20 gpurun_out/r2_pytest_gpu_2.log
