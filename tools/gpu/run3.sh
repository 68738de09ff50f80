set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q --timeout 850 > gpurun_out/r2_pytest_peer.log 2>&1; echo "peer exit $?"
tail -30 gpurun_out/r2_pytest_peer.log
