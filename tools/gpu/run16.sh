set -x; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_peer.py -x -q --timeout 900 -k "ranks_on_one_gpu or bench_two" > gpurun_out/r2_pytest_peer_multi.log 2>&1; echo "peer exit $?"; tail -15 gpurun_out/r2_pytest_peer_multi.log
