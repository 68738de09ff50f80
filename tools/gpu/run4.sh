set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q --timeout 850 -k two_ranks > gpurun_out/r2_pytest_peer2.log 2>&1; echo "peer exit $?"
tail -3 gpurun_out/r2_pytest_peer2.log
timeout 900 python tools/epi_sweep.py base "o4s4=15:4,16:4" "o6s3=15:6,4:3" "o7s3=15:7,4:3" "o5s3=15:5,4:3" "noload=12:0" "o7s3nl=15:7,4:3,12:0" "spin=5:2" > gpurun_out/r2_epi_sweep.txt 2>&1; echo "sweep exit $?"
cat gpurun_out/r2_epi_sweep.txt | grep sweep
