cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 900 -k "benched" > gpurun_out/g1_benched.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q --timeout 1200 -k "not benched" > gpurun_out/g1_fullsize.log 2>&1
tail -3 gpurun_out/g1_benched.log gpurun_out/g1_fullsize.log
