set -x; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -x -q --timeout 900 > gpurun_out/r2_pytest_nary2.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_pytest_nary2.log
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.loop 3 > gpurun_out/r2_pull_steps_loop.txt 2>&1; grep reduce gpurun_out/r2_pull_steps_loop.txt | head -5
timeout 300 python tools/pull_profile.py alexconv_b128.data 2 > gpurun_out/r2_pull_steps_conv.txt 2>&1; grep reduce gpurun_out/r2_pull_steps_conv.txt | head -5
