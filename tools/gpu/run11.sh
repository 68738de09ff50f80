set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -x -q --timeout 600 -k "seeded or chained or peer_self or fused_reduce or unfused or two_ranks or loop" > gpurun_out/r2_pytest_nary.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_pytest_nary.log
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.opt 3 > gpurun_out/r2_pull_steps.txt 2>&1; head -8 gpurun_out/r2_pull_steps.txt
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.data 3 > gpurun_out/r2_pull_steps_data.txt 2>&1; grep upd gpurun_out/r2_pull_steps_data.txt | head -4
timeout 300 python tools/pull_profile.py alexconv_b128.data 2 > gpurun_out/r2_pull_steps_conv.txt 2>&1; head -12 gpurun_out/r2_pull_steps_conv.txt
