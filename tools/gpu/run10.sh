set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -x -q --timeout 600 -k "seeded or chained_fp32 or peer_self or fused_reduce or unfused or two_ranks" > gpurun_out/r2_pytest_nary.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_pytest_nary.log
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.opt 3 > gpurun_out/r2_pull_steps.txt 2>&1; head -8 gpurun_out/r2_pull_steps.txt
timeout 300 python tools/pull_profile.py alexconv_b128.data 2 > gpurun_out/r2_pull_steps_conv.txt 2>&1; head -12 gpurun_out/r2_pull_steps_conv.txt
timeout 900 python tools/epi_sweep.py base "dyn=10:0" "promo128=7:3" "promo256=7:4" "nostream=8:1" > gpurun_out/r2_epi_sweep2.txt 2>&1; grep sweep gpurun_out/r2_epi_sweep2.txt
