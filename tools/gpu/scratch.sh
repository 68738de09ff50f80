timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -q -x --timeout 900 -k "peer or forced or loop or graph" 2>&1 | tail -2
TPX_SOLO=0,8 timeout 300 python tools/step_profile.py cfg2_mlp5x8192_b512.loop.k3 3 | head -8
TPX_SOLO=0,4 timeout 300 python tools/step_profile.py cfg2_mlp5x8192_b512.loop.k2 3 | head -8
