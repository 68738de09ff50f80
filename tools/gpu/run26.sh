timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.loop 3 | head -3
timeout 300 python tools/pull_profile.py cfg1_mlp3x1024_b64.loop 3 | head -3
