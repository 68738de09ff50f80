timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.loop 3 > /tmp/a.txt; head -1 /tmp/a.txt
timeout 300 python tools/pull_profile.py cfg1_mlp3x1024_b64.loop 3 > /tmp/b.txt; head -1 /tmp/b.txt
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q --timeout 900 -k "ranks_on_one_gpu or peer_self" 2>&1 | tail -2
