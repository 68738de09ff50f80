"""bench.py's own N > 1 launcher on CPU: `--gpus 2` without a torchrun environment re-launches
itself as 2 ranks through torch.distributed.run on 127.0.0.1; with the reference arm (CPU, no GPU
needed) rank 0 prints the one JSON line and rank 1 exits 0 without work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
def test_bench_self_launches_two_ranks_reference_arm():
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library not built")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--config", "cfg1_mlp3x1024_b64", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=560, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "launching 2 ranks" in out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "cfg1_mlp3x1024_b64"
