"""One plan, a few steps: the process ncu wraps for per-kernel captures of a whole train step.

    ncu ... -k regex:gemm -s 30 -c 15 python tools/ncu_step.py [config] [steps]
(2 warm-up steps of 15 GEMM launches for cfg2 at k=0 are skipped by -s 30.)"""
import gzip
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_04170_b200.executor import FLAG_FUSE, Context, PlanExecutor  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2_mlp5x8192_b512"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
text = gzip.open(os.path.join(ROOT, "plans", f"{cfg}.opt.k0.plan.json.gz"), "rt").read()
ex = PlanExecutor(Context(0), text, precision=0, flags=FLAG_FUSE)
ex.init_inputs(7)
for _ in range(steps):
    ex.execute()
ex.synchronize()
print("steps", steps, [(s["op"], s.get("shapes", [[0]])[0]) for s in ex.describe()["main"]["steps"] if s["kind"] == "gemm"])
