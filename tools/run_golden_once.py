"""Execute one golden plan once (e.g. under compute-sanitizer) and print its GEMM launches.

    python tools/run_golden_once.py [stem under tests/golden/] [precision]"""
import gzip
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_04170_b200.executor import Context, PlanExecutor  # noqa: E402

stem = sys.argv[1] if len(sys.argv) > 1 else "alexr_conv_b4.data.k1.s7"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
text = gzip.open(os.path.join(ROOT, "tests", "golden", stem + ".plan.json.gz"), "rt").read()
ex = PlanExecutor(Context(0), text, precision=prec, flags=1)
for s in ex.describe()["main"]["steps"]:
    if s["kind"] == "gemm":
        print(s)
ex.init_inputs(int(stem.rsplit(".s", 1)[1]))
ex.execute()
ex.synchronize()
print("ok")
