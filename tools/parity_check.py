"""Quick GPU parity sweep over the golden plans (development tool; tests/ hold the gates).

For each golden plan: (1) chained run from seeded inputs vs the numpy fp64 oracle, every
holder; (2) per-op teacher-forced run (oracle values written into the input holders, only
that op's steps executed) vs the oracle output holders.
"""
import glob
import gzip
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import tileplan_oracle as O  # noqa: E402
from paper_1805_04170_b200.executor import Context, PlanExecutor  # noqa: E402


def normwise(got, want):
    d = np.abs(got - want).max() if got.size else 0.0
    return d / max(np.abs(want).max(), 1e-30) if got.size else 0.0


PREC = 1 if "--fp32" in sys.argv else 0


def run_case(ctx, path, flags):
    plan_text = gzip.open(path, "rt").read()
    P = json.loads(plan_text)
    seed = int(path.split(".s")[-1].split(".")[0])
    serial = O.serial_execute(P["graph"], seed)
    vals = O.execute_nodes(P, serial)
    ex = PlanExecutor(ctx, plan_text, precision=PREC, flags=flags)
    ex.init_inputs(seed)
    ex.execute()
    ex.synchronize()
    worst_chain = 0.0
    worst_t = ""
    for t, hs in P["holders"].items():
        for hid in hs:
            e = normwise(ex.read_node(hid), vals[hid])
            if e > worst_chain:
                worst_chain, worst_t = e, t
    # teacher-forced per op
    worst_op = 0.0
    worst_o = ""
    ex2 = PlanExecutor(ctx, plan_text, precision=PREC, flags=0)
    ex2.init_inputs(seed)
    for op in P["graph"]["ops"]:
        for t in op["inputs"]:
            for hid in P["holders"][t]:
                ex2.write_node(hid, vals[hid])
        ex2.execute_op(op["id"])
        ex2.synchronize()
        for hid in P["holders"][op["output"]]:
            e = normwise(ex2.read_node(hid), vals[hid])
            if e > worst_op:
                worst_op, worst_o = e, op["id"]
    ex.close()
    ex2.close()
    return worst_chain, worst_t, worst_op, worst_o


def main():
    ctx = Context(0)
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    pat = args[0] if args else "*"
    files = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", pat + ".plan.json.gz")))
    bad = 0
    for f in files:
        t0 = time.time()
        try:
            wc, wt, wo, woo = run_case(ctx, f, 1)
            ok = wo <= 2e-3
            bad += not ok
            print(f"{'ok ' if ok else 'BAD'} {os.path.basename(f)[:-13]:45s} chained={wc:.2e}({wt}) "
                  f"per-op={wo:.2e}({woo}) {time.time() - t0:.1f}s", flush=True)
        except Exception as ex:  # noqa: BLE001
            bad += 1
            print(f"ERR {os.path.basename(f)}: {ex}", flush=True)
    print("BAD", bad, "of", len(files))


if __name__ == "__main__":
    main()
