"""One tiled-on-one-GPU train step through the peer-pull path, for ncu (profiles/r2_ncu_pull*):
    python tools/pull_profile.py [plan-stem] [k]
Runs plans/<stem>.k<k> with FUSE | FORCE_XCHG | PEER (every cross-device fetch one pull
launch per phase, against the rank's own arena), prints every pull / reduce step with its
algorithmic bytes (read + write, as describe() counts them) in launch order, so the ncu launch
list can be matched step by step."""
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_04170_b200.executor import FLAG_FORCE_XCHG, FLAG_FUSE, FLAG_PEER, Context, PlanExecutor  # noqa: E402

stem = sys.argv[1] if len(sys.argv) > 1 else "cfg2_mlp5x8192_b512.opt"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
text = gzip.open(os.path.join(ROOT, "plans", f"{stem}.k{k}.plan.json.gz"), "rt").read()
ex = PlanExecutor(Context(0), text, precision=0, flags=FLAG_FUSE | FLAG_FORCE_XCHG | FLAG_PEER)
ex.init_inputs(7)
for _ in range(2):
    ex.execute()
ex.synchronize()
ex.enable_timing(True)
ex.execute()
times = ex.last_step_times()
steps = ex.describe()["main"]["steps"]
rows = []
syncs = [t for t, s in zip(times, steps) if s["kind"] == "sync"]
if syncs:
    print(f"sync steps: {len(syncs)}, {sum(syncs) * 1e3:.1f} us total, {sum(syncs) / len(syncs) * 1e3:.2f} us each "
          f"(step total {sum(times) * 1e3:.1f} us)")
for t, s in zip(times, steps):
    if s["kind"] == "nary":
        gbs = s["bytes"] / (t * 1e-3) / 1e9 if t > 0 else 0
        rows.append({"op": s["op"], "what": s["what"], "descs": s["descs"], "bytes": s["bytes"], "ms": t,
                     "GB/s": gbs, "pull": s.get("pull", 0), "chained": s.get("chained", 0)})
        print(f"{s['op']:10s} {s['what']:8s} descs={s['descs']:4d} bytes={s['bytes']:12d} {t * 1e3:8.1f} us {gbs:7.0f} GB/s")
with open(os.path.join(ROOT, "gpurun_out", f"pull_steps_{stem}.k{k}.json"), "w") as f:
    json.dump(rows, f, indent=1)
