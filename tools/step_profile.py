"""Per lowered step device times (CUDA events) of one plan: where a train step's time goes.

    python tools/step_profile.py <plan stem under plans/> [top]"""
import gzip
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_04170_b200.executor import FLAG_FUSE, Context, PlanExecutor  # noqa: E402

for kv in filter(None, os.environ.get("TPX_GEMM_KNOBS", "").split(",")):  # gemm.cu debug knobs
    import ctypes
    from paper_1805_04170_b200 import native
    k, v = kv.split(":")
    native.lib().tpx_debug_gemm_mn_desc(ctypes.c_uint(int(k)), ctypes.c_uint(int(v)))
stem = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
text = gzip.open(os.path.join(ROOT, "plans", stem + ".plan.json.gz"), "rt").read()
# TPX_SOLO=rank,world: that rank of a world-rank peer plan alone (TPX_FLAG_PEER_SOLO timing)
solo = os.environ.get("TPX_SOLO")
ctx = Context(0, *[int(x) for x in solo.split(",")]) if solo else Context(0)
ex = PlanExecutor(ctx, text, precision=0,
                  flags=FLAG_FUSE | int(os.environ.get("TPX_EXTRA_FLAGS", "0")) | (32 | 128 if solo else 0))
ex.init_inputs(7)
for _ in range(3):
    ex.execute()
ex.enable_timing(True)
runs = []
for _ in range(5):
    ex.execute()
    runs.append(ex.last_step_times())
ms = [statistics.median(x) for x in zip(*runs)]
steps = ex.describe()["main"]["steps"]
tot = sum(ms)
print(f"{stem}: {len(steps)} steps, {tot:.3f} ms")
by = {}
for st, t in zip(steps, ms):
    key = (st["kind"], st["what"])
    by[key] = by.get(key, 0.0) + t
for key, t in sorted(by.items(), key=lambda kv: -kv[1]):
    print(f"  {key[0]:5s} {key[1]:12s} {t:8.3f} ms {100 * t / tot:5.1f}%")
for st, t in sorted(zip(steps, ms), key=lambda p: -p[1])[:top]:
    extra = st.get("shapes", [[]])[0] if st["kind"] == "gemm" else st.get("descs", "")
    gbs = f"{st['bytes'] / (t * 1e-3) / 1e9:7.0f} GB/s" if st.get("bytes") and st["kind"] != "gemm" else ""
    print(f"  {t:8.3f} ms  {st['kind']:5s} {st['what']:12s} {st['op']:10s} {extra} {gbs}")
