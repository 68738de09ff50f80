import gzip, json, os, sys
sys.path.insert(0, os.getcwd())
from paper_1805_04170_b200.executor import FLAG_FUSE, Context, PlanExecutor
for stem in ["cfg2_mlp5x8192_b512.loop.k3", "cfg2_mlp5x8192_b512.opt.k0"]:
    text = gzip.open(f"plans/{stem}.plan.json.gz", "rt").read()
    ex = PlanExecutor(Context(0), text, precision=0, flags=FLAG_FUSE)
    for s in ex.describe()["main"]["steps"]:
        if s["kind"] == "gemm":
            print(stem, {k: s.get(k) for k in ("op", "shapes", "bn", "pair", "swap", "stream_k", "group", "nprob", "units")})
