"""Small launches of every kernel family for compute-sanitizer (racecheck / synccheck / memcheck):
the CTA-pair GEMM with the fused SGD epilogue and the operand-loader warp, a stream-K GEMM
(partial tiles + flags), a 3xTF32 GEMM, bf16 pair, and a plan step through the peer-pull path
(FORCE_XCHG | PEER: pulls, sync counters, barrier, fused reduce + SGD).  Prints each GEMM's
variant so the log shows what was covered.  Development / evidence tool, not a test."""
import gzip
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_04170_b200 import native  # noqa: E402

SHAPES = [("pair TN + scale/sub", 2048, 2048, 512, True, False, [3, 6], 0),
          ("pair NN", 512, 4096, 1024, False, False, None, 0),
          ("stream-K small-M", 64, 2048, 4096, False, False, [1], 0),
          ("3xTF32", 256, 512, 1024, False, True, [2], 1),
          ("bf16 pair TN + scale/sub", 2048, 2048, 512, True, False, [3, 6], 2)]
for label, M, N, K, ta, tb, epi, prec in SHAPES:
    dt = torch.bfloat16 if prec == 2 else torch.float32
    A = torch.rand((K, M) if ta else (M, K), device="cuda").to(dt)
    B = torch.rand((N, K) if tb else (K, N), device="cuda").to(dt)
    C = torch.empty((M, N), device="cuda", dtype=dt)
    W = torch.rand((M, N), device="cuda").to(dt)
    outs = [torch.empty((M, N), device="cuda", dtype=dt) for _ in (epi or [])]
    e = [(op, 0.01, W if op >= 4 else None, o) for op, o in zip(epi or [], outs)]
    native.gemm(A, B, ta, tb, C, epi=e, precision=1 if prec == 1 else prec)
    torch.cuda.synchronize()
    print(label, (M, N, K, ta, tb), native.last_launch(), flush=True)

from paper_1805_04170_b200.executor import FLAG_FORCE_XCHG, FLAG_FUSE, FLAG_PEER, Context, PlanExecutor  # noqa: E402
ctx = Context(0)
for stem in ("mlp_train_d2.data.k2.s33", "cfg1_mlp3x1024_b64.opt.k1.s7"):
    text = gzip.open(os.path.join(ROOT, "tests", "golden", stem + ".plan.json.gz"), "rt").read()
    ex = PlanExecutor(ctx, text, precision=0, flags=FLAG_FUSE | FLAG_FORCE_XCHG | FLAG_PEER)
    ex.init_inputs(7)
    ex.execute()
    ex.execute()
    ex.synchronize()
    print("peer plan", stem, ex.describe()["sync_points"], "sync points", flush=True)
    ex.close()
print("sanitize run done")
