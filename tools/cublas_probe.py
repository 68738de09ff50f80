"""ncu probe of cuBLAS on the cfg2 GEMM shapes (not product): one launch per shape after warm-up,
so `ncu --set full -k regex:'^(?!.*tpx)'` captures cuBLAS's kernel choice (name = tile/cluster
shape), its tensor-pipe activity and smem traffic next to our own kernels' captures."""
import sys
import torch

torch.backends.cuda.matmul.allow_tf32 = True
dt = torch.bfloat16 if "bf16" in sys.argv else torch.float32
for (M, N, K, ta, tb) in [(512, 8192, 8192, False, False), (512, 8192, 8192, False, True),
                          (8192, 8192, 512, True, False)]:
    A = torch.rand((K, M) if ta else (M, K), device="cuda", dtype=dt)
    B = torch.rand((N, K) if tb else (K, N), device="cuda", dtype=dt)
    a = A.t() if ta else A
    b = B.t() if tb else B
    torch.cuda.nvtx.range_push(f"probe {M}x{N}x{K} ta={ta} tb={tb}")
    torch.matmul(a, b)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
