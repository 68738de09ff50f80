"""Same-box sanity reference: cuBLAS (torch.matmul, TF32 and BF16) on the executor's GEMM shapes.
Not part of the product; prints median ms and TFLOP/s per shape."""
import torch

torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cudnn.allow_tf32 = True


def t(M, N, K, ta, tb, dtype, reps=5, iters=20):
    A = torch.rand((K, M) if ta else (M, K), device="cuda", dtype=dtype)
    B = torch.rand((N, K) if tb else (K, N), device="cuda", dtype=dtype)
    a = A.t() if ta else A
    b = B.t() if tb else B
    for _ in range(3):
        torch.matmul(a, b)
    res = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        res.append(s.elapsed_time(e) / iters)
    ms = sorted(res)[len(res) // 2]
    return ms, 2 * M * N * K / ms / 1e9


for shape in [(512, 8192, 8192, False, False), (512, 8192, 8192, False, True), (8192, 8192, 512, True, False),
              (64, 8192, 8192, False, False), (4, 32768, 32768, False, False), (4096, 4096, 4096, False, False),
              (8192, 8192, 8192, False, True)]:
    for dt in (torch.float32, torch.bfloat16):
        ms, tf = t(*shape, dt)
        print(f"cublas {str(dt).split('.')[-1]:9s} {shape}: {ms:.3f} ms {tf:.1f} TFLOP/s")
