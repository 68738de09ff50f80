"""HBM practical bandwidth for the bwd_w epilogue's traffic mix (torch kernels, for reference)."""
import torch

n = 8192 * 8192
gw, w = torch.rand(n, device="cuda"), torch.rand(n, device="cuda")
wd, wn, c = torch.empty_like(gw), torch.empty_like(gw), torch.empty_like(gw)


def t(f, reps=20):
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


ms = t(lambda: c.copy_(gw)); print(f"hbm copy 1r1w: {ms*1e3:.1f} us {2*4*n/ms/1e9:.2f} TB/s")
ms = t(lambda: torch.mul(gw, 0.01, out=wd)); print(f"hbm scale 1r1w: {ms*1e3:.1f} us {2*4*n/ms/1e9:.2f} TB/s")
ms = t(lambda: torch.sub(w, wd, out=wn)); print(f"hbm sub 2r1w: {ms*1e3:.1f} us {3*4*n/ms/1e9:.2f} TB/s")
ms = t(lambda: c.fill_(1.0)); print(f"hbm fill 0r1w: {ms*1e3:.1f} us {4*n/ms/1e9:.2f} TB/s")
ms = t(lambda: gw.sum()); print(f"hbm sum 1r0w: {ms*1e3:.1f} us {4*n/ms/1e9:.2f} TB/s")
