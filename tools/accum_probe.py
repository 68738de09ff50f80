"""Tensor-core accumulation probe on the reference's own data (GPU): the cfg2 k=0 bwd_w4 and the
AlexNet-style conv bwd_k5 operands as the fp64 oracle produces them (oracle/torch_oracle.py),
through the kernel (TF32 and 3xTF32), against emulations of the MMA's arithmetic on the same
operands: tf32 operand truncation with the products summed exactly (floor), summed per
8-deep MMA step into an fp32 accumulator rounded to nearest, or toward zero, and the same with
the k range cut into chains of C k-blocks summed in fp32 (round to nearest).

    python tools/accum_probe.py   (writes gpurun_out/accum_probe.json)
"""
import gzip
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import torch_oracle as T  # noqa: E402
from paper_1805_04170_b200 import native  # noqa: E402


def nw(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max()).item()


def trunc(x):
    return (x.float().contiguous().view(torch.int32) & ~0x1FFF).view(torch.float32)


def rz(v64):
    f = v64.float()
    over = f.double().abs() > v64.abs()
    return torch.where(over, torch.nextafter(f, torch.zeros_like(f)), f)


def emulate(A, B, mode, chain_kb=0, step=8):
    """A [K, M], B [K, N] fp32 (already tf32-valued), out = A^T B with an fp32 accumulator
    updated once per `step` k (one MMA instruction); chains of chain_kb*32 k summed in fp32."""
    K = A.shape[0]
    chain = chain_kb * 32 if chain_kb else K
    total = torch.zeros((A.shape[1], B.shape[1]), dtype=torch.float32, device=A.device)
    for c0 in range(0, K, chain):
        acc = torch.zeros_like(total)
        for k0 in range(c0, min(K, c0 + chain), step):
            part = A[k0:k0 + step].double().t() @ B[k0:k0 + step].double()
            v = acc.double() + part
            acc = rz(v) if mode == "rz" else v.float()
        total = (total.double() + acc.double()).float()
    return total


def main():
    out = {}
    cases = []
    P = json.loads(gzip.open(os.path.join(ROOT, "plans", "cfg2_mlp5x8192_b512.opt.k0.plan.json.gz"), "rt").read())
    serial = T.serial_execute(P["graph"], 7, device="cuda")
    cases.append(("cfg2_bwd_w4", serial["x3"].float(), serial["g4"].float()))
    cases.append(("cfg2_bwd_w1", serial["x0"].float(), serial["g1"].float()))
    del serial
    torch.cuda.empty_cache()
    for name, A, B in cases:
        M, N = A.shape[1], B.shape[1]
        ref = A.double().t() @ B.double()
        At, Bt = trunc(A), trunc(B)
        row = {"floor_trunc_exact_sum": nw(At.double().t() @ Bt.double(), ref)}
        for prec, label in ((0, "kernel_tf32"), (1, "kernel_3xtf32")):
            C = torch.empty((M, N), device="cuda")
            native.gemm(A, B, True, False, C, precision=prec)
            torch.cuda.synchronize()
            row[label] = nw(C, ref)
            if prec == 0:
                Ck = C
        # emulations on a slice of rows (the full 8192 x 8192 is 64 x 512 sequential updates)
        rows = slice(0, 1024)
        refs = ref[rows]
        for mode in ("rn", "rz"):
            for ch in (0, 16, 4, 1):
                e = emulate(At[:, rows], Bt, mode, ch)
                row[f"emul_tf32_{mode}_chain{ch or 'all'}"] = nw(e, refs)
                if mode == "rz" and ch == 0:
                    row["kernel_vs_emul_rz"] = nw(Ck[rows], e.double())
                    row["kernel_tf32_rows"] = nw(Ck[rows], refs)
        out[name] = row
        print(name, json.dumps(row, indent=1), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "accum_probe.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
