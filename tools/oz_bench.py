"""A/B timing of the FP64 products on config-2 shapes: DMMA kernels vs the int8 Ozaki kernels
(CUDA events, median of 10 after warm-up).  python tools/oz_bench.py [n] [m]"""
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import kernels as K

n = int(sys.argv[1]) if len(sys.argv) > 1 else 110592
m = int(sys.argv[2]) if len(sys.argv) > 2 else 523
g = torch.Generator(device="cuda").manual_seed(0)
ld = (m + 15) // 16 * 16
X = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
AX = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
W = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
P = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
G = torch.randn((m, m), generator=g, device="cuda", dtype=torch.float64) / 30
R = torch.triu(G)
s = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) + 0.5
outs = [torch.empty((n, ld), device="cuda", dtype=torch.float64)[:, :m] for _ in range(4)]
C = torch.empty((m, m), device="cuda", dtype=torch.float64)
metric = torch.zeros(1, device="cuda", dtype=torch.float64)

cases = {
    "gram X^T AX": lambda: K.gram(X, AX, C),
    "gram X^T X sym": lambda: K.gram(X, X, C, symmetric=True),
    "tsgemm W=s(AX-XG)": lambda: K.tsgemm([X], [G], [outs[0]], alpha=-1.0, beta=1.0, zs=[AX], rowscale=s),
    "tsgemm +metric": lambda: K.tsgemm([X], [G], [outs[0]], alpha=-1.0, beta=1.0, zs=[AX], metric=metric,
                                       ksplit=m - 10, nsplit=m - 10),
    "tsgemm x4 proj": lambda: K.tsgemm([X, AX, X, AX], [G, G, G, G], outs, alpha=-1.0, beta=1.0,
                                       zs=[W, P, W, P]),
    "tsgemm upper X R^-1": lambda: K.tsgemm([X], [R], [outs[0]], upper=True),
}


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for name, fn in cases.items():
    with K.fp64_emulation(False):
        td = t(fn)
    with K.fp64_emulation(True):
        te = t(fn)
    print(f"{name:24s} dmma {td:7.3f} ms   ozaki {te:7.3f} ms   x{td / te:5.2f}", flush=True)
