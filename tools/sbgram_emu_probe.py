"""Would the q = 64 pencil Grams gain from the emulated products?  17 subblocks of [X_j W_j P_j]
(n x 192) at config-3 size: DMMA Grams vs emulated Grams with S sliced once (coldigits)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import kernels as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
nb, d = 17, 192
g = torch.Generator(device="cuda").manual_seed(0)
S = [torch.randn((n, d), generator=g, device="cuda", dtype=torch.float64) for _ in range(nb)]
AS = [torch.randn((n, d), generator=g, device="cuda", dtype=torch.float64) for _ in range(nb)]
A = torch.empty((d, d), device="cuda", dtype=torch.float64)
B = torch.empty((d, d), device="cuda", dtype=torch.float64)
buf = None


def dmma():
    with K.fp64_emulation(False):
        for j in range(nb):
            K.gram(S[j], AS[j], A)
            K.gram(S[j], S[j], B, symmetric=True)


def emu():
    global buf
    with K.fp64_emulation(True):
        for j in range(nb):
            dg = K.coldigits(S[j], buf)
            buf = dg.buf
            K.gram(S[j], AS[j], A, xdig=dg)
            K.gram(S[j], S[j], B, symmetric=True, xdig=dg)


def t(fn, reps=5):
    for _ in range(2):
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


print(f"n = {n}: 17 x (S^T AS, S^T S) with d = 192: DMMA {t(dmma):.2f} ms, emulated (S sliced once) {t(emu):.2f} ms")
