"""One emulated product on config-2 shapes for ncu: python tools/oz_one.py {ts|gram|ts4}"""
import os
import sys
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import kernels as K

what = sys.argv[1] if len(sys.argv) > 1 else "ts"
n, m = 110592, 523
ld = 528
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
AX = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
G = torch.randn((m, m), generator=g, device="cuda", dtype=torch.float64) / 30
s = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) + 0.5
Y = torch.empty((n, ld), device="cuda", dtype=torch.float64)[:, :m]
C = torch.empty((m, m), device="cuda", dtype=torch.float64)
with K.fp64_emulation(True):
    for _ in range(2):
        if what == "ts":
            K.tsgemm([X], [G], [Y], alpha=-1.0, beta=1.0, zs=[AX], rowscale=s)
        else:
            K.gram(X, AX, C)
torch.cuda.synchronize()
