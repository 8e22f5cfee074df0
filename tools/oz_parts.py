"""Per-kernel times of one emulated Gram / tall GEMM on config-2 shapes (torch profiler)."""
import os
import sys
import torch
from torch.profiler import profile, ProfilerActivity

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import kernels as K

n, m, ld = 110592, 523, 528
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
AX = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
G = torch.randn((m, m), generator=g, device="cuda", dtype=torch.float64) / 30
Y = torch.empty((n, ld), device="cuda", dtype=torch.float64)[:, :m]
C = torch.empty((m, m), device="cuda", dtype=torch.float64)
for what, fn in [("gram", lambda: K.gram(X, AX, C)), ("ts", lambda: K.tsgemm([X], [G], [Y], alpha=-1.0, beta=1.0, zs=[AX]))]:
    with K.fp64_emulation(True):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
    tot = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            tot[e.name] = tot.get(e.name, 0.0) + e.device_time / 5 / 1000
    print(what, {k[:40]: round(v, 4) for k, v in sorted(tot.items(), key=lambda x: -x[1])})
