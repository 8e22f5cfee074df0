"""Tall-GEMM core time vs shape and column offset of the views (bench's live state uses a
513-wide view at column offset 10 of 528-stride blocks)."""
import os
import sys
import statistics
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import kernels as K, _lib

lib = _lib.load()
n = 110592
g = torch.Generator(device="cuda").manual_seed(0)
for (m, off) in [(523, 0), (513, 0), (513, 10), (513, 2), (512, 0), (512, 16)]:
    ld = 528
    Xb = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)
    Zb = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)
    Yb = torch.empty((n, ld), device="cuda", dtype=torch.float64)
    X, Z, Y = Xb[:, off:off + m], Zb[:, off:off + m], Yb[:, off:off + m]
    G = torch.randn((m, m), generator=g, device="cuda", dtype=torch.float64) / 30
    with K.fp64_emulation(True):
        f = lambda: K.tsgemm([X], [G], [Y], alpha=-1.0, beta=1.0, zs=[Z])
        f()
        torch.cuda.synchronize()
        ks = []
        for _ in range(5):
            lib.bk_ozaki_timing(1)
            f()
            ks.append(lib.bk_ozaki_kernel_ms())
        lib.bk_ozaki_timing(0)
    print(f"m {m} off {off}: kernel {statistics.median(ks):.3f} ms", flush=True)
