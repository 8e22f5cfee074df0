"""Tall-GEMM core time cold vs after 6 s of back-to-back emulated products, with the SM clock."""
import os
import subprocess
import sys
import statistics
import time
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import kernels as K, _lib

lib = _lib.load()
n, m, ld = 110592, 523, 528
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
Z = torch.randn((n, ld), generator=g, device="cuda", dtype=torch.float64)[:, :m]
Y = torch.empty((n, ld), device="cuda", dtype=torch.float64)[:, :m]
G = torch.randn((m, m), generator=g, device="cuda", dtype=torch.float64) / 30
f = lambda: K.tsgemm([X], [G], [Y], alpha=-1.0, beta=1.0, zs=[Z])  # noqa: E731


def clk():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                           "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()


def kt():
    ks = []
    for _ in range(5):
        lib.bk_ozaki_timing(1)
        f()
        ks.append(lib.bk_ozaki_kernel_ms())
    lib.bk_ozaki_timing(0)
    return statistics.median(ks)


with K.fp64_emulation(True):
    f()
    torch.cuda.synchronize()
    print("cold:", kt(), clk(), flush=True)
    t0 = time.time()
    while time.time() - t0 < 6:
        for _ in range(20):
            f()
        torch.cuda.synchronize()
    print("hot :", kt(), clk(), flush=True)
    time.sleep(3)
    print("rest:", kt(), clk(), flush=True)
