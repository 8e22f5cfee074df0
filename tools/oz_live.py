"""Tall-GEMM core time on the live config-2 solver state vs random operands of the same shape."""
import os
import sys
import statistics
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import kernels as K, _lib
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner

lib = _lib.load()
a, k, q, tol = config_problem(2)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10**6)).start()
for _ in range(6):
    s.step()
torch.cuda.synchronize()
L = s.L
ka = s.kt - L
x, ax = s.X(), s.AX()
G = s.Gm[:ka, :ka]
tmp = torch.empty_like(s.W)[:, L:]


def kt(f):
    f()
    torch.cuda.synchronize()
    ks = []
    for _ in range(5):
        lib.bk_ozaki_timing(1)
        f()
        ks.append(lib.bk_ozaki_kernel_ms())
    lib.bk_ozaki_timing(0)
    return statistics.median(ks)


print("L", L, "ka", ka, "x stride", x.stride(), "G stride", G.stride())
print("live  :", kt(lambda: K.tsgemm([x], [G], [tmp], alpha=-1.0, beta=1.0, zs=[ax])))
Gr = torch.randn_like(G.contiguous()) / 30
print("rand G:", kt(lambda: K.tsgemm([x], [Gr], [tmp], alpha=-1.0, beta=1.0, zs=[ax])))
xr = torch.randn_like(x)
print("rand X:", kt(lambda: K.tsgemm([xr], [G], [tmp], alpha=-1.0, beta=1.0, zs=[ax])))
Gc = G.contiguous()
print("G contiguous:", kt(lambda: K.tsgemm([x], [Gc], [tmp], alpha=-1.0, beta=1.0, zs=[ax])))
print("G abs stats: max", G.abs().max().item(), "min diag", G.diagonal().abs().min().item(),
      "zero cols", int((G.abs().amax(0) == 0).sum().item()))
