"""Sub-phases of PPCGSolver.start() at config 2 (warm): allocation, X0 draw + upload, the
initial Gram / CholQR, SpMM, residual.  usage: python tools/start_phases.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import ppcg as PP  # noqa: E402
from paper_1407_7506_b200.operators import SparseHermitian  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

a0, k, q, tol = config_problem(2)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for rep in range(reps):
    a = SparseHermitian(a0._csr.copy(), "symmetric")
    s = PP.PPCGSolver(a, jacobi_preconditioner(a), None, PP.SolverOptions(k=k, sbsize=q, tol=tol, max_iter=20))
    K = s.K
    T = {}

    def mark(name, t0):
        torch.cuda.synchronize()
        T[name] = 1e3 * (time.perf_counter() - t0)
        return time.perf_counter()

    t = time.perf_counter()
    s._alloc()
    t = mark("alloc", t)
    raw = s.XF[1]
    src = PP.initial_block_source(s.n, s.kt, s.cplx, s.opts.seed, s.x0, 0, s.n)
    t = mark("x0 source", t)
    K.from_host(src, raw)
    t = mark("x0 draw+upload", t)
    G = s.Gm
    K.gram(raw, raw, G, symmetric=True)
    t = mark("gram", t)
    s.xi = 1
    s.L = 0
    s._cholqr_inplace_swap(G, 1)
    t = mark("cholqr", t)
    s._A(s.X(), s.AX())
    t = mark("spmm", t)
    s._residual_w()
    t = mark("residual", t)
    print(f"rep {rep}: " + "  ".join(f"{k_} {v:6.1f}" for k_, v in T.items()), flush=True)
