"""Host-side phase timing of the public ppcg_solve path at config 2 (what bench.py's e2e
number is made of).  usage: python tools/e2e_profile.py [cfg] [iters]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_7506_b200 import ppcg as PP  # noqa: E402
from paper_1407_7506_b200.operators import SparseHermitian  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
a0, k, q, tol = config_problem(cfg)
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
T = {}


def mark(name, t0):
    torch.cuda.synchronize()
    T[name] = time.perf_counter() - t0
    return time.perf_counter()


for rep in range(2):
    T.clear()
    a = SparseHermitian(a0._csr.copy(), "symmetric")
    t = jacobi_preconditioner(a)
    tt = time.perf_counter()
    t0 = tt
    opts = PP.SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=iters)
    s = PP.PPCGSolver(a, t, None, opts)
    t0 = mark("construct (device CSR upload)", t0)
    s._alloc()
    t0 = mark("alloc + cusolver handle", t0)
    x = PP.draw_initial_block(s.n, s.kt, s.cplx, 0, None)
    t0 = mark("X0 draw (numpy PCG64)", t0)
    xt = torch.from_numpy(np.ascontiguousarray(x)).to("cuda")
    t0 = mark("X0 upload", t0)
    del xt
    s2 = PP.PPCGSolver(a, t, None, opts)
    t1 = time.perf_counter()
    s2.start()
    t0 = mark("start() total", t1)
    while not s2.step():
        pass
    t0 = mark(f"{iters} steps", t0)
    r = s2.finish()
    t0 = mark("finish()", t0)
    V = s2.XF[s2.xi][:, :k]
    t0 = time.perf_counter()
    vv = V.cpu().numpy()
    t0 = mark("  (of which: vectors download, pageable)", t0)
    T["TOTAL (ppcg_solve equivalent)"] = T["start() total"] + T[f"{iters} steps"] + T["finish()"] + T[
        "construct (device CSR upload)"]
    print(f"--- rep {rep}")
    for kk, v in T.items():
        print(f"{v * 1e3:10.1f} ms  {kk}")
