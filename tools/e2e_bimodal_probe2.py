"""Per-iteration wall time inside consecutive public-path solves (PPCGSolver start/step/finish as
ppcg_solve runs them), to see whether a slow call is slow uniformly or in spikes."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200.operators import SparseHermitian  # noqa: E402
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

a0, k, q, tol = config_problem(2)
opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=20)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    a = SparseHermitian(a0._csr.copy(), "symmetric")
    t = jacobi_preconditioner(a)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    s = PPCGSolver(a, t, None, opts).start()
    ts = [time.perf_counter()]
    while not s.step():
        ts.append(time.perf_counter())
    ts.append(time.perf_counter())
    r = s.finish()
    torch.cuda.synchronize()
    w = time.perf_counter() - w0
    d = [1e3 * (b - a_) for a_, b in zip(ts, ts[1:])]
    print(f"rep {rep}: wall {1e3 * w:6.1f} ms, start {1e3 * (ts[0] - w0):5.1f}, threads {threading.active_count()}, steps: "
          + " ".join(f"{x:4.0f}" for x in d), flush=True)
    del r, s
