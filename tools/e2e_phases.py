"""Phase timing of the public ppcg_solve path (what bench.py's e2e number is made of), on
fresh host inputs each repetition: construction (device operator: CSR upload + stencil plan,
preconditioner), start() (X0 draw + upload, initial CholQR / SpMM / residual), the steps,
finish() (final RR, vectors download).  usage: python tools/e2e_phases.py [cfg] [iters] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200.operators import SparseHermitian  # noqa: E402
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a0, k, q, tol = config_problem(cfg)
torch.zeros(1, device="cuda")
rep_ = None
for rep in range(reps):
    rep_ = None  # like bench.py: the previous result is released before the next call
    a = SparseHermitian(a0._csr.copy(), "symmetric" if a0.dtype.kind == "f" else "hermitian")
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=iters)
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    s = PPCGSolver(a, t, None, opts)
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    s.start()
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    while not s.step():
        pass
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    rep_ = s.finish()
    torch.cuda.synchronize()
    T.append(time.perf_counter())
    d = [1e3 * (T[i + 1] - T[i]) for i in range(4)]
    print(f"rep {rep}: construct {d[0]:7.1f} ms  start {d[1]:7.1f} ms  {rep_.iterations} steps {d[2]:7.1f} ms  "
          f"finish {d[3]:7.1f} ms  total {sum(d):7.1f} ms  -> {rep_.iterations / (sum(d) / 1e3):.2f} it/s",
          flush=True)
