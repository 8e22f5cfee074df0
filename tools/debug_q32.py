"""Debug: device vs oracle trajectories for q = 32 problems (small grids)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from oracle import ppcg_oracle as O  # noqa: E402
from paper_1407_7506_b200 import SolverOptions, ppcg_solve  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402
from util import HostCsr, HostDiag  # noqa: E402

for N, k, q, iters in ((16, 64, 32, 3), (20, 96, 32, 3), (16, 64, 16, 3), (16, 60, 20, 3)):
    a, _, _, _ = config_problem(2, N=N)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=k, sbsize=q, tol=1e-6, seed=0, max_iter=iters)
    rep = ppcg_solve(a, t, opts=opts)
    ref = O.oracle_solve(HostCsr(a._csr), HostDiag(t.d), opts=opts)
    print(f"N={N} k={k} q={q}")
    for r1, r2 in zip(rep.trace, ref.trace):
        print(f"  it {r1.iteration}: dev trace {r1.trace_value:.12g} ref {r2.trace_value:.12g}  rel {r1.rel_resid:.6g} / {r2.rel_resid:.6g}")
    print("  values maxrel", float(np.max(np.abs(rep.values - ref.values) / np.abs(ref.values))))
