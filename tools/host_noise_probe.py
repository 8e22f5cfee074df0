"""Is e2e jitter host noise?  Alternates the e2e call with a fixed single-thread CPU task and a fixed
16-thread task (numpy normals), printing all three timings per repetition."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import SolverOptions, ppcg_solve  # noqa: E402
from paper_1407_7506_b200.operators import SparseHermitian  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

a0, k, q, tol = config_problem(2)
opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=20)
pool = ThreadPoolExecutor(max_workers=16)


def cpu1():
    t = time.perf_counter()
    np.random.default_rng(1).standard_normal(4_000_000)
    return 1e3 * (time.perf_counter() - t)


def cpu16():
    t = time.perf_counter()
    list(pool.map(lambda s: np.random.default_rng(s).standard_normal(3_000_000), range(16)))
    return 1e3 * (time.perf_counter() - t)


a = SparseHermitian(a0._csr.copy(), "symmetric")
ppcg_solve(a, jacobi_preconditioner(a), opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=2))
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    c1, c16 = cpu1(), cpu16()
    a = SparseHermitian(a0._csr.copy(), "symmetric")
    t = jacobi_preconditioner(a)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    r = ppcg_solve(a, t, opts=opts)
    torch.cuda.synchronize()
    w = time.perf_counter() - w0
    steps = r.trace[-1].wall_ms - r.trace[0].wall_ms
    del r
    print(f"rep {rep}: 1-thread task {c1:6.1f} ms   16-thread task {c16:6.1f} ms   e2e {1e3 * w:6.1f} ms "
          f"({20 / w:5.1f} it/s; iterations 2..20 {steps:6.1f} ms)", flush=True)
