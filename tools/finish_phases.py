"""Sub-phases of PPCGSolver.finish() at config 2: the final RR on the device vs the vector
download (to_host: pinned staging + multi-threaded copy into a fresh numpy array)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_7506_b200 import kernels as K  # noqa: E402
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

a, k, q, tol = config_problem(2)
for rep in range(3):
    s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=3)).start()
    while not s.step():
        pass
    torch.cuda.synchronize()
    V = s.XF[s.xi][:, :k]
    t0 = time.perf_counter()
    out = K.to_host(V)
    t1 = time.perf_counter()
    buf = np.empty((V.shape[0], k))
    t2 = time.perf_counter()
    buf[:] = 0.0
    t3 = time.perf_counter()
    t4 = time.perf_counter()
    rep_ = s.finish()
    t5 = time.perf_counter()
    print(f"rep {rep}: to_host {1e3*(t1-t0):.1f} ms; fault-in of a fresh array {1e3*(t3-t2):.1f} ms; "
          f"finish() {1e3*(t5-t4):.1f} ms", flush=True)
