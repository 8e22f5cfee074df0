"""Debug: full-size config 2, device vs oracle state after iteration 1."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ppcg_oracle as O  # noqa: E402
from paper_1407_7506_b200 import SolverOptions  # noqa: E402
from paper_1407_7506_b200.ppcg import PPCGSolver  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402
from util import HostCsr, HostDiag  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 48
k = int(sys.argv[2]) if len(sys.argv) > 2 else 512
q = int(sys.argv[3]) if len(sys.argv) > 3 else 32
a, _, _, _ = config_problem(2, N=N)
t = jacobi_preconditioner(a)
opts = SolverOptions(k=k, sbsize=q, tol=1e-6, seed=0, max_iter=5)
s = PPCGSolver(a, t, None, opts).start()
t0 = time.time()
r = O.OracleRun(HostCsr(a._csr), HostDiag(t.d), None, opts, blas_threads=len(os.sched_getaffinity(0))).start()
print("oracle start", time.time() - t0, flush=True)


def cmp(name, dev, ref):
    dev = dev.cpu().numpy() if hasattr(dev, "cpu") else dev
    out = []
    for j in range(ref.shape[1]):
        e = min(np.linalg.norm(dev[:, j] - ref[:, j]), np.linalg.norm(dev[:, j] + ref[:, j]))
        out.append(e / max(np.linalg.norm(ref[:, j]), 1e-300))
    out = np.array(out)
    print(f"  {name}: max col rel err {out.max():.3e} (argmax {out.argmax()}), median {np.median(out):.3e}", flush=True)


cmp("X0", s.X(), r.x)
cmp("AX0", s.AX(), r.ax)
for it in range(2):
    # compare W before preconditioning (oracle keeps raw W; device stores T(W))
    wdev = s.W[:, s.L:].cpu().numpy() / t.d[:, None]
    cmp(f"it{it+1} W(raw)", wdev, r.w)
    s.step()
    r.step()
    cmp(f"it{it+1} X", s.X(), r.x)
    cmp(f"it{it+1} AX", s.AX(), r.ax)
    if r.p is not None:
        cmp(f"it{it+1} P", s.Pa(), r.p)
    print(f"  trace dev {s.trace[-1].trace_value!r} ref {r.trace[-1].trace_value!r}", flush=True)
