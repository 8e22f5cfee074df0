"""Are the step-loop spikes Python garbage collections?  Times every collection (gc.callbacks)
inside consecutive public-path solves."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import SolverOptions, ppcg_solve  # noqa: E402
from paper_1407_7506_b200.operators import SparseHermitian  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

acc = {"t0": 0.0, "ms": [0.0, 0.0, 0.0], "n": [0, 0, 0]}


def cb(phase, info):
    if phase == "start":
        acc["t0"] = time.perf_counter()
    else:
        g = info["generation"]
        acc["ms"][g] += 1e3 * (time.perf_counter() - acc["t0"])
        acc["n"][g] += 1


gc.callbacks.append(cb)
a0, k, q, tol = config_problem(2)
opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=20)
a = SparseHermitian(a0._csr.copy(), "symmetric")
ppcg_solve(a, jacobi_preconditioner(a), opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=2))
print("objects tracked:", len(gc.get_objects()), "thresholds", gc.get_threshold())
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 16):
    a = SparseHermitian(a0._csr.copy(), "symmetric")
    t = jacobi_preconditioner(a)
    torch.cuda.synchronize()
    acc["ms"], acc["n"] = [0.0, 0.0, 0.0], [0, 0, 0]
    w0 = time.perf_counter()
    r = ppcg_solve(a, t, opts=opts)
    torch.cuda.synchronize()
    w = time.perf_counter() - w0
    steps = r.trace[-1].wall_ms - r.trace[0].wall_ms
    del r
    print(f"rep {rep}: wall {1e3 * w:6.1f} ms, iterations 2..20 {steps:6.1f} ms, gc time by generation "
          f"{acc['ms'][0]:.1f}/{acc['ms'][1]:.1f}/{acc['ms'][2]:.1f} ms in {acc['n']} collections", flush=True)
