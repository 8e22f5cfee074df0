"""All-in time-to-solution of the public ppcg_solve on BASELINE configs.
usage: python tools/time_to_solution.py cfg [max_iter]   -> one JSON line"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_7506_b200 import SolverOptions, ppcg_solve  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1])
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
a, k, q, tol = config_problem(cfg)
t = jacobi_preconditioner(a)
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
w0 = time.perf_counter()
rep = ppcg_solve(a, t, opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=max_iter))
torch.cuda.synchronize()
wall = time.perf_counter() - w0
rn = np.array(rep.diagnostics["final_residual_norms"])
print(json.dumps({"config": cfg, "n": a.n, "k": k, "sbsize": q, "tol": tol, "status": rep.status,
                  "iterations": rep.iterations, "rr_count": rep.rr_count, "matvecs": rep.matvecs,
                  "wall_s": wall, "ms_per_iteration": 1e3 * wall / max(rep.iterations, 1),
                  "final_rel_resid": rep.trace[-1].rel_resid if rep.trace else None,
                  "lambda_min": float(rep.values[0]), "lambda_k": float(rep.values[-1]),
                  "max_final_residual_norm": float(rn.max()), "recoveries": rep.breakdown_recoveries}))
