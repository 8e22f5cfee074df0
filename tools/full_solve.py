"""Full public ppcg_solve of a BASELINE config on one GPU; writes values / trace / residual
norms (and the wall time) to an npz for offline parity checks (eigsh, reference goldens).

usage: python tools/full_solve.py CFG OUT.npz [max_iter] [N]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_7506_b200 import SolverOptions, ppcg_solve  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg, out = int(sys.argv[1]), sys.argv[2]
max_iter = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
kw = {"N": int(sys.argv[4])} if len(sys.argv) > 4 else {}
a, k, q, tol = config_problem(cfg, **kw)
t = jacobi_preconditioner(a)
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
w0 = time.perf_counter()
rep = ppcg_solve(a, t, opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=max_iter))
torch.cuda.synchronize()
wall = time.perf_counter() - w0
rn = np.array(rep.diagnostics["final_residual_norms"])
tr = np.array([[r.iteration, r.trace_value, r.rel_resid, r.n_locked, r.n_matvec, r.wall_ms] for r in rep.trace])
np.savez_compressed(out, values=rep.values, trace=tr, final_rn=rn,
                    meta=np.array([rep.iterations, rep.matvecs, rep.rr_count, rep.breakdown_recoveries,
                                   1 if rep.status == "converged" else 0]),
                    vhist=np.array(rep.values_history, dtype=object) if False else np.zeros(0),
                    wall_s=np.array(wall),
                    peak_mem=np.array(torch.cuda.max_memory_allocated()))
print(json.dumps({"config": cfg, "n": a.n, "k": k, "sbsize": q, "tol": tol, "status": rep.status,
                  "iterations": rep.iterations, "rr_count": rep.rr_count, "matvecs": rep.matvecs,
                  "wall_s": wall, "ms_per_iteration": 1e3 * wall / max(rep.iterations, 1),
                  "final_rel_resid": rep.trace[-1].rel_resid if rep.trace else None,
                  "lambda_min": float(rep.values[0]), "lambda_k": float(rep.values[-1]),
                  "max_final_residual_norm": float(rn.max()), "recoveries": rep.breakdown_recoveries,
                  "max_memory_allocated_GB": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
