"""Warm time to solution: the public ppcg_solve twice in one process (the second run timed),
plus the per-iteration wall-clock trace.  usage: python tools/tts_warm.py cfg"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import SolverOptions, ppcg_solve  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1])
a, k, q, tol = config_problem(cfg)
t = jacobi_preconditioner(a)
out = []
for rep in range(2):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    r = ppcg_solve(a, t, opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=5000))
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    ms = [tr.wall_ms for tr in r.trace]
    out.append({"rep": rep, "wall_s": wall, "iterations": r.iterations,
                "first_iter_ms": ms[0] if ms else None,
                "per_iter_ms_10_50": (ms[50] - ms[10]) / 40 if len(ms) > 50 else None,
                "last_trace_ms": ms[-1] if ms else None})
print(json.dumps({"config": cfg, "runs": out}))
