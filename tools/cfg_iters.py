"""Per-iteration device time of a BASELINE config over a few iterations (for configs whose
full solve is long, e.g. 4).  usage: python tools/cfg_iters.py cfg steps  -> JSON line"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.perf_counter()
a, k, q, tol = config_problem(cfg)
t_gen = time.perf_counter() - t0
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6))
t0 = time.perf_counter()
s.start()
torch.cuda.synchronize()
t_start = time.perf_counter() - t0
ms = []
for _ in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.step()
    e1.record()
    e1.synchronize()
    ms.append(e0.elapsed_time(e1))
print(json.dumps({"config": cfg, "n": a.n, "nnz": int(a.nnz) if hasattr(a, "nnz") else None, "k": k, "sbsize": q,
                  "k_total": s.kt, "host_generate_s": t_gen, "start_s": t_start, "iteration_ms": ms,
                  "rel_resid": [r.rel_resid for r in s.trace],
                  "max_memory_allocated_GB": torch.cuda.max_memory_allocated() / 1e9}))
