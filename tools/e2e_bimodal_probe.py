"""Why are some e2e calls 50% slower?  Profiles consecutive ppcg_solve calls (CUPTI) and prints, per
call, the wall time, the summed kernel time and the largest kernels' totals."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1407_7506_b200 import SolverOptions, ppcg_solve  # noqa: E402
from paper_1407_7506_b200.operators import SparseHermitian  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

a0, k, q, tol = config_problem(2)
opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=20)
a = SparseHermitian(a0._csr.copy(), "symmetric")
ppcg_solve(a, jacobi_preconditioner(a), opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=2))
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    a = SparseHermitian(a0._csr.copy(), "symmetric")
    t = jacobi_preconditioner(a)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        w0 = time.perf_counter()
        r = ppcg_solve(a, t, opts=opts)
        torch.cuda.synchronize()
        w = time.perf_counter() - w0
    steps = r.trace[-1].wall_ms - r.trace[0].wall_ms
    del r
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name.split("(")[0][-40:]] += ev.device_time_total / 1e3
    tot = sum(agg.values())
    top = sorted(agg.items(), key=lambda kv: -kv[1])[:4]
    print(f"rep {rep}: wall {1e3 * w:6.1f} ms, iterations 2..20 {steps:6.1f} ms, kernel sum {tot:6.1f} ms; "
          + "; ".join(f"{n} {v:.0f}" for n, v in top), flush=True)
