"""Kernel timeline (stream, start, duration) of one steady-state config-2 iteration, from
torch.profiler / CUPTI.  usage: python tools/timeline.py [cfg] [skip]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 6
count = int(sys.argv[3]) if len(sys.argv) > 3 else 1
filt = sys.argv[4] if len(sys.argv) > 4 else ""
a, k, q, tol = config_problem(cfg)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6)).start()
for _ in range(skip):
    s.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(count):
        s.step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    d = e.time_range.end - e.time_range.start
    if d < 20 and "Memcpy" not in e.name:
        continue
    if filt and not any(f in e.name for f in filt.split(",")):
        continue
    print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  +{d / 1e3:7.3f}  s{getattr(e, 'device_resource_id', '?')}  {e.name[:70]}")
