"""Per-iteration GPU kernel-time breakdown of the config-2 solver (torch.profiler / CUPTI),
over a window of steady-state iterations.
usage: python tools/iter_breakdown.py [cfg] [skip] [count] [N (grid edge override)] [k override]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 5
count = int(sys.argv[3]) if len(sys.argv) > 3 else 10
kw = {"N": int(sys.argv[4])} if len(sys.argv) > 4 else {}
a, k, q, tol = config_problem(cfg, **kw)
if len(sys.argv) > 5:
    k = int(sys.argv[5])
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10**6)).start()
for _ in range(skip):
    s.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0.record()
    for _ in range(count):
        s.step()
    e1.record()
    torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / count
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name
        for pre in ("void ", "bk::"):
            if name.startswith(pre):
                name = name[len(pre):]
        name = name.split("(")[0][:60]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total / 1e3
tot = sum(v for _, v in agg.values())
print(f"cfg {cfg}: {count} iterations {skip + 1}..{skip + count}, L={s.L}, event wall {wall:.3f} ms/iter, "
      f"kernel sum {tot / count:.3f} ms/iter")
rows = sorted(agg.items(), key=lambda x: -x[1][1])
for name, (c, v) in rows[:30]:
    print(f"{v / count:8.3f} ms/iter {100 * v / tot:5.1f}%  {c / count:6.1f}/iter  {name}")
json.dump({"cfg": cfg, "wall_ms": wall, "kernel_ms": tot / count,
           "kernels": {n: {"ms_per_iter": v / count, "launches_per_iter": c / count} for n, (c, v) in rows}},
          open(os.path.join("gpurun_out", f"breakdown_cfg{cfg}.json"), "w"), indent=1)
