"""GPU idle time per iteration of the config-2 step loop: wall minus the union of all kernel /
memcpy intervals (CUPTI via torch.profiler), and the largest gaps with the kernels around them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

a, k, q, tol = config_problem(2)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6)).start()
for _ in range(6):
    s.step()
torch.cuda.synchronize()
count = 8
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(count):
        s.step()
    torch.cuda.synchronize()
ev = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
             if e.device_type == torch.autograd.DeviceType.CUDA), key=lambda t: t[0])
t0, t1 = ev[0][0], max(e[1] for e in ev)
busy, cur_s, cur_e, gaps, last_name = 0.0, ev[0][0], ev[0][1], [], ev[0][2]
for a_, b_, nm in ev[1:]:
    if a_ > cur_e:
        busy += cur_e - cur_s
        gaps.append((a_ - cur_e, last_name[:40], nm[:40]))
        cur_s, cur_e = a_, b_
    else:
        cur_e = max(cur_e, b_)
    last_name = nm if b_ >= cur_e else last_name
busy += cur_e - cur_s
span = t1 - t0
print(f"{count} iterations: span {span / 1e3 / count:.3f} ms/iter, GPU busy {busy / 1e3 / count:.3f}, idle "
      f"{(span - busy) / 1e3 / count:.3f} ms/iter in {len(gaps) / count:.1f} gaps/iter")
agg = {}
for g, before, after in gaps:
    key = (before, after)
    agg.setdefault(key, [0, 0.0])
    agg[key][0] += 1
    agg[key][1] += g
for (before, after), (c, g) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {g / 1e3 / count:7.3f} ms/iter  {c / count:4.1f}/iter  after {before:40s} before {after}")
