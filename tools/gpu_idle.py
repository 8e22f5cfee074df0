"""GPU idle time inside solver iterations: union of kernel/memcpy intervals (torch.profiler /
CUPTI) vs the event-timed wall, and the largest gaps with the kernels around them.
usage: python tools/gpu_idle.py [cfg] [skip] [count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 5
count = int(sys.argv[3]) if len(sys.argv) > 3 else 5
a, k, q, tol = config_problem(cfg)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6)).start()
for _ in range(skip):
    s.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(count):
        s.step()
    torch.cuda.synchronize()
iv = []
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and ev.time_range.elapsed_us() > 0:
        iv.append((ev.time_range.start, ev.time_range.end, ev.name[:50]))
iv.sort()
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
gaps = []
last_name = iv[0][2]
for st, en, nm in iv[1:]:
    if st > cur_e:
        busy += cur_e - cur_s
        gaps.append((st - cur_e, last_name, nm))
        cur_s, cur_e = st, en
    else:
        cur_e = max(cur_e, en)
    if en >= cur_e:
        last_name = nm
busy += cur_e - cur_s
span = t1 - t0
print(f"cfg {cfg}: {count} iterations, span {span / 1e3 / count:.3f} ms/iter, busy {busy / 1e3 / count:.3f}, "
      f"idle {(span - busy) / 1e3 / count:.3f} ms/iter in {len(gaps) / count:.1f} gaps/iter")
gaps.sort(reverse=True)
for g, a_, b_ in gaps[:25]:
    print(f"  {g:8.1f} us  after {a_:50s} before {b_}")
