"""Per-call device time of the kernel wrappers inside solver iterations (CUDA events around
each paper_1407_7506_b200.kernels call, labelled by the calling line of ppcg.py), with the
algorithmic flops of the GEMM-shaped calls.  usage: python tools/call_timing.py [cfg] [skip] [count]"""
import collections
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import kernels as K  # noqa: E402
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 5
count = int(sys.argv[3]) if len(sys.argv) > 3 else 5
REC = []
ON = [False]


def flops_of(name, args, kw):
    try:
        if name == "gram":
            x, y = args[0], args[1]
            f = 2.0 * x.shape[0] * x.shape[1] * y.shape[1]
            return f / 2 if kw.get("symmetric") else f
        if name == "gram2":
            return 2.0 * args[0].shape[0] * (args[0].shape[1] * args[1].shape[1] + args[3].shape[1] * args[4].shape[1])
        if name == "tsgemm":
            xs, gs = args[0], args[1]
            f = sum(2.0 * x.shape[0] * x.shape[1] * g.shape[1] for x, g in zip(xs, gs))
            return f / 2 if kw.get("upper") else f
    except Exception:
        return 0.0
    return 0.0


def wrap(name):
    fn = getattr(K, name)

    def inner(*args, **kw):
        if not ON[0]:
            return fn(*args, **kw)
        st = traceback.extract_stack(limit=3)[-2]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn(*args, **kw)
        e1.record()
        REC.append((f"{name} @{os.path.basename(st.filename)}:{st.lineno}", e0, e1, flops_of(name, args, kw)))
        return r
    setattr(K, name, inner)


for nm in ["gram", "gram2", "tsgemm", "subblock_grams", "subblock_pencils", "subblock_recombine", "sumsq",
           "small_stats", "rr_residual", "spmm_csr"]:
    wrap(nm)

a, k, q, tol = config_problem(cfg)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6)).start()
for _ in range(skip):
    s.step()
torch.cuda.synchronize()
ON[0] = True
for _ in range(count):
    s.step()
torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for lab, e0, e1, f in REC:
    ms = e0.elapsed_time(e1)
    agg[lab][0] += 1
    agg[lab][1] += ms
    agg[lab][2] += f
tot = sum(v[1] for v in agg.values())
print(f"cfg {cfg}: iterations {skip + 1}..{skip + count}, wrapped-call time {tot / count:.2f} ms/iter")
for lab, (c, ms, f) in sorted(agg.items(), key=lambda x: -x[1][1]):
    tf = f / (ms / 1e3) / 1e12 if f else 0.0
    print(f"{ms / count:8.3f} ms/iter  {c / count:4.1f}x  {tf:6.2f} TF/s  {lab}")
