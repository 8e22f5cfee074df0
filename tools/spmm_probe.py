"""One SpMM launch per kernel on the config-2 (or CFG) operator for ncu captures, plus a
device copy of the same block (the streaming reference at this size).

usage: python tools/spmm_probe.py [cfg] [col_offset]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200.operators import DeviceCsr  # noqa: E402
from paper_1407_7506_b200.problems import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
off = int(sys.argv[2]) if len(sys.argv) > 2 else 10
lib = _lib.load()
a, k, q, tol = config_problem(cfg, **({"N": 64} if cfg == 5 else {}))
DeviceCsr.stencil_kinds = ("slot", "march")
d = DeviceCsr(a._csr)
kt = k + -(-k * 2 // 100)
ld = (kt + 15) // 16 * 16
dt = torch.complex128 if d.complex else torch.float64
xb = torch.randn(a.n, ld, dtype=dt, device="cuda")
yb = torch.zeros(a.n, ld, dtype=dt, device="cuda")
x, y = xb[:, off:kt], yb[:, off:kt]
for name, slot in (("march", False), ("slot", True)):
    d.stencil.use_slot = slot
    for _ in range(3):
        d.apply_into(x, y)
    torch.cuda.synchronize()
for _ in range(3):
    y.copy_(x)
torch.cuda.synchronize()
# CUDA-event times (not under ncu these are the numbers to quote): each kernel and the copy
res = {}
for name, fn in (("march", lambda: (setattr(d.stencil, "use_slot", False), d.apply_into(x, y))),
                 ("slot", lambda: (setattr(d.stencil, "use_slot", True), d.apply_into(x, y))),
                 ("copy", lambda: y.copy_(x))):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    e1.synchronize()
    res[name] = e0.elapsed_time(e1) / 20
m = kt - off
s = 16 if d.complex else 8
byts = 2.0 * a.n * m * s + d.nnz * (s + 4) + 4 * (a.n + 1)
print({k: (round(v, 4), round(byts / v / 1e6, 1)) for k, v in res.items()}, "bytes", byts)
