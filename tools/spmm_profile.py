"""Launch each SpMM variant once on config 2 (m = 523) for ncu: gather, vec, march."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200.operators import DeviceCsr, as_device_operator  # noqa: E402
from paper_1407_7506_b200.problems import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, k, q, tol = config_problem(cfg)
d = as_device_operator(a)
kt = k + -(-k * 2 // 100)
ld = (kt + 15) // 16 * 16
dt = torch.complex128 if d.complex else torch.float64
x = torch.randn(a.n, ld, dtype=dt, device="cuda")[:, :kt]
y = torch.zeros(a.n, ld, dtype=dt, device="cuda")[:, :kt]
lib = _lib.load()
for variant in sys.argv[2:] or ["gather", "vec", "march"]:
    lib.bk_spmm_set_variant({"gather": 0, "tiled": 1}.get(variant, 2))
    DeviceCsr.use_stencil = variant == "march"
    for _ in range(2):
        d.apply_into(x, y)
torch.cuda.synchronize()
print("ok")
