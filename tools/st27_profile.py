"""One launch of each requested stencil-slot configuration on a config-4-structure grid, for ncu.
usage: python tools/st27_profile.py N m cfg [cfg ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200.operators import DeviceCsr  # noqa: E402
from paper_1407_7506_b200.problems import config_problem  # noqa: E402

N, m = int(sys.argv[1]), int(sys.argv[2])
a, k, q, tol = config_problem(4, N=N)
DeviceCsr.stencil_kinds = ("slot",)
d = DeviceCsr(a._csr)
ld = (m + 15) // 16 * 16
x = torch.randn(a.n, ld, dtype=torch.float64, device="cuda")[:, :m]
y = torch.zeros(a.n, ld, dtype=torch.float64, device="cuda")[:, :m]
lib = _lib.load()
for c in sys.argv[3:]:
    lib.bk_spmm_stencil_set_config(int(c))
    d.apply_into(x, y)
    d.apply_into(x, y)
torch.cuda.synchronize()
print("ok")
