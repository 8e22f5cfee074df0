"""Symmetric / X^T Y Gram timing under both loaders (env knobs are read once per process:
run once per setting).  usage: GRAM_LOADER=1 PPCG_GRAM_MINWAVES=8 python tools/sym_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200 import kernels as K  # noqa: E402

_lib.load().bk_gram_set_loader(int(os.environ.get("GRAM_LOADER", "1")))


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


n = 110592
res = {k: os.environ.get(k) for k in ("GRAM_LOADER", "PPCG_GRAM_MINWAVES", "PPCG_GRAM_SPLIT")}
for m in (512, 523, 533):
    x = torch.randn(n, 534, dtype=torch.float64, device="cuda")[:, :m]
    g = torch.zeros(m, 534, dtype=torch.float64, device="cuda")[:, :m]
    res[f"sym{m}_ms"] = round(t(lambda: K.gram(x, x, g, symmetric=True)), 4)
    res[f"xy{m}_ms"] = round(t(lambda: K.gram(x, x, g)), 4)
print(json.dumps(res))
