"""Microbenchmark of the FP64 DMMA Gram / tall-GEMM kernels at config-2 shapes
(n = 110,592, m = 523, row stride 524).  Tile overrides via PPCG_GRAM_TILE / PPCG_TS_TILE."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200 import kernels as K  # noqa: E402

if "GRAM_LOADER" in os.environ:  # 1 = bulk-copy pipeline, 0 = cp.async ring
    _lib.load().bk_gram_set_loader(int(os.environ["GRAM_LOADER"]))


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


n, m, ld = 110592, 523, 524
x = torch.randn(n, ld, dtype=torch.float64, device="cuda")[:, :m]
y = torch.randn(n, ld, dtype=torch.float64, device="cuda")[:, :m]
g = torch.zeros(m, ld, dtype=torch.float64, device="cuda")[:, :m]
out = torch.zeros(n, ld, dtype=torch.float64, device="cuda")[:, :m]
fl = 2.0 * n * m * m
res = {"gram_tile": os.environ.get("PPCG_GRAM_TILE", "default"), "ts_tile": os.environ.get("PPCG_TS_TILE", "default")}
res["gram_loader"] = _lib.load().bk_gram_set_loader(-1)
res["gram_xy_tflops"] = fl / t(lambda: K.gram(x, y, g)) / 1e9
xo = torch.randn(n, 534, dtype=torch.float64, device="cuda")[:, 11:534]  # odd column start (odd L)
res["gram_xy_oddcol_tflops"] = fl / t(lambda: K.gram(xo, y, g)) / 1e9
res["gram_sym_tflops"] = 0.5 * fl / t(lambda: K.gram(x, x, g, symmetric=True)) / 1e9
gg = torch.randn(m, ld, dtype=torch.float64, device="cuda")[:, :m]
res["tsgemm_tflops"] = fl / t(lambda: K.tsgemm([x], [gg], [out], alpha=-1.0, beta=1.0, zs=[y])) / 1e9
res["tsgemm_x2_tflops"] = 2 * fl / t(lambda: K.tsgemm([x, y], [gg, gg], [out, out])) / 1e9
# the solver's call shapes: projection (4 in-place updates, +- metric), residual (row scale + metric)
bufs = [torch.randn(n, ld, dtype=torch.float64, device="cuda")[:, :m] for _ in range(4)]
xs = [x, y, x, y]
gs = [gg, gg, gg, gg]
st = torch.zeros(4, dtype=torch.float64, device="cuda")
res["proj4_inplace_tflops"] = 4 * fl / t(lambda: K.tsgemm(xs, gs, bufs, alpha=-1.0, beta=1.0, zs=bufs)) / 1e9
res["proj4_inplace_metric_tflops"] = 4 * fl / t(lambda: K.tsgemm(xs, gs, bufs, alpha=-1.0, beta=1.0, zs=bufs,
                                                                  metric=st[0:1], ksplit=m, nsplit=m)) / 1e9
rs = torch.rand(n, dtype=torch.float64, device="cuda")
res["resid_rowscale_tflops"] = fl / t(lambda: K.tsgemm([x], [gg], [out], alpha=-1.0, beta=1.0, zs=[y], rowscale=rs)) / 1e9
res["resid_rowscale_metric_tflops"] = fl / t(lambda: K.tsgemm([x], [gg], [out], alpha=-1.0, beta=1.0, zs=[y], rowscale=rs,
                                                               metric=st[0:1], ksplit=512, nsplit=512)) / 1e9
res["cholqr_upper_tflops"] = 0.5 * 2 * fl / t(lambda: K.tsgemm([x, y], [gg, gg], [out, bufs[0]], upper=True)) / 1e9
res["gram2_tflops"] = 2 * fl / t(lambda: K.gram2(x, y, g, x, bufs[1], gg)) / 1e9
# edge-tile effect: widths that are / are not multiples of the 64-wide tile
for mm in (512, 576, 520):
    xx = torch.randn(n, 580, dtype=torch.float64, device="cuda")[:, :mm]
    gg2 = torch.zeros(mm, 580, dtype=torch.float64, device="cuda")[:, :mm]
    res[f"gram_m{mm}_tflops"] = 2.0 * n * mm * mm / t(lambda: K.gram(xx, xx, gg2)) / 1e9
    oo = torch.zeros(n, 580, dtype=torch.float64, device="cuda")[:, :mm]
    res[f"tsgemm_m{mm}_tflops"] = 2.0 * n * mm * mm / t(lambda: K.tsgemm([xx], [gg2], [oo])) / 1e9
print(json.dumps(res))
