"""Time the batched subblock pencils (block_update's dense part, pencil.cu) at the BASELINE
shapes: config 2 (17 real d = 96), config 3 (17 real d = 192), config 4 (33 real d = 192),
config 5 (66 complex d = 192; 9 per rank when split over 8 GPUs).  The raw Grams come from
bk_subblock_grams on random blocks (X orthonormalised, W, P random) so the pencils have the
production structure.  usage: python tools/pencil_batch_time.py  -> JSON lines"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import kernels as K  # noqa: E402


def case(name, nb, q, cplx, n=4096):
    ka = nb * q
    dt = torch.complex128 if cplx else torch.float64
    g = torch.Generator(device="cuda").manual_seed(nb)
    blocks = [torch.randn(n, ka, dtype=dt, device="cuda", generator=g) for _ in range(6)]
    blocks[0] = torch.linalg.qr(blocks[0])[0].contiguous()
    dmax = 3 * q
    araw = torch.zeros(nb * dmax * dmax, dtype=dt, device="cuda")
    braw = torch.zeros_like(araw)
    tmp = None
    if cplx:
        tmp = (torch.zeros(nb * 4 * dmax * dmax, dtype=torch.float64, device="cuda"),
               torch.zeros(nb * 4 * dmax * dmax, dtype=torch.float64, device="cuda"))
    K.subblock_grams(n, ka, q, True, *[b.data_ptr() for b in blocks], ka, 0, araw, braw, tmp=tmp)
    coef = torch.zeros(nb * dmax * q, dtype=dt, device="cuda")
    theta = torch.zeros(ka, dtype=torch.float64, device="cuda")
    info = torch.zeros(nb * 4, dtype=torch.int32, device="cuda")
    cscale = torch.zeros(nb, dtype=torch.float64, device="cuda")
    run = lambda: K.subblock_pencils(ka, q, True, araw, braw, coef, theta, info, cscale)  # noqa: E731
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    e1.synchronize()
    st = info.view(nb, 4).cpu()
    print(json.dumps({"case": name, "nb": nb, "d": dmax, "complex": cplx, "ms": e0.elapsed_time(e1) / 5,
                      "errors": int((st[:, 2] != 0).sum()), "fallbacks": int(st[:, 0].sum())}), flush=True)


case("config 2 (q 32)", 17, 32, False)
case("config 3 (q 64)", 17, 64, False)
case("config 4 (q 64)", 33, 64, False)
case("config 5 (q 64, complex, 1 GPU)", 66, 64, True)
case("config 5 (q 64, complex, per rank of 8)", 9, 64, True)
