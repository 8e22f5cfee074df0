"""One batched pencil launch at config-3 shape (17 real d = 192) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import kernels as K  # noqa: E402

nb, q, n = 17, 64, 4096
ka = nb * q
g = torch.Generator(device="cuda").manual_seed(nb)
blocks = [torch.randn(n, ka, dtype=torch.float64, device="cuda", generator=g) for _ in range(6)]
blocks[0] = torch.linalg.qr(blocks[0])[0].contiguous()
dmax = 3 * q
araw = torch.zeros(nb * dmax * dmax, dtype=torch.float64, device="cuda")
braw = torch.zeros_like(araw)
K.subblock_grams(n, ka, q, True, *[b.data_ptr() for b in blocks], ka, 0, araw, braw)
coef = torch.zeros(nb * dmax * q, dtype=torch.float64, device="cuda")
theta = torch.zeros(ka, dtype=torch.float64, device="cuda")
info = torch.zeros(nb * 4, dtype=torch.int32, device="cuda")
cscale = torch.zeros(nb, dtype=torch.float64, device="cuda")
for _ in range(2):
    K.subblock_pencils(ka, q, True, araw, braw, coef, theta, info, cscale)
torch.cuda.synchronize()
