import numpy as np, torch, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from util import gauss
from paper_1407_7506_b200 import kernels as K
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
n, m = 20000, 70
x, ax = gauss(n, m, 10), gauss(n, m, 11)
g = x.T @ ax
for k, ns in [(64, 64), (70, 70), (70, 64), (64, 70), (32, 64)]:
    for emu in (True, False):
        metric = torch.zeros(1, dtype=torch.float64, device="cuda")
        w = torch.empty((n, m), dtype=torch.float64, device="cuda")
        with K.fp64_emulation(emu):
            K.tsgemm([d(x)], [d(g)], [w], alpha=-1.0, beta=1.0, zs=[d(ax)], metric=metric, ksplit=k, nsplit=ns)
        ref = np.linalg.norm(ax[:, :ns] - x[:, :k] @ g[:k, :ns], "fro") ** 2
        wr = ax - x @ g
        print(k, ns, "emu" if emu else "dmma", "metric rel err", abs(metric.item() - ref) / ref, "W err", np.abs(w.cpu().numpy() - wr).max(), "W max", np.abs(wr).max())
