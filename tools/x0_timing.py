"""Host<->device staging costs of the e2e path at config 2: the X0 draw (hostrng phases),
its upload, and the final vectors download, plus alternatives.  usage: python tools/x0_timing.py"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_7506_b200 import hostrng as H  # noqa: E402
from paper_1407_7506_b200 import kernels as K  # noqa: E402

n, kt, ldp = 110592, 524, 524
count = n * kt
print("cores", len(os.sched_getaffinity(0)), "count", count)
torch.zeros(1, device="cuda")
dev = torch.empty((n, ldp), dtype=torch.float64, device="cuda")


def t(name, f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{best * 1e3:9.1f} ms  {name}")
    return r


x = t("standard_normal (all)", lambda: H.standard_normal(0, count))
t("numpy empty+fill (page faults, 1 thread)", lambda: np.empty(count).fill(0.0))
t("from_host (pinned double-buffer)", lambda: K.from_host(x.reshape(n, kt), dev[:, :kt]))
t("torch pageable .to(cuda)", lambda: torch.from_numpy(x).to("cuda"))
t("to_host (pinned double-buffer)", lambda: K.to_host(dev[:, :523]))
t("torch pageable .cpu()", lambda: dev[:, :523].cpu())


def par_copy(dst, src, nt=16):
    rows = dst.shape[0]
    step = -(-rows // nt)

    def cp(i):
        dst[i * step:(i + 1) * step] = src[i * step:(i + 1) * step]

    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(cp, range(nt)))


for nt in (4, 8, 16):
    t(f"parallel numpy copy into fresh array, {nt} threads",
      lambda: par_copy(np.empty((n, kt)), x.reshape(n, kt), nt))
pin = torch.empty((n, kt), dtype=torch.float64, pin_memory=True)
t("pinned alloc 463 MB (cached after first)", lambda: torch.empty((n, kt), dtype=torch.float64, pin_memory=True), 1)
t("parallel copy into pinned, 16 threads", lambda: par_copy(pin.numpy(), x.reshape(n, kt), 16))
t("H2D from pinned (one copy)", lambda: dev[:, :kt].copy_(pin, non_blocking=True))
t("D2H into pinned", lambda: pin.copy_(dev[:, :kt], non_blocking=True))
t("normal_draw (fresh chunks)", lambda: H.normal_draw(0, count))
t("normal_draw (reused chunks)", lambda: H.normal_draw(0, count, reuse=True))
d = H.normal_draw(0, count, reuse=True)
assert np.array_equal(d.array(), x)
