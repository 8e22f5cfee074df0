import ctypes, torch, sys, os
sys.path.insert(0, '/root/repo')
from paper_1407_7506_b200 import kernels as K
n, m = 20000, 130
X = torch.randn((n, m), device="cuda", dtype=torch.float64)
G = torch.randn((m, m), device="cuda", dtype=torch.float64)
Y = torch.empty((n, m), device="cuda", dtype=torch.float64)
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
try:
    with K.fp64_emulation(True):
        K.tsgemm([X], [G], [Y])
    torch.cuda.synchronize()
    print("ok", (Y - X @ G).abs().max().item())
except Exception as e:
    print("ERR", e)
    try:
        torch.cuda.synchronize()
    except Exception as e2:
        print("sync:", e2)
