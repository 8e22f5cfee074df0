import torch
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2):
    c = a @ b
x = torch.randn(110592, 523, dtype=torch.float64, device="cuda")
for _ in range(2):
    g = x.T @ x
    y = x @ g
torch.cuda.synchronize()
print("ok")
