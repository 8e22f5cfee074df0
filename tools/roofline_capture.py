"""Run config 2 to steady state, then issue exactly the bench's roofline launches inside a
cudaProfilerStart/Stop window (ncu --profile-from-start off captures only these):
  gram   : X^T AX on the live state (main 64-aligned launch + strip launch)
  tsgemm : the residual update AX - X G
usage: ncu --profile-from-start off ... python tools/roofline_capture.py [gram|tsgemm]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import kernels as K  # noqa: E402
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "gram"
a, k, q, tol = config_problem(2)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6)).start()
for _ in range(3):
    s.step()
L, ka = s.L, s.kt - s.L
x, ax = s.X(), s.AX()
G = s.Gm[:ka, :ka]
K.gram(x, ax, G)
tmp = torch.empty_like(s.W)[:, L:]
K.tsgemm([x], [G], [tmp], alpha=-1.0, beta=1.0, zs=[ax])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
if what == "gram":
    K.gram(x, ax, G)
else:
    K.tsgemm([x], [G], [tmp], alpha=-1.0, beta=1.0, zs=[ax])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", what, ka)
