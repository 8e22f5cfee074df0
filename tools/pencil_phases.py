"""Phase clocks of the subblock pencil kernel (subblock 0) on live solver state.  Needs a
profiling build of the library (pencil.cu compiled with -DPPCG_PENCIL_PROFILE):
  PPCG_B200_LIB=.../libppcg_b200_prof.so python tools/pencil_phases.py [cfg] [steps] [N] [k]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kw = {"N": int(sys.argv[3])} if len(sys.argv) > 3 else {}
a, k, q, tol = config_problem(cfg, **kw)
if len(sys.argv) > 4:
    k = int(sys.argv[4])
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6)).start()
lib = ctypes.CDLL(_lib.LIB_PATH)
lib.bk_pencil_phase_clocks.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
names = {0: "kernel start", 1: "attempt start (norms, masks, assembly)", 2: "Cholesky (singular-Gram test)",
         3: "reload + Cholesky (reduction)", 4: "triangular inverse", 5: "L^-1 A L^-H + symmetrise",
         6: "tridiagonalisation", 7: "bisection", 8: "inverse iteration", 9: "Gram-Schmidt x2",
         10: "Rayleigh-Ritz in span(Z)", 11: "back-transformation", 12: "eigenvector copy", 13: "C = L^-H Z",
         14: "rank test setup", 15: "sigma_min(C_X) (one-sided Jacobi)", 16: "coefficients out"}
for it in range(steps):
    s.step()
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 32)()
    rc = lib.bk_pencil_phase_clocks(buf)
    if rc != 1:
        print("not a profiling build", rc)
        break
    c = list(buf)
    if it >= steps - 2:
        tot = c[16] - c[0]
        print(f"iteration {s.it}: L = {s.L}, subblock 0: {tot} clocks")
        prev = c[0]
        for i in range(1, 17):
            print(f"  {names[i]:42s} {c[i] - prev:9d}  {100.0 * (c[i] - prev) / tot:5.1f}%")
            prev = c[i]
