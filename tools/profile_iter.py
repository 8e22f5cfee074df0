"""Run the config-2 solver for a few iterations (for ncu launch lists / captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
a, k, q, tol = config_problem(cfg)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10**6)).start()
for _ in range(steps):
    s.step()
torch.cuda.synchronize()
print("ok", s.it, s.L)
