"""Jacobi sweeps per subblock pencil (info[3] >> 8) over a few solver iterations.
usage: python tools/pencil_sweeps.py [cfg] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1407_7506_b200.ppcg import PPCGSolver, SolverOptions  # noqa: E402
from paper_1407_7506_b200.problems import config_problem, jacobi_preconditioner  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
a, k, q, tol = config_problem(cfg)
s = PPCGSolver(a, jacobi_preconditioner(a), None, SolverOptions(k=k, sbsize=q, tol=tol, max_iter=10 ** 6)).start()
for i in range(steps):
    s.step()
    torch.cuda.synchronize()
    info = s.info.cpu().numpy().reshape(-1, 4)
    nb = (s.kt - s.L + q - 1) // q
    sw = (info[:nb, 3] >> 8).tolist()
    print(f"iteration {s.it}: sweeps per pencil {sw}")
