"""Independent eigenvalues of a full-size BASELINE operator (scipy ARPACK, not PPCG) for the
GPU solves' parity ("Ritz values vs ... eigsh on the same CSR").

usage: python tools/eigsh_check.py CFG NEV OUT.npz [shift-invert|lanczos]
Writes the NEV lowest eigenvalues and ARPACK's residual norms; the committed fixture lives
under tests/golden/ (generated here, on the host, once).
"""
import sys
import time

import numpy as np
import scipy.sparse.linalg as sla

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1407_7506_b200.problems import config_problem  # noqa: E402

cfg, nev, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
mode = sys.argv[4] if len(sys.argv) > 4 else "shift-invert"
a, k, q, tol = config_problem(cfg)
A = a._csr.tocsc() if mode == "shift-invert" else a._csr
t0 = time.time()
if mode == "shift-invert":
    # shift just below the spectrum (Gershgorin lower bound of the diagonal-dominant part is
    # loose; use the smallest diagonal minus the largest off-diagonal row sum)
    d = A.diagonal()
    off = np.asarray(abs(A).sum(axis=1)).ravel() - abs(d)
    sigma = float(np.min(d - off)) - 1e-3
    vals, vecs = sla.eigsh(A, k=nev, sigma=sigma, which="LM", tol=1e-14, ncv=max(2 * nev + 1, 64))
else:
    vals, vecs = sla.eigsh(A, k=nev, which="SA", tol=1e-12, ncv=max(3 * nev, 96), maxiter=100000)
o = np.argsort(vals)
vals, vecs = vals[o], vecs[:, o]
res = np.linalg.norm(a._csr @ vecs - vecs * vals, axis=0)
np.savez_compressed(out, values=vals, resid=res, wall_s=np.array(time.time() - t0), mode=np.array(mode))
print(cfg, mode, "wall", round(time.time() - t0, 1), "lowest", vals[:4], "max resid", res.max())
