"""North-star acceptance beyond config 2 (BASELINE configs 3-5): converged eigenpairs vs the
reference's own CPU PPCG and vs an independent eigensolver.

* configs 3, 4, 5 on scaled grids with the production block shape (q = 64: the d = 192
  pencils, the 7-point / 27-point / complex stencil SpMMs in their production mode) against the
  reference's full solves (tests/golden/scaled.npz, make_golden.py --scaled): iteration count
  +-1, lock schedule, eigenvalues within relative 1e-10, the locked-column residual criterion
  (rayleigh_ritz.py:95-108), principal angles <= 1e-6;
* config 3 at full size (n = 262,144, k = 1,024): the lowest 48 eigenvalues against scipy
  ARPACK in shift-invert mode (tests/golden/eigsh_cfg3.npz, tools/eigsh_check.py; residuals
  1e-14) within relative 1e-9 -- the reference CPU solve itself needs ~a day here;
* config 4 at full size (n = 884,736, 27-point, k = 2,048): lambda_1 = 1 exactly (A = I + a
  weighted graph Laplacian, constant null vector), the locked-column criterion, and ARPACK
  eigenvalues when that fixture exists.
"""

import os

import numpy as np
import pytest

from util import sine_angle

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCALED = {"cfg3_n32": (3, 32, dict(k=256, sbsize=64, tol=1e-6)),
          "cfg4_n24": (4, 24, dict(k=256, sbsize=64, tol=1e-5)),
          "cfg5_n24": (5, 24, dict(k=256, sbsize=64, tol=1e-5))}


def _locked_ok(rep, tol):
    rn = np.array(rep.diagnostics["final_residual_norms"])
    L = rep.trace[-1].n_locked if rep.trace else 0
    bound = tol * np.maximum(np.abs(rep.values), 1.0)
    assert np.all(rn[:L] <= bound[:L]), float(np.max(rn[:L] / bound[:L]))
    return L


@pytest.mark.parametrize("name", list(SCALED))
def test_scaled_config_vs_reference(cuda, name):
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner, ppcg_solve

    z = np.load(os.path.join(G, "scaled.npz"))
    cfg, N, kw = SCALED[name]
    a, _, _, _ = config_problem(cfg, N=N)
    rep = ppcg_solve(a, jacobi_preconditioner(a), opts=SolverOptions(seed=0, max_iter=3000, **kw))
    meta, tr = z[f"{name}_meta"], z[f"{name}_trace"]
    assert rep.status == "converged" and bool(meta[4])
    assert abs(rep.iterations - int(meta[0])) <= 1
    n = min(len(rep.trace), tr.shape[0])
    for r, t in zip(rep.trace[:n], tr[:n]):
        assert r.n_locked == int(t[3]) and r.n_matvec == int(t[4]), r.iteration
        assert abs(r.trace_value - t[1]) <= 1e-10 * abs(t[1]), r.iteration
    ref = z[f"{name}_values"]
    assert np.max(np.abs(rep.values - ref) / np.abs(ref)) <= 1e-10
    assert _locked_ok(rep, kw["tol"]) == int(tr[-1][3])
    assert sine_angle(z[f"{name}_vec_lo"], rep.vectors[:, :4]) <= 1e-6
    assert sine_angle(z[f"{name}_vec_hi"], rep.vectors[:, -4:]) <= 1e-6
    assert max(rep.diagnostics["proj_defect"]) <= 1e-10


def test_config3_full_size_vs_arpack(cuda):
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner, ppcg_solve

    z = np.load(os.path.join(G, "eigsh_cfg3.npz"))
    a, k, q, tol = config_problem(3)
    rep = ppcg_solve(a, jacobi_preconditioner(a), opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=3000))
    assert rep.status == "converged"
    ev = z["values"]
    assert np.max(np.abs(rep.values[:ev.size] - ev) / np.abs(ev)) <= 1e-9
    _locked_ok(rep, tol)


def test_config4_full_size(cuda):
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner, ppcg_solve

    a, k, q, tol = config_problem(4)
    rep = ppcg_solve(a, jacobi_preconditioner(a), opts=SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=3000))
    assert rep.status == "converged"
    assert abs(rep.values[0] - 1.0) <= 1e-10  # exact: A = I + weighted graph Laplacian
    assert np.all(np.diff(rep.values) >= -1e-12)
    _locked_ok(rep, tol)
    path = os.path.join(G, "eigsh_cfg4.npz")
    if os.path.exists(path):
        ev = np.load(path)["values"]
        assert np.max(np.abs(rep.values[:ev.size] - ev) / np.abs(ev)) <= 1e-9
