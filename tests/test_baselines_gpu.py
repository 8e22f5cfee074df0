"""LOBPCG / Davidson baselines on the device kernels vs the reference
baselines.py run in the build container (tests/golden/baselines.npz, make_golden.py
--baselines), and the reference's own baseline tests (test_baselines.py,
test_acceptance.py:90-106) replayed on the device."""

import os

import numpy as np
import pytest

from util import sine_angle

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "baselines.npz"))


def _problem(name):
    from paper_1407_7506_b200 import (SparseHermitian, config_problem, jacobi_preconditioner, laplacian_1d,
                                      random_hermitian)

    if name == "rand90":
        return random_hermitian(90, 0.25, seed=17), None, dict(k=6, tol=1e-9, seed=9, max_iter=200)
    if name == "lap1d":
        a = laplacian_1d(300)
        return a, jacobi_preconditioner(a), dict(k=8, tol=1e-7, seed=0, max_iter=1500)
    if name == "cfg1s":
        a = SparseHermitian(config_problem(1, N=24)[0]._csr, "symmetric")
        return a, jacobi_preconditioner(a), dict(k=16, tol=1e-7, seed=0, max_iter=600)
    if name == "randz60":
        return random_hermitian(60, 0.5, seed=4, complex_field=True), None, dict(k=4, tol=1e-9, seed=1, max_iter=400)
    if name == "cfg5s":
        a = SparseHermitian(config_problem(5, N=8)[0]._csr, "hermitian")
        return a, jacobi_preconditioner(a), dict(k=16, tol=1e-6, seed=0, max_iter=600)
    raise KeyError(name)


@pytest.mark.parametrize("tag", ["lob", "dav"])
@pytest.mark.parametrize("name", ["rand90", "lap1d", "cfg1s", "randz60", "cfg5s"])
def test_baseline_matches_reference(cuda, tag, name):
    from paper_1407_7506_b200 import BaselineOptions, davidson_solve, lobpcg_solve

    a, t, kw = _problem(name)
    solve = lobpcg_solve if tag == "lob" else davidson_solve
    rep = solve(a, t, opts=BaselineOptions(**kw))
    pre = f"{tag}_{name}"
    meta = GOLD[f"{pre}_meta"]
    ref_tr = GOLD[f"{pre}_trace"]
    assert (rep.status == "converged") == bool(meta[4])
    n = min(len(rep.trace), len(ref_tr), 30)
    for r, g in zip(rep.trace[:n], ref_tr[:n]):
        assert r.n_locked == int(g[3]) and r.n_matvec == int(g[4])
        assert abs(r.trace_value - g[1]) <= 1e-10 * abs(g[1])
    # rounding-level differences can move a lock by an iteration or two late in a run
    assert abs(rep.iterations - int(meta[0])) <= max(1, int(0.05 * meta[0]))
    vals = GOLD[f"{pre}_values"]
    tol = 1e-9 if rep.status == "converged" else 1e-7  # a max_iter stop is mid-trajectory
    assert np.max(np.abs(rep.values - vals) / np.maximum(np.abs(vals), 1e-300)) <= tol
    if f"{pre}_vectors" in GOLD.files and rep.status == "converged":
        assert sine_angle(GOLD[f"{pre}_vectors"], rep.vectors) <= 1e-5


def test_whole_block_ppcg_tracks_lobpcg(cuda):
    """test_acceptance.py:90-106: whole-block PPCG with rr_period 1 follows LOBPCG's Ritz
    values to 1e-8 for 10 iterations (both on the device, and LOBPCG vs the reference)."""
    from paper_1407_7506_b200 import BaselineOptions, SolverOptions, lobpcg_solve, ppcg_solve, random_hermitian

    a = random_hermitian(100, 0.2, seed=12)
    x0 = GOLD["equiv_x0"]
    rp = ppcg_solve(a, x0=x0, opts=SolverOptions(k=8, nbuf=0, sbsize=8, rr_period=1, tol=1e-14, seed=5, max_iter=10))
    rl = lobpcg_solve(a, x0=x0, opts=BaselineOptions(k=8, nbuf=0, tol=1e-14, seed=5, max_iter=10))
    assert len(rp.values_history) >= 10 and len(rl.values_history) >= 10
    worst = max(float(np.max(np.abs(vp - vl))) for vp, vl in zip(rp.values_history[:10], rl.values_history[:10]))
    assert worst <= 1e-8
    ref = GOLD["equiv_lob_vhist"]
    assert max(float(np.max(np.abs(v - r))) for v, r in zip(rl.values_history[:10], ref)) <= 1e-10


def test_baseline_options_validation():
    from paper_1407_7506_b200 import BaselineOptions

    with pytest.raises(ValueError):
        BaselineOptions(k=0).validate()
    with pytest.raises(ValueError):
        BaselineOptions(k=2, restart_dim_multiple=1).validate()
    assert BaselineOptions(k=100).resolved_nbuf() == 2
