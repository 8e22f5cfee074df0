"""Pin the CPU oracle (oracle/ppcg_oracle.py) against golden vectors produced by the
reference itself (tests/golden/make_golden.py), and pin our host-side problem generators
against the reference's.  CPU only."""

import math
import os

import numpy as np
import pytest

from oracle import ppcg_oracle as O
from util import HostCsr, HostDense, HostDiag

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


class Opts:
    def __init__(self, **kw):
        base = dict(k=1, nbuf=None, sbsize=5, rr_period=5, tol=1e-6, trace_tol=None, max_iter=500,
                    orth_policy="every", orth_period=1, orth_threshold=0.1, orth_scheme="cholesky-qr",
                    taylor_terms=4, seed=0, project_w=True, project_p=True)
        base.update(kw)
        self.__dict__.update(base)


def test_block_inner_golden():
    z = load("kernels.npz")
    assert np.allclose(O.herm_gram(z["gram_x"], z["gram_y"]), z["gram_out"], rtol=0, atol=1e-13)
    assert np.allclose(O.herm_gram(z["gramz_x"], z["gramz_y"]), z["gramz_out"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("tag", ["p24", "p96", "pz12"])
def test_solve_pencil_golden(tag):
    z = load("kernels.npz")
    a, b, om, c = z[f"{tag}_a"], z[f"{tag}_b"], z[f"{tag}_omega"], z[f"{tag}_c"]
    w, cc = O.solve_small_pencil(a, b, om.shape[0])
    assert np.allclose(w, om, rtol=0, atol=1e-12 * max(1.0, np.abs(om).max()))
    # eigenvectors up to a unit-modulus column factor
    for j in range(cc.shape[1]):
        ph = np.vdot(cc[:, j], c[:, j])
        ph /= abs(ph)
        assert np.allclose(cc[:, j] * ph, c[:, j], atol=1e-9)


def test_cholesky_qr_golden_and_rank_column():
    z = load("kernels.npz")
    q, r = O.cholqr(z["cqr_x"])
    assert np.allclose(q, z["cqr_q"], atol=1e-13) and np.allclose(r, z["cqr_r"], atol=1e-13)
    with pytest.raises(O.OracleRankDeficiency) as e:
        O.cholqr(z["cqr_xd"])
    assert e.value.column == int(z["cqr_fail_col"]) == 2


def test_polar_and_metrics_golden():
    z = load("kernels.npz")
    assert np.allclose(O.taylor_poly(z["polar_gram"], 4), z["polar_poly"], atol=1e-14)
    rel, tr, chg = O.stop_metrics(z["met_x"], z["met_ax"], 1.5)
    assert np.allclose([rel, tr, chg], z["met_out"], rtol=1e-13, atol=0)


def test_block_update_golden():
    z = load("kernels.npz")
    a, x, w, p = z["bu_a"], z["bu_x"], z["bu_w"], z["bu_p"]
    r = O.subblock_update(x, w, p, a @ x, a @ w, a @ p)
    assert np.allclose(r.theta, z["bu_theta"], atol=1e-12)
    assert int(r.used_fallback) == int(z["bu_fb"])
    for c in range(x.shape[1]):
        s = np.sign(np.dot(r.x[:, c], z["bu_xo"][:, c]))
        assert np.allclose(s * r.x[:, c], z["bu_xo"][:, c], atol=1e-10)
        assert np.allclose(s * r.p[:, c], z["bu_po"][:, c], atol=1e-10)
    assert abs(r.coeff_scale - float(z["bu_cs"])) <= 1e-10 * float(z["bu_cs"])
    d2 = np.diag([1.0, 2.0])
    rf = O.subblock_update(np.eye(2)[:, 1:2], np.eye(2)[:, 0:1], None, d2 @ np.eye(2)[:, 1:2], d2 @ np.eye(2)[:, 0:1], None)
    assert rf.used_fallback and int(z["fb_used"]) == 1
    assert np.allclose(abs(rf.x), abs(z["fb_x"]), atol=1e-12)


def test_generators_match_reference():
    from paper_1407_7506_b200 import problems as P

    z = load("generators.npz")
    ours = {"lap3d": P.laplacian_3d(5, 4, 3), "well": P.well_problem(6, 6, 6, depth=40.0, seed=3),
            "rand": P.random_hermitian(40, 0.3, seed=5), "randz": P.random_hermitian(30, 0.4, seed=6, complex_field=True)}
    for k, op in ours.items():
        c = op._csr
        assert np.array_equal(c.indptr, z[f"{k}_indptr"]) and np.array_equal(c.indices, z[f"{k}_indices"])
        assert np.array_equal(c.data, z[f"{k}_data"])
    t = P.jacobi_preconditioner(ours["well"], shift=-90.0)
    assert np.array_equal(t.d, z["well_jacobi"])


def _check_solve(rep, z, prefix, exact_iters=True):
    meta = z[f"{prefix}_meta"]
    assert rep.iterations == int(meta[0]) if exact_iters else abs(rep.iterations - int(meta[0])) <= 1
    assert rep.matvecs == int(meta[1]) and rep.rr_count == int(meta[2])
    assert (rep.status == "converged") == bool(meta[4])
    assert np.allclose(rep.values, z[f"{prefix}_values"], rtol=1e-12, atol=1e-14)
    tr = z[f"{prefix}_trace"]
    assert len(rep.trace) == tr.shape[0]
    for r, t in zip(rep.trace, tr):
        assert r.iteration == int(t[0]) and r.n_locked == int(t[3]) and r.n_matvec == int(t[4])
        assert abs(r.trace_value - t[1]) <= 1e-12 * max(1.0, abs(t[1]))


def test_oracle_config1_matches_reference_run():
    """The oracle reproduces the reference's config-1 run (162 it, 33 RR, 7929 matvecs)."""
    from paper_1407_7506_b200 import config_problem, jacobi_preconditioner

    a, k, q, tol = config_problem(1)
    t = jacobi_preconditioner(a)
    rep = O.oracle_solve(HostCsr(a._csr), HostDiag(t.d), opts=Opts(k=k, sbsize=q, tol=tol, seed=0, max_iter=2000))
    z = load("cfg1.npz")
    _check_solve(rep, z, "cfg1")
    assert np.allclose(rep.diagnostics["final_residual_norms"], z["cfg1_final_rn"], rtol=1e-6, atol=1e-14)


@pytest.mark.parametrize("name", ["lap1d", "rand90", "randz60", "well_tol4", "well_tol6", "cfg4_n12", "cfg5_n8"])
def test_oracle_small_solves_match_reference(name):
    from paper_1407_7506_b200 import problems as P

    z = load("solves.npz")
    if name == "lap1d":
        a, t, kw = P.laplacian_1d(500), None, dict(k=10, tol=1e-6, seed=0, max_iter=2000)
    elif name == "rand90":
        a, t, kw = P.random_hermitian(90, 0.25, seed=17), None, dict(k=6, sbsize=2, tol=1e-9, seed=9, max_iter=80)
    elif name == "randz60":
        a, t, kw = P.random_hermitian(60, 0.5, seed=4, complex_field=True), None, dict(k=4, tol=1e-9, seed=1, max_iter=400)
    elif name.startswith("well"):
        a = P.well_problem(8, 8, 8, depth=80.0, seed=3)
        t = P.jacobi_preconditioner(a, shift=-90.0)
        kw = dict(k=10, nbuf=2, sbsize=5, rr_period=5, tol=1e-4 if name == "well_tol4" else 1e-6, seed=1,
                  max_iter=140 if name == "well_tol4" else 210)
    elif name == "cfg4_n12":
        a, _, _, _ = P.config_problem(4, N=12)
        t = P.jacobi_preconditioner(a)
        kw = dict(k=32, sbsize=8, tol=1e-5, seed=0, max_iter=400)
    else:
        a, _, _, _ = P.config_problem(5, N=8)
        t = P.jacobi_preconditioner(a)
        kw = dict(k=16, sbsize=4, tol=1e-5, seed=0, max_iter=400)
    rep = O.oracle_solve(HostCsr(a._csr), None if t is None else HostDiag(t.d), opts=Opts(**kw))
    _check_solve(rep, z, name)
    if name == "well_tol4":
        assert rep.iterations <= 14  # PROJECTION_BASELINE_ITERS, test_acceptance.py:30-33
    if name == "well_tol6":
        assert rep.iterations <= 21  # RR5_ITERS, test_acceptance.py:34-36


@pytest.mark.skipif(not os.path.exists(os.path.join(G, "cfg2_iter2.npz")) or not os.environ.get("PPCG_SLOW"),
                    reason="config-2 golden pin is slow (set PPCG_SLOW=1)")
def test_oracle_config2_first_iterations():
    from paper_1407_7506_b200 import config_problem, jacobi_preconditioner

    a, k, q, tol = config_problem(2)
    t = jacobi_preconditioner(a)
    rep = O.oracle_solve(HostCsr(a._csr), HostDiag(t.d), opts=Opts(k=k, sbsize=q, tol=tol, seed=0, max_iter=2),
                         blas_threads=None)
    z = load("cfg2_iter2.npz")
    tr = z["cfg2_trace"]
    for r, t_ in zip(rep.trace, tr):
        assert abs(r.trace_value - t_[1]) <= 1e-12 * abs(t_[1])
        assert abs(r.rel_resid - t_[2]) <= 1e-10 * abs(t_[2])
    assert np.allclose(rep.values, z["cfg2_values"], rtol=1e-11)
