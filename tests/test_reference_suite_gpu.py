"""The reference's solver-level tests (test_ppcg.py::TestPpcgSolve, TestLockAndCompact's
end-to-end case) replayed on the device solver, with the same problems, options and bars
(restated here; the reference itself does not travel to the GPU box)."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gram(x):
    return x.conj().T @ x


def test_complex_hermitian_field(cuda):
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    a = random_hermitian(60, 0.5, seed=4, complex_field=True)
    ref = np.linalg.eigvalsh(a.to_dense())[:4]
    rep = ppcg_solve(a, opts=SolverOptions(k=4, tol=1e-9, seed=1, max_iter=400))
    assert rep.status == "converged"
    assert np.allclose(rep.values, ref, atol=1e-8)
    assert np.iscomplexobj(rep.vectors)


def test_report_invariants(cuda):
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    k = 6
    rep = ppcg_solve(random_hermitian(80, 0.3, seed=6), opts=SolverOptions(k=k, tol=1e-8, seed=2, max_iter=300))
    assert np.all(np.diff(rep.values) >= -1e-14)
    assert np.linalg.norm(_gram(rep.vectors) - np.eye(k)) <= 1e-8 * math.sqrt(k)


def test_projection_invariant_every_iteration(cuda):
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    rep = ppcg_solve(random_hermitian(70, 0.4, seed=11), opts=SolverOptions(k=5, tol=1e-9, seed=3, max_iter=150))
    assert max(rep.diagnostics["proj_defect"]) <= 1e-10


def test_orthonormality_maintained_under_every_policy(cuda):
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    rep = ppcg_solve(random_hermitian(70, 0.4, seed=12),
                     opts=SolverOptions(k=5, tol=1e-9, seed=4, max_iter=150, orth_policy="every"))
    assert max(rep.diagnostics["orth_loss"]) < 0.5


def test_trace_tol_secondary_criterion(cuda):
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    rep = ppcg_solve(random_hermitian(60, 0.4, seed=16),
                     opts=SolverOptions(k=4, tol=1e-30, trace_tol=1e-10, seed=8, max_iter=400))
    assert rep.status == "converged"


def test_locked_values_are_accurate_when_locked(cuda):
    from paper_1407_7506_b200 import DenseHermitian, SolverOptions, ppcg_solve

    rep = ppcg_solve(DenseHermitian(np.diag(np.arange(1.0, 51.0))),
                     opts=SolverOptions(k=10, nbuf=0, tol=1e-9, seed=8, max_iter=200))
    rows = [r for r in rep.trace if r.n_locked > 0]
    assert rows
    nl = rows[0].n_locked
    assert np.allclose(rep.values[:nl], np.arange(1.0, nl + 1.0), atol=1e-6)


def test_x0_wider_than_block_rejected(cuda):
    from paper_1407_7506_b200 import DimensionError, SolverOptions, ppcg_solve, random_hermitian

    with pytest.raises(DimensionError):
        ppcg_solve(random_hermitian(20, 0.5, seed=19), x0=np.eye(20)[:, :8], opts=SolverOptions(k=3, nbuf=0))


def test_k_total_larger_than_n_rejected(cuda):
    from paper_1407_7506_b200 import DimensionError, SolverOptions, ppcg_solve, random_hermitian

    with pytest.raises(DimensionError):
        ppcg_solve(random_hermitian(10, 0.5, seed=1), opts=SolverOptions(k=10, nbuf=2))


def test_partial_x0_is_padded_with_the_seeded_draw(cuda):
    """x0 narrower than k_total is padded with the seed's normals (ppcg.py:414-438): the run
    equals one started from the explicitly padded block."""
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian
    from paper_1407_7506_b200.ppcg import draw_initial_block

    a = random_hermitian(50, 0.4, seed=21)
    opts = SolverOptions(k=4, nbuf=2, tol=1e-9, seed=3, max_iter=100)
    x0 = np.random.default_rng(9).standard_normal((50, 2))
    full = draw_initial_block(50, 6, False, 3, x0)
    r1 = ppcg_solve(a, x0=x0, opts=opts)
    r2 = ppcg_solve(a, x0=full, opts=opts)
    assert np.array_equal(r1.values, r2.values) and r1.iterations == r2.iterations


def test_singular_user_operator_block_reports_rank_deficiency(cuda):
    """A rank-deficient x0 fails the initial Cholesky-QR with the failing column
    (core.py:67-83), as in the reference."""
    from paper_1407_7506_b200 import RankDeficiencyError, SolverOptions, ppcg_solve, random_hermitian

    a = random_hermitian(30, 0.5, seed=2)
    x0 = np.random.default_rng(0).standard_normal((30, 3))
    x0[:, 2] = x0[:, 0]
    with pytest.raises(RankDeficiencyError) as exc:
        ppcg_solve(a, x0=x0, opts=SolverOptions(k=3, nbuf=0, tol=1e-8))
    assert exc.value.column == 2
