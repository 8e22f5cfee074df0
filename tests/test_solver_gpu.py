"""Solver-level parity of the device PPCG against the CPU oracle (numpy restatement of the
reference ppcg_solve) and against the reference's own solver-level tests
(test_ppcg.py::TestPpcgSolve, test_acceptance.py) replayed on the device solver."""

import math

import numpy as np
import pytest

from oracle import ppcg_oracle as O
from util import HostCsr, HostDense, HostDiag, sine_angle

pytestmark = pytest.mark.gpu


def _solve_both(a_dev, a_host, t_dev, t_host, opts, x0=None):
    from paper_1407_7506_b200 import ppcg_solve

    rep = ppcg_solve(a_dev, t_dev, x0=x0, opts=opts)
    ref = O.oracle_solve(a_host, t_host, x0=x0, opts=opts)
    return rep, ref


def test_config1_parity_vs_oracle(cuda):
    """BASELINE config 1 (2-D 5-pt 64^2 + V, k=64, q=8, Jacobi, tol 1e-6), same seeded X0."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner

    a, k, q, tol = config_problem(1)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=2000)
    rep, ref = _solve_both(a, HostCsr(a._csr), t, HostDiag(t.d), opts)
    assert rep.status == ref.status == "converged"
    # trajectory parity: same iteration count (+-1) and lock schedule
    assert abs(rep.iterations - ref.iterations) <= 1
    assert rep.rr_count in (ref.rr_count, ref.rr_count + 1, ref.rr_count - 1)
    # eigenvalues: relative 1e-10
    assert np.max(np.abs(rep.values - ref.values) / np.abs(ref.values)) <= 1e-10
    # subspace: max principal angle (sine form) <= 1e-6 vs the oracle's converged subspace
    assert sine_angle(ref.vectors, rep.vectors) <= 1e-6
    # residual criterion in the reference's own metric
    assert rep.trace[-1].rel_resid > opts.tol
    assert max(rep.diagnostics["proj_defect"]) <= 1e-10
    n = min(len(rep.trace), len(ref.trace), 40)
    for r1, r2 in zip(rep.trace[:n], ref.trace[:n]):
        assert r1.n_locked == r2.n_locked
        assert r1.n_matvec == r2.n_matvec
        assert abs(r1.trace_value - r2.trace_value) <= 1e-12 * abs(r2.trace_value)


def test_laplacian_analytic_spectrum(cuda):
    from paper_1407_7506_b200 import SolverOptions, laplacian_1d, ppcg_solve

    n, k = 500, 10
    rep = ppcg_solve(laplacian_1d(n), opts=SolverOptions(k=k, tol=1e-6, seed=0, max_iter=2000))
    analytic = 2.0 - 2.0 * np.cos(np.arange(1, k + 1) * np.pi / (n + 1))
    assert rep.status == "converged"
    assert np.allclose(rep.values, analytic, atol=1e-8)


def test_jacobi_preconditioned_laplacian(cuda):
    from paper_1407_7506_b200 import SolverOptions, jacobi_preconditioner, laplacian_1d, ppcg_solve

    n, k = 300, 6
    a = laplacian_1d(n)
    rep = ppcg_solve(a, jacobi_preconditioner(a), opts=SolverOptions(k=k, tol=1e-7, seed=0, max_iter=1500))
    analytic = 2.0 - 2.0 * np.cos(np.arange(1, k + 1) * np.pi / (n + 1))
    assert rep.status == "converged"
    assert np.allclose(rep.values, analytic, atol=1e-8)


def test_random_sparse_matches_oracle_trajectory(cuda):
    from paper_1407_7506_b200 import SolverOptions, random_hermitian

    a = random_hermitian(90, 0.25, seed=17)
    opts = SolverOptions(k=6, sbsize=2, tol=1e-9, seed=9, max_iter=80)
    rep, ref = _solve_both(a, HostCsr(a._csr), None, None, opts)
    assert rep.status == ref.status
    assert abs(rep.iterations - ref.iterations) <= 1
    assert np.allclose(rep.values, ref.values, rtol=1e-10, atol=1e-12)


def test_determinism_bitwise(cuda):
    """test_ppcg.py:325-341: reruns (and any `threads`) are bitwise identical."""
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    a = random_hermitian(90, 0.25, seed=17)

    def run(threads):
        return ppcg_solve(a, opts=SolverOptions(k=6, sbsize=2, tol=1e-9, seed=9, max_iter=80), threads=threads)

    r1, r2, r4 = run(1), run(1), run(4)
    for other in (r2, r4):
        assert len(r1.trace) == len(other.trace)
        for t1, t2 in zip(r1.trace, other.trace):
            assert t1.trace_value == t2.trace_value and t1.rel_resid == t2.rel_resid
            assert t1.n_locked == t2.n_locked and t1.n_matvec == t2.n_matvec
        assert np.array_equal(r1.values, other.values)
        assert np.array_equal(r1.vectors, other.vectors)


def test_dense_diag_problem(cuda):
    from paper_1407_7506_b200 import DenseHermitian, DiagonalOperator, SolverOptions, ppcg_solve

    a = DenseHermitian(np.diag(np.arange(1.0, 101.0)))
    opts = SolverOptions(k=5, nbuf=2, sbsize=1, rr_period=5, tol=1e-8, seed=3, max_iter=400)
    rep = ppcg_solve(a, DiagonalOperator(np.ones(100)), opts=opts)
    assert rep.status == "converged"
    assert np.allclose(rep.values, [1, 2, 3, 4, 5], atol=1e-7)


def test_exact_invariant_start(cuda):
    from paper_1407_7506_b200 import DenseHermitian, SolverOptions, ppcg_solve

    a = DenseHermitian(np.diag(np.arange(1.0, 11.0)))
    rep = ppcg_solve(a, x0=np.eye(10)[:, :2], opts=SolverOptions(k=2, nbuf=0, tol=1e-10))
    assert rep.status == "converged" and rep.iterations == 0 and len(rep.trace) == 0
    assert np.allclose(rep.values, [1.0, 2.0], atol=1e-12)


def test_max_iter_zero_and_trace_rows(cuda):
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    a = random_hermitian(30, 0.5, seed=18)
    rep = ppcg_solve(a, opts=SolverOptions(k=3, tol=1e-12, seed=1, max_iter=0))
    assert rep.status == "max_iter" and rep.iterations == 0 and len(rep.trace) == 0
    assert rep.values.shape == (3,)
    b = random_hermitian(50, 0.4, seed=15)
    rep = ppcg_solve(b, opts=SolverOptions(k=4, tol=1e-20, seed=7, max_iter=9))
    assert rep.status == "max_iter" and rep.iterations == 9 and len(rep.trace) == 9


def test_rr_period_inf(cuda):
    from paper_1407_7506_b200 import DenseHermitian, SolverOptions, ppcg_solve

    a = DenseHermitian(np.diag(np.arange(1.0, 41.0)))
    rep = ppcg_solve(a, opts=SolverOptions(k=3, nbuf=0, rr_period=math.inf, tol=1e-8, seed=2, max_iter=60))
    assert rep.rr_count == 1 and len(rep.values_history) == 0


def test_policies_and_taylor(cuda):
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian

    a = random_hermitian(80, 0.3, seed=13)
    w_ref = np.linalg.eigvalsh(a.to_dense())[:4]
    rep = ppcg_solve(a, opts=SolverOptions(k=4, tol=1e-8, seed=5, max_iter=300, orth_scheme="taylor-polar"))
    assert rep.status == "converged" and np.allclose(rep.values, w_ref, atol=1e-7)
    b = random_hermitian(80, 0.3, seed=14)
    w_ref = np.linalg.eigvalsh(b.to_dense())[:4]
    rep = ppcg_solve(b, opts=SolverOptions(k=4, tol=1e-8, seed=6, max_iter=400, orth_policy="adaptive"))
    assert rep.status == "converged" and np.allclose(rep.values, w_ref, atol=1e-7)


def test_well_problem_golden_iterations(cuda):
    """Acceptance C3/C5 golden counts (test_acceptance.py:30-36): 14 and 21 iterations."""
    from paper_1407_7506_b200 import SolverOptions, jacobi_preconditioner, ppcg_solve, well_problem

    a = well_problem(8, 8, 8, depth=80.0, seed=3)
    t = jacobi_preconditioner(a, shift=-90.0)
    rep = ppcg_solve(a, t, opts=SolverOptions(k=10, nbuf=2, sbsize=5, rr_period=5, tol=1e-4, seed=1, max_iter=140))
    assert rep.status == "converged" and rep.iterations <= 14
    rep5 = ppcg_solve(a, t, opts=SolverOptions(k=10, nbuf=2, sbsize=5, rr_period=5, tol=1e-6, seed=1, max_iter=210))
    assert rep5.status == "converged" and rep5.iterations <= 21


@pytest.mark.parametrize("cfg,N,k,iters", [(3, 14, 128, 12), (4, 8, 128, 10), (5, 8, 124, 10)])
def test_q64_scaled_configs_match_oracle_trajectory(cuda, cfg, N, k, iters):
    """Configs 3-5 run with sbsize 64 (pencils of dimension 192, the global-workspace pencil
    variant; complex at cfg5): scaled-down instances of the same operators, first iterations
    of the trace vs the oracle from the same seeded X0."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner

    a, _, q, tol = config_problem(cfg, N=N)
    assert q == 64
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=iters)
    rep, ref = _solve_both(a, HostCsr(a._csr), t, HostDiag(t.d), opts)
    assert rep.iterations == ref.iterations == iters
    for r1, r2 in zip(rep.trace, ref.trace):
        assert r1.n_locked == r2.n_locked and r1.n_matvec == r2.n_matvec
        assert abs(r1.trace_value - r2.trace_value) <= 1e-11 * abs(r2.trace_value)
        assert abs(r1.rel_resid - r2.rel_resid) <= 1e-6 * r2.rel_resid
    assert np.max(np.abs(rep.values - ref.values) / np.abs(ref.values)) <= 1e-9
    assert max(rep.diagnostics["proj_defect"]) <= 1e-10


@pytest.mark.parametrize("cfg,N,k,sb,iters", [(1, 24, 64, 66, 14), (5, 8, 64, 66, 10), (3, 9, 80, 41, 8)])
def test_large_pencils_whole_block_vs_oracle(cuda, cfg, N, k, sb, iters):
    """Subblocks whose pencil exceeds the batched kernels (3q > 192: whole-block PPCG, the
    LOBPCG-equivalent mode of test_acceptance.py:90-106) go through bigblock.py: host-side
    block_update branches, device Grams/cuSOLVER/tsgemm.  Real and complex, vs the oracle
    trajectory from the same X0 (iteration 1 has no P and still uses the batched pencils)."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner

    a, _, _, tol = config_problem(cfg, N=N)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=k, sbsize=sb, tol=1e-9, seed=0, max_iter=iters)
    rep, ref = _solve_both(a, HostCsr(a._csr), t, HostDiag(t.d), opts)
    assert rep.iterations == ref.iterations
    for r1, r2 in zip(rep.trace, ref.trace):
        assert r1.n_locked == r2.n_locked and r1.n_matvec == r2.n_matvec
        assert abs(r1.trace_value - r2.trace_value) <= 1e-11 * abs(r2.trace_value)
    assert rep.breakdown_recoveries == ref.breakdown_recoveries
    assert np.max(np.abs(rep.values - ref.values) / np.abs(ref.values)) <= 1e-9


@pytest.mark.parametrize("which", ["refresh", "breakdown"])
def test_guard_branches_match_oracle(cuda, monkeypatch, which):
    """The cache-refresh (coeff_scale > threshold: two extra operator applies, ppcg.py:718-724)
    and breakdown-recovery (max |X|,|P| > threshold: Householder QR of the pre-update X, P
    dropped, ppcg.py:698-717) branches, forced by lowering their thresholds in both the device
    solver and the oracle: same recoveries/refresh counts, matvec counts and trajectory."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner
    from paper_1407_7506_b200 import ppcg as PP

    if which == "refresh":
        monkeypatch.setattr(PP, "_COEFF_REFRESH", 0.99)   # coeff_scale >= 1: refresh every iteration
        monkeypatch.setattr(O, "COEFF_REFRESH", 0.99)
    else:
        monkeypatch.setattr(PP, "_BREAKDOWN_MAX", 0.27)   # one recovery in the oracle's run
        monkeypatch.setattr(O, "BREAKDOWN_MAX", 0.27)
    a, _, _, _ = config_problem(1, N=16)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=12, sbsize=4, tol=1e-8, seed=0, max_iter=25)
    rep, ref = _solve_both(a, HostCsr(a._csr), t, HostDiag(t.d), opts)
    assert rep.iterations == ref.iterations
    assert rep.breakdown_recoveries == ref.breakdown_recoveries
    assert rep.diagnostics["cache_refreshes"] == ref.diagnostics["cache_refreshes"]
    if which == "refresh":
        assert ref.diagnostics["cache_refreshes"] > 0
    else:
        assert ref.breakdown_recoveries > 0
    for r1, r2 in zip(rep.trace, ref.trace):
        assert r1.n_locked == r2.n_locked and r1.n_matvec == r2.n_matvec
        assert abs(r1.trace_value - r2.trace_value) <= 1e-10 * abs(r2.trace_value)


def test_operator_arrays_replaced_after_solve(cuda):
    """The device copy of an operator follows its host arrays: replacing the CSR values after
    a solve (here A -> 2A) gives the new spectrum, not the cached one (operators.py
    as_device_operator, keyed by the source arrays)."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, ppcg_solve

    a, _, _, _ = config_problem(1, N=12)
    opts = SolverOptions(k=4, sbsize=4, tol=1e-9, seed=0, max_iter=400)
    v1 = ppcg_solve(a, opts=opts).values
    a._csr.data = a._csr.data * 2.0
    v2 = ppcg_solve(a, opts=opts).values
    np.testing.assert_allclose(v2, 2.0 * v1, rtol=1e-9)


def test_result_vectors_pool_never_aliases_live_results(cuda):
    """The page-locked result pool (ppcg._pinned_take): a solve's vectors stay intact while the
    caller holds them (or any view of them) -- the next solve gets other memory -- and the
    buffer is reused once they are dropped; results are the same either way."""
    import gc

    from paper_1407_7506_b200 import SolverOptions, ppcg_solve, random_hermitian
    from paper_1407_7506_b200 import ppcg as PP

    a = random_hermitian(400, 0.05, seed=21)
    b = random_hermitian(400, 0.05, seed=22)
    opts = SolverOptions(k=6, sbsize=3, tol=1e-8, seed=1, max_iter=60)
    r1 = ppcg_solve(a, opts=opts)
    v1 = r1.vectors.copy()
    view = r1.vectors[5:, :2]          # a view keeps the buffer leased
    p1 = r1.vectors.ctypes.data
    del r1
    gc.collect()
    r2 = ppcg_solve(b, opts=opts)      # same shape: must not land in the leased buffer
    assert r2.vectors.ctypes.data != p1
    assert np.array_equal(view, v1[5:, :2])
    del view
    gc.collect()
    r3 = ppcg_solve(a, opts=opts)
    assert np.array_equal(r3.vectors, v1) and np.array_equal(r3.values, ppcg_solve(a, opts=opts).values)
    leased = [e for e in PP._RESULT_POOL if e[1]() is not None]
    assert len(PP._RESULT_POOL) >= 1 and len(leased) <= len(PP._RESULT_POOL)
