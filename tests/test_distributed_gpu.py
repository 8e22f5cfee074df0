"""Row-partitioned solver on the GPU: ranks emulated as threads of one process
on one device (ThreadComm: host-side barriers, sums in rank order), so the whole sharded
path -- local CSR over the extended block, halo exchange, Gram/norm allreduces, replicated
small solves, gathered vectors -- runs through the CUDA kernels and is compared with the
single-GPU solver and the oracle.  (Real NCCL ranks need one GPU each; the CPU suite
covers TorchComm itself with gloo.)"""

import threading

import numpy as np
import pytest

from oracle import ppcg_oracle as O
from util import HostCsr, HostDiag, sine_angle

pytestmark = pytest.mark.gpu


def _run_ranks(size, a, t, opts):
    from paper_1407_7506_b200.distributed import dist_ppcg_solve, thread_comms

    comms = thread_comms(size)
    out, err = [None] * size, [None] * size

    def work(r):
        try:
            out[r] = dist_ppcg_solve(a, t, None, opts, comm=comms[r])
        except BaseException as e:  # noqa: BLE001
            err[r] = e
            comms[r].sh.barrier.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for x in th:
        x.start()
    for x in th:
        x.join(600)
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    assert all(o is not None for o in out)
    return out


@pytest.mark.parametrize("size", [2, 3])
def test_row_partition_matches_single_gpu(cuda, size):
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner, ppcg_solve

    a, _, _, _ = config_problem(1, N=24)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=16, sbsize=8, tol=1e-7, seed=0, max_iter=400)
    one = ppcg_solve(a, t, opts=opts)
    reps = _run_ranks(size, a, t, opts)
    for r in reps[1:]:  # every rank holds the same report
        assert np.array_equal(r.values, reps[0].values)
        assert r.iterations == reps[0].iterations and r.matvecs == reps[0].matvecs
    rep = reps[0]
    assert rep.status == one.status == "converged"
    assert abs(rep.iterations - one.iterations) <= 1
    assert np.max(np.abs(rep.values - one.values) / np.abs(one.values)) <= 1e-10
    assert sine_angle(one.vectors, rep.vectors) <= 1e-6
    n = min(len(rep.trace), len(one.trace), 30)
    for r1, r2 in zip(rep.trace[:n], one.trace[:n]):
        assert r1.n_locked == r2.n_locked and r1.n_matvec == r2.n_matvec
        assert abs(r1.trace_value - r2.trace_value) <= 1e-11 * abs(r2.trace_value)
    assert max(rep.diagnostics["proj_defect"]) <= 1e-10


def test_row_partition_complex_and_q64_vs_oracle(cuda):
    """complex Hermitian (Peierls, cfg5 structure) and sbsize 64 (cfg3 structure) over 2
    ranks vs the oracle trajectory from the same X0."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner

    for cfg, N, k, q, iters in ((5, 6, 12, 4, 12), (3, 10, 100, 64, 8)):
        a, _, _, tol = config_problem(cfg, N=N)
        t = jacobi_preconditioner(a)
        opts = SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=iters)
        rep = _run_ranks(2, a, t, opts)[0]
        ref = O.oracle_solve(HostCsr(a._csr), HostDiag(t.d), opts=opts)
        assert rep.iterations == ref.iterations
        for r1, r2 in zip(rep.trace, ref.trace):
            assert r1.n_locked == r2.n_locked and r1.n_matvec == r2.n_matvec
            assert abs(r1.trace_value - r2.trace_value) <= 1e-11 * abs(r2.trace_value)
        assert np.max(np.abs(rep.values - ref.values) / np.abs(ref.values)) <= 1e-9


def test_torchrun_two_ranks_cli(cuda, tmp_path):
    """Real processes: `torchrun --nproc-per-node 2 -m paper_1407_7506_b200 solve --ngpus 2`
    (TorchComm; gloo with host staging so both ranks fit one GPU -- NCCL needs one GPU per
    rank) gives the single-GPU eigenvalues."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    args = ["solve", "--solver", "ppcg", "--problem", "config:1,16", "--k", "12", "--sbsize", "4",
            "--precond", "jacobi", "--tol", "1e-8", "--max-iter", "300"]
    env = dict(os.environ, PPCG_DIST_BACKEND="gloo", PYTHONPATH=root)
    one = subprocess.run([sys.executable, "-m", "paper_1407_7506_b200"] + args, cwd=root, env=env,
                         capture_output=True, text=True, timeout=300)
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29571", "-m", "paper_1407_7506_b200"]
                         + args + ["--ngpus", "2"], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0 and two.returncode == 0, two.stderr[-2000:]

    def values(out):
        lines = out.splitlines()
        i = lines.index("eigenvalues:")
        return np.array([float(v) for v in lines[i + 1:i + 13]])

    v1, v2 = values(one.stdout), values(two.stdout)
    assert np.max(np.abs(v1 - v2) / np.abs(v1)) <= 1e-10


def test_row_partition_more_ranks_than_pencils(cuda):
    """The split pencils (reduce-scatter, a chunk of subblocks per rank, all-gather) when the
    subblocks do not divide over the ranks: 2 subblocks on 3 ranks (rank 2 solves none)."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner

    a, _, _, _ = config_problem(1, N=12)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=4, sbsize=4, tol=1e-9, seed=0, max_iter=60)
    rep = _run_ranks(3, a, t, opts)[0]
    ref = O.oracle_solve(HostCsr(a._csr), HostDiag(t.d), opts=opts)
    assert rep.iterations == ref.iterations
    for r1, r2 in zip(rep.trace, ref.trace):
        assert r1.n_locked == r2.n_locked and r1.n_matvec == r2.n_matvec
        assert abs(r1.trace_value - r2.trace_value) <= 1e-11 * abs(r2.trace_value)
    assert np.max(np.abs(rep.values - ref.values) / np.abs(ref.values)) <= 1e-10


def test_row_partition_breakdown_recovery(cuda, monkeypatch):
    """Breakdown recovery over a row partition (ppcg.py:698-717): the orthonormal basis of the
    pre-update X comes from shifted Cholesky-QR3 over the ranks instead of a gathered
    Householder QR (same Q up to column signs, which PPCG is equivariant to): the trajectory
    still follows the oracle's."""
    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner
    from paper_1407_7506_b200 import ppcg as PP

    monkeypatch.setattr(PP, "_BREAKDOWN_MAX", 0.27)
    monkeypatch.setattr(O, "BREAKDOWN_MAX", 0.27)
    a, _, _, _ = config_problem(1, N=16)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=12, sbsize=4, tol=1e-8, seed=0, max_iter=25)
    rep = _run_ranks(2, a, t, opts)[0]
    ref = O.oracle_solve(HostCsr(a._csr), HostDiag(t.d), opts=opts)
    assert ref.breakdown_recoveries > 0
    assert rep.iterations == ref.iterations and rep.breakdown_recoveries == ref.breakdown_recoveries
    for r1, r2 in zip(rep.trace, ref.trace):
        assert r1.n_locked == r2.n_locked and r1.n_matvec == r2.n_matvec
        assert abs(r1.trace_value - r2.trace_value) <= 1e-10 * abs(r2.trace_value)


def test_root_gather_and_memory_plan(cuda):
    """gather="root": rank 0 holds the (n, k) vectors, the others their own rows only; and the
    device memory the solver allocates stays within device_bytes_plan's per-rank budget."""
    import threading

    import torch

    from paper_1407_7506_b200 import SolverOptions, config_problem, jacobi_preconditioner
    from paper_1407_7506_b200.distributed import dist_ppcg_solve, thread_comms
    from paper_1407_7506_b200.ppcg import PPCGSolver, device_bytes_plan

    a, _, _, _ = config_problem(3, N=16)
    t = jacobi_preconditioner(a)
    opts = SolverOptions(k=60, sbsize=16, tol=1e-6, seed=0, max_iter=6)
    comms = thread_comms(2)
    out = [None, None]

    def work(r):
        out[r] = dist_ppcg_solve(a, t, None, opts, comm=comms[r], gather="root")

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(300)
    assert out[0].vectors.shape == (a.n, 60)
    lo, hi = out[1].diagnostics["vector_rows"]
    np.testing.assert_array_equal(out[1].vectors, out[0].vectors[lo:hi])
    # single-rank allocation vs the plan (state blocks, Grams, pencils, operator, workspaces)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    s = PPCGSolver(a, t, None, opts).start()
    for _ in range(3):
        s.step()
    torch.cuda.synchronize()
    used = torch.cuda.max_memory_allocated() - base
    kt = s.kt
    plan = device_bytes_plan(a.n, a.n, kt, 16, False, a._csr.nnz, 1)
    assert used <= plan["total"], (used, plan)
    assert plan["state_blocks"] >= 8 * a.n * ((kt + 15) // 16 * 16) * 8
    del s
