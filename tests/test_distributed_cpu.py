"""Host side of the row-partitioned solver on CPU: the partition, the halo
plan and local CSR, and the torch.distributed communicator over gloo with world_size 2
(allreduce sum/max, the halo exchange feeding a sharded SpMM, gathered rows)."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from paper_1407_7506_b200.distributed import HaloPlan, local_rows_csr, partition_rows


def _problems():
    from paper_1407_7506_b200 import config_problem, random_hermitian

    return [("cfg1", config_problem(1, N=16)[0]._csr), ("cfg4", config_problem(4, N=6)[0]._csr),
            ("cfg5", config_problem(5, N=6)[0]._csr), ("rand", random_hermitian(90, 0.25, seed=17)._csr)]


def test_partition_rows_covers_and_balances():
    rp = np.arange(0, 7 * 1001, 7)
    for size in (1, 2, 3, 7, 8):
        for b in (partition_rows(1000, size), partition_rows(1000, size, rp)):
            assert b[0][0] == 0 and b[-1][1] == 1000
            assert all(lo < hi for lo, hi in b)
            assert all(b[i][1] == b[i + 1][0] for i in range(size - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition_rows(3, 4)


@pytest.mark.parametrize("size", [1, 2, 3, 4])
def test_halo_plan_local_spmm_equals_global(size):
    rng = np.random.default_rng(0)
    for name, csr in _problems():
        n = csr.shape[0]
        bounds = partition_rows(n, size, csr.indptr)
        x = rng.standard_normal((n, 5))
        if np.iscomplexobj(csr.data):
            x = x + 1j * rng.standard_normal((n, 5))
        y = csr @ x
        plans = [HaloPlan(csr, bounds, r) for r in range(size)]
        for r, p in enumerate(plans):
            loc = local_rows_csr(csr, p.lo, p.hi, p.g_lo, p.n_ext)
            assert loc.shape == (p.hi - p.lo, p.n_ext)
            # the extended block = owned rows + received ghost rows, nothing else is read
            ext = np.zeros((p.n_ext, 5), dtype=x.dtype)
            ext[p.top:p.top + p.hi - p.lo] = x[p.lo:p.hi]
            for peer, a, b in p.recv:
                assert bounds[peer][0] <= a < b <= bounds[peer][1]
                ext[a - p.g_lo:b - p.g_lo] = x[a:b]
            np.testing.assert_allclose(loc @ ext, y[p.lo:p.hi], rtol=1e-13, atol=1e-13)
            # what r receives from s is exactly what s sends to r, in the same order
            for s_ in range(size):
                got = [(a, b) for peer, a, b in p.recv if peer == s_]
                sent = [(a, b) for peer, a, b in plans[s_].send if peer == r]
                assert got == sent, (name, r, s_)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, size, port, q):
    import torch
    import torch.distributed as dist

    from paper_1407_7506_b200 import config_problem
    from paper_1407_7506_b200.distributed import HaloPlan, TorchComm, local_rows_csr, partition_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        comm = TorchComm()
        res = {}
        # sums / max exactly as the solver uses them
        t = torch.arange(6, dtype=torch.float64) * (rank + 1)
        comm.allreduce_sum(t)
        res["sum"] = t.tolist()
        z = torch.tensor([1 + 2j, rank - 1j], dtype=torch.complex128)
        comm.allreduce_sum(z)
        res["zsum"] = z.tolist()
        f = torch.tensor([rank, 10 - rank, 0], dtype=torch.int64)
        comm.allreduce_max(f)
        res["max"] = f.tolist()
        # sharded SpMM through the halo exchange
        csr = config_problem(4, N=6)[0]._csr
        n = csr.shape[0]
        bounds = partition_rows(n, size, csr.indptr)
        p = HaloPlan(csr, bounds, rank)
        x = np.random.default_rng(3).standard_normal((n, 4))
        base = torch.zeros((p.n_ext, 4), dtype=torch.float64)
        base[p.top:p.top + p.hi - p.lo] = torch.from_numpy(x[p.lo:p.hi])
        comm.exchange([(peer, base[a - p.g_lo:b - p.g_lo]) for peer, a, b in p.send],
                      [(peer, base[a - p.g_lo:b - p.g_lo]) for peer, a, b in p.recv])
        loc = local_rows_csr(csr, p.lo, p.hi, p.g_lo, p.n_ext)
        y = loc @ base.numpy()
        res["spmm_err"] = float(np.max(np.abs(y - (csr @ x)[p.lo:p.hi])))
        full = comm.allgather_rows(torch.from_numpy(y), bounds)
        res["gather_err"] = float(np.max(np.abs(full.numpy() - csr @ x)))
        # the split pencils' collectives and the host assembly of the vectors
        rs = (torch.arange(8, dtype=torch.float64) + 1) * (rank + 1)
        comm.reduce_scatter_sum(rs, 4)
        res["rs"] = rs[4 * rank:4 * rank + 4].tolist()
        ag = torch.zeros(6, dtype=torch.complex128)
        ag[3 * rank:3 * rank + 3] = torch.tensor([rank + 1j, 2.0 * rank, -1j * rank])
        comm.allgather_chunks(ag, 3)
        res["ag"] = ag.tolist()
        res["host_all"] = comm.gather_rows_host(y, bounds, mode="all")
        res["host_root"] = comm.gather_rows_host(y, bounds, mode="root")
        res["y_full"] = csr @ x
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_torchcomm_gloo_world2():
    import torch.multiprocessing as mp

    size = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(size))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(size):
        res = out[r]
        assert res["sum"] == [3.0 * i for i in range(6)]
        assert res["zsum"] == [2 + 4j, 1 - 2j]
        assert res["max"] == [1, 10, 0]
        assert res["spmm_err"] <= 1e-12 and res["gather_err"] <= 1e-12
        assert res["rs"] == [3.0 * (4 * r + i + 1) for i in range(4)]
        assert res["ag"] == [1j, 0j, 0j, 1 + 1j, 2 + 0j, -1j]
        np.testing.assert_allclose(res["host_all"], res["y_full"], rtol=0, atol=1e-12)
        if r == 0:
            np.testing.assert_allclose(res["host_root"], res["y_full"], rtol=0, atol=1e-12)
        else:
            assert res["host_root"] is None


def test_threadcomm_split_collectives():
    """ThreadComm (ranks as threads): reduce-scatter / chunk all-gather / host row assembly
    with sums in rank order (bitwise what its allreduce gives)."""
    import threading

    import torch

    from paper_1407_7506_b200.distributed import thread_comms

    size = 3
    comms = thread_comms(size)
    out = [None] * size

    def work(r):
        c = comms[r]
        a = torch.arange(9, dtype=torch.float64) * (r + 1) + 0.1
        b = a.clone()
        c.allreduce_sum(b)
        c.reduce_scatter_sum(a, 3)
        g = torch.full((6,), -1.0, dtype=torch.float64)
        g[2 * r:2 * r + 2] = r
        c.allgather_chunks(g, 2)
        rows = [(0, 2), (2, 3), (3, 5)]
        loc = np.full((rows[r][1] - rows[r][0], 2), float(r))
        out[r] = (a[3 * r:3 * r + 3].tolist(), b[3 * r:3 * r + 3].tolist(), g.tolist(),
                  c.gather_rows_host(loc, rows, "all"), c.gather_rows_host(loc, rows, "root"))

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    for r in range(size):
        rs, ar, g, hall, hroot = out[r]
        assert rs == ar
        assert g == [0.0, 0.0, 1.0, 1.0, 2.0, 2.0]
        assert hall.tolist() == [[0.0, 0.0]] * 2 + [[1.0, 1.0]] + [[2.0, 2.0]] * 2
        assert (hroot is None) == (r != 0)


def test_config5_fits_eight_b200():
    """Per-rank device bytes of config 5 (complex 128^3 Peierls, k_total 4178, q 64) on 8
    GPUs: 8 state blocks (P, AP updated in place), ghost planes, Grams, pencil buffers,
    workspaces and the largest transients stay under 170 GB of the 183 GB HBM; the vectors
    are assembled on the host (PPCGSolver.finish), never on a device."""
    from paper_1407_7506_b200.ppcg import device_bytes_plan

    n, P, kt = 128 ** 3, 128 * 128, 4096 + 82
    plan = device_bytes_plan(n // 8, n // 8 + 2 * P, kt, 64, True, 14581760 // 8 + 2 * P, 8)
    assert plan["total"] < 170e9, plan
    one_block = (n // 8) * ((kt + 15) // 16 * 16) * 16
    assert plan["state_blocks"] < 8.6 * one_block  # 8 blocks (+ ghost planes), not 10
    # config 4 on one GPU keeps the same accounting
    assert device_bytes_plan(96 ** 3, 96 ** 3, 2048 + 41, 64, False, 23393656, 1)["total"] < 170e9


def test_partition_rows_plane_aligned_for_stencils():
    """Stencil operators are cut at grid-plane boundaries (ppcg.py uses the plane inferred
    from the CSR), so each rank's ghost-extended local CSR is again a whole-plane stencil the
    plane-marching SpMM can run (spmm_plan.StencilPlan), with one ghost plane per side."""
    from paper_1407_7506_b200 import config_problem
    from paper_1407_7506_b200.ppcg import _stencil_plane
    from paper_1407_7506_b200.spmm_plan import StencilPlan
    from test_spmm_plan import replay

    for cfg, N in ((2, 10), (4, 7), (5, 9)):
        csr = config_problem(cfg, N=N)[0]._csr
        n, P = csr.shape[0], _stencil_plane(csr)
        assert P == N * N
        for size in (2, 3, 4):
            bounds = partition_rows(n, size, csr.indptr, plane=P)
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(lo % P == 0 and hi % P == 0 and lo < hi for lo, hi in bounds)
            for r in range(size):
                hp = HaloPlan(csr, bounds, r)
                loc = local_rows_csr(csr, hp.lo, hp.hi, hp.g_lo, hp.n_ext)
                sp_ = StencilPlan(loc.indptr, loc.indices, loc.shape[0], loc.shape[1])
                assert sp_.ok and sp_.grid[1:] == (N, N)
                # (a one-plane slab may be read as shifted by a plane: an equally exact decoding)
                x = np.random.default_rng(r).standard_normal((hp.n_ext, 2))
                if np.iscomplexobj(loc.data):
                    x = x + 1j * np.random.default_rng(r + 9).standard_normal((hp.n_ext, 2))
                np.testing.assert_allclose(replay(loc, sp_, x), loc @ x, rtol=0, atol=1e-12)
    # fewer planes than ranks: ordinary row cuts
    csr = config_problem(2, N=3)[0]._csr
    b = partition_rows(27, 4, csr.indptr, plane=9)
    assert len(b) == 4 and b[-1][1] == 27 and not all(lo % 9 == 0 for lo, _ in b)
    assert _stencil_plane(config_problem(1, N=8)[0]._csr) == 64  # 2-D: one plane
