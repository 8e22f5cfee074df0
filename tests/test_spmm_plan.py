"""Host side of the plane-marching SpMM (spmm_plan.py): grid inference from a CSR alone and
the ring-offset encoding, checked by replaying the kernel's addressing in numpy against
scipy's ``csr @ X`` (the reference's SparseHermitian.apply, problems.py:72-73)."""

import numpy as np
import pytest

from paper_1407_7506_b200.distributed import local_rows_csr
from paper_1407_7506_b200.problems import config_problem, laplacian_1d, random_hermitian
from paper_1407_7506_b200.spmm_plan import TY, StencilPlan
from util import gauss


def replay(csr, plan, x):
    """Y = A X through the plan: each ELL entry's offset decoded to (dx, dy, dz) exactly as
    the kernel maps it to a ring slot / halo row, values in ELL order."""
    nx, ny, nz = plan.grid
    vals = plan.ell_values(csr.data).numpy()
    offs = plan.ell_off.numpy().view(np.uint16)
    y = np.zeros((csr.shape[0], x.shape[1]), dtype=np.result_type(vals, x))
    for r in range(csr.shape[0]):
        ix, iy, iz = r // (ny * nz), (r // nz) % ny, r % nz
        for t in range(plan.width):
            o = int(offs[r, t])
            if o == 0xFFFF:
                break
            dx = (o >> 14) - 1
            h = o & 0x3FFF
            dy, dz = h // (TY + 2) - 1, h % (TY + 2) - 1
            src = plan.d0 + ((ix + dx) * ny + iy + dy) * nz + iz + dz
            y[r] += vals[r, t] * x[src]
    return y


@pytest.mark.parametrize("cfg,kw,grid", [(1, {"N": 12}, (1, 12, 12)), (2, {"N": 6}, (6, 6, 6)),
                                         (3, {"N": 5}, (5, 5, 5)), (4, {"N": 5}, (5, 5, 5)),
                                         (5, {"N": 5}, (5, 5, 5))])
def test_plan_replays_csr(cfg, kw, grid):
    a, _, _, _ = config_problem(cfg, **kw)
    csr = a._csr
    p = StencilPlan(csr.indptr, csr.indices, csr.shape[0])
    assert p.ok and p.grid == grid and p.d0 == 0 and (p.xlo, p.xhi) == (0, grid[0])
    assert p.width == (5 if cfg == 1 else 27 if cfg == 4 else 7) and p.woff % 8 == 0
    x = gauss(csr.shape[0], 3, 5, cplx=cfg == 5)
    np.testing.assert_allclose(replay(csr, p, x), csr @ x, rtol=0, atol=1e-12)


def test_plan_ghost_extended_local_rows():
    """The row partition's local CSR (columns of the ghost-extended block): d0 = the ghost
    shift, planes -1 .. nx_local referenced."""
    a, _, _, _ = config_problem(4, N=6)
    csr = a._csr
    P = 36
    x = gauss(csr.shape[0], 2, 7)
    full = csr @ x
    for lo, hi in ((2 * P, 4 * P), (0, 2 * P), (4 * P, 6 * P)):
        g_lo, g_hi = max(lo - P, 0), min(hi + P, csr.shape[0])
        loc = local_rows_csr(csr, lo, hi, g_lo, g_hi - g_lo)
        p = StencilPlan(loc.indptr, loc.indices, loc.shape[0], loc.shape[1])
        assert p.ok and p.grid == (2, 6, 6) and p.d0 == lo - g_lo
        assert p.xlo == (-1 if lo > 0 else 0) and p.xhi == (3 if hi < csr.shape[0] else 2)
        np.testing.assert_allclose(replay(loc, p, x[g_lo:g_hi]), full[lo:hi], rtol=0, atol=1e-12)


def test_plan_rejects_non_stencils():
    assert not StencilPlan(*(lambda c: (c.indptr, c.indices, c.shape[0]))(random_hermitian(90, 0.25, seed=1)._csr)).ok
    # periodic wrap-around (offset nz - 1 inside a z-line) needs a wider halo: rejected (the
    # offsets do fit a shifted 2 x 2 grid, but not with whole planes of X rows)
    import scipy.sparse as sp

    n = 4 * 4 * 4
    a = sp.lil_matrix((n, n))
    for r in range(n):
        a[r, r] = 2.0
        a[r, (r // 4) * 4 + (r + 1) % 4] = -1.0
    a = ((a + a.T) / 2).tocsr()
    assert not StencilPlan(a.indptr, a.indices, n).ok
    # 1-D Laplacian: a 1 x 1 x n grid
    c = laplacian_1d(50)._csr
    p = StencilPlan(c.indptr, c.indices, 50)
    assert p.ok and p.grid == (1, 1, 50)


_CROSS_POS = ((-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0))


def replay_slots(csr, plan, x):
    """Y = A X through the stencil-slot layout exactly as bk_spmm_stencil_* reads it: slot s of
    a row is stencil position s (cross order for st = 7, (dx, dy, dz) lexicographic for 27),
    skipped unless its presence bit is set."""
    nx, ny, nz = plan.grid
    sv = plan.slot_values(csr.data).numpy()
    cplx = np.iscomplexobj(csr.data)
    vals = sv[:, :2 * plan.st].view(np.complex128) if cplx else sv[:, :plan.st]
    masks = sv[:, plan.vd - 1].view(np.int64)
    pos = _CROSS_POS if plan.st == 7 else [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    y = np.zeros((csr.shape[0], x.shape[1]), dtype=np.result_type(vals, x))
    for r in range(csr.shape[0]):
        ix, iy, iz = r // (ny * nz), (r // nz) % ny, r % nz
        for s, (dx, dy, dz) in enumerate(pos):
            if (int(masks[r]) >> s) & 1:
                y[r] += vals[r, s] * x[plan.d0 + ((ix + dx) * ny + iy + dy) * nz + iz + dz]
    return y


@pytest.mark.parametrize("cfg,kw,st", [(1, {"N": 12}, 7), (2, {"N": 6}, 7), (3, {"N": 5}, 7), (4, {"N": 5}, 27),
                                       (5, {"N": 5}, 7)])
def test_slot_layout_replays_csr(cfg, kw, st):
    a, _, _, _ = config_problem(cfg, **kw)
    csr = a._csr
    p = StencilPlan(csr.indptr, csr.indices, csr.shape[0])
    assert p.ok and p.st == st
    sv = p.slot_values(csr.data)
    assert sv.shape == (csr.shape[0], p.vd) and p.vd % 2 == 0
    # every stored entry has its presence bit, and nothing else
    bits = sv[:, p.vd - 1].numpy().view(np.int64)
    assert [bin(int(b)).count("1") for b in bits] == list(np.diff(csr.indptr))
    x = gauss(csr.shape[0], 3, 5, cplx=cfg == 5)
    np.testing.assert_allclose(replay_slots(csr, p, x), csr @ x, rtol=0, atol=1e-12)
    # ghost-extended local rows keep the layout (d0 shift)
    if cfg in (3, 4):
        P = kw["N"] ** 2
        lo, hi = 2 * P, 4 * P
        loc = local_rows_csr(csr, lo, hi, lo - P, 4 * P)
        pl = StencilPlan(loc.indptr, loc.indices, loc.shape[0], loc.shape[1])
        assert pl.ok and pl.st == st
        np.testing.assert_allclose(replay_slots(loc, pl, x[lo - P:hi + P]), (csr @ x)[lo:hi], rtol=0, atol=1e-12)


def test_slot_layout_needs_sorted_rows():
    """Unsorted column indices within a row (legal CSR) keep the offset-ELL march: the slot
    kernel's FMA order is the stencil order, which equals CSR order only for sorted rows."""
    a, _, _, _ = config_problem(3, N=5)
    c = a._csr.copy()
    r = 40
    lo, hi = c.indptr[r], c.indptr[r + 1]
    c.indices[lo:hi] = c.indices[lo:hi][::-1].copy()
    c.data[lo:hi] = c.data[lo:hi][::-1].copy()
    p = StencilPlan(c.indptr, c.indices, c.shape[0])
    assert p.ok and p.st == 0
