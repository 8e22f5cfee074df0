"""SpMM kernels (SparseHermitian.apply, problems.py:72-73 / scipy csr_matvecs): the plane-
marching stencil kernel, the whole-row vector gather and the row gather must agree with each
other bit for bit (all three run every row's FMAs in CSR order) and with scipy to fp64
rounding, on the BASELINE operator structures (2-D 5-pt, 3-D 7-pt, 27-pt, complex Peierls),
non-stencil CSRs, column views at odd / even offsets (locked columns), and the ghost-
extended local CSR of a row partition."""

import numpy as np
import pytest

from paper_1407_7506_b200.distributed import local_rows_csr
from paper_1407_7506_b200.problems import config_problem, laplacian_1d, random_hermitian
from util import gauss

pytestmark = pytest.mark.gpu


def run_variants(torch, dc, xb, off, m, cplx):
    """Y = A X[:, off:off+m] by march (when planned), vector gather, row gather."""
    from paper_1407_7506_b200 import _lib
    from paper_1407_7506_b200.operators import DeviceCsr

    lib = _lib.load()
    dt = torch.complex128 if cplx else torch.float64
    x = xb[:, off:off + m]
    outs = {}
    # stencil-slot configurations: variant + 100 x (forced x segment count); 4..7 hold X planes in
    # registers (27-point; the 7-point kernel ignores the variant)
    variants = (("slot", 2, True, True, 0), ("slot_v1", 2, True, True, 1), ("slot_v4", 2, True, True, 4),
                ("slot_v5", 2, True, True, 5), ("slot_v6", 2, True, True, 6), ("slot_v7", 2, True, True, 7),
                ("slot_v4x2", 2, True, True, 204), ("slot_v5x3", 2, True, True, 305), ("slot_v7x2", 2, True, True, 207),
                ("march", 2, True, False, 0), ("vec", 2, False, False, 0), ("gather", 0, False, False, 0))
    try:
        for name, variant, stencil, slot, cfg in variants:
            if stencil and dc.stencil is None:
                continue
            if slot and getattr(dc.stencil, "sval", None) is None:
                continue
            lib.bk_spmm_set_variant(variant)
            lib.bk_spmm_stencil_set_config(cfg)
            DeviceCsr.use_stencil = stencil
            if dc.stencil is not None:
                dc.stencil.use_slot = slot
            yb = torch.full((dc.n, xb.shape[1]), float("nan"), dtype=dt, device="cuda")
            y = yb[:, off:off + m]
            dc.apply_into(x, y)
            torch.cuda.synchronize()
            outs[name] = yb.cpu().numpy()
    finally:
        lib.bk_spmm_set_variant(2)
        lib.bk_spmm_stencil_set_config(0)
        DeviceCsr.use_stencil = True
        if dc.stencil is not None:
            dc.stencil.use_slot = True
    return outs


def check(torch, csr, xh, ncols=None, expect_march=True, expect_st=None):
    from paper_1407_7506_b200.operators import DeviceCsr

    cplx = np.iscomplexobj(csr.data) or np.iscomplexobj(xh)
    prev = DeviceCsr.min_stencil_rows, DeviceCsr.stencil_kinds
    DeviceCsr.min_stencil_rows = 0  # the test problems are small; production plans from 32768 rows
    DeviceCsr.stencil_kinds = ("slot", "march")  # both plan layouts: every kernel is compared
    try:
        dc = DeviceCsr(csr)
    finally:
        DeviceCsr.min_stencil_rows, DeviceCsr.stencil_kinds = prev
    assert (dc.stencil is not None) == expect_march
    if expect_st is not None:
        assert dc.stencil.st == expect_st
    xb = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    kt = xh.shape[1]
    for off in (0, 1, 10, 11):
        m = kt - off - (3 if off == 11 else 0)
        outs = run_variants(torch, dc, xb, off, m, cplx)
        ref = csr @ xh[:, off:off + m]
        base = outs["gather"]
        for name, yb in outs.items():
            # columns outside the view untouched, the view bitwise equal across kernels
            assert np.all(np.isnan(yb[:, :off])) and np.all(np.isnan(yb[:, off + m:])), name
            np.testing.assert_array_equal(yb[:, off:off + m], base[:, off:off + m], err_msg=name)
            err = np.max(np.abs(yb[:, off:off + m] - ref))
            assert err <= 1e-13 * max(np.max(np.abs(ref)), 1.0), (name, err)


@pytest.mark.parametrize("cfg,kw,kt", [(1, {"N": 24}, 70), (2, {"N": 20}, 131), (2, {"N": 17}, 64),
                                       (3, {"N": 12}, 200), (4, {"N": 10}, 90), (5, {"N": 10}, 48),
                                       (4, {"N": 13}, 37), (5, {"N": 11}, 70)])
def test_spmm_kernels_agree(cuda, cfg, kw, kt):
    a, _, _, _ = config_problem(cfg, **kw)
    csr = a._csr
    kt = kt + kt % 2  # solver blocks have an even leading dimension
    check(cuda, csr, gauss(csr.shape[0], kt, cfg, cplx=cfg == 5), expect_st=27 if cfg == 4 else 7)


def test_spmm_non_stencil_and_1d(cuda):
    check(cuda, random_hermitian(300, 0.05, seed=3)._csr, gauss(300, 40, 1), expect_march=False)
    check(cuda, random_hermitian(200, 0.05, seed=4, complex_field=True)._csr, gauss(200, 24, 2, True),
          expect_march=False)
    check(cuda, laplacian_1d(500)._csr, gauss(500, 36, 3))


def test_spmm_ghost_extended_local(cuda):
    """Rows [lo, hi) of a 7-pt and a 27-pt operator with one ghost plane per side, applied to
    the extended block (the row partition's SpMM): march with d0 = P and planes -1 .. nx."""
    for cfg, N in ((3, 12), (4, 10)):
        a, _, _, _ = config_problem(cfg, N=N)
        csr = a._csr
        P = N * N
        x = gauss(csr.shape[0], 66, 9)
        for lo, hi in ((3 * P, 7 * P), (0, 4 * P), (6 * P, N * P)):
            g_lo, g_hi = max(lo - P, 0), min(hi + P, csr.shape[0])
            loc = local_rows_csr(csr, lo, hi, g_lo, g_hi - g_lo)
            check(cuda, loc, x[g_lo:g_hi])
