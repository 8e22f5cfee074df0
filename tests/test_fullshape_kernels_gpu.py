"""Kernel-level parity at the BASELINE configs' full shapes (the solver-level full-size tests are in
test_fullsize_gpu.py): the emulated Gram / tall GEMM at config 3's 262,144 x 1,045 blocks against
extended-precision dot products of sampled entries, and the stencil SpMM kernels on config 4's
96^3 27-point operator (blocks of 1.85e9 elements: byte offsets beyond 2^32) and a 64^3 complex
Peierls operator -- bitwise against the CSR gather on the whole block, against scipy on sampled
columns (SparseHermitian.apply, problems.py:72-73; block_inner, core.py:43-49)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def test_emulated_products_at_config3_shape(cuda):
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, m = 262144, 1045
    ld = (m + 15) // 16 * 16
    g = torch.Generator(device="cuda").manual_seed(3)
    scale = torch.logspace(-2, 2, m, dtype=torch.float64, device="cuda")
    x = (torch.randn((n, ld), generator=g, dtype=torch.float64, device="cuda") * 0.05)[:, :m] * scale
    y = torch.randn((n, ld), generator=g, dtype=torch.float64, device="cuda")[:, :m]
    assert K.fp64_emulation_enabled()
    gm = K.gram(x, y)
    rng = np.random.default_rng(0)
    ii, jj = rng.integers(0, m, 24), rng.integers(0, m, 24)
    xs = x[:, torch.as_tensor(ii, device="cuda")].cpu().numpy().astype(np.longdouble)
    ys = y[:, torch.as_tensor(jj, device="cuda")].cpu().numpy().astype(np.longdouble)
    got = gm.cpu().numpy()
    for a in range(24):
        ref = np.sum(xs[:, a] * ys[:, a])
        bound = 4 * U * float(np.sum(np.abs(xs[:, a] * ys[:, a])))
        assert abs(float(got[ii[a], jj[a]] - ref)) <= bound, (a, got[ii[a], jj[a]], ref, bound)
    # tall GEMM W = s (.) (Z - X G) with the fused metric (ksplit = m - 21): sampled rows
    gmat = torch.randn((m, m), generator=g, dtype=torch.float64, device="cuda") / 40
    s = torch.rand(n, generator=g, dtype=torch.float64, device="cuda") + 0.5
    w = torch.empty((n, ld), dtype=torch.float64, device="cuda")[:, :m]
    K.tsgemm([x], [gmat], [w], alpha=-1.0, beta=1.0, zs=[y], rowscale=s)
    rows = torch.as_tensor(rng.integers(0, n, 40), device="cuda")
    xr = x[rows].cpu().numpy().astype(np.longdouble)
    gh = gmat.cpu().numpy().astype(np.longdouble)
    zr, sr = y[rows].cpu().numpy(), s[rows].cpu().numpy()[:, None]
    prod = xr @ gh
    ref = (sr * (zr - prod)).astype(np.float64)
    bound = sr * (4 * U * (np.abs(xr.astype(np.float64)) @ np.abs(gh.astype(np.float64)))
                  + 2 * U * np.abs(zr - prod.astype(np.float64)))
    assert np.all(np.abs(w[rows].cpu().numpy() - ref) <= bound + 1e-300)


def _variants(torch, dc, x, y_out):
    """y by the stencil-slot kernel, the offset-ELL march and the CSR gather (device tensors)."""
    from paper_1407_7506_b200 import _lib
    from paper_1407_7506_b200.operators import DeviceCsr

    lib = _lib.load()
    outs = {}
    try:
        for name, variant, stencil, slot in (("slot", 2, True, True), ("march", 2, True, False),
                                             ("gather", 0, False, False)):
            lib.bk_spmm_set_variant(variant)
            DeviceCsr.use_stencil = stencil
            dc.stencil.use_slot = slot
            y = y_out[name]
            y.fill_(float("nan"))
            dc.apply_into(x, y)
            torch.cuda.synchronize()
            outs[name] = y
    finally:
        lib.bk_spmm_set_variant(2)
        DeviceCsr.use_stencil = True
        dc.stencil.use_slot = True
    return outs


@pytest.mark.parametrize("cfg,kw,m,st", [(4, {}, 2089, 27), (5, {"N": 64}, 523, 7)])
def test_stencil_spmm_at_full_grid(cuda, cfg, kw, m, st):
    from paper_1407_7506_b200.operators import DeviceCsr
    from paper_1407_7506_b200.problems import config_problem

    torch = cuda
    a, _, _, _ = config_problem(cfg, **kw)
    csr = a._csr
    prev = DeviceCsr.stencil_kinds
    DeviceCsr.stencil_kinds = ("slot", "march")
    try:
        dc = DeviceCsr(csr)
    finally:
        DeviceCsr.stencil_kinds = prev
    assert dc.stencil is not None and dc.stencil.st == st
    cplx = np.iscomplexobj(csr.data)
    dt = torch.complex128 if cplx else torch.float64
    n = csr.shape[0]
    ld = (m + 15) // 16 * 16
    g = torch.Generator(device="cuda").manual_seed(cfg)
    xb = torch.randn((n, ld), generator=g, dtype=torch.float64, device="cuda").to(dt)
    if cplx:
        xb = xb + 1j * torch.randn((n, ld), generator=g, dtype=torch.float64, device="cuda")
    off = 11  # a locked-column offset: views start off the 128-byte line
    x = xb[:, off:off + m - off]
    bufs = {k: torch.full((n, ld), float("nan"), dtype=dt, device="cuda") for k in ("slot", "march", "gather")}
    outs = _variants(torch, dc, x, {k: v[:, off:off + m - off] for k, v in bufs.items()})
    assert torch.equal(outs["slot"], outs["gather"])
    assert torch.equal(outs["march"], outs["gather"])
    for b in bufs.values():  # nothing written outside the view
        assert bool(torch.isnan(b[:, :off].real).all()) and bool(torch.isnan(b[:, m:].real).all())
    cols = torch.as_tensor([0, 1, (m - off) // 2, m - off - 2, m - off - 1], device="cuda")
    xh = x[:, cols].cpu().numpy()
    ref = csr @ xh
    got = outs["slot"][:, cols].cpu().numpy()
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(np.max(np.abs(ref)), 1.0)
