"""FP64 products emulated on the int8 tensor cores (csrc/ozaki.cu, Ozaki scheme with 8 signed
8-bit digits) against exact references.

The bar is DGEMM's error bound class: every sampled entry within 4 * 2^-53 * (|X|^T |Y|) of the
product computed in extended precision (np.longdouble).  Also: non-finite inputs propagate as NaN (the solver's
breakdown guards rely on it, ppcg.py:698-724), zero columns / rows, wide dynamic range,
super-chunked slicing, the fused stopping-metric snapshot, bitwise determinism."""

import numpy as np
import pytest

from util import gauss

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def dev(x, torch):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def exact_gram(x, y, cols1=None, cols2=None):
    """X^T Y in extended precision (np.longdouble: 64-bit significand, i.e. 11 bits beyond fp64),
    optionally only on sampled columns; returns (reference, |X|^T |Y|)."""
    if cols1 is not None:
        x, y = x[:, cols1], y[:, cols2]
    xl = x.astype(np.longdouble)
    yl = y.astype(np.longdouble)
    return (xl.T @ yl).astype(np.float64), (np.abs(x).T @ np.abs(y))


def sample(m, k, seed):
    return np.sort(np.random.default_rng(seed).choice(m, size=min(m, k), replace=False))


def emu(torch, on=True):
    from paper_1407_7506_b200 import kernels as K

    return K.fp64_emulation(on)


@pytest.mark.parametrize("n,m1,m2", [(20000, 64, 64), (40000, 200, 130), (110592, 523, 523), (70001, 97, 333)])
def test_ozaki_gram_within_dgemm_bound(cuda, n, m1, m2):
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    rng = np.random.default_rng(n + m1)
    x = gauss(n, m1, 1) * np.exp(rng.uniform(-6, 6, m1))[None, :]
    y = gauss(n, m2, 2) * np.exp(rng.uniform(-6, 6, m2))[None, :]
    x[:, 3] = 0.0  # an all-zero column
    with emu(torch):
        c = K.gram(dev(x, torch), dev(y, torch)).cpu().numpy()
    c1, c2 = sample(m1, 24, 1), sample(m2, 24, 2)
    c1[0] = 3
    ref, absprod = exact_gram(x, y, c1, c2)
    err = np.abs(c[np.ix_(c1, c2)] - ref)
    assert np.all(err <= 4 * U * absprod + 1e-300), (err / (absprod + 1e-300)).max()
    assert np.all(c[3] == 0.0)


def test_ozaki_gram_symmetric_and_views(cuda):
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, m = 50000, 300
    big = dev(gauss(n, m + 20, 3), torch)
    v = big[:, 11 : 11 + m]
    x = v.cpu().numpy()
    cs = sample(m, 40, 3)
    ref, absprod = exact_gram(x, x, cs, cs)
    with emu(torch):
        g = K.gram(v, v, symmetric=True).cpu().numpy()
        g2 = K.gram(v, v, symmetric=True).cpu().numpy()
        gn = K.gram(v, v).cpu().numpy()
    assert np.array_equal(g, g.T)
    assert np.array_equal(g, g2)  # deterministic
    assert np.all(np.abs(g[np.ix_(cs, cs)] - ref) <= 4 * U * absprod)
    assert np.all(np.abs(gn[np.ix_(cs, cs)] - ref) <= 4 * U * absprod)


def test_ozaki_gram_complex(cuda):
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, m1, m2 = 30000, 70, 90
    x = gauss(n, m1, 4) + 1j * gauss(n, m1, 5)
    y = gauss(n, m2, 6) + 1j * gauss(n, m2, 7)
    with emu(torch):
        c = K.gram(dev(x, torch), dev(y, torch)).cpu().numpy()
    c1, c2 = sample(m1, 20, 6), sample(m2, 20, 7)
    xs, ys = x[:, c1], y[:, c2]
    ref = (xs.conj().T.astype(np.clongdouble) @ ys.astype(np.clongdouble)).astype(np.complex128)
    bound = 8 * U * (np.abs(xs).T @ np.abs(ys))
    assert np.all(np.abs(c[np.ix_(c1, c2)] - ref) <= bound)


def test_ozaki_gram_nonfinite_propagates(cuda):
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, m = 20000, 80
    x = gauss(n, m, 8)
    y = gauss(n, m, 9)
    x[123, 5] = np.nan
    y[77, 9] = np.inf
    with emu(torch):
        c = K.gram(dev(x, torch), dev(y, torch)).cpu().numpy()
    assert np.all(np.isnan(c[5, :]))
    assert np.all(np.isnan(c[:, 9]))
    ok = np.ones_like(c, dtype=bool)
    ok[5, :] = False
    ok[:, 9] = False
    assert np.all(np.isfinite(c[ok]))


def test_ozaki_gram_superchunks_match(cuda):
    """A workspace that holds a third of the digits: rows are sliced in super-chunks and the
    partial Grams accumulate in order; same bound (and same chunk partials) as one pass."""
    from paper_1407_7506_b200 import _lib
    from paper_1407_7506_b200.kernels import stream_ptr

    torch = cuda
    lib = _lib.load()
    n, m = 100000, 128
    x = dev(gauss(n, m, 10), torch)
    y = dev(gauss(n, m, 11), torch)
    full = lib.bk_ozaki_gram_ws_bytes(n, m, m, 0, 0)
    outs = []
    for frac in (1.0, 0.34):
        nb = int(full * frac)
        ws = torch.zeros(max(nb, full), dtype=torch.uint8, device="cuda")
        c = torch.empty((m, m), dtype=torch.float64, device="cuda")
        _lib.call("bk_ozaki_gram_d", n, m, m, x.data_ptr(), m, y.data_ptr(), m, c.data_ptr(), m, 0, ws.data_ptr(),
                  nb if frac < 1 else full, stream_ptr())
        outs.append(c.cpu().numpy())
    xn, yn = x.cpu().numpy(), y.cpu().numpy()
    cs = sample(m, 32, 4)
    ref, absprod = exact_gram(xn, yn, cs, cs)
    for c in outs:
        assert np.all(np.abs(c[np.ix_(cs, cs)] - ref) <= 4 * U * absprod)


@pytest.mark.parametrize("n,K_,N,nprob", [(40000, 523, 523, 2), (16384, 64, 200, 1), (30001, 300, 77, 4)])
def test_ozaki_tsgemm(cuda, n, K_, N, nprob):
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    rng = np.random.default_rng(K_)
    xs = [gauss(n, K_, 20 + b) * np.exp(rng.uniform(-5, 5, n))[:, None] for b in range(nprob)]
    gs = [gauss(K_, N, 30 + b) * np.exp(rng.uniform(-5, 5, N))[None, :] for b in range(nprob)]
    zs = [gauss(n, N, 40 + b) for b in range(nprob)]
    s = np.abs(gauss(n, 1, 50))[:, 0] + 0.5
    ys = [torch.empty((n, N), dtype=torch.float64, device="cuda") for _ in range(nprob)]
    with emu(torch):
        K.tsgemm([dev(x, torch) for x in xs], [dev(g, torch) for g in gs], ys, alpha=-1.0, beta=1.0,
                 zs=[dev(z, torch) for z in zs], rowscale=dev(s, torch))
    rows = sample(n, 300, 5)
    for b in range(nprob):
        xr, zr, sr = xs[b][rows], zs[b][rows], s[rows, None]
        prod = xr.astype(np.longdouble) @ gs[b].astype(np.longdouble)
        ref = (sr * (zr - prod)).astype(np.float64)
        bound = sr * (4 * U * (np.abs(xr) @ np.abs(gs[b])) + 2 * U * np.abs(zr - prod.astype(np.float64)))
        assert np.all(np.abs(ys[b].cpu().numpy()[rows] - ref) <= bound + 1e-300), b


def test_ozaki_tsgemm_metric_snapshot_and_inplace(cuda):
    """The fused stopping metric: sum over cols < nsplit of (alpha X[:, :ksplit] G[:ksplit] + beta Z)^2,
    with Z aliasing Y (in-place update) and a metric-only launch (Y = None)."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, Kt, N, ks, ns = 50000, 523, 523, 513, 500
    x, g, ax = gauss(n, Kt, 60), gauss(Kt, N, 61) * 0.1, gauss(n, N, 62)
    ref_metric = np.sum((ax[:, :ns] - x[:, :ks] @ g[:ks, :ns]) ** 2)
    ref_w = ax - x @ g
    with emu(torch):
        w = dev(ax, torch)
        metric = torch.zeros(1, dtype=torch.float64, device="cuda")
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [w], alpha=-1.0, beta=1.0, zs=[w], metric=metric, ksplit=ks,
                 nsplit=ns)
        m2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [None], alpha=-1.0, beta=1.0, zs=[dev(ax, torch)], metric=m2,
                 ksplit=ks, nsplit=ns)
        m3 = torch.zeros(1, dtype=torch.float64, device="cuda")
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [None], alpha=-1.0, beta=1.0, zs=[dev(ax, torch)], metric=m3,
                 ksplit=Kt, nsplit=N)
    assert abs(metric.item() - ref_metric) <= 1e-12 * ref_metric
    assert metric.item() == m2.item()
    assert abs(m3.item() - np.sum(ref_w ** 2)) <= 1e-12 * np.sum(ref_w ** 2)
    assert np.max(np.abs(w.cpu().numpy() - ref_w)) <= 1e-13 * np.abs(ref_w).max() * 10


@pytest.mark.parametrize("ks,ns", [(300, 499), (491, 523), (522, 1), (513, 33)])
def test_ozaki_tsgemm_metric_modes(cuda, ks, ns):
    """The three forms of the fused metric give the same number: a long K tail takes the partial-K
    snapshot (MMA warp paused), a short one (K - ksplit <= 32) the full-K accumulator minus the
    tail's fp64 product, ksplit = K the final accumulator; odd nsplit, row scale, edge tiles."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, Kt, N = 40000, 523, 523
    x, g, ax = gauss(n, Kt, 160), gauss(Kt, N, 161) * 0.1, gauss(n, N, 162)
    s = np.abs(gauss(n, 1, 163))[:, 0] + 0.5
    ref_metric = np.sum((ax[:, :ns] - x[:, :ks] @ g[:ks, :ns]) ** 2)
    ref_w = s[:, None] * (ax - x @ g)
    with emu(torch):
        w = torch.empty((n, N), dtype=torch.float64, device="cuda")
        metric = torch.zeros(1, dtype=torch.float64, device="cuda")
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [w], alpha=-1.0, beta=1.0, zs=[dev(ax, torch)],
                 rowscale=dev(s, torch), metric=metric, ksplit=ks, nsplit=ns)
        w0 = torch.empty_like(w)
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [w0], alpha=-1.0, beta=1.0, zs=[dev(ax, torch)],
                 rowscale=dev(s, torch))
    assert abs(metric.item() - ref_metric) <= 1e-12 * ref_metric
    assert np.max(np.abs(w.cpu().numpy() - ref_w)) <= 1e-12 * np.abs(ref_w).max()
    if Kt - ks <= 32:  # no k split: the same digits as the plain product
        assert torch.equal(w, w0)


def test_ozaki_coldigits_reused_across_grams(cuda):
    """Column digits sliced once (kernels.coldigits) and handed to several Grams -- full block,
    column ranges at odd offsets (locked columns), gram2, symmetric, complex views -- give
    bitwise the results of the Grams that slice X themselves; an operand that is not a column
    range of the sliced block is sliced as usual."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, m = 40000, 212
    xb = dev(gauss(n, m + 12, 170) * np.logspace(-3, 3, m + 12)[None, :], torch)
    x = xb[:, 5:5 + m]
    w, p = dev(gauss(n, 150, 171), torch), dev(gauss(n, 97, 172), torch)
    with emu(torch):
        d = K.coldigits(x)
        assert d is not None and d.m == m
        for a, b in ((0, m), (11, m), (3, 140)):
            xs = x[:, a:b]
            assert torch.equal(K.gram(xs, w, xdig=d), K.gram(xs, w))
            assert torch.equal(K.gram(xs, xs, symmetric=True, xdig=d), K.gram(xs, xs, symmetric=True))
            g1, g2 = (torch.empty((b - a, 150), dtype=torch.float64, device="cuda"),
                      torch.empty((b - a, 97), dtype=torch.float64, device="cuda"))
            h1, h2 = torch.empty_like(g1), torch.empty_like(g2)
            K.gram2(xs, w, g1, xs, p, g2, xdig=d)
            K.gram2(xs, w, h1, xs, p, h2)
            assert torch.equal(g1, h1) and torch.equal(g2, h2)
        assert torch.equal(K.gram(w, p, xdig=d), K.gram(w, p))  # not a range of the sliced block
        z = dev(gauss(n, 90, 173, cplx=True), torch)
        zw = dev(gauss(n, 70, 174, cplx=True), torch)
        dz = K.coldigits(z)
        assert torch.equal(K.gram(z[:, 7:], zw, xdig=dz), K.gram(z[:, 7:], zw))
        # a buffer that is too small is replaced, a large one reused
        d2 = K.coldigits(x, d.buf)
        assert d2.buf is d.buf
        assert K.coldigits(x[:, :40]) is None  # below the emulation threshold: DMMA Grams


def test_ozaki_tsgemm_nonfinite_row(cuda):
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, Kt, N = 20000, 100, 100
    x, g = gauss(n, Kt, 70), gauss(Kt, N, 71)
    x[9, 4] = np.nan
    g[3, 7] = np.inf
    y = torch.empty((n, N), dtype=torch.float64, device="cuda")
    with emu(torch):
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [y])
    yn = y.cpu().numpy()
    assert np.all(np.isnan(yn[9]))
    assert np.all(np.isnan(yn[:, 7]))
    ok = np.ones_like(yn, dtype=bool)
    ok[9] = False
    ok[:, 7] = False
    assert np.all(np.isfinite(yn[ok]))


def test_ozaki_gram2_shares_x_and_batched_tsgemm_shares_digits(cuda):
    """gram2 with one basis (X sliced once) agrees with two single Grams to the DGEMM-class bound
    (its split-K chunking follows both products' tile counts, so the chunk sums round
    differently); a batched tall GEMM whose problems repeat X / G (the projection update
    [X, X, AX] x [G1, G3, G3]) equals the unbatched products bitwise."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, m = 30000, 150
    x, w, p = (dev(gauss(n, m, 80 + i), torch) for i in range(3))
    with emu(torch):
        a1 = torch.empty((m, m), dtype=torch.float64, device="cuda")
        a2 = torch.empty_like(a1)
        K.gram2(x, w, a1, x, p, a2)
        b1, b2 = K.gram(x, w), K.gram(x, p)
        xa = x.abs()
        for a, b, y in [(a1, b1, w), (a2, b2, p)]:
            bound = 8 * U * (xa.T @ y.abs())
            assert bool(((a - b).abs() <= bound).all())
        ax = dev(gauss(n, m, 90), torch)
        g1, g3 = dev(gauss(m, m, 91), torch), dev(gauss(m, m, 92), torch)
        ys = [torch.zeros((n, m), dtype=torch.float64, device="cuda") for _ in range(3)]
        K.tsgemm([x, x, ax], [g1, g3, g3], ys, alpha=-1.0, beta=0.0)
        for y, (xx, gg) in zip(ys, [(x, g1), (x, g3), (ax, g3)]):
            r = torch.zeros_like(y)
            K.tsgemm([xx], [gg], [r], alpha=-1.0, beta=0.0)
            assert torch.equal(y, r)


def test_ozaki_tsgemm_last_stage_snapshots_back_to_back(cuda):
    """Metric launches whose snapshot is the last k stage (ksplit = K) on many consecutive
    tiles: the MMA warp must not run a second snapshot phase ahead of the epilogue (a hang, not
    a wrong number, if it does)."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, Kt, N = 60000, 96, 300
    x, g, z = gauss(n, Kt, 100), gauss(Kt, N, 101), gauss(n, N, 102)
    with emu(torch):
        m = torch.zeros(1, dtype=torch.float64, device="cuda")
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [None], alpha=-1.0, beta=1.0, zs=[dev(z, torch)], metric=m,
                 ksplit=Kt, nsplit=N)
        torch.cuda.synchronize()
    ref = np.sum((z - x @ g) ** 2)
    assert abs(m.item() - ref) <= 1e-12 * ref


def test_ozaki_tsgemm_superchunks_bitwise(cuda):
    """A workspace that holds the row digits of a fraction of the rows: the tall GEMM runs in
    row super-chunks (the 4-problem projection update at config 2 does); rows are independent,
    so Y is bitwise the one-pass result and the metric agrees to rounding of its partial sums."""
    from paper_1407_7506_b200 import _lib
    from paper_1407_7506_b200.kernels import stream_ptr

    torch = cuda
    lib = _lib.load()
    n, Kt, N, ks = 70000, 200, 150, 190
    x, g, z = dev(gauss(n, Kt, 110), torch), dev(gauss(Kt, N, 111), torch), dev(gauss(n, N, 112), torch)
    s = dev(np.abs(gauss(n, 1, 113))[:, 0] + 0.5, torch)
    full = lib.bk_ozaki_tsgemm_ws_bytes(1, n, Kt, N, ks)
    outs = []
    for frac in (1.0, 0.3):
        nb = int(full * frac)
        ws = torch.empty(full, dtype=torch.uint8, device="cuda")
        y = torch.empty((n, N), dtype=torch.float64, device="cuda")
        m = torch.zeros(1, dtype=torch.float64, device="cuda")
        XP, _a = _lib.ptr_array([x.data_ptr()])
        GP, _b = _lib.ptr_array([g.data_ptr()])
        ZP, _c = _lib.ptr_array([z.data_ptr()])
        YP, _d = _lib.ptr_array([y.data_ptr()])
        _lib.call("bk_ozaki_tsgemm_d", 1, n, Kt, N, -1.0, XP, Kt, GP, N, 1.0, ZP, N, YP, N, s.data_ptr(), 0, ks, N,
                  m.data_ptr(), ws.data_ptr(), nb, stream_ptr())
        outs.append((y.cpu().numpy(), m.item()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert abs(outs[0][1] - outs[1][1]) <= 1e-14 * abs(outs[0][1])
    xn, gn, zn = x.cpu().numpy(), g.cpu().numpy(), z.cpu().numpy()
    ref = np.sum((zn - xn[:, :ks] @ gn[:ks]) ** 2)
    assert abs(outs[0][1] - ref) <= 1e-12 * ref


def test_ozaki_extreme_scales(cuda):
    """Columns / rows scaled to 1e-300 and 1e+150 (products down to the subnormal range and up
    to 1e300): the power-of-two factors leave the fast path and go through exact ldexp; the
    results stay within the DGEMM-class bound of the longdouble reference, and pure
    subnormal inputs are represented (not flushed)."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n, m = 20000, 96
    x, y = gauss(n, m, 120), gauss(n, m, 121)
    x[:, :8] *= 1e-300
    y[:, 8:16] *= 1e150
    x[:, 16:24] *= 1e150
    x[:, 24] = 5e-324 * np.sign(x[:, 24])  # subnormal column
    with emu(torch):
        c = K.gram(dev(x, torch), dev(y, torch)).cpu().numpy()
        g = gauss(m, m, 122)
        g[:, :4] *= 1e-200
        w = torch.empty((n, m), dtype=torch.float64, device="cuda")
        K.tsgemm([dev(x, torch)], [dev(g, torch)], [w])
    cs = np.arange(0, 40)
    ref, absprod = exact_gram(x, y, cs, cs)
    assert np.all(np.abs(c[np.ix_(cs, cs)] - ref) <= 4 * U * absprod + 1e-320)
    assert np.count_nonzero(c[24]) > 0
    rows = sample(n, 200, 123)
    prod = (x[rows].astype(np.longdouble) @ g.astype(np.longdouble)).astype(np.float64)
    bound = 4 * U * (np.abs(x[rows]) @ np.abs(g))
    assert np.all(np.abs(w.cpu().numpy()[rows] - prod) <= bound + 1e-320)


@pytest.mark.parametrize("m1,m2", [(64, 64), (127, 129), (128, 64), (129, 200), (255, 65), (256, 256), (300, 64),
                                   (65, 300)])
def test_ozaki_gram_segments_edges(cuda, m1, m2):
    """The Gram's segments (main 128 x 64 block, narrow right strip, bottom rows computed
    transposed) at tile boundaries: every entry, the last rows and columns included, within
    the DGEMM-class bound."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n = 16384
    x, y = gauss(n, m1, 130 + m1), gauss(n, m2, 140 + m2)
    with emu(torch):
        c = K.gram(dev(x, torch), dev(y, torch)).cpu().numpy()
    c1 = np.unique(np.r_[0, m1 // 2, np.arange(max(0, m1 - 12), m1)])
    c2 = np.unique(np.r_[0, m2 // 2, np.arange(max(0, m2 - 12), m2)])
    ref, absprod = exact_gram(x, y, c1, c2)
    assert np.all(np.abs(c[np.ix_(c1, c2)] - ref) <= 4 * U * absprod)


@pytest.mark.parametrize("m", [64, 127, 128, 129, 191, 192, 257])
def test_ozaki_gram_symmetric_segments(cuda, m):
    """Symmetric Grams: upper main tiles, the right strip and the diagonal corner, mirrored --
    exactly symmetric, and the corner / strip entries within the bound."""
    from paper_1407_7506_b200 import kernels as K

    torch = cuda
    n = 16384
    xd = dev(gauss(n, m, 150 + m), torch)
    with emu(torch):
        g = K.gram(xd, xd, symmetric=True).cpu().numpy()
    assert np.array_equal(g, g.T)
    x = xd.cpu().numpy()
    cs = np.unique(np.r_[0, m // 2, np.arange(max(0, m - 12), m)])
    ref, absprod = exact_gram(x, x, cs, cs)
    assert np.all(np.abs(g[np.ix_(cs, cs)] - ref) <= 4 * U * absprod)
