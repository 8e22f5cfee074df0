"""Torch-tensor wrappers over the C ABI (include/ppcg_b200.h).

Tensors are 2-D row-major CUDA tensors, possibly column-sliced views (stride (ld, 1)).
Complex128 tensors are passed as interleaved real views: a complex n x m block with
leading dimension ld is a real n x 2m block with leading dimension 2*ld, so every FP64
tensor-core kernel is real; complex products are assembled by small expand/combine kernels.
"""

from __future__ import annotations

import threading

import torch

from . import _lib
from .errors import DeviceError

F64 = torch.float64
C128 = torch.complex128


def stream_ptr():
    return torch.cuda.current_stream().cuda_stream


def _check2d(t, name):
    if t.dim() != 2:
        raise DeviceError(f"{name}: expected 2-D tensor, got {tuple(t.shape)}")
    if not t.is_cuda:
        raise DeviceError(f"{name}: expected a CUDA tensor")
    if t.shape[0] > 0 and t.shape[1] > 0 and t.stride(1) != 1:
        raise DeviceError(f"{name}: inner stride must be 1 (row-major view)")


def ld_of(t):
    """Leading dimension (in elements of t's dtype)."""
    if t.shape[0] <= 1:
        return max(t.shape[1], 1) if t.dim() == 2 else 1
    return t.stride(0)


def real_view(t):
    """(ptr, rows, real_cols, real_ld) of a 2-D float64/complex128 tensor view."""
    _check2d(t, "block")
    if t.dtype == F64:
        return t.data_ptr(), t.shape[0], t.shape[1], ld_of(t)
    if t.dtype == C128:
        return t.data_ptr(), t.shape[0], 2 * t.shape[1], 2 * ld_of(t)
    raise DeviceError(f"unsupported dtype {t.dtype}")


class Workspace:
    """Zero-initialised scratch shared by the split-K / ticketed reductions (stream-ordered)."""

    def __init__(self, device=None, nbytes=1 << 22):
        self.device = device or torch.device("cuda")
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)

    def get(self, nbytes):
        nbytes = int(nbytes)
        if nbytes > self.buf.numel():
            grow = max(nbytes, int(self.buf.numel() * 1.5))
            torch.cuda.current_stream().synchronize()
            self.buf = torch.zeros(grow, dtype=torch.uint8, device=self.device)
        return self.buf.data_ptr(), self.buf.numel()


_WS = {}


def workspace(kind="gram"):
    """One zeroed scratch buffer per reduction family, device and stream.  Each family keeps
    its tickets at offset 0 and resets them after use; families must not share a buffer (one
    family's partials would overwrite another's tickets), and neither may two streams."""
    key = (torch.cuda.current_device(), kind, torch.cuda.current_stream().cuda_stream)
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = Workspace(torch.device("cuda", key[0]))
    return ws


# ----------------------------------------------------------------------------- FP64 emulation
# FP64 products of at least EMU_MIN_ROWS rows and EMU_MIN_COLS columns on each side run on the
# int8 tensor cores (Ozaki scheme, csrc/ozaki.cu); smaller ones on the FP64 DMMA kernels.
EMU_MIN_ROWS = 16384
EMU_MIN_COLS = 64


def fp64_emulation_enabled():
    return bool(_lib.load().bk_fp64_emu_enabled())


class fp64_emulation:
    """Context manager (and setter): ``with fp64_emulation(False): ...`` pins the DMMA kernels."""

    def __init__(self, on):
        lib = _lib.load()
        self.prev = lib.bk_fp64_emu_enabled()
        lib.bk_fp64_emu_set(1 if on else 0)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        _lib.load().bk_fp64_emu_set(self.prev)
        return False


def _emu(n, m1, m2):
    return n >= EMU_MIN_ROWS and min(m1, m2) >= EMU_MIN_COLS and _lib.load().bk_fp64_emu_enabled()


class ColDigits:
    """Exponents and column digits of an n x m real block (view), kept between the emulated
    Grams that have (a column range of) it as their left operand: ``coldigits(x)`` slices once,
    ``gram(x[:, a:b], y, xdig=d)`` / ``gram2(..., xdig=d)`` skip the slicing of X.  The caller
    keeps the block unchanged while the digits are in use."""

    __slots__ = ("buf", "ptr", "ld", "n", "m")

    def col0(self, px, lx, n, m1):
        """Column offset of the operand (px, lx, n rows, m1 real columns) inside the sliced
        block, or -1 when it is not a column range of it."""
        d = px - self.ptr
        if lx != self.ld or n != self.n or d < 0 or d % 8:
            return -1
        c0 = d // 8
        return c0 if c0 + m1 <= self.m else -1


def coldigits(x, buf=None):
    """ColDigits of the block x (float64, or complex128 as its interleaved real view), into
    ``buf`` (a uint8 CUDA tensor, grown if too small) -- or None when the emulated Grams would
    not be used for it."""
    px, n, mr, lx = real_view(x)
    if not _emu(n, mr, EMU_MIN_COLS):
        return None
    nbytes = int(_lib.load().bk_ozaki_coldigits_bytes(n, mr))
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    d = ColDigits()
    d.buf, d.ptr, d.ld, d.n, d.m = buf, px, lx, n, mr
    _lib.call("bk_ozaki_coldigits_d", n, mr, px, lx, buf.data_ptr(), buf.numel(), stream_ptr())
    return d


def _ozaki_gram(n, m1, m2, px, lx, py, ly, out_ptr, ldo, symmetric, ws_kind, xdig=None):
    lib = _lib.load()
    same = 1 if (px == py and lx == ly and m1 == m2) else 0
    sym = 1 if (symmetric and same) else 0
    c0 = xdig.col0(px, lx, n, m1) if xdig is not None else -1
    if c0 >= 0:
        wp, wb = workspace(ws_kind + "/oz").get(lib.bk_ozaki_gram_pre_ws_bytes(n, m1, m2, same, sym))
        _lib.call("bk_ozaki_gram_pre_d", n, m1, m2, px, lx, xdig.buf.data_ptr(), xdig.m, c0, py, ly, out_ptr, ldo, sym,
                  wp, wb, stream_ptr())
        return
    wp, wb = workspace(ws_kind + "/oz").get(lib.bk_ozaki_gram_ws_bytes(n, m1, m2, same, sym))
    _lib.call("bk_ozaki_gram_d", n, m1, m2, px, lx, py, ly, out_ptr, ldo, sym, wp, wb, stream_ptr())


# ----------------------------------------------------------------------------- Grams
_STRIP = threading.local()


def set_strip_stream(stream):
    """Second stream for the narrow strip launches of split Grams (None: same stream).  The
    compute-bound 64-aligned main launch and the memory-bound strips then overlap."""
    _STRIP.stream = stream


def _split_launch(splits, call_part, ws_kind, nbytes):
    """call_part(part, ws_ptr, ws_bytes, stream): whole Gram on the current stream, or the
    main block there and the strips on the strip stream (own workspace), fenced by events."""
    side = getattr(_STRIP, "stream", None)
    main = torch.cuda.current_stream()
    if side is None or not splits or side == main:
        wp, wb = workspace(ws_kind).get(nbytes)
        call_part(0, wp, wb, stream_ptr())
        return
    ev = torch.cuda.Event()
    ev.record(main)
    wp, wb = workspace(ws_kind).get(nbytes)
    call_part(1, wp, wb, stream_ptr())
    side.wait_event(ev)
    with torch.cuda.stream(side):
        sp, sb = workspace("strip").get(nbytes)
        call_part(2, sp, sb, stream_ptr())
    main.wait_stream(side)


def gram(x, y, out=None, symmetric=False, ws_kind="gram", xdig=None):
    """out = X^H Y (m1 x m2).  symmetric=True requires x is y (same view).  Launches on a
    second stream must pass their own ``ws_kind`` (split-K tickets live in the workspace).
    ``xdig``: ColDigits of a block that contains x as a column range (emulated Grams only)."""
    n = x.shape[0]
    if y.shape[0] != n:
        raise DeviceError(f"row dimensions differ: {n} vs {y.shape[0]}")
    m1, m2 = x.shape[1], y.shape[1]
    if out is None:
        out = torch.empty((m1, m2), dtype=x.dtype, device=x.device)
    if m1 == 0 or m2 == 0:
        return out
    lib = _lib.load()
    if x.dtype == F64:
        px, _, _, lx = real_view(x)
        py, _, _, ly = real_view(y)
        if _emu(n, m1, m2):
            _ozaki_gram(n, m1, m2, px, lx, py, ly, out.data_ptr(), ld_of(out), symmetric, ws_kind, xdig)
            return out
        _split_launch(lib.bk_gram_splits(m1, m2), lambda part, wp, wb, st: _lib.call(
            "bk_gram_part_d", n, m1, m2, px, lx, py, ly, out.data_ptr(), ld_of(out), 1 if symmetric else 0, part,
            wp, wb, st), ws_kind, lib.bk_gram_ws_bytes(n, m1, m2))
        return out
    # complex: real Gram of the interleaved views, then combine
    px, _, r1, lx = real_view(x)
    py, _, r2, ly = real_view(y)
    tmp = torch.empty((r1, r2), dtype=F64, device=x.device)
    if _emu(n, r1, r2):
        _ozaki_gram(n, r1, r2, px, lx, py, ly, tmp.data_ptr(), r2, symmetric, ws_kind, xdig)
        _lib.call("bk_cplx_gram_combine_d", m1, m2, tmp.data_ptr(), r2, out.data_ptr(), ld_of(out),
                  stream_ptr())
        return out
    _split_launch(lib.bk_gram_splits(r1, r2), lambda part, wp, wb, st: _lib.call(
        "bk_gram_part_d", n, r1, r2, px, lx, py, ly, tmp.data_ptr(), r2, 1 if symmetric else 0, part, wp, wb, st),
        ws_kind, lib.bk_gram_ws_bytes(n, r1, r2))
    _lib.call("bk_cplx_gram_combine_d", m1, m2, tmp.data_ptr(), r2, out.data_ptr(), ld_of(out),
              stream_ptr())
    return out


def gram2(x1, y1, out1, x2, y2, out2, xdig=None):
    """Two independent Grams in one launch (real only; complex falls back to two launches).
    Emulated: X^T Y1 and X^T Y2 of one basis X share its digits (``xdig``: already sliced)."""
    n = x1.shape[0]
    if (x1.dtype == F64 and x1.data_ptr() == x2.data_ptr() and x1.shape == x2.shape and x1.stride() == x2.stride()
            and _emu(n, x1.shape[1], min(y1.shape[1], y2.shape[1]))):
        lib = _lib.load()
        px, _, _, lx = real_view(x1)
        pa, _, _, la = real_view(y1)
        pb, _, _, lb = real_view(y2)
        c0 = xdig.col0(px, lx, n, x1.shape[1]) if xdig is not None else -1
        if c0 >= 0:
            wp, wb = workspace("gram/oz").get(lib.bk_ozaki_gram2_pre_ws_bytes(n, x1.shape[1], y1.shape[1], y2.shape[1]))
            _lib.call("bk_ozaki_gram2_pre_d", n, x1.shape[1], px, lx, xdig.buf.data_ptr(), xdig.m, c0, y1.shape[1], pa,
                      la, out1.data_ptr(), ld_of(out1), y2.shape[1], pb, lb, out2.data_ptr(), ld_of(out2), wp, wb,
                      stream_ptr())
            return
        wp, wb = workspace("gram/oz").get(lib.bk_ozaki_gram2_ws_bytes(n, x1.shape[1], y1.shape[1], y2.shape[1]))
        _lib.call("bk_ozaki_gram2_d", n, x1.shape[1], px, lx, y1.shape[1], pa, la, out1.data_ptr(), ld_of(out1),
                  y2.shape[1], pb, lb, out2.data_ptr(), ld_of(out2), wp, wb, stream_ptr())
        return
    if x1.dtype != F64 or _emu(x1.shape[0], min(x1.shape[1], x2.shape[1]), min(y1.shape[1], y2.shape[1])):
        gram(x1, y1, out1, xdig=xdig)
        gram(x2, y2, out2, xdig=xdig)
        return
    n = x1.shape[0]
    p1, _, _, l1 = real_view(x1)
    q1, _, _, k1 = real_view(y1)
    p2, _, _, l2 = real_view(x2)
    q2, _, _, k2 = real_view(y2)
    lib = _lib.load()
    nb = 2 * max(lib.bk_gram_ws_bytes(n, x1.shape[1], y1.shape[1]), lib.bk_gram_ws_bytes(n, x2.shape[1], y2.shape[1]))
    splits = lib.bk_gram_splits(x1.shape[1], y1.shape[1]) and lib.bk_gram_splits(x2.shape[1], y2.shape[1])
    _split_launch(splits, lambda part, wp, wb, st: _lib.call(
        "bk_gram2_part_d", n, x1.shape[1], y1.shape[1], p1, l1, q1, k1, out1.data_ptr(), ld_of(out1), x2.shape[1],
        y2.shape[1], p2, l2, q2, k2, out2.data_ptr(), ld_of(out2), part, wp, wb, st), "gram", nb)


# ----------------------------------------------------------------------------- tall GEMM
def _expand_cplx(g):
    K, N = g.shape
    gr = torch.empty((2 * K, 2 * N), dtype=F64, device=g.device)
    _lib.call("bk_cplx_expand_d", K, N, g.data_ptr(), ld_of(g), gr.data_ptr(), 2 * N, stream_ptr())
    return gr


def tsgemm(xs, gs, ys, alpha=1.0, beta=0.0, zs=None, rowscale=None, upper=False,
           metric=None, ksplit=0, nsplit=0):
    """Y_b = s (.) (alpha X_b G_b + beta Z_b) for up to 4 problems with equal shapes.

    ``metric`` (a 1-element float64 CUDA tensor) receives
    sum (alpha X_0[:, :ksplit] G_0[:ksplit] + beta Z_0)[:, :nsplit]^2.
    Y may be None for metric-only launches.  Y must not alias X.
    """
    nprob = len(xs)
    x0 = xs[0]
    n, K = x0.shape
    N = gs[0].shape[1]
    cplx = x0.dtype == C128
    if cplx:
        gs = [_expand_cplx(g) for g in gs]
        K, N, ksplit, nsplit = 2 * K, 2 * N, 2 * ksplit, 2 * nsplit
    xp = [real_view(x)[0] for x in xs]
    ldx = real_view(x0)[3]
    gp = [g.data_ptr() for g in gs]
    ldg = ld_of(gs[0]) if gs[0].dtype == F64 else 2 * ld_of(gs[0])
    yp = [real_view(y)[0] if y is not None else 0 for y in ys]
    ldy = real_view(ys[0])[3] if ys[0] is not None else 1
    if zs is not None:
        zp = [real_view(z)[0] for z in zs]
        ldz = real_view(zs[0])[3]
    else:
        zp, ldz = None, 1
    XP, _a = _lib.ptr_array(xp)
    GP, _b = _lib.ptr_array(gp)
    YP, _c = _lib.ptr_array(yp)
    ZP, _d = _lib.ptr_array(zp) if zp is not None else (None, None)
    if metric is not None:
        nbytes = _lib.load().bk_tsgemm_ws_bytes(n, N)
        wp, wb = workspace("metric").get(nbytes)
        mp = metric.data_ptr()
    else:
        wp, wb, mp = None, 0, None
    if rowscale is not None and cplx:
        pass  # rowscale is per row: identical on the real view
    if _emu(n, K, N) and K <= 16320:
        lib = _lib.load()
        nbytes = lib.bk_ozaki_tsgemm_ws_bytes(nprob, n, K, N, int(ksplit) if metric is not None else 0)
        wp, wb = workspace("tsgemm/oz").get(nbytes)
        _lib.call("bk_ozaki_tsgemm_d", nprob, n, K, N, float(alpha), XP, ldx, GP, ldg, float(beta), ZP, ldz, YP,
                  ldy, rowscale.data_ptr() if rowscale is not None else None, 1 if upper else 0, int(ksplit),
                  int(nsplit),
                  metric.data_ptr() if metric is not None else None, wp, wb, stream_ptr())
        return
    _lib.call("bk_tsgemm_batched_d", nprob, n, K, N, float(alpha), XP, ldx, GP, ldg, float(beta), ZP,
              ldz, YP, ldy, rowscale.data_ptr() if rowscale is not None else None,
              1 if upper else 0, int(ksplit), int(nsplit), mp, wp, wb, stream_ptr())


# ----------------------------------------------------------------------------- elementwise / reductions
def scale_rows(d, x, out):
    px, n, mr, lx = real_view(x)
    po, _, _, lo = real_view(out)
    _lib.call("bk_scale_rows_d", n, mr, d.data_ptr(), px, lx, po, lo, stream_ptr())
    return out


def sumsq(x, out):
    """out[0] = ||x||_F^2 (deterministic)."""
    px, n, mr, lx = real_view(x)
    lib = _lib.load()
    wp, wb = workspace("sumsq").get(lib.bk_sumsq_ws_bytes())
    _lib.call("bk_sumsq_d", n, mr, px, lx, out.data_ptr(), wp, wb, stream_ptr())
    return out


def small_stats(c, out):
    """out[0:3] = (||C||_F^2, ||C - I||_F^2, Re tr C)."""
    _check2d(c, "C")
    cplx = 1 if c.dtype == C128 else 0
    _lib.call("bk_small_stats_d", c.shape[0], c.shape[1], c.data_ptr(), ld_of(c), cplx, out.data_ptr(),
              stream_ptr())
    return out


def copy_cols(src, dst):
    """dst[:, :] = src[:, :] for equal-shaped column views of row-major buffers."""
    es = 16 if src.dtype == C128 else 8
    _lib.call("bk_copy_cols", src.shape[0], src.shape[1], es, src.data_ptr(), ld_of(src), 0,
              dst.data_ptr(), ld_of(dst), 0, stream_ptr())


def zero_cols(dst):
    es = 16 if dst.dtype == C128 else 8
    _lib.call("bk_zero_cols", dst.shape[0], dst.shape[1], es, dst.data_ptr(), ld_of(dst), 0, stream_ptr())


def rr_residual(v, av, omega, rowscale, w_out, colnorm2):
    """R = AV - V diag(omega); w_out = s (.) R (optional); colnorm2 = ||R(:, j)||^2."""
    n, kt = v.shape
    cplx = 1 if v.dtype == C128 else 0
    lib = _lib.load()
    wp, wb = workspace("rr").get(lib.bk_rr_residual_ws_bytes(kt))
    _lib.call("bk_rr_residual_d", n, kt, cplx, v.data_ptr(), ld_of(v), av.data_ptr(), ld_of(av),
              omega.data_ptr(), rowscale.data_ptr() if rowscale is not None else None,
              w_out.data_ptr() if w_out is not None else None,
              ld_of(w_out) if w_out is not None else 1, colnorm2.data_ptr(), wp, wb, stream_ptr())


# ----------------------------------------------------------------------------- operator apply
def spmm_csr(rowptr, col, val, x, y):
    n = y.shape[0]
    m = x.shape[1]
    if x.dtype == F64:
        _lib.call("bk_spmm_csr_d", n, rowptr.data_ptr(), col.data_ptr(), val.data_ptr(), m, x.data_ptr(),
                  ld_of(x), y.data_ptr(), ld_of(y), stream_ptr())
    else:
        _lib.call("bk_spmm_csr_z", n, rowptr.data_ptr(), col.data_ptr(), val.data_ptr(), m, x.data_ptr(),
                  ld_of(x), y.data_ptr(), ld_of(y), stream_ptr())
    return y


def _row_align(t):
    """Byte alignment every row start of t's underlying buffer has (128 or 16)."""
    base = t.untyped_storage().data_ptr()
    rowb = ld_of(t) * t.element_size()
    return 128 if base % 128 == 0 and rowb % 128 == 0 else 16


def spmm_march(plan, x, y):
    """Plane-marching stencil SpMM (bk_spmm_march_*) with a device StencilPlan; returns False
    when the views' alignment does not allow it (the caller then uses spmm_csr)."""
    m = x.shape[1]
    ldx, ldy = ld_of(x), ld_of(y)
    if x.dtype == F64:
        if ldx % 2 or ldy % 2 or (x.data_ptr() % 16) != (y.data_ptr() % 16) or x.data_ptr() % 8:
            return False
        name = "bk_spmm_march_d"
    else:
        name = "bk_spmm_march_z"
    nx, ny, nz = plan.grid
    align = min(_row_align(x), _row_align(y))
    if getattr(plan, "sval", None) is not None and plan.use_slot:
        _lib.call(name.replace("march", "stencil"), nx, ny, nz, plan.xlo, plan.xhi, plan.d0, plan.sval.data_ptr(),
                  plan.vd, plan.st, m, x.data_ptr(), ldx, y.data_ptr(), ldy, align, stream_ptr())
        return True
    if plan.ell_val is None:
        return False
    _lib.call(name, nx, ny, nz, plan.xlo, plan.xhi, plan.d0, plan.ell_val.data_ptr(), plan.ell_off.data_ptr(),
              plan.width, plan.woff, m, x.data_ptr(), ldx, y.data_ptr(), ldy, align, stream_ptr())
    return True


# ----------------------------------------------------------------------------- subblock path
def subblock_grams(n, k_act, q, has_p, X, W, P, AX, AW, AP, ld, c0, araw, braw, tmp=None):
    """Raw pencil Grams of every subblock.  Pointers are raw device addresses of the state
    buffers (ld, c0 in elements of the state dtype); complex needs real scratch ``tmp``
    (two tensors of nb*(2*dmax)^2 doubles)."""
    lib = _lib.load()
    hp = 1 if has_p else 0
    if araw.dtype == C128:
        wp, wb = workspace().get(lib.bk_subblock_grams_ws_bytes(n, 2 * k_act, 2 * q, hp))
        _lib.call("bk_subblock_grams_z", n, k_act, q, hp, X, W, P if has_p else None, AX, AW,
                  AP if has_p else None, ld, c0, araw.data_ptr(), braw.data_ptr(), tmp[0].data_ptr(),
                  tmp[1].data_ptr(), wp, wb, stream_ptr())
        return
    wp, wb = workspace().get(lib.bk_subblock_grams_ws_bytes(n, k_act, q, hp))
    _lib.call("bk_subblock_grams_d", n, k_act, q, hp, X, W, P if has_p else None, AX, AW,
              AP if has_p else None, ld, c0, araw.data_ptr(), braw.data_ptr(), wp, wb, stream_ptr())


def _pencil_ws(nb, d, cplx):
    """Global scratch of the large (d > 96 real / 64 complex) pencil variant, else (None, 0)."""
    nbytes = _lib.load().bk_pencil_ws_bytes(nb, d, 1 if cplx else 0)
    return workspace("pencil").get(nbytes) if nbytes else (None, 0)


def subblock_pencils(k_act, q, has_p, araw, braw, coef, theta, info, cscale, force_fallback=False):
    cplx = araw.dtype == C128
    name = "bk_subblock_pencils_z" if cplx else "bk_subblock_pencils_d"
    wp, wb = _pencil_ws((k_act + q - 1) // q, (3 if has_p else 2) * q, cplx)
    _lib.call(name, k_act, q, 1 if has_p else 0, araw.data_ptr(), braw.data_ptr(),
              coef.data_ptr(), theta.data_ptr(), info.data_ptr(), cscale.data_ptr(),
              1 if force_fallback else 0, wp, wb, stream_ptr())


def subblock_pencils_range(j0, j1, k_act, q, has_p, araw, braw, coef, theta, info, cscale):
    """subblock_pencils for subblocks [j0, j1) only (the row-partitioned solver's chunk):
    the same kernel on pointer-offset views -- block j's pencil, coefficients, Ritz values,
    status and scale live at fixed strides, and only the global last block is narrower."""
    cplx = araw.dtype == C128
    dmax = (3 if has_p else 2) * q
    es = araw.element_size()
    ka = min(k_act - j0 * q, (j1 - j0) * q)
    name = "bk_subblock_pencils_z" if cplx else "bk_subblock_pencils_d"
    wp, wb = _pencil_ws(j1 - j0, dmax, cplx)
    _lib.call(name, ka, q, 1 if has_p else 0, araw.data_ptr() + j0 * dmax * dmax * es,
              braw.data_ptr() + j0 * dmax * dmax * es, coef.data_ptr() + j0 * dmax * q * coef.element_size(),
              theta.data_ptr() + j0 * q * 8, info.data_ptr() + j0 * 4 * 4, cscale.data_ptr() + j0 * 8,
              0, wp, wb, stream_ptr())


def subblock_recombine(n, k_act, q, has_p, coef, X, W, P, AX, AW, AP, Xo, Po, AXo, APo, ld, c0, flags,
                       coef_tmp=None):
    if coef.dtype == C128:
        _lib.call("bk_subblock_recombine_z", n, k_act, q, 1 if has_p else 0, coef.data_ptr(), X, W,
                  P if has_p else None, AX, AW, AP if has_p else None, Xo, Po, AXo, APo, ld, c0,
                  flags.data_ptr(), coef_tmp.data_ptr(), stream_ptr())
        return
    _lib.call("bk_subblock_recombine_d", n, k_act, q, 1 if has_p else 0, coef.data_ptr(), X, W,
              P if has_p else None, AX, AW, AP if has_p else None, Xo, Po, AXo, APo, ld, c0,
              flags.data_ptr(), stream_ptr())


# ----------------------------------------------------------------------------- large subblocks
def pencil_max_dim():
    """Largest pencil dimension the batched device pencils solve (larger: bigblock.py)."""
    return int(_lib.load().bk_pencil_max_dim())


def block_assemble(d, idx, sf, araw, braw, ldr, a, b):
    """a, b (d x d) = scaled symmetrised pencil of the kept raw columns idx (int32) / scales sf."""
    cplx = 1 if a.dtype == C128 else 0
    _lib.call("bk_block_assemble", d, cplx, idx.data_ptr(), sf.data_ptr(), araw.data_ptr(), braw.data_ptr(), ldr,
              a.data_ptr(), b.data_ptr(), ld_of(a), stream_ptr())


def block_coef(d, w, nrows, idx, sf, c, coef, cmax):
    cplx = 1 if c.dtype == C128 else 0
    _lib.call("bk_block_coef", d, w, nrows, cplx, idx.data_ptr(), sf.data_ptr(), c.data_ptr(), ld_of(c),
              coef.data_ptr(), cmax.data_ptr(), stream_ptr())


def block_stats(x, flags, slot):
    cplx = 1 if x.dtype == C128 else 0
    _lib.call("bk_block_stats", x.shape[0], x.shape[1], cplx, x.data_ptr(), ld_of(x), flags.data_ptr(), slot,
              stream_ptr())


def pencil_batched(a, b, want, omega, c, status):
    """a, b: (nb, ldm, ldm) float64/complex128; solves nb pencils of dimension ldm."""
    nb, d, _ = a.shape
    cplx = a.dtype == C128
    name = "bk_pencil_batched_z" if cplx else "bk_pencil_batched_d"
    wp, wb = _pencil_ws(nb, d, cplx)
    _lib.call(name, nb, d, d, a.data_ptr(), b.data_ptr(), want, omega.data_ptr(),
              c.data_ptr(), status.data_ptr(), wp, wb, stream_ptr())


# ----------------------------------------------------------------------------- dense (cuSOLVER)
_DENSE = threading.local()


def dense_context():
    """The calling thread's cached Dense context for the current device (creating a
    cuSOLVER handle costs tens of ms; a handle must not be shared between host threads)."""
    cache = getattr(_DENSE, "by_dev", None)
    if cache is None:
        cache = _DENSE.by_dev = {}
    dev = torch.cuda.current_device()
    ctx = cache.get(dev)
    if ctx is None or ctx.h is None:
        ctx = cache[dev] = Dense()
    return ctx


_STAGE = threading.local()
_POOL = []
_POOL_LOCK = threading.Lock()


def _par_rows(fn, r0, r1, row_bytes, min_bytes=1 << 20):
    """fn(a, b) over [r0, r1) split across a shared host thread pool (numpy copies release
    the GIL; spreading them also spreads the page faults of a freshly allocated target)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    with _POOL_LOCK:
        if not _POOL:
            try:
                nt = len(os.sched_getaffinity(0))
            except Exception:
                nt = os.cpu_count() or 1
            _POOL.append((ThreadPoolExecutor(max_workers=max(1, min(16, nt))), max(1, min(16, nt))))
    pool, nt = _POOL[0]
    parts = max(1, min(nt, (r1 - r0) * row_bytes // min_bytes))
    if parts == 1:
        fn(r0, r1)
        return
    step = -(-(r1 - r0) // parts)
    futs = [pool.submit(fn, a, min(r1, a + step)) for a in range(r0, r1, step)]
    for f in futs:
        f.result()


def to_host(x, chunk_bytes=32 << 20, out=None):
    """numpy copy of a (possibly row-strided) 2-D device block through two pinned staging
    buffers: the device->pinned copy of one row chunk overlaps the (multi-threaded)
    pinned->numpy copy of the previous one (a pageable .cpu() of a large block runs at a
    few GB/s).  ``out``: a C-contiguous destination of the right shape / dtype (e.g. one
    whose pages were faulted in ahead of time)."""
    import numpy as np

    n, m = x.shape
    dt = np.complex128 if x.dtype == C128 else np.float64
    if out is None or out.shape != (n, m) or out.dtype != dt or not out.flags.c_contiguous:
        out = np.empty((n, m), dtype=dt)
    if n == 0 or m == 0:
        return out
    rb = m * x.element_size()
    rows = max(1, chunk_bytes // rb)
    key = (x.dtype, m, rows)
    st = getattr(_STAGE, "bufs", None)
    if st is None or st[0] != key:
        bufs = [torch.empty((rows, m), dtype=x.dtype, pin_memory=True) for _ in range(2)]
        st = _STAGE.bufs = (key, bufs, [torch.cuda.Event(), torch.cuda.Event()])
    _, bufs, evs = st
    pend = None

    def drain(pb, p0, p1):
        evs[pb].synchronize()
        src = bufs[pb].numpy()

        def cp(a, b):
            out[a:b] = src[a - p0:b - p0]
        _par_rows(cp, p0, p1, rb)

    for k, r0 in enumerate(range(0, n, rows)):
        r1 = min(n, r0 + rows)
        b = k & 1
        bufs[b][: r1 - r0].copy_(x[r0:r1], non_blocking=True)
        evs[b].record()
        if pend is not None:
            drain(*pend)
        pend = (b, r0, r1)
    drain(*pend)
    return out


def to_host_pinned(x, out, chunk_bytes=128 << 20):
    """numpy view of the page-locked tensor ``out`` after out[:, :] = x: row chunks of the
    (row-strided) device block are packed on the device and copied straight into ``out`` --
    no host staging pass.  The array keeps ``out`` alive (its base)."""
    n, m = x.shape
    rows = max(1, chunk_bytes // max(1, m * x.element_size()))
    for r0 in range(0, n, rows):
        out[r0:r0 + rows].copy_(x[r0:r0 + rows], non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def from_host(src, x, chunk_bytes=32 << 20):
    """x[:, :] = src through two pinned staging buffers: the pinned->device copy of one row
    chunk overlaps the (multi-threaded) fill of the next.  src is a C-contiguous numpy
    array, or any object with ``fill_rows(r0, r1, dst)`` (dst: a contiguous
    (r1 - r0) x m numpy view) -- the X0 draw fills staging straight from its chunks."""
    n, m = x.shape
    if n == 0 or m == 0:
        return x
    rb = m * x.element_size()
    rows = max(1, chunk_bytes // rb)
    key = (x.dtype, m, rows)
    st = getattr(_STAGE, "up", None)
    if st is None or st[0] != key:
        st = _STAGE.up = (key, [torch.empty((rows, m), dtype=x.dtype, pin_memory=True) for _ in range(2)])
    bufs = st[1]
    fill = getattr(src, "fill_rows", None)
    evs = [None, None]
    for k, r0 in enumerate(range(0, n, rows)):
        r1 = min(n, r0 + rows)
        b = k & 1
        if evs[b] is not None:
            evs[b].synchronize()
        dst = bufs[b].numpy()

        def cp(a, c, dst=dst, r0=r0):
            if fill is not None:
                fill(a, c, dst[a - r0:c - r0])
            else:
                dst[a - r0:c - r0] = src[a:c]
        _par_rows(cp, r0, r1, rb)
        x[r0:r1].copy_(bufs[b][: r1 - r0], non_blocking=True)
        evs[b] = torch.cuda.Event()
        evs[b].record()
    for e in evs:
        if e is not None:
            e.synchronize()
    return x


class Dense:
    """Owns a bk_dense context (cuSOLVER handle + workspace) bound to the current stream."""

    def __init__(self):
        import ctypes

        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.call("bk_dense_create", ctypes.byref(h), stream_ptr())
        self.h = h
        self._lib = lib

    def _sync_stream(self):
        _lib.call("bk_dense_set_stream", self.h, stream_ptr())

    def close(self):
        if self.h is not None and self.h.value:
            self._lib.bk_dense_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def chol_upper_floor(self, g, fail_col):
        self._sync_stream()
        name = "bk_chol_upper_floor_z" if g.dtype == C128 else "bk_chol_upper_floor_d"
        _lib.call(name, self.h, g.shape[0], g.data_ptr(), ld_of(g), fail_col.data_ptr())

    def tri_inv_upper(self, r):
        self._sync_stream()
        name = "bk_tri_inv_upper_z" if r.dtype == C128 else "bk_tri_inv_upper_d"
        _lib.call(name, self.h, r.shape[0], r.data_ptr(), ld_of(r))

    def rr_pencil(self, a, b, omega, c, status):
        self._sync_stream()
        name = "bk_rr_pencil_z" if a.dtype == C128 else "bk_rr_pencil_d"
        _lib.call(name, self.h, a.shape[0], a.data_ptr(), ld_of(a), b.data_ptr(), ld_of(b),
                  omega.data_ptr(), c.data_ptr(), ld_of(c), status.data_ptr())

    def svals(self, m, s):
        """s[:min(m.shape)] = singular values of the (row-major view) m, descending."""
        self._sync_stream()
        name = "bk_svals_z" if m.dtype == C128 else "bk_svals_d"
        _lib.call(name, self.h, m.shape[0], m.shape[1], m.data_ptr(), ld_of(m), s.data_ptr())

    def householder_q(self, x, tmp):
        self._sync_stream()
        name = "bk_householder_q_z" if x.dtype == C128 else "bk_householder_q_d"
        _lib.call(name, self.h, x.shape[0], x.shape[1], x.data_ptr(), ld_of(x), tmp.data_ptr())
