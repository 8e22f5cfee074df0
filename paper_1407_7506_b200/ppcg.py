"""PPCG block eigensolver on B200: host orchestration of the device kernels.

Drop-in for ``blockeig.ppcg.ppcg_solve`` (ppcg.py:587-787): same signature, options
(``SolverOptions``, ppcg.py:48-103), result (``SolveReport``, ppcg.py:149-163), trace
records and exceptions.  All n-length arithmetic runs in libppcg_b200.so; the host keeps
only the control flow of the reference loop (ppcg.py:653-758) and reads a handful of
scalars per iteration.

Device state: every block is an n x k_total row-major CUDA buffer and a
column keeps its global position for the whole run, so
  * [X_lock | X] is one buffer ``XF`` (locked columns lead, ppcg.py:110-112) and the full
    basis of _full_basis / _orth_loss / _extract_ritz is a free view (no concatenation);
  * the active block is the column range [L, k_total) of XF, AXF, W, AW, P, AP;
  * P realignment in lock_and_compact (ppcg.py:399-408) is a zeroing of re-activated
    columns only;
  * X/AX are ping-pong pairs: the subblock update, CholQR and Rayleigh-Ritz write the other
    buffer, so the pre-update X survives for the breakdown and rank-deficiency recoveries
    (ppcg.py:694-717, 456-472) without copies;
  * P/AP are updated in place (no recovery path reads the pre-update P: both drop P), so the
    state is 8 full-width blocks -- config 5 fits 8 GPUs (device_bytes_plan).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionError, RankDeficiencyError, SingularGramError
from .trace import TraceRecord

__all__ = ["SolverOptions", "SolveReport", "split_blocks", "ppcg_solve", "PPCGSolver", "device_bytes_plan"]

# host-sync trimming (bit 0: projections queued before the metric is read; bit 1: the
# orthonormality Gram queued before the update's flags are read); PPCG_SPECULATE overrides
_SPECULATE = int(os.environ.get("PPCG_SPECULATE", "7"))
# column digits of X kept between the emulated Grams of an iteration (PPCGSolver._slice_x);
# the buffer is as large as one state block, so only up to this size
_DIGIT_CACHE = int(os.environ.get("PPCG_DIGIT_CACHE", "1"))
_DIGIT_CACHE_MAX = 4 << 30
_COEFF_REFRESH = 100.0   # ppcg.py:41
_BREAKDOWN_MAX = 1e8     # ppcg.py:705
_TAYLOR_OK = 0.1         # core.py:127


@dataclass
class SolverOptions:
    """Tunables of the PPCG iteration; identical fields, defaults and validation to
    blockeig SolverOptions (ppcg.py:48-103)."""

    k: int
    nbuf: int | None = None
    sbsize: int = 5
    rr_period: float = 5
    tol: float = 1e-6
    trace_tol: float | None = None
    max_iter: int = 500
    orth_policy: str = "every"
    orth_period: int = 1
    orth_threshold: float = 0.1
    orth_scheme: str = "cholesky-qr"
    taylor_terms: int = 4
    seed: int = 0
    project_w: bool = True
    project_p: bool = True

    def resolved_nbuf(self):
        if self.nbuf is not None:
            return self.nbuf
        return math.ceil(0.02 * self.k)

    def validate(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.nbuf is not None and self.nbuf < 0:
            raise ValueError("nbuf must be >= 0")
        if self.sbsize < 1:
            raise ValueError("sbsize must be >= 1")
        if not (self.rr_period >= 1):
            raise ValueError("rr_period must be >= 1 (math.inf disables RR)")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.trace_tol is not None and self.trace_tol <= 0:
            raise ValueError("trace_tol must be positive")
        if self.max_iter < 0:
            raise ValueError("max_iter must be >= 0")
        if self.orth_policy not in ("every", "periodic", "adaptive"):
            raise ValueError(f"unknown orth_policy {self.orth_policy!r}")
        if self.orth_period < 1:
            raise ValueError("orth_period must be >= 1")
        if self.orth_scheme not in ("cholesky-qr", "taylor-polar"):
            raise ValueError(f"unknown orth_scheme {self.orth_scheme!r}")


@dataclass
class SolveReport:
    """Final eigenpairs plus the convergence record (ppcg.py:149-163)."""

    values: np.ndarray
    vectors: np.ndarray = field(repr=False)
    trace: list
    status: str
    iterations: int
    matvecs: int
    rr_count: int
    breakdown_recoveries: int
    wall_ms: float
    values_history: list = field(default_factory=list, repr=False)
    diagnostics: dict = field(default_factory=dict, repr=False)


def split_blocks(k_act, sbsize):
    """Contiguous column ranges of width sbsize; the last may be narrower (ppcg.py:189-195)."""
    if k_act < 0:
        raise ValueError("k_act must be >= 0")
    if sbsize < 1:
        raise ValueError("sbsize must be >= 1")
    return [(lo, min(lo + sbsize, k_act)) for lo in range(0, k_act, sbsize)]


def lock_count(values, rnorms, tol):
    """Prefix-closed convergence (detect_converged, rayleigh_ritz.py:95-108)."""
    n = 0
    for th, rn in zip(values, rnorms):
        if rn <= tol * max(abs(th), 1.0):
            n += 1
        else:
            break
    return n


def draw_initial_block(n, kt, complex_field, seed, x0=None):
    """Host draw of X0 exactly as _initial_block (ppcg.py:414-438) before orthonormalisation:
    numpy PCG64 normals (real block then imaginary block), x0 padded on the right."""
    from .hostrng import standard_normal

    dtype = np.complex128 if complex_field else np.float64

    def draw(cols):
        # one stream: n*cols real parts, then n*cols imaginary parts (multi-threaded,
        # bit-identical to rng.standard_normal((n, cols)) twice; hostrng.py)
        flat = standard_normal(seed, n * cols * (2 if complex_field else 1))
        blk = flat[: n * cols].reshape(n, cols)
        if complex_field:
            blk = blk + 1j * flat[n * cols:].reshape(n, cols)
        return blk

    if x0 is None:
        return draw(kt).astype(dtype)
    x0 = np.asarray(x0, dtype=dtype)
    if x0.ndim != 2 or x0.shape[0] != n:
        raise DimensionError(f"x0 must be {n} x m, got {x0.shape}")
    if x0.shape[1] > kt:
        raise DimensionError(f"x0 has {x0.shape[1]} columns, at most k + nbuf = {kt} allowed")
    if not np.all(np.isfinite(x0)):
        raise ValueError("x0 contains non-finite entries")
    pad = kt - x0.shape[1]
    return np.column_stack([x0, draw(pad).astype(dtype)]) if pad else x0.copy()


class _DrawRows:
    """Rows [lo, hi) of the real X0 draw without assembling it: from_host fills its pinned
    staging straight from the generator chunks (hostrng.FlatDraw)."""

    def __init__(self, draw, kt, lo):
        self.d, self.kt, self.lo = draw, kt, lo

    def fill_rows(self, r0, r1, dst):
        self.d.copy_range((self.lo + r0) * self.kt, (self.lo + r1) * self.kt, dst.reshape(-1))


_X0 = {"pool": None, "gen": 0, "lock": None}


def _x0_draw_locked(n, kt, seed):
    with _X0["lock"]:
        return initial_block_source(n, kt, False, seed, None, 0, n)


_RESULT_POOL = []          # [page-locked (n, k) tensor, lease: weakref (dead = free)]
_RESULT_POOL_TRIED = set()
_RESULT_POOL_MAX = 2 << 30
_RESULT_POOL_LOCK = __import__("threading").Lock()


def _pinned_take(n, k, cplx, device, owner):
    """A free page-locked (n, k) result tensor from the pool, leased to ``owner`` (a weakref),
    or None.  The pool keeps one buffer per result shape: finish() hands the caller a numpy view
    of it and the lease follows that array (and every view of it), so the buffer is reused
    only after the caller has dropped the previous result -- a caller that keeps results gets
    pageable arrays instead.  The one cold cudaHostAlloc per shape (~0.45 ms per MB, holding a
    driver lock that stalls kernel launches) happens here, on the worker thread."""
    import torch

    dtype = torch.complex128 if cplx else torch.float64
    nbytes = n * k * (16 if cplx else 8)
    if nbytes > _RESULT_POOL_MAX or nbytes == 0:
        return None
    key = (n, k, cplx, int(device))
    with _RESULT_POOL_LOCK:
        for ent in _RESULT_POOL:
            if ent[2] == key and ent[1]() is None:
                ent[1] = owner
                return ent
        if key in _RESULT_POOL_TRIED:
            return None
        _RESULT_POOL_TRIED.add(key)
        while _RESULT_POOL and sum(e[0].numel() * e[0].element_size() for e in _RESULT_POOL) + nbytes > _RESULT_POOL_MAX:
            _RESULT_POOL.pop(0)
    try:
        with torch.cuda.device(device):
            t = torch.empty((n, k), dtype=dtype, pin_memory=True)
    except Exception:
        return None
    ent = [t, owner, key]
    with _RESULT_POOL_LOCK:
        _RESULT_POOL.append(ent)
    return ent


def _result_buffer(n, k, cplx, device, owner):
    """The (n, k) result array, prepared on the X0 worker while the GPU iterates: a page-locked
    pool buffer when one is free (_pinned_take), so the final vector download is one device ->
    host copy at PCIe rate straight into the array the caller receives -- no staging copy, no
    page faults; otherwise a pageable array with its pages faulted in (a fresh 453 MB array
    costs ~60 ms of page faults at config 2)."""
    ent = _pinned_take(n, k, cplx, device, owner)
    if ent is not None:
        return ent
    import ctypes

    arr = np.empty((n, k), dtype=np.complex128 if cplx else np.float64)
    # libc memset through ctypes: the GIL is released, so the thread that launches the GPU
    # work is never held up (a numpy strided write keeps the GIL)
    ctypes.memset(arr.ctypes.data, 0, arr.nbytes)
    return arr


def _vectors_prefault(n, k, cplx, device, owner):
    if _X0["pool"] is None:
        return None
    return _X0["pool"].submit(_result_buffer, n, k, cplx, device, owner)


def _x0_prefetch(n, kt, seed):
    """Start the real X0 draw on one persistent worker thread (its reuse scratch persists
    across calls); returns a job token for _x0_take."""
    import threading
    from concurrent.futures import ThreadPoolExecutor

    if _X0["pool"] is None:
        _X0["pool"] = ThreadPoolExecutor(max_workers=1, thread_name_prefix="ppcg-x0")
        _X0["lock"] = threading.Lock()
    _X0["gen"] += 1
    fut = _X0["pool"].submit(_x0_draw_locked, n, kt, seed)
    return (_X0["gen"], n, kt, seed, fut)


class _x0_take:
    """Context manager over a prefetched draw: ``src`` is the draw if it is still the
    worker's latest (its scratch buffers are reused by the next prefetch) and for the same
    problem, else None (draw again).  The worker's lock is held while the draw is consumed."""

    def __init__(self, job, n, kt, seed):
        self.job, self.key, self.src, self.held = job, (n, kt, seed), None, False

    def __enter__(self):
        if self.job is not None:
            gen, n0, kt0, seed0, fut = self.job
            res = fut.result()
            _X0["lock"].acquire()
            self.held = True
            if gen == _X0["gen"] and (n0, kt0, seed0) == self.key:
                self.src = res
        return self

    def __exit__(self, *exc):
        if self.held:
            _X0["lock"].release()
        return False


def initial_block_source(n, kt, complex_field, seed, x0=None, lo=0, hi=None):
    """Rows [lo, hi) of draw_initial_block(...) in a form K.from_host accepts."""
    from .hostrng import normal_draw

    hi = n if hi is None else hi
    if x0 is None and not complex_field:
        return _DrawRows(normal_draw(seed, n * kt, reuse=True), kt, lo)
    return np.ascontiguousarray(draw_initial_block(n, kt, complex_field, seed, x0)[lo:hi])


class PPCGSolver:
    """Step-wise device PPCG (``start`` / ``step`` / ``finish``), used by ``ppcg_solve`` and
    by bench.py to time single outer iterations."""

    _metric_ev = None  # event after the queued metric copy (speculative projection, step)

    def __init__(self, a, t=None, x0=None, opts=None, comm=None):
        import torch

        from . import kernels as K
        from .operators import as_device_operator, as_device_preconditioner

        if opts is None:
            raise ValueError("opts is required")
        opts.validate()
        from . import _lib

        _lib.load()  # DeviceError without the library or a GPU: there is no CPU fallback
        self.torch, self.K = torch, K
        self.opts = opts
        self.a = a
        self.n = int(a.n)
        # row partition (distributed.py): comm with size > 1 -> this rank owns rows [lo, hi)
        self.comm = comm if comm is not None and comm.size > 1 else None
        self.plan = None
        # the host X0 draw (~70 ms at config 2, bit-identical to numpy's stream) depends only on
        # (seed, n, k_total): start it now, beside the operator upload and the allocations
        self._x0_job = None
        if (self.comm is None and x0 is None and opts.k + opts.resolved_nbuf() <= self.n
                and not np.issubdtype(np.dtype(a.dtype), np.complexfloating)):
            self._x0_job = _x0_prefetch(self.n, opts.k + opts.resolved_nbuf(), opts.seed)
        if self.comm is not None:
            from .distributed import HaloPlan, host_csr_of, local_rows_csr, partition_rows
            from .operators import DeviceCsr

            csr = host_csr_of(a)
            self.bounds = partition_rows(self.n, self.comm.size, csr.indptr, plane=_stencil_plane(csr))
            self.plan = p = HaloPlan(csr, self.bounds, self.comm.rank)
            self.dev_a = DeviceCsr(local_rows_csr(csr, p.lo, p.hi, p.g_lo, p.n_ext))
            self.prec = as_device_preconditioner(t)
            if self.prec is not None and self.prec[0] != "diag":
                raise NotImplementedError("row-partitioned runs support diagonal preconditioners only")
            self.rowscale = self.prec[1][p.lo:p.hi] if self.prec is not None else None
            self.nl = p.hi - p.lo
            self.cplx = bool(np.iscomplexobj(csr.data)) or bool(
                np.issubdtype(np.dtype(a.dtype), np.complexfloating))
        else:
            self.dev_a = as_device_operator(a)
            self.prec = as_device_preconditioner(t)
            self.rowscale = self.prec[1] if self.prec is not None and self.prec[0] == "diag" else None
            self.nl = self.n
            self.cplx = bool(np.issubdtype(np.dtype(a.dtype), np.complexfloating)) or self.dev_a.complex
        self.tdt = torch.complex128 if self.cplx else torch.float64
        self.k = opts.k
        self.kt = opts.k + opts.resolved_nbuf()
        if self.kt > self.n:
            raise DimensionError(f"k + nbuf = {self.kt} exceeds operator dimension {self.n}")
        self.x0 = x0
        self.matvecs = 0
        self._pmax = None
        self._overlap = None

    # ------------------------------------------------------------------ helpers
    def _A(self, x, y):
        """y = A x on device, counted in matvec units (operators.py:122-124)."""
        self.matvecs += x.shape[1]
        if not x.shape[1]:
            return
        if self.plan is None:
            self.dev_a.apply_into(x, y)
            return
        # row partition: fill the ghost rows of x's extended buffer, then the local CSR
        # (columns relative to the extended buffer's first row) multiplies it
        base, owned = self._ext_of(x)
        p = self.plan
        es = x.element_size()
        c0 = (x.data_ptr() - owned.data_ptr()) // es
        w = x.shape[1]
        if 4 * w <= 3 * base.shape[1]:
            # narrow active block (locked columns, padding): exchange only its columns, packed
            # into contiguous buffers, instead of whole ld-wide rows
            sends = [(peer, base[a - p.g_lo:b - p.g_lo, c0:c0 + w].contiguous()) for peer, a, b in p.send]
            recvs = [(peer, a, b, torch_empty_like_rows(base, b - a, w)) for peer, a, b in p.recv]
            self.comm.exchange(sends, [(peer, t) for peer, _, _, t in recvs])
            for _, a, b, t in recvs:
                base[a - p.g_lo:b - p.g_lo, c0:c0 + w].copy_(t)
        else:
            self.comm.exchange([(peer, base[a - p.g_lo:b - p.g_lo]) for peer, a, b in p.send],
                               [(peer, base[a - p.g_lo:b - p.g_lo]) for peer, a, b in p.recv])
        self.dev_a.apply_into(base[:, c0:c0 + x.shape[1]], y)

    def _ext_of(self, x):
        for base, owned in self._ext:
            lo = base.data_ptr()
            if lo <= x.data_ptr() < lo + base.numel() * base.element_size():
                return base, owned
        raise DimensionError("operator applied to a block without ghost rows")

    def _red(self, *ts):
        """Sum the row-partial results of a Gram / norm over the ranks (no-op on one GPU).
        A padded-row view (rows of ld > columns, unit column stride) is reduced as the
        contiguous span from its first to its last element: no gather/scatter copies; the
        padding in between is summed too and never read."""
        if self.comm is None:
            return
        for t in ts:
            if t.numel() == 0:
                continue
            if t.is_contiguous():
                self.comm.allreduce_sum(t)
            elif t.dim() == 2 and t.stride(1) == 1:
                span = (t.shape[0] - 1) * t.stride(0) + t.shape[1]
                self.comm.allreduce_sum(t.as_strided((span,), (1,)))
            else:
                tmp = t.contiguous()
                self.comm.allreduce_sum(tmp)
                t.copy_(tmp)

    def _precond_general(self, w):
        if self.prec is not None and self.prec[0] == "op":
            tmp = self.torch.empty_like(w)
            self.prec[1].apply_into(w, tmp)
            w.copy_(tmp)

    def _fetch(self, *pairs):
        """Copy device tensors into pinned host mirrors and synchronise once."""
        for dev, host in pairs:
            host.copy_(dev, non_blocking=True)
        self.torch.cuda.current_stream().synchronize()

    def _alloc(self):
        torch = self.torch
        kt = self.kt
        z = lambda *s, dt=None: torch.zeros(s, dtype=dt or self.tdt, device="cuda")  # noqa: E731
        # n x k_total blocks with the row stride padded to a multiple of 4 elements (16/32-byte
        # aligned rows for vector and bulk-tensor loads); columns keep global positions
        self.ldp = (kt + 15) // 16 * 16  # 128-byte rows (real): aligned TMA / bulk-copy row pieces
        self.side = torch.cuda.Stream()  # diagnostics that overlap the subblock pencils
        # the pencils run on a high-priority stream: when they and the side stream's Gram
        # become runnable together, the CTA scheduler dispatches the pencil CTAs first (a
        # pencil CTA needs a whole SM's shared memory, so it cannot start on an SM that
        # already holds Gram CTAs)
        self.hi = torch.cuda.Stream(priority=-5)
        # (kernels.set_strip_stream can run the narrow strips of split Grams on a second
        # stream beside the main launch; measured slower end to end at config 2 -- the strip
        # CTAs only start as main CTAs retire and the fences add host work -- so it is off)
        nl = self.nl
        blk = lambda: z(nl, self.ldp)[:, :kt]  # noqa: E731
        self._ext = []

        def xblk():
            # blocks the operator is applied to (X, W, P): with a row partition they carry
            # the ghost rows above and below the owned slab in one contiguous buffer
            if self.plan is None:
                return blk()
            base = z(self.plan.n_ext, self.ldp)
            owned = base[self.plan.top:self.plan.top + nl, :kt]
            self._ext.append((base, owned))
            return owned

        self.XF = [xblk(), xblk()]
        self.AXF = [blk(), blk()]
        self.W = xblk()
        self.AW = blk()
        self.P = [xblk()]   # updated in place (subblock recombination writes P', AP' over P, AP)
        self.AP = [blk()]
        self.xi = 0   # current X/AX buffer
        self.pi = 0   # the P/AP buffer
        sq = lambda: z(kt, self.ldp)[:, :kt]  # noqa: E731  (even ld: 16-byte operand loads)
        self.Gm = sq()
        self.Gl = sq()
        self.Gp = sq()
        self.Gp2 = sq()
        self.Gfull = sq()
        self.Gstack = sq()
        self.Rm = sq()
        self.Ahat = sq()
        self.Bhat = sq()
        self.Cm = sq()
        self.omega = z(kt, dt=torch.float64)
        self.colnorm2 = z(kt, dt=torch.float64)
        self.stats = z(32, dt=torch.float64)
        self.iflags = torch.full((8,), -1, dtype=torch.int32, device="cuda")
        self.flags64 = z(3, dt=torch.int64)
        self.h_stats = torch.zeros(32, dtype=torch.float64).pin_memory()
        self.h_iflags = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.h_flags64 = torch.zeros(3, dtype=torch.int64).pin_memory()
        self.h_omega = torch.zeros(kt, dtype=torch.float64).pin_memory()
        self.h_colnorm2 = torch.zeros(kt, dtype=torch.float64).pin_memory()
        self.rr_status = torch.zeros(4, dtype=torch.int32, device="cuda")
        self.h_rr_status = torch.zeros(4, dtype=torch.int32).pin_memory()
        q = self.opts.sbsize
        nbmax = (kt + q - 1) // q
        if self.comm is not None:  # pencils split over the ranks: a whole chunk per rank
            nbmax = -(-nbmax // self.comm.size) * self.comm.size
        dmax = 3 * q
        self.araw = z(nbmax * dmax * dmax)
        self.braw = z(nbmax * dmax * dmax)
        self.coef = z(nbmax * dmax * q)
        if self.cplx:  # real scratch for Grams of interleaved views and expanded coefficients
            self.gtmp = (z(nbmax * 4 * dmax * dmax, dt=torch.float64), z(nbmax * 4 * dmax * dmax, dt=torch.float64))
            self.coef_tmp = z(nbmax * 4 * dmax * q, dt=torch.float64)
        else:
            self.gtmp, self.coef_tmp = None, None
        self.theta = z(max(kt, nbmax * q), dt=torch.float64)
        self.info = torch.zeros(nbmax * 4, dtype=torch.int32, device="cuda")
        self.cscale = z(nbmax, dt=torch.float64)
        self.h_info = torch.zeros(nbmax * 4, dtype=torch.int32).pin_memory()
        self.h_cscale = torch.zeros(nbmax, dtype=torch.float64).pin_memory()
        self.eye = torch.eye(kt, dtype=self.tdt, device="cuda")
        from .bigblock import LargeBlocks
        from .kernels import dense_context

        self.dense = dense_context()
        self.large = LargeBlocks(self)

    # views
    def X(self):
        return self.XF[self.xi][:, self.L:]

    def AX(self):
        return self.AXF[self.xi][:, self.L:]

    def Pa(self):
        return self.P[self.pi][:, self.L:]

    def APa(self):
        return self.AP[self.pi][:, self.L:]

    # ------------------------------------------------------------------ orthonormalisation
    # Column digits of [X_lock X] for the emulated Grams (kernels.ColDigits): sliced once by
    # _residual_w, then reused by the Grams that have the unchanged block as left operand --
    # the next iteration's projections X^H W / X^H P and proj_defect, the final Rayleigh-Ritz.
    # Every method that writes X drops them; the buffer index is checked on use.
    _xdig = None
    _xdig_buf = None

    def _slice_x(self, other_cols):
        """Slice XF[xi] for Grams whose right operands have at least ``other_cols`` columns."""
        self._xdig = None
        K = self.K
        xf = self.XF[self.xi]
        if not _DIGIT_CACHE or other_cols < K.EMU_MIN_COLS:
            return None
        if xf.shape[0] * xf.shape[1] * xf.element_size() > _DIGIT_CACHE_MAX:
            return None
        d = K.coldigits(xf, self._xdig_buf)
        if d is None:
            return None
        self._xdig_buf = d.buf
        self._xdig = (d, self.xi)
        return d

    def _xd(self):
        t = self._xdig
        return t[0] if t is not None and t[1] == self.xi else None

    def _cholqr_inplace_swap(self, gram_act, x_src_idx):
        """CholQR of the active block (core.py:86-100 / ppcg.py:483-484): R from the Gram
        with the pivot floor; X <- X R^{-1}, AX <- AX R^{-1} into the other buffer; swap.
        Raises RankDeficiencyError(column) like _cholesky_upper."""
        K = self.K
        self._xdig = None
        L, ka = self.L, self.kt - self.L
        R = self.Rm[:ka, :ka]
        spec = self._spec_R == L and gram_act.data_ptr() == self.Gfull[L:, L:].data_ptr()
        self._spec_R = None
        if not spec:
            self._cholqr_factor(gram_act)
            self._fetch((self.iflags, self.h_iflags))  # (speculated: fetched with the step's flags)
        col = int(self.h_iflags[0])
        if col >= 0:
            raise RankDeficiencyError(col)
        src, dst = x_src_idx, 1 - x_src_idx
        K.tsgemm([self.XF[src][:, L:], self.AXF[src][:, L:]], [R, R],
                 [self.XF[dst][:, L:], self.AXF[dst][:, L:]], upper=True)
        self.xi = dst

    _spec_R = None  # L of a CholQR factor already queued from Gfull (step)

    def _cholqr_factor(self, gram_act):
        """R^{-1} (upper) of the Gram with _cholesky_upper's pivot floor (core.py:67-83); the
        failing column (or -1) goes to iflags[0] -- read by the caller."""
        ka = gram_act.shape[0]
        R = self.Rm[:ka, :ka]
        R.copy_(gram_act)
        self.dense.chol_upper_floor(R, self.iflags[0:1])
        self.dense.tri_inv_upper(R)  # garbage when the factor failed; never used then

    def _taylor_swap(self, gram_act):
        """Taylor-polar correction X <- X p(G - I) (core.py:106-124, ppcg.py:477-481)."""
        K, torch = self.K, self.torch
        self._xdig = None
        L, ka = self.L, self.kt - self.L
        terms = self.opts.taylor_terms
        eye = self.eye[:ka, :ka]
        y = (gram_act - eye).contiguous()
        cf = [1.0]
        for i in range(1, terms + 1):
            cf.append(-cf[-1] * (2 * i - 1) / (2 * i))
        p = (cf[-1] * eye).contiguous()
        for c in reversed(cf[:-1]):
            pn = torch.empty_like(p)
            K.tsgemm([y], [p], [pn], alpha=1.0, beta=c, zs=[eye.contiguous()])
            p = pn
        src, dst = self.xi, 1 - self.xi
        K.tsgemm([self.XF[src][:, L:], self.AXF[src][:, L:]], [p, p],
                 [self.XF[dst][:, L:], self.AXF[dst][:, L:]])
        self.xi = dst

    def _residual_w(self):
        """W = T(AX - X (X^H AX)) (ppcg.py:630, 716, 758) with the Jacobi apply of
        ppcg.py:678 fused as a row scale and, when no column is locked, the next
        iteration's stopping metric fused as a partial-K snapshot."""
        K = self.K
        L, ka, k = self.L, self.kt - self.L, self.k
        x, ax = self.X(), self.AX()
        G = self.Gm[:ka, :ka]
        xd = self._slice_x(ka)
        if not (0 < L < k):  # (the locked form builds its own stacked Gram)
            K.gram(x, ax, G, xdig=xd)
            self._red(G)
        w = self.W[:, L:]
        if L == 0:
            K.tsgemm([x], [G], [w], alpha=-1.0, beta=1.0, zs=[ax], rowscale=self.rowscale,
                     metric=self.stats[0:1], ksplit=k, nsplit=k)
            self._red(self.stats[0:1])
            K.small_stats(G[:k, :k], self.stats[1:4])
            self.metric_cached = True
        elif L < k:
            self._residual_w_locked(x, ax, w)
            return
        else:
            K.tsgemm([x], [G], [w], alpha=-1.0, beta=1.0, zs=[ax], rowscale=self.rowscale)
            self.metric_cached = False
        self._precond_general(w)

    def _residual_w_locked(self, x, ax, w):
        """0 < L < k: the residual of the active block AND the next stopping metric over the
        leading k columns of [X_lock X] (ppcg.py:655-664) without the separate k x k Gram
        and metric GEMM (2 n k^2 flops each):
          Gs = [X_lock X]^H AX                  one Gram; its lower ka rows are X^H AX
          Y  = AX - [X_lock X] Gs               snapshot after K = k: ||AX_lead - X_lead G_lead||^2
                                                on the active lead columns
          W  = T(Y + X_lock Gs[:L])             = T(AX - X (X^H AX)), ppcg.py:630/758
          Glk = X_lead^H AX_lock, ||AX_lock - X_lead Glk||^2 for the locked lead columns,
          ||G_lead||_F^2 and Re tr G_lead from the blocks [Glk | Gs[:k, :k-L]]."""
        K = self.K
        L, k, ka = self.L, self.k, self.kt - self.L
        ma = k - L
        XFc, AXFc = self.XF[self.xi], self.AXF[self.xi]
        xl, axl = XFc[:, :L], AXFc[:, :L]
        Gs = self.Gstack[:, :ka]
        xd = self._xd()
        K.gram(XFc, ax, Gs, xdig=xd)
        self._red(Gs)
        K.tsgemm([XFc], [Gs], [w], alpha=-1.0, beta=1.0, zs=[ax], metric=self.stats[0:1], ksplit=k, nsplit=ma)
        K.tsgemm([xl], [Gs[:L]], [w], alpha=1.0, beta=1.0, zs=[w], rowscale=self.rowscale)
        Glk = self.Gl[:k, :L]
        K.gram(XFc[:, :k], axl, Glk, xdig=xd)
        self._red(Glk)
        K.tsgemm([XFc[:, :k]], [Glk], [None], alpha=-1.0, beta=1.0, zs=[axl], metric=self.stats[11:12], ksplit=k,
                 nsplit=L)
        self._red(self.stats[0:1], self.stats[11:12])
        K.sumsq(Glk, self.stats[12:13])
        K.sumsq(Gs[:k, :ma], self.stats[13:14])
        K.small_stats(Glk[:L], self.stats[14:17])
        K.small_stats(Gs[L:k, :ma], self.stats[17:20])
        self.metric_cached = "locked"
        self._precond_general(w)

    def _householder_refresh(self):
        """X <- qr(X)[0], AX <- A X (ppcg.py:712-713, 756-757)."""
        self._xdig = None
        x = self.X()
        if self.comm is None:
            self.dense.householder_q(x, self.AW)
        else:
            self._shifted_cholqr3()
            x = self.X()
        self._A(x, self.AX())

    def _shifted_cholqr3(self):
        """Row partition: the orthonormal basis of ppcg.py:712-713's qr(X) without gathering
        the block -- shifted Cholesky-QR (G + s I, s = 11 (n k + k (k+1)) u ||X||_F^2 keeps the
        factor positive definite at any conditioning) followed by two plain Cholesky-QR
        passes, each a Gram + allreduce + k x k factor + tall triangular GEMM.  Spans the same
        subspace as the Householder Q with columns equal up to sign/rounding (column signs
        are equivariant in PPCG); this path runs only after a breakdown or a
        rank-deficient CholQR, both of which drop P."""
        K, torch = self.K, self.torch
        self._xdig = None
        L, ka = self.L, self.kt - self.L
        for shift in (True, False, False):
            x = self.X()
            G = self.Gm[:ka, :ka]
            K.gram(x, x, G, symmetric=True)
            self._red(G)
            if shift:
                tr = float(torch.real(torch.diagonal(G)).sum().item())
                s_ = 11.0 * (self.n * ka + ka * (ka + 1)) * 2.220446049250313e-16 * max(tr, 1e-300)
                torch.diagonal(G).add_(s_)
            self._cholqr_factor(G)
            src, dst = self.xi, 1 - self.xi
            K.tsgemm([self.XF[src][:, L:]], [self.Rm[:ka, :ka]], [self.XF[dst][:, L:]], upper=True)
            self.xi = dst

    # ------------------------------------------------------------------ Rayleigh-Ritz
    def _ritz(self, fresh):
        """_extract_ritz (ppcg.py:553-584) over [X_lock, X].  Writes the Ritz vectors (and
        A V) into the other X buffer and returns host (omega, colnorm2)."""
        K = self.K
        kt = self.kt
        for attempt in range(2):
            S, AS = self.XF[self.xi], self.AXF[self.xi]
            xd = self._xd()
            if xd is None:  # S is the left operand of both Grams: slice it once
                xd = self._slice_x(self.kt)
            K.gram(S, AS, self.Ahat, xdig=xd)
            K.gram(S, S, self.Bhat, symmetric=True, xdig=xd)
            self._xdig = None
            self._red(self.Ahat, self.Bhat)
            self.dense.rr_pencil(self.Ahat, self.Bhat, self.omega, self.Cm, self.rr_status)
            self._fetch((self.rr_status, self.h_rr_status))
            if int(self.h_rr_status[0]) == 0:
                break
            if attempt == 1:
                raise SingularGramError("Gram matrix numerically singular in Rayleigh-Ritz")
            # clean the active block and retry once (ppcg.py:558-572)
            ka = kt - self.L
            G = self.Gm[:ka, :ka]
            K.gram(self.X(), self.X(), G, symmetric=True)
            self._red(G)
            try:
                self._cholqr_inplace_swap(G, self.xi)
            except RankDeficiencyError:
                self._householder_refresh()
        src, dst = self.xi, 1 - self.xi
        V = self.XF[dst]
        AV = self.AXF[dst]
        if fresh:
            K.tsgemm([S], [self.Cm], [V])
            self._A(V, AV)
        else:
            K.tsgemm([S, AS], [self.Cm, self.Cm], [V, AV])
        return src, dst

    def _rr_and_lock(self):
        K = self.K
        kt = self.kt
        src, dst = self._ritz(fresh=True)
        V, AV = self.XF[dst], self.AXF[dst]
        K.rr_residual(V, AV, self.omega, self.rowscale, self.W, self.colnorm2)
        self._red(self.colnorm2)
        self._fetch((self.omega, self.h_omega), (self.colnorm2, self.h_colnorm2))
        omega = self.h_omega.numpy().copy()
        rn = np.sqrt(self.h_colnorm2.numpy())
        self.rr_count += 1
        self.values_history.append(omega.copy())
        L_old = self.L
        L_new = lock_count(omega, rn, self.opts.tol)
        # lock_and_compact (ppcg.py:381-411): W <- residual (already in W, global columns)
        if self.has_p and L_new < L_old:
            K.zero_cols(self.P[self.pi][:, L_new:L_old])
            K.zero_cols(self.AP[self.pi][:, L_new:L_old])
        self.xi = dst
        if L_new > 0:
            K.copy_cols(self.XF[dst][:, :L_new], self.XF[src][:, :L_new])
            K.copy_cols(self.AXF[dst][:, :L_new], self.AXF[src][:, :L_new])
        self.L = L_new
        self.values_lock = omega[:L_new]
        self._precond_general(self.W[:, L_new:])
        self.metric_cached = False

    # ------------------------------------------------------------------ run
    def start(self):
        torch, K = self.torch, self.K
        self._alloc()
        self.t0 = time.perf_counter()
        self.L = 0
        self.has_p = False
        self.metric_cached = False
        # cholesky_qr of the initial block (ppcg.py:437-438)
        raw = self.XF[1]
        lo, hi = (self.plan.lo, self.plan.hi) if self.plan is not None else (0, self.n)
        with _x0_take(self._x0_job if not self.cplx else None, self.n, self.kt, self.opts.seed) as pre:
            src = pre.src
            if src is None:
                src = initial_block_source(self.n, self.kt, self.cplx, self.opts.seed, self.x0, lo, hi)
            K.from_host(src, raw)
        self._x0_job = None
        # the result array's pages, faulted in on the worker while the GPU iterates (finish)
        import weakref

        self._vec_job = (_vectors_prefault(self.n, self.k, self.cplx, torch.cuda.current_device(), weakref.ref(self))
                         if self.comm is None else None)
        G = self.Gm
        K.gram(raw, raw, G, symmetric=True)
        self._red(G)
        self.xi = 1
        self._cholqr_inplace_swap(G, 1)
        self._A(self.X(), self.AX())
        self._residual_w()
        self.trace, self.values_history = [], []
        self.orth_loss, self.proj_defect = [], []
        self.rr_count = self.recoveries = self.refreshes = 0
        self._metric_ev = None
        self.prev_trace = None
        self.status, self.iterations = "max_iter", self.opts.max_iter
        self.it = 0
        self.values_lock = np.zeros(0)
        self.done = self.opts.max_iter == 0
        return self

    def _metrics(self):
        """Stopping metrics on the leading k columns (ppcg.py:655-664)."""
        K = self.K
        k = self.k
        if not self.metric_cached:
            xl, axl = self.XF[self.xi][:, :k], self.AXF[self.xi][:, :k]
            Gk = self.Gl[:k, :k]
            K.gram(xl, axl, Gk, xdig=self._xd())
            self._red(Gk)
            K.small_stats(Gk, self.stats[1:4])
            K.tsgemm([xl], [Gk], [None], alpha=-1.0, beta=1.0, zs=[axl], metric=self.stats[0:1],
                     ksplit=k, nsplit=k)
            self._red(self.stats[0:1])
        if self._metric_ev is None:
            self._fetch((self.stats, self.h_stats))
        else:  # copy issued before the speculative projection launches (step)
            self._metric_ev.synchronize()
            self._metric_ev = None
        s = self.h_stats.numpy()
        if self.metric_cached == "locked":  # assembled from the locked/active blocks
            rel = math.sqrt(max(s[0] + s[11], 0.0)) / max(math.sqrt(max(s[12] + s[13], 0.0)), 1e-300)
            return float(rel), float(s[16] + s[19])
        rel = math.sqrt(max(s[0], 0.0)) / max(math.sqrt(max(s[1], 0.0)), 1e-300)
        return float(rel), float(s[3])

    def step(self):
        """One outer iteration (ppcg.py:653-758).  Returns True once the run has stopped."""
        if self.done:
            return True
        K, torch, o = self.K, self.torch, self.opts
        it = self.it = self.it + 1
        L, kt = self.L, self.kt
        ka = kt - L
        w, aw = self.W[:, L:], self.AW[:, L:]
        mv0 = self.matvecs
        # The stopping metric is already on the device (fused into the last residual): queue
        # its copy, then the projections of this iteration, then wait for the copy only -- the
        # GPU runs the projections while the host tests convergence.  On convergence the
        # speculative work (W, AW, stats[4] of an iteration that does not happen) is dropped:
        # finish() reads only X and AX, and the matvec count is rolled back.
        spec = bool(self.metric_cached) and ka > 0 and _SPECULATE & 1
        if spec:
            self.h_stats.copy_(self.stats, non_blocking=True)
            self._metric_ev = self.torch.cuda.Event()
            self._metric_ev.record()
            # W = T(W) is already applied (fused into the producer); AW = A W and the
            # projections (ppcg.py:678-687)
            self._project(L, ka, w, aw)
        rel, tr = self._metrics()
        chg = math.inf if self.prev_trace is None else abs(tr - self.prev_trace) / max(abs(tr), 1e-300)
        self.prev_trace = tr
        done = rel <= o.tol or (o.trace_tol is not None and chg <= o.trace_tol)
        if done or ka == 0:
            self.matvecs = mv0
            self.status, self.iterations, self.done = "converged", it - 1, True
            return True
        self.trace.append(TraceRecord(iteration=it, trace_value=tr, rel_resid=rel, n_locked=L,
                                      n_matvec=mv0,
                                      wall_ms=(time.perf_counter() - self.t0) * 1e3))
        if not spec:
            self._project(L, ka, w, aw)
        # proj_defect = ||[X_lock X]^H W||_F / ||W||_F (ppcg.py:688-692): a diagnostic that
        # nothing downstream reads, so it runs on a side stream concurrently with the
        # subblock pencils (one CTA per subblock leaves most SMs idle)
        Gd = self.Gp[:kt, :ka]
        main = torch.cuda.current_stream()
        xfull = self.XF[self.xi]
        xd = self._xd()  # last use of X's digits: the subblock update writes the other buffer,
        self._xdig = None  # the orthonormalisation after it this one
        if self.comm is None:
            def overlap(ready):  # after the pencil Grams (event `ready`): runs beside the pencils
                self.side.wait_event(ready)
                with torch.cuda.stream(self.side):
                    K.gram(xfull, w, Gd, ws_kind="side", xdig=xd)
                    K.small_stats(Gd, self.stats[5:8])
            self._overlap = overlap
        else:  # collectives stay on one stream, in the same order on every rank
            K.gram(xfull, w, Gd, xdig=xd)
            self._red(Gd)
            K.small_stats(Gd, self.stats[5:8])

        # subblock updates (ppcg.py:694-696) -> other buffers
        q = o.sbsize
        src, dst = self.xi, 1 - self.xi
        psrc = pdst = self.pi  # P, AP in place
        self._subblock_update(ka, q, src, psrc, dst, pdst)
        nb = (ka + q - 1) // q
        main.wait_stream(self.side)
        # orthonormality Gram of the updated [X_lock, X] (ppcg.py:726-729), queued before the
        # host reads the update's flags so one sync serves both; a breakdown (rare) restores
        # the previous X and leaves this Gram unused, a coefficient refresh keeps X
        early = bool(_SPECULATE & 2)
        self._spec_R = None
        if early:
            K.gram(self.XF[dst], self.XF[dst], self.Gfull, symmetric=True)
            self._red(self.Gfull)
            K.small_stats(self.Gfull, self.stats[8:11])
            # the CholQR factor of the coming orthonormalisation (ppcg.py:483-484) depends only on
            # this Gram: factor and invert it before the host reads the flags, so the GPU is not
            # idle across two host round trips (unused when the iteration ends otherwise)
            rr_now = math.isfinite(o.rr_period) and it % int(o.rr_period) == 0
            if (_SPECULATE & 4 and not rr_now and o.orth_scheme == "cholesky-qr"
                    and o.orth_policy in ("every", "adaptive", "periodic")):
                self._cholqr_factor(self.Gfull[L:, L:])
                self._spec_R = L
        fetch = [(self.info, self.h_info), (self.cscale, self.h_cscale), (self.flags64, self.h_flags64),
                 (self.stats, self.h_stats)]
        if self._spec_R is not None:
            fetch.append((self.iflags, self.h_iflags))  # the speculated factor's pivot flag: same sync
        self._fetch(*fetch)
        s = self.h_stats.numpy()
        wn = math.sqrt(max(s[4], 0.0))
        self.proj_defect.append(float(math.sqrt(max(s[5], 0.0)) / max(wn, 1e-300)))
        info = self.h_info.numpy()[: 4 * nb].reshape(nb, 4)
        if np.any(info[:, 2] != 0):
            raise SingularGramError("Gram matrix numerically singular in a subblock pencil")
        self.recoveries += int(np.sum(info[:, 0]))
        cs = max(1.0, float(np.max(self.h_cscale.numpy()[:nb])))
        f64 = self.h_flags64.numpy()
        mx = float(np.frombuffer(np.int64(f64[1]).tobytes(), dtype=np.float64)[0])
        mp = float(np.frombuffer(np.int64(f64[2]).tobytes(), dtype=np.float64)[0])
        broken = bool(f64[0] != 0) or max(mx, mp) > _BREAKDOWN_MAX
        prev_idx, prev_pidx = src, psrc
        if broken:
            # ppcg.py:706-717: restore pre-update X, Householder QR, drop P
            self._spec_R = None
            self.recoveries += 1
            self.orth_loss.append(math.inf)
            self.xi = prev_idx
            self._householder_refresh()
            self.has_p = False
            self._residual_w()
            self._check_max_iter()
            return self.done
        self.xi, self.pi = dst, pdst
        self.has_p = True
        if cs > _COEFF_REFRESH:
            # ppcg.py:718-724: refresh the cached products with real operator applications
            self.refreshes += 1
            self._A(self.X(), self.AX())
            self._A(self.Pa(), self.APa())
        # orthonormality loss of [X_lock, X] (ppcg.py:726-729): its Gram came with the flags
        if not early:
            K.gram(self.XF[self.xi], self.XF[self.xi], self.Gfull, symmetric=True)
            self._red(self.Gfull)
            K.small_stats(self.Gfull, self.stats[8:11])
            self._fetch((self.stats, self.h_stats))
        loss = float(math.sqrt(max(s[9], 0.0)))
        self.orth_loss.append(loss)
        gact = self.Gfull[L:, L:]
        if math.isfinite(o.rr_period) and it % int(o.rr_period) == 0:
            self._rr_and_lock()
        else:
            do = (o.orth_policy == "every"
                  or (o.orth_policy == "periodic" and it % o.orth_period == 0)
                  or (o.orth_policy == "adaptive" and loss >= o.orth_threshold))
            if do:
                try:
                    self._orth(gact, loss)
                except RankDeficiencyError as err:
                    self.recoveries += 1
                    self._redo_without_p(prev_idx, prev_pidx, err.column)
                    try:
                        K.gram(self.XF[self.xi], self.XF[self.xi], self.Gfull, symmetric=True)
                        self._red(self.Gfull)
                        self._orth(self.Gfull[L:, L:], loss)
                    except RankDeficiencyError:
                        self._householder_refresh()
            self._residual_w()
        self._check_max_iter()
        return self.done

    # AW = A W after the projections instead of updating A W with AX G: the same operator
    # applications (one per iteration on W, so matvec counts and traces match), one fewer
    # n x k_total x k_total GEMM per iteration, and an AW that is exact for the projected W
    # rather than carrying the drift of the cached AX (ppcg.py:679-687 apply first and update).
    FRESH_AW = True

    def _project(self, L, ka, w, aw):
        """W = T(R) arrives preconditioned; projections of W and P against X, then X_lock
        (ppcg.py:680-687; the same sequence as LOBPCG's, baselines.py:259-268), W and P
        batched per basis; AW = A W (ppcg.py:679, see FRESH_AW); ||W||_F^2 into stats[4]
        (fused into the last W update when possible)."""
        K, o = self.K, self.opts
        fresh = self.FRESH_AW and o.project_w
        if not fresh:
            self._A(w, aw)
        p, ap = (self.Pa(), self.APa()) if self.has_p else (None, None)
        proj_p = self.has_p and o.project_p

        def update(xb, axb, gw, gp, ks, metric):
            xs, gs, ys = [], [], []
            if o.project_w:
                xs.append(xb), gs.append(gw), ys.append(w)
                if not fresh:
                    xs.append(axb), gs.append(gw), ys.append(aw)
            if proj_p:
                xs += [xb, axb]
                gs += [gp, gp]
                ys += [p, ap]
            K.tsgemm(xs, gs, ys, alpha=-1.0, beta=1.0, zs=ys, metric=metric if o.project_w else None,
                     ksplit=ks, nsplit=ka)

        xd = self._xd()

        def grams(xb, gw, gp):
            if o.project_w and proj_p:
                K.gram2(xb, w, gw, xb, p, gp, xdig=xd)
                self._red(gw, gp)
            elif o.project_w:
                K.gram(xb, w, gw, xdig=xd)
                self._red(gw)
            else:
                K.gram(xb, p, gp, xdig=xd)
                self._red(gp)

        wnorm_done = False
        if o.project_w or proj_p:
            last_w = o.project_w and L == 0
            x, ax = self.X(), self.AX()
            G1, G3 = self.Gm[:ka, :ka], self.Gp2[:ka, :ka]
            grams(x, G1, G3)
            update(x, ax, G1, G3, ka, self.stats[4:5] if last_w else None)
            wnorm_done = last_w
            if L:
                xl, axl = self.XF[self.xi][:, :L], self.AXF[self.xi][:, :L]
                G2, G4 = self.Gl[:L, :ka], self.Gp[:L, :ka]
                grams(xl, G2, G4)
                update(xl, axl, G2, G4, L, self.stats[4:5])
                wnorm_done = o.project_w
        if not wnorm_done:
            K.sumsq(w, self.stats[4:5])
        self._red(self.stats[4:5])
        if fresh:
            self._A(w, aw)

    def _subblock_update(self, ka, q, src, psrc, dst, pdst):
        """block_update of every q-wide subblock of the active block (ppcg.py:487-533):
        batched device pencils, or bigblock.py beyond their limits; writes XF[dst], P[pdst],
        AXF[dst], AP[pdst], theta, info, cscale and the breakdown flags."""
        K, L = self.K, self.L
        XFs, AXFs = self.XF[src], self.AXF[src]
        Ps, APs = self.P[psrc], self.AP[psrc]
        overlap, self._overlap = self._overlap, None
        if self._large((3 if self.has_p else 2) * q, q):
            # pencils beyond the batched kernel (whole-block mode, sbsize >= 65): bigblock.py
            if overlap:
                ready = self.torch.cuda.Event()
                ready.record()
                overlap(ready)
            self.flags64.zero_()
            self.large.update(ka, q, self.has_p, src, psrc, dst, pdst)
        else:
            K.subblock_grams(self.nl, ka, q, self.has_p, XFs.data_ptr(), self.W.data_ptr(), Ps.data_ptr(),
                             AXFs.data_ptr(), self.AW.data_ptr(), APs.data_ptr(), self._ldr(), self._c0r(L),
                             self.araw, self.braw, tmp=self.gtmp)
            ready = self.torch.cuda.Event()
            ready.record()
            if self.comm is not None:
                self._pencils_split(ka, q)
            elif overlap:
                # pencils on the high-priority stream, the side-stream diagnostic beside them
                torch = self.torch
                self.hi.wait_event(ready)
                with torch.cuda.stream(self.hi):
                    K.subblock_pencils(ka, q, self.has_p, self.araw, self.braw, self.coef, self.theta, self.info,
                                       self.cscale)
                done = torch.cuda.Event()
                done.record(self.hi)
                overlap(ready)
                torch.cuda.current_stream().wait_event(done)
            else:
                K.subblock_pencils(ka, q, self.has_p, self.araw, self.braw, self.coef, self.theta, self.info,
                                   self.cscale)
            self.flags64.zero_()
            K.subblock_recombine(self.nl, ka, q, self.has_p, self.coef, XFs.data_ptr(), self.W.data_ptr(),
                                 Ps.data_ptr(), AXFs.data_ptr(), self.AW.data_ptr(), APs.data_ptr(),
                                 self.XF[dst].data_ptr(), self.P[pdst].data_ptr(), self.AXF[dst].data_ptr(),
                                 self.AP[pdst].data_ptr(), self._ldr(), self._c0r(L), self.flags64,
                                 coef_tmp=self.coef_tmp)
        if self.comm is not None:
            self.comm.allreduce_max(self.flags64)

    def _pencils_split(self, ka, q):
        """Row partition: the nb subblock pencils are independent (ppcg.py:515-519), so each
        rank solves a contiguous chunk of them.  The raw pencil Grams are reduce-scattered
        (rank r receives the sums of its chunk only), the chunk is solved, and the
        coefficients, Ritz values, status words and coefficient scales are all-gathered --
        instead of an allreduce of every Gram and nb replicated solves per rank."""
        K, comm = self.K, self.comm
        size, r = comm.size, comm.rank
        nb = (ka + q - 1) // q
        per = -(-nb // size)
        dmax = (3 if self.has_p else 2) * q
        dd = dmax * dmax
        comm.reduce_scatter_sum(self.araw[: size * per * dd], per * dd)
        comm.reduce_scatter_sum(self.braw[: size * per * dd], per * dd)
        j0, j1 = r * per, min(nb, (r + 1) * per)
        if j0 < j1:
            K.subblock_pencils_range(j0, j1, ka, q, self.has_p, self.araw, self.braw, self.coef, self.theta,
                                     self.info, self.cscale)
        comm.allgather_chunks(self.coef[: size * per * dmax * q], per * dmax * q)
        comm.allgather_chunks(self.theta[: size * per * q], per * q)
        comm.allgather_chunks(self.info[: size * per * 4], per * 4)
        comm.allgather_chunks(self.cscale[: size * per], per)

    def _orth(self, gact, loss):
        """_orth_active (ppcg.py:475-484)."""
        if self.opts.orth_scheme == "taylor-polar" and loss <= _TAYLOR_OK:
            self._taylor_swap(gact)
        else:
            self._cholqr_inplace_swap(gact, self.xi)

    def _redo_without_p(self, prev_idx, prev_pidx, column):
        """_redo_subblock_without_p (ppcg.py:456-472): fallback_steepest_descent on the
        pre-update subblock owning ``column``, written into the current buffers."""
        K = self.K
        q, L = self.opts.sbsize, self.L
        ka = self.kt - L
        lo = None
        for a, b in split_blocks(ka, q):
            if a <= column < b:
                lo, hi = a, b
        if lo is None:
            raise RankDeficiencyError(column, "failing column outside the active partition")
        w = hi - lo
        c0 = self._c0r(L + lo)
        XFp, AXFp = self.XF[prev_idx], self.AXF[prev_idx]
        if self._large(2 * w, w):
            self.flags64.zero_()
            self.large.update(ka, q, False, prev_idx, self.pi, self.xi, self.pi, force_fallback=True,
                              blocks=[(lo, hi)])
            self._fetch((self.info, self.h_info))
            if int(self.h_info.numpy()[2]) != 0:
                raise SingularGramError("Gram matrix numerically singular in fallback pencil")
            return
        K.subblock_grams(self.nl, w, w, False, XFp.data_ptr(), self.W.data_ptr(), 0, AXFp.data_ptr(),
                         self.AW.data_ptr(), 0, self._ldr(), c0, self.araw, self.braw, tmp=self.gtmp)
        self._red(self.araw, self.braw)
        K.subblock_pencils(w, w, False, self.araw, self.braw, self.coef, self.theta, self.info, self.cscale,
                           force_fallback=True)
        self.flags64.zero_()
        K.subblock_recombine(self.nl, w, w, False, self.coef, XFp.data_ptr(), self.W.data_ptr(), 0,
                             AXFp.data_ptr(), self.AW.data_ptr(), 0, self.XF[self.xi].data_ptr(),
                             self.P[self.pi].data_ptr(), self.AXF[self.xi].data_ptr(),
                             self.AP[self.pi].data_ptr(), self._ldr(), c0, self.flags64, coef_tmp=self.coef_tmp)
        self._fetch((self.info, self.h_info))
        if int(self.h_info.numpy()[2]) != 0:
            raise SingularGramError("Gram matrix numerically singular in fallback pencil")

    def _large(self, dmax, q):
        """Pencils beyond the batched kernels (dimension > 192 or subblocks wider than 64)
        go through bigblock.py."""
        if self._pmax is None:
            self._pmax = self.K.pencil_max_dim()
        return dmax > self._pmax or q > 64

    def _ldr(self):
        return self.ldp  # all state buffers share the padded row stride (complex: in complex elements)

    def _c0r(self, c):
        return c

    def _check_max_iter(self):
        if self.it >= self.opts.max_iter:
            self.done = True

    def finish(self, gather=None):
        """Final extraction (ppcg.py:760-787) and the host report.  Row partition: each rank
        downloads its own rows of the Ritz vectors and the (n, k) array is assembled on the
        host (dist_ppcg_solve's ``gather``), never on a device."""
        K, torch = self.K, self.torch
        wall = (time.perf_counter() - self.t0) * 1e3
        k = self.k
        src, dst = self._ritz(fresh=False)
        V, AV = self.XF[dst][:, :k], self.AXF[dst][:, :k]
        K.rr_residual(V, AV, self.omega, None, None, self.colnorm2)
        self._red(self.colnorm2)
        self.rr_count += 1
        self._fetch((self.omega, self.h_omega), (self.colnorm2, self.h_colnorm2))
        values = self.h_omega.numpy()[:k].copy()
        rn = np.sqrt(self.h_colnorm2.numpy()[:k]).tolist()
        pre = getattr(self, "_vec_job", None)
        self._vec_job = None
        buf = pre.result() if pre is not None else None
        if isinstance(buf, list):  # pool entry: the lease passes to the array (all its views hold arr.base)
            import weakref

            vectors = K.to_host_pinned(V, buf[0])
            buf[1] = weakref.ref(vectors.base)
        else:
            vectors = K.to_host(V, out=buf)
        extra = {}
        if self.comm is not None:
            if gather is None:
                gather = "all" if self.n * k * V.element_size() <= 8 << 30 else "root"
            full = self.comm.gather_rows_host(vectors, self.bounds, mode=gather)
            if full is not None:
                vectors = full
            else:
                extra["vector_rows"] = (self.plan.lo, self.plan.hi)
        self.xi = dst
        inc = [b.iteration for a_, b in zip(self.trace, self.trace[1:]) if b.trace_value > a_.trace_value]
        return SolveReport(values=values, vectors=vectors, trace=self.trace, status=self.status,
                           iterations=self.iterations, matvecs=self.matvecs, rr_count=self.rr_count,
                           breakdown_recoveries=self.recoveries, wall_ms=wall,
                           values_history=self.values_history,
                           diagnostics={"orth_loss": self.orth_loss, "proj_defect": self.proj_defect,
                                        "final_residual_norms": rn, "cache_refreshes": self.refreshes,
                                        "trace_increases": inc, **extra})


def device_bytes_plan(n_loc, n_ext, kt, q, cplx, nnz_loc=0, size=1):
    """Device bytes one rank of PPCGSolver allocates (``_alloc``), by buffer family, plus the
    largest transient scratch of an iteration: the budget check that config 5 (complex,
    128^3, k_total 4178) fits 8 B200s.  n_loc rows owned, n_ext = owned + ghost rows."""
    s = 16 if cplx else 8
    ldp = (kt + 15) // 16 * 16
    nb = -(-kt // q)
    nb = -(-nb // size) * size if size > 1 else nb
    dmax = 3 * q
    out = {
        # XF x2, W, P carry the ghost rows (operator inputs); AXF x2, AW, AP own rows only
        "state_blocks": 4 * n_ext * ldp * s + 4 * n_loc * ldp * s,
        "square_grams": 10 * kt * ldp * s + kt * kt * s,          # Gm .. Cm, eye
        "pencil_buffers": nb * dmax * dmax * s * 2 + nb * dmax * q * s
                          + ((nb * 4 * dmax * dmax * 8 * 2 + nb * 4 * dmax * q * 8) if cplx else 0),
        "operator": nnz_loc * (s + 4) + (n_loc + 1) * 4 + n_loc * 58 * 8 + n_loc * 8,
    }
    try:
        from . import _lib

        lib = _lib.load(require_cuda=False)
        r = 2 * kt if cplx else kt
        gram_ws = int(lib.bk_gram_ws_bytes(n_ext, r, r))
        sb_ws = int(lib.bk_subblock_grams_ws_bytes(n_ext, 2 * kt if cplx else kt, 2 * q if cplx else q, 1))
        # emulated FP64 products (csrc/ozaki.cu): digits + split-K partials, capped per call
        oz = int(lib.bk_ozaki_gram_ws_bytes(n_ext, r, r, 0, 0)) + int(lib.bk_ozaki_tsgemm_ws_bytes(4, n_loc, r, r, r))
    except Exception:  # library not built: the measured sizes at config 5 (~0.6 / 0.2 / 4.6 GB)
        gram_ws, sb_ws, oz = 6 << 27, 2 << 27, 37 << 27
    dig = n_ext * ldp * s  # column digits of [X_lock X] kept between Grams (PPCGSolver._slice_x)
    out["digit_cache"] = dig if dig <= _DIGIT_CACHE_MAX and _DIGIT_CACHE else 0
    out["workspaces"] = 3 * gram_ws + sb_ws  # main / side / rr families
    # main and side-stream emulated Grams + the tall GEMM (small products keep the DMMA kernels)
    out["fp64_emulation_workspaces"] = 2 * oz
    # transients: the complex Gram's real (2k x 2k) product, cuSOLVER's k_total eigensolver
    out["transient"] = ((2 * kt) ** 2 * 8 if cplx else 0) + 2 * (kt * kt + 64 * kt) * s
    out["total"] = sum(out.values())
    return out


def torch_empty_like_rows(base, rows, cols):
    """Contiguous (rows, cols) receive buffer of base's dtype and device (packed halo)."""
    import torch

    return torch.empty((rows, cols), dtype=base.dtype, device=base.device)


def _stencil_plane(csr):
    """Rows per grid plane when the CSR is a nearest-neighbour stencil (spmm_plan.infer_grid)."""
    import torch

    from .spmm_plan import infer_grid

    g = infer_grid(torch.from_numpy(csr.indptr.astype(np.int64)), torch.from_numpy(csr.indices.astype(np.int64)),
                   csr.shape[0])
    return None if g is None else g[0][1] * g[0][2]


def ppcg_solve(a, t=None, x0=None, opts=None, threads=1):
    """Lowest eigenpairs of a Hermitian operator with PPCG on the GPU.

    Same contract as blockeig.ppcg.ppcg_solve (ppcg.py:587-614); ``threads`` is accepted
    for API compatibility and has no effect (results are identical for any value).
    """
    if opts is None:
        raise ValueError("opts is required")
    opts.validate()
    s = PPCGSolver(a, t, x0, opts).start()
    while not s.step():
        pass
    return s.finish()
