"""CPU oracle for the PPCG hot path: a numpy restatement of the reference algorithm.

TEST INFRASTRUCTURE ONLY.  This module is the checker, never the product: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The product package never imports it and has no CPU
fallback.

It restates, in its own structure, the arithmetic of the reference package ``blockeig``
(``/root/reference/pkg/src/blockeig``; cited below as ``ppcg.py:L``, ``core.py:L``,
``rayleigh_ritz.py:L``).  Every floating-point operation is the same numpy/LAPACK call in
the same order as the reference, so on one machine it reproduces the reference's results
to the last bit; ``tests/test_oracle_golden.py`` pins it against golden vectors produced
by the reference itself (``tests/golden/make_golden.py``).

The solver is written as a stepper (``OracleRun.start`` / ``step`` / ``finish``) so that a
single outer iteration can be timed on its own (bench.py's CPU baseline).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

try:  # BLAS thread pinning, as the reference does (ppcg.py:610-613)
    from threadpoolctl import threadpool_limits
except Exception:  # pragma: no cover
    threadpool_limits = None


# --- thresholds (ppcg.py:39-45, core.py:64, core.py:175, rayleigh_ritz.py:22, problems.py:276)
CX_RANK_FLOOR = 1e-14
COEFF_REFRESH = 100.0
BREAKDOWN_MAX = 1e8   # ppcg.py:705
DIRECTION_FLOOR = 1e-14
PIVOT_FLOOR = 1e-14
GRAM_RTOL = 1e-12
DEN_FLOOR = 1e-300
TAYLOR_OK = 0.1


class OracleSingularGram(Exception):
    """Mirror of blockeig.errors.SingularGramError (errors.py:31-32)."""


class OracleRankDeficiency(Exception):
    """Mirror of blockeig.errors.RankDeficiencyError (errors.py:12-20)."""

    def __init__(self, column):
        self.column = column
        super().__init__(f"rank deficiency detected at column {column}")


# ----------------------------------------------------------------------------- dense kernels
def herm_gram(x, y):
    """X^H Y (core.py:43-49)."""
    return x.conj().T @ y


def chol_upper_with_floor(g):
    """Column-by-column upper Cholesky with the relative pivot floor (core.py:67-83)."""
    m = g.shape[0]
    r = np.zeros_like(g)
    ref = max(float(np.max(np.abs(np.diag(g)).real)), 1e-300)
    for j in range(m):
        piv = g[j, j].real - np.sum(np.abs(r[:j, j]) ** 2)
        if piv <= PIVOT_FLOOR * ref or not np.isfinite(piv):
            raise OracleRankDeficiency(j)
        r[j, j] = np.sqrt(piv)
        if j + 1 < m:
            r[j, j + 1:] = (g[j, j + 1:] - r[:j, j].conj() @ r[:j, j + 1:]) / r[j, j]
    return r


def right_solve_upper(r, b):
    """B R^{-1} through the transposed lower solve (core.py:99, ppcg.py:484)."""
    return sla.solve_triangular(r.T, b.T, lower=True).T


def cholqr(x, gram=None):
    """Cholesky QR (core.py:86-100)."""
    if gram is None:
        gram = herm_gram(x, x)
    r = chol_upper_with_floor(gram)
    return right_solve_upper(r, x), r


def taylor_poly(gram, terms):
    """Horner evaluation of the (1+Y)^{-1/2} series, Y = G - I (core.py:106-124)."""
    m = gram.shape[0]
    eye = np.eye(m, dtype=gram.dtype)
    y = gram - eye
    cf = [1.0]
    for i in range(1, terms + 1):
        cf.append(-cf[-1] * (2 * i - 1) / (2 * i))
    acc = cf[-1] * eye
    for c in reversed(cf[:-1]):
        acc = c * eye + y @ acc
    return acc


def solve_small_pencil(a_hat, b_hat, want):
    """Symmetrise, singular-Gram test, dense generalized eigensolve (core.py:143-202).

    Returns (omega[:want], C[:, :want]).
    """
    a = np.atleast_2d(np.asarray(a_hat))
    b = np.atleast_2d(np.asarray(b_hat))
    a = 0.5 * (a + a.conj().T)
    b = 0.5 * (b + b.conj().T)
    d = a.shape[0]
    if not 1 <= want <= d:
        raise ValueError(f"want must be in [1, {d}], got {want}")
    bn = np.linalg.norm(b, "fro")
    flo = GRAM_RTOL * max(bn, 1e-300)
    try:
        np.linalg.cholesky(b - flo * np.eye(d))
    except np.linalg.LinAlgError:
        raise OracleSingularGram("singular Gram") from None
    try:
        om, c = sla.eigh(a, b)
    except sla.LinAlgError:
        raise OracleSingularGram("not positive definite") from None
    return om[:want], c[:, :want]


# ----------------------------------------------------------------------------- subblock update
@dataclass
class BlockStep:
    """Per-subblock outcome (ppcg.py:166-186)."""

    x: np.ndarray
    p: np.ndarray
    theta: np.ndarray
    c_x: np.ndarray
    c_w: np.ndarray
    c_p: np.ndarray
    used_fallback: bool = False
    zero_residual: bool = False
    coeff_scale: float = 1.0


def _colnorms(b):
    return np.linalg.norm(b, axis=0)


def _kept(b, scale):
    """Columns above the direction floor (ppcg.py:198-203)."""
    if b is None or b.shape[1] == 0:
        return np.array([], dtype=int)
    return np.nonzero(_colnorms(b) > DIRECTION_FLOOR * scale)[0]


def _rq(x, ax):
    """Per-column Rayleigh quotients (ppcg.py:214-217)."""
    return np.real(np.sum(x.conj() * ax, axis=0)) / np.real(np.sum(x.conj() * x, axis=0))


def _normalised(b, idx):
    """Kept columns at unit norm, and their norms (ppcg.py:220-228)."""
    cols = b[:, idx]
    nrm = _colnorms(cols)
    return cols / nrm[None, :], nrm


def _pencil_over(parts, aparts, want):
    """[X|W|P] pencil (ppcg.py:206-211)."""
    s = np.concatenate(parts, axis=1)
    as_ = np.concatenate(aparts, axis=1)
    return solve_small_pencil(herm_gram(s, as_), herm_gram(s, s), want)


def _passthrough(x, ax, w, p, fallback, zero):
    q = x.shape[1]
    return BlockStep(
        x=x.copy(), p=np.zeros_like(x), theta=_rq(x, ax), c_x=np.eye(q, dtype=x.dtype),
        c_w=np.zeros((0 if w is None else w.shape[1], q), dtype=x.dtype),
        c_p=np.zeros((0 if p is None else p.shape[1], q), dtype=x.dtype),
        used_fallback=fallback, zero_residual=zero)


def steepest_fallback(x, w, ax, aw):
    """Pencil over [X, W] only (ppcg.py:231-275)."""
    q = x.shape[1]
    scale = max(np.max(_colnorms(x)), 1e-300)
    kw = _kept(w, scale)
    if kw.size == 0:
        res = _passthrough(x, ax, w, None, True, True)
        res.c_p = np.zeros((0, q), dtype=x.dtype)
        return res
    wu, wn = _normalised(w, kw)
    om, c = _pencil_over([x, wu], [ax, aw[:, kw] / wn[None, :]], q)
    cw = np.zeros((w.shape[1], q), dtype=c.dtype)
    cw[kw] = c[q:] / wn[:, None]
    pn = w @ cw
    return BlockStep(x=x @ c[:q] + pn, p=pn, theta=om, c_x=c[:q], c_w=cw,
                     c_p=np.zeros((0, q), dtype=c.dtype), used_fallback=True,
                     coeff_scale=float(np.max(np.abs(c))))


def subblock_update(x, w, p, ax, aw, ap):
    """One subblock of the PPCG update (ppcg.py:278-378)."""
    q = x.shape[1]
    scale = max(np.max(_colnorms(x)), 1e-300)
    kw = _kept(w, scale)
    kp = _kept(p, scale)
    if kw.size == 0 and kp.size == 0:
        return _passthrough(x, ax, w, p, False, kw.size == 0)

    def attempt(iw, ip):
        parts, aparts, wn, pn = [x], [ax], np.zeros(0), np.zeros(0)
        if iw.size:
            wu, wn = _normalised(w, iw)
            parts.append(wu)
            aparts.append(aw[:, iw] / wn[None, :])
        if ip.size:
            pu, pn = _normalised(p, ip)
            parts.append(pu)
            aparts.append(ap[:, ip] / pn[None, :])
        return _pencil_over(parts, aparts, q), wn, pn

    kp_used = kp
    try:
        (om, c), wn, pn = attempt(kw, kp_used)
    except OracleSingularGram:
        kp_used = np.array([], dtype=int)
        trial = kw.copy()
        while True:
            try:
                (om, c), wn, pn = attempt(trial, kp_used)
                break
            except OracleSingularGram:
                if trial.size == 0:
                    raise
                trial = np.delete(trial, int(np.argmin(_colnorms(w[:, trial]))))
        kw = trial

    nw = kw.size
    cx = c[:q]
    smin = np.linalg.svd(cx, compute_uv=False)[-1]
    if smin < CX_RANK_FLOOR * max(np.linalg.norm(c, 2), 1.0):
        return steepest_fallback(x, w, ax, aw)
    cw = np.zeros((0 if w is None else w.shape[1], q), dtype=c.dtype)
    if nw:
        cw[kw] = c[q:q + nw] / wn[:, None]
    cp = np.zeros((0 if p is None else p.shape[1], q), dtype=c.dtype)
    if kp_used.size:
        cp[kp_used] = c[q + nw:] / pn[:, None]
    pnew = np.zeros((x.shape[0], q), dtype=np.result_type(x.dtype, c.dtype))
    if nw:
        pnew = w @ cw
    if kp_used.size:
        pnew = pnew + p @ cp
    return BlockStep(x=x @ cx + pnew, p=pnew, theta=om, c_x=cx, c_w=cw, c_p=cp,
                     coeff_scale=float(np.max(np.abs(c))))


def partition(k_act, q):
    """Contiguous column spans (ppcg.py:189-195)."""
    if k_act < 0 or q < 1:
        raise ValueError("bad partition arguments")
    return [(lo, min(lo + q, k_act)) for lo in range(0, k_act, q)]


# ----------------------------------------------------------------------------- metrics
def stop_metrics(x, ax, prev):
    """(rel_subspace_residual, trace, rel_trace_change) (rayleigh_ritz.py:71-92)."""
    g = herm_gram(x, ax)
    r = ax - x @ g
    rel = np.linalg.norm(r, "fro") / max(np.linalg.norm(g, "fro"), DEN_FLOOR)
    tr = float(np.trace(g).real)
    chg = math.inf if prev is None else abs(tr - prev) / max(abs(tr), DEN_FLOOR)
    return float(rel), tr, float(chg)


def leading_lock_count(values, rnorms, tol):
    """Prefix-closed convergence (rayleigh_ritz.py:95-108)."""
    n = 0
    for th, rn in zip(values, rnorms):
        if rn <= tol * max(abs(th), 1.0):
            n += 1
        else:
            break
    return n


# ----------------------------------------------------------------------------- the solver
@dataclass
class OracleTraceRow:
    iteration: int
    trace_value: float
    rel_resid: float
    n_locked: int
    n_matvec: int
    wall_ms: float


@dataclass
class OracleReport:
    values: np.ndarray
    vectors: np.ndarray
    trace: list
    status: str
    iterations: int
    matvecs: int
    rr_count: int
    breakdown_recoveries: int
    wall_ms: float
    values_history: list = field(default_factory=list)
    diagnostics: dict = field(default_factory=dict)


class OracleRun:
    """Step-wise restatement of ppcg_solve/_ppcg_solve (ppcg.py:587-787).

    ``op`` needs ``n``, ``dtype`` and ``apply(block)``; ``prec`` is None or has
    ``apply``.  ``opts`` is any object with the SolverOptions fields (ppcg.py:48-81).
    """

    def __init__(self, op, prec=None, x0=None, opts=None, blas_threads=1):
        if opts is None:
            raise ValueError("opts is required")
        self.op, self.prec, self.opts = op, prec, opts
        self.x0 = x0
        self.blas_threads = blas_threads
        self.matvecs = 0

    # operator counting (operators.py:113-124)
    def _A(self, b):
        self.matvecs += np.asarray(b).shape[1]
        return self.op.apply(b)

    def _limit(self):
        if threadpool_limits is None or self.blas_threads is None:
            import contextlib
            return contextlib.nullcontext()
        return threadpool_limits(limits=self.blas_threads)

    # -- initial block (ppcg.py:414-438)
    def _x_init(self, kt):
        n = self.op.n
        cplx = np.issubdtype(np.dtype(self.op.dtype), np.complexfloating)
        dt = np.complex128 if cplx else np.float64
        g = np.random.default_rng(self.opts.seed)

        def draw(c):
            blk = g.standard_normal((n, c))
            if cplx:
                blk = blk + 1j * g.standard_normal((n, c))
            return blk

        if self.x0 is None:
            x = draw(kt).astype(dt)
        else:
            x0 = np.asarray(self.x0, dtype=dt)
            if x0.ndim != 2 or x0.shape[0] != n:
                raise ValueError(f"x0 must be {n} x m, got {x0.shape}")
            if x0.shape[1] > kt:
                raise ValueError("x0 too wide")
            pad = kt - x0.shape[1]
            x = np.column_stack([x0, draw(pad).astype(dt)]) if pad else x0.copy()
        return cholqr(x)[0]

    def start(self):
        o = self.opts
        with self._limit():
            self.k = o.k
            nbuf = o.nbuf if o.nbuf is not None else math.ceil(0.02 * o.k)
            self.kt = o.k + nbuf
            if self.kt > self.op.n:
                raise ValueError("k + nbuf exceeds operator dimension")
            self.t0 = time.perf_counter()
            x = self._x_init(self.kt)
            ax = self._A(x)
            empty = np.zeros((self.op.n, 0), dtype=x.dtype)
            self.x, self.ax = x, ax
            self.w = ax - x @ herm_gram(x, ax)
            self.p = self.ap = self.aw = None
            self.xl, self.axl = empty, empty
            self.vals_lock = np.zeros(0)
            self.spans = partition(self.kt, o.sbsize)
            self.trace, self.values_history = [], []
            self.orth_loss, self.proj_defect = [], []
            self.rr_count = self.recoveries = self.refreshes = 0
            self.prev_trace = None
            self.status, self.iterations = "max_iter", o.max_iter
            self.it = 0
            self.done = o.max_iter == 0
        return self

    @property
    def n_locked(self):
        return self.xl.shape[1]

    def _lead(self):
        """Leading k columns of [X_lock, X] (ppcg.py:536-544)."""
        L = self.n_locked
        if L >= self.k:
            return self.xl[:, :self.k], self.axl[:, :self.k]
        need = self.k - L
        return (np.concatenate([self.xl, self.x[:, :need]], axis=1),
                np.concatenate([self.axl, self.ax[:, :need]], axis=1))

    def _project(self, basis, abasis, blk, ablk):
        """ppcg.py:441-445."""
        g = herm_gram(basis, blk)
        blk -= basis @ g
        if ablk is not None:
            ablk -= abasis @ g

    def _gram_full(self):
        """Orthonormality loss and the active Gram (ppcg.py:448-453)."""
        s = np.concatenate([self.xl, self.x], axis=1)
        g = herm_gram(s, s)
        return float(np.linalg.norm(g - np.eye(s.shape[1]), "fro")), g[self.n_locked:, self.n_locked:]

    def _subblocks(self):
        """ppcg.py:487-533 (single-threaded; the reference is result-invariant in threads)."""
        n, m = self.x.shape
        xn = np.empty((n, m), dtype=self.x.dtype)
        pn, axn, apn = np.empty_like(xn), np.empty_like(xn), np.empty_like(xn)
        nfb, cs = 0, 1.0
        for lo, hi in self.spans:
            pj = self.p[:, lo:hi] if self.p is not None else None
            apj = self.ap[:, lo:hi] if self.ap is not None else None
            r = subblock_update(self.x[:, lo:hi], self.w[:, lo:hi], pj,
                                self.ax[:, lo:hi], self.aw[:, lo:hi], apj)
            xn[:, lo:hi] = r.x
            pn[:, lo:hi] = r.p
            aps = np.zeros_like(r.p)
            if r.c_w.shape[0]:
                aps += self.aw[:, lo:hi] @ r.c_w
            if r.c_p.shape[0] and self.ap is not None:
                aps += self.ap[:, lo:hi] @ r.c_p
            apn[:, lo:hi] = aps
            axn[:, lo:hi] = self.ax[:, lo:hi] @ r.c_x + aps
            nfb += int(r.used_fallback)
            cs = max(cs, r.coeff_scale)
        return xn, pn, axn, apn, nfb, cs

    def _orth(self, gram, loss):
        """ppcg.py:475-484."""
        if self.opts.orth_scheme == "taylor-polar" and loss <= TAYLOR_OK:
            poly = taylor_poly(gram, self.opts.taylor_terms)
            self.x = self.x @ poly
            self.ax = self.ax @ poly
            return
        q, r = cholqr(self.x, gram=gram)
        self.x = q
        self.ax = right_solve_upper(r, self.ax)

    def _redo_without_p(self, prev, col):
        """ppcg.py:456-472."""
        x0, w0, p0, ax0, aw0, ap0 = prev
        for lo, hi in self.spans:
            if lo <= col < hi:
                r = steepest_fallback(x0[:, lo:hi], w0[:, lo:hi], ax0[:, lo:hi], aw0[:, lo:hi])
                self.x[:, lo:hi] = r.x
                self.p[:, lo:hi] = r.p
                aps = np.zeros_like(r.p)
                if r.c_w.shape[0]:
                    aps += aw0[:, lo:hi] @ r.c_w
                self.ap[:, lo:hi] = aps
                self.ax[:, lo:hi] = ax0[:, lo:hi] @ r.c_x + aps
                return
        raise OracleRankDeficiency(col)

    def _ritz(self, fresh):
        """ppcg.py:553-584."""
        s = np.concatenate([self.xl, self.x], axis=1)
        as_ = np.concatenate([self.axl, self.ax], axis=1)
        kt = s.shape[1]
        try:
            om, c = solve_small_pencil(herm_gram(s, as_), herm_gram(s, s), kt)
        except OracleSingularGram:
            try:
                q, r = cholqr(self.x)
                self.ax = right_solve_upper(r, self.ax)
            except OracleRankDeficiency:
                q = np.linalg.qr(self.x)[0]
                self.ax = self._A(q)
            self.x = q
            s = np.concatenate([self.xl, self.x], axis=1)
            as_ = np.concatenate([self.axl, self.ax], axis=1)
            om, c = solve_small_pencil(herm_gram(s, as_), herm_gram(s, s), kt)
        vecs = s @ c
        axf = self._A(vecs) if fresh else as_ @ c
        res = axf - vecs * om[None, :]
        return om, vecs, _colnorms(res), axf, res

    def _lock(self, om, vecs, rn, res):
        """ppcg.py:381-411."""
        L_old = self.n_locked
        kt = vecs.shape[1]
        L = leading_lock_count(om, rn, self.opts.tol)
        self.xl = vecs[:, :L]
        self.vals_lock = om[:L]
        self.x = vecs[:, L:]
        self.w = res[:, L:]
        if self.p is not None:
            ka = kt - L
            pn = np.zeros((self.p.shape[0], ka), dtype=self.p.dtype)
            apn = np.zeros_like(pn) if self.ap is not None else None
            for g in range(max(L_old, L), kt):
                pn[:, g - L] = self.p[:, g - L_old]
                if apn is not None:
                    apn[:, g - L] = self.ap[:, g - L_old]
            self.p, self.ap = pn, apn
        self.spans = partition(self.x.shape[1], self.opts.sbsize)
        return L

    def step(self):
        """One outer iteration (ppcg.py:653-758).  Returns True when the run has stopped."""
        if self.done:
            return True
        o = self.opts
        with self._limit():
            it = self.it + 1
            self.it = it
            xl, axl = self._lead()
            rel, tr, chg = stop_metrics(xl, axl, self.prev_trace)
            self.prev_trace = tr
            stop = rel <= o.tol or (o.trace_tol is not None and chg <= o.trace_tol)
            if stop or self.x.shape[1] == 0:
                self.status, self.iterations, self.done = "converged", it - 1, True
                return True
            self.trace.append(OracleTraceRow(it, tr, rel, self.n_locked, self.matvecs,
                                             (time.perf_counter() - self.t0) * 1e3))
            if self.prec is not None:
                self.w = self.prec.apply(self.w)
            self.aw = self._A(self.w)
            if o.project_w:
                self._project(self.x, self.ax, self.w, self.aw)
                if self.n_locked:
                    self._project(self.xl, self.axl, self.w, self.aw)
            if self.p is not None and o.project_p:
                self._project(self.x, self.ax, self.p, self.ap)
                if self.n_locked:
                    self._project(self.xl, self.axl, self.p, self.ap)
            basis = np.concatenate([self.xl, self.x], axis=1)
            wn = np.linalg.norm(self.w)
            self.proj_defect.append(float(np.linalg.norm(herm_gram(basis, self.w)) / max(wn, 1e-300)))

            prev = (self.x, self.w, self.p, self.ax, self.aw, self.ap)
            self.x, self.p, self.ax, self.ap, nfb, cs = self._subblocks()
            self.recoveries += nfb
            broken = not all(np.isfinite(b).all() for b in (self.x, self.p, self.ax, self.ap))
            if not broken:
                broken = max(float(np.max(np.abs(self.x))), float(np.max(np.abs(self.p)))) > BREAKDOWN_MAX
            if broken:
                self.recoveries += 1
                self.orth_loss.append(math.inf)
                self.x = np.linalg.qr(prev[0])[0]
                self.ax = self._A(self.x)
                self.p = self.ap = None
                self.w = self.ax - self.x @ herm_gram(self.x, self.ax)
                self._check_max_iter()
                return self.done
            if cs > COEFF_REFRESH:
                self.refreshes += 1
                self.ax = self._A(self.x)
                self.ap = self._A(self.p)
            loss, gact = self._gram_full()
            self.orth_loss.append(loss)
            if math.isfinite(o.rr_period) and it % int(o.rr_period) == 0:
                om, vecs, rn, axf, res = self._ritz(True)
                self.rr_count += 1
                self.values_history.append(om.copy())
                L = self._lock(om, vecs, rn, res)
                self.axl, self.ax = axf[:, :L], axf[:, L:]
            else:
                do = (o.orth_policy == "every"
                      or (o.orth_policy == "periodic" and it % o.orth_period == 0)
                      or (o.orth_policy == "adaptive" and loss >= o.orth_threshold))
                if do:
                    try:
                        self._orth(gact, loss)
                    except OracleRankDeficiency as err:
                        self.recoveries += 1
                        self._redo_without_p(prev, err.column)
                        try:
                            _, gact = self._gram_full()
                            self._orth(gact, loss)
                        except OracleRankDeficiency:
                            self.x = np.linalg.qr(self.x)[0]
                            self.ax = self._A(self.x)
                self.w = self.ax - self.x @ herm_gram(self.x, self.ax)
            self._check_max_iter()
        return self.done

    def _check_max_iter(self):
        if self.it >= self.opts.max_iter:
            self.done = True

    def finish(self):
        """Final extraction and report (ppcg.py:760-787)."""
        with self._limit():
            wall = (time.perf_counter() - self.t0) * 1e3
            om, vecs, rn, _, _ = self._ritz(False)
            self.rr_count += 1
        inc = [b.iteration for a, b in zip(self.trace, self.trace[1:]) if b.trace_value > a.trace_value]
        k = self.k
        return OracleReport(
            values=om[:k], vectors=vecs[:, :k], trace=self.trace, status=self.status,
            iterations=self.iterations, matvecs=self.matvecs, rr_count=self.rr_count,
            breakdown_recoveries=self.recoveries, wall_ms=wall, values_history=self.values_history,
            diagnostics={"orth_loss": self.orth_loss, "proj_defect": self.proj_defect,
                         "final_residual_norms": rn[:k].tolist(), "cache_refreshes": self.refreshes,
                         "trace_increases": inc})


def oracle_solve(op, prec=None, x0=None, opts=None, blas_threads=1):
    """Run the oracle to completion (ppcg_solve, ppcg.py:587-614)."""
    if opts is None:
        raise ValueError("opts is required")
    run = OracleRun(op, prec, x0, opts, blas_threads).start()
    while not run.step():
        pass
    return run.finish()
