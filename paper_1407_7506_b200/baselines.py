"""LOBPCG and Davidson-Liu baselines on the same device kernels as the PPCG solver.

Drop-in for ``blockeig.baselines`` (baselines.py:1-315): same ``BaselineOptions`` (fields,
defaults, validation), ``lobpcg_solve`` / ``davidson_solve`` signatures and ``SolveReport``
layout, so head-to-head runs like the paper's Table 4 compare algorithms on identical
kernels.

* LOBPCG (baselines.py:198-315): per iteration the Ritz residual W = T(AX - X Theta), AW = A W,
  projections of W and P against X then X_lock, one block_update over the whole active
  block (batched device pencil when 3 k_act <= 192, else bigblock.py), prefix locking by
  the reference's residual test.  Built on PPCGSolver's buffers: the whole-block update
  is PPCG with sbsize = k_act and a Rayleigh-Ritz every iteration.
* Davidson (baselines.py:78-195): trial basis accumulated in one n x cap device buffer with
  its A-products, projected pencil blocks grown in place, two-pass projection +
  norm filter + Cholesky-QR with column deletion for new directions, thick restart at
  ``restart_dim_multiple * k_total`` columns, dense pencil by cuSOLVER sygvd.
Both run on one GPU.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .errors import DimensionError, RankDeficiencyError, SingularGramError
from .ppcg import PPCGSolver, SolveReport, SolverOptions, initial_block_source, lock_count
from .trace import TraceRecord

__all__ = ["BaselineOptions", "lobpcg_solve", "davidson_solve", "LOBPCGSolver"]


@dataclass
class BaselineOptions:
    """Tunables shared by the baseline solvers (baselines.py:25-54)."""

    k: int
    nbuf: int | None = None
    tol: float = 1e-6
    max_iter: int = 500
    seed: int = 0
    restart_dim_multiple: int = 2

    def resolved_nbuf(self):
        if self.nbuf is not None:
            return self.nbuf
        return math.ceil(0.02 * self.k)

    def validate(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.nbuf is not None and self.nbuf < 0:
            raise ValueError("nbuf must be >= 0")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iter < 0:
            raise ValueError("max_iter must be >= 0")
        if self.restart_dim_multiple < 2:
            raise ValueError("restart_dim_multiple must be >= 2")


def _solver_options(opts):
    kt = opts.k + opts.resolved_nbuf()
    return SolverOptions(k=opts.k, nbuf=opts.resolved_nbuf(), sbsize=max(kt, 1), rr_period=math.inf, tol=opts.tol,
                         max_iter=opts.max_iter, seed=opts.seed)


# ----------------------------------------------------------------------------- LOBPCG
class LOBPCGSolver(PPCGSolver):
    """Step-wise device LOBPCG (baselines.py:198-315)."""

    def __init__(self, a, t=None, x0=None, opts=None, comm=None):
        if opts is None:
            raise ValueError("opts is required")
        opts.validate()
        self.bopts = opts
        super().__init__(a, t, x0, _solver_options(opts), comm)

    def start(self):
        # X0 = cholesky_qr(draw), AX = A X, first W = T(AX - X (X^H AX)) with the leading-k
        # metric cached (baselines.py:211-246; same _initial_block as PPCG)
        super().start()
        self.values_lock = np.zeros(0)
        self.have_theta = False
        return self

    def step(self):
        if self.done:
            return True
        K = self.K
        it = self.it = self.it + 1
        rel, tr = self._metrics()
        self.prev_trace = tr
        L, kt = self.L, self.kt
        ka = kt - L
        if rel <= self.opts.tol or ka == 0:
            self.status, self.iterations, self.done = "converged", it - 1, True
            return True
        self.trace.append(TraceRecord(iteration=it, trace_value=tr, rel_resid=rel, n_locked=L, n_matvec=self.matvecs,
                                      wall_ms=(time.perf_counter() - self.t0) * 1e3))
        w, aw = self.W[:, L:], self.AW[:, L:]
        self._project(L, ka, w, aw)         # AW = A W + projections, baselines.py:259-268
        src, dst = self.xi, 1 - self.xi
        psrc = pdst = self.pi  # P, AP in place
        self._subblock_update(ka, ka, src, psrc, dst, pdst)   # whole-block block_update
        self._fetch((self.info, self.h_info))
        info = self.h_info.numpy()[:4]
        if info[2] != 0:
            raise SingularGramError("Gram matrix numerically singular in the LOBPCG pencil")
        self.recoveries += int(info[0])
        self.xi, self.pi = dst, pdst
        self.has_p = True
        self.have_theta = True
        # Ritz residual R = AX - X Theta: norms for locking, and next W = T(R)
        x, ax = self.X(), self.AX()
        K.rr_residual(x, ax, self.theta[:ka], self.rowscale, self.W[:, L:], self.colnorm2[:ka])
        self._red(self.colnorm2)
        self._fetch((self.theta, self.h_omega), (self.colnorm2, self.h_colnorm2))
        theta = self.h_omega.numpy()[:ka].copy()
        self.rr_count += 1
        self.values_history.append(np.concatenate([self.values_lock, theta]))
        newly = lock_count(theta, np.sqrt(np.maximum(self.h_colnorm2.numpy()[:ka], 0.0)), self.opts.tol)
        if newly:
            self.values_lock = np.concatenate([self.values_lock, theta[:newly]])
            self.L = L + newly
            self.theta[: ka - newly].copy_(self.theta[newly:ka].clone())
        self.metric_cached = False
        self._check_max_iter()
        return self.done

    def finish(self):
        K = self.K
        wall = (time.perf_counter() - self.t0) * 1e3
        k = self.k
        if not self.have_theta:
            # converged before the first update: extract once (baselines.py:296-301)
            src, dst = self._ritz(fresh=False)
            self.xi = dst
            self._fetch((self.omega, self.h_omega))
            values = self.h_omega.numpy()[:self.kt].copy()
            self.rr_count += 1
        else:
            ka = self.kt - self.L
            self._fetch((self.theta, self.h_omega))
            values = np.concatenate([self.values_lock, self.h_omega.numpy()[:ka]])
        vals = self.torch.from_numpy(np.ascontiguousarray(values[:k])).cuda()
        V, AV = self.XF[self.xi][:, :k], self.AXF[self.xi][:, :k]
        K.rr_residual(V, AV, vals, None, None, self.colnorm2)
        self._red(self.colnorm2)
        self._fetch((self.colnorm2, self.h_colnorm2))
        rn = np.sqrt(np.maximum(self.h_colnorm2.numpy()[:k], 0.0)).tolist()
        if self.comm is not None:
            V = self.comm.allgather_rows(V.contiguous(), self.bounds)
        vectors = K.to_host(V)
        return SolveReport(values=values[:k].copy(), vectors=vectors, trace=self.trace, status=self.status,
                           iterations=self.iterations, matvecs=self.matvecs, rr_count=self.rr_count,
                           breakdown_recoveries=self.recoveries, wall_ms=wall, values_history=self.values_history,
                           diagnostics={"final_residual_norms": rn})


def lobpcg_solve(a, t=None, x0=None, opts=None, threads=1):
    """Locally optimal block preconditioned conjugate gradient on the device
    (baselines.py:198-210); ``threads`` is accepted for API compatibility."""
    if opts is None:
        raise ValueError("opts is required")
    opts.validate()
    s = LOBPCGSolver(a, t, x0, opts).start()
    while not s.step():
        pass
    return s.finish()


# ----------------------------------------------------------------------------- Davidson
def davidson_solve(a, t=None, x0=None, opts=None, threads=1):
    """Simplest Davidson-Liu iteration with thick restart on the device (baselines.py:78-89)."""
    if opts is None:
        raise ValueError("opts is required")
    opts.validate()
    return _Davidson(a, t, x0, opts).run()


class _Davidson:
    def __init__(self, a, t, x0, opts):
        import torch

        from . import _lib
        from . import kernels as K
        from .operators import as_device_operator, as_device_preconditioner

        _lib.load()
        self.torch, self.K = torch, K
        self.opts = opts
        self.n = int(a.n)
        self.dev_a = as_device_operator(a)
        self.prec = as_device_preconditioner(t)
        self.cplx = bool(np.issubdtype(np.dtype(a.dtype), np.complexfloating)) or self.dev_a.complex
        self.tdt = torch.complex128 if self.cplx else torch.float64
        self.k = opts.k
        self.kt = opts.k + opts.resolved_nbuf()
        if self.kt > self.n:
            raise DimensionError(f"k + nbuf = {self.kt} exceeds operator dimension {self.n}")
        self.x0 = x0
        self.matvecs = 0
        self.cap = opts.restart_dim_multiple * self.kt
        self.dense = K.dense_context()

    # helpers --------------------------------------------------------------
    def _A(self, x, y):
        self.matvecs += x.shape[1]
        if x.shape[1]:
            self.dev_a.apply_into(x, y)

    def _T(self, w):
        if self.prec is None:
            return
        if self.prec[0] == "diag":
            self.K.scale_rows(self.prec[1], w, w)
        else:
            tmp = self.torch.empty_like(w)
            self.prec[1].apply_into(w, tmp)
            w.copy_(tmp)

    def _gram(self, x, y):
        out = self.torch.empty((x.shape[1], y.shape[1]), dtype=self.tdt, device="cuda")
        self.K.gram(x, y, out)
        return out

    def _metrics(self, x, ax, prev):
        """convergence_metrics on the leading k columns (rayleigh_ritz.py:71-92)."""
        K, torch = self.K, self.torch
        k = self.k
        G = self._gram(x[:, :k], ax[:, :k])
        st = torch.zeros(4, dtype=torch.float64, device="cuda")
        K.small_stats(G, st[1:4])
        K.tsgemm([x[:, :k]], [G], [None], alpha=-1.0, beta=1.0, zs=[ax[:, :k]], metric=st[0:1], ksplit=k, nsplit=k)
        s = st.cpu().numpy()
        return math.sqrt(max(s[0], 0.0)) / max(math.sqrt(max(s[1], 0.0)), 1e-300), float(s[3])

    def _solve_pencil(self, ga, gb, want):
        """solve_pencil(SmallPencil(ga, gb), want) (core.py:175-202) via cuSOLVER sygvd."""
        torch = self.torch
        d = ga.shape[0]
        A, B = ga.clone(), gb.clone()
        om = torch.empty(d, dtype=torch.float64, device="cuda")
        C = torch.empty((d, d), dtype=self.tdt, device="cuda")
        st = torch.zeros(4, dtype=torch.int32, device="cuda")
        self.dense.rr_pencil(A, B, om, C, st)
        if int(st.cpu()[0]) != 0:
            raise SingularGramError("Gram matrix numerically singular in the Davidson pencil")
        return om[:want], C[:, :want]

    def _expand(self, nb, w):
        """_expand_orthonormal (baselines.py:56-70): two projection passes against the
        current basis, drop columns of norm <= 1e-12 max norm, Cholesky-QR with column
        deletion.  Returns the surviving (orthonormal) columns as a new tensor."""
        K, torch = self.K, self.torch
        basis = self.basis[:, :nb]
        for _ in range(2):
            g = self._gram(basis, w)
            K.tsgemm([basis], [g], [w], alpha=-1.0, beta=1.0, zs=[w])
        nrm = np.sqrt(np.maximum(np.real(torch.diagonal(self._gram(w, w)).cpu().numpy()), 0.0))
        keep = np.flatnonzero(nrm > 1e-12 * max(float(np.max(nrm)) if nrm.size else 0.0, 1e-300))
        w = w[:, torch.from_numpy(keep).cuda()] if keep.size < w.shape[1] else w
        fail = torch.full((1,), -1, dtype=torch.int32, device="cuda")
        while w.shape[1]:
            R = self._gram(w, w)
            self.dense.chol_upper_floor(R, fail)
            col = int(fail.cpu()[0])
            if col >= 0:
                idx = [i for i in range(w.shape[1]) if i != col]
                w = w[:, torch.tensor(idx, dtype=torch.long, device="cuda")].contiguous()
                continue
            self.dense.tri_inv_upper(R)
            q = torch.empty_like(w)
            K.tsgemm([w], [R], [q], upper=True)
            return q
        return w

    def run(self):
        K, torch = self.K, self.torch
        n, kt, k, opts = self.n, self.kt, self.k, self.opts
        t_start = time.perf_counter()
        z = lambda *s: torch.zeros(s, dtype=self.tdt, device="cuda")  # noqa: E731
        self.basis = z(n, self.cap)
        self.abasis = z(n, self.cap)
        # X0 = cholesky_qr(draw) (ppcg.py:414-438), AX = A X
        x = z(n, kt)
        K.from_host(initial_block_source(n, kt, self.cplx, opts.seed, self.x0), x)
        g = self._gram(x, x)
        fail = torch.full((1,), -1, dtype=torch.int32, device="cuda")
        self.dense.chol_upper_floor(g, fail)
        col = int(fail.cpu()[0])
        if col >= 0:
            raise RankDeficiencyError(col)
        self.dense.tri_inv_upper(g)
        xq = z(n, kt)
        K.tsgemm([x], [g], [xq], upper=True)
        x = xq
        ax = z(n, kt)
        self._A(x, ax)
        self.basis[:, :kt].copy_(x)
        self.abasis[:, :kt].copy_(ax)
        nb = kt
        ga = self._gram(self.basis[:, :nb], self.abasis[:, :nb])
        gb = self._gram(self.basis[:, :nb], self.basis[:, :nb])
        theta = None
        trace, values_history = [], []
        prev = None
        status, iterations = "max_iter", opts.max_iter
        n_locked = 0
        rr_count = 0
        colnorm2 = torch.zeros(kt, dtype=torch.float64, device="cuda")
        for it in range(1, opts.max_iter + 1):
            rel, tr = self._metrics(x, ax, prev)
            prev = tr
            if rel <= opts.tol or n_locked >= kt:
                status, iterations = "converged", it - 1
                break
            trace.append(TraceRecord(iteration=it, trace_value=tr, rel_resid=rel, n_locked=n_locked,
                                     n_matvec=self.matvecs, wall_ms=(time.perf_counter() - t_start) * 1e3))
            if theta is None:
                gx = self._gram(x, ax)
                w = ax.clone()
                K.tsgemm([x], [gx], [w], alpha=-1.0, beta=1.0, zs=[ax])
            else:
                w = z(n, kt - n_locked)
                K.rr_residual(x[:, n_locked:], ax[:, n_locked:], theta[n_locked:], None, w, colnorm2)
            self._T(w)
            if nb + w.shape[1] > self.cap:  # thick restart to the current Ritz block
                self.basis[:, :kt].copy_(x)
                self.abasis[:, :kt].copy_(ax)
                nb = kt
                ga = self._gram(self.basis[:, :nb], self.abasis[:, :nb])
                gb = self._gram(self.basis[:, :nb], self.basis[:, :nb])
            w = self._expand(nb, w)
            m = w.shape[1]
            if m:
                self.basis[:, nb:nb + m].copy_(w)
                wv = self.basis[:, nb:nb + m]
                awv = self.abasis[:, nb:nb + m]
                self._A(wv, awv)
                cross_a = self._gram(self.basis[:, :nb], awv)
                cross_b = self._gram(self.basis[:, :nb], wv)
                ga2 = z(nb + m, nb + m)
                gb2 = z(nb + m, nb + m)
                ga2[:nb, :nb] = ga
                ga2[:nb, nb:] = cross_a
                ga2[nb:, :nb] = cross_a.conj().T
                ga2[nb:, nb:] = self._gram(wv, awv)
                gb2[:nb, :nb] = gb
                gb2[:nb, nb:] = cross_b
                gb2[nb:, :nb] = cross_b.conj().T
                gb2[nb:, nb:] = self._gram(wv, wv)
                ga, gb = ga2, gb2
                nb += m
            theta, c = self._solve_pencil(ga, gb, kt)
            c = c.contiguous()
            x, ax = z(n, kt), z(n, kt)
            K.tsgemm([self.basis[:, :nb], self.abasis[:, :nb]], [c, c], [x, ax])
            rr_count += 1
            th = theta.cpu().numpy()
            values_history.append(th.copy())
            K.rr_residual(x, ax, theta, None, None, colnorm2)
            rn = np.sqrt(np.maximum(colnorm2.cpu().numpy(), 0.0))
            n_locked = lock_count(th, rn, opts.tol)
        if theta is None:
            theta, c = self._solve_pencil(ga, gb, kt)
            c = c.contiguous()
            xn, axn = z(n, kt), z(n, kt)
            K.tsgemm([x, ax], [c, c], [xn, axn])
            x, ax = xn, axn
            rr_count += 1
        wall = (time.perf_counter() - t_start) * 1e3
        K.rr_residual(x, ax, theta, None, None, colnorm2)
        rn = np.sqrt(np.maximum(colnorm2.cpu().numpy(), 0.0))
        th = theta.cpu().numpy()
        return SolveReport(values=th[:k].copy(), vectors=K.to_host(x[:, :k]), trace=trace, status=status,
                           iterations=iterations, matvecs=self.matvecs, rr_count=rr_count, breakdown_recoveries=0,
                           wall_ms=wall, values_history=values_history,
                           diagnostics={"final_residual_norms": rn[:k].tolist()})
