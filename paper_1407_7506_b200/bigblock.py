"""Subblock updates whose pencil exceeds the batched device pencils (3q > 192): whole-block
PPCG (sbsize >= 65, e.g. the LOBPCG-equivalent mode of test_acceptance.py:90-106) and
LOBPCG's block_update over the whole active block.

The arithmetic stays on the device -- raw Grams (gram_kernel), pencil assembly / coefficient
scatter / breakdown statistics (bigblock.cu), Cholesky probe + sygvd and gesvd (cuSOLVER),
recombination (tsgemm) -- while the host runs block_update's branch logic (ppcg.py:278-378)
one subblock at a time, in the same order as the batched pencil kernel:
dropped directions (198-203), unit scaling (220-228), SingularGramError retry ladder
(332-349: drop P, then shed the weakest W column), rank test sigma_min(C_X) <
1e-14 max(||C||_2, 1) (351-356), fallback_steepest_descent (231-275), coefficient un-scaling
and coeff_scale (358-363, 376).
"""

from __future__ import annotations

import numpy as np

_DIR_FLOOR = 1e-14   # ppcg.py:198-203
_CX_FLOOR = 1e-14    # ppcg.py:351-356


class LargeBlocks:
    """Scratch and state for the large-subblock path of one PPCGSolver."""

    def __init__(self, solver):
        self.s = solver
        self.bufs = {}

    def _buf(self, key, shape, dtype):
        import torch

        t = self.bufs.get(key)
        if t is None or t.numel() < int(np.prod(shape)):
            t = torch.zeros(int(np.prod(shape)), dtype=dtype, device="cuda")
            self.bufs[key] = t
        return t[: int(np.prod(shape))].view(*shape)

    def update(self, ka, q, has_p, src, psrc, dst, pdst, force_fallback=False, blocks=None):
        """Run every subblock (or the given (lo, hi) ranges) of the active block [L, L+ka):
        writes XF[dst], P[pdst], AXF[dst], AP[pdst] columns, theta, info, cscale, flags64
        exactly as subblock_grams/pencils/recombine do for small pencils."""
        import torch

        from .ppcg import split_blocks

        s = self.s
        K = s.K
        parts = split_blocks(ka, q) if blocks is None else blocks
        info = np.zeros((len(parts), 4), dtype=np.int32)
        cs = np.ones(len(parts))
        for j, (lo, hi) in enumerate(parts):
            info[j], cs[j] = self._one(lo, hi - lo, has_p, src, psrc, dst, pdst, force_fallback)
        s.info[: info.size].copy_(torch.from_numpy(info.reshape(-1)))
        s.cscale[: len(parts)].copy_(torch.from_numpy(cs))

    # ------------------------------------------------------------------ one subblock
    def _one(self, lo, w, has_p, src, psrc, dst, pdst, force):
        import torch

        s = self.s
        K, L = s.K, s.L
        tdt = s.tdt
        nparts = 3 if has_p else 2
        d0 = nparts * w
        c0 = L + lo
        XFs, AXFs = s.XF[src], s.AXF[src]
        Ps, APs = s.P[psrc], s.AP[psrc]
        # raw Grams S^H [AX AW AP], S^H S of S = [X_j W_j P_j]  (ppcg.py:206-211)
        K.subblock_grams(s.nl, w, w, has_p, XFs.data_ptr(), s.W.data_ptr(), Ps.data_ptr(), AXFs.data_ptr(),
                         s.AW.data_ptr(), APs.data_ptr(), s._ldr(), c0, s.araw, s.braw, tmp=s.gtmp)
        s._red(s.araw[: d0 * d0], s.braw[: d0 * d0])
        araw = s.araw[: d0 * d0].view(d0, d0)
        braw = s.braw[: d0 * d0].view(d0, d0)
        bd = np.real(torch.diagonal(braw).cpu().numpy()).astype(np.float64)
        ad = np.real(torch.diagonal(araw).cpu().numpy()).astype(np.float64)
        nrm = np.sqrt(np.maximum(bd, 0.0))
        sc = max(float(np.max(nrm[:w])) if w else 0.0, 1e-300)
        floor = _DIR_FLOOR * sc
        keptw = [i for i in range(w) if nrm[w + i] > floor]
        keptp = [i for i in range(w) if has_p and nrm[2 * w + i] > floor]

        coef = self._buf("coef", (d0, w), tdt)
        theta = s.theta[lo: lo + w]
        fallback = zero_res = err = attempts = 0
        cmax = 1.0
        sol = None

        def passthrough(fb):
            nonlocal fallback, zero_res, cmax
            eye = torch.zeros((d0, w), dtype=tdt, device="cuda")
            eye[:w].copy_(torch.eye(w, dtype=tdt, device="cuda"))
            coef.copy_(eye)
            theta.copy_(torch.from_numpy(ad[:w] / bd[:w]))
            fallback, zero_res, cmax = int(fb), 1, 1.0

        def attempt(mw, mp):
            idx = list(range(w)) + [w + i for i in mw] + [2 * w + i for i in mp]
            sf = [1.0] * w + [1.0 / nrm[w + i] for i in mw] + [1.0 / nrm[2 * w + i] for i in mp]
            d = len(idx)
            idx_t = torch.tensor(idx, dtype=torch.int32, device="cuda")
            sf_t = torch.tensor(sf, dtype=torch.float64, device="cuda")
            A = self._buf("A", (d, d), tdt)
            B = self._buf("B", (d, d), tdt)
            C = self._buf("C", (d, d), tdt)
            om = self._buf("om", (d,), torch.float64)
            st = self._buf("st", (4,), torch.int32)
            K.block_assemble(d, idx_t, sf_t, araw, braw, d0, A, B)
            s.dense.rr_pencil(A, B, om, C, st)
            singular = int(st.cpu()[0]) != 0
            return singular, (idx_t, sf_t, d, C, om)

        if not force and not keptw and not keptp:
            passthrough(False)
        else:
            mw, mp = list(keptw), list(keptp)
            do_fb = bool(force)
            if not do_fb:
                bad, sol = attempt(mw, mp)
                attempts += 1
                if bad:
                    mp = []  # drop P first, then shed the weakest W column (ppcg.py:335-349)
                    while True:
                        bad, sol = attempt(mw, mp)
                        attempts += 1
                        if not bad:
                            break
                        if not mw:
                            err = 1
                            break
                        worst = min(mw, key=lambda i: (nrm[w + i], i))
                        mw.remove(worst)
                if not err:
                    _, _, d, C, _ = sol
                    sv = self._buf("sv", (d,), torch.float64)
                    s.dense.svals(C[:, :w], sv)
                    cn = float(sv[:min(d, w)].max().cpu())
                    s.dense.svals(C[:w, :w], sv)
                    smin = float(sv[:w].min().cpu())
                    if smin < _CX_FLOOR * max(cn, 1.0):
                        do_fb = True
            if do_fb:  # fallback_steepest_descent over [X, kept W] (ppcg.py:231-275)
                fallback = 1
                mw, mp = list(keptw), []
                if not mw:
                    passthrough(True)
                else:
                    bad, sol = attempt(mw, mp)
                    attempts += 1
                    if bad:
                        err = 1
            if not err and not (fallback and zero_res):
                idx_t, sf_t, d, C, om = sol
                cm = self._buf("cm", (1,), torch.float64)
                K.block_coef(d, w, d0, idx_t, sf_t, C, coef, cm)
                theta.copy_(om[:w])
                cmax = float(cm.cpu()[0])
        if not err:
            self._recombine(lo, w, has_p, coef, src, psrc, dst, pdst)
        return np.array([fallback, zero_res, err, attempts], dtype=np.int32), cmax

    # ------------------------------------------------------------------ X C, W C_W + P C_P
    def _recombine(self, lo, w, has_p, coef, src, psrc, dst, pdst):
        """P' = W C_W + P C_P, X' = X C_X + P' and the A-side alike (ppcg.py:365-369,
        521-532) with the tall DMMA GEMM, plus the breakdown statistics (701-705)."""
        s = self.s
        K = s.K
        c0 = s.L + lo
        cs = slice(c0, c0 + w)
        x, ax = s.XF[src][:, cs], s.AXF[src][:, cs]
        wv, awv = s.W[:, cs], s.AW[:, cs]
        xo, axo = s.XF[dst][:, cs], s.AXF[dst][:, cs]
        po, apo = s.P[pdst][:, cs], s.AP[pdst][:, cs]
        inplace = has_p and pdst == psrc
        if inplace:  # P' = W C_W + P C_P reads P: build it in scratch, copy over P at the end
            po_f, apo_f = po, apo
            po = self._buf("po", (s.nl, w), s.tdt)
            apo = self._buf("apo", (s.nl, w), s.tdt)
        cx, cw = coef[:w], coef[w: 2 * w]
        K.tsgemm([wv, awv], [cw, cw], [po, apo])
        if has_p:
            p, ap = s.P[psrc][:, cs], s.AP[psrc][:, cs]
            cp = coef[2 * w: 3 * w]
            K.tsgemm([p, ap], [cp, cp], [po, apo], beta=1.0, zs=[po, apo])
        K.tsgemm([x, ax], [cx, cx], [xo, axo], beta=1.0, zs=[po, apo])
        if inplace:
            K.copy_cols(po, po_f)
            K.copy_cols(apo, apo_f)
            po, apo = po_f, apo_f
        K.block_stats(xo, s.flags64, 1)
        K.block_stats(po, s.flags64, 2)
        K.block_stats(axo, s.flags64, 0)
        K.block_stats(apo, s.flags64, 0)
