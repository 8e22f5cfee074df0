"""Stencil plan for the plane-marching CSR SpMM (bk_spmm_march_*; replaces problems.py:72-73).

A row gather reads each X row once per nonzero that references it (7x for a 7-point
stencil, 27x for a 27-point one).  Even at full memory-level parallelism that traffic runs
into the L2 throughput cap long before HBM (profiles/spmm_sweep_r01.jsonl).  The march
kernel instead stages X tiles in shared memory and reuses them: a work unit is an 8 x 8 tile
of a grid plane and a column slice (512 bytes for real rows of <= 8 entries, else 256), and it
marches along the slowest grid axis, keeping planes x-1, x, x+1 of the tile (with its one-row
y/z halo) in a 4-6 slot ring fed by TMA.  Every X row is then read ~(10 x 10)/(8 x 8) = 1.56
times instead of 7 or 27 times.

The kernel computes from the CSR values in CSR order (so the result equals the gather's bit
for bit), re-laid out as a grid-ordered ELL (each row's entries contiguous, padded to the
widest row) together with 16 bits per entry that encode the stencil offset ``(dx, dy, dz)``
of its column relative to its row as the kernel's shared-memory ring position, so that a plane
tile's entries arrive with one TMA load like the X tile.  The grid is inferred
from the CSR alone, so the reference's own ``SparseHermitian`` objects qualify:

* every offset ``col - row - d0`` (``d0`` = the diagonal's shift: 0 for a global CSR,
  the ghost shift for the ghost-extended local CSR of a row partition) must be
  ``a*P + b*nz + c`` with ``|a|, |b|, |c| <= 1``, ``P = ny*nz`` and ``n = nx*P``;
* decoding row and column to grid coordinates must give ``|dx|, |dy|, |dz| <= 1`` for
  every nonzero (this rejects periodic wrap-around, which would need a wider halo).

Anything else keeps the gather kernels; so do operators under 32,768 rows (operators.py).

Stencil-slot layout (bk_spmm_stencil_*, the default where it applies): when every row's
columns are sorted (CSR order = stencil order (dx, dy, dz) lexicographic) and the offsets are
the 7-point cross or lie in the 27-point cube, the values are laid out per stencil POSITION
instead (slot s of a row = the value at position s, presence bits in the row's last double).
The kernel then knows every X address at compile time and reuses X rows from registers.
"""

from __future__ import annotations

import numpy as np

TY = TZ = 8  # grid tile per CTA (the kernel's compile-time tile)

# 27-point position (dx+1)*9 + (dy+1)*3 + dz+1 -> 7-point cross slot
_CROSS = {4: 0, 10: 1, 12: 2, 13: 3, 14: 4, 16: 5, 22: 6}
# doubles per stencil-slot row (values + mask, even; padded so that the rows of one warp's
# value loads fall in different shared-memory banks)
_SLOT_VD = {(7, False): 10, (27, False): 28, (7, True): 18, (27, True): 58}


def _torch():
    import torch

    return torch


def _row_ids(indptr):
    torch = _torch()
    n = indptr.shape[0] - 1
    return torch.repeat_interleave(torch.arange(n, dtype=torch.int64, device=indptr.device), indptr[1:] - indptr[:-1])


def infer_grid(indptr, indices, n):
    """((nx, ny, nz), d0) such that every offset col - row - d0 lies in the 27-point stencil
    set of an nx x ny x nz C-order grid, or None.  indptr / indices: int64 torch tensors."""
    torch = _torch()
    if n == 0 or indices.shape[0] == 0:
        return None
    off = indices - _row_ids(indptr)
    vals, counts = torch.unique(off, return_counts=True)
    if vals.shape[0] > 27:
        return None
    vals, counts = vals.cpu().numpy(), counts.cpu().numpy()
    # the diagonal's shift d0: the most frequent offsets first (ties: the one nearest the
    # middle of the offset range, e.g. interior slabs where +-P are as frequent as 0)
    mid = int(vals.min()) + int(vals.max())
    for i in sorted(range(vals.shape[0]), key=lambda i: (-int(counts[i]), abs(2 * int(vals[i]) - mid))):
        d0 = int(vals[i])
        g = _grid_for(vals - d0, n)
        if g is not None:
            return g, d0
    return None


def _grid_for(o, n):
    pos = o[o > 0]
    if pos.shape[0] == 0:
        return (1, 1, n) if np.all(o == 0) else None

    def fits(nz, P):
        allowed = {a * P + b * nz + c for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)}
        return all(int(v) in allowed for v in o)

    cands = sorted({int(v) for v in pos if v >= 2})
    for nz in cands:  # 3-D: nz and P = ny*nz both appear as offsets
        for P in cands:
            if P <= nz or P % nz or n % P:
                continue
            if fits(nz, P):
                return (n // P, P // nz, nz)
    for nz in cands:  # 2-D (nx = 1)
        if n % nz == 0 and fits(nz, n):
            return (1, n // nz, nz)
    if fits(n, n):  # 1-D: offsets -1, 0, 1 only
        return (1, 1, n)
    return None


class StencilPlan:
    use_slot = True  # bk_spmm_stencil_* when slot values exist (tests flip it to compare kernels)

    """The march SpMM's plan: grid (nx, ny, nz), shift d0, planes [xlo, xhi) the columns
    reach, and the grid-ordered ELL arrays ``ell_off`` (n x woff int16 holding uint16 bit
    patterns: the ring position (plane slot, halo row) of each entry's X row, 0xffff = padding) and
    ``ell_values(data)``, as torch tensors on ``indptr``'s device (built on the GPU in
    production: a few elementwise passes over the nonzeros).  ``ok`` is False when the CSR is
    not a nearest-neighbour stencil on an inferred grid."""

    def __init__(self, indptr, indices, n, ncols=None, device=None):
        torch = _torch()
        self.ok = False
        ncols = n if ncols is None else ncols
        indptr = torch.as_tensor(np.asarray(indptr) if not torch.is_tensor(indptr) else indptr,
                                 device=device).to(torch.int64)
        indices = torch.as_tensor(np.asarray(indices) if not torch.is_tensor(indices) else indices,
                                  device=indptr.device).to(torch.int64)
        g = infer_grid(indptr, indices, n)
        if g is None:
            return
        (nx, ny, nz), d0 = g
        rows = _row_ids(indptr)
        c = indices - d0
        P = ny * nz
        cx = torch.div(c, P, rounding_mode="floor")
        rem = c - cx * P
        dx = cx - torch.div(rows, P, rounding_mode="floor")
        dy = torch.div(rem, nz, rounding_mode="floor") - torch.div(rows, nz, rounding_mode="floor") % ny
        dz = rem % nz - rows % nz
        amax = torch.stack([dx.abs().max(), dy.abs().max(), dz.abs().max(), cx.min(), cx.max()]).cpu().tolist()
        if max(amax[:3]) > 1:
            return
        # planes the column indices reach (ghost planes of a row partition: -1 and nx); the
        # kernel stages whole planes [xlo, xhi) of X rows d0 + p*P .., which must exist
        xlo, xhi = int(amax[3]), int(amax[4]) + 1
        if d0 % P or d0 + xlo * P < 0 or d0 + xhi * P > ncols:
            return
        self.grid = (int(nx), int(ny), int(nz))
        self.d0 = d0
        self.xlo, self.xhi = xlo, xhi
        # grid-ordered ELL (row r's entries in CSR order, then padding 0xffff): the kernel stages
        # a plane tile's entries with one TMA load, like the X tile.  Per entry the kernel's
        # ring position of its X row: (dx+1) << 14 | (dy+1)*(TY+2) + dz+1
        offs = ((dx + 1) << 14) | ((dy + 1) * (TY + 2) + (dz + 1))
        cnt = indptr[1:] - indptr[:-1]
        w = max(int(cnt.max().item()), 1)
        self.width = w
        self.woff = -(-w // 8) * 8                         # 16-byte rows of uint16
        slot = torch.arange(indices.shape[0], dtype=torch.int64, device=indptr.device) - indptr[rows]
        ell_off = torch.full((n, self.woff), -1, dtype=torch.int16, device=indptr.device)
        ell_off[rows, slot] = offs.to(torch.int32).to(torch.int16)  # uint16 bit patterns
        self.ell_off = ell_off
        self._rows, self._slot = rows, slot
        # stencil-slot layout: rows sorted (strictly increasing positions) -> 7 or 27 slots
        pos = (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1)
        same = rows[1:] == rows[:-1]
        self.st = 0
        if not bool((pos[1:][same] <= pos[:-1][same]).any().item()):
            lut = torch.full((27,), -1, dtype=torch.int64, device=indptr.device)
            for p27, c in _CROSS.items():
                lut[p27] = c
            cross = lut[pos]
            if bool((cross >= 0).all().item()):
                self.st, self._spos = 7, cross
            else:
                self.st, self._spos = 27, pos
        self.ok = True

    def ell_values(self, data):
        """Values (torch tensor or numpy, on any device) in the grid-ordered ELL layout: real
        rows padded to an even width (16-byte rows), complex rows of ``width`` elements;
        padding is zero (never read)."""
        torch = _torch()
        data = torch.as_tensor(data).to(self.ell_off.device)
        if data.is_complex():
            out = torch.zeros((self.ell_off.shape[0], self.width), dtype=torch.complex128, device=data.device)
        else:
            out = torch.zeros((self.ell_off.shape[0], -(-self.width // 2) * 2), dtype=torch.float64,
                              device=data.device)
        out[self._rows, self._slot] = data.to(out.dtype)
        return out

    def slot_values(self, data):
        """Stencil-slot layout for bk_spmm_stencil_* (``st`` 7 or 27): an n x vd float64
        tensor, row r = the values of its stencil positions (real, or interleaved complex) and
        the presence bit mask (int64 bit pattern) in the last double; absent slots are zero and
        never read."""
        torch = _torch()
        data = torch.as_tensor(data).to(self.ell_off.device)
        cplx = data.is_complex()
        self.vd = _SLOT_VD[(self.st, cplx)]
        n = self.ell_off.shape[0]
        out = torch.zeros((n, self.vd), dtype=torch.float64, device=data.device)
        if cplx:
            vals = out[:, :2 * self.st].view(torch.complex128)
            vals[self._rows, self._spos] = data.to(torch.complex128)
        else:
            out[self._rows, self._spos] = data.to(torch.float64)
        mask = torch.zeros(n, dtype=torch.int64, device=data.device)
        mask.index_add_(0, self._rows, torch.ones_like(self._spos) << self._spos)
        out[:, self.vd - 1] = mask.view(torch.float64)
        return out

    def release_host_index(self):
        """Drop the per-nonzero scatter indices once the values are laid out."""
        del self._rows, self._slot
        self.__dict__.pop("_spos", None)
