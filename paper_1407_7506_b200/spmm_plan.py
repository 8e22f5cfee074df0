"""Stencil plan for the plane-marching CSR SpMM (bk_spmm_march_*; replaces problems.py:72-73).

A row gather reads each X row once per nonzero that references it (7x for a 7-point
stencil, 27x for a 27-point one).  Even at full memory-level parallelism that traffic runs
into the L2 throughput cap long before HBM (profiles/spmm_sweep_r01.jsonl).  The march
kernel instead stages X tiles in shared memory and reuses them: a CTA owns an 8 x 8 tile of
a grid plane and a 256-byte column slice and marches along the slowest grid axis, keeping
planes x-1, x, x+1 of the tile (with its one-row y/z halo) in a 4-slot ring.  Every X row
is then read ~(10 x 10)/(8 x 8) = 1.56 times instead of 7 or 27 times.

The kernel computes from the CSR values in CSR order (so the result equals the gather's bit
for bit), re-laid out as a grid-ordered ELL (each row's entries contiguous, padded to the
widest row) together with 16 bits per entry that encode the stencil offset ``(dx, dy, dz)``
of its column relative to its row as the kernel's shared-memory ring offset, so that a plane
tile's entries arrive with one TMA load like the X tile.  The grid is inferred
from the CSR alone, so the reference's own ``SparseHermitian`` objects qualify:

* every offset ``col - row - d0`` (``d0`` = the diagonal's shift: 0 for a global CSR,
  the ghost shift for the ghost-extended local CSR of a row partition) must be
  ``a*P + b*nz + c`` with ``|a|, |b|, |c| <= 1``, ``P = ny*nz`` and ``n = nx*P``;
* decoding row and column to grid coordinates must give ``|dx|, |dy|, |dz| <= 1`` for
  every nonzero (this rejects periodic wrap-around, which would need a wider halo).

Anything else keeps the gather kernels.
"""

from __future__ import annotations

import numpy as np

TY = TZ = 8         # grid tile per CTA (the kernel's compile-time tile)
SLICE_DOUBLES = 32  # doubles per staged X row slice (the kernel's M_COLS)


def _row_ids(indptr):
    n = indptr.shape[0] - 1
    return np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr).astype(np.int64))


def infer_grid(indptr, indices, n):
    """((nx, ny, nz), d0) such that every offset col - row - d0 lies in the 27-point stencil
    set of an nx x ny x nz C-order grid, or None."""
    if n == 0 or indices.shape[0] == 0:
        return None
    rows = _row_ids(indptr)
    off = indices.astype(np.int64) - rows
    vals, counts = np.unique(off, return_counts=True)
    if vals.shape[0] > 27:
        return None
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
    """Host side of the march SpMM: grid (nx, ny, nz), shift d0, planes [xlo, xhi) the
    columns reach, and the grid-ordered ELL arrays: ``ell_off`` (n x woff uint16, the ring
    offset of each entry's X row, 0xffff = padding) and ``ell_values(data)``.  ``ok`` is False when the
    CSR is not a nearest-neighbour stencil on an inferred grid."""

    def __init__(self, indptr, indices, n, ncols=None):
        self.ok = False
        ncols = n if ncols is None else ncols
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        g = infer_grid(indptr, indices, n)
        if g is None:
            return
        (nx, ny, nz), d0 = g
        rows = _row_ids(indptr)
        c = indices - d0
        P = ny * nz
        rx, ry, rz = rows // P, (rows // nz) % ny, rows % nz
        cx = np.floor_divide(c, P)
        rem = c - cx * P
        cy, cz = rem // nz, rem % nz
        dx, dy, dz = cx - rx, cy - ry, cz - rz
        if indices.shape[0] and (np.abs(dx).max() > 1 or np.abs(dy).max() > 1 or np.abs(dz).max() > 1):
            return
        # planes the column indices reach (ghost planes of a row partition: -1 and nx); the
        # kernel stages whole planes [xlo, xhi) of X rows d0 + p*P .., which must exist
        xlo = int(cx.min()) if indices.shape[0] else 0
        xhi = int(cx.max()) + 1 if indices.shape[0] else nx
        if d0 % P or d0 + xlo * P < 0 or d0 + xhi * P > ncols:
            return
        self.grid = (int(nx), int(ny), int(nz))
        self.d0 = d0
        self.xlo, self.xhi = xlo, xhi
        # grid-ordered ELL (row r's entries in CSR order, then padding 0xffff): the kernel stages
        # a plane tile's entries with one TMA load, like the X tile.  Per entry the kernel's
        # ring offset of its X row: (dx+1) << 14 | ((dy+1)*(TY+2) + dz+1) * SLICE_DOUBLES
        offs = (((dx + 1) << 14) | (((dy + 1) * (TY + 2) + (dz + 1)) * SLICE_DOUBLES)).astype(np.uint16)
        cnt = np.diff(indptr)
        w = int(cnt.max(initial=1))
        self.width = w
        self.woff = -(-w // 8) * 8                         # 16-byte rows of uint16
        slot = np.arange(indices.shape[0], dtype=np.int64) - indptr[rows]
        ell_off = np.full((n, self.woff), 0xFFFF, dtype=np.uint16)
        ell_off[rows, slot] = offs
        self.ell_off = ell_off
        self.rows_, self.slot_ = rows, slot
        self.ok = True

    def ell_values(self, data):
        """Values in the grid-ordered ELL layout: real rows padded to an even width (16-byte
        rows), complex rows of ``width`` elements; padding is zero (never read)."""
        if np.iscomplexobj(data):
            out = np.zeros((self.ell_off.shape[0], self.width), dtype=np.complex128)
        else:
            out = np.zeros((self.ell_off.shape[0], -(-self.width // 2) * 2), dtype=np.float64)
        out[self.rows_, self.slot_] = data
        return out
