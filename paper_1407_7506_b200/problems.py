"""Seeded problem generators producing scipy CSR matrices (host-side input construction).

Two families:

* mirrors of the reference's own model problems (``problems.py:191-276`` in
  ``blockeig``): ``laplacian_1d``, ``laplacian_3d``, ``laplacian_plus_potential``,
  ``two_well_potential``, ``well_problem``, ``random_hermitian`` and
  ``jacobi_preconditioner`` (``problems.py:279-286``), so reference tests can be replayed
  on the GPU box, where ``/root/reference`` does not exist;
* the BASELINE.json configurations 1-5, which the reference does not
  ship.  Draw order and sign conventions are fixed here and recorded in DESIGN.md.

Every builder returns a ``SparseHermitian`` from this package (CSR, duplicates summed,
full mirrored storage, ``problems.py:29-45``).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .errors import DimensionError
from .operators import DiagonalPreconditioner, SparseHermitian

__all__ = [
    "laplacian_1d", "laplacian_2d", "laplacian_3d", "laplacian_plus_potential",
    "two_well_potential", "well_problem", "random_hermitian", "jacobi_preconditioner",
    "config_problem", "CONFIGS",
]

_JACOBI_FLOOR = 1e-8


def _lap1d_csr(n):
    if n < 1:
        raise ValueError("n must be >= 1")
    main = np.full(n, 2.0)
    off = -np.ones(n - 1)
    return sp.diags([off, main, off], [-1, 0, 1], format="csr")


def laplacian_1d(n):
    """(-1, 2, -1) Dirichlet Laplacian (reference problems.py:191-198)."""
    return SparseHermitian(_lap1d_csr(n), "symmetric")


def _lap3d_csr(nx, ny, nz):
    if min(nx, ny, nz) < 1:
        raise ValueError("grid dimensions must be >= 1")
    lx, ly, lz = _lap1d_csr(nx), _lap1d_csr(ny), _lap1d_csr(nz)
    ix, iy, iz = sp.identity(nx), sp.identity(ny), sp.identity(nz)
    return (sp.kron(sp.kron(lx, iy), iz) + sp.kron(sp.kron(ix, ly), iz)
            + sp.kron(sp.kron(ix, iy), lz)).tocsr()


def laplacian_3d(nx, ny, nz):
    """7-point Dirichlet Laplacian, C-order flattening (reference problems.py:201-214)."""
    return SparseHermitian(_lap3d_csr(nx, ny, nz), "symmetric")


def laplacian_2d(nx, ny):
    """5-point Dirichlet Laplacian kron(L1,I)+kron(I,L1) (config 1; NOT laplacian_3d(nx,ny,1))."""
    lx, ly = _lap1d_csr(nx), _lap1d_csr(ny)
    return (sp.kron(lx, sp.identity(ny)) + sp.kron(sp.identity(nx), ly)).tocsr()


def laplacian_plus_potential(nx, ny, nz, potential):
    """3-D Laplacian plus a diagonal potential (reference problems.py:217-225)."""
    potential = np.asarray(potential, dtype=np.float64)
    n = nx * ny * nz
    if potential.shape != (n,):
        raise DimensionError(f"potential has shape {potential.shape}, grid needs ({n},)")
    return SparseHermitian((_lap3d_csr(nx, ny, nz) + sp.diags(potential)).tocsr(), "symmetric")


def two_well_potential(nx, ny, nz, depth, seed=0):
    """Mirror-image Gaussian double well on the unit cube (reference problems.py:228-254)."""
    g = np.random.default_rng(seed)
    c1 = np.array([0.28, 0.28, 0.28]) + g.uniform(-0.06, 0.06, size=3)
    centres = np.array([c1, 1.0 - c1])
    width = 0.11
    axes = [(np.arange(k) + 0.5) / k for k in (nx, ny, nz)]
    px, py, pz = np.meshgrid(*axes, indexing="ij")
    pts = np.stack([px.ravel(), py.ravel(), pz.ravel()], axis=1)
    v = np.zeros(nx * ny * nz)
    for c in centres:
        d2 = np.sum((pts - c[None, :]) ** 2, axis=1)
        v -= depth * np.exp(-d2 / (2.0 * width ** 2))
    return v


def well_problem(nx, ny, nz, depth, seed=0):
    return laplacian_plus_potential(nx, ny, nz, two_well_potential(nx, ny, nz, depth, seed))


def _from_triangle(n, rows, cols, vals, symmetry):
    """Mirror one stored triangle (reference problems.py:47-63)."""
    rows, cols, vals = np.asarray(rows), np.asarray(cols), np.asarray(vals)
    off = rows != cols
    r = np.concatenate([rows, cols[off]])
    c = np.concatenate([cols, rows[off]])
    mv = vals[off].conj() if symmetry == "hermitian" else vals[off]
    v = np.concatenate([vals, mv])
    return SparseHermitian(sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr(), symmetry)


def random_hermitian(n, density, seed, complex_field=False):
    """Seeded sparse Hermitian with N(0,1) entries (reference problems.py:257-276)."""
    if not 0 < density <= 1:
        raise ValueError("density must be in (0, 1]")
    g = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n)
    keep = g.random(iu.shape[0]) < density if density < 1 else np.ones(iu.shape[0], bool)
    iu, ju = iu[keep], ju[keep]
    vals = g.standard_normal(iu.shape[0])
    if complex_field:
        im = g.standard_normal(iu.shape[0])
        im[iu == ju] = 0.0
        return _from_triangle(n, iu, ju, vals + 1j * im, "hermitian")
    return _from_triangle(n, iu, ju, vals, "symmetric")


def jacobi_preconditioner(op, shift=0.0):
    """d_i = 1/max(Re A_ii - shift, 1e-8) (reference problems.py:279-286)."""
    diag = np.real(op.diagonal())
    return DiagonalPreconditioner(1.0 / np.maximum(diag - shift, _JACOBI_FLOOR))


# ----------------------------------------------------------------------------- BASELINE configs
def _grid_index(shape):
    nx, ny, nz = shape
    return np.arange(nx * ny * nz).reshape(nx, ny, nz)


def _cfg1(seed=0, N=64):
    """2-D 5-pt Dirichlet Laplacian on N x N plus V ~ U[0,1)."""
    v = np.random.default_rng(seed).random(N * N)
    return SparseHermitian((laplacian_2d(N, N) + sp.diags(v)).tocsr(), "symmetric")


def _cfg2(seed=0, N=48, wells=8):
    """3-D 7-pt Laplacian N^3 plus 8 Gaussian wells."""
    g = np.random.default_rng(seed)
    centres = g.uniform(0, N, (wells, 3))
    depths = g.uniform(1, 5, wells)
    widths = g.uniform(2, 4, wells)
    ax = np.arange(N, dtype=np.float64)
    px, py, pz = np.meshgrid(ax, ax, ax, indexing="ij")
    pts = np.stack([px.ravel(), py.ravel(), pz.ravel()], axis=1)
    v = np.zeros(N ** 3)
    for c, dep, w in zip(centres, depths, widths):
        d2 = np.sum((pts - c[None, :]) ** 2, axis=1)
        v -= dep * np.exp(-d2 / (2.0 * w * w))
    return laplacian_plus_potential(N, N, N, v)


def _cfg3(seed=0, N=64):
    """3-D 7-pt Laplacian N^3 plus V ~ U[0,2)."""
    return laplacian_plus_potential(N, N, N, np.random.default_rng(seed).uniform(0, 2, N ** 3))


def _cfg4(seed=0, N=96, margin=1.0):
    """27-pt symmetric stencil on N^3, off-diagonals U[-0.1,0] per undirected edge, diag =
    row-sum |w| + margin."""
    idx = _grid_index((N, N, N))
    offsets = [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
               if (dx, dy, dz) > (0, 0, 0)]
    rows, cols = [], []
    for dx, dy, dz in offsets:
        sx = slice(max(0, -dx), N - max(0, dx))
        sy = slice(max(0, -dy), N - max(0, dy))
        sz = slice(max(0, -dz), N - max(0, dz))
        src = idx[sx, sy, sz]
        dst = idx[sx.start + dx:sx.stop + dx, sy.start + dy:sy.stop + dy, sz.start + dz:sz.stop + dz]
        rows.append(src.ravel())
        cols.append(dst.ravel())
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    w = np.random.default_rng(seed).uniform(-0.1, 0.0, rows.shape[0])
    n = N ** 3
    off = sp.coo_matrix((w, (rows, cols)), shape=(n, n)).tocsr()
    off = (off + off.T).tocsr()
    diag = np.asarray(abs(off).sum(axis=1)).ravel() + margin
    return SparseHermitian((off + sp.diags(diag)).tocsr(), "symmetric")


def _cfg5(seed=0, N=128, flux=0.01):
    """Complex Hermitian 7-pt tight binding on N^3 with Peierls phases on y-links,
    theta = 2*pi*flux*x, diag = 6 + V, V ~ U[0,1)."""
    idx = _grid_index((N, N, N))
    n = N ** 3
    v = np.random.default_rng(seed).random(n)
    rows = [np.arange(n)]
    cols = [np.arange(n)]
    vals = [(6.0 + v).astype(np.complex128)]
    # x-links
    rows.append(idx[:-1].ravel()); cols.append(idx[1:].ravel())
    vals.append(np.full(rows[-1].shape[0], -1.0 + 0j))
    # y-links with Peierls phase exp(i theta(x))
    src = idx[:, :-1, :]
    xs = np.broadcast_to(np.arange(N)[:, None, None], src.shape).ravel()
    rows.append(src.ravel()); cols.append(idx[:, 1:, :].ravel())
    vals.append(-np.exp(1j * 2.0 * np.pi * flux * xs))
    # z-links
    rows.append(idx[:, :, :-1].ravel()); cols.append(idx[:, :, 1:].ravel())
    vals.append(np.full(rows[-1].shape[0], -1.0 + 0j))
    return _from_triangle(n, np.concatenate(rows), np.concatenate(cols),
                          np.concatenate(vals), "hermitian")


# name -> (builder, k, sbsize, tol, description)
CONFIGS = {
    1: (_cfg1, 64, 8, 1e-6, "2-D 5-pt 64^2 + V~U[0,1), n=4096, k=64, q=8"),
    2: (_cfg2, 512, 32, 1e-6, "3-D 7-pt 48^3 + 8 Gaussian wells, n=110592, k=512, q=32"),
    3: (_cfg3, 1024, 64, 1e-6, "3-D 7-pt 64^3 + V~U[0,2), n=262144, k=1024, q=64"),
    4: (_cfg4, 2048, 64, 1e-5, "3-D 27-pt 96^3, n=884736, k=2048, q=64"),
    5: (_cfg5, 4096, 64, 1e-5, "complex 7-pt Peierls 128^3, n=2097152, k=4096, q=64"),
}


def config_problem(cfg, seed=0, **kw):
    """Return (operator, k, sbsize, tol) for BASELINE config ``cfg``; ``kw`` may shrink the
    grid (``N=``) for scaled-down instances of the same structure."""
    build, k, q, tol, _ = CONFIGS[cfg]
    return build(seed=seed, **kw), k, q, tol
