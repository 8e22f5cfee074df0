"""Operator and preconditioner types (same API as blockeig operators.py / problems.py:29-89),
backed by device kernels.

The solver only needs ``n``, ``dtype`` and ``apply(block)`` (operators.py:1-7).  Here
``apply`` accepts a numpy block (uploads, computes on the GPU, returns numpy) or a CUDA
tensor (stays on the device).  ``as_device_operator`` / ``as_device_preconditioner``
turn any operator — these classes, the reference's own ``blockeig`` objects, or a duck-typed
user object — into a device apply used inside the solver:

* anything exposing a scipy CSR as ``_csr`` (SparseHermitian, both packages) -> CSR SpMM
  (replaces problems.py:72-73): the plane-marching stencil kernel (bk_spmm_march_*) when the
  CSR is a nearest-neighbour stencil on a grid inferred from its offsets (spmm_plan.py),
  the whole-row gather (bk_spmm_csr_*) otherwise;
* ``DenseHermitian`` (``matrix``) -> DMMA tall GEMM;
* ``DiagonalOperator`` (``diag``) / ``DiagonalPreconditioner`` (``d``) -> row scaling, which
  the solver fuses into the residual epilogue for preconditioners (operators.py:96-110);
* other user operators keep their own ``apply`` (host callback); that is the user's code,
  not a fallback of this package.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .errors import DimensionError

__all__ = [
    "LinearBlockOperator", "DenseHermitian", "DiagonalOperator", "MatrixFreeOperator",
    "IdentityPreconditioner", "DiagonalPreconditioner", "CountingOperator", "SparseHermitian",
    "as_device_operator", "as_device_preconditioner",
]


def _torch():
    import torch

    return torch


def _is_tensor(x):
    try:
        torch = _torch()
    except Exception:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


class LinearBlockOperator:
    """Square operator applied to n x m blocks via ``apply`` (operators.py:24-42)."""

    n = 0
    dtype = np.float64

    def apply(self, block):
        raise NotImplementedError

    def __matmul__(self, block):
        return self.apply(block)

    def _check(self, block):
        shape = tuple(block.shape)
        if len(shape) != 2 or shape[0] != self.n:
            raise DimensionError(f"operator of dimension {self.n} applied to block of shape {shape}")
        return block

    def _device_apply(self, block):
        """numpy -> device -> numpy through this operator's device kernel."""
        torch = _torch()
        dev = as_device_operator(self)
        if _is_tensor(block):
            x = block
            y = torch.empty_like(x)
            dev.apply_into(x, y)
            return y
        arr = np.ascontiguousarray(self._check(np.asarray(block)))
        tdt = torch.complex128 if (np.iscomplexobj(arr) or dev.complex) else torch.float64
        x = torch.from_numpy(arr.astype(np.complex128 if tdt == torch.complex128 else np.float64)).cuda()
        y = torch.empty_like(x)
        dev.apply_into(x, y)
        return y.cpu().numpy()


class SparseHermitian(LinearBlockOperator):
    """CSR Hermitian operator (problems.py:29-89); ``apply`` runs the device SpMM."""

    def __init__(self, csr, symmetry):
        if symmetry not in ("symmetric", "hermitian"):
            raise ValueError(f"unknown symmetry {symmetry!r}")
        self._csr = csr.tocsr()
        self._csr.sum_duplicates()
        self.n = csr.shape[0]
        self.symmetry = symmetry
        self.dtype = self._csr.dtype
        self._dev = None

    @classmethod
    def from_triangle(cls, n, rows, cols, values, symmetry):
        rows, cols, values = np.asarray(rows), np.asarray(cols), np.asarray(values)
        off = rows != cols
        r = np.concatenate([rows, cols[off]])
        c = np.concatenate([cols, rows[off]])
        mv = values[off].conj() if symmetry == "hermitian" else values[off]
        v = np.concatenate([values, mv])
        return cls(sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr(), symmetry)

    @classmethod
    def from_dense(cls, matrix):
        matrix = np.asarray(matrix)
        symmetry = "hermitian" if np.iscomplexobj(matrix) else "symmetric"
        return cls(sp.csr_matrix(0.5 * (matrix + matrix.conj().T)), symmetry)

    def apply(self, block):
        return self._device_apply(block)

    def diagonal(self):
        return self._csr.diagonal()

    def to_dense(self):
        return self._csr.toarray()

    def to_coo_lower(self):
        low = sp.tril(self._csr, format="coo")
        order = np.lexsort((low.col, low.row))
        return low.row[order], low.col[order], low.data[order]

    @property
    def nnz(self):
        return self._csr.nnz


class DenseHermitian(LinearBlockOperator):
    """Explicit dense Hermitian matrix (operators.py:45-60)."""

    def __init__(self, matrix):
        matrix = np.asarray(matrix)
        if matrix.ndim != 2 or matrix.shape[0] != matrix.shape[1]:
            raise DimensionError(f"expected a square matrix, got shape {matrix.shape}")
        self.matrix = 0.5 * (matrix + matrix.conj().T)
        self.n = matrix.shape[0]
        self.dtype = self.matrix.dtype
        self._dev = None

    def apply(self, block):
        return self._device_apply(block)

    def to_dense(self):
        return self.matrix


class DiagonalOperator(LinearBlockOperator):
    """Diagonal operator (operators.py:63-73)."""

    def __init__(self, diag):
        self.diag = np.asarray(diag)
        self.n = self.diag.shape[0]
        self.dtype = self.diag.dtype
        self._dev = None

    def apply(self, block):
        return self._device_apply(block)

    def to_dense(self):
        return np.diag(self.diag)


class MatrixFreeOperator(LinearBlockOperator):
    """Wrap a block-apply callable (operators.py:76-85).  ``device=True`` means the callable
    takes and returns CUDA tensors."""

    def __init__(self, n, apply_fn, dtype=np.float64, device=False):
        self.n = n
        self._apply_fn = apply_fn
        self.dtype = np.dtype(dtype)
        self.device = device

    def apply(self, block):
        return self._apply_fn(self._check(block))


class IdentityPreconditioner(LinearBlockOperator):
    def __init__(self, n):
        self.n = n

    def apply(self, block):
        b = self._check(block)
        return b.clone() if _is_tensor(b) else np.array(b, copy=True)


class DiagonalPreconditioner(LinearBlockOperator):
    """HPD diagonal preconditioner (operators.py:96-110)."""

    def __init__(self, d):
        d = np.asarray(d, dtype=np.float64)
        if d.ndim != 1:
            raise DimensionError("diagonal must be a 1-D array")
        if not np.all(d > 0):
            raise ValueError("preconditioner diagonal must be strictly positive")
        self.d = d
        self.n = d.shape[0]
        self.dtype = d.dtype
        self._dev = None

    def apply(self, block):
        return self._device_apply(block)


class CountingOperator(LinearBlockOperator):
    """Counts applications column by column (operators.py:113-124)."""

    def __init__(self, inner):
        self.inner = inner
        self.n = inner.n
        self.dtype = inner.dtype
        self.matvecs = 0

    def apply(self, block):
        self.matvecs += block.shape[1]
        return self.inner.apply(block)


# ----------------------------------------------------------------------------- device views
class DeviceCsr:
    """CSR on the device: int32 row pointers / column indices, fp64 or complex128 values."""

    kind = "csr"

    def __init__(self, csr):
        torch = _torch()
        csr = csr.tocsr()
        if csr.nnz >= 2 ** 31 or csr.shape[0] >= 2 ** 31:
            raise DimensionError("CSR too large for int32 indices")
        self.n = csr.shape[0]
        self.complex = np.iscomplexobj(csr.data)
        self.nnz = csr.nnz
        self.rowptr = torch.from_numpy(csr.indptr.astype(np.int32)).cuda()
        self.col = torch.from_numpy(csr.indices.astype(np.int32)).cuda()
        vals = csr.data.astype(np.complex128 if self.complex else np.float64)
        self.val = torch.from_numpy(vals).cuda()
        self.diag = np.real(csr.diagonal())
        self.ncols = csr.shape[1]
        # small operators (config 1: n = 4096) stay on the gather: the march pipeline does not pay
        # at that size, and the plan's first torch ops would dominate a sub-second solve
        self.stencil = (_device_stencil_plan(self)
                        if DeviceCsr.use_stencil and self.n >= DeviceCsr.min_stencil_rows else None)

    # plane-marching stencil kernel when the CSR is a nearest-neighbour stencil on an inferred
    # grid (spmm_plan.py); the whole-row gather otherwise
    use_stencil = True
    min_stencil_rows = 1 << 15
    stencil_kinds = ("slot",)  # plan layouts built: "slot" (preferred where it applies), "march"

    def apply_into(self, x, y):
        from . import kernels

        if self.complex and x.dtype != _torch().complex128:
            raise DimensionError("complex operator applied to a real block")
        if (self.stencil is not None and DeviceCsr.use_stencil
                and kernels.spmm_march(self.stencil, x, y)):
            return
        kernels.spmm_csr(self.rowptr, self.col, self.val, x, y)


def _device_stencil_plan(dc):
    """StencilPlan built on the GPU from the already uploaded CSR (spmm_plan.py)."""
    from .spmm_plan import StencilPlan

    if dc.n == 0 or dc.nnz == 0:
        return None
    plan = StencilPlan(dc.rowptr, dc.col, dc.n, dc.ncols)
    if not plan.ok:
        return None
    # stencil-slot values when the rows qualify (bk_spmm_stencil_*), else the offset ELL
    # (bk_spmm_march_*); DeviceCsr.stencil_kinds can keep both (tests compare the kernels)
    plan.sval = plan.slot_values(dc.val) if plan.st and "slot" in DeviceCsr.stencil_kinds else None
    plan.ell_val = plan.ell_values(dc.val) if plan.sval is None or "march" in DeviceCsr.stencil_kinds else None
    plan.release_host_index()
    return plan


class DeviceDense:
    kind = "dense"

    def __init__(self, matrix):
        torch = _torch()
        self.n = matrix.shape[0]
        self.complex = np.iscomplexobj(matrix)
        dt = torch.complex128 if self.complex else torch.float64
        self.a = torch.from_numpy(np.ascontiguousarray(matrix).astype(
            np.complex128 if self.complex else np.float64)).cuda()
        self.diag = np.real(np.diag(matrix))
        self.dtype = dt

    def apply_into(self, x, y):
        from . import kernels

        a = self.a if x.dtype == self.a.dtype else self.a.to(x.dtype)
        kernels.tsgemm([a], [x], [y])


class DeviceDiag:
    kind = "diag"

    def __init__(self, d):
        torch = _torch()
        d = np.asarray(d)
        if np.iscomplexobj(d):
            if np.any(np.imag(d) != 0):
                raise DimensionError("complex diagonal operators are not supported on the device")
            d = np.real(d)
        self.n = d.shape[0]
        self.complex = False
        self.d = torch.from_numpy(d.astype(np.float64)).cuda()
        self.diag = d

    def apply_into(self, x, y):
        from . import kernels

        kernels.scale_rows(self.d, x, y)


class DeviceCallback:
    """A user operator without a device form: its own apply runs on host copies."""

    kind = "callback"

    def __init__(self, op):
        self.op = op
        self.n = op.n
        self.complex = np.issubdtype(np.dtype(op.dtype), np.complexfloating)
        self.device = bool(getattr(op, "device", False))
        self.diag = None

    def apply_into(self, x, y):
        if self.device:
            y.copy_(self.op.apply(x))
            return
        torch = _torch()
        out = np.asarray(self.op.apply(x.cpu().numpy()))
        y.copy_(torch.from_numpy(np.ascontiguousarray(out).astype(
            np.complex128 if y.dtype == torch.complex128 else np.float64)))


def _source_key(op):
    """What the device copy was made from: the identity and shape of the host arrays plus a
    sampled fingerprint of their values, so replacing (or editing) an operator's arrays after a
    solve rebuilds the device form instead of silently reusing a stale one (the reference reads
    the operator on every apply)."""
    def fp(a):
        a = np.asarray(a)
        if a.size == 0:
            return (id(a), 0)
        step = max(1, a.size // 4096)
        flat = a.reshape(-1)[::step]
        return (id(a), a.shape, a.dtype.str, complex(np.sum(flat * (1.0 + np.arange(flat.size) % 7))))

    if hasattr(op, "_csr"):
        c = op._csr
        return ("csr", fp(c.data), fp(c.indices), fp(c.indptr), c.shape)
    for attr in ("matrix", "diag", "d"):
        if hasattr(op, attr):
            return (attr, fp(getattr(op, attr)))
    return ("callback", id(op))


def as_device_operator(op):
    """Device form of an operator (cached on the object, keyed by its source arrays)."""
    if isinstance(op, CountingOperator):
        return as_device_operator(op.inner)
    key = _source_key(op)
    cached = getattr(op, "_dev", None)
    if cached is not None and getattr(op, "_dev_key", None) == key:
        return cached
    if hasattr(op, "_csr"):
        dev = DeviceCsr(op._csr)
    elif hasattr(op, "matrix") and type(op).__name__ == "DenseHermitian":
        dev = DeviceDense(np.asarray(op.matrix))
    elif hasattr(op, "diag") and type(op).__name__ == "DiagonalOperator":
        dev = DeviceDiag(op.diag)
    elif hasattr(op, "d") and type(op).__name__ == "DiagonalPreconditioner":
        dev = DeviceDiag(op.d)
    else:
        dev = DeviceCallback(op)
    try:
        op._dev, op._dev_key = dev, key
    except Exception:
        pass
    return dev


def as_device_preconditioner(t):
    """None (identity), ('diag', d_tensor) for fused row scaling, or ('op', device operator)."""
    if t is None or type(t).__name__ == "IdentityPreconditioner":
        return None
    dev = as_device_operator(t)
    if isinstance(dev, DeviceDiag):
        return ("diag", dev.d)
    return ("op", dev)
