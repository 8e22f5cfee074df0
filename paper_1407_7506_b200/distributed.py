"""Row-partitioned (multi-GPU) PPCG: partition, halo plan and communicators.

SURVEY §8(e): every n-length quantity of the PPCG iteration (SpMM, residual, Gram
partials, update GEMMs, subblock recombination) is row-local, so the state blocks are split
into contiguous row slabs, one per rank (one process per GPU).  Per iteration the ranks
exchange
  * one halo per operator apply: the ghost rows of the block being multiplied, as
    contiguous row ranges of the neighbouring slabs (P2P send/recv; for 7/27-point
    stencils one grid plane per side), and
  * one sum-allreduce per Gram (metrics, projections, subblock pencils, orthonormality,
    Rayleigh-Ritz) plus the scalar partial sums and the breakdown flags (max).
Everything k_total x k_total or smaller (CholQR factor, pencils, RR eigenproblem) is then
computed redundantly on every rank from identical reduced inputs: the kernels are
deterministic, so every rank takes the same branch of the reference's control flow
(ppcg.py:653-758) without further traffic.

The reference itself is single-process (ppcg.py:587-614); this module is the B200 scale-out
of the same iteration.  Communicators:
  * ``TorchComm``  -- torch.distributed (NCCL between GPUs; gloo for CPU tests);
  * ``ThreadComm`` -- ranks as threads of one process (sums in rank order), used to run the
    sharded solver on a single GPU in tests; collectives are host-side barriers, no
    kernel ever waits on another rank's kernel.
"""

from __future__ import annotations

import threading

import numpy as np

__all__ = ["partition_rows", "HaloPlan", "local_rows_csr", "Comm", "TorchComm", "ThreadComm",
           "thread_comms", "host_csr_of", "dist_ppcg_solve"]


def partition_rows(n, size, rowptr=None, plane=None):
    """Contiguous row slabs [lo, hi) for ``size`` ranks.  With CSR row pointers the cuts
    balance nonzeros (SpMM work), otherwise rows; every slab is non-empty when n >= size.
    ``plane``: rows per grid plane of a stencil operator (spmm_plan.infer_grid); when the grid
    has at least ``size`` planes the cuts fall on plane boundaries, so every rank's local CSR
    is again a whole-plane stencil for the plane-marching SpMM and its halo is one plane."""
    if size < 1:
        raise ValueError("size must be >= 1")
    if n < size:
        raise ValueError(f"cannot split {n} rows over {size} ranks")
    if plane is not None and plane > 0 and n % plane == 0 and n // plane >= size:
        npl = n // plane
        if rowptr is None:
            pc = [(npl * r) // size for r in range(size + 1)]
        else:
            rp = np.asarray(rowptr, dtype=np.int64)
            work = (rp + np.arange(n + 1, dtype=np.int64))[::plane]  # work at plane boundaries
            tot = int(work[-1])
            pc = [0]
            for r in range(1, size):
                c = int(np.searchsorted(work, (tot * r) // size, side="left"))
                pc.append(min(max(c, pc[-1] + 1), npl - (size - r)))
            pc.append(npl)
        return [(pc[r] * plane, pc[r + 1] * plane) for r in range(size)]
    if rowptr is None:
        cuts = [(n * r) // size for r in range(size + 1)]
    else:
        rp = np.asarray(rowptr, dtype=np.int64)
        nnz = int(rp[-1])
        # balance rows + nnz (row-length work of the dense blocks plus the SpMM gathers)
        work = rp + np.arange(n + 1, dtype=np.int64)
        tot = int(work[-1])
        cuts = [0]
        for r in range(1, size):
            c = int(np.searchsorted(work, (tot * r) // size, side="left"))
            c = min(max(c, cuts[-1] + 1), n - (size - r))
            cuts.append(c)
        cuts.append(n)
        del nnz
    return [(cuts[r], cuts[r + 1]) for r in range(size)]


class HaloPlan:
    """Ghost-row exchange of one rank for a CSR operator split into ``bounds``.

    The ghost rows are kept contiguous with the slab: rank r's extended block covers global
    rows [g_lo, g_hi) = [min col referenced, max col referenced + 1] of its rows, owned rows
    sit at offset ``top = lo - g_lo``, and the local CSR addresses the extended block
    (column index - g_lo).  recv: (peer, a, b) global rows this rank receives; send: (peer,
    a, b) global rows of this rank's slab another rank needs.  Every rank derives the whole
    plan from the host CSR alone (no setup traffic)."""

    def __init__(self, csr, bounds, rank):
        self.bounds = bounds
        self.rank = rank
        ext = [self._extent(csr, lo, hi) for lo, hi in bounds]
        self.ext = ext
        lo, hi = bounds[rank]
        self.lo, self.hi = lo, hi
        self.g_lo, self.g_hi = ext[rank]
        self.top = lo - self.g_lo
        self.n_ext = self.g_hi - self.g_lo
        self.recv = self._ranges(rank, bounds, ext[rank])
        self.send = []
        for peer in range(len(bounds)):
            if peer == rank:
                continue
            for p, a, b in self._ranges(peer, bounds, ext[peer]):
                if p == rank:
                    self.send.append((peer, a, b))

    @staticmethod
    def _extent(csr, lo, hi):
        idx = csr.indices[csr.indptr[lo]:csr.indptr[hi]]
        if idx.size == 0:
            return lo, hi
        return min(lo, int(idx.min())), max(hi, int(idx.max()) + 1)

    @staticmethod
    def _ranges(rank, bounds, extent):
        """(owner, a, b) pieces of [g_lo, lo) and [hi, g_hi) for ``rank``."""
        lo, hi = bounds[rank]
        g_lo, g_hi = extent
        out = []
        for peer, (plo, phi) in enumerate(bounds):
            if peer == rank:
                continue
            for a, b in ((max(plo, g_lo), min(phi, lo)), (max(plo, hi), min(phi, g_hi))):
                if a < b:
                    out.append((peer, a, b))
        return out

    def ghost_rows(self):
        return sum(b - a for _, a, b in self.recv)


def local_rows_csr(csr, lo, hi, col_offset, ncols):
    """Rows [lo, hi) of a scipy CSR with column indices shifted by -col_offset (columns of
    the rank's extended block, ``ncols`` rows of it)."""
    import scipy.sparse as sp

    sub = csr[lo:hi].tocsr()
    sub.sort_indices()
    return sp.csr_matrix((sub.data, sub.indices - col_offset, sub.indptr), shape=(hi - lo, ncols))


def host_csr_of(a):
    """Host CSR of an operator for row partitioning (sparse and diagonal operators)."""
    import scipy.sparse as sp

    if hasattr(a, "_csr"):
        return a._csr.tocsr()
    inner = getattr(a, "inner", None)
    if inner is not None:
        return host_csr_of(inner)
    if type(a).__name__ == "DiagonalOperator":
        return sp.diags(np.asarray(a.diag)).tocsr()
    raise NotImplementedError("row-partitioned runs need a sparse (CSR) or diagonal operator")


# ----------------------------------------------------------------------------- communicators
class Comm:
    """Collectives the row-partitioned solver needs.  Tensors are contiguous and in place."""

    rank = 0
    size = 1

    def allreduce_sum(self, t):
        raise NotImplementedError

    def allreduce_max(self, t):
        raise NotImplementedError

    def exchange(self, sends, recvs):
        """sends/recvs: lists of (peer, tensor); the k-th send to a peer matches that
        peer's k-th recv from this rank."""
        raise NotImplementedError

    def allgather_rows(self, local, bounds):
        """Concatenate every rank's (rows_r x c) block in rank order."""
        raise NotImplementedError

    def reduce_scatter_sum(self, full, chunk):
        """``full`` (contiguous, size * chunk elements): rank r's chunk [r chunk, (r+1) chunk)
        becomes the sum over ranks of that chunk (the other chunks are left undefined)."""
        raise NotImplementedError

    def allgather_chunks(self, full, chunk):
        """``full`` (contiguous, size * chunk elements) holding this rank's chunk at r chunk:
        afterwards every chunk holds its owner's values, on every rank."""
        raise NotImplementedError

    def gather_rows_host(self, local, bounds, mode="all"):
        """Host assembly of a row-partitioned result (numpy rows_r x c per rank) without any
        device-side gather: mode "all" -> the (n x c) array on every rank, "root" -> on rank
        0 (other ranks get None)."""
        raise NotImplementedError

    def barrier(self):
        raise NotImplementedError


def _real(t):
    import torch

    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t.reshape(-1)


class TorchComm(Comm):
    """torch.distributed process group (NCCL across GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        # gloo moves CPU tensors: device tensors are staged through host copies (used to
        # exercise the multi-rank path where only one GPU is available; NCCL is the product)
        self.stage = dist.get_backend(group) == "gloo"

    def _staged(self, t, fn):
        if self.stage and t.is_cuda:
            h = t.cpu()
            fn(h)
            t.copy_(h)
        else:
            fn(t)

    def allreduce_sum(self, t):
        self._staged(t, lambda x: self.dist.all_reduce(x, op=self.dist.ReduceOp.SUM, group=self.group))

    def allreduce_max(self, t):
        self._staged(t, lambda x: self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX, group=self.group))

    def _global(self, peer):
        return peer if self.group is None else self.dist.get_global_rank(self.group, peer)

    def exchange(self, sends, recvs):
        dist = self.dist
        if self.stage:
            sends = [(p, t.cpu()) for p, t in sends]
            hrecv = [(p, t, t.new_empty(t.shape, device="cpu")) for p, t in recvs]
            recvs = [(p, h) for p, _, h in hrecv]
        ops = [dist.P2POp(dist.isend, t, self._global(p), self.group) for p, t in sends]
        ops += [dist.P2POp(dist.irecv, t, self._global(p), self.group) for p, t in recvs]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if self.stage:
            for _, t, h in hrecv:
                t.copy_(h)

    def allgather_rows(self, local, bounds):
        import torch

        dev = "cpu" if self.stage else local.device
        rows = max(b - a for a, b in bounds)
        pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
        pad[: local.shape[0]] = local
        out = torch.empty((self.size * rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
        self.dist.all_gather_into_tensor(out, pad, group=self.group)
        full = torch.cat([out[r * rows: r * rows + (b - a)] for r, (a, b) in enumerate(bounds)])
        return full.to(local.device)

    def reduce_scatter_sum(self, full, chunk):
        if self.stage:  # gloo: no reduce-scatter on staged tensors -- a sum-allreduce is a superset
            self.allreduce_sum(full)
            return
        f = _real(full)
        c = chunk * (2 if full.is_complex() else 1)
        # in place: the output chunk is this rank's slice of the input (NCCL's in-place form)
        self.dist.reduce_scatter_tensor(f[self.rank * c:(self.rank + 1) * c], f, group=self.group)

    def allgather_chunks(self, full, chunk):
        f = _real(full)
        c = chunk * (2 if full.is_complex() else 1)
        if self.stage:
            h = f.cpu()
            parts = list(h.split(c))
            self.dist.all_gather(parts, parts[self.rank].clone(), group=self.group)
            f.copy_(h)
            return
        self.dist.all_gather_into_tensor(f, f[self.rank * c:(self.rank + 1) * c], group=self.group)

    def _host_group(self):
        g = getattr(self, "_gloo", None)
        if g is None:
            g = self._gloo = self.dist.new_group(backend="gloo") if not self.stage else self.group
        return g

    def gather_rows_host(self, local, bounds, mode="all"):
        """Rows over a host (gloo) group: rank order, padded to the largest slab.  One
        process per GPU on one node in practice, so this is a host-memory copy per rank."""
        import torch

        g = self._host_group()
        rows = max(b - a for a, b in bounds)
        pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=torch.from_numpy(local[:0]).dtype)
        pad[: local.shape[0]] = torch.from_numpy(local)
        if mode == "root":
            parts = [torch.empty_like(pad) for _ in range(self.size)] if self.rank == 0 else None
            self.dist.gather(pad, parts, dst=self._global(0), group=g)
        else:
            parts = [torch.empty_like(pad) for _ in range(self.size)]
            self.dist.all_gather(parts, pad, group=g)
        if parts is None:
            return None
        return np.concatenate([p[: b - a].numpy() for p, (a, b) in zip(parts, bounds)])

    def barrier(self):
        self.dist.barrier(group=self.group)


class _ThreadShared:
    def __init__(self, size):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size
        self.mail = {}


class ThreadComm(Comm):
    """Ranks as threads of one process (sharded solver on one device, for tests).  Sums are
    taken in rank order, so every rank holds bitwise the same result."""

    def __init__(self, shared, rank):
        self.sh = shared
        self.rank = rank
        self.size = shared.size

    @staticmethod
    def _sync(t):
        if t.is_cuda:
            import torch

            torch.cuda.current_stream(t.device).synchronize()

    def _gather(self, t):
        self._sync(t)
        self.sh.slots[self.rank] = t.clone()
        self._sync(t)
        self.sh.barrier.wait()
        vals = list(self.sh.slots)
        self.sh.barrier.wait()
        return vals

    def allreduce_sum(self, t):
        vals = self._gather(t)
        acc = vals[0].clone()
        for v in vals[1:]:
            acc += v
        t.copy_(acc)
        self._sync(t)

    def allreduce_max(self, t):
        import torch

        vals = self._gather(t)
        acc = vals[0].clone()
        for v in vals[1:]:
            acc = torch.maximum(acc, v)
        t.copy_(acc)
        self._sync(t)

    def exchange(self, sends, recvs):
        for p, t in sends:
            self._sync(t)
        for k, (p, t) in enumerate(sends):
            key = (self.rank, p, sum(1 for q, _ in sends[:k] if q == p))
            self.sh.mail[key] = t.clone()
            self._sync(t)
        self.sh.barrier.wait()
        for k, (p, t) in enumerate(recvs):
            key = (p, self.rank, sum(1 for q, _ in recvs[:k] if q == p))
            t.copy_(self.sh.mail[key])
            self._sync(t)
        self.sh.barrier.wait()
        if self.rank == 0:
            self.sh.mail.clear()
        self.sh.barrier.wait()

    def allgather_rows(self, local, bounds):
        import torch

        vals = self._gather(local.contiguous())
        return torch.cat(vals)

    def reduce_scatter_sum(self, full, chunk):
        vals = self._gather(full)
        lo, hi = self.rank * chunk, (self.rank + 1) * chunk
        acc = vals[0].reshape(-1)[lo:hi].clone()
        for v in vals[1:]:
            acc += v.reshape(-1)[lo:hi]
        full.reshape(-1)[lo:hi].copy_(acc)
        self._sync(full)

    def allgather_chunks(self, full, chunk):
        vals = self._gather(full)
        f = full.reshape(-1)
        for r, v in enumerate(vals):
            if r != self.rank:
                f[r * chunk:(r + 1) * chunk].copy_(v.reshape(-1)[r * chunk:(r + 1) * chunk])
        self._sync(full)

    def gather_rows_host(self, local, bounds, mode="all"):
        self.sh.slots[self.rank] = local
        self.sh.barrier.wait()
        vals = list(self.sh.slots)
        self.sh.barrier.wait()
        if mode == "root" and self.rank != 0:
            return None
        return np.concatenate(vals)

    def barrier(self):
        self.sh.barrier.wait()


def thread_comms(size):
    sh = _ThreadShared(size)
    return [ThreadComm(sh, r) for r in range(size)]


def dist_ppcg_solve(a, t=None, x0=None, opts=None, comm=None, gather=None):
    """ppcg_solve over a row partition (one rank per GPU).  Every rank passes the same
    operator, preconditioner, x0 and options.  The eigenvectors are assembled on the host
    from each rank's row slab (no device-side gather; PPCGSolver.finish):
      gather="all"  -- every rank receives the full (n, k) vectors;
      gather="root" -- rank 0 does, the other ranks receive their own rows [lo, hi)
                       (``diagnostics["vector_rows"]``);
      None          -- "all" up to 8 GB of vectors, else "root" (config 5: 137 GB).
    Everything else in the SolveReport is identical on every rank."""
    from .ppcg import PPCGSolver

    if opts is None:
        raise ValueError("opts is required")
    opts.validate()
    s = PPCGSolver(a, t, x0, opts, comm=comm).start()
    while not s.step():
        pass
    return s.finish(gather=gather)
