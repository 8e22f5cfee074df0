"""Multi-threaded host draw of ``numpy.random.default_rng(seed).standard_normal(count)``,
bit-identical to the sequential draw.

The reference draws the initial block X0 with numpy's PCG64 generator (ppcg.py:414-438) and
parity requires the same X0, so it cannot come from a device RNG.  At
config 2 the sequential draw (110,592 x 523 normals) takes ~0.7 s on one core, longer than
20 solver iterations on the GPU.  It parallelises because PCG64 can jump ahead:

  * numpy's normal sampler (a ziggurat) consumes one 64-bit draw per normal on its fast
    path and a few more on its rare slow paths, so chunk c of the output starts at an
    unknown stream position near c*M;
  * every chunk is therefore drawn speculatively from stream position c*M (PCG64.advance);
    that chain coincides with the true sequence from the first stream position where both
    start a normal -- within a few normals, since almost every normal is a one-draw fast
    path;
  * the chains are spliced where a run of ``_RUN`` consecutive values of chunk c appears in
    chunk c-1's overlap (32 identical doubles cannot occur by accident), and any shortfall
    at the end is drawn sequentially from the last chunk's generator, which by then sits on
    the true stream.
If a splice point is not found the function falls back to the sequential draw, so the
result is always exactly the sequential one.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_RUN = 32
_MIN_PARALLEL = 1 << 21


def _threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return max(1, os.cpu_count() or 1)


def _find_splice(prev, prev_from, nxt):
    """(t, j): prev[t:t+_RUN] == nxt[j:j+_RUN] with t >= prev_from and the smallest j, or None."""
    lo = max(prev_from, len(prev) - len(prev) // 8 - 4 * _RUN)
    win = prev[lo:len(prev) - _RUN]
    for j in range(0, min(256, len(nxt) - _RUN)):
        for t in np.flatnonzero(win == nxt[j]):
            t = int(t) + lo
            if np.array_equal(prev[t:t + _RUN], nxt[j:j + _RUN]):
                return t, j
    return None


class FlatDraw:
    """The draw as spliced segments, never assembled unless asked: ``segs`` holds
    (i0, i1, arr, j0) with output[i0:i1] == arr[j0:j0 + i1 - i0], covering [0, count).
    ``copy_range`` lets an upload fill pinned staging straight from the chunk buffers
    (one host pass over the data instead of two)."""

    def __init__(self, count, segs):
        self.count = count
        self.segs = segs

    def _resolve(self, upto):
        return self.segs

    def copy_range(self, a, b, dst):
        """dst[:] = output[a:b] (dst: 1-D float64 view of length b - a)."""
        for i0, i1, arr, j0 in self._resolve(b):
            lo, hi = max(a, i0), min(b, i1)
            if lo < hi:
                dst[lo - a:hi - a] = arr[j0 + lo - i0:j0 + hi - i0]

    def array(self, threads=None):
        out = np.empty(self.count)
        segs = self._resolve(self.count)
        if len(segs) == 1:
            i0, i1, arr, j0 = segs[0]
            out[:] = arr[j0:j0 + i1 - i0]
            return out

        def copy(sg):
            i0, i1, arr, j0 = sg
            out[i0:i1] = arr[j0:j0 + i1 - i0]

        with ThreadPoolExecutor(max_workers=min(len(segs), threads or _threads())) as ex:
            list(ex.map(copy, segs))
        return out


class ChainedDraw(FlatDraw):
    """FlatDraw whose chains are still being drawn: the chunks run on a thread pool in stream
    order (several per thread), and a range of the output becomes available once the chunks
    up to the one after it are drawn and spliced -- so an upload of the first rows overlaps
    the draw of the later ones.  ``_resolve(upto)`` blocks until output [0, upto) is covered."""

    def __init__(self, seed, count, nchunk, M, extra, bufs, threads):
        self.count, self.seed, self.nchunk = count, seed, nchunk
        self.segs = []
        self._starts = [(0, 0)]   # (output index, chunk offset) where chunk c takes over
        self._next = 0            # next chunk to splice
        self._filled = 0
        self._lock = threading.Lock()

        def draw(c):
            bg = np.random.PCG64(seed)
            if c:
                bg.advance(c * M)
            g = np.random.Generator(bg)
            if bufs is not None:
                return g, g.standard_normal(M + extra, out=bufs[c])
            return g, g.standard_normal(M + extra)

        self._pool = ThreadPoolExecutor(max_workers=min(threads, nchunk))
        self._futs = [self._pool.submit(draw, c) for c in range(nchunk)]
        self._pool.shutdown(wait=False)

    def wait(self):
        """All chains drawn (their buffers may be reused after this)."""
        for f in self._futs:
            f.exception()

    def _sequential(self):
        self.segs = [(0, self.count, np.random.default_rng(self.seed).standard_normal(self.count), 0)]
        self._filled = self.count
        self._next = self.nchunk

    def _resolve(self, upto):
        upto = min(upto, self.count)
        with self._lock:
            while self._filled < upto:
                c = self._next
                if c >= self.nchunk:  # shortfall: the last chain sits on the true stream
                    g, _ = self._futs[-1].result()
                    self.segs.append((self._filled, self.count, g.standard_normal(self.count - self._filled), 0))
                    self._filled = self.count
                    break
                _, arr = self._futs[c].result()
                i, j = self._starts[c]
                if c + 1 < self.nchunk:
                    sp = _find_splice(arr, j, self._futs[c + 1].result()[1])
                    if sp is None:  # never seen; the result stays exactly the sequential draw
                        self.wait()
                        self._sequential()
                        break
                    t, jn = sp
                    end = i + (t - j)
                    self._starts.append((end, jn))
                else:
                    end = i + len(arr) - j
                end = min(end, self.count)
                if end > i:
                    self.segs.append((i, end, arr, j))
                    self._filled = end
                self._next = c + 1
            return list(self.segs)


_SCRATCH = threading.local()
_CHUNKS_PER_THREAD = 4


def normal_draw(seed, count, threads=None, reuse=False):
    """FlatDraw of ``np.random.default_rng(seed).standard_normal(count)``; returns at once,
    the chains complete in the background (ChainedDraw).  With ``reuse`` the chunks are drawn
    into this thread's scratch buffers from the previous call (no fresh pages to fault in), so
    the result is only valid until the thread's next ``reuse`` call -- for callers that consume
    it at once (the X0 upload)."""
    threads = threads or _threads()
    if count < _MIN_PARALLEL or threads < 2:
        return FlatDraw(count, [(0, count, np.random.default_rng(seed).standard_normal(count), 0)])
    nchunk = min(_CHUNKS_PER_THREAD * threads, max(2, count // (_MIN_PARALLEL // 2)))
    M = -(-count // nchunk)           # nominal stream draws per chunk
    extra = M // 16 + 4096            # overlap covering the slow-path surplus of a chunk

    bufs = None
    if reuse:
        last = getattr(_SCRATCH, "last", None)
        if last is not None:
            last.wait()  # its chains write the scratch buffers
        bufs = getattr(_SCRATCH, "bufs", None)
        if bufs is None or len(bufs) != nchunk or len(bufs[0]) != M + extra:
            bufs = _SCRATCH.bufs = [np.empty(M + extra) for _ in range(nchunk)]
    d = ChainedDraw(seed, count, nchunk, M, extra, bufs, threads)
    if reuse:
        _SCRATCH.last = d
    return d


def standard_normal(seed, count, threads=None):
    """Flat float64 array equal to ``np.random.default_rng(seed).standard_normal(count)``."""
    return normal_draw(seed, count, threads).array(threads)
