// Tall-skinny Gram products C = X^T Y on FP64 tensor cores (DMMA, mma.sync m8n8k4).
//
// Replaces the reference's block_inner (blockeig core.py:43-49, `x.conj().T @ y`, OpenBLAS
// dgemm) at every call site on the PPCG hot path: the full Grams of _apply_projection
// (ppcg.py:441-445), the orthonormality Gram (ppcg.py:448-453), the residual Gram
// (ppcg.py:630,758), proj_defect (ppcg.py:688-692) and the per-q-block pencil Grams of
// _solve_subblock_pencil (ppcg.py:206-211).
//
// Design:
//  * the reduction dimension is the row count n (huge); the output is small.  Rows are
//    split into chunks; each CTA computes one BM x BN output tile over one chunk, 16 rows
//    per stage through a cp.async ring (16-byte copies when offsets allow, else 8-byte).
//  * configurations follow the shape that saturates the B200 DMMA pipe (measured: cuBLAS'
//    64x128x16, 3-stage, 4-warp DGEMM runs the tensor pipe at 96%): 4 warps with 32x64 warp
//    tiles, two CTAs per SM so one CTA's barrier waits are covered by the other's DMMAs.
//    "big" = 64x128 (k_total-wide Grams), "small" = 64x64 (pencil-sized outputs).
//  * fragments are double buffered; warps with a fully valid tile issue unpredicated DMMAs
//    (a predicated mma.sync costs a WARPSYNC + NOP per instruction).
//  * split-K partials go to a workspace; the LAST CTA to finish a tile (atomic ticket)
//    sums the partials in fixed chunk order -> bitwise run-to-run deterministic, one launch.
//  * operands are virtual concatenations of up to 3 column segments of row-major blocks,
//    so S = [X_j | W_j | P_j] of a subblock is never materialised.
//  * symmetric mode (X == Y) skips tiles below the diagonal and mirrors the upper triangle,
//    so the result is exactly symmetric.
//  * row strides of BM+4 / BN+4 (= 4 mod 16 doubles) make the half-warp fragment loads
//    (4 rows x 4 doubles) conflict-free.
#include <cuda.h>
#include "common.cuh"

namespace bk {

constexpr int G_BK = 16;

struct Seg {
  const double* p;
  int64_t ld;
  int64_t col0;
  int width;
};

struct GramProblem {
  Seg xs[3];
  Seg ys[3];
  int nxs, nys;
  int M, N;
  double* C;
  int64_t ldc;
  int symmetric;
  int tiles_m, tiles_n, ntiles;
  // strip problems of a split Gram: entry (i, j) lands at C[(i + row_off)][(j + col_off)],
  // transposed if trans; mirror also writes the transpose position when it lies outside
  // the strip (global row < col_off)
  int row_off, col_off, trans, mirror;
};

struct GramParams {
  int nprob;
  int explicit_list;          // 1: problems in `prob`; 0: subblock mode
  GramProblem prob[4];
  // subblock mode (ppcg.py:206-211): per block j two problems: S^T(AS) and S^T S
  const double* sX;
  const double* sW;
  const double* sP;
  const double* sAX;
  const double* sAW;
  const double* sAP;
  int64_t sld;
  int64_t sc0;
  int k_act, q, has_p, dmax;
  double* outA;               // nb blocks of dmax x dmax (A_hat raw)
  double* outB;               // nb blocks of dmax x dmax (B_hat raw)
  // common
  int64_t nrows;
  int nchunks;
  int64_t chunk_rows;
  int max_tiles;              // tiles per problem slot in the grid
  int vec16;                  // all segment offsets/leading dims even: 16-byte copies
  int allow_fast;             // fast-path switch (PPCG_GRAM_FAST=0 disables, for A/B checks)
  int bulk;                   // host: run gram_bulk_kernel (even row strides; PPCG_GRAM_BULK=0 disables)
  int chunk_major;            // block order (tile, problem, chunk) instead of (tile, chunk, problem)
  int force_chunks;           // host: split-K chunk count fixed by the caller (0 = choose)
  double* ws;                 // partials: [prob][tile][chunk][BM*BN]
  int* tickets;               // [prob][tile]
};

template <int BM, int BN>
BK_DEV void subblock_problem(const GramParams& P, int b, GramProblem& g) {
  g = GramProblem{};  // no strip offsets / transposition / mirroring in subblock mode
  int j = b >> 1, kind = b & 1;
  int lo = j * P.q;
  int w = min(P.q, P.k_act - lo);
  int nseg = P.has_p ? 3 : 2;
  const double* xs[3] = {P.sX, P.sW, P.sP};
  const double* as[3] = {P.sAX, P.sAW, P.sAP};
  for (int s = 0; s < 3; ++s) {
    g.xs[s] = {xs[s], P.sld, P.sc0 + lo, w};
    g.ys[s] = {kind ? xs[s] : as[s], P.sld, P.sc0 + lo, w};
  }
  g.nxs = g.nys = nseg;
  g.M = g.N = nseg * w;
  g.C = (kind ? P.outB : P.outA) + (int64_t)j * P.dmax * P.dmax;
  g.ldc = P.dmax;
  g.symmetric = kind;
  g.tiles_m = (g.M + BM - 1) / BM;
  g.tiles_n = (g.N + BN - 1) / BN;
  g.ntiles = g.tiles_m * g.tiles_n;
}

// pointer to virtual column c (nullptr if outside the segments); ld of its segment
BK_DEV const double* seg_col(const Seg* segs, int nseg, int c, int64_t& ld, int& seg) {
  int off = 0;
  for (int s = 0; s < nseg; ++s) {
    if (c < off + segs[s].width) {
      ld = segs[s].ld;
      seg = s;
      return segs[s].p + segs[s].col0 + (c - off);
    }
    off += segs[s].width;
  }
  ld = 0;
  seg = -1;
  return nullptr;
}

// Per-thread loader for a pair of adjacent virtual columns
struct PairCol {
  const double* p0;   // column c
  const double* p1;   // column c+1
  int64_t ld0, ld1;
  bool v0, v1, fused; // fused: c and c+1 contiguous and 16-byte aligned -> one 16-byte copy
};

BK_DEV PairCol make_pair(const Seg* segs, int nseg, int M, int c, bool vec16) {
  PairCol pc;
  int s0, s1;
  pc.p0 = seg_col(segs, nseg, c, pc.ld0, s0);
  pc.p1 = seg_col(segs, nseg, c + 1, pc.ld1, s1);
  pc.v0 = pc.p0 != nullptr && c < M;
  pc.v1 = pc.p1 != nullptr && c + 1 < M;
  pc.fused = vec16 && pc.v0 && pc.v1 && s0 == s1 && ((reinterpret_cast<uintptr_t>(pc.p0) & 15) == 0);
  if (!pc.v0) pc.p0 = segs[0].p;
  if (!pc.v1) pc.p1 = segs[0].p;
  return pc;
}

// Fast-path source of a column pair: a 16-byte aligned address readable on every row.
//  * both columns valid and contiguous                -> the pair itself;
//  * last valid column c with c + 1 past the operand  -> the pair if c + 1 is still inside the
//    row stride (the padding column: read, never used);
//  * both columns past the operand                    -> the tile's first pair (read, never used).
// Values of columns >= M only reach accumulator rows/columns that are never stored, so edge
// tiles can run the unpredicated full-tile loop.  ok = false: this tile takes the general path.
BK_DEV const double* fast_pair(const Seg* segs, int nseg, int M, int c, int c_tile0, bool vec16, int64_t& ld,
                               bool& ok) {
  ok = false;
  ld = 0;
  if (!vec16) return nullptr;
  int64_t ld0, ld1;
  int s0, s1;
  const double* p0 = seg_col(segs, nseg, c, ld0, s0);
  const double* p1 = seg_col(segs, nseg, c + 1, ld1, s1);
  const bool v0 = p0 != nullptr && c < M, v1 = p1 != nullptr && c + 1 < M;
  if (v0 && v1) {
    ok = s0 == s1 && (reinterpret_cast<uintptr_t>(p0) & 15) == 0;
    ld = ld0;
    return p0;
  }
  if (v0) {  // c + 1 past the operand: inside the row stride?
    int off = 0;
    for (int s = 0; s < s0; ++s) off += segs[s].width;
    const int64_t phys = segs[s0].col0 + (c - off) + 1;
    ok = phys < segs[s0].ld && (reinterpret_cast<uintptr_t>(p0) & 15) == 0;
    ld = ld0;
    return p0;
  }
  const double* pt = seg_col(segs, nseg, c_tile0, ld0, s0);
  const double* pt1 = seg_col(segs, nseg, c_tile0 + 1, ld1, s1);
  ok = pt != nullptr && pt1 != nullptr && s0 == s1 && c_tile0 + 1 < M && (reinterpret_cast<uintptr_t>(pt) & 15) == 0;
  ld = ld0;
  return pt;
}

BK_DEV void load_pair(double* dst, const PairCol& pc, int64_t row, bool rv) {
  if (pc.fused) {
    cp_async16(dst, rv ? pc.p0 + row * pc.ld0 : pc.p0, rv ? 16 : 0);
  } else {
    cp_async8(dst, rv && pc.v0 ? pc.p0 + row * pc.ld0 : pc.p0, rv && pc.v0);
    cp_async8(dst + 1, rv && pc.v1 ? pc.p1 + row * pc.ld1 : pc.p1, rv && pc.v1);
  }
}

template <int BM_, int BN_, int STAGES_, int MINB_, int SLOTS_, int WARPS_M_ = 2, int WARPS_N_ = 2>
struct GCfg {
  static constexpr int BM = BM_, BN = BN_, STAGES = STAGES_, MINB = MINB_, SLOTS_PER_SM = SLOTS_;
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int WM = BM / WARPS_M / 8, WN = BN / WARPS_N / 8;
  static constexpr int LDX = BM + 4, LDY = BN + 4; // = 4 mod 16
  static constexpr int XPAIRS = G_BK * BM / 2 / THREADS, YPAIRS = G_BK * BN / 2 / THREADS;
  static constexpr int XSTAGE = G_BK * LDX, YSTAGE = G_BK * LDY;
  static constexpr int SMEM = STAGES * (XSTAGE + YSTAGE) * (int)sizeof(double);
};
using Big = GCfg<64, 128, 4, 2, 2>;
using Small = GCfg<64, 64, 4, 3, 3>;
// subblock pencil Grams of width 3q = 96 (q = 32, config 2): one 96 x 96 tile, 3 x 2 warps
// of 32 x 48 -- 64 x 64 tiles would leave 44% of the DMMA work on padding (4 tiles for 96^2)
using Sb96 = GCfg<96, 96, 4, 2, 2, 3, 2>;
// narrow strips left over when a Gram's width is not a multiple of 64 (523 = 8 x 64 + 11):
// 64 x 16 tiles, 4 warps of 16 x 16, small enough for 4 CTAs per SM
using Strip = GCfg<64, 16, 4, 4, 4, 4, 1>;

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gram_kernel(const __grid_constant__ GramParams P) {
  constexpr int BM = C::BM, BN = C::BN, LDX = C::LDX, LDY = C::LDY, WM = C::WM, WN = C::WN, ST = C::STAGES;
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                    // [STAGES][BK][LDX]
  double* Ys = smem + ST * C::XSTAGE;   // [STAGES][BK][LDY]
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bid = blockIdx.x;
  const int slot = (int)(bid % P.max_tiles);
  const int chunk = P.chunk_major ? (int)(bid / ((int64_t)P.max_tiles * P.nprob))
                                  : (int)((bid / P.max_tiles) % P.nchunks);
  const int pidx = P.chunk_major ? (int)((bid / P.max_tiles) % P.nprob) : (int)(bid / ((int64_t)P.max_tiles * P.nchunks));

  GramProblem g;
  if (P.explicit_list) g = P.prob[pidx];
  else subblock_problem<BM, BN>(P, pidx, g);
  if (slot >= g.ntiles) return;
  const int ti = slot / g.tiles_n, tj = slot % g.tiles_n;
  const int m0 = ti * BM, n0 = tj * BN;
  if (g.symmetric && n0 + BN <= m0) return;  // entirely below the diagonal: mirrored

  const int64_t r_begin = (int64_t)chunk * P.chunk_rows;
  const int64_t r_end = lmin(P.nrows, r_begin + P.chunk_rows);
  const int nstages = (int)((r_end - r_begin + G_BK - 1) / G_BK);

  // loader: X pairs: column (tid % (BM/2)) * 2, rows tid / (BM/2) + step i; Y likewise
  constexpr int XCPR = BM / 2, YCPR = BN / 2;
  const int xc = (tid % XCPR) * 2, xr = tid / XCPR;
  const int yc = (tid % YCPR) * 2, yr = tid / YCPR;
  const PairCol px = make_pair(g.xs, g.nxs, g.M, m0 + xc, P.vec16);
  const PairCol py = make_pair(g.ys, g.nys, g.N, n0 + yc, P.vec16);

  // Fast path (CTA-uniform): every column pair of the tile is one aligned 16-byte copy and
  // the chunk is whole stages -> unpredicated cp.async with per-thread running pointers and
  // full warp tiles only.  Edge tiles, odd offsets and ragged chunks take the general path.
  int64_t fldx, fldy;
  bool okx, oky;
  const double* fpx = fast_pair(g.xs, g.nxs, g.M, m0 + xc, m0, P.vec16, fldx, okx);
  const double* fpy = fast_pair(g.ys, g.nys, g.N, n0 + yc, n0, P.vec16, fldy, oky);
  const bool fast = __syncthreads_and(okx && oky) && ((r_end - r_begin) % G_BK) == 0 && P.allow_fast;

  auto load_stage = [&](int s, int st) {
    const int64_t rb = r_begin + (int64_t)s * G_BK;
    double* xd = Xs + st * C::XSTAGE;
    double* yd = Ys + st * C::YSTAGE;
#pragma unroll
    for (int i = 0; i < C::XPAIRS; ++i) {
      const int kr = xr + (C::THREADS / XCPR) * i;
      const int64_t row = rb + kr;
      load_pair(xd + kr * LDX + xc, px, row, row < r_end);
    }
#pragma unroll
    for (int i = 0; i < C::YPAIRS; ++i) {
      const int kr = yr + (C::THREADS / YCPR) * i;
      const int64_t row = rb + kr;
      load_pair(yd + kr * LDY + yc, py, row, row < r_end);
    }
  };
  const double* fx = fpx + (r_begin + xr) * fldx;
  const double* fy = fpy + (r_begin + yr) * fldy;
  const int64_t fxs = (int64_t)(C::THREADS / XCPR) * fldx, fys = (int64_t)(C::THREADS / YCPR) * fldy;
  auto load_stage_fast = [&](int s, int st) {
    double* xd = Xs + st * C::XSTAGE + xr * LDX + xc;
    double* yd = Ys + st * C::YSTAGE + yr * LDY + yc;
    const double* gx = fx + (int64_t)s * G_BK * fldx;
    const double* gy = fy + (int64_t)s * G_BK * fldy;
#pragma unroll
    for (int i = 0; i < C::XPAIRS; ++i) cp_async16(xd + (C::THREADS / XCPR) * i * LDX, gx + i * fxs, 16);
#pragma unroll
    for (int i = 0; i < C::YPAIRS; ++i) cp_async16(yd + (C::THREADS / YCPR) * i * LDY, gy + i * fys, 16);
  };

  // warp placement (2 x 2); valid DMMA tiles (skip tiles outside M x N / below the diagonal)
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int wm0 = m0 + wm * 8 * WM, wn0 = n0 + wn * 8 * WN;
  const int mtv = max(0, min(WM, (g.M - wm0 + 7) / 8));
  const int ntv = max(0, min(WN, (g.N - wn0 + 7) / 8));
  const bool below = g.symmetric && (wn0 + 8 * WN <= wm0);
  const bool warp_active = mtv > 0 && ntv > 0 && !below;
  const bool full_tile = mtv == WM && ntv == WN;

  double acc[WM][WN][2];
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int fr = lane & 3, fc = lane >> 2;  // fragment: k = lane%4, m/n = lane/4
  const int xoff = fr * LDX + wm * 8 * WM + fc, yoff = fr * LDY + wn * 8 * WN + fc;
  if (fast) {
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
      if (s < nstages) load_stage_fast(s, s);
      cp_async_commit();
    }
    for (int s = 0; s < nstages; ++s) {
      cp_async_wait<ST - 2>();
      __syncthreads();
      {
        const int sn = s + ST - 1;
        if (sn < nstages) load_stage_fast(sn, sn % ST);
        cp_async_commit();
      }
      if (warp_active) {  // partially valid warps run the full tile (extra entries are never stored)
        const double* xs = Xs + (s % ST) * C::XSTAGE + xoff;
        const double* ys = Ys + (s % ST) * C::YSTAGE + yoff;
        double af[2][WM], bf[2][WN];
#pragma unroll
        for (int a = 0; a < WM; ++a) af[0][a] = lds64(xs + a * 8);
#pragma unroll
        for (int b = 0; b < WN; ++b) bf[0][b] = lds64(ys + b * 8);
#pragma unroll
        for (int kq = 0; kq < G_BK / 4; ++kq) {
          const int cur = kq & 1;
          dmma_step_il<WM, WN>(acc, af[cur], bf[cur], af[cur ^ 1], bf[cur ^ 1], xs + (kq + 1) * 4 * LDX, 8,
                               ys + (kq + 1) * 4 * LDY, 8, kq + 1 < G_BK / 4);
        }
      }
    }
  } else {
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nstages) load_stage(s, s);
    cp_async_commit();
  }
  for (int s = 0; s < nstages; ++s) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    {
      const int sn = s + ST - 1;
      if (sn < nstages) load_stage(sn, sn % ST);
      cp_async_commit();
    }
    if (warp_active) {
      const double* xs = Xs + (s % ST) * C::XSTAGE + xoff;
      const double* ys = Ys + (s % ST) * C::YSTAGE + yoff;
      double af[2][WM], bf[2][WN];
#pragma unroll
      for (int a = 0; a < WM; ++a) af[0][a] = lds64(xs + a * 8);
#pragma unroll
      for (int b = 0; b < WN; ++b) bf[0][b] = lds64(ys + b * 8);
      if (full_tile) {
#pragma unroll
        for (int kq = 0; kq < G_BK / 4; ++kq) {
          const int cur = kq & 1;
          dmma_step_il<WM, WN>(acc, af[cur], bf[cur], af[cur ^ 1], bf[cur ^ 1], xs + (kq + 1) * 4 * LDX, 8,
                               ys + (kq + 1) * 4 * LDY, 8, kq + 1 < G_BK / 4);
        }
      } else {
#pragma unroll
        for (int kq = 0; kq < G_BK / 4; ++kq) {
          const int cur = kq & 1;
          if (kq + 1 < G_BK / 4) {
#pragma unroll
            for (int a = 0; a < WM; ++a) af[cur ^ 1][a] = xs[(kq + 1) * 4 * LDX + a * 8];
#pragma unroll
            for (int b = 0; b < WN; ++b) bf[cur ^ 1][b] = ys[(kq + 1) * 4 * LDY + b * 8];
          }
          dmma_block<WM, WN, false>(acc, af[cur], bf[cur], mtv, ntv);
        }
      }
    }
  }
  }
  cp_async_wait<0>();

  // ---- epilogue: (a,b,e) -> tile row wm*8WM + a*8 + lane/4, col wn*8WN + b*8 + 2*(lane%4) + e
  auto store_final = [&](int lrow, int lcol, double v) {
    const int gi = m0 + lrow, gj = n0 + lcol;
    if (gi >= g.M || gj >= g.N) return;
    if (g.symmetric) {
      if (gi > gj) return;  // upper triangle, mirrored
      g.C[(int64_t)gi * g.ldc + gj] = v;
      g.C[(int64_t)gj * g.ldc + gi] = v;
    } else {
      int r = gi + g.row_off, c = gj + g.col_off;
      if (g.trans) { const int t = r; r = c; c = t; }
      g.C[(int64_t)r * g.ldc + c] = v;
      if (g.mirror && r < g.col_off) g.C[(int64_t)c * g.ldc + r] = v;
    }
  };

  if (P.nchunks == 1) {
    if (!warp_active) return;
#pragma unroll
    for (int a = 0; a < WM; ++a)
#pragma unroll
      for (int b = 0; b < WN; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          store_final(wm * 8 * WM + a * 8 + (lane >> 2), wn * 8 * WN + b * 8 + 2 * (lane & 3) + e, acc[a][b][e]);
    return;
  }

  const int64_t tile_id = (int64_t)pidx * P.max_tiles + slot;
  double* part = P.ws + (tile_id * P.nchunks + chunk) * (BM * BN);
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b)
      *reinterpret_cast<double2*>(part + (wm * 8 * WM + a * 8 + (lane >> 2)) * BN + wn * 8 * WN + b * 8 +
                                  2 * (lane & 3)) = make_double2(acc[a][b][0], acc[a][b][1]);
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&P.tickets[tile_id], 1) == P.nchunks - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double* base = P.ws + tile_id * P.nchunks * (BM * BN);
  for (int e = tid; e < BM * BN; e += C::THREADS) {
    double v = 0.0;
    for (int c = 0; c < P.nchunks; ++c) v += __ldcg(base + (int64_t)c * (BM * BN) + e);
    store_final(e / BN, e % BN, v);
  }
  if (tid == 0) P.tickets[tile_id] = 0;  // reset for the next launch (stream-ordered)
}

// ---------------------------------------------------------------------------------------
// Warp-specialised variant (the default wherever row strides are even): one producer warp
// streams each stage with bulk async copies (cp.async.bulk, one per row piece, completing
// on the stage's "full" mbarrier); the MMA warps wait on it and release the stage through an
// "empty" mbarrier.  The MMA warps issue no copy instructions and no CTA-wide barriers:
// the DMMA mainloop probe measured 34.2 TF/s for this scheme vs 31.2 for the cp.async ring
// on the same HBM stream (profiles/dmma_loop_probe_r01.json).
//  * explicit problems (one segment per operand) may start at an odd column: the copy starts
//    one column early and the tile sits one double right in shared memory (sh = 1), so every
//    copy is 16-byte aligned -- odd locked counts L no longer drop to 8-byte copies;
//  * subblock problems lay segments out at even ("padded") offsets: segment s, column off at
//    tile column s * wp + off, wp = w rounded up to even; the epilogue maps back;
//  * rows past the chunk end in a partial last stage are zero-filled by the producer.
// Copies never run past an even row stride (host-checked), and tile columns past the
// operand only feed accumulator entries that are never stored.
struct Pieces {
  const double* src[3];  // global address of the piece's first copied column in row 0
  int soff[3];           // shared-memory column of that column
  int len[3];            // doubles per row (even)
  int n;
  int64_t ld;
};

BK_DEV int pad_map(int p, int wp, int w) {  // padded tile column -> virtual column (or -1)
  if (wp == 0) return p;
  const int s = p / wp, off = p - s * wp;
  return off < w ? s * w + off : -1;
}

// pieces of a tile [c0, c0 + B) of one operand; sh = shared-memory shift of column 0
BK_DEV void tile_pieces(const GramProblem& g, bool xop, int c0, int B, int wp, Pieces& pc, int& sh) {
  const Seg* segs = xop ? g.xs : g.ys;
  const int nseg = xop ? g.nxs : g.nys;
  const int M = xop ? g.M : g.N;
  pc.n = 0;
  pc.ld = segs[0].ld;
  sh = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    pc.src[i] = segs[0].p;
    pc.soff[i] = 0;
    pc.len[i] = 0;
  }
  if (wp == 0) {  // one segment, any column parity
    const double* p0 = segs[0].p + segs[0].col0;
    sh = (int)((reinterpret_cast<uintptr_t>(p0) >> 3) & 1);
    const int width = min(B, M - c0);
    pc.src[0] = p0 + c0 - sh;
    pc.soff[0] = 0;
    pc.len[0] = (width + sh + 1) & ~1;
    pc.n = 1;
    return;
  }
  for (int s = 0; s < nseg; ++s) {
    const int lo = s * wp, hi = lo + wp;
    const int a = max(c0, lo), b = min(c0 + B, hi);
    if (a >= b) continue;
    pc.src[pc.n] = segs[s].p + segs[s].col0 + (a - lo);
    pc.soff[pc.n] = a - c0;
    pc.len[pc.n] = b - a;
    ++pc.n;
  }
}

// CTA body of the bulk-loader Gram for block `bid` of problem set P (gram_bulk_kernel runs one
// set; gram_bulk_combo runs a main-block set and a strip set interleaved by chunk)
// TMA subblock variant (TMA = true, subblock mode with q <= 32, 3 segments): each segment of a
// stage arrives as two 16 x 16 boxes (128-byte rows, 128-byte swizzle) of a 2-D tensor map
// over its block -- 12 copies per stage instead of 96 row copies of 256 bytes, which kept the
// MMA warps waiting on the single producer warp.  Segment s occupies tile columns
// [32 s, 32 s + 32); element (row k, tile column p) of a stage sits at
//   (p >> 4) * 256 + k * 16 + (((p >> 1) & 7) ^ (k & 7)) * 2 + (p & 1).
// The 4-row k slices of the DMMA fragments take rows {0,2,4,6}, {1,3,5,7}, {8,..,14}, {9,..,15}:
// a 64-bit fragment load is served per half-warp (4 rows x 4 columns = 2 chunks per row), and
// under the swizzle rows 0, 2, 4, 6 put those chunk pairs in four disjoint 32-byte bank groups,
// so each load is two conflict-free wavefronts (rows {0,4,1,5} measured 2-way conflicted).  The
// k order inside a stage only permutes the summation of the Gram.
constexpr int SB_TMA_BOX = 16 * 16;      // doubles per box
constexpr int SB_TMA_STAGE = 6 * SB_TMA_BOX;  // 3 segments x 2 boxes per operand stage
constexpr int SB_PAIR_STAGES = 8;
struct SbMaps {
  CUtensorMap m[6];  // X, W, P, AX, AW, AP: dims (ld, n), box (16, 16), 128-byte swizzle
};

BK_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

BK_DEV int sb_tma_row(int kq, int fr) { return (kq >> 1) * 8 + (kq & 1) + fr * 2; }

// PAIR (TMA subblock mode only): one CTA computes both Grams of a subblock -- warps of group 0
// S^T (AS), group 1 S^T S -- from one staged copy of S and AS per stage (2 operand loads per
// stage for the two Grams instead of 3), one CTA per SM with an 8-deep ring.  13 warps put 4
// on one SM sub-partition, whose 16K registers cap the kernel at 128 per thread.  Config 2:
// 2.60 -> 2.28 ms for the 16 subblocks (PPCG_GRAM_SBPAIR=0: two CTAs, one per Gram).
template <class C, bool TMA = false, bool PAIR = false>
BK_DEV void gram_bulk_body(const GramParams& P, int64_t bid, const CUtensorMap* maps = nullptr) {
  static_assert(!PAIR || TMA, "pair mode loads through TMA boxes");
  constexpr int BM = C::BM, BN = C::BN, LDX = C::LDX, LDY = C::LDY, WM = C::WM, WN = C::WN;
  constexpr int ST = PAIR ? SB_PAIR_STAGES : C::STAGES;
  constexpr int GW = C::THREADS / 32;          // MMA warps per group
  constexpr int NCW = (PAIR ? 2 : 1) * GW;     // MMA warps
  constexpr int XSTG = TMA ? SB_TMA_STAGE : C::XSTAGE, YSTG = TMA ? SB_TMA_STAGE : C::YSTAGE;
  static_assert(!TMA || (BM == 96 && BN == 96), "TMA subblock variant: one 96 x 96 tile");
  extern __shared__ __align__(16) double smem_raw[];
  // 128-byte swizzled boxes need 1024-byte aligned destinations (1 KB of slack allocated)
  double* smem = TMA ? reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023))
                     : smem_raw;
  double* Xs = smem;                    // [STAGES][BK][LDX]
  double* Ys = smem + ST * XSTG;        // [STAGES][BK][LDY]
  uint64_t* full = reinterpret_cast<uint64_t*>(Ys + ST * YSTG);
  uint64_t* empty = full + ST;
  __shared__ int s_last_g[2];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = (PAIR && warp < NCW) ? warp / GW : 0;  // pair mode: Gram of this warp group
  const int gwarp = warp - grp * GW, gtid = tid - grp * C::THREADS;
  int& s_last = s_last_g[grp];
  // block order: tile fastest, then chunk, then problem; chunk_major: then problem, then chunk
  // (pair mode: chunk fastest, then subblock; problem 2 j + group)
  const int slot = PAIR ? 0 : (int)(bid % P.max_tiles);
  const int chunk = PAIR ? (int)(bid % P.nchunks)
                         : P.chunk_major ? (int)(bid / ((int64_t)P.max_tiles * P.nprob))
                                         : (int)((bid / P.max_tiles) % P.nchunks);
  const int pidx = PAIR ? (int)(2 * (bid / P.nchunks) + grp)
                        : P.chunk_major ? (int)((bid / P.max_tiles) % P.nprob)
                                        : (int)(bid / ((int64_t)P.max_tiles * P.nchunks));

  GramProblem g;
  int wp = 0, w = 0;  // padded segment stride (subblock mode) and real segment width
  int Mp, Np;
  if (P.explicit_list) {
    g = P.prob[pidx];
    Mp = g.M;
    Np = g.N;
  } else {
    subblock_problem<BM, BN>(P, pidx, g);
    w = g.xs[0].width;
    wp = TMA ? 32 : (w + 1) & ~1;
    Mp = Np = g.nxs * wp;
    g.tiles_m = (Mp + BM - 1) / BM;
    g.tiles_n = (Np + BN - 1) / BN;
    g.ntiles = g.tiles_m * g.tiles_n;
  }
  if (slot >= g.ntiles) return;
  const int ti = slot / g.tiles_n, tj = slot % g.tiles_n;
  const int m0 = ti * BM, n0 = tj * BN;
  if (g.symmetric && n0 + BN <= m0) return;  // entirely below the diagonal: mirrored

  const int64_t r_begin = (int64_t)chunk * P.chunk_rows;
  const int64_t r_end = lmin(P.nrows, r_begin + P.chunk_rows);
  const int nstages = (int)((r_end - r_begin + G_BK - 1) / G_BK);

  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // a diagonal tile of a symmetric Gram (X == Y, m0 == n0): both operands are the same rows and
  // columns, so only the X stage is copied and the MMA warps read Y fragments from it
  const bool same = BM == BN && g.symmetric && m0 == n0;

  if (TMA && warp == NCW) {  // ---- producer (TMA): one lane, 6 or 12 boxes per stage
    if (lane == 0) {
      const int kind = pidx & 1, col = (int)(P.sc0 + (int64_t)(pidx >> 1) * P.q);
      const uint32_t bytes = (same ? 6u : 12u) * SB_TMA_BOX * 8u;
      for (int s = 0; s < nstages; ++s) {
        const int st = s % ST;
        if (s >= ST) mbar_wait(empty + st, ((s / ST) - 1) & 1);
        const int rb = (int)(r_begin + (int64_t)s * G_BK);
        mbar_arrive_expect_tx(full + st, bytes);
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          const int sg = b >> 1, c = col + (b & 1) * 16;
          tma_load_2d(Xs + st * XSTG + b * SB_TMA_BOX, maps + sg, c, rb, full + st);
          if (!same) tma_load_2d(Ys + st * YSTG + b * SB_TMA_BOX, maps + (kind ? sg : 3 + sg), c, rb, full + st);
        }
      }
    }
    return;
  }
  if (!TMA && warp == NCW) {  // ---- producer warp: lane = (operand, row); pieces held in registers
    const int r = lane & 15;
    const bool xop = lane < 16;
    Pieces pc;
    int sh, bx = 0, by = 0;
    tile_pieces(g, true, m0, BM, wp, pc, sh);
#pragma unroll
    for (int i = 0; i < 3; ++i) bx += i < pc.n ? pc.len[i] : 0;
    Pieces py;
    tile_pieces(g, false, n0, BN, wp, py, sh);
#pragma unroll
    for (int i = 0; i < 3; ++i) by += i < py.n ? py.len[i] : 0;
    if (!xop) pc = py;
    const uint32_t stage_row_bytes = (uint32_t)(bx + (same ? 0 : by)) * 8;
    const bool copies = xop || !same;
    double* dbase = xop ? Xs + r * LDX : Ys + r * LDY;
    const int dstage = xop ? C::XSTAGE : C::YSTAGE;
    const double* src0 = pc.src[0] + (r_begin + r) * pc.ld;
    const double* src1 = pc.src[1] + (r_begin + r) * pc.ld;
    const double* src2 = pc.src[2] + (r_begin + r) * pc.ld;
    const int64_t sstep = (int64_t)G_BK * pc.ld;
    for (int s = 0; s < nstages; ++s) {
      const int st = s % ST;
      if (s >= ST) mbar_wait(empty + st, ((s / ST) - 1) & 1);
      const int64_t rb = r_begin + (int64_t)s * G_BK;
      const int nvalid = (int)lmin(G_BK, r_end - rb);
      double* dst = dbase + st * dstage;
      if (copies && r >= nvalid) {  // partial last stage: zero rows (generic stores, before the arrive)
        const int ld = xop ? LDX : LDY;
        for (int c = 0; c < ld; ++c) dst[c] = 0.0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(full + st, (uint32_t)nvalid * stage_row_bytes);
      __syncwarp();
      if (copies && r < nvalid) {
        const int64_t o = (int64_t)s * sstep;
        bulk_g2s(dst + pc.soff[0], src0 + o, pc.len[0] * 8, full + st);
        if (pc.n > 1) bulk_g2s(dst + pc.soff[1], src1 + o, pc.len[1] * 8, full + st);
        if (pc.n > 2) bulk_g2s(dst + pc.soff[2], src2 + o, pc.len[2] * 8, full + st);
      }
    }
    return;
  }

  // ---- MMA warps
  int shx = 0, shy = 0;
  if (wp == 0) {
    shx = (int)((reinterpret_cast<uintptr_t>(g.xs[0].p + g.xs[0].col0) >> 3) & 1);
    shy = (int)((reinterpret_cast<uintptr_t>(g.ys[0].p + g.ys[0].col0) >> 3) & 1);
  }
  const int wm = gwarp / C::WARPS_N, wn = gwarp % C::WARPS_N;
  const int wm0 = m0 + wm * 8 * WM, wn0 = n0 + wn * 8 * WN;
  const bool below = g.symmetric && (wn0 + 8 * WN <= wm0);
  const bool warp_active = wm0 < Mp && wn0 < Np && !below;

  double acc[WM][WN][2];
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int fr = lane & 3, fc = lane >> 2;
  const int xoff = fr * LDX + wm * 8 * WM + fc + shx, yoff = fr * LDY + wn * 8 * WN + fc + shy;
  // TMA layout: the warp's first fragment column starts a box (8 WM, 8 WN multiples of 16), so a
  // fragment's box is (first box) + a / 2 and its 16-byte chunk ((a & 1) << 2 | fc >> 1)
  static_assert(!TMA || ((8 * WM) % 16 == 0 && (8 * WN) % 16 == 0), "warp tiles start on boxes");
  const int tbx = (wm * 8 * WM >> 4) * SB_TMA_BOX + (fc & 1), tby = (wn * 8 * WN >> 4) * SB_TMA_BOX + (fc & 1);
  for (int s = 0; s < nstages; ++s) {
    const int st = s % ST;
    mbar_wait(full + st, (s / ST) & 1);
    if constexpr (TMA) {
      if (warp_active) {
        const double* xs = Xs + st * XSTG;
        const double* ys = (same ? Xs : Ys) + st * YSTG;
        double af[2][WM], bf[2][WN];
        auto load = [&](int kq, double* fa, double* fb) {
          const int k = sb_tma_row(kq, fr), t = ((fc >> 1) ^ k) & 7;
          const double* xr = xs + tbx + k * 16;
          const double* yr = ys + tby + k * 16;
#pragma unroll
          for (int a = 0; a < WM; ++a) fa[a] = lds64(xr + (a >> 1) * SB_TMA_BOX + ((t ^ ((a & 1) << 2)) << 1));
#pragma unroll
          for (int b = 0; b < WN; ++b) fb[b] = lds64(yr + (b >> 1) * SB_TMA_BOX + ((t ^ ((b & 1) << 2)) << 1));
        };
        // pair mode (13 warps: 4 on one SM sub-partition, so <= 128 registers): no fragment
        // double buffering -- the other MMA warps of the sub-partition cover the load latency
        if (!PAIR) load(0, af[0], bf[0]);
#pragma unroll
        for (int kq = 0; kq < G_BK / 4; ++kq) {
          const int cur = PAIR ? 0 : kq & 1;
          if (PAIR) load(kq, af[0], bf[0]);
          else if (kq + 1 < G_BK / 4) load(kq + 1, af[cur ^ 1], bf[cur ^ 1]);
#pragma unroll
          for (int a = 0; a < WM; ++a)
#pragma unroll
            for (int b = 0; b < WN; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[cur][a], bf[cur][b]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      continue;
    }
    if (warp_active) {
      const double* xs = Xs + st * C::XSTAGE + xoff;
      const double* ys = (same ? Xs : Ys) + st * C::YSTAGE + yoff;  // (BM == BN: same stage shape)
      double af[2][WM], bf[2][WN];
#pragma unroll
      for (int a = 0; a < WM; ++a) af[0][a] = lds64(xs + a * 8);
#pragma unroll
      for (int b = 0; b < WN; ++b) bf[0][b] = lds64(ys + b * 8);
#pragma unroll
      for (int kq = 0; kq < G_BK / 4; ++kq) {
        const int cur = kq & 1;
        dmma_step_il<WM, WN>(acc, af[cur], bf[cur], af[cur ^ 1], bf[cur ^ 1], xs + (kq + 1) * 4 * LDX, 8,
                             ys + (kq + 1) * 4 * LDY, 8, kq + 1 < G_BK / 4);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }

  // ---- epilogue (MMA warps only): tile (lrow, lcol) -> virtual (gi, gj)
  auto store_final = [&](int lrow, int lcol, double v) {
    const int pi = m0 + lrow, pj = n0 + lcol;
    if (pi >= Mp || pj >= Np) return;
    const int gi = pad_map(pi, wp, w), gj = pad_map(pj, wp, w);
    if (gi < 0 || gj < 0 || gi >= g.M || gj >= g.N) return;
    if (g.symmetric) {
      if (gi > gj) return;  // upper triangle, mirrored
      g.C[(int64_t)gi * g.ldc + gj] = v;
      g.C[(int64_t)gj * g.ldc + gi] = v;
    } else {
      int r = gi + g.row_off, c = gj + g.col_off;
      if (g.trans) { const int t = r; r = c; c = t; }
      g.C[(int64_t)r * g.ldc + c] = v;
      if (g.mirror && r < g.col_off) g.C[(int64_t)c * g.ldc + r] = v;
    }
  };

  if (P.nchunks == 1) {
    if (!warp_active) return;
#pragma unroll
    for (int a = 0; a < WM; ++a)
#pragma unroll
      for (int b = 0; b < WN; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          store_final(wm * 8 * WM + a * 8 + (lane >> 2), wn * 8 * WN + b * 8 + 2 * (lane & 3) + e, acc[a][b][e]);
    return;
  }

  const int64_t tile_id = (int64_t)pidx * P.max_tiles + slot;
  double* part = P.ws + (tile_id * P.nchunks + chunk) * (BM * BN);
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b)
      *reinterpret_cast<double2*>(part + (wm * 8 * WM + a * 8 + (lane >> 2)) * BN + wn * 8 * WN + b * 8 +
                                  2 * (lane & 3)) = make_double2(acc[a][b][0], acc[a][b][1]);
  __threadfence();
  named_bar_sync(1 + grp, C::THREADS);
  if (gtid == 0) s_last = (atomicAdd(&P.tickets[tile_id], 1) == P.nchunks - 1);
  named_bar_sync(1 + grp, C::THREADS);
  if (!s_last) return;
  __threadfence();
  const double* base = P.ws + tile_id * P.nchunks * (BM * BN);
  for (int e = gtid; e < BM * BN; e += C::THREADS) {
    double v = 0.0;
    for (int c = 0; c < P.nchunks; ++c) v += __ldcg(base + (int64_t)c * (BM * BN) + e);
    store_final(e / BN, e % BN, v);
  }
  if (gtid == 0) P.tickets[tile_id] = 0;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS + 32, C::MINB) gram_bulk_kernel(const __grid_constant__ GramParams P) {
  gram_bulk_body<C>(P, blockIdx.x);
}

template <class C>
__global__ void __launch_bounds__(C::THREADS + 32, C::MINB)
    gram_sb_tma_kernel(const __grid_constant__ GramParams P, const __grid_constant__ SbMaps M) {
  gram_bulk_body<C, true>(P, blockIdx.x, M.m);
}

template <class C>
__global__ void __launch_bounds__(2 * C::THREADS + 32, 1)
    gram_sb_pair_kernel(const __grid_constant__ GramParams P, const __grid_constant__ SbMaps M) {
  gram_bulk_body<C, true, true>(P, blockIdx.x, M.m);
}

// Main block (CA tiles) and strips (CB tiles) of split Grams in ONE launch, both chunk-major
// with the same row chunks: the CTAs of chunk c of both sets are adjacent, so the strip CTAs
// read the chunk's X / Y rows while the main tiles hold them in L2 -- the separate strip launch
// re-read X and AX from DRAM (1 GB per config-2 Gram) at 4x lower tensor-pipe use.
template <class CA, class CB>
__global__ void __launch_bounds__(CA::THREADS + 32, CA::MINB) gram_bulk_combo(const __grid_constant__ GramParams PA,
                                                                            const __grid_constant__ GramParams PB) {
  static_assert(CA::THREADS == CB::THREADS, "one block size");
  const int64_t na = (int64_t)PA.max_tiles * PA.nprob, nb = (int64_t)PB.max_tiles * PB.nprob;
  const int64_t c = blockIdx.x / (na + nb), l = blockIdx.x % (na + nb);
  if (l < na) gram_bulk_body<CA>(PA, c * na + l);
  else gram_bulk_body<CB>(PB, c * nb + (l - na));
}

// 1: split Grams run main block + strips in one interleaved launch (PPCG_GRAM_COMBO=0: two)
static int g_combo = [] {
  const char* e = getenv("PPCG_GRAM_COMBO");
  return e ? atoi(e) : 1;
}();

static int g_bulk_loader = [] {
  const char* e = getenv("PPCG_GRAM_BULK");
  return e ? atoi(e) : 1;
}();

static int choose_chunks(int64_t nrows, int64_t total_tiles, int slots_per_sm) {
  // Wave-aware split-K: the smallest chunk count whose last wave is >= 92% full (each chunk
  // >= 32 stages when possible); a 1.1-wave grid idles most of the second wave.
  // At least 8 waves: short CTAs let the dynamic block scheduler even out CTAs of unequal
  // cost (edge tiles of 523 = 8 x 64 + 11) and shrink the tail; measured at config 2:
  // 22.5 -> 24.1 TF/s (X^T Y), 17.2 -> 20.2 (symmetric), 22.8 -> 24.6 (two Grams)
  // (profiles/gemm_sweep_r01c.json).  PPCG_GRAM_MINWAVES overrides (0 = off).
  static const int min_waves = [] {
    const char* e = getenv("PPCG_GRAM_MINWAVES");
    return e ? atoi(e) : 8;
  }();
  const int64_t slots = (int64_t)slots_per_sm * kSMs;
  total_tiles = lmax(total_tiles, 1);
  const int64_t cmax = lmax(1, lmin(256, nrows / (32 * G_BK)));
  if (total_tiles >= 8 * slots || cmax == 1) return 1;
  if (min_waves > 0) {
    for (int64_t c = 1; c <= cmax; ++c) {
      const int64_t ctas = total_tiles * c;
      const int64_t waves = (ctas + slots - 1) / slots;
      if (waves >= min_waves && (double)ctas / (double)(waves * slots) >= 0.92) return (int)c;
    }
  }
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t c = 1; c <= cmax; ++c) {
    const int64_t ctas = total_tiles * c;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (eff >= 0.92) return (int)c;
    if (eff > best_eff) { best_eff = eff; best = c; }
  }
  return (int)best;
}

// workspace layout: [tickets: 64 KB][partials]
constexpr int64_t kTicketBytes = 1 << 16;

template <class C>
static int64_t ws_bytes_for(int64_t nrows, int64_t tiles) {
  const int c = choose_chunks(nrows, tiles, C::SLOTS_PER_SM);
  return kTicketBytes + tiles * c * C::BM * C::BN * (int64_t)sizeof(double);
}

template <class C>
static int launch_gram_cfg(GramParams& P, int64_t total_tiles_slots, void* ws, int64_t ws_bytes, cudaStream_t st,
                           const SbMaps* maps = nullptr) {
  static const int fast_on = [] {
    const char* e = getenv("PPCG_GRAM_FAST");
    return e ? atoi(e) : 1;
  }();
  P.allow_fast = fast_on;
  P.nchunks = P.force_chunks > 0 ? P.force_chunks : choose_chunks(P.nrows, total_tiles_slots, C::SLOTS_PER_SM);
  int64_t part_bytes = (int64_t)total_tiles_slots * P.nchunks * C::BM * C::BN * sizeof(double);
  if (P.nchunks > 1) {
    while (P.nchunks > 1 && kTicketBytes + part_bytes > ws_bytes) {  // fit the workspace
      P.nchunks = (P.nchunks + 1) / 2;
      part_bytes = (int64_t)total_tiles_slots * P.nchunks * C::BM * C::BN * sizeof(double);
    }
    if (P.nchunks > 1 && total_tiles_slots * (int64_t)sizeof(int) > kTicketBytes) P.nchunks = 1;
  }
  P.chunk_rows = (P.nrows + P.nchunks - 1) / P.nchunks;
  P.chunk_rows = ((P.chunk_rows + G_BK - 1) / G_BK) * G_BK;
  P.nchunks = (int)lmax(1, (P.nrows + P.chunk_rows - 1) / P.chunk_rows);
  P.tickets = reinterpret_cast<int*>(ws);
  P.ws = reinterpret_cast<double*>(static_cast<char*>(ws) + kTicketBytes);
  const int64_t grid = (int64_t)P.nprob * P.max_tiles * P.nchunks;
  if (grid <= 0) return BK_OK;
  if (grid > 0x7fffffff) return BK_ERR_UNSUPPORTED;
  // per launch (cheap): the attribute belongs to the current device's context
  cudaFuncSetAttribute(gram_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  cudaFuncSetAttribute(gram_bulk_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::SMEM + 16 * C::STAGES);
  BK_COUNT();
  if constexpr (C::BM == 96 && C::BN == 96) if (maps) {
    constexpr int tsmem = C::STAGES * 2 * SB_TMA_STAGE * (int)sizeof(double) + 16 * C::STAGES + 1024;
    static bool tattr = false;
    if (!tattr) {
      cudaFuncSetAttribute(gram_sb_tma_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
      tattr = true;
    }
    gram_sb_tma_kernel<C><<<(unsigned)grid, C::THREADS + 32, tsmem, st>>>(P, *maps);
    BK_CHECK_LAUNCH();
    return BK_OK;
  }
  if (P.bulk && g_bulk_loader)
    gram_bulk_kernel<C><<<(unsigned)grid, C::THREADS + 32, C::SMEM + 16 * C::STAGES, st>>>(P);
  else
    gram_kernel<C><<<(unsigned)grid, C::THREADS, C::SMEM, st>>>(P);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

static bool even_segs(const GramProblem& g) {
  for (int s = 0; s < g.nxs; ++s)
    if ((g.xs[s].ld & 1) || (g.xs[s].col0 & 1) || (reinterpret_cast<uintptr_t>(g.xs[s].p) & 15)) return false;
  for (int s = 0; s < g.nys; ++s)
    if ((g.ys[s].ld & 1) || (g.ys[s].col0 & 1) || (reinterpret_cast<uintptr_t>(g.ys[s].p) & 15)) return false;
  return true;
}

template <class C>
static void fill_tiles(GramProblem& g) {
  g.tiles_m = (g.M + C::BM - 1) / C::BM;
  g.tiles_n = (g.N + C::BN - 1) / C::BN;
  g.ntiles = g.tiles_m * g.tiles_n;
}

// tile choice: 64x64 at 3 CTAs/SM measured fastest at config-2 shapes (22.6 vs 17.3
// TFLOP/s for 64x128 at 2 CTAs/SM, profiles/gemm_sweep_r01.json); PPCG_GRAM_TILE=128
// selects the wide tile for tuning
static bool use_big(int m2) {
  static int force = [] {
    const char* e = getenv("PPCG_GRAM_TILE");
    return e ? atoi(e) : 0;
  }();
  return force == 128 && m2 >= 192;
}

template <class C>
static int prepare_explicit(int nprob, GramParams& P) {
  int maxt = 0;
  P.vec16 = 1;
  P.bulk = 1;
  for (int i = 0; i < nprob; ++i) {
    GramProblem& g = P.prob[i];
    fill_tiles<C>(g);
    if (g.M == 0 || g.N == 0) g.ntiles = 0;
    maxt = max(maxt, g.ntiles);
    if (!even_segs(g)) P.vec16 = 0;
    if (g.nxs != 1 || g.nys != 1 || (g.xs[0].ld & 1) || (g.ys[0].ld & 1) ||
        (reinterpret_cast<uintptr_t>(g.xs[0].p) & 7) || (reinterpret_cast<uintptr_t>(g.ys[0].p) & 7))
      P.bulk = 0;
  }
  P.nprob = nprob;
  P.explicit_list = 1;
  P.max_tiles = maxt;
  return maxt;
}

// workspace of a combined launch: [tickets A | tickets B (one 64 KB ticket region, the only
// place any launch keeps tickets, so they are always zero between launches)][partials A][partials B]
template <class CA, class CB>
static int64_t combo_ws_bytes(int64_t nrows, int64_t tiles_a, int64_t tiles_b, int nchunks) {
  return kTicketBytes + (tiles_a * CA::BM * CA::BN + tiles_b * CB::BM * CB::BN) * nchunks * (int64_t)sizeof(double);
}

template <class CA, class CB>
static int combo_chunks(int64_t nrows, int64_t tiles_a, int64_t tiles_b) {
  return choose_chunks(nrows, tiles_a + tiles_b, CA::SLOTS_PER_SM);
}

// A (main blocks, CA tiles) and B (strips, CB tiles) prepared by prepare_explicit; one launch
template <class CA, class CB>
static int launch_combo(GramParams& A, GramParams& B, void* ws, int64_t ws_bytes, cudaStream_t st) {
  const int64_t ta = (int64_t)A.max_tiles * A.nprob, tb = (int64_t)B.max_tiles * B.nprob;
  int nch = A.force_chunks;
  if (combo_ws_bytes<CA, CB>(A.nrows, ta, tb, nch) > ws_bytes || (ta + tb) * (int64_t)sizeof(int) > kTicketBytes)
    return BK_ERR_UNSUPPORTED;
  int64_t rows = (A.nrows + nch - 1) / nch;
  rows = ((rows + G_BK - 1) / G_BK) * G_BK;
  nch = (int)lmax(1, (A.nrows + rows - 1) / rows);
  static const int fast_on = [] {
    const char* e = getenv("PPCG_GRAM_FAST");
    return e ? atoi(e) : 1;
  }();
  char* w = static_cast<char*>(ws);
  for (GramParams* P : {&A, &B}) {
    P->allow_fast = fast_on;
    P->nchunks = nch;
    P->chunk_rows = rows;
    P->chunk_major = 1;
  }
  A.tickets = reinterpret_cast<int*>(w);
  B.tickets = A.tickets + ta;
  A.ws = reinterpret_cast<double*>(w + kTicketBytes);
  B.ws = A.ws + ta * nch * CA::BM * CA::BN;
  const int64_t grid = (ta + tb) * nch;
  if (grid > 0x7fffffff) return BK_ERR_UNSUPPORTED;
  const int smem = max(CA::SMEM + 16 * CA::STAGES, CB::SMEM + 16 * CB::STAGES);
  // per launch (cheap): the attribute belongs to the current device's context
  cudaFuncSetAttribute(gram_bulk_combo<CA, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  BK_COUNT();
  gram_bulk_combo<CA, CB><<<(unsigned)grid, CA::THREADS + 32, smem, st>>>(A, B);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

template <class C>
static int gram_explicit(int nprob, GramParams& P, void* ws, int64_t ws_bytes, cudaStream_t st) {
  int maxt = 0;
  P.vec16 = 1;
  P.bulk = 1;
  for (int i = 0; i < nprob; ++i) {
    GramProblem& g = P.prob[i];
    fill_tiles<C>(g);
    if (g.M == 0 || g.N == 0) g.ntiles = 0;
    maxt = max(maxt, g.ntiles);
    if (!even_segs(g)) P.vec16 = 0;
    // bulk copies: one segment per operand, even row strides (copies end within the row)
    if (g.nxs != 1 || g.nys != 1 || (g.xs[0].ld & 1) || (g.ys[0].ld & 1) ||
        (reinterpret_cast<uintptr_t>(g.xs[0].p) & 7) || (reinterpret_cast<uintptr_t>(g.ys[0].p) & 7))
      P.bulk = 0;
  }
  if (maxt == 0) return BK_OK;
  P.nprob = nprob;
  P.explicit_list = 1;
  P.max_tiles = maxt;
  return launch_gram_cfg<C>(P, (int64_t)maxt * nprob, ws, ws_bytes, st);
}

// Split of a Gram whose width is not a multiple of 64 (k_total = 523 = 8 x 64 + 11): the
// 64-aligned main block runs full 64 x 64 tiles (30+ TF/s, vs ~24 when a ninth, mostly empty
// tile row/column rides along -- such edge CTAs stream as many rows as full ones), the
// remainder strips run 64 x 16 tiles in a second launch.  The right strip covers all rows
// (incl. the corner); the bottom strip is computed transposed (Y^T X) so it also has a
// 64-aligned long side; a symmetric Gram needs only the right strip, mirrored.
static int env_flag(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

static bool split_worth(const GramProblem& g) {
  static const int on = env_flag("PPCG_GRAM_SPLIT", 1);
  return on && g.M >= 128 && g.N >= 128 && (g.M % 64 != 0 || g.N % 64 != 0) && g.nxs == 1 && g.nys == 1 && !use_big(g.N);
}

static int split_parts(const GramProblem& g, GramProblem& main, GramProblem* strips) {
  const int M1 = g.M / 64 * 64, N1 = g.N / 64 * 64;
  main = g;
  main.M = M1;
  main.N = N1;
  main.xs[0].width = M1;
  main.ys[0].width = N1;
  int ns = 0;
  if (g.N > N1) {  // right strip: rows [0, M) x cols [N1, N)
    GramProblem r = g;
    r.symmetric = 0;
    r.ys[0].col0 += N1;
    r.ys[0].width = g.N - N1;
    r.N = g.N - N1;
    r.col_off = N1;
    r.mirror = g.symmetric;
    strips[ns++] = r;
  }
  if (!g.symmetric && g.M > M1) {  // bottom strip rows [M1, M) x cols [0, N1), as (Y^T X)^T
    GramProblem b = g;
    b.symmetric = 0;
    b.xs[0] = g.ys[0];
    b.xs[0].width = N1;
    b.ys[0] = g.xs[0];
    b.ys[0].col0 += M1;
    b.ys[0].width = g.M - M1;
    b.M = N1;
    b.N = g.M - M1;
    b.col_off = M1;
    b.trans = 1;
    strips[ns++] = b;
  }
  return ns;
}

// part: 0 = whole Gram (main then strips on `st`), 1 = main block only, 2 = strips only
// (parts 1/2 let the caller run the memory-bound strips on a second stream beside the
// compute-bound main launch; an unsplit Gram is all "main").
static int gram_problems(int nprob, const GramProblem* probs, int64_t n, void* ws, int64_t ws_bytes,
                         cudaStream_t st, int part = 0) {
  bool split = true;
  for (int i = 0; i < nprob; ++i) split = split && split_worth(probs[i]);
  GramParams A{};
  A.nrows = n;
  if (!split) {
    if (part == 2) return BK_OK;
    for (int i = 0; i < nprob; ++i) A.prob[i] = probs[i];
    if (use_big(probs[0].N)) return gram_explicit<Big>(nprob, A, ws, ws_bytes, st);
    return gram_explicit<Small>(nprob, A, ws, ws_bytes, st);
  }
  GramParams B{};
  B.nrows = n;
  int nb = 0;
  for (int i = 0; i < nprob; ++i) nb += split_parts(probs[i], A.prob[i], B.prob + nb);
  {
    // main block and strips share one split-K chunking (that of the combined launch), so
    // the combined launch and the two-launch path (parts, cp.async loader) agree bit for bit
    GramParams A2 = A, B2 = B;
    const int ma = prepare_explicit<Small>(nprob, A2), mb = prepare_explicit<Strip>(nb, B2);
    const int64_t ta = (int64_t)ma * nprob, tb = (int64_t)mb * nb;
    int nch = combo_chunks<Small, Strip>(n, ta, tb);
    while (nch > 1 && combo_ws_bytes<Small, Strip>(n, ta, tb, nch) > ws_bytes) nch = (nch + 1) / 2;
    A.force_chunks = B.force_chunks = nch;
    if (part == 0 && nb > 0 && g_combo && g_bulk_loader && ma > 0 && mb > 0 && A2.bulk && B2.bulk) {
      A2.force_chunks = B2.force_chunks = nch;
      const int rc = launch_combo<Small, Strip>(A2, B2, ws, ws_bytes, st);
      if (rc != BK_ERR_UNSUPPORTED) return rc;
    }
  }
  if (part != 2) {
    int rc = gram_explicit<Small>(nprob, A, ws, ws_bytes, st);
    if (rc != BK_OK) return rc;
  }
  if (part == 1 || nb == 0) return BK_OK;
  return gram_explicit<Strip>(nb, B, ws, ws_bytes, st);
}

}  // namespace bk

using namespace bk;

extern "C" int64_t bk_gram_ws_bytes(int64_t n, int m1, int m2) {
  if (use_big(m2)) return ws_bytes_for<Big>(n, (int64_t)((m1 + 63) / 64) * ((m2 + 127) / 128));
  const int64_t full = ws_bytes_for<Small>(n, (int64_t)((m1 + 63) / 64) * ((m2 + 63) / 64));
  // split launches (sequential, sharing the buffer): up to two strip problems per Gram
  const int64_t right = (int64_t)((m1 + 63) / 64) * (((m2 % 64) + 15) / 16);
  const int64_t bottom = (int64_t)(m2 / 64) * (((m1 % 64) + 15) / 16);
  // one combined launch (main 64-aligned tiles + both strips, shared chunking)
  const int64_t main_t = (int64_t)(m1 / 64) * (m2 / 64), strip_t = 2 * lmax(right, bottom);
  const int64_t combo = combo_ws_bytes<Small, Strip>(n, main_t, strip_t, combo_chunks<Small, Strip>(n, main_t, strip_t));
  return lmax(lmax(full, combo), ws_bytes_for<Strip>(n, 2 * lmax(right, bottom)));
}

// C (m1 x m2, ldc) = X(:, 0:m1)^T Y(:, 0:m2) over n rows.  symmetric != 0 requires X == Y,
// m1 == m2 and computes only the tiles meeting the upper triangle.  (core.py:43-49)
static int gram_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C,
                  int64_t ldc, int symmetric, void* ws, int64_t ws_bytes, void* stream, int part);

extern "C" int bk_gram_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y,
                         int64_t ldy, double* C, int64_t ldc, int symmetric, void* ws, int64_t ws_bytes,
                         void* stream) {
  return gram_d(n, m1, m2, X, ldx, Y, ldy, C, ldc, symmetric, ws, ws_bytes, stream, 0);
}

// 1 / 0: split Grams as one combined launch / as main + strip launches; -1: query
extern "C" int bk_gram_set_combo(int mode) {
  const int prev = g_combo;
  if (mode >= 0) g_combo = mode ? 1 : 0;
  return prev;
}

extern "C" int bk_gram_set_loader(int mode) {
  const int prev = g_bulk_loader;
  if (mode >= 0) g_bulk_loader = mode ? 1 : 0;
  return prev;
}

// 1 if bk_gram_d / bk_gram2_d split this width into a main block and strips (see gram_problems)
extern "C" int bk_gram_splits(int m1, int m2) {
  GramProblem g{};
  g.M = m1;
  g.N = m2;
  g.nxs = g.nys = 1;
  return split_worth(g) ? 1 : 0;
}

// One part of a Gram (part 1 = main block, 2 = strips; 0 = all): callers run part 2 on a
// second stream with its own workspace, fenced by events, beside part 1.
extern "C" int bk_gram_part_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y,
                              int64_t ldy, double* C, int64_t ldc, int symmetric, int part, void* ws,
                              int64_t ws_bytes, void* stream) {
  if (part < 0 || part > 2) return BK_ERR_ARG;
  return gram_d(n, m1, m2, X, ldx, Y, ldy, C, ldc, symmetric, ws, ws_bytes, stream, part);
}

static int gram_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C,
                  int64_t ldc, int symmetric, void* ws, int64_t ws_bytes, void* stream, int part) {
  if (n < 0 || m1 < 0 || m2 < 0 || (symmetric && m1 != m2)) return BK_ERR_ARG;
  if (m1 == 0 || m2 == 0) return BK_OK;
  if (n == 0) {
    for (int i = 0; i < m1; ++i)
      if (cudaMemsetAsync(C + (int64_t)i * ldc, 0, sizeof(double) * m2, (cudaStream_t)stream) != cudaSuccess)
        return BK_ERR_CUDA;
    return BK_OK;
  }
  GramParams P{};
  GramProblem& g = P.prob[0];
  g.xs[0] = {X, ldx, 0, m1};
  g.ys[0] = {Y, ldy, 0, m2};
  g.nxs = g.nys = 1;
  g.M = m1;
  g.N = m2;
  g.C = C;
  g.ldc = ldc;
  g.symmetric = symmetric ? 1 : 0;
  return gram_problems(1, &g, n, ws, ws_bytes, (cudaStream_t)stream, part);
}

// Two Grams sharing the row range in one launch: C1 = X1^T Y1, C2 = X2^T Y2 (e.g. the
// projection Grams X^T W and X^T P of ppcg.py:680-687).
static int gram2_d(int64_t n, int m1a, int m2a, const double* X1, int64_t ldx1, const double* Y1, int64_t ldy1,
                   double* C1, int64_t ldc1, int m1b, int m2b, const double* X2, int64_t ldx2, const double* Y2,
                   int64_t ldy2, double* C2, int64_t ldc2, void* ws, int64_t ws_bytes, void* stream, int part);

extern "C" int bk_gram2_d(int64_t n, int m1a, int m2a, const double* X1, int64_t ldx1, const double* Y1,
                          int64_t ldy1, double* C1, int64_t ldc1, int m1b, int m2b, const double* X2,
                          int64_t ldx2, const double* Y2, int64_t ldy2, double* C2, int64_t ldc2, void* ws,
                          int64_t ws_bytes, void* stream) {
  return gram2_d(n, m1a, m2a, X1, ldx1, Y1, ldy1, C1, ldc1, m1b, m2b, X2, ldx2, Y2, ldy2, C2, ldc2, ws, ws_bytes,
                 stream, 0);
}

extern "C" int bk_gram2_part_d(int64_t n, int m1a, int m2a, const double* X1, int64_t ldx1, const double* Y1,
                               int64_t ldy1, double* C1, int64_t ldc1, int m1b, int m2b, const double* X2,
                               int64_t ldx2, const double* Y2, int64_t ldy2, double* C2, int64_t ldc2, int part,
                               void* ws, int64_t ws_bytes, void* stream) {
  if (part < 0 || part > 2) return BK_ERR_ARG;
  return gram2_d(n, m1a, m2a, X1, ldx1, Y1, ldy1, C1, ldc1, m1b, m2b, X2, ldx2, Y2, ldy2, C2, ldc2, ws, ws_bytes,
                 stream, part);
}

static int gram2_d(int64_t n, int m1a, int m2a, const double* X1, int64_t ldx1, const double* Y1, int64_t ldy1,
                   double* C1, int64_t ldc1, int m1b, int m2b, const double* X2, int64_t ldx2, const double* Y2,
                   int64_t ldy2, double* C2, int64_t ldc2, void* ws, int64_t ws_bytes, void* stream, int part) {
  if (n <= 0) return BK_ERR_ARG;
  GramParams P{};
  const double* xs[2] = {X1, X2};
  const double* ys[2] = {Y1, Y2};
  int64_t lx[2] = {ldx1, ldx2}, ly[2] = {ldy1, ldy2}, lc[2] = {ldc1, ldc2};
  int ma[2] = {m1a, m1b}, na[2] = {m2a, m2b};
  double* cs[2] = {C1, C2};
  for (int i = 0; i < 2; ++i) {
    GramProblem& g = P.prob[i];
    g.xs[0] = {xs[i], lx[i], 0, ma[i]};
    g.ys[0] = {ys[i], ly[i], 0, na[i]};
    g.nxs = g.nys = 1;
    g.M = ma[i];
    g.N = na[i];
    g.C = cs[i];
    g.ldc = lc[i];
    g.symmetric = 0;
  }
  return gram_problems(2, P.prob, n, ws, ws_bytes, (cudaStream_t)stream, part);
}

// split-K grid of the paired subblock Grams: `waves` CTA waves (one CTA per SM): fewer, longer
// chunks than choose_chunks' 8 waves halve the partial-sum traffic and the last-CTA
// reductions; config 2 measured 36.9 (8 waves), 36.9 (4), 37.1 (2), 36.9 (1) it/s -- within
// the ~1% run-to-run spread, so 2 is kept for the traffic.  0 = choose_chunks.  A chunk keeps
// >= 32 stages (the choose_chunks floor), and the count depends on n and nb only, never on the
// workspace a caller happens to hold (bk_subblock_grams_ws_bytes sizes it exactly).
static int g_sbpair_waves = [] {
  const char* e = getenv("PPCG_SBPAIR_WAVES");
  return e ? atoi(e) : 2;
}();

static int sb_pair_chunks(int64_t n, int nb) {
  const int64_t cmax = lmax(1, lmin(256, n / (32 * G_BK)));
  if (g_sbpair_waves <= 0) return choose_chunks(n, nb, 1);
  return (int)lmax(1, lmin(cmax, (int64_t)g_sbpair_waves * kSMs / lmax(1, nb)));
}

extern "C" int bk_subblock_grams_set_waves(int waves) {
  if (waves < -1 || waves > 64) return BK_ERR_ARG;
  const int prev = g_sbpair_waves;
  if (waves >= 0) g_sbpair_waves = waves;
  return prev;
}

extern "C" int64_t bk_subblock_grams_ws_bytes(int64_t n, int k_act, int q, int has_p) {
  const int nb = (k_act + q - 1) / q;
  const int dmax = (has_p ? 3 : 2) * q;
  if (use_big(dmax)) return ws_bytes_for<Big>(n, (int64_t)2 * nb * ((dmax + 63) / 64) * ((dmax + 127) / 128));
  if (dmax > 64 && dmax <= 96) {
    // the paired launch (exactly its chunk count) or the per-Gram fallback, whichever is larger
    const int64_t pair = kTicketBytes + (int64_t)2 * nb * sb_pair_chunks(n, nb) * Sb96::BM * Sb96::BN * 8;
    return lmax(pair, ws_bytes_for<Sb96>(n, (int64_t)2 * nb));
  }
  const int t = (dmax + 63) / 64;
  return ws_bytes_for<Small>(n, (int64_t)2 * nb * t * t);
}

// both Grams of each subblock in one CTA (gram_sb_pair_kernel): grid nb x chunks, one CTA per SM
template <class C>
static int launch_sb_pair(GramParams& P, int nb, void* ws, int64_t ws_bytes, cudaStream_t st, const SbMaps& M) {
  P.nchunks = P.force_chunks > 0 ? P.force_chunks : sb_pair_chunks(P.nrows, nb);
  auto part_bytes = [&] { return (int64_t)P.nprob * P.nchunks * C::BM * C::BN * (int64_t)sizeof(double); };
  if (P.nchunks > 1) {
    while (P.nchunks > 1 && kTicketBytes + part_bytes() > ws_bytes) P.nchunks = (P.nchunks + 1) / 2;
    if (P.nchunks > 1 && (int64_t)P.nprob * (int64_t)sizeof(int) > kTicketBytes) P.nchunks = 1;
  }
  P.chunk_rows = (P.nrows + P.nchunks - 1) / P.nchunks;
  P.chunk_rows = ((P.chunk_rows + G_BK - 1) / G_BK) * G_BK;
  P.nchunks = (int)lmax(1, (P.nrows + P.chunk_rows - 1) / P.chunk_rows);
  P.tickets = reinterpret_cast<int*>(ws);
  P.ws = reinterpret_cast<double*>(static_cast<char*>(ws) + kTicketBytes);
  const int64_t grid = (int64_t)nb * P.nchunks;
  if (grid <= 0) return BK_OK;
  if (grid > 0x7fffffff) return BK_ERR_UNSUPPORTED;
  constexpr int smem = SB_PAIR_STAGES * 2 * SB_TMA_STAGE * (int)sizeof(double) + 16 * SB_PAIR_STAGES + 1024;
  // per launch (cheap): the attribute belongs to the current device's context
  cudaFuncSetAttribute(gram_sb_pair_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  BK_COUNT();
  gram_sb_pair_kernel<C><<<(unsigned)grid, 2 * C::THREADS + 32, smem, st>>>(P, M);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

typedef CUresult (*SbEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D map over an n x ld row-major block: box 16 columns x 16 rows, 128-byte swizzle; rows past n
// arrive zero-filled
static bool encode_sb_map(CUtensorMap* map, const double* base, int64_t ld, int64_t n) {
  static SbEncodeFn enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (SbEncodeFn) nullptr;
    return reinterpret_cast<SbEncodeFn>(p);
  }();
  if (!enc || !base) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  const cuuint32_t box[2] = {16, 16};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Per-subblock raw pencil Grams (ppcg.py:206-211 before unit scaling, ppcg.py:220-228):
// for block j (columns c0 + [j*q, min((j+1)*q, k_act))), S_j = [X_j | W_j | P_j] and
// A_j = S_j^T [AX_j | AW_j | AP_j], B_j = S_j^T S_j, each stored dmax x dmax (ld dmax).
extern "C" int bk_subblock_grams_d(int64_t n, int k_act, int q, int has_p, const double* X, const double* W,
                                   const double* P_, const double* AX, const double* AW, const double* AP,
                                   int64_t ld, int64_t c0, double* Araw, double* Braw, void* ws,
                                   int64_t ws_bytes, void* stream) {
  if (n <= 0 || k_act <= 0 || q <= 0) return BK_ERR_ARG;
  GramParams P{};
  const int nb = (k_act + q - 1) / q;
  P.explicit_list = 0;
  P.nprob = 2 * nb;
  P.sX = X; P.sW = W; P.sP = P_; P.sAX = AX; P.sAW = AW; P.sAP = AP;
  P.sld = ld;
  P.sc0 = c0;
  P.k_act = k_act;
  P.q = q;
  P.has_p = has_p ? 1 : 0;
  P.dmax = (has_p ? 3 : 2) * q;
  P.outA = Araw;
  P.outB = Braw;
  P.nrows = n;
  // 16-byte copies need even offsets/ld everywhere (q even keeps every block start even)
  const double* ptrs[6] = {X, W, P_, AX, AW, AP};
  bool aligned = !(ld & 1) && !(c0 & 1) && !(q & 1);
  for (int i = 0; i < 6; ++i)
    if (ptrs[i] && (reinterpret_cast<uintptr_t>(ptrs[i]) & 15)) aligned = false;
  P.vec16 = aligned ? 1 : 0;
  P.bulk = aligned ? 1 : 0;  // padded segment layout needs even q, offsets and stride
  // PPCG_GRAM_SBORDER=1: block order (tile, problem, chunk), all subblocks' Grams reading a row
  // chunk together -- measured no faster than problem-major (2.76 vs 2.73 ms at config 2); the
  // partial sums keep their fixed chunk order either way (same result)
  static const int sb_chunk_major = [] {
    const char* e = getenv("PPCG_GRAM_SBORDER");
    return e ? atoi(e) : 0;
  }();
  P.chunk_major = sb_chunk_major;
  if (use_big(P.dmax)) {
    P.bulk = 0;
    P.max_tiles = ((P.dmax + 63) / 64) * ((P.dmax + 127) / 128);
    return launch_gram_cfg<Big>(P, (int64_t)P.nprob * P.max_tiles, ws, ws_bytes, (cudaStream_t)stream);
  }
  if (P.dmax > 64 && P.dmax <= 96) {
    P.max_tiles = 1;
    // TMA boxes: 3 segments of <= 32 columns, 16-byte aligned bases and row strides
    static const int sb_tma = [] {
      const char* e = getenv("PPCG_GRAM_SBTMA");
      return e ? atoi(e) : 1;
    }();
    if (sb_tma && P.has_p && q <= 32 && P.bulk && n < 0x7fffffff && c0 + (int64_t)k_act <= ld) {
      SbMaps M;
      bool ok = true;
      for (int i = 0; i < 6 && ok; ++i) ok = encode_sb_map(&M.m[i], ptrs[i], ld, n);
      static const int sb_pair = [] {
        const char* e = getenv("PPCG_GRAM_SBPAIR");
        return e ? atoi(e) : 1;
      }();
      if (ok && sb_pair) return launch_sb_pair<Sb96>(P, nb, ws, ws_bytes, (cudaStream_t)stream, M);
      if (ok) return launch_gram_cfg<Sb96>(P, (int64_t)P.nprob, ws, ws_bytes, (cudaStream_t)stream, &M);
    }
    return launch_gram_cfg<Sb96>(P, (int64_t)P.nprob, ws, ws_bytes, (cudaStream_t)stream);
  }
  const int t = (P.dmax + 63) / 64;
  P.max_tiles = t * t;
  return launch_gram_cfg<Small>(P, (int64_t)P.nprob * P.max_tiles, ws, ws_bytes, (cudaStream_t)stream);
}

namespace bk {
// per-block combine of real Grams of interleaved views into complex X^H Y blocks
__global__ void k_subblock_combine(int nb, int k_act, int q, int nparts, int dmax, const double* __restrict__ tr,
                                   double* __restrict__ out) {
  const int j = blockIdx.y;
  const int w = min(q, k_act - j * q);
  const int d0 = nparts * w;
  const int ldr = 2 * dmax;
  const double* t = tr + (int64_t)j * ldr * ldr;
  double* o = out + (int64_t)j * dmax * dmax * 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d0 * d0; e += gridDim.x * blockDim.x) {
    const int a = e / d0, b = e % d0;
    const double rr = t[(2 * a) * ldr + 2 * b], ri = t[(2 * a) * ldr + 2 * b + 1];
    const double ir = t[(2 * a + 1) * ldr + 2 * b], ii = t[(2 * a + 1) * ldr + 2 * b + 1];
    o[2 * (a * dmax + b)] = rr + ii;
    o[2 * (a * dmax + b) + 1] = ri - ir;
  }
}
}  // namespace bk

// complex128 variant: X..AP interleaved complex, ld/c0 in complex elements; Araw/Braw are
// nb x dmax x dmax complex; tmpA/tmpB are real scratch of nb x (2 dmax)^2 doubles.
extern "C" int bk_subblock_grams_z(int64_t n, int k_act, int q, int has_p, const double* X, const double* W,
                                   const double* P_, const double* AX, const double* AW, const double* AP,
                                   int64_t ld, int64_t c0, double* Araw, double* Braw, double* tmpA, double* tmpB,
                                   void* ws, int64_t ws_bytes, void* stream) {
  int rc = bk_subblock_grams_d(n, 2 * k_act, 2 * q, has_p, X, W, P_, AX, AW, AP, 2 * ld, 2 * c0, tmpA, tmpB, ws,
                               ws_bytes, stream);
  if (rc != BK_OK) return rc;
  const int nb = (k_act + q - 1) / q;
  const int nparts = has_p ? 3 : 2;
  const int dmax = nparts * q;
  dim3 grid((unsigned)lmin(64, (dmax * dmax + 255) / 256), nb);
  BK_COUNT();
  k_subblock_combine<<<grid, 256, 0, (cudaStream_t)stream>>>(nb, k_act, q, nparts, dmax, tmpA, Araw);
  BK_COUNT();
  k_subblock_combine<<<grid, 256, 0, (cudaStream_t)stream>>>(nb, k_act, q, nparts, dmax, tmpB, Braw);
  BK_CHECK_LAUNCH();
  return BK_OK;
}
