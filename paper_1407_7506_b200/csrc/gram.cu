// Tall-skinny Gram products C = X^T Y on FP64 tensor cores (DMMA, mma.sync m8n8k4).
//
// Replaces the reference's block_inner (blockeig core.py:43-49, `x.conj().T @ y`, OpenBLAS
// dgemm) at every call site on the PPCG hot path: the full Grams of _apply_projection
// (ppcg.py:441-445), the orthonormality Gram (ppcg.py:448-453), the residual Gram
// (ppcg.py:630,758) and the per-q-block pencil Grams of _solve_subblock_pencil
// (ppcg.py:206-211).
//
// Design:
//  * reduction dimension = rows n (huge); the output is small (m1 x m2).  The row range is
//    split into `nchunks` contiguous chunks; each CTA computes one 64x64 output tile over
//    one chunk, 16 rows per pipeline stage, 4-stage cp.async ring.
//  * split-K partials go to a workspace; the LAST CTA to finish a tile (atomic ticket)
//    sums the partials in fixed chunk order -> results are bitwise run-to-run
//    deterministic, with a single launch.
//  * operands are "virtual concatenations" of up to 3 column segments of row-major
//    blocks, so S = [X_j | W_j | P_j] of a subblock is never materialised.
//  * symmetric mode (X == Y) computes only tiles ti <= tj and mirrors; diagonal tiles
//    write the upper triangle and mirror it, so the result is exactly symmetric.
//  * warps skip 8x8 MMA tiles that lie entirely outside the output, so ragged widths
//    (m = 523, 1045, ...) waste at most 7 columns of tensor work.
#include "common.cuh"

namespace bk {

constexpr int G_BM = 64, G_BN = 64, G_BK = 16, G_STAGES = 4, G_THREADS = 128;
constexpr int G_PAD = 4;  // row stride 68 = 4 mod 16 doubles: half-warp fragment loads hit 4 disjoint 8-bank groups
constexpr int G_LDS = G_BM + G_PAD;
constexpr int G_WM = 4, G_WN = 4;           // warp tile = 32 x 32 (4 x 4 MMA tiles)

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
  int tiles_dim;              // tiles per dim for dmax
  // common
  int64_t nrows;
  int nchunks;
  int64_t chunk_rows;
  int max_tiles;              // tiles per problem slot in the grid
  double* ws;                 // partials: [prob][tile][chunk][64*64]
  int* tickets;               // [prob][tile]
};

BK_DEV void subblock_problem(const GramParams& P, int b, GramProblem& g) {
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
  g.tiles_m = g.tiles_n = (g.M + G_BM - 1) / G_BM;
  g.ntiles = g.symmetric ? g.tiles_m * (g.tiles_m + 1) / 2 : g.tiles_m * g.tiles_n;
}

BK_DEV const double* seg_col_ptr(const Seg* segs, int nseg, int c, int64_t& ld, bool& valid) {
  int off = 0;
  for (int s = 0; s < nseg; ++s) {
    if (c < off + segs[s].width) {
      ld = segs[s].ld;
      valid = true;
      return segs[s].p + segs[s].col0 + (c - off);
    }
    off += segs[s].width;
  }
  valid = false;
  ld = 0;
  return nullptr;
}

__global__ void __launch_bounds__(G_THREADS, 2) gram_kernel(const __grid_constant__ GramParams P) {
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                                   // [STAGES][BK][LDS]
  double* Ys = smem + G_STAGES * G_BK * G_LDS;         // [STAGES][BK][LDS]
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = blockIdx.x % P.max_tiles;
  const int chunk = (blockIdx.x / P.max_tiles) % P.nchunks;
  const int pidx = blockIdx.x / (P.max_tiles * P.nchunks);

  GramProblem g;
  if (P.explicit_list) g = P.prob[pidx];
  else subblock_problem(P, pidx, g);
  if (slot >= g.ntiles) return;

  int ti, tj;
  if (g.symmetric) {  // slot -> (ti, tj), ti <= tj, row-major over the upper triangle
    int t = slot, r = 0, len = g.tiles_m;
    while (t >= len) { t -= len; ++r; --len; }
    ti = r; tj = r + t;
  } else {
    ti = slot / g.tiles_n; tj = slot % g.tiles_n;
  }
  const int m0 = ti * G_BM, n0 = tj * G_BN;

  const int64_t r_begin = (int64_t)chunk * P.chunk_rows;
  const int64_t r_end = min(P.nrows, r_begin + P.chunk_rows);
  const int nstages = (int)((r_end - r_begin + G_BK - 1) / G_BK);

  // each thread loads a fixed column of each operand: col = tid % 64, rows tid/64 + 2i
  const int lc = tid & 63, lr = tid >> 6;
  int64_t ldx, ldy;
  bool vx, vy;
  const double* px = seg_col_ptr(g.xs, g.nxs, m0 + lc, ldx, vx);
  const double* py = seg_col_ptr(g.ys, g.nys, n0 + lc, ldy, vy);
  vx = vx && (m0 + lc < g.M);
  vy = vy && (n0 + lc < g.N);

  auto load_stage = [&](int s, int st) {
    const int64_t rb = r_begin + (int64_t)s * G_BK;
    double* xd = Xs + st * G_BK * G_LDS;
    double* yd = Ys + st * G_BK * G_LDS;
#pragma unroll
    for (int i = 0; i < G_BK / 2; ++i) {
      const int kr = lr + 2 * i;
      const int64_t row = rb + kr;
      const bool rv = row < r_end;
      cp_async8(xd + kr * G_LDS + lc, rv && vx ? px + row * ldx : px, rv && vx);
      cp_async8(yd + kr * G_LDS + lc, rv && vy ? py + row * ldy : py, rv && vy);
    }
  };

  // warp tile placement and valid MMA-tile counts (skip tiles entirely outside M x N)
  const int wm = warp >> 1, wn = warp & 1;
  const int wm0 = m0 + wm * 8 * G_WM, wn0 = n0 + wn * 8 * G_WN;
  const int mtv = max(0, min(G_WM, (g.M - wm0 + 7) / 8));
  const int ntv = max(0, min(G_WN, (g.N - wn0 + 7) / 8));
  const bool warp_active = mtv > 0 && ntv > 0 && !(g.symmetric && ti == tj && wm > wn);

  double acc[G_WM][G_WN][2];
#pragma unroll
  for (int a = 0; a < G_WM; ++a)
#pragma unroll
    for (int b = 0; b < G_WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < G_STAGES - 1; ++s) {
    if (s < nstages) load_stage(s, s);
    cp_async_commit();
  }

  const int fr = lane & 3, fc = lane >> 2;  // fragment: k = lane%4, m/n = lane/4
  for (int s = 0; s < nstages; ++s) {
    cp_async_wait<G_STAGES - 2>();
    __syncthreads();
    {
      const int sn = s + G_STAGES - 1;
      if (sn < nstages) load_stage(sn, sn % G_STAGES);
      cp_async_commit();
    }
    if (warp_active) {
      const double* xs = Xs + (s % G_STAGES) * G_BK * G_LDS;
      const double* ys = Ys + (s % G_STAGES) * G_BK * G_LDS;
#pragma unroll
      for (int kk = 0; kk < G_BK; kk += 4) {
        double af[G_WM], bf[G_WN];
#pragma unroll
        for (int a = 0; a < G_WM; ++a) af[a] = xs[(kk + fr) * G_LDS + wm * 8 * G_WM + a * 8 + fc];
#pragma unroll
        for (int b = 0; b < G_WN; ++b) bf[b] = ys[(kk + fr) * G_LDS + wn * 8 * G_WN + b * 8 + fc];
#pragma unroll
        for (int a = 0; a < G_WM; ++a)
#pragma unroll
          for (int b = 0; b < G_WN; ++b)
            if (a < mtv && b < ntv) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: accumulator element (a,b,e) -> tile row wm*32+a*8+lane/4, col wn*32+b*8+2*(lane%4)+e
  auto store_final = [&](int lrow, int lcol, double v) {
    const int gi = m0 + lrow, gj = n0 + lcol;
    if (gi >= g.M || gj >= g.N) return;
    if (g.symmetric) {
      if (ti == tj && lrow > lcol) return;  // diagonal tile: upper triangle then mirror
      g.C[(int64_t)gi * g.ldc + gj] = v;
      g.C[(int64_t)gj * g.ldc + gi] = v;
    } else {
      g.C[(int64_t)gi * g.ldc + gj] = v;
    }
  };

  if (P.nchunks == 1) {
#pragma unroll
    for (int a = 0; a < G_WM; ++a)
#pragma unroll
      for (int b = 0; b < G_WN; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          store_final(wm * 8 * G_WM + a * 8 + (lane >> 2), wn * 8 * G_WN + b * 8 + 2 * (lane & 3) + e,
                      acc[a][b][e]);
    return;
  }

  const int64_t tile_id = (int64_t)pidx * P.max_tiles + slot;
  double* part = P.ws + (tile_id * P.nchunks + chunk) * (G_BM * G_BN);
#pragma unroll
  for (int a = 0; a < G_WM; ++a)
#pragma unroll
    for (int b = 0; b < G_WN; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        part[(wm * 8 * G_WM + a * 8 + (lane >> 2)) * G_BN + wn * 8 * G_WN + b * 8 + 2 * (lane & 3) + e] =
            acc[a][b][e];
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int t = atomicAdd(&P.tickets[tile_id], 1);
    s_last = (t == P.nchunks - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double* base = P.ws + tile_id * P.nchunks * (G_BM * G_BN);
  for (int e = tid; e < G_BM * G_BN; e += G_THREADS) {
    double v = 0.0;
    for (int c = 0; c < P.nchunks; ++c) v += __ldcg(base + (int64_t)c * (G_BM * G_BN) + e);
    store_final(e / G_BN, e % G_BN, v);
  }
  if (tid == 0) P.tickets[tile_id] = 0;  // reset for the next launch (stream-ordered)
}

static int g_smem_bytes() { return 2 * G_STAGES * G_BK * G_LDS * (int)sizeof(double); }

static void fill_tiles(GramProblem& g) {
  g.tiles_m = (g.M + G_BM - 1) / G_BM;
  g.tiles_n = (g.N + G_BN - 1) / G_BN;
  g.ntiles = g.symmetric ? g.tiles_m * (g.tiles_m + 1) / 2 : g.tiles_m * g.tiles_n;
}

static int choose_chunks(int64_t nrows, int64_t total_tiles) {
  // Wave-aware split-K: 3 resident CTAs per SM -> 444 slots.  Pick the chunk count (each
  // chunk >= 32 stages when possible) whose last wave is fullest: a 1.1-wave grid idles
  // most of the second wave.
  const int64_t slots = 3LL * kSMs;
  total_tiles = lmax(total_tiles, 1);
  const int64_t cmax = lmax(1, lmin(256, nrows / (32 * G_BK)));
  if (total_tiles >= 8 * slots || cmax == 1) return 1;
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t c = 1; c <= cmax; ++c) {
    const int64_t ctas = total_tiles * c;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (eff >= 0.92) return (int)c;  // smallest chunk count with a >= 92% full last wave
    if (eff > best_eff) { best_eff = eff; best = c; }
  }
  return (int)best;
}

// workspace layout: [tickets: 64 KB][partials]
constexpr int64_t kTicketBytes = 1 << 16;

static int launch_gram(GramParams& P, int64_t total_tiles_slots, void* ws, int64_t ws_bytes,
                       cudaStream_t st) {
  P.nchunks = choose_chunks(P.nrows, total_tiles_slots);
  int64_t part_bytes = (int64_t)total_tiles_slots * P.nchunks * G_BM * G_BN * sizeof(double);
  if (P.nchunks > 1) {
    // shrink chunks until the partials fit the workspace
    while (P.nchunks > 1 && kTicketBytes + part_bytes > ws_bytes) {
      P.nchunks = (P.nchunks + 1) / 2;
      part_bytes = (int64_t)total_tiles_slots * P.nchunks * G_BM * G_BN * sizeof(double);
    }
    if (P.nchunks > 1 && total_tiles_slots * (int64_t)sizeof(int) > kTicketBytes) P.nchunks = 1;
  }
  P.chunk_rows = (P.nrows + P.nchunks - 1) / P.nchunks;
  P.chunk_rows = ((P.chunk_rows + G_BK - 1) / G_BK) * G_BK;
  P.nchunks = (int)lmax(1, (P.nrows + P.chunk_rows - 1) / P.chunk_rows);
  P.tickets = reinterpret_cast<int*>(ws);
  P.ws = reinterpret_cast<double*>(static_cast<char*>(ws) + kTicketBytes);
  int64_t grid = (int64_t)P.nprob * P.max_tiles * P.nchunks;
  if (grid <= 0) return BK_OK;
  if (grid > 0x7fffffff) return BK_ERR_UNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, g_smem_bytes());
    attr = true;
  }
  BK_COUNT();
  gram_kernel<<<(unsigned)grid, G_THREADS, g_smem_bytes(), st>>>(P);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

}  // namespace bk

using namespace bk;

extern "C" int64_t bk_gram_ws_bytes(int64_t n, int m1, int m2) {
  int64_t tiles = (int64_t)((m1 + G_BM - 1) / G_BM) * ((m2 + G_BN - 1) / G_BN);
  int c = choose_chunks(n, tiles);
  return kTicketBytes + tiles * c * G_BM * G_BN * (int64_t)sizeof(double);
}

// C (m1 x m2, ldc) = X(:, 0:m1)^T Y(:, 0:m2) over n rows.  symmetric != 0 requires X == Y,
// m1 == m2 and computes half the tiles.  (core.py:43-49)
extern "C" int bk_gram_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y,
                         int64_t ldy, double* C, int64_t ldc, int symmetric, void* ws, int64_t ws_bytes,
                         void* stream) {
  if (n < 0 || m1 < 0 || m2 < 0 || (symmetric && m1 != m2)) return BK_ERR_ARG;
  if (m1 == 0 || m2 == 0) return BK_OK;
  if (n == 0) {
    for (int i = 0; i < m1; ++i)
      if (cudaMemsetAsync(C + (int64_t)i * ldc, 0, sizeof(double) * m2, (cudaStream_t)stream) != cudaSuccess)
        return BK_ERR_CUDA;
    return BK_OK;
  }
  GramParams P{};
  P.nprob = 1;
  P.explicit_list = 1;
  GramProblem& g = P.prob[0];
  g.xs[0] = {X, ldx, 0, m1};
  g.ys[0] = {Y, ldy, 0, m2};
  g.nxs = g.nys = 1;
  g.M = m1;
  g.N = m2;
  g.C = C;
  g.ldc = ldc;
  g.symmetric = symmetric ? 1 : 0;
  fill_tiles(g);
  P.max_tiles = g.ntiles;
  P.nrows = n;
  return launch_gram(P, g.ntiles, ws, ws_bytes, (cudaStream_t)stream);
}

// Two Grams sharing the row range in one launch: C1 = X1^T Y1, C2 = X2^T Y2 (e.g. the
// projection Grams X^T W and X^T P of ppcg.py:680-687).
extern "C" int bk_gram2_d(int64_t n, int m1a, int m2a, const double* X1, int64_t ldx1, const double* Y1,
                          int64_t ldy1, double* C1, int64_t ldc1, int m1b, int m2b, const double* X2,
                          int64_t ldx2, const double* Y2, int64_t ldy2, double* C2, int64_t ldc2, void* ws,
                          int64_t ws_bytes, void* stream) {
  if (n <= 0) return BK_ERR_ARG;
  GramParams P{};
  P.nprob = 2;
  P.explicit_list = 1;
  GramProblem* gs[2] = {&P.prob[0], &P.prob[1]};
  const double* xs[2] = {X1, X2};
  const double* ys[2] = {Y1, Y2};
  int64_t lx[2] = {ldx1, ldx2}, ly[2] = {ldy1, ldy2}, lc[2] = {ldc1, ldc2};
  int ma[2] = {m1a, m1b}, na[2] = {m2a, m2b};
  double* cs[2] = {C1, C2};
  int maxt = 0;
  for (int i = 0; i < 2; ++i) {
    GramProblem& g = *gs[i];
    g.xs[0] = {xs[i], lx[i], 0, ma[i]};
    g.ys[0] = {ys[i], ly[i], 0, na[i]};
    g.nxs = g.nys = 1;
    g.M = ma[i];
    g.N = na[i];
    g.C = cs[i];
    g.ldc = lc[i];
    g.symmetric = 0;
    fill_tiles(g);
    if (ma[i] == 0 || na[i] == 0) g.ntiles = 0;
    maxt = max(maxt, g.ntiles);
  }
  if (maxt == 0) return BK_OK;
  P.max_tiles = maxt;
  P.nrows = n;
  return launch_gram(P, (int64_t)maxt * 2, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int64_t bk_subblock_grams_ws_bytes(int64_t n, int k_act, int q, int has_p) {
  int nb = (k_act + q - 1) / q;
  int dmax = (has_p ? 3 : 2) * q;
  int t = (dmax + G_BM - 1) / G_BM;
  int64_t tiles = (int64_t)2 * nb * t * t;
  int c = choose_chunks(n, tiles);
  return kTicketBytes + tiles * c * G_BM * G_BN * (int64_t)sizeof(double);
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
  int nb = (k_act + q - 1) / q;
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
  int t = (P.dmax + G_BM - 1) / G_BM;
  P.max_tiles = t * t;  // non-symmetric slot count bounds the symmetric one
  P.nrows = n;
  return launch_gram(P, (int64_t)P.nprob * P.max_tiles, ws, ws_bytes, (cudaStream_t)stream);
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
