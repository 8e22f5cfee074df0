// Tall-skinny update GEMMs on FP64 tensor cores (DMMA):
//     Y = s (.) (alpha * X G + beta * Z)        X: n x K (row-major), G: K x N small
//
// Covers every n-tall product of the PPCG iteration:
//   * projection updates  W -= X G, AW -= AX G     (ppcg.py:443-445, four problems per launch)
//   * residual            W = T (.) (AX - X G)     (ppcg.py:630,758 + the Jacobi apply of
//                         ppcg.py:678 fused as the row scale s = d, operators.py:110)
//   * CholQR              X R^{-1}, AX R^{-1}      (core.py:99, ppcg.py:484; R^{-1} upper
//                         triangular -> K-tiles below the diagonal are skipped)
//   * Rayleigh-Ritz       S C, AS C                (ppcg.py:574-577)
//   * Taylor-polar        X p(Y), AX p(Y)          (ppcg.py:477-481)
// and, fused into the residual launch, the stopping metric of the NEXT iteration
// (rayleigh_ritz.py:71-92 on the leading k columns): ||AX_k - X_k G_kk||_F^2 is the
// partial-K accumulator snapshot after the first k columns of X, reduced deterministically
// (never written to HBM).
//
// Tiles: 64 rows x BN (BN = 128 for k_total-wide outputs, 64 otherwise), 4 warps (2 x 2,
// warp tile 32 x BN/2), two or three CTAs per SM; K in 16-column stages through a cp.async
// ring (16-byte copies when aligned), fragments double buffered, unpredicated DMMAs for full
// warp tiles.
#include "common.cuh"

namespace bk {

constexpr int T_BK = 16, T_THREADS = 128, T_BM = 64;
constexpr int T_XLD = T_BK + 4;  // 20 doubles = 4 mod 16: conflict-free A fragments

struct TsProblem {
  const double* X;
  const double* G;
  const double* Z;
  double* Y;
};

struct TsParams {
  TsProblem prob[4];
  int nprob;
  int64_t n;
  int K, N;
  int64_t ldx, ldg, ldz, ldy;
  double alpha, beta;
  const double* rowscale;  // may be null
  int upper_tri;           // G upper triangular: skip rows i >= col tile end
  int ksplit, nsplit;      // metric snapshot after K columns [0, ksplit) on output cols < nsplit
  int col_off;             // global index of output column 0 (strip launch of a split GEMM)
  int metric_accum;        // add to *metric_out instead of overwriting (second launch)
  int vec_x, vec_g;        // 16-byte copies allowed for X (even k offsets) / G
  double* metric_out;      // device scalar (sum of squares); null -> no metric
  double* metric_ws;       // per-CTA partials
  int* metric_ticket;
};

BK_DEV void cp_pair(double* dst, const double* src, int nvalid, bool vec, const double* fb) {
  if (vec) {
    cp_async16(dst, nvalid > 0 ? src : fb, nvalid * 8);
  } else {
    cp_async8(dst, nvalid > 0 ? src : fb, nvalid > 0);
    cp_async8(dst + 1, nvalid > 1 ? src + 1 : fb, nvalid > 1);
  }
}

template <int BN_, int STAGES_, int MINB_>
struct TCfg {
  static constexpr int BN = BN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int GLD = BN + 4;                 // = 4 mod 16
  static constexpr int WM = T_BM / 2 / 8, WN = BN / 2 / 8;
  static constexpr int XROWSTEP = T_THREADS / 8;     // X: 8 pairs per 16-column row
  static constexpr int XNLOAD = T_BM / XROWSTEP;
  static constexpr int GCPR = BN / 2;
  static constexpr int GROWSTEP = T_THREADS / GCPR;
  static constexpr int GNLOAD = T_BK / GROWSTEP;
  static constexpr int XSTAGE = T_BM * T_XLD, GSTAGE = T_BK * GLD;
  static constexpr int SMEM = STAGES * (XSTAGE + GSTAGE) * (int)sizeof(double);
};
using TBig = TCfg<128, 4, 2>;
using TSmall = TCfg<64, 4, 3>;
// right strip of a GEMM whose width is not a multiple of 64 (N = 523 = 8 x 64 + 11): the
// 64-wide tiles then all run full (~30.5 TF/s instead of ~27.5 when every ninth CTA streams
// its X rows for 11 columns), the strip runs 16-wide tiles in a second launch
using TStrip = TCfg<16, 4, 4>;

template <class C>
__global__ void __launch_bounds__(T_THREADS, C::MINB) tsgemm_kernel(const __grid_constant__ TsParams P) {
  constexpr int BN = C::BN, WM = C::WM, WN = C::WN, GLD = C::GLD, ST = C::STAGES;
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                   // [STAGES][BM][XLD]
  double* Gs = smem + ST * C::XSTAGE;  // [STAGES][BK][GLD]
  __shared__ double s_red[T_THREADS / 32];
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const TsProblem pr = P.prob[blockIdx.z];
  const int n0 = blockIdx.x * BN;
  const int64_t r0 = (int64_t)blockIdx.y * T_BM;
  const int kend_all = P.upper_tri ? min(P.K, P.col_off + n0 + BN) : P.K;

  const int xc = (tid & 7) * 2, xr = tid >> 3;
  const int gc = (tid % C::GCPR) * 2, gr = tid / C::GCPR;
  const int gnv = max(0, min(2, P.N - (n0 + gc)));

  auto load_stage = [&](int kb, int kstop, int st, bool vx) {
    double* xd = Xs + st * C::XSTAGE;
    double* gd = Gs + st * C::GSTAGE;
    const int kx = kb + xc;
    const int xnv = max(0, min(2, kstop - kx));
#pragma unroll
    for (int i = 0; i < C::XNLOAD; ++i) {
      const int lr = xr + C::XROWSTEP * i;
      const int64_t row = r0 + lr;
      cp_pair(xd + lr * T_XLD + xc, pr.X + row * P.ldx + kx, row < P.n ? xnv : 0, vx, pr.X);
    }
#pragma unroll
    for (int i = 0; i < C::GNLOAD; ++i) {
      const int lk = gr + C::GROWSTEP * i;
      const int k = kb + lk;
      cp_pair(gd + lk * GLD + gc, pr.G + (int64_t)k * P.ldg + n0 + gc, k < kstop ? gnv : 0, P.vec_g != 0, pr.G);
    }
  };

  const int wm = warp >> 1, wn = warp & 1;
  const int64_t wr0 = r0 + wm * 8 * WM;
  const int wc0 = n0 + wn * 8 * WN;
  const int mtv = (int)lmax(0, lmin(WM, (P.n - wr0 + 7) / 8));
  const int ntv = max(0, min(WN, (P.N - wc0 + 7) / 8));
  const bool active = mtv > 0 && ntv > 0;
  const bool full_tile = mtv == WM && ntv == WN;

  double acc[WM][WN][2];
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int fk = lane & 3, fm = lane >> 2;

  // the epilogue's Z tile (and row scales) are known now: pull them into L2 while the K loop
  // runs, so the epilogue loads do not expose an HBM round trip at the end of every CTA
  if (P.beta != 0.0 && pr.Z != nullptr && pr.Y != nullptr) {
    constexpr int LINES = BN * 8 / 128 > 0 ? BN * 8 / 128 : 1;  // 128-byte lines per tile row
    for (int e = tid; e < T_BM * LINES; e += T_THREADS) {
      const int64_t row = r0 + e / LINES;
      const int col = n0 + (e % LINES) * 16;
      if (row < P.n && col < P.N) prefetch_l2(pr.Z + row * P.ldz + col);
    }
  }
  if (P.rowscale != nullptr && pr.Y != nullptr && tid < T_BM / 16) {
    const int64_t row = r0 + tid * 16;
    if (row < P.n) prefetch_l2(P.rowscale + row);
  }

  // one K phase over [kbeg, kstop); after stage `snap` (if >= 0) runs snap_fn() on the
  // partial accumulators without draining the cp.async pipeline
  auto run_phase = [&](int kbeg, int kstop, int snap, auto&& snap_fn) {
    if (kstop <= kbeg) return;
    const bool vx = P.vec_x && !(kbeg & 1);
    const int nst = (kstop - kbeg + T_BK - 1) / T_BK;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
      if (s < nst) load_stage(kbeg + s * T_BK, kstop, s, vx);
      cp_async_commit();
    }
    for (int s = 0; s < nst; ++s) {
      cp_async_wait<ST - 2>();
      __syncthreads();
      {
        const int sn = s + ST - 1;
        if (sn < nst) load_stage(kbeg + sn * T_BK, kstop, sn % ST, vx);
        cp_async_commit();
      }
      if (active) {
        const double* xs = Xs + (s % ST) * C::XSTAGE + (wm * 8 * WM + fm) * T_XLD + fk;
        const double* gs = Gs + (s % ST) * C::GSTAGE + fk * GLD + wn * 8 * WN + fm;
        double af[2][WM], bf[2][WN];
#pragma unroll
        for (int a = 0; a < WM; ++a) af[0][a] = lds64(xs + a * 8 * T_XLD);
#pragma unroll
        for (int b = 0; b < WN; ++b) bf[0][b] = lds64(gs + b * 8);
        if (full_tile) {
#pragma unroll
          for (int kq = 0; kq < T_BK / 4; ++kq) {
            const int cur = kq & 1;
            dmma_step_il<WM, WN>(acc, af[cur], bf[cur], af[cur ^ 1], bf[cur ^ 1], xs + (kq + 1) * 4, 8 * T_XLD,
                                 gs + (kq + 1) * 4 * GLD, 8, kq + 1 < T_BK / 4);
          }
        } else {
#pragma unroll
          for (int kq = 0; kq < T_BK / 4; ++kq) {
            const int cur = kq & 1;
            if (kq + 1 < T_BK / 4) {
#pragma unroll
              for (int a = 0; a < WM; ++a) af[cur ^ 1][a] = xs[a * 8 * T_XLD + (kq + 1) * 4];
#pragma unroll
              for (int b = 0; b < WN; ++b) bf[cur ^ 1][b] = gs[(kq + 1) * 4 * GLD + b * 8];
            }
            dmma_block<WM, WN, false>(acc, af[cur], bf[cur], mtv, ntv);
          }
        }
      }
      if (s == snap) snap_fn();
    }
    cp_async_wait<0>();
    __syncthreads();
  };
  auto no_snap = [] {};

  // element (a,b,e) -> row wr0 + a*8 + lane/4, col wc0 + b*8 + 2*(lane%4) + e
  auto metric = [&] {
    double ss = 0.0;
    if (blockIdx.z == 0) {
#pragma unroll
      for (int a = 0; a < WM; ++a) {
        const int64_t row = wr0 + a * 8 + (lane >> 2);
        if (row >= P.n) continue;
#pragma unroll
        for (int b = 0; b < WN; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = wc0 + b * 8 + 2 * (lane & 3) + e;
            if (col < P.nsplit && col < P.N) {
              const double zv = P.beta != 0.0 ? pr.Z[row * P.ldz + col] : 0.0;
              const double v = P.alpha * acc[a][b][e] + P.beta * zv;
              ss = fma(v, v, ss);
            }
          }
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) s_red[warp] = ss;
    __syncthreads();
    const int64_t total = (int64_t)gridDim.x * gridDim.y * gridDim.z;
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < T_THREADS / 32; ++w) t += s_red[w];
      const int64_t cta = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      P.metric_ws[cta] = t;
      __threadfence();
      s_last = (atomicAdd(P.metric_ticket, 1) == total - 1);
    }
    __syncthreads();
    if (s_last) {  // block-uniform: the last CTA sums the partials with all its threads,
      __threadfence();  // each over a fixed strided subset, then a fixed-order tree
      double sum = 0.0;
      for (int64_t c = tid; c < total; c += T_THREADS) sum += __ldcg(P.metric_ws + c);
      sum = warp_sum(sum);
      if (lane == 0) s_red[warp] = sum;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < T_THREADS / 32; ++w) t += s_red[w];
        *P.metric_out = P.metric_accum ? *P.metric_out + t : t;
        *P.metric_ticket = 0;
      }
    }
  };
  if (P.metric_out != nullptr) {
    const int ks = min(P.ksplit, kend_all);
    if (ks > 0 && ks % T_BK == 0) {
      // snapshot at a stage boundary inside one pipelined K loop (same summation order)
      run_phase(0, kend_all, ks / T_BK - 1, metric);
    } else {
      run_phase(0, ks, -1, no_snap);
      metric();
      run_phase(ks, kend_all, -1, no_snap);
    }
  } else {
    run_phase(0, kend_all, -1, no_snap);
  }

  // ---- epilogue (metric-only launches pass Y = null)
  if (pr.Y == nullptr) return;
#pragma unroll
  for (int a = 0; a < WM; ++a) {
    const int64_t row = wr0 + a * 8 + (lane >> 2);
    if (row >= P.n) continue;
    const double sr = P.rowscale ? P.rowscale[row] : 1.0;
#pragma unroll
    for (int b = 0; b < WN; ++b) {
      const int col = wc0 + b * 8 + 2 * (lane & 3);
      double v0 = P.alpha * acc[a][b][0];
      double v1 = P.alpha * acc[a][b][1];
      const int64_t zo = row * P.ldz + col, yo = row * P.ldy + col;
      // 16-byte accesses when both columns exist and the pair is aligned (the usual case)
      const bool pair = col + 1 < P.N && ((reinterpret_cast<uintptr_t>(pr.Y + yo) & 15) == 0) &&
                        (P.beta == 0.0 || (reinterpret_cast<uintptr_t>(pr.Z + zo) & 15) == 0);
      if (pair) {
        if (P.beta != 0.0) {
          const double2 z = *reinterpret_cast<const double2*>(pr.Z + zo);
          v0 = fma(P.beta, z.x, v0);
          v1 = fma(P.beta, z.y, v1);
        }
        *reinterpret_cast<double2*>(pr.Y + yo) = make_double2(sr * v0, sr * v1);
        continue;
      }
      if (P.beta != 0.0) {
        if (col < P.N) v0 = fma(P.beta, pr.Z[zo], v0);
        if (col + 1 < P.N) v1 = fma(P.beta, pr.Z[zo + 1], v1);
      }
      if (col < P.N) pr.Y[yo] = sr * v0;
      if (col + 1 < P.N) pr.Y[yo + 1] = sr * v1;
    }
  }
}

template <class C>
static int launch_ts(TsParams& P, cudaStream_t st) {
  dim3 grid((P.N + C::BN - 1) / C::BN, (unsigned)((P.n + T_BM - 1) / T_BM), P.nprob);
  if (grid.y > 65535) return BK_ERR_UNSUPPORTED;
  // per launch (cheap): the attribute belongs to the current device's context
  cudaFuncSetAttribute(tsgemm_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  BK_COUNT();
  tsgemm_kernel<C><<<grid, T_THREADS, C::SMEM, st>>>(P);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// tile choice: 64x64 at 3 CTAs/SM measured fastest at config-2 shapes (28.1 vs 21.5
// TFLOP/s for 64x128, profiles/gemm_sweep_r01.json); PPCG_TS_TILE=128 selects the wide tile
static bool ts_big(int N) {
  static int force = [] {
    const char* e = getenv("PPCG_TS_TILE");
    return e ? atoi(e) : 0;
  }();
  return force == 128 && N >= 192;
}

}  // namespace bk

using namespace bk;

extern "C" int64_t bk_tsgemm_ws_bytes(int64_t n, int N) {
  const int bn = ts_big(N) ? TBig::BN : TSmall::BN;
  const int64_t ctas = ((n + T_BM - 1) / T_BM) * ((N + bn - 1) / bn) * 4;
  return 256 + ctas * (int64_t)sizeof(double);
}

// Batched Y_b = s (.) (alpha X_b G_b + beta Z_b), b < nprob <= 4; all problems share shapes
// and leading dimensions.  Y must not alias X.  Z may alias Y (in-place update).
// flags: bit0 = G upper triangular.  metric: if metric_out != null, also returns
// sum over rows, cols < nsplit of (alpha X[:, :ksplit] G[:ksplit, :] + beta Z)^2 for problem 0.
extern "C" int bk_tsgemm_batched_d(int nprob, int64_t n, int K, int N, double alpha, const double* const* Xs,
                                   int64_t ldx, const double* const* Gs, int64_t ldg, double beta,
                                   const double* const* Zs, int64_t ldz, double* const* Ys, int64_t ldy,
                                   const double* rowscale, int flags, int ksplit, int nsplit, double* metric_out,
                                   void* ws, int64_t ws_bytes, void* stream) {
  if (nprob < 1 || nprob > 4 || n < 0 || K < 0 || N < 0) return BK_ERR_ARG;
  if (n == 0 || N == 0) return BK_OK;
  TsParams P{};
  P.nprob = nprob;
  P.vec_x = !(ldx & 1);
  P.vec_g = !(ldg & 1);
  for (int b = 0; b < nprob; ++b) {
    P.prob[b].X = Xs[b];
    P.prob[b].G = Gs[b];
    P.prob[b].Z = Zs ? Zs[b] : nullptr;
    P.prob[b].Y = Ys[b];
    if (beta != 0.0 && P.prob[b].Z == nullptr) return BK_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(Xs[b]) & 15) P.vec_x = 0;
    if (reinterpret_cast<uintptr_t>(Gs[b]) & 15) P.vec_g = 0;
  }
  P.n = n;
  P.K = K;
  P.N = N;
  P.ldx = ldx;
  P.ldg = ldg;
  P.ldz = ldz;
  P.ldy = ldy;
  P.alpha = alpha;
  P.beta = beta;
  P.rowscale = rowscale;
  P.upper_tri = flags & 1;
  P.ksplit = ksplit;
  P.nsplit = nsplit;
  const int bn = ts_big(N) ? TBig::BN : TSmall::BN;
  if (metric_out) {
    const int64_t ctas = ((n + T_BM - 1) / T_BM) * ((N + bn - 1) / bn) * nprob;
    const int64_t need = 256 + ctas * (int64_t)sizeof(double);
    if (ws == nullptr || ws_bytes < need) return BK_ERR_ARG;
    P.metric_ticket = reinterpret_cast<int*>(ws);
    P.metric_ws = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
    P.metric_out = metric_out;
  }
  if (ts_big(N)) return launch_ts<TBig>(P, (cudaStream_t)stream);
  static const int split_on = [] {
    const char* e = getenv("PPCG_TS_SPLIT");
    return e ? atoi(e) : 1;
  }();
  const int N1 = N / 64 * 64;
  if (!split_on || N < 128 || N1 == N) return launch_ts<TSmall>(P, (cudaStream_t)stream);
  // main: columns [0, N1); strip: [N1, N) with the metric (if any) accumulated
  TsParams S = P;
  P.N = N1;
  P.nsplit = min(P.nsplit, N1);
  int rc = launch_ts<TSmall>(P, (cudaStream_t)stream);
  if (rc != BK_OK) return rc;
  S.N = N - N1;
  S.col_off = N1;
  for (int b = 0; b < nprob; ++b) {
    S.prob[b].G = S.prob[b].G + N1;
    if (S.prob[b].Z) S.prob[b].Z = S.prob[b].Z + N1;
    if (S.prob[b].Y) S.prob[b].Y = S.prob[b].Y + N1;
  }
  S.vec_g = S.vec_g && !(N1 & 1);
  if (S.metric_out) {
    S.nsplit = max(0, S.nsplit - N1);
    S.metric_accum = 1;
    if (S.nsplit == 0) S.metric_out = nullptr;  // nothing of the metric lies in the strip
  }
  bool any_y = false;
  for (int b = 0; b < nprob; ++b) any_y = any_y || S.prob[b].Y != nullptr;
  if (!any_y && !S.metric_out) return BK_OK;  // metric-only launch fully covered by the main part
  return launch_ts<TStrip>(S, (cudaStream_t)stream);
}

extern "C" int bk_tsgemm_d(int64_t n, int K, int N, double alpha, const double* X, int64_t ldx, const double* G,
                           int64_t ldg, double beta, const double* Z, int64_t ldz, double* Y, int64_t ldy,
                           const double* rowscale, int flags, void* stream) {
  const double* xs[1] = {X};
  const double* gs[1] = {G};
  const double* zs[1] = {Z};
  double* ys[1] = {Y};
  return bk_tsgemm_batched_d(1, n, K, N, alpha, xs, ldx, gs, ldg, beta, Z ? zs : nullptr, ldz, ys, ldy, rowscale,
                             flags, 0, 0, nullptr, nullptr, 0, stream);
}
