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
#include "common.cuh"

namespace bk {

constexpr int T_BM = 128, T_BN = 64, T_BK = 16, T_STAGES = 3, T_THREADS = 256;
constexpr int T_XLD = T_BK + 4;    // 20 doubles: conflict-free A fragments
constexpr int T_GLD = T_BN + 4;    // 68 = 4 mod 16 doubles: conflict-free B fragments
constexpr int T_WM = 4, T_WN = 4;  // warp tile 32 x 32, warps 4 (rows) x 2 (cols)

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
  double* metric_out;      // device scalar (sum of squares); null -> no metric
  double* metric_ws;       // per-CTA partials
  int* metric_ticket;
};

__global__ void __launch_bounds__(T_THREADS, 2) tsgemm_kernel(const __grid_constant__ TsParams P) {
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                              // [STAGES][BM][XLD]
  double* Gs = smem + T_STAGES * T_BM * T_XLD;    // [STAGES][BK][GLD]
  __shared__ double s_red[T_THREADS / 32];
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const TsProblem pr = P.prob[blockIdx.z];
  const int n0 = blockIdx.x * T_BN;
  const int64_t r0 = (int64_t)blockIdx.y * T_BM;

  const int kend_all = P.upper_tri ? min(P.K, n0 + T_BN) : P.K;

  // loader geometry
  const int xc = tid & 15, xr = tid >> 4;   // X: col fixed, rows xr + 16 i (i < 8)
  const int gc = tid & 63, gr = tid >> 6;   // G: col fixed, rows gr + 4 i (i < 4)

  auto load_stage = [&](int kb, int kstop, int st) {
    double* xd = Xs + st * T_BM * T_XLD;
    double* gd = Gs + st * T_BK * T_GLD;
    const int kx = kb + xc;
    const bool kxv = kx < kstop;
#pragma unroll
    for (int i = 0; i < T_BM / 16; ++i) {
      const int lr = xr + 16 * i;
      const int64_t row = r0 + lr;
      const bool v = kxv && row < P.n;
      cp_async8(xd + lr * T_XLD + xc, v ? pr.X + row * P.ldx + kx : pr.X, v);
    }
    const bool gcv = n0 + gc < P.N;
#pragma unroll
    for (int i = 0; i < T_BK / 4; ++i) {
      const int lk = gr + 4 * i;
      const int k = kb + lk;
      const bool v = gcv && k < kstop;
      cp_async8(gd + lk * T_GLD + gc, v ? pr.G + (int64_t)k * P.ldg + n0 + gc : pr.G, v);
    }
  };

  const int wm = warp >> 1, wn = warp & 1;
  const int64_t wr0 = r0 + wm * 32;
  const int wc0 = n0 + wn * 32;
  const int mtv = (int)lmax(0, lmin(T_WM, (P.n - wr0 + 7) / 8));
  const int ntv = max(0, min(T_WN, (P.N - wc0 + 7) / 8));
  const bool active = mtv > 0 && ntv > 0;

  double acc[T_WM][T_WN][2];
#pragma unroll
  for (int a = 0; a < T_WM; ++a)
#pragma unroll
    for (int b = 0; b < T_WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int fk = lane & 3, fm = lane >> 2;

  // one K phase over [kbeg, kstop)
  auto run_phase = [&](int kbeg, int kstop) {
    if (kstop <= kbeg) return;
    const int nst = (kstop - kbeg + T_BK - 1) / T_BK;
#pragma unroll
    for (int s = 0; s < T_STAGES - 1; ++s) {
      if (s < nst) load_stage(kbeg + s * T_BK, kstop, s);
      cp_async_commit();
    }
    for (int s = 0; s < nst; ++s) {
      cp_async_wait<T_STAGES - 2>();
      __syncthreads();
      {
        const int sn = s + T_STAGES - 1;
        if (sn < nst) load_stage(kbeg + sn * T_BK, kstop, sn % T_STAGES);
        cp_async_commit();
      }
      if (active) {
        const double* xs = Xs + (s % T_STAGES) * T_BM * T_XLD;
        const double* gs = Gs + (s % T_STAGES) * T_BK * T_GLD;
#pragma unroll
        for (int kk = 0; kk < T_BK; kk += 4) {
          double af[T_WM], bf[T_WN];
#pragma unroll
          for (int a = 0; a < T_WM; ++a) af[a] = xs[(wm * 32 + a * 8 + fm) * T_XLD + kk + fk];
#pragma unroll
          for (int b = 0; b < T_WN; ++b) bf[b] = gs[(kk + fk) * T_GLD + wn * 32 + b * 8 + fm];
#pragma unroll
          for (int a = 0; a < T_WM; ++a)
#pragma unroll
            for (int b = 0; b < T_WN; ++b)
              if (a < mtv && b < ntv) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
  };

  // element (a,b,e) -> row wr0 + a*8 + lane/4, col wc0 + b*8 + 2*(lane%4) + e
  if (P.metric_out != nullptr) {
    const int ks = min(P.ksplit, kend_all);
    run_phase(0, ks);
    double ss = 0.0;
    if (blockIdx.z == 0) {
#pragma unroll
      for (int a = 0; a < T_WM; ++a) {
        const int64_t row = wr0 + a * 8 + (lane >> 2);
        if (row >= P.n) continue;
#pragma unroll
        for (int b = 0; b < T_WN; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = wc0 + b * 8 + 2 * (lane & 3) + e;
            if (col < P.nsplit && col < P.N) {
              double zv = P.beta != 0.0 ? pr.Z[row * P.ldz + col] : 0.0;
              double v = P.alpha * acc[a][b][e] + P.beta * zv;
              ss = fma(v, v, ss);
            }
          }
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) s_red[warp] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < T_THREADS / 32; ++w) t += s_red[w];
      const int64_t cta = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      P.metric_ws[cta] = t;
      __threadfence();
      const int64_t total = (int64_t)gridDim.x * gridDim.y * gridDim.z;
      int tk = atomicAdd(P.metric_ticket, 1);
      s_last = (tk == total - 1);
      if (s_last) {
        __threadfence();
        double sum = 0.0;
        for (int64_t c = 0; c < total; ++c) sum += __ldcg(P.metric_ws + c);
        *P.metric_out = sum;
        *P.metric_ticket = 0;
      }
    }
    run_phase(ks, kend_all);
  } else {
    run_phase(0, kend_all);
  }

  // ---- epilogue (metric-only launches pass Y = null)
  if (pr.Y == nullptr) return;
#pragma unroll
  for (int a = 0; a < T_WM; ++a) {
    const int64_t row = wr0 + a * 8 + (lane >> 2);
    if (row >= P.n) continue;
    const double sr = P.rowscale ? P.rowscale[row] : 1.0;
#pragma unroll
    for (int b = 0; b < T_WN; ++b) {
      const int col = wc0 + b * 8 + 2 * (lane & 3);
      double v0 = P.alpha * acc[a][b][0];
      double v1 = P.alpha * acc[a][b][1];
      if (P.beta != 0.0) {
        if (col < P.N) v0 = fma(P.beta, pr.Z[row * P.ldz + col], v0);
        if (col + 1 < P.N) v1 = fma(P.beta, pr.Z[row * P.ldz + col + 1], v1);
      }
      if (col < P.N) pr.Y[row * P.ldy + col] = sr * v0;
      if (col + 1 < P.N) pr.Y[row * P.ldy + col + 1] = sr * v1;
    }
  }
}

static int t_smem_bytes() { return (T_STAGES * T_BM * T_XLD + T_STAGES * T_BK * T_GLD) * (int)sizeof(double); }

}  // namespace bk

using namespace bk;

extern "C" int64_t bk_tsgemm_ws_bytes(int64_t n, int N) {
  int64_t ctas = ((n + T_BM - 1) / T_BM) * ((N + T_BN - 1) / T_BN) * 4;
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
  for (int b = 0; b < nprob; ++b) {
    P.prob[b].X = Xs[b];
    P.prob[b].G = Gs[b];
    P.prob[b].Z = Zs ? Zs[b] : nullptr;
    P.prob[b].Y = Ys[b];
    if (beta != 0.0 && P.prob[b].Z == nullptr) return BK_ERR_ARG;
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
  dim3 grid((N + T_BN - 1) / T_BN, (unsigned)((n + T_BM - 1) / T_BM), nprob);
  if (grid.y > 65535) return BK_ERR_UNSUPPORTED;
  if (metric_out) {
    int64_t need = 256 + (int64_t)grid.x * grid.y * grid.z * sizeof(double);
    if (ws == nullptr || ws_bytes < need) return BK_ERR_ARG;
    P.metric_ticket = reinterpret_cast<int*>(ws);
    P.metric_ws = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
    P.metric_out = metric_out;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tsgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, t_smem_bytes());
    attr = true;
  }
  BK_COUNT();
  tsgemm_kernel<<<grid, T_THREADS, t_smem_bytes(), (cudaStream_t)stream>>>(P);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_tsgemm_d(int64_t n, int K, int N, double alpha, const double* X, int64_t ldx, const double* G,
                           int64_t ldg, double beta, const double* Z, int64_t ldz, double* Y, int64_t ldy,
                           const double* rowscale, int flags, void* stream) {
  const double* xs[1] = {X};
  const double* gs[1] = {G};
  const double* zs[1] = {Z};
  double* ys[1] = {Y};
  return bk_tsgemm_batched_d(1, n, K, N, alpha, xs, ldx, gs, ldg, beta, Z ? zs : nullptr, ldz, ys, ldy,
                             rowscale, flags, 0, 0, nullptr, nullptr, 0, stream);
}
