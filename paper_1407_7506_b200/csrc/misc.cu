// Elementwise and reduction kernels of the PPCG iteration (HBM-bound or tiny).
//
//   bk_scale_rows_d       Y = d (.) X : DiagonalPreconditioner / DiagonalOperator apply
//                         (operators.py:63-73, 96-110) when not fused into a GEMM epilogue
//   bk_sumsq_d            ||X||_F^2, deterministic (ppcg.py:689 norm of W)
//   bk_small_stats_d      ||C||_F^2, ||C - I||_F^2, Re tr C of a small matrix
//                         (rayleigh_ritz.py:83-85, ppcg.py:452, ppcg.py:690)
//   bk_rr_residual_d      R = AV - V diag(omega), W = s (.) R, ||R(:,j)||^2
//                         (ppcg.py:576-582 and the W hand-off of ppcg.py:396-397 + 678)
//   bk_cplx_expand_d      complex K x N G -> real 2K x 2N so complex X G runs on the real
//                         DMMA kernel over the interleaved real view
//   bk_cplx_gram_combine  real Gram of interleaved views -> complex X^H Y
//   bk_copy_cols_d        strided column-range copy (cudaMemcpy2DAsync)
#include "common.cuh"

namespace bk {

__global__ void k_scale_rows(int64_t n, int m, const double* __restrict__ d, const double* __restrict__ X,
                             int64_t ldx, double* __restrict__ Y, int64_t ldy) {
  const int64_t tot = n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / m;
    const int c = (int)(e % m);
    Y[r * ldy + c] = d[r] * X[r * ldx + c];
  }
}

constexpr int SQ_CTAS = 2 * kSMs, SQ_THREADS = 256;

__global__ void __launch_bounds__(SQ_THREADS) k_sumsq(int64_t n, int m, const double* __restrict__ X, int64_t ldx,
                                                      double* part, int* ticket, double* out) {
  __shared__ double red[SQ_THREADS / 32];
  __shared__ int last;
  const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t rb = blockIdx.x * rows_per, re = min(n, rb + rows_per);
  double s = 0.0;
  const int64_t tot = (re > rb) ? (re - rb) * m : 0;
  for (int64_t e = threadIdx.x; e < tot; e += SQ_THREADS) {
    const double v = X[(rb + e / m) * ldx + e % m];
    s = fma(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < SQ_THREADS / 32; ++i) t += red[i];
    part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
    if (last) {
      __threadfence();
      double a = 0.0;
      for (int i = 0; i < (int)gridDim.x; ++i) a += __ldcg(part + i);
      out[0] = a;
      *ticket = 0;
    }
  }
}

__global__ void k_small_stats(int m1, int m2, const double* C, int64_t ldc, int cplx, double* out) {
  __shared__ double r0[32], r1[32], r2[32];
  double s = 0.0, si = 0.0, tr = 0.0;
  const int w = cplx ? 2 : 1;
  // warps own rows, lanes columns (coalesced, no index division)
  const int nw = blockDim.x >> 5, wq = threadIdx.x >> 5, ln = threadIdx.x & 31;
  for (int i = wq; i < m1; i += nw) {
    const double* rowp = C + (int64_t)i * ldc * w;
    for (int j = ln; j < m2; j += 32) {
      const double* p = rowp + (int64_t)j * w;
      double a2 = p[0] * p[0];
      if (cplx) a2 += p[1] * p[1];
      s += a2;
      if (i == j) {
        const double dr = p[0] - 1.0;
        si += dr * dr + (cplx ? p[1] * p[1] : 0.0);
        tr += p[0];
      } else {
        si += a2;
      }
    }
  }
  s = warp_sum(s);
  si = warp_sum(si);
  tr = warp_sum(tr);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  if (lane == 0) { r0[wp] = s; r1[wp] = si; r2[wp] = tr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a += r0[i]; b += r1[i]; c += r2[i]; }
    out[0] = a;
    out[1] = b;
    out[2] = c;
  }
}

// rows split over CTAs; each CTA writes partial column sums; last CTA reduces in order
constexpr int RR_THREADS = 256;
__global__ void __launch_bounds__(RR_THREADS) k_rr_residual(int64_t n, int kt, int cplx, const double* __restrict__ V,
                                                           int64_t ldv, const double* __restrict__ AV, int64_t ldav,
                                                           const double* __restrict__ omega,
                                                           const double* __restrict__ rowscale, double* W,
                                                           int64_t ldw, double* part, int* ticket,
                                                           double* colnorm2) {
  extern __shared__ double colacc[];  // kt doubles
  __shared__ int last;
  const int w = cplx ? 2 : 1;
  const int mr = kt * w;  // real columns
  for (int c = threadIdx.x; c < kt; c += RR_THREADS) colacc[c] = 0.0;
  __syncthreads();
  const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t rb = blockIdx.x * rows_per, re = min(n, rb + rows_per);
  // each thread owns real columns c = threadIdx.x + k*RR_THREADS; loops its rows
  for (int c = threadIdx.x; c < mr; c += RR_THREADS) {
    const int jc = c / w;
    const double om = omega[jc];
    double s = 0.0;
    for (int64_t r = rb; r < re; ++r) {
      const double rv = AV[r * ldav * w + c] - V[r * ldv * w + c] * om;
      s = fma(rv, rv, s);
      if (W) W[r * ldw * w + c] = (rowscale ? rowscale[r] : 1.0) * rv;
    }
    if (w == 1) colacc[jc] = s;
    else atomicAdd(&colacc[jc], s);  // two real columns per complex column; order irrelevant (2 terms)
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kt; c += RR_THREADS) part[(int64_t)blockIdx.x * kt + c] = colacc[c];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = threadIdx.x; c < kt; c += RR_THREADS) {
    double a = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) a += __ldcg(part + (int64_t)b * kt + c);
    colnorm2[c] = a;
  }
  if (threadIdx.x == 0) *ticket = 0;
}

__global__ void k_cplx_expand(int K, int N, const double* G, int64_t ldg, double* Gr, int64_t ldr) {
  const int64_t tot = (int64_t)K * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / N), j = (int)(e % N);
    const double gr = G[2 * (i * ldg + j)], gi = G[2 * (i * ldg + j) + 1];
    Gr[(2 * i) * ldr + 2 * j] = gr;
    Gr[(2 * i) * ldr + 2 * j + 1] = gi;
    Gr[(2 * i + 1) * ldr + 2 * j] = -gi;
    Gr[(2 * i + 1) * ldr + 2 * j + 1] = gr;
  }
}

__global__ void k_cplx_gram_combine(int m1, int m2, const double* Cr, int64_t ldr, double* C, int64_t ldc) {
  const int64_t tot = (int64_t)m1 * m2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / m2), j = (int)(e % m2);
    const double rr = Cr[(2 * i) * ldr + 2 * j], ri = Cr[(2 * i) * ldr + 2 * j + 1];
    const double ir = Cr[(2 * i + 1) * ldr + 2 * j], ii = Cr[(2 * i + 1) * ldr + 2 * j + 1];
    C[2 * (i * ldc + j)] = rr + ii;
    C[2 * (i * ldc + j) + 1] = ri - ir;
  }
}

static unsigned gridn(int64_t tot) { return (unsigned)lmin(8 * kSMs * 4, lmax(1, (tot + 255) / 256)); }

}  // namespace bk

using namespace bk;

extern "C" int bk_scale_rows_d(int64_t n, int m, const double* d, const double* X, int64_t ldx, double* Y,
                               int64_t ldy, void* stream) {
  if (n < 0 || m < 0) return BK_ERR_ARG;
  if (n == 0 || m == 0) return BK_OK;
  BK_COUNT();
  k_scale_rows<<<gridn(n * m), 256, 0, (cudaStream_t)stream>>>(n, m, d, X, ldx, Y, ldy);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int64_t bk_sumsq_ws_bytes(void) { return 256 + SQ_CTAS * sizeof(double); }

extern "C" int bk_sumsq_d(int64_t n, int m, const double* X, int64_t ldx, double* out, void* ws, int64_t ws_bytes,
                          void* stream) {
  if (n < 0 || m < 0 || ws_bytes < bk_sumsq_ws_bytes()) return BK_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0 || m == 0) return cudaMemsetAsync(out, 0, sizeof(double), st) == cudaSuccess ? BK_OK : BK_ERR_CUDA;
  int* ticket = reinterpret_cast<int*>(ws);
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  BK_COUNT();
  k_sumsq<<<SQ_CTAS, SQ_THREADS, 0, st>>>(n, m, X, ldx, part, ticket, out);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// out[0] = sum |c|^2, out[1] = sum |c - delta|^2, out[2] = Re trace (cplx: interleaved)
extern "C" int bk_small_stats_d(int m1, int m2, const double* C, int64_t ldc, int cplx, double* out, void* stream) {
  if (m1 < 0 || m2 < 0) return BK_ERR_ARG;
  BK_COUNT();
  k_small_stats<<<1, 1024, 0, (cudaStream_t)stream>>>(m1, m2, C, ldc, cplx, out);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int64_t bk_rr_residual_ws_bytes(int kt) { return 256 + (int64_t)2 * kSMs * kt * sizeof(double); }

extern "C" int bk_rr_residual_d(int64_t n, int kt, int cplx, const double* V, int64_t ldv, const double* AV,
                                int64_t ldav, const double* omega, const double* rowscale, double* W, int64_t ldw,
                                double* colnorm2, void* ws, int64_t ws_bytes, void* stream) {
  if (n <= 0 || kt <= 0 || ws_bytes < bk_rr_residual_ws_bytes(kt)) return BK_ERR_ARG;
  const int ctas = 2 * kSMs;
  const int smem = kt * (int)sizeof(double);
  if (smem > 200 * 1024) return BK_ERR_UNSUPPORTED;
  static int attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(k_rr_residual, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = smem;
  }
  int* ticket = reinterpret_cast<int*>(ws);
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  BK_COUNT();
  k_rr_residual<<<ctas, RR_THREADS, smem, (cudaStream_t)stream>>>(n, kt, cplx, V, ldv, AV, ldav, omega, rowscale, W,
                                                                  ldw, part, ticket, colnorm2);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_cplx_expand_d(int K, int N, const double* G, int64_t ldg, double* Gr, int64_t ldr, void* stream) {
  if (K < 0 || N < 0) return BK_ERR_ARG;
  if (K == 0 || N == 0) return BK_OK;
  BK_COUNT();
  k_cplx_expand<<<gridn((int64_t)K * N), 256, 0, (cudaStream_t)stream>>>(K, N, G, ldg, Gr, ldr);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_cplx_gram_combine_d(int m1, int m2, const double* Cr, int64_t ldr, double* C, int64_t ldc,
                                      void* stream) {
  if (m1 < 0 || m2 < 0) return BK_ERR_ARG;
  if (m1 == 0 || m2 == 0) return BK_OK;
  BK_COUNT();
  k_cplx_gram_combine<<<gridn((int64_t)m1 * m2), 256, 0, (cudaStream_t)stream>>>(m1, m2, Cr, ldr, C, ldc);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// dst[r][dc0 + c] = src[r][sc0 + c] for r < n, c < w  (elem_bytes 8 or 16)
extern "C" int bk_copy_cols(int64_t n, int w, int elem_bytes, const void* src, int64_t lds, int64_t sc0, void* dst,
                            int64_t ldd, int64_t dc0, void* stream) {
  if (n < 0 || w < 0) return BK_ERR_ARG;
  if (n == 0 || w == 0) return BK_OK;
  const char* s = static_cast<const char*>(src) + sc0 * elem_bytes;
  char* d = static_cast<char*>(dst) + dc0 * elem_bytes;
  return cudaMemcpy2DAsync(d, ldd * elem_bytes, s, lds * elem_bytes, (size_t)w * elem_bytes, n,
                           cudaMemcpyDeviceToDevice, (cudaStream_t)stream) == cudaSuccess
             ? BK_OK
             : BK_ERR_CUDA;
}

extern "C" int bk_zero_cols(int64_t n, int w, int elem_bytes, void* dst, int64_t ldd, int64_t dc0, void* stream) {
  if (n < 0 || w < 0) return BK_ERR_ARG;
  if (n == 0 || w == 0) return BK_OK;
  char* d = static_cast<char*>(dst) + dc0 * elem_bytes;
  return cudaMemset2DAsync(d, ldd * elem_bytes, 0, (size_t)w * elem_bytes, n, (cudaStream_t)stream) == cudaSuccess
             ? BK_OK
             : BK_ERR_CUDA;
}

extern "C" int bk_version(void) { return 1; }

unsigned long long bk_launch_counter = 0;
extern "C" unsigned long long bk_launch_count(void) { return __atomic_load_n(&bk_launch_counter, __ATOMIC_RELAXED); }
