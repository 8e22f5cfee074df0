// Block operator apply Y = A X for CSR matrices (real and complex), HBM-bound.
//
// Replaces SparseHermitian.apply (blockeig problems.py:72-73, scipy csr_matvecs) called
// once per iteration on W (ppcg.py:679), on the full block at initialisation and at each
// Rayleigh-Ritz pass (ppcg.py:626, 575), and for cache refreshes (ppcg.py:718-724).
//
// Row-major blocks make each CSR row a gather of whole X rows: one warp per output row,
// lanes over columns (coalesced 256 B per warp load), the row's (col, val) pairs loaded
// once per 32-entry batch by the lanes and broadcast with shuffles.  Row-major X rows of
// 7/27-point stencils have reuse distances of one grid plane, far inside the 126 MB L2, so
// DRAM traffic is ~ read X once + write Y once + the CSR arrays.
#include "common.cuh"

namespace bk {

constexpr int S_THREADS = 256;

template <int NV>
__global__ void __launch_bounds__(S_THREADS) spmm_csr_real(int64_t n, const int32_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ val, int m,
                                                           const double* __restrict__ X, int64_t ldx,
                                                           double* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (S_THREADS / 32) + (threadIdx.x >> 5);
  if (row >= n) return;
  const int kb = rowptr[row], ke = rowptr[row + 1];
  for (int c0 = 0; c0 < m; c0 += 32 * NV) {
    double acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
    for (int k0 = kb; k0 < ke; k0 += 32) {
      const int kk = k0 + lane;
      const int cj = kk < ke ? col[kk] : 0;
      const double aj = kk < ke ? val[kk] : 0.0;
      const int cnt = min(32, ke - k0);
      for (int t = 0; t < cnt; ++t) {
        const int64_t jr = __shfl_sync(0xffffffffu, cj, t);
        const double a = __shfl_sync(0xffffffffu, aj, t);
        const double* xr = X + jr * ldx;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int c = c0 + v * 32 + lane;
          if (c < m) acc[v] = fma(a, __ldg(xr + c), acc[v]);
        }
      }
    }
    double* yr = Y + row * ldy;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = c0 + v * 32 + lane;
      if (c < m) yr[c] = acc[v];
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(S_THREADS) spmm_csr_cplx(int64_t n, const int32_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ col,
                                                           const double2* __restrict__ val, int m,
                                                           const double2* __restrict__ X, int64_t ldx,
                                                           double2* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (S_THREADS / 32) + (threadIdx.x >> 5);
  if (row >= n) return;
  const int kb = rowptr[row], ke = rowptr[row + 1];
  for (int c0 = 0; c0 < m; c0 += 32 * NV) {
    double2 acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = make_double2(0.0, 0.0);
    for (int k0 = kb; k0 < ke; k0 += 32) {
      const int kk = k0 + lane;
      const int cj = kk < ke ? col[kk] : 0;
      const double2 aj = kk < ke ? val[kk] : make_double2(0.0, 0.0);
      const int cnt = min(32, ke - k0);
      for (int t = 0; t < cnt; ++t) {
        const int64_t jr = __shfl_sync(0xffffffffu, cj, t);
        const double ar = __shfl_sync(0xffffffffu, aj.x, t);
        const double ai = __shfl_sync(0xffffffffu, aj.y, t);
        const double2* xr = X + jr * ldx;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int c = c0 + v * 32 + lane;
          if (c < m) {
            const double2 x = __ldg(xr + c);
            acc[v].x = fma(ar, x.x, fma(-ai, x.y, acc[v].x));
            acc[v].y = fma(ar, x.y, fma(ai, x.x, acc[v].y));
          }
        }
      }
    }
    double2* yr = Y + row * ldy;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = c0 + v * 32 + lane;
      if (c < m) yr[c] = acc[v];
    }
  }
}

}  // namespace bk

using namespace bk;

// Y(:, 0:m) = A X(:, 0:m) for a CSR A with n rows (int32 indices).  X and Y row-major.
extern "C" int bk_spmm_csr_d(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, int m,
                             const double* X, int64_t ldx, double* Y, int64_t ldy, void* stream) {
  if (n < 0 || m < 0) return BK_ERR_ARG;
  if (n == 0 || m == 0) return BK_OK;
  const unsigned grid = (unsigned)((n + S_THREADS / 32 - 1) / (S_THREADS / 32));
  cudaStream_t st = (cudaStream_t)stream;
  BK_COUNT();
  if (m <= 32) spmm_csr_real<1><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, val, m, X, ldx, Y, ldy);
  else if (m <= 64) spmm_csr_real<2><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, val, m, X, ldx, Y, ldy);
  else if (m <= 128) spmm_csr_real<4><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, val, m, X, ldx, Y, ldy);
  else spmm_csr_real<8><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, val, m, X, ldx, Y, ldy);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// complex128: val, X, Y are interleaved (re, im); ld in complex elements
extern "C" int bk_spmm_csr_z(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, int m,
                             const double* X, int64_t ldx, double* Y, int64_t ldy, void* stream) {
  if (n < 0 || m < 0) return BK_ERR_ARG;
  if (n == 0 || m == 0) return BK_OK;
  const unsigned grid = (unsigned)((n + S_THREADS / 32 - 1) / (S_THREADS / 32));
  cudaStream_t st = (cudaStream_t)stream;
  auto v2 = reinterpret_cast<const double2*>(val);
  auto x2 = reinterpret_cast<const double2*>(X);
  auto y2 = reinterpret_cast<double2*>(Y);
  BK_COUNT();
  if (m <= 32) spmm_csr_cplx<1><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, v2, m, x2, ldx, y2, ldy);
  else if (m <= 64) spmm_csr_cplx<2><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, v2, m, x2, ldx, y2, ldy);
  else spmm_csr_cplx<4><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, v2, m, x2, ldx, y2, ldy);
  BK_CHECK_LAUNCH();
  return BK_OK;
}
