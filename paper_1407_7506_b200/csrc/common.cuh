// Shared device helpers for the PPCG sm_100a kernels.
//
// Layout convention: every n x m block is row-major with leading
// dimension ld (element (r, c) at p[r * ld + c]), exactly the C-order numpy layout of the
// reference (SURVEY.md §8 preamble).  Complex blocks are interleaved (re, im) pairs, so a
// complex n x m block is also a real n x 2m block; the FP64 tensor kernels only ever see
// real views and complex products are assembled from them.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/ppcg_b200.h"

#define BK_DEV __device__ __forceinline__

// host-side count of kernels launched by this library (exported as bk_launch_count)
extern unsigned long long bk_launch_counter;
#define BK_COUNT() __atomic_fetch_add(&bk_launch_counter, 1ull, __ATOMIC_RELAXED)

#define BK_CHECK_LAUNCH()                                   \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return BK_ERR_CUDA;              \
  } while (0)

namespace bk {

constexpr int kSMs = 148;

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

// ---- FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col)  -> SASS DMMA.8x8x4
BK_DEV void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- cp.async (LDGSTS) with zero-fill: copies src_bytes (0..cp) and zero-fills the rest
BK_DEV void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
BK_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
BK_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
BK_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

BK_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
BK_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// monotone bit pattern for non-negative doubles: lets atomicMax on uint64 act as a max
BK_DEV unsigned long long dbits(double v) { return static_cast<unsigned long long>(__double_as_longlong(v)); }

struct cplx {
  double re, im;
};
BK_DEV cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
BK_DEV cplx cfma(cplx a, cplx b, cplx c) {  // a*b + c
  return {fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}

}  // namespace bk
