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
#include <cstdlib>
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

// WM x WN DMMA tiles of one warp.  FULL: every tile valid -> unpredicated mma.sync (a
// predicated mma.sync costs a WARPSYNC + NOP + fixed-latency wait per instruction).
template <int WM, int WN, bool FULL>
BK_DEV void dmma_block(double (&acc)[WM][WN][2], const double* af, const double* bf, int mtv, int ntv) {
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b)
      if (FULL || (a < mtv && b < ntv)) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
}

BK_DEV double lds64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
  return v;
}

// One k4 step of a WM x WN warp tile with the NEXT step's fragment loads interleaved
// between the DMMAs (one ld.shared after each of the first WM+WN DMMAs).  Both are volatile
// asm, so program order is kept: the loads fill the issue gap a back-to-back DMMA pair
// would otherwise fill with NOPs.  xn/yn: next fragments' addresses (stride 8 / xs, ys
// element strides between tiles); has_next false on the last step.
template <int WM, int WN>
BK_DEV void dmma_step_il(double (&acc)[WM][WN][2], const double* af, const double* bf, double* afn, double* bfn,
                         const double* xn, int xs, const double* yn, int ys, bool has_next) {
#pragma unroll
  for (int a = 0; a < WM; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) {
      dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      const int i = a * WN + b;
      if (has_next) {
        if (i < WM) afn[i] = lds64(xn + i * xs);
        else if (i < WM + WN) bfn[i - WM] = lds64(yn + (i - WM) * ys);
      }
    }
  // thin warp tiles (WM * WN < WM + WN, e.g. 4 x 1): the fragments left over
#pragma unroll
  for (int i = WM * WN; i < WM + WN; ++i)
    if (has_next) {
      if (i < WM) afn[i] = lds64(xn + i * xs);
      else bfn[i - WM] = lds64(yn + (i - WM) * ys);
    }
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

// ---- mbarrier pipeline helpers (producer/consumer rings without CTA-wide barriers)
BK_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
BK_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
BK_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive once all of this thread's prior cp.async copies have landed (count pre-set at init)
BK_DEV void mbar_cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
BK_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "BK_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BK_WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bulk (TMA-unit) copy global -> shared, completion counted in bytes on an mbarrier
BK_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
BK_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
BK_DEV void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}
BK_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

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

namespace bk {
// hint a 128-byte line into L2 (no register result, no ordering)
BK_DEV void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p)); }
}  // namespace bk
