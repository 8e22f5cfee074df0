// FP64 products on the int8 tensor cores (tcgen05.mma kind::i8, TMEM accumulators): the Ozaki
// scheme.  sm_100a has no FP64 tcgen05 kind; its FP64 tensor path (DMMA, mma.sync) peaks at
// 37 TFLOP/s, while the int8 tensor cores run at ~4.5 POPS.  Every FP64 operand element is
// split into S = 8 signed 8-bit digits against a per-row / per-column power-of-two scale:
//
//     x = 2^(E - 6) * sum_{i<S} d_i 2^(-8 i) + O(2^(E - 8S + 2)),   d_i in [-128, 127],
//
// (Z = trunc(x 2^(8S-2-E)), |Z| < 2^(8S-2); the lower digits are the bytes of Z + 0x80..80
// minus 128, the top digit its arithmetic high byte), so a dot product of two such vectors is
// sum_{i,j} 2^(EA+EB-12-8(i+j)) <dA_i, dB_j>, each <dA_i, dB_j> an exact int32 sum
// (|d_i d_j| <= 2^14, at most S pairs per accumulator, chunks of <= 16,320 rows).  The pairs
// with i + j <= S - 1 are kept (36 products); the digit truncation (2^-62 of max|x|) and the
// dropped tail (~2^-59 of max|x| max|y| per term) sit far below fp64 rounding, so the result is
// within DGEMM's error bound class (u |X|^T |Y|) even for rows / columns whose entries span many
// binades.  (7 digits with i + j <= 6, 28 products, measured 2^-52.5 of max|x| max|y| per term --
// above DGEMM's bound for short sums -- tools/ozaki_probe.cu.)
//
// The pairs of one group t = i + j share a scale, so they accumulate in one TMEM block; B's
// digit blocks are consecutive 64-row blocks of shared memory and the groups consecutive
// 64-column blocks of TMEM, so A_i x [B_j0 .. B_j0+3] is ONE tcgen05.mma with N = 256 writing
// groups i+j0 .. i+j0+3 (12 MMAs per 32-deep k step instead of 36: fewer shared-memory re-reads
// of A, the limiter of this kernel -- ncu: tensor-core shared-memory path 80% busy).
//
// Kernels: digit slicing (column-wise with a transpose for Grams, row-wise for the tall GEMM),
// the tcgen05 mainloop (TMA producer warp, single-thread MMA issue, 4 epilogue warps reading
// TMEM), a fixed-order split-K reduction.  Results are deterministic (fixed summation orders).
// Replaces the FP64 products of block_inner (core.py:43-49) and the tall updates
// (ppcg.py:443-445, 630, 758; core.py:99; ppcg.py:574-577).
#include <cuda.h>
#include <cstdio>
#include "common.cuh"

#define BK_HD __host__ __device__ __forceinline__

namespace bk {
namespace oz {

constexpr int S = 8;            // digits per element (and digit groups t = i + j <= S - 1 kept)
constexpr int BM = 128;         // output rows per CTA (TMEM lanes)
constexpr int BN = 64;          // output columns per digit group (TMEM columns per group)
#ifndef OZ_KB
#define OZ_KB 64
#define OZ_STAGES 2
#endif
constexpr int KB = OZ_KB;       // k bytes (= k elements) per pipeline stage (swizzle width)
constexpr int STAGES = OZ_STAGES;
constexpr int A_BYTES = S * BM * KB, B_BYTES = S * BN * KB;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TS_STAGE_OUT = 8 * 32 * 16 * 8;  // tall GEMM: per epilogue warp a 32 x 16 fp64 staging tile
constexpr int TS_SMEM = SMEM + TS_STAGE_OUT;
constexpr int THREADS = 192;    // warp 0 TMA, warp 1 MMA (+TMEM alloc), warps 2-5 epilogue
constexpr int TS_THREADS = 320; // tall GEMM: 8 epilogue warps (lane quadrant x column half)
constexpr int MAX_CHUNK = 16320;  // rows per int32 accumulation: S pairs * 2^14 * 16320 < 2^31
constexpr int KPAD = 64;

BK_DEV void tma3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 64-byte swizzle, SBO = 8 rows x 64 B, LBO = 1 (unused
// for swizzled K-major), version 1 (sm_100)
BK_DEV uint64_t umma_desc(uint32_t saddr) {
  constexpr uint64_t layout = KB == 128 ? 2 : KB == 64 ? 4 : 6;  // SWIZZLE_128B / 64B / 32B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((8 * KB) >> 4) << 32) |
         ((uint64_t)1 << 46) | (layout << 61);
}

// instruction descriptor kind::i8: s32 accumulate, signed A and B, K-major both, N, M = 128
BK_DEV uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

BK_DEV void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

// 16 accumulator columns [cc, cc+16) of this thread's TMEM lane, digit groups combined in fp64
// (smallest group first): sum_t 2^(-12-8t) acc_t
BK_DEV void combine16(uint32_t tmem_lane, int cc, double (&acc)[16]) {
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0;
#pragma unroll
  for (int t = S - 1; t >= 0; --t) {
    uint32_t v[16];
    tmem_ld16(tmem_lane + t * BN + cc, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const double w = ldexp(1.0, -12 - 8 * t);
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = fma((double)(int)v[e], w, acc[e]);
  }
}

// Same as combine16 but exact in integers first: H = sum_{t<4} acc_t 2^(8(3-t)), L likewise for
// t >= 4 (|H|, |L| < 2^56 fit int64), result = 2^-36 (H + 2^-32 L): two int64 -> fp64
// conversions per column instead of eight.  Caller applies the 2^-36 (folded into the exponent).
template <int GS = BN>  // TMEM columns between digit groups
BK_DEV void combine16_i64(uint32_t tmem_lane, int cc, double (&acc)[16]) {
  static_assert(S == 8, "two halves of four digit groups");
  long long h[16];
  {
    uint32_t v[4][16];
#pragma unroll
    for (int t = 0; t < 4; ++t) tmem_ld16(tmem_lane + t * GS + cc, v[t]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      long long x = (long long)(int)v[0][e];
      x = (x << 8) + (long long)(int)v[1][e];
      x = (x << 8) + (long long)(int)v[2][e];
      h[e] = (x << 8) + (long long)(int)v[3][e];
    }
  }
  {
    uint32_t v[4][16];
#pragma unroll
    for (int t = 0; t < 4; ++t) tmem_ld16(tmem_lane + (4 + t) * GS + cc, v[t]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      long long x = (long long)(int)v[0][e];
      x = (x << 8) + (long long)(int)v[1][e];
      x = (x << 8) + (long long)(int)v[2][e];
      x = (x << 8) + (long long)(int)v[3][e];
      acc[e] = fma((double)x, 0x1p-32, (double)h[e]);
    }
  }
}

// int32 -> fp64 exactly without the conversion unit: the double with high word 0x43300000 and
// low word u is 2^52 + u, and v + 2^31 = v ^ 0x80000000 as an unsigned word
BK_DEV double i2d(uint32_t v) {
  return __hiloint2double(0x43300000, (int)(v ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}

// combine16_i64 in fp64 arithmetic, for short sums: with K <= TS_F64_COMBINE_K accumulated rows
// every |acc_t| <= 8 K 2^14, so H and L (Horner in base 256 over four groups) stay below 2^53
// and each fma is exact -- bitwise the int64 result, with half the instructions (one LOP and one
// DADD per conversion, no 64-bit shifts / carries, no I2F.F64.S64).  An experiment
// (PPCG_OZ_F64COMB=1): the FP64 pipe's latency makes it slightly slower than the int64 form.
constexpr int TS_F64_COMBINE_K = 4032;
template <int GS>
BK_DEV void combine16_f64(uint32_t tmem_lane, int cc, double (&acc)[16]) {
  static_assert(S == 8, "two halves of four digit groups");
  double h[16];
  {
    uint32_t v[4][16];
#pragma unroll
    for (int t = 0; t < 4; ++t) tmem_ld16(tmem_lane + t * GS + cc, v[t]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      double x = i2d(v[0][e]);
      x = fma(x, 256.0, i2d(v[1][e]));
      x = fma(x, 256.0, i2d(v[2][e]));
      h[e] = fma(x, 256.0, i2d(v[3][e]));
    }
  }
  {
    uint32_t v[4][16];
#pragma unroll
    for (int t = 0; t < 4; ++t) tmem_ld16(tmem_lane + (4 + t) * GS + cc, v[t]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      double x = i2d(v[0][e]);
      x = fma(x, 256.0, i2d(v[1][e]));
      x = fma(x, 256.0, i2d(v[2][e]));
      x = fma(x, 256.0, i2d(v[3][e]));
      acc[e] = fma(x, 0x1p-32, h[e]);
    }
  }
}

BK_DEV void combine16_i64_rt(uint32_t tmem_lane, int gs, int cc, double (&acc)[16]) {
  long long h[16];
  {
    uint32_t v[4][16];
#pragma unroll
    for (int t = 0; t < 4; ++t) tmem_ld16(tmem_lane + t * gs + cc, v[t]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      long long x = (long long)(int)v[0][e];
      x = (x << 8) + (long long)(int)v[1][e];
      x = (x << 8) + (long long)(int)v[2][e];
      h[e] = (x << 8) + (long long)(int)v[3][e];
    }
  }
  {
    uint32_t v[4][16];
#pragma unroll
    for (int t = 0; t < 4; ++t) tmem_ld16(tmem_lane + (4 + t) * gs + cc, v[t]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      long long x = (long long)(int)v[0][e];
      x = (x << 8) + (long long)(int)v[1][e];
      x = (x << 8) + (long long)(int)v[2][e];
      x = (x << 8) + (long long)(int)v[3][e];
      acc[e] = fma((double)x, 0x1p-32, (double)h[e]);
    }
  }
}

// signed base-256 digits of x 2^sh, sh = 8S-2-E (|x 2^sh| < 2^(8S-2)): packs digit s of 4 consecutive
// elements into w[s] (byte e of the word = element e)
BK_DEV void digits4(const double (&v)[4], int sh, uint32_t (&w)[S]) {
  unsigned long long B = 0;
#pragma unroll
  for (int q = 0; q < S - 1; ++q) B |= 0x80ull << (8 * q);
#pragma unroll
  for (int s = 0; s < S; ++s) w[s] = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const long long U = (long long)ldexp(v[e], sh) + (long long)B;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int d = (s == 0) ? (int)(U >> (8 * (S - 1))) : (int)((U >> (8 * (S - 1 - s))) & 255) - 128;
      w[s] |= ((uint32_t)(d & 255)) << (8 * e);
    }
  }
}

// exponent E with max|x| < 2^E; NON_FINITE marks a column / row holding Inf or NaN: its products
// come out NaN (the breakdown guards of ppcg.py:698-724 then see them, as with DGEMM)
constexpr int NON_FINITE = 0x40000000;
BK_DEV int exp_of(double mx) { return !isfinite(mx) ? NON_FINITE : mx > 0 ? ilogb(mx) + 1 : 0; }
BK_DEV int shift_of(int E) { return E == NON_FINITE ? -2000 : 8 * S - 2 - E; }
BK_DEV double scaled(double acc, int e1, int e2) {
  if (e1 == NON_FINITE || e2 == NON_FINITE) return __longlong_as_double(0x7ff8000000000000ll);
  const int e = e1 + e2;
  // 2^e as a normal double from its bits (one multiply); ldexp only outside the normal range
  if (e >= -1022 && e <= 1023) return acc * __longlong_as_double((long long)(e + 1023) << 52);
  return ldexp(acc, e);
}

// ---------------------------------------------------------------------------------------- slicing
// column maxima (|x| bit patterns, atomicMax; zeroed by the caller) of an n x m row-major block;
// CTA = 64 rows x 256 columns
__global__ void __launch_bounds__(256) k_colmax(int64_t n, int m, const double* __restrict__ X, int64_t ld,
                                                unsigned long long* colmax) {
  const int c = blockIdx.y * 256 + threadIdx.x;
  if (c >= m) return;
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  const int nr = (int)lmin(64, n - r0);
  const double* p = X + r0 * ld + c;
  double mx = 0;
  bool bad = false;
  if (nr == 64) {
#pragma unroll 16
    for (int r = 0; r < 64; ++r) {
      const double v = fabs(__ldg(p + r * ld));
      mx = fmax(mx, v);
      bad |= !(v <= 1.7976931348623157e308);
    }
  } else {
    for (int r = 0; r < nr; ++r) {
      const double v = fabs(__ldg(p + r * ld));
      mx = fmax(mx, v);
      bad |= !(v <= 1.7976931348623157e308);
    }
  }
  // NaN bits order above every finite / infinite magnitude
  atomicMax(colmax + c, bad ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(mx));
}

__global__ void k_exponents(int m, const unsigned long long* colmax, int* E, double* pow2) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < m) {
    const int e = exp_of(__longlong_as_double((long long)colmax[c]));
    E[c] = e;
    if (pow2)
      pow2[c] = e == NON_FINITE ? __longlong_as_double(0x7ff8000000000000ll)
                : (e >= -1000 && e <= 1000) ? __longlong_as_double((long long)(e + 1023) << 52)
                                            : 0.0;
  }
}

// column digits, transposed: out[s][c][k - r_base] for rows k in [r0, r0 + 128) of the n x m block
// (rows >= n -> 0; k offsets >= klim not written).  CTA = 128 rows x 32 columns, 256 threads: thread (column, 16 rows).
__global__ void __launch_bounds__(256) k_slice_cols(int64_t n, int m, const double* __restrict__ X, int64_t ld,
                                                    const int* E, int64_t r_base, int8_t* out, int64_t kld,
                                                    int64_t slice_stride, int64_t klim) {
  __shared__ __align__(16) int8_t t[S][32][128 + 16];
  const int64_t r0 = r_base + (int64_t)blockIdx.x * 128;
  const int c0 = blockIdx.y * 32;
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = c0 + cl;
  const int sh = c < m ? shift_of(E[c]) : 0;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    double v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t r = r0 + g * 16 + h * 4 + e;
      v[e] = (c < m && r < n) ? __ldg(X + r * ld + c) : 0.0;
    }
    uint32_t w[S];
    digits4(v, sh, w);
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(&t[s][cl][g * 16 + h * 4]) = w[s];
  }
  __syncthreads();
  const int64_t kofs = r0 - r_base;
  for (int i = threadIdx.x; i < S * 32 * 8; i += blockDim.x) {
    const int p = i & 7, cc = (i >> 3) & 31, s = i >> 8;
    if (c0 + cc < m && kofs + p * 16 < klim)
      *reinterpret_cast<int4*>(out + s * slice_stride + (int64_t)(c0 + cc) * kld + kofs + p * 16) =
          *reinterpret_cast<const int4*>(&t[s][cc][p * 16]);
  }
}

// row digits (no transpose): out[s][r - r_base][kk] for row r of the n x K block, exponent over
// the row; k layout split at ksplit: columns [0, ksplit) -> [0, ksplit), columns [ksplit, K) ->
// [kp1, kp1 + K - ksplit), zeros elsewhere up to kp.  One warp per row; lane = 4 columns.
__global__ void __launch_bounds__(256) k_slice_rows(int64_t r_base, int64_t nrows, int K, const double* __restrict__ X,
                                                    int64_t ld, int ksplit, int kp1, int kp, int8_t* out,
                                                    int64_t slice_stride, int* E) {
  const int64_t rl = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (rl >= nrows) return;
  const double* x = X + (r_base + rl) * ld;
  double mx = 0;
  bool bad = false;
  for (int c = lane; c < K; c += 32) {
    const double v = fabs(__ldg(x + c));
    mx = fmax(mx, v);
    bad |= !(v <= 1.7976931348623157e308);
  }
  mx = warp_max(mx);
  bad = __any_sync(0xffffffffu, bad);
  const int e = bad ? NON_FINITE : exp_of(mx);
  if (lane == 0) E[r_base + rl] = e;
  const int sh = shift_of(e);
  int8_t* o = out + rl * kp;
  for (int p0 = lane * 4; p0 < kp; p0 += 128) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = p0 + q;
      const int c = p < kp1 ? (p < ksplit ? p : -1) : (p - kp1 + ksplit < K ? p - kp1 + ksplit : -1);
      v[q] = c >= 0 ? __ldg(x + c) : 0.0;
    }
    uint32_t w[S];
    digits4(v, sh, w);
#pragma unroll
    for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(o + s * slice_stride + p0) = w[s];
  }
}

// ---------------------------------------------------------------------------------------- mainloop
// A Gram is cut into up to three segments, all in one launch (one tile list): the main block in
// 128 x 64 tiles without padding, a narrow right strip (tiles of 16 / 32 / 64 columns), and the
// bottom rows computed transposed (C[m1a:, :]^T = Y^T X[:, m1a:], the remainder on the N side
// where the granularity is 16 instead of 128) -- or, for a symmetric Gram, the bottom-right
// corner.  A segment reads A's digits (box 128 rows) and B's (box tbn rows) from its own maps.
struct GramSeg {
  int rowA0, rowB0;   // first operand column of the A / B side
  int ta, tb;         // tile grid (128 A columns x tbn B columns per tile)
  int tbn;            // 16, 32 or 64
  int sym;            // upper tiles only (main block / corner of a symmetric Gram; equal origins)
  int mirror;         // symmetric Gram: write the upper part (B col >= A col) and its mirror
  int trans;          // writes C[B col][A col]
  int limA, limB;     // operand column limits (exclusive)
  int mapA, mapB;     // tensor map index of each side
  int tile0;          // first tile of the segment in the launch's tile list
  const int* EA;      // exponents of the A side's columns (indexed by operand column)
  const int* EB;
  int64_t part_off;   // this segment's partial sums, doubles: [chunk][tile][128][tbn]
};

struct GramEpi {
  GramSeg seg[3];
  int nseg;
  int ntiles;         // tiles of all segments
  int64_t chunk_rows;  // rows per CTA (multiple of KB)
  int64_t nrows;      // rows in this launch
  double* part;
  int dbg;            // experiments (PPCG_OZ_DBG): 1 = no MMAs, 4 = no TMA
};

struct TsEpi {
  int64_t nrows;      // rows in this launch (from row r_base)
  int64_t r_base;
  int N;
  int nk;             // k stages (kp / KB)
  int snap_stage;     // metric snapshot after this stage (-1: none)
  int upper;          // G upper triangular (no metric): skip k stages below the tile
  int kp1, kv1, kv2;  // k layout: [0, kv1) valid, zeros to kp1, [kp1, kp1 + kv2) valid (32-deep steps
                      // wholly in the zero padding are skipped)
  int nsplit;
  int f64comb;        // K short enough for the fp64 digit-group combine (combine16_f64)
  double alpha, beta;
  const int* ER[4];   // row exponents (indexed by global row)
  const int* EG[4];   // G column exponents
  const double* EGf[4];  // 2^EG when |EG| <= 1000, NaN for non-finite columns, else 0 (exact path)
  const double* Z[4];
  double* Y[4];
  int64_t ldz, ldy;
  const double* rowscale;  // indexed by global row
  double* metric_ws;  // per-CTA partial sums of squares (problem 0)
  int dbg;            // experiments (PPCG_OZ_DBG): 1 = no MMAs, 2 = no epilogue stores, 4 = no TMA
};

// upper tiles (b*tbn + tbn - 1 >= a*BM) of a ta x tb grid, enumerated row by row
BK_HD int sym_bmin(int a, int tbn) {
  const int v = a * BM - (tbn - 1);
  return v <= 0 ? 0 : (v + tbn - 1) / tbn;
}
BK_DEV void sym_tile(int idx, int ta, int tb, int tbn, int& a, int& b) {
  for (a = 0; a < ta; ++a) {
    const int cnt = tb - sym_bmin(a, tbn);
    if (cnt > 0 && idx < cnt) {
      b = sym_bmin(a, tbn) + idx;
      return;
    }
    if (cnt > 0) idx -= cnt;
  }
  a = ta - 1;
  b = tb - 1;
}

BK_DEV const GramSeg& seg_of(const GramEpi& P, int tile, int& local) {
  int i = 0;
  while (i + 1 < P.nseg && tile >= P.seg[i + 1].tile0) ++i;
  local = tile - P.seg[i].tile0;
  return P.seg[i];
}

BK_DEV void seg_tile(const GramSeg& g, int local, int& a, int& b) {
  if (g.sym) {
    sym_tile(local, g.ta, g.tb, g.tbn, a, b);
  } else {
    a = local / g.tb;
    b = local % g.tb;
  }
}

// Gram partial of one (tile, row chunk); grid (tiles of all segments, chunks).  The B tile
// width is per segment (16 / 32 / 64): the digit groups sit tbn TMEM columns apart, and one MMA
// covers up to 256 / tbn digit blocks of B.
__global__ void __launch_bounds__(THREADS, 1)
    k_oz_gram(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
              const __grid_constant__ CUtensorMap mapA2, const __grid_constant__ CUtensorMap mapA3,
              const __grid_constant__ CUtensorMap mapB0, const __grid_constant__ CUtensorMap mapB1,
              const __grid_constant__ CUtensorMap mapB2, const __grid_constant__ CUtensorMap mapB3,
              const GramEpi P) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int local;
  const GramSeg& g = seg_of(P, blockIdx.x, local);
  int ta_, tb_;
  seg_tile(g, local, ta_, tb_);
  const int tbn = g.tbn;
  const int rowA = g.rowA0 + ta_ * BM, rowB = g.rowB0 + tb_ * tbn;
  const int kc0 = (int)(blockIdx.y * P.chunk_rows);
  const int64_t k1 = lmin(P.nrows, (int64_t)kc0 + P.chunk_rows);
  const int nk = (int)((k1 - kc0 + KB - 1) / KB);
  const CUtensorMap* mA = g.mapA == 0 ? &mapA0 : g.mapA == 1 ? &mapA1 : g.mapA == 2 ? &mapA2 : &mapA3;
  const CUtensorMap* mB = g.mapB == 0 ? &mapB0 : g.mapB == 1 ? &mapB1 : g.mapB == 2 ? &mapB2 : &mapB3;
  const uint32_t stage_bytes = A_BYTES + S * tbn * KB;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(mA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(mB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int st = kb % STAGES;
        mbar_wait(empty + st, ((kb / STAGES) & 1) ^ 1);
        uint8_t* sa = sm + st * STAGE_BYTES;
        if (P.dbg & 4) {
          mbar_arrive(full + st);
          continue;
        }
        mbar_arrive_expect_tx(full + st, stage_bytes);
        const int kc = kc0 + kb * KB;
        tma3d(sa, mA, kc, rowA, 0, full + st);
        tma3d(sa + A_BYTES, mB, kc, rowB, 0, full + st);
      }
    }
  } else if (warp == 1) {
    const int nj_max = 256 / tbn;
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % STAGES;
      mbar_wait(full + st, (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0 && !(P.dbg & 1)) {
        const uint32_t sa = smem_u32(sm + st * STAGE_BYTES);
        const uint32_t sb = sa + A_BYTES;
#pragma unroll
        for (int ks = 0; ks < KB / 32; ++ks) {
#pragma unroll
          for (int i = 0; i < S; ++i) {
            for (int j0 = 0; j0 < S - i; j0 += nj_max) {
              const int nj = (S - i - j0) < nj_max ? (S - i - j0) : nj_max;
              const uint64_t da = umma_desc(sa + i * BM * KB + ks * 32);
              const uint64_t db = umma_desc(sb + j0 * tbn * KB + ks * 32);
              const uint32_t accf = (kb > 0 || ks > 0 || i > 0) ? 1u : 0u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (i + j0) * tbn),
                  "l"(da), "l"(db), "r"(idesc_i8(nj * tbn)), "r"(accf));
            }
          }
        }
      }
      if (lane == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(empty + st))
                     : "memory");
        if (kb == nk - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(done))
                       : "memory");
      }
      __syncwarp();
    }
  } else {
    // epilogue warps: TMEM lane quadrant = warp % 4 (hardware rule), lane = A column of the tile
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int ga = rowA + r;
    const int ea0 = ga < g.limA ? g.EA[ga] : 0;
    const int ea = ea0 == NON_FINITE ? NON_FINITE : ea0 - 36;  // combine16_i64 leaves 2^-36
    const int seg_tiles = g.ta * g.tb;  // partial slots per chunk (sym: the full grid, sparse)
    double* out = P.part + g.part_off + (((int64_t)blockIdx.y * seg_tiles + ta_ * g.tb + tb_) * BM + r) * tbn;
    for (int cc = 0; cc < tbn; cc += 16) {
      double acc[16];
      combine16_i64_rt(tl, tbn, cc, acc);
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        const int gb = rowB + cc + e;
        const int e0 = gb < g.limB ? g.EB[gb] : 0;
        const int e1 = gb + 1 < g.limB ? g.EB[gb + 1] : 0;
        *reinterpret_cast<double2*>(out + cc + e) = make_double2(scaled(acc[e], ea, e0), scaled(acc[e + 1], ea, e1));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

// Tall GEMM, persistent: one CTA per SM walks the tiles tau = blockIdx.x + i * gridDim.x (column
// tiles fastest, so the column tiles of a row block run side by side and share its X digits in
// L2).  Tiles are 128 rows x TBN columns; with TBN = 32 the 8 digit groups take 256 TMEM columns
// and two accumulators alternate: the MMA warp fills one while the epilogue drains the other.
// The producer runs ahead across tile boundaries; the epilogue drains TMEM into registers
// (digit groups combined exactly in int64, then fp64), releases the accumulator, and only then
// scales, reads Z and writes Y through a swizzled shared staging tile (whole-line traffic).
// Metric tiles (problem 0, columns < nsplit) pause the MMA warp after the snapshot stage until
// the epilogue has read the snapshot.
template <int TBN>
__global__ void __launch_bounds__(TS_THREADS, 1)  // 10 warps: 3 share a sub-partition -> <= 168 registers
    k_oz_ts(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
            const __grid_constant__ CUtensorMap mapA2, const __grid_constant__ CUtensorMap mapA3,
            const __grid_constant__ CUtensorMap mapB0, const __grid_constant__ CUtensorMap mapB1,
            const __grid_constant__ CUtensorMap mapB2, const __grid_constant__ CUtensorMap mapB3, const TsEpi P,
            int ctn, int rtn, int nprob) {
  constexpr int NACC = TBN == 32 ? 2 : 1;               // TMEM accumulators (S * TBN columns each)
  constexpr int B_BYTES_T = S * TBN * KB;
  constexpr int STAGE_T = A_BYTES + B_BYTES_T;
  constexpr int CPW = TBN / 2;                          // columns per epilogue warp (2 column halves)
  constexpr int NJ = 256 / TBN;                          // digit blocks of B per MMA (N <= 256)
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE_T);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;     // [NACC]
  uint64_t* tmem_free = done + 2;      // [NACC]
  uint64_t* snap_full = done + 4;
  uint64_t* snap_free = done + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 6);
  double* stage_out = reinterpret_cast<double*>(sm + STAGES * STAGE_T + 256);
  __shared__ double s_red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = ctn * rtn * nprob;

  struct Tile {
    int prob, rowA, rowB, nk, snap;
  };
  auto tile_of = [&](int tau) {
    Tile t;
    t.prob = tau / (ctn * rtn);
    const int r = tau - t.prob * ctn * rtn;
    t.rowA = (r / ctn) * BM;
    t.rowB = (r % ctn) * TBN;
    t.nk = P.nk;
    if (P.upper) t.nk = min(t.nk, (t.rowB + TBN + KB - 1) / KB);
    t.snap = (t.prob == 0 && P.snap_stage >= 0 && t.rowB < P.nsplit) ? P.snap_stage : -1;
    return t;
  };
  auto mapA = [&](int b) { return b == 0 ? &mapA0 : b == 1 ? &mapA1 : b == 2 ? &mapA2 : &mapA3; };
  auto mapB = [&](int b) { return b == 0 ? &mapB0 : b == 1 ? &mapB1 : b == 2 ? &mapB2 : &mapB3; };

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(done + i, 1);
      mbar_init(tmem_free + i, 256);
    }
    mbar_init(snap_full, 1);
    mbar_init(snap_free, 256);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < nprob; ++b) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(mapA(b)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(mapB(b)) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;  // global stage counter
      for (int tau = blockIdx.x; tau < ntiles; tau += gridDim.x) {
        const Tile t = tile_of(tau);
        const CUtensorMap* mA = mapA(t.prob);
        const CUtensorMap* mB = mapB(t.prob);
        for (int kb = 0; kb < t.nk; ++kb, ++it) {
          const int st = it % STAGES;
          mbar_wait(empty + st, ((it / STAGES) & 1) ^ 1);
          uint8_t* sa = sm + st * STAGE_T;
          if (P.dbg & 4) {
            mbar_arrive(full + st);
            continue;
          }
          mbar_arrive_expect_tx(full + st, STAGE_T);
          tma3d(sa, mA, kb * KB, t.rowA, 0, full + st);
          tma3d(sa + A_BYTES, mB, kb * KB, t.rowB, 0, full + st);
        }
      }
    }
  } else if (warp == 1) {
    int it = 0, ti = 0, si = 0;
    for (int tau = blockIdx.x; tau < ntiles; tau += gridDim.x, ++ti) {
      const Tile t = tile_of(tau);
      const int ab = ti % NACC;                     // accumulator of this tile
      const uint32_t acc_base = tmem + ab * S * TBN;
      mbar_wait(tmem_free + ab, ((ti / NACC) & 1) ^ 1);  // epilogue has drained this accumulator
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kb = 0; kb < t.nk; ++kb, ++it) {
        const int st = it % STAGES;
        mbar_wait(full + st, (it / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t sa = smem_u32(sm + st * STAGE_T);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int ks = 0; ks < KB / 32; ++ks) {
            if (P.dbg & 1) break;
            const int k0 = kb * KB + ks * 32;  // skip 32-deep steps that lie in the zero padding
            if (ks > 0 && ((k0 >= P.kv1 && k0 < P.kp1) || k0 >= P.kp1 + P.kv2)) break;
#pragma unroll
            for (int i = 0; i < S; ++i) {
#pragma unroll
              for (int j0 = 0; j0 < S - i; j0 += NJ) {
                const int nj = (S - i - j0) < NJ ? (S - i - j0) : NJ;
                const uint64_t da = umma_desc(sa + i * BM * KB + ks * 32);
                const uint64_t db = umma_desc(sb + j0 * TBN * KB + ks * 32);
                const uint32_t accf = (kb > 0 || ks > 0 || i > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(acc_base + (i + j0) * TBN),
                    "l"(da), "l"(db), "r"(idesc_i8(nj * TBN)), "r"(accf));
              }
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(empty + st))
                       : "memory");
          if (kb == t.snap)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(snap_full))
                         : "memory");
          if (kb == t.nk - 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(done + ab))
                         : "memory");
        }
        __syncwarp();
        if (kb == t.snap) {
          // epilogue has read the snapshot -- also after a last-stage snapshot: with two
          // accumulators the next tile's snapshot commit must not run a second phase ahead
          mbar_wait(snap_free, si & 1);
          ++si;
        }
      }
    }
  } else {
    // 8 epilogue warps: TMEM lane quadrant q = warp % 4 (hardware rule), column half h
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int c0 = h * CPW;
    double ss = 0;  // metric partial (problem 0 tiles with columns < nsplit)
    int ti = 0, si = 0;
    for (int tau = blockIdx.x; tau < ntiles; tau += gridDim.x, ++ti) {
      const Tile t = tile_of(tau);
      const int ab = ti % NACC;
      const uint32_t tl = tmem + ab * S * TBN + ((uint32_t)(q * 32) << 16);
      const int64_t lrow = t.rowA + r;
      const bool live = lrow < P.nrows;
      const int64_t grow = P.r_base + lrow;
      const int er0 = live ? P.ER[t.prob][grow] : 0;
      const int er = er0 == NON_FINITE ? NON_FINITE : er0 - 36;  // combine leaves 2^-36
      const int* EG = P.EG[t.prob];
      const double* Z = P.Z[t.prob];
      double* Y = P.Y[t.prob];
      const int ncol = min(CPW, P.N - (t.rowB + c0));  // valid columns of this warp (may be <= 0)
      if (live && ncol > 0 && Z != nullptr && P.beta != 0.0) {
        // this row's Z segment into L2 while the tile's MMAs run (metric and stores)
        const double* zr = Z + grow * P.ldz + t.rowB + c0;
#pragma unroll
        for (int c = 0; c < CPW; c += 16) prefetch_l2(zr + c);
      }
      if (t.snap >= 0) {
        mbar_wait(snap_full, si & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int cc = 0; cc < CPW; cc += 16) {
          if (t.rowB + c0 + cc < P.nsplit && cc < ncol) {
            double acc[16];
            if (P.f64comb)
              combine16_f64<TBN>(tl, c0 + cc, acc);
            else
              combine16_i64<TBN>(tl, c0 + cc, acc);
            double z[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int gc = t.rowB + c0 + cc + e;
              z[e] = (live && P.beta != 0.0 && e + cc < ncol) ? Z[grow * P.ldz + gc] : 0.0;
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int gc = t.rowB + c0 + cc + e;
              if (live && gc < P.nsplit && e + cc < ncol) {
                const double v = fma(P.beta, z[e], P.alpha * scaled(acc[e], er, EG[gc]));
                ss = fma(v, v, ss);
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(snap_free);
        ++si;
      }
      mbar_wait(done + ab, (ti / NACC) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      double acc[CPW];
#pragma unroll
      for (int cc = 0; cc < CPW; cc += 16) {
        if (cc < ncol) {
          double a16[16];
          if (P.f64comb)
            combine16_f64<TBN>(tl, c0 + cc, a16);
          else
            combine16_i64<TBN>(tl, c0 + cc, a16);
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[cc + e] = a16[e];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tmem_free + ab);
      if (Y == nullptr || ncol <= 0 || (P.dbg & 2)) continue;
      const bool vec = ncol == CPW && !(P.ldy & 1) && (P.beta == 0.0 || !(P.ldz & 1)) &&
                       ((reinterpret_cast<uintptr_t>(Y + t.rowB + c0) & 15) == 0) &&
                       (P.beta == 0.0 || (reinterpret_cast<uintptr_t>(Z + t.rowB + c0) & 15) == 0);
      if (vec) {
        // rows -> shared (16-byte pairs, XOR-swizzled by row), then 8 lanes per 128-byte row
        // segment: Z loads and Y stores move whole lines
        double* wb = stage_out + (warp - 2) * 512;
        // row factor 2^er (exact power of two when er is in the normal range; otherwise, and for
        // NaN markers, the exact per-element path)
        const bool rfast = live && er >= -1000 && er <= 1000;
        const double fr = rfast ? P.alpha * __longlong_as_double((long long)(er + 1023) << 52) : 0.0;
        const double* EGf = P.EGf[t.prob];
#pragma unroll
        for (int cc = 0; cc < CPW; cc += 16) {
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const int gc = t.rowB + c0 + cc + 2 * p;
            const double2 fc = *reinterpret_cast<const double2*>(EGf + gc);
            double u0, u1;
            if (rfast && fc.x != 0.0 && fc.y != 0.0) {
              u0 = acc[cc + 2 * p] * fc.x * fr;
              u1 = acc[cc + 2 * p + 1] * fc.y * fr;
            } else {
              u0 = live ? P.alpha * scaled(acc[cc + 2 * p], er, EG[gc]) : 0.0;
              u1 = live ? P.alpha * scaled(acc[cc + 2 * p + 1], er, EG[gc + 1]) : 0.0;
            }
            *reinterpret_cast<double2*>(wb + lane * 16 + ((p ^ (lane & 7)) * 2)) = make_double2(u0, u1);
          }
          __syncwarp();
          // all eight Z pairs (and row scales) first: Y may alias Z, so the compiler would keep
          // each load behind the previous store; every lane reads and writes only its own
          // elements, so hoisting is safe and the load latencies overlap
          const int p = lane & 7;
          const int gc = t.rowB + c0 + cc + 2 * p;
          double2 z[8];
          double srr[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + (lane >> 3);
            const int64_t lr = t.rowA + q * 32 + rr;
            const int64_t gr = P.r_base + (lr < P.nrows ? lr : 0);
            z[i] = P.beta != 0.0 ? __ldcg(reinterpret_cast<const double2*>(Z + gr * P.ldz + gc)) : make_double2(0.0, 0.0);
            srr[i] = P.rowscale ? __ldg(P.rowscale + gr) : 1.0;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + (lane >> 3);
            const int64_t lr = t.rowA + q * 32 + rr;
            if (lr < P.nrows) {
              const int64_t gr = P.r_base + lr;
              const double2 u = *reinterpret_cast<const double2*>(wb + rr * 16 + ((p ^ (rr & 7)) * 2));
              const double v0 = fma(P.beta, z[i].x, u.x), v1 = fma(P.beta, z[i].y, u.y);
              *reinterpret_cast<double2*>(Y + gr * P.ldy + gc) = make_double2(srr[i] * v0, srr[i] * v1);
            }
          }
          __syncwarp();
        }
      } else if (live) {
        const double sr = P.rowscale ? P.rowscale[grow] : 1.0;
        const int64_t zo = grow * P.ldz + t.rowB + c0, yo = grow * P.ldy + t.rowB + c0;
#pragma unroll
        for (int e = 0; e < CPW; ++e) {
          if (e < ncol) {
            const int gc = t.rowB + c0 + e;
            double v = P.alpha * scaled(acc[e], er, EG[gc]);
            if (P.beta != 0.0) v = fma(P.beta, Z[zo + e], v);
            Y[yo + e] = sr * v;
          }
        }
      }
    }
    if (P.snap_stage >= 0) {
      ss = warp_sum(ss);
      if (lane == 0) s_red[warp - 2] = ss;
      named_bar_sync(1, 256);
      if (threadIdx.x == 64) {
        double tsum = 0;
        for (int w = 0; w < 8; ++w) tsum += s_red[w];
        P.metric_ws[blockIdx.x] = tsum;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

// 32-column tall-GEMM tiles with two TMEM accumulators (epilogue overlapped with the MMAs);
// 64-column tiles (PPCG_OZ_TBN=64) read the X digits half as often but drain TMEM between tiles
static int ts_tbn() {
  static const int tbn = [] {
    const char* e = getenv("PPCG_OZ_TBN");
    return (e && atoi(e) == 64) ? 64 : 32;
  }();
  return tbn;
}

template <int TBN>
constexpr int ts_smem() {
  return STAGES * (A_BYTES + S * TBN * KB) + 1024 + 256 + TS_STAGE_OUT;
}

// C (+)= sum over chunks of the partials, fixed chunk order, compensated; symmetric segments
// write their upper part and its mirror, transposed segments C[B col][A col].
// grid (tiles of all segments, 16): 8 A columns x tbn B columns per CTA
__global__ void k_gram_reduce(GramEpi P, int nch, double* C, int64_t ldc, int accumulate) {
  int local;
  const GramSeg& g = seg_of(P, blockIdx.x, local);
  int a, b;
  seg_tile(g, local, a, b);
  const int r = blockIdx.y * 8 + (threadIdx.x >> 6), c = threadIdx.x & 63;
  if (c >= g.tbn) return;
  const int gA = g.rowA0 + a * BM + r, gB = g.rowB0 + b * g.tbn + c;
  if (gA >= g.limA || gB >= g.limB) return;
  if (g.mirror && gB < gA) return;
  double* dst = g.trans ? C + (int64_t)gB * ldc + gA : C + (int64_t)gA * ldc + gB;
  // compensated (Neumaier) sum: the chunk partials are each rounded once, so the total error stays
  // ~u sum_chunks |partial| <= u |X|^T |Y| whatever the chunk count
  double s = accumulate ? *dst : 0.0, comp = 0.0;
  const int64_t per_chunk = (int64_t)g.ta * g.tb * BM * g.tbn;
  const double* src = P.part + g.part_off + ((int64_t)(a * g.tb + b) * BM + r) * g.tbn + c;
  for (int ch = 0; ch < nch; ++ch) {
    const double v = __ldcg(src + ch * per_chunk);
    const double t = s + v;
    comp += fabs(s) >= fabs(v) ? (s - t) + v : (v - t) + s;
    s = t;
  }
  s += comp;
  *dst = s;
  if (g.mirror && gB > gA) C[(int64_t)gB * ldc + gA] = s;
}

// metric: fixed-order sum of the per-CTA partials (one thread block)
__global__ void k_metric_sum(const double* ws, int64_t cnt, double* out, int accumulate) {
  __shared__ double red[32];
  double s = 0;
  for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) s += ws[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = accumulate ? *out + t : t;
  }
}

// ---------------------------------------------------------------------------------------- host
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// digit array [S][rows][kld] (int8, K contiguous): box 64 k x box_rows rows x S digits, 64-byte
// swizzle; rows >= `rows` and k >= kdim arrive zero-filled
static bool encode_digits(CUtensorMap* map, const int8_t* base, int64_t kld, int64_t kdim, int64_t rows,
                          int box_rows, int64_t slice_stride) {
  static EncodeFn enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeFn) nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)kdim, (cuuint64_t)rows, (cuuint64_t)S};
  const cuuint64_t strides[2] = {(cuuint64_t)kld, (cuuint64_t)slice_stride};
  const cuuint32_t box[3] = {(cuuint32_t)KB, (cuuint32_t)box_rows, (cuuint32_t)S};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             KB == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
             : KB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                        : CU_TENSOR_MAP_SWIZZLE_32B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int g_emu_mode = -1;  // -1: from PPCG_FP64_EMU (default on), 0 off, 1 on

// optional CUDA-event timing of the GEMM-core launches (k_oz_gram / k_oz_ts) on their stream,
// for bench.py's roofline (the kernel's own duration, digit slicing excluded)
struct OzTimer {
  int on = 0;
  int n = 0;
  cudaEvent_t ev[16][2];
  bool made = false;
  void begin(cudaStream_t st) {
    if (!on) return;
    if (!made) {
      for (auto& e : ev) {
        cudaEventCreate(&e[0]);
        cudaEventCreate(&e[1]);
      }
      made = true;
    }
    if (n < 16) cudaEventRecord(ev[n][0], st);
  }
  void end(cudaStream_t st) {
    if (!on) return;
    if (n < 16) cudaEventRecord(ev[n][1], st);
    ++n;
  }
};
static OzTimer g_timer;

static int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// rows per chunk: <= MAX_CHUNK, a multiple of KB, chosen for whole waves of 148 CTAs
static int64_t gram_chunk_rows(int64_t n, int ntiles) {
  const int64_t cmin = (n + MAX_CHUNK - 1) / MAX_CHUNK;
  int64_t best = cmin;
  double best_eff = -1;
  for (int64_t c = cmin; c <= cmin * 8 + 8; ++c) {
    const int64_t rows = align_up((n + c - 1) / c, KB);
    const int64_t nch = (n + rows - 1) / rows;
    const int64_t ctas = nch * ntiles;
    const int64_t waves = (ctas + kSMs - 1) / kSMs;
    const double eff = (double)ctas / (double)(waves * kSMs) - 0.004 * (double)nch / (double)cmin;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = c;
    }
  }
  return align_up((n + best - 1) / best, KB);
}

static int narrow_tbn(int w) { return w <= 16 ? 16 : w <= 32 ? 32 : 64; }

static int sym_count(int ta, int tb, int tbn) {
  int cnt = 0;
  for (int a = 0; a < ta; ++a) cnt += tb - sym_bmin(a, tbn) > 0 ? tb - sym_bmin(a, tbn) : 0;
  return cnt;
}

// segments of C = X^T Y (operand 0 = X, 1 = Y), see GramSeg
struct GramPlan {
  GramSeg seg[3];
  int opA[3], opB[3];
  int nseg, ntiles;
  int64_t part_per_chunk;  // doubles
};

static GramPlan gram_plan(int m1, int m2, int sym) {
  GramPlan G{};
  auto add = [&](int opA, int rowA0, int limA, int opB, int rowB0, int limB, int tbn, int symf, int mirror,
                 int trans) {
    if (limA <= rowA0 || limB <= rowB0) return;
    GramSeg& g = G.seg[G.nseg];
    g = GramSeg{};
    g.rowA0 = rowA0;
    g.limA = limA;
    g.rowB0 = rowB0;
    g.limB = limB;
    g.tbn = tbn;
    g.ta = (limA - rowA0 + BM - 1) / BM;
    g.tb = (limB - rowB0 + tbn - 1) / tbn;
    g.sym = symf;
    g.mirror = mirror;
    g.trans = trans;
    g.tile0 = G.ntiles;
    g.part_off = G.part_per_chunk;  // scaled by the chunk count when the launch is set up
    G.ntiles += symf ? sym_count(g.ta, g.tb, tbn) : g.ta * g.tb;
    G.part_per_chunk += (int64_t)g.ta * g.tb * BM * tbn;
    G.opA[G.nseg] = opA;
    G.opB[G.nseg] = opB;
    ++G.nseg;
  };
  const int m1a = m1 / BM * BM, m2a = m2 / BN * BN;
  if (sym) {  // X^T X: upper main tiles, the right strip (all above the diagonal), the corner
    add(0, 0, m1a, 0, 0, m2a, BN, 1, 1, 0);
    add(0, 0, m1a, 0, m2a, m2, narrow_tbn(m2 - m2a), 0, 1, 0);
    add(0, m1a, m1, 0, m1a, m2, narrow_tbn(m2 - m1a), 1, 1, 0);
  } else {
    add(0, 0, m1a, 1, 0, m2a, BN, 0, 0, 0);
    add(0, 0, m1a, 1, m2a, m2, narrow_tbn(m2 - m2a), 0, 0, 0);
    add(1, 0, m2, 0, m1a, m1, narrow_tbn(m1 - m1a), 0, 0, 1);  // bottom rows, transposed
  }
  return G;
}

struct GramLayout {
  int nq;                      // B operands sharing the A digits (1 or 2)
  GramPlan plan[2];
  int64_t chunk_rows, sc_rows;  // rows per chunk, rows per super-chunk (digits held at once)
  int64_t off_cmA, off_EA, off_sA, off_cmB[2], off_EB[2], off_part[2], off_sB[2], total;
};

// same: B operand q is X itself (one set of digits); sym (requires same): symmetric segments
// preA: X's digits come pre-sliced from the caller (all rows: one super-chunk, no cap)
static GramLayout gram_layout(int64_t n, int m1, int nq, const int* m2, const int* same, int sym, int64_t ws_cap,
                              int preA = 0) {
  GramLayout L{};
  L.nq = nq;
  int tt = 0;
  for (int q = 0; q < nq; ++q) {
    L.plan[q] = gram_plan(m1, m2[q], sym);
    tt = tt > L.plan[q].ntiles ? tt : L.plan[q].ntiles;
  }
  L.chunk_rows = gram_chunk_rows(n, tt);
  // digits of at most ~1.5 GB at once (or what the caller's workspace holds)
  int64_t sc_chunks = (n + L.chunk_rows - 1) / L.chunk_rows;
  const int64_t cap = preA ? ((int64_t)1 << 62) : ws_cap > 0 ? ws_cap : ((int64_t)3 << 29);
  auto layout = [&](int64_t chunks) {
    const int64_t rows = chunks * L.chunk_rows;
    int64_t o = 0;
    L.off_cmA = o; o += align_up(8 * (int64_t)m1, 256);
    L.off_EA = o;  o += align_up(4 * (int64_t)m1, 256);
    for (int q = 0; q < nq; ++q) {
      L.off_cmB[q] = o; o += align_up(8 * (int64_t)m2[q], 256);
      L.off_EB[q] = o;  o += align_up(4 * (int64_t)m2[q], 256);
      L.off_part[q] = o; o += align_up(chunks * L.plan[q].part_per_chunk * 8, 1024);
    }
    L.off_sA = o; o += preA ? 0 : align_up((int64_t)S * m1 * rows, 1024);
    for (int q = 0; q < nq; ++q) {
      L.off_sB[q] = o;
      o += same[q] ? 0 : align_up((int64_t)S * m2[q] * rows, 1024);
    }
    return o;
  };
  while (sc_chunks > 1 && layout(sc_chunks) > cap) sc_chunks = (sc_chunks + 1) / 2;
  L.sc_rows = sc_chunks * L.chunk_rows;
  L.total = layout(sc_chunks);
  return L;
}

// Column digits kept by the caller between products (bk_ozaki_coldigits_d): exponents E[m],
// digits [S][m][kld] of all n rows, kld = align_up(n, KPAD)
struct ColDigits {
  const int* E;
  const int8_t* dig;
  int64_t kld;
  int m;
};
static int64_t coldigits_hdr(int m) { return align_up(8 * (int64_t)m, 256) + align_up(4 * (int64_t)m, 256); }
static ColDigits coldigits_view(void* buf, int64_t n, int m) {
  char* w = static_cast<char*>(buf);
  ColDigits d;
  d.E = reinterpret_cast<const int*>(w + align_up(8 * (int64_t)m, 256));
  d.dig = reinterpret_cast<const int8_t*>(w + coldigits_hdr(m));
  d.kld = align_up(n, KPAD);
  d.m = m;
  return d;
}

// C_q = X^T Y_q for nq <= 2 operands Y_q that share X's digits; pre (optional): the digits of
// the block whose columns [pre_c0, pre_c0 + m1) are X
static int ozaki_gram_multi(int64_t n, int m1, const double* X, int64_t ldx, int nq, const int* m2,
                            const double* const* Y, const int64_t* ldy, double* const* C, const int64_t* ldc,
                            int symmetric, void* ws, int64_t ws_bytes, cudaStream_t st,
                            const ColDigits* pre = nullptr, int pre_c0 = 0) {
  if (n <= 0 || m1 <= 0 || !X) return BK_ERR_ARG;
  if (pre && (pre_c0 < 0 || pre_c0 + m1 > pre->m)) return BK_ERR_ARG;
  int same[2] = {0, 0};
  for (int q = 0; q < nq; ++q) {
    if (m2[q] <= 0 || !Y[q] || !C[q]) return BK_ERR_ARG;
    same[q] = (X == Y[q] && ldx == ldy[q] && m1 == m2[q]) ? 1 : 0;
    if (symmetric && !same[q]) return BK_ERR_ARG;
  }
  const GramLayout L = gram_layout(n, m1, nq, m2, same, symmetric, ws_bytes, pre ? 1 : 0);
  if (!ws || ws_bytes < L.total) return BK_ERR_ARG;
  char* w = static_cast<char*>(ws);
  auto* cmA = reinterpret_cast<unsigned long long*>(w + L.off_cmA);
  int* EA = reinterpret_cast<int*>(w + L.off_EA);
  int8_t* sA = reinterpret_cast<int8_t*>(w + L.off_sA);
  int* EB[2];
  int8_t* sB[2];
  if (pre) {
    EA = const_cast<int*>(pre->E) + pre_c0;
    sA = const_cast<int8_t*>(pre->dig) + (int64_t)pre_c0 * pre->kld;
  } else {
    // exponents over all rows
    cudaMemsetAsync(cmA, 0, 8 * (size_t)m1, st);
    BK_COUNT();
    k_colmax<<<dim3((unsigned)((n + 63) / 64), (m1 + 255) / 256), 256, 0, st>>>(n, m1, X, ldx, cmA);
    BK_COUNT();
    k_exponents<<<(m1 + 255) / 256, 256, 0, st>>>(m1, cmA, EA, nullptr);
  }
  for (int q = 0; q < nq; ++q) {
    EB[q] = same[q] ? EA : reinterpret_cast<int*>(w + L.off_EB[q]);
    sB[q] = same[q] ? sA : reinterpret_cast<int8_t*>(w + L.off_sB[q]);
    if (same[q]) continue;
    auto* cmB = reinterpret_cast<unsigned long long*>(w + L.off_cmB[q]);
    cudaMemsetAsync(cmB, 0, 8 * (size_t)m2[q], st);
    BK_COUNT();
    k_colmax<<<dim3((unsigned)((n + 63) / 64), (m2[q] + 255) / 256), 256, 0, st>>>(n, m2[q], Y[q], ldy[q], cmB);
    BK_COUNT();
    k_exponents<<<(m2[q] + 255) / 256, 256, 0, st>>>(m2[q], cmB, EB[q], nullptr);
  }
  cudaFuncSetAttribute(k_oz_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  static const int dbg = [] {
    const char* e = getenv("PPCG_OZ_DBG");
    return e ? atoi(e) : 0;
  }();
  for (int64_t r0 = 0; r0 < n; r0 += L.sc_rows) {
    const int64_t rows = lmin(L.sc_rows, n - r0);
    const int64_t kld = align_up(rows, KPAD);
    const unsigned gx = (unsigned)((rows + 127) / 128);
    if (!pre) {
      BK_COUNT();
      k_slice_cols<<<dim3(gx, (m1 + 31) / 32), 256, 0, st>>>(r0 + rows, m1, X, ldx, EA, r0, sA, kld,
                                                             kld * (int64_t)m1, kld);
    }
    const int64_t strideA = pre ? kld * (int64_t)pre->m : kld * (int64_t)m1;  // between digit planes
    const int nch = (int)((rows + L.chunk_rows - 1) / L.chunk_rows);
    for (int q = 0; q < nq; ++q) {
      if (!same[q]) {
        BK_COUNT();
        k_slice_cols<<<dim3(gx, (m2[q] + 31) / 32), 256, 0, st>>>(r0 + rows, m2[q], Y[q], ldy[q], EB[q], r0, sB[q],
                                                                 kld, kld * (int64_t)m2[q], kld);
      }
      // tensor maps: one per (operand, box rows) pair the segments use
      const GramPlan& G = L.plan[q];
      const int8_t* dig[2] = {sA, sB[q]};
      const int mcols[2] = {m1, m2[q]};
      const int64_t dstride[2] = {strideA, same[q] ? strideA : kld * (int64_t)m2[q]};
      const int* ex[2] = {EA, EB[q]};
      CUtensorMap mapsA[4], mapsB[4];
      int keyA[4], keyB[4], na = 0, nb = 0;
      GramEpi P{};
      P.nseg = G.nseg;
      P.ntiles = G.ntiles;
      P.chunk_rows = L.chunk_rows;
      P.nrows = rows;
      P.part = reinterpret_cast<double*>(w + L.off_part[q]);
      P.dbg = dbg;
      for (int i = 0; i < G.nseg; ++i) {
        P.seg[i] = G.seg[i];
        P.seg[i].part_off = G.seg[i].part_off * nch;
        P.seg[i].EA = ex[G.opA[i]];
        P.seg[i].EB = ex[G.opB[i]];
        const int ka = G.opA[i], kbk = G.opB[i] * 1000 + G.seg[i].tbn;
        int ia = -1, ib = -1;
        for (int j = 0; j < na; ++j)
          if (keyA[j] == ka) ia = j;
        for (int j = 0; j < nb; ++j)
          if (keyB[j] == kbk) ib = j;
        if (ia < 0) {
          ia = na++;
          keyA[ia] = ka;
          if (!encode_digits(&mapsA[ia], dig[ka], kld, rows, mcols[ka], BM, dstride[ka]))
            return BK_ERR_UNSUPPORTED;
        }
        if (ib < 0) {
          ib = nb++;
          keyB[ib] = kbk;
          const int ob = G.opB[i];
          if (!encode_digits(&mapsB[ib], dig[ob], kld, rows, mcols[ob], G.seg[i].tbn, dstride[ob]))
            return BK_ERR_UNSUPPORTED;
        }
        P.seg[i].mapA = ia;
        P.seg[i].mapB = ib;
      }
      for (int j = na; j < 4; ++j) mapsA[j] = mapsA[0];
      for (int j = nb; j < 4; ++j) mapsB[j] = mapsB[0];
      BK_COUNT();
      g_timer.begin(st);
      k_oz_gram<<<dim3(G.ntiles, nch), THREADS, SMEM, st>>>(mapsA[0], mapsA[1], mapsA[2], mapsA[3], mapsB[0],
                                                            mapsB[1], mapsB[2], mapsB[3], P);
      g_timer.end(st);
      BK_CHECK_LAUNCH();
      BK_COUNT();
      k_gram_reduce<<<dim3(G.ntiles, 16), 512, 0, st>>>(P, nch, C[q], ldc[q], r0 > 0 ? 1 : 0);
    }
  }
  BK_CHECK_LAUNCH();
  return BK_OK;
}

}  // namespace oz
}  // namespace bk

using namespace bk;
using namespace bk::oz;

extern "C" int bk_fp64_emu_set(int mode) {
  g_emu_mode = mode;
  return BK_OK;
}

// Kernel timing: bk_ozaki_timing(1) clears and arms the CUDA-event pairs recorded around each
// GEMM-core launch; bk_ozaki_kernel_ms() waits for them and returns the summed milliseconds of
// the launches since (up to 16); bk_ozaki_timing(0) disarms.
extern "C" int bk_ozaki_timing(int on) {
  g_timer.on = on;
  g_timer.n = 0;
  return BK_OK;
}

extern "C" double bk_ozaki_kernel_ms(void) {
  double t = 0.0;
  const int n = g_timer.n < 16 ? g_timer.n : 16;
  for (int i = 0; i < n; ++i) {
    float ms = 0.f;
    cudaEventSynchronize(g_timer.ev[i][1]);
    if (cudaEventElapsedTime(&ms, g_timer.ev[i][0], g_timer.ev[i][1]) == cudaSuccess) t += ms;
  }
  return t;
}

extern "C" int bk_fp64_emu_enabled(void) {
  if (g_emu_mode < 0) {
    const char* e = getenv("PPCG_FP64_EMU");
    g_emu_mode = e ? atoi(e) : 1;
  }
  return g_emu_mode;
}

extern "C" int64_t bk_ozaki_gram_ws_bytes(int64_t n, int m1, int m2, int same, int symmetric) {
  if (n <= 0 || m1 <= 0 || m2 <= 0) return 0;
  const int m2s[1] = {m2}, sm[1] = {same};
  return gram_layout(n, m1, 1, m2s, sm, symmetric, 0).total;
}

// C = X^T Y (m1 x m2) with the Ozaki scheme; X and Y the same block -> one set of digits;
// symmetric (requires that): upper tiles computed, mirrored.
extern "C" int bk_ozaki_gram_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                               double* C, int64_t ldc, int symmetric, void* ws, int64_t ws_bytes, void* stream) {
  const int m2s[1] = {m2};
  const double* Ys[1] = {Y};
  const int64_t lds[1] = {ldy}, ldcs[1] = {ldc};
  double* Cs[1] = {C};
  return ozaki_gram_multi(n, m1, X, ldx, 1, m2s, Ys, lds, Cs, ldcs, symmetric, ws, ws_bytes, (cudaStream_t)stream);
}

// C1 = X^T Y1, C2 = X^T Y2 (the projections of W and P against one basis, ppcg.py:680-687):
// X is sliced once
extern "C" int64_t bk_ozaki_gram2_ws_bytes(int64_t n, int m1, int m2a, int m2b) {
  if (n <= 0 || m1 <= 0 || m2a <= 0 || m2b <= 0) return 0;
  const int m2s[2] = {m2a, m2b}, sm[2] = {0, 0};
  return gram_layout(n, m1, 2, m2s, sm, 0, 0).total;
}

extern "C" int bk_ozaki_gram2_d(int64_t n, int m1, const double* X, int64_t ldx, int m2a, const double* Ya,
                                int64_t ldya, double* Ca, int64_t ldca, int m2b, const double* Yb, int64_t ldyb,
                                double* Cb, int64_t ldcb, void* ws, int64_t ws_bytes, void* stream) {
  const int m2s[2] = {m2a, m2b};
  const double* Ys[2] = {Ya, Yb};
  const int64_t lds[2] = {ldya, ldyb}, ldcs[2] = {ldca, ldcb};
  double* Cs[2] = {Ca, Cb};
  return ozaki_gram_multi(n, m1, X, ldx, 2, m2s, Ys, lds, Cs, ldcs, 0, ws, ws_bytes, (cudaStream_t)stream);
}

// ---- column digits kept between products: the same block is the left operand of several Grams
// of an iteration (X^H AX, the projections X^H W / X^H P, proj_defect), so its exponents and
// digits are computed once (bk_ozaki_coldigits_d) and handed to the *_pre_d Grams together with
// the column offset of the operand inside the sliced block.
extern "C" int64_t bk_ozaki_coldigits_bytes(int64_t n, int m) {
  if (n <= 0 || m <= 0) return 0;
  return coldigits_hdr(m) + align_up((int64_t)S * m * align_up(n, KPAD), 1024);
}

extern "C" int bk_ozaki_coldigits_d(int64_t n, int m, const double* X, int64_t ldx, void* dig, int64_t dig_bytes,
                                    void* stream) {
  if (n <= 0 || m <= 0 || !X || !dig || dig_bytes < bk_ozaki_coldigits_bytes(n, m)) return BK_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const ColDigits d = coldigits_view(dig, n, m);
  auto* cm = reinterpret_cast<unsigned long long*>(dig);
  cudaMemsetAsync(cm, 0, 8 * (size_t)m, st);
  BK_COUNT();
  k_colmax<<<dim3((unsigned)((n + 63) / 64), (m + 255) / 256), 256, 0, st>>>(n, m, X, ldx, cm);
  BK_COUNT();
  k_exponents<<<(m + 255) / 256, 256, 0, st>>>(m, cm, const_cast<int*>(d.E), nullptr);
  BK_COUNT();
  k_slice_cols<<<dim3((unsigned)((n + 127) / 128), (m + 31) / 32), 256, 0, st>>>(
      n, m, X, ldx, d.E, 0, const_cast<int8_t*>(d.dig), d.kld, d.kld * (int64_t)m, d.kld);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int64_t bk_ozaki_gram_pre_ws_bytes(int64_t n, int m1, int m2, int same, int symmetric) {
  if (n <= 0 || m1 <= 0 || m2 <= 0) return 0;
  const int m2s[1] = {m2}, sm[1] = {same};
  return gram_layout(n, m1, 1, m2s, sm, symmetric, 0, 1).total;
}

// bk_ozaki_gram_d with X = columns [c0, c0 + m1) of the block (n x mdig) whose digits are `dig`
extern "C" int bk_ozaki_gram_pre_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const void* dig, int mdig,
                                   int c0, const double* Y, int64_t ldy, double* C, int64_t ldc, int symmetric,
                                   void* ws, int64_t ws_bytes, void* stream) {
  if (!dig || mdig <= 0) return BK_ERR_ARG;
  const ColDigits d = coldigits_view(const_cast<void*>(dig), n, mdig);
  const int m2s[1] = {m2};
  const double* Ys[1] = {Y};
  const int64_t lds[1] = {ldy}, ldcs[1] = {ldc};
  double* Cs[1] = {C};
  return ozaki_gram_multi(n, m1, X, ldx, 1, m2s, Ys, lds, Cs, ldcs, symmetric, ws, ws_bytes, (cudaStream_t)stream, &d,
                          c0);
}

extern "C" int64_t bk_ozaki_gram2_pre_ws_bytes(int64_t n, int m1, int m2a, int m2b) {
  if (n <= 0 || m1 <= 0 || m2a <= 0 || m2b <= 0) return 0;
  const int m2s[2] = {m2a, m2b}, sm[2] = {0, 0};
  return gram_layout(n, m1, 2, m2s, sm, 0, 0, 1).total;
}

extern "C" int bk_ozaki_gram2_pre_d(int64_t n, int m1, const double* X, int64_t ldx, const void* dig, int mdig, int c0,
                                    int m2a, const double* Ya, int64_t ldya, double* Ca, int64_t ldca, int m2b,
                                    const double* Yb, int64_t ldyb, double* Cb, int64_t ldcb, void* ws,
                                    int64_t ws_bytes, void* stream) {
  if (!dig || mdig <= 0) return BK_ERR_ARG;
  const ColDigits d = coldigits_view(const_cast<void*>(dig), n, mdig);
  const int m2s[2] = {m2a, m2b};
  const double* Ys[2] = {Ya, Yb};
  const int64_t lds[2] = {ldya, ldyb}, ldcs[2] = {ldca, ldcb};
  double* Cs[2] = {Ca, Cb};
  return ozaki_gram_multi(n, m1, X, ldx, 2, m2s, Ys, lds, Cs, ldcs, 0, ws, ws_bytes, (cudaStream_t)stream, &d, c0);
}

// ---- tall GEMM: Y_b = s (.) (alpha X_b G_b + beta Z_b), b < nprob <= 4 (semantics of
// bk_tsgemm_batched_d; flags bit0 = G upper triangular: k stages below a tile are skipped)
namespace bk {
namespace oz {
struct TsLayout {
  int kp1, kp;
  int64_t sc_rows;
  int64_t off_ER, off_EG, off_EGf, off_cmG, off_sG, off_mws, off_sX, total;
};
static TsLayout ts_layout(int nprob, int64_t n, int K, int N, int ksplit, int64_t ws_cap) {
  TsLayout L{};
  const bool split = ksplit > 0 && ksplit < K;
  L.kp1 = split ? (int)align_up(ksplit, KB) : (int)align_up(K, KB);
  L.kp = split ? L.kp1 + (int)align_up(K - ksplit, KB) : L.kp1;
  const int64_t cap = ws_cap > 0 ? ws_cap : ((int64_t)3 << 29);
  int64_t o = 0;
  L.off_ER = o;  o += align_up(4 * (int64_t)nprob * n, 256);
  L.off_EG = o;  o += align_up(4 * (int64_t)nprob * N, 256);
  L.off_EGf = o; o += align_up(8 * (int64_t)nprob * (N + 1), 256);
  L.off_cmG = o; o += align_up(8 * (int64_t)nprob * N, 256);
  L.off_sG = o;  o += align_up((int64_t)nprob * S * N * L.kp, 1024);
  const int64_t ctas_max = ((n + BM - 1) / BM) * ((N + BN - 1) / BN);
  L.off_mws = o; o += align_up(8 * ctas_max, 256);
  L.off_sX = o;
  const int64_t per_row = (int64_t)nprob * S * L.kp;
  int64_t rows = align_up(n, BM);
  while (rows > BM && o + per_row * rows > cap) rows = align_up(rows / 2, BM);
  L.sc_rows = rows;
  L.total = o + align_up(per_row * rows, 1024);
  return L;
}
}  // namespace oz
}  // namespace bk

extern "C" int64_t bk_ozaki_tsgemm_ws_bytes(int nprob, int64_t n, int K, int N, int ksplit) {
  if (nprob < 1 || nprob > 4 || n <= 0 || K <= 0 || N <= 0) return 0;
  return ts_layout(nprob, n, K, N, ksplit, 0).total;
}

extern "C" int bk_ozaki_tsgemm_d(int nprob, int64_t n, int K, int N, double alpha, const double* const* Xs,
                                 int64_t ldx, const double* const* Gs, int64_t ldg, double beta,
                                 const double* const* Zs, int64_t ldz, double* const* Ys, int64_t ldy,
                                 const double* rowscale, int flags, int ksplit, int nsplit, double* metric_out,
                                 void* ws, int64_t ws_bytes, void* stream) {
  if (nprob < 1 || nprob > 4 || n < 0 || K <= 0 || N < 0) return BK_ERR_ARG;
  if (n == 0 || N == 0) return BK_OK;
  if (K > MAX_CHUNK) return BK_ERR_UNSUPPORTED;  // int32 accumulation bound
  const int ks = metric_out ? ksplit : 0;
  const TsLayout L = ts_layout(nprob, n, K, N, ks, ws_bytes);
  if (!ws || ws_bytes < L.total) return BK_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  int* ER = reinterpret_cast<int*>(w + L.off_ER);
  int* EG = reinterpret_cast<int*>(w + L.off_EG);
  double* EGf = reinterpret_cast<double*>(w + L.off_EGf);
  auto* cmG = reinterpret_cast<unsigned long long*>(w + L.off_cmG);
  int8_t* sG = reinterpret_cast<int8_t*>(w + L.off_sG);
  double* mws = reinterpret_cast<double*>(w + L.off_mws);
  int8_t* sX = reinterpret_cast<int8_t*>(w + L.off_sX);
  const bool split = metric_out && ksplit > 0 && ksplit < K;
  TsEpi P{};
  P.N = N;
  P.nk = L.kp / KB;
  P.snap_stage = -1;
  P.nsplit = nsplit;
  P.alpha = alpha;
  P.beta = beta;
  P.ldz = ldz;
  P.ldy = ldy;
  P.rowscale = rowscale;
  P.upper = (flags & 1) && !metric_out;
  P.kp1 = L.kp1;
  P.kv1 = split ? ksplit : K;
  P.kv2 = split ? K - ksplit : 0;
  static const int f64c = [] {
    const char* e = getenv("PPCG_OZ_F64COMB");
    return e ? atoi(e) : 0;  // measured 1-4% slower than the int64 combine (profiles/ozaki_ab_r02g.txt)
  }();
  P.f64comb = (f64c && L.kp <= TS_F64_COMBINE_K) ? 1 : 0;
  static const int dbg = [] {
    const char* e = getenv("PPCG_OZ_DBG");
    return e ? atoi(e) : 0;
  }();
  P.dbg = dbg;
  P.metric_ws = mws;
  if (metric_out) P.snap_stage = split ? L.kp1 / KB - 1 : P.nk - 1;
  bool any = metric_out != nullptr;
  // G^T digits per problem: column exponents over the K rows of G; k layout split like X's
  CUtensorMap mA[4], mB[4];
  // problems that share X (or G) share its digits: xa[b] / ga[b] = first problem with the same block
  int xa[4], ga[4];
  for (int b = 0; b < nprob; ++b) {
    xa[b] = ga[b] = b;
    for (int c = 0; c < b; ++c) {
      if (xa[b] == b && Xs[c] == Xs[b]) xa[b] = c;
      if (ga[b] == b && Gs[c] == Gs[b]) ga[b] = c;
    }
  }
  cudaMemsetAsync(cmG, 0, 8 * (size_t)nprob * N, st);
  for (int b = 0; b < nprob; ++b) {
    if (beta != 0.0 && (!Zs || !Zs[b])) return BK_ERR_ARG;
    P.Z[b] = Zs ? Zs[b] : nullptr;
    P.Y[b] = Ys[b];
    any = any || Ys[b] != nullptr;
    P.ER[b] = ER + (int64_t)xa[b] * n;
    P.EG[b] = EG + (int64_t)ga[b] * N;
    P.EGf[b] = EGf + (int64_t)ga[b] * ((N + 1) & ~1);  // 16-byte aligned per problem
    if (ga[b] != b) {
      mB[b] = mB[ga[b]];
      continue;
    }
    BK_COUNT();
    k_colmax<<<dim3((unsigned)((K + 63) / 64), (N + 255) / 256), 256, 0, st>>>(K, N, Gs[b], ldg, cmG + (int64_t)b * N);
    BK_COUNT();
    k_exponents<<<(N + 255) / 256, 256, 0, st>>>(N, cmG + (int64_t)b * N, EG + (int64_t)b * N,
                                                 EGf + (int64_t)b * ((N + 1) & ~1));
    int8_t* g = sG + (int64_t)b * S * N * L.kp;
    const int64_t sstr = (int64_t)N * L.kp;
    cudaMemsetAsync(g, 0, (size_t)S * N * L.kp, st);
    // rows [0, ksplit) of G -> k [0, ksplit); rows [ksplit, K) -> k [kp1, ...)
    const int k1 = split ? ksplit : K;
    BK_COUNT();
    k_slice_cols<<<dim3((unsigned)((k1 + 127) / 128), (N + 31) / 32), 256, 0, st>>>(k1, N, Gs[b], ldg,
                                                                                   EG + (int64_t)b * N, 0, g,
                                                                                   L.kp, sstr, L.kp1);
    if (split) {
      // second k range: rows [ksplit, K) of G written at k offset kp1 (k_slice_cols writes
      // out[(c * kld) + (r - r_base)], so shift the output base by kp1 - ksplit)
      BK_COUNT();
      k_slice_cols<<<dim3((unsigned)((K - ksplit + 127) / 128), (N + 31) / 32), 256, 0, st>>>(
          K, N, Gs[b], ldg, EG + (int64_t)b * N, ksplit, g + L.kp1, L.kp, sstr, L.kp - L.kp1);
    }
    if (!encode_digits(&mB[b], g, L.kp, L.kp, N, ts_tbn(), sstr)) return BK_ERR_UNSUPPORTED;
  }
  if (!any) return BK_OK;
  for (int b = nprob; b < 4; ++b) mB[b] = mB[0];
  const int tbn = ts_tbn();
  if (tbn == 32)
    cudaFuncSetAttribute(k_oz_ts<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, ts_smem<32>());
  else
    cudaFuncSetAttribute(k_oz_ts<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, ts_smem<64>());
  const int ctn = (N + tbn - 1) / tbn;
  int64_t metric_ctas = 0;
  for (int64_t r0 = 0; r0 < n; r0 += L.sc_rows) {
    const int64_t rows = lmin(L.sc_rows, n - r0);
    for (int b = 0; b < nprob; ++b) {
      if (xa[b] != b) {
        mA[b] = mA[xa[b]];
        continue;
      }
      int8_t* x = sX + (int64_t)b * S * L.sc_rows * L.kp;
      BK_COUNT();
      k_slice_rows<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(r0, rows, K, Xs[b], ldx, split ? ksplit : K, L.kp1,
                                                              L.kp, x, L.sc_rows * L.kp, ER + (int64_t)b * n);
      if (!encode_digits(&mA[b], x, L.kp, L.kp, rows, BM, L.sc_rows * L.kp)) return BK_ERR_UNSUPPORTED;
    }
    for (int b = nprob; b < 4; ++b) mA[b] = mA[0];
    P.nrows = rows;
    P.r_base = r0;
    P.metric_ws = mws + metric_ctas;
    const int rtn = (int)((rows + BM - 1) / BM);
    const int64_t tiles = (int64_t)ctn * rtn * nprob;
    const int grid = (int)lmin(tiles, kSMs);
    BK_COUNT();
    g_timer.begin(st);
    if (tbn == 32)
      k_oz_ts<32><<<grid, TS_THREADS, ts_smem<32>(), st>>>(mA[0], mA[1], mA[2], mA[3], mB[0], mB[1], mB[2], mB[3], P,
                                                          ctn, rtn, nprob);
    else
      k_oz_ts<64><<<grid, TS_THREADS, ts_smem<64>(), st>>>(mA[0], mA[1], mA[2], mA[3], mB[0], mB[1], mB[2], mB[3], P,
                                                          ctn, rtn, nprob);
    g_timer.end(st);
    {
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        fprintf(stderr, "bk_ozaki_tsgemm_d: launch failed: %s\n", cudaGetErrorString(e));
        return BK_ERR_CUDA;
      }
    }
    metric_ctas += grid;
  }
  if (metric_out) {
    BK_COUNT();
    k_metric_sum<<<1, 512, 0, st>>>(mws, metric_ctas, metric_out, 0);
  }
  BK_CHECK_LAUNCH();
  return BK_OK;
}
