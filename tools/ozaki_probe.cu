// Probe: FP64 Gram C = X^T Y emulated on the int8 tensor cores (tcgen05.mma kind::i8, TMEM
// accumulators), Ozaki scheme with S 7-bit slices per element and per-column exponents.
// Standalone (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o oz tools/ozaki_probe.cu -lcublas -lcuda).
// Compares against cuBLAS DGEMM and a long-double host sum of sampled entries; times each phase.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}\n" ::"r"(smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------- prepass
// column max |x| as monotone uint64 bit patterns (colmax zeroed by the caller); CTA = 64 rows x
// 256 columns, 16 loads in flight per thread
__global__ void __launch_bounds__(256) oz_colmax(int64_t n, int m, const double* X, int64_t ld, unsigned long long* colmax) {
  const int c = blockIdx.y * 256 + threadIdx.x;
  if (c >= m) return;
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  const int nr = (int)min((int64_t)64, n - r0);
  const double* p = X + r0 * ld + c;
  double mx = 0;
  if (nr == 64) {
#pragma unroll 16
    for (int r = 0; r < 64; ++r) mx = fmax(mx, fabs(__ldg(p + r * ld)));
  } else {
    for (int r = 0; r < nr; ++r) mx = fmax(mx, fabs(__ldg(p + r * ld)));
  }
  atomicMax(colmax + c, (unsigned long long)__double_as_longlong(mx));
}

// slices: out[s][c][k] (k = row index, Kld bytes per column), exponent E[c] with max|x_c| < 2^E.
// CTA = 128 rows x 32 columns, 256 threads; thread (column cl, rows 16 g .. 16 g + 15) builds one
// 16-byte vector per slice
template <int S, bool DIG8>
__global__ void __launch_bounds__(256) oz_slice_cols(int64_t n, int m, const double* X, int64_t ld,
                                                     const unsigned long long* colmax, int8_t* out, int64_t Kld,
                                                     int64_t slice_stride) {
  __shared__ __align__(16) int8_t t[S][32][128 + 16];
  const int64_t r0 = (int64_t)blockIdx.x * 128;
  const int c0 = blockIdx.y * 32;
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = c0 + cl;
  double scale = 0;
  if (c < m) {
    const double mx = __longlong_as_double((long long)colmax[c]);
    const int E = (mx > 0) ? ilogb(mx) + 1 : 0;
    scale = DIG8 ? ldexp(1.0, 8 * S - 2 - E) : ldexp(1.0, 7 * S - E);  // |x| 2^-E 2^(7S) < 2^(7S)
  }
  double v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int64_t r = r0 + g * 16 + e;
    v[e] = (c < m && r < n) ? __ldg(X + r * ld + c) : 0.0;
  }
  uint32_t w[S][4];
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) w[s][q] = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    if (DIG8) {
      // signed base-256 digits: Z = trunc(x 2^(8S-2-E)), |Z| < 2^(8S-2); Z + B (B = 0x80 in every lower
      // byte) has unsigned lower bytes u_i, digit_i = u_i - 128, top digit = (Z + B) >> 8(S-1)
      const long long Z = (long long)(v[e] * scale);
      unsigned long long B = 0;
#pragma unroll
      for (int q = 0; q < S - 1; ++q) B |= 0x80ull << (8 * q);
      const long long U = Z + (long long)B;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        int d = (s == 0) ? (int)(U >> (8 * (S - 1))) : (int)((U >> (8 * (S - 1 - s))) & 255) - 128;
        w[s][e >> 2] |= ((uint32_t)(d & 255)) << (8 * (e & 3));
      }
    } else {
      const unsigned long long Y = (unsigned long long)(fabs(v[e]) * scale);
      const bool neg = v[e] < 0;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        int d = (int)((Y >> (7 * (S - 1 - s))) & 127);
        d = neg ? -d : d;
        w[s][e >> 2] |= ((uint32_t)(d & 255)) << (8 * (e & 3));
      }
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s)
    *reinterpret_cast<uint4*>(&t[s][cl][g * 16]) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
  __syncthreads();
  // write: per (s, col) 128 bytes = 8 x 16-byte pieces
  for (int i = threadIdx.x; i < S * 32 * 8; i += blockDim.x) {
    const int p = i & 7, cc = (i >> 3) & 31, s = i >> 8;
    if (c0 + cc < m && r0 + p * 16 < Kld)
      *reinterpret_cast<int4*>(out + s * slice_stride + (int64_t)(c0 + cc) * Kld + r0 + p * 16) =
          *reinterpret_cast<const int4*>(&t[s][cc][p * 16]);
  }
}

__global__ void oz_exponents(int m, const unsigned long long* colmax, int* E) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < m) {
    double mx = __longlong_as_double((long long)colmax[c]);
    E[c] = (mx > 0) ? ilogb(mx) + 1 : 0;
  }
}

// ---------------------------------------------------------------- Ozaki Gram (tcgen05 i8)
constexpr int BM = 128, BN = 64;

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, int kb) {
  // K-major, swizzle = kb bytes (32/64/128), SBO = 8 rows * kb bytes, LBO = 1, version 1
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(((8 * kb) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  uint64_t lt = kb == 128 ? 2 : kb == 64 ? 4 : 6;
  d |= lt << 61;
  return d;
}

template <int S, int KB, int STAGES>
struct OzCfg {
  static constexpr int A_BYTES = S * BM * KB, B_BYTES = S * BN * KB;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

// grid: (tiles, chunks); C partial[chunk][tile][128][64] in fp64 (scaled by 2^(E1+E2))
template <int S, int KB, int STAGES, bool DIG8>
__global__ void __launch_bounds__(192, 1)
oz_gram_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int m1, int m2,
               int64_t n, int64_t rows_per_chunk, const int* EA, const int* EB, const int2* tiles, double* part) {
  using C = OzCfg<S, KB, STAGES>;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 tile = tiles[blockIdx.x];
  const int row0 = tile.x * BM, col0 = tile.y * BN;
  const int64_t k0 = (int64_t)blockIdx.y * rows_per_chunk;
  const int64_t k1 = min(n, k0 + rows_per_chunk);
  const int nk = (int)((k1 - k0 + KB - 1) / KB);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(512));
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
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(empty + st, ph ^ 1);
        uint8_t* sa = sm + st * C::STAGE;
        mbar_expect_tx(full + st, C::STAGE);
        const int kc = (int)(k0 + (int64_t)kb * KB);
        tma3d(sa, &mapA, kc, row0, 0, full + st);
        tma3d(sa + C::A_BYTES, &mapB, kc, col0, 0, full + st);
      }
    }
  } else if (warp == 1) {
    // instruction descriptor: S32 accum (bits 4-5 = 2), A/B signed int8 (bits 7-9, 10-12 = 1), K-major,
    // N >> 3 at bit 17, M >> 4 at bit 24
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(full + st, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t sa = smem_u32(sm + st * C::STAGE);
        const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
        for (int ks = 0; ks < KB / 32; ++ks) {
          // A_i x [B_j0 .. B_j0+nj-1] in one MMA (B slices are consecutive 64-row blocks in shared
          // memory; accumulators acc[t] are consecutive 64-column blocks of TMEM, t = i + j)
#pragma unroll
          for (int i = 0; i < S; ++i) {
#pragma unroll
            for (int j0 = 0; j0 < S - i; j0 += 4) {
              const int nj = (S - i - j0) < 4 ? (S - i - j0) : 4;
              const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((nj * BN) >> 3) << 17) |
                                     ((uint32_t)(BM >> 4) << 24);
              const uint64_t da = make_desc(sa + i * BM * KB + ks * 32, KB);
              const uint64_t db = make_desc(sb + j0 * BN * KB + ks * 32, KB);
              const uint32_t acc = (kb > 0 || ks > 0 || i > 0) ? 1u : 0u;
              const uint32_t dt = tmem + (i + j0) * BN;
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                           ::"r"(dt), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(empty + st)) : "memory");
        if (kb == nk - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(done)) : "memory");
      }
      __syncwarp();
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lane quadrant warp % 4
    const int q = warp & 3;
    const int r = q * 32 + lane;  // tile row
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int gr = row0 + r;
    const int ea = gr < m1 ? EA[gr] : 0;
    double* out = part + (((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * BM + r) * BN;
#pragma unroll 1
    for (int cc = 0; cc < BN; cc += 16) {
      double acc[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[e] = 0;
#pragma unroll
      for (int t = S - 1; t >= 0; --t) {
        uint32_t v[16];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + t * BN + cc;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const double w = DIG8 ? ldexp(1.0, -12 - 8 * t) : ldexp(1.0, -7 * (t + 2));
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[e] = fma((double)(int)v[e], w, acc[e]);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int gc = col0 + cc + e;
        const int eb = gc < m2 ? EB[gc] : 0;
        out[cc + e] = ldexp(acc[e], ea + eb);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

// C = sum over chunks of the partials (fixed order); grid (tiles, 16 row groups of 8 rows)
__global__ void oz_reduce(int m1, int m2, int ntiles, int nchunks, const int2* tiles, const double* part, double* Cm,
                          int64_t ldc, int sym) {
  const int tix = blockIdx.x;
  const int2 tile = tiles[tix];
  const int r = blockIdx.y * 8 + (threadIdx.x >> 6), c = threadIdx.x & 63;
  const int gr = tile.x * BM + r, gc = tile.y * BN + c;
  if (gr >= m1 || gc >= m2) return;
  double s = 0;
  for (int ch = 0; ch < nchunks; ++ch) s += part[(((int64_t)ch * ntiles + tix) * BM + r) * BN + c];
  if (!sym || gc >= gr) Cm[(int64_t)gr * ldc + gc] = s;
  if (sym && gc > gr) Cm[(int64_t)gc * ldc + gr] = s;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncFn get_enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (EncFn)p;
}
static void make_map(CUtensorMap* map, const int8_t* base, int64_t Kld, int m, int S, int box_rows, int kb) {
  static EncFn enc = get_enc();
  cuuint64_t dims[3] = {(cuuint64_t)Kld, (cuuint64_t)m, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)Kld, (cuuint64_t)(Kld * m)};
  cuuint32_t box[3] = {(cuuint32_t)kb, (cuuint32_t)box_rows, (cuuint32_t)S};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = kb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : kb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
}

template <int S, int KB, int STAGES, bool DIG8 = false>
static void run(int64_t n, int m, int nchunks_req, bool sym, int reps) {
  using Cfg = OzCfg<S, KB, STAGES>;
  printf("== S=%d dig8=%d KB=%d STAGES=%d n=%lld m=%d sym=%d smem=%d\n", S, (int)DIG8, KB, STAGES, (long long)n, m, (int)sym, Cfg::SMEM);
  const int64_t ld = (m + 15) / 16 * 16;
  std::vector<double> hX(n * ld), hY(n * ld);
  std::mt19937_64 g(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (int64_t r = 0; r < n; ++r)
    for (int c = 0; c < ld; ++c) {
      double sc = 1.0 / sqrt((double)n) * (1.0 + 3.0 * (c % 7 == 0)) * (c % 11 == 0 ? 1e-3 : 1.0);
      hX[r * ld + c] = c < m ? nd(g) * sc : 0;
      hY[r * ld + c] = c < m ? (nd(g) * sc + 0.5 * hX[r * ld + c]) * (1.0 + 0.001 * c) : 0;
    }
  double *X, *Y, *Cr, *Co, *part;
  CK(cudaMalloc(&X, n * ld * 8)); CK(cudaMalloc(&Y, n * ld * 8));
  CK(cudaMemcpy(X, hX.data(), n * ld * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(Y, hY.data(), n * ld * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&Cr, (int64_t)m * m * 8)); CK(cudaMalloc(&Co, (int64_t)m * m * 8));
  const int64_t Kld = (n + 127) / 128 * 128;
  int8_t *SA, *SB;
  CK(cudaMalloc(&SA, (int64_t)S * m * Kld)); CK(cudaMalloc(&SB, (int64_t)S * m * Kld));
  unsigned long long *cmA, *cmB;
  int *EA, *EB;
  CK(cudaMalloc(&cmA, m * 8)); CK(cudaMalloc(&cmB, m * 8)); CK(cudaMalloc(&EA, m * 4)); CK(cudaMalloc(&EB, m * 4));
  // tiles
  std::vector<int2> ht;
  const int ta = (m + BM - 1) / BM, tb = (m + BN - 1) / BN;
  for (int a = 0; a < ta; ++a)
    for (int b = 0; b < tb; ++b)
      if (!sym || b * BN + BN - 1 >= a * BM) ht.push_back(make_int2(a, b));
  const int ntiles = (int)ht.size();
  int2* dt;
  CK(cudaMalloc(&dt, ntiles * sizeof(int2)));
  CK(cudaMemcpy(dt, ht.data(), ntiles * sizeof(int2), cudaMemcpyHostToDevice));
  int nchunks = nchunks_req;
  int64_t rpc = (n + nchunks - 1) / nchunks;
  rpc = (rpc + KB - 1) / KB * KB;
  nchunks = (int)((n + rpc - 1) / rpc);
  if (rpc * 127 * 127 * S > (1ll << 31)) printf("WARNING: chunk of %lld rows can overflow int32\n", (long long)rpc);
  CK(cudaMalloc(&part, (int64_t)nchunks * ntiles * BM * BN * 8));
  CUtensorMap mA, mB;
  make_map(&mA, SA, Kld, m, S, BM, KB);
  make_map(&mB, SB, Kld, m, S, BN, KB);
  CK(cudaFuncSetAttribute(oz_gram_kernel<S, KB, STAGES, DIG8>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));

  cublasHandle_t hb;
  cublasCreate(&hb);
  double one = 1, zero = 0;
  cudaEvent_t e[6];
  for (auto& x : e) cudaEventCreate(&x);
  auto prepass = [&]() {
    cudaMemsetAsync(cmA, 0, m * 8); cudaMemsetAsync(cmB, 0, m * 8);
    dim3 gc((unsigned)((n + 63) / 64), (m + 255) / 256);
    oz_colmax<<<gc, 256>>>(n, m, X, ld, cmA);
    oz_colmax<<<gc, 256>>>(n, m, Y, ld, cmB);
    oz_exponents<<<(m + 255) / 256, 256>>>(m, cmA, EA);
    oz_exponents<<<(m + 255) / 256, 256>>>(m, cmB, EB);
  };
  auto slice = [&]() {
    dim3 gs((unsigned)((n + 127) / 128), (m + 31) / 32);
    oz_slice_cols<S, DIG8><<<gs, 256>>>(n, m, X, ld, cmA, SA, Kld, Kld * m);
    oz_slice_cols<S, DIG8><<<gs, 256>>>(n, m, Y, ld, cmB, SB, Kld, Kld * m);
  };
  auto gemm = [&]() {
    dim3 gg(ntiles, nchunks);
    oz_gram_kernel<S, KB, STAGES, DIG8><<<gg, 192, Cfg::SMEM>>>(mA, mB, m, m, n, rpc, EA, EB, dt, part);
  };
  auto red = [&]() { oz_reduce<<<dim3(ntiles, 16), 512>>>(m, m, ntiles, nchunks, dt, part, Co, m, 0); };
  CK(cudaMemset(Co, 0, (int64_t)m * m * 8));
  prepass(); slice(); gemm(); red();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  // reference: C = X^T Y ; column-major view: X row-major n x ld == col-major ld x n
  // C_rowmajor (m x m) == C^T col-major; compute col-major Cr' = Y^T X ... simpler: Cr(col-major) = X^T Y with
  // A = X (col-major ld x n) op N? we want sum_r X[r][i] Y[r][j] = (Xcm * Ycm^T)(i,j) with Xcm = ld x n.
  cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, m, m, (int)n, &one, Y, (int)ld, X, (int)ld, &zero, Cr, m);
  // Cr col-major (i=row from Y, j=col from X) -> Cr[j*m + i] = sum Y[.,i] X[.,j] = C[j][i] row-major: C[j][i]= X_j.Y_i
  CK(cudaDeviceSynchronize());
  std::vector<double> hC(m * m), hR(m * m);
  CK(cudaMemcpy(hC.data(), Co, m * m * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hR.data(), Cr, m * m * 8, cudaMemcpyDeviceToHost));
  // hR[j*m+i] = sum_r Y[r][i] X[r][j] = C[j][i] (row j = X col j) -> matches hC[j*m + i] (row-major, rows = X cols)
  double maxrel = 0, maxabs_vs = 0;
  int bad = 0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      if (sym && j < i) continue;
      bool need = true;
      (void)need;
      int a = i / BM, b = j / BN;
      if (sym && !(b * BN + BN - 1 >= a * BM)) continue;
      double d = fabs(hC[i * m + j] - hR[i * m + j]);
      if (!(d <= 1e300)) ++bad;
      maxabs_vs = fmax(maxabs_vs, d);
    }
  // long-double samples: error relative to sum |x||y|
  std::mt19937 g2(3);
  double worst_oz = 0, worst_cb = 0;
  for (int smp = 0; smp < 48; ++smp) {
    int i = g2() % m, j = g2() % m;
    if (sym && j < i) std::swap(i, j);
    if (sym && !((j / BN) * BN + BN - 1 >= (i / BM) * BM)) continue;
    long double s = 0, sa = 0;
    for (int64_t r = 0; r < n; ++r) {
      s += (long double)hX[r * ld + i] * hY[r * ld + j];
      sa += fabsl((long double)hX[r * ld + i] * hY[r * ld + j]);
    }
    worst_oz = fmax(worst_oz, (double)(fabsl(hC[i * m + j] - s) / sa));
    worst_cb = fmax(worst_cb, (double)(fabsl(hR[i * m + j] - s) / sa));
  }
  (void)maxrel;
  printf("nonfinite %d, max |oz - cublas| %.3e; sampled err / sum|xy|: ozaki %.3e cublas %.3e\n", bad, maxabs_vs, worst_oz, worst_cb);
  // timing
  float t[5] = {0};
  for (int rep = 0; rep < reps; ++rep) {
    cudaEventRecord(e[0]); prepass(); cudaEventRecord(e[1]); slice(); cudaEventRecord(e[2]); gemm(); cudaEventRecord(e[3]);
    red(); cudaEventRecord(e[4]);
    cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, m, m, (int)n, &one, Y, (int)ld, X, (int)ld, &zero, Cr, m);
    cudaEventRecord(e[5]);
    CK(cudaEventSynchronize(e[5]));
    for (int i = 0; i < 5; ++i) { float ms; cudaEventElapsedTime(&ms, e[i], e[i + 1]); t[i] += ms / reps; }
  }
  double flops = 2.0 * n * m * m;
  double tot = t[0] + t[1] + t[2] + t[3];
  printf("ms: colmax %.3f slice %.3f gemm %.3f reduce %.3f | total %.3f (%.1f TF/s fp64-equiv, full) | cublas %.3f (%.1f TF/s)\n",
         t[0], t[1], t[2], t[3], tot, flops / tot * 1e-9, t[4], flops / t[4] * 1e-9);
  double macs = (double)ntiles * BM * BN * (double)nchunks * rpc * (S * (S + 1) / 2);
  printf("gemm kernel: tiles %d chunks %d (%d CTAs) rows/chunk %lld, int8 TOPS (padded) %.0f\n", ntiles, nchunks,
         ntiles * nchunks, (long long)rpc, 2 * macs / t[2] * 1e-9);
  cudaFree(X); cudaFree(Y); cudaFree(Cr); cudaFree(Co); cudaFree(part); cudaFree(SA); cudaFree(SB);
  cudaFree(cmA); cudaFree(cmB); cudaFree(EA); cudaFree(EB); cudaFree(dt);
  cublasDestroy(hb);
}

int main(int argc, char** argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 110592;
  int m = argc > 2 ? atoi(argv[2]) : 523;
  int chunks = argc > 3 ? atoi(argv[3]) : 17;
  int reps = 5;
  if (argc > 4) { run<7, 64, 2, true>(n, m, chunks, false, 1); return 0; }
  run<8, 64, 2>(n, m, chunks, true, reps);
  run<7, 64, 2, true>(8192, 200, 1, false, 2);
  run<7, 64, 2, true>(n, m, chunks, true, reps);
  run<7, 64, 2, true>(n, m, chunks, false, reps);
  run<6, 64, 3, true>(n, m, chunks, true, reps);
  return 0;
}
