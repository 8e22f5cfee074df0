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
#include <cuda.h>
#include <type_traits>

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


// ---- one warp per row, whole row in one pass (default for blocks up to 1024 real / 512
// complex columns).
//
// The row gather above is latency-bound (ncu: long-scoreboard stalls, DRAM ~35% busy): per
// nonzero it issues one 8-byte load per lane and waits for it before the next nonzero.
// Here every lane owns NV 16-byte pieces of the row (real: the aligned column pairs
// (2p - off, 2p + 1 - off); complex: one element), so a warp moves a whole X row per
// nonzero with 16-byte loads, and the loads of U nonzeros are issued before their FMAs.
// The loop body is branch-free: padded nonzero slots and pieces outside the row reload a
// valid piece and are discarded at the (warp-uniform) FMA predicate / the store.  Real
// blocks whose first or last column is half of a 16-byte pair leave those (at most two)
// columns to spmm_csr_edge.  Each warp walks RPW consecutive rows and loads the next row's
// (col, val) batch while the current row computes.  FMAs stay in nonzero order: the result
// equals the gather's and scipy's csr_matvecs bit for bit.
constexpr int V_THREADS = 256;
constexpr int V_RPW = 4;  // rows per warp

template <bool CPLX>
BK_DEV void vec_load_nz(const int32_t* col, const double* val, int kk, int ke, int& cj, double& ar, double& ai) {
  cj = 0;
  ar = ai = 0.0;
  if (kk < ke) {
    cj = __ldg(col + kk);
    if (CPLX) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(val) + kk);
      ar = t.x;
      ai = t.y;
    } else {
      ar = __ldg(val + kk);
    }
  }
}

// pieces [p_lo, p_hi] of each row are computed (16-byte aligned pairs / complex elements)
template <bool CPLX, int NV, int U, int MINB>
__global__ void __launch_bounds__(V_THREADS, MINB) spmm_csr_vec(int64_t n, const int32_t* __restrict__ rowptr,
                                                                const int32_t* __restrict__ col,
                                                                const double* __restrict__ val, int p_lo, int p_hi,
                                                                const double2* __restrict__ X, int64_t ldx,
                                                                double2* __restrict__ Y, int64_t ldy) {
  // X, Y: 16-byte aligned bases, ldx/ldy in 16-byte pieces
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (V_THREADS / 32) + (threadIdx.x >> 5);
  const int64_t rbeg = warp * V_RPW;
  if (rbeg >= n) return;
  const int64_t rend = lmin(n, rbeg + V_RPW);
  int pc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) pc[v] = min(max(v * 32 + lane, p_lo), p_hi);
  int kb = __ldg(rowptr + rbeg), ke = __ldg(rowptr + rbeg + 1);
  int cj;
  double ar, ai;
  vec_load_nz<CPLX>(col, val, kb + lane, ke, cj, ar, ai);
  for (int64_t row = rbeg; row < rend; ++row) {
    int nkb = 0, nke = 0, ncj = 0;
    double nar = 0.0, nai = 0.0;
    if (row + 1 < rend) {  // prefetch the next row's first (col, val) batch
      nkb = ke;
      nke = __ldg(rowptr + row + 2);
      vec_load_nz<CPLX>(col, val, nkb + lane, nke, ncj, nar, nai);
    }
    double2 acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = make_double2(0.0, 0.0);
    for (int k0 = kb; k0 < ke; k0 += 32) {
      if (k0 > kb) vec_load_nz<CPLX>(col, val, k0 + lane, ke, cj, ar, ai);  // > 32 nonzeros
      const int cnt = min(32, ke - k0);
      for (int t0 = 0; t0 < cnt; t0 += U) {
        double2 xv[U][NV];
        double a_r[U], a_i[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src = t0 + u < cnt ? t0 + u : t0;  // padded slots reload slot t0's row
          const int64_t jr = __shfl_sync(0xffffffffu, cj, src);
          a_r[u] = __shfl_sync(0xffffffffu, ar, src);
          a_i[u] = CPLX ? __shfl_sync(0xffffffffu, ai, src) : 0.0;
          const double2* xr = X + jr * ldx;
#pragma unroll
          for (int v = 0; v < NV; ++v) xv[u][v] = __ldg(xr + pc[v]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (t0 + u < cnt) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              if (CPLX) {
                acc[v].x = fma(a_r[u], xv[u][v].x, fma(-a_i[u], xv[u][v].y, acc[v].x));
                acc[v].y = fma(a_r[u], xv[u][v].y, fma(a_i[u], xv[u][v].x, acc[v].y));
              } else {
                acc[v].x = fma(a_r[u], xv[u][v].x, acc[v].x);
                acc[v].y = fma(a_r[u], xv[u][v].y, acc[v].y);
              }
            }
          }
      }
    }
    double2* yr = Y + row * ldy;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int p = v * 32 + lane;
      if (p >= p_lo && p <= p_hi) yr[p] = acc[v];
    }
    kb = nkb;
    ke = nke;
    cj = ncj;
    ar = nar;
    ai = nai;
  }
}

// the (at most two) real columns c0, c1 (-1 = none) that are half of a 16-byte pair: one
// thread per row, nonzeros in CSR order
__global__ void spmm_csr_edge(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                              const double* __restrict__ val, int c0, int c1, const double* __restrict__ X,
                              int64_t ldx, double* __restrict__ Y, int64_t ldy) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int kb = __ldg(rowptr + row), ke = __ldg(rowptr + row + 1);
  double a0 = 0.0, a1 = 0.0;
  for (int k = kb; k < ke; ++k) {
    const int64_t j = __ldg(col + k);
    const double a = __ldg(val + k);
    if (c0 >= 0) a0 = fma(a, __ldg(X + j * ldx + c0), a0);
    if (c1 >= 0) a1 = fma(a, __ldg(X + j * ldx + c1), a1);
  }
  if (c0 >= 0) Y[row * ldy + c0] = a0;
  if (c1 >= 0) Y[row * ldy + c1] = a1;
}

// experiment knob for the real NV = 9 case (config 2 widths): 0 = default (U 2, MINB 1)
static int bk_vec_cfg = 0;

template <bool CPLX>
static void launch_vec(int nv, int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, int p_lo,
                       int p_hi, const double* X, int64_t ldx, double* Y, int64_t ldy, cudaStream_t st) {
  const int64_t rows_per_cta = (int64_t)V_RPW * (V_THREADS / 32);
  const unsigned grid = (unsigned)((n + rows_per_cta - 1) / rows_per_cta);
  auto x2 = reinterpret_cast<const double2*>(X);
  auto y2 = reinterpret_cast<double2*>(Y);
  const int64_t lx = ldx / 2, ly = ldy / 2;
#define BK_VEC(NV_, U_, MB_) \
  spmm_csr_vec<CPLX, NV_, U_, MB_><<<grid, V_THREADS, 0, st>>>(n, rowptr, col, val, p_lo, p_hi, x2, lx, y2, ly)
  if (!CPLX && nv == 9 && bk_vec_cfg != 0) {
    switch (bk_vec_cfg) {
      case 1: BK_VEC(9, 1, 1); break;
      case 2: BK_VEC(9, 1, 2); break;
      case 3: BK_VEC(9, 2, 2); break;
      case 4: BK_VEC(9, 4, 1); break;
      case 5: BK_VEC(9, 1, 3); break;
      default: BK_VEC(9, 2, 1); break;
    }
    return;
  }
  // two CTAs per SM (<= 128 registers) beat deeper per-warp MLP (config 2, NV = 9: U 1 x 2 CTAs
  // 0.27 ms, U 2 x 1 CTA 0.37 ms; profiles/spmm_sweep_r01.jsonl)
  switch (nv) {
    case 1: BK_VEC(1, 4, 2); break;
    case 2: BK_VEC(2, 4, 2); break;
    case 3: BK_VEC(3, 2, 2); break;
    case 4: BK_VEC(4, 2, 2); break;
    case 5: BK_VEC(5, 2, 2); break;
    case 6: BK_VEC(6, 1, 2); break;
    case 7: BK_VEC(7, 1, 2); break;
    case 8: BK_VEC(8, 1, 2); break;
    case 9: BK_VEC(9, 1, 2); break;
    case 10: BK_VEC(10, 1, 2); break;
    case 11: BK_VEC(11, 1, 2); break;
    case 12: BK_VEC(12, 1, 2); break;
    case 13: BK_VEC(13, 1, 1); break;
    case 14: BK_VEC(14, 1, 1); break;
    case 15: BK_VEC(15, 1, 1); break;
    case 16: BK_VEC(16, 1, 1); break;
    default: break;
  }
#undef BK_VEC
}

}  // namespace bk

using namespace bk;

// 2: whole-row vector gather (default where it applies); 0: row gather.  3..7 select the
// vector kernel's (U, MINB) experiment variants for NV = 9 (tools/spmm_sweep.py).
static int bk_spmm_variant = 2;
extern "C" int bk_spmm_set_variant(int variant) {
  if (variant < 0 || variant == 1 || variant > 2 + 5) return BK_ERR_ARG;
  bk_spmm_variant = variant > 2 ? 2 : variant;
  bk_vec_cfg = variant > 2 ? variant - 2 : 0;
  return BK_OK;
}

// Y(:, 0:m) = A X(:, 0:m) for a CSR A with n rows (int32 indices).  X and Y row-major.
extern "C" int bk_spmm_csr_d(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, int m,
                             const double* X, int64_t ldx, double* Y, int64_t ldy, void* stream) {
  if (n < 0 || m < 0) return BK_ERR_ARG;
  if (n == 0 || m == 0) return BK_OK;
  const unsigned grid = (unsigned)((n + S_THREADS / 32 - 1) / (S_THREADS / 32));
  cudaStream_t st = (cudaStream_t)stream;
  BK_COUNT();
  const int off = (int)((reinterpret_cast<uintptr_t>(X) >> 3) & 1);
  const bool vec_ok = (ldx % 2) == 0 && (ldy % 2) == 0 && off == (int)((reinterpret_cast<uintptr_t>(Y) >> 3) & 1);
  const int nv = (m + off + 63) / 64;
  const int p_lo = off, p_hi = (m + off) / 2 - 1;  // full 16-byte pairs of X - off
  if (bk_spmm_variant == 2 && vec_ok && nv <= 16 && p_hi >= p_lo) {
    launch_vec<false>(nv, n, rowptr, col, val, p_lo, p_hi, X - off, ldx, Y - off, ldy, st);
    const int c0 = off ? 0 : -1, c1 = ((m + off) & 1) ? m - 1 : -1;
    if (c0 >= 0 || c1 >= 0) {
      BK_COUNT();
      spmm_csr_edge<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, rowptr, col, val, c0, c1, X, ldx, Y, ldy);
    }
  } else if (m <= 32) spmm_csr_real<1><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, val, m, X, ldx, Y, ldy);
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
  const int nvz = (m + 31) / 32;
  if (bk_spmm_variant == 2 && nvz <= 16) {
    launch_vec<true>(nvz, n, rowptr, col, val, 0, m - 1, X, 2 * ldx, Y, 2 * ldy, st);
  } else if (m <= 32) spmm_csr_cplx<1><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, v2, m, x2, ldx, y2, ldy);
  else if (m <= 64) spmm_csr_cplx<2><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, v2, m, x2, ldx, y2, ldy);
  else spmm_csr_cplx<4><<<grid, S_THREADS, 0, st>>>(n, rowptr, col, v2, m, x2, ldx, y2, ldy);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// ---- plane-marching stencil SpMM (default when the CSR is a nearest-neighbour stencil on an
// inferred grid, spmm_plan.py StencilPlan).
//
// Work unit = an 8 x 8 tile (y, z) of the grid x one 256-byte column slice x a range of
// planes x.  The unit marches along x.  A producer warp streams, per plane, the 10 x 10 halo
// tile of X and the tile rows' CSR entries (grid-ordered ELL: values, and per entry the
// 16-bit ring offset of its X row) into an NS-slot shared-memory ring with three 4-D TMA
// loads (cp.async.bulk.tensor; grid-edge halo rows arrive zero-filled); 16 consumer warps
// compute plane x from the X slots of planes x-1, x, x+1.  Full/empty mbarriers replace CTA
// barriers; the kernel is persistent and each CTA walks its units as one continuous load
// stream, so loads run ahead across unit boundaries.  Every X row crosses L2 -> SM ~1.56
// times instead of once per referencing nonzero (7x / 27x), and consumers touch global
// memory only for the stores.
//
// Consumers: thread t computes row t/8 of the tile, 16-byte pieces t%8 and t%8 + 8 of the
// slice (a quarter-warp reads one row's 128 contiguous bytes: no bank conflicts).  A row's
// entries are processed in chunks whose offsets / values / X pieces are all loaded before
// the chunk's first FMA; FMAs run in CSR order, so the result equals bk_spmm_csr_* bit for
// bit.  Plane x's entries travel with X plane x + 1 (both are first needed by plane x).
// Real blocks are addressed in 16-byte pairs of X - off (off = 8-byte misalignment); the
// at most two half-valid edge pairs are computed like the rest (the extra element is the
// preceding buffer column or a zero-filled one) and stored element-wise.
namespace bk {

constexpr int M_T = 8;                   // tile edge (y and z)
constexpr int M_H = M_T + 2;             // halo tile edge
constexpr int M_HR = M_H * M_H;          // X rows per ring slot
// doubles per staged row slice: 64 (512 B) for real rows of <= 8 entries, else 32 (the ring
// must still hold 4 slots of X + ELL in 227 KB); pieces per consumer thread and row = COLS / 16
constexpr int M_NSMAX = 6;               // ring slots (3 planes in use, up to 3 in flight)
constexpr int M_CONS = 512;              // consumer threads (8 per tile row)
constexpr int M_THREADS = M_CONS + 32;   // + producer warp
constexpr uint16_t M_PAD = 0xffff;       // ELL padding offset

struct MarchArgs {
  int nx, ny, nz;
  int xlo;             // first plane the X tensor map covers
  int gy, gz, nslices, xseg, nunits;
  int m, off;          // columns, and leading columns of the slices before column 0 (alignment)
  int order;           // stencil-slot unit order: 0 = slice fastest, 1 = (y, z) tile fastest
  int nodir;           // stencil-slot: every x segment marches upward (plane-holding variants)
  int npieces;         // 16-byte pieces of a row from the slices' origin to the block's end
  int vdoubles;        // ELL value row in doubles (real: even width; complex: 2 x width)
  int woff;            // ELL offset row in uint16 (multiple of 8)
  int width;           // ELL entries per row
  int slot_bytes, vals_off, offs_off, ns;
  double* Y;           // 16-byte aligned base (Y - off for real), ldy in doubles
  int64_t ldy;
};

struct MarchUnit {
  int s, y0, z0, xa, xb;
};

BK_DEV MarchUnit march_unit(const MarchArgs& A, int u) {
  MarchUnit U;
  U.s = u % A.nslices;
  u /= A.nslices;
  U.z0 = (u % A.gz) * M_T;
  u /= A.gz;
  U.y0 = (u % A.gy) * M_T;
  const int seg = u / A.gy;
  U.xa = (int)((int64_t)seg * A.nx / A.xseg);
  U.xb = (int)((int64_t)(seg + 1) * A.nx / A.xseg);
  return U;
}

BK_DEV void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

template <bool CPLX>
using march_vt = typename std::conditional<CPLX, double2, double>::type;

// one row: entries [0, W) (W > 0: compile-time width, chunks of C; W == 0: runtime width);
// this thread's pieces g + 8 k (k < COLS / 16) of the slice
template <bool CPLX, int W, int C, int COLS>
BK_DEV void march_row(const uint16_t* orow, const march_vt<CPLX>* vrow, int width, const double* sb0,
                      const double* sb1, const double* sb2, int hb, double2 (&acc)[COLS / 16]) {
  constexpr int M_NP = COLS / 16;
  const int wd = W > 0 ? W : width;
#pragma unroll(W > 0 ? 32 : 1)
  for (int c0 = 0; c0 < wd; c0 += C) {
    uint16_t o[C];
    march_vt<CPLX> a[C];
    double2 v[C][M_NP];
    if (W > 0 && W <= 8) {  // one 16-byte load of the row's offsets, values in 16-byte pairs
      const uint4 ow = *reinterpret_cast<const uint4*>(orow);
      const uint32_t wds[4] = {ow.x, ow.y, ow.z, ow.w};
#pragma unroll
      for (int t = 0; t < C; ++t) o[t] = (uint16_t)(wds[t >> 1] >> (16 * (t & 1)));
      if constexpr (CPLX) {
#pragma unroll
        for (int t = 0; t < C; ++t) a[t] = vrow[t];
      } else {
#pragma unroll
        for (int t = 0; t < C; t += 2) {
          const double2 pr = *reinterpret_cast<const double2*>(vrow + t);
          a[t] = pr.x;
          if (t + 1 < C) a[t + 1] = pr.y;
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < C; ++t) {
        o[t] = c0 + t < wd ? orow[c0 + t] : M_PAD;
        a[t] = c0 + t < wd ? vrow[c0 + t] : march_vt<CPLX>{};
      }
    }
#pragma unroll
    for (int t = 0; t < C; ++t) {
      const int e = o[t] == M_PAD ? (1 << 14) : o[t];  // padding reads the centre slot, never used
      const int d = e >> 14;
      const double* xr = (d == 0 ? sb0 : d == 1 ? sb1 : sb2) + (e & 0x3fff) * COLS + hb;
#pragma unroll
      for (int k = 0; k < M_NP; ++k) v[t][k] = *reinterpret_cast<const double2*>(xr + 16 * k);
    }
#pragma unroll
    for (int t = 0; t < C; ++t) {
      if (o[t] == M_PAD) continue;
#pragma unroll
      for (int k = 0; k < M_NP; ++k) {
        if constexpr (CPLX) {
          acc[k].x = fma(a[t].x, v[t][k].x, fma(-a[t].y, v[t][k].y, acc[k].x));
          acc[k].y = fma(a[t].x, v[t][k].y, fma(a[t].y, v[t][k].x, acc[k].y));
        } else {
          acc[k].x = fma(a[t], v[t][k].x, acc[k].x);
          acc[k].y = fma(a[t], v[t][k].y, acc[k].y);
        }
      }
    }
  }
}

// store one 16-byte piece pc of a row (real: element-wise where the pair is half valid)
template <bool CPLX>
BK_DEV void march_store(const MarchArgs& A, double* yr, int pc, double2 v) {
  if (CPLX) {
    if (pc >= A.off && pc - A.off < A.m) *reinterpret_cast<double2*>(yr + 2 * pc) = v;
  } else {
    const int c = 2 * pc - A.off;  // first column of the pair
    if (c >= 0 && c + 1 < A.m) {
      *reinterpret_cast<double2*>(yr + 2 * pc) = v;
    } else {
      if (c >= 0 && c < A.m) yr[2 * pc] = v.x;
      if (c + 1 >= 0 && c + 1 < A.m) yr[2 * pc + 1] = v.y;
    }
  }
}

template <bool CPLX, int W, int COLS>
__global__ void __launch_bounds__(M_THREADS, 1) spmm_march_kernel(const __grid_constant__ CUtensorMap xmap,
                                                                  const __grid_constant__ CUtensorMap vmap,
                                                                  const __grid_constant__ CUtensorMap omap,
                                                                  MarchArgs A) {
  extern __shared__ __align__(128) unsigned char msm[];
  __shared__ __align__(8) uint64_t full[M_NSMAX], empty[M_NSMAX];
  const int NS = A.ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], M_CONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == M_CONS / 32) {
    // ---------------- producer: one elected lane streams the planes of every unit
    if (lane == 0) {
      const uint32_t csr_bytes = M_T * M_T * (A.vdoubles * 8 + A.woff * 2);
      int k = 0;
      for (int u = blockIdx.x; u < A.nunits; u += gridDim.x) {
        const MarchUnit U = march_unit(A, u);
        for (int p = U.xa - 1; p <= U.xb; ++p, ++k) {
          const int slot = k % NS;
          unsigned char* sb = msm + (size_t)slot * A.slot_bytes;
          if (k >= NS) mbar_wait(&empty[slot], ((k / NS) - 1) & 1);
          const bool csr = p - 1 >= U.xa && p - 1 < U.xb;  // entries of plane p - 1 ride along
          mbar_arrive_expect_tx(&full[slot], M_HR * COLS * 8 + (csr ? csr_bytes : 0));
          tma_load_4d(sb, &xmap, U.s * COLS, U.z0 - 1, U.y0 - 1, p - A.xlo, &full[slot]);
          if (csr) {
            tma_load_4d(sb + A.vals_off, &vmap, 0, U.z0, U.y0, p - 1, &full[slot]);
            tma_load_4d(sb + A.offs_off, &omap, 0, U.z0, U.y0, p - 1, &full[slot]);
          }
        }
      }
    }
    return;
  }
  // ---------------- consumers
  using VT = march_vt<CPLX>;
  constexpr int M_NP = COLS / 16;
  constexpr int C = W == 27 ? (M_NP > 2 ? 5 : 9) : (W > 0 ? W : 4);
  const int g = threadIdx.x & 7, r = threadIdx.x >> 3;
  const int iy = r / M_T, iz = r % M_T;
  const int hb = (iy * M_H + iz) * COLS + 2 * g;  // X row of (dy, dz) = (-1, -1), this piece
  const int64_t plane = (int64_t)A.ny * A.nz;
  int k = 0;  // load index of the unit's first plane
  for (int u = blockIdx.x; u < A.nunits; u += gridDim.x) {
    const MarchUnit U = march_unit(A, u);
    const bool act = U.y0 + iy < A.ny && U.z0 + iz < A.nz;
    int64_t row = ((int64_t)U.xa * A.ny + U.y0 + iy) * A.nz + U.z0 + iz;
    mbar_wait(&full[k % NS], (k / NS) & 1);
    mbar_wait(&full[(k + 1) % NS], ((k + 1) / NS) & 1);
    for (int x = U.xa; x < U.xb; ++x, row += plane) {
      const int kx = k + (x - U.xa);  // load index of plane x - 1
      const int s0 = kx % NS, s1 = (kx + 1) % NS, s2 = (kx + 2) % NS;
      mbar_wait(&full[s2], ((kx + 2) / NS) & 1);
      // rows whose pieces all lie past the block (the last slice) skip the work
      const int pc = U.s * (COLS / 2) + g;
      if (act && pc < A.npieces) {
        const unsigned char* b2 = msm + (size_t)s2 * A.slot_bytes;
        double2 acc[M_NP];
#pragma unroll
        for (int k2 = 0; k2 < M_NP; ++k2) acc[k2] = make_double2(0.0, 0.0);
        march_row<CPLX, W, C, COLS>(reinterpret_cast<const uint16_t*>(b2 + A.offs_off) + r * A.woff,
                              reinterpret_cast<const VT*>(reinterpret_cast<const double*>(b2 + A.vals_off) +
                                                          r * A.vdoubles),
                              A.width, reinterpret_cast<const double*>(msm + (size_t)s0 * A.slot_bytes),
                              reinterpret_cast<const double*>(msm + (size_t)s1 * A.slot_bytes),
                              reinterpret_cast<const double*>(b2), hb, acc);
        double* yr = A.Y + row * A.ldy;
#pragma unroll
        for (int k2 = 0; k2 < M_NP; ++k2) march_store<CPLX>(A, yr, pc + 8 * k2, acc[k2]);
      }
      // plane x - 1's slot is not needed again
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s0]);
    }
    // release the unit's last two planes
    const int kl = k + (U.xb - U.xa);
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty[kl % NS]);
      mbar_arrive(&empty[(kl + 1) % NS]);
    }
    k = kl + 2;
  }
}

}  // namespace bk

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 4-D tiled tensor map: dims d0 (contiguous) .. d3, strides in elements, box (b0, b1, b2, 1)
static int encode_4d(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* base, int64_t d0, int64_t d1,
                     int64_t d2, int64_t d3, int64_t s1, int64_t s2, int64_t s3, int b0, int b1, int b2) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return BK_ERR_CUDA;
  const cuuint64_t dims[4] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2, (cuuint64_t)d3};
  const cuuint64_t strides[3] = {(cuuint64_t)(s1 * esize), (cuuint64_t)(s2 * esize), (cuuint64_t)(s3 * esize)};
  const cuuint32_t box[4] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (enc(map, dt, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return BK_ERR_UNSUPPORTED;
  return BK_OK;
}

static int march_launch(bool cplx, int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* ell_val,
                        const uint16_t* ell_off, int width, int woff, int m, const double* X, int64_t ldx, double* Y,
                        int64_t ldy, int row_align, void* stream) {
  if (nx < 0 || ny <= 0 || nz <= 0 || m < 0 || xhi < xlo || width <= 0 || woff < width || (woff % 8)) return BK_ERR_ARG;
  if (nx == 0 || m == 0) return BK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  MarchArgs A;
  A.nodir = 0;
  A.nx = nx;
  A.ny = ny;
  A.nz = nz;
  A.xlo = xlo;
  A.width = width;
  A.woff = woff;
  A.m = m;
  const double* xbase;  // 16-byte aligned base of row-space row 0
  int64_t ldxd, cols;   // leading dimension and tensor width in doubles
  if (cplx) {
    // off: leading complex columns (before column 0) the slices start at, for 128-byte lines
    const uintptr_t xa = reinterpret_cast<uintptr_t>(X), ya = reinterpret_cast<uintptr_t>(Y);
    A.off = (row_align % 128 == 0 && ldx % 8 == 0 && ldy % 8 == 0 && xa % 128 == ya % 128) ? (int)((xa % 128) / 16)
                                                                                       : 0;
    xbase = X + 2 * (d0 * ldx - A.off);
    ldxd = 2 * ldx;
    cols = 2 * ((int64_t)m + A.off);
    A.Y = Y - 2 * A.off;
    A.ldy = 2 * ldy;
    A.vdoubles = 2 * width;
  } else {
    A.off = (int)((reinterpret_cast<uintptr_t>(X) >> 3) & 1);
    if ((ldx & 1) || (ldy & 1) || A.off != (int)((reinterpret_cast<uintptr_t>(Y) >> 3) & 1)) return BK_ERR_UNSUPPORTED;
    // rows that start on 128-byte boundaries (caller's row_align): start the slices on the
    // 128-byte boundary at or before column 0, so every TMA row piece covers whole lines
    const uintptr_t xa = reinterpret_cast<uintptr_t>(X), ya = reinterpret_cast<uintptr_t>(Y);
    if (row_align % 128 == 0 && ldx % 16 == 0 && ldy % 16 == 0 && xa % 128 == ya % 128)
      A.off = (int)((xa % 128) / 8);
    xbase = X - A.off + d0 * ldx;
    ldxd = ldx;
    cols = m + A.off;
    A.Y = Y - A.off;
    A.ldy = ldy;
    A.vdoubles = (width + 1) / 2 * 2;
  }
  if (A.vdoubles > 256 || woff > 256) return BK_ERR_UNSUPPORTED;  // TMA box limit
  const int COLS = (!cplx && width <= 8) ? 64 : 32;
  A.vals_off = M_HR * COLS * 8;
  A.offs_off = A.vals_off + M_T * M_T * A.vdoubles * 8;
  A.slot_bytes = (A.offs_off + M_T * M_T * woff * 2 + 127) / 128 * 128;
  A.ns = (int)lmin(M_NSMAX, (227 * 1024) / A.slot_bytes);
  if (A.ns < 4) return BK_ERR_UNSUPPORTED;
  const size_t smem = (size_t)A.ns * A.slot_bytes;
  CUtensorMap xmap, vmap, omap;
  const int64_t P = (int64_t)ny * nz;
  int rc = encode_4d(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, xbase + (int64_t)xlo * P * ldxd, cols, nz, ny,
                     xhi - xlo, ldxd, nz * ldxd, P * ldxd, COLS, M_H, M_H);
  if (rc == BK_OK)
    rc = encode_4d(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, ell_val, A.vdoubles, nz, ny, nx, A.vdoubles,
                   nz * A.vdoubles, P * A.vdoubles, A.vdoubles, M_T, M_T);
  if (rc == BK_OK)
    rc = encode_4d(&omap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, ell_off, woff, nz, ny, nx, woff, nz * woff, P * woff,
                   woff, M_T, M_T);
  if (rc != BK_OK) return rc;
  A.gy = (ny + M_T - 1) / M_T;
  A.gz = (nz + M_T - 1) / M_T;
  A.nslices = (int)((cols + COLS - 1) / COLS);
  A.npieces = (int)((cols + 1) / 2);
  // x segments: >= 8 units per CTA (balance) while a segment keeps >= 8 planes
  const int64_t per_seg = (int64_t)A.gy * A.gz * A.nslices;
  // x segments: minimise waves x (planes per segment + 2 halo planes); units of one wave run
  // the same planes of neighbouring tiles (shared halo rows and whole X rows stay in L2)
  A.xseg = 1;
  int64_t best = -1;
  for (int xs = 1; xs <= lmax(1, nx / 8); ++xs) {
    const int64_t waves = (per_seg * xs + kSMs - 1) / kSMs;
    const int64_t cost = waves * ((nx + xs - 1) / xs + 2);
    if (best < 0 || cost < best) {
      best = cost;
      A.xseg = xs;
    }
  }
  A.nunits = (int)(per_seg * A.xseg);
  // the 7-point (3-D), 27-point and 5-point (2-D) widths run with compile-time chunks
  auto kern = cplx ? (width == 7 ? spmm_march_kernel<true, 7, 32> : width == 5 ? spmm_march_kernel<true, 5, 32>
                      : width == 27 ? spmm_march_kernel<true, 27, 32> : spmm_march_kernel<true, 0, 32>)
                   : (width == 7 ? spmm_march_kernel<false, 7, 64> : width == 5 ? spmm_march_kernel<false, 5, 64>
                      : width == 27 ? spmm_march_kernel<false, 27, 32>
                      : width <= 8 ? spmm_march_kernel<false, 0, 64> : spmm_march_kernel<false, 0, 32>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = (unsigned)lmin(A.nunits, kSMs);
  BK_COUNT();
  kern<<<grid, M_THREADS, smem, st>>>(xmap, vmap, omap, A);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// Y = A X for a CSR A that is a nearest-neighbour stencil on an nx x ny x nz C-order grid,
// from the plan of spmm_plan.py StencilPlan (grid-ordered ELL values and 16-bit ring offsets,
// d0 = column shift, planes [xlo, xhi) referenced); same result as bk_spmm_csr_d.  Real: ldx,
// ldy even and X, Y equally 16-byte aligned, else BK_ERR_UNSUPPORTED.  row_align: the caller's
// guarantee that the rows of the buffers X and Y are views of start on row_align-byte
// boundaries (128 lets the slices start on 128-byte lines).
extern "C" int bk_spmm_march_d(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* ell_val,
                               const uint16_t* ell_off, int width, int woff, int m, const double* X, int64_t ldx,
                               double* Y, int64_t ldy, int row_align, void* stream) {
  return march_launch(false, nx, ny, nz, xlo, xhi, d0, ell_val, ell_off, width, woff, m, X, ldx, Y, ldy, row_align,
                      stream);
}

// complex128: ell_val, X, Y interleaved; ld in complex elements
extern "C" int bk_spmm_march_z(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* ell_val,
                               const uint16_t* ell_off, int width, int woff, int m, const double* X, int64_t ldx,
                               double* Y, int64_t ldy, int row_align, void* stream) {
  return march_launch(true, nx, ny, nz, xlo, xhi, d0, ell_val, ell_off, width, woff, m, X, ldx, Y, ldy, row_align,
                      stream);
}

// ---- stencil-slot march (default for 7-point and 27-point stencils whose CSR rows are
// sorted: spmm_plan.py StencilPlan.slot_values).
//
// Same work units, TMA X ring and plane march as spmm_march_kernel, but the entries arrive
// as a stencil-slot ELL: row r holds the value of stencil position s (CSR order = (dx, dy,
// dz) lexicographic) in slot s and a presence mask in its last double, so every X address is
// a compile-time offset and the kernel reuses X from registers:
//  * 7-point (ST = 7): the centre column of the tile walks along x in registers (planes
//    x-1, x, x+1), only the four in-plane neighbours come from shared memory, and a step
//    holds two ring slots (planes x, x+1) instead of three -- more planes in flight.
//  * 27-point (ST = 27): a thread computes RZ consecutive z rows and loads each (dx, dy)
//    line of RZ + 2 X rows once for all of them: 9 (RZ + 2) / RZ shared loads per output
//    row instead of 27.
// FMAs run in CSR order (absent positions are skipped by the mask), so the result equals
// bk_spmm_csr_* bit for bit.
namespace bk {

constexpr int ST_NSMAX = 8;

// stencil-slot units: slice fastest, then x segment, then (y, z) tile, so the segments of one
// tile run in the same wave; odd segments march down (dir = -1).  Two neighbouring segments
// then read their shared boundary plane at the same moment (both at their start, or both at
// their end) and the second read hits L2 instead of DRAM.
struct StUnit {
  int s, y0, z0, xa, xb, dir;
};

BK_DEV StUnit st_unit(const MarchArgs& A, int u) {
  StUnit U;
  int seg, tile;
  if (A.order == 0) {  // slice fastest: the slices of a tile share its entries (27-point: > L2)
    U.s = u % A.nslices;
    u /= A.nslices;
    seg = u % A.xseg;
    tile = u / A.xseg;
  } else if (A.order == 2) {  // slice, then tile, x segment slowest
    U.s = u % A.nslices;
    u /= A.nslices;
    const int ntiles = A.gy * A.gz;
    tile = u % ntiles;
    seg = u / ntiles;
  } else {  // tile fastest: a wave covers whole planes of one slice, so every halo row is read
            // by all tiles needing it at the same time (7-point: entries of all slices fit L2)
    const int ntiles = A.gy * A.gz;
    tile = u % ntiles;
    u /= ntiles;
    seg = u % A.xseg;
    U.s = u / A.xseg;
  }
  U.z0 = (tile % A.gz) * M_T;
  U.y0 = (tile / A.gz) * M_T;
  U.xa = (int)((int64_t)seg * A.nx / A.xseg);
  U.xb = (int)((int64_t)(seg + 1) * A.nx / A.xseg);
  U.dir = (seg & 1) && !A.nodir ? -1 : 1;
  return U;
}

template <int COLS, int NP, int RZ>
constexpr int st_consumers() {
  return M_T * M_T / RZ * (COLS / 2 / NP);
}
template <int COLS, int NP, int RZ, int RY>
constexpr int st_consumers_y() {
  return M_T * M_T / (RZ * RY) * (COLS / 2 / NP);
}

template <bool CPLX>
BK_DEV void st_fma(double2& acc, march_vt<CPLX> a, double2 v) {
  if constexpr (CPLX) {
    acc.x = fma(a.x, v.x, fma(-a.y, v.y, acc.x));
    acc.y = fma(a.x, v.y, fma(a.y, v.x, acc.y));
  } else {
    acc.x = fma(a, v.x, acc.x);
    acc.y = fma(a, v.y, acc.y);
  }
}

template <bool CPLX, int ST, int COLS, int NP, int RZ, int RY = 1, int HOLD = 0>
__global__ void __launch_bounds__(st_consumers_y<COLS, NP, RZ, RY>() + 32, 1)
    spmm_stencil_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap vmap,
                        MarchArgs A) {
  static_assert(ST == 7 || ST == 27, "stencil");
  static_assert(ST == 27 || (RZ == 1 && RY == 1), "7-point: one row per thread");
  static_assert(HOLD == 0 || (ST == 27 && RY == 1), "plane holding: 27-point, z row blocks");
  constexpr int TPR = COLS / 2 / NP;  // threads per row (16-byte pieces g + TPR k)
  constexpr int NCONS = st_consumers_y<COLS, NP, RZ, RY>();
  constexpr int NR = RY * RZ;         // output rows per thread: RY (y) x RZ (z) block
  using VT = march_vt<CPLX>;
  extern __shared__ __align__(128) unsigned char msm[];
  __shared__ __align__(8) uint64_t full[ST_NSMAX], empty[ST_NSMAX];
  const int NS = A.ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NCONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == NCONS / 32) {
    if (lane == 0) {
      const uint32_t ell_bytes = M_T * M_T * A.vdoubles * 8;
      int k = 0;
      for (int u = blockIdx.x; u < A.nunits; u += gridDim.x) {
        const StUnit U = st_unit(A, u);
        const int nload = U.xb - U.xa + 2;
        for (int i = 0; i < nload; ++i, ++k) {
          const int p = U.dir > 0 ? U.xa - 1 + i : U.xb - i;  // planes in march order
          const int pe = p - U.dir;                             // entries of plane p - dir ride along
          const int slot = k % NS;
          unsigned char* sb = msm + (size_t)slot * A.slot_bytes;
          if (k >= NS) mbar_wait(&empty[slot], ((k / NS) - 1) & 1);
          const bool ell = pe >= U.xa && pe < U.xb;
          mbar_arrive_expect_tx(&full[slot], M_HR * COLS * 8 + (ell ? ell_bytes : 0));
          tma_load_4d(sb, &xmap, U.s * COLS, U.z0 - 1, U.y0 - 1, p - A.xlo, &full[slot]);
          if (ell) tma_load_4d(sb + A.vals_off, &vmap, 0, U.z0, U.y0, pe, &full[slot]);
        }
      }
    }
    return;
  }
  // ---------------- consumers: thread -> (tile row group, piece g)
  const int g = threadIdx.x % TPR, grp = threadIdx.x / TPR;
  constexpr int ZG = M_T / RZ;  // z groups per tile row
  const int iy = (grp / ZG) * RY, iz0 = (grp % ZG) * RZ;
  const int64_t plane = (int64_t)A.ny * A.nz;
  const int pc0 = g;  // first piece of this thread within the slice
  auto xrow = [&](int slot, int hy, int hz) {  // halo-tile row (hy, hz) of a slot, this thread's pieces
    return reinterpret_cast<const double*>(msm + (size_t)slot * A.slot_bytes) + (hy * M_H + hz) * COLS + 2 * pc0;
  };
  auto ld = [&](const double* p, double2 (&v)[NP]) {
#pragma unroll
    for (int k = 0; k < NP; ++k) v[k] = *reinterpret_cast<const double2*>(p + 2 * TPR * k);
  };
  int k = 0;
  for (int u = blockIdx.x; u < A.nunits; u += gridDim.x) {
    const StUnit U = st_unit(A, u);
    const int pcs = U.s * (COLS / 2) + pc0;  // piece index in the row (from the slices' origin)
    bool act[NR];  // output (iy + i / RZ, iz0 + i % RZ)
#pragma unroll
    for (int i = 0; i < NR; ++i)
      act[i] = U.y0 + iy + i / RZ < A.ny && U.z0 + iz0 + i % RZ < A.nz && pcs < A.npieces;
    const int nsteps = U.xb - U.xa;
    const int64_t rstep = U.dir * plane;
    int64_t row = ((int64_t)(U.dir > 0 ? U.xa : U.xb - 1) * A.ny + U.y0 + iy) * A.nz + U.z0 + iz0;
    if constexpr (ST == 7) {
      // centre column in march order: ctp = plane x - dir, ccur = x, ctn = x + dir
      double2 ctp[NP], ccur[NP], ctn[NP];
      mbar_wait(&full[k % NS], (k / NS) & 1);
      ld(xrow(k % NS, iy + 1, iz0 + 1), ctp);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[k % NS]);
      mbar_wait(&full[(k + 1) % NS], ((k + 1) / NS) & 1);
      ld(xrow((k + 1) % NS, iy + 1, iz0 + 1), ccur);
      for (int i = 0; i < nsteps; ++i, row += rstep) {
        const int kx = k + 1 + i;  // load index of plane x
        const int s1 = kx % NS, s2 = (kx + 1) % NS;
        mbar_wait(&full[s2], ((kx + 1) / NS) & 1);
        ld(xrow(s2, iy + 1, iz0 + 1), ctn);
        if (act[0]) {
          const double* ev = reinterpret_cast<const double*>(msm + (size_t)s2 * A.slot_bytes + A.vals_off) +
                             (iy * M_T + iz0) * A.vdoubles;
          const uint32_t mask = (uint32_t)__double_as_longlong(ev[A.vdoubles - 1]);
          const VT* av = reinterpret_cast<const VT*>(ev);
          double2 nb[4][NP];
          ld(xrow(s1, iy, iz0 + 1), nb[0]);      // (0, -1, 0)
          ld(xrow(s1, iy + 1, iz0), nb[1]);      // (0, 0, -1)
          ld(xrow(s1, iy + 1, iz0 + 2), nb[2]);  // (0, 0, +1)
          ld(xrow(s1, iy + 2, iz0 + 1), nb[3]);  // (0, +1, 0)
          double2 acc[NP];
#pragma unroll
          for (int q = 0; q < NP; ++q) acc[q] = make_double2(0.0, 0.0);
#pragma unroll
          for (int s = 0; s < 7; ++s) {
            if (!((mask >> s) & 1u)) continue;
            const VT a = av[s];
#pragma unroll
            for (int q = 0; q < NP; ++q) {
              // dx = -1 / +1: the planes before / after x in grid order
              const double2 v = s == 0 ? (U.dir > 0 ? ctp[q] : ctn[q]) : s == 1 ? nb[0][q] : s == 2 ? nb[1][q]
                                : s == 3 ? ccur[q] : s == 4 ? nb[2][q] : s == 5 ? nb[3][q]
                                : (U.dir > 0 ? ctn[q] : ctp[q]);
              st_fma<CPLX>(acc[q], a, v);
            }
          }
          double* yr = A.Y + row * A.ldy;
#pragma unroll
          for (int q = 0; q < NP; ++q) march_store<CPLX>(A, yr, pcs + TPR * q, acc[q]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s1]);  // plane x: neighbours done, centre kept in registers
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          ctp[q] = ccur[q];
          ccur[q] = ctn[q];
        }
      }
      const int kl = k + 1 + nsteps;  // the last halo plane
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[kl % NS]);
      k = kl + 1;
    } else if constexpr (HOLD > 0) {
      // 27-point with X planes held in registers across the march (always upward).  HOLD = 1:
      // plane x stays in registers from the step that loaded it as x + 1, so a step reads two
      // planes from shared memory (x - 1 line by line, x + 1 into the held array once plane
      // x's FMAs are done).  HOLD = 2: planes x - 1 and x are both held (two arrays swapping
      // roles, the loop unrolled by two), a step reads only plane x + 1 -- into the array
      // plane x - 1 has just left -- and a ring slot is released by the step that loaded it.
      // The real values of a row are read as 16-byte pairs (14 loads for 27 slots + mask).
      double2 pa[3][RZ + 2][NP];
      double2 pb[HOLD == 2 ? 3 : 1][HOLD == 2 ? RZ + 2 : 1][NP];
      auto ldline = [&](int slot, int dyi, double2 (&v)[RZ + 2][NP]) {
#pragma unroll
        for (int j = 0; j < RZ + 2; ++j) ld(xrow(slot, iy + dyi, iz0 + j), v[j]);
      };
      // the three values (dz = -1, 0, 1) of slot group s0 = 9 dx + 3 dy of one row
      auto vals3 = [&](const double* evi, int s0, double2& carry, VT (&a)[3]) {
        const double2* av = reinterpret_cast<const double2*>(evi);
        if constexpr (CPLX) {
          a[0] = av[s0];
          a[1] = av[s0 + 1];
          a[2] = av[s0 + 2];
        } else if (s0 & 1) {  // (s0 - 1, s0) came with the previous group
          const double2 t = av[(s0 + 1) >> 1];
          a[0] = carry.y;
          a[1] = t.x;
          a[2] = t.y;
        } else {
          const double2 t = av[s0 >> 1];
          carry = av[(s0 >> 1) + 1];
          a[0] = t.x;
          a[1] = t.y;
          a[2] = carry.x;
        }
      };
      auto fma_line = [&](const double* ev, const uint32_t (&mask)[RZ], double2 (&carry)[RZ], int dxi, int dyi,
                          const double2 (&v)[RZ + 2][NP], double2 (&acc)[RZ][NP]) {
#pragma unroll
        for (int i = 0; i < RZ; ++i) {
          VT a[3];
          vals3(ev + i * A.vdoubles, dxi * 9 + dyi * 3, carry[i], a);
#pragma unroll
          for (int dzi = 0; dzi < 3; ++dzi) {
            if (!((mask[i] >> (dxi * 9 + dyi * 3 + dzi)) & 1u)) continue;
#pragma unroll
            for (int q = 0; q < NP; ++q) st_fma<CPLX>(acc[i][q], a[dzi], v[i + dzi][q]);
          }
        }
      };
      bool any = false;
#pragma unroll
      for (int i = 0; i < NR; ++i) any |= act[i];
      // one step: plane x - 1 = `prev` (HOLD 2) or ring slot s0 (HOLD 1), plane x = `cur`, plane
      // x + 1 from ring slot s2 into `prev` (HOLD 2) / `cur` (HOLD 1)
      auto step = [&](int i, double2 (&prev)[3][RZ + 2][NP], double2 (&cur)[3][RZ + 2][NP]) {
        const int kx = k + i;  // load index of plane x - 1
        const int s0 = kx % NS, s2 = (kx + 2) % NS;
        mbar_wait(&full[s2], ((kx + 2) / NS) & 1);
        if (any) {
          const double* ev = reinterpret_cast<const double*>(msm + (size_t)s2 * A.slot_bytes + A.vals_off) +
                             (iy * M_T + iz0) * A.vdoubles;
          uint32_t mask[RZ];
          double2 carry[RZ];
          double2 acc[RZ][NP];
#pragma unroll
          for (int r = 0; r < RZ; ++r) {
            mask[r] = (uint32_t)__double_as_longlong(ev[r * A.vdoubles + A.vdoubles - 1]);
            carry[r] = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < NP; ++q) acc[r][q] = make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int dyi = 0; dyi < 3; ++dyi) {
            if constexpr (HOLD == 2) {
              fma_line(ev, mask, carry, 0, dyi, prev[dyi], acc);
            } else {
              double2 v[RZ + 2][NP];
              ldline(s0, dyi, v);
              fma_line(ev, mask, carry, 0, dyi, v, acc);
            }
          }
          if constexpr (HOLD == 2) {
#pragma unroll
            for (int dyi = 0; dyi < 3; ++dyi) ldline(s2, dyi, prev[dyi]);
          }
#pragma unroll
          for (int dyi = 0; dyi < 3; ++dyi) fma_line(ev, mask, carry, 1, dyi, cur[dyi], acc);
#pragma unroll
          for (int dyi = 0; dyi < 3; ++dyi) {
            if constexpr (HOLD == 2) {
              fma_line(ev, mask, carry, 2, dyi, prev[dyi], acc);
            } else {
              ldline(s2, dyi, cur[dyi]);
              fma_line(ev, mask, carry, 2, dyi, cur[dyi], acc);
            }
          }
#pragma unroll
          for (int r = 0; r < RZ; ++r)
            if (act[r]) {
              double* yr = A.Y + (row + r) * A.ldy;
#pragma unroll
              for (int q = 0; q < NP; ++q) march_store<CPLX>(A, yr, pcs + TPR * q, acc[r][q]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[HOLD == 2 ? s2 : s0]);
        row += rstep;
      };
      mbar_wait(&full[k % NS], (k / NS) & 1);
      mbar_wait(&full[(k + 1) % NS], ((k + 1) / NS) & 1);
      if constexpr (HOLD == 2) {
#pragma unroll
        for (int dyi = 0; dyi < 3; ++dyi) {
          ldline(k % NS, dyi, pa[dyi]);
          ldline((k + 1) % NS, dyi, pb[dyi]);
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[k % NS]);
          mbar_arrive(&empty[(k + 1) % NS]);
        }
        for (int i = 0; i < nsteps; i += 2) {
          step(i, pa, pb);
          if (i + 1 < nsteps) step(i + 1, pb, pa);
        }
      } else {
#pragma unroll
        for (int dyi = 0; dyi < 3; ++dyi) ldline((k + 1) % NS, dyi, pa[dyi]);
        for (int i = 0; i < nsteps; ++i) step(i, pa, pa);
        const int kl = k + nsteps;
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[kl % NS]);
          mbar_arrive(&empty[(kl + 1) % NS]);
        }
      }
      k += nsteps + 2;
    } else {
      mbar_wait(&full[k % NS], (k / NS) & 1);
      mbar_wait(&full[(k + 1) % NS], ((k + 1) / NS) & 1);
      for (int i = 0; i < nsteps; ++i, row += rstep) {
        const int kx = k + i;  // load index of plane x - dir
        const int s0 = kx % NS, s2 = (kx + 2) % NS;
        mbar_wait(&full[s2], ((kx + 2) / NS) & 1);
        bool any = false;
#pragma unroll
        for (int i = 0; i < NR; ++i) any |= act[i];
        if (any) {
          const double* ev = reinterpret_cast<const double*>(msm + (size_t)s2 * A.slot_bytes + A.vals_off) +
                             (iy * M_T + iz0) * A.vdoubles;
          // values of output i at ev + ((i / RZ) M_T + i % RZ) vdoubles
          uint32_t mask[NR];
#pragma unroll
          for (int i = 0; i < NR; ++i)
            mask[i] = (uint32_t)__double_as_longlong(ev[((i / RZ) * M_T + i % RZ) * A.vdoubles + A.vdoubles - 1]);
          double2 acc[NR][NP];
#pragma unroll
          for (int i = 0; i < NR; ++i)
#pragma unroll
            for (int q = 0; q < NP; ++q) acc[i][q] = make_double2(0.0, 0.0);
#pragma unroll
          for (int dxi = 0; dxi < 3; ++dxi) {
            const int sl = (U.dir > 0 ? kx + dxi : kx + 2 - dxi) % NS;  // plane x + dxi - 1
            if constexpr (RY == 1) {
#pragma unroll
              for (int dyi = 0; dyi < 3; ++dyi) {
                double2 v[RZ + 2][NP];
#pragma unroll
                for (int j = 0; j < RZ + 2; ++j) ld(xrow(sl, iy + dyi, iz0 + j), v[j]);
#pragma unroll
                for (int i = 0; i < RZ; ++i) {
                  const VT* av = reinterpret_cast<const VT*>(ev + i * A.vdoubles);
#pragma unroll
                  for (int dzi = 0; dzi < 3; ++dzi) {
                    const int s = dxi * 9 + dyi * 3 + dzi;
                    if (!((mask[i] >> s) & 1u)) continue;
                    const VT a = av[s];
#pragma unroll
                    for (int q = 0; q < NP; ++q) st_fma<CPLX>(acc[i][q], a, v[i + dzi][q]);
                  }
                }
              }
            } else {
              // the (RY + 2) x (RZ + 2) halo rows of the block once per plane: 3 (RY+2)(RZ+2) /
              // (RY RZ) X loads per output row instead of 3 (RZ+2) (3 / RZ)
              double2 v[RY + 2][RZ + 2][NP];
#pragma unroll
              for (int jy = 0; jy < RY + 2; ++jy)
#pragma unroll
                for (int jz = 0; jz < RZ + 2; ++jz) ld(xrow(sl, iy + jy, iz0 + jz), v[jy][jz]);
#pragma unroll
              for (int i = 0; i < NR; ++i) {
                const int yi = i / RZ, zi = i % RZ;
                const VT* av = reinterpret_cast<const VT*>(ev + (yi * M_T + zi) * A.vdoubles);
#pragma unroll
                for (int dyi = 0; dyi < 3; ++dyi)
#pragma unroll
                  for (int dzi = 0; dzi < 3; ++dzi) {
                    const int s = dxi * 9 + dyi * 3 + dzi;
                    if (!((mask[i] >> s) & 1u)) continue;
                    const VT a = av[s];
#pragma unroll
                    for (int q = 0; q < NP; ++q) st_fma<CPLX>(acc[i][q], a, v[yi + dyi][zi + dzi][q]);
                  }
              }
            }
          }
#pragma unroll
          for (int i = 0; i < NR; ++i)
            if (act[i]) {
              double* yr = A.Y + (row + (int64_t)(i / RZ) * A.nz + i % RZ) * A.ldy;
#pragma unroll
              for (int q = 0; q < NP; ++q) march_store<CPLX>(A, yr, pcs + TPR * q, acc[i][q]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s0]);
      }
      const int kl = k + nsteps;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[kl % NS]);
        mbar_arrive(&empty[(kl + 1) % NS]);
      }
      k = kl + 2;
    }
  }
}

// stencil-slot kernel variants: (COLS, NP, RZ) per stencil; the knob selects among them for sweeps
static int bk_stencil_cfg = 0;
static int bk_stencil_order = -1;  // unit order override (sweeps): -1 = per stencil default
static int bk_stencil_xseg = 0;    // x segment count override (sweeps): 0 = cost model

}  // namespace bk

// cfg = variant + 10 (order + 1) + 100 xseg: variant 0/1; order 0 slice-(segment)-tile, 1 tile
// fastest, 2 slice-tile-segment; xseg forces the x segment count (0: cost model)
extern "C" int bk_spmm_stencil_set_config(int cfg) {
  if (cfg < 0 || cfg % 100 > 39) return BK_ERR_ARG;
  bk::bk_stencil_cfg = cfg % 10;
  bk::bk_stencil_order = (cfg / 10) % 10 - 1;
  bk::bk_stencil_xseg = cfg / 100;
  return BK_OK;
}

static int stencil_launch(bool cplx, int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* sval,
                          int vd, int st, int m, const double* X, int64_t ldx, double* Y, int64_t ldy, int row_align,
                          void* stream) {
  using namespace bk;
  if (nx < 0 || ny <= 0 || nz <= 0 || m < 0 || xhi < xlo || (st != 7 && st != 27) || vd % 2 ||
      vd < (cplx ? 2 * st + 1 : st + 1) || vd > 256)
    return BK_ERR_ARG;
  if (nx == 0 || m == 0) return BK_OK;
  cudaStream_t strm = (cudaStream_t)stream;
  MarchArgs A;
  A.nx = nx;
  A.ny = ny;
  A.nz = nz;
  A.xlo = xlo;
  A.width = st;
  A.woff = 0;
  A.nodir = 0;
  A.m = m;
  A.vdoubles = vd;
  const double* xbase;
  int64_t ldxd, cols;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(X), ya = reinterpret_cast<uintptr_t>(Y);
  if (cplx) {
    A.off = (row_align % 128 == 0 && ldx % 8 == 0 && ldy % 8 == 0 && xa % 128 == ya % 128) ? (int)((xa % 128) / 16)
                                                                                       : 0;
    xbase = X + 2 * (d0 * ldx - A.off);
    ldxd = 2 * ldx;
    cols = 2 * ((int64_t)m + A.off);
    A.Y = Y - 2 * A.off;
    A.ldy = 2 * ldy;
  } else {
    A.off = (int)((xa >> 3) & 1);
    if ((ldx & 1) || (ldy & 1) || A.off != (int)((ya >> 3) & 1)) return BK_ERR_UNSUPPORTED;
    if (row_align % 128 == 0 && ldx % 16 == 0 && ldy % 16 == 0 && xa % 128 == ya % 128) A.off = (int)((xa % 128) / 8);
    xbase = X - A.off + d0 * ldx;
    ldxd = ldx;
    cols = m + A.off;
    A.Y = Y - A.off;
    A.ldy = ldy;
  }
  // variants: 7-point (COLS, NP) = (32, 2) default / (64, 4); 27-point RZ = 2 default / 4
  const int cfg = bk_stencil_cfg;
  int COLS, NCONS;
  void (*kern)(const CUtensorMap, const CUtensorMap, MarchArgs);
  if (st == 7) {
    if (cfg == 1) {
      COLS = 64;
      NCONS = st_consumers<64, 4, 1>();
      kern = cplx ? spmm_stencil_kernel<true, 7, 64, 4, 1> : spmm_stencil_kernel<false, 7, 64, 4, 1>;
    } else {
      COLS = 32;
      NCONS = st_consumers<32, 2, 1>();
      kern = cplx ? spmm_stencil_kernel<true, 7, 32, 2, 1> : spmm_stencil_kernel<false, 7, 32, 2, 1>;
    }
  } else {
    COLS = 32;
    if (cfg == 1) {
      NCONS = st_consumers<32, 1, 4>();
      kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 4> : spmm_stencil_kernel<false, 27, 32, 1, 4>;
    } else if (cfg == 2) {  // 2 (y) x 2 (z) rows per thread
      NCONS = st_consumers_y<32, 1, 2, 2>();
      kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 2, 2> : spmm_stencil_kernel<false, 27, 32, 1, 2, 2>;
    } else if (cfg == 3) {  // 2 (y) x 4 (z)
      NCONS = st_consumers_y<32, 1, 4, 2>();
      kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 4, 2> : spmm_stencil_kernel<false, 27, 32, 1, 4, 2>;
    } else if (cfg >= 4 && cfg <= 7) {  // planes held in registers: (RZ, HOLD) = (2,1) (2,2) (4,1) (4,2)
      A.nodir = 1;
      if (cfg == 4) {
        NCONS = st_consumers<32, 1, 2>();
        kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 2, 1, 1> : spmm_stencil_kernel<false, 27, 32, 1, 2, 1, 1>;
      } else if (cfg == 5) {
        NCONS = st_consumers<32, 1, 2>();
        kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 2, 1, 2> : spmm_stencil_kernel<false, 27, 32, 1, 2, 1, 2>;
      } else if (cfg == 6) {
        NCONS = st_consumers<32, 1, 4>();
        kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 4, 1, 1> : spmm_stencil_kernel<false, 27, 32, 1, 4, 1, 1>;
      } else {
        NCONS = st_consumers<32, 1, 4>();
        kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 4, 1, 2> : spmm_stencil_kernel<false, 27, 32, 1, 4, 1, 2>;
      }
    } else {
      NCONS = st_consumers<32, 1, 2>();
      kern = cplx ? spmm_stencil_kernel<true, 27, 32, 1, 2> : spmm_stencil_kernel<false, 27, 32, 1, 2>;
    }
  }
  A.vals_off = M_HR * COLS * 8;
  A.offs_off = 0;
  A.slot_bytes = (A.vals_off + M_T * M_T * vd * 8 + 127) / 128 * 128;
  A.ns = (int)lmin(ST_NSMAX, (227 * 1024) / A.slot_bytes);
  if (A.ns < 4 && cfg != 0) {  // variant does not fit (complex 512-byte slices): the default
    bk_stencil_cfg = 0;
    const int rc0 = stencil_launch(cplx, nx, ny, nz, xlo, xhi, d0, sval, vd, st, m, X, ldx, Y, ldy, row_align, stream);
    bk_stencil_cfg = cfg;
    return rc0;
  }
  if (A.ns < 4) return BK_ERR_UNSUPPORTED;
  const size_t smem = (size_t)A.ns * A.slot_bytes;
  CUtensorMap xmap, vmap;
  const int64_t P = (int64_t)ny * nz;
  int rc = encode_4d(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, xbase + (int64_t)xlo * P * ldxd, cols, nz, ny,
                     xhi - xlo, ldxd, nz * ldxd, P * ldxd, COLS, M_H, M_H);
  if (rc == BK_OK)
    rc = encode_4d(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, sval, vd, nz, ny, nx, vd, nz * vd, P * vd, vd, M_T,
                   M_T);
  if (rc != BK_OK) return rc;
  A.gy = (ny + M_T - 1) / M_T;
  A.gz = (nz + M_T - 1) / M_T;
  A.nslices = (int)((cols + COLS - 1) / COLS);
  A.npieces = (int)((cols + 1) / 2);
  const int64_t per_seg = (int64_t)A.gy * A.gz * A.nslices;
  A.xseg = 1;
  int64_t best = -1;
  for (int xs = 1; xs <= lmax(1, nx / 8); ++xs) {
    const int64_t waves = (per_seg * xs + kSMs - 1) / kSMs;
    const int64_t cost = waves * ((nx + xs - 1) / xs + 2);
    if (best < 0 || cost < best) {
      best = cost;
      A.xseg = xs;
    }
  }
  // 7-point: segments of ~12 planes, segment slowest (every wave marches one segment in
  // lockstep over all slices of a band of tiles), odd segments downward: measured best over
  // xseg 1..16 x three unit orders at configs 2, 3 and 5 (profiles/stencil_sweep_r02.jsonl:
  // config 2 0.212 -> 0.175 ms, 0.68 -> 0.82 of HBM)
  if (st == 7) A.xseg = (int)lmax(1, (nx + 6) / 12);
  if (bk_stencil_xseg > 0) A.xseg = (int)lmin(bk_stencil_xseg, nx);
  A.nunits = (int)(per_seg * A.xseg);
  A.order = st == 7 ? (bk_stencil_order >= 0 ? bk_stencil_order : 2) : (bk_stencil_order >= 0 ? bk_stencil_order : 0);
  // per launch: the attribute belongs to the current device's context (cheap)
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = (unsigned)lmin(A.nunits, kSMs);
  BK_COUNT();
  kern<<<grid, NCONS + 32, smem, strm>>>(xmap, vmap, A);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// Y = A X for a nearest-neighbour stencil CSR with sorted rows, from the stencil-slot values of
// spmm_plan.py StencilPlan (sval: n x vd doubles per row -- st = 7 or 27 slot values, real or
// interleaved complex, the presence mask's bits in the row's last double); same result as
// bk_spmm_csr_*.  Other arguments as bk_spmm_march_*.
extern "C" int bk_spmm_stencil_d(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* sval, int vd,
                                 int st, int m, const double* X, int64_t ldx, double* Y, int64_t ldy, int row_align,
                                 void* stream) {
  return stencil_launch(false, nx, ny, nz, xlo, xhi, d0, sval, vd, st, m, X, ldx, Y, ldy, row_align, stream);
}

extern "C" int bk_spmm_stencil_z(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* sval, int vd,
                                 int st, int m, const double* X, int64_t ldx, double* Y, int64_t ldy, int row_align,
                                 void* stream) {
  return stencil_launch(true, nx, ny, nz, xlo, xhi, d0, sval, vd, st, m, X, ldx, Y, ldy, row_align, stream);
}
