// Large subblock updates (pencil dimension d > 192, e.g. whole-block PPCG with sbsize >= 65,
// or LOBPCG's block_update over the whole [X, W, P]): the same block_update decision tree as
// pencil.cu (blockeig ppcg.py:278-378), with the host running the branch logic and these
// kernels plus cuSOLVER (dense.cu: potrf probe + sygvd, gesvd) doing the arithmetic.
//
//   bk_block_assemble_*  scaled, symmetrised pencil of the kept basis      ppcg.py:312-330, core.py:143-164
//   bk_block_coef_*      un-scaled coefficients onto the raw columns,      ppcg.py:358-363, 376
//                        coeff_scale = max |C|
//   bk_block_stats_*     non-finite / max|.| breakdown statistics          ppcg.py:701-705
#include "common.cuh"

namespace bk {

// A[a][b] = (Ar[ia][ib] + conj(Ar[ib][ia])) / 2 * sf[a] sf[b]  (same for B), real diagonal
__global__ void k_block_assemble(int d, const int* __restrict__ idx, const double* __restrict__ sf,
                                 const double* __restrict__ Ar, const double* __restrict__ Br, int64_t ldr,
                                 double* __restrict__ A, double* __restrict__ B, int64_t ld, int cplx) {
  const int64_t tot = (int64_t)d * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / d), b = (int)(e % d);
    const int ia = idx[a], ib = idx[b];
    const double s = 0.5 * sf[a] * sf[b];
    if (!cplx) {
      A[a * ld + b] = (Ar[ia * ldr + ib] + Ar[ib * ldr + ia]) * s;
      B[a * ld + b] = (Br[ia * ldr + ib] + Br[ib * ldr + ia]) * s;
    } else {
      const double* x1 = Ar + 2 * (ia * ldr + ib);
      const double* x2 = Ar + 2 * (ib * ldr + ia);
      const double* y1 = Br + 2 * (ia * ldr + ib);
      const double* y2 = Br + 2 * (ib * ldr + ia);
      A[2 * (a * ld + b)] = (x1[0] + x2[0]) * s;
      A[2 * (a * ld + b) + 1] = a == b ? 0.0 : (x1[1] - x2[1]) * s;
      B[2 * (a * ld + b)] = (y1[0] + y2[0]) * s;
      B[2 * (a * ld + b) + 1] = a == b ? 0.0 : (y1[1] - y2[1]) * s;
    }
  }
}

// coef (nparts*w x w, ld w) = 0; coef[idx[a]][c] = C[a][c] * sf[a]; cmax = max |C[:, :w]|
__global__ void k_block_coef(int d, int w, int nrows, const int* __restrict__ idx, const double* __restrict__ sf,
                             const double* __restrict__ C, int64_t ldc, double* __restrict__ coef, int cplx,
                             double* cmax) {
  __shared__ double red[32];
  const int e2 = cplx ? 2 : 1;
  for (int64_t e = threadIdx.x; e < (int64_t)nrows * w * e2; e += blockDim.x) coef[e] = 0.0;
  __syncthreads();
  double m = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)d * w; e += blockDim.x) {
    const int a = (int)(e / w), c = (int)(e % w);
    if (!cplx) {
      const double v = C[a * ldc + c];
      m = fmax(m, fabs(v));
      coef[(int64_t)idx[a] * w + c] = v * sf[a];
    } else {
      const double re = C[2 * (a * ldc + c)], im = C[2 * (a * ldc + c) + 1];
      m = fmax(m, sqrt(re * re + im * im));
      coef[2 * ((int64_t)idx[a] * w + c)] = re * sf[a];
      coef[2 * ((int64_t)idx[a] * w + c) + 1] = im * sf[a];
    }
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmax(t, red[i]);
    cmax[0] = t;
  }
}

// flags[0] |= any non-finite; flags[slot] = max(flags[slot], max |x|) (bit pattern of a
// non-negative double, monotone as an integer; modulus for complex); slot 0: non-finite only
__global__ void k_block_stats(int64_t n, int m, const double* __restrict__ X, int64_t ldx, int cplx,
                              unsigned long long* flags, int slot) {
  const int e2 = cplx ? 2 : 1;
  double mx = 0.0;
  bool bad = false;
  const int64_t tot = n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / m;
    const int c = (int)(e % m);
    const double* p = X + (r * ldx + c) * e2;
    if (!cplx) {
      bad |= !isfinite(p[0]);
      mx = fmax(mx, fabs(p[0]));
    } else {
      bad |= !isfinite(p[0]) || !isfinite(p[1]);
      mx = fmax(mx, sqrt(p[0] * p[0] + p[1] * p[1]));
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicOr(&flags[0], 1ull);
    if (slot > 0 && mx > 0.0) atomicMax(&flags[slot], dbits(mx));
  }
}

static unsigned grid_of(int64_t tot) { return (unsigned)lmin(4096, lmax(1, (tot + 255) / 256)); }

}  // namespace bk

using namespace bk;

// A, B: d x d row-major (ld, in scalars of the field) from raw Grams Ar/Br (ldr); idx/sf: device
extern "C" int bk_block_assemble(int d, int cplx, const int* idx, const double* sf, const double* Ar,
                                 const double* Br, int64_t ldr, double* A, double* B, int64_t ld, void* stream) {
  if (d <= 0) return BK_ERR_ARG;
  BK_COUNT();
  k_block_assemble<<<grid_of((int64_t)d * d), 256, 0, (cudaStream_t)stream>>>(d, idx, sf, Ar, Br, ldr, A, B, ld,
                                                                              cplx);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// coef: nrows x w (ld w) with nrows = nparts * w; C: d x >= w (ldc); cmax: device scalar
extern "C" int bk_block_coef(int d, int w, int nrows, int cplx, const int* idx, const double* sf, const double* C,
                             int64_t ldc, double* coef, double* cmax, void* stream) {
  if (d <= 0 || w <= 0) return BK_ERR_ARG;
  BK_COUNT();
  k_block_coef<<<1, 1024, 0, (cudaStream_t)stream>>>(d, w, nrows, idx, sf, C, ldc, coef, cplx, cmax);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_block_stats(int64_t n, int m, int cplx, const double* X, int64_t ldx, unsigned long long* flags,
                              int slot, void* stream) {
  if (n < 0 || m < 0 || slot < 0 || slot > 2) return BK_ERR_ARG;
  if (n == 0 || m == 0) return BK_OK;
  BK_COUNT();
  k_block_stats<<<grid_of(n * m), 256, 0, (cudaStream_t)stream>>>(n, m, X, ldx, cplx, flags, slot);
  BK_CHECK_LAUNCH();
  return BK_OK;
}
