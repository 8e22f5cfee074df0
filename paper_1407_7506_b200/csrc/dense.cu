// Periodic dense work (north-star item 5): Cholesky-QR factor, triangular inverse,
// k_total x k_total generalized eigenproblem, Householder QR (recovery only), plus the small
// elementwise/reduction kernels the host orchestration needs.  cuSOLVER is used only here,
// outside the per-iteration subblock path, as BASELINE.json permits.
//
//   bk_chol_upper_floor_*   _cholesky_upper with the 1e-14 pivot floor    core.py:67-83
//   bk_tri_inv_upper_*      R^{-1} for Q = X R^{-1}                        core.py:99
//   bk_rr_pencil_*          solve_pencil(SmallPencil(S^H AS, S^H S), kt)   core.py:175-202,
//                           used by _extract_ritz                          ppcg.py:553-584
//   bk_householder_q_*      np.linalg.qr(x)[0]                             ppcg.py:567,712,756
//
// Row-major <-> column-major: a row-major buffer seen by cuSOLVER is the transpose (for
// Hermitian matrices: the conjugate).  Potrf(LOWER) on a row-major Gram therefore returns
// the row-major UPPER factor R with R^H R = G directly, and trtri(LOWER) its inverse.
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include "common.cuh"

namespace bk {

struct DenseCtx {
  cusolverDnHandle_t h = nullptr;
  cudaStream_t st = nullptr;
  void* dwork = nullptr;
  size_t dbytes = 0;
  void* hwork = nullptr;
  size_t hbytes = 0;
  int* dinfo = nullptr;  // 4 ints
  double* dscal = nullptr;  // 8 doubles
};

static int ensure(DenseCtx* c, size_t dbytes, size_t hbytes) {
  if (dbytes > c->dbytes) {
    if (c->dwork) cudaFree(c->dwork);
    size_t nb = dbytes + (dbytes >> 2) + 4096;
    if (cudaMalloc(&c->dwork, nb) != cudaSuccess) { c->dwork = nullptr; c->dbytes = 0; return BK_ERR_CUDA; }
    c->dbytes = nb;
  }
  if (hbytes > c->hbytes) {
    free(c->hwork);
    c->hwork = malloc(hbytes + 64);
    if (!c->hwork) { c->hbytes = 0; return BK_ERR_CUDA; }
    c->hbytes = hbytes + 64;
  }
  return BK_OK;
}

// ---------------------------------------------------------------- small kernels
__global__ void k_symmetrize(int n, double* A, int64_t lda, int cplx) {
  // A <- (A + A^H) / 2 on an n x n matrix (real or interleaved complex)
  const int64_t tot = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (i > j) continue;
    if (!cplx) {
      const double v = 0.5 * (A[i * lda + j] + A[j * lda + i]);
      A[i * lda + j] = v;
      A[j * lda + i] = v;
    } else {
      double* a = A + 2 * (i * lda + j);
      double* b = A + 2 * (j * lda + i);
      const double re = 0.5 * (a[0] + b[0]);
      const double im = 0.5 * (a[1] - b[1]);
      a[0] = re; a[1] = im;
      b[0] = re; b[1] = -im;
    }
  }
}

// out[0] = ||A||_F^2 (single CTA)
__global__ void k_fro2(int n, const double* A, int64_t lda, int cplx, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  const int w = cplx ? 2 : 1;
  for (int64_t e = threadIdx.x; e < (int64_t)n * n * w; e += blockDim.x) {
    const int64_t i = e / (n * w), jj = e % (n * w);
    const double v = A[i * lda * w + jj];
    s = fma(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    out[0] = t;
  }
}

// B <- A (n x n) then B -= 1e-12 * max(sqrt(fro2), 1e-300) * I
__global__ void k_copy_shift(int n, const double* A, int64_t lda, double* B, int64_t ldb, int cplx,
                             const double* fro2) {
  const double flo = 1e-12 * fmax(sqrt(fro2[0]), 1e-300);
  const int w = cplx ? 2 : 1;
  const int64_t tot = (int64_t)n * n * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / (n * w), jj = e % (n * w);
    double v = A[i * lda * w + jj];
    if (jj == i * w) v -= flo;
    B[i * ldb * w + jj] = v;
  }
}

// row-major C[i][j] = Z(i, j) (conj for complex), Z column-major with ldz
__global__ void k_colmajor_to_rowmajor(int n, int ncols, const double* Z, int64_t ldz, double* C, int64_t ldc,
                                       int cplx) {
  const int64_t tot = (int64_t)n * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / ncols), j = (int)(e % ncols);
    if (!cplx) {
      C[i * ldc + j] = Z[(int64_t)j * ldz + i];
    } else {
      C[2 * (i * ldc + j)] = Z[2 * ((int64_t)j * ldz + i)];
      C[2 * (i * ldc + j) + 1] = -Z[2 * ((int64_t)j * ldz + i) + 1];
    }
  }
}

// pivot-floor check after potrf: fail column = first j with R_jj^2 <= 1e-14 * max|G_jj|
// (G diagonal saved in gdiag), or info-1 if potrf failed; zero the strictly lower part
// (row-major) of R.  out: fail_col (-1 if none)
__global__ void k_chol_check(int m, double* R, int64_t ldr, const double* gdiag, const int* info, int cplx,
                             int* fail_col) {
  __shared__ double s_scale;
  __shared__ int s_fail;
  const int w = cplx ? 2 : 1;
  if (threadIdx.x == 0) {
    double sc = 0.0;
    for (int j = 0; j < m; ++j) sc = fmax(sc, fabs(gdiag[j]));
    s_scale = fmax(sc, 1e-300);
    int f = -1;
    const int inf = info[0];
    const int lim = inf > 0 ? inf - 1 : m;
    for (int j = 0; j < lim; ++j) {
      const double r = R[(j * ldr + j) * w];
      const double piv = r * r;
      if (!(piv > 1e-14 * s_scale) || !isfinite(piv)) { f = j; break; }
    }
    if (f < 0 && inf > 0) f = inf - 1;
    s_fail = f;
    fail_col[0] = f;
  }
  __syncthreads();
  const int64_t tot = (int64_t)m * m;
  for (int64_t e = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; e < tot; e += (int64_t)blockDim.x * gridDim.x) {
    const int i = (int)(e / m), j = (int)(e % m);
    if (i > j) {
      R[(i * ldr + j) * w] = 0.0;
      if (cplx) R[(i * ldr + j) * w + 1] = 0.0;
    }
  }
}

__global__ void k_save_diag(int m, const double* G, int64_t ldg, int cplx, double* out) {
  const int w = cplx ? 2 : 1;
  for (int j = threadIdx.x + blockIdx.x * blockDim.x; j < m; j += blockDim.x * gridDim.x) out[j] = G[(j * ldg + j) * w];
}

__global__ void k_status(const int* info_a, const int* info_b, int* status) {
  status[0] = (info_a[0] != 0 || info_b[0] != 0) ? 1 : 0;
  status[1] = info_a[0];
  status[2] = info_b[0];
}

static unsigned grid_for(int64_t tot) { return (unsigned)lmin(4096, lmax(1, (tot + 255) / 256)); }

}  // namespace bk

using namespace bk;

extern "C" int bk_dense_create(void** ctx, void* stream) {
  DenseCtx* c = new DenseCtx();
  c->st = (cudaStream_t)stream;
  if (cusolverDnCreate(&c->h) != CUSOLVER_STATUS_SUCCESS) { delete c; return BK_ERR_SOLVER; }
  cusolverDnSetStream(c->h, c->st);
  if (cudaMalloc(&c->dinfo, 4 * sizeof(int)) != cudaSuccess) { cusolverDnDestroy(c->h); delete c; return BK_ERR_CUDA; }
  if (cudaMalloc(&c->dscal, 8 * sizeof(double)) != cudaSuccess) { cudaFree(c->dinfo); cusolverDnDestroy(c->h); delete c; return BK_ERR_CUDA; }
  *ctx = c;
  return BK_OK;
}

extern "C" int bk_dense_destroy(void* ctx) {
  DenseCtx* c = static_cast<DenseCtx*>(ctx);
  if (!c) return BK_OK;
  cudaStreamSynchronize(c->st);
  if (c->dwork) cudaFree(c->dwork);
  free(c->hwork);
  cudaFree(c->dinfo);
  cudaFree(c->dscal);
  cusolverDnDestroy(c->h);
  delete c;
  return BK_OK;
}

extern "C" int bk_dense_set_stream(void* ctx, void* stream) {
  DenseCtx* c = static_cast<DenseCtx*>(ctx);
  c->st = (cudaStream_t)stream;
  return cusolverDnSetStream(c->h, c->st) == CUSOLVER_STATUS_SUCCESS ? BK_OK : BK_ERR_SOLVER;
}

// In place: G (m x m Gram, row-major) -> R upper with R^H R = G; fail_col (device int) =
// first column whose pivot is <= 1e-14 max|diag G| (or -1).  (core.py:67-83)
static int chol_upper_floor(DenseCtx* c, int m, double* G, int64_t ldg, int cplx, int* fail_col) {
  if (m <= 0) return BK_ERR_ARG;
  cudaDataType dt = cplx ? CUDA_C_64F : CUDA_R_64F;
  cusolverDnParams_t prm;
  cusolverDnCreateParams(&prm);
  size_t db = 0, hb = 0;
  if (cusolverDnXpotrf_bufferSize(c->h, prm, CUBLAS_FILL_MODE_LOWER, m, dt, G, ldg, dt, &db, &hb) !=
      CUSOLVER_STATUS_SUCCESS) { cusolverDnDestroyParams(prm); return BK_ERR_SOLVER; }
  size_t diag_bytes = ((size_t)m * sizeof(double) + 255) & ~(size_t)255;
  if (ensure(c, db + diag_bytes, hb) != BK_OK) { cusolverDnDestroyParams(prm); return BK_ERR_CUDA; }
  double* gdiag = reinterpret_cast<double*>(c->dwork);
  void* work = static_cast<char*>(c->dwork) + diag_bytes;
  BK_COUNT();
  k_save_diag<<<grid_for(m), 256, 0, c->st>>>(m, G, ldg, cplx, gdiag);
  cusolverStatus_t s = cusolverDnXpotrf(c->h, prm, CUBLAS_FILL_MODE_LOWER, m, dt, G, ldg, dt, work, db,
                                        hb ? c->hwork : nullptr, hb, c->dinfo);
  cusolverDnDestroyParams(prm);
  if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  BK_COUNT();
  k_chol_check<<<grid_for((int64_t)m * m), 256, 0, c->st>>>(m, G, ldg, gdiag, c->dinfo, cplx, fail_col);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_chol_upper_floor_d(void* ctx, int m, double* G, int64_t ldg, int* fail_col) {
  return chol_upper_floor(static_cast<DenseCtx*>(ctx), m, G, ldg, 0, fail_col);
}
extern "C" int bk_chol_upper_floor_z(void* ctx, int m, double* G, int64_t ldg, int* fail_col) {
  return chol_upper_floor(static_cast<DenseCtx*>(ctx), m, G, ldg, 1, fail_col);
}

// In place R (upper, row-major) -> R^{-1}
static int tri_inv_upper(DenseCtx* c, int m, double* R, int64_t ldr, int cplx) {
  cudaDataType dt = cplx ? CUDA_C_64F : CUDA_R_64F;
  size_t db = 0, hb = 0;
  if (cusolverDnXtrtri_bufferSize(c->h, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, m, dt, R, ldr, &db, &hb) !=
      CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  if (ensure(c, db, hb) != BK_OK) return BK_ERR_CUDA;
  if (cusolverDnXtrtri(c->h, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, m, dt, R, ldr, c->dwork, db,
                       hb ? c->hwork : nullptr, hb, c->dinfo) != CUSOLVER_STATUS_SUCCESS)
    return BK_ERR_SOLVER;
  return BK_OK;
}
extern "C" int bk_tri_inv_upper_d(void* ctx, int m, double* R, int64_t ldr) {
  return tri_inv_upper(static_cast<DenseCtx*>(ctx), m, R, ldr, 0);
}
extern "C" int bk_tri_inv_upper_z(void* ctx, int m, double* R, int64_t ldr) {
  return tri_inv_upper(static_cast<DenseCtx*>(ctx), m, R, ldr, 1);
}

// Generalized Hermitian-definite pencil of dimension d (row-major, ld lda; A and B are
// overwritten).  omega: d ascending eigenvalues; C: d x d row-major B-orthonormal
// eigenvectors (ld ldc); status (device, 3 ints): [0] = 1 if singular (the Cholesky of
// B - 1e-12 ||B||_F I failed, or sygvd's own Cholesky failed).
static int rr_pencil(DenseCtx* c, int d, double* A, int64_t lda, double* B, int64_t ldb, double* omega, double* C,
                     int64_t ldc, int cplx, int* status) {
  if (d <= 0 || lda > 0x7fffffff || ldb > 0x7fffffff) return BK_ERR_ARG;
  const int w = cplx ? 2 : 1;
  BK_COUNT();
  k_symmetrize<<<grid_for((int64_t)d * d), 256, 0, c->st>>>(d, A, lda, cplx);
  BK_COUNT();
  k_symmetrize<<<grid_for((int64_t)d * d), 256, 0, c->st>>>(d, B, ldb, cplx);
  BK_COUNT();
  k_fro2<<<1, 1024, 0, c->st>>>(d, B, ldb, cplx, c->dscal);
  // singular-Gram probe on a shifted copy
  int lw = 0, lwp = 0;
  const size_t tmp_bytes = (((size_t)d * d * w * sizeof(double)) + 255) & ~(size_t)255;
  cusolverStatus_t s;
  if (!cplx) {
    s = cusolverDnDpotrf_bufferSize(c->h, CUBLAS_FILL_MODE_LOWER, d, B, d, &lwp);
    if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
    s = cusolverDnDsygvd_bufferSize(c->h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d,
                                    A, (int)lda, B, (int)ldb, omega, &lw);
  } else {
    s = cusolverDnZpotrf_bufferSize(c->h, CUBLAS_FILL_MODE_LOWER, d, reinterpret_cast<cuDoubleComplex*>(B), d, &lwp);
    if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
    s = cusolverDnZhegvd_bufferSize(c->h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d,
                                    reinterpret_cast<cuDoubleComplex*>(A), (int)lda,
                                    reinterpret_cast<cuDoubleComplex*>(B), (int)ldb, omega, &lw);
  }
  if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  const size_t wbytes = (size_t)max(lw, lwp) * w * sizeof(double);
  if (ensure(c, tmp_bytes + wbytes, 0) != BK_OK) return BK_ERR_CUDA;
  double* tmp = reinterpret_cast<double*>(c->dwork);
  double* work = reinterpret_cast<double*>(static_cast<char*>(c->dwork) + tmp_bytes);
  BK_COUNT();
  k_copy_shift<<<grid_for((int64_t)d * d * w), 256, 0, c->st>>>(d, B, ldb, tmp, d, cplx, c->dscal);
  if (!cplx) {
    s = cusolverDnDpotrf(c->h, CUBLAS_FILL_MODE_LOWER, d, tmp, d, work, max(lw, lwp), c->dinfo);
    if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
    s = cusolverDnDsygvd(c->h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d, A, (int)lda,
                         B, (int)ldb, omega, work, max(lw, lwp), c->dinfo + 1);
  } else {
    s = cusolverDnZpotrf(c->h, CUBLAS_FILL_MODE_LOWER, d, reinterpret_cast<cuDoubleComplex*>(tmp), d,
                         reinterpret_cast<cuDoubleComplex*>(work), max(lw, lwp), c->dinfo);
    if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
    s = cusolverDnZhegvd(c->h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, d,
                         reinterpret_cast<cuDoubleComplex*>(A), (int)lda, reinterpret_cast<cuDoubleComplex*>(B),
                         (int)ldb, omega, reinterpret_cast<cuDoubleComplex*>(work), max(lw, lwp), c->dinfo + 1);
  }
  if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  BK_COUNT();
  k_status<<<1, 1, 0, c->st>>>(c->dinfo, c->dinfo + 1, status);
  BK_COUNT();
  k_colmajor_to_rowmajor<<<grid_for((int64_t)d * d), 256, 0, c->st>>>(d, d, A, lda, C, ldc, cplx);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_rr_pencil_d(void* ctx, int d, double* A, int64_t lda, double* B, int64_t ldb, double* omega,
                              double* C, int64_t ldc, int* status) {
  return rr_pencil(static_cast<DenseCtx*>(ctx), d, A, lda, B, ldb, omega, C, ldc, 0, status);
}
extern "C" int bk_rr_pencil_z(void* ctx, int d, double* A, int64_t lda, double* B, int64_t ldb, double* omega,
                              double* C, int64_t ldc, int* status) {
  return rr_pencil(static_cast<DenseCtx*>(ctx), d, A, lda, B, ldb, omega, C, ldc, 1, status);
}

// Q factor of a Householder QR of X (n x m, row-major, ld ldx), written back into X.
// tmp must hold n*m elements (caller-provided, column-major scratch).
__global__ void k_rm_to_cm(int64_t n, int m, const double* X, int64_t ldx, double* T, int cplx) {
  const int64_t tot = n * m;
  const int w = cplx ? 2 : 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / m;
    const int c = (int)(e % m);
    for (int t = 0; t < w; ++t) T[(c * n + r) * w + t] = X[(r * ldx + c) * w + t];
  }
}
__global__ void k_cm_to_rm(int64_t n, int m, const double* T, double* X, int64_t ldx, int cplx) {
  const int64_t tot = n * m;
  const int w = cplx ? 2 : 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / m;
    const int c = (int)(e % m);
    for (int t = 0; t < w; ++t) X[(r * ldx + c) * w + t] = T[(c * n + r) * w + t];
  }
}

static int householder_q(DenseCtx* c, int64_t n, int m, double* X, int64_t ldx, double* tmp, int cplx) {
  if (n > 0x7fffffff || m <= 0 || n < m) return BK_ERR_ARG;
  const int w = cplx ? 2 : 1;
  BK_COUNT();
  k_rm_to_cm<<<4096, 256, 0, c->st>>>(n, m, X, ldx, tmp, cplx);
  int l1 = 0, l2 = 0;
  cusolverStatus_t s;
  const size_t tau_bytes = (((size_t)m * w * sizeof(double)) + 255) & ~(size_t)255;
  if (!cplx) {
    s = cusolverDnDgeqrf_bufferSize(c->h, (int)n, m, tmp, (int)n, &l1);
    if (s == CUSOLVER_STATUS_SUCCESS) s = cusolverDnDorgqr_bufferSize(c->h, (int)n, m, m, tmp, (int)n, nullptr, &l2);
  } else {
    auto t = reinterpret_cast<cuDoubleComplex*>(tmp);
    s = cusolverDnZgeqrf_bufferSize(c->h, (int)n, m, t, (int)n, &l1);
    if (s == CUSOLVER_STATUS_SUCCESS) s = cusolverDnZungqr_bufferSize(c->h, (int)n, m, m, t, (int)n, nullptr, &l2);
  }
  if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  const int lw = max(l1, l2);
  if (ensure(c, tau_bytes + (size_t)lw * w * sizeof(double), 0) != BK_OK) return BK_ERR_CUDA;
  double* tau = reinterpret_cast<double*>(c->dwork);
  double* work = reinterpret_cast<double*>(static_cast<char*>(c->dwork) + tau_bytes);
  if (!cplx) {
    s = cusolverDnDgeqrf(c->h, (int)n, m, tmp, (int)n, tau, work, lw, c->dinfo);
    if (s == CUSOLVER_STATUS_SUCCESS) s = cusolverDnDorgqr(c->h, (int)n, m, m, tmp, (int)n, tau, work, lw, c->dinfo);
  } else {
    auto t = reinterpret_cast<cuDoubleComplex*>(tmp);
    auto tt = reinterpret_cast<cuDoubleComplex*>(tau);
    auto wk = reinterpret_cast<cuDoubleComplex*>(work);
    s = cusolverDnZgeqrf(c->h, (int)n, m, t, (int)n, tt, wk, lw, c->dinfo);
    if (s == CUSOLVER_STATUS_SUCCESS) s = cusolverDnZungqr(c->h, (int)n, m, m, t, (int)n, tt, wk, lw, c->dinfo);
  }
  if (s != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  BK_COUNT();
  k_cm_to_rm<<<4096, 256, 0, c->st>>>(n, m, tmp, X, ldx, cplx);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_householder_q_d(void* ctx, int64_t n, int m, double* X, int64_t ldx, double* tmp) {
  return householder_q(static_cast<DenseCtx*>(ctx), n, m, X, ldx, tmp, 0);
}
extern "C" int bk_householder_q_z(void* ctx, int64_t n, int m, double* X, int64_t ldx, double* tmp) {
  return householder_q(static_cast<DenseCtx*>(ctx), n, m, X, ldx, tmp, 1);
}

// Singular values of a row-major m x n matrix M (ld ldm, scalars of the field) into s
// (min(m, n) device doubles, descending), via gesvd on a column-major copy (m >= n arranged
// by transposing when needed: singular values are transpose-invariant).  Used by the large
// subblock path for the rank test sigma_min(C_X) < 1e-14 max(||C||_2, 1) (ppcg.py:351-356).
namespace bk {
__global__ void k_to_colmajor(int rows, int cols, const double* M, int64_t ldm, int trans, double* T, int cplx) {
  // trans == 0: T (rows x cols, col-major, ld rows) = M;  trans == 1: T (cols x rows) = M^T
  const int64_t tot = (int64_t)rows * cols;
  const int w = cplx ? 2 : 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e % cols);
    const int64_t dst = trans ? ((int64_t)i * cols + j) : ((int64_t)j * rows + i);
    for (int t = 0; t < w; ++t) T[dst * w + t] = M[(i * ldm + j) * w + t];
  }
}
}  // namespace bk

static int svals(DenseCtx* c, int m, int n, const double* M, int64_t ldm, double* s, int cplx) {
  if (m <= 0 || n <= 0) return BK_ERR_ARG;
  const int w = cplx ? 2 : 1;
  const int trans = m < n ? 1 : 0;
  const int mm = trans ? n : m, nn = trans ? m : n;  // column-major mm x nn with mm >= nn
  int lw = 0;
  cusolverStatus_t st = cplx ? cusolverDnZgesvd_bufferSize(c->h, mm, nn, &lw) : cusolverDnDgesvd_bufferSize(c->h, mm, nn, &lw);
  if (st != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  const size_t abytes = (((size_t)mm * nn * w * sizeof(double)) + 255) & ~(size_t)255;
  const size_t rbytes = (((size_t)nn * 5 * sizeof(double)) + 255) & ~(size_t)255;
  if (ensure(c, abytes + rbytes + (size_t)lw * w * sizeof(double), 0) != BK_OK) return BK_ERR_CUDA;
  double* T = reinterpret_cast<double*>(c->dwork);
  double* rwork = reinterpret_cast<double*>(static_cast<char*>(c->dwork) + abytes);
  double* work = reinterpret_cast<double*>(static_cast<char*>(c->dwork) + abytes + rbytes);
  BK_COUNT();
  k_to_colmajor<<<grid_for((int64_t)m * n), 256, 0, c->st>>>(m, n, M, ldm, trans, T, cplx);
  if (!cplx) {
    st = cusolverDnDgesvd(c->h, 'N', 'N', mm, nn, T, mm, s, nullptr, 1, nullptr, 1, work, lw, rwork, c->dinfo);
  } else {
    st = cusolverDnZgesvd(c->h, 'N', 'N', mm, nn, reinterpret_cast<cuDoubleComplex*>(T), mm, s, nullptr, 1, nullptr,
                          1, reinterpret_cast<cuDoubleComplex*>(work), lw, rwork, c->dinfo);
  }
  if (st != CUSOLVER_STATUS_SUCCESS) return BK_ERR_SOLVER;
  BK_CHECK_LAUNCH();
  return BK_OK;
}

extern "C" int bk_svals_d(void* ctx, int m, int n, const double* M, int64_t ldm, double* s) {
  return svals(static_cast<DenseCtx*>(ctx), m, n, M, ldm, s, 0);
}
extern "C" int bk_svals_z(void* ctx, int m, int n, const double* M, int64_t ldm, double* s) {
  return svals(static_cast<DenseCtx*>(ctx), m, n, M, ldm, s, 1);
}
