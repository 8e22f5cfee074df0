// Batched projected eigenproblems of the PPCG subblock update, one CTA per subblock.
//
// Replaces, per subblock j, the host logic of block_update (blockeig ppcg.py:278-378)
// from the raw Grams onwards, including
//   * the direction-drop test and unit scaling     ppcg.py:198-203, 220-228, 296-299
//   * SmallPencil symmetrisation                    core.py:143-164
//   * solve_pencil: singular-Gram test (Cholesky of B - 1e-12||B||_F I) and the dense
//     generalized eigensolve (LAPACK sygvd: potrf, reduce, eig)   core.py:175-202
//   * the SingularGramError retry ladder (drop P, shed weakest W)  ppcg.py:332-349
//   * the sigma_min(C_X) rank test and fallback_steepest_descent   ppcg.py:351-356, 231-275
//   * coefficient un-scaling and coeff_scale                       ppcg.py:358-363, 376
// The dense eigensolve is Cholesky reduction C = L^{-1} A L^{-T} followed by a two-sided
// parallel cyclic Jacobi (round-robin ordering, d/2 disjoint rotations per round) with the
// whole working set in shared memory.  Singular values for the rank test come from
// one-sided (Hestenes) Jacobi.  No host round trip: every branch of the reference's retry
// logic runs on the device and only counters/flags are returned.
//
// Mode 1 ("raw") solves one plain pencil per CTA: solve_pencil(SmallPencil(A, B), want).
#include <cfloat>
#include "common.cuh"

namespace bk {

constexpr int PD = 96;            // max pencil dimension of the shared-memory path
constexpr int PLD = PD + 1;       // odd leading dimension: conflict-free column access
constexpr int P_THREADS = 512;
constexpr double kGramRtol = 1e-12, kDirFloor = 1e-14, kCxFloor = 1e-14;

struct PencilParams {
  int nb;
  int k_act, q, has_p, dmax;
  const double* Araw;  // nb x dmax x dmax
  const double* Braw;
  double* coef;        // nb x (dmax x q): block j rows [part*w + i], ld = w
  double* theta;       // k_act (block mode) / nb x want (raw mode)
  int* info;           // nb x 4: fallback, zero_residual, error, attempts
  double* cscale;      // nb
  int mode;            // 0 = block_update, 1 = raw pencil
  int want;            // raw mode
  int rawd;            // raw mode pencil dimension
  int force_fallback;  // 1: fallback_steepest_descent directly (ppcg.py:456-472 redo)
};

struct PSmem {
  double* M0;  // PD x PLD : A (reduced), later temps
  double* M1;  // PD x PLD : B -> L -> T -> V
  double* M2;  // PD x PLD : Linv
  double* nrm;   // PD column norms of [X|W|P]
  double* sf;    // PD scale factor of the assembled basis (1 or 1/norm)
  double* ev;    // PD eigenvalues
  double* rc;    // PD/2 rotation c
  double* rs;    // PD/2 rotation s
  double* red;   // 32 reduction slots
  int* idx;      // PD assembled basis -> raw column
  int* ord;      // PD eigen order
  int* pp;       // PD/2
  int* pq;       // PD/2
  int* misc;     // 8 ints: [0] flag, [1] rotation count
};

// ---------------------------------------------------------------- block reductions
BK_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    red[31] = t;
  }
  __syncthreads();
  return red[31];
}
BK_DEV double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) t = fmax(t, red[i]);
    red[31] = t;
  }
  __syncthreads();
  return red[31];
}

// ---------------------------------------------------------------- in-place lower Cholesky
// Returns true on success (all pivots > 0 and finite), like LAPACK potrf.
// Work is mapped 2-D without integer division: warps over rows, lanes over columns.
#define BK_WARP (threadIdx.x >> 5)
#define BK_LANE (threadIdx.x & 31)
#define BK_NWARP (blockDim.x >> 5)

BK_DEV bool smem_cholesky(double* M, int ld, int d, int* flag) {
  // right-looking, one column per step; the pivot test is uniform (all threads read the
  // same shared value after the barrier)
  for (int j = 0; j < d; ++j) {
    __syncthreads();
    const double piv = M[j * ld + j];
    if (!(piv > 0.0) || !isfinite(piv)) return false;
    const double ljj = sqrt(piv);
    const double inv = 1.0 / ljj;
    // trailing update of rows i > j uses the scaled column: l_ij = a_ij / ljj
    for (int i = j + 1 + BK_WARP; i < d; i += BK_NWARP) {
      const double lij = M[i * ld + j] * inv;
      for (int k = j + 1 + BK_LANE; k <= i; k += 32) M[i * ld + k] = fma(-lij, M[k * ld + j] * inv, M[i * ld + k]);
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < d; i += blockDim.x) M[i * ld + j] *= inv;
    if (threadIdx.x == 0) M[j * ld + j] = ljj;
  }
  __syncthreads();
  return true;
}

// Linv (lower, ld li) from L (lower, ld ll): right-looking column sweep
//   X = I; for j: X[j,:] /= l_jj; X[i,:] -= l_ij X[j,:] (i > j)
BK_DEV void smem_lower_inverse(const double* L, int ll, double* Li, int li, int d) {
  for (int i = BK_WARP; i < d; i += BK_NWARP)
    for (int c = BK_LANE; c < d; c += 32) Li[i * li + c] = (i == c) ? 1.0 / L[i * ll + i] : 0.0;
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    // row j of X is final (already divided by l_jj); eliminate below
    for (int i = j + 1 + BK_WARP; i < d; i += BK_NWARP) {
      const double f = L[i * ll + j] / L[i * ll + i];
      for (int c = BK_LANE; c <= j; c += 32) Li[i * li + c] = fma(-f, Li[j * li + c], Li[i * li + c]);
    }
    __syncthreads();
  }
}

// C (d x d, ldc) = op(A) * op(B) over shared memory, 6x3 register block per thread for
// d <= 96 (warps -> rows w, w+16, ...; lanes -> cols l, l+32, l+64).
//   tb = false: C[i][j] = sum_k A[i][k] B[k][j]
//   tb = true : C[i][j] = sum_k A[i][k] B[j][k]
template <bool TA, bool TB>
BK_DEV void smem_gemm(const double* A, int la, const double* B, int lb, double* C, int lc, int d, int kmax,
                      int ncols = -1) {
  constexpr int RI = 6, RJ = 3;
  const int nc = ncols < 0 ? d : ncols;
  for (int i0 = BK_WARP; i0 < d; i0 += BK_NWARP * RI) {
    double acc[RI][RJ];
#pragma unroll
    for (int a = 0; a < RI; ++a)
#pragma unroll
      for (int b = 0; b < RJ; ++b) acc[a][b] = 0.0;
    for (int k = 0; k < kmax; ++k) {
      double av[RI], bv[RJ];
#pragma unroll
      for (int a = 0; a < RI; ++a) {
        const int i = i0 + a * BK_NWARP;
        av[a] = i < d ? (TA ? A[k * la + i] : A[i * la + k]) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < RJ; ++b) {
        const int j = BK_LANE + 32 * b;
        bv[b] = j < nc ? (TB ? B[j * lb + k] : B[k * lb + j]) : 0.0;
      }
#pragma unroll
      for (int a = 0; a < RI; ++a)
#pragma unroll
        for (int b = 0; b < RJ; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < RI; ++a) {
      const int i = i0 + a * BK_NWARP;
#pragma unroll
      for (int b = 0; b < RJ; ++b) {
        const int j = BK_LANE + 32 * b;
        if (i < d && j < nc) C[i * lc + j] = acc[a][b];
      }
    }
  }
}

// ---------------------------------------------------------------- parallel cyclic Jacobi
BK_DEV void rr_pair(int r, int i, int dd, int& p, int& q) {
  const int np = dd - 1;  // circle players 0..np-1, fixed player np
  int a, b;
  if (i == 0) { a = r; b = np; }
  else { a = (r + i) % np; b = (r - i + np) % np; }
  p = min(a, b);
  q = max(a, b);
}

// Diagonalises symmetric A (d x d, ld la) in place; accumulates V (ld lv) if withV.
// Returns the number of sweeps.
BK_DEV int smem_jacobi(double* A, int la, double* V, int lv, int d, bool withV, PSmem& S) {
  if (withV) {
    for (int i = BK_WARP; i < d; i += BK_NWARP)
      for (int c = BK_LANE; c < d; c += 32) V[i * lv + c] = (i == c) ? 1.0 : 0.0;
  }
  if (d == 1) { __syncthreads(); return 0; }
  {
    double f = 0.0;
    for (int i = BK_WARP; i < d; i += BK_NWARP)
      for (int c = BK_LANE; c < d; c += 32) {
        const double v = A[i * la + c];
        f = fma(v, v, f);
      }
    f = sqrt(block_sum(f, S.red));
    if (threadIdx.x == 0) S.red[30] = 0.5 * DBL_EPSILON * f / (double)d;
    __syncthreads();
  }
  const int dd = d + (d & 1);
  const int npairs = dd / 2;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) S.misc[1] = 0;
    __syncthreads();
    for (int r = 0; r < dd - 1; ++r) {
      // 1. rotation parameters
      for (int i = threadIdx.x; i < npairs; i += blockDim.x) {
        int p, q;
        rr_pair(r, i, dd, p, q);
        double c = 1.0, s = 0.0;
        if (q < d) {
          const double apq = A[p * la + q];
          const double app = A[p * la + p], aqq = A[q * la + q];
          // rotate unless |a_pq| is below both the relative (Demmel-Veselic) and the
          // absolute eps*||A||_F/d floor: an entry that small moves eigenvalues by less than
          // the rounding already in the diagonal (avoids endless sweeps on noise when a
          // diagonal entry is ~0)
          if (apq != 0.0 && fabs(apq) > DBL_EPSILON * 0.5 * sqrt(fabs(app) * fabs(aqq)) &&
              fabs(apq) > S.red[30]) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            atomicAdd(&S.misc[1], 1);
          }
        }
        S.pp[i] = p;
        S.pq[i] = q;
        S.rc[i] = c;
        S.rs[i] = s;
      }
      __syncthreads();
      // 2. row rotations  A <- J^T A   (warp per pair, lanes over columns: stride-1 rows)
      for (int i = BK_WARP; i < npairs; i += BK_NWARP) {
        const double s = S.rs[i];
        if (s == 0.0) continue;  // warp-uniform
        const double c = S.rc[i];
        double* ap_ = A + S.pp[i] * la;
        double* aq_ = A + S.pq[i] * la;
        for (int j = BK_LANE; j < d; j += 32) {
          const double ap = ap_[j], aq = aq_[j];
          ap_[j] = c * ap - s * aq;
          aq_[j] = s * ap + c * aq;
        }
      }
      __syncthreads();
      // 3. column rotations  A <- A J, V <- V J (lanes over rows: odd stride, conflict-free);
      //    the annihilated pair is set to exact zero
      for (int i = BK_WARP; i < npairs; i += BK_NWARP) {
        const double s = S.rs[i];
        if (s == 0.0) continue;
        const double c = S.rc[i];
        const int p = S.pp[i], q = S.pq[i];
        for (int row = BK_LANE; row < d; row += 32) {
          const double ap = A[row * la + p], aq = A[row * la + q];
          double np_ = c * ap - s * aq, nq = s * ap + c * aq;
          if (row == p) nq = 0.0;
          if (row == q) np_ = 0.0;
          A[row * la + p] = np_;
          A[row * la + q] = nq;
          if (withV) {
            const double vp = V[row * lv + p], vq = V[row * lv + q];
            V[row * lv + p] = c * vp - s * vq;
            V[row * lv + q] = s * vp + c * vq;
          }
        }
      }
      __syncthreads();
    }
    if (S.misc[1] == 0) break;
    __syncthreads();
  }
  __syncthreads();
  return sweep;
}

// One-sided Jacobi on M (rows x cols, ld lm), in place; returns singular values in sv[0:cols]
BK_DEV void smem_svals(double* M, int lm, int rows, int cols, double* sv, PSmem& S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (cols > 1) {
    const int dd = cols + (cols & 1), npairs = dd / 2;
    for (int sweep = 0; sweep < 60; ++sweep) {
      if (threadIdx.x == 0) S.misc[1] = 0;
      __syncthreads();
      for (int r = 0; r < dd - 1; ++r) {
        for (int i = warp; i < npairs; i += nw) {
          int p, q;
          rr_pair(r, i, dd, p, q);
          if (q >= cols) continue;
          double a = 0.0, b = 0.0, g = 0.0;
          for (int k = lane; k < rows; k += 32) {
            const double x = M[k * lm + p], y = M[k * lm + q];
            a = fma(x, x, a);
            b = fma(y, y, b);
            g = fma(x, y, g);
          }
          a = warp_sum(a);
          b = warp_sum(b);
          g = warp_sum(g);
          if (g == 0.0 || fabs(g) <= DBL_EPSILON * sqrt(a * b)) continue;
          const double zeta = (b - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int k = lane; k < rows; k += 32) {
            const double x = M[k * lm + p], y = M[k * lm + q];
            M[k * lm + p] = c * x - s * y;
            M[k * lm + q] = s * x + c * y;
          }
          if (lane == 0) atomicAdd(&S.misc[1], 1);
        }
        __syncthreads();
      }
      if (S.misc[1] == 0) break;
      __syncthreads();
    }
  }
  __syncthreads();
  for (int j = warp; j < cols; j += nw) {
    double a = 0.0;
    for (int k = lane; k < rows; k += 32) a = fma(M[k * lm + j], M[k * lm + j], a);
    a = warp_sum(a);
    if (lane == 0) sv[j] = sqrt(a);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- one pencil attempt
// Assembled basis: idx[0:d] raw columns, sf[0:d] scale factors.  Raw Grams at (Ar, Br, ldr).
// On success: ev[0:want] ascending eigenvalues (ord applied), C (d x want) in M1 (ld PLD).
// Returns 0 ok, 1 singular (either Cholesky failed).
BK_DEV int pencil_attempt(const double* Ar, const double* Br, int ldr, int d, int want, PSmem& S) {
  double* A = S.M0;
  double* B = S.M1;
  double* Li = S.M2;
  // assemble symmetrised, scaled B and its Frobenius norm
  double fro = 0.0;
  for (int a = BK_WARP; a < d; a += BK_NWARP) {
    const int ia = S.idx[a];
    const double sa = S.sf[a];
    for (int b = BK_LANE; b < d; b += 32) {
      const int ib = S.idx[b];
      const double v = 0.5 * (Br[ia * ldr + ib] + Br[ib * ldr + ia]) * sa * S.sf[b];
      B[a * PLD + b] = v;
      fro = fma(v, v, fro);
    }
  }
  fro = sqrt(block_sum(fro, S.red));
  const double flo = kGramRtol * fmax(fro, 1e-300);
  for (int a = threadIdx.x; a < d; a += blockDim.x) B[a * PLD + a] -= flo;
  __syncthreads();
  if (!smem_cholesky(B, PLD, d, S.misc)) return 1;  // core.py:193-197
  // reload B (exact) and factor it for the reduction (sygvd's potrf)
  for (int a = BK_WARP; a < d; a += BK_NWARP) {
    const int ia = S.idx[a];
    const double sa = S.sf[a];
    for (int b = BK_LANE; b < d; b += 32) {
      const int ib = S.idx[b];
      const double sab = sa * S.sf[b];
      B[a * PLD + b] = 0.5 * (Br[ia * ldr + ib] + Br[ib * ldr + ia]) * sab;
      A[a * PLD + b] = 0.5 * (Ar[ia * ldr + ib] + Ar[ib * ldr + ia]) * sab;
    }
  }
  __syncthreads();
  if (!smem_cholesky(B, PLD, d, S.misc)) return 1;  // core.py:198-201
  smem_lower_inverse(B, PLD, Li, PLD, d);
  smem_gemm<false, false>(Li, PLD, A, PLD, B, PLD, d, d);  // T = Linv A -> B (L no longer needed)
  __syncthreads();
  smem_gemm<false, true>(B, PLD, Li, PLD, A, PLD, d, d);   // Ared = T Linv^T -> A
  __syncthreads();
  // symmetrise (the reduced matrix is symmetric in exact arithmetic)
  for (int i = BK_WARP; i < d; i += BK_NWARP)
    for (int j = i + 1 + BK_LANE; j < d; j += 32) {
      const double v = 0.5 * (A[i * PLD + j] + A[j * PLD + i]);
      A[i * PLD + j] = v;
      A[j * PLD + i] = v;
    }
  __syncthreads();
  smem_jacobi(A, PLD, B, PLD, d, true, S);  // V in B
  for (int i = threadIdx.x; i < d; i += blockDim.x) S.ev[i] = A[i * PLD + i];
  __syncthreads();
  // ascending order (ties by index)
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const double v = S.ev[i];
    int rank = 0;
    for (int j = 0; j < d; ++j) {
      const double u = S.ev[j];
      rank += (u < v) || (u == v && j < i);
    }
    S.ord[rank] = i;
  }
  __syncthreads();
  // gather V[:, ord[0:want]] -> A, then C = Linv^T Vsel -> B (ld PLD)
  for (int k = BK_WARP; k < d; k += BK_NWARP)
    for (int r = BK_LANE; r < want; r += 32) A[k * PLD + r] = B[k * PLD + S.ord[r]];
  __syncthreads();
  smem_gemm<true, false>(Li, PLD, A, PLD, B, PLD, d, d, want);
  // sorted eigenvalues
  for (int r = threadIdx.x; r < want; r += blockDim.x) A[PD * PLD - 1 - r] = S.ev[S.ord[r]];
  __syncthreads();
  for (int r = threadIdx.x; r < want; r += blockDim.x) S.ev[r] = A[PD * PLD - 1 - r];
  __syncthreads();
  return 0;
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(P_THREADS, 1) pencil_kernel(const __grid_constant__ PencilParams P) {
  extern __shared__ __align__(16) double sm[];
  PSmem S;
  S.M0 = sm;
  S.M1 = S.M0 + PD * PLD;
  S.M2 = S.M1 + PD * PLD;
  S.nrm = S.M2 + PD * PLD;
  S.sf = S.nrm + PD;
  S.ev = S.sf + PD;
  S.rc = S.ev + PD;
  S.rs = S.rc + PD / 2;
  S.red = S.rs + PD / 2;
  S.idx = reinterpret_cast<int*>(S.red + 32);
  S.ord = S.idx + PD;
  S.pp = S.ord + PD;
  S.pq = S.pp + PD / 2;
  S.misc = S.pq + PD / 2;

  const int j = blockIdx.x;
  const int tid = threadIdx.x;
  const double* Ar = P.Araw + (int64_t)j * P.dmax * P.dmax;
  const double* Br = P.Braw + (int64_t)j * P.dmax * P.dmax;
  const int ldr = P.dmax;

  if (P.mode == 1) {  // plain solve_pencil(SmallPencil(A, B), want)
    const int d = P.rawd;
    for (int i = tid; i < d; i += blockDim.x) { S.idx[i] = i; S.sf[i] = 1.0; }
    __syncthreads();
    const int st = pencil_attempt(Ar, Br, ldr, d, P.want, S);
    double* cout = P.coef + (int64_t)j * P.dmax * P.want;
    if (st == 0) {
      for (int e = tid; e < d * P.want; e += blockDim.x) cout[e] = S.M1[(e / P.want) * PLD + e % P.want];
      for (int r = tid; r < P.want; r += blockDim.x) P.theta[(int64_t)j * P.want + r] = S.ev[r];
    }
    if (tid == 0) { P.info[4 * j + 2] = st; P.info[4 * j + 0] = 0; P.info[4 * j + 1] = 0; P.info[4 * j + 3] = 1; }
    return;
  }

  const int lo = j * P.q;
  const int w = min(P.q, P.k_act - lo);
  const int nparts = P.has_p ? 3 : 2;
  const int d0 = nparts * w;
  double* cout = P.coef + (int64_t)j * P.dmax * P.q;  // rows part*w + i, ld w

  // column norms of the raw basis from the Gram diagonal (ppcg.py:202, 226)
  for (int i = tid; i < d0; i += blockDim.x) S.nrm[i] = sqrt(fmax(Br[i * ldr + i], 0.0));
  __syncthreads();
  double sc = 0.0;
  for (int i = 0; i < w; ++i) sc = fmax(sc, S.nrm[i]);
  sc = fmax(sc, 1e-300);
  const double floor_ = kDirFloor * sc;  // ppcg.py:198-203

  // kept masks as bit sets (w <= 32 -> fits 64-bit masks for 3 parts)
  unsigned long long keptw = 0ull, keptp = 0ull;
  for (int i = 0; i < w; ++i) {
    if (S.nrm[w + i] > floor_) keptw |= 1ull << i;
    if (P.has_p && S.nrm[2 * w + i] > floor_) keptp |= 1ull << i;
  }

  int fallback = 0, zero_res = 0, err = 0, attempts = 0;
  double cmax = 1.0;
  int status = 0;
  int nw_used = 0, np_used = 0;

  auto assemble = [&](unsigned long long mw, unsigned long long mp) -> int {
    // basis order: X (all), kept W, kept P (ppcg.py:312-330)
    int d = 0;
    if (tid == 0) {
      for (int i = 0; i < w; ++i) { S.idx[d] = i; S.sf[d] = 1.0; ++d; }
      for (int i = 0; i < w; ++i)
        if (mw >> i & 1ull) { S.idx[d] = w + i; S.sf[d] = 1.0 / S.nrm[w + i]; ++d; }
      for (int i = 0; i < w; ++i)
        if (mp >> i & 1ull) { S.idx[d] = 2 * w + i; S.sf[d] = 1.0 / S.nrm[2 * w + i]; ++d; }
      S.misc[0] = d;
    }
    __syncthreads();
    d = S.misc[0];
    __syncthreads();
    return d;
  };

  auto write_passthrough = [&](bool fb) {
    // x unchanged, p = 0, theta = Rayleigh quotients (ppcg.py:300-310, 255-265)
    for (int e = tid; e < nparts * w * w; e += blockDim.x) {
      const int r = e / w, c = e % w;
      cout[e] = (r < w && r == c) ? 1.0 : 0.0;
    }
    for (int i = tid; i < w; i += blockDim.x) P.theta[lo + i] = Ar[i * ldr + i] / Br[i * ldr + i];
    fallback = fb;
    zero_res = 1;
    cmax = 1.0;
  };

  if (!P.force_fallback && keptw == 0ull && keptp == 0ull) {
    write_passthrough(false);
  } else {
    unsigned long long mw = keptw, mp = keptp;
    int d = 0;
    bool do_fallback = P.force_fallback != 0;
    if (!do_fallback) {
    d = assemble(mw, mp);
    status = pencil_attempt(Ar, Br, ldr, d, w, S);
    ++attempts;
    if (status != 0) {
      mp = 0ull;  // drop P first, then shed the weakest W column (ppcg.py:335-349)
      while (true) {
        d = assemble(mw, mp);
        status = pencil_attempt(Ar, Br, ldr, d, w, S);
        ++attempts;
        if (status == 0) break;
        if (mw == 0ull) { err = 1; break; }
        int worst = -1;
        double wv = 0.0;
        for (int i = 0; i < w; ++i)
          if ((mw >> i & 1ull) && (worst < 0 || S.nrm[w + i] < wv)) { worst = i; wv = S.nrm[w + i]; }
        mw &= ~(1ull << worst);
      }
    }
    if (!err) {
      nw_used = __popcll(mw);
      np_used = __popcll(mp);
      // rank test: sigma_min(C_X) < 1e-14 max(||C||_2, 1)  (ppcg.py:351-356)
      double* T1 = S.M2;                 // C copy (d x w, ld w)  -- Linv no longer needed
      double* T2 = S.M0;                 // C_X copy (w x w, ld w); C itself stays in M1
      for (int e = tid; e < d * w; e += blockDim.x) T1[e] = S.M1[(e / w) * PLD + e % w];
      for (int e = tid; e < w * w; e += blockDim.x) T2[e] = S.M1[(e / w) * PLD + e % w];
      __syncthreads();
      smem_svals(T1, w, d, w, S.rc, S);
      double cn = 0.0;
      for (int i = 0; i < w; ++i) cn = fmax(cn, S.rc[i]);
      __syncthreads();
      smem_svals(T2, w, w, w, S.rc, S);
      double smin = S.rc[0];
      for (int i = 1; i < w; ++i) smin = fmin(smin, S.rc[i]);
      __syncthreads();
      if (smin < kCxFloor * fmax(cn, 1.0)) do_fallback = true;
    }
    }  // !force_fallback
    if (do_fallback) {
      // fallback_steepest_descent: pencil over [X, kept W] (ppcg.py:231-275), no retries
      fallback = 1;
      mw = keptw;
      mp = 0ull;
      if (mw == 0ull) {
        write_passthrough(true);
      } else {
        d = assemble(mw, mp);
        status = pencil_attempt(Ar, Br, ldr, d, w, S);
        ++attempts;
        if (status != 0) err = 1;
        nw_used = __popcll(mw);
        np_used = 0;
      }
    }
    if (!err && !(fallback && zero_res)) {
      // coefficients: X rows direct, W/P rows un-scaled onto original columns (ppcg.py:358-363)
      double m = 0.0;
      for (int e = tid; e < d * w; e += blockDim.x) m = fmax(m, fabs(S.M1[(e / w) * PLD + e % w]));
      cmax = block_max(m, S.red);
      for (int e = tid; e < nparts * w * w; e += blockDim.x) cout[e] = 0.0;
      __syncthreads();
      for (int e = tid; e < d * w; e += blockDim.x) {
        const int a = e / w, c = e % w;
        const int raw = S.idx[a];
        cout[raw * w + c] = S.M1[a * PLD + c] * S.sf[a];
      }
      for (int i = tid; i < w; i += blockDim.x) P.theta[lo + i] = S.ev[i];
    }
  }
  __syncthreads();
  if (tid == 0) {
    P.info[4 * j + 0] = fallback;
    P.info[4 * j + 1] = zero_res;
    P.info[4 * j + 2] = err;
    P.info[4 * j + 3] = attempts;
    P.cscale[j] = cmax;
  }
}

static int p_smem_bytes() {
  return (3 * PD * PLD + 3 * PD + PD + 32) * (int)sizeof(double) + (2 * PD + PD + 8) * (int)sizeof(int);
}

}  // namespace bk

using namespace bk;

extern "C" int bk_pencil_max_dim(void) { return PD; }

// Device-side block_update for every subblock (see file header).  Araw/Braw from
// bk_subblock_grams_d.  coef: nb x (dmax x q) doubles; theta: k_act; info: nb x 4 ints
// (used_fallback, zero_residual, error, attempts); cscale: nb doubles.
extern "C" int bk_subblock_pencils_d(int k_act, int q, int has_p, const double* Araw, const double* Braw,
                                     double* coef, double* theta, int* info, double* cscale, int force_fallback,
                                     void* stream) {
  if (k_act <= 0 || q <= 0) return BK_ERR_ARG;
  const int dmax = (has_p ? 3 : 2) * q;
  if (dmax > PD || q > 32) return BK_ERR_UNSUPPORTED;
  PencilParams P{};
  P.nb = (k_act + q - 1) / q;
  P.k_act = k_act;
  P.q = q;
  P.has_p = has_p ? 1 : 0;
  P.dmax = dmax;
  P.Araw = Araw;
  P.Braw = Braw;
  P.coef = coef;
  P.theta = theta;
  P.info = info;
  P.cscale = cscale;
  P.mode = 0;
  P.force_fallback = force_fallback ? 1 : 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pencil_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p_smem_bytes());
    attr = true;
  }
  BK_COUNT();
  pencil_kernel<<<P.nb, P_THREADS, p_smem_bytes(), (cudaStream_t)stream>>>(P);
  BK_CHECK_LAUNCH();
  return BK_OK;
}

// Batched plain pencils: nb problems of dimension d (stride ldm*ldm, ld ldm), want smallest
// pairs.  omega: nb x want; C: nb x (ldm x want) (ld want); status: nb x 4 ints ([2] = 1 if
// singular).  (core.py:175-202)
extern "C" int bk_pencil_batched_d(int nb, int d, int ldm, const double* A, const double* B, int want,
                                   double* omega, double* C, int* status, void* stream) {
  if (nb <= 0 || d <= 0 || want < 1 || want > d || ldm < d) return BK_ERR_ARG;
  if (d > PD) return BK_ERR_UNSUPPORTED;
  PencilParams P{};
  P.nb = nb;
  P.dmax = ldm;
  P.Araw = A;
  P.Braw = B;
  P.coef = C;
  P.theta = omega;
  P.info = status;
  P.mode = 1;
  P.want = want;
  P.rawd = d;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pencil_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p_smem_bytes());
    attr = true;
  }
  BK_COUNT();
  pencil_kernel<<<nb, P_THREADS, p_smem_bytes(), (cudaStream_t)stream>>>(P);
  BK_CHECK_LAUNCH();
  return BK_OK;
}
