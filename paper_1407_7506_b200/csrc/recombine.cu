// Batched subblock recombination on FP64 tensor cores (DMMA).
//
// Replaces the per-subblock products of block_update and _run_subblocks:
//   P_j' = W_j C_W + P_j C_P,  X_j' = X_j C_X + P_j'           (ppcg.py:365-369)
//   AP_j' = AW_j C_W + AP_j C_P, AX_j' = AX_j C_X + AP_j'      (ppcg.py:521-532)
// for every subblock j in one launch (grid: row tiles x blocks x {X side, A side}),
// writing into separate output buffers so the pre-update blocks survive for the
// breakdown and rank-deficiency recovery paths (ppcg.py:694, 698-717, 456-472).
// The breakdown test of ppcg.py:701-705 (non-finite entries in X, P, AX, AP; max|X|,
// max|P| > 1e8) is fused into the epilogue as device-wide flags.
#include "common.cuh"

namespace bk {

constexpr int R_BM = 64, R_THREADS = 128;  // 4 warps x 16 rows
constexpr int R_QMAX = 64;

struct RecombParams {
  int64_t n;
  int k_act, q, has_p;
  int64_t ld, c0;      // shared by all state blocks
  int dmax;
  const double* coef;  // nb x (dmax x q), block rows part*w + i, ld w
  const double* in[2][3];   // side -> {X, W, P} / {AX, AW, AP}
  double* outX[2];          // side -> X' / AX'
  double* outP[2];          // side -> P' / AP'
  unsigned long long* flags;  // [0] nonfinite (0/1), [1] max|X'| bits, [2] max|P'| bits
  int cplx;                   // real view of complex data: columns pair up as (re, im)
};

// complex coefficients (block j: nparts*w x w, ld w, stride dmax*q) -> real expanded
// (2 nparts w x 2w, ld 2w, stride (2 dmax)(2 q)) so the real kernel applies X C on views
__global__ void k_expand_coef(int k_act, int q, int nparts, const double* __restrict__ cz, double* __restrict__ cr) {
  const int j = blockIdx.y;
  const int w = min(q, k_act - j * q);
  const int dmax = nparts * q;
  const double* src = cz + (int64_t)j * dmax * q * 2;
  double* dst = cr + (int64_t)j * (2 * dmax) * (2 * q);
  const int rows = nparts * w;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * w; e += gridDim.x * blockDim.x) {
    const int i = e / w, c = e % w;
    const double gr = src[2 * (i * w + c)], gi = src[2 * (i * w + c) + 1];
    const int ld = 2 * w;
    dst[(2 * i) * ld + 2 * c] = gr;
    dst[(2 * i) * ld + 2 * c + 1] = gi;
    dst[(2 * i + 1) * ld + 2 * c] = -gi;
    dst[(2 * i + 1) * ld + 2 * c + 1] = gr;
  }
}

BK_DEV int pad_a(int w) { int l = (w + 3) & ~3; if ((l & 7) == 0) l += 4; return l; }   // l % 8 == 4
BK_DEV int pad_b(int w) { int l = (w + 7) & ~7; return l + 4; }  // l % 8 == 4: 4 rows -> 4 disjoint 8-bank groups

__global__ void __launch_bounds__(R_THREADS) recombine_kernel(const __grid_constant__ RecombParams P) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = blockIdx.y, side = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.x * R_BM;
  const int lo = j * P.q;
  const int w = min(P.q, P.k_act - lo);
  const int nparts = P.has_p ? 3 : 2;
  const int la = pad_a(w), lb = pad_b(w);
  double* In = sm;                                  // [part][R_BM][la]
  double* Cf = sm + 3 * R_BM * la;                  // [nparts*w][lb]
  const double* cg = P.coef + (int64_t)j * P.dmax * P.q;

  // stage inputs (rows r0..r0+63, cols c0+lo .. +w of each part) and coefficients
  for (int part = 0; part < nparts; ++part) {
    const double* src = P.in[side][part];
    for (int e = tid; e < R_BM * w; e += R_THREADS) {
      const int r = e / w, c = e % w;
      const int64_t row = r0 + r;
      const bool v = row < P.n;
      cp_async8(In + (part * R_BM + r) * la + c, v ? src + row * P.ld + P.c0 + lo + c : src, v);
    }
  }
  for (int e = tid; e < nparts * w * w; e += R_THREADS) {
    const int r = e / w, c = e % w;
    cp_async8(Cf + r * lb + c, cg + e, true);
  }
  cp_async_commit();
  // zero the MMA padding: columns w..(w rounded to 8) of inputs and coefficient rows
  const int w8 = (w + 7) & ~7, k4 = (w + 3) & ~3;
  for (int e = tid; e < nparts * R_BM * (k4 - w); e += R_THREADS) {
    const int part = e / (R_BM * (k4 - w)), rem = e % (R_BM * (k4 - w));
    In[(part * R_BM + rem / (k4 - w)) * la + w + rem % (k4 - w)] = 0.0;
  }
  for (int e = tid; e < nparts * w * (w8 - w); e += R_THREADS) Cf[(e / (w8 - w)) * lb + w + e % (w8 - w)] = 0.0;
  cp_async_wait<0>();
  __syncthreads();

  // warp: rows warp*16 .. +16 (2 MMA rows), cols 0..w8 (<= 8 MMA cols)
  double accX[2][R_QMAX / 8][2], accP[2][R_QMAX / 8][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < R_QMAX / 8; ++b) accX[a][b][0] = accX[a][b][1] = accP[a][b][0] = accP[a][b][1] = 0.0;
  const int ntv = w8 / 8;
  const int fk = lane & 3, fm = lane >> 2;
  for (int part = 0; part < nparts; ++part) {
    const double* ia = In + part * R_BM * la;
    for (int kk = 0; kk < k4; kk += 4) {
      double af[2], bf[R_QMAX / 8];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = ia[(warp * 16 + a * 8 + fm) * la + kk + fk];
      const int crow = part * w + kk + fk;
      const bool kv = kk + fk < w;
#pragma unroll
      for (int b = 0; b < R_QMAX / 8; ++b)
        if (b < ntv) bf[b] = kv ? Cf[crow * lb + b * 8 + fm] : 0.0;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < R_QMAX / 8; ++b)
          if (b < ntv) {
            if (part == 0) dmma_8x8x4(accX[a][b][0], accX[a][b][1], af[a], bf[b]);
            else dmma_8x8x4(accP[a][b][0], accP[a][b][1], af[a], bf[b]);
          }
    }
  }

  // epilogue: P' = accP, X' = accX + accP; breakdown statistics
  bool nonfin = false;
  double mx = 0.0, mp = 0.0;
  double* ox = P.outX[side];
  double* op = P.outP[side];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int64_t row = r0 + warp * 16 + a * 8 + fm;
    if (row >= P.n) continue;
#pragma unroll
    for (int b = 0; b < R_QMAX / 8; ++b) {
      if (b >= ntv) continue;
      double x2 = 0.0, p2 = 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = b * 8 + 2 * fk + e;
        if (c >= w) continue;
        const double pv = accP[a][b][e];
        const double xv = accX[a][b][e] + pv;
        const int64_t off = row * P.ld + P.c0 + lo + c;
        ox[off] = xv;
        op[off] = pv;
        nonfin |= !isfinite(xv) || !isfinite(pv);
        if (P.cplx) {  // (re, im) pair of one complex entry: modulus like np.abs
          x2 = fma(xv, xv, x2);
          p2 = fma(pv, pv, p2);
        } else {
          mx = fmax(mx, fabs(xv));
          mp = fmax(mp, fabs(pv));
        }
      }
      if (P.cplx) {
        mx = fmax(mx, sqrt(x2));
        mp = fmax(mp, sqrt(p2));
      }
    }
  }
  nonfin = __any_sync(0xffffffffu, nonfin);
  mx = warp_max(mx);
  mp = warp_max(mp);
  if (lane == 0) {
    if (nonfin) atomicOr(&P.flags[0], 1ull);
    if (side == 0) {
      if (mx > 0.0) atomicMax(&P.flags[1], dbits(mx));
      if (mp > 0.0) atomicMax(&P.flags[2], dbits(mp));
    }
  }
}

}  // namespace bk

using namespace bk;

static int recombine(int64_t n, int k_act, int q, int has_p, const double* coef, const double* X, const double* W,
                     const double* P_, const double* AX, const double* AW, const double* AP, double* Xo, double* Po,
                     double* AXo, double* APo, int64_t ld, int64_t c0, unsigned long long* flags, int cplx,
                     void* stream);

// flags: 3 x uint64 on device, zeroed by the caller.  Outputs may not alias inputs.
extern "C" int bk_subblock_recombine_d(int64_t n, int k_act, int q, int has_p, const double* coef,
                                       const double* X, const double* W, const double* P_, const double* AX,
                                       const double* AW, const double* AP, double* Xo, double* Po, double* AXo,
                                       double* APo, int64_t ld, int64_t c0, unsigned long long* flags,
                                       void* stream) {
  return recombine(n, k_act, q, has_p, coef, X, W, P_, AX, AW, AP, Xo, Po, AXo, APo, ld, c0, flags, 0, stream);
}

// complex128: blocks interleaved, ld/c0 in complex elements, coef complex (nb x dmax x q);
// coef_tmp: real scratch of nb x (2 dmax)(2 q) doubles for the expanded coefficients.
extern "C" int bk_subblock_recombine_z(int64_t n, int k_act, int q, int has_p, const double* coef,
                                       const double* X, const double* W, const double* P_, const double* AX,
                                       const double* AW, const double* AP, double* Xo, double* Po, double* AXo,
                                       double* APo, int64_t ld, int64_t c0, unsigned long long* flags,
                                       double* coef_tmp, void* stream) {
  if (n <= 0 || k_act <= 0 || q <= 0) return BK_ERR_ARG;
  const int nb = (k_act + q - 1) / q;
  const int nparts = has_p ? 3 : 2;
  dim3 grid((unsigned)lmin(64, (nparts * q * q + 255) / 256), nb);
  BK_COUNT();
  k_expand_coef<<<grid, 256, 0, (cudaStream_t)stream>>>(k_act, q, nparts, coef, coef_tmp);
  BK_CHECK_LAUNCH();
  return recombine(n, 2 * k_act, 2 * q, has_p, coef_tmp, X, W, P_, AX, AW, AP, Xo, Po, AXo, APo, 2 * ld, 2 * c0,
                   flags, 1, stream);
}

static int recombine(int64_t n, int k_act, int q, int has_p, const double* coef, const double* X, const double* W,
                     const double* P_, const double* AX, const double* AW, const double* AP, double* Xo, double* Po,
                     double* AXo, double* APo, int64_t ld, int64_t c0, unsigned long long* flags, int cplx,
                     void* stream) {
  if (n <= 0 || k_act <= 0 || q <= 0) return BK_ERR_ARG;
  if (q > R_QMAX) return BK_ERR_UNSUPPORTED;
  RecombParams R{};
  R.cplx = cplx;
  R.n = n;
  R.k_act = k_act;
  R.q = q;
  R.has_p = has_p ? 1 : 0;
  R.ld = ld;
  R.c0 = c0;
  R.dmax = (has_p ? 3 : 2) * q;
  R.coef = coef;
  R.in[0][0] = X; R.in[0][1] = W; R.in[0][2] = P_;
  R.in[1][0] = AX; R.in[1][1] = AW; R.in[1][2] = AP;
  R.outX[0] = Xo; R.outX[1] = AXo;
  R.outP[0] = Po; R.outP[1] = APo;
  R.flags = flags;
  int la = (q + 3) & ~3;
  if ((la & 7) == 0) la += 4;
  const int lb = ((q + 7) & ~7) + 4;
  const int smem = (3 * R_BM * la + 3 * q * lb) * (int)sizeof(double);
  static int attr_bytes = 0;
  if (smem > attr_bytes) {
    cudaFuncSetAttribute(recombine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_bytes = smem;
  }
  const int nb = (k_act + q - 1) / q;
  dim3 grid((unsigned)((n + R_BM - 1) / R_BM), nb, 2);
  if (nb > 65535) return BK_ERR_UNSUPPORTED;
  BK_COUNT();
  recombine_kernel<<<grid, R_THREADS, smem, (cudaStream_t)stream>>>(R);
  BK_CHECK_LAUNCH();
  return BK_OK;
}
