// Batched subblock recombination on FP64 tensor cores (DMMA).
//
// Replaces the per-subblock products of block_update and _run_subblocks:
//   P_j' = W_j C_W + P_j C_P,  X_j' = X_j C_X + P_j'           (ppcg.py:365-369)
//   AP_j' = AW_j C_W + AP_j C_P, AX_j' = AX_j C_X + AP_j'      (ppcg.py:521-532)
// for every subblock j in one launch (grid: row tiles x blocks x {X side, A side}).  X'
// and AX' go to separate output buffers so the pre-update X survives for the breakdown and
// rank-deficiency recovery paths (ppcg.py:694, 698-717, 456-472); P' and AP' may overwrite
// P and AP in place (nothing reads the pre-update P after the update), which keeps the
// state at 8 full-width blocks (config 5 on 8 GPUs).  A CTA reads its rows of P_j before it
// writes them; where a subblock needs several column tiles (complex q = 64) one CTA runs the
// tiles in turn and stages the earlier tiles' outputs in shared memory until the last tile
// has read its inputs.
// The breakdown test of ppcg.py:701-705 (non-finite entries in X, P, AX, AP; max|X|,
// max|P| > 1e8) is fused into the epilogue as device-wide flags.
#include "common.cuh"

namespace bk {

constexpr int R_BM = 64, R_THREADS = 128;  // 4 warps x 16 rows
constexpr int R_QMAX = 128;  // real-view width (complex q <= 64)

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

// Tiling: a CTA owns 64 rows x NT output columns of one subblock and one side; it streams
// the concatenated basis [X_j | W_j | P_j] (3w columns) through a 3-stage cp.async ring in
// chunks of 16 columns together with the matching 16 x NT coefficient rows, and accumulates
// X_j C_X and W_j C_W + P_j C_P in separate DMMA accumulators (the first part is X).  A
// CTA therefore reads its rows once per column tile (NT covers w for real q <= 64) and the
// coefficients stream from L2.  Strides of 20 / NT+4 doubles (== 4 mod 16) keep the
// fragment loads conflict-free.
constexpr int R_KC = 16, R_STAGES = 3, R_LA = R_KC + 4;

// SEQ (several column tiles per CTA, earlier tiles' outputs staged): a two-stage ring, so that
// two CTAs fit an SM beside the 64 KB of staging (one 4-warp CTA per SM left the DMMA pipe idle)
template <int NT, int MINB = 1, bool SEQ = false>
__global__ void __launch_bounds__(R_THREADS, MINB) recombine_kernel(const __grid_constant__ RecombParams P) {
  constexpr int R_STAGES = SEQ ? 2 : bk::R_STAGES;
  constexpr int LB = NT + 4, WN = NT / 8;
  constexpr int IN_STAGE = R_BM * R_LA, CF_STAGE = R_KC * LB;
  extern __shared__ __align__(16) double sm[];
  double* In = sm;                          // [stage][R_BM][R_LA]
  double* Cf = sm + R_STAGES * IN_STAGE;    // [stage][R_KC][LB]
  double* Stg = Cf + R_STAGES * CF_STAGE;   // SEQ: [tile][X', P'][R_BM][NT] of the earlier tiles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = blockIdx.y;
  const int side = blockIdx.z & 1;
  const int64_t r0 = (int64_t)blockIdx.x * R_BM;
  const int lo = j * P.q;
  const int w = min(P.q, P.k_act - lo);
  const int ntiles = SEQ ? (w + NT - 1) / NT : 1;
  bool nonfin = false;
  double mx = 0.0, mp = 0.0;
  for (int tile = 0; tile < ntiles; ++tile) {
  const int ct0 = SEQ ? tile * NT : (blockIdx.z >> 1) * NT;   // first output column of this tile
  if (ct0 >= w) return;
  if (SEQ && tile > 0) __syncthreads();  // the previous tile's stages are free
  const int nparts = P.has_p ? 3 : 2;
  const int cpp = (w + R_KC - 1) / R_KC;    // chunks per part
  const int nchunks = nparts * cpp;
  const double* cg = P.coef + (int64_t)j * P.dmax * P.q;
  const bool al16 = ((P.ld | (P.c0 + lo)) & 1) == 0;  // 16-byte aligned row segments

  auto load_chunk = [&](int c, int stage) {
    const int part = c / cpp, k0 = (c % cpp) * R_KC;
    const int kw = min(R_KC, w - k0);
    const double* src = P.in[side][part] + P.c0 + lo + k0;
    double* in = In + stage * IN_STAGE;
    if (al16) {
      for (int e = tid; e < R_BM * (R_KC / 2); e += R_THREADS) {
        const int r = e / (R_KC / 2), c2 = 2 * (e % (R_KC / 2));
        const int64_t row = r0 + r;
        const int nbytes = (row < P.n) ? 8 * max(0, min(2, kw - c2)) : 0;
        cp_async16(in + r * R_LA + c2, nbytes ? src + row * P.ld + c2 : src, nbytes);
      }
    } else {
      for (int e = tid; e < R_BM * R_KC; e += R_THREADS) {
        const int r = e / R_KC, cc = e % R_KC;
        const int64_t row = r0 + r;
        const bool v = row < P.n && cc < kw;
        cp_async8(in + r * R_LA + cc, v ? src + row * P.ld + cc : src, v);
      }
    }
    double* cf = Cf + stage * CF_STAGE;
    const double* csrc = cg + (int64_t)(part * w + k0) * w + ct0;
    for (int e = tid; e < R_KC * NT; e += R_THREADS) {
      const int r = e / NT, cc = e % NT;
      const bool v = r < kw && ct0 + cc < w;
      cp_async8(cf + r * LB + cc, v ? csrc + r * w + cc : cg, v);
    }
  };

  double accX[2][WN][2], accP[2][WN][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < WN; ++b) accX[a][b][0] = accX[a][b][1] = accP[a][b][0] = accP[a][b][1] = 0.0;
  const int fk = lane & 3, fm = lane >> 2;

#pragma unroll
  for (int s = 0; s < R_STAGES - 1; ++s) {
    if (s < nchunks) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<R_STAGES - 2>();
    __syncthreads();
    if (c + R_STAGES - 1 < nchunks) load_chunk(c + R_STAGES - 1, (c + R_STAGES - 1) % R_STAGES);
    cp_async_commit();
    const double* ia = In + (c % R_STAGES) * IN_STAGE + (warp * 16 + fm) * R_LA + fk;
    const double* cb = Cf + (c % R_STAGES) * CF_STAGE + fk * LB + fm;
    const bool xpart = c < cpp;
#pragma unroll
    for (int kk = 0; kk < R_KC; kk += 4) {
      double af[2], bf[WN];
      af[0] = ia[kk];
      af[1] = ia[8 * R_LA + kk];
#pragma unroll
      for (int b = 0; b < WN; ++b) bf[b] = cb[kk * LB + b * 8];
      if (xpart) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < WN; ++b) dmma_8x8x4(accX[a][b][0], accX[a][b][1], af[a], bf[b]);
      } else {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < WN; ++b) dmma_8x8x4(accP[a][b][0], accP[a][b][1], af[a], bf[b]);
      }
    }
  }
  cp_async_wait<0>();

  // epilogue: P' = accP, X' = accX + accP; breakdown statistics
  double* ox = P.outX[side];
  double* op = P.outP[side];
  if (SEQ && tile + 1 < ntiles) {  // stage this tile until the last tile has read its inputs
    double* sx = Stg + (size_t)tile * 2 * R_BM * NT;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < WN; ++b) {
        const int rr = warp * 16 + a * 8 + fm, cc = b * 8 + 2 * fk;
        sx[rr * NT + cc] = accX[a][b][0] + accP[a][b][0];
        sx[rr * NT + cc + 1] = accX[a][b][1] + accP[a][b][1];
        sx[R_BM * NT + rr * NT + cc] = accP[a][b][0];
        sx[R_BM * NT + rr * NT + cc + 1] = accP[a][b][1];
      }
    continue;
  }
  for (int tt = SEQ ? 0 : tile; tt <= tile; ++tt) {
  const int cb0 = SEQ ? tt * NT : ct0;
  const double* sx = Stg + (size_t)tt * 2 * R_BM * NT;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int64_t row = r0 + warp * 16 + a * 8 + fm;
    if (row >= P.n) continue;
#pragma unroll
    for (int b = 0; b < WN; ++b) {
      const int c = cb0 + b * 8 + 2 * fk;  // this lane's two adjacent columns c, c+1
      if (c >= w) continue;
      double p0 = accP[a][b][0], p1 = accP[a][b][1];
      double x0 = accX[a][b][0] + p0, x1 = accX[a][b][1] + p1;
      if (SEQ && tt < tile) {
        const int rr = warp * 16 + a * 8 + fm, cc = b * 8 + 2 * fk;
        x0 = sx[rr * NT + cc];
        x1 = sx[rr * NT + cc + 1];
        p0 = sx[R_BM * NT + rr * NT + cc];
        p1 = sx[R_BM * NT + rr * NT + cc + 1];
      }
      const int64_t off = row * P.ld + P.c0 + lo + c;
      if (c + 1 < w) {
        if ((off & 1) == 0) {
          *reinterpret_cast<double2*>(ox + off) = make_double2(x0, x1);
          *reinterpret_cast<double2*>(op + off) = make_double2(p0, p1);
        } else {
          ox[off] = x0; ox[off + 1] = x1;
          op[off] = p0; op[off + 1] = p1;
        }
        nonfin |= !isfinite(x0) || !isfinite(x1) || !isfinite(p0) || !isfinite(p1);
        if (P.cplx) {  // (re, im) of one complex entry: modulus like np.abs
          mx = fmax(mx, sqrt(fma(x0, x0, x1 * x1)));
          mp = fmax(mp, sqrt(fma(p0, p0, p1 * p1)));
        } else {
          mx = fmax(mx, fmax(fabs(x0), fabs(x1)));
          mp = fmax(mp, fmax(fabs(p0), fabs(p1)));
        }
      } else {  // odd real width: last column alone
        ox[off] = x0;
        op[off] = p0;
        nonfin |= !isfinite(x0) || !isfinite(p0);
        mx = fmax(mx, fabs(x0));
        mp = fmax(mp, fabs(p0));
      }
    }
  }
  }  // tt
  }  // tile
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

template <int NT, int MINB>
static void launch_recombine_m(const RecombParams& R, unsigned nrt, int nb, int nct, cudaStream_t st) {
  constexpr int smem = R_STAGES * (R_BM * R_LA + R_KC * (NT + 4)) * (int)sizeof(double);
  // per launch: the attribute belongs to the current device's context
  cudaFuncSetAttribute(recombine_kernel<NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  recombine_kernel<NT, MINB><<<dim3(nrt, nb, 2 * nct), R_THREADS, smem, st>>>(R);
}

// in-place P' over several column tiles: one CTA per (row tile, subblock, side) runs the tiles
template <int NT>
static void launch_recombine_seq(const RecombParams& R, unsigned nrt, int nb, int nct, cudaStream_t st) {
  const int smem = (2 * (R_BM * R_LA + R_KC * (NT + 4)) + (nct - 1) * 2 * R_BM * NT) * (int)sizeof(double);
  cudaFuncSetAttribute(recombine_kernel<NT, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  recombine_kernel<NT, 2, true><<<dim3(nrt, nb, 2), R_THREADS, smem, st>>>(R);
}

template <int NT>
static void launch_recombine(const RecombParams& R, unsigned nrt, int nb, int nct, cudaStream_t st) {
  // 5 CTAs per SM (94 registers, no spills): the short 6-chunk pipelines of a CTA need the
  // extra resident CTAs to keep bytes in flight (config 2: 1.30 -> 1.25 ms); 6 spills
  static const int minb = [] {
    const char* e = getenv("PPCG_RECOMB_MINB");
    return e ? atoi(e) : 5;
  }();
  if constexpr (NT >= 64) {
    // 64-column tiles (q = 64: configs 3-5) hold twice the accumulators: 208 registers without
    // a cap, and the 96 of five CTAs per SM cost 2 KB of spills per thread.  Three CTAs per SM
    // (164 registers, no spills) measured at config 3: 23.1 ms (5 CTAs) / 14.4 (4) / 9.8 (3) /
    // 11.9 (2)
    static const int minb64 = [] {
      const char* e = getenv("PPCG_RECOMB_MINB64");
      return e ? atoi(e) : 3;
    }();
    if (minb64 == 5) launch_recombine_m<NT, 5>(R, nrt, nb, nct, st);
    else if (minb64 == 2) launch_recombine_m<NT, 2>(R, nrt, nb, nct, st);
    else if (minb64 == 4) launch_recombine_m<NT, 4>(R, nrt, nb, nct, st);
    else launch_recombine_m<NT, 3>(R, nrt, nb, nct, st);
    return;
  }
  if (minb == 5) launch_recombine_m<NT, 5>(R, nrt, nb, nct, st);
  else if (minb == 6) launch_recombine_m<NT, 6>(R, nrt, nb, nct, st);
  else launch_recombine_m<NT, 1>(R, nrt, nb, nct, st);
}

}  // namespace bk

using namespace bk;

static int recombine(int64_t n, int k_act, int q, int has_p, const double* coef, const double* X, const double* W,
                     const double* P_, const double* AX, const double* AW, const double* AP, double* Xo, double* Po,
                     double* AXo, double* APo, int64_t ld, int64_t c0, unsigned long long* flags, int cplx,
                     void* stream);

// flags: 3 x uint64 on device, zeroed by the caller.  X', AX' may not alias inputs; P', AP'
// may be P, AP themselves (in-place update).
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
  const int nb = (k_act + q - 1) / q;
  if (nb > 65535) return BK_ERR_UNSUPPORTED;
  const unsigned nrt = (unsigned)((n + R_BM - 1) / R_BM);
  cudaStream_t st = (cudaStream_t)stream;
  BK_COUNT();
  const bool inplace = Po == P_ || APo == AP;
  if ((Xo == X || AXo == AX || Xo == W || AXo == AW) ||
      (inplace && !(Po == P_ && APo == AP)))  // X' may not alias inputs; P' in place on both sides or neither
    return BK_ERR_ARG;
  if (q <= 16) launch_recombine<16>(R, nrt, nb, 1, st);
  else if (q <= 32) launch_recombine<32>(R, nrt, nb, 1, st);
  else if (q <= 64 || !inplace) launch_recombine<64>(R, nrt, nb, (q + 63) / 64, st);
  else launch_recombine_seq<64>(R, nrt, nb, (q + 63) / 64, st);
  BK_CHECK_LAUNCH();
  return BK_OK;
}
