/* ppcg_b200.h — C ABI of the B200-native PPCG hot path (libppcg_b200.so).
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t (as void*), never
 * allocates caller-visible memory, and returns a status code (BK_OK = 0).  Blocks are
 * row-major (element (r, c) at p[r*ld + c]) — the C-order numpy layout of the reference
 * package — and complex128 data is interleaved (re, im).
 *
 * The reference (blockeig, pure Python over numpy/scipy) has no FFI of its own; each
 * function below replaces one numpy/scipy call site of its hot path, cited as
 * file:line under /root/reference/pkg/src/blockeig.  INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 */
#ifndef PPCG_B200_H
#define PPCG_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BK_OK 0
#define BK_ERR_ARG (-1)
#define BK_ERR_CUDA (-2)
#define BK_ERR_SOLVER (-3)
#define BK_ERR_UNSUPPORTED (-4)

int bk_version(void);
/* number of kernels this library has launched (host-side counter; evidence for gpu_launches) */
unsigned long long bk_launch_count(void);

/* ---- operator apply: SparseHermitian.apply, problems.py:72-73 (scipy csr_matvecs) */
int bk_spmm_csr_d(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, int m,
                  const double* X, int64_t ldx, double* Y, int64_t ldy, void* stream);
int bk_spmm_csr_z(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, int m,
                  const double* X, int64_t ldx, double* Y, int64_t ldy, void* stream);
/* SpMM kernel choice for bk_spmm_csr_*: 2 = whole-row vector gather (default), 0 = one warp
 * per row gather (3..7: experiment variants of the vector kernel) */
int bk_spmm_set_variant(int variant);
/* Plane-marching stencil SpMM, same result as bk_spmm_csr_*: for a CSR that is a
 * nearest-neighbour stencil on an nx x ny x nz C-order grid, with the plan of
 * paper_1407_7506_b200/spmm_plan.py: the CSR entries re-laid out as a grid-ordered ELL
 * (ell_val: n x width values, real rows padded to an even width; ell_off: n x woff uint16,
 * woff a multiple of 8, per entry (dx+1) << 14 | (dy+1)*10 + dz+1, 0xffff = padding),
 * d0 = column shift of a ghost-extended local CSR, planes [xlo, xhi) referenced.  X tiles and
 * entries are staged in shared memory by TMA and reused across the stencil.  Real: ldx, ldy
 * even and X, Y equally 16-byte aligned, else BK_ERR_UNSUPPORTED (use bk_spmm_csr_d). */
int bk_spmm_march_d(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* ell_val,
                    const uint16_t* ell_off, int width, int woff, int m, const double* X, int64_t ldx, double* Y,
                    int64_t ldy, int row_align, void* stream);
int bk_spmm_march_z(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* ell_val,
                    const uint16_t* ell_off, int width, int woff, int m, const double* X, int64_t ldx, double* Y,
                    int64_t ldy, int row_align, void* stream);
/* Stencil-slot SpMM (default where it applies), same result as bk_spmm_csr_*: for a
 * nearest-neighbour stencil CSR whose rows are sorted (CSR order = (dx, dy, dz) lexicographic)
 * and whose offsets form the 7-point cross (st = 7) or lie in the 27-point cube (st = 27).
 * sval: n x vd doubles (StencilPlan.slot_values): row r holds the value of stencil position s
 * in slot s (complex: interleaved) and the presence bit mask (int64 bit pattern) in its last
 * double.  X tiles are staged by TMA; the 7-point kernel keeps the tile's centre column in
 * registers along the march, the 27-point kernel computes 2 z rows per thread from shared
 * X lines.  Other arguments and the alignment rules as bk_spmm_march_*. */
int bk_spmm_stencil_d(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* sval, int vd, int st,
                      int m, const double* X, int64_t ldx, double* Y, int64_t ldy, int row_align, void* stream);
int bk_spmm_stencil_z(int nx, int ny, int nz, int xlo, int xhi, int64_t d0, const double* sval, int vd, int st,
                      int m, const double* X, int64_t ldx, double* Y, int64_t ldy, int row_align, void* stream);
/* kernel variant of bk_spmm_stencil_* (sweeps): 0 default; 1 = 7-point 512-byte slices /
 * 27-point 4 rows per thread */
int bk_spmm_stencil_set_config(int cfg);

/* ---- diagonal apply: DiagonalPreconditioner.apply operators.py:110, DiagonalOperator
 *      operators.py:68-69 (real d; complex blocks as real views with 2m columns) */
int bk_scale_rows_d(int64_t n, int m, const double* d, const double* X, int64_t ldx, double* Y,
                    int64_t ldy, void* stream);

/* ---- Gram X^T Y: block_inner, core.py:43-49 (complex: real Gram of interleaved views +
 *      bk_cplx_gram_combine_d).  ws: see bk_gram_ws_bytes; must be zero-initialised once. */
int64_t bk_gram_ws_bytes(int64_t n, int m1, int m2);
int bk_gram_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y, int64_t ldy,
              double* C, int64_t ldc, int symmetric, void* ws, int64_t ws_bytes, void* stream);
int bk_gram2_d(int64_t n, int m1a, int m2a, const double* X1, int64_t ldx1, const double* Y1,
               int64_t ldy1, double* C1, int64_t ldc1, int m1b, int m2b, const double* X2,
               int64_t ldx2, const double* Y2, int64_t ldy2, double* C2, int64_t ldc2, void* ws,
               int64_t ws_bytes, void* stream);
/* Grams whose width is not a multiple of 64 run as a 64-aligned main block plus narrow
 * strips; bk_gram_splits says whether a width splits, and the _part variants launch one
 * part (1 = main block, 2 = strips, 0 = both) so the strips can run on a second stream with
 * their own workspace beside the main block */
int bk_gram_splits(int m1, int m2);
/* Gram loader: 1 = warp-specialised bulk-copy pipeline (default where row strides are even),
 * 0 = the cp.async ring of every thread; returns the previous mode (mode < 0: query only).
 * Both give bitwise identical results; the switch exists for A/B measurement and tests. */
int bk_gram_set_loader(int mode);
/* Split Grams (bk_gram_splits): 1 = main 64-aligned block and the narrow strips in one launch,
 * interleaved by row chunk so the strips read X / Y rows while they are in L2 (default);
 * 0 = two launches.  Returns the previous mode (mode < 0: query only). */
int bk_gram_set_combo(int mode);
int bk_gram_part_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y,
                   int64_t ldy, double* C, int64_t ldc, int symmetric, int part, void* ws,
                   int64_t ws_bytes, void* stream);
int bk_gram2_part_d(int64_t n, int m1a, int m2a, const double* X1, int64_t ldx1, const double* Y1,
                    int64_t ldy1, double* C1, int64_t ldc1, int m1b, int m2b, const double* X2,
                    int64_t ldx2, const double* Y2, int64_t ldy2, double* C2, int64_t ldc2, int part,
                    void* ws, int64_t ws_bytes, void* stream);
int bk_cplx_gram_combine_d(int m1, int m2, const double* Cr, int64_t ldr, double* C, int64_t ldc,
                           void* stream);

/* ---- per-subblock pencil Grams: _solve_subblock_pencil, ppcg.py:206-211 */
int64_t bk_subblock_grams_ws_bytes(int64_t n, int k_act, int q, int has_p);
int bk_subblock_grams_d(int64_t n, int k_act, int q, int has_p, const double* X, const double* W,
                        const double* P, const double* AX, const double* AW, const double* AP,
                        int64_t ld, int64_t c0, double* Araw, double* Braw, void* ws,
                        int64_t ws_bytes, void* stream);
/* split-K waves of the paired (q = 32) subblock Grams (default 2; 0 = choose_chunks; -1 =
 * query); returns the previous value */
int bk_subblock_grams_set_waves(int waves);
/* complex128 blocks (interleaved; ld, c0 in complex elements); tmpA/tmpB: nb*(2*dmax)^2 doubles */
int bk_subblock_grams_z(int64_t n, int k_act, int q, int has_p, const double* X, const double* W,
                        const double* P, const double* AX, const double* AW, const double* AP,
                        int64_t ld, int64_t c0, double* Araw, double* Braw, double* tmpA,
                        double* tmpB, void* ws, int64_t ws_bytes, void* stream);

/* ---- batched subblock update (block_update ppcg.py:278-378 incl. fallback 231-275,
 *      solve_pencil core.py:175-202) and plain batched pencils */
/* Dense eigensolver of real shared-memory pencils (d <= 96, want <= 32): 0 = Householder
 * tridiagonalisation + bisection + inverse iteration (default), 1 = two-sided Jacobi.
 * Returns the previous mode (mode < 0: query only). */
int bk_pencil_set_eig(int mode);
int bk_pencil_max_dim(void);
/* Profiling builds only (pencil.cu compiled with -DPPCG_PENCIL_PROFILE): clock64 stamps of subblock 0's
 * phases in the last pencil launch (32 values; tools/pencil_phases.py).  Returns 1, or 0 in normal builds. */
int bk_pencil_phase_clocks(long long* out);
/* global workspace for nb pencils of dimension dmax (0 when d <= 96 real / 64 complex, which
 * run entirely in shared memory; larger ones keep their matrices and, real, the Jacobi
 * rotation log here); pass it as ws/ws_bytes below */
int64_t bk_pencil_ws_bytes(int nb, int dmax, int cplx);
int bk_subblock_pencils_d(int k_act, int q, int has_p, const double* Araw, const double* Braw,
                          double* coef, double* theta, int* info, double* cscale, int force_fallback,
                          void* ws, int64_t ws_bytes, void* stream);
int bk_pencil_batched_d(int nb, int d, int ldm, const double* A, const double* B, int want,
                        double* omega, double* C, int* status, void* ws, int64_t ws_bytes, void* stream);
int bk_subblock_pencils_z(int k_act, int q, int has_p, const double* Araw, const double* Braw,
                          double* coef, double* theta, int* info, double* cscale, int force_fallback,
                          void* ws, int64_t ws_bytes, void* stream);
int bk_pencil_batched_z(int nb, int d, int ldm, const double* A, const double* B, int want,
                        double* omega, double* C, int* status, void* ws, int64_t ws_bytes, void* stream);

/* ---- large subblock updates (pencil dimension > bk_pencil_max_dim(): whole-block PPCG,
 *      LOBPCG): block_update ppcg.py:278-378 with the branch logic on the host
 *      (bigblock.py); cplx selects interleaved complex128 data */
/* A, B (d x d, ld) = scaled symmetrised pencil of the kept basis columns idx[0:d] with
 * scales sf[0:d] from raw Grams Ar/Br (ld ldr)  (ppcg.py:312-330, core.py:143-164) */
int bk_block_assemble(int d, int cplx, const int* idx, const double* sf, const double* Ar,
                      const double* Br, int64_t ldr, double* A, double* B, int64_t ld, void* stream);
/* coef (nrows x w, ld w) = C[:, :w] rows scattered to raw columns idx and un-scaled by sf;
 * cmax = max |C[:, :w]| (coeff_scale, ppcg.py:358-363, 376) */
int bk_block_coef(int d, int w, int nrows, int cplx, const int* idx, const double* sf, const double* C,
                  int64_t ldc, double* coef, double* cmax, void* stream);
/* breakdown statistics of an n x m block (ppcg.py:701-705): flags[0] |= non-finite,
 * flags[slot] = max(flags[slot], bits(max |x|)), slot 1 = X, 2 = P, 0 = non-finite test only */
int bk_block_stats(int64_t n, int m, int cplx, const double* X, int64_t ldx, unsigned long long* flags,
                   int slot, void* stream);
/* singular values (descending) of a row-major m x n matrix (gesvd); rank test ppcg.py:351-356 */
int bk_svals_d(void* ctx, int m, int n, const double* M, int64_t ldm, double* s);
int bk_svals_z(void* ctx, int m, int n, const double* M, int64_t ldm, double* s);

/* ---- recombination: ppcg.py:365-369 and _run_subblocks ppcg.py:521-532 (+ breakdown
 *      flags of ppcg.py:701-705).  Xo, AXo must not alias any input; Po == P and APo == AP
 *      (both, or neither) update P, AP in place; other aliasing is BK_ERR_ARG. */
int bk_subblock_recombine_d(int64_t n, int k_act, int q, int has_p, const double* coef,
                            const double* X, const double* W, const double* P, const double* AX,
                            const double* AW, const double* AP, double* Xo, double* Po,
                            double* AXo, double* APo, int64_t ld, int64_t c0,
                            unsigned long long* flags, void* stream);
/* complex128: coef complex (nb x dmax x q); coef_tmp: nb*(2*dmax)*(2*q) doubles */
int bk_subblock_recombine_z(int64_t n, int k_act, int q, int has_p, const double* coef,
                            const double* X, const double* W, const double* P, const double* AX,
                            const double* AW, const double* AP, double* Xo, double* Po,
                            double* AXo, double* APo, int64_t ld, int64_t c0,
                            unsigned long long* flags, double* coef_tmp, void* stream);

/* ---- tall update GEMM Y = s.*(alpha X G + beta Z): _apply_projection ppcg.py:443-445,
 *      residual ppcg.py:630/758 (+Jacobi ppcg.py:678 as s), CholQR core.py:99 (flags bit0:
 *      G upper triangular), RR ppcg.py:574-577, Taylor-polar ppcg.py:477-481; optional
 *      fused stopping metric rayleigh_ritz.py:71-92 (ksplit/nsplit/metric_out) */
int64_t bk_tsgemm_ws_bytes(int64_t n, int N);
int bk_tsgemm_d(int64_t n, int K, int N, double alpha, const double* X, int64_t ldx, const double* G,
                int64_t ldg, double beta, const double* Z, int64_t ldz, double* Y, int64_t ldy,
                const double* rowscale, int flags, void* stream);
int bk_tsgemm_batched_d(int nprob, int64_t n, int K, int N, double alpha, const double* const* Xs,
                        int64_t ldx, const double* const* Gs, int64_t ldg, double beta,
                        const double* const* Zs, int64_t ldz, double* const* Ys, int64_t ldy,
                        const double* rowscale, int flags, int ksplit, int nsplit,
                        double* metric_out, void* ws, int64_t ws_bytes, void* stream);
int bk_cplx_expand_d(int K, int N, const double* G, int64_t ldg, double* Gr, int64_t ldr,
                     void* stream);

/* ---- FP64 products on the int8 tensor cores (tcgen05 kind::i8, Ozaki scheme: 8 signed 8-bit
 *      digits per element against per-row / per-column power-of-two scales, 36 digit products
 *      accumulated exactly in int32 TMEM, combined in fp64; error within DGEMM's bound class).
 *      Same results contract as bk_gram_d / bk_tsgemm_batched_d (the products of block_inner,
 *      core.py:43-49, and of the tall updates listed above); deterministic; Inf/NaN in a
 *      row / column make that row / column of the product NaN.  bk_fp64_emu_set(0/1) selects
 *      the DMMA or the emulated kernels in the host layer (default: PPCG_FP64_EMU, else on). */
int bk_fp64_emu_set(int mode);
int bk_fp64_emu_enabled(void);
/* CUDA-event timing of the emulated GEMM-core launches (digit slicing excluded), for the
 * roofline: bk_ozaki_timing(1) arms and clears, bk_ozaki_kernel_ms() syncs and returns the summed
 * milliseconds of the launches since (up to 16), bk_ozaki_timing(0) disarms. */
int bk_ozaki_timing(int on);
double bk_ozaki_kernel_ms(void);
/* ws bytes for one call (same: X and Y are one block; symmetric requires same).  A smaller ws
 * (>= the size for one row chunk) is accepted: rows are then sliced in super-chunks. */
int64_t bk_ozaki_gram_ws_bytes(int64_t n, int m1, int m2, int same, int symmetric);
int bk_ozaki_gram_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                    double* C, int64_t ldc, int symmetric, void* ws, int64_t ws_bytes, void* stream);
/* C1 = X^T Y1, C2 = X^T Y2 with X's digits computed once (the W / P projections) */
int64_t bk_ozaki_gram2_ws_bytes(int64_t n, int m1, int m2a, int m2b);
int bk_ozaki_gram2_d(int64_t n, int m1, const double* X, int64_t ldx, int m2a, const double* Ya, int64_t ldya,
                     double* Ca, int64_t ldca, int m2b, const double* Yb, int64_t ldyb, double* Cb, int64_t ldcb,
                     void* ws, int64_t ws_bytes, void* stream);
/* Column digits kept between products.  One block is the left operand of several Grams of an
 * iteration -- X^H AX (ppcg.py:630/758), the projections X^H W / X^H P (680-687), proj_defect
 * (688-692) -- so its exponents and digits are computed once into a caller-owned buffer
 * (bk_ozaki_coldigits_bytes(n, m) bytes) and the *_pre_d Grams read them: X there is columns
 * [c0, c0 + m1) of the sliced n x mdig block.  Same results as the plain entries bit for bit
 * (the digits are the same); the pre-sliced operand is never re-sliced in row super-chunks, so
 * ws holds the other operand's digits of all rows (*_pre_ws_bytes). */
int64_t bk_ozaki_coldigits_bytes(int64_t n, int m);
int bk_ozaki_coldigits_d(int64_t n, int m, const double* X, int64_t ldx, void* dig, int64_t dig_bytes, void* stream);
int64_t bk_ozaki_gram_pre_ws_bytes(int64_t n, int m1, int m2, int same, int symmetric);
int bk_ozaki_gram_pre_d(int64_t n, int m1, int m2, const double* X, int64_t ldx, const void* dig, int mdig, int c0,
                        const double* Y, int64_t ldy, double* C, int64_t ldc, int symmetric, void* ws,
                        int64_t ws_bytes, void* stream);
int64_t bk_ozaki_gram2_pre_ws_bytes(int64_t n, int m1, int m2a, int m2b);
int bk_ozaki_gram2_pre_d(int64_t n, int m1, const double* X, int64_t ldx, const void* dig, int mdig, int c0, int m2a,
                         const double* Ya, int64_t ldya, double* Ca, int64_t ldca, int m2b, const double* Yb,
                         int64_t ldyb, double* Cb, int64_t ldcb, void* ws, int64_t ws_bytes, void* stream);
/* K <= 16320; flags bit0: G upper triangular (k stages below a column tile are skipped) */
int64_t bk_ozaki_tsgemm_ws_bytes(int nprob, int64_t n, int K, int N, int ksplit);
int bk_ozaki_tsgemm_d(int nprob, int64_t n, int K, int N, double alpha, const double* const* Xs, int64_t ldx,
                      const double* const* Gs, int64_t ldg, double beta, const double* const* Zs, int64_t ldz,
                      double* const* Ys, int64_t ldy, const double* rowscale, int flags, int ksplit,
                      int nsplit, double* metric_out, void* ws, int64_t ws_bytes, void* stream);

/* ---- reductions: norms of ppcg.py:689-691, rayleigh_ritz.py:83-85, ppcg.py:452 */
int64_t bk_sumsq_ws_bytes(void);
int bk_sumsq_d(int64_t n, int m, const double* X, int64_t ldx, double* out, void* ws,
               int64_t ws_bytes, void* stream);
int bk_small_stats_d(int m1, int m2, const double* C, int64_t ldc, int cplx, double* out,
                     void* stream);

/* ---- Rayleigh-Ritz residual: ppcg.py:576-582 (W hand-off ppcg.py:396-397) */
int64_t bk_rr_residual_ws_bytes(int kt);
int bk_rr_residual_d(int64_t n, int kt, int cplx, const double* V, int64_t ldv, const double* AV,
                     int64_t ldav, const double* omega, const double* rowscale, double* W,
                     int64_t ldw, double* colnorm2, void* ws, int64_t ws_bytes, void* stream);

/* ---- strided column-range copy / zero (P realignment, lock_and_compact ppcg.py:399-408) */
int bk_copy_cols(int64_t n, int w, int elem_bytes, const void* src, int64_t lds, int64_t sc0,
                 void* dst, int64_t ldd, int64_t dc0, void* stream);
int bk_zero_cols(int64_t n, int w, int elem_bytes, void* dst, int64_t ldd, int64_t dc0,
                 void* stream);

/* ---- periodic dense work (north-star item 5, cuSOLVER inside; context owns workspace) */
int bk_dense_create(void** ctx, void* stream);
int bk_dense_destroy(void* ctx);
int bk_dense_set_stream(void* ctx, void* stream);
/* _cholesky_upper core.py:67-83: G -> R (row-major upper), fail_col (device) = first pivot
 * <= 1e-14 max|diag G|, or -1 */
int bk_chol_upper_floor_d(void* ctx, int m, double* G, int64_t ldg, int* fail_col);
int bk_chol_upper_floor_z(void* ctx, int m, double* G, int64_t ldg, int* fail_col);
int bk_tri_inv_upper_d(void* ctx, int m, double* R, int64_t ldr);
int bk_tri_inv_upper_z(void* ctx, int m, double* R, int64_t ldr);
/* solve_pencil core.py:175-202 at k_total (sygvd/hegvd); status[0] = 1 if singular */
int bk_rr_pencil_d(void* ctx, int d, double* A, int64_t lda, double* B, int64_t ldb, double* omega,
                   double* C, int64_t ldc, int* status);
int bk_rr_pencil_z(void* ctx, int d, double* A, int64_t lda, double* B, int64_t ldb, double* omega,
                   double* C, int64_t ldc, int* status);
/* np.linalg.qr(x)[0] (recovery paths ppcg.py:567, 712, 756); tmp: n*m scratch elements */
int bk_householder_q_d(void* ctx, int64_t n, int m, double* X, int64_t ldx, double* tmp);
int bk_householder_q_z(void* ctx, int64_t n, int m, double* X, int64_t ldx, double* tmp);

#ifdef __cplusplus
}
#endif
#endif /* PPCG_B200_H */
