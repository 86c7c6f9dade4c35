/*
 * cmf_b200.h -- C ABI of the B200-native ALS half-iteration.
 *
 * The reference (`cmf`, /root/reference/pkg/src/cmf) has no FFI: its hot path
 * is a set of Python functions over numba kernels.  Each entry point below is
 * the stateless C replacement for one of those functions; the Python package
 * paper_1808_03843_b200 keeps the reference's Python names and signatures and
 * binds these symbols with ctypes (see INTEGRATION.md for the stub a `cmf`
 * maintainer would add to route the reference's own functions here).
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer owned by the caller (e.g. a torch CUDA
 *     tensor's data_ptr()), unless the parameter name ends in `_host`.
 *   - Sizes and offsets are 64-bit.  `indptr` holds absolute positions into
 *     `indices`/`values`, so a row block [r0, r1) is processed by passing
 *     `indptr + r0` with `nrows = r1 - r0` (outputs offset by the caller).
 *   - Packed symmetric storage is the reference's row-major lower triangle:
 *     entry (i, j<=i) at i*(i+1)/2 + j (gram.py:20-21, :113-129).  `a_stride`
 *     is the element distance between consecutive systems (>= f*(f+1)/2).
 *   - All work is enqueued on `stream` (a cudaStream_t); nothing synchronises
 *     except where a function documents a device->host read.
 *   - Return value: one of the CMF_* status codes.  `cmf_last_error()` gives a
 *     thread-local message for the last non-zero status.
 */
#ifndef CMF_B200_H
#define CMF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMF_OK 0
#define CMF_EINVAL 1     /* -> DataError            (errors.py:14-15)   */
#define CMF_EOVERFLOW 2  /* -> NumericalError       (gram.py:139-145)   */
#define CMF_ESINGULAR 3  /* -> SingularSystemError  (solvers.py:225-235)*/
#define CMF_ECUDA 4      /* -> CmfError (CUDA runtime failure)          */

#define CMF_PREC_FP32 0
#define CMF_PREC_FP16 1

/* Gram kernels (K1).  BITWISE reproduces the reference's float32
 * mul-then-add in CSR order bit for bit (gram.py:149-187); FMA fuses the
 * multiply-add (one rounding).  The tcgen05 tensor-core path (fp16 operands,
 * fp32 TMEM accumulation; CG route) has its own entry point,
 * cmf_gram_assemble_tc, because it reads a binary16 shadow of the fixed
 * factors; CMF_GRAM_TC is accepted only by cmf_half_update. */
#define CMF_GRAM_BITWISE 0
#define CMF_GRAM_FMA 1
#define CMF_GRAM_TC 2

/* CG vector arithmetic.  FP32 is the paper's mixed-precision design
 * (fp16/fp32 A, fp32 vectors); FP64 restates solvers.py:70-145 operation for
 * operation (float64, sequential dot products) and is bitwise equal to it. */
#define CMF_CG_FP32 0
#define CMF_CG_FP64 1

const char *cmf_last_error(void);
int cmf_version(void);
/* SM count and compute capability of the current device (host query). */
int cmf_device_info(int *sm_count, int *cc_major, int *cc_minor);

/*
 * K1+K2: per-row Gram matrix and right-hand side for one half-update.
 * Replaces gram.assemble_side (gram.py:236-314) with its kernels
 * _accumulate_chunk (gram.py:190-206), pack_half (gram.py:132-146) and
 * _bias_chunk (gram.py:209-220) fused into one pass over the gathered rows.
 *
 *   A_u = base + sum_p fl(a_w[p] * theta_i) * theta_j  + reg * I
 *   b_u = sum_p b_w[p] * theta_{indices[p]}     (float64 accumulation)
 *   reg = float32(lam * n_u) if weighted_reg else float32(lam)
 *
 * a_weights NULL = all ones; b_weights NULL = skip the bias (b_out unused);
 * base_packed NULL = zeros.  a_out is float32 or binary16 (RNE) per
 * `precision`; a finite entry that overflows binary16 sets *overflow_flag
 * (device int, caller zeroes it) and the call still returns CMF_OK -- the
 * caller reads the flag and raises NumericalError.  nu_out (int64, nullable)
 * receives n_u.  kernel: CMF_GRAM_*.
 */
int cmf_gram_assemble(const int64_t *indptr, const int32_t *indices,
                      const float *a_weights, const float *b_weights,
                      int64_t nrows, const float *fixed, int64_t ncols, int32_t f,
                      double lam, int32_t weighted_reg, const float *base_packed,
                      int32_t precision, int32_t kernel, void *a_out, int64_t a_stride,
                      float *b_out, int64_t *nu_out, int32_t *overflow_flag,
                      void *stream);

/*
 * K1+K2 on the tensor cores (tcgen05.mma kind::f16, TMEM accumulators).
 * Same contract as cmf_gram_assemble with a_weights == NULL, except that the
 * fixed factors are read from `fixed16`, the binary16 shadow written by
 * cmf_factors_to_half (row width `w16` = cmf_tc_width(f) halves, ncols + 1
 * rows, the last one zero; column ids >= ncols gather as that zero row), and
 * the bias accumulates in fp32 in the same MMAs (the ratings ride as two extra
 * operand rows).  Requires f <= 120, even a_stride.
 *
 * Split precision (the exact route): pass `fixed16_lo` and `split_scale` from
 * cmf_factors_to_half_split; the kernel accumulates H H^T + H L^T + L H^T
 * (hi/lo binary16 halves of scale*theta, ~2^-22 relative) and undoes the
 * scale, which gives an fp32-faithful Gram for the exact solver's 1e-4 bar.
 * fixed16_lo == NULL selects the single-pass fp16 Gram (CG route).
 */
int cmf_gram_assemble_tc(const int64_t *indptr, const int32_t *indices, const float *b_weights,
                         int64_t nrows, const void *fixed16, const void *fixed16_lo,
                         int64_t ncols, float split_scale, int32_t w16, int32_t f, double lam,
                         int32_t weighted_reg, const float *base_packed, int32_t precision,
                         void *a_out, int64_t a_stride, float *b_out, int64_t *nu_out,
                         int32_t *overflow_flag, void *stream);
/*
 * cmf_gram_assemble_tc with the rows' rating count and a device workspace:
 * the split-precision (fp32) Gram over long rows (nnz >= 1024 * nrows) whose
 * hi + lo shadow exceeds 72 MB runs P <= 8 passes over equal fixed-side id
 * ranges (each pass's shadow slice stays in L2), accumulating into a_out /
 * b_out; P - 1 arrays of nrows int64 segment bounds go to `ws`
 * (cmf_gram_tc_workspace_bytes; too small or NULL: one pass).  Same results as
 * cmf_gram_assemble_tc up to fp32 summation order.  No base_packed.
 * Replaces the same reference path (gram.py:161-236 assemble_side).
 */
int cmf_gram_assemble_tc_ws(const int64_t *indptr, const int32_t *indices, const float *b_weights,
                            int64_t nrows, int64_t nnz, const void *fixed16, const void *fixed16_lo,
                            int64_t ncols, float split_scale, int32_t w16, int32_t f, double lam,
                            int32_t weighted_reg, int32_t precision, void *a_out, int64_t a_stride,
                            float *b_out, int64_t *nu_out, int32_t *overflow_flag, void *ws,
                            int64_t ws_bytes, void *stream);
int64_t cmf_gram_tc_workspace_bytes(int64_t nrows, int64_t nnz, int64_t ncols, int32_t f, int32_t split);
/* hi = fp16(scale*x), lo = fp16(scale*x - hi), both (rows + 1, w16), zero padded
 * (row `rows` all zero, as cmf_factors_to_half);
 * a finite value whose hi overflows binary16 sets *overflow_flag. */
int cmf_factors_to_half_split(const float *x, int64_t rows, int32_t f, void *hi16, void *lo16,
                              int32_t w16, float scale, int32_t *overflow_flag, void *stream);
/*
 * Fused half-update on the CG route (tensor-core Gram -> TMEM -> truncated CG
 * in registers): for every row with n_u > 0, A_u and b_u are accumulated by
 * tcgen05.mma into TMEM (fp16 operands from `fixed16`, fp32 accumulation) and
 * solved in place, target[u] <- CG_{f_s}(A_u + reg*I, b_u, x0 = target[u]),
 * eps = cg_tol * ||b_u||.  A_u never reaches HBM.  Replaces als.update_side
 * (als.py:54-74) for SolverConfig(method="cg").  f <= 120.  *breakdowns
 * (device int, nullable) accumulates p^T A p <= 0 exits.  A_u is used by the
 * CG in binary16 (RNE, the reference's precision="fp16" Hermitian storage,
 * gram.py:132-146): an entry of a row's A_u (or a rating) whose binary16
 * rounding overflows sets *overflow_flag (device int, nullable, caller zeroes
 * it; the caller raises NumericalError).  nnz =
 * indptr[nrows] - indptr[0], counted on the host: rows averaging >= 1024
 * ratings (the item side) run a CTA shape with fewer CG warps.
 */
int cmf_fused_cg_update(const int64_t *indptr, const int32_t *indices, const float *values,
                        int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16, int32_t f, double lam,
                        int32_t weighted_reg, float *target, int32_t f_s, double cg_tol,
                        int32_t *breakdowns, int32_t *overflow_flag, void *stream);
/*
 * Multi-GPU form of cmf_fused_cg_update: every solved row is also stored into
 * npeers replicas of `target` (peer_targets: a DEVICE array of device
 * pointers, e.g. CUDA-IPC mappings of the other ranks' factor matrices over
 * NVLink, each offset like `target`), so the all-gather after the half-update
 * disappears.  The caller orders the halves (stream sync + rank barrier).
 * Replaces the update + NCCL all-gather of the sharded driver.
 */
int cmf_fused_cg_update_peers(const int64_t *indptr, const int32_t *indices, const float *values,
                              int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16,
                              int32_t f, double lam, int32_t weighted_reg, float *target,
                              float *const *peer_targets, int32_t npeers, int32_t f_s, double cg_tol,
                              int32_t *breakdowns, int32_t *overflow_flag, void *stream);
/*
 * cmf_fused_cg_update_peers with a caller-supplied device workspace: for long
 * rows (avg >= 1024 ratings) over a fixed side whose binary16 shadow exceeds
 * L2 (> 48 MB), the half-update runs as two passes over the fixed side's row
 * range (first half of the column ids, then the second half), parking each
 * row's fp32 partial Gram in the workspace, so each pass's gather stays
 * L2-resident.  Same results up to fp32 summation order.  The workspace must
 * hold cmf_fused_cg_workspace_bytes(nrows, f) bytes (256-byte aligned); with
 * less (or NULL) the single pass runs.  CMF_TWO_PASS=0/1 forces the choice.
 */
int cmf_fused_cg_update_ws(const int64_t *indptr, const int32_t *indices, const float *values,
                           int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16,
                           int32_t f, double lam, int32_t weighted_reg, float *target,
                           float *const *peer_targets, int32_t npeers, int32_t f_s, double cg_tol,
                           int32_t *breakdowns, int32_t *overflow_flag, void *workspace,
                           int64_t workspace_bytes, void *stream);
/*
 * Implicit-feedback half-update on the fused CG route (f1 in SURVEY 8):
 * replaces implicit.implicit_update_side (implicit.py:63-84) with
 * precision="fp16" for every row with observations:
 *   A_u = gram_full + sum_k alpha r_k theta_k theta_k^T + lam I   (plain lambda)
 *   b_u = sum_k (1 + alpha r_k) theta_k
 * gram_full: F^T F of the fixed factors as a full row-major float32 matrix,
 * f rows of stride cmf_fused_base_ld(f) floats (implicit.precompute_gram,
 * unpacked; the stride is the kernel instance's compile-time row width).  The Gram runs on tcgen05 with
 * the gathered binary16 rows against a weighted copy (alpha r_k theta_k,
 * binary16) written by the producer warps; the CG, the overflow flag and the
 * workspace are as cmf_fused_cg_update_ws.  Rows with n_u == 0 are NOT touched
 * (their system is gram_full + lam I with b = 0, one shared matrix: the caller
 * solves them with cmf_batch_cg and a_stride = 0).  values must be >= 0.
 */
int cmf_fused_cg_update_implicit(const int64_t *indptr, const int32_t *indices, const float *values,
                                 int64_t nrows, int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16,
                                 int32_t f, double alpha, double lam, const float *gram_full, float *target,
                                 float *const *peer_targets, int32_t npeers, int32_t f_s, double cg_tol,
                                 int32_t *breakdowns, int32_t *overflow_flag, void *workspace,
                                 int64_t workspace_bytes, void *stream);
int64_t cmf_fused_cg_workspace_bytes(int64_t nrows, int32_t f);
/* Row stride (floats) of cmf_fused_cg_update_implicit's gram_full; -1 if f > 120. */
int32_t cmf_fused_base_ld(int32_t f);
/*
 * One pass of the fused kernel's two-pass scheme with a caller-owned segment
 * split and partial-accumulator buffer (the multi-GPU reduce-scatter exchange
 * for tall-skinny data):
 *   pass 1: gathers positions [indptr[u], seg[u]) of each row and stores the
 *           fp32 accumulator (Gram + the two bias columns) of row u at
 *           partial + (u*f + i) * pws, i < f, pws = roundup4(cmf_tc_width(f) + 2);
 *           nothing is solved.  Rows without ratings store nothing (zero the
 *           buffer first when it is summed across ranks).
 *   pass 2: gathers [seg[u], indptr[u+1]), adds the row's partial, adds
 *           lam*n_u (n_u = indptr[u+1] - indptr[u]) and solves into target.
 *           With seg[u] == indptr[u+1] the row is solved from the partial alone.
 * cmf_fused_cg_partial_floats(nrows, f) = floats of the partial buffer.  f <= 104.
 */
int cmf_fused_cg_pass(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                      int64_t nnz, const void *fixed16, int64_t ncols, int32_t w16, int32_t f, double lam,
                      int32_t weighted_reg, float *target, float *const *peer_targets, int32_t npeers,
                      const int64_t *seg, float *partial, int32_t pass, int32_t f_s, double cg_tol,
                      int32_t *breakdowns, int32_t *overflow_flag, void *stream);
int64_t cmf_fused_cg_partial_floats(int64_t nrows, int32_t f);
/* CUDA IPC for the peer replicas: export a device pointer (any address inside
 * an allocation) as a 64-byte handle + offset; open it in another process
 * (peer access enabled lazily over NVLink); close with the same offset. */
int cmf_ipc_export(const void *ptr, void *handle64, int64_t *offset);
int cmf_ipc_open(const void *handle64, int64_t offset, void **ptr_out);
int cmf_ipc_close(void *ptr, int64_t offset);
/* Debugging aid: a device buffer of 8 * 4096 int64 (or NULL to switch off) that
 * CTA 0 of the tensor-core kernels fills with clock64 stamps per operand stage
 * (producer wait / slot free / copies issued / MMA sees data / MMA commit). */
int cmf_debug_trace(void *buf);
/* Row width (halves) of the binary16 factor shadow for a given f. */
int cmf_tc_width(int32_t f);
/* fp32 (rows, f) -> binary16 (rows + 1, w16), RNE, zero padded columns, plus an
 * all-zero row `rows`: the tensor-core gather reads it for padding positions
 * (and for column ids >= ncols), so out16 must hold (rows + 1) * w16 halves.
 * A finite value whose binary16 rounding overflows sets *overflow_flag
 * (nullable). */
int cmf_factors_to_half(const float *x, int64_t rows, int32_t f, void *out16, int32_t w16,
                        int32_t *overflow_flag, void *stream);

/*
 * K2 alone: b_u = sum_p b_w[p] * theta_{indices[p]}, float64 accumulation in
 * CSR order, rounded once to float32.  Replaces gram.get_bias /
 * gram._bias_chunk (gram.py:209-220, :334-344).
 */
int cmf_spmm_bias(const int64_t *indptr, const int32_t *indices, const float *b_weights,
                  int64_t nrows, const float *fixed, int64_t ncols, int32_t f,
                  float *b_out, void *stream);

/*
 * K3: truncated CG on a batch of packed systems.  Replaces
 * solvers._cg_batch (solvers.py:121-145) as called by batch_solve
 * (solvers.py:238-245) and cg_solve/cg_solve_half (solvers.py:173-202).
 *   eps (float64 per system, nullable): absolute residual tolerance; when NULL
 *   the kernel uses cg_tol * ||b_s||_2 (solvers.py:240).
 *   nu (int64, nullable): systems with nu[s] == 0 are skipped and x_out[s] is
 *   not written (als.py:69-72 compaction, done in place).
 *   x0 and x_out may alias (in-place warm start).  iters/broke nullable.
 *   *breakdowns (device int, nullable) accumulates the breakdown count.
 *   a_stride == 0: every system shares the one matrix at `a` (the implicit
 *   engine's rows without observations: F^T F + lam I, b = 0).
 */
int cmf_batch_cg(const void *a, int32_t a_precision, int64_t a_stride, const float *b,
                 const float *x0, const double *eps, double cg_tol, const int64_t *nu,
                 int64_t nsys, int32_t f, int32_t f_s, int32_t accum, float *x_out,
                 int32_t *iters, int32_t *broke, int32_t *breakdowns, void *stream);

/*
 * K4: batched exact solve (Cholesky + two triangular solves) of packed
 * float32 systems.  Replaces solvers.exact_solve (solvers.py:148-164) and the
 * exact branch of batch_solve (solvers.py:221-237).  info[s] = 0 or k+1 for a
 * non-positive k-th pivot (LAPACK convention); x_out[s] is not written for
 * such systems and *nbad (device int, nullable) counts them.  nu as above.
 * accum: CMF_CG_FP32 (float32 factorisation) or CMF_CG_FP64.
 */
int cmf_batch_cholesky(const float *a, int64_t a_stride, const float *b, const int64_t *nu,
                       int64_t nsys, int32_t f, int32_t accum, float *x_out, int32_t *info,
                       int32_t *nbad, void *stream);

/*
 * Fused half-update for the streaming row-block path: Gram (+bias) into a
 * caller-supplied workspace, then the solve, block by block, writing the
 * solutions into `target` in place for rows with n_u > 0.  Replaces
 * als.update_side (als.py:54-74).  method: 0 = cg, 1 = exact.  The workspace
 * must hold ws_rows systems of a_stride elements (fp16 or fp32 per
 * precision) plus ws_rows*f floats (b) and ws_rows int64 (n_u).  With
 * kernel == CMF_GRAM_TC, ws16 must hold (ncols + 1) * cmf_tc_width(f) halves for
 * the binary16 shadow of `fixed` (ignored otherwise).
 * flags (4 device ints): [0] fp16 overflow, [1] CG breakdowns, [2] singular.
 */
int cmf_half_update(const int64_t *indptr, const int32_t *indices, const float *values,
                    int64_t nrows, const float *fixed, int64_t ncols, float *target,
                    int32_t f, double lam, int32_t weighted_reg, int32_t method,
                    int32_t precision, int32_t kernel, int32_t f_s, double cg_tol,
                    int32_t accum, void *ws_a, int64_t a_stride, float *ws_b,
                    int64_t *ws_nu, int64_t ws_rows, void *ws16, int32_t *flags, void *stream);

/* float32 -> binary16 RNE over n elements; *overflow_flag as above.
 * Replaces gram.pack_half (gram.py:132-146). */
int cmf_pack_half(const float *in, void *out, int64_t n, int32_t *overflow_flag,
                  void *stream);

/*
 * Evaluation (f2 in SURVEY 8(f)).  Squared-error partial sums of
 * (r - x_u . theta_v) over `count` (user, item, rating) triples, float64,
 * reduced deterministically into *out (one float64).  Replaces the data
 * term of als.objective (als.py:77-97) and als.rmse (als.py:100-107).
 * users/items are int64 when idx64 != 0, else int32.
 */
int cmf_sq_error(const void *users, const void *items, int32_t idx64, const float *ratings,
                 int64_t count, const float *x, const float *theta, int32_t f,
                 double *out, void *stream);
/* Same over a CSR view (row index implied by indptr). */
int cmf_sq_error_csr(const int64_t *indptr, const int32_t *indices, const float *values,
                     int64_t nrows, const float *x, const float *theta, int32_t f,
                     double *out, void *stream);
/* sum_r weight_r * ||x_r||^2 in float64 (weight = n_r from indptr, or 1 when
 * indptr is NULL) -> *out.  The regulariser of als.objective (als.py:86-93). */
int cmf_weighted_sqnorm(const int64_t *indptr, const float *x, int64_t nrows, int32_t f,
                        double *out, void *stream);
/* pred[k] = x_{users[k]} . theta_{items[k]} (float32).  factors.predict_pairs
 * (factors.py:41-54). */
int cmf_predict_pairs(const void *users, const void *items, int32_t idx64, int64_t count,
                      const float *x, const float *theta, int32_t f, float *pred,
                      void *stream);

/*
 * CSR + CSC construction (a13 / f3 in SURVEY 8).  Replaces data.build
 * (data.py:205-249): triples (user, item, rating) in file order -> the
 * reference's paired structure, bit for bit: rows ordered by (user, item),
 * duplicate (user, item) pairs collapsed to the LAST occurrence in file order,
 * CSC ordered by (item, user).  Hand-written stable LSD radix sorts (u64 key
 * user*n + item, then u32 key item), deterministic.
 *
 * user/item: int64 when idx64 != 0, else int32.  mn[2] (host, in/out): m, n;
 * a negative entry means "max id + 1" (the reference's default for None) and
 * is replaced by the resolved value (row_ptr == NULL: resolve m, n and return
 * without building, so the caller can size the outputs).  Outputs are caller-allocated device
 * arrays sized for the worst case: row_ptr[m+1], col_ptr[n+1] (int64),
 * col_idx/row_idx (int32) and csr_val/csc_val (float32) of length k.
 * ws: device workspace of cmf_build_workspace_bytes(k) bytes.
 * Synchronises `stream` (device->host reads of m/n, the validation result and
 * nnz): *nnz_host = entries after dedup.  An out-of-range triple returns
 * CMF_EINVAL with *bad_host = its index (the reference names the first one),
 * else *bad_host = -1.  Limits: k < 2^32 - 1, m < 2^32, n < 2^31.
 */
int cmf_build(const void *user, const void *item, int32_t idx64, const float *rating, int64_t k,
              int64_t *mn, int64_t *row_ptr, int32_t *col_idx, float *csr_val, int64_t *col_ptr,
              int32_t *row_idx, float *csc_val, void *ws, int64_t ws_bytes, int64_t *nnz_host,
              int64_t *bad_host, void *stream);
int64_t cmf_build_workspace_bytes(int64_t k);

/*
 * Implicit-feedback helpers (f1 in SURVEY 8; implicit.py:57-131).
 *
 * cmf_dense_gram: packed lower triangle of F^T F for a row-major (rows, f)
 * float32 matrix -- implicit.precompute_gram (implicit.py:57-60).  fp64 != 0:
 * float64 accumulation and output (the objective's Gram trick), else float32.
 * Deterministic (per-block partials summed in block order).  f <= 124.
 * ws: cmf_dense_gram_workspace_bytes(rows, f, fp64) bytes.
 */
int64_t cmf_dense_gram_workspace_bytes(int64_t rows, int32_t f, int32_t fp64);
int cmf_dense_gram(const float *F, int64_t rows, int32_t f, int32_t fp64, void *out_packed, void *ws,
                   int64_t ws_bytes, void *stream);
/* sum over a CSR view of c (1 - x_u.theta_v)^2 - (x_u.theta_v)^2, c = 1 + alpha r,
 * float64, deterministic -> *out (CMF_REDUCE_SLOTS doubles, like cmf_sq_error):
 * the sparse part of implicit_objective (implicit.py:87-104). */
int cmf_implicit_loss_csr(const int64_t *indptr, const int32_t *indices, const float *values, int64_t nrows,
                          const float *x, const float *theta, int32_t f, double alpha, double *out, void *stream);
/* Stable grouping of (row, col) pairs by row, duplicates kept: indptr[nrows+1],
 * cols_out[k] (int32).  rows/cols int64 when idx64 != 0.  ws: cmf_group_workspace_bytes(k). */
int64_t cmf_group_workspace_bytes(int64_t k);
int cmf_group_rows(const void *rows, const void *cols, int32_t idx64, int64_t k, int64_t nrows, int64_t *indptr,
                   int32_t *cols_out, void *ws, int64_t ws_bytes, void *stream);
/* Mean percentile rank numerator (implicit.py:115-131) over positives grouped
 * by user (pos_ptr[m+1], pos_item): *out (uint64, device) = sum over positives
 * of 2 #{i: s_ui > s_uv} + #{i != v: s_ui == s_uv}, s = float32 x_u.theta_i;
 * MPR = *out / (2 (n - 1) #positives).  Exact integer sum. */
int cmf_mpr_count(const int64_t *pos_ptr, const int32_t *pos_item, int64_t m, const float *x, const float *theta,
                  int64_t n, int32_t f, uint64_t *out, void *stream);

/*
 * Streaming synthetic generator (f3 in SURVEY 8; a counter-based restatement
 * of gen_synthetic's model, data.py:270-302, that any rank evaluates for its
 * own shard).  Cell (u, v) is present iff H(s_cell, u, v) < thr_cell, held out
 * iff also H(s_test, u, v) < thr_test; truth X / Theta entries and the rating
 * noise are hashes of (seed, index) too (gen.cu header).  Three calls:
 *   cmf_gen_truth:  which = 0 -> X (rows = m), 1 -> Theta (rows = n), (rows, f) float32;
 *   cmf_gen_count:  majors [lo, hi) (users when by_user != 0, else items) ->
 *                   ptr[hi-lo+1] (train cells per major, exclusive scan; ptr[hi-lo] = total)
 *                   and, for users only, tptr (test cells, nullable);
 *                   scratch: 2 (hi - lo) int64;
 *   cmf_gen_fill:   minor ids (ascending: build() order) and ratings of the
 *                   train cells at ptr; with tptr, the test triples (int64
 *                   user, item; float32 rating) of those users at tptr.
 * by_user = 1 gives a CSR shard, 0 a CSC shard; concatenated shards equal
 * data.build of the generated triples byte for byte (tests/test_gpu_gen.py).
 * Minors (items for a CSR shard, users for a CSC shard) are restricted to
 * [minor_lo, minor_hi) and written relative to minor_lo (a rank's local CSC
 * over its own users for the reduce-scatter exchange); the full range gives
 * global ids.
 */
int cmf_gen_truth(uint64_t seed, int32_t which, int64_t rows, int32_t f, float *out, void *stream);
int cmf_gen_count(uint64_t seed, int64_t m, int64_t n, uint64_t thr_cell, uint64_t thr_test, int32_t by_user,
                  int64_t lo, int64_t hi, int64_t minor_lo, int64_t minor_hi, int64_t *ptr, int64_t *tptr,
                  int64_t *scratch, void *stream);
int cmf_gen_fill(uint64_t seed, int64_t m, int64_t n, int32_t f, uint64_t thr_cell, uint64_t thr_test,
                 float noise_scale, int32_t by_user, int64_t lo, int64_t hi, int64_t minor_lo, int64_t minor_hi,
                 const float *X, const float *T, const int64_t *ptr, int32_t *minor_out, float *val_out,
                 const int64_t *tptr, int64_t *test_u, int64_t *test_v, float *test_r, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CMF_B200_H */
