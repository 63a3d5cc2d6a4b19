/*
 * bk_kernels.h — internal thin C ABI between the host driver (C++) and the
 * hand-written sm_100a CUDA kernels of libblockeig_b200.so.
 *
 * Plain pointers and sizes only: every function takes raw DEVICE pointers,
 * an explicit leading dimension per dense operand and a cudaStream_t (passed
 * as void*), never throws, and returns 0 on success or a cudaError_t code.
 *
 * Device layout: dense blocks are ROW-MAJOR n x k with leading dimension ld
 * (element (i, j) at p[i*ld + j]); a column range of a block is the same
 * pointer offset by the first column, so the shrink/expand column selection
 * of the reference (take_leading, rightCols, hcat: proj/src/solvers.cpp:12-23)
 * is pointer arithmetic plus, where contiguity is needed, bk_copy_cols.
 * The matrix is full (both triangles) CSR with int32 row_ptr / col.
 *
 * Each entry names the reference code it replaces.
 */
#ifndef BK_KERNELS_H
#define BK_KERNELS_H

#include <stddef.h>
#include <stdint.h>

#if defined(_WIN32)
#define BK_API __declspec(dllexport)
#else
#define BK_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- K1 SpMM: Y = A X  (replaces spmv / spmv_block, proj/src/kernel.cpp:8-33) ---- */
BK_API int bk_spmm_d(int n, const int32_t* row_ptr, const int32_t* col, const double* val,
                     const double* x, int ldx, int k, double* y, int ldy, void* stream);
/* Window-staged form K1w (same Y, bit-identical): a HOST plan regroups the rows into
 * tiles of graph-local rows and lists, per tile t, the X rows it needs — window
 * wrow[wptr[t] .. wptr[t+1]): the tile's own rows first (they are also the Y rows
 * it writes), then the distinct out-of-tile columns (halo).  rp2 / val2: the full
 * CSR in tile order (each row's nonzeros in their original order); code[p]: the
 * window slot of nonzero p.  The kernel stages a window's X rows (a column chunk
 * at a time) and the tile's index slice in shared memory and reads every
 * nonzero's X row on chip.  bk_spmm_win_plan: tile = 0 takes 64 rows per tile; wcap = 0
 * applies the kernel's shared-memory rule (three CTAs per SM with >= 32-column chunks),
 * wcap > 0 a plain cap on the slots per window; ok = 0 when the windows are too large or
 * the graph has too little locality (the plain bk_spmm_d is then the kernel to use).
 * All plan pointers are host memory owned by the plan; the caller uploads them.
 * bk_spmm_win_d takes even ldx / ldy and x, y either both 16-byte aligned or both at an
 * odd column of a 16-byte aligned block (the column in front is then read, never written);
 * it returns cudaErrorMisalignedAddress otherwise. */
BK_API int bk_spmm_win_plan(int n, const int32_t* row_ptr, const int32_t* col, const double* val, int tile,
                            int wcap, void** plan);
BK_API int bk_spmm_win_plan_info(const void* plan, int* ok, int* tile, int* ntiles, int* wmax, int* nzmax,
                                 double* loads_per_row);
BK_API int bk_spmm_win_plan_arrays(const void* plan, const int32_t** rp2, const int32_t** code,
                                   const double** val2, const int32_t** wptr, const int32_t** wrow,
                                   int64_t* wrow_len);
BK_API void bk_spmm_win_plan_free(void* plan);
BK_API int bk_spmm_win_d(int n, int tile, int ntiles, int wmax, int nzmax, const int32_t* rp2,
                         const int32_t* code, const double* val2, const int32_t* wptr, const int32_t* wrow,
                         const double* x, int ldx, int k, double* y, int ldy, void* stream);
/* complex Hermitian twin: x, y, val interleaved (re, im); ld in complex elements */
BK_API int bk_spmm_z(int n, const int32_t* row_ptr, const int32_t* col, const double* val,
                     const double* x, int ldx, int k, double* y, int ldy, void* stream);

/* ---- K2 Gram: C = X^H Y, X n x a, Y n x b; C a x b row-major (ldc) ----
 * (replaces s.transpose()*as, proj/src/rr.cpp:11, and q.transpose()*v in CGS2,
 * proj/src/kernel.cpp:76,79).  FP64 DMMA tensor cores, split-K over n with a
 * fixed-order reduction (deterministic).  work: >= bk_gram_work_bytes(n, a, b). */
BK_API size_t bk_gram_work_bytes(int n, int a, int b);
BK_API int bk_gram_d(int n, const double* x, int ldx, int a, const double* y, int ldy, int b,
                     double* c, int ldc, void* work, void* stream);
/* symmetric-result variant for the Rayleigh-Ritz matrix H = S^T (A S) (d x d):
 * only the 96 x 96 tiles on and above the diagonal are computed; the strictly
 * lower tiles are mirrored (the reference symmetrises, kernel.cpp:97) */
BK_API int bk_gram_sym_d(int n, const double* x, int ldx, const double* y, int ldy, int d, double* c,
                         int ldc, void* work, void* stream);

/* ---- K3 update: Y = alpha X C + beta Y, X n x d, C d x k (row-major, ldc) ----
 * (replaces s*e.vectors, proj/src/rr.cpp:13; s*z1 / s*o.q, proj/src/solvers.cpp:195;
 * q*(q^T v), proj/src/kernel.cpp:76,79).  FP64 DMMA.  Y must not alias X. */
BK_API int bk_gemm_d(int n, const double* x, int ldx, int d, const double* c, int ldc, int k,
                     double alpha, double beta, double* y, int ldy, void* stream);

/* predicated launches: the kernels return at once unless *run_if != 0 (device
 * flag), so a data-dependent step costs no host round trip */
BK_API int bk_gram_if_d(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c,
                        int ldc, void* work, const int* run_if, void* stream);
BK_API int bk_gemm_if_d(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                        double beta, double* y, int ldy, const int* run_if, void* stream);
/* K4 "twice is enough" test after the first projection pass (DGKS, eta^2 = eta2):
 * flag[0] = 1 iff some column j has ||c_j||^2 > (1 - eta2) ||w_j||^2 (ref2), i.e.
 * lost more than 1 - eta2 of its squared norm; c: m x a (ldc elements, cw = 1 real
 * / 2 complex) */
BK_API int bk_dgks_flag_d(int m, int a, const double* c, int ldc, int cw, const double* ref2, double eta2,
                          int* flag, void* stream);

/* ---- column sums of squares: out[j] = sum_i |X_ij|^2 (deterministic) ---- */
BK_API size_t bk_colnorm2_work_bytes(int n, int k);
BK_API int bk_colnorm2_d(int n, const double* x, int ldx, int k, double* out, void* work,
                         void* stream);

/* ---- K6 residual + norms: R = AV - V diag(lambda); optional W = t .* R ----
 * (replaces residual_block + apply_precond, proj/src/rr.cpp:16-20,
 * proj/src/solvers.cpp:105-107).  Column norms of R and V land in
 * rn2[k], vn2[k] (sums of squares, deterministic).  r may be NULL when only
 * W is wanted; w (ldw) receives t.*R for columns [w_from, k) when non-NULL
 * (t == NULL means identity). */
BK_API size_t bk_residual_work_bytes(int n, int k);
BK_API int bk_residual_d(int n, const double* v, int ldv, const double* av, int ldav,
                         const double* lambda, int k, double* r, int ldr, const double* t,
                         double* w, int ldw, int w_from, double* rn2, double* vn2, void* work,
                         void* stream);
/* ... and the squared column norms of W (columns >= w_from) into wn2 (k - w_from
 * doubles; nullptr: none) — K4's reference norms without re-reading W */
BK_API int bk_residual_w_d(int n, const double* v, int ldv, const double* av, int ldav,
                           const double* lambda, int k, double* r, int ldr, const double* t,
                           double* w, int ldw, int w_from, double* rn2, double* vn2, double* wn2,
                           void* work, void* stream);

/* convergence finish (replaces assess_convergence, proj/src/rr.cpp:22-38):
 * per_pair[i] = sqrt(rn2)/(norm_a*sqrt(vn2) + sqrt(vn2)*|lambda|), overall =
 * max over i < n_ev, converged = leading prefix with per_pair <= tol.
 * rec receives {overall, converged, nonfinite_flag} as 3 doubles. */
BK_API int bk_convergence_d(int k, const double* rn2, const double* vn2, const double* lambda,
                            double norm_a, int n_ev, double tol, double* per_pair, double* rec,
                            void* stream);

/* ---- K4 pieces: skip-pivot Cholesky of a Gram block with the CGS2 drop rule ----
 * (replaces the keep/drop test of project_orthonormalize, proj/src/kernel.cpp:83-85).
 * g: a x a Gram (row-major, ldg) of the externally projected block; ref2[j] =
 * squared norm of column j BEFORE any projection (ref2 == NULL: no dropping,
 * every positive pivot kept).  A column is dropped when its Cholesky pivot is
 * below drop*ref (or ref == 0).  Output m (a x a, ldm, row-major): W*m has the
 * kept columns orthonormalised and packed left (rows of R^-1 in kept order,
 * zero rows for dropped columns).  info[0] = kept; info[1] = 1 when a pivot
 * decision was not certain (heavy cancellation in the Schur complement, so the
 * caller re-runs the block with exact column CGS2); info[2] = 1 on a
 * non-finite value.  work >= bk_chol_work_bytes(a). */
BK_API size_t bk_chol_work_bytes(int a);
BK_API int bk_chol_drop_d(int a, const double* g, int ldg, const double* ref2, double drop,
                          double* m, int ldm, int* info, void* work, void* stream);
/* the same, also writing cond[0] = 1 when some kept pivot kept less than 1e-3 of
 * its projected norm squared (g_jj / p_j > 1e3: the fused CholQR + Newton-Schulz
 * update would lose orthogonality, eps g_jj / p_j), cond[1] = 1 for a nonempty
 * well-conditioned block — device predicates for the bk_*_if_* kernels */
BK_API int bk_chol_drop_cond_d(int a, const double* g, int ldg, const double* ref2, double drop,
                               double* m, int ldm, int* info, int* cond, void* work, void* stream);

/* ---- K5 symmetric eigensolver (replaces sym_eig_small, proj/src/kernel.cpp:95-100) ----
 * Eigendecomposition of 0.5(H + H^T) (d x d row-major, ldh): values ascending
 * (the n_need smallest; n_need <= 0 means all), z (ldz) row-major with
 * eigenvector j in column j.  info[0] = Jacobi sweeps used (0 for the
 * tridiagonal path), info[1] = 1 if not converged.  d <= 2048.
 * bk_syev_d dispatches: d <= 48 one-CTA cyclic Jacobi (bk_syev_jacobi_d, H is
 * destroyed), else Householder tridiagonalisation + multisection bisection +
 * inverse iteration + CholQR2 + back-transformation (bk_syev_tri_d, H kept). */
BK_API size_t bk_syev_work_bytes(int d);
BK_API int bk_syev_d(int d, double* h, int ldh, int n_need, double* values, double* z, int ldz,
                     void* work, int* info, void* stream);
BK_API size_t bk_syev_jacobi_work_bytes(int d);
BK_API int bk_syev_jacobi_d(int d, double* h, int ldh, double* values, double* z, int ldz,
                            void* work, int* info, void* stream);
BK_API size_t bk_syev_tri_work_bytes(int d);
BK_API int bk_syev_tri_d(int d, const double* h, int ldh, int n_need, double* values, double* z,
                         int ldz, void* work, int* info, void* stream);

/* ---- K7 column movement / elementwise ---- */
/* dst[:, 0:k] = src[:, 0:k] (row-major; src and dst may overlap in the same rows) */
BK_API int bk_copy_cols_d(int n, const double* src, int lds, int k, double* dst, int ldd,
                          void* stream);
/* column-major host layout <-> row-major device layout */
BK_API int bk_cm_to_rm_d(int n, int k, const double* cm, int ldcm, double* rm, int ldrm,
                         void* stream);
BK_API int bk_rm_to_cm_d(int n, int k, const double* rm, int ldrm, double* cm, int ldcm,
                         void* stream);
/* y = a*x + b*y over n x k (row-major) */
BK_API int bk_axpby_d(int n, int k, double a, const double* x, int ldx, double b, double* y,
                      int ldy, void* stream);
/* zero rows [r0, r1) of columns [0, k) */
BK_API int bk_zero_rows_d(double* x, int ldx, int k, int r0, int r1, void* stream);
/* out = a*x + b*y over n x k (out may alias x or y) */
BK_API int bk_lincomb_d(int n, int k, double a, const double* x, int ldx, double b, const double* y,
                        int ldy, double* out, int ldo, void* stream);
/* y[i][c] = t[i] * x[i][c] (t == NULL: plain copy); the diagonal preconditioner
 * W = diag(T) R of proj/src/solvers.cpp:98-107 */
BK_API int bk_scale_rows_d(int n, int k, const double* t, const double* x, int ldx, double* y,
                           int ldy, void* stream);
/* out[c] = sum_i x[i][c] * y[i][c] (deterministic two-level sum) */
BK_API int bk_coldot_d(int n, const double* x, int ldx, const double* y, int ldy, int k,
                       double* out, void* work, void* stream);
/* batched CG bookkeeping for TraceMIN (cg_solve, proj/src/kernel.cpp:139-164):
 * state per column c: rs[c], bnorm[c], active[c] (1/0).
 * bk_cg_check: deactivate columns with sqrt(rs) < 1e-14*bnorm; count[0] = #active.
 * bk_cg_step1: for active c: pap <= 0 deactivates, else alpha = rs/pap,
 *              x += alpha p, r -= alpha ap.
 * bk_cg_step2: for active c: beta = rs_new/rs, p = r + beta p, rs = rs_new. */
/* CG start for the TraceMIN solves (kernel.cpp:143-145): bnorm = sqrt(rs), active = bnorm != 0 */
BK_API int bk_cg_init_d(int k, const double* rs, double* bnorm, int* active, void* stream);
BK_API int bk_cg_check_d(int k, const double* rs, const double* bnorm, int* active, int* count,
                         void* stream);
BK_API int bk_cg_step1_d(int n, int k, const double* rs, const double* pap, int* active, double* x,
                         int ldx, double* r, int ldr, const double* p, int ldp, const double* ap,
                         int ldap, void* stream);
BK_API int bk_cg_step2_d(int n, int k, double* rs, const double* rs_new, const int* active,
                         const double* r, int ldr, double* p, int ldp, void* stream);

/* Newton-Schulz re-orthonormalisation coefficients: m = (3I - g)/2 (a x a), so
 * that W m is orthonormal to O(||W^T W - I||^2).  Second pass of CholQR2 and
 * the final polish of the eigenvector block (no sequential factorisation). */
BK_API int bk_ns_coeff_d(int a, const double* g, int ldg, double* m, int ldm, void* stream);

/* device-side CGS2 column step (the exact fallback of K4, kernel.cpp:83-87):
 * given nrm2 = ||v||^2 after the projections and ref2 = ||w_j||^2 before them,
 * keep v when sqrt(nrm2) >= drop * sqrt(ref2) (and ref2 > 0): write v / ||v||
 * into column counter[0] of out and increment counter[0].  No host sync. */
BK_API int bk_cgs2_commit_d(int n, const double* v, const double* nrm2, const double* ref2, double drop,
                            double* out, int ldo, int* counter, void* stream);

/* ---- complex128 (Hermitian) variants — config 5 (no reference counterpart:
 * the reference is real-only).  Complex blocks are interleaved
 * (re, im) row-major; every ld / column count below is in COMPLEX elements.
 * Tall-skinny products run on the real views (n x 2k) through the real DMMA
 * kernels (bk_complex.cu explains the rearrangements).  Same contracts as the
 * _d functions above; the work sizes differ. */
BK_API size_t bk_gram_z_work_bytes(int n, int a, int b);
BK_API int bk_gram_z(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c,
                     int ldc, void* work, void* stream);
/* Hermitian H = X^H Y (d x d) when X^H Y is known to be Hermitian (Rayleigh-Ritz):
 * upper tiles only; work: bk_gram_z_work_bytes(n, d, d) */
BK_API int bk_gram_sym_z(int n, const double* x, int ldx, const double* y, int ldy, int d, double* c, int ldc,
                         void* work, void* stream);
BK_API size_t bk_gemm_z_work_bytes(int d, int k);
BK_API int bk_gram_if_z(int n, const double* x, int ldx, int a, const double* y, int ldy, int b, double* c,
                        int ldc, void* work, const int* run_if, void* stream);
BK_API int bk_gemm_if_z(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                        double beta, double* y, int ldy, void* work, const int* run_if, void* stream);
BK_API int bk_gemm_z(int n, const double* x, int ldx, int d, const double* c, int ldc, int k, double alpha,
                     double beta, double* y, int ldy, void* work, void* stream);
BK_API size_t bk_colnorm2_z_work_bytes(int n, int k);
BK_API int bk_colnorm2_z(int n, const double* x, int ldx, int k, double* out, void* work, void* stream);
BK_API size_t bk_coldot_z_work_bytes(int n, int k); /* out[c] = Re sum conj(x) y */
BK_API int bk_coldot_z(int n, const double* x, int ldx, const double* y, int ldy, int k, double* out,
                       void* work, void* stream);
BK_API size_t bk_residual_z_work_bytes(int n, int k);
BK_API int bk_residual_z(int n, const double* v, int ldv, const double* av, int ldav, const double* lambda,
                         int k, double* r, int ldr, const double* t, double* w, int ldw, int w_from,
                         double* rn2, double* vn2, void* work, void* stream);
BK_API int bk_residual_w_z(int n, const double* v, int ldv, const double* av, int ldav, const double* lambda,
                           int k, double* r, int ldr, const double* t, double* w, int ldw, int w_from,
                           double* rn2, double* vn2, double* wn2, void* work, void* stream);
BK_API int bk_ns_coeff_z(int a, const double* g, int ldg, double* m, int ldm, void* stream);
BK_API size_t bk_chol_z_work_bytes(int a);
BK_API int bk_chol_drop_z(int a, const double* g, int ldg, const double* ref2, double drop, double* m,
                          int ldm, int* info, void* work, void* stream);
BK_API int bk_chol_drop_cond_z(int a, const double* g, int ldg, const double* ref2, double drop, double* m,
                               int ldm, int* info, int* cond, void* work, void* stream);
BK_API int bk_cm_to_rm_z(int n, int k, const double* cm, int ldcm, double* rm, int ldrm, void* stream);
BK_API int bk_rm_to_cm_z(int n, int k, const double* rm, int ldrm, double* cm, int ldcm, void* stream);
/* Hermitian projected eigenproblem: grid-cooperative Householder reduction to a
 * REAL tridiagonal (LAPACK zhetd2 conventions), bisection + inverse iteration
 * as for bk_syev_tri_d, complex back-transformation.  d <= 1200. */
BK_API size_t bk_syev_z_work_bytes(int d);
BK_API int bk_syev_z(int d, const double* h, int ldh, int n_need, double* values, double* z, int ldz,
                     void* work, int* info, void* stream);
BK_API int bk_cg_step1_z(int n, int k, const double* rs, const double* pap, int* active, double* x, int ldx,
                         double* r, int ldr, const double* p, int ldp, const double* ap, int ldap, void* stream);
BK_API int bk_cg_step2_z(int n, int k, double* rs, const double* rs_new, const int* active, const double* r,
                         int ldr, double* p, int ldp, void* stream);
BK_API int bk_cgs2_commit_z(int n, const double* v, const double* nrm2, const double* ref2, double drop,
                            double* out, int ldo, int* counter, void* stream);

/* host-only hook: nblocks consecutive random blocks (sizes[i] values each) from
 * the solver's per-solve normal stream; bit-identical to drawing each block
 * with a fresh std::normal_distribution over one std::mt19937_64(seed) */
BK_API int bk_host_normal_blocks(uint64_t seed, const int* sizes, int nblocks, double* out);

/* host-only hook (no device use): the product's strategy state machine driven
 * over a residual sequence, for CPU tests of decide() parity */
BK_API int bk_host_decide_sequence(int kind, int j_e, int j_s, double mu, int j_p, int j_warm,
                                   double r_warm, const double* r, int count, int n_es, int n_ex,
                                   int start_n_now, int start_shrunk, int apply_changes,
                                   int* decisions);

/* ---- sparse shift-and-invert factor (reference SpdFactor sparse path,
 * proj/src/kernel.cpp:110-134) ----
 * The symbolic structure comes from the host analysis (host/spchol.cpp): L in
 * CSC (colptr, rowind with the diagonal first, val), its row patterns (rptr, rk
 * ascending, rpos = position of L(j, rk) in val), the etree level sets (order,
 * lvlptr; lvlptr_host is the same array in host memory), C = P (sgn A - shift I)
 * P^T's lower entries as (aidx = destination in val, aval).
 * factor: fail = 1 when a pivot is not positive (not SPD).
 * solve: y = P^T L^-T L^-1 P x for m right-hand sides (row-major, x != y), t a
 * scratch n x ldt block, perm[new] = old. */
BK_API int bk_spchol_factor_d(int n, int nlev, const int* lvlptr_host, const int* order, const int64_t* colptr,
                              const int* rowind, double* val, int64_t nnz_l, const int64_t* rptr, const int* rk,
                              const int64_t* rpos, int64_t nnz_c, const int64_t* aidx, const double* aval,
                              int* fail, void* stream);
BK_API int bk_spchol_solve_d(int n, int m, const double* x, int ldx, double* y, int ldy, double* t, int ldt,
                             const int* perm, int nlev, const int* lvlptr, const int* order,
                             const int64_t* colptr, const int* rowind, const double* val, const int64_t* rptr,
                             const int* rk, const int64_t* rpos, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BK_KERNELS_H */
