/*
 * bt200 -- C-ABI of the B200-native (sm_100a) hot path behind the
 * reference package `blockten` (arXiv 2105.01170 structure-preserving
 * approximations).  Plain pointers, int64 extents, an explicit CUDA stream
 * (passed as void*), caller-owned device memory and workspaces.  Every
 * entry point returns a status code; bt_last_error() gives a thread-local
 * message.  Bit-reproducible: no floating-point atomics anywhere.
 *
 * The reference has no FFI of its own: each entry point
 * below replaces the numpy/LAPACK work inside the named reference function
 * (paths relative to /root/reference/pkg/src/blockten/).
 * shows the ctypes binding a maintainer would add to blockten.
 *
 * Layouts: all arrays are C-order (row-major) fp64 unless stated; tensors
 * are (m, p, n) = (block rows, class, block cols) (blocks.py:445-448); CP
 * factors are (extent, R) row-major like numpy's (decomp.py:90-117).
 */
#ifndef BT200_H
#define BT200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BT_ABI_VERSION 1

/* status codes (errors.py:11-32) */
#define BT_OK 0
#define BT_E_SHAPE 1   /* ShapeError */
#define BT_E_PATTERN 2 /* PatternMismatchError */
#define BT_E_NOT_PD 3  /* NotPositiveDefiniteError */
#define BT_E_CONV 4    /* ConvergenceError */
#define BT_E_CUDA 5    /* RuntimeError (CUDA failure) */
#define BT_E_VALUE 6   /* ValueError */

int bt_version(void);
const char* bt_last_error(void);
/* number of kernels this library has launched in the process (monotonic) */
int64_t bt_launch_count(void);

/* ------------------------------------------------------------------------
 * Strided-batched FP64 GEMM on the DMMA tensor pipe (building block of the
 * mode products and Grams: tensor.py:75-90 mode_multiply, decomp.py:220-234
 * unfolding Grams).  C[b][m][n] = alpha * sum_{ko,ki} A(b,m,ko,ki) *
 * B(b,ko,ki,n) * scale(b,ko,n) + beta * C.  A must have unit stride along m
 * or ki; B along n or ki.  symmetric=1 computes the lower tiles of a square
 * C and mirrors them (SYRK).
 * ---------------------------------------------------------------------- */
typedef struct bt_gemm_desc {
  int64_t M, N, Kin, Kout, batch;
  const double* A;
  int64_t sAm, sAko, sAki, sAb;
  const double* B;
  int64_t sBn, sBko, sBki, sBb;
  const double* bscale; /* optional: B(k,n) *= bscale[b*s_scale_b + ko*s_scale_ko + n] */
  int64_t s_scale_ko, s_scale_b;
  const double* ascale; /* optional: A(m,k) *= ascale[b*s_ascale_b + ko*s_ascale_ko + ki] */
  int64_t s_ascale_ko, s_ascale_b;
  double* C;
  int64_t sCm, sCn, sCb;
  double alpha, beta;
  int symmetric;
  int splits; /* 0 = heuristic */
} bt_gemm_desc;

int64_t bt_gemm_f64_ws_bytes(const bt_gemm_desc* d);
int bt_gemm_f64(const bt_gemm_desc* d, double* ws, int64_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * K1/K2: block gather T_E and scatter M_E.
 * Pattern maps (built on the host from BlockPattern.placements,
 * blocks.py:42-123): cell_class[ell*q] (int32, -1 = uncovered),
 * cell_order[ell*q] (int64: rank of the cell in the reference's scan order:
 * classes in order then cells in placement order; uncovered cells get
 * nnz + i*q + j, i.e. argwhere order), rep_cell[p] (int64, i*q+j of each
 * class's first placement), eta[p] (int64 counts).
 * ---------------------------------------------------------------------- */
typedef struct bt_pattern_dev {
  int64_t ell, q, m, n, p, nnz;
  const int32_t* cell_class;
  const int64_t* cell_order;
  const int64_t* rep_cell;
  const int64_t* eta;
  /* optional (may be NULL): the cells of class k are class_cells[class_ptr[k]
   * .. class_ptr[k+1]) (i*q+j, placement order) -- lets the scatter write a
   * class's block from one read of its representative */
  const int64_t* class_ptr;
  const int64_t* class_cells;
} bt_pattern_dev;

/* workspace: 2 * ell * q int32 flags + 2 int64 */
int64_t bt_gather_ws_bytes(const bt_pattern_dev* pat);
/* blocks.py:395-449 extract_blocks + mat_to_tensor.  a: (ell*m, q*n) with
 * row stride lda (>= q*n).  t: (m, p, n).  On mismatch returns BT_E_PATTERN
 * and writes the offending cell's order rank into *bad_order (host int64;
 * -1 if none).  Synchronises `stream` to read the verdict. */
int bt_gather_blocks_f64(const double* a, int64_t lda, const bt_pattern_dev* pat, double tol,
                         int weighted, double* t, void* ws, int64_t* bad_order, void* stream);
/* blocks.py:452-462 tensor_to_mat / 363-381 struct_expand: a[cell of k] =
 * t[:, k, :] / sqrt(eta_k) for a (m, p, n) tensor (t_sm, t_sp, t_sn
 * strides), uncovered cells zero.  a: (ell*m, q*n) with row stride lda. */
int bt_scatter_blocks_f64(const double* t, int64_t t_sm, int64_t t_sp, int64_t t_sn,
                          const bt_pattern_dev* pat, double* a, int64_t lda, void* stream);

/* blocks.py:266-329 detect_pattern, device passes.  Digest: per grid cell
 * (row-major, ell*q) a 128-bit order-independent digest (h1, h2) of the
 * block's bytes and nz = the reference's keep predicate (tol == 0: some
 * entry not +-0.0, i.e. blk.any(); tol > 0: NOT max|blk| <= tol, NaN kept).
 * Match: for every cell with cand[cell] >= 0, eq[cell] = 1 iff the block
 * equals block cand[cell] (exact != 0: bit for bit; else max|d| <= tol,
 * NaN failing).  Group: leader[cell] = the row-major first cell with the same
 * (h1, h2) among the cells with nz != 0 (-1 for a cell with nz == 0) and
 * cand[cell] = leader[cell] if another cell leads, else -1 -- the host's
 * first-occurrence grouping (blocks.py:300-318) on the device, so digest,
 * grouping and match queue without a host round trip.  ws: at least
 * bt_block_group_ws_bytes(cells) bytes (-1: cell count out of range).
 * Asynchronous. */
int64_t bt_block_group_ws_bytes(int64_t cells);
int bt_block_group(const uint64_t* h1, const uint64_t* h2, const int* nz, int64_t cells,
                   int64_t* leader, int64_t* cand, void* ws, int64_t ws_bytes, void* stream);
int bt_block_digest_f64(const double* a, int64_t lda, int64_t ell, int64_t q, int64_t m, int64_t n,
                        double tol, uint64_t* h1, uint64_t* h2, int* nz, void* stream);
int bt_block_match_f64(const double* a, int64_t lda, int64_t ell, int64_t q, int64_t m, int64_t n,
                       const int64_t* cand, double tol, int exact, int* eq, void* stream);

/* ------------------------------------------------------------------------
 * K3: weighted tensor builders for the configs.
 * ---------------------------------------------------------------------- */
/* apps.py:193-201: t[a, k, b] = sqrt(eta_k) * params[k, a, b]; t is (d_out, p, d_in) */
int bt_build_hankel_f64(const double* params, int64_t p, int64_t d_out, int64_t d_in,
                        const int64_t* eta, double* t, void* stream);
/* C3 Gneiting space-time tensor, t[i, k, j] = sqrt(eta_k) * phi(|x_i - x_j|, k / lag_scale),
 * phi(h, u) = exp(-10 h / (u+1)^0.25) / (u+1); points: (npts, 2) */
int bt_build_gneiting_f64(const double* points, int64_t npts, int64_t lags, double lag_scale,
                          const int64_t* eta, double* t, void* stream);
/* multilevel.py:268-298 generalised: x[i1,i2,i3] = sqrt(eta_i1 eta_i2 eta_i3) *
 * psf[i3,i2,i1], eta_i = grid - |i - h| (psf K^3, K odd) */
int bt_build_psf_f64(const double* psf, int64_t k, int64_t grid, double* x, void* stream);
/* C5: x[i,j,k] = sum_r a0[i,r] b0[j,r] c0[k,r] + noise * N(0,1)_philox(key, lin index),
 * only rows k in [k0, k1) (x is (I, J, k1-k0)); lin index uses the global K */
int bt_build_cp_model_f64(const double* a0, const double* b0, const double* c0, int64_t I,
                          int64_t J, int64_t K, int64_t R, int64_t k0, int64_t k1, double noise,
                          uint64_t key, double* x, void* ws, int64_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * K4-K6: CP-ALS (decomp.py:344-410) on a C-order (I, J, K) tensor.
 * ---------------------------------------------------------------------- */
typedef struct bt_cp_problem {
  const double* x; /* (I, J, K) C-order, device */
  int64_t I, J, K, R;
  double norm_x; /* ||x||_F (<= 0: computed on device) */
} bt_cp_problem;

/* Whole ALS loop, device resident.  factors a (I,R), b (J,R), c (K,R) hold
 * the initialisation on entry; on exit a holds KruskalRep.x = F0 * lam
 * (decomp.py:403), b and c the normalised factors, lam (R) the mode-3
 * column norms (decomp.py:391-392).  phase_ms (host, 4 doubles, optional)
 * accumulates CUDA-event times of the phases [mode 1 (tree kernel), mode 2
 * (P tree: stream P; Q tree: the Q GEMM + reduction), mode 3 (P tree: GEMM;
 * Q tree: stream Q), solves + fit] (bt_cp_tree_variant).  fit_history (host, max_iters) receives the fit
 * per sweep; *n_iters and *converged follow decomp.py:397-410.
 * fit_mode: 0 auto (Gram identity, explicit residual when the identity loses
 * precision), 1 always explicit (reference semantics decomp.py:395-396),
 * 2 Gram identity only.  The host loop reads the fit back once per sweep only
 * when tol > 0 (convergence test); with tol <= 0 the sweeps run without host
 * synchronisation.
 * Without phase_ms the call picks the path by size: a tensor that fits the
 * shared memory of 8 SMs (I*J*K <= 2^17, R <= 16) runs every sweep in ONE
 * launch on a thread-block cluster (cp_cluster.cuh; one-CTA fallback); R <= 16
 * beyond that (I, J <= 576, K <= 512) runs the two-pass sweep of cp_mid.cu,
 * where fit_mode 0 and 1 both report the explicit fit (its residual rides on
 * the X x3 C pass); everything else the dimension-tree phases below. */
int64_t bt_cp_als_ws_bytes(const bt_cp_problem* pb);
/* Dimension-tree root the CP phases use for this problem: 0 = P = X x3 C
 * (modes 1/2 from P, mode 3 a full GEMM), 1 = Q = X x1 A (mode 1 from the
 * tree kernel without a P store -- or, for K <= 256, from T[i] = X[i]^T B
 * batched over i --, Q by one GEMM, modes 2/3 from Q; chosen when R > 16
 * and K <= I).  Same MTTKRPs as decomp.py:384-388 either way; only the summation
 * order differs. */
int bt_cp_tree_variant(const bt_cp_problem* pb);
int bt_cp_als_f64(const bt_cp_problem* pb, double* a, double* b, double* c, double* lam,
                  int max_iters, double tol, int fit_mode, double* fit_history, int* n_iters,
                  int* converged, double* phase_ms, void* ws, int64_t ws_bytes, void* stream);

/* Phase API of the same loop, for a tensor sharded along mode 3 across
 * ranks (A, B replicated; C and X row-sharded; I, J global, K local).  A sweep:
 *   bt_cp_mttkrp(1, m1) -> SUM(m1) -> bt_cp_solve(1, m1, g) -> bt_cp_solve_finish(1, it, g)
 *   bt_cp_mttkrp(2, m2) -> SUM(m2) -> bt_cp_solve(2, m2, g) -> bt_cp_solve_finish(2, it, g)
 *   bt_cp_mttkrp(3, m3) ->            bt_cp_solve(3, m3, g) -> SUM(g) -> bt_cp_solve_finish(3, it, g)
 *   bt_cp_residual(r)   -> SUM(r)  -> bt_cp_residual_finish(it, r)
 * after bt_cp_init_local(buf) -> SUM(buf) -> bt_cp_init_finish(buf).
 * SUM is the caller's cross-rank sum (NCCL allreduce); with one rank it is
 * the identity.  Buffers: m1 (I,R), m2 (J,R), m3 (K,R), g and buf (R*R+2),
 * r (1), all device, caller owned.  bt_cp_state_finish writes x = a * lam. */
int64_t bt_cp_state_ws_bytes(const bt_cp_problem* pb);
int bt_cp_state_create(const bt_cp_problem* pb, double* a, double* b, double* c, double* lam,
                       int max_iters, int fit_mode, void* ws, int64_t ws_bytes, void* stream,
                       void** state);
int bt_cp_state_destroy(void* state);
int bt_cp_init_local(void* state, double norm_x, double* buf);
int bt_cp_init_finish(void* state, const double* buf);
int bt_cp_mttkrp(void* state, int mode, double* out);
int bt_cp_solve(void* state, int mode, const double* m, double* gbuf);
int bt_cp_solve_finish(void* state, int mode, int it, const double* gbuf);
int bt_cp_residual(void* state, double* res2);
int bt_cp_residual_finish(void* state, int it, const double* res2);
int bt_cp_read_fit(void* state, int it, double* fit);
int bt_cp_state_finish(void* state, int n_iters, double* fit_history);

/* Single MTTKRP (decomp.py:385-387 unfold(t,k) @ khatri_rao(...)): out (extent_mode, R).
 * mode in {1,2,3}.  Fused Khatri-Rao; no unfolding copy. */
int64_t bt_mttkrp_ws_bytes(const bt_cp_problem* pb, int mode);
int bt_mttkrp_f64(const bt_cp_problem* pb, int mode, const double* a, const double* b,
                  const double* c, double* out, void* ws, int64_t ws_bytes, void* stream);

/* Pseudo-inverse of a symmetric R x R matrix with numpy's pinv cutoff
 * (rcond 1e-15 * max |eig|) via an on-chip cyclic Jacobi eigensolver. */
int bt_pinv_sym_f64(const double* v, int64_t R, double* vp, void* stream);

/* ------------------------------------------------------------------------
 * K7-K9: Tucker pieces (decomp.py:220-321)
 * ---------------------------------------------------------------------- */
/* Gram of the mode-`mode` unfolding of a C-order tensor of order `order`
 * (dims[order]); g: (dims[mode-1])^2.  Unique-half SYRK on DMMA. */
int64_t bt_unfold_gram_ws_bytes(const int64_t* dims, int order, int mode);
int bt_unfold_gram_f64(const double* x, const int64_t* dims, int order, int mode, double* g,
                       void* ws, int64_t ws_bytes, void* stream);
/* Symmetric eigensolver: w (n) descending, v (n, n) row-major with column i
 * the eigenvector of w[i], each column sign-normalised so its largest-|.|
 * entry (first on ties) is positive (decomp.py:176-179). */
int64_t bt_syevd_ws_bytes(int64_t n);
int bt_syevd_f64(const double* a, int64_t n, double* w, double* v, void* ws, int64_t ws_bytes,
                 void* stream);
/* Leading nvec eigenpairs (n >= 3): Householder tridiagonalisation,
 * bisection, inverse iteration, back-transformation.  w (nvec) descending,
 * v (n x nvec) row-major, sign rule as bt_syevd_f64.  Eigenvectors are
 * computed only for w > tau * |w[0]| (tau < 0: all); the other columns are 0. */
int64_t bt_syevx_ws_bytes(int64_t n, int64_t nvec);
int bt_syevx_f64(const double* a, int64_t n, int64_t nvec, double tau, double* w, double* v,
                 void* ws, int64_t ws_bytes, void* stream);
/* Thin QR with nonnegative diag(R) (decomp.py:182-193): a (m x n, m >= n),
 * q (m x n), r (n x n), row-major. */
int64_t bt_qr_thin_ws_bytes(int64_t m, int64_t n);
int bt_qr_thin_f64(const double* a, int64_t m, int64_t n, double* q, double* r, void* ws,
                   int64_t ws_bytes, void* stream);
/* Lower Cholesky factor (decomp.py:196-212 / numpy potrf; lower triangle of
 * a read, a == l allowed): blocked, 64-wide panels, DMMA trailing updates.
 * BT_E_NOT_PD with *bad_pivot = 1-based failing pivot.  Synchronises the
 * stream.  bt_tri_inv_lower_f64: linv = L^-1 (blocked forward substitution;
 * replaces the two solve_triangular calls per block of psd.py:248-257). */
int64_t bt_cholesky_ws_bytes(int64_t n);
int bt_cholesky_f64(const double* a, int64_t n, double* l, void* ws, int64_t* bad_pivot,
                    void* stream);
int64_t bt_tri_inv_lower_ws_bytes(int64_t n);
int bt_tri_inv_lower_f64(const double* l, int64_t n, double* linv, void* ws, void* stream);
/* Mode product y = x x_mode u (tensor.py:75-90): u is (rows, dims[mode-1])
 * row-major (transpose=0) or u^T is given as (dims[mode-1], rows) (transpose=1). */
int64_t bt_ttm_ws_bytes(const int64_t* dims, int order, int mode, int64_t rows);
int bt_ttm_f64(const double* x, const int64_t* dims, int order, int mode, const double* u,
               int64_t rows, int transpose, double* y, void* ws, int64_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * K11: structured matvecs (reconstruct.py:271-315) for nrhs right-hand sides.
 * x: (nrhs, q*n) row-major (each row one RHS vector), y: (nrhs, ell*m).
 * ---------------------------------------------------------------------- */
/* Kron-sum: coeffs (p, r), terms (r, m, n). */
int64_t bt_matvec_kron_ws_bytes(const bt_pattern_dev* pat, int64_t r, int64_t nrhs);
int bt_matvec_kron_f64(const bt_pattern_dev* pat, const int64_t* row_ptr, const int64_t* row_cells,
                       const double* coeffs, const double* terms, int64_t r, const double* x,
                       int64_t nrhs, double* y, void* ws, int64_t ws_bytes, void* stream);
/* BLR: left (m, rl), right (n, rr), middles (p, rl, rr).  row_ptr (ell+1) /
 * row_cells (nnz: j * p + k, cells of block row i sorted by j) describe the
 * pattern rows. */
int64_t bt_matvec_blr_ws_bytes(const bt_pattern_dev* pat, int64_t rl, int64_t rr, int64_t nrhs);
int bt_matvec_blr_f64(const bt_pattern_dev* pat, const int64_t* row_ptr, const int64_t* row_cells,
                      const double* left, int64_t rl, const double* right, int64_t rr,
                      const double* middles, const double* x, int64_t nrhs, double* y, void* ws,
                      int64_t ws_bytes, void* stream);
/* Multilevel Kronecker sum of `nterms` 3-level terms with dense level
 * matrices s1 (nterms, N3o, N3i), s2 (nterms, N2o, N2i), s3 (nterms, N1o, N1i)
 * applied to volumes x (nrhs, N3i, N2i, N1i) -> y (nrhs, N3o, N2o, N1o). */
int64_t bt_ml_matvec_ws_bytes(int64_t nterms, const int64_t* nin, const int64_t* nout,
                              int64_t nrhs);
int bt_ml_matvec_f64(int64_t nterms, const int64_t* nin, const int64_t* nout, const double* s1,
                     const double* s2, const double* s3, const double* x, int64_t nrhs, double* y,
                     void* ws, int64_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * misc device reductions used by the host mirror
 * ---------------------------------------------------------------------- */
/* max |x| over n doubles into a device double (ws: bt_sumsq_ws_bytes) */
int bt_maxabs_f64(const double* x, int64_t n, double* out, void* ws, int64_t ws_bytes,
                  void* stream);
/* psd.py:141-161 block comparison: blocks (p, n, n), partner[p] (device
 * int64); returns BT_E_PATTERN with *bad_class = first failing class.
 * ws: p ints.  Synchronises the stream. */
int bt_transpose_check_f64(const double* blocks, int64_t p, int64_t n, const int64_t* partner,
                           double tol, void* ws, int64_t* bad_class, void* stream);
/* out = 1 / sqrt(x) elementwise */
int bt_inv_sqrt_f64(const double* x, int64_t n, double* out, void* stream);
/* Leading eigenpairs of a symmetric n x n Gram by block subspace iteration
 * with Rayleigh-Ritz (block b = min(min(need, hint>0 ? hint : need), 80) + 16;
 * optional warm-start columns start (n x start_cols)).  On *status == 0:
 * w[0..bq) Ritz values descending, v (n x bq, row-major) sign-normalised
 * Ritz vectors, *k_out leading pairs above tau*w[0] with residual
 * <= 32 eps w[0].  *status 1: no convergence (use bt_syevx_f64), 2: block
 * shape not applicable.  Synchronises the stream (host-side decisions). */
int64_t bt_leading_subspace_ws_bytes(int64_t n, int64_t need, int64_t hint);
int bt_leading_subspace_f64(const double* g, int64_t n, int64_t need, double tau,
                            const double* start, int64_t start_cols, int64_t hint, double* w,
                            double* v, int64_t* bq_out, int64_t* k_out, int* status, void* ws,
                            int64_t ws_bytes, void* stream);
/* Diagnostic: 13 clock64 values: stamps (9) of sweep 1's phases in the fused one-CTA
 * small CP-ALS kernel of bt_cp_als_f64, then 4 pinv timings (tools/prof_c1_small.py). */
int bt_cp_small_clocks(long long* out);
/* detect_pattern representatives: out[k] (m x n, contiguous) = the block at
 * cell cells[k] (= i*q + j, device int64) of a (row stride lda). */
int bt_copy_cells_f64(const double* a, int64_t lda, const int64_t* cells, int64_t p, int64_t q,
                      int64_t m, int64_t n, double* out, void* stream);
/* out[0] = trace(m), m n x n row-major (device double out) */
int bt_trace_f64(const double* m, int64_t n, double* out, void* stream);
/* SVQB column scaling: dinv = diag(m)^-1/2 (0 for a zero diagonal), out = D (m + m^T)/2 D */
int bt_sym_scale_f64(const double* m, int64_t b, double* dinv, double* out, void* stream);
/* sign rule (decomp.py:176-179) on every column of a row-major matrix */
int bt_sign_fix_f64(double* x, int64_t rows, int64_t cols, void* stream);
/* Same rule on x, with every flipped column also flipped in y (yrows x cols):
 * the u / v pair of svd_truncated (decomp.py:176-179). */
int bt_sign_fix_pair_f64(double* x, int64_t rows, int64_t cols, double* y, int64_t yrows,
                         void* stream);
/* Container payload layout (container.py:111-159): out = x's elements in
 * first-index-fastest order (the C-order array of the axis-reversed tensor),
 * rank 1..6; the same call with the reversed extents inverts it. */
int bt_reverse_axes_f64(const double* x, const int64_t* dims, int ndim, double* out, void* stream);
/* out[i] = Philox4x32-10 Box-Muller normal of index i under key. */
int bt_fill_normal_f64(double* out, int64_t n, uint64_t key, void* stream);
/* out (cols x rows) = x (rows x cols)^T, row-major, tiled through shared
 * memory (the RHS layout flips of the batched matvecs). */
int bt_transpose_f64(const double* x, int64_t rows, int64_t cols, double* out, void* stream);
/* SVD of a small square matrix m (n x n, n <= 32, row-major) by one-sided
 * Jacobi in one warp (high relative accuracy for small singular values; the
 * reference's np.linalg.svd of decomp.py:172 restricted to the projected
 * factor of a basis refinement): s descending, u (n x n) with the sign rule
 * of decomp.py:176-179 per column, v (n x n) compensated; m = u diag(s) v^T. */
int bt_svd_small_f64(const double* m, int64_t n, double* u, double* s, double* v, void* stream);
/* Tall-skinny Householder QR of x (m x n row-major, n <= 32, m up to ~6.6k
 * rows): q (m x n) orthonormal, r (n x n) upper triangular with diag >= 0
 * (decomp.py:182-193's normalisation); two-level TSQR, no Gram. */
int64_t bt_tsqr_ws_bytes(int64_t m, int64_t n);
/* Cholesky of a small SPD Gram g (n x n, n <= 32) for a CholeskyQR step:
 * lt = L^T, linvt = L^-T (both upper, row-major); *flag (device int) = 1
 * when a pivot is not above 1e-12 of the largest diagonal entry. */
int bt_chol_small_f64(const double* g, int64_t n, double* lt, double* linvt, int* flag,
                      void* stream);
/* `need` (<= 1024) orthonormal columns orthogonal to basis (n x k) into out
 * (n x need), from a Philox Gaussian block under key: blockwise projection +
 * column-scaled CholeskyQR2, sign rule per column; *status (host) 1 when a
 * block was rejected (numerically dependent), 0 otherwise. */
int64_t bt_complete_basis_ws_bytes(int64_t n, int64_t k, int64_t need);
int bt_complete_basis_f64(const double* basis, int64_t n, int64_t k, int64_t need, uint64_t key,
                          double* out, int* status, void* ws, int64_t ws_bytes, void* stream);
int bt_tsqr_f64(const double* x, int64_t m, int64_t n, double* q, double* r, void* ws,
                int64_t ws_bytes, void* stream);
/* out[i][j] = left[i] x[i][j] right[j] (left / right may be NULL). */
int bt_diag_scale_f64(const double* x, int64_t rows, int64_t cols, const double* left,
                      const double* right, double* out, void* stream);
/* out[c] = ||x[:, c]||_2 of a row-major rows x cols matrix. */
int bt_col_norms_f64(const double* x, int64_t rows, int64_t cols, double* out, void* stream);
/* s = sqrt(max(w, 0)) and sinv = 1 / s (1 where s == 0), elementwise. */
int bt_svals_f64(const double* w, int64_t n, double* s, double* sinv, void* stream);
/* normalise every column of a row-major (rows x cols) matrix to unit 2-norm */
int bt_col_normalize_f64(double* x, int64_t rows, int64_t cols, void* stream);
/* Ritz residual norms out[c] = ||gv[:, c] - theta[c] v[:, c]|| over the first
 * cols columns of row-major (rows x ld) gv and v. */
int bt_ritz_resid_f64(const double* gv, const double* v, const double* theta, int64_t rows,
                      int64_t cols, int64_t ld, double* out, void* stream);
/* z = alpha * x + beta * y elementwise (n doubles) */
int bt_axpby_f64(int64_t n, double alpha, const double* x, double beta, const double* y, double* z,
                 void* stream);
/* sum of squares of n doubles, deterministic tree; out is a device double */
int bt_sumsq_f64(const double* x, int64_t n, double* out, void* ws, int64_t ws_bytes,
                 void* stream);
int64_t bt_sumsq_ws_bytes(int64_t n);

/* FP64 peak microbenchmarks (bench only): DMMA.8x8x4 chains / DFMA chains on
 * all SMs; *flops receives the executed flop count. */
int bt_peak_dmma(int64_t iters, int blocks, int threads, double* sink, double* flops, void* stream);
int bt_peak_dmma_chains(int64_t iters, int blocks, int threads, int chains, double* sink,
                        double* flops, void* stream);
int bt_peak_dfma(int64_t iters, int blocks, int threads, double* sink, double* flops, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BT200_H */
