/* hps_b200.h — C ABI of the B200-native HPS (hierarchical Poincare-Steklov) solver kernels.
 *
 * The reference (arXiv 1612.02736, Python package `specdtn`) has no FFI: its operator API is
 * the Python functions build_stage / FactorizedSolver.solve (pkg/src/specdtn/solver.py:357,
 * :337). This library is what those entry points bind to on the GPU side; the Python host
 * package paper_1612_02736_b200 loads it with ctypes (INTEGRATION.md shows the binding).
 * Each entry point below replaces one numeric step of the reference:
 *
 *   hps_leaf_build        leaf.py:138-163 build_leaf_operators (assembly model.py:153-177,
 *                         LU + gecon leaf.py:104-121, S/T/F/H leaf.py:152-162) for a batch of
 *                         same-shape leaves
 *   hps_merge_build       solver.py:122-143 merge_siblings (+ _factor_interface :108-119) for a
 *                         batch of same-shape parents
 *   hps_sweep_gemv        solver.py:255-335 one level of the upward / downward solve sweeps
 *   hps_gemm_batched      the dense products of solver.py:146-188 (2:1 wraps) and any batched
 *                         A.B the host needs
 *   hps_gj_invert_batched the batched FP64 pivoted inverse used by the two build steps
 *   hps_leaf_apply        timestepping.py:117-167 the explicit side (1/k + A/2) u_n of
 *                         Crank-Nicolson (or u_n/k for backward Euler) on every leaf
 *
 * Conventions: all matrices are row-major FP64 in DEVICE memory owned by the caller; every
 * call enqueues work on `stream` (a cudaStream_t, NULL = legacy default stream) and returns
 * immediately with HPS_OK or an error code (hps_status_string). Calls never allocate device
 * memory: callers size workspaces with the *_workspace_bytes queries. Numerical failures
 * (exactly zero / NaN pivot) are reported per batch item in `status` (bit 0); condition
 * numbers are reported as exact 1-norms (`*norm` outputs) so the host can apply the
 * reference's rcond < 1e-13 rule (leaf.py:37, solver.py:52) with kappa_1 = |A|_1 |A^-1|_1.
 * Stateless and re-entrant; safe to call concurrently on different streams.
 */
#ifndef HPS_B200_H
#define HPS_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_ABI_VERSION 7

enum hps_status { HPS_OK = 0, HPS_EINVAL = 1, HPS_ECUDA = 2 };

/* A batch of equally shaped matrices: item i starts at (ptrs ? ptrs[i] : base + i*stride) + off,
 * rows are `ld` elements apart. */
typedef struct {
  double* base;
  long long stride;
  double* const* ptrs;
  int ld;
  long long off;
} hps_mat_batch;

int hps_abi_version(void);
const char* hps_status_string(int code);

/* C_i = alpha A_i B_i + beta C_i (+ bias, an M x N matrix shared by the batch, if non-null). */
int hps_gemm_batched(int batch, int M, int N, int K, double alpha, const hps_mat_batch* A,
                     const hps_mat_batch* B, double beta, const hps_mat_batch* C,
                     const double* bias, int ldbias, void* stream);

/* In-place inverse of the leading n x n block of M_i (n x ncols); trailing columns become
 * inv(A_i) * rhs_i. piv: batch*n ints; workspace: hps_gj_workspace_bytes; anorm / ainvnorm
 * (nullable): 1-norms of A_i and inv(A_i); status (nullable): per-item flags.
 * perm (nullable, batch*n ints): if given, the inverse's columns are left in pivot order,
 * M_i[:, j] = inv(A_i)[:, perm_i[j]] (so inv(A_i) b = M_i[:, :n] b[perm_i]) and perm is
 * written — saves the un-permutation pass; else the columns are restored. */
long long hps_gj_workspace_bytes(int batch, int n, int ncols);
int hps_gj_invert_batched(int batch, int n, int ncols, const hps_mat_batch* M, int* piv,
                          void* workspace, double* anorm, double* ainvnorm, int* status,
                          int* perm, void* stream);

/* Leaf stage for `nleaf` leaves of one shape (p Chebyshev nodes per side, q Gauss nodes per
 * edge; m = (p-2)^2 interior, b = 4q Gauss, c = 4(p-1) exterior Chebyshev, P = p^2).
 * Outputs per leaf (contiguous batches):
 *   fs  m x (m+b) = [F_ii | S_ie]   F_ii = inv(A_ii), S_ie = -inv(A_ii) A_ie L   (retained)
 *   h   b x m     = H restricted to interior columns                          (retained)
 *   t   b x b     = T (DtN map), consumed by the parent merge                 (transient)
 *   anorm/ainvnorm: |A_ii|_1, |inv(A_ii)|_1 ; status: pivot flags. */
typedef struct {
  int nleaf, p, q;
  const double* coef;   /* [6][nleaf][P]: c11,c12,c22,c1,c2,c at the Chebyshev points */
  const double* dx;     /* p x p 1D differentiation matrices of this leaf shape */
  const double* dy;
  const double* dxx;    /* dx @ dx */
  const double* dyy;    /* dy @ dy */
  const int* int_pos;   /* [P]: index in i_ci or -1 */
  const int* ext_pos;   /* [P]: index in i_ce or -1 */
  const double* lift;   /* c x b  Gauss -> exterior Chebyshev (spectral.py:282-319) */
  const double* dfi;    /* b x m  flux extractor, interior columns */
  const double* t0;     /* b x b  flux extractor exterior columns @ lift */
  double* fs;
  double* h;
  double* t;
  double* anorm;
  double* ainvnorm;
  int* status;
  int* perm;            /* nullable: F_ii left in pivot column order, perm (nleaf x m) written
                           (see hps_gj_invert_batched); H then shares the same column order */
  void* workspace;      /* hps_leaf_workspace_bytes */
} hps_leaf_batch;
long long hps_leaf_workspace_bytes(int nleaf, int p, int q);
int hps_leaf_build(const hps_leaf_batch* b, void* stream);

/* Merge stage for `npar` parents with the same interface shape: m3 = |J3|, n1 = |J1|,
 * n2 = |J2|, e = n1 + n2. ta[i] / tb[i]: DtN maps of the children (lda / ldb columns).
 * idx + i*idx_stride: [pos1_a(n1) | pos3_a(m3) | pos2_b(n2) | pos3_b(m3)] (geometry.py:622-639).
 * Outputs (contiguous batches):
 *   xs   m3 x (m3+e) = [X | S],  X = inv(T^a_33 - T^b_33), S = X [-T^a_31 | T^b_32]  (retained)
 *   tei  e x m3      = [T^a_13 ; T^b_23]                                           (retained)
 *   tnew e x e       = blkdiag(T^a_11, T^b_22) + tei S                              (transient)
 *   dnorm/xnorm: |Delta|_1, |X|_1 ; status: pivot flags. */
typedef struct {
  int npar, m3, n1, n2;
  double* const* ta;
  double* const* tb;
  int lda, ldb;
  const int* idx;
  long long idx_stride;
  double* xs;
  double* tei;
  double* tnew;
  double* dnorm;
  double* xnorm;
  int* status;
  int* perm;            /* nullable: X left in pivot column order, perm (npar x m3) written */
  void* workspace;      /* hps_merge_workspace_bytes */
  double* delta;        /* nullable: Delta = T^a_33 - T^b_33 (npar x m3 x m3) copied out before
                           the elimination, for the reference's (lu, piv) archive sections
                           (reference archive.py:55-57) */
} hps_merge_batch;
long long hps_merge_workspace_bytes(int npar, int m3, int e);
int hps_merge_build(const hps_merge_batch* b, void* stream);

/* One batched gather-GEMV of the solve sweeps. pool: rows x nrhs vector arena (RHS fastest).
 *   x_i[k][j] = pool[xidx[i][k]][j] - (x2idx && x2idx[i][k] >= 0 ? pool[x2idx[i][k]][j] : 0)
 *   y1 = pool[oidx[i][r]][j] = sum_k A_i[r][k] x_i[k][j] + (aidx ? pool[aidx[i][r]][j] : 0)
 * Optional fused second stage (mode2), same launch:
 *   mode2 = 1 (tail):  pool[o2idx[i][r]] = A2_i x_i[K-K2 .. K)          (leaf down, exterior rows)
 *   mode2 = 2 (chain): pool[o2idx[i][r]] = A2_i y1 + pool[a2idx[i][r]]  (parent up: w3 -> h)
 *   mode2 = 3 (split): pool[o2idx[i][r]] = sum_{k < K2} A_i[r][k] x_i[k]  (R2 = R, aidx null;
 *                      parent down: u3 = [X | S][d; u_ext] also yields w3 = X d)
 * Output rows must not alias input rows within one call. nrhs <= 16. */
typedef struct {
  int nitems, R, K, nrhs;
  hps_mat_batch A;
  double* pool;
  const int* xidx;
  const int* x2idx;
  const int* aidx;
  const int* oidx;
  int mode2, R2, K2;
  hps_mat_batch A2;
  const int* a2idx;
  const int* o2idx;
  int kparts;           /* 0/1: item i is A_i (R x K). kparts > 1 (split-K, nrhs >= 3): item i is
                           the column block [(i % kparts) K, (i % kparts + 1) K) of operator
                           A_{i / kparts}, which A describes unsplit (base/stride/ld/off, no ptrs);
                           single-RHS split-K parts are addressed through A.ptrs instead */
  int kscale;           /* > 0: the gathered x_i[k] of columns k < kscale are multiplied by xscale
                           (backward Euler: the body load g = u_n / dt is read straight from the
                           leaf tabulations). Multi-RHS (nrhs >= 3) steps only. */
  double xscale;
} hps_gemv_batch;
int hps_sweep_gemv(const hps_gemv_batch* g, void* stream);

/* Time-stepping right-hand side on the leaves (timestepping.py:117-167 _RhsContext.apply):
 *   g_l[r][j] = alpha u_l[k_r][j] + beta (A u_l)[k_r][j]   at the interior nodes k_r (i_ci order),
 * A = the collocation operator with coefficient samples coef ([6][nleaf][P]; null if beta = 0).
 * u_l = u + l*u_stride (P rows x nrhs, x1-fastest grid), g_l = g + l*g_stride (m rows x nrhs).
 * Crank-Nicolson: alpha = 1/k, beta = 1/2 (operator of the parabolic problem);
 * backward Euler (config 5): alpha = 1/dt, beta = 0. */
typedef struct {
  int nleaf, p, nrhs;
  double alpha, beta;
  const double* coef;
  const double* dx;
  const double* dy;
  const double* dxx;
  const double* dyy;
  const double* u;
  long long u_stride;
  double* g;
  long long g_stride;
} hps_leaf_apply_args;
int hps_leaf_apply(const hps_leaf_apply_args* a, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HPS_B200_H */
