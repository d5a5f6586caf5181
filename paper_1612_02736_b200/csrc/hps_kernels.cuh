// Internal launch interface shared by the kernel translation units and the C-ABI layer.
#pragma once
#include "hps_common.cuh"

namespace hps {

enum { MODE_GEMM = 0, MODE_GJ_UPD = 1 };

struct GemmArgs {
  int M, N, K;
  double alpha, beta;
  MatB A, B, C;
  const double* bias;  // MODE_GEMM: optional M x N matrix shared by the batch, added in the epilogue
  int ldbias;
  int k0, kb;          // MODE_GJ_UPD: pivot rows [k0, k0+kb) get beta = 0
  int kc;              // MODE_GJ_UPD: logical column where the kb panel columns are skipped
};

int launch_gemm(const GemmArgs& g, int batch, int mode, cudaStream_t s);

// Blocked Gauss-Jordan inversion with partial pivoting of the leading n x n block of each
// M_i (n x ncols, row-major, ld); the trailing ncols-n columns are right-hand sides that end
// up multiplied by the inverse. piv: batch x n (LAPACK-style row interchanges), wbuf:
// workspace (see gj_workspace_doubles). On exit M_i[:, :n] = inv(A_i) (columns un-permuted),
// M_i[:, n:] = inv(A_i) * rhs_i. anorm/ainvnorm (may be null): 1-norms before/after.
long long gj_workspace_doubles(int batch, int n, int ncols);
// perm_out (nullable): leave the inverse's columns permuted, M[:, j] = inv(A)[:, perm[j]], and
// write perm (batch x n); consumers then gather right-hand sides as x[j] = b[perm[j]].
int gj_invert(int batch, int n, int ncols, MatB M, int* piv, double* wbuf, double* anorm,
              double* ainvnorm, int* status, cudaStream_t s, int* perm_out = nullptr);

int launch_colnorm1(int batch, int n, MatB M, double* out, cudaStream_t s);

struct FusedArgs {
  int batch, n, ncols;
  MatB M;
  int* piv;            // batch x n
  int* status;
  double* anorm;       // full mode only
  double* ainvnorm;
  int k_begin, k_end;  // pivot columns processed
  int col_lo, col_hi;  // columns updated (must contain [k_begin, k_end))
  int full;            // 1: norms + column un-permutation
  int* perm_out;       // full mode: if set, columns stay permuted and perm (batch x n) is written
  int ldp, ldw, cw;    // set by the launcher
};
int gj_fused_panel_width(int n, int full);
// cluster block factorisation for few large matrices (gj_cluster.cu)
bool gj_cluster_ok(int n, int nb);
int launch_gj_cluster(int batch, int n, int k0, int nb, MatB M, int* piv, int* status, cudaStream_t s);
int launch_gj_fused(const FusedArgs& a, int grid, cudaStream_t s);
// small matrices resident in a 2-CTA cluster's shared memory (gj_pair.cu; full mode)
bool gj_pair_ok(int n, int ncols);
int launch_gj_pair(const FusedArgs& a, cudaStream_t s);
// warp-specialised look-ahead kernel for the p = 16 leaf blocks (gj_la.cu; full mode)
bool gj_la_ok(int n, int ncols);
int launch_gj_la(const FusedArgs& a, cudaStream_t s);

// Leaf-stage assembly: interior rows of the collocation matrix for each leaf.
struct LeafAsmArgs {
  int nleaf, p;
  const double* coef;      // [6][nleaf][p*p]
  const double* dx;        // p x p 1D operators of this leaf shape
  const double* dy;
  const double* dxx;
  const double* dyy;
  const int* int_pos;      // [p*p] position in i_ci or -1
  const int* ext_pos;      // [p*p] position in i_ce or -1
  MatB Aii;                // m x (m+b) (only the first m columns written)
  MatB Aie;                // m x c
  double* colpart;         // nullable: [nleaf][row blocks][m] partial column sums of |A_ii|
  double* anorm;           // with colpart: |A_ii|_1 per leaf (leaf_assemble_rows() rows per block)
};
int leaf_assemble_rows(int p, int q);  // rows per CTA = row blocks of colpart
int launch_leaf_assemble(const LeafAsmArgs& a, cudaStream_t s);
// fused assembly + right-hand sides FS[:, m:] = -A_ie L (A_ie stays on chip); -1: not applicable
int launch_leaf_assemble_fused(const LeafAsmArgs& a, MatB FS, const double* lift, int q, cudaStream_t s);

// Merge gather: builds [Delta | -Ta31 | Tb32], Tei = [Ta13; Tb23], Tnew = blkdiag(Ta11, Tb22)
struct MergeGatherArgs {
  int npar, m3, n1, n2;
  MatB Ta, Tb;              // child DtN maps (ld = child exterior size)
  const int* idx;           // per parent: [p1a(n1) | p3a(m3) | p2b(n2) | p3b(m3)]
  long long idx_stride;     // 0 when all parents share one index set
  MatB XS;                  // m3 x (m3 + e)
  MatB Tei;                 // e x m3
  MatB Tnew;                // e x e
};
int launch_merge_gather(const MergeGatherArgs& a, cudaStream_t s);

// Solve-stage batched gather-GEMV: for item i, rows r < R, rhs j < nrhs:
//   y[oidx[i][r]][j] = sum_k A_i[r][k] * x_i[k][j] + (aidx ? pool[aidx[i][r]][j] : 0)
//   x_i[k][j] = pool[xidx[i][k]][j] - (x2idx ? pool[x2idx[i][k]][j] : 0)
// pool is a single (rows x nrhs) vector arena; every index is an absolute pool row.
struct GemvArgs {
  int nitems, R, K, nrhs;
  MatB A;
  double* pool;
  const int* xidx;   // [nitems][K]
  const int* x2idx;  // [nitems][K] or null
  const int* aidx;   // [nitems][R] or null
  const int* oidx;   // [nitems][R]
  // optional second stage: 1 = tail  y2 = A2 x[K-K2:K)   (leaf down: exterior rows = L u_ge)
  //                        2 = chain y2 = A2 y1 + add2   (parent up: h = T_ei w3 + [h_a; h_b])
  int mode2, R2, K2;
  MatB A2;
  const int* a2idx;  // [nitems][R2] or null
  const int* o2idx;  // [nitems][R2]
  long long xstride; // per-item stride of xidx/x2idx (default K) and of aidx/oidx (default R)
  long long ostride;
  int pre_mask;      // which kernels load static gather indices before the launch wait
                     // (bit mask, HPS_PRE_INDEX, set per launch by launch_gemv_gather)
  int kparts;        // split-K: item i = column block i % kparts of operator i / kparts (ABI)
  int kscale;        // x columns k < kscale are scaled by xscale after the gather (ABI)
  double xscale;
};
// Operator rows of item i, split-K aware (multi-RHS kernels; the single-RHS kernels address
// split-K parts through per-part pointer arrays, which keeps their hot loops branch-free)
__device__ __forceinline__ const double* gemv_a(const GemvArgs& a, int i) {
  return a.kparts > 1 ? a.A.get(i / a.kparts) + (long long)(i % a.kparts) * a.K : a.A.get(i);
}
int launch_gemv_gather(const GemvArgs& a, cudaStream_t s);
// programmatic dependent launch for a step with this many right-hand sides on a persistent (one
// CTA per SM, TMA-fed) or many-CTA kernel (HPS_PDL; sweep.cu)
bool sweep_pdl_for(int nrhs, bool persistent);
// TMA-fed multi-RHS path for large leaf levels (sweep_tma.cu); false = not applicable
bool launch_gemv_tma(const GemvArgs& a, cudaStream_t s);
// TMA-streamed multi-RHS path for large operator items (top levels, split-K parts; sweep_tma.cu)
bool launch_gemv_stream(const GemvArgs& a, cudaStream_t s);

// Leaf operator application for time stepping (leaf_apply.cu)
struct LeafApplyArgs {
  int nleaf, p, nrhs;
  double alpha, beta;
  const double* coef;   // [6][nleaf][P] or null when beta == 0
  const double* dx;
  const double* dy;
  const double* dxx;
  const double* dyy;
  const double* u;      // leaf l: u + l*u_stride, P rows x nrhs
  long long u_stride;
  double* g;            // leaf l: g + l*g_stride, m rows x nrhs
  long long g_stride;
};
int launch_leaf_apply(const LeafApplyArgs& a, cudaStream_t s);

}  // namespace hps
