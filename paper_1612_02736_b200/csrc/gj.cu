// Batched blocked Gauss-Jordan inversion with partial pivoting (FP64).
//
// Replaces the reference's LU + gecon + lu_solve(I) / lu_solve(rhs) chain
// (pkg/src/specdtn/leaf.py:104-121,152-161 and solver.py:108-136): the leading n x n block
// of each M_i = [A | R] (n x ncols) is inverted in place and the trailing columns become
// inv(A) R. The pivot sequence is that of LAPACK dgetrf (the candidate rows of column j
// in GJ are exactly the rows of LU's Schur complement; ties keep the smallest row index).
//
// Per column block J = [k0, k0+kb):
//   1. gj_panel    : one CTA per matrix factors the n x kb panel in shared memory (warp
//                    argmax pivot search, row swap, scale, eliminate all other rows) giving
//                    panel = [inv(B_JJ) ; -B_RJ inv(B_JJ)] (rows J after swaps).
//   2. gj_swapcopy : applies the kb row interchanges to every other column and saves the
//                    kb pivot rows W = B_J,C (they are overwritten by step 3).
//   3. DMMA update (gemm_dmma.cu MODE_GJ_UPD): B_J,C = panel_J W,  B_R,C += panel_R W.
// Finally the column interchanges are undone: inv(A)[:, perm[j]] = M[:, j].
//
// Work: 2 n^2 ncols flops (= (2/3)n^3 LU + (4/3)n^3 inverse + 2 n^2 (ncols-n) for the RHS),
// all but the 2 n kb^2 per panel on DMMA tiles.
#include <cstdlib>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

constexpr int GJ_THREADS = 256;
// Outer block width of the two-level scheme (inner: fused kernel on the NB-column block;
// outer: row interchanges + one DMMA GEMM with K = NB over all other columns).
constexpr int GJ_OUTER_NB_DEFAULT = 64;
// Blocking schemes of the batched inversion:
//   TWO_LEVEL   fused kernel on a 64-column block (panel + update of the block), then row
//               interchanges + one K = 64 DMMA GEMM over all other columns;
//   THREE_FEW   few large matrices (top merges): the block itself is factored by narrow panels
//               (or one 8-CTA cluster per matrix) with multi-CTA updates, look-ahead on a side stream;
//   THREE_MANY  many large matrices (p = 32 leaves, 1024 x 900 x 1024): 192-wide outer blocks, each
//               factored as 64-wide fused panels + K = 64 updates inside the block, then ONE outer
//               K ~ 180 update of the other columns: a third of the read-modify-write passes over
//               the 7.4 MB matrices (leaf stage 120 -> 112 ms on the B200).
enum { GJ_TWO_LEVEL = 0, GJ_THREE_FEW = 1, GJ_THREE_MANY = 2 };
static int gj_scheme(int batch, int n) {
  static int many = -1, force3 = -1;
  if (many < 0) {
    const char* e = getenv("HPS_GJ_MANY");
    many = e ? atoi(e) : 1;
    e = getenv("HPS_GJ_THREE");  // 1: three-level (few-large form) for every blocked inversion
    force3 = e ? atoi(e) : 0;
  }
  if (force3 == 1 || batch * ((n + 255) / 256) < 64) return GJ_THREE_FEW;
  if (many && n >= 512) return GJ_THREE_MANY;
  return GJ_TWO_LEVEL;
}
static int gj_outer_nb(int batch, int n) {
  static int nb = -1;
  if (nb < 0) {
    const char* e = getenv("HPS_GJ_NB");
    nb = e ? atoi(e) : 0;
    if (nb && nb < 16) nb = 16;
    if (nb > 256) nb = 256;
  }
  if (nb) return nb;
  const int sc = gj_scheme(batch, n);
  if (sc == GJ_THREE_MANY) return 192;
  // few matrices too small for the cluster panel kernel (n <= 768, e.g. 8-16 merges of m3 = 480):
  // wider outer blocks, fewer read-modify-write passes (config 5 levels 3-4: 4.7 -> 4.4 ms)
  if (sc == GJ_THREE_FEW && n <= 768 && n >= 384 && batch > 8) return 96;
  return GJ_OUTER_NB_DEFAULT;
}
constexpr int GJ_SMEM_BUDGET = 220 * 1024;

static int gj_panel_width(int n) {
  int kb = GJ_SMEM_BUDGET / (8 * n) - 2;  // n*(kb+1) doubles of panel + pivot row + scratch
  if (kb > 32) kb = 32;
  if (kb > n) kb = n;
  if (kb > 4) kb &= ~3;
  return kb < 1 ? 1 : kb;
}

// W (batch x kb x ncols doubles) followed by the inverse column permutation (batch x n ints)
static int sm_count();
static bool gj_is_fused_full(int batch, int n) { return n <= 256 && (batch >= sm_count() || n <= 64); }

long long gj_workspace_doubles(int batch, int n, int ncols) {
  if (gj_is_fused_full(batch, n)) return 1;  // the fused kernel needs no global workspace
  return (long long)batch * gj_outer_nb(batch, n) * ncols + ((long long)batch * n + 1) / 2 + 1;
}

__global__ void __launch_bounds__(GJ_THREADS) gj_panel_kernel(int n, int k0, int kb, MatB M, int* piv,
                                                              int* status, int batch_off) {
  extern __shared__ double sm[];
  const int ldp = kb + 1;  // odd stride: row-per-thread access is bank-conflict free
  double* P = sm;
  double* prow = P + (size_t)n * ldp;
  double* rv = prow + 32;
  int* ri = reinterpret_cast<int*>(rv + 8);

  const int item = blockIdx.x + batch_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Mi = M.get(item);
  const long long ld = M.ld;

  for (int e = tid; e < n * kb; e += GJ_THREADS) {
    const int r = e / kb, c = e - r * kb;
    P[r * ldp + c] = Mi[r * ld + k0 + c];
  }
  __syncthreads();

  for (int j = 0; j < kb; ++j) {
    const int cj = k0 + j;
    double best = -1.0;
    int bi = n;
    for (int i = cj + tid; i < n; i += GJ_THREADS) {
      const double v = fabs(P[i * ldp + j]);
      if (v > best) { best = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { rv[warp] = best; ri[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = rv[0];
      int bix = ri[0];
      for (int w = 1; w < GJ_THREADS / 32; ++w)
        if (rv[w] > b || (rv[w] == b && ri[w] < bix)) { b = rv[w]; bix = ri[w]; }
      if (bix >= n) bix = cj;  // all candidates NaN: keep the diagonal, NaN propagates
      if (!(b > 0.0) && status) status[item] |= 1;
      ri[8] = bix;
      piv[(long long)item * n + cj] = bix;
    }
    __syncthreads();
    const int pr = ri[8];
    if (pr != cj && tid < kb) {
      const double t = P[pr * ldp + tid];
      P[pr * ldp + tid] = P[cj * ldp + tid];
      P[cj * ldp + tid] = t;
    }
    __syncthreads();
    if (tid < kb) {
      const double inv = 1.0 / P[cj * ldp + j];
      prow[tid] = (tid == j) ? inv : P[cj * ldp + tid] * inv;
    }
    __syncthreads();
    for (int i = tid; i < n; i += GJ_THREADS) {
      double* row = P + i * ldp;
      if (i == cj) {
        for (int jj = 0; jj < kb; ++jj) row[jj] = prow[jj];
      } else {
        const double f = row[j];
        row[j] = 0.0;
        for (int jj = 0; jj < kb; ++jj) row[jj] -= f * prow[jj];
      }
    }
    __syncthreads();
  }

  for (int e = tid; e < n * kb; e += GJ_THREADS) {
    const int r = e / kb, c = e - r * kb;
    Mi[r * ld + k0 + c] = P[r * ldp + c];
  }
}

// One thread per non-panel column: apply the panel's kb row interchanges and save the kb
// pivot rows to W. The interchanges are composed once per CTA in shared memory (rowid), so
// each column needs only independent loads: W[j] = M[rowid[k0+j]] and, for the displaced
// rows outside the panel (which always receive original panel rows), M[x] = M[rowid[x]].
// Rows inside the panel are not written: the GJ update overwrites them with panel_J W.
__global__ void gj_swapcopy_kernel(int n, int col_lo, int nlog, int kskip, int k0, int kb, MatB M, const int* piv,
                                   MatB W, int batch_off) {
  extern __shared__ int rowid[];  // n - k0 entries + moves
  int* moves = rowid + (n - k0);  // [0] count, then (dst, src)
  const int item = blockIdx.y + batch_off;
  const int* pv = piv + (long long)item * n + k0;
  for (int x = threadIdx.x; x < n - k0; x += blockDim.x) rowid[x] = x + k0;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < kb; ++j) {
      const int p = pv[j] - k0;
      const int t = rowid[j];
      rowid[j] = rowid[p];
      rowid[p] = t;
    }
    int nm = 0;
    for (int j = 0; j < kb; ++j) {
      const int x = pv[j];
      if (x >= k0 + kb && rowid[x - k0] != x) {
        moves[1 + 2 * nm] = x;
        moves[2 + 2 * nm] = rowid[x - k0];
        ++nm;
      }
    }
    moves[0] = nm;
  }
  __syncthreads();
  const int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= nlog) return;
  int c = col_lo + cl;
  if (c >= kskip) c += kb;  // the panel's own columns are skipped when they lie inside the range
  double* Mi = M.get(item);
  const long long ld = M.ld;
  double* Wi = W.get(item);
#pragma unroll 8
  for (int j = 0; j < kb; ++j) Wi[(long long)j * W.ld + c] = Mi[(long long)rowid[j] * ld + c];
  // displaced rows (after the W reads of this column: a W source can be a move destination).
  // Every move source is an original panel row and every destination lies outside the panel,
  // so the loads of a group can all be issued before its stores (8 in flight instead of one
  // dependent round trip per move)
  const int nm = moves[0];
  const int m0 = 0, m1 = nm;
  for (int mb = m0; mb < m1; mb += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (mb + u < m1) v[u] = Mi[(long long)moves[2 + 2 * (mb + u)] * ld + c];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (mb + u < m1) Mi[(long long)moves[1 + 2 * (mb + u)] * ld + c] = v[u];
  }
}

// inverse column permutation pinv (pinv[perm[j]] = j) from the LAPACK interchange list, or
// perm itself when want_perm
__global__ void gj_perm_kernel(int n, const int* piv, int* pinv, int batch_off, int want_perm) {
  extern __shared__ int perm[];
  const int item = blockIdx.x + batch_off;
  const int* pv = piv + (long long)item * n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) perm[j] = j;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) {
      const int r = pv[j];
      const int t = perm[j];
      perm[j] = perm[r];
      perm[r] = t;
    }
  }
  __syncthreads();
  int* out = pinv + (long long)item * n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    if (want_perm)
      out[j] = perm[j];
    else
      out[perm[j]] = j;
  }
}

// F[r][c] = M[r][pinv[c]] for c < n, one warp per row, row staged in shared memory
__global__ void gj_unpermute_kernel(int n, MatB M, const int* pinv, int rows_per_cta, int batch_off) {
  extern __shared__ double rowbuf[];
  const int item = blockIdx.y + batch_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  double* buf = rowbuf + (size_t)warp * n;
  double* Mi = M.get(item);
  const int* pi = pinv + (long long)item * n;
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(n, r0 + rows_per_cta);
  for (int r = r0 + warp; r < r1; r += nw) {
    double* row = Mi + (long long)r * M.ld;
    for (int c = lane; c < n; c += 32) buf[c] = row[c];
    __syncwarp();
    for (int c = lane; c < n; c += 32) row[c] = buf[pi[c]];
    __syncwarp();
  }
}

// out[item] = max_c sum_r |M[r][c]| over the leading n x n block (atomic max on the bit
// pattern: valid for non-negative doubles and lets NaN win)
__global__ void colnorm1_kernel(int n, MatB M, unsigned long long* out, int batch_off) {
  const int item = blockIdx.y + batch_off;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (c < n) {
    const double* Mi = M.get(item);
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int r = 0;
#pragma unroll 4
    for (; r + 4 <= n; r += 4) {
      s += fabs(Mi[(long long)r * M.ld + c]);
      s1 += fabs(Mi[(long long)(r + 1) * M.ld + c]);
      s2 += fabs(Mi[(long long)(r + 2) * M.ld + c]);
      s3 += fabs(Mi[(long long)(r + 3) * M.ld + c]);
    }
    for (; r < n; ++r) s += fabs(Mi[(long long)r * M.ld + c]);
    s = (s + s1) + (s2 + s3);
  }
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, s, o);
    s = (t > s || t != t) ? t : s;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = (red[w] > m || red[w] != red[w]) ? red[w] : m;
    atomicMax(out + item, (unsigned long long)__double_as_longlong(m));
  }
}

int launch_colnorm1(int batch, int n, MatB M, double* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double) * batch, s);
  for (int off = 0; off < batch; off += 65535) {
    const int nb = min(65535, batch - off);
    dim3 grid((n + 255) / 256, nb);
    colnorm1_kernel<<<grid, 256, 0, s>>>(n, M, reinterpret_cast<unsigned long long*>(out), off);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}


// Row interchanges of the panel [k0, k0+kb) applied to the columns [col_lo, col_hi) \ panel
// (the panel may lie inside or outside the range), saving the pivot rows to W.
static void swapcopy_range(int batch, int n, int col_lo, int col_hi, int k0, int kb, MatB M, const int* piv,
                           MatB W, cudaStream_t s) {
  const bool inside = k0 >= col_lo && k0 < col_hi;
  const int nlog = (col_hi - col_lo) - (inside ? kb : 0);
  if (nlog <= 0) return;
  for (int off = 0; off < batch; off += 65535) {
    const int bb = min(65535, batch - off);
    // one thread per column; few matrices: 32-thread CTAs so the pass spreads over the SMs
    const int nt = (long long)((nlog + 127) / 128) * bb >= 2 * sm_count() ? 128 : 32;
    dim3 g2((nlog + nt - 1) / nt, bb);
    gj_swapcopy_kernel<<<g2, nt, sizeof(int) * (n - k0 + 2 * kb + 4), s>>>(n, col_lo, nlog, inside ? k0 : (1 << 30),
                                                                           k0, kb, M, piv, W, off);
  }
}

// DMMA trailing update of the columns [c_lo, c_hi) by the factored panel [k0, k0+kb); the panel
// columns are skipped when they lie inside the range.
static int gemm_range(int batch, int n, int c_lo, int c_hi, int k0, int kb, MatB M, MatB W, cudaStream_t s) {
  const bool inside = k0 >= c_lo && k0 < c_hi;
  const int nlog = (c_hi - c_lo) - (inside ? kb : 0);
  if (nlog <= 0) return 0;
  GemmArgs g{};
  g.M = n;
  g.N = nlog;
  g.K = kb;
  g.alpha = 1.0;
  g.beta = 1.0;
  g.A = M;
  g.A.off = M.off + k0;
  g.B = W;
  g.B.off = W.off + c_lo;
  g.C = M;
  g.C.off = M.off + c_lo;
  g.k0 = k0;
  g.kb = kb;
  g.kc = inside ? k0 - c_lo : (1 << 30);
  return launch_gemm(g, batch, MODE_GJ_UPD, s);
}

static int update_range(int batch, int n, int col_lo, int col_hi, int k0, int kb, MatB M, const int* piv,
                        MatB W, cudaStream_t s) {
  swapcopy_range(batch, n, col_lo, col_hi, k0, kb, M, piv, W, s);
  return gemm_range(batch, n, col_lo, col_hi, k0, kb, M, W, s);
}

// Side stream + events for the look-ahead (created once, reused; stream-ordered use only).
struct Lookahead {
  cudaStream_t side = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  bool ok = false;
  Lookahead() {
    // highest priority: the latency-bound block factorisation gets SMs first as the
    // trailing-update GEMM's CTAs retire
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    ok = cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming) == cudaSuccess;
  }
};

// Factor the NB-column block starting at K0 (pivot columns [K0, K0+nb), columns of the block
// only): one fused CTA per matrix, or for few large matrices panel-only fused launches plus
// multi-CTA updates inside the block.
static int factor_block(int batch, int n, int ncols, int K0, int nb, int scheme, MatB M, int* piv,
                        int* status, MatB W, cudaStream_t s) {
  const bool three_level = scheme != GJ_TWO_LEVEL;
  int rc;
  static int use_cluster = -1;
  if (use_cluster < 0) {
    const char* e = getenv("HPS_GJ_CLUSTER");
    use_cluster = e ? atoi(e) : 1;
  }
  // the 8-CTA cluster panel: large n, or medium n (>= 384) with at most 8 matrices (config 5
  // level 3: 4.54 -> 4.23 ms; with 16 matrices the fused panels win)
  if (scheme == GJ_THREE_FEW && use_cluster && (n > 768 || batch <= 8) && gj_cluster_ok(n, nb))
    return launch_gj_cluster(batch, n, K0, nb, M, piv, status, s);
  const int kin = scheme == GJ_THREE_FEW ? gj_fused_panel_width(n, 0) : (scheme == GJ_THREE_MANY ? 64 : nb);
  for (int k0 = K0; k0 < K0 + nb; k0 += kin) {
    const int kb = min(kin, K0 + nb - k0);
    FusedArgs f{};
    f.batch = batch;
    f.n = n;
    f.ncols = ncols;
    f.M = M;
    f.piv = piv;
    f.status = status;
    f.k_begin = k0;
    f.k_end = k0 + kb;
    f.col_lo = three_level ? k0 : K0;
    f.col_hi = three_level ? k0 + kb : K0 + nb;
    f.full = 0;
    if ((rc = launch_gj_fused(f, batch, s))) return rc;
    if (three_level && (rc = update_range(batch, n, K0, K0 + nb, k0, kb, M, piv, W, s))) return rc;
  }
  return 0;
}

int gj_invert(int batch, int n, int ncols, MatB M, int* piv, double* wbuf, double* anorm,
              double* ainvnorm, int* status, cudaStream_t s, int* perm_out) {
  if (batch <= 0 || n <= 0) return 0;
  const int sms = sm_count();
  const bool fused_full = gj_is_fused_full(batch, n);
  if (fused_full) {
    // |A|_1 as a separate bandwidth-bound pass: inside the persistent kernel the column sums
    // were a latency-bound sweep over each matrix (~13 % of its time at n = 196)
    if (anorm) {
      const int rc = launch_colnorm1(batch, n, M, anorm, s);
      if (rc) return rc;
    }
    FusedArgs f{};
    f.batch = batch;
    f.n = n;
    f.ncols = ncols;
    f.M = M;
    f.piv = piv;
    f.status = status;
    f.anorm = nullptr;
    f.ainvnorm = ainvnorm;
    f.k_begin = 0;
    f.k_end = n;
    f.col_lo = 0;
    f.col_hi = ncols;
    f.full = 1;
    f.perm_out = perm_out;
    static int per_sm = -1;
    if (per_sm < 0) {
      const char* e = getenv("HPS_GJ_FUSED_PER_SM");
      per_sm = e ? atoi(e) : 2;
    }
    if (gj_la_ok(n, ncols) && batch >= sms) return launch_gj_la(f, s);
    if (gj_pair_ok(n, ncols)) return launch_gj_pair(f, s);
    const int grid = batch < per_sm * sms ? batch : per_sm * sms;
    return launch_gj_fused(f, grid, s);
  }
  if (anorm) {
    int rc = launch_colnorm1(batch, n, M, anorm, s);
    if (rc) return rc;
  }
  // few large matrices: the inner level is itself split (panel-only fused kernel + multi-CTA
  // update of the block) so the whole GPU works on each block instead of one SM per matrix
  const int scheme = gj_scheme(batch, n);
  const bool three_level = scheme != GJ_TWO_LEVEL;
  // equal outer blocks (multiple of 4) so no narrow tail update is left over; many matrices
  // use K = 128 outer updates (half the read-modify-write passes over the trailing columns)
  const int nbmax = gj_outer_nb(batch, n);
  const int nblk = (n + nbmax - 1) / nbmax;
  const int NB = (((n + nblk - 1) / nblk) + 3) & ~3;
  MatB W{wbuf, (long long)NB * ncols, nullptr, ncols, 0};
  // Look-ahead: once block K0's interchanges and the update of the NEXT block's columns are
  // done, the next block is factored on a side stream while the main stream updates the
  // remaining columns (disjoint column sets) — the latency-bound panel work hides under the
  // bandwidth/compute-bound trailing GEMM.
  static Lookahead la;
  static int la_mode = -1;  // HPS_GJ_LOOKAHEAD: 0 never, 1 few-large only (default), 2 always
  if (la_mode < 0) {
    const char* e = getenv("HPS_GJ_LOOKAHEAD");
    la_mode = e ? atoi(e) : 1;
  }
  const bool use_la = la.ok && (la_mode == 2 || (la_mode == 1 && scheme == GJ_THREE_FEW));
  int rc;
  if ((rc = factor_block(batch, n, ncols, 0, min(NB, n), scheme, M, piv, status, W, s))) return rc;
  for (int K0 = 0; K0 < n; K0 += NB) {
    const int nb = min(NB, n - K0);
    const int K1 = K0 + nb;
    const int nb1 = min(NB, n - K1);
    // with look-ahead the next block's columns get their interchanges + update first, so the
    // side stream starts factoring them while the main stream swaps and updates all the others
    // (the full-width interchange pass was ~35 us per block on the critical path of the top merges)
    const bool early = use_la && nb1 > 0;
    if (early) {
      swapcopy_range(batch, n, K1, K1 + nb1, K0, nb, M, piv, W, s);
    } else {
      swapcopy_range(batch, n, 0, ncols, K0, nb, M, piv, W, s);
    }
    if (nb1 > 0) {
      if ((rc = gemm_range(batch, n, K1, K1 + nb1, K0, nb, M, W, s))) return rc;
      if (use_la) {
        cudaEventRecord(la.ev_a, s);
        cudaStreamWaitEvent(la.side, la.ev_a, 0);
        if ((rc = factor_block(batch, n, ncols, K1, nb1, scheme, M, piv, status, W, la.side))) return rc;
        cudaEventRecord(la.ev_b, la.side);
        swapcopy_range(batch, n, 0, K1, K0, nb, M, piv, W, s);
        swapcopy_range(batch, n, K1 + nb1, ncols, K0, nb, M, piv, W, s);
      }
    }
    if ((rc = gemm_range(batch, n, 0, K0, K0, nb, M, W, s))) return rc;
    if ((rc = gemm_range(batch, n, K1 + (nb1 > 0 ? nb1 : 0), ncols, K0, nb, M, W, s))) return rc;
    if (nb1 > 0) {
      if (use_la)
        cudaStreamWaitEvent(s, la.ev_b, 0);
      else if ((rc = factor_block(batch, n, ncols, K1, nb1, scheme, M, piv, status, W, s)))
        return rc;
    }
  }
  // undo the column interchanges of the inverse block (pinv lives in the workspace after W)
  int* pinv = reinterpret_cast<int*>(wbuf + (size_t)batch * gj_outer_nb(batch, n) * ncols);
  for (int off = 0; off < batch; off += 65535) {
    const int bb = min(65535, batch - off);
    if (perm_out) {
      gj_perm_kernel<<<bb, 128, sizeof(int) * n, s>>>(n, piv, perm_out, off, 1);
      continue;
    }
    gj_perm_kernel<<<bb, 128, sizeof(int) * n, s>>>(n, piv, pinv, off, 0);
    const int rows_per_cta = 32;
    const size_t usmem = sizeof(double) * (size_t)n * 4;
    if (usmem > 48 * 1024)
      cudaFuncSetAttribute(gj_unpermute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usmem);
    dim3 g3((n + rows_per_cta - 1) / rows_per_cta, bb);
    gj_unpermute_kernel<<<g3, 128, usmem, s>>>(n, M, pinv, rows_per_cta, off);
  }
  if (ainvnorm) {
    int rc = launch_colnorm1(batch, n, M, ainvnorm, s);
    if (rc) return rc;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
