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
#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

constexpr int GJ_THREADS = 256;
constexpr int GJ_SMEM_BUDGET = 220 * 1024;

static int gj_panel_width(int n) {
  int kb = GJ_SMEM_BUDGET / (8 * n) - 2;  // n*(kb+1) doubles of panel + pivot row + scratch
  if (kb > 32) kb = 32;
  if (kb > n) kb = n;
  if (kb > 4) kb &= ~3;
  return kb < 1 ? 1 : kb;
}

// W (batch x kb x ncols doubles) followed by the inverse column permutation (batch x n ints)
long long gj_workspace_doubles(int batch, int n, int ncols) {
  return (long long)batch * 64 * ncols + ((long long)batch * n + 1) / 2 + 1;
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
__global__ void gj_swapcopy_kernel(int n, int ncols, int k0, int kb, MatB M, const int* piv, MatB W,
                                   int batch_off) {
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
  if (cl >= ncols - kb) return;
  const int c = cl < k0 ? cl : cl + kb;
  double* Mi = M.get(item);
  const long long ld = M.ld;
  double* Wi = W.get(item);
#pragma unroll 8
  for (int j = 0; j < kb; ++j) Wi[(long long)j * W.ld + c] = Mi[(long long)rowid[j] * ld + c];
  const int nm = moves[0];
  for (int m = 0; m < nm; ++m) {
    const int dst = moves[1 + 2 * m], src = moves[2 + 2 * m];
    Mi[(long long)dst * ld + c] = Mi[(long long)src * ld + c];
  }
}

// inverse column permutation pinv (pinv[perm[j]] = j) from the LAPACK interchange list
__global__ void gj_perm_kernel(int n, const int* piv, int* pinv, int batch_off) {
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
  for (int j = threadIdx.x; j < n; j += blockDim.x) out[perm[j]] = j;
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
    for (int r = 0; r < n; ++r) s += fabs(Mi[(long long)r * M.ld + c]);
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

// Outer block width of the two-level scheme (inner: fused kernel on the NB-column block;
// outer: row interchanges + one DMMA GEMM with K = NB over all other columns).
constexpr int GJ_OUTER_NB = 64;

int gj_invert(int batch, int n, int ncols, MatB M, int* piv, double* wbuf, double* anorm,
              double* ainvnorm, int* status, cudaStream_t s) {
  if (batch <= 0 || n <= 0) return 0;
  const int sms = sm_count();
  const bool fused_full = n <= 256 && (batch >= sms || n <= 64);
  if (fused_full) {
    FusedArgs f{};
    f.batch = batch;
    f.n = n;
    f.ncols = ncols;
    f.M = M;
    f.piv = piv;
    f.status = status;
    f.anorm = anorm;
    f.ainvnorm = ainvnorm;
    f.k_begin = 0;
    f.k_end = n;
    f.col_lo = 0;
    f.col_hi = ncols;
    f.full = 1;
    const int grid = batch < 2 * sms ? batch : 2 * sms;
    return launch_gj_fused(f, grid, s);
  }
  if (anorm) {
    int rc = launch_colnorm1(batch, n, M, anorm, s);
    if (rc) return rc;
  }
  // equal outer blocks (multiple of 4, <= 64) so no narrow tail update is left over
  const int nblk = (n + GJ_OUTER_NB - 1) / GJ_OUTER_NB;
  const int NB = (((n + nblk - 1) / nblk) + 3) & ~3;
  MatB W{wbuf, (long long)NB * ncols, nullptr, ncols, 0};
  for (int K0 = 0; K0 < n; K0 += NB) {
    const int nb = min(NB, n - K0);
    FusedArgs f{};
    f.batch = batch;
    f.n = n;
    f.ncols = ncols;
    f.M = M;
    f.piv = piv;
    f.status = status;
    f.k_begin = K0;
    f.k_end = K0 + nb;
    f.col_lo = K0;
    f.col_hi = K0 + nb;
    f.full = 0;
    int rc = launch_gj_fused(f, batch, s);
    if (rc) return rc;
    if (ncols > nb) {
      for (int off = 0; off < batch; off += 65535) {
        const int bb = min(65535, batch - off);
        dim3 g2((ncols - nb + 127) / 128, bb);
        gj_swapcopy_kernel<<<g2, 128, sizeof(int) * (n - K0 + 2 * nb + 4), s>>>(n, ncols, K0, nb, M, piv, W, off);
      }
      GemmArgs g{};
      g.M = n;
      g.N = ncols - nb;
      g.K = nb;
      g.alpha = 1.0;
      g.beta = 1.0;
      g.A = M;
      g.A.off = M.off + K0;
      g.B = W;
      g.C = M;
      g.k0 = K0;
      g.kb = nb;
      if ((rc = launch_gemm(g, batch, MODE_GJ_UPD, s))) return rc;
    }
  }
  // undo the column interchanges of the inverse block (pinv lives in the workspace after W)
  int* pinv = reinterpret_cast<int*>(wbuf + (size_t)batch * NB * ncols);
  for (int off = 0; off < batch; off += 65535) {
    const int bb = min(65535, batch - off);
    gj_perm_kernel<<<bb, 128, sizeof(int) * n, s>>>(n, piv, pinv, off);
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
