// Block factorisation for FEW LARGE matrices (top-of-tree merges): one thread-block cluster of
// CL CTAs per matrix holds the n x nb column block in distributed shared memory (CTA c owns rows
// [c*rl, (c+1)*rl)), and runs Gauss-Jordan with partial pivoting column by column:
//   1. every CTA finds its best candidate row (|value|, ties -> smallest row) and publishes it,
//   2. cluster barrier; every CTA reads the CL candidates through DSMEM and picks the winner
//      (LAPACK rule), then copies the pivot row and the displaced row cj into local buffers,
//   3. cluster barrier; every CTA eliminates its own rows over the nb block columns, the owners
//      of rows cj / pr write the scaled pivot row / the displaced row.
// Two cluster barriers per column and no global traffic inside the block; the whole GPU works
// on the trailing update afterwards (gj.cu). Replaces, for batch x ceil(n/256) < 64, the
// one-SM-per-matrix inner level whose latency dominated the root merges.
#include <cooperative_groups.h>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace cg = cooperative_groups;

namespace hps {

constexpr int GC_CL = 8;         // CTAs per cluster (portable size)
constexpr int GC_THREADS = 256;
constexpr int GC_NBMAX = 64;

struct GcArgs {
  int batch, n, k0, nb;
  MatB M;
  int* piv;
  int* status;
  int rl;  // rows per CTA
};

__global__ void __cluster_dims__(GC_CL, 1, 1) __launch_bounds__(GC_THREADS, 1) gj_cluster_kernel(GcArgs a) {
  extern __shared__ double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int item = blockIdx.x / GC_CL;
  const int n = a.n, nb = a.nb, k0 = a.k0, rl = a.rl;
  const int ldb = nb + 1;                       // odd stride: conflict-free row-wise access
  constexpr int SL = 2 + 2 * GC_NBMAX;          // slot: best value, best row, candidate row, row cj
  double* B = sm;                               // rl x ldb  (own rows of the block)
  double* slots = B + (size_t)rl * ldb;         // [2][SL]  double-buffered per column parity
  double* prow = slots + 2 * SL;                // scaled pivot row (local)
  double* drow = prow + GC_NBMAX;               // displaced row cj (local)
  double* red = drow + GC_NBMAX;                // [warps][2]
  int* sel = reinterpret_cast<int*>(red + 2 * (GC_THREADS / 32));  // [2]: pr, owner
  int* spiv = sel + 2;                          // [nb] pivots, written to global at the end
                                                // (a global store inside the loop would make
                                                // every cluster barrier's release wait for it)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Mi = a.M.get(item);
  const long long ld = a.M.ld;
  const int r0 = rank * rl;

  for (int e = tid; e < rl * nb; e += GC_THREADS) {
    const int r = e / nb, c = e - r * nb;
    const int gi = r0 + r;
    B[r * ldb + c] = gi < n ? Mi[gi * ld + k0 + c] : 0.0;
  }
  __syncthreads();
  int flag = 0;
  for (int j = 0; j < nb; ++j) {
    const int cj = k0 + j;
    double* myslot = slots + (j & 1) * SL;
    // 1. local candidate among own rows gi >= cj
    double best = -1.0;
    int bi = n;
    for (int r = tid; r < rl; r += GC_THREADS) {
      const int gi = r0 + r;
      if (gi < n && gi >= cj) {
        const double v = fabs(B[r * ldb + j]);
        if (v > best) { best = v; bi = gi; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) {
      red[2 * warp] = best;
      red[2 * warp + 1] = (double)bi;
    }
    __syncthreads();
    // every warp reduces the 8 warp results itself (no extra barrier)
    {
      double b = red[0];
      int bix = (int)red[1];
#pragma unroll
      for (int w = 1; w < GC_THREADS / 32; ++w) {
        const double vw = red[2 * w];
        const int iw = (int)red[2 * w + 1];
        if (vw > b || (vw == b && iw < bix)) { b = vw; bix = iw; }
      }
      if (tid == 0) {
        myslot[0] = b;
        myslot[1] = (double)bix;
      }
      // 2. publish the candidate row and, if owned, the row cj (slots only: B can be
      //    overwritten right after the single cluster barrier)
      if (bix < n && bix >= r0 && bix < r0 + rl)
        for (int c = tid; c < nb; c += GC_THREADS) myslot[2 + c] = B[(bix - r0) * ldb + c];
      if (cj >= r0 && cj < r0 + rl)
        for (int c = tid; c < nb; c += GC_THREADS) myslot[2 + GC_NBMAX + c] = B[(cj - r0) * ldb + c];
    }
    cluster.sync();  // the only cluster barrier per column
    // 3. winner over the CL candidates: lanes 0..CL-1 of warp 0 read one remote slot each
    if (warp == 0) {
      double vc = -2.0;
      int ic = n;
      if (lane < GC_CL) {
        const double* rs = cluster.map_shared_rank(myslot, lane);
        vc = rs[0];
        ic = (int)rs[1];
      }
      int oc = lane;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, vc, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ic, o);
        const int oo = __shfl_xor_sync(0xffffffffu, oc, o);
        if (ov > vc || (ov == vc && oi < ic)) { vc = ov; ic = oi; oc = oo; }
      }
      if (lane == 0) {
        if (ic >= n) ic = -1;  // all NaN: keep the diagonal (row cj)
        sel[0] = ic;
        sel[1] = oc;
        if (!(vc > 0.0)) flag = 1;
      }
    }
    __syncthreads();
    int pr = sel[0];
    const int owner = sel[1];
    const int owner_cj = cj / rl;
    if (pr < 0) pr = cj;
    {
      const double* dsl = cluster.map_shared_rank(myslot, owner_cj) + 2 + GC_NBMAX;
      const double* psl = cluster.map_shared_rank(myslot, owner) + 2;
      for (int c = tid; c < nb; c += GC_THREADS) {
        const double d = dsl[c];
        drow[c] = d;
        prow[c] = (pr == cj) ? d : psl[c];
      }
    }
    if (tid == 0) spiv[j] = pr;
    __syncthreads();
    const double inv = 1.0 / prow[j];
    __syncthreads();
    for (int c = tid; c < nb; c += GC_THREADS) prow[c] = (c == j) ? inv : prow[c] * inv;
    __syncthreads();
    // 4. eliminate own rows: two threads per row, 32 columns each, all loads issued first
    for (int e = tid; e < 2 * rl; e += GC_THREADS) {
      const int r = e >> 1, part = e & 1;
      const int gi = r0 + r;
      if (gi >= n) continue;
      double* row = B + r * ldb;
      const int c0 = part * 32;
      const double* src = (gi == pr && gi != cj) ? drow : row;
      double v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = (c0 + u < nb) ? src[c0 + u] : 0.0;
      if (gi == cj) {
#pragma unroll
        for (int u = 0; u < 32; ++u)
          if (c0 + u < nb) row[c0 + u] = prow[c0 + u];
        continue;
      }
      const double f = src[j];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int c = c0 + u;
        if (c < nb) row[c] = (c == j ? 0.0 : v[u]) - f * prow[c];
      }
    }
    __syncthreads();
  }
  cluster.sync();
  for (int e = tid; e < rl * nb; e += GC_THREADS) {
    const int r = e / nb, c = e - r * nb;
    const int gi = r0 + r;
    if (gi < n) Mi[gi * ld + k0 + c] = B[r * ldb + c];
  }
  if (rank == 0)
    for (int j = tid; j < nb; j += GC_THREADS) a.piv[(long long)item * n + k0 + j] = spiv[j];
  if (tid == 0 && rank == 0 && flag && a.status) a.status[item] |= 1;
}

size_t gj_cluster_smem(int n, int nb) {
  const int rl = (n + GC_CL - 1) / GC_CL;
  return sizeof(double) * ((size_t)rl * (nb + 1) + 2 * (2 + 2 * GC_NBMAX) + 2 * GC_NBMAX + 2 * (GC_THREADS / 32) + 2 +
                           GC_NBMAX / 2 + 2);
}

// measured faster than the three-level fused path only for n >= ~900 (root and level-1 merges)
bool gj_cluster_ok(int n, int nb) { return n > 768 && nb <= GC_NBMAX && gj_cluster_smem(n, nb) <= 200 * 1024; }

int launch_gj_cluster(int batch, int n, int k0, int nb, MatB M, int* piv, int* status, cudaStream_t s) {
  if (!gj_cluster_ok(n, nb)) return 1;
  GcArgs a{};
  a.batch = batch;
  a.n = n;
  a.k0 = k0;
  a.nb = nb;
  a.M = M;
  a.piv = piv;
  a.status = status;
  a.rl = (n + GC_CL - 1) / GC_CL;
  const size_t smem = gj_cluster_smem(n, nb);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gj_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  gj_cluster_kernel<<<batch * GC_CL, GC_THREADS, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
