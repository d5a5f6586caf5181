#include <cstdlib>
// Block factorisation for FEW LARGE matrices (top-of-tree merges): one thread-block cluster of
// CL CTAs per matrix holds the n x nb column block in distributed shared memory (CTA c owns rows
// [c*rl, (c+1)*rl)), and runs Gauss-Jordan with partial pivoting column by column:
//   1. every CTA finds its best candidate row (|value|, ties -> smallest row) and publishes it
//      together with the row currently at the pivot position,
//   2. one cluster barrier; every CTA reads the CL candidates through DSMEM and picks the winner
//      (LAPACK rule), then swaps / eliminates its own rows.
// The elimination is blocked (SB = 8 columns): inside a sub-block only its 8 columns are
// eliminated (row interchanges are applied to all nb columns at once), and at the end of the
// sub-block the other nb - 8 columns get the accumulated transform as one DMMA product
//     C <- D C + W C_piv     (W: the sub-block's n x 8 GJ multipliers, C_piv: its 8 pivot
//                             rows before the transform, D: identity with pivot rows zeroed)
// — the same identity the outer blocked scheme (gj.cu) uses with K = nb. Per column that leaves
// a 8-wide rank-1 update instead of a 64-wide one (the r01 profile had the 64-wide scalar
// elimination at ~40 % of the kernel's stall samples, 373 us per 1920 x 64 block).
// The whole GPU works on the trailing update afterwards (gj.cu). Replaces, for batch x
// ceil(n/256) < 64, the one-SM-per-matrix inner level whose latency dominated the root merges.
#include <cooperative_groups.h>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace cg = cooperative_groups;

namespace hps {

#ifdef GC_PROFILE
__device__ long long gc_prof[8];
#define GC_T(i)                                                  \
  if (threadIdx.x == 0 && blockIdx.x == 0) {                     \
    const long long now = clock64();                             \
    gc_prof[i] += now - gc_last;                                 \
    gc_last = now;                                               \
  }
#else
#define GC_T(i)
#endif

// CTAs per cluster: 8 (portable) or 16 (non-portable, opt-in; HPS_GJ_CL=16)
constexpr int GC_THREADS = 256;
constexpr int GC_NBMAX = 64;
constexpr int GC_SB = 8;         // sub-block width

struct GcArgs {
  int batch, n, k0, nb;
  MatB M;
  int* piv;
  int* status;
  int rl;  // rows per CTA
};

// shared-memory layout (doubles) shared by the kernel and gj_cluster_smem
template <int CL>
struct GcLayout {
  int rl, nb, ldb;
  __host__ __device__ GcLayout(int rl_, int nb_) : rl(rl_), nb(nb_), ldb(nb_ + 1) {}
  static constexpr int BOX = 2 + GC_NBMAX;                           // best, row id, candidate row
  __host__ __device__ size_t b() const { return 0; }                   // rl x ldb own rows
  __host__ __device__ size_t box() const { return (size_t)rl * ldb; }  // [2][CL][BOX] inbox
  __host__ __device__ size_t cjrow() const { return box() + 2 * CL * BOX; }  // [2][NBMAX]
  __host__ __device__ size_t cp() const { return cjrow() + 2 * GC_NBMAX; }      // [SB][NBMAX+1]
  __host__ __device__ size_t red() const { return cp() + GC_SB * (GC_NBMAX + 1); }  // [warps][2]
  __host__ __device__ size_t ints() const { return red() + 2 * (GC_THREADS / 32); }  // spiv[nb]
  __host__ __device__ size_t total() const { return ints() + GC_NBMAX / 2 + 1; }
};

template <int CL>
__global__ void __launch_bounds__(GC_THREADS, 1) gj_cluster_kernel(GcArgs a) {
  extern __shared__ double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int item = blockIdx.x / CL;
  const int n = a.n, nb = a.nb, k0 = a.k0, rl = a.rl;
  const GcLayout<CL> L(rl, nb);
  const int ldb = L.ldb;
  constexpr int BOX = GcLayout<CL>::BOX;
  constexpr int CPLD = GC_NBMAX + 1;
  double* B = sm + L.b();
  double* box = sm + L.box();
  double* cjrow = sm + L.cjrow();
  double* cp = sm + L.cp();
  double* red = sm + L.red();
  int* spiv = reinterpret_cast<int*>(sm + L.ints());  // pivots, written to global at the end
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Mi = a.M.get(item);
  const long long ld = a.M.ld;
  const int r0 = rank * rl;
  // warp w pushes this CTA's candidate (and row cj when owned) into CTA w's inbox
  // (CL = 16: warp w also serves CTA w + 8)
  double* peer_box = cluster.map_shared_rank(box, warp);
  double* peer_cj = cluster.map_shared_rank(cjrow, warp);
  double* peer_box2 = CL > 8 ? cluster.map_shared_rank(box, warp + 8) : nullptr;
  double* peer_cj2 = CL > 8 ? cluster.map_shared_rank(cjrow, warp + 8) : nullptr;

  for (int e = tid; e < rl * nb; e += GC_THREADS) {
    const int r = e / nb, c = e - r * nb;
    const int gi = r0 + r;
    B[r * ldb + c] = gi < n ? Mi[gi * ld + k0 + c] : 0.0;
  }
  __syncthreads();
#ifdef GC_PROFILE
  long long gc_last = clock64();
#endif
  int flag = 0;
  bool have_cand = false;  // warp candidates for column j already in red (found during elimination)
  for (int j = 0; j < nb; ++j) {
    const int cj = k0 + j;
    const int j0 = j & ~(GC_SB - 1), j1 = min(nb, j0 + GC_SB);
    const int par = j & 1;
    // 1. local candidate among own rows gi >= cj (|value|, ties -> smallest row)
    if (!have_cand) {
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
    }
    {
      double b = red[0];
      int bix = (int)red[1];
#pragma unroll
      for (int w = 1; w < GC_THREADS / 32; ++w) {
        const double vw = red[2 * w];
        const int iw = (int)red[2 * w + 1];
        if (vw > b || (vw == b && iw < bix)) { b = vw; bix = iw; }
      }
      // 2. push: warp w writes {best, row, candidate row} into CTA w's inbox slot [par][rank]
#pragma unroll
      for (int h = 0; h < (CL > 8 ? 2 : 1); ++h) {
        double* dst = (h ? peer_box2 : peer_box) + ((size_t)par * CL + rank) * BOX;
        if (lane == 0) {
          dst[0] = b;
          dst[1] = (double)bix;
        }
        if (bix < n)
          for (int c = lane; c < nb; c += 32) dst[2 + c] = B[(bix - r0) * ldb + c];
        if (cj >= r0 && cj < r0 + rl)
          for (int c = lane; c < nb; c += 32) (h ? peer_cj2 : peer_cj)[par * GC_NBMAX + c] = B[(cj - r0) * ldb + c];
      }
    }
    GC_T(0);
    cluster.sync();  // the only cluster barrier per column (release / acquire of the pushes)
    GC_T(1);
    // 3. winner from the local inbox (every warp: lane c < CL reads candidate c, shuffle reduce)
    const double* mybox = box + (size_t)par * CL * BOX;
    double vb = -2.0;
    int pr = n, owner = lane;
    if (lane < CL) {
      vb = mybox[lane * BOX];
      pr = (int)mybox[lane * BOX + 1];
    }
#pragma unroll
    for (int o = CL / 2; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, vb, o);
      const int oi = __shfl_xor_sync(0xffffffffu, pr, o);
      const int oo = __shfl_xor_sync(0xffffffffu, owner, o);
      if (ov > vb || (ov == vb && oi < pr)) { vb = ov; pr = oi; owner = oo; }
    }
    vb = __shfl_sync(0xffffffffu, vb, 0);
    pr = __shfl_sync(0xffffffffu, pr, 0);
    owner = __shfl_sync(0xffffffffu, owner, 0);
    if (pr >= n) pr = -1;  // all NaN: keep the diagonal (row cj)
    if (!(vb > 0.0)) flag = 1;
    if (pr < 0) pr = cj;
    const double* drow = cjrow + par * GC_NBMAX;
    const double* prow = (pr == cj) ? drow : mybox + owner * BOX + 2;
    if (tid == 0) spiv[j] = pr;
    GC_T(2);
    // 4. own rows: interchange over all nb columns, elimination over the sub-block only.
    //    Position cj <- pivot row: sub-block columns scaled (column j <- 1/pivot), the other
    //    columns keep the unscaled values (their transform is applied at the sub-block end).
    const double inv = 1.0 / prow[j];
    const int lcj = cj - r0, lpr = pr - r0;
    for (int c = tid; c < nb; c += GC_THREADS) {
      const bool insb = c >= j0 && c < j1;
      const double pc = prow[c];
      cp[(j - j0) * CPLD + c] = pc;  // C_piv row of this step: the pivot row, other columns
      if (lcj >= 0 && lcj < rl) B[lcj * ldb + c] = insb ? (c == j ? inv : pc * inv) : pc;
      if (pr != cj && lpr >= 0 && lpr < rl && !insb) B[lpr * ldb + c] = drow[c];
    }
    // the next column's candidates come out of the same pass when it lies in this sub-block
    const bool fuse = j + 1 < j1;
    double nbest = -1.0;
    int nbi = n;
    for (int r = tid; r < rl; r += GC_THREADS) {
      const int gi = r0 + r;
      if (gi >= n || gi == cj) continue;
      double* row = B + r * ldb;
      const bool moved = (gi == pr);  // receives the displaced row cj
      const double f = moved ? drow[j] : row[j];
#pragma unroll
      for (int u = 0; u < GC_SB; ++u) {
        const int c = j0 + u;
        if (c < j1) {
          const double v = moved ? drow[c] : row[c];
          const double pv = (c == j) ? inv : prow[c] * inv;
          const double nv = (c == j ? 0.0 : v) - f * pv;
          row[c] = nv;
          if (c == j + 1 && gi > cj && fabs(nv) > nbest) {  // rows below the next pivot position
            nbest = fabs(nv);
            nbi = gi;
          }
        }
      }
    }
    if (fuse) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, nbest, o);
        const int oi = __shfl_xor_sync(0xffffffffu, nbi, o);
        if (ov > nbest || (ov == nbest && oi < nbi)) { nbest = ov; nbi = oi; }
      }
      if (lane == 0) {
        red[2 * warp] = nbest;
        red[2 * warp + 1] = (double)nbi;
      }
    }
    have_cand = fuse;
    __syncthreads();
    GC_T(3);
    if (j == j1 - 1 && nb > j1 - j0) {
      // 5. sub-block end: C <- D C + W C_piv on the other nb - sb columns (local data only: every
      //    CTA captured the pivot rows from its inbox). One m-tile per warp pass, all n-tiles.
      const int sb = j1 - j0;
      const int g = lane >> 2, t = lane & 3;
      const int mtiles = (rl + 7) >> 3, ocols = nb - sb, ntiles = (ocols + 7) >> 3;
      const int pr_lo = k0 + j0 - r0, pr_hi = k0 + j1 - r0;  // pivot rows in local numbering
      for (int mt = warp; mt < mtiles; mt += GC_THREADS / 32) {
        const int r = mt * 8 + g;
        const bool rok = r < rl && r0 + r < n;
        const bool pivrow = r >= pr_lo && r < pr_hi;
        const double* wrow = B + (size_t)(rok ? r : 0) * ldb + j0;
        const double a0 = (rok && t < sb) ? wrow[t] : 0.0;
        const double a1 = (rok && t + 4 < sb) ? wrow[t + 4] : 0.0;
#pragma unroll
        for (int nt = 0; nt < GC_NBMAX / 8; ++nt) {
          if (nt >= ntiles) break;
          double d[2];
          int cc[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int x = nt * 8 + 2 * t + h;
            cc[h] = x < ocols ? (x < j0 ? x : x + sb) : -1;
            d[h] = (rok && cc[h] >= 0 && !pivrow) ? B[r * ldb + cc[h]] : 0.0;
          }
          const int xb = nt * 8 + g;
          const int cb = xb < ocols ? (xb < j0 ? xb : xb + sb) : -1;
          const double b0 = (t < sb && cb >= 0) ? cp[t * CPLD + cb] : 0.0;
          const double b1 = (t + 4 < sb && cb >= 0) ? cp[(t + 4) * CPLD + cb] : 0.0;
          dmma8x8x4(d[0], d[1], a0, b0);
          dmma8x8x4(d[0], d[1], a1, b1);
          if (rok) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (cc[h] >= 0) B[r * ldb + cc[h]] = d[h];
          }
        }
      }
      __syncthreads();
      GC_T(4);
    }
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

static int gc_cl() {
  static int cl = -1;  // HPS_GJ_CL: CTAs per cluster, 8 (portable) or 16 (non-portable)
  if (cl < 0) {
    const char* e = getenv("HPS_GJ_CL");
    cl = (e && atoi(e) == 16) ? 16 : 8;
  }
  return cl;
}

size_t gj_cluster_smem(int n, int nb) {
  const int cl = gc_cl();
  const int rl = (n + cl - 1) / cl;
  return sizeof(double) * (cl == 16 ? GcLayout<16>(rl, nb).total() : GcLayout<8>(rl, nb).total());
}

// measured faster than the three-level fused path only for n >= ~900 (root and level-1 merges)
bool gj_cluster_ok(int n, int nb) {
  static int nmin = -1;  // HPS_GJ_CLUSTER_NMIN: smallest n for the cluster panel kernel
  if (nmin < 0) {
    const char* e = getenv("HPS_GJ_CLUSTER_NMIN");
    nmin = e ? atoi(e) : 384;
  }
  return n >= nmin && nb <= GC_NBMAX && gj_cluster_smem(n, nb) <= 200 * 1024;
}

template <int CL>
static int launch_cl(const GcArgs& a, size_t smem, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gj_cluster_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (CL > 8) cudaFuncSetAttribute(gj_cluster_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.batch * CL);
  cfg.blockDim = dim3(GC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gj_cluster_kernel<CL>, a) == cudaSuccess ? 0 : 2;
}

int launch_gj_cluster(int batch, int n, int k0, int nb, MatB M, int* piv, int* status, cudaStream_t s) {
  if (!gj_cluster_ok(n, nb)) return 1;
  const int cl = gc_cl();
  GcArgs a{};
  a.batch = batch;
  a.n = n;
  a.k0 = k0;
  a.nb = nb;
  a.M = M;
  a.piv = piv;
  a.status = status;
  a.rl = (n + cl - 1) / cl;
  const size_t smem = gj_cluster_smem(n, nb);
  return cl == 16 ? launch_cl<16>(a, smem, s) : launch_cl<8>(a, smem, s);
}

}  // namespace hps

#ifdef GC_PROFILE
extern "C" void hps_gc_prof(long long* h, int reset) {
  cudaMemcpyFromSymbol(h, hps::gc_prof, 8 * sizeof(long long));
  if (reset) {
    long long z[8] = {};
    cudaMemcpyToSymbol(hps::gc_prof, z, sizeof(z));
  }
}
#endif
