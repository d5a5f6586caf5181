// Solve-stage sweeps: batched gather-GEMV over one level of the tree (reference
// solver.py:255-335). Every vector lives in one pool (rows x nrhs, RHS fastest) and every
// gather/scatter is an absolute pool-row index, so leaf and parent steps — including the
// 2:1 wrap interpolations — all run through this one kernel:
//   leaf up      h      = H g                                   (solver.py:278)
//   parent up    w3     = X (h_b[pos3_b] - h_a[pos3_a])           (solver.py:284)
//                h_ge   = [h_a[pos1_a]; h_b[pos2_b]] + T_ei w3    (solver.py:285-286)
//   parent down  u[j3]  = S u[ext] + w[j3]                        (solver.py:335)
//   leaf down    u_c    = [F_ii | S_ie] [g; u_ge],  u_ce = L u_ge  (solver.py:325-327)
// Bandwidth-bound: each operator entry is read once per call and used for nrhs FMAs.
#include <cstdlib>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

constexpr int SW_THREADS = 256;

// 1: single-RHS kernels load their (static) gather indices before the programmatic-launch wait
// (bit mask: 1 staged-x row kernel, 2 gather kernel, 4 multi-item kernel, 8 one-row kernel)
#define pre_index(bit) ((a.pre_mask & (bit)) != 0)

// every sweep launch carries the programmatic-serialization attribute (HPS_PDL=0 disables)
// Programmatic dependent launch (the next step's prologue overlaps this step's tail). HPS_PDL:
// 0 = never, 2 = every step, 1 (default) = every step with <= 2 right-hand sides, and with more
// only the persistent TMA kernels (one CTA per SM that streams its operator before the launch
// wait). At 16 RHS the early CTAs of a many-CTA register-streaming step hold shared memory and
// registers that the tail of the current step still needs: config 5, 16 RHS runs 3.62 ms with
// PDL everywhere, 3.51 ms with none and 3.48 ms with this rule, while the single-RHS sweeps gain
// from it everywhere (config 2 0.72 ms without, 0.67 ms with).
static int pdl_mode() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HPS_PDL");
    on = e ? atoi(e) : 1;
  }
  return on;
}
bool sweep_pdl_for(int nrhs, bool persistent) {
  return pdl_mode() == 2 || (pdl_mode() == 1 && (nrhs <= 2 || persistent));
}
static thread_local bool g_pdl_now = true;  // set per hps_sweep_gemv call (launch_gemv_gather)
// many-CTA kernels of multi-RHS steps: dependent launch only for steps that stream at most this
// many MB of operator (HPS_PDL_MAX_MB). Short steps gain from the hidden launch latency, long ones
// lose more to the early CTAs of their successor (config 2 at 16 RHS: 1.09 ms without, 1.04 ms
// with; config 5: 3.62 ms with, 3.47 ms without)
static double pdl_max_mb() {
  static double v = -1.0;
  if (v < 0) {
    const char* e = getenv("HPS_PDL_MAX_MB");
    v = e ? atof(e) : 64.0;
  }
  return v;
}
static bool pdl_enabled() { return g_pdl_now; }

template <typename... KArgs, typename... Args>
static void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// x gather into shared memory: dst[k*ld + j] = pool[xi[k]][j] (- pool[x2[k]][j] if x2[k] >= 0) for k < kc,
// j < nrhs; zero for kc <= k < kp or j >= nrhs. GU elements per thread are issued together so
// the index -> value load chains overlap: one memory round trip per GU elements, not per element
// (the per-element loop left the multi-RHS leaf steps stalled on the gather, r01 ncu).
template <int NRP, int GU = 8, bool PLAIN = false>
__device__ __forceinline__ void gather_x(double* dst, int ld, const int* __restrict__ xi,
                                         const int* __restrict__ x2, const double* pool, int nrhs, int kc,
                                         int kp, int tid = -1, int nth = 0, int ksc = 0, double sc = 1.0) {
  // (ksc, sc): columns k < ksc of this chunk are scaled by sc (GemvArgs::kscale / xscale)
  // (tid, nth): the gathering thread group (default: the whole CTA)
  if (tid < 0) {
    tid = threadIdx.x;
    nth = blockDim.x;
  }
  const int tot = kp * NRP;
  for (int e0 = tid; e0 < tot; e0 += GU * nth) {
    int i1[GU], i2[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int e = e0 + u * nth, k = e / NRP;
      const bool ok = e < tot && k < kc && e - k * NRP < nrhs;
      // PLAIN: the index arrays were staged in shared memory (no read-only-path load)
      i1[u] = ok ? (PLAIN ? xi[k] : __ldg(xi + k)) : -1;
      i2[u] = (ok && x2) ? (PLAIN ? x2[k] : __ldg(x2 + k)) : -1;
    }
    double v[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int e = e0 + u * nth, k = e / NRP, j = e - k * NRP;
      v[u] = i1[u] >= 0 ? pool[(long long)i1[u] * nrhs + j] : 0.0;
      if (i2[u] >= 0) v[u] -= pool[(long long)i2[u] * nrhs + j];
      if (k < ksc) v[u] *= sc;
    }
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int e = e0 + u * nth, k = e / NRP, j = e - k * NRP;
      if (e < tot) dst[k * ld + j] = v[u];
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(SW_THREADS) gemv_gather_kernel(GemvArgs a, int rows_per_cta, int kchunk,
                                                                 int batch_off) {
  extern __shared__ double sm[];
  double* xs = sm;                          // kchunk x NR
  double* part = xs + (size_t)kchunk * NR;  // rows_per_cta x NR
  const int item = blockIdx.y + batch_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarp = SW_THREADS / 32;
  const int R = a.R, K = a.K, nrhs = a.nrhs;
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(R, r0 + rows_per_cta);
  const double* Ai = a.A.get(item);
  const long long lda = a.A.ld;
  const int* xi = a.xidx + (long long)item * a.xstride;
  const int* x2 = a.x2idx ? a.x2idx + (long long)item * a.xstride : nullptr;
  double* pool = a.pool;

  pdl_trigger();
  for (int e = tid; e < (r1 - r0) * NR; e += SW_THREADS) part[e] = 0.0;
  for (int r = r0 + tid; r < r1; r += SW_THREADS) {
    // start streaming this CTA's operator rows into L2 while x is gathered
    const double* rp = Ai + (long long)r * lda;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(rp) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(rp + K) + 15) & ~(uintptr_t)15;
    prefetch_l2_bulk(reinterpret_cast<const void*>(lo), (unsigned)(hi - lo));
  }
  // single RHS, one chunk: the static gather indices are loaded before the launch wait
  const bool pre = NR == 1 && a.mode2 == 0 && K <= kchunk && K <= 2 * SW_THREADS && pre_index(2);
  if (pre) {
    int i1[2], i2[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = tid + u * SW_THREADS;
      i1[u] = k < K ? __ldg(xi + k) : -1;
      i2[u] = (k < K && x2) ? __ldg(x2 + k) : -1;
    }
    pdl_wait();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = tid + u * SW_THREADS;
      double v = i1[u] >= 0 ? pool[i1[u]] : 0.0;
      if (i2[u] >= 0) v -= pool[i2[u]];
      if (k < K) xs[k] = v;
    }
  } else {
    pdl_wait();
  }

  // mode2 = 3: chunk boundaries align with K2 and the partial sum over columns [0, K2) is also
  // stored at o2idx (parent down: u3 = [X | S][d; u_ext] writes w3 = X d on the way)
  const int ksplit = a.mode2 == 3 ? a.K2 : K;
  for (int k0 = 0, kc = 0; k0 < K; k0 += kc) {
    kc = min(kchunk, (k0 < ksplit ? ksplit : K) - k0);
    if (k0 == ksplit) {
      __syncthreads();
      const int* o2 = a.o2idx + (long long)item * a.ostride;
      for (int e = tid; e < (r1 - r0) * NR; e += SW_THREADS) {
        const int rr = e / NR, j = e - rr * NR;
        if (j < nrhs) pool[(long long)o2[r0 + rr] * nrhs + j] = part[e];
      }
    }
    __syncthreads();
    for (int e = pre ? kc * NR : tid; e < kc * NR; e += SW_THREADS) {  // pre: x already staged
      const int k = e / NR, j = e - k * NR;
      double v = 0.0;
      if (j < nrhs) {
        v = pool[(long long)xi[k0 + k] * nrhs + j];
        if (x2 && x2[k0 + k] >= 0) v -= pool[(long long)x2[k0 + k] * nrhs + j];
      }
      xs[e] = v;
    }
    __syncthreads();
    for (int r = r0 + warp; r < r1; r += nwarp) {
      const double* row = Ai + (long long)r * lda + k0;
      double acc[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[j] = 0.0;
      for (int k = lane; k < kc; k += 32) {
        const double av = row[k];
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[j] = fma(av, xs[k * NR + j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[j] = warp_sum(acc[j]);
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < NR; ++j) part[(r - r0) * NR + j] += acc[j];
      }
    }
  }
  __syncthreads();
  const int* ai = a.aidx ? a.aidx + (long long)item * a.ostride : nullptr;
  const int* oi = a.oidx + (long long)item * a.ostride;
  for (int e = tid; e < (r1 - r0) * NR; e += SW_THREADS) {
    const int rr = e / NR, j = e - rr * NR;
    if (j >= nrhs) continue;
    const int r = r0 + rr;
    double v = part[e];
    if (ai) v += pool[(long long)ai[r] * nrhs + j];
    pool[(long long)oi[r] * nrhs + j] = v;
  }
}

// Multi-RHS variant on DMMA tiles: Y (R x NRP) = A (R x K) X (K x NRP), NRP = 8 or 16 padded
// right-hand sides. A CTA owns rpc rows (16..128) of one item; its 8 warps are split into
// WR = rpc/16 row groups x WK = 8/WR k-slices (k4 steps dealt round-robin), partial sums are
// reduced through shared memory. A fragments are streamed straight from global memory (each
// lane group reads one 32-byte sector per row, 8 loads in flight per lane), X is gathered into
// shared memory chunk by chunk with a padded stride (conflict-free B fragments).
// L2 bulk prefetch of rows [r0, r1) of an item's operator (static data: issued before the
// programmatic-launch wait, so the DMMA loop after it reads L2 instead of HBM); one request per
// row, spread over the calling threads (tid of nth)
__device__ __forceinline__ void prefetch_rows(const double* Ai, long long ld, int r0, int r1, int K, int tid,
                                              int nth) {
  for (int r = r0 + tid; r < r1; r += nth) {
    const double* rp = Ai + (long long)r * ld;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(rp) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(rp + K) + 15) & ~(uintptr_t)15;
    prefetch_l2_bulk(reinterpret_cast<const void*>(lo), (unsigned)(hi - lo));
  }
}

#ifndef HPS_DMMA_U2
#define HPS_DMMA_U2 6  // A-fragment loads in flight per lane and row tile for K >= 96 (4 below)
#endif
// UA: A-fragment loads in flight per lane and row tile. 6 instead of 4 for the longer rows keeps
// more bytes in flight per SM at the same 4 CTAs (config 5, 16 RHS: leaf upward step 514 -> 487 us,
// K = 240 split parts 57 -> 53.5 us); 8 needs 3 CTAs per SM or spills and measured slower
template <int NRP, bool VEC, int UA = 4>
__global__ void __launch_bounds__(256, 4) gemv_dmma_kernel(GemvArgs a, int rpc, int kchunk, int batch_off,
                                                            int stage_idx) {
  extern __shared__ double xs[];
  // VEC: each lane loads A[r][k+2t .. k+2t+1] as one 16-byte load and uses the two halves as
  // the A fragments of two "virtual" k4 steps; B fragments follow the same k permutation.
  // Stride NRP+2 keeps those B loads conflict free, NRP+4 the natural-order ones.
  constexpr int XLD = VEC ? NRP + 2 : NRP + 4;
  constexpr int NT = NRP / 8;
  const int item = blockIdx.y + batch_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int WR = rpc >> 4, WK = 8 / WR;
  const int wr = warp % WR, wk = warp / WR;
  double* red = xs + (size_t)kchunk * XLD;
  const int R = a.R, K = a.K, nrhs = a.nrhs;
  const int rbase = blockIdx.x * rpc + wr * 16;
  const double* Ai = gemv_a(a, item);
  const long long lda = a.A.ld;
  const int* xi = a.xidx + (long long)item * a.xstride;
  const int* x2 = a.x2idx ? a.x2idx + (long long)item * a.xstride : nullptr;
  const double* pool = a.pool;
  const int ra = rbase + gq, rb = rbase + 8 + gq;
  const double* rowa = Ai + (long long)(ra < R ? ra : 0) * lda;
  const double* rowb = Ai + (long long)(rb < R ? rb : 0) * lda;
  const bool la = ra < R, lb = rb < R;

  double acc[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
  pdl_trigger();
  if (a.pre_mask & 16) prefetch_rows(Ai, lda, blockIdx.x * rpc, min(R, (int)(blockIdx.x + 1) * rpc), K, tid, blockDim.x);
  // stage_idx: the (static) gather indices go to shared memory before the launch wait, so after
  // it the x gather is one dependent global load per element instead of two
  int* sidx = reinterpret_cast<int*>(red + (size_t)(WK - 1) * WR * 32 * (4 * NT));
  if (stage_idx) {
    for (int k = tid; k < K; k += blockDim.x) {
      sidx[k] = __ldg(xi + k);
      sidx[K + k] = x2 ? __ldg(x2 + k) : -1;
    }
  }
  pdl_wait();

  for (int k0 = 0; k0 < K; k0 += kchunk) {
    const int kc = min(kchunk, K - k0);
    const int kcp = VEC ? (kc + 7) & ~7 : (kc + 3) & ~3;
    __syncthreads();
    if (stage_idx)
      gather_x<NRP, 4, true>(xs, XLD, sidx + k0, x2 ? sidx + K + k0 : nullptr, pool, nrhs, kc, kcp, -1, 0,
                             a.kscale - k0, a.xscale);
    else
      gather_x<NRP, 4>(xs, XLD, xi + k0, x2 ? x2 + k0 : nullptr, pool, nrhs, kc, kcp, -1, 0, a.kscale - k0,
                       a.xscale);
    __syncthreads();
    if (VEC) {
      const int step = WK * 8;
      int k = wk * 8;
      for (; k < kcp; k += 4 * step) {
        double2 va[4], vb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = k + u * step + 2 * tq;
          va[u] = make_double2(0.0, 0.0);
          vb[u] = make_double2(0.0, 0.0);
          if (kk + 1 < kc) {
            if (la) va[u] = __ldg(reinterpret_cast<const double2*>(rowa + k0 + kk));
            if (lb) vb[u] = __ldg(reinterpret_cast<const double2*>(rowb + k0 + kk));
          } else if (kk < kc) {
            if (la) va[u].x = __ldg(rowa + k0 + kk);
            if (lb) vb[u].x = __ldg(rowb + k0 + kk);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kb = k + u * step;
          if (kb >= kcp) break;
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const double b0 = xs[(kb + 2 * tq) * XLD + n * 8 + gq];
            const double b1 = xs[(kb + 2 * tq + 1) * XLD + n * 8 + gq];
            dmma8x8x4(acc[0][n][0], acc[0][n][1], va[u].x, b0);
            dmma8x8x4(acc[1][n][0], acc[1][n][1], vb[u].x, b0);
            dmma8x8x4(acc[0][n][0], acc[0][n][1], va[u].y, b1);
            dmma8x8x4(acc[1][n][0], acc[1][n][1], vb[u].y, b1);
          }
        }
      }
      continue;
    }
    const int kc4 = kcp;
    const int step = WK * 4;
    int k = wk * 4;
    for (; k + (UA - 1) * step < kc4; k += UA * step) {
      double va[UA], vb[UA];
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        const int kk = k + u * step + tq;
        const bool kin = kk < kc;
        va[u] = (kin && la) ? __ldg(rowa + k0 + kk) : 0.0;
        vb[u] = (kin && lb) ? __ldg(rowb + k0 + kk) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UA; ++u)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const double bv = xs[(k + u * step + tq) * XLD + n * 8 + gq];
          dmma8x8x4(acc[0][n][0], acc[0][n][1], va[u], bv);
          dmma8x8x4(acc[1][n][0], acc[1][n][1], vb[u], bv);
        }
    }
    for (; k < kc4; k += step) {
      const int kk = k + tq;
      const bool kin = kk < kc;
      const double va = (kin && la) ? __ldg(rowa + k0 + kk) : 0.0;
      const double vb = (kin && lb) ? __ldg(rowb + k0 + kk) : 0.0;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double bv = xs[(k + tq) * XLD + n * 8 + gq];
        dmma8x8x4(acc[0][n][0], acc[0][n][1], va, bv);
        dmma8x8x4(acc[1][n][0], acc[1][n][1], vb, bv);
      }
    }
  }
  // reduce the k-slices of each row group through shared memory
  if (WK > 1) {
    __syncthreads();
    if (wk > 0) {
      double* dst = red + ((size_t)((wk - 1) * WR + wr) * 32 + lane) * (4 * NT);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          dst[(i * NT + n) * 2] = acc[i][n][0];
          dst[(i * NT + n) * 2 + 1] = acc[i][n][1];
        }
    }
    __syncthreads();
    if (wk > 0) return;
    for (int w = 1; w < WK; ++w) {
      const double* src = red + ((size_t)((w - 1) * WR + wr) * 32 + lane) * (4 * NT);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          acc[i][n][0] += src[(i * NT + n) * 2];
          acc[i][n][1] += src[(i * NT + n) * 2 + 1];
        }
    }
  }
  const int* ai = a.aidx ? a.aidx + (long long)item * a.ostride : nullptr;
  const int* oi = a.oidx + (long long)item * a.ostride;
  double* pw = a.pool;
  // even nrhs on a 16-byte aligned pool: the pair (j, j + 1) of a lane is one 16-byte access (the
  // deep levels move more vector bytes than operator bytes)
  const bool wide = (nrhs & 1) == 0 && (reinterpret_cast<uintptr_t>(pw) & 15) == 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = i ? rb : ra;
    if (r >= R) continue;
    const long long orow = (long long)oi[r] * nrhs;
    const long long arow = ai ? (long long)ai[r] * nrhs : -1;
    if (wide) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int j = n * 8 + tq * 2;
        if (j < nrhs) {
          double2 v = make_double2(acc[i][n][0], acc[i][n][1]);
          if (arow >= 0) {
            const double2 w = *reinterpret_cast<const double2*>(pool + arow + j);
            v.x += w.x;
            v.y += w.y;
          }
          *reinterpret_cast<double2*>(pw + orow + j) = v;
        }
      }
      continue;
    }
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = n * 8 + tq * 2 + h;
        if (j < nrhs) {
          double v = acc[i][n][h];
          if (arow >= 0) v += pool[arow + j];
          pw[orow + j] = v;
        }
      }
  }
}

// Multi-RHS (3..16) steps of small items (deep tree levels: thousands of items of 15..360 rows
// and K <= ~300): IPC items per CTA, each owned by a group of 8/IPC warps. A group stages its
// item's whole x (K x NRP, padded stride) in shared memory, then each warp takes 16-row groups
// of the item and runs the k4 steps on DMMA tiles with A fragments straight from global memory.
// No k-split, no cross-warp reduction. The one-item-per-CTA kernel above left the 8192-item
// levels of config 5 at 0.4-0.9 TB/s. mode2 = 3 (w3 = X d as a partial sum over [0, K2)) is
// two passes over the column ranges.
template <int NRP, int IPC>
__global__ void __launch_bounds__(256) gemv_dmma_multi_kernel(GemvArgs a) {
  extern __shared__ double xsm[];
  constexpr int XLD = NRP + 4;
  constexpr int NT = NRP / 8;
  constexpr int GW = 8 / IPC;  // warps per item
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp / GW, gw = warp % GW;
  const int item = blockIdx.x * IPC + grp;
  const int gq = lane >> 2, tq = lane & 3;
  const int R = a.R, K = a.K, nrhs = a.nrhs;
  const int kp = (K + 3) & ~3;
  double* xs = xsm + (size_t)grp * kp * XLD;
  // per-group index slice after all the x slices: [2][kp] ints, staged before the launch wait
  int* sidx = reinterpret_cast<int*>(xsm + (size_t)IPC * kp * XLD) + (size_t)grp * 2 * kp;
  pdl_trigger();
  const bool live = item < a.nitems;
  const int* xi = a.xidx + (long long)(live ? item : 0) * a.xstride;
  const int* x2 = a.x2idx ? a.x2idx + (long long)(live ? item : 0) * a.xstride : nullptr;
  const int gtid = (int)threadIdx.x - grp * GW * 32;
  if (live) {
    for (int k = gtid; k < K; k += GW * 32) {
      sidx[k] = __ldg(xi + k);
      sidx[kp + k] = x2 ? __ldg(x2 + k) : -1;
    }
    if (a.pre_mask & 16) prefetch_rows(gemv_a(a, item), a.A.ld, 0, R, K, gtid, GW * 32);
  }
  pdl_wait();
  if (!live) return;  // whole group
  if (GW == 1)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(GW * 32) : "memory");
  gather_x<NRP, 4, true>(xs, XLD, sidx, x2 ? sidx + kp : nullptr, a.pool, nrhs, K, kp, gtid, GW * 32, a.kscale,
                         a.xscale);
  if (GW == 1)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(GW * 32) : "memory");
  const double* Ai = gemv_a(a, item);
  const long long lda = a.A.ld;
  const int* ai = a.aidx ? a.aidx + (long long)item * a.ostride : nullptr;
  const int* oi = a.oidx + (long long)item * a.ostride;
  const int* o2 = a.mode2 == 3 ? a.o2idx + (long long)item * a.ostride : nullptr;
  const int ksplit = a.mode2 == 3 ? a.K2 : 0;
  double* pool = a.pool;
  for (int rbase = gw * 16; rbase < R; rbase += GW * 16) {
    const int ra = rbase + gq, rb = rbase + 8 + gq;
    const bool la = ra < R, lb = rb < R;
    const double* rowa = Ai + (long long)(la ? ra : 0) * lda;
    const double* rowb = Ai + (long long)(lb ? rb : 0) * lda;
    double acc[2][NT][2], accw[2][NT][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[i][n][0] = acc[i][n][1] = accw[i][n][0] = accw[i][n][1] = 0.0;
    // pass 0: columns [0, ksplit) into accw (mode2 = 3 only); pass 1: [ksplit, K) into acc
    for (int pass = ksplit > 0 ? 0 : 1; pass < 2; ++pass) {
      const int klo = pass ? ksplit : 0, khi = pass ? K : ksplit;
      for (int k = klo & ~3; k < khi; k += 16) {
        double va[4], vb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = k + 4 * u + tq;
          const bool kin = kk >= klo && kk < khi;
          va[u] = (kin && la) ? __ldg(rowa + kk) : 0.0;
          vb[u] = (kin && lb) ? __ldg(rowb + kk) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kb = k + 4 * u;
          if (kb >= khi) break;
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const double bv = xs[(kb + tq) * XLD + n * 8 + gq];
            if (pass) {
              dmma8x8x4(acc[0][n][0], acc[0][n][1], va[u], bv);
              dmma8x8x4(acc[1][n][0], acc[1][n][1], vb[u], bv);
            } else {
              dmma8x8x4(accw[0][n][0], accw[0][n][1], va[u], bv);
              dmma8x8x4(accw[1][n][0], accw[1][n][1], vb[u], bv);
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = i ? rb : ra;
      if (r >= R) continue;
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = n * 8 + tq * 2 + h;
          if (j >= nrhs) continue;
          double v = acc[i][n][h] + accw[i][n][h];
          if (o2) pool[(long long)o2[r] * nrhs + j] = accw[i][n][h];
          if (ai) v += pool[(long long)ai[r] * nrhs + j];
          pool[(long long)oi[r] * nrhs + j] = v;
        }
    }
  }
}

template <int NRP>
static bool launch_dmma_multi(const GemvArgs& a, cudaStream_t s) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HPS_DMMA_MULTI");
    on = e ? atoi(e) : 1;
  }
  // measured (config 5, 16 RHS): faster than the one-item-per-CTA kernel only for the split-output
  // downward steps of the deepest levels (R <= 32: one launch instead of two; 8192 items 232 ->
  // 123 us); slower for the upward steps, whose rows the 8 warps of a CTA split better
  if (!on || a.mode2 != 3 || a.aidx || a.R > 32) return false;
  const size_t per_item = sizeof(double) * (size_t)((a.K + 3) & ~3) * (NRP + 4) +
                          sizeof(int) * 2 * (size_t)((a.K + 3) & ~3);
  int ipc = 1;
  while (ipc < 8 && (long long)a.nitems / (2 * ipc) >= 2 * 148 && per_item * 2 * ipc <= 96 * 1024) ipc *= 2;
  if (ipc == 1 || a.R > 16 * 8 * 4) return false;  // one item per CTA: the kernel above
  const size_t smem = per_item * ipc;
  const dim3 grid((unsigned)((a.nitems + ipc - 1) / ipc));
  switch (ipc) {
    case 2:
      cudaFuncSetAttribute(gemv_dmma_multi_kernel<NRP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      launch_k(gemv_dmma_multi_kernel<NRP, 2>, grid, dim3(256), smem, s, a);
      break;
    case 4:
      cudaFuncSetAttribute(gemv_dmma_multi_kernel<NRP, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      launch_k(gemv_dmma_multi_kernel<NRP, 4>, grid, dim3(256), smem, s, a);
      break;
    default:
      cudaFuncSetAttribute(gemv_dmma_multi_kernel<NRP, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      launch_k(gemv_dmma_multi_kernel<NRP, 8>, grid, dim3(256), smem, s, a);
      break;
  }
  return true;
}

// Staged-x sweep kernel for nrhs <= 2 with an optional fused second stage (tail / chain).
// Rows are processed by groups of L lanes (L = 4..32 chosen from K so short rows do not idle
// lanes), 8 independent loads in flight per lane, group-wide shuffle reduction.
// Scalar accumulation of columns [kb, ke) of RB rows: lane kl of an L-lane group takes columns
// kb + kl + t*L, U loads per row in flight.
// SA: the rows live in shared memory (staged by a bulk copy), plain loads instead of __ldg
template <int NR, int RB, int U, bool SA = false>
__device__ __forceinline__ void dot_cols(double (&acc)[RB][NR], const double* const (&row)[RB],
                                         const bool (&live)[RB], int kb, int ke, int L, int kl,
                                         const double* xs) {
  int k = kb + kl;
  for (; k + (U - 1) * L < ke; k += U * L) {
    double v[RB][U];
#pragma unroll
    for (int q = 0; q < RB; ++q)
#pragma unroll
      for (int u = 0; u < U; ++u) v[q][u] = live[q] ? (SA ? row[q][k + u * L] : __ldg(row[q] + k + u * L)) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const double xv = xs[(k + u * L) * NR + j];
#pragma unroll
        for (int q = 0; q < RB; ++q) acc[q][j] = fma(v[q][u], xv, acc[q][j]);
      }
  }
  for (; k < ke; k += L) {
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const double v = live[q] ? (SA ? row[q][k] : __ldg(row[q] + k)) : 0.0;
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[q][j] = fma(v, xs[k * NR + j], acc[q][j]);
    }
  }
}

// ksplit < K (mode2 = 3): the partial sum over columns [0, ksplit) is also stored at o2idx[r].
template <int NR, bool VEC, int RB = 2, int U = 4, bool SA = false>
__device__ __forceinline__ void rows_dot(const double* __restrict__ A, long long lda, int R, int r0, int r1,
                                         int K, int L, const double* xs, const int* aidx, const int* oidx,
                                         double* pool, int nrhs, double* ys, int ksplit = 1 << 30,
                                         const int* o2idx = nullptr, int warp = -1, int nw = 0, int arow0 = 0) {
  // each warp streams RB row groups at once (RB x U independent loads in flight per lane);
  // (warp, nw): this warp's index in the row-processing group (default: the whole CTA)
  const int lane = threadIdx.x & 31;
  if (warp < 0) {
    warp = threadIdx.x >> 5;
    nw = blockDim.x >> 5;
  }
  const int G = 32 / L, sub = lane / L, kl = lane % L;
  const bool split = ksplit < K;
  for (int rb = r0 + warp * G * RB; rb < r1; rb += nw * G * RB) {
    double acc[RB][NR], accw[RB][NR];
    const double* row[RB];
    bool live[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int r = rb + q * G + sub;
      live[q] = r < r1;
      row[q] = A + (long long)((live[q] ? r : r0) - arow0) * lda;  // arow0: first row held at A
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[q][j] = accw[q][j] = 0.0;
    }
    if (split) {
      dot_cols<NR, RB, U, SA>(accw, row, live, 0, ksplit, L, kl, xs);
      dot_cols<NR, RB, U, SA>(acc, row, live, ksplit, K, L, kl, xs);
#pragma unroll
      for (int o = L >> 1; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < RB; ++q)
#pragma unroll
          for (int j = 0; j < NR; ++j) accw[q][j] += __shfl_xor_sync(0xffffffffu, accw[q][j], o);
    } else if (VEC) {
      // 16-byte loads: lane kl covers columns 2kl, 2kl+1 of each 2L-wide strip
      for (int k = 2 * kl; k < K; k += 2 * L * U) {
        double2 v[RB][U];
#pragma unroll
        for (int q = 0; q < RB; ++q)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int kk = k + u * 2 * L;
            v[q][u] = make_double2(0.0, 0.0);
            if (live[q]) {
              if (kk + 1 < K) v[q][u] = __ldg(reinterpret_cast<const double2*>(row[q] + kk));
              else if (kk < K) v[q][u].x = __ldg(row[q] + kk);
            }
          }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = k + u * 2 * L;
          if (kk >= K) break;
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const double x0 = xs[kk * NR + j];
            const double x1 = (kk + 1 < K) ? xs[(kk + 1) * NR + j] : 0.0;
#pragma unroll
            for (int q = 0; q < RB; ++q) acc[q][j] = fma(v[q][u].y, x1, fma(v[q][u].x, x0, acc[q][j]));
          }
        }
      }
    } else {
      dot_cols<NR, RB, U, SA>(acc, row, live, 0, K, L, kl, xs);
    }
#pragma unroll
    for (int o = L >> 1; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < RB; ++q)
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[q][j] += __shfl_xor_sync(0xffffffffu, acc[q][j], o);
    if (kl == 0) {
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const int r = rb + q * G + sub;
        if (!live[q]) continue;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          if (j >= nrhs) break;
          double y = acc[q][j];
          if (split) {
            pool[(long long)o2idx[r] * nrhs + j] = accw[q][j];
            y += accw[q][j];
          }
          if (aidx) y += pool[(long long)aidx[r] * nrhs + j];
          pool[(long long)oidx[r] * nrhs + j] = y;
          if (ys) ys[(r - r0) * NR + j] = y;
        }
      }
    }
  }
}

__host__ __device__ inline int lanes_for(int K) { return K <= 16 ? 4 : (K <= 48 ? 8 : (K <= 128 ? 16 : 32)); }

// One work unit of a sweep step: item `item`, row chunk `chunk` of `nchunks` (rows_per_cta rows).
__device__ __forceinline__ uint32_t sw_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Shared-memory tile of the unit's operator rows (SA): doubles reserved in front of x
__host__ __device__ inline int sa_tile_doubles(int rows, int ld) { return ((rows * ld + 2) + 1) & ~1; }

template <int NR, bool VEC, int RB = 2, int U = 4, bool PDL = false, bool SA = false>
__device__ __forceinline__ void sweep_unit(const GemvArgs& a, int item, int chunk, int nchunks, int rows_per_cta,
                                           double* sm, int pf_rows = 1 << 30) {
  // SA: the unit's operator rows (one contiguous range) are bulk-copied into shared memory
  // BEFORE the launch wait (operators are static), so the dot products after it read on-chip
  const int tdoubles = SA ? sa_tile_doubles(rows_per_cta, a.A.ld) : 0;
  double* tile = sm;
  double* xs = sm + tdoubles;             // K x NR
  double* ys = xs + (size_t)a.K * NR;     // R x NR (chain mode)
  const int K = a.K, nrhs = a.nrhs;
  const int* xi = a.xidx + (long long)item * a.xstride;
  const int* x2 = a.x2idx ? a.x2idx + (long long)item * a.xstride : nullptr;
  const double* pool = a.pool;
  const double* Ai = a.A.get(item);
  const int r0 = chunk * rows_per_cta;
  const int r1 = min(a.R, r0 + rows_per_cta);
  __shared__ __align__(8) uint64_t sa_bar;
  int shift = 0;
  if (SA) {
    const uintptr_t src = reinterpret_cast<uintptr_t>(Ai + (long long)r0 * a.A.ld);
    const uintptr_t s0 = src & ~(uintptr_t)15;
    const uintptr_t s1 = (reinterpret_cast<uintptr_t>(Ai + (long long)(r1 - 1) * a.A.ld + K) + 15) & ~(uintptr_t)15;
    shift = (int)((src - s0) / 8);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sw_smem(&sa_bar)));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sw_smem(&sa_bar)),
                   "r"((unsigned)(s1 - s0)) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              sw_smem(tile)),
          "l"(s0), "r"((unsigned)(s1 - s0)), "r"(sw_smem(&sa_bar))
          : "memory");
    }
  }
  // start streaming this unit's operator rows into L2 while x is gathered (the first pf_rows:
  // a grid's worth of prefetches must fit in L2 or it evicts rows before they are used)
  for (int r = r0 + threadIdx.x; r < min(r1, r0 + (SA ? 0 : pf_rows)); r += blockDim.x) {
    const double* rp = Ai + (long long)r * a.A.ld;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(rp) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(rp + K) + 15) & ~(uintptr_t)15;
    prefetch_l2_bulk(reinterpret_cast<const void*>(lo), (unsigned)(hi - lo));
  }
  if (NR == 1 && PDL && K <= 2 * (int)blockDim.x && pre_index(1)) {
    // single RHS, short x: the gather indices are static, so they are loaded before the
    // programmatic-launch wait; after it only the pool rows remain on the critical path
    int i1[2], i2[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = threadIdx.x + u * blockDim.x;
      i1[u] = k < K ? __ldg(xi + k) : -1;
      i2[u] = (k < K && x2) ? __ldg(x2 + k) : -1;
    }
    pdl_wait();
    double v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      v[u] = i1[u] >= 0 ? pool[i1[u]] : 0.0;
      if (i2[u] >= 0) v[u] -= pool[i2[u]];
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = threadIdx.x + u * blockDim.x;
      if (k < K) xs[k] = v[u];
    }
  } else {
    if (PDL) pdl_wait();
    gather_x<NR>(xs, NR, xi, x2, pool, nrhs, K, K);
  }
  __syncthreads();
  if (SA)
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "SAW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n"
        "@!P bra SAW_%=;\n"
        "}\n" ::"r"(sw_smem(&sa_bar))
        : "memory");
  rows_dot<NR, VEC, RB, U, SA>(SA ? tile + shift : Ai, a.A.ld, a.R, r0, r1, K, lanes_for(K), xs,
                               a.aidx ? a.aidx + (long long)item * a.ostride : nullptr,
                               a.oidx + (long long)item * a.ostride, a.pool, nrhs, a.mode2 == 2 ? ys : nullptr,
                               a.mode2 == 3 ? a.K2 : 1 << 30,
                               a.mode2 == 3 ? a.o2idx + (long long)item * a.ostride : nullptr, -1, 0,
                               SA ? r0 : 0);
  if (a.mode2 == 1) {
    // tail stage rows split evenly over the row chunks of this item
    const int per = (a.R2 + nchunks - 1) / nchunks;
    const int s0 = chunk * per, s1 = min(a.R2, s0 + per);
    rows_dot<NR, false>(a.A2.get(item), a.A2.ld, a.R2, s0, s1, a.K2, lanes_for(a.K2), xs + (size_t)(K - a.K2) * NR,
                        a.a2idx ? a.a2idx + (long long)item * a.R2 : nullptr, a.o2idx + (long long)item * a.R2,
                        a.pool, nrhs, nullptr);
  } else if (a.mode2 == 2) {
    __syncthreads();
    rows_dot<NR, false>(a.A2.get(item), a.A2.ld, a.R2, 0, a.R2, a.K2, lanes_for(a.K2), ys,
                        a.a2idx ? a.a2idx + (long long)item * a.R2 : nullptr, a.o2idx + (long long)item * a.R2,
                        a.pool, nrhs, nullptr);
  }
}

template <int NR, bool VEC, int RB = 2, int U = 4, bool SA = false>
__global__ void __launch_bounds__(256) sweep_kernel(GemvArgs a, int rows_per_cta, int batch_off, int pf_rows) {
  extern __shared__ __align__(16) double sm[];
  pdl_trigger();
  sweep_unit<NR, VEC, RB, U, true, SA>(a, blockIdx.y + batch_off, blockIdx.x, gridDim.x, rows_per_cta, sm, pf_rows);
}

// Several small items per CTA (deep tree levels: thousands of 15..60-row items): the CTA's warps
// are split into IPC groups of 256/IPC threads, each group gathers its item's x into its own slice
// of shared memory (named barrier per group) and streams the item's rows. One wave of CTAs covers
// the level instead of several waves of one-item CTAs. Single row chunk per item; mode2 0 or 3.
template <int NR, int IPC, bool SA = false>
__global__ void __launch_bounds__(256) sweep_multi_kernel(GemvArgs a, int batch_off, int pf_rows) {
  extern __shared__ __align__(16) double sm[];
  constexpr int GT = 256 / IPC;
  const int grp = threadIdx.x / GT, gtid = threadIdx.x % GT;
  const int item = (blockIdx.x + batch_off) * IPC + grp;
  const int K = a.K, nrhs = a.nrhs;
  // SA: per-group operator tiles (whole item, bulk copy before the launch wait) after the x slices
  const int tdoubles = SA ? sa_tile_doubles(a.R, a.A.ld) : 0;
  const size_t xall = ((size_t)IPC * K * NR + 1) & ~(size_t)1;
  double* xs = sm + (size_t)grp * K * NR;
  double* tile = sm + xall + (size_t)grp * tdoubles;
  __shared__ __align__(8) uint64_t sa_bars[IPC];
  pdl_trigger();
  const bool live = item < a.nitems;
  const double* Ai = live ? a.A.get(item) : nullptr;
  int shift = 0;
  if (SA && live) {
    const uintptr_t src = reinterpret_cast<uintptr_t>(Ai);
    const uintptr_t s0 = src & ~(uintptr_t)15;
    const uintptr_t s1 = (reinterpret_cast<uintptr_t>(Ai + (long long)(a.R - 1) * a.A.ld + K) + 15) & ~(uintptr_t)15;
    shift = (int)((src - s0) / 8);
    if (gtid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sw_smem(&sa_bars[grp])));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sw_smem(&sa_bars[grp])),
                   "r"((unsigned)(s1 - s0)) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       sw_smem(tile)),
                   "l"(s0), "r"((unsigned)(s1 - s0)), "r"(sw_smem(&sa_bars[grp]))
                   : "memory");
    }
  }
  if (live && !SA) {
    for (int r = gtid; r < min(a.R, pf_rows); r += GT) {
      const double* rp = Ai + (long long)r * a.A.ld;
      const uintptr_t lo = reinterpret_cast<uintptr_t>(rp) & ~(uintptr_t)15;
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(rp + K) + 15) & ~(uintptr_t)15;
      prefetch_l2_bulk(reinterpret_cast<const void*>(lo), (unsigned)(hi - lo));
    }
  }
  const int* xi = live ? a.xidx + (long long)item * a.xstride : nullptr;
  const int* x2 = (live && a.x2idx) ? a.x2idx + (long long)item * a.xstride : nullptr;
  if (NR == 1 && K <= 2 * GT && pre_index(4)) {
    // single RHS: the static gather indices are loaded before the launch wait
    int i1[2], i2[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = gtid + u * GT;
      i1[u] = (live && k < K) ? __ldg(xi + k) : -1;
      i2[u] = (k < K && x2) ? __ldg(x2 + k) : -1;
    }
    pdl_wait();
    if (!live) return;  // the whole group shares the item
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = gtid + u * GT;
      double v = i1[u] >= 0 ? a.pool[i1[u]] : 0.0;
      if (i2[u] >= 0) v -= a.pool[i2[u]];
      if (k < K) xs[k] = v;
    }
  } else {
    pdl_wait();
    if (!live) return;  // the whole group shares the item
    gather_x<NR>(xs, NR, xi, x2, a.pool, nrhs, K, K, gtid, GT);
  }
  if (GT == 32)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(GT) : "memory");
  if (SA)
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "SMW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n"
        "@!P bra SMW_%=;\n"
        "}\n" ::"r"(sw_smem(&sa_bars[grp]))
        : "memory");
  rows_dot<NR, false, 2, 4, SA>(SA ? tile + shift : Ai, a.A.ld, a.R, 0, a.R, K, lanes_for(K), xs,
                      a.aidx ? a.aidx + (long long)item * a.ostride : nullptr,
                      a.oidx + (long long)item * a.ostride, a.pool, nrhs, nullptr,
                      a.mode2 == 3 ? a.K2 : 1 << 30, a.mode2 == 3 ? a.o2idx + (long long)item * a.ostride : nullptr,
                      gtid >> 5, GT / 32);
}

static int sweep_ctas_target() { return 4 * 148; }

template <int NR>
static void launch_nr(const GemvArgs& a, cudaStream_t s) {
  int rows = 64;
  while (rows > 8 && (long long)a.nitems * ((a.R + rows - 1) / rows) < sweep_ctas_target()) rows >>= 1;
  if (rows > a.R) rows = a.R;
  int kchunk = (48 * 1024 / 8 - rows * NR) / NR;
  if (kchunk > a.K) kchunk = a.K;
  if (kchunk < 32) kchunk = 32;
  const size_t smem = sizeof(double) * ((size_t)kchunk * NR + (size_t)rows * NR);
  const int gx = (a.R + rows - 1) / rows;
  for (int off = 0; off < a.nitems; off += 65535) {
    dim3 grid(gx, min(65535, a.nitems - off));
    launch_k(gemv_gather_kernel<NR>, grid, dim3(SW_THREADS), smem, s, a, rows, kchunk, off);
  }
}

static bool vec16(const MatB& m) {
  if (m.ptrs) return false;
  return (reinterpret_cast<uintptr_t>(m.base + m.off) % 16 == 0) && m.ld % 2 == 0 && m.stride % 2 == 0;
}

template <int NRP>
static void launch_dmma(const GemvArgs& a, cudaStream_t s) {
  const bool vec = false && vec16(a.A);  // 16-byte path measured slower (r01); kept for tuning
  int rpc = 128;
  while (rpc > 16 && (rpc >= 2 * a.R || (long long)a.nitems * ((a.R + rpc - 1) / rpc) < 2 * 148)) rpc >>= 1;
  const int WR = rpc / 16, WK = 8 / WR;
  const size_t red = (size_t)(WK - 1) * WR * 32 * (4 * (NRP / 8));
  const int xld = vec ? NRP + 2 : NRP + 4;
  static int stage_env = -1;  // HPS_STAGE_IDX=0: gather indices read after the launch wait
  if (stage_env < 0) {
    const char* e = getenv("HPS_STAGE_IDX");
    stage_env = e ? atoi(e) : 1;
  }
  const int stage = stage_env && a.K <= 1024;
  const size_t idx_doubles = stage ? ((size_t)2 * a.K * sizeof(int) + 7) / 8 : 0;
  int kchunk = (int)((48 * 1024 / 8 - red - idx_doubles) / xld) & ~7;
  const int k8 = (a.K + 7) & ~7;
  if (kchunk > k8) kchunk = k8;
  const size_t smem = sizeof(double) * ((size_t)kchunk * xld + red + idx_doubles);
  const int gx = (a.R + rpc - 1) / rpc;
  for (int off = 0; off < a.nitems; off += 65535) {
    dim3 grid(gx, min(65535, a.nitems - off));
    if (vec)
      launch_k(gemv_dmma_kernel<NRP, true, 4>, grid, dim3(256), smem, s, a, rpc, kchunk, off, stage);
    else if (a.K >= 96)
      launch_k(gemv_dmma_kernel<NRP, false, HPS_DMMA_U2>, grid, dim3(256), smem, s, a, rpc, kchunk, off, stage);
    else
      launch_k(gemv_dmma_kernel<NRP, false, 4>, grid, dim3(256), smem, s, a, rpc, kchunk, off, stage);
  }
}

static int sweep_rows_per_cta(const GemvArgs& a) {
  static int rmax = -1;  // HPS_ROWS_MAX: cap on rows per CTA (tuning)
  if (rmax < 0) {
    const char* e = getenv("HPS_ROWS_MAX");
    rmax = e ? atoi(e) : 0;
  }
  int rows = a.R;
  if (a.mode2 != 2) {
    const int G = 32 / lanes_for(a.K);
    const int minrows = 8 * G * 2;
    static int rcap = -1;  // HPS_ROWS_CAP: most rows per CTA (each CTA gathers its item's x once)
    if (rcap < 0) {
      const char* e = getenv("HPS_ROWS_CAP");
      rcap = e ? atoi(e) : 64;
    }
    rows = a.R < rcap ? a.R : rcap;
    while (rows > minrows && (long long)a.nitems * ((a.R + rows - 1) / rows) < 4 * 148) rows = (rows + 1) / 2;
    if (rows < minrows) rows = minrows < a.R ? minrows : a.R;
    if (rmax > 0 && rows > rmax) rows = rmax;
  }
  return rows;
}

static int variant_of_env() {
  static int variant = -1;
  if (variant < 0) {
    const char* e = getenv("HPS_SWEEP_VARIANT");
    variant = e ? atoi(e) : 0;
  }
  return variant;
}

template <int NR>
static bool launch_sweep(const GemvArgs& a, cudaStream_t s) {
  {
    static int old = -1;
    if (old < 0) {
      const char* e = getenv("HPS_SWEEP_VARIANT");
      old = (e && atoi(e) != 9) ? 0 : 1;  // default: previous gemv_gather kernel for single-stage steps
    }
    // single-stage steps with long rows keep the gemv_gather kernel (HPS_GATHER_MINK: shortest K)
    static int mink = -1;
    if (mink < 0) {
      const char* e = getenv("HPS_GATHER_MINK");
      mink = e ? atoi(e) : 1 << 30;  // default: the staged-x kernel for every step whose x fits
    }
    if (old && a.mode2 == 0 && a.K >= mink) return false;
    if (old && a.mode2 == 3 && a.K >= mink && getenv("HPS_SPLIT3_GATHER")) return false;
  }
  const size_t smem = sizeof(double) * NR * ((size_t)a.K + (a.mode2 == 2 ? a.R : 0));
  if (smem > 48 * 1024) return false;
  {
    // chain steps (one CTA per item, two dependent stages) with too few items to fill the GPU
    // run as two row-chunked launches instead (HPS_CHAIN_SPLIT: item threshold)
    static int split = -1;
    if (split < 0) {
      const char* e = getenv("HPS_CHAIN_SPLIT");
      split = e ? atoi(e) : 300;
    }
    if (a.mode2 == 2 && a.nitems < split) return false;
  }
  if (a.mode2 == 3 && variant_of_env() != 0 && variant_of_env() != 3) return false;  // split needs the scalar path
  const int rows = sweep_rows_per_cta(a);
  const int gx = (a.R + rows - 1) / rows;
  {
    // deep levels: pack IPC items per CTA while a level still fills ~4 CTAs per SM (HPS_MULTI=0: off)
    static int multi = -1, min_ctas = 0;
    if (multi < 0) {
      const char* e = getenv("HPS_MULTI");
      multi = e ? atoi(e) : 1;
      e = getenv("HPS_MULTI_CTAS");
      min_ctas = e ? atoi(e) : 2 * 148;
    }
    int ipc = 1;
    static int msa = -1;  // HPS_MULTI_SA=0: no shared-memory operator tiles in the multi-item kernel
    if (msa < 0) {
      const char* e = getenv("HPS_MULTI_SA");
      msa = e ? atoi(e) : 1;
    }
    const size_t tile = sizeof(double) * (size_t)sa_tile_doubles(a.R, a.A.ld);
    const bool sa = msa && a.A.ptrs == nullptr && a.kparts <= 1 && tile <= 40 * 1024;  // larger: ipc = 1
    const size_t per_item = smem + (sa ? tile : 0);
    if (multi && gx == 1 && (a.mode2 == 0 || a.mode2 == 3)) {
      // next ipc: the level still gives min_ctas CTAs, x (and the tiles) fit, and the group's
      // warps cover the item's rows in at most 4 passes (warps x row groups per warp x 2 rows)
      // (+ the kernel's static shared memory: one 8-byte mbarrier per item, plus 16 B)
      while (ipc < 8 && (long long)a.nitems / (2 * ipc) >= min_ctas && (per_item + 8) * 2 * ipc + 16 <= 48 * 1024 &&
             a.R <= (8 / (2 * ipc)) * (32 / lanes_for(a.K)) * 2 * 4)
        ipc *= 2;
    }
    if (ipc > 1) {
      const long long ctas = (a.nitems + ipc - 1) / ipc;
      const int pf_rows = 1 << 30;
      const size_t sm2 = sa ? (((size_t)ipc * a.K * NR + 1) & ~(size_t)1) * sizeof(double) + tile * ipc : smem * ipc;
      for (long long off = 0; off < ctas; off += 2147483647LL) {
        const dim3 grid((unsigned)ctas);
        if (sa) {
          switch (ipc) {
            case 2: launch_k(sweep_multi_kernel<NR, 2, true>, grid, dim3(256), sm2, s, a, 0, pf_rows); break;
            case 4: launch_k(sweep_multi_kernel<NR, 4, true>, grid, dim3(256), sm2, s, a, 0, pf_rows); break;
            default: launch_k(sweep_multi_kernel<NR, 8, true>, grid, dim3(256), sm2, s, a, 0, pf_rows); break;
          }
          continue;
        }
        switch (ipc) {
          case 2: launch_k(sweep_multi_kernel<NR, 2>, grid, dim3(256), sm2, s, a, 0, pf_rows); break;
          case 4: launch_k(sweep_multi_kernel<NR, 4>, grid, dim3(256), sm2, s, a, 0, pf_rows); break;
          default: launch_k(sweep_multi_kernel<NR, 8>, grid, dim3(256), sm2, s, a, 0, pf_rows); break;
        }
      }
      return true;
    }
  }
  const int variant = variant_of_env();
  // L2 prefetch per CTA: all rows while a grid's worth (~4 CTAs x 148 SMs) fits in the 126 MB L2,
  // else the first 16 KB (p = 32 leaves: 588 KB per CTA, full prefetch ran at 4.3 TB/s vs 7.0)
  static long long pf_kb = -2;
  if (pf_kb == -2) {
    const char* e = getenv("HPS_PREFETCH_KB");
    pf_kb = e ? atoll(e) : -1;
  }
  const long long cta_bytes = 8LL * a.K * rows;
  const long long cap = pf_kb >= 0 ? pf_kb * 1024 : (cta_bytes <= 160 * 1024 ? cta_bytes : 16 * 1024);
  const int pf_rows = (int)(cap / (8LL * a.K));
  // SA: small operator tiles (latency-bound parent levels) go to shared memory by bulk copy
  static int sa_kb = -1;  // HPS_SA_KB: largest tile staged this way (0 = off)
  if (sa_kb < 0) {
    const char* e = getenv("HPS_SA_KB");
    sa_kb = e ? atoi(e) : 40;
  }
  const size_t sa_bytes = sizeof(double) * (size_t)sa_tile_doubles(rows, a.A.ld);
  // (+ 64 B of static shared memory: the tile's mbarrier)
  const bool sa = variant == 0 && sa_kb > 0 && sa_bytes <= (size_t)sa_kb * 1024 && smem + sa_bytes + 64 <= 48 * 1024;
  for (int off = 0; off < a.nitems; off += 65535) {
    dim3 grid(gx, min(65535, a.nitems - off));
    if (sa) {
      launch_k(sweep_kernel<NR, false, 2, 4, true>, grid, dim3(256), smem + sa_bytes, s, a, rows, off, pf_rows);
      continue;
    }
    switch (variant) {
      case 1: launch_k(sweep_kernel<NR, false, 1, 8>, grid, dim3(256), smem, s, a, rows, off, pf_rows); break;
      case 2: launch_k(sweep_kernel<NR, true, 1, 4>, grid, dim3(256), smem, s, a, rows, off, pf_rows); break;
      case 3: launch_k(sweep_kernel<NR, false, 1, 4>, grid, dim3(256), smem, s, a, rows, off, pf_rows); break;
      case 4: launch_k(sweep_kernel<NR, true, 2, 2>, grid, dim3(256), smem, s, a, rows, off, pf_rows); break;
      default: launch_k(sweep_kernel<NR, false, 2, 4>, grid, dim3(256), smem, s, a, rows, off, pf_rows); break;
    }
  }
  return true;
}

// One-row steps (split-K reductions with A = ones, the Dirichlet copy): one thread per
// (item, rhs), so thousands of tiny items do not each occupy a CTA.
__global__ void __launch_bounds__(256) gemv_row1_kernel(GemvArgs a) {
  pdl_trigger();
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = e < (long long)a.nitems * a.nrhs;
  const int item = live ? (int)(e / a.nrhs) : 0, j = live ? (int)(e - (long long)item * a.nrhs) : 0;
  const int* xi = a.xidx + (long long)item * a.xstride;
  const int* x2 = a.x2idx ? a.x2idx + (long long)item * a.xstride : nullptr;
  // the indices (static) before the launch wait, the pool values after it
  constexpr int KP = 8;
  const bool pre = pre_index(8);
  int i1[KP], i2[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    i1[k] = (pre && live && k < a.K) ? __ldg(xi + k) : -1;
    i2[k] = (pre && live && k < a.K && x2) ? __ldg(x2 + k) : -1;
  }
  pdl_wait();
  if (!pre && live) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      i1[k] = k < a.K ? xi[k] : -1;
      i2[k] = (k < a.K && x2) ? x2[k] : -1;
    }
  }
  if (!live) return;
  const double* A = a.A.get(item);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    if (k >= a.K) break;
    double v = a.pool[(long long)i1[k] * a.nrhs + j];
    if (i2[k] >= 0) v -= a.pool[(long long)i2[k] * a.nrhs + j];
    acc = fma(A[k], v, acc);
  }
  for (int k = KP; k < a.K; ++k) {
    double v = a.pool[(long long)xi[k] * a.nrhs + j];
    if (x2 && x2[k] >= 0) v -= a.pool[(long long)x2[k] * a.nrhs + j];
    acc = fma(A[k], v, acc);
  }
  const long long o = (long long)a.oidx[(long long)item * a.ostride] * a.nrhs + j;
  if (a.aidx) acc += a.pool[(long long)a.aidx[(long long)item * a.ostride] * a.nrhs + j];
  a.pool[o] = acc;
}

int launch_gemv_gather(const GemvArgs& a0, cudaStream_t s) {
  if (a0.nitems <= 0 || a0.R <= 0) return 0;
  GemvArgs a = a0;
  g_pdl_now = sweep_pdl_for(a.nrhs, false) ||
              (sweep_pdl_for(a.nrhs, true) && 8.0e-6 * a.nitems * a.R * a.K <= pdl_max_mb());
  // the L2 prefetch of a CTA's operator rows pays when it runs ahead of the launch wait; without
  // a dependent launch it only doubles the L2 requests (config 5, 16 RHS: 3.47 -> 3.41 ms)
  if (!g_pdl_now && a.nrhs > 2) a.pre_mask &= ~16;
  if (a.R == 1 && !a.mode2 && a.K <= 64) {
    const long long n = (long long)a.nitems * a.nrhs;
    launch_k(gemv_row1_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, a);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  if (a.nrhs <= 2) {
    const bool ok = a.nrhs == 1 ? launch_sweep<1>(a, s) : launch_sweep<2>(a, s);
    if (ok) return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  if (a.nrhs > 2 && a.mode2 == 1 && launch_gemv_stream(a, s)) return cudaGetLastError() == cudaSuccess ? 0 : 2;
  if (a.nrhs > 2 && launch_gemv_tma(a, s)) return cudaGetLastError() == cudaSuccess ? 0 : 2;
  if (a.nrhs > 2 && launch_gemv_stream(a, s)) return cudaGetLastError() == cudaSuccess ? 0 : 2;
  if (a.nrhs > 2 && a.nrhs <= 16 && a.R > 1 && !a.A.ptrs) {
    const bool ok = a.nrhs <= 8 ? launch_dmma_multi<8>(a, s) : launch_dmma_multi<16>(a, s);
    if (ok) return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  if (a.mode2 == 3 && a.nrhs > 2) {
    // split output on the multi-RHS path: w = A[:, :K2] x[:K2] -> o2idx, then
    // y = A[:, K2:] x[K2:] + w -> oidx (the same operator bytes, two launches)
    GemvArgs b = a;
    b.mode2 = 0;
    b.K = a.K2;
    b.oidx = a.o2idx;
    int rc = launch_gemv_gather(b, s);
    if (rc) return rc;
    GemvArgs c = a;
    c.mode2 = 0;
    c.K = a.K - a.K2;
    c.A.off += a.K2;
    c.xidx = a.xidx + a.K2;
    c.x2idx = a.x2idx ? a.x2idx + a.K2 : nullptr;
    c.aidx = a.o2idx;
    return launch_gemv_gather(c, s);
  }
  if (a.mode2 && a.mode2 != 3) {
    // second stage for the chunked / multi-RHS paths: separate launch after the first
    GemvArgs b = a;
    b.mode2 = 0;
    int rc = launch_gemv_gather(b, s);
    if (rc) return rc;
    GemvArgs c{};
    c.nitems = a.nitems;
    c.nrhs = a.nrhs;
    c.pre_mask = a.pre_mask;
    c.pool = a.pool;
    c.A = a.A2;
    c.R = a.R2;
    c.K = a.K2;
    c.aidx = a.a2idx;
    c.oidx = a.o2idx;
    c.ostride = a.R2;
    if (a.mode2 == 1) {
      // tail: the last K2 gather indices of the first stage (no difference operand)
      if (a.x2idx) return 1;
      c.xidx = a.xidx + (a.K - a.K2);
      c.xstride = a.xstride;
    } else {
      c.xidx = a.oidx;  // chain: x of the second stage = y1 rows in the pool
      c.xstride = a.ostride;
    }
    return launch_gemv_gather(c, s);
  }
  if (a.nrhs <= 1)
    launch_nr<1>(a, s);
  else if (a.nrhs <= 2)
    launch_nr<2>(a, s);
  else if (a.nrhs <= 8)
    launch_dmma<8>(a, s);
  else if (a.nrhs <= 16)
    launch_dmma<16>(a, s);
  else
    return 1;
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
