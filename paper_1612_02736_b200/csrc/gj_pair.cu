// Batched Gauss-Jordan inversion with partial pivoting for many SMALL matrices (p = 16 leaves:
// M = [A_ii | -A_ie L], 196 x 256), one 2-CTA thread-block cluster per matrix with the whole
// matrix resident in the pair's shared memory (column split: CTA c owns columns
// [c*C0, min(ncols, (c+1)*C0)), C0 = ncols/2 rounded up to 8; 196 x 128 doubles = 200 KB each).
//
// Blocked right-looking GJ with panels of NB = 8 pivot columns and a one-panel look-ahead:
//   step p, CTA owning panel p+1:  warp 0 updates panel p+1's columns with panel p, factors
//                                   panel p+1 (rows in registers, warp-shuffle argmax, LAPACK
//                                   tie rule) and pushes P_{p+1} + pivots into the peer's shared
//                                   memory (DSMEM) with a remote mbarrier arrive;
//                                   warps 1..7 meanwhile apply panel p to every other column;
//   step p, other CTA:              all 8 warps apply panel p to its columns.
// Applying a panel = its 8 row interchanges, then C <- D C + P W on DMMA tiles (W: the 8 pivot
// rows before the update, D: identity with the pivot rows zeroed; gj.cu / gj_cluster.cu use the
// same identity). The factored panel stays in place in its owner's columns; the peer gets a
// copy in a double buffer whose reuse is released by a remote arrive (back-pressure).
//
// Why: the one-CTA-per-matrix persistent kernel (gj_fused.cu) cannot hold the 401 KB augmented
// matrix on chip, so every panel streamed the whole matrix through L2 with 2 CTAs per SM at
// 25 % occupancy (config 5 leaf stage 51 ms). Here the matrix crosses HBM once each way and the
// serial pivot chain of the next panel runs under the DMMA update of the current one.
//
// Shared-memory layout of the owned columns: row-major, 128 doubles per row (cw <= 128), the
// 16-byte chunk index XOR-ed with ((row & 1) << 2) so the C-fragment accesses of a quarter warp
// (rows g, g+1 x 4 column pairs) fall into 8 distinct bank groups without padding.
//
// Outputs as gj_fused full mode: inverse columns left in pivot order (perm_out) or un-permuted,
// the right-hand-side columns multiplied by the inverse, LAPACK pivots, |A^-1|_1, status flags.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace cg = cooperative_groups;

namespace hps {

namespace {

constexpr int GP_THREADS = 256;
constexpr int GP_WARPS = GP_THREADS / 32;
constexpr int GP_NB = 8;
constexpr int GP_LD = 128;  // owned-column capacity (row length in shared memory)
constexpr int GP_RPL = 6;   // register-resident panel rows per lane in the factor warp (n <= 224)

__device__ __forceinline__ int sw(int r, int c) {
  // swizzled position of (row r, column c): 16-byte chunk index ^ ((r & 1) << 2)
  return r * GP_LD + ((((c >> 1) ^ ((r & 1) << 2))) << 1) + (c & 1);
}

struct GpLayout {
  int n;
  __host__ __device__ explicit GpLayout(int n_) : n(n_) {}
  __host__ __device__ size_t ms() const { return 0; }                               // n x 128
  __host__ __device__ size_t pb() const { return (size_t)n * GP_LD; }               // [2][n][NB] peer panels
  __host__ __device__ size_t prow() const { return pb() + 2 * (size_t)n * GP_NB; }  // [2][NB] rows pr, cj
  __host__ __device__ size_t bars() const { return prow() + 2 * GP_NB; }            // 4 mbarriers
  __host__ __device__ size_t red() const { return bars() + 4; }                      // [16]
  __host__ __device__ size_t ints() const { return red() + 16; }
  // ints: piv[n], spiv[2][NB], perm[n]
  __host__ __device__ size_t total_doubles() const { return ints() + (2 * (size_t)n + 2 * GP_NB + 1) / 2 + 1; }
};

__device__ __forceinline__ uint32_t s_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_addr(b)), "r"(cnt));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n}\n" ::"r"(s_addr(b)),
      "r"(parity)
      : "memory");
}
// arrive on the peer CTA's mbarrier (release at cluster scope: our earlier DSMEM stores are
// visible to a thread that completes a wait on it)
__device__ __forceinline__ void bar_arrive_remote(uint64_t* local_bar, int rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(s_addr(local_bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}

}  // namespace

// One DMMA sweep applying a factored panel (OWNP: in place in the shared matrix at columns
// pc0.., else P: n x NB dense) to the columns [cbeg, cend): non-pivot rows C += P W, then
// (after a barrier among the nw warps) the pivot rows k0.. C = P_J W. W = rows k0.. (read in
// place). Columns in [skip_lo, skip_hi) are left untouched. Executed by warps [w0, w0 + nw).
template <bool OWNP>
__device__ __forceinline__ void gp_apply(double* Ms, int n, int k0, int kb, const double* P, int pc0, int cbeg,
                                         int cend, int skip_lo, int skip_hi, int w0, int nw, int bar_id) {
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - w0;
  const int g = lane >> 2, t = lane & 3;
  auto pval = [&](int r, int kk) -> double {
    if (r >= n || kk >= kb) return 0.0;
    return OWNP ? Ms[sw(r, pc0 + kk)] : P[r * GP_NB + kk];
  };
  auto wval = [&](int kk, int c) -> double { return (c < cend && kk < kb) ? Ms[sw(k0 + kk, c)] : 0.0; };
  auto skip = [&](int c) { return c >= skip_lo && c < skip_hi; };
  const int ncol = cend - cbeg;
  const int mt = (n + 15) >> 4, ntl = (ncol + 15) >> 4;
  // (a) every 16 x 16 block outside the pivot tile
  for (int blk = warp; blk < mt * ntl; blk += nw) {
    const int rb = (blk / ntl) * 16, cb = cbeg + (blk % ntl) * 16;
    double d[2][2][2], af[2][2];
    bool live[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int tr = rb + mi * 8, r = tr + g;
      live[mi] = tr < n && tr != k0;
#pragma unroll
      for (int k4 = 0; k4 < 2; ++k4) af[mi][k4] = live[mi] ? pval(r, k4 * 4 + t) : 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int c = cb + nt * 8 + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (live[mi] && r < n && c < cend) v = *reinterpret_cast<const double2*>(Ms + sw(r, c));
        d[mi][nt][0] = v.x;
        d[mi][nt][1] = v.y;
      }
    }
    if (!live[0] && !live[1]) continue;
#pragma unroll
    for (int k4 = 0; k4 < 2; ++k4) {
      const double b0 = wval(k4 * 4 + t, cb + g), b1 = wval(k4 * 4 + t, cb + 8 + g);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        dmma8x8x4(d[mi][0][0], d[mi][0][1], af[mi][k4], b0);
        dmma8x8x4(d[mi][1][0], d[mi][1][1], af[mi][k4], b1);
      }
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r = rb + mi * 8 + g;
      if (!live[mi] || r >= n) continue;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int c = cb + nt * 8 + 2 * t;
        if (c >= cend) continue;
        const bool s0 = !skip(c), s1 = c + 1 < cend && !skip(c + 1);
        if (s0 && s1) {
          *reinterpret_cast<double2*>(Ms + sw(r, c)) = make_double2(d[mi][nt][0], d[mi][nt][1]);
        } else {
          if (s0) Ms[sw(r, c)] = d[mi][nt][0];
          if (s1) Ms[sw(r, c + 1)] = d[mi][nt][1];
        }
      }
    }
  }
  // every W read of (a) before the pivot rows are overwritten
  if (nw == 1)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(nw * 32) : "memory");
  // (b) the pivot tile: rows k0 .. k0 + kb
  for (int ct = warp; ct < (ncol + 7) >> 3; ct += nw) {
    const int cb = cbeg + ct * 8, c = cb + 2 * t, r = k0 + g;
    const double a0 = pval(r, t), a1 = pval(r, 4 + t);
    const double b0 = wval(t, cb + g), b1 = wval(4 + t, cb + g);
    __syncwarp();  // every lane has read W before any lane overwrites the pivot rows
    double dd[2] = {0.0, 0.0};
    dmma8x8x4(dd[0], dd[1], a0, b0);
    dmma8x8x4(dd[0], dd[1], a1, b1);
    if (g < kb && c < cend) {
      if (!skip(c)) Ms[sw(r, c)] = dd[0];
      if (c + 1 < cend && !skip(c + 1)) Ms[sw(r, c + 1)] = dd[1];
    }
  }
}

// Warp-level factorisation of panel [k0, k0+kb) held in columns pc0.. of the shared matrix:
// rows lane + 32 s (s < GP_RPL) live in registers, the overflow rows GP_RPL*32 + lane (n up to
// 32 (GP_RPL + 1)) are updated in place in shared memory; per column: argmax with the LAPACK tie
// rule, interchange, scaling, elimination. Returns the status flag (zero / NaN pivot).
#ifdef GP_TRACE
// phase timestamps (clock64) of the first item of cluster 0, printed after the item: debug only
__device__ long long gp_tr[2][2][32][8];
#define GP_T(tag, p)                                                                   \
  if (blockIdx.x < 2 && item == 0 && (threadIdx.x == 0 || threadIdx.x == 32) && (p) < 32) \
    gp_tr[blockIdx.x][threadIdx.x >> 5][(p)][(tag)] = clock64();
__device__ long long gp_tf[32][8][6];
#define GP_F(tag) if (gp_trc) gp_tf[k0 >> 3][j][(tag)] = clock64();
#else
#define GP_F(tag)
#define GP_T(tag, p)
#endif

__device__ __forceinline__ int gp_factor_warp(double* Ms, double* prow, int n, int k0, int kb, int pc0, int* spiv,
                                              int* piv_s) {
  const int lane = threadIdx.x & 31;
#ifdef GP_TRACE
  const bool gp_trc = blockIdx.x == 0 && lane == 0 && k0 < 256;
#endif
  const int rx = GP_RPL * 32 + lane;  // overflow row of this lane (shared memory)
  double v[GP_RPL][GP_NB];
#pragma unroll
  for (int s = 0; s < GP_RPL; ++s) {
    const int r = lane + 32 * s;
#pragma unroll
    for (int c = 0; c < GP_NB; ++c) v[s][c] = (r < n && c < kb) ? Ms[sw(r, pc0 + c)] : 0.0;
  }
  int flag = 0;
  double* crow = prow + GP_NB;
#pragma unroll
  for (int j = 0; j < GP_NB; ++j) {
    if (j >= kb) break;
    const int cj = k0 + j;
    GP_F(0)
    double best = -1.0;
    int bi = n;
#pragma unroll
    for (int s = 0; s < GP_RPL; ++s) {
      const int r = lane + 32 * s;
      const double av = fabs(v[s][j]);
      if (r < n && r >= cj && av > best) {
        best = av;
        bi = r;
      }
    }
    if (rx < n && rx >= cj) {
      const double av = fabs(Ms[sw(rx, pc0 + j)]);
      if (av > best) {
        best = av;
        bi = rx;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    GP_F(1)
    const int pr = bi >= n ? cj : bi;  // all NaN: keep the diagonal, NaN propagates
    if (!(best > 0.0)) flag = 1;
    // rows pr (the pivot row) and cj (moves to pr) through shared memory, from their owner lanes
    const int sp = pr >> 5, sc = cj >> 5;
#pragma unroll
    for (int s = 0; s < GP_RPL; ++s) {
      if (s == sp && lane == (pr & 31))
#pragma unroll
        for (int c = 0; c < GP_NB; ++c) prow[c] = v[s][c];
      if (s == sc && lane == (cj & 31))
#pragma unroll
        for (int c = 0; c < GP_NB; ++c) crow[c] = v[s][c];
    }
    // (overflow rows: only the kb panel columns are read or written; the rest of the 8-column
    // window may belong to other columns of the matrix, updated concurrently by other warps)
    if (sp >= GP_RPL && lane == (pr & 31))
#pragma unroll
      for (int c = 0; c < GP_NB; ++c) prow[c] = c < kb ? Ms[sw(pr, pc0 + c)] : 0.0;
    if (sc >= GP_RPL && lane == (cj & 31))
#pragma unroll
      for (int c = 0; c < GP_NB; ++c) crow[c] = c < kb ? Ms[sw(cj, pc0 + c)] : 0.0;
    __syncwarp();
    GP_F(2)
    const double inv = 1.0 / prow[j];
    GP_F(3)
#pragma unroll
    for (int s = 0; s < GP_RPL; ++s) {
      const int r = lane + 32 * s;
      if (r >= n) continue;
      if (r == cj) {
#pragma unroll
        for (int c = 0; c < GP_NB; ++c) v[s][c] = (c == j) ? inv : prow[c] * inv;
        continue;
      }
      if (r == pr) {
#pragma unroll
        for (int c = 0; c < GP_NB; ++c) v[s][c] = crow[c];
      }
      const double f = v[s][j];
#pragma unroll
      for (int c = 0; c < GP_NB; ++c) v[s][c] = (c == j ? 0.0 : v[s][c]) - f * ((c == j) ? inv : prow[c] * inv);
    }
    GP_F(4)
    if (rx < n) {
      if (rx == cj) {
#pragma unroll
        for (int c = 0; c < GP_NB; ++c)
          if (c < kb) Ms[sw(rx, pc0 + c)] = (c == j) ? inv : prow[c] * inv;
      } else {
        double w[GP_NB];
#pragma unroll
        for (int c = 0; c < GP_NB; ++c) w[c] = c >= kb ? 0.0 : ((rx == pr) ? crow[c] : Ms[sw(rx, pc0 + c)]);
        const double f = w[j];
#pragma unroll
        for (int c = 0; c < GP_NB; ++c)
          if (c < kb) Ms[sw(rx, pc0 + c)] = (c == j ? 0.0 : w[c]) - f * ((c == j) ? inv : prow[c] * inv);
      }
    }
    if (lane == 0) {
      spiv[j] = pr;
      piv_s[cj] = pr;
    }
    __syncwarp();  // prow / crow are rewritten by the next column
    GP_F(5)
  }
#pragma unroll
  for (int s = 0; s < GP_RPL; ++s) {
    const int r = lane + 32 * s;
    if (r < n)
#pragma unroll
      for (int c = 0; c < GP_NB; ++c)
        if (c < kb) Ms[sw(r, pc0 + c)] = v[s][c];
  }
  __syncwarp();
  return flag;
}


__global__ void __launch_bounds__(GP_THREADS, 1) gj_pair_kernel(FusedArgs a, int C0) {
  extern __shared__ double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int peer = rank ^ 1;
  const int n = a.n, ncols = a.ncols;
  const int c0 = rank * C0;
  const int cw = min(ncols, c0 + C0) - c0;  // columns owned by this CTA
  const GpLayout L(n);
  double* Ms = sm + L.ms();
  double* Pb = sm + L.pb();
  double* prow = sm + L.prow();
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars());
  uint64_t* pready = bars;     // [2]: a peer panel landed in Pb[b] (remote arrive by its producer)
  uint64_t* pfree = bars + 2;  // [2]: the peer released our copy in its Pb[b] (back-pressure)
  double* red = sm + L.red();
  int* piv_s = reinterpret_cast<int*>(sm + L.ints());
  int* spiv = piv_s + n;  // [2][NB] pivots of the panels in flight (by buffer)
  int* perm = spiv + 2 * GP_NB;
  double* peer_Pb = cluster.map_shared_rank(Pb, peer);
  int* peer_spiv = cluster.map_shared_rank(spiv, peer);
  double* peer_red = cluster.map_shared_rank(red, peer);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pairs = gridDim.x / 2;
  const int npan = (n + GP_NB - 1) / GP_NB;
  auto owner_of = [&](int p) { return p * GP_NB < C0 ? 0 : 1; };
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) bar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // completed-phase counters per buffer (uniform across the CTA)
  unsigned ready_cnt[2] = {0, 0}, free_cnt[2] = {0, 0};
  cluster.sync();

  // (warp 0 of the owner) P_p -> the peer's Pb[p & 1] + its pivots, then the peer's pready
  // arrive; first wait until the peer released that buffer (its step p - 2 is complete,
  // whoever owned panel p - 2)
  auto push = [&](int p, int pc0) {
    const int b = p & 1, kb = min(GP_NB, n - p * GP_NB);
    if (p >= 2) {
      bar_wait(pfree + b, free_cnt[b] & 1u);
      ++free_cnt[b];
    }
    for (int e = lane; e < n * GP_NB; e += 32) {
      const int r = e / GP_NB, c = e - r * GP_NB;
      peer_Pb[(size_t)b * n * GP_NB + e] = c < kb ? Ms[sw(r, pc0 + c)] : 0.0;
    }
    if (lane < GP_NB) peer_spiv[b * GP_NB + lane] = spiv[b * GP_NB + lane];
    __syncwarp();
    if (lane == 0) bar_arrive_remote(pready + b, peer);
  };

  for (int item = blockIdx.x / 2; item < a.batch; item += pairs) {
    double* Mi = a.M.get(item);
    const long long ld = a.M.ld;
    for (int e = tid; e < n * cw; e += GP_THREADS) {
      const int r = e / cw, c = e - r * cw;
      Ms[sw(r, c)] = Mi[(long long)r * ld + c0 + c];
    }
    int flag = 0;
    cluster.sync();  // both halves loaded; no DSMEM traffic of the previous item outstanding

    // panel 0: factored by its owner (warp 0) before the loop
    if (owner_of(0) == rank && warp == 0) {
      flag |= gp_factor_warp(Ms, prow, n, 0, min(GP_NB, n), 0, spiv, piv_s);
      push(0, 0);
    }
    __syncthreads();

    for (int p = 0; p < npan; ++p) {
      const int k0 = p * GP_NB, kb = min(GP_NB, n - k0), b = p & 1;
      const bool own = owner_of(p) == rank;
      const bool own_next = p + 1 < npan && owner_of(p + 1) == rank;
      const int lk0 = k0 - c0;  // local column of panel p (owner)
      GP_T(0, p)
      if (!own) {
        bar_wait(pready + b, ready_cnt[b] & 1u);  // P_p and its pivots landed in Pb[b]
        ++ready_cnt[b];
      }
      GP_T(1, p)
      const int* pv = spiv + b * GP_NB;
      const double* P = own ? nullptr : Pb + (size_t)b * n * GP_NB;
      const int skip_lo = own ? lk0 : -1, skip_hi = own ? lk0 + kb : -1;
      // 1. the panel's row interchanges on every other own column
      for (int c = tid; c < cw; c += GP_THREADS) {
        if (c >= skip_lo && c < skip_hi) continue;
#pragma unroll 1
        for (int j = 0; j < kb; ++j) {
          const int pr = pv[j], cj = k0 + j;
          if (pr != cj) {
            const double x = Ms[sw(cj, c)];
            Ms[sw(cj, c)] = Ms[sw(pr, c)];
            Ms[sw(pr, c)] = x;
          }
        }
      }
      __syncthreads();
      GP_T(2, p)
      // 2. apply panel p; the owner of panel p+1 factors it on warp 0 meanwhile
      if (own_next) {
        const int nk0 = k0 + GP_NB, nlk = nk0 - c0, nkb = min(GP_NB, n - nk0);
        if (warp == 0) {
          if (own)
            gp_apply<true>(Ms, n, k0, kb, nullptr, lk0, nlk, nlk + nkb, skip_lo, skip_hi, 0, 1, 0);
          else
            gp_apply<false>(Ms, n, k0, kb, P, 0, nlk, nlk + nkb, skip_lo, skip_hi, 0, 1, 0);
          GP_T(3, p)
          flag |= gp_factor_warp(Ms, prow, n, nk0, nkb, nlk, spiv + ((p + 1) & 1) * GP_NB, piv_s);
          GP_T(4, p)
          push(p + 1, nlk);
          GP_T(5, p)
        } else {
          // columns [0, nlk) and [nlk + nkb, cw) on warps 1..7 (named barrier 1)
          if (own) {
            gp_apply<true>(Ms, n, k0, kb, nullptr, lk0, 0, nlk, skip_lo, skip_hi, 1, GP_WARPS - 1, 1);
            gp_apply<true>(Ms, n, k0, kb, nullptr, lk0, nlk + nkb, cw, skip_lo, skip_hi, 1, GP_WARPS - 1, 1);
          } else {
            gp_apply<false>(Ms, n, k0, kb, P, 0, 0, nlk, skip_lo, skip_hi, 1, GP_WARPS - 1, 1);
            gp_apply<false>(Ms, n, k0, kb, P, 0, nlk + nkb, cw, skip_lo, skip_hi, 1, GP_WARPS - 1, 1);
          }
        }
      } else {
        if (own)
          gp_apply<true>(Ms, n, k0, kb, nullptr, lk0, 0, cw, skip_lo, skip_hi, 0, GP_WARPS, 1);
        else
          gp_apply<false>(Ms, n, k0, kb, P, 0, 0, cw, skip_lo, skip_hi, 0, GP_WARPS, 1);
      }
      GP_T(6, p)
      __syncthreads();
      // 3. buffers (Pb, spiv)[p & 1] are done with: release them to the peer if it is the one
      //    that will fill them next (panel p + 2)
      if (tid == 0 && p + 2 < npan && owner_of(p + 2) != rank) bar_arrive_remote(pfree + b, peer);
    }

#ifdef GP_TRACE
    if (blockIdx.x == 0 && item == 0 && threadIdx.x == 0)
      for (int q = 0; q < 8; ++q)
        for (int j = 0; j < 8; ++j)
          printf("GPF p=%d j=%d %lld %lld %lld %lld %lld %lld\n", q, j, gp_tf[q][j][0], gp_tf[q][j][1], gp_tf[q][j][2],
                 gp_tf[q][j][3], gp_tf[q][j][4], gp_tf[q][j][5]);
    if (blockIdx.x < 2 && item == 0 && (threadIdx.x == 0 || threadIdx.x == 32))
      for (int q = 0; q < npan && q < 32; ++q)
        printf("GPT r%d t%d p=%d %lld %lld %lld %lld %lld %lld %lld\n", (int)blockIdx.x, (int)threadIdx.x, q,
               gp_tr[blockIdx.x][threadIdx.x >> 5][q][0], gp_tr[blockIdx.x][threadIdx.x >> 5][q][1],
               gp_tr[blockIdx.x][threadIdx.x >> 5][q][2], gp_tr[blockIdx.x][threadIdx.x >> 5][q][3],
               gp_tr[blockIdx.x][threadIdx.x >> 5][q][4], gp_tr[blockIdx.x][threadIdx.x >> 5][q][5],
               gp_tr[blockIdx.x][threadIdx.x >> 5][q][6]);
#endif
    // ---------------- epilogue: pivots, column order, |A^-1|_1, write back
    cluster.sync();  // both halves factored; piv_s complete on both sides
    {
      int* peer_piv = cluster.map_shared_rank(piv_s, peer);
      for (int j = tid; j < n; j += GP_THREADS)
        if (owner_of(j / GP_NB) != rank) piv_s[j] = peer_piv[j];
    }
    __syncthreads();
    if (rank == 0)
      for (int j = tid; j < n; j += GP_THREADS) a.piv[(long long)item * n + j] = piv_s[j];
    if (tid == 0) {
      for (int j = 0; j < n; ++j) perm[j] = j;
      for (int j = 0; j < n; ++j) {
        const int r = piv_s[j];
        const int x = perm[j];
        perm[j] = perm[r];
        perm[r] = x;
      }
    }
    __syncthreads();
    if (rank == 0 && a.perm_out) {
      int* po = a.perm_out + (long long)item * n;
      for (int j = tid; j < n; j += GP_THREADS) po[j] = perm[j];
    }
    // |A^-1|_1: max column sum over the inverse columns (the first n global columns)
    double best = 0.0;
    for (int c = tid; c < cw; c += GP_THREADS) {
      if (c0 + c >= n) continue;
      double s = 0.0;
      for (int r = 0; r < n; ++r) s += fabs(Ms[sw(r, c)]);
      best = (s > best || s != s) ? s : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      best = (ov > best || ov != ov) ? ov : best;
    }
    if (lane == 0) red[warp] = best;
    __syncthreads();
    if (tid == 0) {
      double bb = red[0];
      for (int w = 1; w < GP_WARPS; ++w) bb = (red[w] > bb || red[w] != red[w]) ? red[w] : bb;
      if (rank == 1) peer_red[8] = bb;  // CTA 0 combines
      red[9] = bb;
    }
    // write back: inverse columns stay in pivot order when perm_out is set, else un-permuted
    // (inverse column perm[j] = stored column j)
    for (int e = tid; e < n * cw; e += GP_THREADS) {
      const int r = e / cw, c = e - r * cw, gc = c0 + c;
      const int dst = (a.perm_out || gc >= n) ? gc : perm[gc];
      Mi[(long long)r * ld + dst] = Ms[sw(r, c)];
    }
    cluster.sync();  // peer_red written; every DSMEM read of this item done
    if (rank == 0 && tid == 0 && a.ainvnorm) {
      const double b0 = red[9], b1 = red[8];
      a.ainvnorm[item] = (b1 > b0 || b1 != b1) ? b1 : b0;
    }
    if (tid == 0 && flag && a.status) atomicOr(a.status + item, 1);
  }
}

size_t gj_pair_smem(int n) { return sizeof(double) * GpLayout(n).total_doubles(); }

bool gj_pair_ok(int n, int ncols) {
  static int on = -1;  // opt-in (HPS_GJ_PAIR=1): slower than the one-CTA fused kernel so far
  if (on < 0) {
    const char* e = getenv("HPS_GJ_PAIR");
    on = e ? atoi(e) : 0;
  }
  const int C0 = (((ncols + 1) / 2) + 7) & ~7;
  return on && n <= 32 * (GP_RPL + 1) && n >= 64 && ncols >= n && C0 <= GP_LD && ncols <= 2 * C0 &&
         gj_pair_smem(n) <= 227 * 1024;
}

int launch_gj_pair(const FusedArgs& a, cudaStream_t s) {
  if (!gj_pair_ok(a.n, a.ncols)) return 1;
  const int C0 = (((a.ncols + 1) / 2) + 7) & ~7;
  const size_t smem = gj_pair_smem(a.n);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gj_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int pairs = a.batch < sms / 2 ? a.batch : sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(GP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gj_pair_kernel, a, C0) == cudaSuccess ? 0 : 2;
}

}  // namespace hps
