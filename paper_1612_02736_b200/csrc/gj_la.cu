// Batched Gauss-Jordan inversion with partial pivoting for the p = 16 leaf blocks (n <= 224,
// [A | R] of 196 x 256): one persistent 512-thread CTA per SM with WARP-SPECIALISED LOOK-AHEAD.
//
// gj_fused_kernel runs the phases of a panel one after the other (pivot-column loop 39 % of its
// time, DMMA trailing update 35 %, 2 CTAs per SM for overlap by chance). Here the two phases of
// consecutive panels run side by side inside one CTA:
//   panel group P (warps 0..6, one matrix row per thread, panel rows in registers):
//       factor panel k  ->  publish it (shared memory + global)  ->  apply it to the columns of
//       panel k+1 only (one 32-column DMMA tile per warp)  ->  load panel k+1  ->  factor ...
//   update group U (warps 7..15): apply panel k to every other column, the columns of panel k+2
//       first (P needs them next), while P is already factoring panel k+1.
// Panels k, k+1, k+2 are adjacent, so U's column set is "everything but one contiguous range".
// Hand-offs are CTA-scope mbarriers (full[2]: panel published; empty[2]: panel buffer free;
// la[2]: look-ahead columns ready); every wait is bounded (trap instead of a hang).
// The arithmetic per column (arg-max rule, scaling, elimination order) and the composed row
// interchanges are those of gj_fused_kernel, so pivots and results are identical.
#include <cstdlib>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

namespace {

constexpr int LA_KB = 28;
constexpr int LA_PW = 7, LA_UW = 9;
constexpr int LA_PT = 32 * LA_PW, LA_UT = 32 * LA_UW, LA_THREADS = LA_PT + LA_UT;
constexpr int LA_LDWP = 36;  // look-ahead W: 32 columns + 4 (== 4 mod 16)

__device__ __forceinline__ void la_bar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void la_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
#ifdef LA_DEBUG
__device__ int* la_dbg = nullptr;  // host-mapped buffer: (code, k, parity, tid, block) of a timed-out wait
#define LA_DBG_ARGS , int code, int kk
#define LA_DBG(code, kk) , code, kk
#else
#define LA_DBG_ARGS
#define LA_DBG(code, kk)
#endif

__device__ __forceinline__ void la_wait(uint64_t* b, unsigned parity LA_DBG_ARGS) {
  unsigned done = 0, spins = 0;
  while (!done) {
    asm volatile(
        "{\n.reg .pred P;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
#ifdef LA_DEBUG
    if (!done && ++spins > (1u << 14)) {
      if (la_dbg && atomicCAS(la_dbg, 0, code) == 0) {
        la_dbg[1] = kk;
        la_dbg[2] = (int)parity;
        la_dbg[3] = (int)threadIdx.x;
        la_dbg[4] = (int)blockIdx.x;
        __threadfence_system();
      }
      __trap();
    }
#else
    if (!done && ++spins > (1u << 24)) __trap();  // never a silent hang
#endif
  }
}
#ifdef LA_DEBUG
__device__ long long la_prof[16];
#define LA_T(idx)                                                     \
  if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == LA_PT)) { \
    const long long now_ = clock64();                                 \
    atomicAdd((unsigned long long*)&la_prof[idx], (unsigned long long)(now_ - la_last)); \
    la_last = now_;                                                   \
  }
#else
#define LA_T(idx)
#endif

__device__ __forceinline__ void bar_p() { asm volatile("bar.sync 1, %0;\n" ::"n"(LA_PT) : "memory"); }
__device__ __forceinline__ void bar_u() { asm volatile("bar.sync 2, %0;\n" ::"n"(LA_UT) : "memory"); }

struct LaCtrl {
  int spiv[LA_KB];
  int wsrc[LA_KB];
  int moves[2 * LA_KB + 4];  // [0] = count, then (dst, src) pairs
};

size_t la_smem_bytes(int n, int ldp, int ldw) {
  return sizeof(double) * ((size_t)2 * LA_KB * ldp + (size_t)LA_KB * ldw + (size_t)LA_KB * LA_LDWP +
                           2 * (LA_PW + 1) * (LA_KB + 2) + 2 * LA_KB + 16 + 8) +
         2 * sizeof(LaCtrl) + sizeof(int) * ((size_t)n + 8);
}

// Apply the factored panel (Pk: column-major [KB][ldp], pivot columns [k0, k0 + kbc)) to cw columns
// whose pivot rows are staged in Wt ([KB][ldwt]); physical column of local column cl = cmap(cl).
// Tiles of 32 x 32 dealt to the nw warps of the calling group (warp index wi).
template <typename CMap>
__device__ __forceinline__ void la_update_tiles(double* Mi, long long ld, int n, int k0, int kbc, const double* Pk,
                                                int ldp, const double* Wt, int ldwt, int cw, CMap cmap, int wi,
                                                int nw, int lane) {
  const int gq = lane >> 2, tq = lane & 3;
  const int ntr = (n + 31) >> 5, ntc = (cw + 31) >> 5;
  for (int tile = wi; tile < ntr * ntc; tile += nw) {
    const int r0 = (tile / ntc) * 32, cc0 = (tile % ntc) * 32;
    double acc[4][4][2];
    int pcol[4][2];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cl = cc0 + jj * 8 + tq * 2 + h;
        pcol[jj][h] = (cl < cw) ? cmap(cl) : -1;
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + i * 8 + gq;
      const bool live = r < n && !(r >= k0 && r < k0 + kbc);
      const double* crow = Mi + (long long)(r < n ? r : 0) * ld;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[i][jj][h] = (live && pcol[jj][h] >= 0) ? crow[pcol[jj][h]] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < LA_KB; k += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Pk[(k + tq) * ldp + r0 + i * 8 + gq];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) bf[jj] = Wt[(k + tq) * ldwt + cc0 + jj * 8 + gq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) dmma8x8x4(acc[i][jj][0], acc[i][jj][1], af[i], bf[jj]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + i * 8 + gq;
      if (r >= n) continue;
      double* crow = Mi + (long long)r * ld;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (pcol[jj][h] >= 0) crow[pcol[jj][h]] = acc[i][jj][h];
    }
  }
}

// Stage the pivot rows of cw columns into Wt and apply the displaced-row moves to them (one
// column per thread of the calling group: thread gt of gn).
template <typename CMap>
__device__ __forceinline__ void la_stage_w(double* Mi, long long ld, const LaCtrl& c, int kbc, double* Wt, int ldwt,
                                           int cw, int wcols, CMap cmap, int gt, int gn) {
  const int nm = c.moves[0];
  for (int cc = gt; cc < wcols; cc += gn) {
    if (cc < cw) {
      const int pc = cmap(cc);
#pragma unroll
      for (int j = 0; j < LA_KB; ++j) {
        if (j < kbc) cp_async8(&Wt[j * ldwt + cc], Mi + (long long)c.wsrc[j] * ld + pc, true);
        else Wt[j * ldwt + cc] = 0.0;
      }
      cp_async_commit();
      for (int m0 = 0; m0 < nm; m0 += 8) {
        double mvv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (m0 + u < nm) mvv[u] = Mi[(long long)c.moves[2 + 2 * (m0 + u)] * ld + pc];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (m0 + u < nm) Mi[(long long)c.moves[1 + 2 * (m0 + u)] * ld + pc] = mvv[u];
      }
      cp_async_wait<0>();
    } else {
#pragma unroll
      for (int j = 0; j < LA_KB; ++j) Wt[j * ldwt + cc] = 0.0;
    }
  }
}

__device__ double la_colnorm(const double* Mi, long long ld, int n, double* red) {
  double best = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int r = 0;
#pragma unroll 4
    for (; r + 4 <= n; r += 4) {
      s0 += fabs(Mi[(r + 0) * ld + c]);
      s1 += fabs(Mi[(r + 1) * ld + c]);
      s2 += fabs(Mi[(r + 2) * ld + c]);
      s3 += fabs(Mi[(r + 3) * ld + c]);
    }
    for (; r < n; ++r) s0 += fabs(Mi[r * ld + c]);
    const double s = (s0 + s1) + (s2 + s3);
    best = (s > best || s != s) ? s : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, best, o);
    best = (t > best || t != t) ? t : best;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  double m = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = (red[w] > m || red[w] != red[w]) ? red[w] : m;
  return m;
}

__global__ void __launch_bounds__(LA_THREADS, 1) gj_la_kernel(FusedArgs a) {
  extern __shared__ double sm[];
  const int n = a.n, ncols = a.ncols, ldp = a.ldp, ldw = a.ldw, CW = a.cw;
  // shared-memory carve by plain pointer arithmetic on the shared array: pointers kept in a struct
  // (and indexed by k & 1) end up in local memory, lose their address space and turn every
  // shared access of the pivot loop into a generic LD/ST behind a long scoreboard
  const int pbsz = LA_KB * ldp;
  double* const Pb0 = sm;                       // factored panels, column-major [2][KB][ldp]
  double* const Wu = Pb0 + 2 * (size_t)pbsz;     // U: pivot rows of the current chunk [KB][ldw]
  double* const Wp = Wu + (size_t)LA_KB * ldw;   // P: pivot rows of the look-ahead columns [KB][LA_LDWP]
  double* const slots0 = Wp + (size_t)LA_KB * LA_LDWP;  // [2][LA_PW + 1][KB + 2]
  double* const disp0 = slots0 + 2 * (LA_PW + 1) * (LA_KB + 2);  // [2][KB]
  double* const red = disp0 + 2 * LA_KB;         // [16]
  uint64_t* const bars = reinterpret_cast<uint64_t*>(red + 16);  // full[2], empty[2], la[2]
  LaCtrl* const ctrl0 = reinterpret_cast<LaCtrl*>(bars + 8);     // [2]
  int* const rowid = reinterpret_cast<int*>(ctrl0 + 2);          // [n]
  uint64_t* full = bars;
  uint64_t* empty = bars + 2;
  uint64_t* lab = bars + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int np = (n + LA_KB - 1) / LA_KB;
  const bool isP = tid < LA_PT;

  for (int item = blockIdx.x; item < a.batch; item += gridDim.x) {
    double* Mi = a.M.get(item);
    const long long ld = a.M.ld;
    int* piv = a.piv + (long long)item * n;
    if (tid == 0) {
      // fresh phase counters for every matrix (an mbarrier must be invalidated before it is
      // initialised again)
      for (int b = 0; b < 6; ++b) {
        if (item != (int)blockIdx.x)
          asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars + b)) : "memory");
        la_bar_init(bars + b, 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

#ifdef LA_DEBUG
    long long la_last = clock64();
#endif
    if (isP) {
      // ------------------------------------------------------------------ panel group
      const int i = tid;  // matrix row of this thread
      int flag = 0;
      double row[LA_KB];
#pragma unroll
      for (int t = 0; t < LA_KB; ++t) row[t] = (i < n && t < n) ? Mi[(long long)i * ld + t] : 0.0;
      for (int k = 0; k < np; ++k) {
        const int k0 = k * LA_KB, kbc = min(LA_KB, n - k0);
        LaCtrl& C = *(ctrl0 + (k & 1));
        for (int x = k0 + tid; x < n; x += LA_PT) rowid[x] = x;
        // (the first barrier of the column loop orders the rowid reset before thread 0's swaps)
#pragma unroll 1
        for (int jb = 0; jb < LA_KB; jb += 4) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = jb + q;
            if (j < kbc) {
              const int cj = k0 + j;
              double* slots = slots0 + (j & 1) * (LA_PW + 1) * (LA_KB + 2);
              double* disp = disp0 + (j & 1) * LA_KB;
              // arg-max on the bit pattern of |value| (non-negative doubles order like unsigned
              // integers; NaN and zero map to key 0 = "no candidate"): integer compares keep the
              // FP64 pipe, whose dependent latency dominated this loop, out of the reduction
              unsigned long long key = 0ull;
              int bi = n;
              if (i < n && i >= cj) {
                const double av = fabs(row[q]);
                key = (av == av) ? (unsigned long long)__double_as_longlong(av) : 0ull;
                if (key) bi = i;
              }
              // reciprocal of the own candidate, in flight while the reduction runs
              const double rinv = 1.0 / row[q];
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ok > key || (ok == key && oi < bi)) { key = ok; bi = oi; }
              }
              double* my = slots + warp * (LA_KB + 2);
              if (lane == 0) {
                my[0] = __longlong_as_double((long long)key);
                my[1] = (double)bi;
                // no candidate in this warp: poison the pivot entry (used only when no warp has one)
                if (bi >= n) my[2 + q] = __longlong_as_double(0x7ff8000000000000LL);
              }
              // warp-uniform branches: the loop is bound by instructions issued per warp, and only
              // two threads of the group have a row to publish
              if (__any_sync(0xffffffffu, i == bi)) {
                if (i == bi) {
                  // the candidate row already scaled by 1 / pivot (entry q: the reciprocal itself)
#pragma unroll
                  for (int t = 0; t < LA_KB; ++t) my[2 + t] = (t == q) ? rinv : row[t] * rinv;
                }
              }
              if (cj >> 5 == warp) {
                if (i == cj) {
#pragma unroll
                  for (int t = 0; t < LA_KB; ++t) disp[t] = row[t];
                }
              }
              bar_p();
              unsigned long long kb = 0ull;
              int pr = n, ws = lane;
              if (lane < LA_PW) {
                kb = (unsigned long long)__double_as_longlong(slots[lane * (LA_KB + 2)]);
                pr = (int)slots[lane * (LA_KB + 2) + 1];
              }
#pragma unroll
              for (int o = 4; o > 0; o >>= 1) {
                const unsigned long long ok = __shfl_xor_sync(0xffffffffu, kb, o);
                const int oi = __shfl_xor_sync(0xffffffffu, pr, o);
                const int ow = __shfl_xor_sync(0xffffffffu, ws, o);
                if (ok > kb || (ok == kb && oi < pr)) { kb = ok; pr = oi; ws = ow; }
              }
              kb = __shfl_sync(0xffffffffu, kb, 0);
              pr = __shfl_sync(0xffffffffu, pr, 0);
              ws = __shfl_sync(0xffffffffu, ws, 0);
              const double* pvs = slots + ws * (LA_KB + 2) + 2;  // scaled pivot row
              if (pr >= n) pr = cj;  // no positive candidate anywhere: keep the diagonal (flagged)
              if (tid == 0) {
                if (kb == 0ull) flag = 1;
                C.spiv[j] = pr;
                piv[cj] = pr;
                const int tr = rowid[cj];
                rowid[cj] = rowid[pr];
                rowid[pr] = tr;
              }
              if (pr != cj && (pr >> 5) == warp) {
                if (i == pr) {
#pragma unroll
                  for (int t = 0; t < LA_KB; ++t) row[t] = disp[t];
                }
              }
              if (i == cj) {
#pragma unroll
                for (int t = 0; t < LA_KB; ++t) row[t] = pvs[t];
              } else {
                const double f = row[q];
#pragma unroll
                for (int t = 0; t < LA_KB; ++t) row[t] = ((t == q) ? 0.0 : row[t]) - f * pvs[t];
              }
            }
          }
          // rotate by 4: the next group of columns to the front
          double t0[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) t0[u] = row[u];
#pragma unroll
          for (int t = 0; t < LA_KB - 4; ++t) row[t] = row[t + 4];
#pragma unroll
          for (int u = 0; u < 4; ++u) row[LA_KB - 4 + u] = t0[u];
        }
        LA_T(0);  // column loop
        // publish panel k: its buffer must be free (U finished pass k - 2)
        if (k >= 2) {
          // one thread polls, the group waits at its (free) named barrier: polling warps would
          // take issue slots from the working group
          if (tid == 0) la_wait(empty + (k & 1), ((k >> 1) - 1) & 1 LA_DBG(1, k));
          bar_p();
        }
        LA_T(1);  // wait empty
        double* Pk = Pb0 + (size_t)(k & 1) * pbsz;
        if (i < n) {
          double* dst = Mi + (long long)i * ld + k0;
#pragma unroll
          for (int t = 0; t < LA_KB; ++t) {
            if (t < kbc) dst[t] = row[t];
            Pk[t * ldp + i] = (t < kbc) ? row[t] : 0.0;
          }
        } else if (i < ldp) {
#pragma unroll
          for (int t = 0; t < LA_KB; ++t) Pk[t * ldp + i] = 0.0;
        }
        bar_p();  // spiv / rowid complete, panel in shared memory
        if (warp == 0) {
          const int x = lane < kbc ? C.spiv[lane] : -1;
          if (lane < kbc) C.wsrc[lane] = rowid[k0 + lane];
          const bool mv = x >= k0 + kbc && rowid[x] != x;
          const unsigned bal = __ballot_sync(0xffffffffu, mv);
          if (mv) {
            const int slot = __popc(bal & ((1u << lane) - 1u));
            C.moves[1 + 2 * slot] = x;
            C.moves[2 + 2 * slot] = rowid[x];
          }
          if (lane == 0) C.moves[0] = __popc(bal);
        }
        __threadfence_block();
        bar_p();
        if (tid == 0) la_arrive(full + (k & 1));
        LA_T(2);  // publish
        if (k + 1 < np) {
          // look-ahead: panel k applied to the columns of panel k + 1 (ready once U has applied
          // panel k - 1 to them), then those columns into registers
          const int k1 = k0 + kbc, kb1 = min(LA_KB, n - k1);
          if (k >= 1) {
            if (tid == 0) la_wait(lab + ((k + 1) & 1), (((k + 1) >> 1) - 1) & 1 LA_DBG(2, k));
            bar_p();
          }
          LA_T(3);  // wait look-ahead columns
          auto cmap = [k1](int cl) { return k1 + cl; };
          la_stage_w(Mi, ld, C, kbc, Wp, LA_LDWP, kb1, 32, cmap, tid, LA_PT);
          bar_p();
          LA_T(4);  // stage W (look-ahead)
          la_update_tiles(Mi, ld, n, k0, kbc, Pk, ldp, Wp, LA_LDWP, kb1, cmap, warp, LA_PW, lane);
          __threadfence_block();
          bar_p();
#pragma unroll
          LA_T(5);  // look-ahead tiles
          for (int t = 0; t < LA_KB; ++t) row[t] = (i < n && t < kb1) ? Mi[(long long)i * ld + k1 + t] : 0.0;
          LA_T(6);  // load next panel
        }
      }
      if (tid == 0 && flag && a.status) a.status[item] |= 1;
    } else {
      // ------------------------------------------------------------------ update group
      const int ut = tid - LA_PT, uw = warp - LA_PW;
      for (int k = 0; k < np; ++k) {
        const int k0 = k * LA_KB, kbc = min(LA_KB, n - k0);
        if (ut == 0) la_wait(full + (k & 1), (k >> 1) & 1 LA_DBG(3, k));
        bar_u();
        LA_T(8);  // U: wait full
        const LaCtrl& C = *(ctrl0 + (k & 1));
        const double* Pk = Pb0 + (size_t)(k & 1) * pbsz;
        const int k1 = k0 + kbc, kb1 = (k + 1 < np) ? min(LA_KB, n - k1) : 0;
        const int k2 = k1 + kb1, kb2 = (k + 2 < np) ? min(LA_KB, n - k2) : 0;
        if (kb2 > 0) {
          // the columns of panel k + 2 first: P applies panel k + 1 to them next
          auto cmap = [k2](int cl) { return k2 + cl; };
          la_stage_w(Mi, ld, C, kbc, Wu, ldw, kb2, 32, cmap, ut, LA_UT);
          bar_u();
          la_update_tiles(Mi, ld, n, k0, kbc, Pk, ldp, Wu, ldw, kb2, cmap, uw, LA_UW, lane);
          __threadfence_block();
          bar_u();
          if (ut == 0) la_arrive(lab + ((k + 2) & 1));
          LA_T(9);  // U: look-ahead chunk
        }
        // every other column: all but the contiguous range of panels k, k + 1, k + 2
        const int skipw = kbc + kb1 + kb2;
        const int nlog = ncols - skipw;
        for (int c0 = 0; c0 < nlog; c0 += CW) {
          const int cw = min(CW, nlog - c0);
          auto cmap = [c0, k0, skipw](int cl) {
            const int pc = c0 + cl;
            return pc >= k0 ? pc + skipw : pc;
          };
          la_stage_w(Mi, ld, C, kbc, Wu, ldw, cw, ldw, cmap, ut, LA_UT);
          bar_u();
          LA_T(10);  // U: stage W
#ifndef LA_SKIP_U  // (timing experiment: panel group alone; results are wrong)
          la_update_tiles(Mi, ld, n, k0, kbc, Pk, ldp, Wu, ldw, cw, cmap, uw, LA_UW, lane);
#endif
          bar_u();
          LA_T(11);  // U: tiles
        }
        __threadfence_block();
        bar_u();
        if (ut == 0) la_arrive(empty + (k & 1));
      }
    }
    __threadfence_block();
    __syncthreads();

    if (a.full) {
      // undo the column interchanges of the inverse: inv[:, perm[j]] = M[:, j]
      int* perm = rowid;
      for (int j = tid; j < n; j += LA_THREADS) perm[j] = j;
      __syncthreads();
      if (tid == 0) {
        for (int j = 0; j < n; ++j) {
          const int r = piv[j];
          const int t = perm[j];
          perm[j] = perm[r];
          perm[r] = t;
        }
      }
      __syncthreads();
      if (a.perm_out) {
        int* po = a.perm_out + (long long)item * n;
        for (int j = tid; j < n; j += LA_THREADS) po[j] = perm[j];
      } else {
        double* buf = Pb0 + (size_t)warp * n;  // 16 warps x n doubles <= 2 panel buffers
        for (int r = warp; r < n; r += LA_THREADS / 32) {
          double* rowp = Mi + (long long)r * ld;
          for (int c = lane; c < n; c += 32) buf[c] = rowp[c];
          __syncwarp();
          for (int c = lane; c < n; c += 32) rowp[perm[c]] = buf[c];
          __syncwarp();
        }
      }
      __syncthreads();
      if (a.ainvnorm) {
        const double v = la_colnorm(Mi, ld, n, red);
        if (tid == 0) a.ainvnorm[item] = v;
      }
    }
    __syncthreads();
  }
}

int la_round_ldp(int n) { return ((n + 15) & ~15) + 4; }

}  // namespace

// Look-ahead kernel applicable: full inversions of blocks with 3..8 panels of 28 columns whose
// rows fit one thread each in the 7 panel warps. HPS_GJ_LA=0 keeps gj_fused_kernel.
bool gj_la_ok(int n, int ncols) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HPS_GJ_LA");
    on = e ? atoi(e) : 0;
  }
  return on && n > 2 * LA_KB && n <= LA_PT && ncols >= n && ncols <= 1024;
}

int launch_gj_la(const FusedArgs& a0, cudaStream_t s) {
  FusedArgs a = a0;
  if (!a.full || a.k_begin != 0 || a.k_end != a.n || a.col_lo != 0 || a.col_hi != a.ncols) return 1;
  a.ldp = la_round_ldp(a.n);
  if (a.ldp < LA_PT) a.ldp = ((LA_PT + 15) & ~15) + 4;  // DMMA row tiles read up to row 32 * 7 - 1
  int cw = a.ncols - LA_KB;
  if (cw > 256) cw = 256;
  if (cw < 32) cw = 32;
  size_t smem = 0;
  for (;;) {
    a.ldw = ((cw + 15) & ~15) + 4;
    smem = la_smem_bytes(a.n, a.ldp, a.ldw);
    if (smem <= 200 * 1024 || cw <= 32) break;
    cw -= 32;
  }
  a.cw = cw;
  if (smem > 227 * 1024) return 1;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gj_la_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.batch < sms ? a.batch : sms;
  gj_la_kernel<<<grid, LA_THREADS, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps

#ifdef LA_DEBUG
extern "C" void hps_la_debug_buffer(int* mapped) { cudaMemcpyToSymbol(hps::la_dbg, &mapped, sizeof(mapped)); }
extern "C" void hps_la_prof(long long* h) { cudaMemcpyFromSymbol(h, hps::la_prof, 16 * sizeof(long long)); }
#endif

