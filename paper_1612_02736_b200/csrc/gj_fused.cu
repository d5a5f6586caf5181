// Fused, persistent Gauss-Jordan kernel: one CTA owns one matrix at a time and runs every
// panel of a pivot-column range back to back, so a whole batch of small inverses (leaf
// interior blocks at p=16: 196 x 256 augmented; low tree levels) costs one launch and the
// matrix stays hot in L2 between panels.
//
// Per panel of KB columns:
//   1. each thread holds its RPT rows of the panel in registers (row i = tid + r*256);
//      per column: warp-shuffle argmax + one cross-warp exchange (2 __syncthreads), the
//      pivot row and the displaced row swap through shared memory, elimination in registers;
//   2. the factored panel goes to shared memory (column-major, stride ldp = 4 mod 16, so the
//      DMMA A-fragment loads are bank-conflict free) and back to global;
//   3. the KB row interchanges are composed once (rowid) so every other column needs only
//      independent loads: W[j] = M[rowid[k0+j]] and the few displaced rows outside the panel;
//   4. DMMA (mma.sync.m8n8k4.f64) trailing update of the other columns, in chunks of CW
//      columns: rows in the panel get panel_J W, the rest += panel_R W.
// Modes: full (k = 0..n over all columns, plus |A|_1, |A^-1|_1 and the final column
// un-permutation) or sub-range (pivot columns [k_begin,k_end) updating [col_lo,col_hi)
// only) — the inner level of the two-level blocking used for large n (gj.cu).
#include <cstdlib>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

constexpr int FU_THREADS = 256;

#ifdef FU_PROFILE
__device__ long long fu_prof[8];
#define FU_T(i)                                  \
  if (threadIdx.x == 0 && blockIdx.x == 0) {     \
    const long long now = clock64();             \
    fu_prof[i] += now - fu_last;                 \
    fu_last = now;                               \
  }
#else
#define FU_T(i)
#endif

__device__ __forceinline__ double block_max_nan(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, v, o);
    v = (t > v || t != t) ? t : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = (red[w] > m || red[w] != red[w]) ? red[w] : m;
  return m;
}

__device__ double colnorm_block(const double* Mi, long long ld, int n, double* red) {
  double best = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int r = 0;
    // 16 independent loads in flight per thread (the column sum is latency-bound otherwise)
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
  return block_max_nan(best, red);
}

struct FusedSmem {
  double* P;
  double* W;
  double* slots;  // [2][warps][KB+2]: candidate value, row index, row values
  double* bufB;   // [2][KB]: displaced row
  double* red_v;
  int* red_i;
  int* spiv;
  int* wsrc;
  int* moves;  // [0] = count, then (dst, src) pairs
  int* rowid;
};

template <int KB>
__device__ __forceinline__ FusedSmem carve(double* sm, int n, int ldp, int ldw) {
  constexpr int KB4 = (KB + 3) & ~3;
  FusedSmem s;
  s.P = sm;
  s.W = s.P + (size_t)KB4 * ldp;
  s.slots = s.W + (size_t)KB4 * ldw;
  s.bufB = s.slots + 2 * 16 * (KB + 2);
  s.red_v = s.bufB + 2 * KB4;
  s.red_i = reinterpret_cast<int*>(s.red_v + 16);
  s.spiv = s.red_i + 24;
  s.wsrc = s.spiv + KB4;
  s.moves = s.wsrc + KB4;
  s.rowid = s.moves + 2 * KB4 + 4;
  return s;
}

template <int KB, int RPT, int NTH = 256>
__global__ void __launch_bounds__(NTH, (RPT >= 8 || NTH > 256 ? 1 : 2)) gj_fused_kernel(FusedArgs a) {
  constexpr int FU_THREADS = NTH;
  constexpr int KB4 = (KB + 3) & ~3;
  extern __shared__ double sm[];
  const int n = a.n, ldp = a.ldp, ldw = a.ldw, CW = a.cw;
  FusedSmem S = carve<KB>(sm, n, ldp, ldw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;

#ifdef FU_PROFILE
  long long fu_last = clock64();
#endif
  for (int item = blockIdx.x; item < a.batch; item += gridDim.x) {
    double* Mi = a.M.get(item);
    const long long ld = a.M.ld;
    int* piv = a.piv + (long long)item * n;
    int flag = 0;
    if (a.full && a.anorm) {
      const double v = colnorm_block(Mi, ld, n, S.red_v);
      if (tid == 0) a.anorm[item] = v;
    }
    for (int k0 = a.k_begin; k0 < a.k_end; k0 += KB) {
      const int kbc = min(KB, a.k_end - k0);
      __syncthreads();  // previous panel's smem (P, W, rowid) fully consumed

      // ---- 1. panel rows -> registers
      double row[RPT][KB];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = tid + r * FU_THREADS;
        const double* src = Mi + (long long)(i < n ? i : 0) * ld + k0;
#pragma unroll
        for (int t = 0; t < KB; ++t) row[r][t] = (i < n && t < kbc) ? src[t] : 0.0;
      }
      FU_T(0);
      // composed interchanges of this panel, built by thread 0 as the pivots are chosen
      for (int x = k0 + tid; x < n; x += FU_THREADS) S.rowid[x] = x;
      // Column loop with the panel row rotated in registers by 4 columns at a time: the 4
      // columns of a group use static register indices (row[.][q]), one 4-way rotation per
      // group brings the next group to the front (KB/4 rotations restore the column order).
      // One barrier per column: every warp publishes its best candidate row (double-buffered
      // slots), every warp then picks the global winner (LAPACK rule: largest |value|, ties
      // -> smallest row) with a shuffle reduction over the warp slots.
      static_assert(KB % 4 == 0, "panel width must be a multiple of 4");
#pragma unroll 1
      for (int jb = 0; jb < KB; jb += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = jb + q;
          if (j < kbc) {
            const int cj = k0 + j;
            double* slots = S.slots + (j & 1) * (FU_THREADS / 32) * (KB + 2);
            double* disp = S.bufB + (j & 1) * KB;
            double best = -1.0;
            int bi = n;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
              const int i = tid + r * FU_THREADS;
              if (i < n && i >= cj) {
                const double v = fabs(row[r][q]);
                if (v > best) { best = v; bi = i; }
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const double ov = __shfl_xor_sync(0xffffffffu, best, o);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
              if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
            }
            double* my = slots + warp * (KB + 2);
            if (lane == 0) {
              my[0] = best;
              my[1] = (double)bi;
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
              const int i = tid + r * FU_THREADS;
              if (i == bi) {
#pragma unroll
                for (int t = 0; t < KB; ++t) my[2 + t] = row[r][t];
              }
              if (i == cj) {
#pragma unroll
                for (int t = 0; t < KB; ++t) disp[t] = row[r][t];
              }
            }
            __syncthreads();
            // winner over the warp candidates: lane w reads warp w's slot, shuffle reduction
            constexpr int NWARP = FU_THREADS / 32;
            double b = -2.0;
            int pr = n, ws = lane;
            if (lane < NWARP) {
              b = slots[lane * (KB + 2)];
              pr = (int)slots[lane * (KB + 2) + 1];
            }
#pragma unroll
            for (int o = NWARP / 2; o > 0; o >>= 1) {
              const double ov = __shfl_xor_sync(0xffffffffu, b, o);
              const int oi = __shfl_xor_sync(0xffffffffu, pr, o);
              const int ow = __shfl_xor_sync(0xffffffffu, ws, o);
              if (ov > b || (ov == b && oi < pr)) { b = ov; pr = oi; ws = ow; }
            }
            b = __shfl_sync(0xffffffffu, b, 0);
            pr = __shfl_sync(0xffffffffu, pr, 0);
            ws = __shfl_sync(0xffffffffu, ws, 0);
            const double* pvr = slots + ws * (KB + 2) + 2;
            if (pr >= n) {  // all candidates NaN: keep the diagonal, NaN propagates
              pr = cj;
              pvr = disp;
            }
            if (tid == 0) {
              if (!(b > 0.0)) flag = 1;
              S.spiv[j] = pr;
              piv[cj] = pr;
              const int tr = S.rowid[cj];
              S.rowid[cj] = S.rowid[pr];
              S.rowid[pr] = tr;
            }
            const double inv = 1.0 / pvr[q];
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
              const int i = tid + r * FU_THREADS;
              if (i == pr && pr != cj) {
#pragma unroll
                for (int t = 0; t < KB; ++t) row[r][t] = disp[t];
              }
              if (i == cj) {
#pragma unroll
                for (int t = 0; t < KB; ++t) row[r][t] = (t == q) ? inv : pvr[t] * inv;
              } else {
                const double f = row[r][q];
#pragma unroll
                for (int t = 0; t < KB; ++t)
                  row[r][t] = ((t == q) ? 0.0 : row[r][t]) - f * ((t == q) ? inv : pvr[t] * inv);
              }
            }
          }
        }
        // rotate by 4: the next group of columns to the front
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          double t0[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) t0[u] = row[r][u];
#pragma unroll
          for (int t = 0; t < KB - 4; ++t) row[r][t] = row[r][t + 4];
#pragma unroll
          for (int u = 0; u < 4; ++u) row[r][KB - 4 + u] = t0[u];
        }
      }
      FU_T(1);
      // ---- 2. factored panel -> shared (column-major) and global; composed interchanges
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = tid + r * FU_THREADS;
        if (i < n) {
          double* dst = Mi + (long long)i * ld + k0;
#pragma unroll
          for (int t = 0; t < KB; ++t) {
            if (t < kbc) dst[t] = row[r][t];
            S.P[t * ldp + i] = (t < kbc) ? row[r][t] : 0.0;
          }
        }
      }
      for (int e = tid; e < (KB4 - KB) * ldp; e += FU_THREADS) S.P[KB * ldp + e] = 0.0;
      __syncthreads();
      if (warp == 0) {
        // W sources and the displaced rows outside the panel (lane j: pivot step j)
        const int x = lane < kbc ? S.spiv[lane] : -1;
        if (lane < kbc) S.wsrc[lane] = S.rowid[k0 + lane];
        const bool mv = x >= k0 + kbc && S.rowid[x] != x;
        const unsigned bal = __ballot_sync(0xffffffffu, mv);
        if (mv) {
          const int slot = __popc(bal & ((1u << lane) - 1u));
          S.moves[1 + 2 * slot] = x;
          S.moves[2 + 2 * slot] = S.rowid[x];
        }
        if (lane == 0) S.moves[0] = __popc(bal);
      }
      __syncthreads();

      FU_T(2);
      // ---- 3./4. other columns of [col_lo, col_hi), chunks of CW
      const int nlog = (a.col_hi - a.col_lo) - kbc;
      const int nm = S.moves[0];
      for (int c0 = 0; c0 < nlog; c0 += CW) {
        const int cw = min(CW, nlog - c0);
        if (c0 > 0) __syncthreads();
        for (int cc = tid; cc < ldw; cc += FU_THREADS) {
          if (cc < cw) {
            int pc = a.col_lo + c0 + cc;
            if (pc >= k0) pc += kbc;
            // W rows via cp.async (no registers, all in flight), then the displaced rows in
            // groups of 8 loads before their stores. Safe in any grouping: a displaced row
            // outside the panel always receives an original panel row (a row outside the panel
            // only ever swaps with the current pivot position), so no source is a destination.
#pragma unroll
            for (int j = 0; j < KB4; ++j) {
              if (j < kbc) cp_async8(&S.W[j * ldw + cc], Mi + (long long)S.wsrc[j] * ld + pc, true);
              else S.W[j * ldw + cc] = 0.0;
            }
            cp_async_commit();
            for (int m0 = 0; m0 < nm; m0 += 8) {
              double mvv[8];
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (m0 + u < nm) mvv[u] = Mi[(long long)S.moves[2 + 2 * (m0 + u)] * ld + pc];
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (m0 + u < nm) Mi[(long long)S.moves[1 + 2 * (m0 + u)] * ld + pc] = mvv[u];
            }
            cp_async_wait<0>();
          } else {
#pragma unroll
            for (int j = 0; j < KB4; ++j) S.W[j * ldw + cc] = 0.0;
          }
        }
        __syncthreads();
        FU_T(3);
        const int ntr = (n + 31) >> 5, ntc = (cw + 31) >> 5;
        for (int tile = warp; tile < ntr * ntc; tile += FU_THREADS / 32) {
          const int r0 = (tile / ntc) * 32, cc0 = (tile % ntc) * 32;
          double acc[4][4][2];
          int pcol[4][2];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cl = cc0 + jj * 8 + tq * 2 + h;
              int pc = a.col_lo + c0 + cl;
              if (pc >= k0) pc += kbc;
              pcol[jj][h] = (cl < cw) ? pc : -1;
            }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = r0 + i * 8 + gq;
            const bool live = r < n && !(r >= k0 && r < k0 + kbc);
            const double* crow = Mi + (long long)(r < n ? r : 0) * ld;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                acc[i][jj][h] = (live && pcol[jj][h] >= 0) ? crow[pcol[jj][h]] : 0.0;
          }
#pragma unroll
          for (int k = 0; k < KB4; k += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = S.P[(k + tq) * ldp + r0 + i * 8 + gq];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) bf[jj] = S.W[(k + tq) * ldw + cc0 + jj * 8 + gq];
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
        FU_T(4);
      }
    }
    __syncthreads();
    if (tid == 0 && flag && a.status) a.status[item] |= 1;
    FU_T(5);

    if (a.full) {
      // undo the column interchanges of the inverse: inv[:, perm[j]] = M[:, j]
      int* perm = S.rowid;
      for (int j = tid; j < n; j += FU_THREADS) perm[j] = j;
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
        // leave the columns permuted; consumers gather their right-hand side with perm
        int* po = a.perm_out + (long long)item * n;
        for (int j = tid; j < n; j += FU_THREADS) po[j] = perm[j];
      } else {
        double* buf = S.P + (size_t)warp * n;
        for (int r = warp; r < n; r += FU_THREADS / 32) {
          double* rowp = Mi + (long long)r * ld;
#pragma unroll 8
          for (int c = lane; c < n; c += 32) buf[c] = rowp[c];
          __syncwarp();
#pragma unroll 8
          for (int c = lane; c < n; c += 32) rowp[perm[c]] = buf[c];
          __syncwarp();
        }
      }
      __syncthreads();
      if (a.ainvnorm) {
        const double v = colnorm_block(Mi, ld, n, S.red_v);
        if (tid == 0) a.ainvnorm[item] = v;
      }
    }
  }
}

static int round_ldp(int n) { return ((n + 15) & ~15) + 4; }

template <int KB>
static size_t fused_smem_bytes(int n, int ldw) {
  constexpr int KB4 = (KB + 3) & ~3;
  return sizeof(double) * ((size_t)KB4 * round_ldp(n) + (size_t)KB4 * ldw + 2 * 16 * (KB + 2) + 2 * KB4 + 16) +
         sizeof(int) * (24 + 2 * KB4 + 2 * KB4 + 4 + (size_t)n + 4);
}

template <int KB, int RPT, int NTH = 256>
static int launch_variant(FusedArgs a, int grid, cudaStream_t s) {
  a.ldp = round_ldp(a.n);
  // chunk width: all other columns at once when they fit the budget, else 128
  const int others = (a.col_hi - a.col_lo) - 1;
  int cw = others < 256 ? others : 256;
  size_t smem = 0;
  for (;;) {
    const int ldw = ((cw + 15) & ~15) + 4;
    smem = fused_smem_bytes<KB>(a.n, ldw);
    if (smem <= 110 * 1024 || cw <= 32) {
      a.cw = cw;
      a.ldw = ldw;
      break;
    }
    cw -= 32;
  }
  if (smem > 227 * 1024) return 1;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(gj_fused_kernel<KB, RPT, NTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gj_fused_kernel<KB, RPT, NTH><<<grid, NTH, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int gj_fused_panel_width(int n, int full) {
  if (full && n <= 256) return 28;
  if (n <= 512) return 16;
  if (n <= 1024) {
    const char* e = getenv("HPS_GJ_INNER");
    return (e && atoi(e) == 0) ? 8 : 16;
  }
  return 8;
}

int launch_gj_fused(const FusedArgs& a, int grid, cudaStream_t s) {
  const int kb = gj_fused_panel_width(a.n, a.full);
  if (a.n <= 256 && kb == 28) return launch_variant<28, 1>(a, grid, s);
  if (a.n <= 512) return launch_variant<16, 2>(a, grid, s);
  if (a.n <= 1024) {
    static int v = -1;
    if (v < 0) {
      const char* e = getenv("HPS_GJ_INNER");
      v = e ? atoi(e) : 1;
    }
    if (v == 0) return launch_variant<8, 4>(a, grid, s);
    return launch_variant<16, 2, 512>(a, grid, s);
  }
  if (a.n <= 2048) return launch_variant<8, 4, 512>(a, grid, s);
  return 1;
}

}  // namespace hps

#ifdef FU_PROFILE
extern "C" void hps_fu_prof(long long* h, int reset) {
  cudaMemcpyFromSymbol(h, hps::fu_prof, 8 * sizeof(long long));
  if (reset) {
    long long z[8] = {};
    cudaMemcpyToSymbol(hps::fu_prof, z, sizeof(z));
  }
}
#endif
