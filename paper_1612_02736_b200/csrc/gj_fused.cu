// Fused, persistent Gauss-Jordan kernel: one CTA owns one matrix at a time and runs every
// panel of a pivot-column range back to back (panel factorisation in shared memory, row
// interchanges, pivot-row snapshot, DMMA trailing update), so a whole batch of small
// inverses (leaf interior blocks at p=16: 196 x 256 augmented; low-level merges) costs one
// launch and the matrix stays hot in L2 between panels.
//
// Layout in shared memory (column-major panel so both the row-per-thread elimination and
// the DMMA A-fragment loads are bank-conflict free; stride ldp = 4 mod 16 doubles):
//   P[j*ldp + i]  panel column j, row i       (kb4 x ldp)
//   W[j*LDW + c]  pivot row j, chunk column c (kb4 x LDW), LDW = 132 (= 4 mod 16)
//
// Modes: full (k = 0..n over all columns, plus |A|_1, |A^-1|_1 and the final column
// un-permutation) or sub-range (pivot columns [k_begin,k_end) updating columns
// [col_lo,col_hi) only) — the inner level of the two-level blocking used for large n.
#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

constexpr int FU_THREADS = 256;
constexpr int FU_CW = 128;
constexpr int FU_LDW = FU_CW + 4;

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
  for (int w = 1; w < FU_THREADS / 32; ++w) m = (red[w] > m || red[w] != red[w]) ? red[w] : m;
  return m;
}

__device__ double colnorm_block(const double* Mi, long long ld, int n, double* red) {
  double best = 0.0;
  for (int c = threadIdx.x; c < n; c += FU_THREADS) {
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += fabs(Mi[r * ld + c]);
    best = (s > best || s != s) ? s : best;
  }
  return block_max_nan(best, red);
}

__global__ void __launch_bounds__(FU_THREADS, 2) gj_fused_kernel(FusedArgs a) {
  extern __shared__ double sm[];
  const int n = a.n, ldp = a.ldp, kbmax4 = (a.kb + 3) & ~3;
  double* P = sm;
  double* W = P + (size_t)kbmax4 * ldp;
  double* prow = W + (size_t)kbmax4 * FU_LDW;
  double* red_v = prow + 32;
  int* red_i = reinterpret_cast<int*>(red_v + 8);
  int* spiv = red_i + 16;
  int* perm = spiv + 32;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;

  for (int item = blockIdx.x; item < a.batch; item += gridDim.x) {
    double* Mi = a.M.get(item);
    const long long ld = a.M.ld;
    int* piv = a.piv + (long long)item * n;
    int flag = 0;
    if (a.full && a.anorm) {
      const double v = colnorm_block(Mi, ld, n, red_v);
      if (tid == 0) a.anorm[item] = v;
    }
    for (int k0 = a.k_begin; k0 < a.k_end; k0 += a.kb) {
      const int kb = min(a.kb, a.k_end - k0);
      const int kb4 = (kb + 3) & ~3;
      __syncthreads();
      for (int e = tid; e < n * kb; e += FU_THREADS) {
        const int i = e / kb, j = e - i * kb;
        P[j * ldp + i] = Mi[i * ld + k0 + j];
      }
      for (int e = tid; e < (kb4 - kb) * ldp; e += FU_THREADS) P[kb * ldp + e] = 0.0;
      __syncthreads();

      // ---- panel factorisation (pivot rows searched from k0+j, ties -> smallest index)
      for (int j = 0; j < kb; ++j) {
        const int cj = k0 + j;
        double best = -1.0;
        int bi = n;
        for (int i = cj + tid; i < n; i += FU_THREADS) {
          const double v = fabs(P[j * ldp + i]);
          if (v > best) { best = v; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if (lane == 0) { red_v[warp] = best; red_i[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
          double b = red_v[0];
          int bix = red_i[0];
          for (int w = 1; w < FU_THREADS / 32; ++w)
            if (red_v[w] > b || (red_v[w] == b && red_i[w] < bix)) { b = red_v[w]; bix = red_i[w]; }
          if (bix >= n) bix = cj;
          if (!(b > 0.0)) flag = 1;
          red_i[8] = bix;
          spiv[j] = bix;
          piv[cj] = bix;
        }
        __syncthreads();
        const int pr = red_i[8];
        if (pr != cj && tid < kb) {
          const double t = P[tid * ldp + pr];
          P[tid * ldp + pr] = P[tid * ldp + cj];
          P[tid * ldp + cj] = t;
        }
        __syncthreads();
        if (tid < kb) {
          const double inv = 1.0 / P[j * ldp + cj];
          prow[tid] = (tid == j) ? inv : P[tid * ldp + cj] * inv;
        }
        __syncthreads();
        for (int i = tid; i < n; i += FU_THREADS) {
          if (i == cj) {
            for (int t = 0; t < kb; ++t) P[t * ldp + i] = prow[t];
          } else {
            const double f = P[j * ldp + i];
            P[j * ldp + i] = 0.0;
            for (int t = 0; t < kb; ++t) P[t * ldp + i] -= f * prow[t];
          }
        }
        __syncthreads();
      }
      for (int e = tid; e < n * kb; e += FU_THREADS) {
        const int i = e / kb, j = e - i * kb;
        Mi[i * ld + k0 + j] = P[j * ldp + i];
      }

      // ---- trailing update of the other columns of [col_lo, col_hi), in chunks of FU_CW
      const int nlog = (a.col_hi - a.col_lo) - kb;
      for (int c0 = 0; c0 < nlog; c0 += FU_CW) {
        const int cw = min(FU_CW, nlog - c0);
        __syncthreads();
        for (int cc = tid; cc < FU_CW; cc += FU_THREADS) {
          if (cc < cw) {
            int pc = a.col_lo + c0 + cc;
            if (pc >= k0) pc += kb;
            for (int j = 0; j < kb; ++j) {
              const int r = spiv[j];
              if (r != k0 + j) {
                const double t = Mi[r * ld + pc];
                Mi[r * ld + pc] = Mi[(k0 + j) * ld + pc];
                Mi[(k0 + j) * ld + pc] = t;
              }
            }
            for (int j = 0; j < kb; ++j) W[j * FU_LDW + cc] = Mi[(k0 + j) * ld + pc];
            for (int j = kb; j < kb4; ++j) W[j * FU_LDW + cc] = 0.0;
          } else {
            for (int j = 0; j < kb4; ++j) W[j * FU_LDW + cc] = 0.0;
          }
        }
        __syncthreads();
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
              if (pc >= k0) pc += kb;
              pcol[jj][h] = (cl < cw) ? pc : -1;
            }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = r0 + i * 8 + gq;
            const bool live = r < n && !(r >= k0 && r < k0 + kb);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                acc[i][jj][h] = (live && pcol[jj][h] >= 0) ? Mi[r * ld + pcol[jj][h]] : 0.0;
          }
          for (int k = 0; k < kb4; k += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = P[(k + tq) * ldp + r0 + i * 8 + gq];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) bf[jj] = W[(k + tq) * FU_LDW + cc0 + jj * 8 + gq];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) dmma8x8x4(acc[i][jj][0], acc[i][jj][1], af[i], bf[jj]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = r0 + i * 8 + gq;
            if (r >= n) continue;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                if (pcol[jj][h] >= 0) Mi[r * ld + pcol[jj][h]] = acc[i][jj][h];
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0 && flag && a.status) a.status[item] |= 1;

    if (a.full) {
      // undo the column interchanges of the inverse: inv[:, perm[j]] = M[:, j]
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
      double* buf = P + (size_t)warp * n;
      for (int r = warp; r < n; r += FU_THREADS / 32) {
        double* row = Mi + r * ld;
        for (int c = lane; c < n; c += 32) buf[c] = row[c];
        __syncwarp();
        for (int c = lane; c < n; c += 32) row[perm[c]] = buf[c];
        __syncwarp();
      }
      __syncthreads();
      if (a.ainvnorm) {
        const double v = colnorm_block(Mi, ld, n, red_v);
        if (tid == 0) a.ainvnorm[item] = v;
      }
    }
  }
}

size_t gj_fused_smem(int n, int kb) {
  const int kb4 = (kb + 3) & ~3;
  const int ldp = ((n + 15) & ~15) + 4;
  return sizeof(double) * ((size_t)kb4 * ldp + (size_t)kb4 * FU_LDW + 32 + 8) + sizeof(int) * (16 + 32 + n + 8);
}

int gj_fused_ldp(int n) { return ((n + 15) & ~15) + 4; }

int launch_gj_fused(const FusedArgs& a0, int grid, cudaStream_t s) {
  FusedArgs a = a0;
  a.ldp = gj_fused_ldp(a.n);
  const size_t smem = gj_fused_smem(a.n, a.kb);
  if (smem > 227 * 1024) return 1;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(gj_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = 227 * 1024;
  }
  gj_fused_kernel<<<grid, FU_THREADS, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
