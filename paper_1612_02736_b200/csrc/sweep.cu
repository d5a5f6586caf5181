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
#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

constexpr int SW_THREADS = 256;

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
  const int* xi = a.xidx + (long long)item * K;
  const int* x2 = a.x2idx ? a.x2idx + (long long)item * K : nullptr;
  double* pool = a.pool;

  for (int e = tid; e < (r1 - r0) * NR; e += SW_THREADS) part[e] = 0.0;

  for (int k0 = 0; k0 < K; k0 += kchunk) {
    const int kc = min(kchunk, K - k0);
    __syncthreads();
    for (int e = tid; e < kc * NR; e += SW_THREADS) {
      const int k = e / NR, j = e - k * NR;
      double v = 0.0;
      if (j < nrhs) {
        v = pool[(long long)xi[k0 + k] * nrhs + j];
        if (x2) v -= pool[(long long)x2[k0 + k] * nrhs + j];
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
  const int* ai = a.aidx ? a.aidx + (long long)item * R : nullptr;
  const int* oi = a.oidx + (long long)item * R;
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
// right-hand sides. Warp tile 16 rows x NRP; A fragments come straight from global memory
// (each lane group reads 4 consecutive doubles = one 32-byte sector per row), X is staged
// (gathered) in shared memory with a padded stride so B-fragment loads are conflict free.
template <int NRP>
__global__ void __launch_bounds__(128) gemv_dmma_kernel(GemvArgs a, int kchunk, int batch_off) {
  extern __shared__ double xs[];
  constexpr int XLD = NRP + 4;
  constexpr int NT = NRP / 8;
  const int item = blockIdx.y + batch_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int R = a.R, K = a.K, nrhs = a.nrhs;
  const int rbase = blockIdx.x * (blockDim.x >> 5) * 16 + warp * 16;
  const double* Ai = a.A.get(item);
  const long long lda = a.A.ld;
  const int* xi = a.xidx + (long long)item * K;
  const int* x2 = a.x2idx ? a.x2idx + (long long)item * K : nullptr;
  const double* pool = a.pool;
  const int ra = rbase + gq, rb = rbase + 8 + gq;
  const double* rowa = Ai + (long long)(ra < R ? ra : 0) * lda;
  const double* rowb = Ai + (long long)(rb < R ? rb : 0) * lda;

  double acc[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;

  for (int k0 = 0; k0 < K; k0 += kchunk) {
    const int kc = min(kchunk, K - k0);
    const int kc4 = (kc + 3) & ~3;
    __syncthreads();
    for (int e = tid; e < kc4 * NRP; e += blockDim.x) {
      const int k = e / NRP, j = e - k * NRP;
      double v = 0.0;
      if (j < nrhs && k < kc) {
        v = pool[(long long)xi[k0 + k] * nrhs + j];
        if (x2) v -= pool[(long long)x2[k0 + k] * nrhs + j];
      }
      xs[k * XLD + j] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kc4; k += 4) {
      const int kk = k0 + k + tq;
      const bool kin = (k + tq) < kc;
      const double a0 = (kin && ra < R) ? __ldg(rowa + kk) : 0.0;
      const double a1 = (kin && rb < R) ? __ldg(rowb + kk) : 0.0;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double bv = xs[(k + tq) * XLD + n * 8 + gq];
        dmma8x8x4(acc[0][n][0], acc[0][n][1], a0, bv);
        dmma8x8x4(acc[1][n][0], acc[1][n][1], a1, bv);
      }
    }
  }
  const int* ai = a.aidx ? a.aidx + (long long)item * R : nullptr;
  const int* oi = a.oidx + (long long)item * R;
  double* pw = a.pool;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = i ? rb : ra;
    if (r >= R) continue;
    const long long orow = (long long)oi[r] * nrhs;
    const long long arow = ai ? (long long)ai[r] * nrhs : -1;
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
    gemv_gather_kernel<NR><<<grid, SW_THREADS, smem, s>>>(a, rows, kchunk, off);
  }
}

template <int NRP>
static void launch_dmma(const GemvArgs& a, cudaStream_t s) {
  int warps = (a.R + 15) / 16;
  if (warps > 4) warps = 4;
  const int rows = warps * 16;
  int kchunk = (48 * 1024 / 8) / (NRP + 4);
  kchunk &= ~3;
  const int k4 = (a.K + 3) & ~3;
  if (kchunk > k4) kchunk = k4;
  const size_t smem = sizeof(double) * (size_t)kchunk * (NRP + 4);
  const int gx = (a.R + rows - 1) / rows;
  for (int off = 0; off < a.nitems; off += 65535) {
    dim3 grid(gx, min(65535, a.nitems - off));
    gemv_dmma_kernel<NRP><<<grid, warps * 32, smem, s>>>(a, kchunk, off);
  }
}

int launch_gemv_gather(const GemvArgs& a, cudaStream_t s) {
  if (a.nitems <= 0 || a.R <= 0) return 0;
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
