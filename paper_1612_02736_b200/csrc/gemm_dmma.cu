// Batched FP64 GEMM on DMMA tiles (mma.sync.m8n8k4.f64), cp.async double-buffered smem staging.
//
//   MODE_GEMM   : C_i = alpha * A_i B_i + beta * C_i            (M x N x K, row-major, any ld)
//   MODE_GJ_UPD : blocked Gauss-Jordan trailing update of matrix M_i (n x ncols):
//                 logical column c -> physical c' = c < k0 ? c : c + kb (the panel is skipped),
//                 C[r,c'] = (r in [k0,k0+kb) ? 0 : C[r,c']) + panel[r,:] . W[:, c']
//                 with panel = M_i[:, k0:k0+kb] (already factored) and W = the kb pivot rows
//                 saved before this update (gj.cu).
//
// CTA tile 64x64, BK 16, 4 warps (2x2), warp tile 32x32 = 4x4 DMMA 8x8 blocks, 32 f64
// accumulators per thread. smem: A tile row-major [64][20], B tile [16][68] — paddings chosen
// so the 8-byte fragment loads (A[g][t], B[t][g]) are bank-conflict free.
#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

constexpr int GB_M = 64, GB_N = 64, GB_K = 16;
constexpr int GA_LD = GB_K + 4;  // 20
constexpr int GBS_LD = GB_N + 4; // 68

template <int MODE>
__global__ void __launch_bounds__(128) gemm_dmma_kernel(GemmArgs g, int batch_off) {
  __shared__ __align__(16) double As[2][GB_M * GA_LD];
  __shared__ __align__(16) double Bs[2][GB_K * GBS_LD];

  const int item = blockIdx.z + batch_off;
  const int m0 = blockIdx.y * GB_M;
  const int n0 = blockIdx.x * GB_N;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int gq = lane >> 2, tq = lane & 3;

  const double* A = g.A.get(item);
  const double* B = g.B.get(item);
  double* C = g.C.get(item);
  const int lda = g.A.ld, ldb = g.B.ld, ldc = g.C.ld;
  const int M = g.M, N = g.N, K = g.K;

  auto colmap = [&](int c) { return (MODE == MODE_GJ_UPD && c >= g.k0) ? c + g.kb : c; };

  auto load_tile = [&](int stage, int k) {
    // A: 64 rows x 16 k  -> 1024 elements, 8 per thread; consecutive threads walk k
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int idx = tid + it * 128;
      int kk = idx & 15, mm = idx >> 4;
      int r = m0 + mm, kc = k + kk;
      bool ok = (r < M) && (kc < K);
      const double* src = ok ? (A + (long long)r * lda + kc) : A;
      cp_async8(&As[stage][mm * GA_LD + kk], src, ok);
    }
    // B: 16 k x 64 cols
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int idx = tid + it * 128;
      int nn = idx & 63, kk = idx >> 6;
      int c = n0 + nn, kr = k + kk;
      bool ok = (c < N) && (kr < K);
      const double* src = ok ? (B + (long long)kr * ldb + colmap(c)) : B;
      cp_async8(&Bs[stage][kk * GBS_LD + nn], src, ok);
    }
    cp_async_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = (K + GB_K - 1) / GB_K;
  if (ktiles > 0) load_tile(0, 0);
  for (int kt = 0; kt < ktiles; ++kt) {
    const int st = kt & 1;
    if (kt + 1 < ktiles) {
      load_tile(st ^ 1, (kt + 1) * GB_K);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As[st];
    const double* bs = Bs[st];
#pragma unroll
    for (int k4 = 0; k4 < GB_K; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(wm + i * 8 + gq) * GA_LD + k4 + tq];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(k4 + tq) * GBS_LD + wn + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + gq;
    if (r >= M) continue;
    double beta = g.beta;
    if (MODE == MODE_GJ_UPD) beta = (r >= g.k0 && r < g.k0 + g.kb) ? 0.0 : 1.0;
    double* crow = C + (long long)r * ldc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + j * 8 + tq * 2 + h;
        if (c < N) {
          const int pc = colmap(c);
          double v = g.alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * crow[pc];
          if (MODE == MODE_GEMM && g.bias) v += g.bias[(long long)r * g.ldbias + c];
          crow[pc] = v;
        }
      }
    }
  }
}

int launch_gemm(const GemmArgs& g, int batch, int mode, cudaStream_t s) {
  if (batch <= 0 || g.M <= 0 || g.N <= 0) return 0;
  dim3 block(128);
  const int gx = (g.N + GB_N - 1) / GB_N, gy = (g.M + GB_M - 1) / GB_M;
  for (int off = 0; off < batch; off += 65535) {
    int nb = batch - off < 65535 ? batch - off : 65535;
    dim3 grid(gx, gy, nb);
    if (mode == MODE_GEMM)
      gemm_dmma_kernel<MODE_GEMM><<<grid, block, 0, s>>>(g, off);
    else
      gemm_dmma_kernel<MODE_GJ_UPD><<<grid, block, 0, s>>>(g, off);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
