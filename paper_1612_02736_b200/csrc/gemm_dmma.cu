#include <cstdlib>
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

  auto colmap = [&](int c) { return (MODE == MODE_GJ_UPD && c >= g.kc) ? c + g.kb : c; };

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

// ------------------------------------------------------------------------------------------
// Large-tile variant for the big contractions (GJ trailing updates with K = 64, merge
// T_new = T_ei S, wraps): CTA tile 128x128, BK 16, 8 warps (2 x 4), warp tile 64x32
// (8 x 4 DMMA blocks, 64 f64 accumulators / thread), 3-stage cp.async pipeline with 16-byte
// copies when every operand is 16-byte aligned (else 8-byte copies). Fragment loads use the
// same conflict-free paddings (A row stride 20, B row stride 132 doubles).
constexpr int BB_M = 128, BB_K = 16;
constexpr int BA_LD = BB_K + 4;
constexpr int BA_STAGE = BB_M * BA_LD;
template <int BN, int STAGES = 3> struct BigCfg {
  static constexpr int THREADS = BN * 2;          // warps = BN / 16, warp tile 64 x 32
  static constexpr int BS_LD = BN + 4;            // = 4 mod 16 doubles
  static constexpr int B_STAGE = BB_K * BS_LD;
  // 128x64 tiles: two CTAs per SM overlap (three with a 2-stage pipeline)
  static constexpr int MINB = BN == 128 ? 1 : (STAGES == 2 ? 3 : 2);
  static constexpr size_t SMEM = sizeof(double) * STAGES * (BA_STAGE + B_STAGE);
};

__device__ __forceinline__ void cp_async16_part(void* smem, const void* gmem, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes));
}

template <int MODE, bool VEC, int BN, int BB_STAGES = 3>
__global__ void __launch_bounds__(BigCfg<BN, BB_STAGES>::THREADS, BigCfg<BN, BB_STAGES>::MINB)
    gemm_big_kernel(GemmArgs g, int batch_off) {
  using Cfg = BigCfg<BN, BB_STAGES>;
  constexpr int NT = Cfg::THREADS;
  constexpr int WN = BN / 32;  // warps along n
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;
  double* Bs = gsm + BB_STAGES * BA_STAGE;
  const int item = blockIdx.z + batch_off;
  const int m0 = blockIdx.y * BB_M, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / WN) * 64, wn = (warp % WN) * 32;
  const int gq = lane >> 2, tq = lane & 3;
  const double* A = g.A.get(item);
  const double* B = g.B.get(item);
  double* C = g.C.get(item);
  const long long lda = g.A.ld, ldb = g.B.ld, ldc = g.C.ld;
  const int M = g.M, N = g.N, K = g.K;
  auto colmap = [&](int c) { return (MODE == MODE_GJ_UPD && c >= g.kc) ? c + g.kb : c; };

  auto load_tile = [&](int stage, int k) {
    double* as = As + stage * BA_STAGE;
    double* bs = Bs + stage * Cfg::B_STAGE;
    if (VEC) {
#pragma unroll
      for (int it = 0; it < (BB_M * BB_K / 2) / NT; ++it) {
        const int idx = tid + it * NT;
        const int mm = idx >> 3, kk = (idx & 7) * 2;
        const int r = m0 + mm, kc = k + kk;
        const int bytes = (r < M) ? min(16, max(0, (K - kc) * 8)) : 0;
        cp_async16_part(as + mm * BA_LD + kk, bytes ? (A + r * lda + kc) : A, bytes);
      }
#pragma unroll
      for (int it = 0; it < (BB_K * BN / 2) / NT; ++it) {
        const int idx = tid + it * NT;
        const int kk = idx / (BN / 2), nn = (idx % (BN / 2)) * 2;
        const int c = n0 + nn, kr = k + kk;
        const int bytes = (kr < K) ? min(16, max(0, (N - c) * 8)) : 0;
        cp_async16_part(bs + kk * Cfg::BS_LD + nn, bytes ? (B + kr * ldb + colmap(c)) : B, bytes);
      }
    } else {
#pragma unroll
      for (int it = 0; it < (BB_M * BB_K) / NT; ++it) {
        const int idx = tid + it * NT;
        const int mm = idx >> 4, kk = idx & 15;
        const int r = m0 + mm, kc = k + kk;
        const bool ok = r < M && kc < K;
        cp_async8(as + mm * BA_LD + kk, ok ? (A + r * lda + kc) : A, ok);
      }
#pragma unroll
      for (int it = 0; it < (BB_K * BN) / NT; ++it) {
        const int idx = tid + it * NT;
        const int kk = idx / BN, nn = idx % BN;
        const int c = n0 + nn, kr = k + kk;
        const bool ok = c < N && kr < K;
        cp_async8(bs + kk * Cfg::BS_LD + nn, ok ? (B + kr * ldb + colmap(c)) : B, ok);
      }
    }
  };

  const int ktiles = (K + BB_K - 1) / BB_K;
#pragma unroll
  for (int st = 0; st < BB_STAGES - 1; ++st) {
    if (st < ktiles) load_tile(st, st * BB_K);
    cp_async_commit();
  }

  // alpha == 1: accumulators start from C (rows outside the GJ panel / beta != 0), loaded
  // straight into the accumulator registers so all C reads are in flight together while the
  // pipeline fills; beta and the bias are applied in registers afterwards.
  const bool preload = (g.alpha == 1.0);
  double acc[8][4][2];
  int pcol[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) pcol[j] = colmap(n0 + wn + j * 8 + tq * 2);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = m0 + wm + i * 8 + gq;
    const bool rowload = preload && r < M && (MODE == MODE_GJ_UPD ? !(r >= g.k0 && r < g.k0 + g.kb) : g.beta != 0.0);
    const double* crow = C + (long long)(r < M ? r : 0) * ldc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + wn + j * 8 + tq * 2;
      if (VEC) {
        double2 o = make_double2(0.0, 0.0);
        if (rowload && c + 1 < N) o = *reinterpret_cast<const double2*>(crow + pcol[j]);
        else if (rowload && c < N) o.x = crow[pcol[j]];
        acc[i][j][0] = o.x;
        acc[i][j][1] = o.y;
      } else {
        acc[i][j][0] = (rowload && c < N) ? crow[colmap(c)] : 0.0;
        acc[i][j][1] = (rowload && c + 1 < N) ? crow[colmap(c + 1)] : 0.0;
      }
    }
  }
  if (preload && MODE == MODE_GEMM && (g.beta != 1.0 || g.bias)) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = m0 + wm + i * 8 + gq;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + tq * 2 + h;
          double v = acc[i][j][h] * g.beta;
          if (g.bias && r < M && c < N) v += g.bias[(long long)r * g.ldbias + c];
          acc[i][j][h] = v;
        }
    }
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<BB_STAGES - 2>();
    __syncthreads();
    const int nxt = kt + BB_STAGES - 1;
    if (nxt < ktiles) load_tile(nxt % BB_STAGES, nxt * BB_K);
    cp_async_commit();
    const double* as = As + (kt % BB_STAGES) * BA_STAGE;
    const double* bs = Bs + (kt % BB_STAGES) * Cfg::B_STAGE;
#pragma unroll
    for (int k4 = 0; k4 < BB_K; k4 += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = as[(wm + i * 8 + gq) * BA_LD + k4 + tq];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(k4 + tq) * Cfg::BS_LD + wn + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = m0 + wm + i * 8 + gq;
    if (r >= M) continue;
    double beta = g.beta;
    if (MODE == MODE_GJ_UPD) beta = (r >= g.k0 && r < g.k0 + g.kb) ? 0.0 : 1.0;
    double* crow = C + r * ldc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + wn + j * 8 + tq * 2;
      if (preload) {
        if (VEC && c + 1 < N) {
          *reinterpret_cast<double2*>(crow + pcol[j]) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (c < N) crow[colmap(c)] = acc[i][j][0];
          if (c + 1 < N) crow[colmap(c + 1)] = acc[i][j][1];
        }
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + h < N) {
          const int pc = colmap(c + h);
          double v = g.alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * crow[pc];
          if (MODE == MODE_GEMM && g.bias) v += g.bias[(long long)r * g.ldbias + c + h];
          crow[pc] = v;
        }
      }
    }
  }
}

static bool aligned16(const MatB& m) {
  if (m.ptrs) return false;
  const uintptr_t p = reinterpret_cast<uintptr_t>(m.base + m.off);
  return (p % 16 == 0) && (m.ld % 2 == 0) && (m.stride % 2 == 0);
}

template <int MODE, int BN, int ST = 3>
static void launch_big(const GemmArgs& g, int batch, cudaStream_t s) {
  using Cfg = BigCfg<BN, ST>;
  const bool vec = aligned16(g.A) && aligned16(g.B) && aligned16(g.C) &&
                   (MODE != MODE_GJ_UPD || (g.kc % 2 == 0 && g.kb % 2 == 0));
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gemm_big_kernel<MODE, true, BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg::SMEM);
    cudaFuncSetAttribute(gemm_big_kernel<MODE, false, BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg::SMEM);
    configured = true;
  }
  const int gx = (g.N + BN - 1) / BN, gy = (g.M + BB_M - 1) / BB_M;
  for (int off = 0; off < batch; off += 65535) {
    dim3 grid(gx, gy, min(65535, batch - off));
    if (vec)
      gemm_big_kernel<MODE, true, BN, ST><<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(g, off);
    else
      gemm_big_kernel<MODE, false, BN, ST><<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(g, off);
  }
}

static int gemm_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HPS_GEMM_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

int launch_gemm(const GemmArgs& g, int batch, int mode, cudaStream_t s) {
  if (batch <= 0 || g.M <= 0 || g.N <= 0) return 0;
  // (N >= 48: the 60-column next-block updates of the p = 32 leaf GJ; the masked tile tail costs
  // less than the 64x64 kernel's lower efficiency)
  if (g.M >= 96 && g.N >= 48 && g.K >= 16) {
    // read-modify-write updates with short K are memory-heavy: 128x64 tiles with a 2-stage
    // pipeline, 3 CTAs/SM (measured +3 % over 3 stages / 2 CTAs on the K = 64 GJ updates)
    const bool rmw = mode == MODE_GJ_UPD || g.beta != 0.0;
    if (mode == MODE_GEMM) {
      // 64-wide tiles also when they pad N much less than 128-wide ones (H = D F at p = 32:
      // N = 900 -> 960 instead of 1024); HPS_GEMM_PAD64=0 disables
      static int pad64 = -1;
      if (pad64 < 0) {
        const char* e = getenv("HPS_GEMM_PAD64");
        pad64 = e ? atoi(e) : 1;
      }
      const bool narrow_pad = pad64 && 100 * ((g.N + 63) / 64 * 64) < 95 * ((g.N + 127) / 128 * 128);
      if (rmw || g.N < 96 || narrow_pad) {
        if (gemm_variant() == 3) launch_big<MODE_GEMM, 64>(g, batch, s);
        else launch_big<MODE_GEMM, 64, 2>(g, batch, s);
      } else {
        launch_big<MODE_GEMM, 128>(g, batch, s);
      }
    } else {
      // long-K outer updates of the three-level GJ: C traffic is amortised over K >= 128, the
      // 128 x 128 tile's higher math density wins (HPS_GJ_BIG_K: smallest K for it)
      static int bigk = -1;
      if (bigk < 0) {
        const char* e = getenv("HPS_GJ_BIG_K");
        bigk = e ? atoi(e) : 1 << 30;
      }
      if (g.K >= bigk && g.N >= 96)
        launch_big<MODE_GJ_UPD, 128>(g, batch, s);
      else if (gemm_variant() == 3)
        launch_big<MODE_GJ_UPD, 64>(g, batch, s);
      else
        launch_big<MODE_GJ_UPD, 64, 2>(g, batch, s);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
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
