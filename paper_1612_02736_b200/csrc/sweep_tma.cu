// Multi-RHS leaf sweep steps (3..16 right-hand sides) fed by TMA: Y (R x nrhs) = A (R x K) X.
//
// The leaf operators of one shape group are one contiguous [nitems*R][K] row-major array, so a
// single 2D tensor map covers the whole level. A persistent CTA (one per SM) walks its items;
// a producer warp streams 16-column slabs of an item's R rows (R <= 256) into a ring of
// shared-memory stages with cp.async.bulk.tensor (128-byte swizzle, mbarrier complete_tx), so
// up to NS x R x 128 bytes per SM are in flight regardless of the consumers' progress. The 8
// consumer warps own fixed 8-row m-tiles (tile w, w+8, w+16, w+24) and run DMMA m8n8k4 on
// conflict-free swizzled A fragments against the item's gathered X (K x NRP, padded stride).
// X of the next item is gathered with cp.async while the current item computes (double
// buffer). mode2 = 1 (leaf down) also applies the tail y2 = A2 x[K-K2:K) (the shared lift L).
//
// Why: at 16 RHS the leaf steps are 4 flop/byte, so the kernel has to keep HBM and the DMMA
// pipes busy at once; the register-streaming gemv_dmma_kernel (sweep.cu) ran the config-5 leaf
// downward step at 3.2 TB/s with its loads exposed (long-scoreboard stalls); this kernel runs it
// at 4.1 TB/s (1.62 vs 2.05 ms, 16 RHS). Measured pitfalls: a guarded DMMA compiles to a
// predicated one that still occupies the tensor pipe (hence the per-tile-count dispatch), and
// with only 8 consumer warps per SM the short leaf upward operators (R = 4q) stay faster on
// the 32-warp register kernel, so only R >= 128 comes here.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

namespace {

// NC consumer warps (template parameter, 8 or 16) + 1 producer warp; a consumer warp owns up to
// 32 / NC m-tiles of 8 rows (R <= 256)

__device__ __forceinline__ uint32_t tma_smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tma_smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tma_smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tma_smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(tma_smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          tma_smem_addr(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(tma_smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(tma_smem_addr(dst)), "l"(src) : "memory");
}
// DMMA without the volatile qualifier: no side effects, so the compiler may interleave the
// fragment loads of the next k-step with the current tensor ops
__device__ __forceinline__ void dmma_nv(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
template <int NC>
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(NC * 32) : "memory"); }


}  // namespace

// One pipeline stage of MMAs for a warp owning T m-tiles (tile = warp + 8 i): SPS slabs of 16
// columns, 4 k4-steps each; even / odd k4 steps accumulate into separate sets.
template <int T, int NT, int XLD, int SPS, int NC, int MT>
__device__ __forceinline__ void stage_mma(double (&acc)[2][MT][NT][2], const unsigned char* base, int slot,
                                          int sb_bytes, int nq, const double* xc, int k0, const int (&aoff)[4],
                                          int warp, int g, int t) {
#pragma unroll
  for (int q = 0; q < SPS; ++q) {
    if (q >= nq) break;
    const double* slab = reinterpret_cast<const double*>(base + (size_t)(slot * SPS + q) * sb_bytes);
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int kk = k0 + q * 16 + k4 * 4 + t;
      double bv[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) bv[n] = xc[kk * XLD + n * 8 + g];
      double av[T];
#pragma unroll
      for (int i = 0; i < T; ++i) av[i] = slab[(warp + i * NC) * 128 + aoff[k4]];
#pragma unroll
      for (int i = 0; i < T; ++i)
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma_nv(acc[k4 & 1][i][n][0], acc[k4 & 1][i][n][1], av[i], bv[n]);
    }
  }
}

constexpr int TM_GUNITS = 12 * 256;  // x-gather copy units per CTA (K * units per row)

template <int NRP, int SPS, int NC>
__global__ void __launch_bounds__(32 * (NC + 1), 1)
    gemv_tma_kernel(const __grid_constant__ CUtensorMap tm, GemvArgs a, int ns, int kst, int sb_bytes, int a2ld) {
  constexpr int sps = SPS;
  constexpr int MT = 32 / NC;                // m-tiles per consumer warp
  constexpr int TM_GMAX = TM_GUNITS / (NC * 32);  // x-gather copy units per consumer thread
  extern __shared__ unsigned char smraw[];
  // 1024-byte aligned (128B swizzle) by pointer arithmetic on the shared array itself: a round
  // trip through an integer would lose the address space and turn every fragment load into a
  // generic LD instead of LDS
  unsigned char* base = smraw + ((1024u - (tma_smem_addr(smraw) & 1023u)) & 1023u);
  constexpr int XLD = NRP + 4;
  constexpr int NT = NRP / 8;
  const int R = a.R, K = a.K, nrhs = a.nrhs;
  // kst: stages per item, each sps 16-column slabs of sb_bytes (one TMA box each)
  const int kp = kst * sps * 16;
  const int nslab = (K + 15) >> 4;
  double* xbuf = reinterpret_cast<double*>(base + (size_t)ns * sps * sb_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + 2 * (size_t)kp * XLD);
  uint64_t* empty = full + ns;
  // a2ld > 0: the level-shared tail operator (leaf down: the lift L) staged here once per CTA,
  // rows padded to a2ld (== 4 mod 16: conflict-free fragments), rows past R2 zero
  double* a2s = reinterpret_cast<double*>(empty + ns);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const unsigned slab_tx = (unsigned)R * 128u;

  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();

  if (warp == NC) {
    // ---- producer: operator slabs never depend on the previous kernel, start right away
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
      int slot = 0;
      unsigned ph = 0;
      bool first = true;
      for (int item = blockIdx.x; item < a.nitems; item += gridDim.x) {
        for (int ks = 0; ks < kst; ++ks) {
          if (!first) mbar_wait(empty + slot, ph ^ 1u);
          const int nq = min(sps, nslab - ks * sps);  // no fully out-of-range boxes
          mbar_expect_tx(full + slot, slab_tx * nq);
          for (int q = 0; q < nq; ++q)
            tma_load_2d(base + (size_t)(slot * sps + q) * sb_bytes, &tm, (ks * sps + q) * 16, item * R, full + slot);
          if (++slot == ns) {
            slot = 0;
            ph ^= 1u;
            first = false;
          }
        }
      }
    }
    return;
  }

  // ---- consumers
  // x-gather plan (same for every item): unit u of this thread = (row, first rhs, width)
  const bool wide = (nrhs % 2 == 0);
  const int upr = wide ? nrhs / 2 : nrhs;  // copy units per row
  const int nunits = K * upr;
  int urow[TM_GMAX], ucol[TM_GMAX];
#pragma unroll
  for (int u = 0; u < TM_GMAX; ++u) {
    const int e = tid + u * NC * 32;
    urow[u] = e < nunits ? e / upr : -1;
    ucol[u] = e < nunits ? (e - (e / upr) * upr) * (wide ? 2 : 1) : 0;
  }
  int nidx[TM_GMAX];
  auto load_idx = [&](int item) {
    const int* xi = a.xidx + (long long)item * a.xstride;
#pragma unroll
    for (int u = 0; u < TM_GMAX; ++u) nidx[u] = urow[u] >= 0 ? __ldg(xi + urow[u]) : 0;
  };
  auto issue_copies = [&](double* xb) {
#pragma unroll
    for (int u = 0; u < TM_GMAX; ++u) {
      if (urow[u] < 0) continue;
      const double* src = a.pool + (long long)nidx[u] * nrhs + ucol[u];
      double* dst = xb + urow[u] * XLD + ucol[u];
      if (wide)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(tma_smem_addr(dst)), "l"(src) : "memory");
      else
        cp_async8(dst, src);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  for (int e = tid; e < 2 * kp * XLD; e += NC * 32) xbuf[e] = 0.0;
  if (a2ld) {
    // static data: before the launch wait
    const double* A2 = a.A2.get(0);
    const int r2p = (a.R2 + 7) & ~7;
    for (int e = tid; e < r2p * a2ld; e += NC * 32) {
      const int r = e / a2ld, k = e - r * a2ld;
      a2s[e] = (r < a.R2 && k < a.K2) ? __ldg(A2 + (long long)r * a.A2.ld + k) : 0.0;
    }
  }
  consumers_sync<NC>();
  pdl_wait();  // the pool (x) is produced by the previous step
  if (blockIdx.x < a.nitems) {
    load_idx(blockIdx.x);
    issue_copies(xbuf);
  }
  // indices of the item after next are loaded one item ahead of their copies, so neither the
  // index loads nor the copies sit on the consumers' critical path
  if (blockIdx.x + gridDim.x < a.nitems) load_idx(blockIdx.x + gridDim.x);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  consumers_sync<NC>();

  // A fragment rows: lanes g = 0..3 take even rows, 4..7 odd rows of an 8-row tile, so both
  // half-warps read 8 distinct 16-byte chunks of the 128B-swizzled slab (no bank conflicts)
  const int rg = ((g & 3) << 1) | (g >> 2);
  int aoff[4];
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) {
    const int c = k4 * 4 + t;
    aoff[k4] = rg * 16 + ((((c >> 1) ^ rg) << 1) | (c & 1));
  }
  const int mt = (R + 7) >> 3;
  const int ntw = warp < mt ? (mt - warp + NC - 1) / NC : 0;  // m-tiles of this warp
  int slot = 0;
  unsigned ph = 0;
  int it = 0;
  for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, ++it) {
    double* xc = xbuf + (size_t)(it & 1) * kp * XLD;
    double* xn = xbuf + (size_t)((it + 1) & 1) * kp * XLD;
    if (a.kscale > 0) {
      // backward Euler: the first kscale gathered columns (the body load u_n) times 1/dt
      for (int e = tid; e < a.kscale * NRP; e += NC * 32) xc[(e / NRP) * XLD + (e % NRP)] *= a.xscale;
      consumers_sync<NC>();
    }
    // two accumulator sets (even / odd k4 steps): twice the independent DMMA chains per warp
    double acc[2][MT][NT][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[h][i][n][0] = acc[h][i][n][1] = 0.0;
    const int nxt = item + gridDim.x;
    if (nxt < a.nitems) issue_copies(xn);  // indices loaded during the previous item
    if (nxt + (int)gridDim.x < a.nitems) load_idx(nxt + gridDim.x);
    // output rows of this item, loaded ahead of the epilogue
    const int* oi = a.oidx + (long long)item * a.ostride;
    const int* ai = a.aidx ? a.aidx + (long long)item * a.ostride : nullptr;
    int orows[MT], arows[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int r = (warp + i * NC) * 8 + rg;
      orows[i] = r < R ? __ldg(oi + r) : 0;
      arows[i] = (ai && r < R) ? __ldg(ai + r) : -1;
    }
    if (a.mode2 == 1) {
      // tail: y2 = A2 x[K-K2:K); A2 shared by the level (lift L). It depends on x only, so it runs
      // BEFORE the main loop, on the warps that own fewer m-tiles (the upper half), while the
      // first slabs of the item are still in flight: no serial tail phase at the end of an item
      const double* A2 = a.A2.get(item);
      const int ld2 = a.A2.ld, K2 = a.K2, R2 = a.R2, x0 = K - K2;
      const int* o2 = a.o2idx + (long long)item * R2;
      const int* a2 = a.a2idx ? a.a2idx + (long long)item * R2 : nullptr;
      for (int tile = (warp + NC / 2) % NC; tile * 8 < R2; tile += NC) {
        const int ra = tile * 8 + g;
        const double* arow2 = A2 + (long long)(ra < R2 ? ra : 0) * ld2;
        double c2[NT][2];
#pragma unroll
        for (int n = 0; n < NT; ++n) c2[n][0] = c2[n][1] = 0.0;
        int k = 0;
        if (a2ld) {
          // staged tail operator: two independent accumulator chains over alternating k4 steps
          const double* as = a2s + (size_t)ra * a2ld;
          double c3[NT][2];
#pragma unroll
          for (int n = 0; n < NT; ++n) c3[n][0] = c3[n][1] = 0.0;
          for (; k + 8 <= K2; k += 8) {
            const double a0 = as[k + t], a1 = as[k + 4 + t];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              dmma_nv(c2[n][0], c2[n][1], a0, xc[(x0 + k + t) * XLD + n * 8 + g]);
              dmma_nv(c3[n][0], c3[n][1], a1, xc[(x0 + k + 4 + t) * XLD + n * 8 + g]);
            }
          }
          for (; k < K2; k += 4) {
            const double a0 = as[k + t];
#pragma unroll
            for (int n = 0; n < NT; ++n) dmma_nv(c2[n][0], c2[n][1], a0, xc[(x0 + k + t) * XLD + n * 8 + g]);
          }
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            c2[n][0] += c3[n][0];
            c2[n][1] += c3[n][1];
          }
        }
        for (; k + 16 <= K2; k += 16) {
          double av[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) av[q] = ra < R2 ? __ldg(arow2 + k + 4 * q + t) : 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int n = 0; n < NT; ++n)
              dmma8x8x4(c2[n][0], c2[n][1], av[q], xc[(x0 + k + 4 * q + t) * XLD + n * 8 + g]);
        }
        for (; k < K2; k += 4) {
          const int kk = k + t;
          const double av = (ra < R2 && kk < K2) ? __ldg(arow2 + kk) : 0.0;
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const double bv = (kk < K2) ? xc[(x0 + kk) * XLD + n * 8 + g] : 0.0;
            dmma8x8x4(c2[n][0], c2[n][1], av, bv);
          }
        }
        if (ra < R2) {
          const long long orow = (long long)o2[ra] * nrhs;
          const long long arow = a2 ? (long long)a2[ra] * nrhs : -1;
#pragma unroll
          for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = n * 8 + 2 * t + h;
              if (j < nrhs) {
                double v = c2[n][h];
                if (arow >= 0) v += a.pool[arow + j];
                a.pool[orow + j] = v;
              }
            }
        }
      }
    }
    for (int ks = 0; ks < kst; ++ks) {
      mbar_wait(full + slot, ph);
      const int nq = min(sps, nslab - ks * sps);
      // the tile count is warp-uniform: dispatch to a branch-free body per count (a guarded
      // DMMA compiles to a predicated one, which still occupies the tensor pipe)
      switch (ntw) {
        case 1: stage_mma<1, NT, XLD, SPS, NC, MT>(acc, base, slot, sb_bytes, nq, xc, (ks * sps) * 16, aoff, warp, g, t); break;
        case 2: stage_mma<(MT >= 2 ? 2 : 1), NT, XLD, SPS, NC, MT>(acc, base, slot, sb_bytes, nq, xc, (ks * sps) * 16, aoff, warp, g, t); break;
        case 3: stage_mma<(MT >= 3 ? 3 : 1), NT, XLD, SPS, NC, MT>(acc, base, slot, sb_bytes, nq, xc, (ks * sps) * 16, aoff, warp, g, t); break;
        case 4: stage_mma<(MT >= 4 ? 4 : 1), NT, XLD, SPS, NC, MT>(acc, base, slot, sb_bytes, nq, xc, (ks * sps) * 16, aoff, warp, g, t); break;
        default: break;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if (++slot == ns) {
        slot = 0;
        ph ^= 1u;
      }
    }
    // epilogue: y rows -> pool (+ add rows)
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int r = (warp + i * NC) * 8 + rg;
      if (r >= R) continue;
      const long long orow = (long long)orows[i] * nrhs;
      const long long arow = arows[i] >= 0 ? (long long)arows[i] * nrhs : -1;
      if (wide) {
        // even nrhs: the pair (j, j + 1) of a lane is one 16-byte access
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int j = n * 8 + 2 * t;
          if (j < nrhs) {
            double2 v = make_double2(acc[0][i][n][0] + acc[1][i][n][0], acc[0][i][n][1] + acc[1][i][n][1]);
            if (arow >= 0) {
              const double2 w = *reinterpret_cast<const double2*>(a.pool + arow + j);
              v.x += w.x;
              v.y += w.y;
            }
            *reinterpret_cast<double2*>(a.pool + orow + j) = v;
          }
        }
        continue;
      }
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = n * 8 + 2 * t + h;
          if (j < nrhs) {
            double v = acc[0][i][n][h] + acc[1][i][n][h];
            if (arow >= 0) v += a.pool[arow + j];
            a.pool[orow + j] = v;
          }
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    consumers_sync<NC>();  // next X landed for everyone; this X no longer read
  }
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool tma_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HPS_SWEEP_TMA");
    on = (e && atoi(e) == 0) ? 0 : 1;
  }
  return on != 0;
}

}  // namespace

// Returns true when the step was launched here; false leaves it to the generic kernels.
bool launch_gemv_tma(const GemvArgs& a, cudaStream_t s) {
  if (!tma_enabled()) return false;
  if (a.nrhs <= 2 || a.nrhs > 16 || a.x2idx || a.A.ptrs || a.kparts > 1 || a.mode2 == 2) return false;
  // the leaf downward step (R = (p-2)^2 >= 128 rows); shorter operators (leaf upward, R = 4q)
  // measured faster on the register-streaming kernel, whose 32 warps/SM hide more latency
  static const int min_r = [] {  // HPS_TMA_MINR: shortest operator routed here
    const char* e = getenv("HPS_TMA_MINR");
    return e ? atoi(e) : 128;
  }();
  if (a.R < min_r || a.R > 256 || a.K < 16 || a.nitems < 148) return false;
  if (a.A.stride != (long long)a.R * a.A.ld || (a.A.ld * 8) % 16 != 0) return false;
  const double* gbase = a.A.base + a.A.off;
  if (reinterpret_cast<uintptr_t>(gbase) % 16 != 0) return false;
  if (a.mode2 == 1 && (a.K2 > a.K || a.R2 <= 0)) return false;
  const int upr = a.nrhs % 2 == 0 ? a.nrhs / 2 : a.nrhs;
  if ((long long)a.K * upr > TM_GUNITS) return false;  // x-gather copy units per CTA
  if (a.nrhs % 2 == 0 && reinterpret_cast<uintptr_t>(a.pool) % 16 != 0) return false;
  auto enc = encode_fn();
  if (!enc) return false;

  const int nrp = a.nrhs <= 8 ? 8 : 16;
  const int xld = nrp + 4;
  const int nslab = (a.K + 15) / 16;
  const int sb = ((a.R * 128 + 1023) / 1024) * 1024;
  const size_t budget = 226 * 1024;
  // the level-shared tail operator (lift) staged in shared memory when a ring of >= 4 stages
  // still fits (HPS_TMA_A2S=0: read it through L1/L2 instead)
  static const int a2s_on = [] {
    const char* e = getenv("HPS_TMA_A2S");
    return e ? atoi(e) : 1;
  }();
  int a2ld = 0;
  size_t a2bytes = 0;
  if (a2s_on && a.mode2 == 1 && a.A2.stride == 0 && !a.A2.ptrs && a.K2 % 4 == 0 && a.K2 > 0) {
    a2ld = ((a.K2 + 11) & ~15) + 4;
    a2bytes = sizeof(double) * (size_t)((a.R2 + 7) & ~7) * a2ld;
  }
  // one 16-column slab per stage (wider stages measured no faster on config 5)
  int sps = 1;
  int ns = 0, kst = 0;
  size_t smem = 0;
  for (int pass = 0; pass < 2; ++pass) {
    kst = (nslab + sps - 1) / sps;
    const size_t xbytes = 2 * sizeof(double) * (size_t)kst * sps * 16 * xld;
    ns = 8;
    while (ns > 2 && 1024 + (size_t)ns * sps * sb + xbytes + 16 * ns + a2bytes > budget) --ns;
    smem = 1024 + (size_t)ns * sps * sb + xbytes + 16 * (size_t)ns + a2bytes;
    if (smem <= budget && (ns >= 4 || !a2ld)) break;
    a2ld = 0;  // not enough room for the staged tail operator and a deep enough ring
    a2bytes = 0;
  }
  if (smem > budget || ns < 2) return false;

  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.nitems * a.R};
  const cuuint64_t strides[1] = {(cuuint64_t)a.A.ld * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)a.R};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(gbase), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;

  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.nitems < sms ? a.nitems : sms;
  // consumer warps per CTA (HPS_TMA_NC = 8 or 16): 16 puts 4 DMMA warps on each SM sub-partition
  static const int nc = [] {
    const char* e = getenv("HPS_TMA_NC");
    return (e && atoi(e) == 8) ? 8 : 16;
  }();
  using KFn = void (*)(const CUtensorMap, GemvArgs, int, int, int, int);
  const KFn k = nc == 16 ? (nrp == 16 ? gemv_tma_kernel<16, 1, 16> : gemv_tma_kernel<8, 1, 16>)
                         : (nrp == 16 ? gemv_tma_kernel<16, 1, 8> : gemv_tma_kernel<8, 1, 8>);
  static bool configured[2] = {};
  if (!configured[nrp == 16]) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget);
    configured[nrp == 16] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * (nc + 1));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = sweep_pdl_for(a.nrhs, true) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, tm, a, ns, kst, sb, a2ld) == cudaSuccess;
}

// ---------------------------------------------------------------------------------------------
// Multi-RHS (3..16) steps with LARGE operator items (top tree levels, split-K parts): the
// operator is streamed by TMA in row blocks of RB <= 256 rows, so every item size maps onto
// one persistent CTA per SM with ~150 KB of operator in flight.
//
// Units = (item, row block); item i may be a split-K part (kparts > 1: column block i % kparts
// of operator i / kparts), described to TMA as (row, column) coordinates in one 2D view of the
// whole operator array. Warp roles per CTA:
//   warp 8       producer: 16-column slabs of the unit's RB rows -> smem ring (128B swizzle)
//   warps 9..10  gather:   x chunks of KX columns (x = pool[xidx] - pool[x2idx], zero padded)
//                          -> a double-buffered smem ring, with the x2 difference applied
//   warps 0..7   DMMA consumers, 4 m-tiles of 8 rows each (tile w, w+8, w+16, w+24)
// The two accumulator sets take alternating k4 steps (two independent DMMA chains per tile);
// mode2 = 3 (parent downward [X | S][d; u_ext]) stores their sum at column K2 as w3 = X d.
// Why: the register-streaming gemv_dmma_kernel kept ~16 KB per SM in flight and ran the config-5
// top levels at 0.2-2.5 TB/s (root downward partials: 147 MB in 123 us).
constexpr int ST_NC = 8, ST_GW = 4, ST_THREADS = 32 * (ST_NC + 1 + ST_GW);

struct StreamCfg {
  int RB, nrb, KX, ns, sb_bytes;
  int ld2;  // mode2 = 1: padded row length of the shared tail operator A2 staged in smem
  int nxb;  // x chunk buffers in the gather ring (2..4)
};

// One 16-column slab for T m-tiles: 4 k4 steps into the two accumulator sets by parity. ksnap:
// chunk-local column where w3 = the partial sum is taken (mode2 = 3), else negative.
template <int T, int NT, int XLD>
__device__ __forceinline__ void stream_slab(double (&acc)[2][4][NT][2], const double* slab, const double* xc, int kl0,
                                            int ksnap, const int (&aoff)[4], int warp, int g, int t,
                                            const int (&wrows)[4], double* pool, int nrhs) {
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) {
    const int kl = kl0 + k4 * 4;
    if (kl == ksnap) {
      // w3 = the partial sum over [0, K2) is final here: stored straight to its pool rows
#pragma unroll
      for (int i = 0; i < T; ++i)
        if (wrows[i] >= 0)
#pragma unroll
          for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int j = n * 8 + 2 * t + hh;
              if (j < nrhs) pool[(long long)wrows[i] * nrhs + j] = acc[0][i][n][hh] + acc[1][i][n][hh];
            }
    }
    double bv[NT], av[T];
#pragma unroll
    for (int n = 0; n < NT; ++n) bv[n] = xc[(kl + t) * XLD + n * 8 + g];
#pragma unroll
    for (int i = 0; i < T; ++i) av[i] = slab[(warp + i * ST_NC) * 128 + aoff[k4]];
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma_nv(acc[k4 & 1][i][n][0], acc[k4 & 1][i][n][1], av[i], bv[n]);
  }
}

template <int NRP>
__global__ void __launch_bounds__(ST_THREADS, 1)
    gemv_stream_kernel(const __grid_constant__ CUtensorMap tm, GemvArgs a, StreamCfg c) {
  extern __shared__ unsigned char smraw[];
  unsigned char* base = smraw + ((1024u - (tma_smem_addr(smraw) & 1023u)) & 1023u);
  constexpr int XLD = NRP + 4;
  constexpr int NT = NRP / 8;
  const int R = a.R, K = a.K, nrhs = a.nrhs, RB = c.RB, KX = c.KX, ns = c.ns;
  const int kp = a.kparts > 1 ? a.kparts : 1;
  const int nslab = (K + 15) >> 4, nchunk = (K + KX - 1) / KX, spc = KX >> 4;
  const long long units = (long long)a.nitems * c.nrb;
  double* xbuf = reinterpret_cast<double*>(base + (size_t)ns * c.sb_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + (size_t)c.nxb * KX * XLD);
  uint64_t* empty = full + ns;
  uint64_t* xfull = empty + ns;
  uint64_t* xempty = xfull + 4;
  double* a2s = reinterpret_cast<double*>(xempty + 4);  // mode2 = 1: R2 x ld2
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, ST_NC);
    }
    for (int i = 0; i < c.nxb; ++i) {
      mbar_init(xfull + i, ST_GW * 32);
      mbar_init(xempty + i, ST_NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();

  if (warp == ST_NC) {
    // ---- producer: static operator, streams before the launch wait
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
      int slot = 0;
      unsigned ph = 0;
      bool first = true;
      const unsigned tx = (unsigned)RB * 128u;
      for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = (int)(u / c.nrb), rb = (int)(u - (long long)item * c.nrb);
        const int row0 = (item / kp) * R + rb * RB, col0 = (item % kp) * K;
        for (int j = 0; j < nslab; ++j) {
          if (!first) mbar_wait(empty + slot, ph ^ 1u);
          mbar_expect_tx(full + slot, tx);
          tma_load_2d(base + (size_t)slot * c.sb_bytes, &tm, col0 + j * 16, row0, full + slot);
          if (++slot == ns) {
            slot = 0;
            ph ^= 1u;
            first = false;
          }
        }
      }
    }
    return;
  }
  if (warp > ST_NC) {
    // ---- gather: x chunks (pool rows written by the previous step: after the launch wait)
    pdl_wait();
    const int gt = tid - (ST_NC + 1) * 32;
    const int upr = nrhs / 2 + (nrhs & 1);  // two RHS per copy unit
    int xs = 0;
    unsigned xph = 0;
    int uses = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
      const int item = (int)(u / c.nrb);
      const int* xi = a.xidx + (long long)item * a.xstride;
      const int* x2 = a.x2idx ? a.x2idx + (long long)item * a.xstride : nullptr;
      for (int ch = 0; ch < nchunk; ++ch, ++uses) {
        if (uses >= c.nxb) mbar_wait(xempty + xs, xph ^ 1u);
        double* xb = xbuf + (size_t)xs * KX * XLD;
        const int k0 = ch * KX;
        if (!x2) {
          // plain gather: 16-byte cp.async copies; the indices of 8 units are loaded together so
          // their latencies overlap, then all copies go out at once; rows past K are zeroed
          for (int e0 = gt; e0 < KX * upr; e0 += 8 * ST_GW * 32) {
            int i1[8];
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const int e = e0 + v * ST_GW * 32, kk = e / upr, k = k0 + kk;
              i1[v] = (e < KX * upr && k < K) ? __ldg(xi + k) : -1;
            }
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const int e = e0 + v * ST_GW * 32, kk = e / upr, j = 2 * (e - kk * upr);
              if (e >= KX * upr) continue;
              double* dst = xb + kk * XLD + j;
              if (i1[v] >= 0 && j + 1 < nrhs && !(nrhs & 1)) {  // 16-byte copies need an even row length
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(tma_smem_addr(dst)),
                             "l"(a.pool + (long long)i1[v] * nrhs + j)
                             : "memory");
              } else if (i1[v] >= 0) {
                const double* src = a.pool + (long long)i1[v] * nrhs + j;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(tma_smem_addr(dst)), "l"(src) : "memory");
                if (j + 1 < nrhs)
                  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(tma_smem_addr(dst + 1)), "l"(src + 1)
                               : "memory");
                else if (j + 1 < NRP)
                  dst[1] = 0.0;
              } else {
                dst[0] = 0.0;
                if (j + 1 < NRP) dst[1] = 0.0;
              }
            }
          }
          asm volatile("cp.async.wait_all;\n" ::: "memory");
        } else {
          for (int e0 = gt; e0 < KX * upr; e0 += 8 * ST_GW * 32) {
            int i1[8], i2[8];
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const int e = e0 + v * ST_GW * 32, kk = e / upr, k = k0 + kk;
              const bool ok = e < KX * upr && k < K;
              i1[v] = ok ? __ldg(xi + k) : -1;
              i2[v] = ok ? __ldg(x2 + k) : -1;
            }
            double2 val[8];
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const int e = e0 + v * ST_GW * 32, kk = e / upr, j = 2 * (e - kk * upr);
              val[v] = make_double2(0.0, 0.0);
              if (i1[v] >= 0) {
                const double* p1 = a.pool + (long long)i1[v] * nrhs + j;
                val[v].x = p1[0];
                if (j + 1 < nrhs) val[v].y = p1[1];
                if (i2[v] >= 0) {
                  const double* p2 = a.pool + (long long)i2[v] * nrhs + j;
                  val[v].x -= p2[0];
                  if (j + 1 < nrhs) val[v].y -= p2[1];
                }
              }
            }
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const int e = e0 + v * ST_GW * 32, kk = e / upr, j = 2 * (e - kk * upr);
              if (e < KX * upr) {
                xb[kk * XLD + j] = val[v].x;
                if (j + 1 < NRP) xb[kk * XLD + j + 1] = val[v].y;
              }
            }
          }
        }
        mbar_arrive(xfull + xs);
        if (++xs == c.nxb) {
          xs = 0;
          xph ^= 1u;
        }
      }
    }
    return;
  }

  // ---- consumers
  const bool tail = a.mode2 == 1;
  if (tail) {
    // the level's shared tail operator (leaf down: the lift L) -> smem once per CTA (static data)
    const double* A2 = a.A2.get(0);
    const int r2p = (a.R2 + 7) & ~7;  // whole 8-row tiles (rows past R2 zero)
    for (int e = tid; e < r2p * c.ld2; e += ST_NC * 32) {
      const int r = e / c.ld2, k = e - r * c.ld2;
      a2s[e] = (r < a.R2 && k < a.K2) ? __ldg(A2 + (long long)r * a.A2.ld + k) : 0.0;
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(ST_NC * 32) : "memory");
  }
  pdl_wait();  // the epilogue adds pool rows (aidx) written by the previous step
  const int g = lane >> 2, t = lane & 3;
  const int rg = ((g & 3) << 1) | (g >> 2);
  int aoff[4];
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) {
    const int cc = k4 * 4 + t;
    aoff[k4] = rg * 16 + ((((cc >> 1) ^ rg) << 1) | (cc & 1));
  }
  const int mt = (RB + 7) >> 3;
  const int ntw = warp < mt ? (mt - warp + ST_NC - 1) / ST_NC : 0;
  const bool split = a.mode2 == 3;
  const int K2 = split ? a.K2 : 0;
  int slot = 0, xs = 0;
  unsigned ph = 0, xph = 0;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const int item = (int)(u / c.nrb), rb = (int)(u - (long long)item * c.nrb);
    double acc[2][4][NT][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[h][i][n][0] = acc[h][i][n][1] = 0.0;
    const int* oi = a.oidx + (long long)item * a.ostride;
    const int* ai = a.aidx ? a.aidx + (long long)item * a.ostride : nullptr;
    const int* o2 = split ? a.o2idx + (long long)item * a.ostride : nullptr;
    int orows[4], arows[4], wrows[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = rb * RB + (warp + i * ST_NC) * 8 + rg;
      const bool live = i < ntw && (warp + i * ST_NC) * 8 + rg < RB && r < R;
      orows[i] = live ? __ldg(oi + r) : -1;
      arows[i] = (live && ai) ? __ldg(ai + r) : -1;
      wrows[i] = (live && o2) ? __ldg(o2 + r) : -1;
    }
    for (int ch = 0; ch < nchunk; ++ch) {
      mbar_wait(xfull + xs, xph);
      const double* xc = xbuf + (size_t)xs * KX * XLD;
      const int js = ch * spc, je = min(nslab, js + spc);
      for (int j = js; j < je; ++j) {
        mbar_wait(full + slot, ph);
        const double* slab = reinterpret_cast<const double*>(base + (size_t)slot * c.sb_bytes);
        // the tile count is warp-uniform: one branch-free slab body per count (a guarded DMMA
        // would still occupy the tensor pipe)
        const int kl0 = (j - js) * 16, ksnap = split ? K2 - ch * KX : -1;
        switch (ntw) {
          case 1: stream_slab<1, NT, XLD>(acc, slab, xc, kl0, ksnap, aoff, warp, g, t, wrows, a.pool, nrhs); break;
          case 2: stream_slab<2, NT, XLD>(acc, slab, xc, kl0, ksnap, aoff, warp, g, t, wrows, a.pool, nrhs); break;
          case 3: stream_slab<3, NT, XLD>(acc, slab, xc, kl0, ksnap, aoff, warp, g, t, wrows, a.pool, nrhs); break;
          case 4: stream_slab<4, NT, XLD>(acc, slab, xc, kl0, ksnap, aoff, warp, g, t, wrows, a.pool, nrhs); break;
          default: break;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
        if (++slot == ns) {
          slot = 0;
          ph ^= 1u;
        }
      }
      if (tail && ch == nchunk - 1 && warp * 8 < a.R2) {
        // tail y2 = A2 x[K-K2, K) (leaf down: exterior rows u_ce = L u_ge) from the last x chunk;
        // one 8-row tile per warp
        const int xo = (K - a.K2) - ch * KX;
        double c2[NT][2];
#pragma unroll
        for (int n = 0; n < NT; ++n) c2[n][0] = c2[n][1] = 0.0;
        const double* arow = a2s + (size_t)(warp * 8 + g) * c.ld2;
        for (int k = 0; k < a.K2; k += 4) {
          const double av = arow[k + t];
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma_nv(c2[n][0], c2[n][1], av, xc[(xo + k + t) * XLD + n * 8 + g]);
        }
        const int ra = warp * 8 + g;
        if (ra < a.R2) {
          const long long orow = (long long)__ldg(a.o2idx + (long long)item * a.R2 + ra) * nrhs;
#pragma unroll
          for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int j = n * 8 + 2 * t + hh;
              if (j < nrhs) a.pool[orow + j] = c2[n][hh];
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(xempty + xs);
      if (++xs == c.nxb) {
        xs = 0;
        xph ^= 1u;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (orows[i] < 0) continue;
      const long long orow = (long long)orows[i] * nrhs;
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int j = n * 8 + 2 * t + hh;
          if (j < nrhs) {
            double v = acc[0][i][n][hh] + acc[1][i][n][hh];
            if (arows[i] >= 0) v += a.pool[(long long)arows[i] * nrhs + j];
            a.pool[orow + j] = v;
          }
        }
    }
  }
}

// Returns true when the step was launched on the streaming kernel.
bool launch_gemv_stream(const GemvArgs& a, cudaStream_t s) {
  static const int on = [] {
    const char* e = getenv("HPS_STREAM");
    return e ? atoi(e) : 1;
  }();
  static const long long min_bytes = [] {  // HPS_STREAM_MIN_KB: smallest item routed here
    const char* e = getenv("HPS_STREAM_MIN_KB");
    return 1024LL * (e ? atoll(e) : 48);
  }();
  if (!on || a.nrhs <= 2 || a.nrhs > 16 || a.A.ptrs || a.mode2 == 2 || a.kscale) return false;
  if (a.R < 32 || a.K < 64 || 8LL * a.R * a.K < min_bytes) return false;
  // where it measured faster than the register-streaming DMMA kernels (config 5, 16 RHS): the
  // split-output downward steps of the upper-middle levels and the split-K parts of the top
  // levels; HPS_STREAM=2 routes every eligible step here
  if (on == 1 && !((a.mode2 == 3 && a.R >= 96 && 8LL * a.R * a.K >= 512 * 1024) || (a.kparts > 1 && a.R >= 1536)))
    return false;
  if (a.mode2 == 3 && (a.K2 % 4 != 0 || a.kparts > 1)) return false;
  // mode2 = 1 (tail): a level-shared A2, at most one 8-row tile per consumer warp, K2 % 4 == 0,
  // and the tail's x columns inside the last 128-column x chunk
  if (a.mode2 == 1 && (a.A2.stride != 0 || a.A2.ptrs || a.a2idx || a.R2 > 8 * ST_NC || a.K2 % 4 != 0 ||
                       a.K2 > 128 || (a.K - a.K2) < ((a.K + 127) / 128 - 1) * 128 || a.kparts > 1))
    return false;
  static const int leaf_on = [] {  // HPS_STREAM_LEAF=1: also the leaf downward step (mode2 = 1)
    const char* e = getenv("HPS_STREAM_LEAF");
    return e ? atoi(e) : 0;
  }();
  if (a.mode2 == 1 && !leaf_on) return false;
  const int kp = a.kparts > 1 ? a.kparts : 1;
  const long long nops = a.nitems / kp;  // operator items
  if (a.A.stride != (long long)a.R * a.A.ld || (a.A.ld * 8) % 16 != 0 || (long long)kp * a.K > a.A.ld) return false;
  const double* gbase = a.A.base + a.A.off;
  if (reinterpret_cast<uintptr_t>(gbase) % 16 != 0) return false;
  if (a.nrhs % 2 == 0 && reinterpret_cast<uintptr_t>(a.pool) % 16 != 0) return false;
  auto enc = encode_fn();
  if (!enc) return false;

  StreamCfg c{};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // row blocks: equal blocks of <= 256 rows rounded up to m-tiles. Units (item x row block) are
  // dealt round-robin to one persistent CTA per SM and a 256-row unit is ~10 us of one SM's HBM
  // share, so the block count is chosen for whole waves: the fewest blocks whose unit count fills
  // >= 95 % of its last wave, else the best fill among blocks of >= 64 rows (config 5, 16 RHS:
  // 300-336 units were 2.03-2.27 waves = 68-76 % fill)
  {
    static const int balance = [] {
      const char* e = getenv("HPS_STREAM_BALANCE");
      return e ? atoi(e) : 1;
    }();
    const int nb0 = (a.R + 255) / 256;
    int best_nb = nb0;
    double best_eff = 0.0;
    const int nb_max = balance ? std::max(nb0, (a.R + 63) / 64) : nb0;
    for (int nb = nb0; nb <= nb_max; ++nb) {
      const int rb = nb == 1 ? a.R : (((a.R + nb - 1) / nb) + 7) & ~7;
      const long long u = (long long)a.nitems * ((a.R + rb - 1) / rb);
      const double eff = (double)u / ((double)sms * (double)((u + sms - 1) / sms));
      if (eff > best_eff + 0.02) {
        best_eff = eff;
        best_nb = nb;
      }
      if (eff >= 0.95) break;
    }
    c.RB = best_nb == 1 ? a.R : (((a.R + best_nb - 1) / best_nb) + 7) & ~7;
    c.nrb = (a.R + c.RB - 1) / c.RB;
  }
  c.KX = 128;
  c.sb_bytes = ((c.RB * 128 + 1023) / 1024) * 1024;
  const int nrp = a.nrhs <= 8 ? 8 : 16;
  // x chunk ring: enough buffers for the gather to run two units ahead of the consumers
  c.nxb = std::min(4, std::max(2, 2 * ((a.K + c.KX - 1) / c.KX)));
  const size_t xbytes = (size_t)c.nxb * sizeof(double) * (size_t)c.KX * (nrp + 4);
  const size_t budget = 220 * 1024;
  c.ld2 = a.mode2 == 1 ? ((a.K2 + 11) & ~15) + 4 : 0;  // == 4 mod 16: conflict-free fragments
  const size_t a2bytes = a.mode2 == 1 ? sizeof(double) * (size_t)((a.R2 + 7) & ~7) * c.ld2 : 0;
  c.ns = 8;
  while (c.ns > 2 && 1024 + (size_t)c.ns * c.sb_bytes + xbytes + 16 * (c.ns + 8) + a2bytes > budget) --c.ns;
  const size_t smem = 1024 + (size_t)c.ns * c.sb_bytes + xbytes + 16 * (size_t)(c.ns + 8) + a2bytes;
  if (smem > budget) return false;

  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)a.A.ld, (cuuint64_t)(nops * a.R)};
  const cuuint64_t strides[1] = {(cuuint64_t)a.A.ld * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)c.RB};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(gbase), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const long long units = (long long)a.nitems * c.nrb;
  const int grid = (int)(units < sms ? units : sms);
  using KFn = void (*)(const CUtensorMap, GemvArgs, StreamCfg);
  const KFn k = nrp == 16 ? gemv_stream_kernel<16> : gemv_stream_kernel<8>;
  static bool configured[2] = {};
  if (!configured[nrp == 16]) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget);
    configured[nrp == 16] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ST_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = sweep_pdl_for(a.nrhs, true) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, tm, a, c) == cudaSuccess;
}

}  // namespace hps
