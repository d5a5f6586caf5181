// Microbenchmark: HBM streaming rate of the 16-RHS leaf-down operator pattern through TMA,
// no math (consumers only release the stages). Operator = 16384 items x 196 rows x 256 cols FP64
// (config 5 [F|S], 6.58 GB).
//   layout 0: row-major [item][row][256]; box {16 cols, R rows} = 196 chunks of 128 B, 2 KB apart
//             (what gemv_tma_kernel streams today)
//   layout 1: slab-major [item][slab][row][16]; the same box is one contiguous 25 KB run
//   layout 2: row-major, 3D view {16, 4 slabs, R rows}: 512 B contiguous per row
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_stream tools/tma_stream.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
          sa(b)),
      "r"(ph)
      : "memory");
}

// per item: nbox boxes; box b of item i at coords given by the layout
__global__ void __launch_bounds__(288, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int layout, int nitems,
                                                         int R, int nbox, int box_bytes, int tx_bytes, int ns,
                                                         double* sink) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + (size_t)ns * box_bytes);
  uint64_t* empty = full + ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      int slot = 0;
      unsigned ph = 0;
      bool first = true;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x)
        for (int b = 0; b < nbox; ++b) {
          if (!first) mbar_wait(empty + slot, ph ^ 1u);
          mbar_expect_tx(full + slot, tx_bytes);
          void* dst = base + (size_t)slot * box_bytes;
          if (layout == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                    sa(dst)),
                "l"(&tm), "r"(b * 16), "r"(item * R), "r"(sa(full + slot))
                : "memory");
          } else if (layout == 1) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                    sa(dst)),
                "l"(&tm), "r"(0), "r"((item * nbox + b) * R), "r"(sa(full + slot))
                : "memory");
          } else {
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
                    sa(dst)),
                "l"(&tm), "r"(0), "r"((b & 3) * 4), "r"(item * R + (b >> 2) * (R / 4)), "r"(sa(full + slot))
                : "memory");
          }
          if (++slot == ns) {
            slot = 0;
            ph ^= 1u;
            first = false;
          }
        }
    }
    return;
  }
  int slot = 0;
  unsigned ph = 0;
  double acc = 0.0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x)
    for (int b = 0; b < nbox; ++b) {
      mbar_wait(full + slot, ph);
      acc += ((double*)(base + (size_t)slot * box_bytes))[threadIdx.x];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if (++slot == ns) {
        slot = 0;
        ph ^= 1u;
      }
    }
  if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int nitems = 16384, R = 196, K = 256;
  const size_t n = (size_t)nitems * R * K;
  double* d;
  cudaMalloc(&d, n * 8);
  cudaMemset(d, 0, n * 8);
  double* sink;
  cudaMalloc(&sink, 8);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int layout = 0; layout < 3; ++layout) {
    for (int ns : {3, 5, 8}) {
      CUtensorMap tm;
      int nbox, box_bytes;
      if (layout == 0) {
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)nitems * R};
        cuuint64_t str[1] = {(cuuint64_t)K * 8};
        cuuint32_t box[2] = {16, (cuuint32_t)R};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        nbox = K / 16;
        box_bytes = ((R * 128 + 1023) / 1024) * 1024;
      } else if (layout == 1) {
        cuuint64_t dims[2] = {16, (cuuint64_t)nitems * R * (K / 16)};
        cuuint64_t str[1] = {16 * 8};
        cuuint32_t box[2] = {16, (cuuint32_t)R};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        nbox = K / 16;
        box_bytes = ((R * 128 + 1023) / 1024) * 1024;
      } else {
        cuuint64_t dims[3] = {16, (cuuint64_t)K / 16, (cuuint64_t)nitems * R};
        cuuint64_t str[2] = {16 * 8, (cuuint64_t)K * 8};
        cuuint32_t box[3] = {16, 4, (cuuint32_t)R / 4};
        cuuint32_t es[3] = {1, 1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        // R/4 rows x 4 slabs per box; 4 row-quarters x 4 slab-groups per item
        nbox = 16;
        box_bytes = ((R / 4 * 4 * 128 + 1023) / 1024) * 1024;
      }
      size_t smem = 1024 + (size_t)ns * box_bytes + 16 * ns;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      // layout 2 box coords: rows item*R + quarter*(R/4) handled by treating each box as 1/16 of item
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        const int tx = layout == 2 ? (R / 4) * 4 * 128 : R * 128;  // bytes one box delivers
        stream_kernel<<<sms, 288, smem>>>(tm, layout, nitems, R, nbox, box_bytes, tx, ns, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      printf("layout %d ns %d box %d B: %.3f ms  %.1f GB/s  %s\n", layout, ns, box_bytes, ms, n * 8 / ms / 1e6,
             cudaGetErrorString(err));
    }
  }
  return 0;
}
