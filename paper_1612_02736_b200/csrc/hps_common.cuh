// Shared device helpers for the HPS sm_100a kernels: FP64 tensor-core (DMMA) fragments,
// cp.async staging, batched-matrix descriptors.
//
// FP64 tensor work on Blackwell goes through the warp-level mma.sync f64 path: tcgen05.mma
// has no f64 kind (CUDA 12.9 tcgen05_mma.h lists f16/tf32/f8f6f4/i8/mxf*), so the
// TMEM/UMMA machinery does not apply. mma.sync.m8n8k4.f64 lowers to DMMA.8x8x4 on sm_100a
// (checked with cuobjdump) and a register-resident loop of it reaches 37.1 TFLOP/s on the
// B200 (tools/fp64_peaks.cu, profiles/fp64_peaks_r01.jsonl) — the roofline denominator.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hps {

// Batched matrix operand: either base + i*stride or an explicit device pointer array.
struct MatB {
  double* base;
  long long stride;
  double* const* ptrs;
  int ld;
  long long off;  // element offset added to every item's pointer (e.g. a column block)
  __device__ __forceinline__ double* get(int i) const {
    return (ptrs ? ptrs[i] : base + (long long)i * stride) + off;
  }
};

// D = A(8x4) * B(4x8) + D ; A row-major fragment, B column fragment.
// lane: g = lane>>2, t = lane&3 ; a = A[g][t], b = B[t][g], d0/d1 = D[g][2t], D[g][2t+1]
__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async copy global->shared; src_bytes = 0 gives a zero fill (out-of-range tile element).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// L2 prefetch of a contiguous byte range (bulk; size multiple of 16, address 16-byte aligned)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Programmatic dependent launch: let the next kernel in the stream start (and stream its
// operators into L2) while this one drains; pdl_wait() blocks until the previous grid completed
// and its writes are visible (no-op for a launch without the attribute).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hps
