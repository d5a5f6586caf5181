// Probe: do DMMA (mma.sync m8n8k4 f64) and scalar DFMA share one FP64 pipe on the B200?
// Each warp issues ND DMMAs and NF DFMAs per iteration (independent chains); prints combined TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NF>
__global__ void mixed_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2], f[16];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0.0; c[t][1] = 0.0; }
#pragma unroll
  for (int t = 0; t < 16; ++t) f[t] = t;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (t < ND)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (2 * t + u < NF) asm volatile("fma.rn.f64 %0, %1, %0, %2;\n" : "+d"(f[2 * t + u]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
#pragma unroll
  for (int t = 0; t < 16; ++t) s += f[t];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int ND, int NF>
void run(double* out, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000, grid = sms * 2, block = 512;
  mixed_loop<ND, NF><<<grid, block>>>(out, 100);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); mixed_loop<ND, NF><<<grid, block>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double warps = (double)grid * block / 32;
  const double fd = warps * iters * ND * 512.0, ff = warps * iters * NF * 64.0;
  printf("{\"probe\":\"mixed\",\"dmma_per_iter\":%d,\"dfma_per_iter\":%d,\"ms\":%.3f,\"dmma_tflops\":%.2f,\"dfma_tflops\":%.2f,\"sum\":%.2f}\n",
         ND, NF, best, fd / best / 1e9, ff / best / 1e9, (fd + ff) / best / 1e9);
}

int main() {
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 4096 * 8);
  run<8, 0>(out, sms); run<0, 16>(out, sms); run<8, 4>(out, sms); run<8, 8>(out, sms); run<8, 16>(out, sms); run<4, 16>(out, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
