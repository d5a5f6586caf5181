// FP64 peak probes for the roofline denominators (MEASURED_PEAKS.json has no FP64 entry).
//   dmma : mma.sync.m8n8k4 f64 (DMMA) register-resident loop, all SMs
//   dfma : scalar FP64 FMA register-resident loop, all SMs
// Reported as TFLOP/s with CUDA events, best of several runs; SM clock sampled by the caller.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0.0; c[t][1] = 0.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) c[t] = t;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = fma(a, c[t], b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += c[t];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int sms = prop.multiProcessorCount;
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int iters = 4000;
      int grid = sms * bps, block = 32 * wpb;
      dmma_loop<<<grid, block>>>(out, 100);
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); dmma_loop<<<grid, block>>>(out, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = (double)grid * (block / 32) * iters * 8 * 512.0;
      printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_block\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n",
             wpb, bps, flops / best / 1e9, best);
    }
  }
  for (int wpb : {8, 16, 32}) {
    int iters = 4000, grid = sms * 2, block = 32 * wpb;
    dfma_loop<<<grid, block>>>(out, 100);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_loop<<<grid, block>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = (double)grid * block * iters * 16 * 2.0;
    printf("{\"probe\":\"dfma\",\"warps_per_block\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n", wpb, flops / best / 1e9, best);
  }
  size_t n = (size_t)1 << 27;  // 2 GiB per buffer as double2
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMemset(a, 0, n * 16);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0); copy_kernel<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < best) best = ms;
  }
  printf("{\"probe\":\"copy_f64x2\",\"gbs\":%.1f}\n", 2.0 * n * 16 / best / 1e6);
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, prop.clockRate);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
