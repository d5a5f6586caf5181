// Microbenchmark: latency of cluster barriers and DSMEM reads on the B200 (8-CTA clusters).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_lat tools/cluster_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(8, 1, 1) k_sync(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slot[64];
  if (threadIdx.x < 64) slot[threadIdx.x] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 8) {
      const double* r = cl.map_shared_rank(slot, threadIdx.x);
      acc += r[i & 63];
    }
    __syncthreads();
  }
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 8) {
      const double* r = cl.map_shared_rank(slot, threadIdx.x);
      acc += r[i & 63];
    }
    cl.sync();
  }
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t4 = clock64();
  // barrier.cluster.arrive.relaxed + wait
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  long long t5 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = (t2 - t1) / iters;
    out[2] = (t3 - t2) / iters;
    out[3] = (t4 - t3) / iters;
    out[4] = (t5 - t4) / iters;
    out[5] = (long long)acc;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  k_sync<<<8, 256>>>(10, d);
  cudaDeviceSynchronize();
  k_sync<<<8, 256>>>(2000, d);
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per: cluster.sync %lld | dsmem read + syncthreads %lld | dsmem read + cluster.sync %lld | "
         "syncthreads %lld | relaxed arrive+wait %lld\n", h[0], h[1], h[2], h[3], h[4]);
  k_sync<<<8 * 148 / 8, 256>>>(2000, d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("(148 CTAs) cluster.sync %lld | dsmem+sync %lld | dsmem+cluster %lld | syncthreads %lld | relaxed %lld\n",
         h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
