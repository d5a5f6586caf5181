// Column step with NM independent matrices per thread (interleaved chains, one barrier per column):
// does instruction-level interleaving hide the serial stages? (see colstep_bench.cu)
#include <cstdio>
#include <cuda_runtime.h>
constexpr int KB = 28;

template <int NM, int NT>
__global__ void __launch_bounds__(NT, 1) colstep(double* out, int* piv, int ncol, long long* cycles) {
  __shared__ double slots[2][NM][NT / 32][KB + 2];
  __shared__ double dispb[2][NM][KB];
  __shared__ unsigned long long skey[2][NM][NT / 32];
  __shared__ int sidx[2][NM][NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = NT - 28, i = tid;
  double row[NM][KB];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int t = 0; t < KB; ++t) row[m][t] = 1.0 + 1e-3 * ((tid * 37 + t * 11 + m * 5) % 101) + (t == (tid % KB) ? 3.0 : 0.0);
  __syncthreads();
  const long long t0 = clock64();
  for (int c0 = 0; c0 < ncol; c0 += KB) {
#pragma unroll 1
    for (int jb = 0; jb < KB; jb += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = jb + q, cj = (c0 + j) % n;
        unsigned long long key[NM];
        int bi[NM];
        double rinv[NM];
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          const double av = fabs(row[m][q]);
          const bool ok = i < n && i >= cj;
          key[m] = ok ? (unsigned long long)__double_as_longlong(av) : 0ull;
          bi[m] = ok ? i : n;
          rinv[m] = 1.0 / row[m][q];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int m = 0; m < NM; ++m) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key[m], o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi[m], o);
            if (ok > key[m] || (ok == key[m] && oi < bi[m])) { key[m] = ok; bi[m] = oi; }
          }
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          double* my = &slots[j & 1][m][warp][0];
          if (lane == 0) {
            skey[j & 1][m][warp] = key[m];
            sidx[j & 1][m][warp] = bi[m];
          }
          if (i == bi[m]) {
#pragma unroll
            for (int t = 0; t < KB; t += 2)
              *reinterpret_cast<double2*>(my + 2 + t) =
                  make_double2((t == q) ? rinv[m] : row[m][t] * rinv[m], (t + 1 == q) ? rinv[m] : row[m][t + 1] * rinv[m]);
          }
          if (i == cj) {
#pragma unroll
            for (int t = 0; t < KB; t += 2) *reinterpret_cast<double2*>(&dispb[j & 1][m][t]) = make_double2(row[m][t], row[m][t + 1]);
          }
        }
        __syncthreads();
        int pr[NM], ws[NM];
        unsigned long long kb[NM];
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          kb[m] = 0ull;
          pr[m] = n;
          ws[m] = lane;
          if (lane < NT / 32) {
            kb[m] = skey[j & 1][m][lane];
            pr[m] = sidx[j & 1][m][lane];
          }
        }
#pragma unroll
        for (int o = NT / 64; o > 0; o >>= 1)
#pragma unroll
          for (int m = 0; m < NM; ++m) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, kb[m], o);
            const int oi = __shfl_xor_sync(0xffffffffu, pr[m], o);
            const int ow = __shfl_xor_sync(0xffffffffu, ws[m], o);
            if (ok > kb[m] || (ok == kb[m] && oi < pr[m])) { kb[m] = ok; pr[m] = oi; ws[m] = ow; }
          }
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          pr[m] = __shfl_sync(0xffffffffu, pr[m], 0);
          ws[m] = __shfl_sync(0xffffffffu, ws[m], 0);
          if (pr[m] >= n) pr[m] = cj;
          if (tid == 0) piv[m * 4096 + cj] = pr[m];
          const double* pvr = &slots[j & 1][m][ws[m]][2];
          const double* disp = dispb[j & 1][m];
          if (i == pr[m] && pr[m] != cj) {
#pragma unroll
            for (int t = 0; t < KB; ++t) row[m][t] = disp[t];
          }
          if (i == cj) {
#pragma unroll
            for (int t = 0; t < KB; ++t) row[m][t] = pvr[t];
          } else {
            const double f = row[m][q];
#pragma unroll
            for (int t = 0; t < KB; t += 2) {
              const double2 pv = *reinterpret_cast<const double2*>(pvr + t);
              row[m][t] = ((t == q) ? 0.0 : row[m][t]) - f * pv.x;
              row[m][t + 1] = ((t + 1 == q) ? 0.0 : row[m][t + 1]) - f * pv.y;
            }
          }
        }
      }
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        double t0r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) t0r[u] = row[m][u];
#pragma unroll
        for (int t = 0; t < KB - 4; ++t) row[m][t] = row[m][t + 4];
#pragma unroll
        for (int u = 0; u < 4; ++u) row[m][KB - 4 + u] = t0r[u];
      }
    }
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int t = 0; t < KB; ++t) row[m][t] = 1.0 + 1e-3 * ((tid * 37 + t * 11 + c0 + m) % 101) + (t == (tid % KB) ? 3.0 : 0.0);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int t = 0; t < KB; ++t) s += row[m][t];
  out[blockIdx.x * NT + tid] = s;
  if (blockIdx.x == 0 && tid == 0) cycles[0] = t1 - t0;
}

template <int NM, int NT>
void run(double* out, int* piv, long long* cyc) {
  const int ncol = 28 * 70;
  colstep<NM, NT><<<148, NT>>>(out, piv, ncol, cyc);
  colstep<NM, NT><<<148, NT>>>(out, piv, ncol, cyc);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("NM=%d NT=%d: %8.0f cycles / column step (%.0f per matrix-column)  (%s)\n", NM, NT, (double)h / ncol,
         (double)h / ncol / NM, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out;
  int* piv;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 8);
  cudaMalloc(&piv, 4 * 4096 * 4);
  cudaMalloc(&cyc, 8);
  run<1, 256>(out, piv, cyc);
  run<2, 256>(out, piv, cyc);
  run<3, 256>(out, piv, cyc);
  run<1, 224>(out, piv, cyc);
  run<2, 224>(out, piv, cyc);
  return 0;
}
