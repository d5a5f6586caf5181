// Microbenchmark of ONE pivot-column step of the register-resident Gauss-Jordan panel loop
// (gj_fused_kernel / gj_la_kernel): where do its ~3000 cycles go? One CTA per SM, NT threads, one
// matrix row per thread (KB panel columns in registers). Each variant switches one piece off.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/colstep_bench tools/colstep_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int KB = 28;

enum : unsigned {
  F_REDUCE1 = 1,   // warp shuffle arg-max
  F_PUBLISH = 2,   // candidate row + displaced row to shared memory (predicated stores)
  F_BARRIER = 4,   // __syncthreads
  F_REDUCE2 = 8,   // cross-warp arg-max from the slots
  F_DIVIDE = 16,   // 1 / pivot
  F_ELIM = 32,     // row update (KB x (LDS + DMUL + DFMA))
  F_ROTATE = 64,   // 4-column register rotation
  F_T0 = 128,      // thread 0: pivot bookkeeping (global store + rowid swap)
  F_UNIFORM = 256, // publication behind warp-uniform branches
  F_PRESCALE = 512, // winner publishes the scaled row; elimination is LDS + DFMA only
  F_INTKEY = 1024,  // arg-max on the bit pattern of |v| (integer compares), indices kept as ints
  F_VEC = 2048,     // 16-byte shared stores / loads for the published rows
  F_UELIM = 4096    // elimination: warps without a special row run a bare update
};

template <unsigned F, int NT>
__global__ void __launch_bounds__(NT, 1) colstep(double* out, int* piv, int ncol, long long* cycles) {
  __shared__ double slots[2][NT / 32][KB + 2];
  __shared__ double dispb[2][KB];
  __shared__ int rowid[NT];
  __shared__ unsigned long long skey[2][NT / 32];
  __shared__ int sidx[2][NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = NT - 28, i = tid;
  double row[KB];
#pragma unroll
  for (int t = 0; t < KB; ++t) row[t] = 1.0 + 1e-3 * ((tid * 37 + t * 11) % 101) + (t == (tid % KB) ? 3.0 : 0.0);
  rowid[tid] = tid;
  __syncthreads();
  const long long t0 = clock64();
  for (int c0 = 0; c0 < ncol; c0 += KB) {
#pragma unroll 1
    for (int jb = 0; jb < KB; jb += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = jb + q, cj = (c0 + j) % n;
        double* sl = &slots[j & 1][0][0];
        double* disp = dispb[j & 1];
        double best = -1.0;
        int bi = n;
        if (i < n && i >= cj) {
          best = fabs(row[q]);
          bi = i;
        }
        unsigned long long key = (bi < n) ? (unsigned long long)__double_as_longlong(best) : 0ull;
        if ((F & F_REDUCE1) && (F & F_INTKEY)) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ok > key || (ok == key && oi < bi)) { key = ok; bi = oi; }
          }
        } else if (F & F_REDUCE1) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
          }
        } else {
          bi = cj;  // diagonal
        }
        double* my = sl + warp * (KB + 2);
        double rinv = 1.0;
        if (F & F_PRESCALE) rinv = 1.0 / row[q];
        if (lane == 0) {
          if (F & F_INTKEY) {
            skey[j & 1][warp] = key;
            sidx[j & 1][warp] = bi;
          } else {
            my[0] = best;
            my[1] = (double)bi;
          }
        }
        if (F & F_PUBLISH) {
          if (F & F_UNIFORM) {
            if (__any_sync(0xffffffffu, i == bi)) {
              if (i == bi) {
#pragma unroll
                for (int t = 0; t < KB; t += 2) {
                  const double v0 = (F & F_PRESCALE) ? ((t == q) ? rinv : row[t] * rinv) : row[t];
                  const double v1 = (F & F_PRESCALE) ? ((t + 1 == q) ? rinv : row[t + 1] * rinv) : row[t + 1];
                  if (F & F_VEC) {
                    *reinterpret_cast<double2*>(my + 2 + t) = make_double2(v0, v1);
                  } else {
                    my[2 + t] = v0;
                    my[3 + t] = v1;
                  }
                }
              }
            }
            if ((cj >> 5) == warp) {
              if (i == cj) {
#pragma unroll
                for (int t = 0; t < KB; t += 2) {
                  if (F & F_VEC) {
                    *reinterpret_cast<double2*>(disp + t) = make_double2(row[t], row[t + 1]);
                  } else {
                    disp[t] = row[t];
                    disp[t + 1] = row[t + 1];
                  }
                }
              }
            }
          } else {
            if (i == bi) {
#pragma unroll
              for (int t = 0; t < KB; t += 2) {
                const double v0 = (F & F_PRESCALE) ? ((t == q) ? rinv : row[t] * rinv) : row[t];
                const double v1 = (F & F_PRESCALE) ? ((t + 1 == q) ? rinv : row[t + 1] * rinv) : row[t + 1];
                if (F & F_VEC) {
                  *reinterpret_cast<double2*>(my + 2 + t) = make_double2(v0, v1);
                } else {
                  my[2 + t] = v0;
                  my[3 + t] = v1;
                }
              }
            }
            if (i == cj) {
#pragma unroll
              for (int t = 0; t < KB; t += 2) {
                if (F & F_VEC) {
                  *reinterpret_cast<double2*>(disp + t) = make_double2(row[t], row[t + 1]);
                } else {
                  disp[t] = row[t];
                  disp[t + 1] = row[t + 1];
                }
              }
            }
          }
        }
        if (F & F_BARRIER) __syncthreads();
        double b = -2.0;
        int pr = cj, ws = (cj >> 5);
        if ((F & F_REDUCE2) && (F & F_INTKEY)) {
          unsigned long long kb = 0ull;
          pr = n;
          ws = lane;
          if (lane < NT / 32) {
            kb = skey[j & 1][lane];
            pr = sidx[j & 1][lane];
          }
#pragma unroll
          for (int o = NT / 64; o > 0; o >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, kb, o);
            const int oi = __shfl_xor_sync(0xffffffffu, pr, o);
            const int ow = __shfl_xor_sync(0xffffffffu, ws, o);
            if (ok > kb || (ok == kb && oi < pr)) { kb = ok; pr = oi; ws = ow; }
          }
          pr = __shfl_sync(0xffffffffu, pr, 0);
          ws = __shfl_sync(0xffffffffu, ws, 0);
          if (pr >= n) pr = cj;
        } else if (F & F_REDUCE2) {
          pr = n;
          ws = lane;
          if (lane < NT / 32) {
            b = sl[lane * (KB + 2)];
            pr = (int)sl[lane * (KB + 2) + 1];
          }
#pragma unroll
          for (int o = NT / 64; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, b, o);
            const int oi = __shfl_xor_sync(0xffffffffu, pr, o);
            const int ow = __shfl_xor_sync(0xffffffffu, ws, o);
            if (ov > b || (ov == b && oi < pr)) { b = ov; pr = oi; ws = ow; }
          }
          b = __shfl_sync(0xffffffffu, b, 0);
          pr = __shfl_sync(0xffffffffu, pr, 0);
          ws = __shfl_sync(0xffffffffu, ws, 0);
          if (pr >= n) pr = cj;
        }
        const double* pvr = sl + ws * (KB + 2) + 2;
        if ((F & F_T0) && tid == 0) {
          piv[cj] = pr;
          const int tr = rowid[cj];
          rowid[cj] = rowid[pr];
          rowid[pr] = tr;
        }
        double inv = 0.5;
        if ((F & F_DIVIDE) && !(F & F_PRESCALE)) inv = 1.0 / pvr[q];
        if ((F & F_ELIM) && (F & F_UELIM) && (cj >> 5) != warp && ((pr >> 5) != warp || pr == cj)) {
          // no special row in this warp: bare update
          const double f = row[q];
          if (F & F_PRESCALE) {
#pragma unroll
            for (int t = 0; t < KB; ++t) row[t] = ((t == q) ? 0.0 : row[t]) - f * pvr[t];
          } else {
#pragma unroll
            for (int t = 0; t < KB; ++t) row[t] = ((t == q) ? 0.0 : row[t]) - f * ((t == q) ? inv : pvr[t] * inv);
          }
        } else if (F & F_ELIM) {
          if (i == pr && pr != cj) {
#pragma unroll
            for (int t = 0; t < KB; ++t) row[t] = disp[t];
          }
          if (F & F_PRESCALE) {
            if (i == cj) {
#pragma unroll
              for (int t = 0; t < KB; ++t) row[t] = pvr[t];
            } else if (F & F_VEC) {
              const double f = row[q];
#pragma unroll
              for (int t = 0; t < KB; t += 2) {
                const double2 pv = *reinterpret_cast<const double2*>(pvr + t);
                row[t] = ((t == q) ? 0.0 : row[t]) - f * pv.x;
                row[t + 1] = ((t + 1 == q) ? 0.0 : row[t + 1]) - f * pv.y;
              }
            } else {
              const double f = row[q];
#pragma unroll
              for (int t = 0; t < KB; ++t) row[t] = ((t == q) ? 0.0 : row[t]) - f * pvr[t];
            }
          } else {
            if (i == cj) {
#pragma unroll
              for (int t = 0; t < KB; ++t) row[t] = (t == q) ? inv : pvr[t] * inv;
            } else {
              const double f = row[q];
#pragma unroll
              for (int t = 0; t < KB; ++t)
                row[t] = ((t == q) ? 0.0 : row[t]) - f * ((t == q) ? inv : pvr[t] * inv);
            }
          }
        } else {
          row[q] += inv * 1e-9;
        }
      }
      if (F & F_ROTATE) {
        double t0r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) t0r[u] = row[u];
#pragma unroll
        for (int t = 0; t < KB - 4; ++t) row[t] = row[t + 4];
#pragma unroll
        for (int u = 0; u < 4; ++u) row[KB - 4 + u] = t0r[u];
      }
    }
    // keep the numbers tame between panels
#pragma unroll
    for (int t = 0; t < KB; ++t) row[t] = 1.0 + 1e-3 * ((tid * 37 + t * 11 + c0) % 101) + (t == (tid % KB) ? 3.0 : 0.0);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < KB; ++t) s += row[t];
  out[blockIdx.x * NT + tid] = s;
  if (blockIdx.x == 0 && tid == 0) cycles[0] = t1 - t0;
}

template <unsigned F, int NT>
void run(const char* name, double* out, int* piv, long long* cyc) {
  const int ncol = 28 * 70;
  colstep<F, NT><<<148, NT>>>(out, piv, ncol, cyc);
  colstep<F, NT><<<148, NT>>>(out, piv, ncol, cyc);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-34s NT=%d  %8.0f cycles / column   (%s)\n", name, NT, (double)h / ncol, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out;
  int* piv;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 8);
  cudaMalloc(&piv, 4096 * 4);
  cudaMalloc(&cyc, 8);
  constexpr unsigned ALL = F_REDUCE1 | F_PUBLISH | F_BARRIER | F_REDUCE2 | F_DIVIDE | F_ELIM | F_ROTATE | F_T0;
  run<ALL, 256>("all (gj_fused form)", out, piv, cyc);
  run<ALL & ~F_REDUCE1, 256>("- warp reduce", out, piv, cyc);
  run<ALL & ~F_PUBLISH, 256>("- publish", out, piv, cyc);
  run<ALL & ~F_BARRIER, 256>("- barrier", out, piv, cyc);
  run<ALL & ~F_REDUCE2, 256>("- cross-warp reduce", out, piv, cyc);
  run<ALL & ~F_DIVIDE, 256>("- divide", out, piv, cyc);
  run<ALL & ~F_ELIM, 256>("- eliminate", out, piv, cyc);
  run<ALL & ~F_ROTATE, 256>("- rotate", out, piv, cyc);
  run<ALL & ~F_T0, 256>("- thread-0 bookkeeping", out, piv, cyc);
  run<ALL | F_UNIFORM, 256>("+ uniform publish", out, piv, cyc);
  run<ALL | F_PRESCALE, 256>("+ prescale", out, piv, cyc);
  run<ALL | F_PRESCALE | F_UNIFORM, 256>("+ prescale + uniform", out, piv, cyc);
  run<ALL | F_INTKEY, 256>("+ intkey", out, piv, cyc);
  run<ALL | F_VEC, 256>("+ vec publish", out, piv, cyc);
  run<ALL | F_PRESCALE | F_VEC, 256>("+ prescale + vec", out, piv, cyc);
  run<ALL | F_PRESCALE | F_VEC | F_INTKEY, 256>("+ prescale + vec + intkey", out, piv, cyc);
  run<ALL | F_PRESCALE | F_VEC | F_INTKEY | F_UNIFORM, 256>("+ prescale + vec + intkey + unif", out, piv, cyc);
  run<ALL | F_UELIM, 256>("+ uniform elimination", out, piv, cyc);
  run<ALL | F_UELIM | F_UNIFORM, 256>("+ uniform elim + publish", out, piv, cyc);
  run<ALL | F_UELIM | F_UNIFORM | F_PRESCALE | F_INTKEY, 256>("+ uelim + upub + prescale + intkey", out, piv, cyc);
  run<F_BARRIER, 256>("barrier only", out, piv, cyc);
  run<F_BARRIER | F_ELIM | F_DIVIDE, 256>("barrier + divide + eliminate", out, piv, cyc);
  run<F_REDUCE1 | F_BARRIER | F_REDUCE2, 256>("reduces + barrier", out, piv, cyc);
  run<ALL, 224>("all, 7 warps", out, piv, cyc);
  run<ALL, 128>("all, 4 warps", out, piv, cyc);
  return 0;
}
