// Leaf collocation operator applied to tabulated leaf solutions, for implicit time stepping:
//   g[l][r] = alpha * u[l][k_r] + beta * (A u)[l][k_r]     at the interior nodes k_r (i_ci order)
//   A u = -c11 D1^2 u - 2 c12 D1 D2 u - c22 D2^2 u + c1 D1 u + c2 D2 u + c u
// (reference timestepping.py:117-167 _RhsContext.apply: the explicit side (1/k + A/2) u_n of
// Crank-Nicolson; beta = 0 gives the backward-Euler load u_n / k of config 5).
// One CTA per (leaf, rhs): the p x p tabulation and D2 u are staged in shared memory, the
// tensor-product derivatives are p-term dot products (D1 acts along x1 within a grid row,
// D2 along x2 within a grid column, D1 D2 u = D1 (D2 u)).
#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

__global__ void leaf_apply_kernel(LeafApplyArgs a) {
  extern __shared__ double sm[];
  const int p = a.p, P = p * p, pm = p - 2, m = pm * pm;
  const int leaf = blockIdx.x, j = blockIdx.y;  // j: right-hand side
  const int nrhs = a.nrhs;
  double* U = sm;           // P
  double* V = U + P;        // D2 u (P)
  double* dx = V + P;       // p x p each
  double* dy = dx + p * p;
  double* dxx = dy + p * p;
  double* dyy = dxx + p * p;
  const double* u = a.u + (long long)leaf * a.u_stride;
  for (int e = threadIdx.x; e < P; e += blockDim.x) U[e] = u[(long long)e * nrhs + j];
  const bool op = a.beta != 0.0;
  if (op) {
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      dx[e] = a.dx[e];
      dy[e] = a.dy[e];
      dxx[e] = a.dxx[e];
      dyy[e] = a.dyy[e];
    }
  }
  __syncthreads();
  if (op) {
    for (int e = threadIdx.x; e < P; e += blockDim.x) {
      const int i1 = e % p, i2 = e / p;
      double s = 0.0;
      for (int t = 0; t < p; ++t) s += dy[i2 * p + t] * U[t * p + i1];
      V[e] = s;
    }
    __syncthreads();
  }
  double* g = a.g + (long long)leaf * a.g_stride;
  const long long cs = (long long)a.nleaf * P;
  const double* cf = a.coef ? a.coef + (long long)leaf * P : nullptr;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    const int i1 = 1 + r % pm, i2 = 1 + r / pm, k = i1 + p * i2;
    double out = a.alpha * U[k];
    if (op) {
      double d1 = 0.0, d11 = 0.0, d2 = 0.0, d22 = 0.0, d12 = 0.0;
      for (int t = 0; t < p; ++t) {
        const double ur = U[i2 * p + t], uc = U[t * p + i1];
        d1 += dx[i1 * p + t] * ur;
        d11 += dxx[i1 * p + t] * ur;
        d2 += dy[i2 * p + t] * uc;
        d22 += dyy[i2 * p + t] * uc;
        d12 += dx[i1 * p + t] * V[i2 * p + t];
      }
      double au = -(cf[k] * d11);
      au -= 2.0 * cf[cs + k] * d12;
      au -= cf[2 * cs + k] * d22;
      au += cf[3 * cs + k] * d1;
      au += cf[4 * cs + k] * d2;
      au += cf[5 * cs + k] * U[k];
      out += a.beta * au;
    }
    g[(long long)r * nrhs + j] = out;
  }
}

int launch_leaf_apply(const LeafApplyArgs& a, cudaStream_t s) {
  if (a.nleaf <= 0) return 0;
  if (a.beta != 0.0 && !a.coef) return 1;
  const size_t smem = sizeof(double) * (2 * a.p * a.p + 4 * a.p * a.p);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(leaf_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int threads = a.p * a.p < 256 ? 256 : (a.p * a.p < 1024 ? 512 : 1024);
  for (int off = 0; off < a.nleaf; off += 65535) {
    LeafApplyArgs b = a;
    const int nb = min(65535, a.nleaf - off);
    b.u = a.u + (long long)off * a.u_stride;
    b.g = a.g + (long long)off * a.g_stride;
    if (a.coef) b.coef = a.coef + (long long)off * a.p * a.p;  // coefficient stride stays nleaf*P
    b.nleaf = a.nleaf;
    dim3 grid(nb, a.nrhs);
    leaf_apply_kernel<<<grid, threads, smem, s>>>(b);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
