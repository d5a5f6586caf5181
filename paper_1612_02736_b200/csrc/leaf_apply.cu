// Leaf collocation operator applied to tabulated leaf solutions, for implicit time stepping:
//   g[l][r] = alpha * u[l][k_r] + beta * (A u)[l][k_r]     at the interior nodes k_r (i_ci order)
//   A u = -c11 D1^2 u - 2 c12 D1 D2 u - c22 D2^2 u + c1 D1 u + c2 D2 u + c u
// (reference timestepping.py:117-167 _RhsContext.apply: the explicit side (1/k + A/2) u_n of
// Crank-Nicolson; beta = 0 gives the backward-Euler load u_n / k of config 5).
// The tensor-product derivatives are p-term dot products over the staged tabulation (D1 acts
// along x1 within a grid row, D2 along x2 within a grid column, D1 D2 u = D1 (D2 u)).
#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

// Layout: u and g keep the right-hand sides fastest (the sweep pool layout), so one CTA takes a
// leaf and a chunk of R consecutive right-hand sides and every load/store is a contiguous run of
// R doubles: the staged tiles are [P][R] with the RHS index on the lanes (conflict-free).
__global__ void leaf_apply_copy_kernel(LeafApplyArgs a, const int* __restrict__ kmap) {
  // beta == 0 (backward Euler): g[r][j] = alpha * u[k_r][j], a pure gather-scale
  const int leaf = blockIdx.x, p = a.p, pm = p - 2, m = pm * pm, nrhs = a.nrhs;
  const double* u = a.u + (long long)leaf * a.u_stride;
  double* g = a.g + (long long)leaf * a.g_stride;
  const int tot = m * nrhs;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const int r = e / nrhs, j = e - r * nrhs;
    g[e] = a.alpha * __ldg(u + (long long)kmap[r] * nrhs + j);
  }
}

__global__ void leaf_apply_kernel(LeafApplyArgs a, int R) {
  extern __shared__ double sm[];
  const int p = a.p, P = p * p, pm = p - 2, m = pm * pm;
  const int leaf = blockIdx.x, j0 = blockIdx.y * R;
  const int nrhs = a.nrhs, rc = min(R, nrhs - j0);
  double* dx = sm;          // p x p each
  double* dy = dx + p * p;
  double* dxx = dy + p * p;
  double* dyy = dxx + p * p;
  double* U = dyy + p * p;  // [P][R]
  double* V = U + P * R;    // D2 u, [P][R]
  const double* u = a.u + (long long)leaf * a.u_stride + j0;
  for (int e = threadIdx.x; e < P * rc; e += blockDim.x) {
    const int k = e / rc, jj = e - k * rc;
    U[k * R + jj] = u[(long long)k * nrhs + jj];
  }
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    dx[e] = a.dx[e];
    dy[e] = a.dy[e];
    dxx[e] = a.dxx[e];
    dyy[e] = a.dyy[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < P * rc; e += blockDim.x) {
    const int k = e / rc, jj = e - k * rc;
    const int i1 = k % p, i2 = k / p;
    double s = 0.0;
    for (int t = 0; t < p; ++t) s += dy[i2 * p + t] * U[(t * p + i1) * R + jj];
    V[k * R + jj] = s;
  }
  __syncthreads();
  double* g = a.g + (long long)leaf * a.g_stride + j0;
  const long long cs = (long long)a.nleaf * P;
  const double* cf = a.coef + (long long)leaf * P;
  for (int e = threadIdx.x; e < m * rc; e += blockDim.x) {
    const int r = e / rc, jj = e - r * rc;
    const int i1 = 1 + r % pm, i2 = 1 + r / pm, k = i1 + p * i2;
    double d1 = 0.0, d11 = 0.0, d2 = 0.0, d22 = 0.0, d12 = 0.0;
    for (int t = 0; t < p; ++t) {
      const double ur = U[(i2 * p + t) * R + jj], uc = U[(t * p + i1) * R + jj];
      d1 += dx[i1 * p + t] * ur;
      d11 += dxx[i1 * p + t] * ur;
      d2 += dy[i2 * p + t] * uc;
      d22 += dyy[i2 * p + t] * uc;
      d12 += dx[i1 * p + t] * V[(i2 * p + t) * R + jj];
    }
    const double uk = U[k * R + jj];
    double au = -(cf[k] * d11);
    au -= 2.0 * cf[cs + k] * d12;
    au -= cf[2 * cs + k] * d22;
    au += cf[3 * cs + k] * d1;
    au += cf[4 * cs + k] * d2;
    au += cf[5 * cs + k] * uk;
    g[(long long)r * nrhs + jj] = a.alpha * uk + a.beta * au;
  }
}

namespace {
// interior node k_r (i_ci order) per interior row, cached per p on the device
const int* interior_map(int p, cudaStream_t s) {
  static int* maps[129] = {};
  if (p > 128) return nullptr;
  if (!maps[p]) {
    const int pm = p - 2, m = pm * pm;
    int* h = new int[m];
    for (int r = 0; r < m; ++r) h[r] = (1 + r % pm) + p * (1 + r / pm);
    int* d = nullptr;
    if (cudaMalloc(&d, sizeof(int) * m) != cudaSuccess) { delete[] h; return nullptr; }
    cudaMemcpyAsync(d, h, sizeof(int) * m, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    delete[] h;
    maps[p] = d;
  }
  return maps[p];
}
}  // namespace

int launch_leaf_apply(const LeafApplyArgs& a, cudaStream_t s) {
  if (a.nleaf <= 0) return 0;
  if (a.beta != 0.0 && !a.coef) return 1;
  const int P = a.p * a.p;
  if (a.beta == 0.0) {
    const int* kmap = interior_map(a.p, s);
    if (!kmap) return 2;
    for (int off = 0; off < a.nleaf; off += 1 << 30) {
      LeafApplyArgs b = a;
      const int nb = min(1 << 30, a.nleaf - off);
      b.u = a.u + (long long)off * a.u_stride;
      b.g = a.g + (long long)off * a.g_stride;
      leaf_apply_copy_kernel<<<nb, 256, 0, s>>>(b, kmap);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  // RHS chunk: as many as fit in ~96 KB of staged tiles
  int R = a.nrhs;
  while (R > 1 && sizeof(double) * (4 * P + 2 * (size_t)P * R) > 96 * 1024) R = (R + 1) / 2;
  const size_t smem = sizeof(double) * (4 * P + 2 * (size_t)P * R);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(leaf_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = P * R < 512 ? 256 : 512;
  const int chunks = (a.nrhs + R - 1) / R;
  for (int off = 0; off < a.nleaf; off += 1 << 30) {
    LeafApplyArgs b = a;
    const int nb = min(1 << 30, a.nleaf - off);
    b.u = a.u + (long long)off * a.u_stride;
    b.g = a.g + (long long)off * a.g_stride;
    if (a.coef) b.coef = a.coef + (long long)off * P;  // coefficient stride stays nleaf*P
    dim3 grid(nb, chunks);
    leaf_apply_kernel<<<grid, threads, smem, s>>>(b, R);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
