// Leaf-stage assembly and merge-stage gather kernels (bandwidth-bound producers feeding the
// DMMA Gauss-Jordan and GEMM kernels).
#include "hps_common.cuh"
#include "hps_kernels.cuh"

namespace hps {

// Interior rows of the collocation matrix (reference model.py:153-177, leaf.py:96-101):
//   A = -c11 D1^2 - 2 c12 D1 D2 - c22 D2^2 + c1 D1 + c2 D2 + diag(c)
// with D1 = kron(I, dx), D2 = kron(dy, I) rebuilt from the 1D operators (no P x P constants
// are read): for rows k=(i1,i2), columns j=(j1,j2)
//   D1^2 = [i2==j2] dxx[i1,j1], D1 D2 = dx[i1,j1] dy[i2,j2], D2^2 = [i1==j1] dyy[i2,j2],
//   D1 = [i2==j2] dx[i1,j1],    D2 = [i1==j1] dy[i2,j2].
// The accumulation order matches the reference term by term. A_ii goes to the first m
// columns of the GJ workspace row, A_ie to its own buffer (multiplied by the lift next).
// rows per CTA: the four p x p 1D operators staged in shared memory are amortised over ASM_ROWS
// rows of output (8 rows read 32 KB of constants per 64 KB written at p = 32)
constexpr int ASM_ROWS = 32;

__global__ void __launch_bounds__(256) leaf_assemble_kernel(LeafAsmArgs a, int batch_off) {
  extern __shared__ double sd[];
  const int p = a.p, P = p * p, pm = p - 2;
  const int m = pm * pm;
  double* dx = sd;
  double* dy = dx + p * p;
  double* dxx = dy + p * p;
  double* dyy = dxx + p * p;
  double* cr = dyy + p * p;  // [ASM_ROWS][6] coefficient samples at this CTA's row points
  int* ipos = reinterpret_cast<int*>(cr + 6 * ASM_ROWS);  // [P] position in i_ci, else -(1 + pos in i_ce)
  const int leaf = blockIdx.y + batch_off;
  const long long cstride = (long long)a.nleaf * P;
  const double* cf = a.coef + (long long)leaf * P;
  const int r0 = blockIdx.x * ASM_ROWS;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    dx[e] = a.dx[e];
    dy[e] = a.dy[e];
    dxx[e] = a.dxx[e];
    dyy[e] = a.dyy[e];
  }
  for (int j = threadIdx.x; j < P; j += blockDim.x) {
    const int ip = a.int_pos[j];
    ipos[j] = ip >= 0 ? ip : -1 - a.ext_pos[j];
  }
  // all rows' coefficients staged up front: no dependent global loads inside the row loop
  for (int e = threadIdx.x; e < ASM_ROWS * 6; e += blockDim.x) {
    const int rr = e / 6, t = e - rr * 6, r = r0 + rr;
    if (r < m) cr[e] = cf[t * cstride + (1 + r % pm) + p * (1 + r / pm)];
  }
  __syncthreads();
  double* aii = a.Aii.get(leaf);
  double* aie = a.Aie.get(leaf);
  // |A_ii|_1 on the fly: each thread keeps the |.| sums of its own columns over this CTA's rows
  // (columns of a thread: j = threadIdx.x + t*blockDim.x, t < ASM_COLS)
  constexpr int ASM_COLS = 8;
  double csum[ASM_COLS];
#pragma unroll
  for (int t = 0; t < ASM_COLS; ++t) csum[t] = 0.0;
  for (int r = r0; r < min(m, r0 + ASM_ROWS); ++r) {
    const int i1 = 1 + r % pm, i2 = 1 + r / pm;
    const int k = i1 + p * i2;
    const double* c6 = cr + (r - r0) * 6;
    const double c11 = c6[0], c12 = c6[1], c22 = c6[2], c1 = c6[3], c2 = c6[4], c0 = c6[5];
    auto elem = [&](int j1, int j2) {
      const int j = j1 + p * j2;
      const double d11 = (i2 == j2) ? dxx[i1 * p + j1] : 0.0;
      const double d12 = dy[i2 * p + j2] * dx[i1 * p + j1];
      const double d22 = (i1 == j1) ? dyy[i2 * p + j2] : 0.0;
      const double d1 = (i2 == j2) ? dx[i1 * p + j1] : 0.0;
      const double d2 = (i1 == j1) ? dy[i2 * p + j2] : 0.0;
      double v = -(c11 * d11);
      v -= 2.0 * c12 * d12;
      v -= c22 * d22;
      v += c1 * d1;
      v += c2 * d2;
      if (j == k) v += c0;
      const int ip = ipos[j];
      if (ip >= 0)
        aii[(long long)r * a.Aii.ld + ip] = v;
      else
        aie[(long long)r * a.Aie.ld + (-1 - ip)] = v;
      return ip >= 0 ? fabs(v) : 0.0;
    };
    // (both mappings visit j = threadIdx.x + t*blockDim.x, so csum[t] is always column j's sum)
    if (p >= 32 && (int)blockDim.x % p == 0) {
      // thread -> (j1, first j2) fixed for the CTA: no integer division per element (measured
      // faster at p = 32, slower at p = 16)
      const int j1 = (int)threadIdx.x % p, step = (int)blockDim.x / p;
      int t = 0;
      for (int j2 = (int)threadIdx.x / p; j2 < p; j2 += step, ++t) {
        const double av = elem(j1, j2);
        if (t < ASM_COLS) csum[t] += av;
      }
    } else {
      int t = 0;
      for (int j = threadIdx.x; j < P; j += blockDim.x, ++t) {
        const double av = elem(j % p, j / p);
        if (t < ASM_COLS) csum[t] += av;
      }
    }
  }
  if (a.colpart) {
    double* cp = a.colpart + ((long long)leaf * gridDim.x + blockIdx.x) * m;
    int t = 0;
    for (int j = threadIdx.x; j < P && t < ASM_COLS; j += blockDim.x, ++t)
      if (ipos[j] >= 0) cp[ipos[j]] = csum[t];
  }
}

int leaf_assemble_rows() { return ASM_ROWS; }

// |A_ii|_1 per leaf from the assembly's partial column sums (row blocks summed in order)
__global__ void __launch_bounds__(256) colpart_norm_kernel(int m, int nrb, const double* colpart, double* anorm,
                                                           int batch_off) {
  const int leaf = blockIdx.x + batch_off;
  const double* cp = colpart + (long long)leaf * nrb * m;
  double best = 0.0;
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    double sum = 0.0;
    for (int rb = 0; rb < nrb; ++rb) sum += cp[(long long)rb * m + c];
    best = (sum > best || sum != sum) ? sum : best;
  }
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, best, o);
    best = (t > best || t != t) ? t : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = (red[w] > v || red[w] != red[w]) ? red[w] : v;
    anorm[leaf] = v;
  }
}

int launch_leaf_assemble(const LeafAsmArgs& a, cudaStream_t s) {
  const int m = (a.p - 2) * (a.p - 2);
  const size_t smem = sizeof(double) * (4 * a.p * a.p + 6 * ASM_ROWS) + sizeof(int) * a.p * a.p;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(leaf_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // colpart needs every column of a thread in csum[]: P <= 8 * 256 (p <= 45)
  if (a.colpart && a.p * a.p > 8 * 256) return 1;
  const int nrb = (m + ASM_ROWS - 1) / ASM_ROWS;
  for (int off = 0; off < a.nleaf; off += 65535) {
    dim3 grid(nrb, min(65535, a.nleaf - off));
    leaf_assemble_kernel<<<grid, 256, smem, s>>>(a, off);
  }
  if (a.colpart && a.anorm)
    for (int off = 0; off < a.nleaf; off += 65535)
      colpart_norm_kernel<<<min(65535, a.nleaf - off), 256, 0, s>>>(m, nrb, a.colpart, a.anorm, off);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// Merge gather (reference solver.py:130-141): for each parent,
//   XS   = [ Ta[p3a,p3a] - Tb[p3b,p3b] | -Ta[p3a,p1a] | Tb[p3b,p2b] ]     m3 x (m3+e)
//   Tei  = [ Ta[p1a,p3a] ; Tb[p2b,p3b] ]                                   e x m3
//   Tnew = blkdiag(Ta[p1a,p1a], Tb[p2b,p2b])                               e x e
// One linear element space per parent; consecutive threads walk columns.
__global__ void merge_gather_kernel(MergeGatherArgs a, int batch_off) {
  const int item = blockIdx.y + batch_off;
  const int m3 = a.m3, n1 = a.n1, n2 = a.n2, e = n1 + n2;
  const int* ix = a.idx + (long long)item * a.idx_stride;
  const int* p1a = ix;
  const int* p3a = p1a + n1;
  const int* p2b = p3a + m3;
  const int* p3b = p2b + n2;
  const double* Ta = a.Ta.get(item);
  const double* Tb = a.Tb.get(item);
  const long long lda = a.Ta.ld, ldb = a.Tb.ld;
  double* xs = a.XS.get(item);
  double* tei = a.Tei.get(item);
  double* tnew = a.Tnew.get(item);
  const long long s1 = (long long)m3 * (m3 + e);
  const long long s2 = s1 + (long long)e * m3;
  const long long total = s2 + (long long)e * e;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    if (t < s1) {
      const int r = (int)(t / (m3 + e)), c = (int)(t % (m3 + e));
      double v;
      if (c < m3)
        v = Ta[p3a[r] * lda + p3a[c]] - Tb[p3b[r] * ldb + p3b[c]];
      else if (c < m3 + n1)
        v = -Ta[p3a[r] * lda + p1a[c - m3]];
      else
        v = Tb[p3b[r] * ldb + p2b[c - m3 - n1]];
      xs[(long long)r * a.XS.ld + c] = v;
    } else if (t < s2) {
      const long long u = t - s1;
      const int r = (int)(u / m3), c = (int)(u % m3);
      const double v = (r < n1) ? Ta[p1a[r] * lda + p3a[c]] : Tb[p2b[r - n1] * ldb + p3b[c]];
      tei[(long long)r * a.Tei.ld + c] = v;
    } else {
      const long long u = t - s2;
      const int r = (int)(u / e), c = (int)(u % e);
      double v = 0.0;
      if (r < n1 && c < n1)
        v = Ta[p1a[r] * lda + p1a[c]];
      else if (r >= n1 && c >= n1)
        v = Tb[p2b[r - n1] * ldb + p2b[c - n1]];
      tnew[(long long)r * a.Tnew.ld + c] = v;
    }
  }
}

int launch_merge_gather(const MergeGatherArgs& a, cudaStream_t s) {
  const int e = a.n1 + a.n2;
  const long long total = (long long)a.m3 * (a.m3 + e) + (long long)e * a.m3 + (long long)e * e;
  int gx = (int)((total + 255) / 256);
  const int max_gx = 1184;  // 8 CTAs x 148 SMs per parent is plenty for the big top levels
  if (gx > max_gx) gx = max_gx;
  for (int off = 0; off < a.npar; off += 65535) {
    dim3 grid(gx, min(65535, a.npar - off));
    merge_gather_kernel<<<grid, 256, 0, s>>>(a, off);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace hps
