// Leaf-stage assembly and merge-stage gather kernels (bandwidth-bound producers feeding the
// DMMA Gauss-Jordan and GEMM kernels).
#include <algorithm>
#include <cstdlib>

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

// ---------------------------------------------------------------------------------------------
// Fused leaf assembly: one CTA builds `rows` complete rows [A_ii | A_ie] of one leaf in shared
// memory (columns in output order: the m interior nodes, then the c exterior nodes), multiplies
// the exterior part by the lift on DMMA tiles, R = -A_ie L (rows x b, leaf.py:154), and writes
// [A_ii | R] as whole contiguous rows of the Gauss-Jordan workspace: A_ie never goes to HBM and
// there is no separate GEMM launch (config 5: assembly 4.3 ms + GEMM 3.8 ms before).
//
// Only the 2p - 1 entries of a row that share a grid line with the row's node carry the
// c11/c22/c1/c2/c terms; every other entry is the mixed-derivative term alone,
//   -(2 c12) (dy[i2,j2] dx[i1,j1])
// (the reference's accumulation order adds exact zeros there), so the bulk pass is two
// multiplications per entry and a second pass recomputes the cross entries with the full,
// reference-ordered expression.
struct AsmFusedCfg {
  int rows;     // rows per CTA (multiple of 8)
  int ldt;      // tile row length in doubles (== 4 mod 16: conflict-free DMMA A fragments)
  int b, c;     // Gauss edge nodes / exterior Chebyshev nodes
  int vec;      // 16-byte row stores allowed
  int csc;      // doubles reserved for the column-sum exchange (two row groups in the write-out)
  const double* lift;
  MatB FS;      // m x (m + b) per leaf
};

constexpr int ASMF_MAXT = 4;  // R tiles (8 x 8) held per warp

__global__ void __launch_bounds__(256) leaf_assemble_fused_kernel(LeafAsmArgs a, AsmFusedCfg f, int nrb) {
  extern __shared__ double sd[];
  const int p = a.p, P = p * p, pm = p - 2;
  const int m = pm * pm, b = f.b, c = f.c, rows = f.rows, ldt = f.ldt;
  const int ncol = m + b;
  double* dx = sd;
  double* dy = dx + P;
  double* dxx = dy + P;
  double* dyy = dxx + P;
  double* cr = dyy + P;                 // [rows][6] coefficient samples at the row points
  double* csc = cr + 6 * rows;          // [ncol] column-sum exchange between the two row groups
  double* T = csc + f.csc;              // [rows][ldt] output rows
  int* jof = reinterpret_cast<int*>(T + (size_t)rows * ldt);  // output column -> grid node
  int* qof = jof + P;                                          // grid node -> output column
  int2* ri = reinterpret_cast<int2*>(qof + P);                 // [rows] row offsets (i1 p, i2 p) into the 1D operators
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long cstride = (long long)a.nleaf * P;
  // static data once per CTA (persistent over (leaf, row block) units)
  for (int e = tid; e < P; e += 256) {
    dx[e] = a.dx[e];
    dy[e] = a.dy[e];
    dxx[e] = a.dxx[e];
    dyy[e] = a.dyy[e];
    const int ip = a.int_pos[e];
    const int q = ip >= 0 ? ip : m + a.ext_pos[e];
    qof[e] = q;
    jof[q] = e;
  }
  const long long units = (long long)a.nleaf * nrb;
  // coefficient samples of a unit: at most one value per thread (rows * 6 <= 256), fetched one
  // unit ahead into a register
  auto fetch = [&](long long u) -> double {
    if (u >= units || tid >= rows * 6) return 0.0;
    const int leaf = (int)(u / nrb), rb = (int)(u - (long long)leaf * nrb);
    const int rr = tid / 6, t = tid - rr * 6, r = rb * rows + rr;
    return r < m ? a.coef[(long long)leaf * P + t * cstride + (1 + r % pm) + p * (1 + r / pm)] : 0.0;
  };
  double cnext = fetch(blockIdx.x);
  const int g = lane >> 2, t4 = lane & 3;
  const int mtiles = rows >> 3, ntiles = (b + 7) >> 3, ntile = mtiles * ntiles;
  const int np2 = ncol >> 1;
  const int nh = f.csc ? 2 : 1;  // row groups of the write-out pass
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const int leaf = (int)(u / nrb), rb = (int)(u - (long long)leaf * nrb);
    const int r0 = rb * rows;
    const int nr = min(rows, m - r0);
    __syncthreads();  // previous unit's tile and coefficients fully consumed
    if (tid < rows * 6) cr[tid] = cnext;
    if (tid < rows) {
      const int r = min(r0 + tid, m - 1);
      ri[tid] = make_int2((1 + r % pm) * p, (1 + r / pm) * p);
    }
    cnext = fetch(u + gridDim.x);
    __syncthreads();
    // 1. bulk pass: thread owns output columns q = tid + 256 k
    for (int q = tid; q < P; q += 256) {
      const int j = jof[q], j2 = j / p, j1 = j - j2 * p;
      // four rows per step, all loads before the stores (independent chains: the loop is
      // latency-bound otherwise, shared-memory stores and loads may alias for the compiler)
      int rr = 0;
      for (; rr + 4 <= nr; rr += 4) {
        double cc[4], vy[4], vx[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int2 io = ri[rr + k];
          cc[k] = cr[(rr + k) * 6 + 1];
          vy[k] = dy[io.y + j2];
          vx[k] = dx[io.x + j1];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) T[(rr + k) * ldt + q] = -((2.0 * cc[k]) * (vy[k] * vx[k]));
      }
      for (; rr < nr; ++rr) {
        const int2 io = ri[rr];
        T[rr * ldt + q] = -((2.0 * cr[rr * 6 + 1]) * (dy[io.y + j2] * dx[io.x + j1]));
      }
    }
    __syncthreads();
    // 2. cross entries (same grid line as the row's node): the full expression, reference order
    for (int e = tid; e < nr * (2 * p - 1); e += 256) {
      const int rr = e / (2 * p - 1), sidx = e - rr * (2 * p - 1);
      const int2 io = ri[rr];
      const int i1 = io.x / p, i2 = io.y / p;
      int j1, j2;
      if (sidx < p) {
        j1 = sidx;
        j2 = i2;
      } else {
        j1 = i1;
        j2 = sidx - p;
        if (j2 >= i2) ++j2;
      }
      const double* c6 = cr + rr * 6;
      const double d11 = (i2 == j2) ? dxx[io.x + j1] : 0.0;
      const double d12 = dy[io.y + j2] * dx[io.x + j1];
      const double d22 = (i1 == j1) ? dyy[io.y + j2] : 0.0;
      const double d1 = (i2 == j2) ? dx[io.x + j1] : 0.0;
      const double d2 = (i1 == j1) ? dy[io.y + j2] : 0.0;
      double v = -(c6[0] * d11);
      v -= 2.0 * c6[1] * d12;
      v -= c6[2] * d22;
      v += c6[3] * d1;
      v += c6[4] * d2;
      if (j1 == i1 && j2 == i2) v += c6[5];
      T[rr * ldt + qof[j1 + p * j2]] = v;
    }
    __syncthreads();
    // 3. R = -A_ie L on DMMA tiles (A_ie = T[:, m : m + c]); results held until every warp has
    //    read its A_ie fragments, then written over the A_ie columns
    double acc[ASMF_MAXT][2];
    const double* arow[ASMF_MAXT];
    const double* bcol[ASMF_MAXT];
    bool bok[ASMF_MAXT];
#pragma unroll
    for (int k = 0; k < ASMF_MAXT; ++k) {
      acc[k][0] = acc[k][1] = 0.0;
      const int tile = min(warp + 8 * k, ntile - 1);  // surplus slots repeat the last tile (never stored)
      const int mt = tile % mtiles, nt = tile / mtiles;
      const int col = nt * 8 + g;
      arow[k] = T + (size_t)(mt * 8 + g) * ldt + m + t4;
      bok[k] = col < b;
      bcol[k] = f.lift + (bok[k] ? col : 0) + (long long)t4 * b;
    }
    // k outer, tiles inner: up to ASMF_MAXT independent DMMA chains per warp
    for (int kk = 0; kk < c; kk += 4) {
      double av[ASMF_MAXT], bv[ASMF_MAXT];
#pragma unroll
      for (int k = 0; k < ASMF_MAXT; ++k) {
        av[k] = arow[k][kk];
        bv[k] = bok[k] ? __ldg(bcol[k] + (long long)kk * b) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < ASMF_MAXT; ++k) dmma8x8x4(acc[k][0], acc[k][1], av[k], bv[k]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ASMF_MAXT; ++k) {
      const int tile = warp + 8 * k;
      if (tile < ntile) {
        const int mt = tile % mtiles, nt = tile / mtiles;
        double* drow = T + (size_t)(mt * 8 + g) * ldt + m + nt * 8 + 2 * t4;
        if (nt * 8 + 2 * t4 < b) drow[0] = -acc[k][0];
        if (nt * 8 + 2 * t4 + 1 < b) drow[1] = -acc[k][1];
      }
    }
    __syncthreads();
    // 4. whole rows [A_ii | R] -> global (coalesced); |A_ii|_1 partial column sums on the way
    double* fs = f.FS.get(leaf);
    const long long ld = f.FS.ld;
    double* cp = a.colpart ? a.colpart + ((long long)leaf * nrb + rb) * m : nullptr;
    if (f.vec && nh == 2) {
      // thread = (row group h, column pair q2): all 256 threads store; the second group's
      // column sums reach the first through csc
      const int h = tid / np2, q = 2 * (tid - h * np2);
      double s0 = 0.0, s1 = 0.0;
      if (h < 2) {
        for (int rr = h; rr < nr; rr += 2) {
          const double2 v = *reinterpret_cast<const double2*>(T + (size_t)rr * ldt + q);
          *reinterpret_cast<double2*>(fs + (long long)(r0 + rr) * ld + q) = v;
          s0 += fabs(v.x);
          s1 += fabs(v.y);
        }
        if (h == 1) {
          csc[q] = s0;
          csc[q + 1] = s1;
        }
      }
      __syncthreads();
      if (h == 0 && cp) {
        if (q < m) cp[q] = s0 + csc[q];
        if (q + 1 < m) cp[q + 1] = s1 + csc[q + 1];
      }
    } else if (f.vec) {
      for (int q2 = tid; q2 < np2; q2 += 256) {
        const int q = 2 * q2;
        double s0 = 0.0, s1 = 0.0;
        for (int rr = 0; rr < nr; ++rr) {
          const double2 v = *reinterpret_cast<const double2*>(T + (size_t)rr * ldt + q);
          *reinterpret_cast<double2*>(fs + (long long)(r0 + rr) * ld + q) = v;
          s0 += fabs(v.x);
          s1 += fabs(v.y);
        }
        if (cp) {
          if (q < m) cp[q] = s0;
          if (q + 1 < m) cp[q + 1] = s1;
        }
      }
    } else {
      for (int q = tid; q < ncol; q += 256) {
        double s0 = 0.0;
        for (int rr = 0; rr < nr; ++rr) {
          const double v = T[(size_t)rr * ldt + q];
          fs[(long long)(r0 + rr) * ld + q] = v;
          s0 += fabs(v);
        }
        if (cp && q < m) cp[q] = s0;
      }
    }
  }
}

static int asm_fused_csc(int ncol) { return ncol <= 256 ? ((ncol + 1) & ~1) : 0; }
static size_t asm_fused_smem(int P, int rows, int ncol) {
  const int ldt = ((P + 15) & ~15) + 4;
  return sizeof(double) * (4 * P + 6 * rows + asm_fused_csc(ncol) + (size_t)rows * ldt) +
         sizeof(int) * (2 * P + 2 * rows);
}

// rows per CTA of the fused kernel for this leaf order (0: not applicable, use the two-kernel path)
static int asm_fused_rows(int p, int b) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HPS_ASM_FUSED");
    on = e ? atoi(e) : 1;
  }
  if (!on) return 0;
  const int P = p * p, m = (p - 2) * (p - 2), ntiles = (b + 7) / 8;
  // measured on the B200: p = 16 leaves 5.7 -> 3.8 ms per 16384 (assembly + GEMM before), but
  // p = 32 leaves 4.7 -> 6.1 ms per 1024 (8-row tiles, 2 CTAs per SM): large orders keep the
  // two-kernel path (HPS_ASM_FUSED=2 forces the fused kernel for every order it fits)
  if (on == 1 && P > 576) return 0;
  static int rmax = -1;
  if (rmax < 0) {
    const char* e = getenv("HPS_ASM_ROWS");
    rmax = e ? atoi(e) : 32;
  }
  for (int rows = rmax; rows >= 8; rows -= 8) {
    if (rows / 8 * ntiles > 8 * ASMF_MAXT) continue;
    if (asm_fused_smem(P, rows, m + b) <= (size_t)(rows == 8 ? 200 : 100) * 1024) return rows;  // >= 2 CTAs per SM unless only 8 rows fit
  }
  return 0;
}

int leaf_assemble_rows(int p, int q) {
  const int r = asm_fused_rows(p, 4 * q);
  return r ? r : ASM_ROWS;
}

// Assembly + right-hand sides in one launch; returns -1 when the fused kernel does not apply.
int launch_leaf_assemble_fused(const LeafAsmArgs& a, MatB FS, const double* lift, int q, cudaStream_t s) {
  const int p = a.p, P = p * p, m = (p - 2) * (p - 2), b = 4 * q, c = 4 * (p - 1);
  const int rows = asm_fused_rows(p, b);
  if (!rows || b > c || (a.colpart && P > 8 * 256)) return -1;
  AsmFusedCfg f{};
  f.rows = rows;
  f.ldt = ((P + 15) & ~15) + 4;
  f.b = b;
  f.c = c;
  f.lift = lift;
  f.FS = FS;
  f.vec = !FS.ptrs && FS.base && ((reinterpret_cast<uintptr_t>(FS.base) >> 3) & 1) == 0 &&
          ((FS.stride | FS.off | (long long)FS.ld | (long long)(m + b)) & 1) == 0;
  f.csc = f.vec ? asm_fused_csc(m + b) : 0;
  const size_t smem = asm_fused_smem(P, rows, m + b);
  static int sms = 0, max_smem = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(leaf_assemble_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    max_smem = 200 * 1024;
  }
  if (smem > (size_t)max_smem) return -1;
  const int nrb = (m + rows - 1) / rows;
  // persistent CTAs (the 1D operators and index maps are staged once per CTA): as many as fit
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("HPS_ASM_PER_SM");
    cap = e ? atoi(e) : 4;
  }
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(cap, (227 * 1024) / (smem + 1024)));
  const long long units = (long long)a.nleaf * nrb;
  const int grid = (int)std::min<long long>(units, (long long)per_sm * sms);
  leaf_assemble_fused_kernel<<<grid, 256, smem, s>>>(a, f, nrb);
  if (a.colpart && a.anorm)
    for (int off = 0; off < a.nleaf; off += 65535)
      colpart_norm_kernel<<<min(65535, a.nleaf - off), 256, 0, s>>>(m, nrb, a.colpart, a.anorm, off);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
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
