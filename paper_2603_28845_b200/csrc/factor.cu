// On-GPU factorisation for GPTQ (replaces layerwise.cpp:31-51):
//   hd = fp64(H); damp = percdamp*mean(diag(hd)); hd += damp*I;
//   hp = P hd P^T;  hinv = hp^-1;  U = upper Cholesky factor of hinv.
// Computed as  A = J hp J = L L^T (lower, blocked right-looking fp64),
//              U = J L^-1 J  (blocked triangular inverse).
// Mathematically identical to the reference's LLT -> solve(I) -> LLT (by the
// uniqueness of the Cholesky factor of hinv), 2n^3/3 flops instead of 8n^3/3.
#include <cmath>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int NB = 64;  // panel width
constexpr int kPotrfSmem = 2 * NB * (NB + 1) * int(sizeof(double));

// A[i][j] = double(H[o(i)][o(j)]) (+damp on the diagonal), o(i) = order[n-1-i]
__global__ void build_input_kernel(const float* __restrict__ h, long long n,
                                   const int32_t* __restrict__ order, const double* damp,
                                   double* a) {
  const double dmp = *damp;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n, j = e % n;
    if (j > i) continue;  // lower triangle is all the factorisation reads
    const long long oi = order[n - 1 - i], oj = order[n - 1 - j];
    double v = double(h[oi * n + oj]);
    if (i == j) v = __dadd_rn(v, dmp);
    a[e] = v;
  }
}

// damp = percdamp * mean(diag(fp64 H))  (layerwise.cpp:32-33)
__global__ void damp_kernel(const float* __restrict__ h, long long n, double percdamp,
                            double* damp) {
  __shared__ double part[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += double(h[i * n + i]);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    *damp = percdamp * (t / double(n));
  }
}

// Factor the nb x nb diagonal block at (k0,k0) in shared memory; write L_kk
// back into A and its inverse into dinv (nb x nb, row-major).
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* a, long long n, long long k0,
                                                         double* dinv, unsigned* flag) {
  extern __shared__ double dsm[];
  double(*s)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*inv)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  const int nb = int(min((long long)NB, n - k0));
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int i = e / NB, j = e % NB;
    s[i][j] = (i < nb && j < nb && j <= i) ? a[(k0 + i) * n + k0 + j] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  __shared__ int bad;
  if (tid == 0) bad = 0;
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      const double x = s[j][j];
      if (!(x > 0.0)) bad = 1;  // Eigen: x <= 0 -> NumericalIssue (NaN also rejected here)
      s[j][j] = sqrt(x);
    }
    __syncthreads();
    const double d = s[j][j];
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) s[i][j] = __ddiv_rn(s[i][j], d);
    __syncthreads();
    // trailing update of the block's lower triangle, columns j+1..
    const int m = nb - j - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l <= i) s[i][l] -= s[i][j] * s[l][j];
    }
    __syncthreads();
  }
  // inverse of the lower-triangular block: one column per thread group
  for (int e = tid; e < NB * NB; e += blockDim.x) inv[e / NB][e % NB] = 0.0;
  __syncthreads();
  if (tid < NB) {
    const int col = tid;
    if (col < nb) {
      for (int r = col; r < nb; ++r) {
        double acc = (r == col) ? 1.0 : 0.0;
        for (int l = col; l < r; ++l) acc -= s[r][l] * inv[l][col];
        inv[r][col] = acc / s[r][r];
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int i = e / NB, j = e % NB;
    if (i < nb && j < nb) {
      if (j <= i) a[(k0 + i) * n + k0 + j] = s[i][j];
      dinv[i * NB + j] = inv[i][j];
    }
  }
  if (tid == 0 && bad) atomicOr(flag, kFlagNotPD);
}

__global__ void copy_block_kernel(const double* __restrict__ src, long long lds, double* dst,
                                  long long ldd, long long rows, long long cols) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e % cols;
    dst[i * ldd + j] = src[i * lds + j];
  }
}

__global__ void identity_kernel(double* x, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x)
    x[e] = (e / n == e % n) ? 1.0 : 0.0;
}

// U[r][c] = X[n-1-r][n-1-c] for r <= c (X = L^-1 lower), else 0
__global__ void reverse_to_upper_kernel(const double* __restrict__ x, long long n, double* u) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e % n;
    u[e] = (r <= c) ? x[(n - 1 - r) * n + (n - 1 - c)] : 0.0;
  }
}

inline int blocks_for(long long n) {
  long long g = (n + 255) / 256;
  return int(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

void launch_build_factor_input(const float* h, long long n, const int32_t* order, double percdamp,
                               double* a, double* damp, cudaStream_t st) {
  count_launches(2);
  damp_kernel<<<1, 1024, 0, st>>>(h, n, percdamp, damp);
  build_input_kernel<<<blocks_for(n * n), 256, 0, st>>>(h, n, order, damp, a);
}

// ws layout: [n*NB dinv blocks][n*n scratch]
void factor_upper_inverse(double* a, long long n, double* u, double* ws, unsigned* flag,
                          cudaStream_t st) {
  static const bool attr = [] {
    cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kPotrfSmem);
    return true;
  }();
  (void)attr;
  const long long nblk = (n + NB - 1) / NB;
  double* dinv = ws;                     // nblk * NB * NB
  double* tmp = ws + nblk * NB * NB;     // n * n scratch
  // ---- blocked right-looking Cholesky, lower, in place in A
  for (long long kb = 0; kb < nblk; ++kb) {
    const long long k0 = kb * NB, w = std::min<long long>(NB, n - k0), rest = n - k0 - w;
    potrf_diag_kernel<<<1, 256, kPotrfSmem, st>>>(a, n, k0, dinv + kb * NB * NB, flag);
    count_launches(1);
    if (rest <= 0) continue;
    count_launches(1);  // copy_block
    // panel: L[k+1:, k] = A[k+1:, k] * Linv_kk^T   -> tmp (rest x w), ld NB
    dgemm<double, double>(rest, w, w, 1.0, a + (k0 + w) * n + k0, n, false, dinv + kb * NB * NB,
                          NB, true, 0.0, tmp, NB, false, st);
    copy_block_kernel<<<blocks_for(rest * w), 256, 0, st>>>(tmp, NB, a + (k0 + w) * n + k0, n,
                                                            rest, w);
    // trailing: A[k+1:, k+1:] -= L_panel L_panel^T  (lower tiles only)
    dgemm<double, double>(rest, rest, w, -1.0, tmp, NB, false, tmp, NB, true, 1.0,
                          a + (k0 + w) * n + (k0 + w), n, true, st);
  }
  // ---- X = L^-1, right-looking: X starts as I; for each block row i:
  //   X[i, 0:i+1] = Linv_ii X[i, 0:i+1];  X[i+1:, 0:i+1] -= L[i+1:, i] X[i, 0:i+1]
  double* x = u;  // reuse the U buffer for X, then reverse into tmp and copy
  identity_kernel<<<blocks_for(n * n), 256, 0, st>>>(x, n);
  count_launches(2);  // identity + reverse_to_upper
  for (long long ib = 0; ib < nblk; ++ib) {
    const long long i0 = ib * NB, w = std::min<long long>(NB, n - i0);
    const long long cols = i0 + w, rest = n - i0 - w;
    dgemm<double, double>(w, cols, w, 1.0, dinv + ib * NB * NB, NB, false, x + i0 * n, n, false,
                          0.0, tmp, cols, false, st);
    copy_block_kernel<<<blocks_for(w * cols), 256, 0, st>>>(tmp, cols, x + i0 * n, n, w, cols);
    count_launches(1);
    if (rest > 0)
      dgemm<double, double>(rest, cols, w, -1.0, a + (i0 + w) * n + i0, n, false, x + i0 * n, n,
                            false, 1.0, x + (i0 + w) * n, n, false, st);
  }
  reverse_to_upper_kernel<<<blocks_for(n * n), 256, 0, st>>>(x, n, tmp);
  cudaMemcpyAsync(u, tmp, size_t(n * n) * sizeof(double), cudaMemcpyDeviceToDevice, st);
}

void launch_gram_upper(const double* u, long long n, double* hinv, cudaStream_t st) {
  // hinv = U^T U
  dgemm<double, double>(n, n, n, 1.0, u, n, true, u, n, false, 0.0, hinv, n, false, st);
}

}  // namespace ocwg
