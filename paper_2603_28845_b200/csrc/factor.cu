// On-GPU factorisation for GPTQ (replaces layerwise.cpp:31-51):
//   hd = fp64(H); damp = percdamp*mean(diag(hd)); hd += damp*I;
//   hp = P hd P^T;  hinv = hp^-1;  U = upper Cholesky factor of hinv.
// Computed as  A = J hp J = L L^T (lower, blocked right-looking),
//              U = J L^-1 J  (blocked triangular inverse).
// Mathematically identical to the reference's LLT -> solve(I) -> LLT (by the
// uniqueness of the Cholesky factor of hinv), 2n^3/3 flops instead of 8n^3/3.
// Templated on the compute type T (float default, double reference-class).
#include <cmath>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int NB = 64;  // panel width

// A[i][j] = T(double(H[o(i)][o(j)]) + (i==j)*damp), o(i) = order[n-1-i]; lower only
template <typename T>
__global__ void build_input_kernel(const float* __restrict__ h, long long n,
                                   const int32_t* __restrict__ order, const double* damp, T* a) {
  const double dmp = *damp;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n, j = e % n;
    if (j > i) continue;
    const long long oi = order[n - 1 - i], oj = order[n - 1 - j];
    double v = double(h[oi * n + oj]);
    if (i == j) v = __dadd_rn(v, dmp);
    a[e] = T(v);
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

// Factor the nb x nb diagonal block at (k0,k0) in shared memory with one
// barrier per column (every thread rescales column j itself from the unscaled
// values; the scaled column is written to a separate array), then invert it.
// Writes L_kk back into A and L_kk^-1 into dinv (NB x NB row-major).
template <typename T>
__global__ void __launch_bounds__(256) potrf_diag_kernel(T* a, long long n, long long k0, T* dinv,
                                                         unsigned* flag) {
  extern __shared__ __align__(16) unsigned char dsm_raw[];
  T(*s)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(dsm_raw);
  T(*l)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(dsm_raw + sizeof(T) * NB * (NB + 1));
  T(*x)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(dsm_raw + 2 * sizeof(T) * NB * (NB + 1));
  const int nb = int(min((long long)NB, n - k0));
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) {
    const int i = e / NB, j = e % NB;
    s[i][j] = (i < nb && j < nb && j <= i) ? a[(k0 + i) * n + k0 + j] : T(i == j ? 1 : 0);
    l[i][j] = T(0);
    x[i][j] = T(i == j ? 1 : 0);
  }
  __syncthreads();
  bool bad = false;
  for (int j = 0; j < nb; ++j) {
    const T piv = s[j][j];
    bad |= !(piv > T(0));  // Eigen: x <= 0 -> NumericalIssue (NaN rejected too)
    const T d = sqrt(piv);
    const T rd = T(1) / d;
    for (int e = tid; e < NB * NB; e += 256) {
      const int i = e / NB, c = e % NB;
      if (i <= j || i >= nb) continue;
      if (c == j) {
        l[i][j] = s[i][j] * rd;
      } else if (c > j && c <= i) {
        s[i][c] -= (s[i][j] * rd) * (s[c][j] * rd);
      }
    }
    if (tid == 0) l[j][j] = d;
    __syncthreads();
  }
  // X = L^-1: for each j, rows i > j -= L_ij * (row j / L_jj); then row j /= L_jj
  for (int j = 0; j < nb; ++j) {
    const T rl = T(1) / l[j][j];
    for (int e = tid; e < NB * NB; e += 256) {
      const int i = e / NB, c = e % NB;
      if (c > j || i <= j || i >= nb) continue;
      x[i][c] -= l[i][j] * (x[j][c] * rl);
    }
    __syncthreads();
    if (tid <= j) x[j][tid] *= rl;
    __syncthreads();
  }
  for (int e = tid; e < NB * NB; e += 256) {
    const int i = e / NB, c = e % NB;
    if (i < nb && c < nb) {
      if (c <= i) a[(k0 + i) * n + k0 + c] = l[i][c];
      dinv[i * NB + c] = (c <= i) ? x[i][c] : T(0);
    }
  }
  if (bad) atomicOr(flag, kFlagNotPD);
}

template <typename T>
__global__ void copy_block_kernel(const T* __restrict__ src, long long lds, T* dst, long long ldd,
                                  long long rows, long long cols) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e % cols;
    dst[i * ldd + j] = src[i * lds + j];
  }
}

template <typename T>
__global__ void identity_kernel(T* x, long long n) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x)
    x[e] = T((e / n == e % n) ? 1 : 0);
}

// U[r][c] = X[n-1-r][n-1-c] for r <= c (X = L^-1 lower), else 0
template <typename T>
__global__ void reverse_to_upper_kernel(const T* __restrict__ x, long long n, T* u) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e % n;
    u[e] = (r <= c) ? x[(n - 1 - r) * n + (n - 1 - c)] : T(0);
  }
}

inline int blocks_for(long long n) {
  long long g = (n + 255) / 256;
  return int(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

template <typename T>
constexpr int potrf_smem() {
  return 3 * NB * (NB + 1) * int(sizeof(T));
}

}  // namespace

template <typename T>
void launch_build_factor_input(const float* h, long long n, const int32_t* order, double percdamp,
                               T* a, double* damp, cudaStream_t st) {
  count_launches(2);
  damp_kernel<<<1, 1024, 0, st>>>(h, n, percdamp, damp);
  build_input_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(h, n, order, damp, a);
}

// ws layout: [nblk*NB*NB dinv blocks][n*n scratch]
template <typename T>
void factor_upper_inverse(T* a, long long n, T* u, T* ws, unsigned* flag, cudaStream_t st) {
  static const bool attr = [] {
    cudaFuncSetAttribute(potrf_diag_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         potrf_smem<T>());
    return true;
  }();
  (void)attr;
  const long long nblk = (n + NB - 1) / NB;
  T* dinv = ws;
  T* tmp = ws + nblk * NB * NB;
  for (long long kb = 0; kb < nblk; ++kb) {
    const long long k0 = kb * NB, w = std::min<long long>(NB, n - k0), rest = n - k0 - w;
    count_launches(1);
    potrf_diag_kernel<T><<<1, 256, potrf_smem<T>(), st>>>(a, n, k0, dinv + kb * NB * NB, flag);
    if (rest <= 0) continue;
    gemm<T, T, T>(rest, w, w, 1.0, a + (k0 + w) * n + k0, n, false, dinv + kb * NB * NB, NB, true,
                  0.0, tmp, NB, false, st);
    count_launches(1);
    copy_block_kernel<T><<<blocks_for(rest * w), 256, 0, st>>>(tmp, NB, a + (k0 + w) * n + k0, n,
                                                               rest, w);
    gemm<T, T, T>(rest, rest, w, -1.0, tmp, NB, false, tmp, NB, true, 1.0,
                  a + (k0 + w) * n + (k0 + w), n, true, st);
  }
  T* x = u;
  count_launches(2);
  identity_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(x, n);
  for (long long ib = 0; ib < nblk; ++ib) {
    const long long i0 = ib * NB, w = std::min<long long>(NB, n - i0);
    const long long cols = i0 + w, rest = n - i0 - w;
    gemm<T, T, T>(w, cols, w, 1.0, dinv + ib * NB * NB, NB, false, x + i0 * n, n, false, 0.0, tmp,
                  cols, false, st);
    count_launches(1);
    copy_block_kernel<T><<<blocks_for(w * cols), 256, 0, st>>>(tmp, cols, x + i0 * n, n, w, cols);
    if (rest > 0)
      gemm<T, T, T>(rest, cols, w, -1.0, a + (i0 + w) * n + i0, n, false, x + i0 * n, n, false,
                    1.0, x + (i0 + w) * n, n, false, st);
  }
  reverse_to_upper_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(x, n, tmp);
  cudaMemcpyAsync(u, tmp, size_t(n * n) * sizeof(T), cudaMemcpyDeviceToDevice, st);
}

template <typename T>
void launch_gram_upper(const T* u, long long n, double* hinv, cudaStream_t st) {
  gemm<double, T, T>(n, n, n, 1.0, u, n, true, u, n, false, 0.0, hinv, n, false, st);
}

template void launch_build_factor_input<float>(const float*, long long, const int32_t*, double,
                                               float*, double*, cudaStream_t);
template void launch_build_factor_input<double>(const float*, long long, const int32_t*, double,
                                                double*, double*, cudaStream_t);
template void factor_upper_inverse<float>(float*, long long, float*, float*, unsigned*,
                                          cudaStream_t);
template void factor_upper_inverse<double>(double*, long long, double*, double*, unsigned*,
                                           cudaStream_t);
template void launch_gram_upper<float>(const float*, long long, double*, cudaStream_t);
template void launch_gram_upper<double>(const double*, long long, double*, cudaStream_t);

}  // namespace ocwg
