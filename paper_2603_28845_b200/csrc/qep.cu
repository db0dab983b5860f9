// QEP target correction (replaces layerwise.cpp:95-112, row f1 of SURVEY §8):
//   lambda = eta * mean(diag(gram));  W* = W + alpha * (gram + lambda I)^-1 (cross W)
// in fp64 like the reference (Eigen LLT + solve), on the GPU: the tile
// Cholesky of factor.cu in natural order, L^-1 by recursive doubling, and
// three fp64 GEMMs on the DMMA tensor cores (cross W, L^-1 B, L^-T Y; the two
// triangular products skip the k range of L^-1's zeros).  Non-PD -> kFlagNotPD.
#include <algorithm>

#include "kernels.h"

namespace ocwg {
namespace {

// lambda = eta * mean(diag(gram)) (one CTA), then a = gram + lambda I (grid-wide)
__global__ void qep_lambda_kernel(const double* __restrict__ gram, long long n, double eta,
                                  double* lam) {
  __shared__ double part[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += gram[i * n + i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    *lam = eta * (t / double(n));  // stats.gram.diagonal().mean()
  }
}
__global__ void qep_reg_kernel(const double* __restrict__ gram, long long n,
                               const double* __restrict__ lam, double* __restrict__ a) {
  const double l = *lam;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n, j = e - i * n;
    a[e] = (i == j) ? gram[e] + l : gram[e];
  }
}

__global__ void qep_out_kernel(const float* __restrict__ w, const double* __restrict__ z,
                               long long count, double alpha, float* __restrict__ out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = float(double(w[e]) + alpha * z[e]);  // from_eigen(wd + alpha * correction)
}

}  // namespace

size_t qep_workspace_doubles(long long n, long long m) {
  const long long nblk = (n + 63) / 64;
  return size_t(2 * n * n + nblk * 64 * 64 + n * n + 2 * n * m + 2);
}

void qep_target_f64(const float* w, const double* gram, const double* cross, long long n,
                    long long m, double alpha, double eta, float* out, double* ws, int* flags,
                    unsigned* status, cudaStream_t st) {
  const long long nblk = (n + 63) / 64;
  double* a = ws;                   // n x n: reg, then L
  double* x = a + n * n;            // n x n: L^-1
  double* iws = x + n * n;          // inverse workspace
  double* b = iws + nblk * 64 * 64 + n * n;  // n x m
  double* y = b + n * m;            // n x m
  double* lam = y + n * m;          // 1
  count_launches(2);
  qep_lambda_kernel<<<1, 1024, 0, st>>>(gram, n, eta, lam);
  qep_reg_kernel<<<int(std::min<long long>((n * n + 255) / 256, 148 * 16)), 256, 0, st>>>(gram, n,
                                                                                      lam, a);
  // macro panels of 512 columns: short fp64 pivot chains, the trailing SYRKs on
  // the DMMA tensor cores (mm<double>)
  cholesky_g<double>(a, n, nullptr, nullptr, nullptr, nullptr, flags, status, 512, st);
  lower_inverse<double>(a, n, x, iws, st);
  gemm<double, double, float>(n, m, n, 1.0, cross, n, false, w, m, false, 0.0, b, m, false, st);
  // L^-1 is lower triangular: the tensor-core GEMMs skip the k range of its zeros
  gemm<double, double, double>(n, m, n, 1.0, x, n, false, b, m, false, 0.0, y, m, false, st, 1, 0,
                               0, 0, 1);
  gemm<double, double, double>(n, m, n, 1.0, x, n, true, y, m, false, 0.0, b, m, false, st, 1, 0,
                               0, 0, 2);
  count_launches(1);
  qep_out_kernel<<<int(std::min<long long>((n * m + 255) / 256, 148 * 16)), 256, 0, st>>>(
      w, b, n * m, alpha, out);
}

}  // namespace ocwg
