// QEP target correction (replaces layerwise.cpp:95-112, row f1 of SURVEY §8):
//   lambda = eta * mean(diag(gram));  W* = W + alpha * (gram + lambda I)^-1 (cross W)
// in fp64 like the reference (Eigen LLT + solve), on the GPU: the tile
// Cholesky of factor.cu in natural order, L^-1 by recursive doubling, and
// three fp64 GEMMs (cross W, L^-1 B, L^-T Y).  Non-PD -> kFlagNotPD.
#include "kernels.h"

namespace ocwg {
namespace {

__global__ void qep_reg_kernel(const double* __restrict__ gram, long long n, double eta,
                               double* __restrict__ a) {
  __shared__ double part[32];
  __shared__ double lam;
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += gram[i * n + i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    lam = eta * (t / double(n));  // stats.gram.diagonal().mean()
  }
  __syncthreads();
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n, j = e % n;
    a[e] = (i == j) ? gram[e] + lam : gram[e];
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
  return size_t(2 * n * n + nblk * 64 * 64 + n * n + 2 * n * m);
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
  count_launches(1);
  // one CTA: the diagonal mean must be complete before the copy (grid-stride)
  qep_reg_kernel<<<1, 1024, 0, st>>>(gram, n, eta, a);
  cholesky_g<double>(a, n, nullptr, nullptr, nullptr, nullptr, flags, status, 0, st);
  lower_inverse<double>(a, n, x, iws, st);
  gemm<double, double, float>(n, m, n, 1.0, cross, n, false, w, m, false, 0.0, b, m, false, st);
  gemm<double, double, double>(n, m, n, 1.0, x, n, false, b, m, false, 0.0, y, m, false, st);
  gemm<double, double, double>(n, m, n, 1.0, x, n, true, y, m, false, 0.0, b, m, false, st);
  count_launches(1);
  qep_out_kernel<<<int(std::min<long long>((n * m + 255) / 256, 148 * 16)), 256, 0, st>>>(
      w, b, n * m, alpha, out);
}

}  // namespace ocwg
