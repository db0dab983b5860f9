// FP64 SIMT GEMM used by the factorisation and by the GPTQ trailing update.
// The reference does all of GPTQ in fp64 (Eigen MatrixXd, layerwise.cpp:31-90);
// B200 keeps a full-rate FP64 pipe, so the fp64 contractions stay fp64 here.
//
// Tile 64x64, BK 16, 256 threads, 4x4 outputs per thread with a strided
// (16-apart) thread->element mapping so shared-memory reads broadcast; A/B
// tiles are double-buffered through registers.
#include "kernels.h"

namespace ocwg {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename T>
__device__ inline double ld(const T* p) { return double(__ldg(p)); }

template <typename TA, typename TB>
__global__ void __launch_bounds__(256) dgemm_kernel(long long m, long long n, long long k,
                                                    double alpha, const TA* __restrict__ a,
                                                    long long lda, int ta,
                                                    const TB* __restrict__ b, long long ldb,
                                                    int tb, double beta, double* __restrict__ c,
                                                    long long ldc, int lower_only) {
  const long long row0 = (long long)blockIdx.y * BM, col0 = (long long)blockIdx.x * BN;
  if (lower_only && col0 > row0 + BM - 1) return;
  __shared__ double As[2][BK][BM + 1];
  __shared__ double Bs[2][BK][BN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  double ra[4], rb[4];
  auto load_a = [&](long long k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = tid + q * 256;
      int ii, kk;
      if (ta) { ii = l % BM; kk = l / BM; } else { ii = l / BK; kk = l % BK; }
      const long long gi = row0 + ii, gk = k0 + kk;
      double v = 0.0;
      if (gi < m && gk < k) v = ta ? ld(a + gk * lda + gi) : ld(a + gi * lda + gk);
      ra[q] = v;
    }
  };
  auto load_b = [&](long long k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = tid + q * 256;
      int jj, kk;
      if (tb) { jj = l / BK; kk = l % BK; } else { jj = l % BN; kk = l / BN; }
      const long long gj = col0 + jj, gk = k0 + kk;
      double v = 0.0;
      if (gj < n && gk < k) v = tb ? ld(b + gj * ldb + gk) : ld(b + gk * ldb + gj);
      rb[q] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = tid + q * 256;
      int ii, kk;
      if (ta) { ii = l % BM; kk = l / BM; } else { ii = l / BK; kk = l % BK; }
      As[buf][kk][ii] = ra[q];
      int jj, kb;
      if (tb) { jj = l / BK; kb = l % BK; } else { jj = l % BN; kb = l / BN; }
      Bs[buf][kb][jj] = rb[q];
    }
  };

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  const long long nk = (k + BK - 1) / BK;
  if (nk > 0) {
    load_a(0);
    load_b(0);
    store(0);
  }
  __syncthreads();
  for (long long kt = 0; kt < nk; ++kt) {
    const int buf = int(kt & 1);
    if (kt + 1 < nk) {
      load_a((kt + 1) * BK);
      load_b((kt + 1) * BK);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long gi = row0 + ty + 16 * i;
    if (gi >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long gj = col0 + tx + 16 * j;
      if (gj >= n) continue;
      double* p = c + gi * ldc + gj;
      *p = beta == 0.0 ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *p);
    }
  }
}

}  // namespace

template <typename TA, typename TB>
void dgemm(long long m, long long n, long long k, double alpha, const TA* a, long long lda, bool ta,
           const TB* b, long long ldb, bool tb, double beta, double* c, long long ldc,
           bool lower_only, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  dim3 grid(unsigned((n + BN - 1) / BN), unsigned((m + BM - 1) / BM));
  count_launches(1);
  dgemm_kernel<TA, TB><<<grid, 256, 0, st>>>(m, n, k, alpha, a, lda, ta ? 1 : 0, b, ldb, tb ? 1 : 0,
                                              beta, c, ldc, lower_only ? 1 : 0);
}

template void dgemm<double, double>(long long, long long, long long, double, const double*,
                                    long long, bool, const double*, long long, bool, double,
                                    double*, long long, bool, cudaStream_t);
template void dgemm<float, float>(long long, long long, long long, double, const float*, long long,
                                  bool, const float*, long long, bool, double, double*, long long,
                                  bool, cudaStream_t);
template void dgemm<float, double>(long long, long long, long long, double, const float*,
                                   long long, bool, const double*, long long, bool, double, double*,
                                   long long, bool, cudaStream_t);

}  // namespace ocwg
