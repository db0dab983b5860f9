// SIMT GEMM for the factorisation and the GPTQ trailing update, templated on
// the compute type T (float: default fast path; double: reference-exact
// arithmetic class, the reference runs GPTQ in Eigen MatrixXd).
//
//   C[m x n] = beta*C + alpha * op(A) * op(B)
//   op(A)[i][k] = ta ? A[k*lda + i] : A[i*lda + k]   (same for B with tb)
//
// fp32: 128x128 CTA tile, BK 8, 256 threads, 8x8 outputs per thread.
// fp64: 64x64 CTA tile, BK 16, 256 threads, 4x4 outputs per thread.
// Thread->element mapping is strided so shared-memory reads broadcast;
// tiles are double buffered through registers.
#include <algorithm>

#include "kernels.h"

namespace ocwg {
namespace {

template <typename T>
struct Tile;
template <>
struct Tile<float> {
  static constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;
};
template <>
struct Tile<double> {
  static constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
};

template <typename T, typename S>
__device__ __forceinline__ T ldg_as(const S* p) {
  return T(__ldg(p));
}

template <typename T, typename TA, typename TB>
__global__ void __launch_bounds__(256) gemm_kernel(long long m, long long n, long long k, T alpha,
                                                   const TA* __restrict__ a, long long lda, int ta,
                                                   const TB* __restrict__ b, long long ldb, int tb,
                                                   T beta, T* __restrict__ c, long long ldc,
                                                   int lower_only, long long sa, long long sb,
                                                   long long sc) {
  a += (long long)blockIdx.z * sa;
  b += (long long)blockIdx.z * sb;
  c += (long long)blockIdx.z * sc;
  constexpr int BM = Tile<T>::BM, BN = Tile<T>::BN, BK = Tile<T>::BK;
  constexpr int TM = Tile<T>::TM, TN = Tile<T>::TN;
  constexpr int TX = BN / TN, TY = BM / TM;  // 16 x 16 threads
  static_assert(TX * TY == 256, "256 threads");
  constexpr int LA = BM * BK / 256, LB = BN * BK / 256;  // loads per thread per k-tile
  const long long row0 = (long long)blockIdx.y * BM, col0 = (long long)blockIdx.x * BN;
  if (lower_only && col0 > row0 + BM - 1) return;
  __shared__ T As[2][BK][BM + 4];
  __shared__ T Bs[2][BK][BN + 4];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;

  T ra[LA], rb[LB];
  auto load = [&](long long k0) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int l = tid + q * 256;
      int ii, kk;
      if (ta) { ii = l % BM; kk = l / BM; } else { ii = l / BK; kk = l % BK; }
      const long long gi = row0 + ii, gk = k0 + kk;
      T v = T(0);
      if (gi < m && gk < k) v = ta ? ldg_as<T>(a + gk * lda + gi) : ldg_as<T>(a + gi * lda + gk);
      ra[q] = v;
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int l = tid + q * 256;
      int jj, kk;
      if (tb) { jj = l / BK; kk = l % BK; } else { jj = l % BN; kk = l / BN; }
      const long long gj = col0 + jj, gk = k0 + kk;
      T v = T(0);
      if (gj < n && gk < k) v = tb ? ldg_as<T>(b + gj * ldb + gk) : ldg_as<T>(b + gk * ldb + gj);
      rb[q] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int l = tid + q * 256;
      int ii, kk;
      if (ta) { ii = l % BM; kk = l / BM; } else { ii = l / BK; kk = l % BK; }
      As[buf][kk][ii] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int l = tid + q * 256;
      int jj, kk;
      if (tb) { jj = l / BK; kk = l % BK; } else { jj = l % BN; kk = l / BN; }
      Bs[buf][kk][jj] = rb[q];
    }
  };

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  const long long nk = (k + BK - 1) / BK;
  if (nk > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (long long kt = 0; kt < nk; ++kt) {
    const int buf = int(kt & 1);
    if (kt + 1 < nk) load((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty + TY * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx + TX * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const long long gi = row0 + ty + TY * i;
    if (gi >= m) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const long long gj = col0 + tx + TX * j;
      if (gj >= n) continue;
      T* p = c + gi * ldc + gj;
      *p = beta == T(0) ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *p);
    }
  }
}

// fp64 on the tensor cores (DMMA, mma.sync m8n8k4 .f64 -- tcgen05 has no fp64
// kind): 128 x 128 CTA tile, BK 16, 32 warps as 4 x 8, each warp a 32 x 16
// block = 4 x 2 m8n8 accumulators (16 doubles per lane).  The kernel is
// latency bound: 32 warps beat 16 warps of 32 x 32 (5-15 % on the factor and
// sweep shapes, equal on square 4096) and 8 warps of 64 x 32 (-12 %), see
// profiles/r02_dmma_threads_ab.log.  Operands are staged through registers (any transposition, fp32
// inputs widened exactly) into double-buffered shared tiles stored [row][k]
// for A and [col][k] for B, so a fragment is one 8-byte load per lane; the row
// stride of 20 doubles puts a half-warp's fragment loads on distinct banks.
constexpr int DBM = 128, DBN = 128, DBK = 16, DPAD = 4, DTHREADS = 1024;
constexpr int kDmmaSmem = 2 * (DBM + DBN) * (DBK + DPAD) * 8;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <typename TA, typename TB>
__global__ void __launch_bounds__(DTHREADS, 1) gemm_f64_dmma_kernel(
    long long m, long long n, long long k, double alpha, const TA* __restrict__ a, long long lda,
    int ta, const TB* __restrict__ b, long long ldb, int tb, double beta, double* __restrict__ c,
    long long ldc, int lower_only, long long sa, long long sb, long long sc, int tri) {
  a += (long long)blockIdx.z * sa;
  b += (long long)blockIdx.z * sb;
  c += (long long)blockIdx.z * sc;
  const long long row0 = (long long)blockIdx.y * DBM, col0 = (long long)blockIdx.x * DBN;
  if (lower_only && col0 > row0 + DBM - 1) return;
  // triangular op(A) (tri 1: lower, 2: upper): only the k range that can be nonzero
  const long long kbeg = tri == 2 ? row0 / DBK * DBK : 0;
  const long long kend = tri == 1 ? std::min(k, row0 + DBM) : k;
  extern __shared__ __align__(16) double dsm[];
  double (*As)[DBM][DBK + DPAD] = reinterpret_cast<double (*)[DBM][DBK + DPAD]>(dsm);
  double (*Bs)[DBN][DBK + DPAD] =
      reinterpret_cast<double (*)[DBN][DBK + DPAD]>(dsm + 2 * DBM * (DBK + DPAD));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int WN = 16, NJ = WN / 8;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * WN;
  constexpr int LA = DBM * DBK / DTHREADS, LB = DBN * DBK / DTHREADS;
  double ra[LA], rb[LB];
  auto load = [&](long long k0) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int l = tid + q * DTHREADS;
      const int i = ta ? l % DBM : l / DBK, kk = ta ? l / DBM : l % DBK;
      const long long gi = row0 + i, gk = k0 + kk;
      ra[q] = (gi < m && gk < kend) ? double(ta ? __ldg(a + gk * lda + gi) : __ldg(a + gi * lda + gk))
                                    : 0.0;
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int l = tid + q * DTHREADS;
      const int j = tb ? l / DBK : l % DBN, kk = tb ? l % DBK : l / DBN;
      const long long gj = col0 + j, gk = k0 + kk;
      rb[q] = (gj < n && gk < kend) ? double(tb ? __ldg(b + gj * ldb + gk) : __ldg(b + gk * ldb + gj))
                                    : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int l = tid + q * DTHREADS;
      const int i = ta ? l % DBM : l / DBK, kk = ta ? l / DBM : l % DBK;
      As[buf][i][kk] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int l = tid + q * DTHREADS;
      const int j = tb ? l / DBK : l % DBN, kk = tb ? l % DBK : l / DBN;
      Bs[buf][j][kk] = rb[q];
    }
  };
  double acc[4][NJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const long long nk = kend > kbeg ? (kend - kbeg + DBK - 1) / DBK : 0;
  if (nk > 0) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  const int fr = lane >> 2, fk = lane & 3;
  for (long long kt = 0; kt < nk; ++kt) {
    const int buf = int(kt & 1);
    if (kt + 1 < nk) load(kbeg + (kt + 1) * DBK);
#pragma unroll
    for (int kq = 0; kq < DBK; kq += 4) {
      double av[4], bv[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[buf][wm + 8 * i + fr][kq + fk];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bv[j] = Bs[buf][wn + 8 * j + fr][kq + fk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], av[i], bv[j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long gi = row0 + wm + 8 * i + fr;
    if (gi >= m) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long long gj = col0 + wn + 8 * j + 2 * fk + e;
        if (gj >= n) continue;
        double* p = c + gi * ldc + gj;
        *p = beta == 0.0 ? alpha * acc[i][j][e] : fma(alpha, acc[i][j][e], beta * *p);
      }
  }
}

}  // namespace

template <typename T, typename TA, typename TB>
void gemm(long long m, long long n, long long k, double alpha, const TA* a, long long lda, bool ta,
          const TB* b, long long ldb, bool tb, double beta, T* c, long long ldc, bool lower_only,
          cudaStream_t st, int batch, long long sa, long long sb, long long sc, int tri) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  if constexpr (sizeof(T) == 8) {
    // fp64 on the DMMA tensor cores once a 128 x 128 tile is reasonably filled
    if (m >= 64 && n >= 64 && k >= 8) {
      cudaFuncSetAttribute(gemm_f64_dmma_kernel<TA, TB>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kDmmaSmem);
      dim3 grid(unsigned((n + DBN - 1) / DBN), unsigned((m + DBM - 1) / DBM), unsigned(batch));
      count_launches(1);
      gemm_f64_dmma_kernel<TA, TB><<<grid, DTHREADS, kDmmaSmem, st>>>(
          m, n, k, alpha, a, lda, ta ? 1 : 0, b, ldb, tb ? 1 : 0, beta, c, ldc,
          lower_only ? 1 : 0, sa, sb, sc, tri);
      return;
    }
  }
  (void)tri;  // (the SIMT path multiplies the zeros)
  constexpr int BM = Tile<T>::BM, BN = Tile<T>::BN;
  dim3 grid(unsigned((n + BN - 1) / BN), unsigned((m + BM - 1) / BM), unsigned(batch));
  count_launches(1);
  gemm_kernel<T, TA, TB><<<grid, 256, 0, st>>>(m, n, k, T(alpha), a, lda, ta ? 1 : 0, b, ldb,
                                               tb ? 1 : 0, T(beta), c, ldc, lower_only ? 1 : 0, sa,
                                               sb, sc);
}

namespace {
thread_local float* g_tc_ws = nullptr;
thread_local size_t g_tc_ws_floats = 0;
}  // namespace

void set_tc_workspace(float* ws, size_t floats) {
  g_tc_ws = ws;
  g_tc_ws_floats = floats;
}

template <>
void mm<float>(long long m, long long n, long long k, double alpha, const float* a, long long lda,
               bool ta, const float* b, long long ldb, bool tb, double beta, float* c,
               long long ldc, bool lower_only, cudaStream_t st, int batch, long long sa,
               long long sb, long long sc) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  // tiny problems are latency bound: the SIMT kernel is one launch, the tensor
  // core path is three (split A, split B, MMA)
  const bool big = double(m) * double(n) * double(k) * batch >= double(1 << 22);
  if (g_tc_ws && k > 0 && big &&
      tc_gemm_tf32x3(batch, m, n, k, float(alpha), a, lda, sa, ta, b, ldb, sb, tb, float(beta), c,
                     ldc, sc, lower_only, g_tc_ws, g_tc_ws_floats, st))
    return;
  gemm<float, float, float>(m, n, k, alpha, a, lda, ta, b, ldb, tb, beta, c, ldc, lower_only, st,
                            batch, sa, sb, sc);
}

template <>
void mm<double>(long long m, long long n, long long k, double alpha, const double* a,
                long long lda, bool ta, const double* b, long long ldb, bool tb, double beta,
                double* c, long long ldc, bool lower_only, cudaStream_t st, int batch,
                long long sa, long long sb, long long sc) {
  gemm<double, double, double>(m, n, k, alpha, a, lda, ta, b, ldb, tb, beta, c, ldc, lower_only,
                               st, batch, sa, sb, sc);
}

#define OCWG_GEMM_INST(T, TA, TB)                                                              \
  template void gemm<T, TA, TB>(long long, long long, long long, double, const TA*, long long, \
                                bool, const TB*, long long, bool, double, T*, long long, bool, \
                                cudaStream_t, int, long long, long long, long long, int);
OCWG_GEMM_INST(double, double, double)
OCWG_GEMM_INST(double, float, float)
OCWG_GEMM_INST(double, float, double)
OCWG_GEMM_INST(double, double, float)
OCWG_GEMM_INST(float, float, float)

}  // namespace ocwg
