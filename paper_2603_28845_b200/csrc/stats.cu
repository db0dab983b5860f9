// Operand preparation for the tensor-core statistics (gram_tc.cu), plus
// small conversion / metric kernels.
//   split_bf16:   fp32 calibration inputs of the reference API
//                 (accumulate_stats, stats.cpp:10-19) -> bf16 parts
//                 X_hat = P1 + P2, X - X_hat = D1 + D2 for gram / cross;
//   pad_bf16:     bf16 rows to a TMA-legal row stride (multiple of 8);
//   accumulate_stats_f64: stats.cpp:10-19 in fp64 SIMT GEMMs (OCWG_FP64);
//   hessian_simt: fp64-accumulated X^T X of bf16 X, a test-only cross-check
//                 for the tcgen05 kernel.
#include <cuda_bf16.h>

#include "kernels.h"

namespace ocwg {
namespace {

inline int blocks_for(long long n) {
  long long g = (n + 255) / 256;
  return int(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

__global__ void diff_kernel(const float* __restrict__ xf, const float* __restrict__ xp, long long n,
                            double* d) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    d[e] = __dsub_rn(double(xf[e]), double(xp[e]));
}

__device__ inline float bf16_to_f32(uint16_t v) { return __uint_as_float(uint32_t(v) << 16); }

// 32x32 output tile per block, fp64 accumulation over all tokens
__global__ void hessian_simt_kernel(const uint16_t* __restrict__ x, long long t, long long d,
                                    float* h, int accumulate) {
  __shared__ float xa[32][33], xb[32][33];
  const long long i0 = (long long)blockIdx.y * 32, j0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  double acc[4] = {0, 0, 0, 0};
  for (long long k0 = 0; k0 < t; k0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const long long k = k0 + r;
      xa[r][tx] = (k < t && i0 + tx < d) ? bf16_to_f32(x[k * d + i0 + tx]) : 0.f;
      xb[r][tx] = (k < t && j0 + tx < d) ? bf16_to_f32(x[k * d + j0 + tx]) : 0.f;
    }
    __syncthreads();
    for (int kk = 0; kk < 32; ++kk)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        acc[q] += double(xa[kk][ty + 8 * q]) * double(xb[kk][tx]);
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < d && j < d) {
      float* p = h + i * d + j;
      *p = accumulate ? float(double(*p) + acc[q]) : float(acc[q]);
    }
  }
}

__device__ __forceinline__ uint16_t bf16_bits(float v) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}
__device__ __forceinline__ float bf16_val(uint16_t b) { return __uint_as_float(uint32_t(b) << 16); }

__global__ void split_bf16_kernel(const float* __restrict__ xp, const float* __restrict__ xf,
                                  long long rows, long long dim, long long ld, uint16_t* __restrict__ p1,
                                  uint16_t* __restrict__ p2, uint16_t* __restrict__ d1,
                                  uint16_t* __restrict__ d2, unsigned* flags) {
  bool inexact = false, dnz = false;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * ld;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / ld, c = e % ld;
    uint16_t a = 0, b = 0, u = 0, v = 0;
    if (c < dim) {
      const float x = xp[r * dim + c];
      a = bf16_bits(x);
      b = bf16_bits(__fsub_rn(x, bf16_val(a)));  // exact: x - bf16(x) fits fp32
      inexact |= b != 0;
      if (xf) {
        const double d = double(xf[r * dim + c]) - double(x);
        u = bf16_bits(float(d));
        v = bf16_bits(float(d - double(bf16_val(u))));
        dnz |= d != 0.0;
      }
    }
    p1[e] = a;
    p2[e] = b;
    if (xf) {
      d1[e] = u;
      d2[e] = v;
    }
  }
  // (an integer OR-reduction: nvcc 12.9 miscompiled the two-__any_sync form
  // of this epilogue into votes on the negated predicates)
  const unsigned f = __reduce_or_sync(0xffffffffu, (inexact ? 1u : 0u) | (dnz ? 2u : 0u));
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

__global__ void pad_bf16_kernel(const uint16_t* __restrict__ x, long long rows, long long dim,
                                long long ld, uint16_t* __restrict__ out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * ld;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / ld, c = e % ld;
    out[e] = c < dim ? x[r * dim + c] : uint16_t(0);
  }
}

__global__ void add_f32_to_f64_kernel(const float* __restrict__ in, long long n, double* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] += double(in[e]);
}

__global__ void f64_to_f32_kernel(const double* __restrict__ in, long long n, float* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = float(in[e]);
}
__global__ void f32_to_f64_kernel(const float* __restrict__ in, long long n, double* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = double(in[e]);
}

__global__ void delta_kernel(const float* __restrict__ w, const float* __restrict__ wh, long long n,
                             double* d) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    d[e] = __dsub_rn(double(wh[e]), double(w[e]));
}

// out = sum_e a[e]*b[e] (single block, fixed order -> deterministic)
__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
                           double* out) {
  __shared__ double part[32];
  double s = 0.0;
  for (long long e = threadIdx.x; e < n; e += blockDim.x) s += a[e] * b[e];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    *out = t;
  }
}

}  // namespace

// OCWG_FP64 precision: the reference's arithmetic class (fp64 SIMT GEMMs)
void accumulate_stats_f64(const float* x_fp, const float* x_pert, long long rows, long long dim,
                          double* gram, double* cross, double* diff_ws, cudaStream_t st) {
  gemm<double, float, float>(dim, dim, rows, 1.0, x_pert, dim, true, x_pert, dim, false, 1.0, gram,
                             dim, false, st);
  if (cross) {
    count_launches(1);
    diff_kernel<<<blocks_for(rows * dim), 256, 0, st>>>(x_fp, x_pert, rows * dim, diff_ws);
    gemm<double, float, double>(dim, dim, rows, 1.0, x_pert, dim, true, diff_ws, dim, false, 1.0,
                                cross, dim, false, st);
  }
}

void hessian_simt(const uint16_t* x, long long tokens, long long dim, float* h, int accumulate,
                  cudaStream_t st) {
  dim3 grid(unsigned((dim + 31) / 32), unsigned((dim + 31) / 32));
  count_launches(1);
  hessian_simt_kernel<<<grid, 256, 0, st>>>(x, tokens, dim, h, accumulate);
}

void launch_split_bf16(const float* xp, const float* xf, long long rows, long long dim, long long ld,
                       uint16_t* p1, uint16_t* p2, uint16_t* d1, uint16_t* d2, unsigned* flags,
                       cudaStream_t st) {
  count_launches(1);
  split_bf16_kernel<<<blocks_for(rows * ld), 256, 0, st>>>(xp, xf, rows, dim, ld, p1, p2, d1, d2,
                                                           flags);
}
void launch_pad_bf16(const uint16_t* x, long long rows, long long dim, long long ld, uint16_t* out,
                     cudaStream_t st) {
  count_launches(1);
  pad_bf16_kernel<<<blocks_for(rows * ld), 256, 0, st>>>(x, rows, dim, ld, out);
}
void launch_add_f32_to_f64(const float* in, long long n, double* out, cudaStream_t st) {
  count_launches(1);
  add_f32_to_f64_kernel<<<blocks_for(n), 256, 0, st>>>(in, n, out);
}
void launch_f64_to_f32(const double* in, long long n, float* out, cudaStream_t st) {
  count_launches(1);
  f64_to_f32_kernel<<<blocks_for(n), 256, 0, st>>>(in, n, out);
}
void launch_f32_to_f64(const float* in, long long n, double* out, cudaStream_t st) {
  count_launches(1);
  f32_to_f64_kernel<<<blocks_for(n), 256, 0, st>>>(in, n, out);
}

// ws: 2*n*m doubles
void activation_objective(const float* w, const float* w_hat, const float* h, long long n,
                          long long m, double* out_dev, double* ws, cudaStream_t st) {
  double* d = ws;
  double* hd = ws + n * m;
  count_launches(2);
  delta_kernel<<<blocks_for(n * m), 256, 0, st>>>(w, w_hat, n * m, d);
  gemm<double, float, double>(n, m, n, 1.0, h, n, false, d, m, false, 0.0, hd, m, false, st);
  dot_kernel<<<1, 1024, 0, st>>>(d, hd, n * m, out_dev);
}


// In-place transpose of an n x n fp64 matrix (column-major statistics from a
// caller, ocwg_set_stats_layout): one 32 x 32 tile pair per block, upper pairs.
__global__ void transpose_sq_f64_kernel(double* a, long long n) {
  __shared__ double t1[32][33], t2[32][33];
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;
  const int tx = threadIdx.x;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const long long i1 = (long long)bi * 32 + r, j1 = (long long)bj * 32 + tx;
    const long long i2 = (long long)bj * 32 + r, j2 = (long long)bi * 32 + tx;
    t1[r][tx] = (i1 < n && j1 < n) ? a[i1 * n + j1] : 0.0;
    t2[r][tx] = (i2 < n && j2 < n) ? a[i2 * n + j2] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const long long i1 = (long long)bi * 32 + r, j1 = (long long)bj * 32 + tx;
    const long long i2 = (long long)bj * 32 + r, j2 = (long long)bi * 32 + tx;
    if (i1 < n && j1 < n) a[i1 * n + j1] = t2[tx][r];
    if (i2 < n && j2 < n) a[i2 * n + j2] = t1[tx][r];
  }
}
void transpose_sq_f64(double* a, long long n, cudaStream_t st) {
  if (n <= 1) return;
  const unsigned nb = unsigned((n + 31) / 32);
  transpose_sq_f64_kernel<<<dim3(nb, nb), dim3(32, 8), 0, st>>>(a, n);
  count_launches(1);
}

}  // namespace ocwg
