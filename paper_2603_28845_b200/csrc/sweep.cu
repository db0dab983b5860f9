// GPTQ column-block sweep (replaces layerwise.cpp:62-91), templated on the
// compute type T (float default, double = the reference's arithmetic class).
//
// Reference orientation: W is n x m, rows = input indices processed in
// `order`, columns = output channels, mutually independent.  Per block of B
// rows [ib, ie):
//   in-block (this file): for i in block, for every column j:
//       code = q(float(wp[i,j]), grid[orig_i, j]);  err = (wp[i,j] - w_hat)/U[i,i]
//       wp[k,j] -= U[i,k]*err  for k in (i, ie)             (layerwise.cpp:68-83)
//   trailing (gemm.cu): wp[ie:, :] -= U[ib:ie, ie:]^T * E   (layerwise.cpp:85-90)
//
// In-block mapping: a CTA owns 32 columns (8 warps x 4); lane = cc + 4*rg
// keeps rows rg, rg+8, ... of its column in registers.  The row loop is
// fully unrolled (row li = 8t + o), so the owner lane's register index is a
// compile-time constant; the error is broadcast with one warp shuffle.  The
// U block, the processing->original row map and the block's grids are staged
// in shared memory once per block, off the sequential critical path.
#include "kernels.h"

namespace ocwg {
namespace {

constexpr int kCols = 32;  // columns per CTA

template <typename T>
__global__ void permute_rows_kernel(const float* __restrict__ w, long long n, long long m,
                                    long long ldw, const int32_t* __restrict__ order, T* wp) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * m;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / m, j = e % m;
    wp[e] = T(w[(long long)order[i] * ldw + j]);
  }
}

template <typename T>
__device__ __forceinline__ T err_of(T wv, float wh, T d);
template <>
__device__ __forceinline__ float err_of<float>(float wv, float wh, float d) {
  return __fdiv_rn(__fsub_rn(wv, wh), d);
}
template <>
__device__ __forceinline__ double err_of<double>(double wv, float wh, double d) {
  return __ddiv_rn(__dsub_rn(wv, double(wh)), d);  // (wp - double(w_hat)) / d  (:76-77)
}

template <typename T>
__device__ __forceinline__ T upd(T r, T u, T e);
template <>
__device__ __forceinline__ float upd<float>(float r, float u, float e) {
  return fmaf(-u, e, r);
}
template <>
__device__ __forceinline__ double upd<double>(double r, double u, double e) {
  return __dsub_rn(r, __dmul_rn(u, e));  // two roundings, like the reference (:79-83)
}

template <typename T, int RPT>
__global__ void __launch_bounds__(256) inblock_kernel(
    T* __restrict__ wp, long long n, long long m, const T* __restrict__ u,
    const int32_t* __restrict__ order, QCfg c, const float* __restrict__ scales,
    const int32_t* __restrict__ zeros, long long ib, int bsz, int16_t* __restrict__ codes,
    float* __restrict__ w_hat, long long ldo, T* __restrict__ err_out) {
  constexpr int B = 8 * RPT;
  extern __shared__ __align__(16) unsigned char smem[];
  T* us = reinterpret_cast<T*>(smem);                                   // B x (B+1)
  float* gs = reinterpret_cast<float*>(smem + sizeof(T) * B * (B + 1));  // B x kCols
  int* gz = reinterpret_cast<int*>(gs + B * kCols);                     // B x kCols
  int* og = gz + B * kCols;                                             // B

  const int tid = threadIdx.x;
  const long long j0 = (long long)blockIdx.x * kCols;
  for (int e = tid; e < B; e += 256) og[e] = e < bsz ? order[ib + e] : 0;
  for (int e = tid; e < B * B; e += 256) {
    const int li = e / B, lk = e % B;
    us[li * (B + 1) + lk] = (li < bsz && lk < bsz) ? u[(ib + li) * n + ib + lk] : T(0);
  }
  __syncthreads();
  for (int e = tid; e < B * kCols; e += 256) {
    const int li = e / kCols, cj = e % kCols;
    const long long jj = j0 + cj;
    float s = 1.0f;
    int z = 0;
    if (li < bsz && jj < m) {
      const long long g = group_of(c, og[li], jj);
      s = scales[g];
      z = zeros[g];
    }
    gs[e] = s;
    gz[e] = z;
  }
  __syncthreads();

  const int lane = tid & 31, warp = tid >> 5;
  const int cc = lane & 3, rg = lane >> 2;
  const int cj = warp * 4 + cc;
  const long long j = j0 + cj;
  const bool col_ok = j < m;
  T r[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int li = rg + 8 * t;
    r[t] = (col_ok && li < bsz) ? wp[(ib + li) * m + j] : T(0);
  }
  // Rows li = 8t + o.  r[] is rotated down by one slot after every group of
  // 8 rows, so the owner's value is always r[0] and every register index is
  // a compile-time constant while only the 8-row group body is unrolled
  // (keeps the kernel inside the instruction cache).
#pragma unroll 1
  for (int t = 0; t < RPT; ++t) {
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const int li = 8 * t + o;
      if (li >= bsz) break;
      T e = T(0);
      if (rg == o) {
        const float s = gs[li * kCols + cj];
        const int z = gz[li * kCols + cj];
        const int q = quantize_code(float(r[0]), s, z, c.qmin, c.qmax);  // row_f (:70)
        const float wh = dequantize_code(q, s, z);
        e = err_of<T>(r[0], wh, us[li * (B + 1) + li]);
        if (col_ok) {
          const long long orig = og[li];
          codes[orig * ldo + j] = int16_t(q);  // original row order (:75)
          if (w_hat) w_hat[orig * ldo + j] = wh;
          err_out[(long long)li * m + j] = e;
        }
      }
      e = __shfl_sync(0xffffffffu, e, cc + 4 * o);
      const T* urow = us + li * (B + 1) + rg + 8 * t;
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        if ((k > 0 || rg > o) && t + k < RPT) r[k] = upd<T>(r[k], urow[8 * k], e);
      }
    }
#pragma unroll
    for (int k = 0; k + 1 < RPT; ++k) r[k] = r[k + 1];
  }
}

template <typename T, int RPT>
constexpr int inblock_smem() {
  return int(sizeof(T)) * 8 * RPT * (8 * RPT + 1) + 8 * RPT * kCols * 8 + 8 * RPT * 4;
}

template <typename T, int RPT>
void launch_inblock(T* wp, long long n, long long m, const T* u, const int32_t* order,
                    const QCfg& c, const float* scales, const int32_t* zeros, long long ib, int bsz,
                    int16_t* codes, float* w_hat, long long ldo, T* err, cudaStream_t st) {
  static const bool attr = [] {
    cudaFuncSetAttribute(inblock_kernel<T, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         inblock_smem<T, RPT>());
    return true;
  }();
  (void)attr;
  const unsigned ctas = unsigned((m + kCols - 1) / kCols);
  count_launches(1);
  inblock_kernel<T, RPT><<<ctas, 256, inblock_smem<T, RPT>(), st>>>(
      wp, n, m, u, order, c, scales, zeros, ib, bsz, codes, w_hat, ldo, err);
}

}  // namespace

template <typename T>
void launch_permute_rows(const float* w, long long n, long long m, long long ldw,
                         const int32_t* order, T* wp, cudaStream_t st) {
  long long g = (n * m + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  count_launches(1);
  permute_rows_kernel<T><<<int(g < 1 ? 1 : g), 256, 0, st>>>(w, n, m, ldw, order, wp);
}

template <typename T>
void gptq_sweep(T* wp, long long n, long long m, const T* u, const int32_t* order, const QCfg& c,
                const float* scales, const int32_t* zeros, long long block, int16_t* codes,
                float* w_hat, long long ldo, T* err_ws, cudaStream_t st) {
  // block size is a pure re-association of the trailing update (SURVEY §0
  // item 11); blocks above 128 rows run as 128-row blocks.
  const long long B = block < 1 ? 1 : (block > kMaxSweepBlock ? kMaxSweepBlock : block);
  for (long long ib = 0; ib < n; ib += B) {
    const long long ie = std::min(n, ib + B);
    const int bsz = int(ie - ib);
    if (B <= 32)
      launch_inblock<T, 4>(wp, n, m, u, order, c, scales, zeros, ib, bsz, codes, w_hat, ldo, err_ws,
                           st);
    else if (B <= 64)
      launch_inblock<T, 8>(wp, n, m, u, order, c, scales, zeros, ib, bsz, codes, w_hat, ldo, err_ws,
                           st);
    else
      launch_inblock<T, 16>(wp, n, m, u, order, c, scales, zeros, ib, bsz, codes, w_hat, ldo,
                            err_ws, st);
    if (ie < n)
      mm<T>(n - ie, m, bsz, -1.0, u + ib * n + ie, n, true, err_ws, m, false, 1.0,
                    wp + ie * m, m, false, st);
  }
}

template void launch_permute_rows<float>(const float*, long long, long long, long long,
                                         const int32_t*, float*, cudaStream_t);
template void launch_permute_rows<double>(const float*, long long, long long, long long,
                                          const int32_t*, double*, cudaStream_t);
template void gptq_sweep<float>(float*, long long, long long, const float*, const int32_t*,
                                const QCfg&, const float*, const int32_t*, long long, int16_t*,
                                float*, long long, float*, cudaStream_t);
template void gptq_sweep<double>(double*, long long, long long, const double*, const int32_t*,
                                 const QCfg&, const float*, const int32_t*, long long, int16_t*,
                                 float*, long long, double*, cudaStream_t);

}  // namespace ocwg
