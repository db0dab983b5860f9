// GPTQ column-block sweep (replaces layerwise.cpp:62-91).
//
// Reference orientation: W is n x m, rows = input indices processed in
// `order`, columns = output channels, mutually independent.  Per block of B
// rows [ib, ie):
//   in-block  (this file): for i in block, for every column j:
//       code = q(float(wp[i,j]), grid[orig_i, j]);  err = (wp[i,j] - w_hat)/U[i,i]
//       wp[k,j] -= U[i,k]*err  for k in (i, ie)            (layerwise.cpp:68-83)
//   trailing  (fp64 GEMM): wp[ie:, :] -= U[ib:ie, ie:]^T * E (layerwise.cpp:85-90)
//
// In-block mapping: one warp owns 4 columns; lane = cc + 4*rg holds rows
// rg, rg+8, ... of the block for column cc in registers, so the per-row error
// is broadcast with a warp shuffle and no block-wide barrier is needed.
#include "kernels.h"

namespace ocwg {
namespace {

constexpr int kRPT = 16;          // rows per lane -> blocks up to 8*16 = 128 rows
constexpr int kMaxBlock = 8 * kRPT;
constexpr int kWarps = 4;         // warps per CTA (16 columns)

__global__ void permute_rows_kernel(const float* __restrict__ w, long long n, long long m,
                                    long long ldw, const int32_t* __restrict__ order, double* wp) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * m;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / m, j = e % m;
    wp[e] = double(w[(long long)order[i] * ldw + j]);
  }
}

__global__ void __launch_bounds__(32 * kWarps) inblock_kernel(
    double* __restrict__ wp, long long n, long long m, const double* __restrict__ u,
    const int32_t* __restrict__ order, QCfg c, const float* __restrict__ scales,
    const int32_t* __restrict__ zeros, long long ib, int bsz, int16_t* __restrict__ codes,
    float* __restrict__ w_hat, long long ldo, double* __restrict__ err_out) {
  const int lane = int(threadIdx.x & 31);
  const int cc = lane & 3, rg = lane >> 2;
  const long long j = ((long long)blockIdx.x * kWarps + (threadIdx.x >> 5)) * 4 + cc;
  const bool col_ok = j < m;
  double r[kRPT];
#pragma unroll
  for (int t = 0; t < kRPT; ++t) {
    const int li = rg + 8 * t;
    r[t] = (col_ok && li < bsz) ? wp[(ib + li) * m + j] : 0.0;
  }
  for (int li = 0; li < bsz; ++li) {
    const long long i = ib + li;
    const int owner_rg = li & 7, owner_t = li >> 3;
    double e = 0.0;
    if (rg == owner_rg && col_ok) {
      double wv = 0.0;
#pragma unroll
      for (int t = 0; t < kRPT; ++t)
        if (t == owner_t) wv = r[t];
      const long long orig = order[i];
      const long long g = group_of(c, orig, j);
      const float s = scales[g];
      const int z = zeros[g];
      const int q = quantize_code(float(wv), s, z, c.qmin, c.qmax);   // row_f (layerwise.cpp:70)
      const float wh = dequantize_code(q, s, z);
      codes[orig * ldo + j] = int16_t(q);                               // original order (:75)
      if (w_hat) w_hat[orig * ldo + j] = wh;
      e = __ddiv_rn(__dsub_rn(wv, double(wh)), u[i * n + i]);           // (:76-77)
      err_out[(long long)li * m + j] = e;
    }
    e = __shfl_sync(0xffffffffu, e, cc + 4 * owner_rg);
    // in-block rank-1 update (layerwise.cpp:79-83): two roundings like the ref
#pragma unroll
    for (int t = 0; t < kRPT; ++t) {
      const int lk = rg + 8 * t;
      if (lk > li && lk < bsz) r[t] = __dsub_rn(r[t], __dmul_rn(u[i * n + ib + lk], e));
    }
  }
}

}  // namespace

void launch_permute_rows_f64(const float* w, long long n, long long m, long long ldw,
                             const int32_t* order, double* wp, cudaStream_t st) {
  long long g = (n * m + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  count_launches(1);
  permute_rows_kernel<<<int(g < 1 ? 1 : g), 256, 0, st>>>(w, n, m, ldw, order, wp);
}

void gptq_sweep(double* wp, long long n, long long m, const double* u, const int32_t* order,
                const QCfg& c, const float* scales, const int32_t* zeros, long long block,
                int16_t* codes, float* w_hat, long long ldo, double* err_ws, cudaStream_t st) {
  // block size is a pure re-association of the trailing update (SURVEY §0
  // item 11); blocks above 128 rows are run as 128-row blocks.
  const long long B = block < 1 ? 1 : (block > kMaxBlock ? kMaxBlock : block);
  const long long ctas = (m + 4 * kWarps - 1) / (4 * kWarps);
  for (long long ib = 0; ib < n; ib += B) {
    const long long ie = std::min(n, ib + B);
    const int bsz = int(ie - ib);
    count_launches(1);
    inblock_kernel<<<unsigned(ctas), 32 * kWarps, 0, st>>>(wp, n, m, u, order, c, scales, zeros, ib,
                                                           bsz, codes, w_hat, ldo, err_ws);
    if (ie < n)
      dgemm<double, double>(n - ie, m, bsz, -1.0, u + ib * n + ie, n, true, err_ws, m, false, 1.0,
                            wp + ie * m, m, false, st);
  }
}

}  // namespace ocwg
