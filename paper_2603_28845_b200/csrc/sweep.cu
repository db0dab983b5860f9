// GPTQ column-block sweep (replaces layerwise.cpp:62-91), templated on the
// compute type T (float default, double = the reference's arithmetic class).
//
// Reference orientation: W is n x m, rows = input indices processed in
// `order`, columns = output channels, mutually independent.  The reference
// updates the working copy row by row,
//   err = (wp[i] - w_hat[i]) / U[i,i];  wp[k] -= U[i,k] * err   (k > i)
// which is, in closed form (factor.cu),
//   w_cur[k] = w[k] + sum_{i<k} G[k,i] * D[i],   D[i] = w[i] - w_hat[i],
// with G the unit-lower factor emitted by the Cholesky and w the ORIGINAL
// (permuted) row.  Per block of B rows [ib, ie):
//   in-block (inblock_g_kernel): for i in block: w_cur = w + acc; quantize;
//       D = w - w_hat; acc[k] += G[k,i] D  for the block's later rows k;
//   trailing: acc[ie + B':, :] += G[ie + B':, blk] * D[blk, :]  (tcgen05 3xTF32).
// Lookahead: the trailing update of block b skips block b+1's rows; block
// b+1's in-block kernel applies that slice itself (G[blk b+1, blk b] D_b)
// from shared memory.  In-block kernels run back to back on the calling
// stream while the trailing GEMMs run on an auxiliary stream:
//   inblock(b+1) needs inblock(b) (same stream) and trailing(b-1) (event);
//   trailing(b)  needs inblock(b) (event).
// acc needs no initialisation: trailing(0) writes it with beta = 0 and
// blocks 0 and 1 never read it.
//
// In-block mapping: a CTA owns 32 columns (8 warps x 4); lane = cc + 4*rg
// keeps rows rg, rg+8, ... of its column in registers (with the column's
// original weights, scales and zero points for those rows).  The 8-row group
// body is unrolled and the register arrays rotate by one slot per group, so
// every register index is a compile-time constant; D is broadcast with one
// warp shuffle.  The block's strictly-lower G is staged packed in shared
// memory; D is staged for a coalesced K-major store (the GEMM's B operand).
#include "kernels.h"

namespace ocwg {
namespace {

constexpr int kCols = 32;      // columns per CTA
constexpr int kB = 128;        // max rows per block (D stride)
constexpr int kLaChunk = 64;   // lookahead staging chunk (columns of G)

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t u = __float_as_uint(x);
  u = (u + 0xFFFu + ((u >> 13) & 1u)) & ~0x1FFFu;
  return __uint_as_float(u);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// asynchronous 4/8-byte global -> shared copy (LDGSTS): staging loops keep
// every load in flight instead of round-tripping through registers
template <typename T>
__device__ __forceinline__ void cp_async(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src),
               "n"(int(sizeof(T)))
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ void ld4(const T* p, T (&o)[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    o[0] = f.x, o[1] = f.y, o[2] = f.z, o[3] = f.w;
  } else {
    const double2 f0 = *reinterpret_cast<const double2*>(p);
    const double2 f1 = *reinterpret_cast<const double2*>(p + 2);
    o[0] = f0.x, o[1] = f0.y, o[2] = f1.x, o[3] = f1.y;
  }
}

__host__ __device__ constexpr int packed_off(int li) { return li * kB - li * (li + 1) / 2; }

template <typename T>
struct InblockSmem {
  union {
    T gs[packed_off(kB)];  // strictly-lower G block, column-packed: (k, li) at off(li)+k-li-1
    struct {
      T gc[kB][kLaChunk + 4];     // lookahead: G[ib + li][kprev + q0 + q]
      T dp[kCols][kLaChunk + 4];  // lookahead: D_prev[q0 + q] of column cj
    } la;
  } u;
  T ds[kCols][kB + 1];  // D of this block, staged for the K-major store
  int og[kB];           // processing -> original row of the block
};

template <typename T, int RPT>
__global__ void __launch_bounds__(256) inblock_g_kernel(
    const float* __restrict__ w, long long ldw, const int32_t* __restrict__ order,
    const T* __restrict__ acc, int use_acc, const T* __restrict__ gpl,
    const T* __restrict__ dprev, int bprev, T* __restrict__ dcur, float* __restrict__ dcur_hi,
    float* __restrict__ dcur_lo, QCfg c, const float* __restrict__ scales,
    const int32_t* __restrict__ zeros, long long n, long long m, long long ib, int bsz,
    int16_t* __restrict__ codes, float* __restrict__ w_hat, long long ldo) {
  extern __shared__ __align__(16) unsigned char smraw[];
  InblockSmem<T>& sm = *reinterpret_cast<InblockSmem<T>*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cc = lane & 3, rg = lane >> 2;
  const int cj = warp * 4 + cc;
  const long long j0 = (long long)blockIdx.x * kCols;
  const long long j = j0 + cj;
  const bool col_ok = j < m;

  for (int e = tid; e < kB; e += 256) sm.og[e] = e < bsz ? order[ib + e] : 0;
  __syncthreads();
  // ---- per-lane rows rg + 8t: current partial sums, original weights, grids
  T r[RPT];
  float w0[RPT], s[RPT];
  int z[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int li = rg + 8 * t;
    r[t] = T(0);
    w0[t] = 0.f;
    s[t] = 1.f;
    z[t] = 0;
    if (col_ok && li < bsz) {
      const long long orig = sm.og[li];
      w0[t] = w[orig * ldw + j];
      const long long g = group_of(c, orig, j);
      s[t] = scales[g];
      z[t] = zeros[g];
      if (use_acc) r[t] = acc[(ib + li) * m + j];
    }
  }

  // ---- lookahead: r += G[blk, prev blk] * D_prev  (the slice trailing(b-1) skipped)
  if (bprev > 0) {
    const long long kprev = ib - bprev;
    for (int q0 = 0; q0 < bprev; q0 += kLaChunk) {
      for (int e = tid; e < kB * kLaChunk; e += 256) {
        const int li = e / kLaChunk, q = e % kLaChunk;
        if (li < bsz && q0 + q < bprev)
          cp_async(&sm.u.la.gc[li][q], gpl + (ib + li) * n + kprev + q0 + q);
        else
          sm.u.la.gc[li][q] = T(0);
      }
      for (int e = tid; e < kCols * kLaChunk; e += 256) {
        const int cl = e / kLaChunk, q = e % kLaChunk;
        if (j0 + cl < m && q0 + q < bprev)
          cp_async(&sm.u.la.dp[cl][q], dprev + (j0 + cl) * kB + q0 + q);
        else
          sm.u.la.dp[cl][q] = T(0);
      }
      cp_async_wait_all();
      __syncthreads();
#pragma unroll 2
      for (int q = 0; q < kLaChunk; q += 4) {
        T dv[4];
        ld4(&sm.u.la.dp[cj][q], dv);
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
          T g[4];
          ld4(&sm.u.la.gc[rg + 8 * t][q], g);
          r[t] = fma(g[0], dv[0], r[t]);
          r[t] = fma(g[1], dv[1], r[t]);
          r[t] = fma(g[2], dv[2], r[t]);
          r[t] = fma(g[3], dv[3], r[t]);
        }
      }
      __syncthreads();
    }
  }

  // ---- stage the block's strictly-lower G (packed by column)
  for (int k = 1 + warp; k < bsz; k += 8)
    for (int li = lane; li < k; li += 32)
      cp_async(&sm.u.gs[packed_off(li) + k - li - 1], gpl + (ib + k) * n + ib + li);
  cp_async_wait_all();
  __syncthreads();

  // ---- sequential rows li = 8t + o; owner lane rg == o holds the row in slot 0
#pragma unroll 1
  for (int t = 0; t < RPT; ++t) {
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const int li = 8 * t + o;
      if (li >= bsz) break;
      T d = T(0);
      if (rg == o) {
        const T cur = T(w0[0]) + r[0];  // w_cur = w + sum G D
        const int q = quantize_code(float(cur), s[0], z[0], c.qmin, c.qmax);  // row_f (:70)
        const float wh = dequantize_code(q, s[0], z[0]);
        d = T(w0[0]) - T(wh);
        if (col_ok) {
          const long long orig = sm.og[li];
          codes[orig * ldo + j] = int16_t(q);  // original row order (:75)
          if (w_hat) w_hat[orig * ldo + j] = wh;
        }
        sm.ds[cj][li] = d;
      }
      d = __shfl_sync(0xffffffffu, d, cc + 4 * o);
      const T* gcol = sm.u.gs + packed_off(li) - li - 1;  // gcol[k] = G[k][li]
#pragma unroll
      for (int kk = 0; kk < RPT; ++kk) {
        const int row = rg + 8 * (t + kk);
        if ((kk > 0 || rg > o) && t + kk < RPT && row < bsz) r[kk] = fma(gcol[row], d, r[kk]);
      }
    }
#pragma unroll
    for (int k = 0; k + 1 < RPT; ++k) {
      r[k] = r[k + 1];
      w0[k] = w0[k + 1];
      s[k] = s[k + 1];
      z[k] = z[k + 1];
    }
  }
  __syncthreads();
  // ---- D (K-major: column j's kB values contiguous): plain, and the tf32
  // hi/lo split the tensor-core GEMM consumes
  for (int e = tid; e < kCols * kB; e += 256) {
    const int cl = e / kB, li = e % kB;
    if (j0 + cl >= m) continue;
    const T v = li < bsz ? sm.ds[cl][li] : T(0);
    const long long off = (j0 + cl) * kB + li;
    dcur[off] = v;
    if (dcur_hi) {
      const float hi = tf32_hi(float(v));
      dcur_hi[off] = hi;
      dcur_lo[off] = float(v) - hi;
    }
  }
}

template <typename T, int RPT>
void launch_inblock(const float* w, long long ldw, const int32_t* order, const T* acc, int use_acc,
                    const T* gpl, const T* dprev, int bprev, T* dcur, float* dch, float* dcl,
                    const QCfg& c, const float* scales, const int32_t* zeros, long long n,
                    long long m, long long ib, int bsz, int16_t* codes, float* w_hat, long long ldo,
                    cudaStream_t st) {
  static const bool attr = [] {
    cudaFuncSetAttribute(inblock_g_kernel<T, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(InblockSmem<T>)));
    return true;
  }();
  (void)attr;
  const unsigned ctas = unsigned((m + kCols - 1) / kCols);
  count_launches(1);
  inblock_g_kernel<T, RPT><<<ctas, 256, sizeof(InblockSmem<T>), st>>>(
      w, ldw, order, acc, use_acc, gpl, dprev, bprev, dcur, dch, dcl, c, scales, zeros, n, m, ib,
      bsz, codes, w_hat, ldo);
}

}  // namespace

size_t sweep_delta_elems(long long m) { return size_t(m) * kB; }

template <typename T>
void gptq_sweep_g(const float* w, long long ldw, long long n, long long m, const T* gpl,
                  const T* ghi, const float* glo, const int32_t* order, const QCfg& c,
                  const float* scales, const int32_t* zeros, long long block, int16_t* codes,
                  float* w_hat, long long ldo, T* acc, T* const dpl[2], float* const dhi[2],
                  float* const dlo[2], cudaStream_t st, cudaStream_t aux, cudaEvent_t* ev) {
  // block size is a pure re-association of the trailing update (SURVEY §0
  // item 11); blocks above 128 rows run as 128-row blocks.
  const long long B = block < 1 ? 1 : (block > kB ? kB : block);
  const long long nb = (n + B - 1) / B;
  const bool split = glo != nullptr;
  // ev: [0] fork, [1] in-block done, [2..3] trailing done (by block parity), [4] join
  cudaEventRecord(ev[0], st);
  cudaStreamWaitEvent(aux, ev[0], 0);
  for (long long b = 0; b < nb; ++b) {
    const long long ib = b * B, ie = std::min(n, ib + B);
    const int bsz = int(ie - ib);
    const int p = int(b & 1);
    if (b >= 2) cudaStreamWaitEvent(st, ev[2 + p], 0);  // trailing(b-2) done
    const int bprev = b > 0 ? int(B) : 0;
    const T* dprev = b > 0 ? dpl[p ^ 1] : nullptr;
    float* dch = split ? dhi[p] : nullptr;
    float* dcl = split ? dlo[p] : nullptr;
    if (B <= 32)
      launch_inblock<T, 4>(w, ldw, order, acc, b >= 2, gpl, dprev, bprev, dpl[p], dch, dcl, c,
                           scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, st);
    else if (B <= 64)
      launch_inblock<T, 8>(w, ldw, order, acc, b >= 2, gpl, dprev, bprev, dpl[p], dch, dcl, c,
                           scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, st);
    else
      launch_inblock<T, 16>(w, ldw, order, acc, b >= 2, gpl, dprev, bprev, dpl[p], dch, dcl, c,
                            scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, st);
    // trailing(b): rows [ie + next, n) -- block b+1 takes its slice by lookahead
    const long long r0 = std::min(n, ie + B);
    if (r0 < n) {
      cudaEventRecord(ev[1], st);
      cudaStreamWaitEvent(aux, ev[1], 0);
      const double beta = b == 0 ? 0.0 : 1.0;
      bool done = false;
      if constexpr (sizeof(T) == 4) {
        if (split)
          done = tc_gemm_presplit(n - r0, m, bsz, 1.0f, reinterpret_cast<const float*>(ghi) + r0 * n + ib,
                                  glo + r0 * n + ib, n, dhi[p], dlo[p], kB, float(beta),
                                  reinterpret_cast<float*>(acc) + r0 * m, m, aux);
      }
      if (!done)
        gemm<T, T, T>(n - r0, m, bsz, 1.0, gpl + r0 * n + ib, n, false, dpl[p], kB, true, beta,
                      acc + r0 * m, m, false, aux);
      cudaEventRecord(ev[2 + p], aux);
    }
  }
  cudaEventRecord(ev[4], aux);
  cudaStreamWaitEvent(st, ev[4], 0);
}

template void gptq_sweep_g<float>(const float*, long long, long long, long long, const float*,
                                  const float*, const float*, const int32_t*, const QCfg&,
                                  const float*, const int32_t*, long long, int16_t*, float*,
                                  long long, float*, float* const[2], float* const[2],
                                  float* const[2], cudaStream_t, cudaStream_t, cudaEvent_t*);
template void gptq_sweep_g<double>(const float*, long long, long long, long long, const double*,
                                   const double*, const float*, const int32_t*, const QCfg&,
                                   const float*, const int32_t*, long long, int16_t*, float*,
                                   long long, double*, double* const[2], float* const[2],
                                   float* const[2], cudaStream_t, cudaStream_t, cudaEvent_t*);

}  // namespace ocwg
