// HBM-bound quantisation kernels: grid calibration, RTN quantise/dequantise,
// OCW1 uniform payload pack/unpack and the act-order sort.
// Reference: proj/src/quant.cpp, proj/src/container.cpp:15-35,129-139,168-199,
// proj/src/layerwise.cpp:11-18.
#include <cfloat>
#include <cmath>

#include <type_traits>

#include "kernels.h"

namespace ocwg {

namespace {

constexpr int kWarpsPerBlock = 8;

// warp-wide min/max of one segment w[base + k*stride], k < len
struct Seg {
  long long base, stride, len;
};

__device__ inline Seg segment_of(long long g, long long rows, long long cols, long long ld,
                                const QCfg& c) {
  if (c.gran == 0) return {0, 1, rows * cols};  // per-tensor requires ld == cols
  if (c.gran == 1) return {g * ld, 1, cols};
  const long long r = g / c.gpr, gg = g % c.gpr;
  const long long j0 = gg * c.group;
  const long long len = min(c.group, cols - j0);
  return {r * ld + j0, 1, len};
}

// asymmetric_from_extremes / symmetric_from_extremes (quant.cpp:51-74)
__device__ inline void grid_from_extremes(float lo, float hi, const QCfg& c, float& s, int& z) {
  if (c.scheme == 1) {
    if (hi == lo) {
      s = 1.0f;
      z = clamp_code((long long)ref_rint_to_int(__fsub_rn(float(c.qmin), lo)), c.qmin, c.qmax);
      return;
    }
    s = positive_fp16(__fdiv_rn(__fsub_rn(hi, lo), float(c.qmax - c.qmin)));
    z = clamp_code((long long)ref_rint_to_int(__fsub_rn(float(c.qmin), __fdiv_rn(lo, s))), c.qmin,
                   c.qmax);
  } else {
    const float amax = fmaxf(fabsf(lo), fabsf(hi));
    s = amax == 0.0f ? 1.0f : positive_fp16(__fdiv_rn(amax, float(c.qmax)));
    z = 0;
  }
}

// grid_sq_error (quant.cpp:85-92): fp64 sum in element order
__device__ inline double seq_sq_error(const float* w, const Seg& sg, float s, int z, int qmin,
                                      int qmax) {
  double e = 0.0;
  for (long long k = 0; k < sg.len; ++k) {
    const float v = w[sg.base + k * sg.stride];
    const float wh = dequantize_code(quantize_code(v, s, z, qmin, qmax), s, z);
    const double d = double(__fsub_rn(v, wh));
    e = __dadd_rn(e, __dmul_rn(d, d));
  }
  return e;
}

// One warp per group (per_group / per_channel).  Per-tensor goes through
// the two-pass path below.
__global__ void calibrate_groups_kernel(const float* __restrict__ w, long long rows,
                                        long long cols, long long ld, QCfg c, int mse, long long ngroups,
                                        float* scales, int32_t* zeros, unsigned* flag,
                                        const float* pre_minmax) {
  const long long g = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (g >= ngroups) return;
  const unsigned lane = lane_id();
  const Seg sg = segment_of(g, rows, cols, ld, c);
  float lo, hi;
  if (pre_minmax) {  // per-tensor: extremes from the two-pass reduction
    lo = pre_minmax[0];
    hi = pre_minmax[1];
  } else {
    lo = FLT_MAX;
    hi = -FLT_MAX;
    bool bad = false;
    for (long long k = lane; k < sg.len; k += 32) {
      const float v = w[sg.base + k * sg.stride];
      bad |= !isfinite(v);
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicOr(flag, kFlagNonFinite);
      return;
    }
    for (int o = 16; o; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
  }
  float s;
  int z;
  grid_from_extremes(lo, hi, c, s, z);
  if (mse) {
    // calibrate_grid_mse (quant.cpp:114-140): candidates c = 0..99 split over
    // lanes; each lane sums its candidate's error sequentially (same order as
    // the reference), then first-strict-minimum selection.
    const bool degenerate = c.scheme == 1 ? (hi == lo) : (fmaxf(fabsf(lo), fabsf(hi)) == 0.0f);
    if (!degenerate) {
      const float raw = c.scheme == 1
                            ? __fdiv_rn(__fsub_rn(hi, lo), float(c.qmax - c.qmin))
                            : __fdiv_rn(fmaxf(fabsf(lo), fabsf(hi)), float(c.qmax));
      const double base_err = seq_sq_error(w, sg, s, z, c.qmin, c.qmax);
      double best = INFINITY;
      int best_c = 1 << 30;
      float best_s = s;
      int best_z = z;
      for (int cand = lane; cand < 100; cand += 32) {
        const float mult = __fadd_rn(0.3f, __fdiv_rn(__fmul_rn(0.7f, float(cand)), 99.0f));
        const float cs = positive_fp16(__fmul_rn(mult, raw));
        int cz = z;
        if (c.scheme == 1)
          cz = clamp_code((long long)ref_rint_to_int(__fsub_rn(float(c.qmin), __fdiv_rn(lo, cs))),
                          c.qmin, c.qmax);
        const double e = seq_sq_error(w, sg, cs, cz, c.qmin, c.qmax);
        if (e < best) {  // candidates visited in increasing order per lane
          best = e;
          best_c = cand;
          best_s = cs;
          best_z = cz;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oc = __shfl_xor_sync(0xffffffffu, best_c, o);
        const float os = __shfl_xor_sync(0xffffffffu, best_s, o);
        const int oz = __shfl_xor_sync(0xffffffffu, best_z, o);
        if (ob < best || (ob == best && oc < best_c)) {
          best = ob;
          best_c = oc;
          best_s = os;
          best_z = oz;
        }
      }
      if (best < base_err) {
        s = best_s;
        z = best_z;
      }
    }
  }
  if (lane == 0) {
    scales[g] = s;
    zeros[g] = z;
  }
}

// Min-max grids of per-group quantisation, 8 groups per warp: every lane's
// loads of the 8 groups are in flight together (the one-group-per-warp kernel
// above is latency bound), then lane q computes group q's grid.  Same
// extremes (order-free min / max), same grid arithmetic, same non-finite rule.
template <int IT>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) calibrate_minmax8_kernel(
    const float* __restrict__ w, long long rows, long long cols, long long ld, QCfg c,
    long long ngroups, float* scales, int32_t* zeros, unsigned* flag) {
  const long long g0 = ((long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5)) * 8;
  if (g0 >= ngroups) return;
  const int lane = int(lane_id());
  float v[8][IT];
  int len[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const long long g = g0 + q;
    const Seg sg = g < ngroups ? segment_of(g, rows, cols, ld, c) : Seg{0, 1, 0};
    len[q] = int(sg.len);
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int k = lane + 32 * i;
      v[q][i] = k < len[q] ? __ldg(w + sg.base + k) : 0.f;
    }
  }
  float mlo = 0.f, mhi = 0.f;
  bool mbad = false;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float lo = FLT_MAX, hi = -FLT_MAX;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      if (lane + 32 * i < len[q]) {
        bad |= !isfinite(v[q][i]);
        lo = fminf(lo, v[q][i]);
        hi = fmaxf(hi, v[q][i]);
      }
    }
    for (int o = 16; o; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == q) {
      mlo = lo;
      mhi = hi;
      mbad = bad;
    }
  }
  const long long g = g0 + lane;
  if (lane < 8 && g < ngroups) {
    if (mbad) {
      atomicOr(flag, kFlagNonFinite);
    } else {
      float s;
      int z;
      grid_from_extremes(mlo, mhi, c, s, z);
      scales[g] = s;
      zeros[g] = z;
    }
  }
}

// per-tensor extremes, pass 1: per-block partials; pass 2: one block
__global__ void minmax_partial_kernel(const float* __restrict__ w, long long n, float* part,
                                      unsigned* flag) {
  float lo = FLT_MAX, hi = -FLT_MAX;
  bool bad = false;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const float v = w[k];
    bad |= !isfinite(v);
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(flag, kFlagNonFinite);
  for (int o = 16; o; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ float slo[32], shi[32];
  const int wid = threadIdx.x >> 5;
  if (lane_id() == 0) {
    slo[wid] = lo;
    shi[wid] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < int(blockDim.x >> 5); ++i) {
      lo = fminf(lo, slo[i]);
      hi = fmaxf(hi, shi[i]);
    }
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
  }
}

__global__ void minmax_final_kernel(float* part, int nparts) {
  if (threadIdx.x != 0) return;
  float lo = part[0], hi = part[1];
  for (int i = 1; i < nparts; ++i) {
    lo = fminf(lo, part[2 * i]);
    hi = fmaxf(hi, part[2 * i + 1]);
  }
  part[0] = lo;
  part[1] = hi;
}

__global__ void quantize_rtn_kernel(const float* __restrict__ w, long long rows, long long cols,
                                    long long ld, QCfg c, const float* __restrict__ scales,
                                    const int32_t* __restrict__ zeros, int16_t* codes,
                                    float* w_hat) {
  const long long n = rows * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e % cols;
    const long long g = group_of(c, i, j);
    const float s = scales[g];
    const int z = zeros[g];
    const long long o = i * ld + j;
    const int q = quantize_code(w[o], s, z, c.qmin, c.qmax);
    codes[o] = int16_t(q);
    if (w_hat) w_hat[o] = dequantize_code(q, s, z);
  }
}

__global__ void dequantize_kernel(const int16_t* __restrict__ codes, long long rows, long long cols,
                                  QCfg c, const float* __restrict__ scales,
                                  const int32_t* __restrict__ zeros, float* out) {
  const long long n = rows * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long g = group_of(c, e / cols, e % cols);
    out[e] = dequantize_code(int(codes[e]), scales[g], zeros[g]);
  }
}

// Pack: thread t owns CPT consecutive codes = exactly 16 bytes of the
// LSB-first stream for b | 128 (CPT = 128 / b: 32 codes at 4 bits), else 128
// codes = 16 b bytes (container.cpp:15-35 BitWriter), written as 16-byte
// stores.  The stream's final partial byte is zero-padded (flush()).
template <int B>
constexpr int pack_cpt() { return (128 % B == 0) ? 128 / B : 128; }
template <int B>
__global__ void pack_codes_kernel(const int16_t* __restrict__ codes, long long n_codes, int qmin,
                                  uint8_t* out) {
  constexpr int CPT = pack_cpt<B>(), NW = CPT * B / 32;  // codes, 32-bit words per thread
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long c0 = t * CPT;
  if (c0 >= n_codes) return;
  constexpr uint32_t mask = (1u << B) - 1u;
  uint32_t words[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) words[i] = 0;
  const int cnt = int(min((long long)CPT, n_codes - c0));
  int16_t cv[CPT];
  if (cnt == CPT && (reinterpret_cast<uintptr_t>(codes) & 15) == 0) {  // 16-byte loads
#pragma unroll
    for (int q = 0; q < CPT / 8; ++q) {
      const int4 v4 = __ldg(reinterpret_cast<const int4*>(codes + c0) + q);
      const int16_t* p = reinterpret_cast<const int16_t*>(&v4);
#pragma unroll
      for (int e = 0; e < 8; ++e) cv[8 * q + e] = p[e];
    }
  } else {
#pragma unroll
    for (int k = 0; k < CPT; ++k) cv[k] = k < cnt ? codes[c0 + k] : int16_t(qmin);
  }
  // (codes past the end contribute zero bits: they are never written out)
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const uint32_t v = k < cnt ? (uint32_t(int(cv[k]) - qmin) & mask) : 0u;
    const int bit = k * B, wi = bit >> 5, sh = bit & 31;  // static after unrolling
    words[wi] |= v << sh;
    if (sh + B > 32) words[wi + 1] |= v >> (32 - sh);
  }
  const long long byte0 = t * (4LL * NW);
  if (cnt == CPT && ((reinterpret_cast<uintptr_t>(out + byte0) & 15) == 0)) {
    uint4* o = reinterpret_cast<uint4*>(out + byte0);
#pragma unroll
    for (int q = 0; q < NW / 4; ++q)
      o[q] = make_uint4(words[4 * q], words[4 * q + 1], words[4 * q + 2], words[4 * q + 3]);
  } else {
    const long long nb = min(4LL * NW, (n_codes * B + 7) / 8 - byte0);
#pragma unroll
    for (int b = 0; b < 4 * NW; ++b)
      if (b < nb) out[byte0 + b] = uint8_t(words[b >> 2] >> (8 * (b & 3)));
  }
}

__global__ void pack_meta_kernel(long long n_groups, int asym, const float* __restrict__ scales,
                                 const int32_t* __restrict__ zeros, uint8_t* meta) {
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n_groups;
       g += (long long)gridDim.x * blockDim.x) {
    const uint16_t h = fp16_encode(scales[g]);  // put_fp16 (container.cpp:66-70)
    meta[2 * g] = uint8_t(h & 0xff);
    meta[2 * g + 1] = uint8_t(h >> 8);
    if (asym) meta[2 * n_groups + g] = uint8_t(zeros[g]);
  }
}

__global__ void unpack_codes_kernel(const uint8_t* __restrict__ in, long long n_codes, int bits,
                                    int qmin, int16_t* codes) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n_codes;
       e += (long long)gridDim.x * blockDim.x) {
    const long long bit = e * bits;
    const long long byte = bit >> 3;
    const int sh = int(bit & 7);
    uint32_t v = in[byte];
    if (sh + bits > 8) v |= uint32_t(in[byte + 1]) << 8;
    codes[e] = int16_t(int((v >> sh) & ((1u << bits) - 1u)) + qmin);
  }
}

__global__ void unpack_meta_kernel(const uint8_t* __restrict__ meta, long long n_groups, int asym,
                                   float* scales, int32_t* zeros) {
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n_groups;
       g += (long long)gridDim.x * blockDim.x) {
    scales[g] = fp16_decode(uint16_t(meta[2 * g] | (uint16_t(meta[2 * g + 1]) << 8)));
    zeros[g] = asym ? int(meta[2 * n_groups + g]) : 0;
  }
}

// Stable descending rank of diag(H): rank_i = #{j: d_j > d_i} + #{j < i: d_j == d_i}.
// O(n^2) comparisons: kSplit threads per row i split the j range (diag tiles
// staged in shared memory), then a shuffle reduction; bit-exact with
// std::stable_sort(order, h[a][a] > h[b][b]) for NaN-free diagonals.  The diag
// is read at stride `ds` from `d` (a contiguous copy of diag(H), ds = 1: the
// factor path's damp kernel leaves it beside the factor input).
constexpr int kOrdThreads = 256, kOrdTile = 8192;
template <int kSplit>
__global__ void __launch_bounds__(kOrdThreads) order_rank_kernel(const float* __restrict__ d,
                                                                 long long ds, long long n,
                                                                 int32_t* order) {
  __shared__ float tile[kOrdTile];
  const int part = threadIdx.x % kSplit;
  const long long i = (long long)blockIdx.x * (kOrdThreads / kSplit) + threadIdx.x / kSplit;
  const float di = i < n ? d[i * ds] : 0.0f;
  long long rank = 0;
  for (long long j0 = 0; j0 < n; j0 += kOrdTile) {
    const int cnt = int(min((long long)kOrdTile, n - j0));
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += kOrdThreads) tile[t] = d[(j0 + t) * ds];
    __syncthreads();
    const long long lim = i - j0;  // t < lim  <=>  j0 + t < i
    int cnt_r = 0;
#pragma unroll 4
    for (int t = part; t < cnt; t += kSplit) {
      const float dj = tile[t];
      cnt_r += (dj > di) | ((dj == di) & (t < lim));
    }
    rank += cnt_r;
  }
  for (int o = 1; o < kSplit; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
  if (part == 0 && i < n) order[rank] = int32_t(i);
}

__global__ void iota_kernel(long long n, int32_t* order) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    order[i] = int32_t(i);
}

inline int grid_for(long long n, int threads, int cap = 148 * 16) {
  long long g = (n + threads - 1) / threads;
  return int(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void launch_calibrate_grids(const float* w, long long rows, long long cols, long long ld,
                            const QCfg& c, int mse, float* scales, int32_t* zeros, unsigned* flag, float* ws_minmax,
                            cudaStream_t st) {
  const long long ng = c.gran == 0 ? 1 : (c.gran == 1 ? rows : rows * c.gpr);
  const float* pre = nullptr;
  if (c.gran == 0) {
    const int parts = grid_for(rows * cols, 256, 512);
    minmax_partial_kernel<<<parts, 256, 0, st>>>(w, rows * cols, ws_minmax, flag);
    minmax_final_kernel<<<1, 32, 0, st>>>(ws_minmax, parts);
    pre = ws_minmax;
    count_launches(2);
  }
  count_launches(1);
  if (c.gran == 2 && !mse && c.group <= 128) {
    const int blocks = int((ng + 8 * kWarpsPerBlock - 1) / (8 * kWarpsPerBlock));
    const int it = int((c.group + 31) / 32);
    if (it <= 1)
      calibrate_minmax8_kernel<1><<<blocks, 32 * kWarpsPerBlock, 0, st>>>(w, rows, cols, ld, c, ng, scales, zeros, flag);
    else if (it == 2)
      calibrate_minmax8_kernel<2><<<blocks, 32 * kWarpsPerBlock, 0, st>>>(w, rows, cols, ld, c, ng, scales, zeros, flag);
    else if (it == 3)
      calibrate_minmax8_kernel<3><<<blocks, 32 * kWarpsPerBlock, 0, st>>>(w, rows, cols, ld, c, ng, scales, zeros, flag);
    else
      calibrate_minmax8_kernel<4><<<blocks, 32 * kWarpsPerBlock, 0, st>>>(w, rows, cols, ld, c, ng, scales, zeros, flag);
    return;
  }
  const int blocks = int((ng + kWarpsPerBlock - 1) / kWarpsPerBlock);
  calibrate_groups_kernel<<<blocks, 32 * kWarpsPerBlock, 0, st>>>(w, rows, cols, ld, c, mse, ng, scales,
                                                                  zeros, flag, pre);
}

void launch_quantize_rtn(const float* w, long long rows, long long cols, long long ld,
                         const QCfg& c, const float* scales, const int32_t* zeros, int16_t* codes,
                         float* w_hat, cudaStream_t st) {
  count_launches(1);
  quantize_rtn_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(w, rows, cols, ld, c, scales,
                                                                   zeros, codes, w_hat);
}

void launch_dequantize(const int16_t* codes, long long rows, long long cols, const QCfg& c,
                       const float* scales, const int32_t* zeros, float* out, cudaStream_t st) {
  count_launches(1);
  dequantize_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(codes, rows, cols, c, scales, zeros,
                                                                 out);
}

void launch_pack(const int16_t* codes, long long n_codes, long long n_groups, const QCfg& c,
                 const float* scales, const int32_t* zeros, uint8_t* out, cudaStream_t st) {
  count_launches(2);
  if (n_codes > 0) {
    switch (c.bits) {
#define OCWG_PACK(B)                                                                     \
  case B: {                                                                              \
    const long long thr = (n_codes + pack_cpt<B>() - 1) / pack_cpt<B>();                 \
    pack_codes_kernel<B><<<int((thr + 255) / 256), 256, 0, st>>>(codes, n_codes, c.qmin, out); \
  } break;
      OCWG_PACK(1) OCWG_PACK(2) OCWG_PACK(3) OCWG_PACK(4) OCWG_PACK(5) OCWG_PACK(6) OCWG_PACK(7)
      OCWG_PACK(8)
#undef OCWG_PACK
    }
  }
  const long long code_bytes = (n_codes * c.bits + 7) / 8;
  pack_meta_kernel<<<grid_for(n_groups, 256), 256, 0, st>>>(n_groups, c.scheme == 1, scales, zeros,
                                                             out + code_bytes);
}

void launch_unpack(const uint8_t* payload, long long n_codes, long long n_groups, const QCfg& c,
                   int16_t* codes, float* scales, int32_t* zeros, cudaStream_t st) {
  count_launches(2);
  unpack_codes_kernel<<<grid_for(n_codes, 256), 256, 0, st>>>(payload, n_codes, c.bits, c.qmin,
                                                               codes);
  const long long code_bytes = (n_codes * c.bits + 7) / 8;
  unpack_meta_kernel<<<grid_for(n_groups, 256), 256, 0, st>>>(payload + code_bytes, n_groups,
                                                               c.scheme == 1, scales, zeros);
}

void launch_order(const float* diag, long long n, int actorder, int32_t* order, cudaStream_t st) {
  count_launches(1);
  if (!actorder) {
    iota_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, order);
    return;
  }
  constexpr int split = 16;  // threads per row; diag tiles staged coalesced
  constexpr long long rows = kOrdThreads / split;
  order_rank_kernel<split><<<int((n + rows - 1) / rows), kOrdThreads, 0, st>>>(diag, 1, n, order);
}

// ---- AutoBit's default candidate grid (autobit.cpp:45-61, estimate_error
// :16-34): RTN error of W under bits {2..8} x {per_group 128, per_channel},
// symmetric, for all 14 configurations in one pass over W.  One CTA per row:
// group and row extremes first, then per element and configuration
// code = clamp(rint(w / s)), w_hat = s code, d = w_hat - w (fp64), summed per
// row; a second kernel adds the rows in order.
namespace {
constexpr int kCand = 14, kCandThreads = 256;
__global__ void __launch_bounds__(kCandThreads) candidate_rows_kernel(
    const float* __restrict__ w, long long cols, long long ld, int act,
    const double* __restrict__ in_diag, double* __restrict__ partial, unsigned* flag) {
  extern __shared__ float gmax[];  // per 128-group |w| max, then the row max at [ngroups]
  __shared__ double red[kCandThreads / 32][kCand];
  __shared__ float s_cfg[kCand];
  const long long row = blockIdx.x;
  const float* wr = w + row * ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long ng = (cols + 127) / 128;
  // group extremes: warp w covers columns 32 w.. of each 256-column stride
  bool bad = false;
  for (long long g0 = 0; g0 < ng; g0 += 2) {
    const long long col = g0 * 128 + tid;
    float a = 0.f;
    if (col < cols) {
      const float v = wr[col];
      bad |= !isfinite(v);
      a = fabsf(v);
    }
    for (int o = 16; o; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0) red[warp][0] = a;
    __syncthreads();
    if (tid < 2 && g0 + tid < ng) {
      const int w0 = 4 * tid;
      gmax[g0 + tid] = fmaxf(fmaxf(float(red[w0][0]), float(red[w0 + 1][0])),
                             fmaxf(float(red[w0 + 2][0]), float(red[w0 + 3][0])));
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) atomicOr(flag, kFlagNonFinite);
    return;
  }
  if (tid == 0) {
    float m = 0.f;
    for (long long g = 0; g < ng; ++g) m = fmaxf(m, gmax[g]);
    gmax[ng] = m;
    for (int k = 0; k < kCand; k += 2) {  // per-channel scales (k odd below)
      const int qmax = (1 << (2 + k / 2 - 1)) - 1;
      s_cfg[k + 1] = m == 0.f ? 1.f : positive_fp16(__fdiv_rn(m, float(qmax)));
    }
  }
  __syncthreads();
  double e[kCand];
#pragma unroll
  for (int k = 0; k < kCand; ++k) e[k] = 0.0;
  for (long long col = tid; col < cols; col += kCandThreads) {
    const float v = wr[col];
    const float ga = gmax[col / 128];
#pragma unroll
    for (int b = 0; b < 7; ++b) {
      const int qmax = (1 << (b + 1)) - 1;  // bits b + 2, symmetric
#pragma unroll
      for (int gr = 0; gr < 2; ++gr) {  // grouped first (autobit.cpp:48-49)
        float sv;
        if (gr == 0) sv = ga == 0.f ? 1.f : positive_fp16(__fdiv_rn(ga, float(qmax)));
        else sv = s_cfg[2 * b + 1];
        const int code = quantize_code(v, sv, 0, -qmax, qmax);
        const double d = double(dequantize_code(code, sv, 0)) - double(v);
        e[2 * b + gr] = fma(d, d, e[2 * b + gr]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kCand; ++k) {
    double x = e[k];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][k] = x;
  }
  __syncthreads();
  if (tid < kCand) {
    double x = 0.0;
    for (int q = 0; q < kCandThreads / 32; ++q) x += red[q][tid];
    if (act) x *= 0.5 * (in_diag ? in_diag[row] : 1.0);
    partial[row * kCand + tid] = x;
  }
}
__global__ void candidate_sum_kernel(const double* __restrict__ partial, long long rows,
                                     double* out) {
  const int k = threadIdx.x;
  if (k >= kCand) return;
  double x = 0.0;
  for (long long r = 0; r < rows; ++r) x += partial[r * kCand + k];
  out[k] = x;
}
}  // namespace

void launch_candidate_grid(const float* w, long long rows, long long cols, long long ld, int act,
                           const double* in_diag, double* partial, double* out, unsigned* flag,
                           cudaStream_t st) {
  const long long ng = (cols + 127) / 128;
  const size_t smem = size_t(ng + 1) * sizeof(float);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(candidate_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
  count_launches(2);
  candidate_rows_kernel<<<unsigned(rows), kCandThreads, smem, st>>>(w, cols, ld, act, in_diag,
                                                                    partial, flag);
  candidate_sum_kernel<<<1, 32, 0, st>>>(partial, rows, out);
}

}  // namespace ocwg
