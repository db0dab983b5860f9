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
// (permuted) row.  Two-level blocking, on one stream:
//   super-blocks of 512 rows (4 blocks of B = 128): after the last block of a
//   super-block, ONE trailing GEMM applies it to every later row,
//       acc[se:, :] (+)= G[se:, s0:se] D[s0:se, :]        (tcgen05 3xTF32 pairs);
//   per block, the in-block kernel adds acc, applies the earlier blocks of
//   its own super-block by lookahead (G[blk, s0:ib] D[s0:ib], warp tensor
//   cores), then runs the row chain: quantize; D = w - w_hat; the block's
//   later rows += G[k, i] D.
// acc needs no initialisation: the first super-block's GEMM writes it with
// beta = 0 and the first super-block never reads it.
//
// fp32 path (l4::inblock4_kernel, B = 128): 16 columns per 4-warp CTA, 8
// lanes per column, 16 rotating register slots per lane; a branch-free
// quantise chain (residual division, shifter rounding); the sweep's kernels
// are chained by programmatic dependent launch.  See the kernel.
// Generic path (inblock_g_kernel: fp64, or B != 128): a CTA owns 32 columns
// (8 warps x 4); lane = cc + 4*rg keeps rows rg, rg+8, ... of its column in
// registers, rotating by one slot per 8-row group; D is broadcast with one
// warp shuffle and staged for a coalesced K-major store.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <type_traits>

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
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
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

// Rotated G block: for row li = 8t + o the coefficients a lane (rg) needs are
// G[rg + 8(t + kk)][li], kk = 0..RPT-1 -- its register slot kk after t
// rotations -- stored contiguously at gt[li][rg * kRg + kk] (zero where the row
// is outside the block or not strictly below li), so a row step is RPT/4
// LDS.128 and RPT unconditional FMAs.  kRg = 20 (not 16) spreads the 8
// row groups of a warp over all 32 banks.
constexpr int kRg = 20;

template <typename T>
struct InblockSmem {
  union {
    T gt[kB][8 * kRg];
    struct {
      T gc[kB][kLaChunk + 4];     // lookahead: G[ib + li][kprev + q0 + q]
      T dp[kCols][kLaChunk + 4];  // lookahead: D_prev[q0 + q] of column cj
    } la;
  } u;
  T ds[kCols][kB + 1];  // D of this block, staged for the K-major store
  int og[kB];           // processing -> original row of the block
  long long orow[kB];   // og * ldo: output row offsets
};

template <typename T, int RPT>
__global__ void __launch_bounds__(256) inblock_g_kernel(
    const float* __restrict__ w, long long ldw, const int32_t* __restrict__ order,
    const T* __restrict__ acc, int use_acc, const T* __restrict__ gpl,
    const T* __restrict__ dprev, int bprev, T* __restrict__ dcur, float* __restrict__ dcur_hi,
    float* __restrict__ dcur_lo, QCfg c, const float* __restrict__ scales,
    const int32_t* __restrict__ zeros, long long n, long long m, long long ib, int bsz,
    int16_t* __restrict__ codes, float* __restrict__ w_hat, long long ldo, long long ldd) {
  static_assert(RPT % 4 == 0 && RPT <= kRg, "row slots");
  extern __shared__ __align__(16) unsigned char smraw[];
  InblockSmem<T>& sm = *reinterpret_cast<InblockSmem<T>*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cc = lane & 3, rg = lane >> 2;
  const int cj = warp * 4 + cc;
  const long long j0 = (long long)blockIdx.x * kCols;
  const long long j = j0 + cj;
  const bool col_ok = j < m;

  for (int e = tid; e < kB; e += 256) {
    sm.og[e] = e < bsz ? order[ib + e] : 0;
    sm.orow[e] = (long long)sm.og[e] * ldo;
  }
  __syncthreads();
  // ---- per-lane rows rg + 8t: partial sums, original weights, grids (+ 1/s)
  T r[RPT];
  float w0[RPT], s[RPT], y[RPT], zf[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int li = rg + 8 * t;
    r[t] = T(0);
    w0[t] = 0.f;
    s[t] = 1.f;
    zf[t] = 0.f;
    if (col_ok && li < bsz) {
      const long long orig = sm.og[li];
      w0[t] = w[orig * ldw + j];
      const long long g = group_of(c, orig, j);
      s[t] = scales[g];
      zf[t] = float(zeros[g]);
      if (use_acc) r[t] = acc[(ib + li) * m + j];
    }
    y[t] = rcp_refined(s[t]);
  }
  const float qminf = float(c.qmin), qmaxf = float(c.qmax);

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
          cp_async(&sm.u.la.dp[cl][q], dprev + (j0 + cl) * ldd + q0 + q);
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

  // ---- stage the block's G in the rotated layout (coalesced along li)
  for (int e = tid; e < kB * 8 * RPT; e += 256) {
    const int li = e % kB, slot = e / kB;  // slot = rg * RPT + kk
    const int rgs = slot / RPT, kk = slot % RPT;
    const int k = rgs + 8 * ((li >> 3) + kk);  // row of G this slot multiplies
    T* dst = &sm.u.gt[li][rgs * kRg + kk];
    if (li < bsz && k < bsz && k > li)
      cp_async(dst, gpl + (ib + k) * n + ib + li);
    else
      *dst = T(0);
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- sequential rows li = 8t + o; owner lane rg == o holds the row in slot 0.
  // Every lane quantises its own slot 0 (branch-free); the owner's D is broadcast.
  int16_t* code_col = codes + j;
  float* wh_col = w_hat ? w_hat + j : nullptr;
#pragma unroll 1
  for (int t = 0; t < RPT; ++t) {
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const int li = 8 * t + o;
      if (li >= bsz) break;
      // coefficients of this row first: their smem latency overlaps the chain
      T g[RPT];
      const T* gp = &sm.u.gt[li][rg * kRg];
#pragma unroll
      for (int k4 = 0; k4 < RPT; k4 += 4) {
        T g4[4];
        ld4(gp + k4, g4);
#pragma unroll
        for (int e = 0; e < 4; ++e) g[k4 + e] = g4[e];
      }
      const T cur = T(w0[0]) + r[0];  // w_cur = w + sum G D
      const float cf = quantize_code_f(div_rn_fast(float(cur), s[0], y[0]), zf[0], qminf, qmaxf);
      const float wh = __fmul_rn(s[0], __fsub_rn(cf, zf[0]));  // quant.cpp:33-35
      T d = T(w0[0]) - T(wh);
      if (rg == o) {
        if (col_ok) {
          const long long orow = sm.orow[li];  // original row order (:75)
          code_col[orow] = code_bits(cf);
          if (wh_col) wh_col[orow] = wh;
        }
        sm.ds[cj][li] = d;
      }
      d = __shfl_sync(0xffffffffu, d, cc + 4 * o);
#pragma unroll
      for (int k = 0; k < RPT; ++k) r[k] = fma(g[k], d, r[k]);
    }
#pragma unroll
    for (int k = 0; k + 1 < RPT; ++k) {
      r[k] = r[k + 1];
      w0[k] = w0[k + 1];
      s[k] = s[k + 1];
      y[k] = y[k + 1];
      zf[k] = zf[k + 1];
    }
  }
  __syncthreads();
  // ---- D (K-major: column j's kB values contiguous): plain, and the tf32
  // hi/lo split the tensor-core GEMM consumes
  for (int e = tid; e < kCols * kB; e += 256) {
    const int cl = e / kB, li = e % kB;
    if (j0 + cl >= m || li >= bsz) continue;
    const T v = sm.ds[cl][li];
    const long long off = (j0 + cl) * ldd + li;
    dcur[off] = v;
    if (dcur_hi) {
      const float hi = tf32_hi(float(v));
      dcur_hi[off] = hi;
      dcur_lo[off] = float(v) - hi;
    }
  }
}

// ---------------------------------------------------------------------------
// fp32, 128-row blocks: 4 lanes per column (lane = cc + 8 rg), 8 columns per
// warp, 2 warps (16 columns) per CTA.  Lane group rg owns rows rg + 4s,
// s = 0..31, in registers r[k] <-> s = k + 4T, where T counts 16-row steps: the
// 16-row body is unrolled (the owner of row 4t + o is rg = o, slot k = t % 4,
// static) and the registers rotate by 4 slots after it -- compact code (the
// body fits the instruction cache) with static register indices.  The
// coefficients G[rg + 4s][li] of a row are a contiguous, 16-byte aligned run
// of the diagonal block of G^T that the Cholesky emits in exactly this order
// (factor.cu gp_pos; chunks XOR-swizzled by 2 rg so the 4 lane groups hit
// distinct banks): 8 LDS.128 per row.  The owner's (w, s, 1/s, z) come from a
// per-row table gathered once with cp.async.
namespace l4 {
// 4 warps, all on the row chain: warp w owns columns 4w..4w+3, 8 lanes per
// column; lane (cc, rg) holds rows rg + 8s (s = 0..15) of column 4w + cc.
// Two CTAs per SM give two chain warps per SM sub-partition, whose
// quantise chains interleave.
constexpr int kLpc = 8, kRpt = 16, kCpw = 4, kCols4 = 16, kThreads = 128;
constexpr int kLa4 = 32;      // lookahead K chunk (double-buffered)
constexpr int kGtEarly = 88;  // G rows >= this are staged before the lookahead

struct Smem {
  union {
    float gt[kB * kB + 32];  // block rows of G^T in lane order (+ pad for dead slots)
    struct {
      float gc[2][kB][kLa4 + 4];
      float dp[2][kCols4][kLa4 + 4];
    } la;
  } u;
  float4 tab[kB + 1][kCols4];  // {w, s, 1/s, z} of (row li, column cj); +1 row read ahead
  float ds[kCols4][kB + 1];  // D = w - w_hat of (column, row); lookahead hand-off first
  int16_t cs[kCols4][kB + 2];  // codes of (column, row)
  long long orow[kB];
  int og[kB];
};
static_assert(sizeof(((Smem*)0)->u.la) <= kGtEarly * kB * sizeof(float), "early G rows overlap");

// phase timestamps (globaltimer ns) of one traced launch, per CTA
__device__ unsigned long long g_trace[1024 * 8];
__device__ __forceinline__ void stamp(int trace, int i) {
  if ((trace & 1) && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_trace[blockIdx.x * 8 + i] = t;
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 3xTF32 on the legacy warp-level tensor-core path (m16n8k8): the lookahead
// is a 128 x 16 x K product per CTA, too small for a tcgen05 pipeline.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = h;
  lo = __float_as_uint(x - __uint_as_float(h));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// G^T rows [r0, r1) of the block (zero rows past bsz)
__device__ __forceinline__ void stage_gt(Smem& sm, const float* gpb, long long ib, int bsz, int r0,
                                         int r1, int tid) {
  for (int e = r0 * (kB / 4) + tid; e < r1 * (kB / 4); e += kThreads) {
    const int li = e / (kB / 4), q = (e % (kB / 4)) * 4;
    float* dst = &sm.u.gt[li * kB + q];
    if (li < bsz)
      cp_async16(dst, gpb + (ib + li) * kB + q);
    else
      *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}
// lookahead chunk: G[blk, kprev + q0 : +kLa4] and D_prev[q0 : +kLa4] of the CTA's columns
__device__ __forceinline__ void stage_la(Smem& sm, int buf, const float* gpl, const float* dprev,
                                         long long n, long long m, long long ib, int bsz,
                                         long long kprev, int bprev, int q0, long long j0,
                                         long long ldd, int tid) {
  for (int e = tid; e < kB * kLa4 / 4; e += kThreads) {
    const int li = e / (kLa4 / 4), q = (e % (kLa4 / 4)) * 4;
    float* dst = &sm.u.la.gc[buf][li][q];
    if (li < bsz && q0 + q < bprev)
      cp_async16(dst, gpl + (ib + li) * n + kprev + q0 + q);
    else
      *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int e = tid; e < kCols4 * kLa4 / 4; e += kThreads) {
    const int cl = e / (kLa4 / 4), q = (e % (kLa4 / 4)) * 4;
    float* dst = &sm.u.la.dp[buf][cl][q];
    if (j0 + cl < m && q0 + q < bprev)
      cp_async16(dst, dprev + (j0 + cl) * ldd + q0 + q);
    else
      *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__global__ void __launch_bounds__(kThreads, 1) inblock4_kernel(
    const float* __restrict__ w, long long ldw, const int32_t* __restrict__ order,
    const float* __restrict__ acc, int use_acc, const float* __restrict__ gpl,
    const float* __restrict__ gpb, const float* __restrict__ dprev, int bprev,
    float* __restrict__ dcur, float* __restrict__ dcur_hi, float* __restrict__ dcur_lo, QCfg c,
    const float* __restrict__ scales, const int32_t* __restrict__ zeros, long long n, long long m,
    long long ib, int bsz, int16_t* __restrict__ codes, float* __restrict__ w_hat, long long ldo,
    long long ldd, int trace, const float4* __restrict__ tabb, const int* __restrict__ tab_sbad) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& sm = *reinterpret_cast<Smem*>(smraw);
  stamp(trace, 0);
  // a prepared table block (sweep_table_kernel, built beside the previous
  // trailing GEMM): the {w, s, 1/s, z} rows are one contiguous 32 KB bulk copy
  // instead of a gather.  Its mbarrier lives in the read-ahead row kB, which
  // never holds data (two CTAs per SM leave no spare shared memory).
  const uint32_t tbar = smem_u32(&sm.tab[kB][0]);
  if (tabb && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tbar),
                 "r"(uint32_t(kB * kCols4 * 16))
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(&sm.tab[0][0])),
        "l"(tabb + (long long)blockIdx.x * kB * kCols4), "r"(uint32_t(kB * kCols4 * 16)), "r"(tbar)
        : "memory");
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cc = lane & 3, rg = lane >> 2;
  const int og = tid < bsz ? order[ib + tid] : 0;
  const int cj = warp * kCpw + cc;
  const long long j0 = (long long)blockIdx.x * kCols4;
  const long long j = j0 + cj;
  const bool col_ok = j < m;

  // Up to the table, the prologue reads only what the sweep never writes (order,
  // W, grids, G): as a programmatic dependent it runs beside the previous
  // kernel's tail; acc and the lookahead D (previous kernels' outputs) follow
  // griddepcontrol.wait.
  // ---- async: late G rows (never overlapped by the lookahead buffers)
  const long long kprev = ib - bprev;
  stage_gt(sm, gpb, ib, bsz, bprev > 0 ? kGtEarly : 0, kB, tid);
  if (tid < 8) reinterpret_cast<float4*>(&sm.u.gt[kB * kB])[tid] = make_float4(0.f, 0.f, 0.f, 0.f);
  cp_async_commit();
  sm.og[tid] = og;
  sm.orow[tid] = (long long)og * ldo;
  __syncthreads();
  stamp(trace, 6);

  // ---- per-(row, column) table {w, s, 1/s, z}: task = (row, 4 columns)
  const bool wvec = (ldw & 3) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0;
  bool sbad = tabb ? __ldg(tab_sbad + blockIdx.x) != 0 : false;  // a scale outside scale_safe():
                                                                 // the chain divides exactly
#pragma unroll
  for (int i = 0; i < (tabb ? 0 : kB * kCols4 / 4 / kThreads); ++i) {
    const int e = tid + i * kThreads;
    const int li = e >> 2, q = (e & 3) * 4;
    const long long jj = j0 + q;
    float4* dst = &sm.tab[li][q];
    if (li >= bsz) {
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[u] = make_float4(0.f, 1.f, 1.f, 0.f);
      continue;
    }
    const long long orig = sm.og[li];
    const float* wr = w + orig * ldw + jj;
    float wv[4];
    if (wvec && jj + 3 < m) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(wr));
      wv[0] = f.x, wv[1] = f.y, wv[2] = f.z, wv[3] = f.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) wv[u] = jj + u < m ? __ldg(wr + u) : 0.f;
    }
    const long long g0 = group_of(c, orig, jj), g3 = group_of(c, orig, std::min(jj + 3, m - 1));
    if (g0 == g3) {
      const float sv = __ldg(scales + g0);
      const float y = rcp_refined(sv), zf = float(__ldg(zeros + g0));
      sbad |= !scale_safe(sv);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        dst[u] = jj + u < m ? make_float4(wv[u], sv, y, zf) : make_float4(0.f, 1.f, 1.f, 0.f);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (jj + u < m) {
          const long long g = group_of(c, orig, jj + u);
          const float sv = __ldg(scales + g);
          sbad |= !scale_safe(sv);
          dst[u] = make_float4(wv[u], sv, rcp_refined(sv), float(__ldg(zeros + g)));
        } else {
          dst[u] = make_float4(0.f, 1.f, 1.f, 0.f);
        }
      }
    }
  }
  stamp(trace, 7);
  pdl_wait();
  // ---- this thread's acc rows (earlier super-blocks) and lookahead chunk 0
  float r[kRpt];  // slot s = row rg + 8s
#pragma unroll
  for (int k = 0; k < kRpt; ++k) {
    const int li = rg + 8 * k;
    r[k] = (use_acc && col_ok && li < bsz) ? acc[(ib + li) * m + j] : 0.f;
  }
  if (bprev > 0) stage_la(sm, 0, gpl, dprev, n, m, ib, bsz, kprev, bprev, 0, j0, ldd, tid);
  cp_async_commit();
  stamp(trace, 1);

  // ---- lookahead: G[blk, sb0:ib] D[sb0:ib] on the tensor cores (3xTF32,
  // double-buffered K chunks); warp w owns rows 32w..32w+31, all 16 columns
  if (bprev > 0) {
    float c1[2][2][4] = {}, c2[2][2][4] = {};  // hi*hi, cross terms
    const int gq = lane >> 2, tq = lane & 3, rb = 32 * warp;
    const int nch = (bprev + kLa4 - 1) / kLa4;
#pragma unroll 1
    for (int ch = 0; ch < nch; ++ch) {
      const int buf = ch & 1;
      if (ch + 1 < nch) {
        stage_la(sm, buf ^ 1, gpl, dprev, n, m, ib, bsz, kprev, bprev, (ch + 1) * kLa4, j0, ldd,
                 tid);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
#pragma unroll
      for (int k8 = 0; k8 < kLa4; k8 += 8) {
        uint32_t ah[2][4], al[2][4], bh[2][2], bl[2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const float* g0 = &sm.u.la.gc[buf][rb + 16 * mt + gq][k8 + tq];
          const float* g8 = g0 + 8 * (kLa4 + 4);
          split_tf32(g0[0], ah[mt][0], al[mt][0]);
          split_tf32(g8[0], ah[mt][1], al[mt][1]);
          split_tf32(g0[4], ah[mt][2], al[mt][2]);
          split_tf32(g8[4], ah[mt][3], al[mt][3]);
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const float* d0 = &sm.u.la.dp[buf][8 * nt + gq][k8 + tq];
          split_tf32(d0[0], bh[nt][0], bl[nt][0]);
          split_tf32(d0[4], bh[nt][1], bl[nt][1]);
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            mma_tf32(c1[mt][nt], ah[mt], bh[nt][0], bh[nt][1]);
            mma_tf32(c2[mt][nt], ah[mt], bl[nt][0], bl[nt][1]);
            mma_tf32(c2[mt][nt], al[mt], bh[nt][0], bh[nt][1]);
          }
      }
      __syncthreads();
    }
    // the lookahead buffers are dead: stage the early G rows over them
    stage_gt(sm, gpb, ib, bsz, 0, kGtEarly, tid);
    cp_async_commit();
    // hand the 128 x 16 product to the main warps (ds is free until the chain)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int row = rb + 16 * mt + gq, col = 8 * nt + 2 * tq;
        sm.ds[col][row] = c1[mt][nt][0] + c2[mt][nt][0];
        sm.ds[col + 1][row] = c1[mt][nt][1] + c2[mt][nt][1];
        sm.ds[col][row + 8] = c1[mt][nt][2] + c2[mt][nt][2];
        sm.ds[col + 1][row + 8] = c1[mt][nt][3] + c2[mt][nt][3];
      }
  }
  stamp(trace, 2);
  cp_async_wait<0>();
  if (tabb) {
    uint32_t done;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(tbar)
          : "memory");
    } while (!done);
  }
  const bool exact_div = __syncthreads_or(sbad || (trace & 2));
  stamp(trace, 3);

  // the chain, specialised on the division: the residual step alone (all
  // scales safe, the normal case) or the IEEE routine; no branch per row
  auto chain = [&](auto exact) {
    constexpr bool kExact = decltype(exact)::value;
    if (bprev > 0) {
#pragma unroll
      for (int k = 0; k < kRpt; ++k) r[k] += sm.ds[cj][rg + 8 * k];
    }
    const float qminf = float(c.qmin), qmaxf = float(c.qmax);
    // Rows li >= bsz of a short last block run as padding (w = 0, s = 1, z = 0,
    // zero G rows): finite d that no real row picks up, never stored -- so the
    // step loop has no per-row branch and the next row's loads hoist freely.
    // Per 16 rows (T) the slots rotate by 2; logical slot pair T + mm of lane
    // group rg sits at off[mm] (factor.cu gp_pos: conflict-free 8-byte loads).
    // the table entry of the next row is read one row ahead: the owner's add
    // of row li then never waits on shared memory (this row's stores precede
    // the read in program order, so the compiler cannot hoist it itself)
    float4 tvn = sm.tab[0][cj];
    // 16 rows; LIVE slots: from T = 4 on, slots 8..15 hold rows past the block
    // (16T + 8s + rg >= 128), so half the coefficient loads and FMAs drop out
    auto rows16 = [&](int T, auto live_c) {
      constexpr int LIVE = decltype(live_c)::value;
      int off[LIVE / 2];
#pragma unroll
      for (int mm = 0; mm < LIVE / 2; ++mm)
        off[mm] = 16 * T * kB + rg * 16 + 2 * ((T + mm + 2 * (rg >> 1)) & 7);
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
#pragma unroll
        for (int o = 0; o < kLpc; ++o) {
          const int lj = 8 * tt + o, li = 16 * T + lj;
          const float4 tv = tvn;  // (w, s, 1/s, z) of row li
          tvn = sm.tab[li + 1][cj];
          float g[LIVE];
#pragma unroll
          for (int mm = 0; mm < LIVE / 2; ++mm) {
            const float2 g2 = *reinterpret_cast<const float2*>(&sm.u.gt[off[mm] + lj * kB]);
            g[2 * mm] = g2.x, g[2 * mm + 1] = g2.y;
          }
          const float x = __fadd_rn(tv.x, r[tt]);  // w_cur = w + sum G D (owner lanes)
          const float qv = kExact ? __fdiv_rn(x, tv.y) : div_rn_residual(x, tv.y, tv.z);
          // code - z = clamp(rint(q), qmin - z, qmax - z) (quantize_code_f,
          // shifted by z so W_hat = s (code - z) needs no subtraction on the chain)
          const float loz = __fsub_rn(qminf, tv.w), hiz = __fsub_rn(qmaxf, tv.w);
          const float u = __fsub_rn(__fadd_rn(qv, kRoundShifter), kRoundShifter);
          const float cl = fminf(fmaxf(u, loz), qv < 2147483648.0f ? hiz : loz);
          const float wh = __fmul_rn(tv.y, cl);  // quant.cpp:33-35
          const float d = __shfl_sync(0xffffffffu, __fsub_rn(tv.x, wh), cc + 4 * o);
          if (rg == o) {  // the owner's own d; stores leave with the epilogue
            sm.ds[cj][li] = d;
            sm.cs[cj][li] = code_bits(__fadd_rn(cl, tv.w));
          }
#pragma unroll
          for (int k = 0; k < LIVE; ++k) r[k] = fmaf(g[k], d, r[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < LIVE; ++k) r[k] = k + 2 < LIVE ? r[k + 2] : 0.f;
    };
#pragma unroll 1
    for (int T = 0; T < 4; ++T) {
      if (16 * T >= bsz) return;
      rows16(T, std::integral_constant<int, kRpt>{});
    }
#pragma unroll 1
    for (int T = 4; T < kRpt / 2; ++T) {
      if (16 * T >= bsz) return;
      rows16(T, std::integral_constant<int, kRpt / 2>{});
    }
  };
  if (exact_div)
    chain(std::true_type{});
  else
    chain(std::false_type{});
  pdl_trigger();  // the next kernel's setup may start as these CTAs drain
  __syncthreads();
  stamp(trace, 4);
  // ---- D (K-major, the trailing GEMM's B operand), then codes / W_hat in
  // original row order (layerwise.cpp:75)
  for (int e = tid; e < kCols4 * kB / 4; e += kThreads) {
    const int cl = e / (kB / 4), li = (e % (kB / 4)) * 4;
    if (j0 + cl >= m || li >= bsz) continue;
    const long long off = (j0 + cl) * ldd + li;
    const float4 v = make_float4(sm.ds[cl][li], sm.ds[cl][li + 1], sm.ds[cl][li + 2],
                                 sm.ds[cl][li + 3]);
    if (li + 4 <= bsz) {
      *reinterpret_cast<float4*>(dcur + off) = v;
      if (dcur_hi) {
        const float4 hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        *reinterpret_cast<float4*>(dcur_hi + off) = hi;
        *reinterpret_cast<float4*>(dcur_lo + off) =
            make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
      }
    } else {
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (li + u >= bsz) break;
        dcur[off + u] = vv[u];
        if (dcur_hi) {
          const float hi = tf32_hi(vv[u]);
          dcur_hi[off + u] = hi;
          dcur_lo[off + u] = vv[u] - hi;
        }
      }
    }
  }
  for (int e = tid; e < kB * kCols4; e += kThreads) {
    const int li = e / kCols4, cl = e % kCols4;
    if (li >= bsz || j0 + cl >= m) continue;
    const int16_t q = sm.cs[cl][li];
    const long long o = sm.orow[li] + j0 + cl;
    codes[o] = q;
    if (w_hat) {
      const float4 tv = sm.tab[li][cl];
      w_hat[o] = __fmul_rn(tv.y, __fsub_rn(float(q), tv.w));  // quant.cpp:33-35
    }
  }
  __syncthreads();
  stamp(trace, 5);
}
}  // namespace l4

// The sweep table of one super-block: {w, s, 1/s, z} of W[order[li], j] and its
// grid for rows li in [r0, r1), laid out [block][16-column slab][128 rows][16]
// float4 so an in-block CTA's 128 x 16 block is one contiguous 32 KB copy; rows
// past r1 and columns past m are padding {0, 1, 1, 0}.  sbad[block][slab] != 0:
// a scale outside scale_safe() -- that CTA's chain divides exactly.
__global__ void sweep_table_kernel(const float* __restrict__ w, long long ldw, long long r0,
                                   long long r1, long long m, int slabs,
                                   const int32_t* __restrict__ order, QCfg c,
                                   const float* __restrict__ scales,
                                   const int32_t* __restrict__ zeros, float4* __restrict__ tab,
                                   int* __restrict__ sbad) {
  const long long nblk = (r1 - r0 + kB - 1) / kB;
  const long long per_blk = (long long)slabs * kB * l4::kCols4;
  const long long total = nblk * per_blk;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / per_blk, rem = e % per_blk;
    const long long slab = rem / (kB * l4::kCols4), r2 = rem % (kB * l4::kCols4);
    const long long lr = r2 / l4::kCols4, cl = r2 % l4::kCols4;
    const long long li = r0 + b * kB + lr, jj = slab * l4::kCols4 + cl;
    float4 v = make_float4(0.f, 1.f, 1.f, 0.f);
    if (li < r1 && jj < m) {
      const long long orig = __ldg(order + li);
      const long long g = group_of(c, orig, jj);
      const float sv = __ldg(scales + g);
      v = make_float4(__ldg(w + orig * ldw + jj), sv, rcp_refined(sv), float(__ldg(zeros + g)));
      if (!scale_safe(sv)) atomicOr(sbad + b * slabs + slab, 1);
    }
    tab[e] = v;
  }
}

void launch_inblock4(const float* w, long long ldw, const int32_t* order, const float* acc,
                     int use_acc, const float* gpl, const float* gtt, const float* dprev, int bprev,
                     float* dcur, float* dch, float* dcl, const QCfg& c, const float* scales,
                     const int32_t* zeros, long long n, long long m, long long ib, int bsz,
                     int16_t* codes, float* w_hat, long long ldo, long long ldd, int trace,
                     bool pdl, cudaStream_t st, const float4* tabb = nullptr,
                     const int* tab_sbad = nullptr) {
  // function attributes are per device: set on every launch (cheap)
  cudaFuncSetAttribute(l4::inblock4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(l4::Smem)));
  // OCWG_SWEEP_EXACT_DIV=1 (tests): the IEEE-division chain even with safe scales
  const char* ex = std::getenv("OCWG_SWEEP_EXACT_DIV");
  trace = (trace ? 1 : 0) | (ex && std::atoi(ex) ? 2 : 0);
  const unsigned ctas = unsigned((m + l4::kCols4 - 1) / l4::kCols4);
  count_launches(1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(l4::kThreads);
  cfg.dynamicSmemBytes = sizeof(l4::Smem);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, l4::inblock4_kernel, w, ldw, order, acc, use_acc, gpl, gtt, dprev, bprev,
                     dcur, dch, dcl, c, scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, ldd,
                     trace, tabb, tab_sbad);
}

template <typename T, int RPT>
void launch_inblock(const float* w, long long ldw, const int32_t* order, const T* acc, int use_acc,
                    const T* gpl, const T* dprev, int bprev, T* dcur, float* dch, float* dcl,
                    const QCfg& c, const float* scales, const int32_t* zeros, long long n,
                    long long m, long long ib, int bsz, int16_t* codes, float* w_hat, long long ldo,
                    long long ldd, cudaStream_t st) {
  cudaFuncSetAttribute(inblock_g_kernel<T, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(InblockSmem<T>)));
  const unsigned ctas = unsigned((m + kCols - 1) / kCols);
  count_launches(1);
  inblock_g_kernel<T, RPT><<<ctas, 256, sizeof(InblockSmem<T>), st>>>(
      w, ldw, order, acc, use_acc, gpl, dprev, bprev, dcur, dch, dcl, c, scales, zeros, n, m, ib,
      bsz, codes, w_hat, ldo, ldd);
}

}  // namespace

constexpr long long kSuperRows = 512;  // rows of G D applied per trailing GEMM (K)
// left-looking fp32 sweep: rows per super-block and K parts per GEMM tile
// (OCWG_SWEEP_SUPER caps the super-block as for the right-looking sweep)
// (measured: 256-row super-blocks with 4 K parts per tile are slower -- each
// GEMM launch carries ~28 us of fixed cost and the parts' epilogues chain)
constexpr long long kLeftSuperRows = 512;
constexpr int kLeftSplit = 2;

size_t sweep_delta_elems(long long m) { return size_t(m) * kSuperRows; }
size_t sweep_table_bytes(long long m) {
  const long long slabs = (m + l4::kCols4 - 1) / l4::kCols4;
  const long long blocks = kLeftSuperRows / kB;
  return size_t(blocks * slabs * kB * l4::kCols4) * sizeof(float4) +
         size_t(blocks * slabs) * sizeof(int) + 256;
}

size_t sweep_kflag_ints(long long n, long long m) {
  return size_t(2 * ((kSuperRows + 255) / 256) * ((m + 255) / 256)) + 8;
}

// Two-level blocking: super-blocks of kSuperRows rows (4 blocks of 128).
// In-block kernel b applies, by lookahead, every earlier block of its own
// super-block (G[blk b, sb0:ib] D[sb0:ib]); one trailing GEMM per super-block
// (K = kSuperRows) applies it to all later rows.  Accumulator traffic and
// GEMM launches drop 4x against per-block trailing updates (which could not
// overlap the in-block kernels anyway: they cannot share an SM).
template <typename T>
void gptq_sweep_g(const float* w, long long ldw, long long n, long long m, const T* gpl,
                  const float* gtt, const T* ghi, const float* glo, const int32_t* order,
                  const QCfg& c, const float* scales, const int32_t* zeros, long long block,
                  int16_t* codes, float* w_hat, long long ldo, T* acc, T* const dpl[2],
                  float* const dhi[2], float* const dlo[2], int* kflag, cudaStream_t st,
                  void* tab, cudaStream_t aux, cudaEvent_t* ev) {
  // Block size is a pure re-association of the trailing update (SURVEY §0
  // item 11): the fp32 path always runs the tuned 128-row kernel (so the
  // reference default block_cols = 32, layerwise.hpp:14, is fast too); the
  // fp64 path honours block_cols (blocks above 128 rows run as 128-row blocks).
  const bool fast128 = sizeof(T) == 4 && gtt != nullptr;
  const long long B = fast128 ? kB : (block < 1 ? 1 : (block > kB ? kB : block));
  static const long long super_rows = [] {  // tuning switch: OCWG_SWEEP_SUPER=128..512
    const char* e = getenv("OCWG_SWEEP_SUPER");
    const long long v = e ? atoll(e) : kSuperRows;
    return std::min(kSuperRows, std::max<long long>(kB, v));
  }();
  const long long SB = std::max<long long>(1, super_rows / B);  // blocks per super-block
  const long long SBK = SB * B;
  const bool split = glo != nullptr;
  static const long long trace_ib = [] {
    const char* e = getenv("OCWG_SWEEP_TRACE_IB");
    return e ? atoll(e) : -1LL;
  }();
  // programmatic dependent launches between the sweep's own kernels (not the
  // first: it follows the factorisation and the grids' event); OCWG_SWEEP_PDL=0 off
  static const bool pdl_on = [] {
    const char* e = getenv("OCWG_SWEEP_PDL");
    return !(e && e[0] == '0');
  }();
  // OCWG_SWEEP_EVENTS=1 (debug): an event after every launch, per-launch times
  // printed to stderr at the end (events between launches disable PDL overlap)
  static const bool ev_on = [] {
    const char* e = getenv("OCWG_SWEEP_EVENTS");
    return e && e[0] == '1';
  }();
  std::vector<cudaEvent_t> tl;
  std::vector<char> tl_kind;
  auto mark = [&](char kind) {
    if (!ev_on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tl.push_back(e);
    tl_kind.push_back(kind);
  };
  auto report = [&] {
    if (!ev_on) return;
    cudaEventSynchronize(tl.back());
    float tot = 0.f;
    for (size_t i = 1; i < tl.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tl[i - 1], tl[i]);
      tot += ms;
      fprintf(stderr, "sweep-ev %c %zu %.2f us\n", tl_kind[i], i, ms * 1e3f);
    }
    fprintf(stderr, "sweep-ev total %.2f us\n", tot * 1e3f);
    for (cudaEvent_t e : tl) cudaEventDestroy(e);
  };
  mark('s');
  if constexpr (sizeof(T) == 4) {
    if (fast128 && split && kflag) {
      // Left-looking: before super-block s, ONE GEMM forms its rows' sum over
      // every earlier row, acc[s0:se, :] = G[s0:se, 0:s0] D[0:s0, :] (K = s0,
      // written once: no read-modify-write of the later rows' partial sums),
      // on 2-SM pairs with the K range split in two so 2 x 16 tiles fill the
      // GPU.  D of every row is kept (K-major, ld n: plain for the lookahead,
      // tf32 hi / lo for the GEMM).
      cudaMemsetAsync(kflag, 0, sweep_kflag_ints(n, m) * sizeof(int), st);
      const long long SBL = std::min<long long>(SBK, kLeftSuperRows);
      // Each super-block's {w, s, 1/s, z} table is built just in time on the
      // auxiliary stream, beside the GEMM that precedes the super-block (it is
      // read from L2 right after), so the in-block kernels copy instead of
      // gathering.  One buffer: the build waits for the previous super-block's
      // last in-block kernel.
      const int slabs = int((m + l4::kCols4 - 1) / l4::kCols4);
      const bool jit_tab = tab && aux && ev && SBL == kLeftSuperRows;
      float4* tabf = static_cast<float4*>(tab);
      int* tsbad = jit_tab ? reinterpret_cast<int*>(tabf + (kLeftSuperRows / kB) * slabs * kB *
                                                               l4::kCols4)
                           : nullptr;
      auto build_table = [&](long long s0, long long se, cudaStream_t on) {
        cudaMemsetAsync(tsbad, 0, size_t(kLeftSuperRows / kB) * slabs * sizeof(int), on);
        const long long total = ((se - s0 + kB - 1) / kB) * slabs * kB * l4::kCols4;
        const int blocks = int(std::min<long long>((total + 255) / 256, 148LL * 8));
        count_launches(1);
        sweep_table_kernel<<<blocks, 256, 0, on>>>(w, ldw, s0, se, m, slabs, order, c, scales,
                                                   zeros, tabf, tsbad);
      };
      for (long long s0 = 0, si = 0; s0 < n; s0 += SBL, ++si) {
        const long long se = std::min(n, s0 + SBL);
        if (jit_tab) {
          if (si == 0) {
            build_table(s0, se, st);
          } else {  // fork: the build runs beside this super-block's GEMM
            cudaEventRecord(ev[0], st);
            cudaStreamWaitEvent(aux, ev[0], 0);
            build_table(s0, se, aux);
            cudaEventRecord(ev[1], aux);
          }
        }
        if (si > 0) {
          bool done = tc_gemm2_presplit(se - s0, m, s0, 1.0f,
                                        reinterpret_cast<const float*>(ghi) + s0 * n,
                                        glo + s0 * n, n, dhi[0], dlo[0], n, 0.0f,
                                        reinterpret_cast<float*>(acc) + s0 * m, m, st, pdl_on,
                                        kLeftSplit, kflag, int(si));
          if (!done)
            done = tc_gemm_presplit(se - s0, m, s0, 1.0f,
                                    reinterpret_cast<const float*>(ghi) + s0 * n, glo + s0 * n, n,
                                    dhi[0], dlo[0], n, 0.0f,
                                    reinterpret_cast<float*>(acc) + s0 * m, m, st, 0, pdl_on);
          if (!done)
            gemm<T, T, T>(se - s0, m, s0, 1.0, gpl + s0 * n, n, false, dpl[0], n, true, 0.0,
                          acc + s0 * m, m, false, st);
          mark('g');
        }
        if (jit_tab && si > 0) cudaStreamWaitEvent(st, ev[1], 0);  // join
        for (long long ib = s0; ib < se; ib += B) {
          const int bsz = int(std::min(se, ib + B) - ib);
          const long long tb = (ib - s0) / B;
          launch_inblock4(w, ldw, order, reinterpret_cast<const float*>(acc), si >= 1,
                          reinterpret_cast<const float*>(gpl), gtt,
                          reinterpret_cast<const float*>(dpl[0]) + s0, int(ib - s0),
                          reinterpret_cast<float*>(dpl[0]) + ib, dhi[0] + ib, dlo[0] + ib, c,
                          scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, n, ib == trace_ib,
                          pdl_on && ib > 0, st,
                          jit_tab ? tabf + tb * slabs * kB * l4::kCols4 : nullptr,
                          jit_tab ? tsbad + tb * slabs : nullptr);
          mark('i');
        }
      }
      report();
      return;
    }
  }
  for (long long s0 = 0, si = 0; s0 < n; s0 += SBK, ++si) {
    const long long se = std::min(n, s0 + SBK);
    const int p = int(si & 1);
    for (long long ib = s0; ib < se; ib += B) {
      const int bsz = int(std::min(se, ib + B) - ib);
      const int bprev = int(ib - s0);  // lookahead rows: this super-block's earlier blocks
      const int use_acc = si >= 1;
      T* dcur = dpl[p] + bprev;
      float* dch = split ? dhi[p] + bprev : nullptr;
      float* dcl = split ? dlo[p] + bprev : nullptr;
      if (B <= 32)
        launch_inblock<T, 4>(w, ldw, order, acc, use_acc, gpl, dpl[p], bprev, dcur, dch, dcl, c,
                             scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, kSuperRows, st);
      else if (B <= 64)
        launch_inblock<T, 8>(w, ldw, order, acc, use_acc, gpl, dpl[p], bprev, dcur, dch, dcl, c,
                             scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, kSuperRows, st);
      else if (fast128)
        launch_inblock4(w, ldw, order, reinterpret_cast<const float*>(acc), use_acc,
                        reinterpret_cast<const float*>(gpl), gtt,
                        reinterpret_cast<const float*>(dpl[p]), bprev,
                        reinterpret_cast<float*>(dcur), dch, dcl, c, scales, zeros, n, m, ib, bsz,
                        codes, w_hat, ldo, kSuperRows, ib == trace_ib, pdl_on && ib > 0, st);
      else
        launch_inblock<T, 16>(w, ldw, order, acc, use_acc, gpl, dpl[p], bprev, dcur, dch, dcl, c,
                              scales, zeros, n, m, ib, bsz, codes, w_hat, ldo, kSuperRows, st);
      mark('i');
    }
    // trailing update of this super-block: acc[se:, :] (+)= G[se:, s0:se] D[s0:se, :]
    if (se < n) {
      const double beta = si == 0 ? 0.0 : 1.0;
      const long long kk = se - s0;
      bool done = false;
      if constexpr (sizeof(T) == 4) {
        static const bool pairs = [] {  // OCWG_SWEEP_GEMM2=0: 1-SM 128 x 128 tiles
          const char* e = getenv("OCWG_SWEEP_GEMM2");
          return !(e && e[0] == '0');
        }();
        static const long long pair_min_rows = [] {  // OCWG_SWEEP_GEMM2_MIN: smaller M -> 1-SM tiles
          const char* e = getenv("OCWG_SWEEP_GEMM2_MIN");
          return e ? atoll(e) : 1600LL;  // (measured: 1-SM 128 x 128 tiles win below ~1600 rows)
        }();
        if (split && pairs && n - se >= pair_min_rows)
          done = tc_gemm2_presplit(n - se, m, kk, 1.0f,
                                   reinterpret_cast<const float*>(ghi) + se * n + s0,
                                   glo + se * n + s0, n, dhi[p], dlo[p], kSuperRows, float(beta),
                                   reinterpret_cast<float*>(acc) + se * m, m, st, pdl_on);
        if (split && !done)
          done = tc_gemm_presplit(n - se, m, kk, 1.0f,
                                  reinterpret_cast<const float*>(ghi) + se * n + s0,
                                  glo + se * n + s0, n, dhi[p], dlo[p], kSuperRows, float(beta),
                                  reinterpret_cast<float*>(acc) + se * m, m, st, 0, pdl_on);
      }
      if (!done)
        gemm<T, T, T>(n - se, m, kk, 1.0, gpl + se * n + s0, n, false, dpl[p], kSuperRows, true,
                      beta, acc + se * m, m, false, st);
      mark('g');
    }
  }
  report();
}

int debug_sweep_trace(unsigned long long* out, int cap) {
  const int k = std::min(cap, 1024 * 8);
  return cudaMemcpyFromSymbol(out, l4::g_trace, sizeof(unsigned long long) * k) == cudaSuccess
             ? k
             : -1;
}

template void gptq_sweep_g<float>(const float*, long long, long long, long long, const float*,
                                  const float*, const float*, const float*, const int32_t*, const QCfg&,
                                  const float*, const int32_t*, long long, int16_t*, float*,
                                  long long, float*, float* const[2], float* const[2],
                                  float* const[2], int*, cudaStream_t, void*, cudaStream_t,
                                  cudaEvent_t*);
template void gptq_sweep_g<double>(const float*, long long, long long, long long, const double*,
                                   const float*, const double*, const float*, const int32_t*, const QCfg&,
                                   const float*, const int32_t*, long long, int16_t*, float*,
                                   long long, double*, double* const[2], float* const[2],
                                   float* const[2], int*, cudaStream_t, void*, cudaStream_t,
                                   cudaEvent_t*);

}  // namespace ocwg
