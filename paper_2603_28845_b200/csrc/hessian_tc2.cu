// Calibration Hessian H = X^T X on CTA PAIRS (tcgen05 cta_group::2), the
// production path of hessian_tc (stats.cpp:16, `gram += xp^T xp`, bf16 X).
//
// Same contract, tile scheduling and in-kernel split reduction as
// hessian_tc.cu; what changes is the MMA shape.  A cluster of 2 CTAs on one
// TPC computes a 256 x 256 output tile with tcgen05.mma.cta_group::2 M=256
// N=256 K=16: each CTA stages only ITS half of A (128 channels) and ITS half
// of B (128 channels) per 64-token k-block, and the pair's tensor cores read
// both halves.  Per SM that is 8 KB of shared-memory operand traffic per
// 128x256x16 MMA instead of 12 KB for the single-CTA 128x256 tile -- the
// single-CTA kernel's limiter (sm__mem_tensor ~80 %).  Each CTA's TMEM holds
// its 128 rows x 256 columns of the accumulator (2 x 256 columns,
// double-buffered).
//
// Synchronisation: both CTAs' TMA loads complete on the LEADER's full
// barrier (.cta_group::2 TMA, barrier address mapped into the leader with
// mapa); the leader issues the MMAs and commits (multicast) to both CTAs'
// empty and accumulator-full barriers; both CTAs' epilogue warps arrive on
// the leader's accumulator-empty barrier (remote arrive from the peer).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int TM = 128;          // rows per CTA (M = 256 per pair)
constexpr int TNH = 128;         // B channels per CTA (N = 256 per pair)
constexpr int TK = 64;           // tokens per k-block
constexpr int STAGES = 6;
constexpr int A_BYTES = TM * TK * 2;
constexpr int B_BYTES = TNH * TK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 32 KB per CTA
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 512;
constexpr long long kMaxSplitTokens = 16384;

// kind::f16: D f32, A/B bf16, both MN-major, M = 256, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                            (uint32_t(256 >> 3) << 17) | (uint32_t(256 >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory location in CTA `cta` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag_eq(const int* p, int v) {
  while (ld_acquire(p) != v) __nanosleep(64);
}
// TMA load whose completion is signalled on the pair LEADER's barrier
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// commit the leader's MMAs to the barrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
// SMEM descriptor, SWIZZLE_128B, MN-major: 64-channel strips at LBO, 8-token atoms at SBO
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// upper 256 x 256 tiles (bi <= bj), column block by column block
__device__ __forceinline__ void pair_tile(int tile, int& bi, int& bj) {
  int b = 0, base = 0;
  while (tile >= base + b + 1) {
    base += b + 1;
    ++b;
  }
  bj = b;
  bi = tile - base;
}

__global__ void __launch_bounds__(THREADS, 1)
    hessian_tc2_kernel(const __grid_constant__ CUtensorMap xmap, long long tokens, int dim,
                       int ntiles, int splits, long long kb_total, float* __restrict__ h,
                       int accumulate, int* __restrict__ tile_flag) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_holder;

  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const uint32_t rank = cta_rank();
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const long long nunits = (long long)ntiles * splits;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull_bar[a]), 1);
      mbar_init(smem_u32(&tempty_bar[a]), 8);  // 4 epilogue warps x 2 CTAs (leader's)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();  // barriers initialised in both CTAs before any cross-CTA traffic
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_holder;

  if (warp == 0) {
    // ====================== TMA producer (both CTAs, own halves) ======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (long long u = pair; u < nunits; u += npairs) {
        const int split = int(u / ntiles), tile = int(u % ntiles);
        int bi, bj;
        pair_tile(tile, bi, bj);
        const long long kb0 = kb_total * split / splits, kb1 = kb_total * (split + 1) / splits;
        const int arow = bi * 256 + int(rank) * TM, bcol = bj * 256 + int(rank) * TNH;
        for (long long kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          if (rank == 0) mbar_expect_tx(fb, 2 * STAGE_BYTES);
          const uint32_t fb_leader = mapa(fb, 0);
          const uint32_t sa = sbase + stage * STAGE_BYTES, sb = sa + A_BYTES;
          const int t0 = int(kb * TK);
#pragma unroll
          for (int s = 0; s < TM / 64; ++s)
            tma_load_2d_pair(sa + s * (64 * TK * 2), &xmap, fb_leader, arow + s * 64, t0);
#pragma unroll
          for (int s = 0; s < TNH / 64; ++s)
            tma_load_2d_pair(sb + s * (64 * TK * 2), &xmap, fb_leader, bcol + s * 64, t0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ====================== MMA issuer (leader only) ======================
    if (rank == 0) {
      uint32_t stage = 0, phase = 0;
      long long local = 0;
      for (long long u = pair; u < nunits; u += npairs, ++local) {
        const int split = int(u / ntiles);
        const long long kb0 = kb_total * split / splits, kb1 = kb_total * (split + 1) / splits;
        const uint32_t acc = uint32_t(local & 1), use = uint32_t(local >> 1);
        mbar_wait(smem_u32(&tempty_bar[acc]), (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (long long kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = sbase + stage * STAGE_BYTES, sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < TK / 16; ++k) {
              const uint64_t ad = make_desc_sw128(sa + k * 2048, 64 * TK * 2, 1024);
              const uint64_t bd = make_desc_sw128(sb + k * 2048, 64 * TK * 2, 1024);
              tc_mma_pair(d_tmem, ad, bd, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            tc_commit_pair(smem_u32(&empty_bar[stage]));  // frees the stage in both CTAs
            if (kb + 1 == kb1) tc_commit_pair(smem_u32(&tfull_bar[acc]));
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {
    // ====================== epilogue (warps 2..5, both CTAs) ======================
    const int q = warp & 3;
    long long local = 0;
    for (long long u = pair; u < nunits; u += npairs, ++local) {
      const int split = int(u / ntiles), tile = int(u % ntiles);
      int bi, bj;
      pair_tile(tile, bi, bj);
      const uint32_t acc = uint32_t(local & 1), use = uint32_t(local >> 1);
      const int flag_id = tile * 2 + int(rank);
      if (warp == 2 && lane == 0) wait_flag_eq(tile_flag + flag_id, split);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(smem_u32(&tfull_bar[acc]), use & 1u);
      tc_fence_after();
      const long long row_base = (long long)bi * 256 + rank * TM;
      const long long row = row_base + q * 32 + lane;
      const bool first = split == 0 && !accumulate, last = split == splits - 1;
      auto load_chunk = [&](int c0, float (&v)[32]) {
        const long long col0 = (long long)bj * 256 + c0;
        const float* hrow = h + row * dim + col0;
        if (first || row >= dim || col0 + 31 < row_base) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.f;
        } else if (col0 + 32 <= dim) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 o = __ldcg(reinterpret_cast<const float4*>(hrow) + e);
            v[4 * e] = o.x, v[4 * e + 1] = o.y, v[4 * e + 2] = o.z, v[4 * e + 3] = o.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = col0 + e < dim ? __ldcg(hrow + e) : 0.f;
        }
      };
      float v[32], nv[32];
      load_chunk(0, nv);
#pragma unroll 1
      for (int c0 = 0; c0 < 256; c0 += 32) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = nv[e];
        if (c0 + 32 < 256) load_chunk(c0 + 32, nv);
        uint32_t r[32];
        const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + acc * 256 + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const long long col0 = (long long)bj * 256 + c0;
        if (col0 + 31 < row_base) continue;  // chunk entirely below the diagonal
        if (row < dim) {
          float* hrow = h + row * dim + col0;
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] += __uint_as_float(r[e]);
          if (col0 >= row && col0 + 32 <= dim) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              reinterpret_cast<float4*>(hrow)[e] =
                  make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (col0 + e < dim && col0 + e >= row) hrow[e] = v[e];
          }
        }
        if (last) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const long long col = col0 + e;
            if (row < dim && col < dim && col > row) h[col * dim + row] = v[e];
          }
        }
      }
      __threadfence();
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 2 && lane == 0) st_release(tile_flag + flag_id, split + 1);
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa(smem_u32(&tempty_bar[acc]), 0));
    }
  }

  tc_fence_before();
  cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder2() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiled(nullptr);
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

struct Plan2 {
  int ntiles, splits;
  long long kb_total;
};

Plan2 make_plan2(long long tokens, long long dim, int npairs) {
  Plan2 p;
  const int nb = int((dim + 255) / 256);
  p.ntiles = nb * (nb + 1) / 2;
  p.kb_total = (tokens + TK - 1) / TK;
  const long long min_splits = (p.kb_total * TK + kMaxSplitTokens - 1) / kMaxSplitTokens;
  int best = int(std::max<long long>(1, min_splits));
  double best_eff = -1;
  for (int s = best; s <= best + 16; ++s) {
    if (p.kb_total / s < 16 && s > best) break;
    const long long units = (long long)p.ntiles * s;
    const long long waves = (units + npairs - 1) / npairs;
    const double eff = double(units) / double(waves * npairs);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  p.splits = best;
  return p;
}

int num_sms2() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

size_t hessian_tc2_workspace_bytes(long long tokens, long long dim) {
  const Plan2 p = make_plan2(tokens, dim, num_sms2() / 2);
  return size_t(p.ntiles) * 2 * sizeof(int) + 256;
}

// returns 0 ok, -1 unsupported (caller falls back), >0 cuda error
int hessian_tc2(const uint16_t* x, long long tokens, long long dim, float* h, int accumulate,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  if (dim % 8 != 0 || dim <= 0 || tokens <= 0 || tokens > (1LL << 31) || dim > (1LL << 31))
    return -1;
  EncodeTiled enc = encoder2();
  if (!enc) return -1;
  const int npairs_max = num_sms2() / 2;
  const Plan2 p = make_plan2(tokens, dim, npairs_max);
  if (ws_bytes < size_t(p.ntiles) * 2 * sizeof(int)) return -2;
  CUtensorMap map;
  const cuuint64_t gdim[2] = {cuuint64_t(dim), cuuint64_t(tokens)};
  const cuuint64_t gstride[1] = {cuuint64_t(dim) * 2};
  const cuuint32_t box[2] = {64, TK};
  const cuuint32_t estride[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(x), gdim, gstride, box,
          estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  static const bool attr = [] {
    cudaFuncSetAttribute(hessian_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_BYTES);
    cudaFuncSetAttribute(hessian_tc2_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return true;
  }();
  (void)attr;
  int* tile_flag = static_cast<int*>(ws);
  cudaMemsetAsync(tile_flag, 0, size_t(p.ntiles) * 2 * sizeof(int), st);
  const long long units = (long long)p.ntiles * p.splits;
  const int npairs = int(std::min<long long>(units, npairs_max));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(2 * npairs));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  count_launches(1);
  cudaError_t e = cudaLaunchKernelEx(&cfg, hessian_tc2_kernel, map, tokens, int(dim), p.ntiles,
                                     p.splits, p.kb_total, h, accumulate, tile_flag);
  if (e != cudaSuccess) return int(e);
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : int(e);
}

}  // namespace ocwg
