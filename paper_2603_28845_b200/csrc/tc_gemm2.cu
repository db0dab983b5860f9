// The GPTQ sweep's trailing update on CTA PAIRS (tcgen05 cta_group::2):
//   C[m x n] = beta C + alpha A B^T,  A = a_hi + a_lo (m x k), B = b_hi + b_lo
//   (n x k), both K-major and pre-split (the Cholesky emits G that way, the
//   in-block kernel D) -- layerwise.cpp:85-90 in closed form (sweep.cu).
// 3xTF32 (lo*hi + hi*lo + hi*hi) into one fp32 TMEM accumulator, as
// tc_gemm.cu.  What changes is the tile: a cluster of 2 CTAs computes a
// 256 x 256 output tile with tcgen05.mma.cta_group::2 kind::tf32 M=256 N=256,
// each CTA staging only its 128 rows of A and its 128 rows of B per k-block.
// Per SM that halves the L2 -> shared operand traffic of the 1-CTA 128 x 128
// tile, which is what bounds that kernel (ncu: tensor pipe ~13 % active,
// ~9.6 TB/s of operand traffic across the GPU).
//
// Synchronisation as hessian_tc2.cu: both CTAs' TMA loads complete on the
// leader's full barrier; the leader issues the MMAs and commits (multicast) to
// both CTAs' empty / accumulator-full barriers; both CTAs' epilogue warps
// arrive on the leader's accumulator-empty barrier.
#include <cuda.h>

#include <algorithm>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int TM = 128;   // rows of A per CTA (M = 256 per pair)
constexpr int TNH = 128;  // rows of B per CTA (N = 256 per pair)
constexpr int TK = 32;    // k per block: 32 fp32 = one 128-byte swizzle row
constexpr int STAGES = 3;
constexpr int OPB = 128 * TK * 4;          // 16 KB per operand half-tile
constexpr int STAGE_BYTES = 4 * OPB;       // A_hi, A_lo, B_hi, B_lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int THREADS = 320;  // TMA warp, MMA warp, 8 epilogue warps (2 per TMEM lane quadrant)
constexpr uint32_t TMEM_COLS = 512;

// kind::tf32: D f32, A/B tf32, both K-major, M = 256, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(256 >> 3) << 17) |
                            (uint32_t(256 >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
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
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
// K-major, SWIZZLE_128B: 128-byte k-rows, 8-row atoms at 1024 B; k-step kk at +32 kk
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {
  const uint32_t saddr = base + 32u * kk;
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((16u >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((1024u >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap ahi, const __grid_constant__ CUtensorMap alo,
                    const __grid_constant__ CUtensorMap bhi, const __grid_constant__ CUtensorMap blo,
                    long long m, long long n, long long k, float alpha, float beta,
                    float* __restrict__ c, long long ldc, int tiles_n, int ntiles, int ksplit,
                    int* __restrict__ kflag, int epoch) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_holder;

  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const uint32_t rank = cta_rank();
  const int pair = int(blockIdx.x >> 1), npairs = int(gridDim.x >> 1);
  const int kb_total = int((k + TK - 1) / TK);
  // units: (tile, K part), part-major; part q of a tile covers k-blocks
  // [kb_total q / ksplit, kb_total (q+1) / ksplit).  Part q > 0 adds into C
  // after part q-1 has stored (per-(tile, CTA) flag: part q releases
  // 4 epoch + q + 1): a fixed summation order, deterministic, no zero-fill.  A
  // part is assigned after the parts before it (round-robin over resident
  // pairs), so it never waits on a unit that has not started.
  const int nunits = ntiles * ksplit;
  auto kb_range = [&](int t, int& kb0, int& kb1) {
    const int q = t / ntiles;
    kb0 = int((long long)kb_total * q / ksplit);
    kb1 = int((long long)kb_total * (q + 1) / ksplit);
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull_bar[a]), 1);
      mbar_init(smem_u32(&tempty_bar[a]), 16);  // 8 epilogue warps x 2 CTAs (leader's)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_holder;
  // programmatic dependent launch: setup above overlaps the previous kernel;
  // B (D) and C (acc) are its outputs.  Dependents may start their own setup.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ====================== TMA producer (both CTAs, own halves) ======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int t = pair; t < nunits; t += npairs) {
        const int tile = t % ntiles, tm = tile / tiles_n, tn = tile % tiles_n;
        const int arow = tm * 256 + int(rank) * TM, brow = tn * 256 + int(rank) * TNH;
        int kb0, kb1;
        kb_range(t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          if (rank == 0) mbar_expect_tx(fb, 2 * STAGE_BYTES);
          const uint32_t fb_leader = mapa(fb, 0);
          const uint32_t s0 = sbase + stage * STAGE_BYTES;
          const int k0 = kb * TK;
          tma_load_2d_pair(s0, &ahi, fb_leader, k0, arow);
          tma_load_2d_pair(s0 + OPB, &alo, fb_leader, k0, arow);
          tma_load_2d_pair(s0 + 2 * OPB, &bhi, fb_leader, k0, brow);
          tma_load_2d_pair(s0 + 3 * OPB, &blo, fb_leader, k0, brow);
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
      int local = 0;
      for (int t = pair; t < nunits; t += npairs, ++local) {
        const uint32_t acc = uint32_t(local & 1), use = uint32_t(local >> 1);
        int kb0, kb1;
        kb_range(t, kb0, kb1);
        mbar_wait(smem_u32(&tempty_bar[acc]), (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t s0 = sbase + stage * STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < TK / 8; ++kk) {
              const uint64_t ah = kdesc(s0, kk), al = kdesc(s0 + OPB, kk);
              const uint64_t bh = kdesc(s0 + 2 * OPB, kk), bl = kdesc(s0 + 3 * OPB, kk);
              tc_mma_pair_tf32(d_tmem, al, bh, (kb > kb0 || kk > 0) ? 1u : 0u);  // small terms first
              tc_mma_pair_tf32(d_tmem, ah, bl, 1u);
              tc_mma_pair_tf32(d_tmem, ah, bh, 1u);
            }
            tc_commit_pair(smem_u32(&empty_bar[stage]));
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
    // ====================== epilogue (warps 2..9, both CTAs): C = beta C + alpha D
    // warp w reads TMEM lane quadrant w % 4; warps 2-5 / 6-9 take columns 0-127 / 128-255
    const int q = warp & 3, cbeg = ((warp - 2) >> 2) * 128;
    const bool vec = (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0;
    int local = 0;
    for (int t = pair; t < nunits; t += npairs, ++local) {
      const int tile = t % ntiles, tm = tile / tiles_n, tn = tile % tiles_n;
      const int part = t / ntiles;
      const uint32_t acc = uint32_t(local & 1), use = uint32_t(local >> 1);
      const long long row = (long long)tm * 256 + rank * TM + q * 32 + lane;
      float* crow_base = c + row * ldc + (long long)tn * 256;
      int* flag = kflag + tile * 2 + int(rank);
      const float bt = part == 0 ? beta : 1.f;  // later parts add to the first
      if (part > 0) {  // the previous part of this tile has stored its rows
        if (warp == 2 && lane == 0)
          while (ld_acquire_gpu(flag) != 4 * epoch + part) __nanosleep(64);
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
      auto load_c = [&](int c0, float (&v)[32]) {
        const long long col0 = (long long)tn * 256 + c0;
        const float* cr = crow_base + c0;
        if (bt == 0.f || row >= m) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.f;
        } else if (vec && col0 + 32 <= n) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 o = __ldcg(reinterpret_cast<const float4*>(cr) + e);
            v[4 * e] = o.x, v[4 * e + 1] = o.y, v[4 * e + 2] = o.z, v[4 * e + 3] = o.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = col0 + e < n ? __ldcg(cr + e) : 0.f;
        }
      };
      float cv[32], nv[32];
      load_c(cbeg, nv);
      mbar_wait(smem_u32(&tfull_bar[acc]), use & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = cbeg; c0 < cbeg + 128; c0 += 32) {
#pragma unroll
        for (int e = 0; e < 32; ++e) cv[e] = nv[e];
        if (c0 + 32 < cbeg + 128) load_c(c0 + 32, nv);
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
        const long long col0 = (long long)tn * 256 + c0;
        if (row < m) {
          float* cr = crow_base + c0;
#pragma unroll
          for (int e = 0; e < 32; ++e) cv[e] = fmaf(alpha, __uint_as_float(r[e]), bt * cv[e]);
          if (vec && col0 + 32 <= n) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              reinterpret_cast<float4*>(cr)[e] =
                  make_float4(cv[4 * e], cv[4 * e + 1], cv[4 * e + 2], cv[4 * e + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (col0 + e < n) cr[e] = cv[e];
          }
        }
      }
      tc_fence_before();
      if (part + 1 < ksplit) {  // publish this CTA's rows of the tile to the next part
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (warp == 2 && lane == 0) st_release_gpu(flag, 4 * epoch + part + 1);
      }
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

EncodeTiled encoder3() {
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

bool kmap(CUtensorMap* map, const float* base, long long rows, long long cols, long long ld) {
  const cuuint64_t gdim[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t gstride[1] = {cuuint64_t(ld) * 4};
  const cuuint32_t box[2] = {TK, 128};
  const cuuint32_t es[2] = {1, 1};
  return encoder3()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim,
                    gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms3() { return device_sms(); }

}  // namespace

bool tc_gemm2_presplit(long long m, long long n, long long k, float alpha, const float* a_hi,
                       const float* a_lo, long long lda, const float* b_hi, const float* b_lo,
                       long long ldb, float beta, float* c, long long ldc, cudaStream_t st,
                       bool pdl, int ksplit, int* kflag, int epoch) {
  if (m <= 0 || n <= 0) return true;
  if (!encoder3() || k <= 0 || m >= (1LL << 31) || n >= (1LL << 31)) return false;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if ((lda & 3) || (ldb & 3) || !al16(a_hi) || !al16(a_lo) || !al16(b_hi) || !al16(b_lo))
    return false;
  CUtensorMap mah, mal, mbh, mbl;
  if (!kmap(&mah, a_hi, m, k, lda) || !kmap(&mal, a_lo, m, k, lda) || !kmap(&mbh, b_hi, n, k, ldb) ||
      !kmap(&mbl, b_lo, n, k, ldb))
    return false;
  cudaFuncSetAttribute(tc_gemm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  const int tiles_m = int((m + 255) / 256), tiles_n = int((n + 255) / 256);
  const int ntiles = tiles_m * tiles_n;
  const long long kb_total = (k + TK - 1) / TK;
  if (ksplit < 1 || !kflag) ksplit = 1;
  ksplit = int(std::min<long long>({(long long)ksplit, 4LL, kb_total}));
  const int nunits = ntiles * ksplit;
  int npairs = std::min(nunits, num_sms3() / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(2 * npairs));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  if (ksplit > 1) {  // part-1 units wait on part-0 units: every pair must be resident
    int max_clusters = 0;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, tc_gemm2_kernel, &cfg) == cudaSuccess &&
        max_clusters >= 1)
      npairs = std::min(npairs, max_clusters);
    cudaGetLastError();
    cfg.gridDim = dim3(unsigned(2 * npairs));
    cfg.numAttrs = pdl ? 2 : 1;
  }
  count_launches(1);
  return cudaLaunchKernelEx(&cfg, tc_gemm2_kernel, mah, mal, mbh, mbl, m, n, k, alpha, beta, c,
                            ldc, tiles_n, ntiles, ksplit, kflag, epoch) == cudaSuccess;
}

}  // namespace ocwg
