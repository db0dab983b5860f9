// Calibration Hessian H = X^T X on the 5th-generation tensor cores
// (replaces stats.cpp:16, `gram += xp^T xp`, for bf16 calibration tokens).
//
//   X: tokens x dim, bf16, row-major (token-major, as activations arrive).
//   H: dim x dim fp32, symmetric.
//
// Design (sm_100a):
//   * Only output tiles touching the upper triangle are computed (SYRK:
//     T*N*(N+1) flops instead of 2*T*N^2); the last split mirrors them.
//   * CTA tile 128 (i) x 256 (j) channels, one tcgen05.mma.cta_group::1
//     kind::f16 M=128 N=256 K=16 per 16 tokens, FP32 accumulators in TMEM
//     (2 x 256 columns: the epilogue drains one while the MMA fills the other).
//   * Both operands are channel-contiguous ("MN-major"): A = X[:, i-block]^T,
//     B = X[:, j-block]; staged by TMA (2D map over X, 64-channel x 64-token
//     boxes, 128B swizzle) into a 4-stage mbarrier ring -- no transpose pass.
//   * Warp roles: w0 TMA producer, w1 MMA issuer (+TMEM owner), w2..w5 epilogue.
//   * Persistent CTAs over (split-K, tile) units, split-major so all CTAs
//     stream the same token window (X read from HBM ~once, reused via L2).
//     Splits cap each TMEM accumulation at 16384 tokens (fp32 accuracy).
//   * The split partials are reduced inside the kernel, in split order: the
//     epilogue of (tile, s) waits for the tile's flag to reach s (acquire),
//     adds its accumulator into H's upper entries, and releases s+1; the last
//     split also writes the mirrored lower entries.  Deterministic (fixed
//     order, no data atomics) and overlapped with the MMAs of other units --
//     no partial buffers and no separate finalize pass.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int TM = 128, TN = 256, TK = 64;        // CTA tile and k-block (tokens)
constexpr int STAGES = 4;
constexpr int A_BYTES = TM * TK * 2;              // 16 KB
constexpr int B_BYTES = TN * TK * 2;              // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;    // 48 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 512;
constexpr long long kMaxSplitTokens = 16384;

// ----------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// SMEM matrix descriptor, SWIZZLE_128B, MN-major canonical layout:
//   ((8 x 16B, n strips @ LBO), (8 rows @ 128B, k groups @ SBO))
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (sm_100)
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both MN-major, M=128, N=256
constexpr uint32_t kIdesc = (1u << 4)            // c_format = F32
                            | (1u << 7)          // a_format = BF16
                            | (1u << 10)         // b_format = BF16
                            | (1u << 15)         // a_major = MN
                            | (1u << 16)         // b_major = MN
                            | (uint32_t(TN >> 3) << 17) | (uint32_t(TM >> 4) << 24);

struct TileMap {
  int nbi, nbj, ntiles;
};

__device__ __forceinline__ void tile_coords(int tile, int nbi, int& bi, int& bj) {
  // tiles (bi, bj) with bi*TM <= bj*TN + TN - 1, enumerated column block by
  // column block: column block bj holds min(nbi, 2*bj + 2) row blocks
  int b = 0, base = 0;
  while (true) {
    const int cnt = min(nbi, (b + 1) * (TN / TM));
    if (tile < base + cnt) {
      bi = tile - base;
      bj = b;
      return;
    }
    base += cnt;
    ++b;
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    hessian_tc_kernel(const __grid_constant__ CUtensorMap xmap, long long tokens, int dim,
                      int nbi, int ntiles, int splits, long long kb_total, float* __restrict__ h,
                      int accumulate, int* __restrict__ tile_flag) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_holder;

  const uint32_t base_raw = smem_u32(smem_raw);
  const uint32_t sbase = (base_raw + 1023u) & ~1023u;  // SW128 needs 1024B-aligned atoms
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const long long nunits = (long long)ntiles * splits;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull_bar[a]), 1);
      mbar_init(smem_u32(&tempty_bar[a]), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_holder)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_holder;

  if (warp == 0) {
    // ====================== TMA producer ======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int split = int(u / ntiles), tile = int(u % ntiles);
        int bi, bj;
        tile_coords(tile, nbi, bi, bj);
        const long long kb0 = kb_total * split / splits, kb1 = kb_total * (split + 1) / splits;
        for (long long kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          mbar_expect_tx(fb, STAGE_BYTES);
          const uint32_t sa = sbase + stage * STAGE_BYTES, sb = sa + A_BYTES;
          const int t0 = int(kb * TK);
#pragma unroll
          for (int s = 0; s < TM / 64; ++s)
            tma_load_2d(sa + s * (64 * TK * 2), &xmap, fb, bi * TM + s * 64, t0);
#pragma unroll
          for (int s = 0; s < TN / 64; ++s)
            tma_load_2d(sb + s * (64 * TK * 2), &xmap, fb, bj * TN + s * 64, t0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ====================== MMA issuer ======================
    uint32_t stage = 0, phase = 0;
    long long local = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x, ++local) {
      const int split = int(u / ntiles);
      const long long kb0 = kb_total * split / splits, kb1 = kb_total * (split + 1) / splits;
      const uint32_t acc = uint32_t(local & 1);
      const uint32_t use = uint32_t(local >> 1);
      mbar_wait(smem_u32(&tempty_bar[acc]), (use & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * TN;
      for (long long kb = kb0; kb < kb1; ++kb) {
        mbar_wait(smem_u32(&full_bar[stage]), phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = sbase + stage * STAGE_BYTES, sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < TK / 16; ++k) {
            // 16 tokens = 2 swizzle atoms of 8 rows x 128B
            const uint64_t ad = make_desc_sw128(sa + k * 2048, 64 * TK * 2, 1024);
            const uint64_t bd = make_desc_sw128(sb + k * 2048, 64 * TK * 2, 1024);
            tc_mma_bf16(d_tmem, ad, bd, kIdesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          tc_commit(smem_u32(&empty_bar[stage]));  // frees the smem slot when the MMAs finish
          if (kb + 1 == kb1) tc_commit(smem_u32(&tfull_bar[acc]));
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else {
    // ====================== epilogue (warps 2..5) ======================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    long long local = 0;
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x, ++local) {
      const int split = int(u / ntiles), tile = int(u % ntiles);
      int bi, bj;
      tile_coords(tile, nbi, bi, bj);
      const uint32_t acc = uint32_t(local & 1);
      const uint32_t use = uint32_t(local >> 1);
      // partials of this tile are added in split order
      if (warp == 2 && lane == 0) wait_flag_eq(tile_flag + tile, split);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(smem_u32(&tfull_bar[acc]), use & 1u);
      tc_fence_after();
      const long long row = (long long)bi * TM + q * 32 + lane;
      const bool first = split == 0 && !accumulate, last = split == splits - 1;
      // running partial of this lane's row, one 32-column chunk ahead (loads in flight
      // while the current chunk is added and stored)
      auto load_chunk = [&](int c0, float (&v)[32]) {
        const long long col0 = (long long)bj * TN + c0;
        const float* hrow = h + row * dim + col0;
        if (first || row >= dim || col0 + 31 < (long long)bi * TM) {
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
      for (int c0 = 0; c0 < TN; c0 += 32) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = nv[e];
        if (c0 + 32 < TN) load_chunk(c0 + 32, nv);
        uint32_t r[32];
        const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + acc * TN + c0;
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
        const long long col0 = (long long)bj * TN + c0;
        if (col0 + 31 < (long long)bi * TM) continue;  // chunk entirely below the diagonal
        if (row < dim) {
          float* hrow = h + row * dim + col0;
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] += __uint_as_float(r[e]);
          // upper entries (row <= col) accumulate; the lower half is the mirror
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
          // mirror: H[col][row] = H[row][col] for col > row (coalesced along rows)
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
      if (warp == 2 && lane == 0) st_release(tile_flag + tile, split + 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[acc]));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled get_encoder() {
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

struct Plan {
  int nbi, nbj, ntiles, splits;
  long long kb_total;
};

Plan make_plan(long long tokens, long long dim, int sms) {
  Plan p;
  p.nbi = int((dim + TM - 1) / TM);
  p.nbj = int((dim + TN - 1) / TN);
  p.ntiles = 0;
  for (int b = 0; b < p.nbj; ++b) p.ntiles += std::min(p.nbi, (b + 1) * (TN / TM));
  p.kb_total = (tokens + TK - 1) / TK;
  // split-K factor.  Accuracy bound: the tensor core's fp32 accumulation over
  // one TMEM tile is capped at kMaxSplitTokens tokens (measured: 262144
  // tokens in one accumulator -> 1.6e-4 relative error, above the 1e-4
  // tolerance; 16384 -> ~1e-5); the split partials are chained in fp32 in split order.
  // Within that bound, pick the best wave efficiency.
  const long long min_splits = (p.kb_total * TK + kMaxSplitTokens - 1) / kMaxSplitTokens;
  int best = int(std::max<long long>(1, min_splits));
  double best_eff = -1;
  for (int s = best; s <= best + 16; ++s) {
    if (p.kb_total / s < 16 && s > best) break;
    const long long units = (long long)p.ntiles * s;
    const long long waves = (units + sms - 1) / sms;
    const double eff = double(units) / double(waves * sms);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  p.splits = best;
  return p;
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

bool use_pairs() {
  static const bool on = [] {
    const char* e = getenv("OCWG_HESSIAN_2CTA");
    return !(e && e[0] == '0');
  }();
  return on;
}

size_t hessian_tc_workspace_bytes(long long tokens, long long dim) {
  const Plan p = make_plan(tokens, dim, num_sms());
  return std::max(size_t(p.ntiles) * sizeof(int) + 256, hessian_tc2_workspace_bytes(tokens, dim));
}

// returns 0 ok, -1 unsupported shape (caller must use another kernel), >0 cuda error
int hessian_tc(const uint16_t* x, long long tokens, long long dim, float* h, int accumulate,
               void* ws, size_t ws_bytes, cudaStream_t st) {
  if (use_pairs()) {
    const int r = hessian_tc2(x, tokens, dim, h, accumulate, ws, ws_bytes, st);
    if (r != -1) return r;  // -1: shape unsupported by the pair kernel -> single-CTA kernel
  }
  if (dim % 8 != 0 || dim <= 0 || tokens <= 0 || tokens > (1LL << 31) || dim > (1LL << 31))
    return -1;
  EncodeTiled enc = get_encoder();
  if (!enc) return -1;
  const int sms = num_sms();
  const Plan p = make_plan(tokens, dim, sms);
  if (ws_bytes < size_t(p.ntiles) * sizeof(int)) return -2;

  CUtensorMap map;
  const cuuint64_t gdim[2] = {cuuint64_t(dim), cuuint64_t(tokens)};
  const cuuint64_t gstride[1] = {cuuint64_t(dim) * 2};
  const cuuint32_t box[2] = {64, TK};
  const cuuint32_t estride[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(x), gdim,
                   gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -1;

  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(hessian_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_BYTES);
    attr_set = true;
  }
  int* tile_flag = static_cast<int*>(ws);
  cudaMemsetAsync(tile_flag, 0, size_t(p.ntiles) * sizeof(int), st);
  const long long units = (long long)p.ntiles * p.splits;
  const int grid = int(std::min<long long>(units, sms));
  count_launches(1);
  hessian_tc_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(map, tokens, int(dim), p.nbi, p.ntiles,
                                                       p.splits, p.kb_total, h, accumulate,
                                                       tile_flag);
  if (getenv("OCWG_DEBUG_HESSIAN")) {
    cudaStreamSynchronize(st);
    std::vector<int> f(p.ntiles);
    cudaMemcpy(f.data(), tile_flag, f.size() * 4, cudaMemcpyDeviceToHost);
    int mn = 1 << 30, mx = -1;
    for (int v : f) mn = std::min(mn, v), mx = std::max(mx, v);
    fprintf(stderr, "hessian_tc: dim %lld tok %lld grid %d ntiles %d splits %d flags [%d, %d] err %s ws %p h %p\n",
            dim, tokens, grid, p.ntiles, p.splits, mn, mx, cudaGetErrorString(cudaGetLastError()), ws, (void*)h);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : int(e);
}

}  // namespace ocwg
