// Calibration statistics on the tensor cores (replaces stats.cpp:10-19):
//   gram  (+)= sum_s A_s^T B_s    over a symmetric set of operand pairs
//   cross (+)= sum_s P_s^T Q_s
// where every operand is a T x N bf16 array (token-major, as activations
// arrive).  Uses:
//   * bf16 calibration tokens: gram = X^T X, one segment (the hot path);
//   * fp32 tokens (the reference API, accumulate_stats(stats, x_fp, x_hat)):
//     X_hat = P1 + P2 and D = X - X_hat = D1 + D2 split into bf16 parts, then
//       gram  = P1'P1 + P1'P2 + P2'P1        cross = P1'D1 + P1'D2 + P2'D1
//     (the dropped terms are below 2^-16 relative; fp64 outputs).
//
// Kernel: CTA PAIRS (tcgen05 cta_group::2) compute 256 x 256 output tiles,
// M = 256 x N = 256 x K = 16 MMAs with fp32 accumulation in TMEM (two 256-
// column accumulators per SM, double-buffered).  Each CTA stages its half of
// A and its half of B per 64-token k-block with .cta_group::2 TMA (128B-
// swizzled MN-major boxes straight from the token-major arrays) into a
// 6-stage ring.  Warp roles per CTA: TMA producer, MMA issuer (leader only),
// four epilogue warps.
//
// Work units are (tile, token window): the segments of a tile form one
// virtual K axis, cut into windows of <= 16384 tokens so each TMEM
// accumulation stays short (fp32 accuracy).  Units are CLAIMED from an atomic
// counter in window-major order by the leader's producer and handed to every
// role of both CTAs through a small shared-memory ring, so a claimed unit is
// always held by a running CTA.  The window partials of a tile are added into
// the output in window order (tile flag: acquire w, add, release w+1) --
// deterministic, no partial buffers -- and a unit only waits on units with a
// smaller index, which were claimed earlier by running CTAs: no deadlock
// whatever the number of co-resident pairs.  Gram tiles are the upper ones
// (bi <= bj); the last window mirrors them into the lower triangle.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "tc_ptx.cuh"

namespace ocwg {
namespace {

using namespace ptx;

constexpr int TM = 128;   // rows per CTA (M = 256 per pair)
constexpr int TNH = 128;  // B channels per CTA (N = 256 per pair)
constexpr int TK = 64;    // tokens per k-block
constexpr int STAGES = 6;
constexpr int RING = 4;   // claimed-unit hand-off depth
constexpr int A_BYTES = TM * TK * 2;
constexpr int B_BYTES = TNH * TK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 32 KB per CTA
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 512;
constexpr long long kWindowTokens = 16384;  // default window (GramSpec::window_tokens)
// consumers of a ring slot: leader MMA + 4 leader epilogue warps + peer producer + 4 peer epilogue warps
constexpr uint32_t kRingConsumers = 10;

// kind::f16: D f32, A/B bf16, both MN-major, M = 256, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                            (uint32_t(256 >> 3) << 17) | (uint32_t(256 >> 4) << 24);

struct alignas(64) GramParams {
  CUtensorMap maps[4];
  long long kb_seg;      // k-blocks per segment (ceil(T / 64))
  int dim;
  int nb;                // 256-blocks per side
  int n_gram;            // upper tiles (0 when no gram output)
  int n_cross;           // full tiles (0 when no cross output)
  int splits;            // windows per tile
  int nunits;            // (n_gram + n_cross) * splits
  int gseg, cseg;
  int seg_a[2][3], seg_b[2][3];  // [kind][segment] -> map index
  void* out[2];          // gram, cross (dim x dim, row-major)
  int accumulate;
  int serp;              // serpentine token order across waves
};

// upper 256 x 256 tiles (bi <= bj), column block by column block
__device__ __forceinline__ void upper_tile(int tile, int& bi, int& bj) {
  int b = 0, base = 0;
  while (tile >= base + b + 1) {
    base += b + 1;
    ++b;
  }
  bj = b;
  bi = tile - base;
}

struct Unit {
  int kind, tile, bi, bj, split;
  long long kb0, kb1;
};
__device__ __forceinline__ Unit decode(const GramParams& p, int u) {
  Unit x;
  const int nt = p.n_gram + p.n_cross;
  x.split = u / nt;
  const int t = u % nt;
  x.tile = t;
  if (t < p.n_gram) {
    x.kind = 0;
    upper_tile(t, x.bi, x.bj);
  } else {
    x.kind = 1;
    x.bi = (t - p.n_gram) / p.nb;
    x.bj = (t - p.n_gram) % p.nb;
  }
  const long long kbt = p.kb_seg * (x.kind == 0 ? p.gseg : p.cseg);
  x.kb0 = kbt * x.split / p.splits;
  x.kb1 = kbt * (x.split + 1) / p.splits;
  return x;
}

template <typename OutT>
__global__ void __launch_bounds__(THREADS, 1)
    gram_tc_kernel(const __grid_constant__ GramParams p, int* __restrict__ tile_flag,
                   int* __restrict__ counter) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t ufull_bar[RING], uempty_bar[RING];
  __shared__ int unit_ring[RING];
  __shared__ uint32_t tmem_base_holder;

  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const uint32_t rank = cta_rank();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull_bar[a]), 1);
      mbar_init(smem_u32(&tempty_bar[a]), 8);  // 4 epilogue warps x 2 CTAs (leader's)
    }
    for (int r = 0; r < RING; ++r) {
      mbar_init(smem_u32(&ufull_bar[r]), 1);
      mbar_init(smem_u32(&uempty_bar[r]), kRingConsumers);  // (leader's)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int m = 0; m < 4; ++m) prefetch_tmap(&p.maps[m]);
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

  // next claimed unit from the ring (every role of both CTAs reads every slot
  // once, then frees it on the leader); -1 ends the loop
  auto take_unit = [&](int it, bool arrive) -> int {
    const int slot = it % RING;
    const uint32_t ph = uint32_t(it / RING) & 1u;
    mbar_wait_cluster(smem_u32(&ufull_bar[slot]), ph);
    const int u = *reinterpret_cast<volatile int*>(&unit_ring[slot]);
    if (arrive) mbar_arrive_cluster(mapa(smem_u32(&uempty_bar[slot]), 0));
    return u;
  };

  if (warp == 0) {
    // ====================== unit claims (leader) + TMA producer (both CTAs) ======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int it = 0;; ++it) {
        int u;
        if (rank == 0) {
          const int slot = it % RING;
          const uint32_t ph = uint32_t(it / RING) & 1u;
          mbar_wait(smem_u32(&uempty_bar[slot]), ph ^ 1u);
          u = atomicAdd(counter, 1);
          if (u >= p.nunits) u = -1;
          unit_ring[slot] = u;
          st_cluster_u32(mapa(smem_u32(&unit_ring[slot]), 1), uint32_t(u));
          mbar_arrive_cluster(mapa(smem_u32(&ufull_bar[slot]), 0));
          mbar_arrive_cluster(mapa(smem_u32(&ufull_bar[slot]), 1));
        } else {
          u = take_unit(it, true);
        }
        if (u < 0) break;
        const Unit x = decode(p, u);
        const int arow = x.bi * 256 + int(rank) * TM, bcol = x.bj * 256 + int(rank) * TNH;
        // serpentine: units of odd waves (u / pairs) walk their tokens backwards,
        // starting where the previous wave's units ended -- that stretch of X is
        // still in L2 (DRAM read per launch 5.4 -> 4.3 GB at C2)
        const bool rev = p.serp && ((u / int(gridDim.x >> 1)) & 1);
        int seg = int((rev ? x.kb1 - 1 : x.kb0) / p.kb_seg);
        long long kk = (rev ? x.kb1 - 1 : x.kb0) - seg * p.kb_seg;  // k-block within the segment
        for (long long i = x.kb0; i < x.kb1; ++i) {
          const int t0 = int(kk * TK);
          const CUtensorMap* ma = &p.maps[p.seg_a[x.kind][seg]];
          const CUtensorMap* mb = &p.maps[p.seg_b[x.kind][seg]];
          if (rev) {
            if (--kk < 0) {
              kk = p.kb_seg - 1;
              --seg;
            }
          } else if (++kk == p.kb_seg) {
            kk = 0;
            ++seg;
          }
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          if (rank == 0) mbar_expect_tx(fb, 2 * STAGE_BYTES);
          const uint32_t fb_leader = mapa(fb, 0);
          const uint32_t sa = sbase + stage * STAGE_BYTES, sb = sa + A_BYTES;
#pragma unroll
          for (int s = 0; s < TM / 64; ++s)
            tma_load_2d_pair(sa + s * (64 * TK * 2), ma, fb_leader, arow + s * 64, t0);
#pragma unroll
          for (int s = 0; s < TNH / 64; ++s)
            tma_load_2d_pair(sb + s * (64 * TK * 2), mb, fb_leader, bcol + s * 64, t0);
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
      for (int it = 0;; ++it) {
        int u = 0;
        if (lane == 0) u = take_unit(it, true);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u < 0) break;
        const Unit x = decode(p, u);
        const uint32_t acc = uint32_t(it & 1), use = uint32_t(it >> 1);
        mbar_wait(smem_u32(&tempty_bar[acc]), (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (long long kb = x.kb0; kb < x.kb1; ++kb) {
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = sbase + stage * STAGE_BYTES, sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < TK / 16; ++k) {
              const uint64_t ad = desc_sw128(sa + k * 2048, 64 * TK * 2, 1024);
              const uint64_t bd = desc_sw128(sb + k * 2048, 64 * TK * 2, 1024);
              const uint32_t accum = (kb > x.kb0 || k > 0) ? 1u : 0u;
              asm volatile(
                  "{\n\t.reg .pred q;\n\t"
                  "setp.ne.b32 q, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(d_tmem),
                  "l"(ad), "l"(bd), "r"(kIdesc), "r"(accum)
                  : "memory");
            }
            tc_commit_pair(smem_u32(&empty_bar[stage]));  // frees the stage in both CTAs
            if (kb + 1 == x.kb1) tc_commit_pair(smem_u32(&tfull_bar[acc]));
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
    for (int it = 0;; ++it) {
      int u = 0;
      if (lane == 0) u = take_unit(it, true);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u < 0) break;
      const Unit x = decode(p, u);
      const uint32_t acc = uint32_t(it & 1), use = uint32_t(it >> 1);
      const int flag_id = x.tile * 2 + int(rank);
      if (warp == 2 && lane == 0) {
        while (ld_acquire(tile_flag + flag_id) != x.split) __nanosleep(64);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(smem_u32(&tfull_bar[acc]), use & 1u);
      tc_fence_after();
      const int dim = p.dim;
      const bool gram = x.kind == 0;
      OutT* out = static_cast<OutT*>(p.out[x.kind]);
      const long long row_base = (long long)x.bi * 256 + rank * TM;
      const long long row = row_base + q * 32 + lane;
      const bool first = x.split == 0 && !p.accumulate, last = x.split == p.splits - 1;
      const bool vec_ok = (dim & 3) == 0;  // 16-byte aligned rows
      const long long colt = (long long)x.bj * 256;
      if constexpr (sizeof(OutT) == 4) {
        // fp32 output (the hot path's H): the chunk's old values are loaded one
        // chunk ahead, so their L2 latency overlaps the TMEM load and the adds
        auto load_old = [&](int c0, float (&o)[32]) {
          const long long col0 = colt + c0;
          const float* src = out + row * dim + col0;
          if (first || row >= dim || (gram && col0 + 31 < row_base)) {
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = 0.f;
          } else if (vec_ok && col0 + 32 <= dim) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float4 f = __ldcg(reinterpret_cast<const float4*>(src) + e);
              o[4 * e] = f.x, o[4 * e + 1] = f.y, o[4 * e + 2] = f.z, o[4 * e + 3] = f.w;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = col0 + e < dim ? __ldcg(src + e) : 0.f;
          }
        };
        float v[32], nv[32];
        load_old(0, nv);
#pragma unroll 1
        for (int c0 = 0; c0 < 256; c0 += 32) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = nv[e];
          if (c0 + 32 < 256) load_old(c0 + 32, nv);
          uint32_t r[32];
          tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + acc * 256 + c0, r);
          const long long col0 = colt + c0;
          if (gram && col0 + 31 < row_base) continue;  // chunk entirely below the diagonal
          if (row >= dim) continue;
          float* orow = out + row * dim + col0;
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] += __uint_as_float(r[e]);
          if (vec_ok && col0 + 32 <= dim && (!gram || col0 >= row)) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              reinterpret_cast<float4*>(orow)[e] =
                  make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (col0 + e < dim && (!gram || col0 + e >= row)) orow[e] = v[e];
          }
          if (gram && last) {  // mirror into the lower triangle (coalesced over lanes)
#pragma unroll 4
            for (int e = 0; e < 32; ++e) {
              const long long col = col0 + e;
              if (col < dim && col > row) out[col * dim + row] = v[e];
            }
          }
        }
      } else {
        // fp64 output (the reference API's CalibStats): plain read-modify-write
#pragma unroll 1
        for (int c0 = 0; c0 < 256; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + acc * 256 + c0, r);
          const long long col0 = colt + c0;
          if (gram && col0 + 31 < row_base) continue;
          if (row >= dim) continue;
          double* orow = out + row * dim + col0;
#pragma unroll 4
          for (int e = 0; e < 32; ++e) {
            const long long col = col0 + e;
            if (col < dim && (!gram || col >= row)) {
              const double nvv = (first ? 0.0 : __ldcg(orow + e)) + double(__uint_as_float(r[e]));
              orow[e] = nvv;
              if (gram && last && col > row) out[col * dim + row] = nvv;
            }
          }
        }
      }
      __threadfence();
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 2 && lane == 0) st_release(tile_flag + flag_id, x.split + 1);
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

EncodeTiled encoder() {
  static EncodeTiled fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiled(nullptr);
    return reinterpret_cast<EncodeTiled>(ptr);
  }();
  return fn;
}

int splits_for(long long kb_max, int ntiles, int npairs, long long window) {
  const long long min_splits = (kb_max * TK + window - 1) / window;
  int best = int(std::max<long long>(1, min_splits));
  double best_eff = -1;
  for (int s = best, s0 = best; s <= s0 + 16; ++s) {
    if (kb_max / s < 16 && s > s0) break;
    const long long units = (long long)ntiles * s;
    const long long waves = (units + npairs - 1) / npairs;
    const double eff = double(units) / double(waves * npairs);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

}  // namespace

size_t gram_tc_workspace_bytes(long long dim) {
  const long long nb = (dim + 255) / 256;
  return size_t(nb * (nb + 1) / 2 + nb * nb) * 2 * sizeof(int) + 256;
}

int gram_tc(const GramSpec& s, void* ws, size_t ws_bytes, cudaStream_t st) {
  const long long dim = s.dim, T = s.tokens;
  if (dim <= 0 || T <= 0 || T > (1LL << 31) || dim > (1LL << 30) || s.ld % 8 != 0 || s.ld < dim)
    return -1;
  if (s.nops < 1 || s.nops > 4 || (s.gseg < 1 && s.cseg < 1) || s.gseg > 3 || s.cseg > 3)
    return -1;
  EncodeTiled enc = encoder();
  if (!enc) return -1;
  if (ws_bytes < gram_tc_workspace_bytes(dim)) return -2;
  int dev = 0;
  cudaGetDevice(&dev);
  GramParams p{};
  for (int m = 0; m < 4; ++m) {
    const uint16_t* ptr = s.ops[m < s.nops ? m : 0];
    const cuuint64_t gdim[2] = {cuuint64_t(dim), cuuint64_t(T)};
    const cuuint64_t gstride[1] = {cuuint64_t(s.ld) * 2};
    const cuuint32_t box[2] = {64, TK};
    const cuuint32_t estride[2] = {1, 1};
    if (enc(&p.maps[m], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(ptr), gdim,
            gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -1;
  }
  p.kb_seg = (T + TK - 1) / TK;
  p.dim = int(dim);
  p.nb = int((dim + 255) / 256);
  p.n_gram = s.gseg > 0 ? p.nb * (p.nb + 1) / 2 : 0;
  p.n_cross = s.cseg > 0 ? p.nb * p.nb : 0;
  p.gseg = std::max(1, s.gseg);
  p.cseg = std::max(1, s.cseg);
  for (int k = 0; k < 3; ++k) {
    p.seg_a[0][k] = s.gA[k];
    p.seg_b[0][k] = s.gB[k];
    p.seg_a[1][k] = s.cA[k];
    p.seg_b[1][k] = s.cB[k];
  }
  p.out[0] = s.gram;
  p.out[1] = s.cross;
  p.accumulate = s.accumulate ? 1 : 0;
  p.serp = 1;
  if (const char* e = getenv("OCWG_GRAM_SERP")) p.serp = atoi(e);  // A/B switch
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int npairs_hw = sms / 2;
  const long long kb_max = p.kb_seg * std::max(s.gseg, s.cseg);
  const int ntiles = p.n_gram + p.n_cross;
  const long long window = s.window_tokens > 0 ? std::max<long long>(TK, s.window_tokens) : kWindowTokens;
  p.splits = splits_for(kb_max, ntiles, npairs_hw, window);
  const long long units = (long long)ntiles * p.splits;
  if (units >= (1LL << 31)) return -1;
  p.nunits = int(units);

  auto kern = s.f64 ? gram_tc_kernel<double> : gram_tc_kernel<float>;
  // function attributes are per device: set them on every call (cheap)
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int* tile_flag = static_cast<int*>(ws);
  int* counter = tile_flag + size_t(ntiles) * 2;
  cudaMemsetAsync(ws, 0, size_t(ntiles) * 2 * sizeof(int) + sizeof(int), st);
  cudaLaunchConfig_t cfg{};
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
  // as many pairs as can be resident (any number works: units are claimed)
  int max_clusters = 0;
  cfg.gridDim = dim3(unsigned(2 * npairs_hw));
  if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
    max_clusters = npairs_hw;
  cudaGetLastError();
  const int npairs = int(std::min<long long>({units, (long long)npairs_hw, (long long)max_clusters}));
  cfg.gridDim = dim3(unsigned(2 * npairs));
  count_launches(1);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, tile_flag, counter);
  if (e != cudaSuccess) return int(e);
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : int(e);
}

size_t hessian_tc_workspace_bytes(long long, long long dim) { return gram_tc_workspace_bytes(dim); }

int hessian_tc(const uint16_t* x, long long tokens, long long dim, float* h, int accumulate,
               void* ws, size_t ws_bytes, cudaStream_t st) {
  if (dim % 8 != 0) return -1;
  GramSpec s{};
  s.tokens = tokens;
  s.dim = dim;
  s.ld = dim;
  s.ops[0] = x;
  s.nops = 1;
  s.gseg = 1;
  s.gram = h;
  s.accumulate = accumulate != 0;
  return gram_tc(s, ws, ws_bytes, st);
}

}  // namespace ocwg
