// FP32-accurate GEMM on the 5th-generation tensor cores (3xTF32), used by the
// fp32 factorisation (layerwise.cpp:43-51 restated as blocked Cholesky +
// triangular inverse) and by the GPTQ trailing update
// (layerwise.cpp:85-90, wp[ie:, :] -= U[ib:ie, ie:]^T E).
//
//   C[m x n] = beta * C + alpha * op(A) op(B)          (C fp32 row-major, ldc)
//
// Each fp32 operand x is split once into hi = tf32_rn(x) and lo = x - hi by a
// split kernel that also re-lays the operand out K-major (tiled transpose when
// needed: the MN-major tf32 form is avoided); the MMA warp issues three
// tcgen05.mma kind::tf32 per 8-deep k-step -- lo*hi + hi*lo + hi*hi -- into one
// FP32 TMEM accumulator, reproducing fp32 GEMM accuracy (tests/test_gpu_gemm.py;
// the GPTQ code match is unchanged vs fp32).  TMA with 128B swizzle
// into a 3-stage mbarrier ring; 128 x 128 CTA tiles; persistent CTAs over
// (batch, tile) with double-buffered TMEM so the C read-modify-write epilogue of
// one tile overlaps the MMAs of the next.  Batched form: operand b of a batch
// sits at base + b * stride (used by the log-depth triangular inverse).
#include <cuda.h>

#include <algorithm>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int TM = 128, TN = 128, TK = 32;       // tile; k-block = 32 fp32 = 128 bytes
constexpr int STAGES = 3;
constexpr int OPB = TM * TK * 4;                   // 16 KB per operand tile (TM == TN)
constexpr int STAGE_BYTES = 4 * OPB;               // A_hi, A_lo, B_hi, B_lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 256;

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
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (sm_100)
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}

// smem tile layouts (both 16 KB, 1024B aligned):
//  K-major  (box {32 k, 128 rows}):  row r at r*128B, 8-row atoms at 1024B.
//           MMA k-step kk (8 fp32 = 32B) starts at +32*kk inside the atom row.
//  MN-major (box {32 mn, 32 k} x 4 strips): strip s (32 mn) at s*4096B,
//           k-row at 128B, 8-k atoms at 1024B.  MMA k-step kk = +1024*kk.
__device__ __forceinline__ uint64_t op_desc(uint32_t base, bool mn_major, int kk) {
  return mn_major ? make_desc_sw128(base + 1024u * kk, 4096u, 1024u)
                  : make_desc_sw128(base + 32u * kk, 16u, 1024u);
}

__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap ahi, const __grid_constant__ CUtensorMap alo,
                   const __grid_constant__ CUtensorMap bhi, const __grid_constant__ CUtensorMap blo,
                   int a_mn, int b_mn, long long m, long long n, long long k, float alpha,
                   float beta, float* __restrict__ c, long long ldc, long long sc, int lower_only,
                   int tiles_m, int tiles_n, int ntiles) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_holder;

  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const int kb_total = int((k + TK - 1) / TK);
  // kind::tf32 instruction descriptor: D f32, A/B tf32, majors, N=128, M=128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) |
                         (uint32_t(b_mn) << 16) | (uint32_t(TN >> 3) << 17) |
                         (uint32_t(TM >> 4) << 24);

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
  // programmatic dependent launch (no-op otherwise): setup above overlaps the
  // previous kernel, whose outputs may be B and C
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // t -> (batch, tm, tn); the operand rows of batch b start at b*m (A) / b*n (B)
  const int per_batch = tiles_m * tiles_n;
  auto tile_of = [&](int t, int& tm, int& tn) {
    tm = (t % per_batch) / tiles_n;
    tn = t % tiles_n;
  };

  if (warp == 0) {
    if (lane == 0) {  // ============ TMA producer
      uint32_t stage = 0, phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int tm, tn;
        tile_of(t, tm, tn);
        if (lower_only && (long long)tn * TN > (long long)tm * TM + TM - 1) continue;
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1u);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          mbar_expect_tx(fb, STAGE_BYTES);
          const uint32_t s0 = sbase + stage * STAGE_BYTES;
          const int k0 = kb * TK;
          const CUtensorMap* maps[4] = {&ahi, &alo, &bhi, &blo};
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            const bool mn = (o < 2) ? a_mn : b_mn;
            const int bidx = t / per_batch;
            const int r0 = (o < 2) ? int(bidx * m) + tm * TM : int(bidx * n) + tn * TN;
            const uint32_t dst = s0 + o * OPB;
            if (mn) {
#pragma unroll
              for (int sidx = 0; sidx < 4; ++sidx)
                tma_load_2d(dst + sidx * 4096, maps[o], fb, r0 + sidx * 32, k0);
            } else {
              tma_load_2d(dst, maps[o], fb, k0, r0);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {  // ============ MMA issuer
    uint32_t stage = 0, phase = 0;
    int local = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int tm, tn;
      tile_of(t, tm, tn);
      if (lower_only && (long long)tn * TN > (long long)tm * TM + TM - 1) continue;
      const uint32_t acc = uint32_t(local & 1), use = uint32_t(local >> 1);
      ++local;
      mbar_wait(smem_u32(&tempty_bar[acc]), (use & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * TN;
      for (int kb = 0; kb < kb_total; ++kb) {
        mbar_wait(smem_u32(&full_bar[stage]), phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t s0 = sbase + stage * STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < TK / 8; ++kk) {
            const uint64_t ah = op_desc(s0, a_mn, kk), al = op_desc(s0 + OPB, a_mn, kk);
            const uint64_t bh = op_desc(s0 + 2 * OPB, b_mn, kk),
                           bl = op_desc(s0 + 3 * OPB, b_mn, kk);
            const uint32_t first = (kb > 0 || kk > 0) ? 1u : 0u;
            tc_mma_tf32(d_tmem, al, bh, idesc, first);  // small terms first
            tc_mma_tf32(d_tmem, ah, bl, idesc, 1u);
            tc_mma_tf32(d_tmem, ah, bh, idesc, 1u);
          }
          tc_commit(smem_u32(&empty_bar[stage]));
          if (kb + 1 == kb_total) tc_commit(smem_u32(&tfull_bar[acc]));
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else {  // ============ epilogue: C = beta C + alpha D
    const int q = warp & 3;
    int local = 0;
    const bool vec_ld = ((ldc & 3) == 0);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int tm, tn;
      tile_of(t, tm, tn);
      if (lower_only && (long long)tn * TN > (long long)tm * TM + TM - 1) continue;
      const uint32_t acc = uint32_t(local & 1), use = uint32_t(local >> 1);
      ++local;
      const long long row = (long long)tm * TM + q * 32 + lane;
      float* cbase = c + (long long)(t / per_batch) * sc + row * ldc + (long long)tn * TN;
      // C does not depend on the MMA: its first chunk is read before the
      // accumulator is ready, and each next chunk while the current one is stored
      auto load_c = [&](int c0, float (&v)[32]) {
        const long long col0 = (long long)tn * TN + c0;
        float* crow = cbase + c0;
        if (beta == 0.f || row >= m) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.f;
        } else if (vec_ld && col0 + 32 <= n && ((reinterpret_cast<uintptr_t>(crow) & 15) == 0)) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 o = reinterpret_cast<const float4*>(crow)[e];
            v[4 * e] = o.x, v[4 * e + 1] = o.y, v[4 * e + 2] = o.z, v[4 * e + 3] = o.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = col0 + e < n ? crow[e] : 0.f;
        }
      };
      float cv[32], nv[32];
      load_c(0, nv);
      mbar_wait(smem_u32(&tfull_bar[acc]), use & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < TN; c0 += 32) {
#pragma unroll
        for (int e = 0; e < 32; ++e) cv[e] = nv[e];
        if (c0 + 32 < TN) load_c(c0 + 32, nv);
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
        const long long col0 = (long long)tn * TN + c0;
        if (row < m) {
          float* crow = cbase + c0;
#pragma unroll
          for (int e = 0; e < 32; ++e) cv[e] = fmaf(alpha, __uint_as_float(r[e]), beta * cv[e]);
          if (vec_ld && col0 + 32 <= n && ((reinterpret_cast<uintptr_t>(crow) & 15) == 0)) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              reinterpret_cast<float4*>(crow)[e] =
                  make_float4(cv[4 * e], cv[4 * e + 1], cv[4 * e + 2], cv[4 * e + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (col0 + e < n) crow[e] = cv[e];
          }
        }
      }
      tc_fence_before();
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

// K-major hi/lo split of an fp32 operand: out[r][c] (rows x cols, ld = ldo)
// takes src[r*lds + c] (trans = 0) or src[c*lds + r] (trans = 1, tiled
// transpose through shared memory); hi = tf32 round-to-nearest(x), lo = x - hi.
__global__ void split_tf32_kernel(const float* __restrict__ src, long long lds, int trans,
                                  long long rows, long long cols, float* hi, float* lo,
                                  long long ldo, long long src_batch_stride) {
  __shared__ float tile[32][33];
  src += (long long)blockIdx.z * src_batch_stride;
  hi += (long long)blockIdx.z * rows * ldo;
  lo += (long long)blockIdx.z * rows * ldo;
  const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    float x = 0.f;
    if (trans) {  // read src[(c0+k)*lds + r0+tx] coalesced, store transposed
      if (c0 + k < cols && r0 + tx < rows) x = src[(c0 + k) * lds + r0 + tx];
      tile[tx][k] = x;
    } else {
      if (r0 + k < rows && c0 + tx < cols) x = src[(r0 + k) * lds + c0 + tx];
      tile[k][tx] = x;
    }
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const long long r = r0 + k, c = c0 + tx;
    if (r < rows && c < cols) {
      const float x = tile[k][tx];
      uint32_t u = __float_as_uint(x);
      u = (u + 0xFFFu + ((u >> 13) & 1u)) & ~0x1FFFu;  // RNE to 10 mantissa bits
      const float h = __uint_as_float(u);
      hi[r * ldo + c] = h;
      lo[r * ldo + c] = x - h;
    }
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
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

// 2D map over a compact fp32 matrix (rows x cols, ld), box {32 inner, box_outer}
bool make_map(CUtensorMap* map, const float* base, long long rows, long long cols, long long ld,
              int box_outer) {
  const cuuint64_t gdim[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t gstride[1] = {cuuint64_t(ld) * 4};
  const cuuint32_t box[2] = {32, cuuint32_t(box_outer)};
  const cuuint32_t es[2] = {1, 1};
  return encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms_tc() { return device_sms(); }

inline long long pad4(long long x) { return (x + 3) & ~3LL; }

void ensure_attr() {  // function attributes are per device: set on every call
  cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
}

}  // namespace

size_t tc_gemm_workspace_floats(long long m, long long n, long long k, int batch) {
  return size_t(2 * (m + n) * pad4(k)) * size_t(batch) + 64;
}

// op(A)[i][kk] = ta ? A[kk*lda + i] : A[i*lda + kk];  op(B)[kk][j] = tb ? B[j*ldb + kk] : B[kk*ldb + j]
// Batch b uses A + b*sa, B + b*sb, C + b*sc.  Operands are re-laid out K-major
// (A as m x k, B as n x k per batch, stacked) by the split kernel.
bool tc_gemm_tf32x3(int batch, long long m, long long n, long long k, float alpha, const float* a,
                    long long lda, long long sa, bool ta, const float* b, long long ldb,
                    long long sb, bool tb, float beta, float* c, long long ldc, long long sc,
                    bool lower_only, float* ws, size_t ws_floats, cudaStream_t st) {
  if (m <= 0 || n <= 0 || batch <= 0) return true;
  if (!encoder() || k <= 0) return false;
  if (ws_floats < tc_gemm_workspace_floats(m, n, k, batch)) return false;
  if ((long long)batch * std::max(m, n) >= (1LL << 31)) return false;
  ensure_attr();
  const long long ldk = pad4(k);
  float* a_hi = ws;
  float* a_lo = a_hi + batch * m * ldk;
  float* b_hi = a_lo + batch * m * ldk;
  float* b_lo = b_hi + batch * n * ldk;
  count_launches(3);
  split_tf32_kernel<<<dim3(unsigned((k + 31) / 32), unsigned((m + 31) / 32), unsigned(batch)), 256,
                      0, st>>>(a, lda, ta ? 1 : 0, m, k, a_hi, a_lo, ldk, sa);
  split_tf32_kernel<<<dim3(unsigned((k + 31) / 32), unsigned((n + 31) / 32), unsigned(batch)), 256,
                      0, st>>>(b, ldb, tb ? 0 : 1, n, k, b_hi, b_lo, ldk, sb);
  CUtensorMap mah, mal, mbh, mbl;
  if (!make_map(&mah, a_hi, batch * m, k, ldk, TM) || !make_map(&mal, a_lo, batch * m, k, ldk, TM) ||
      !make_map(&mbh, b_hi, batch * n, k, ldk, TN) || !make_map(&mbl, b_lo, batch * n, k, ldk, TN))
    return false;
  const int tiles_m = int((m + TM - 1) / TM), tiles_n = int((n + TN - 1) / TN);
  const int ntiles = tiles_m * tiles_n * batch;
  const int grid = std::min(ntiles, num_sms_tc());
  tc_gemm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(mah, mal, mbh, mbl, 0, 0, m, n, k, alpha, beta,
                                                    c, ldc, sc, lower_only ? 1 : 0, tiles_m,
                                                    tiles_n, ntiles);
  return cudaGetLastError() == cudaSuccess;
}

// Operands already split and K-major: A = (a_hi + a_lo) is m x k (row stride
// lda), B = (b_hi + b_lo) is n x k (row stride ldb); C = beta C + alpha A B^T.
// Used by the GPTQ sweep, whose G and D are emitted pre-split by the Cholesky
// and in-block kernels (no split launches on the sweep's critical path).
bool tc_gemm_presplit(long long m, long long n, long long k, float alpha, const float* a_hi,
                      const float* a_lo, long long lda, const float* b_hi, const float* b_lo,
                      long long ldb, float beta, float* c, long long ldc, cudaStream_t st,
                      int max_ctas, bool pdl) {
  if (m <= 0 || n <= 0) return true;
  if (!encoder() || k <= 0 || m >= (1LL << 31) || n >= (1LL << 31)) return false;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if ((lda & 3) || (ldb & 3) || !al16(a_hi) || !al16(a_lo) || !al16(b_hi) || !al16(b_lo))
    return false;
  ensure_attr();
  CUtensorMap mah, mal, mbh, mbl;
  if (!make_map(&mah, a_hi, m, k, lda, TM) || !make_map(&mal, a_lo, m, k, lda, TM) ||
      !make_map(&mbh, b_hi, n, k, ldb, TN) || !make_map(&mbl, b_lo, n, k, ldb, TN))
    return false;
  const int tiles_m = int((m + TM - 1) / TM), tiles_n = int((n + TN - 1) / TN);
  const int ntiles = tiles_m * tiles_n;
  const int cap = max_ctas > 0 ? std::min(max_ctas, num_sms_tc()) : num_sms_tc();
  const int grid = std::min(ntiles, cap);
  count_launches(1);
  if (pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, tc_gemm_kernel, mah, mal, mbh, mbl, 0, 0, m, n, k, alpha, beta,
                              c, ldc, 0LL, 0, tiles_m, tiles_n, ntiles) == cudaSuccess;
  }
  tc_gemm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(mah, mal, mbh, mbl, 0, 0, m, n, k, alpha, beta,
                                                    c, ldc, 0, 0, tiles_m, tiles_n, ntiles);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace ocwg
