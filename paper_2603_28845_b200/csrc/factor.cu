// On-GPU factorisation for GPTQ (replaces layerwise.cpp:31-51):
//   hd = fp64(H); damp = percdamp*mean(diag(hd)); hd += damp*I;
//   hp = P hd P^T;  hinv = hp^-1;  U = upper Cholesky factor of hinv.
//
// The reference forms hinv and factors it again (8n^3/3 flops).  Here
//   A = J hp J = L L^T                 (one Cholesky, n^3/3 flops)
// and the sweep consumes L directly.  U = (J L J)^-1 by uniqueness of the
// Cholesky factor, so with D = diag(U) the reference's error propagation
//   wp[k] -= U[i,k] * (wp[i] - w_hat[i]) / U[i,i]              (layerwise.cpp:76-90)
// unrolls to the closed form (V = D^-1 U unit upper)
//   w_cur[k] = w[k] + sum_{i<k} G[k,i] * (w[i] - w_hat[i]),    G = V^-T - I,
//   G[k,i]  = L[n-1-i, n-1-k] / L[n-1-k, n-1-k]                 (i < k).
// i.e. G is the unit-lower LDL^T factor of hp read in processing order.  No
// triangular inverse is on the hot path; the inverse (for the H^-1 / U
// parity artefacts of ocwg_gptq_factor) is computed only on request.
//
// Cholesky: one persistent kernel over 64x64 tiles with acquire/release tile
// flags.  CTA 0 (the owner) runs the critical path alone on its SM: per column
// c it applies the k = c-1 term to S'[c,c], factors it (factor_tile64, which
// also yields X = L[c,c]^-T), and forms L[c+1,c] = S[c+1,c] X, keeping
// L[c+1,c] in shared memory for the next column -- no inter-CTA hand-off on
// the chain.  The other CTAs take work items in column order from an atomic
// counter: partial S'[c..c+1, c] (sum over k < c-1), full tiles (c+2.., c)
// (accumulate, then S X with X read from the diagonal tile's upper triangle)
// and one emission item per column for the owner's tiles.  Tile products run
// as 3xTF32 on the warp tensor cores over cp.async-staged row-major tiles.
// Items only wait on earlier items or on the owner, which only waits on
// earlier items, so with every CTA resident the schedule cannot deadlock.
// Large n runs macro panels: the kernel over a column range, then one tcgen05
// 3xTF32 SYRK for the trailing matrix (gemm.cu / tc_gemm.cu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda.h>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int TB = 64;    // tile
constexpr int CT = 256;   // threads per CTA: 16 x 16, each a 4x4 register block

// A[i][j] = T(double(H[o(i)][o(j)]) + (i==j)*damp), o(i) = order[n-1-i]; lower only
template <typename T>
__global__ void build_input_kernel(const float* __restrict__ h, long long n,
                                   const int32_t* __restrict__ order, const double* damp, T* a) {
  const double dmp = *damp;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n, j = e % n;
    if (j > i) continue;
    const long long oi = order[n - 1 - i], oj = order[n - 1 - j];
    double v = double(h[oi * n + oj]);
    if (i == j) v = __dadd_rn(v, dmp);
    a[e] = T(v);
  }
}

// Same gather, one CTA per output row: H row order[n-1-i] is staged in shared
// memory with coalesced loads, then a[i, j] = row[order[n-1-j]] (j <= i) is
// written coalesced -- the column permutation happens on chip.
template <typename T>
__global__ void __launch_bounds__(256) build_input_rows_kernel(const float* __restrict__ h,
                                                               long long n,
                                                               const int32_t* __restrict__ order,
                                                               const double* damp, T* a) {
  extern __shared__ float hrow[];
  const long long i = blockIdx.x;
  const long long oi = order[n - 1 - i];
  const float* src = h + oi * n;
  if ((n & 3) == 0) {
    for (long long t = threadIdx.x; t < n / 4; t += blockDim.x)
      reinterpret_cast<float4*>(hrow)[t] = __ldg(reinterpret_cast<const float4*>(src) + t);
  } else {
    for (long long t = threadIdx.x; t < n; t += blockDim.x) hrow[t] = __ldg(src + t);
  }
  __syncthreads();
  const double dmp = *damp;
  T* dst = a + i * n;
  for (long long j = threadIdx.x; j <= i; j += blockDim.x) {
    double v = double(hrow[order[n - 1 - j]]);
    if (j == i) v = __dadd_rn(v, dmp);
    dst[j] = T(v);
  }
}

// damp = percdamp * mean(diag(fp64 H))  (layerwise.cpp:32-33)
__global__ void damp_kernel(const float* __restrict__ h, long long n, double percdamp,
                            double* damp, float* __restrict__ diag) {
  __shared__ double part[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = h[i * n + i];
    if (diag) diag[i] = v;
    s += double(v);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
    *damp = percdamp * (t / double(n));
  }
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const int* p) {
  while (!ld_acquire(p)) __nanosleep(20);
}

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
  return __ldcg(p);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_1_n() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Raw copy of a 64 x 64 tile (rows x cols valid, row stride n) into dst
// (row-major, ld 64); 16-byte cp.async when aligned, zero outside.
template <typename T>
__device__ __forceinline__ void stage_tile(T* dst, const T* src, long long n, int rows, int cols,
                                           bool vec_ok, int ldd = TB + 4) {
  constexpr int V = 16 / sizeof(T);
  for (int e = threadIdx.x; e < TB * TB / V; e += CT) {
    const int rr = e / (TB / V), cc = (e % (TB / V)) * V;
    T* d = dst + rr * ldd + cc;
    if (vec_ok && rr < rows && cc + V <= cols) {
      cp_async16(d, src + (long long)rr * n + cc);
    } else {
#pragma unroll
      for (int q = 0; q < V; ++q) d[q] = (rr < rows && cc + q < cols) ? ldcg(src + (long long)rr * n + cc + q) : T(0);
    }
  }
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t u = __float_as_uint(x);
  u = (u + 0xFFFu + ((u >> 13) & 1u)) & ~0x1FFFu;  // RNE to 10 mantissa bits
  return __uint_as_float(u);
}

// Position of block-local row kk (0..127) in a lane-ordered row of G^T for
// the sweep's in-block kernel: lane group rg = kk % 8 owns slots s = kk / 8,
// stored as 8-byte pairs p = s / 2 at rg*16 + 2*((p + 2*(rg/2)) % 8) -- the
// rotation makes the eight lane groups' reads of one slot pair hit distinct
// banks (sweep.cu).
__host__ __device__ inline int gp_pos(int kk) {
  const int rg = kk & 7, s = kk >> 3;
  return rg * 16 + 2 * (((s >> 1) + 2 * (rg >> 1)) & 7) + (s & 1);
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


constexpr int LD = TB + 4;  // row stride of the owner's row-major tiles

// Small fields first: the fp32 workers' tcgen05 operand stages (kUmmaOff on)
// alias the big buffers, which a worker only uses after its k-loop.
template <typename T>
struct CholSmem {
  int item;
  int ready;
  alignas(16) int stg[4];  // owner: which tiles the factor's idle warps staged; [3]: product done
  alignas(16) T rdiag[TB];
  alignas(16) T wcol4[4][72];  // factor_tile64: the producer's pivot-column ring (shared-pivot elimination)
  alignas(16) T ps[TB * LD];   // row-major tiles (ld LD): tile-product operands / staging
  alignas(16) T qs[TB * LD];
  alignas(16) T lt[TB][LD];    // workers: L_cc transposed / G staging; owner: X = L_cc^-T
  alignas(16) T sf[TB][TB + 1];  // diagonal tile being factored
  alignas(16) T sb[2][TB * LD];  // owner: staged partial tiles (row-major, ld LD, cp.async)
};

// Publish the finalised tile (values in t, rows b = 64r + 4ty + u, cols
// a = 64c + 4tx + v) into G: G[n-1-a][n-1-b] = L[b][a] / L[a][a] for b > a.
// `diag` holds L[a][a] for the tile's column range.  Uses sm.lt as staging.
template <typename T>
__device__ void emit_g(const T (&t)[4][4], CholSmem<T>& sm, const T* diag, int r, int c, long long n,
                       T* ghi, float* glo, float* gpl) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) sm.lt[4 * ty + u][4 * tx + v] = t[u][v];
  __syncthreads();
  const long long b0 = (long long)r * TB, a0 = (long long)c * TB;
  for (int e = tid; e < TB * TB; e += CT) {
    const int al = e >> 6, q = e & 63;  // G row k = n-1-(a0+al); col i = n-1-(b0+63-q)
    const int bl = 63 - q;
    const long long a = a0 + al, b = b0 + bl;
    if (a >= n || b >= n) continue;
    T g = T(0);
    if (b > a) g = sm.lt[bl][al] / diag[al];
    const long long off = (n - 1 - a) * n + (n - 1 - b);
    if (sizeof(T) == 4 && glo) {
      const float hi = tf32_hi(float(g));
      ghi[off] = T(hi);
      glo[off] = float(g) - hi;
      gpl[off] = float(g);
    } else {
      ghi[off] = g;
    }
  }
}

// rsqrt to the hardware approximation (pivots are positive normal numbers,
// or the factorisation has failed and is reported)
template <typename T>
__device__ __forceinline__ T rsqrt_fast(T x) {
  if constexpr (sizeof(T) == 4) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  } else {
    return rsqrt(x);
  }
}

// Shared-pivot elimination for factor_tile64: the eliminating warp (producer)
// publishes each pivot column in a 4-deep shared ring (wcol4[j & 3], shifted
// as in warp_chol32) and 1/L[j][j] in rdiag[j]; carrying warps (consumers)
// apply the same pivots to their rows without redoing the elimination.  Per
// ring slot s two named barriers (nthreads = the participating warps):
// full(s) = 2 + s -- the producer arrives once pivot j's column and rdiag[j]
// are written, consumers sync; empty(s) = 6 + s -- consumers arrive once done
// with the slot, the producer syncs before refilling it.  The producer never
// waits for consumers unless it is 4 pivots ahead, so its pivot chain alone
// sets the pace (a full rendezvous per pivot put the consumers' work on it).
__device__ __forceinline__ void bar_sync_id(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_id(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
template <typename T>
__device__ __forceinline__ bool warp_chol32_prod(T (&a)[32], T* out_row, T* rdiag,
                                                 T (*wcol4)[72], int nthreads) {
  const int lane = threadIdx.x & 31;
  const bool cons = nthreads > 32;
  bool ok = true;
  wcol4[0][lane + 3] = a[0];
  // the pivot travels by shuffle (the next pivot is lane j+1's updated entry),
  // so the chain is shuffle -> rsqrt -> 3 FMA-pipe ops; only the column, which
  // the FMAs need later, goes through the shared ring
  T p = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    const int sh = (3 - j) & 3;
    __syncwarp();
    T v[32];
    const T* nxt = wcol4[j & 3] + j + sh + 1;
#pragma unroll
    for (int k4 = 0; k4 < 32; k4 += 4) {
      T v4[4];
      ld4(nxt + k4, v4);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[k4 + e] = v4[e];
    }
    ok &= (p > T(0));
    const T rs = rsqrt_fast(p);
    const T l = a[0] * rs;
    const T lrs = l * rs;
    const T a0 = fma(-lrs, v[0], a[1]);
    // slot (j+1) & 3 last held pivot j-3's column: the consumers must be done with it
    if (cons && j >= 3 && j + 1 < 32) bar_sync_id(6 + ((j + 1) & 3), nthreads);
    if (j + 1 < 32) wcol4[(j + 1) & 3][lane + ((2 - j) & 3)] = a0;
    if (lane == j) rdiag[j] = rs;  // 1 / L[j][j]
    if (cons) bar_arrive_id(2 + (j & 3), nthreads);
    if (j + 1 < 32) p = __shfl_sync(0xffffffffu, a0, j + 1);
#pragma unroll
    for (int k = 1; k + 1 < 32; ++k) a[k] = fma(-lrs, v[k], a[k + 1]);
    a[0] = a0;
    a[31] = T(0);
    out_row[j] = lane >= j ? l : T(0);
  }
  if (cons) {  // balance the empty phases of pivots 28..31
#pragma unroll
    for (int s = 0; s < 4; ++s) bar_sync_id(6 + s, nthreads);
  }
  return ok;
}
template <typename T>
__device__ __forceinline__ void warp_carry32_cons(T (&b)[32], T* out_b, const T* rdiag,
                                                  const T (*wcol4)[72], int nthreads) {
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    const int sh = (3 - j) & 3;
    bar_sync_id(2 + (j & 3), nthreads);
    T v[32];
    const T* nxt = wcol4[j & 3] + j + sh + 1;
#pragma unroll
    for (int k4 = 0; k4 < 32; k4 += 4) {
      T v4[4];
      ld4(nxt + k4, v4);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[k4 + e] = v4[e];
    }
    const T rs = rdiag[j];
    bar_arrive_id(6 + (j & 3), nthreads);  // (slot and rdiag[j] read into registers)
    const T lb = b[0] * rs;  // (b L^-T)[j]
    const T lbrs = lb * rs;
#pragma unroll
    for (int k = 0; k + 1 < 32; ++k) b[k] = fma(-lbrs, v[k], b[k + 1]);
    b[31] = T(0);
    out_b[j] = lb;
  }
}

// Factor the 64 x 64 tile in sm.sf (lower, padded with identity) in place.
// Three warps share the 32-column eliminations (warp_chol32_prod / _cons), on distinct
// SM sub-partitions, so the rows they carry cost no chain length:
//   h = 0: warp 0 -> L11 = chol(A11); warp 2 carries A21 -> L21 = A21 L11^-T;
//          [INV] warp 1 carries identity rows 0-31 -> X rows of L^-T;
//          CTA: A22 -= L21 L21^T  [INV: X[0:32, 32:] = -X[0:32, :32] L21^T];
//   h = 1: warp 0 -> L22 = chol(A22);
//          [INV] warps 1, 2 carry X rows 0-31 / identity rows 32-63.
// With INV, sm.lt receives X = L^-T (upper triangular, ld TB + 4).  Upper
// entries of sf are zeroed; sm.rdiag gets 1 / L[j][j].  All threads call.
struct NoSide {
  __device__ void operator()(int) const {}
};
// Side: work for the warps the eliminations leave idle (warps 3-7 call it at
// the start of each half, side(0) and side(1)).
template <typename T, bool INV = false, typename Side = NoSide>
__device__ bool factor_tile64(CholSmem<T>& sm, long long* prof = nullptr, const Side& side = Side()) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  bool ok = true;
  auto pstamp = [&](int i) {
    if (prof && tid == 0) prof[i] = clock64();
  };
  pstamp(0);
  for (int e = tid; e < 4 * 72; e += CT) (&sm.wcol4[0][0])[e] = T(0);
  __syncthreads();
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int o = 32 * h;  // diagonal block [o, o+32)
    const bool active = warp == 0 || (warp == 2 && h == 0) || (INV && warp <= 2);
    if (warp >= 3) side(h);
    // (votes make the warp-uniform branches visible to ptxas: no divergent-shuffle
    // fallback paths, which would pin the loads behind branch checks)
    if (__any_sync(0xffffffffu, active)) {
      T bv[32];
      T* brow = nullptr;  // carried row (written back in place)
      if (warp == 2 && h == 0) {
        brow = &sm.sf[32 + lane][0];
#pragma unroll
        for (int k = 0; k < 32; ++k) bv[k] = brow[k];
      } else if (warp > 0) {  // INV
        const bool ident = (warp == 1) == (h == 0);
        brow = &sm.lt[32 * (warp - 1) + lane][o];
#pragma unroll
        for (int k = 0; k < 32; ++k) bv[k] = ident ? T(k == lane ? 1 : 0) : brow[k];
        if (h == 1 && warp == 2) {
#pragma unroll
          for (int k = 0; k < 32; ++k) sm.lt[32 + lane][k] = T(0);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) bv[k] = T(0);
      }
      const bool w0 = __any_sync(0xffffffffu, warp == 0);
      // producer + consumers: h = 0 warps 0, 2 (+1 with INV); h = 1 warp 0 (+1, 2 with INV)
      const int nthreads = 32 * (h == 0 ? 2 + (INV ? 1 : 0) : 1 + (INV ? 2 : 0));
      if (w0) {
        T av[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) av[k] = sm.sf[o + lane][o + k];
        ok &= warp_chol32_prod(av, &sm.sf[o + lane][o], &sm.rdiag[o], sm.wcol4, nthreads);
      } else {
        warp_carry32_cons(bv, brow, &sm.rdiag[o], sm.wcol4, nthreads);
      }
      if (w0) {
        if (h == 0) {
#pragma unroll
          for (int k = 0; k < 32; ++k) sm.sf[lane][32 + k] = T(0);
        }
      }
      pstamp(1 + 3 * h);
    }
    __syncthreads();
    if (h == 0) {
      if (!INV || tid < 128) {  // A22 -= L21 L21^T: thread -> row i, (INV ? 8 : 4) columns
        constexpr int NJ = INV ? 8 : 4;
        const int i = tid / (32 / NJ), j0 = (tid % (32 / NJ)) * NJ;
        T s4[NJ] = {};
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const T li = sm.sf[32 + i][k];
#pragma unroll
          for (int jj = 0; jj < NJ; ++jj) s4[jj] = fma(li, sm.sf[32 + j0 + jj][k], s4[jj]);
        }
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
          if (j0 + jj <= i) sm.sf[32 + i][32 + j0 + jj] -= s4[jj];
      } else {  // X[0:32, 32:] = -X[0:32, :32] L21^T: thread -> row i, 8 columns
        const int q = tid - 128, i = q >> 2, j0 = (q & 3) * 8;
        T s8[8] = {};
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const T xi = sm.lt[i][k];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) s8[jj] = fma(xi, sm.sf[32 + j0 + jj][k], s8[jj]);
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) sm.lt[i][32 + j0 + jj] = -s8[jj];
      }
      __syncthreads();
      pstamp(3);
    }
  }
  return ok;
}

// ---- the owner's 64 x 64 x 64 tile products ---------------------------------
// D = src + sgn * A B'  with B' = B^T (B row-major [j][k]) or, BT, B' = B
// ([k][j]); A, B, src: row-major ld LD; D: ld ldd (may alias src).  With
// pad >= 0, D[i][i] = 1 for i >= pad (identity padding of a diagonal tile).
// fp32: 3xTF32 on the warp-level tensor cores (m16n8k8), warp w computes rows
// 16 (w & 3).., columns 32 (w >> 2)..: conflict-free fragment loads at ld 68.
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
// ---- worker tile products on the 5th-gen tensor cores (fp32 path) ----------
// acc (TMEM, 128 lanes x 64 fp32 columns; lanes 0-63 used) += L[r,k] L[c,k]^T
// as 3xTF32 (lo*hi + hi*lo + hi*hi, tcgen05.mma kind::tf32, M = 128, N = 64,
// K = 8 per instruction).  Every published L tile is also stored pre-split
// (lhi = tf32 round-to-nearest of L, llo = L - lhi), and a k-step is four
// 64 x 64 tiles (A hi / lo, B hi / lo) brought in by TMA (SWIZZLE_128B, two
// 32-column boxes each) into a 3-stage ring: one thread of the CTA produces
// (tile flags, then TMA), one issues the MMAs, nobody else is involved until
// the accumulator is read back.  M = 128 costs the same as M = 64 (the
// instruction floor is M = 128); its upper 64 rows read the next 8 KB of the
// stage and land in TMEM lanes never read.
constexpr int kUmmaStage = 65536;  // A hi | A lo | B hi | B lo, 16 KB each
constexpr int kUmmaStages = 3;
constexpr int kUmmaOff = 4096;     // past CholSmem's small fields
constexpr int kUmmaEnd = kUmmaOff + kUmmaStages * kUmmaStage + 1024;
constexpr uint32_t kUmmaIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(64 >> 3) << 17) |
                                (uint32_t(128 >> 4) << 24);
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t umma_kdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;                       // LBO (unused for swizzled K-major)
  d |= uint64_t((1024u >> 4) & 0x3FFFu) << 32;  // SBO: 8-row atoms at 1 KB
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;                       // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(kUmmaIdesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
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
__device__ __forceinline__ void tma_tile(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x,
                                         int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// store the tile's tf32 hi / lo split beside L (rows x cols valid)
__device__ __forceinline__ void store_split(const float (&t)[4][4], float* lhi, float* llo,
                                            long long off, long long n, int rows, int cols) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int rr = 4 * ty + u;
    if (rr >= rows) continue;
    const long long o = off + (long long)rr * n + 4 * tx;
    if (4 * tx + 4 <= cols) {
      const float4 h = make_float4(tf32_hi(t[u][0]), tf32_hi(t[u][1]), tf32_hi(t[u][2]),
                                   tf32_hi(t[u][3]));
      *reinterpret_cast<float4*>(lhi + o) = h;
      *reinterpret_cast<float4*>(llo + o) =
          make_float4(t[u][0] - h.x, t[u][1] - h.y, t[u][2] - h.z, t[u][3] - h.w);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (4 * tx + v < cols) {
          const float h = tf32_hi(t[u][v]);
          lhi[o + v] = h;
          llo[o + v] = t[u][v] - h;
        }
    }
  }
}
struct UmmaMaps {
  CUtensorMap hi, lo;  // lhi / llo: n x n fp32, 32 x 64 boxes, SWIZZLE_128B
};

template <typename T, bool BT>
__device__ __forceinline__ void owner_prod(const T* A, const T* B, const T* src, T* D, int ldd,
                                           T sgn, int pad) {
  const int tid = threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int r0 = 16 * (warp & 3), n0 = 32 * (warp >> 2);
    float c1[4][4] = {}, c2[4][4] = {};
#pragma unroll 2
    for (int k8 = 0; k8 < TB; k8 += 8) {
      uint32_t ah[4], al[4];
      split_tf32(A[(r0 + g) * LD + k8 + t], ah[0], al[0]);
      split_tf32(A[(r0 + g + 8) * LD + k8 + t], ah[1], al[1]);
      split_tf32(A[(r0 + g) * LD + k8 + t + 4], ah[2], al[2]);
      split_tf32(A[(r0 + g + 8) * LD + k8 + t + 4], ah[3], al[3]);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int nn = n0 + 8 * nt + g;
        const float b0 = BT ? B[(k8 + t) * LD + nn] : B[nn * LD + k8 + t];
        const float b1 = BT ? B[(k8 + t + 4) * LD + nn] : B[nn * LD + k8 + t + 4];
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(b0, bh0, bl0);
        split_tf32(b1, bh1, bl1);
        mma_tf32(c1[nt], ah, bh0, bh1);
        mma_tf32(c2[nt], ah, bl0, bl1);
        mma_tf32(c2[nt], al, bh0, bh1);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = r0 + g + 8 * (q >> 1), j = n0 + 8 * nt + 2 * t + (q & 1);
        float v = (src ? src[i * LD + j] : 0.f) + sgn * (c1[nt][q] + c2[nt][q]);
        if (pad >= 0 && i == j && i >= pad) v = 1.f;
        D[i * ldd + j] = v;
      }
  } else {
    const int ty = tid >> 4, tx = tid & 15;
    T acc[4][4] = {};
    for (int k = 0; k < TB; ++k) {
      T av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = A[(4 * ty + u) * LD + k];
        bv[u] = BT ? B[k * LD + 4 * tx + u] : B[(4 * tx + u) * LD + k];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = 4 * ty + u, j = 4 * tx + v;
        T val = (src ? src[i * LD + j] : T(0)) + sgn * acc[u][v];
        if (pad >= 0 && i == j && i >= pad) val = T(1);
        D[i * ldd + j] = val;
      }
  }
}

// D = src - A B^T on warps 4-7 only (fp32): the owner's sub-tile update runs
// beside the factorisation on warps the elimination leaves idle.
__device__ __forceinline__ void owner_prod_w47(const float* A, const float* B, float* D) {
  const int warp = (threadIdx.x >> 5) - 4, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int r0 = 16 * warp;
#pragma unroll 1
  for (int n0 = 0; n0 < TB; n0 += 32) {
    float c1[4][4] = {}, c2[4][4] = {};
#pragma unroll 2
    for (int k8 = 0; k8 < TB; k8 += 8) {
      uint32_t ah[4], al[4];
      split_tf32(A[(r0 + g) * LD + k8 + t], ah[0], al[0]);
      split_tf32(A[(r0 + g + 8) * LD + k8 + t], ah[1], al[1]);
      split_tf32(A[(r0 + g) * LD + k8 + t + 4], ah[2], al[2]);
      split_tf32(A[(r0 + g + 8) * LD + k8 + t + 4], ah[3], al[3]);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int nn = n0 + 8 * nt + g;
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(B[nn * LD + k8 + t], bh0, bl0);
        split_tf32(B[nn * LD + k8 + t + 4], bh1, bl1);
        mma_tf32(c1[nt], ah, bh0, bh1);
        mma_tf32(c2[nt], ah, bl0, bl1);
        mma_tf32(c2[nt], al, bh0, bh1);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = r0 + g + 8 * (q >> 1), j = n0 + 8 * nt + 2 * t + (q & 1);
        D[i * LD + j] -= c1[nt][q] + c2[nt][q];
      }
  }
}

// Running tile product acc += A B^T over k steps (A, B row-major ld LD), in
// the tensor-core fragment layout for fp32 (3xTF32), 4x4 register blocks for
// fp64; acc_store writes it out row-major.
template <typename T>
struct TileAcc {
  T c[4][4];
};
template <>
struct TileAcc<float> {
  float c1[4][4], c2[4][4];
};
template <typename T>
__device__ __forceinline__ void acc_zero(TileAcc<T>& s) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s.c1[i][j] = s.c2[i][j] = 0.f;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s.c[i][j] = T(0);
  }
}
template <typename T>
__device__ __forceinline__ void acc_mma(TileAcc<T>& s, const T* A, const T* B) {
  const int tid = threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int r0 = 16 * (warp & 3), n0 = 32 * (warp >> 2);
#pragma unroll 2
    for (int k8 = 0; k8 < TB; k8 += 8) {
      uint32_t ah[4], al[4];
      split_tf32(A[(r0 + g) * LD + k8 + t], ah[0], al[0]);
      split_tf32(A[(r0 + g + 8) * LD + k8 + t], ah[1], al[1]);
      split_tf32(A[(r0 + g) * LD + k8 + t + 4], ah[2], al[2]);
      split_tf32(A[(r0 + g + 8) * LD + k8 + t + 4], ah[3], al[3]);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int nn = n0 + 8 * nt + g;
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(B[nn * LD + k8 + t], bh0, bl0);
        split_tf32(B[nn * LD + k8 + t + 4], bh1, bl1);
        mma_tf32(s.c1[nt], ah, bh0, bh1);
        mma_tf32(s.c2[nt], ah, bl0, bl1);
        mma_tf32(s.c2[nt], al, bh0, bh1);
      }
    }
  } else {
    const int ty = tid >> 4, tx = tid & 15;
    for (int k = 0; k < TB; ++k) {
      T av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = A[(4 * ty + u) * LD + k];
        bv[u] = B[(4 * tx + u) * LD + k];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) s.c[u][v] = fma(av[u], bv[v], s.c[u][v]);
    }
  }
}
template <typename T>
__device__ __forceinline__ void acc_store(const TileAcc<T>& s, T* D, int ldd) {
  const int tid = threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int r0 = 16 * (warp & 3), n0 = 32 * (warp >> 2);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        D[(r0 + g + 8 * (q >> 1)) * ldd + n0 + 8 * nt + 2 * t + (q & 1)] = s.c1[nt][q] + s.c2[nt][q];
  } else {
    const int ty = tid >> 4, tx = tid & 15;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) D[(4 * ty + u) * ldd + 4 * tx + v] = s.c[u][v];
  }
}

// ---- pieces shared by the owner and the worker CTAs -------------------------
// t (thread block rows 4ty+u, cols 4tx+v) <- tile at ab; identity padding of a
// diagonal tile's rows past n
template <typename T>
__device__ __forceinline__ void load_t(T (&t)[4][4], const T* ab, long long n, int rows, int cols,
                                       bool diag, bool vec_ok) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int rr = 4 * ty + u;
    const T* p = ab + (long long)rr * n + 4 * tx;
    if (vec_ok && rr < rows && 4 * tx + 4 <= cols) {
      if constexpr (sizeof(T) == 4) {
        const float4 f = __ldcg(reinterpret_cast<const float4*>(p));
        t[u][0] = f.x, t[u][1] = f.y, t[u][2] = f.z, t[u][3] = f.w;
      } else {
        const double2 f0 = __ldcg(reinterpret_cast<const double2*>(p));
        const double2 f1 = __ldcg(reinterpret_cast<const double2*>(p + 2));
        t[u][0] = f0.x, t[u][1] = f0.y, t[u][2] = f1.x, t[u][3] = f1.y;
      }
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int cc = 4 * tx + v;
        t[u][v] = (rr < rows && cc < cols) ? ldcg(p + v) : T(0);
      }
    }
    if (diag) {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (rr == 4 * tx + v && rr >= rows) t[u][v] = T(1);
    }
  }
}

template <typename T>
__device__ __forceinline__ void store_t(const T (&t)[4][4], T* ab, long long n, int rows, int cols,
                                        bool lower) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int rr = 4 * ty + u;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int cl = 4 * tx + v;
      if (rr < rows && cl < cols && (!lower || cl <= rr)) ab[(long long)rr * n + cl] = t[u][v];
    }
  }
}



// Publish a finalised tile L[r,c] (values t) into G: the sweep's lane-ordered
// diagonal blocks of G^T (gtt) and the GEMM / lookahead operands (emit_g).
// sm.rdiag holds L[a][a] of column tile c.
template <typename T>
__device__ __forceinline__ void emit_tile(const T (&t)[4][4], CholSmem<T>& sm, int r, int c,
                                          long long n, T* ghi, float* glo, float* gpl,
                                          float* gtt) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  if (gtt) {
    // diagonal 128 x 128 blocks of G^T in the sweep's lane order (sweep.cu
    // gp_pos): row i = n-1-b, column k = n-1-a, only when i, k share a block
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long b = (long long)r * TB + 4 * ty + u;
      if (b >= n) continue;
      const long long i = n - 1 - b;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const long long av = (long long)c * TB + 4 * tx + v;
        if (av >= n || b <= av) continue;
        const long long k = n - 1 - av;
        if ((i >> 7) != (k >> 7)) continue;
        gtt[i * 128 + gp_pos(int(k & 127))] = float(t[u][v] / sm.rdiag[4 * tx + v]);
      }
    }
  }
  if (ghi) emit_g(t, sm, sm.rdiag, r, c, n, ghi, glo, gpl);
}

// CTA 0 is the owner of the critical path: per column c it factors tile
// (c, c) and solves tile (c+1, c), keeping L[c+1, c] in shared memory for the
// next column's k = c terms, so the chain diag -> sub -> diag has no
// inter-CTA hand-off.  The other CTAs take work items of column c, in order:
//   0, 1 -> partial S[c+q,c] = A - sum_{c0<=k<c-1} L[c+q,k] L[c,k]^T, stored in
//           place (the owner applies k = c-1);
//   2..  -> tiles (c+2.., c): full accumulation, then X L[c,c]^T = S;
//   last -> emission of the owner's two tiles into G.
enum ItemKind { kFull = 0, kPartial = 1, kEmit = 2, kOwner = 3 };

template <typename T>
__global__ void __launch_bounds__(CT, 1)
    chol_tile_kernel(T* __restrict__ a, long long n, int nt, int c0, int c1, int* flags,
                     int* pflags, int* counter, unsigned* status, T* ghi, float* glo, float* gpl,
                     float* gtt, unsigned long long* trace, const __grid_constant__ UmmaMaps maps,
                     float* lhi, float* llo, int* sflags) {
  extern __shared__ __align__(16) unsigned char smraw[];
  CholSmem<T>& sm = *reinterpret_cast<CholSmem<T>*>(smraw);
  // optional timeline (debug): per entry {r, c + 1000 kind, start, k-loop done,
  // factor/solve done, published}
  auto stamp = [&](long long e, int slot) {
    if (trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[e * 6 + slot] = t;
    }
  };
  auto tag = [&](long long e, int r, int c, int kind) {
    if (trace && threadIdx.x == 0) {
      trace[e * 6 + 0] = (unsigned long long)r;
      trace[e * 6 + 1] = (unsigned long long)(c + 1000 * kind);
    }
  };
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const bool vec_ok = (sizeof(T) == 4 ? (n & 3) == 0 : (n & 1) == 0);
  long long total = 0;
  for (int c = c0; c < c1; ++c) total += nt - c + 1;
  const long long tile = (long long)TB * n;  // elements per tile row

  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  int* owner_sm = counter + nt;  // panel ci's owner slot (counters: nt item counters, then nt owner slots)
  if (blockIdx.x == 0) {
    if (tid == 0) st_release(owner_sm, int(smid) + 1);
    // ================= owner: the critical path diag(c) -> sub(c+1, c) -> diag(c+1)
    // Row-major tiles (ld LD) in shared memory:
    //   qs: L[c, c-1] (kept from the previous column)    ps: L[c+1, c-1] (staged)
    //   sb[1]: S'[c, c] (partial, staged during column c-1)
    //   sb[0]: S'[c+1, c] -> S[c+1, c]                    lt: X = L[c,c]^-T
    // Tiles are published by one thread of warp 7 (its fence only stalls itself).
    bool staged = false;  // sb[1] holds S'[c, c]
    for (int c = c0; c < c1; ++c) {
      const long long e0 = total + 2LL * (c - c0);
      const int rows = int(std::min<long long>(TB, n - (long long)c * TB));
      const bool sub = c + 1 < nt;
      const int rows1 = sub ? int(std::min<long long>(TB, n - (long long)(c + 1) * TB)) : 0;
      const bool prev = c > c0;
      tag(e0, c, c, kOwner);
      stamp(e0, 2);
      if (!staged) {
        if (tid == 0) wait_flag(pflags + 2 * c);
        __syncthreads();
        stage_tile(sm.sb[1], a + c * tile + (long long)c * TB, n, rows, rows, vec_ok);
      }
      cp_async_wait_all();
      __syncthreads();
      // S[c,c] = S' - L[c,c-1] L[c,c-1]^T  -> sf (identity padding past n)
      if (prev) {
        owner_prod<T, false>(sm.qs, sm.qs, sm.sb[1], &sm.sf[0][0], TB + 1, T(-1), rows);
      } else {
        for (int e = tid; e < TB * TB; e += CT) {
          const int i = e >> 6, j = e & 63;
          sm.sf[i][j] = (i == j && i >= rows) ? T(1) : sm.sb[1][i * LD + j];
        }
      }
      __syncthreads();
      stamp(e0, 3);
      // the factor's idle warps (3-7) stage what is already published: S'[c+1,c],
      // L[c+1,c-1] and the next column's S'[c+1,c+1] (sm.stg bits tell which)
      auto side = [&](int half) {
        const int st = tid - 96;  // 0..159
        if (half == 1 && st < 32 && sub && !sm.stg[2]) {
          // the next column's S'[c+1,c+1] may land during the first half: warp 3
          // checks again and stages it under the second half
          int ready = 0;
          if (st == 0) ready = ld_acquire(pflags + 2 * (c + 1));
          ready = __shfl_sync(0xffffffffu, ready, 0);
          if (ready) {
            constexpr int V = 16 / sizeof(T);
            const T* src = a + (c + 1) * tile + (long long)(c + 1) * TB;
            for (int e = st; e < TB * TB / V; e += 32) {
              const int rr = e / (TB / V), cc = (e % (TB / V)) * V;
              T* d = sm.sb[1] + rr * LD + cc;
              if (vec_ok && rr < rows1 && cc + V <= rows1) {
                cp_async16(d, src + (long long)rr * n + cc);
              } else {
#pragma unroll
                for (int u = 0; u < V; ++u)
                  d[u] = (rr < rows1 && cc + u < rows1) ? ldcg(src + (long long)rr * n + cc + u) : T(0);
              }
            }
            __syncwarp();
            if (st == 0) sm.stg[2] = 1;
          }
        }
        if (half == 1) {
          // S[c+1,c] -= L[c+1,c-1] L[c,c-1]^T beside the h = 1 elimination when both
          // tiles were staged (fp32; otherwise it runs after the factor)
          if (sizeof(T) == 4 && prev && sm.stg[0] && sm.stg[1]) {
            cp_async_wait_all();
            asm volatile("bar.sync 1, 160;" ::: "memory");
            if (tid >= 128)
              owner_prod_w47(reinterpret_cast<const float*>(sm.ps),
                             reinterpret_cast<const float*>(sm.qs),
                             reinterpret_cast<float*>(sm.sb[0]));
            if (st == 0) sm.stg[3] = 1;
          }
          return;
        }
        if (st == 0) sm.stg[3] = 0;
        if (st == 0) sm.stg[0] = sub && ld_acquire(pflags + 2 * c + 1);
        if (st == 32) sm.stg[1] = sub && prev && ld_acquire(flags + (c + 1) * nt + (c - 1));
        if (st == 64) sm.stg[2] = sub && ld_acquire(pflags + 2 * (c + 1));
        asm volatile("bar.sync 1, 160;" ::: "memory");
        constexpr int V = 16 / sizeof(T);
        const T* src[3] = {a + (c + 1) * tile + (long long)c * TB,
                           a + (c + 1) * tile + (long long)(c - 1) * TB,
                           a + (c + 1) * tile + (long long)(c + 1) * TB};
        T* dst[3] = {sm.sb[0], sm.ps, sm.sb[1]};
        const int rws[3] = {rows1, rows1, rows1};
        const int cls[3] = {TB, TB, rows1};
        for (int q = 0; q < 3; ++q) {
          if (!sm.stg[q]) continue;
          for (int e = st; e < TB * TB / V; e += 160) {
            const int rr = e / (TB / V), cc = (e % (TB / V)) * V;
            T* d = dst[q] + rr * LD + cc;
            if (vec_ok && rr < rws[q] && cc + V <= cls[q]) {
              cp_async16(d, src[q] + (long long)rr * n + cc);
            } else {
#pragma unroll
              for (int u = 0; u < V; ++u)
                d[u] = (rr < rws[q] && cc + u < cls[q]) ? ldcg(src[q] + (long long)rr * n + cc + u) : T(0);
            }
          }
        }
      };
      const bool ok = factor_tile64<T, true>(sm, nullptr, side);  // sm.lt = L[c,c]^-T
      if (!ok && tid == 0 && rows > 0) atomicOr(status, kFlagNotPD);
      const bool s_staged = sm.stg[0], l_staged = sm.stg[1];
      stamp(e0, 4);
      {
        T t[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int i = 4 * ty + u, j = 4 * tx + v;
            t[u][v] = j <= i ? sm.sf[i][j] : sm.lt[i][j];
          }
        // lower: L[c,c]; strict upper: X = L[c,c]^-T (the workers' solve operand;
        // the upper triangle of a diagonal tile is otherwise unused)
        store_t(t, a + c * tile + (long long)c * TB, n, rows, rows, false);
      }
      // publish: one thread of warp 7 fences (release is cumulative over the
      // CTA's stores ordered by the barrier); the chain warps go on
      __syncthreads();
      if (tid == CT - 32) {
        __threadfence();
        st_release(flags + c * nt + c, 1);
      }
      stamp(e0, 5);
      if (!sub) break;

      // ---- sub tile (c+1, c): S = S' - L[c+1,c-1] L[c,c-1]^T;  X = S L[c,c]^-T
      const long long e1 = e0 + 1;
      tag(e1, c + 1, c, kOwner);
      stamp(e1, 2);
      if (!s_staged) {
        if (tid == 0) wait_flag(pflags + 2 * c + 1);
        __syncthreads();
        stage_tile(sm.sb[0], a + (c + 1) * tile + (long long)c * TB, n, rows1, TB, vec_ok);
      }
      if (prev && !l_staged) {
        if (tid == 0) wait_flag(flags + (c + 1) * nt + (c - 1));
        __syncthreads();
        stage_tile(sm.ps, a + (c + 1) * tile + (long long)(c - 1) * TB, n, rows1, TB, vec_ok);
      }
      cp_async_wait_all();
      __syncthreads();
      if (prev && !sm.stg[3]) {
        owner_prod<T, false>(sm.ps, sm.qs, sm.sb[0], sm.sb[0], LD, T(-1), -1);
        __syncthreads();
      }
      stamp(e1, 3);
      staged = sm.stg[2];  // the next column's S'[c+1,c+1], staged under the factor
      // not staged yet: look again (relaxed load issued before the solve, so its
      // latency hides under the product) and start the copy for the next column
      int pv = 0;
      if (!staged && tid == 0) pv = ld_relaxed(pflags + 2 * (c + 1));
      owner_prod<T, true>(sm.sb[0], &sm.lt[0][0], nullptr, sm.qs, LD, T(1), -1);  // -> L[c+1,c]
      if (!staged && tid == 0) {
        if (pv) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        sm.stg[2] = pv;
      }
      __syncthreads();
      if (!staged && sm.stg[2]) {  // (completes under the publish; waited at the next column)
        stage_tile(sm.sb[1], a + (c + 1) * tile + (long long)(c + 1) * TB, n, rows1, rows1, vec_ok);
        staged = true;
      }
      stamp(e1, 4);
      {
        T t[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) t[u][v] = sm.qs[(4 * ty + u) * LD + 4 * tx + v];
        store_t(t, a + (c + 1) * tile + (long long)c * TB, n, rows1, TB, false);
      }
      __syncthreads();
      if (tid == CT - 32) {
        __threadfence();
        st_release(flags + (c + 1) * nt + c, 1);
      }
      stamp(e1, 5);
    }
    return;
  }

  // ================= workers (none on the owner's SM: it keeps its issue slots)
  if (tid == 0) {
    int o;
    while ((o = ld_acquire(owner_sm)) == 0) __nanosleep(100);
    sm.ready = o == int(smid) + 1;
  }
  __syncthreads();
  if (sm.ready) return;
  // fp32: tensor-memory accumulator (64 columns) and the MMA completion barrier
  __shared__ __align__(8) unsigned long long full_bar[kUmmaStages], empty_bar[kUmmaStages];
  __shared__ __align__(8) unsigned long long done_bar;
  __shared__ uint32_t tmem_holder;
  uint8_t* ub = nullptr;
  uint32_t tmem = 0;
  // ring position (producer / MMA issuer) and accumulator phase, kept across items
  uint32_t p_stage = 0, p_phase = 0, m_stage = 0, m_phase = 0, d_phase = 0;
  const bool umma = sizeof(T) == 4 && lhi != nullptr;
  if (umma) {
    ub = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + kUmmaOff + 1023) &
                                    ~uintptr_t(1023));
    if (tid == 0) {
      for (int q = 0; q < kUmmaStages; ++q) {
        mbar_init1(smem_addr(&full_bar[q]));
        mbar_init1(smem_addr(&empty_bar[q]));
      }
      mbar_init1(smem_addr(&done_bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.lo)) : "memory");
    }
    if (tid < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                       smem_addr(&tmem_holder))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tmem = tmem_holder;
  }
  while (true) {
    if (tid == 0) sm.item = atomicAdd(counter, 1);
    __syncthreads();
    long long idx = sm.item;
    __syncthreads();
    if (idx >= total) {
      if (umma) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tid < 32)
          asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem)
                       : "memory");
      }
      break;
    }
    const long long item_id = idx;
    int c = c0;
    while (idx >= nt - c + 1) {
      idx -= nt - c + 1;
      ++c;
    }
    const int cols = int(std::min<long long>(TB, n - (long long)c * TB));

    if (idx == nt - c) {
      // ---- emission of the owner's tiles L[c..c+2, c]
      tag(item_id, c, c, kEmit);
      stamp(item_id, 2);
      if (tid == 0) wait_flag(flags + c * nt + c);
      __syncthreads();
      T t[4][4];
      load_t(t, a + c * tile + (long long)c * TB, n, cols, cols, false, vec_ok);
      if (tx == ty) {
#pragma unroll
        for (int u = 0; u < 4; ++u) sm.rdiag[4 * ty + u] = t[u][u];
      }
      __syncthreads();
      emit_tile(t, sm, c, c, n, ghi, glo, gpl, gtt);
      for (int q = 1; q <= 1 && c + q < nt; ++q) {
        const int rq = int(std::min<long long>(TB, n - (long long)(c + q) * TB));
        if (tid == 0) wait_flag(flags + (c + q) * nt + c);
        __syncthreads();
        load_t(t, a + (c + q) * tile + (long long)c * TB, n, rq, TB, false, vec_ok);
        if constexpr (sizeof(T) == 4) {
          if (umma) {  // the owner's sub tile, pre-split for the k-loops (off its chain)
            store_split(t, lhi, llo, (c + q) * tile + (long long)c * TB, n, rq, TB);
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncthreads();
            if (tid == 0) st_release(sflags + (c + q) * nt + c, 1);
          }
        }
        emit_tile(t, sm, c + q, c, n, ghi, glo, gpl, gtt);
      }
      stamp(item_id, 5);
      __syncthreads();
      continue;
    }

    const int r = c + int(idx);
    const bool partial = r <= c + 1;
    tag(item_id, r, c, partial ? kPartial : kFull);
    stamp(item_id, 2);
    const int rows = int(std::min<long long>(TB, n - (long long)r * TB));
    const int kend = partial ? c - 1 : c;  // partial items leave k = c-1 to the owner

    // ---- S = A[r,c] - sum_k L[r,k] L[c,k]^T over the published k (double-
    // buffered staging while the next k is already published)
    if (umma) {
      const int warp = tid >> 5, lane = tid & 31;
      if (c0 < kend) {
        if (warp == 0) {  // ---- producer: tile flags, then four TMA tiles per k
          int horizon = c0;  // every k < horizon is published (rows r and c)
          for (int k = c0; k < kend; ++k) {
            while (horizon <= k) {  // the warp probes the next 32 k of both rows
              const int kk = k + lane;
              const bool ok = kk >= kend || (ld_acquire(sflags + r * nt + kk) != 0 &&
                                             ld_acquire(sflags + c * nt + kk) != 0);
              const unsigned bal = __ballot_sync(0xffffffffu, ok);
              const int run = ~bal ? __ffs(~bal) - 1 : 32;
              horizon = k + run;
              if (run == 0) __nanosleep(40);
            }
            if (lane == 0) {
              asm volatile("fence.proxy.async.global;" ::: "memory");
              mbar_wait_parity(smem_addr(&empty_bar[p_stage]), p_phase ^ 1u);
              const uint32_t fb = smem_addr(&full_bar[p_stage]);
              mbar_expect(fb, kUmmaStage);
              const uint32_t s0 = smem_addr(ub) + p_stage * kUmmaStage;
              const int x0 = k * TB, ya = r * TB, yb = c * TB;
#pragma unroll
              for (int ch = 0; ch < 2; ++ch) {
                tma_tile(s0 + ch * 8192, &maps.hi, fb, x0 + 32 * ch, ya);
                tma_tile(s0 + 16384 + ch * 8192, &maps.lo, fb, x0 + 32 * ch, ya);
                tma_tile(s0 + 32768 + ch * 8192, &maps.hi, fb, x0 + 32 * ch, yb);
                tma_tile(s0 + 49152 + ch * 8192, &maps.lo, fb, x0 + 32 * ch, yb);
              }
              if (++p_stage == kUmmaStages) {
                p_stage = 0;
                p_phase ^= 1u;
              }
            }
            __syncwarp();
          }
        } else if (warp == 1) {  // ---- MMA issuer
          if (lane == 0) {
            for (int k = c0; k < kend; ++k) {
              mbar_wait_parity(smem_addr(&full_bar[m_stage]), m_phase);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              const uint32_t s0 = smem_addr(ub) + m_stage * kUmmaStage;
#pragma unroll
              for (int ch = 0; ch < 2; ++ch)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  const uint32_t off = ch * 8192 + kk * 32;
                  const uint64_t ah = umma_kdesc(s0 + off), al = umma_kdesc(s0 + 16384 + off);
                  const uint64_t bh = umma_kdesc(s0 + 32768 + off), bl = umma_kdesc(s0 + 49152 + off);
                  umma_tf32(tmem, al, bh, (k > c0 || ch > 0 || kk > 0) ? 1u : 0u);
                  umma_tf32(tmem, ah, bl, 1u);
                  umma_tf32(tmem, ah, bh, 1u);
                }
              umma_commit(smem_addr(&empty_bar[m_stage]));
              if (++m_stage == kUmmaStages) {
                m_stage = 0;
                m_phase ^= 1u;
              }
            }
            umma_commit(smem_addr(&done_bar));
          }
          __syncwarp();
        }
        mbar_wait_parity(smem_addr(&done_bar), d_phase);
        d_phase ^= 1u;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (tid < 64) {  // TMEM lanes 0-63 = rows of the product
        T* srow = &sm.sf[tid][0];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v[32];
          if (c0 < kend) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
                "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                  "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                  "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                  "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                  "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + (uint32_t(32 * (tid >> 5)) << 16) + uint32_t(32 * h)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0u;
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) srow[32 * h + e] = T(__uint_as_float(v[e]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
    } else {
      // row-major tiles staged by cp.async
      // (double-buffered while the next k is already published), tensor-core products
      TileAcc<T> acc;
      acc_zero(acc);
      T* const Pb[2] = {sm.ps, sm.sb[0]};
      T* const Qb[2] = {sm.qs, sm.sb[1]};
      if (c0 < kend) {
        if (tid == 0) {
          wait_flag(flags + r * nt + c0);
          wait_flag(flags + c * nt + c0);
        }
        __syncthreads();
        stage_tile(Pb[0], a + (long long)r * tile + (long long)c0 * TB, n, rows, TB, vec_ok);
        stage_tile(Qb[0], a + (long long)c * tile + (long long)c0 * TB, n, cols, TB, vec_ok);
        cp_async_commit();
      }
      int buf = 0;
      int horizon = c0 + 1;  // every k < horizon is known to be published
      for (int k = c0; k < kend; ++k, buf ^= 1) {
        const bool more = k + 1 < kend;
        const int* fr = flags + r * nt + k + 1;
        const int* fc = flags + c * nt + k + 1;
        const bool probe = more && k + 1 >= horizon;
        if (probe && tid < 64) {
          // refresh the horizon: warps 0 / 1 probe the next 32 k of row r / row c
          // (one acquire round trip, all in parallel)
          const int kk = k + 1 + (tid & 31);
          const int* f = flags + (tid < 32 ? r : c) * nt + kk;
          const unsigned bal = __ballot_sync(0xffffffffu, kk < kend && ld_acquire(f));
          if ((tid & 31) == 0) sm.stg[tid >> 5] = ~bal ? __ffs(~bal) - 1 : 32;
        }
        __syncthreads();  // (also: everyone is done with buffer buf ^ 1)
        if (probe) horizon = k + 1 + min(sm.stg[0], sm.stg[1]);
        const bool ready = more && k + 1 < horizon;
        if (ready) {  // prefetch k+1 under this product
          stage_tile(Pb[buf ^ 1], a + (long long)r * tile + (long long)(k + 1) * TB, n, rows, TB, vec_ok);
          stage_tile(Qb[buf ^ 1], a + (long long)c * tile + (long long)(k + 1) * TB, n, cols, TB, vec_ok);
          cp_async_commit();
          cp_async_wait_1();
        } else {
          cp_async_wait_all();
        }
        __syncthreads();
        acc_mma(acc, Pb[buf], Qb[buf]);
        if (more && !ready) {  // at the dependency frontier: wait, then load
          if (tid == 0) wait_flag(fr);
          if (tid == 32) wait_flag(fc);
          __syncthreads();
          horizon = k + 2;
          stage_tile(Pb[buf ^ 1], a + (long long)r * tile + (long long)(k + 1) * TB, n, rows, TB, vec_ok);
          stage_tile(Qb[buf ^ 1], a + (long long)c * tile + (long long)(k + 1) * TB, n, cols, TB, vec_ok);
          cp_async_commit();
        }
      }
      __syncthreads();
      acc_store(acc, &sm.sf[0][0], TB + 1);
    }
    T t[4][4];
    load_t(t, a + (long long)r * tile + (long long)c * TB, n, rows, cols, false, vec_ok);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) t[u][v] -= sm.sf[4 * ty + u][4 * tx + v];
    stamp(item_id, 3);

    if (partial) {
      store_t(t, a + (long long)r * tile + (long long)c * TB, n, rows, cols, false);
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(pflags + 2 * c + (r - c), 1);
      stamp(item_id, 5);
      continue;
    }

    // ---- off-diagonal tile: X = S L[c,c]^-T, with L^-T from the diagonal
    // tile's upper triangle (written by the owner; its diagonal is 1 / L[j][j])
    if (tid == 0) wait_flag(flags + c * nt + c);
    __syncthreads();
    stage_tile(sm.ps, a + (long long)c * tile + (long long)c * TB, n, cols, cols, vec_ok);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) sm.sb[0][(4 * ty + u) * LD + 4 * tx + v] = t[u][v];
    cp_async_wait_all();
    __syncthreads();
    for (int e = tid; e < TB * TB; e += CT) {  // qs = X (row-major [k][j]), rdiag = L[j][j]
      const int i = e >> 6, j = e & 63;
      const T d = sm.ps[i * LD + i];
      sm.qs[i * LD + j] = j > i ? sm.ps[i * LD + j] : (j == i ? (i < cols ? T(1) / d : T(1)) : T(0));
      if (j == 0) sm.rdiag[i] = i < cols ? d : T(1);
    }
    __syncthreads();
    owner_prod<T, true>(sm.sb[0], sm.qs, nullptr, &sm.sf[0][0], TB + 1, T(1), -1);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) t[u][v] = sm.sf[4 * ty + u][4 * tx + v];
    stamp(item_id, 4);
    store_t(t, a + (long long)r * tile + (long long)c * TB, n, rows, cols, false);
    if constexpr (sizeof(T) == 4)
      if (umma) store_split(t, lhi, llo, (long long)r * tile + (long long)c * TB, n, rows, cols);
    __threadfence();
    if (umma) asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      st_release(flags + r * nt + c, 1);
      if (umma) st_release(sflags + r * nt + c, 1);
    }
    stamp(item_id, 5);
    emit_tile(t, sm, r, c, n, ghi, glo, gpl, gtt);
    __syncthreads();
  }
}

// Inverse of each 64x64 diagonal block of L (lower): dinv[b] = L_bb^-1.
// Column-parallel forward substitution (off the hot path: parity artefacts).
template <typename T>
__global__ void diag_inverse_kernel(const T* __restrict__ l, long long n, T* dinv) {
  __shared__ T ls[TB][TB + 1];
  const int b = blockIdx.x, tid = threadIdx.x;
  T* xs = dinv + (long long)b * TB * TB;  // X[i][j] at xs[i*TB + j]
  const long long k0 = (long long)b * TB;
  const int w = int(std::min<long long>(TB, n - k0));
  for (int e = tid; e < TB * TB; e += blockDim.x) {
    const int r = e / TB, c = e % TB;
    T v = (r < w && c < w) ? l[(k0 + r) * n + k0 + c] : T(r == c ? 1 : 0);
    ls[r][c] = (c <= r) ? v : T(0);
  }
  __syncthreads();
  if (tid < TB) {
    const int j = tid;  // column j of the inverse: L x = e_j
    for (int i = 0; i < TB; ++i) {
      T s = (i == j) ? T(1) : T(0);
      for (int k = j; k < i; ++k) s -= ls[i][k] * xs[k * TB + j];
      xs[i * TB + j] = (i < j) ? T(0) : s / ls[i][i];
    }
  }
}

// X = blockdiag(dinv_k), zero elsewhere (lower block triangle is filled by the doubling)
template <typename T>
__global__ void init_inverse_kernel(T* x, long long n, const T* __restrict__ dinv) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e % n;
    const long long br = r / TB, bc = c / TB;
    x[e] = (br == bc) ? dinv[br * TB * TB + (r % TB) * TB + (c % TB)] : T(0);
  }
}

// U[r][c] = X[n-1-r][n-1-c] for r <= c (X = L^-1 lower), else 0
template <typename T>
__global__ void reverse_to_upper_kernel(const T* __restrict__ x, long long n, T* u) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e % n;
    u[e] = (r <= c) ? x[(n - 1 - r) * n + (n - 1 - c)] : T(0);
  }
}

inline int blocks_for(long long n) {
  long long g = (n + 255) / 256;
  return int(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

int num_sms_f() { return device_sms(); }

// Micro-benchmark (debug): one CTA factors a well-conditioned 64 x 64 tile
// `iters` times; cycles[0] = total clocks, cycles[1] = clocks of the last
// factor_tile64 call, out = L (64 x 64) for a correctness check.
template <typename T>
__global__ void __launch_bounds__(CT, 1) factor_bench_kernel(int iters, long long* cycles, T* out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  CholSmem<T>& sm = *reinterpret_cast<CholSmem<T>*>(smraw);
  const int tid = threadIdx.x;
  long long t_last = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int e = tid; e < TB * TB; e += CT) {
      const int r = e >> 6, c = e & 63;
      sm.sf[r][c] = r == c ? T(64 + r) : T(1) / T(1 + r + c);
    }
    __syncthreads();
    const long long t1 = clock64();
    factor_tile64(sm, cycles + 2);
    t_last = clock64() - t1;
  }
  const long long t2 = clock64();
  if (tid == 0) {
    cycles[0] = t2 - t0;
    cycles[1] = t_last;
  }
  for (int e = tid; e < TB * TB; e += CT) out[e] = sm.sf[e >> 6][e & 63];
}

}  // namespace

void debug_factor_bench(int iters, long long* cycles, float* out, cudaStream_t st) {
  cudaFuncSetAttribute(factor_bench_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(CholSmem<float>)));
  count_launches(1);
  factor_bench_kernel<float><<<1, CT, sizeof(CholSmem<float>), st>>>(iters, cycles, out);
}

size_t cholesky_flag_ints(long long n) {
  const long long nt = (n + TB - 1) / TB;
  // tile flags, partial flags, per-panel item counters + owner slots (<= nt panels),
  // split-stored flags (the tcgen05 k-loops' operands)
  return size_t(nt * nt + 2 * nt + 2 * nt + 8 + nt * nt);
}

void launch_damp(const float* h, long long n, double percdamp, double* damp, float* diag,
                 cudaStream_t st) {
  count_launches(1);
  damp_kernel<<<1, 1024, 0, st>>>(h, n, percdamp, damp, diag);
}

template <typename T>
void launch_build_factor_input(const float* h, long long n, const int32_t* order, double percdamp,
                               T* a, double* damp, cudaStream_t st, bool damp_ready) {
  if (!damp_ready) launch_damp(h, n, percdamp, damp, nullptr, st);
  count_launches(1);
  const size_t row_bytes = size_t(n) * sizeof(float);
  if (row_bytes <= 200 * 1024) {
    cudaFuncSetAttribute(build_input_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    build_input_rows_kernel<T><<<unsigned(n), 256, row_bytes, st>>>(h, n, order, damp, a);
  } else {
    build_input_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(h, n, order, damp, a);
  }
}

using EncodeTiledF = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledF encoder_f() {
  static EncodeTiledF fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiledF(nullptr);
    return reinterpret_cast<EncodeTiledF>(ptr);
  }();
  return fn;
}
// n x n fp32 row-major, 32-column x 64-row boxes, SWIZZLE_128B, zero fill out of range
bool split_map(CUtensorMap* m, const float* base, long long n) {
  EncodeTiledF enc = encoder_f();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {cuuint64_t(n), cuuint64_t(n)};
  const cuuint64_t gstride[1] = {cuuint64_t(n) * 4};
  const cuuint32_t box[2] = {32, TB};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T>
void cholesky_g(T* a, long long n, T* ghi, float* glo, float* gpl, float* gtt, int* flags,
                unsigned* status, long long macro_cols, cudaStream_t st, float* lhi, float* llo) {
  // fp32 with the pre-split L (lhi / llo): worker products on tcgen05 (TMA ring
  // after the shared struct's small fields, one CTA per SM)
  UmmaMaps maps{};
  if (sizeof(T) != 4 || n % 4 != 0 || !lhi || !llo || !split_map(&maps.hi, lhi, n) ||
      !split_map(&maps.lo, llo, n))
    lhi = llo = nullptr;
  const int smem = lhi ? std::max<int>(int(sizeof(CholSmem<T>)), kUmmaEnd)
                       : int(sizeof(CholSmem<T>));
  cudaFuncSetAttribute(chol_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);  // (per device: set on every call)
  const int nt = int((n + TB - 1) / TB);
  int* pflags = flags + (long long)nt * nt;
  int* counters = pflags + 2LL * nt;
  int* sflags = counters + 2LL * nt + 8;
  cudaMemsetAsync(flags, 0, cholesky_flag_ints(n) * sizeof(int), st);
  if (gtt) cudaMemsetAsync(gtt, 0, size_t(n) * 128 * sizeof(float), st);  // non-emitted = 0
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_tile_kernel<T>, CT, smem);
  const int max_ctas = std::max(1, occ) * num_sms_f();
  const int step = macro_cols <= 0 ? nt : int(std::max<long long>(1, macro_cols / TB));
  int ci = 0;
  for (int c0 = 0; c0 < nt; c0 += step, ++ci) {
    const int c1 = std::min(nt, c0 + step);
    long long items = 0;  // worker items; CTA 0 is the owner of the critical path
    for (int c = c0; c < c1; ++c) items += nt - c + 1;
    const int grid = 1 + int(std::min<long long>(items, std::max(1, max_ctas - 1)));
    count_launches(1);
    unsigned long long* trace = nullptr;
    const char* tp = getenv("OCWG_CHOL_TRACE");
    const long long entries = items + 2LL * (c1 - c0);
    if (tp) {
      cudaMallocAsync(&trace, size_t(entries) * 6 * 8, st);
      cudaMemsetAsync(trace, 0, size_t(entries) * 6 * 8, st);
    }
    chol_tile_kernel<T><<<grid, CT, smem, st>>>(a, n, nt, c0, c1, flags, pflags, counters + ci,
                                                status, ghi, glo, gpl, gtt, trace, maps, lhi, llo,
                                                sflags);
    if (tp) {
      std::vector<unsigned long long> h(size_t(entries) * 6);
      cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cudaFreeAsync(trace, st);
      if (FILE* f = fopen(tp, "ab")) {
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
      }
    }
    const long long k0 = (long long)c0 * TB, k1 = std::min<long long>(n, (long long)c1 * TB);
    const long long rest = n - k1;
    if (rest > 0)  // trailing SYRK: A22 -= L21 L21^T (lower tiles)
      mm<T>(rest, rest, k1 - k0, -1.0, a + k1 * n + k0, n, false, a + k1 * n + k0, n, true, 1.0,
            a + k1 * n + k1, n, true, st);
  }
}

// X = L^-1 (n x n lower) from the Cholesky factor (a, lower) by recursive
// doubling over the 64x64 diagonal blocks.  ws: nblk*64*64 + n*n elements.
template <typename T>
void lower_inverse(const T* a, long long n, T* x, T* ws, cudaStream_t st) {
  const long long nblk = (n + TB - 1) / TB;
  T* dinv = ws;
  T* tmp = ws + nblk * TB * TB;
  count_launches(2);
  diag_inverse_kernel<T><<<unsigned(nblk), 64, 0, st>>>(a, n, dinv);
  init_inverse_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(x, n, dinv);
  for (long long s = 2 * TB; s < 2 * n; s *= 2) {
    const long long h = s / 2;
    const long long full = n / s;
    if (full > 0) {
      const long long stride = s * (n + 1);
      mm<T>(h, h, h, 1.0, a + h * n, n, false, x, n, false, 0.0, tmp, h, false, st, int(full),
            stride, stride, h * h);
      mm<T>(h, h, h, -1.0, x + h * n + h, n, false, tmp, h, false, 0.0, x + h * n, n, false, st,
            int(full), stride, h * h, stride);
    }
    const long long p0 = full * s, c2 = n - p0 - h;
    if (c2 > 0) {
      mm<T>(c2, h, h, 1.0, a + (p0 + h) * n + p0, n, false, x + p0 * n + p0, n, false, 0.0, tmp, h,
            false, st);
      mm<T>(c2, h, c2, -1.0, x + (p0 + h) * n + (p0 + h), n, false, tmp, h, false, 0.0,
            x + (p0 + h) * n + p0, n, false, st);
    }
  }
}

// U = (J L J)^-1 from the Cholesky factor (a, lower): parity artefact path.
// ws: ceil(n/64)*64*64 + n*n elements; u receives U (n x n upper).
template <typename T>
void upper_from_cholesky(const T* a, long long n, T* u, T* ws, cudaStream_t st) {
  const long long nblk = (n + TB - 1) / TB;
  lower_inverse<T>(a, n, u, ws, st);
  T* tmp = ws + nblk * TB * TB;
  count_launches(1);
  reverse_to_upper_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(u, n, tmp);
  cudaMemcpyAsync(u, tmp, size_t(n * n) * sizeof(T), cudaMemcpyDeviceToDevice, st);
}

template <typename T>
void launch_gram_upper(const T* u, long long n, double* hinv, cudaStream_t st) {
  gemm<double, T, T>(n, n, n, 1.0, u, n, true, u, n, false, 0.0, hinv, n, false, st);
}

template void launch_build_factor_input<float>(const float*, long long, const int32_t*, double,
                                               float*, double*, cudaStream_t, bool);
template void launch_build_factor_input<double>(const float*, long long, const int32_t*, double,
                                                double*, double*, cudaStream_t, bool);
template void cholesky_g<float>(float*, long long, float*, float*, float*, float*, int*,
                                unsigned*, long long, cudaStream_t, float*, float*);
template void cholesky_g<double>(double*, long long, double*, float*, float*, float*, int*,
                                 unsigned*, long long, cudaStream_t, float*, float*);
template void lower_inverse<float>(const float*, long long, float*, float*, cudaStream_t);
template void lower_inverse<double>(const double*, long long, double*, double*, cudaStream_t);
template void upper_from_cholesky<float>(const float*, long long, float*, float*, cudaStream_t);
template void upper_from_cholesky<double>(const double*, long long, double*, double*,
                                          cudaStream_t);
template void launch_gram_upper<float>(const float*, long long, double*, cudaStream_t);
template void launch_gram_upper<double>(const double*, long long, double*, cudaStream_t);

}  // namespace ocwg
