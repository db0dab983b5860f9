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
// Cholesky: one persistent, dataflow-scheduled kernel over 64x64 tiles.
// Work items are the lower tiles (r, c) of a column range [c0, c1) in
// column-major order, handed out by an atomic counter; item (r, c) computes
//   S = A[r,c] - sum_{c0<=k<c} L[r,k] L[c,k]^T
// waiting on per-tile ready flags (acquire/release) for each L[.,k], then
//   r == c: factors S (64-step right-looking elimination, one barrier per step)
//   r >  c: L[r,c] = S L[c,c]^-T by forward substitution (warp shuffles only)
// and publishes L[r,c] (and the matching block of G) with a release flag.
// Items only ever wait on items handed out earlier, so the schedule cannot
// deadlock whatever the residency.  Large n runs macro panels: the dataflow
// kernel over a column range, then one tcgen05 3xTF32 SYRK for the trailing
// matrix (gemm.cu / tc_gemm.cu).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
                            double* damp) {
  __shared__ double part[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += double(h[i * n + i]);
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

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t u = __float_as_uint(x);
  u = (u + 0xFFFu + ((u >> 13) & 1u)) & ~0x1FFFu;  // RNE to 10 mantissa bits
  return __uint_as_float(u);
}

// 1/x and 1/sqrt(x) to fp32 accuracy without the IEEE slow-path checks
// (pivots are positive normal numbers, or the factorisation has failed)
__device__ __forceinline__ float rcp_nr(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return fmaf(y, fmaf(-x, y, 1.0f), y);
}
__device__ __forceinline__ double rcp_nr(double x) { return 1.0 / x; }
__device__ __forceinline__ float rsqrt_nr(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y * fmaf(-0.5f * x * y, y, 1.5f);
}
__device__ __forceinline__ double rsqrt_nr(double x) { return rsqrt(x); }
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  reinterpret_cast<double2*>(p)[0] = make_double2(a, b);
  reinterpret_cast<double2*>(p)[1] = make_double2(c, d);
}

// Position of block-local column kk (0..127) of a sweep block row in the
// in-block kernel's order: lane group rg = kk % 4 owns slots s = kk / 4,
// stored in 16-byte chunks c = s / 4, XOR-swizzled by 2 rg (sweep.cu).
__host__ __device__ inline int gp_pos(int kk) {
  const int rg = kk & 3, s = kk >> 2;
  return rg * 32 + 4 * ((s >> 2) ^ (2 * rg)) + (s & 3);
}

// A 64x64 tile (row-major, ld) <-> 16 elements per thread: rows tid/16 + 16*ii,
// cols 4*(tid%16) + e.  Out-of-range elements read as 0.
template <typename T>
struct TileRegs {
  T v[4][4];
};

template <typename T>
__device__ __forceinline__ void load_tile(TileRegs<T>& R, const T* base, long long ld, int rows,
                                          int cols, bool vec_ok) {
  const int tid = threadIdx.x, c4 = (tid & 15) * 4;
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int r = (tid >> 4) + 16 * ii;
    const T* p = base + (long long)r * ld + c4;
    if (vec_ok && r < rows && c4 + 4 <= cols) {
      if constexpr (sizeof(T) == 4) {
        const float4 f = __ldcg(reinterpret_cast<const float4*>(p));
        R.v[ii][0] = f.x, R.v[ii][1] = f.y, R.v[ii][2] = f.z, R.v[ii][3] = f.w;
      } else {
        const double2 f0 = __ldcg(reinterpret_cast<const double2*>(p));
        const double2 f1 = __ldcg(reinterpret_cast<const double2*>(p + 2));
        R.v[ii][0] = f0.x, R.v[ii][1] = f0.y, R.v[ii][2] = f1.x, R.v[ii][3] = f1.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) R.v[ii][e] = (r < rows && c4 + e < cols) ? ldcg(p + e) : T(0);
    }
  }
}

// Store the tile transposed into swizzled k-major smem: S[k][i] at
// k*64 + ((i/4) ^ ((k/4)&15))*4 + i%4  (conflict-free stores and float4 reads).
template <typename T>
__device__ __forceinline__ void store_tile_t(const TileRegs<T>& R, T* S) {
  const int tid = threadIdx.x, tx = tid & 15;
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int i = (tid >> 4) + 16 * ii;
    const int pg = (i >> 2) ^ tx;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = 4 * tx + e;
      S[k * TB + pg * 4 + (i & 3)] = R.v[ii][e];
    }
  }
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

// acc[u][v] += sum_k P[4ty+u][k] * Q[4tx+v][k]
template <typename T>
__device__ __forceinline__ void tile_mma(T (&acc)[4][4], const T* Ps, const T* Qs) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
#pragma unroll 4
  for (int k = 0; k < TB; ++k) {
    const int sw = (k >> 2) & 15;
    T p[4], q[4];
    ld4(Ps + k * TB + ((ty ^ sw) << 2), p);
    ld4(Qs + k * TB + ((tx ^ sw) << 2), q);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = fma(p[u], q[v], acc[u][v]);
  }
}

template <typename T>
struct CholSmem {
  T ps[TB * TB];
  T qs[TB * TB];
  T lt[TB][TB + 4];   // diag tile L_cc transposed (lt[j][c] = L[c][j]); also G staging
  T col[2][TB];       // (unused)
  T sf[TB][TB + 1];   // diagonal tile being factored
  T wcol[2][72];      // warp elimination: published pivot column (shifted, + zero pad)
  T lt32[32][40];     // warp elimination: L columns, shifted like wcol (for the solve)
  T rdiag[TB];
  int item;
  int ready;
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

// Warp-synchronous right-looking Cholesky of a 32 x 32 block held one row per
// lane (a[k] = A[lane][j0 + k], lower part used), written to out[lane][j0 + j].
// The register array rotates as it is updated (a[0] is always the pivot
// column).  Per pivot each lane publishes its pivot-column entry to shared
// memory (one store + warp sync, double-buffered, zero-padded past 32) and
// reads the others as broadcasts: no block barrier, no shuffles.
// With WITH_B, each lane also carries row 32 + lane (b[k] = A[32 + lane][j0 + k])
// through the same pivots: b ends as L21 = A21 L11^-T (written to out_b), off
// the pivot chain.
template <typename T, bool WITH_B>
__device__ __forceinline__ bool warp_chol32(T (&a)[32], T (&b)[32], T* out_row, T* out_b,
                                            T* rdiag, T (*wcol)[72], T (*lt32)[40] = nullptr) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    // stored at lane + sh so that entry j+1 starts a 16-byte chunk: the 31
    // entries a lane needs are 8 LDS.128 broadcasts
    const int sh = (3 - j) & 3;
    T* cb = wcol[j & 1];
    cb[lane + sh] = a[0];
    const T p = __shfl_sync(0xffffffffu, a[0], j);  // pivot off the shared-memory round trip
    __syncwarp();
    // the column entries first: their load latency overlaps the rsqrt chain
    T v[32];
    const T* nxt = cb + j + sh + 1;  // 16-byte aligned
#pragma unroll
    for (int k4 = 0; k4 < 32; k4 += 4) {
      T v4[4];
      ld4(nxt + k4, v4);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[k4 + e] = v4[e];
    }
    ok &= (p > T(0));
    const T rs = rsqrt_nr(p);
    const T l = a[0] * rs;  // L[lane][j]; lane j: sqrt(p)
    const T lrs = l * rs;   // a[k] -= L[lane][j] L[j+k][j] = lrs * a_{j+k}[j]
#pragma unroll
    for (int k = 0; k + 1 < 32; ++k) a[k] = fma(-lrs, v[k], a[k + 1]);
    a[31] = T(0);
    const T lo = lane >= j ? l : T(0);
    out_row[j] = lo;
    if (lt32) lt32[j][lane + sh] = lo;  // column j of L, shifted like cb (for the solve)
    if (lane == j) rdiag[j] = rs;  // 1 / L[j][j]
    if (WITH_B) {
      const T lb = b[0] * rs;  // L21[lane][j]
      const T lbrs = lb * rs;
#pragma unroll
      for (int k = 0; k + 1 < 32; ++k) b[k] = fma(-lbrs, v[k], b[k + 1]);
      b[31] = T(0);
      out_b[j] = lb;
    }
  }
  return ok;
}

// Factor the 64 x 64 tile in sm.sf (lower, padded with identity) in place:
// L11 = chol(A11) and L21 = A21 L11^-T by warp 0, A22 -= L21 L21^T by the
// CTA, L22 = chol(A22) by warp 0.  Upper entries are zeroed; sm.rdiag gets
// 1 / L[j][j].  All threads call.
template <typename T>
__device__ bool factor_tile64(CholSmem<T>& sm, long long* prof = nullptr) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  bool ok = true;
  auto pstamp = [&](int i) {
    if (prof && tid == 0) prof[i] = clock64();
  };
  pstamp(0);
  for (int e = tid; e < 2 * 72; e += CT) sm.wcol[e / 72][e % 72] = T(0);
  for (int e = tid; e < 32 * 40; e += CT) sm.lt32[e / 40][e % 40] = T(0);
  __syncthreads();
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int o = 32 * h;  // diagonal block [o, o+32)
    if (warp == 0) {
      T av[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) av[k] = sm.sf[o + lane][o + k];
      ok &= warp_chol32<T, false>(av, av, &sm.sf[o + lane][o], nullptr, &sm.rdiag[o], sm.wcol,
                                  sm.lt32);
      pstamp(1 + 3 * h);
      if (h == 0) {
        __syncwarp();
        // L21: rows 32 + lane solve x L11^T = a (forward substitution, rotating)
#pragma unroll
        for (int k = 0; k < 32; ++k) av[k] = sm.sf[32 + lane][k];
#pragma unroll 1
        for (int j = 0; j < 32; ++j) {
          T v[32];
          const T* lcol = &sm.lt32[j][j + ((3 - j) & 3) + 1];  // L11[j+1..][j], aligned
#pragma unroll
          for (int k4 = 0; k4 < 32; k4 += 4) {
            T v4[4];
            ld4(lcol + k4, v4);
#pragma unroll
            for (int e = 0; e < 4; ++e) v[k4 + e] = v4[e];
          }
          const T x = av[0] * sm.rdiag[j];
#pragma unroll
          for (int k = 0; k + 1 < 32; ++k) av[k] = fma(-x, v[k], av[k + 1]);
          av[31] = T(0);
          sm.sf[32 + lane][j] = x;
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) sm.sf[lane][32 + k] = T(0);
        pstamp(2);
      }
    }
    __syncthreads();
    if (h == 0) {  // A22 -= L21 L21^T: thread -> row i, 4 columns
      const int i = tid >> 3, j0 = (tid & 7) * 4;
      T s4[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const T li = sm.sf[32 + i][k];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) s4[jj] = fma(li, sm.sf[32 + j0 + jj][k], s4[jj]);
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        if (j0 + jj <= i) sm.sf[32 + i][32 + j0 + jj] -= s4[jj];
      __syncthreads();
      pstamp(3);
    }
  }
  return ok;
}

template <typename T>
__global__ void __launch_bounds__(CT, sizeof(T) == 4 ? 2 : 1)
    chol_tile_kernel(T* __restrict__ a, long long n, int nt, int c0, int c1, int* flags,
                     int* counter, unsigned* status, T* ghi, float* glo, float* gpl, float* gtt,
                     unsigned long long* trace) {
  extern __shared__ __align__(16) unsigned char smraw[];
  CholSmem<T>& sm = *reinterpret_cast<CholSmem<T>*>(smraw);
  // optional timeline (debug): per item {r, c, start, k-loop done, solve done, published}
  auto stamp = [&](long long item, int slot) {
    if (trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[item * 6 + slot] = t;
    }
  };
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31;
  const bool vec_ok = (sizeof(T) == 4 ? (n & 3) == 0 : (n & 1) == 0);
  long long total = 0;
  for (int c = c0; c < c1; ++c) total += nt - c;

  while (true) {
    if (tid == 0) sm.item = atomicAdd(counter, 1);
    __syncthreads();
    long long idx = sm.item;
    __syncthreads();
    if (idx >= total) break;
    const long long item_id = idx;
    int c = c0;
    while (idx >= nt - c) {
      idx -= nt - c;
      ++c;
    }
    const int r = c + int(idx);
    if (trace && tid == 0) {
      trace[item_id * 6 + 0] = (unsigned long long)r;
      trace[item_id * 6 + 1] = (unsigned long long)c;
    }
    stamp(item_id, 2);
    const int rows = int(std::min<long long>(TB, n - (long long)r * TB));
    const int cols = int(std::min<long long>(TB, n - (long long)c * TB));

    // ---- S = A[r,c] - sum_k L[r,k] L[c,k]^T
    T acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
    TileRegs<T> P, Q;
    if (c0 < c) {
      if (tid == 0) {
        wait_flag(flags + r * nt + c0);
        wait_flag(flags + c * nt + c0);
      }
      __syncthreads();
      load_tile(P, a + (long long)r * TB * n + (long long)c0 * TB, n, rows, TB, vec_ok);
      load_tile(Q, a + (long long)c * TB * n + (long long)c0 * TB, n, cols, TB, vec_ok);
    }
    for (int k = c0; k < c; ++k) {
      store_tile_t(P, sm.ps);
      store_tile_t(Q, sm.qs);
      const bool more = k + 1 < c;
      const int* fr = flags + r * nt + k + 1;
      const int* fc = flags + c * nt + k + 1;
      if (tid == 0) sm.ready = more && ld_acquire(fr) && ld_acquire(fc);
      __syncthreads();
      const bool ready = sm.ready;
      // prefetch k+1 under the MMA when its tiles are already published
      if (ready) {
        load_tile(P, a + (long long)r * TB * n + (long long)(k + 1) * TB, n, rows, TB, vec_ok);
        load_tile(Q, a + (long long)c * TB * n + (long long)(k + 1) * TB, n, cols, TB, vec_ok);
      }
      tile_mma(acc, sm.ps, sm.qs);
      if (more && !ready) {  // at the dependency frontier: wait, then load
        if (tid == 0) {
          wait_flag(fr);
          wait_flag(fc);
        }
        __syncthreads();
        load_tile(P, a + (long long)r * TB * n + (long long)(k + 1) * TB, n, rows, TB, vec_ok);
        load_tile(Q, a + (long long)c * TB * n + (long long)(k + 1) * TB, n, cols, TB, vec_ok);
      }
      __syncthreads();
    }
    // t = A[r,c] - acc (own 4x4 block: rows 4ty+u, cols 4tx+v)
    T t[4][4];
    {
      const T* ab = a + (long long)r * TB * n + (long long)c * TB;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = 4 * ty + u;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int cc = 4 * tx + v;
          T x = (rr < rows && cc < cols) ? ab[(long long)rr * n + cc] : T(0);
          if (r == c && rr == cc && rr >= rows) x = T(1);  // identity padding
          t[u][v] = x - acc[u][v];
        }
      }
    }

    stamp(item_id, 3);
    if (r == c) {
      // ---- diagonal tile: warp-level factorisation in shared memory (factor_tile64)
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) sm.sf[4 * ty + u][4 * tx + v] = t[u][v];
      __syncthreads();
      const bool ok = factor_tile64(sm);
      if (!ok && tid == 0 && cols > 0) atomicOr(status, kFlagNotPD);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) t[u][v] = sm.sf[4 * ty + u][4 * tx + v];
      // diag values for G scaling
      if (tx == ty) {
#pragma unroll
        for (int u = 0; u < 4; ++u) sm.rdiag[4 * ty + u] = t[u][u];
      }
    } else {
      // ---- off-diagonal tile: X L_cc^T = t by forward substitution
      if (tid == 0) wait_flag(flags + c * nt + c);
      __syncthreads();
      {
        const T* lb = a + (long long)c * TB * n + (long long)c * TB;
        T x[TB * TB / CT];
#pragma unroll
        for (int q = 0; q < TB * TB / CT; ++q) {
          const int e = tid + q * CT, rr = e >> 6, cl = e & 63;
          x[q] = (rr < cols && cl <= rr) ? ldcg(lb + (long long)rr * n + cl) : T(rr == cl ? 1 : 0);
        }
#pragma unroll
        for (int q = 0; q < TB * TB / CT; ++q) {
          const int e = tid + q * CT, rr = e >> 6, cl = e & 63;
          sm.lt[cl][rr] = x[q];  // lt[j][c] = L[c][j]
        }
      }
      __syncthreads();
      if (tid < TB) sm.rdiag[tid] = T(1) / sm.lt[tid][tid];
      __syncthreads();
      const int src0 = lane & 16;
#pragma unroll 1
      for (int j0 = 0; j0 < TB; j0 += 4) {
        const bool own = tx == (j0 >> 2), later = tx > (j0 >> 2);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = j0 + jj;
          const T rd = sm.rdiag[j];
          T x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = __shfl_sync(0xffffffffu, t[u][jj] * rd, src0 + (j >> 2));
          if (own) {
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u][jj] = x[u];
          }
          T l[4];
          ld4(&sm.lt[j][4 * tx], l);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (later || (own && v > jj)) {
#pragma unroll
              for (int u = 0; u < 4; ++u) t[u][v] = fma(-x[u], l[v], t[u][v]);
            }
        }
      }
      // diag values of L_cc for G scaling: lt[j][j]
      __syncthreads();
      if (tid < TB) sm.rdiag[tid] = sm.lt[tid][tid];
    }

    stamp(item_id, 4);
    // ---- store L[r,c], publish
    {
      T* ab = a + (long long)r * TB * n + (long long)c * TB;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = 4 * ty + u;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int cl = 4 * tx + v;
          if (rr < rows && cl < cols && (r != c || cl <= rr)) ab[(long long)rr * n + cl] = t[u][v];
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(flags + r * nt + c, 1);
    stamp(item_id, 5);
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
    if (ghi) {
      // rdiag holds L[a][a] of column tile c (written before the last barrier)
      emit_g(t, sm, sm.rdiag, r, c, n, ghi, glo, gpl);
    }
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

int num_sms_f() {
  static int v = [] {
    int dev = 0, s = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    return s;
  }();
  return v;
}

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
  return size_t(nt * nt + 64);
}

template <typename T>
void launch_build_factor_input(const float* h, long long n, const int32_t* order, double percdamp,
                               T* a, double* damp, cudaStream_t st) {
  count_launches(2);
  damp_kernel<<<1, 1024, 0, st>>>(h, n, percdamp, damp);
  const size_t row_bytes = size_t(n) * sizeof(float);
  if (row_bytes <= 200 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(build_input_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr = true;
    }
    build_input_rows_kernel<T><<<unsigned(n), 256, row_bytes, st>>>(h, n, order, damp, a);
  } else {
    build_input_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(h, n, order, damp, a);
  }
}

template <typename T>
void cholesky_g(T* a, long long n, T* ghi, float* glo, float* gpl, float* gtt, int* flags,
                unsigned* status, long long macro_cols, cudaStream_t st) {
  static const bool attr = [] {
    cudaFuncSetAttribute(chol_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(CholSmem<T>)));
    return true;
  }();
  (void)attr;
  const int nt = int((n + TB - 1) / TB);
  int* counters = flags + (long long)nt * nt;
  cudaMemsetAsync(flags, 0, cholesky_flag_ints(n) * sizeof(int), st);
  if (gtt) cudaMemsetAsync(gtt, 0, size_t(n) * 128 * sizeof(float), st);  // non-emitted = 0
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_tile_kernel<T>, CT,
                                                sizeof(CholSmem<T>));
  const int max_ctas = std::max(1, occ) * num_sms_f();
  const int step = macro_cols <= 0 ? nt : int(std::max<long long>(1, macro_cols / TB));
  int ci = 0;
  for (int c0 = 0; c0 < nt; c0 += step, ++ci) {
    const int c1 = std::min(nt, c0 + step);
    long long items = 0;
    for (int c = c0; c < c1; ++c) items += nt - c;
    const int grid = int(std::min<long long>(items, max_ctas));
    count_launches(1);
    unsigned long long* trace = nullptr;
    const char* tp = getenv("OCWG_CHOL_TRACE");
    if (tp) cudaMallocAsync(&trace, size_t(items) * 6 * 8, st);
    chol_tile_kernel<T><<<grid, CT, sizeof(CholSmem<T>), st>>>(a, n, nt, c0, c1, flags,
                                                                counters + ci, status, ghi, glo, gpl,
                                                                gtt, trace);
    if (tp) {
      std::vector<unsigned long long> h(size_t(items) * 6);
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
                                               float*, double*, cudaStream_t);
template void launch_build_factor_input<double>(const float*, long long, const int32_t*, double,
                                                double*, double*, cudaStream_t);
template void cholesky_g<float>(float*, long long, float*, float*, float*, float*, int*,
                                unsigned*, long long, cudaStream_t);
template void cholesky_g<double>(double*, long long, double*, float*, float*, float*, int*,
                                 unsigned*, long long, cudaStream_t);
template void lower_inverse<float>(const float*, long long, float*, float*, cudaStream_t);
template void lower_inverse<double>(const double*, long long, double*, double*, cudaStream_t);
template void upper_from_cholesky<float>(const float*, long long, float*, float*, cudaStream_t);
template void upper_from_cholesky<double>(const double*, long long, double*, double*,
                                          cudaStream_t);
template void launch_gram_upper<float>(const float*, long long, double*, cudaStream_t);
template void launch_gram_upper<double>(const double*, long long, double*, cudaStream_t);

}  // namespace ocwg
