// On-GPU factorisation for GPTQ (replaces layerwise.cpp:31-51):
//   hd = fp64(H); damp = percdamp*mean(diag(hd)); hd += damp*I;
//   hp = P hd P^T;  hinv = hp^-1;  U = upper Cholesky factor of hinv.
// Computed as  A = J hp J = L L^T (lower, blocked right-looking),
//              U = J L^-1 J.
// Mathematically identical to the reference's LLT -> solve(I) -> LLT (by the
// uniqueness of the Cholesky factor of hinv), with 2n^3/3 (Cholesky n^3/3 +
// inverse) instead of 8n^3/3 flops.  Templated on the compute type T (float
// default, double = the reference's arithmetic class).
//
// Cholesky: one fused launch per 64-column panel (every CTA factors + inverts
// the 64x64 diagonal block in shared memory; CTA 0 stores L_kk and L_kk^-1,
// CTA c >= 1 solves its 64-row slice of the panel), then one trailing SYRK
// (tensor cores in fp32 mode).  Triangular inverse: log-depth recursive
// doubling over the diagonal blocks,
//   inv([A 0; B C]) = [A^-1 0; -C^-1 (B A^-1), C^-1],
// each level two batched GEMMs (6 levels for n = 4096).
#include <cmath>

#include "kernels.h"

namespace ocwg {
namespace {

constexpr int NB = 64;  // panel width / base block

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

// Fused panel step at column k0 (block width nb <= 64).
// Every CTA factors and inverts the (already updated) 64x64 diagonal block
// with a 16x16 grid of threads, each holding a 4x4 register tile (static
// register indices, two barriers per elimination step: publish column/row j,
// then rank-1 update).  Rows/cols >= nb are identity padding.  CTA 0 stores
// L_kk (into A) and L_kk^-1 (dinv); CTA c >= 1 computes its 64-row panel slice
// L_slice = A_slice * L_kk^-T and writes it back into A.
template <typename T>
__device__ __forceinline__ T pick4(const T (&v)[4], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : (i == 2 ? v[2] : v[3]));
}

template <typename T>
__global__ void __launch_bounds__(256) panel_kernel(T* a, long long n, long long k0, T* dinv,
                                                    unsigned* flag) {
  extern __shared__ __align__(16) unsigned char dsm_raw[];
  T(*lb)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(dsm_raw);                              // L
  T(*xb)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(dsm_raw + sizeof(T) * NB * (NB + 1));  // L^-1
  T(*ps)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(dsm_raw + 2 * sizeof(T) * NB * (NB + 1));
  T* diag = reinterpret_cast<T*>(dsm_raw + 3 * sizeof(T) * NB * (NB + 1));
  T* vec = diag + NB;  // column j of L / row j of L^-1 being published
  const int nb = int(min((long long)NB, n - k0));
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const long long r0 = k0 + nb + (long long)(blockIdx.x - 1) * NB;  // panel slice rows
  const int pr = blockIdx.x == 0 ? 0 : int(min((long long)NB, n - r0));

  T t[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = 4 * ti + u, c = 4 * tj + v;
      T val = T(0);
      if (r < nb && c < nb) {
        if (c <= r) val = a[(k0 + r) * n + k0 + c];
      } else if (r == c) {
        val = T(1);
      }
      t[u][v] = val;
      if (r == c) diag[r] = val;
    }
  if (blockIdx.x > 0)
    for (int e = tid; e < NB * NB; e += 256) {
      const int r = e / NB, c = e % NB;
      ps[r][c] = (r < pr && c < nb) ? a[(r0 + r) * n + k0 + c] : T(0);
    }
  __syncthreads();

  // ---- Cholesky of the block (right-looking, lower)
  bool bad = false;
  for (int j = 0; j < NB; ++j) {
    const T piv = diag[j];
    const T d = sqrt(piv);
    const T rd = T(1) / d;
    if (tid == 0 && j < nb) bad |= !(piv > T(0));  // Eigen: x <= 0 -> NumericalIssue
    if (tj == (j >> 2) && ti >= tj) {
      const int jj = j & 3;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = 4 * ti + u;
        if (r > j) {
          const T lv = pick4(t[u], jj) * rd;
          vec[r] = lv;
          lb[r][j] = lv;
        } else if (r == j) {
          lb[j][j] = d;
        }
      }
    }
    __syncthreads();
    if (ti >= tj && 4 * ti + 3 > j && 4 * tj + 3 > j) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = 4 * ti + u;
        if (r <= j) continue;
        const T lr = vec[r];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = 4 * tj + v;
          if (c > j && c <= r) t[u][v] -= lr * vec[c];
        }
        if (ti == tj) diag[r] = t[u][u];
      }
    }
    __syncthreads();
  }
  // ---- X = L^-1 (right-looking): publish row j of X scaled by 1/L_jj, update rows below
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) t[u][v] = T((4 * ti + u) == (4 * tj + v) ? 1 : 0);
  for (int j = 0; j < NB; ++j) {
    const T rl = T(1) / lb[j][j];
    if (ti == (j >> 2) && 4 * tj <= j) {
      const int jj = j & 3;
#pragma unroll
      for (int uu = 0; uu < 4; ++uu) {
        if (uu != jj) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = 4 * tj + v;
          if (c <= j) {
            t[uu][v] *= rl;
            vec[c] = t[uu][v];
          }
        }
      }
    }
    __syncthreads();
    if (ti >= (j >> 2) && 4 * tj <= j) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = 4 * ti + u;
        if (r <= j) continue;
        const T lr = lb[r][j];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = 4 * tj + v;
          if (c <= j) t[u][v] -= lr * vec[c];
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = 4 * ti + u, c = 4 * tj + v;
      xb[r][c] = (c <= r) ? t[u][v] : T(0);
    }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int e = tid; e < NB * NB; e += 256) {
      const int r = e / NB, c = e % NB;
      if (r < nb && c < nb) {
        if (c <= r) a[(k0 + r) * n + k0 + c] = lb[r][c];
        dinv[r * NB + c] = xb[r][c];
      }
    }
    if (tid == 0 && bad) atomicOr(flag, kFlagNotPD);
    return;
  }
  // ---- panel slice: out[r][c] = sum_k P[r][k] * X[c][k]
  T acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
  for (int k = 0; k < NB; ++k) {
    T pv[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) pv[u] = ps[4 * ti + u][k];
#pragma unroll
    for (int v = 0; v < 4; ++v) xv[v] = xb[4 * tj + v][k];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] += pv[u] * xv[v];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = 4 * ti + u, c = 4 * tj + v;
      if (r < pr && c < nb) a[(r0 + r) * n + k0 + c] = acc[u][v];
    }
}

// X = blockdiag(dinv_k), zero elsewhere (lower block triangle is filled by the doubling)
template <typename T>
__global__ void init_inverse_kernel(T* x, long long n, const T* __restrict__ dinv) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e % n;
    const long long br = r / NB, bc = c / NB;
    x[e] = (br == bc) ? dinv[br * NB * NB + (r % NB) * NB + (c % NB)] : T(0);
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

template <typename T>
constexpr int panel_smem() {
  return (3 * NB * (NB + 1) + 2 * NB) * int(sizeof(T));
}

}  // namespace

template <typename T>
void launch_build_factor_input(const float* h, long long n, const int32_t* order, double percdamp,
                               T* a, double* damp, cudaStream_t st) {
  count_launches(2);
  damp_kernel<<<1, 1024, 0, st>>>(h, n, percdamp, damp);
  build_input_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(h, n, order, damp, a);
}

// ws layout: [nblk*NB*NB dinv blocks][n*n scratch]
template <typename T>
void factor_upper_inverse(T* a, long long n, T* u, T* ws, unsigned* flag, cudaStream_t st,
                          cudaEvent_t mid) {
  static const bool attr = [] {
    cudaFuncSetAttribute(panel_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         panel_smem<T>());
    return true;
  }();
  (void)attr;
  const long long nblk = (n + NB - 1) / NB;
  T* dinv = ws;
  T* tmp = ws + nblk * NB * NB;
  // ---- Cholesky: fused panel kernel + trailing SYRK per 64 columns
  for (long long kb = 0; kb < nblk; ++kb) {
    const long long k0 = kb * NB, w = std::min<long long>(NB, n - k0), rest = n - k0 - w;
    count_launches(1);
    panel_kernel<T><<<unsigned(1 + (rest + NB - 1) / NB), 256, panel_smem<T>(), st>>>(
        a, n, k0, dinv + kb * NB * NB, flag);
    if (rest > 0)
      mm<T>(rest, rest, w, -1.0, a + (k0 + w) * n + k0, n, false, a + (k0 + w) * n + k0, n, true,
            1.0, a + (k0 + w) * n + (k0 + w), n, true, st);
  }
  if (mid) cudaEventRecord(mid, st);
  // ---- X = L^-1 by recursive doubling over the diagonal blocks (in u)
  T* x = u;
  count_launches(2);
  init_inverse_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(x, n, dinv);
  for (long long s = 2 * NB; s < 2 * n; s *= 2) {
    const long long h = s / 2;
    const long long full = n / s;  // pairs with a full-size second half
    // batched full pairs: base row/col p*s; A-block [p*s, p*s+h), C-block [p*s+h, p*s+s)
    if (full > 0) {
      const long long stride = s * (n + 1);
      // tmp_p = L[C, A] * X[A, A]         (h x h x h)
      mm<T>(h, h, h, 1.0, a + h * n, n, false, x, n, false, 0.0, tmp, h, false, st, int(full),
            stride, stride, h * h);
      // X[C, A] = -X[C, C] * tmp_p         (h x h x h)
      mm<T>(h, h, h, -1.0, x + h * n + h, n, false, tmp, h, false, 0.0, x + h * n, n, false, st,
            int(full), stride, h * h, stride);
    }
    // a trailing partial pair: A-block [p0, p0+h), C-block [p0+h, n) with 0 < n-p0-h < h
    const long long p0 = full * s, c2 = n - p0 - h;
    if (c2 > 0) {
      mm<T>(c2, h, h, 1.0, a + (p0 + h) * n + p0, n, false, x + p0 * n + p0, n, false, 0.0, tmp, h,
            false, st);
      mm<T>(c2, h, c2, -1.0, x + (p0 + h) * n + (p0 + h), n, false, tmp, h, false, 0.0,
            x + (p0 + h) * n + p0, n, false, st);
    }
  }
  reverse_to_upper_kernel<T><<<blocks_for(n * n), 256, 0, st>>>(x, n, tmp);
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
template void factor_upper_inverse<float>(float*, long long, float*, float*, unsigned*,
                                          cudaStream_t, cudaEvent_t);
template void factor_upper_inverse<double>(double*, long long, double*, double*, unsigned*,
                                           cudaStream_t, cudaEvent_t);
template void launch_gram_upper<float>(const float*, long long, double*, cudaStream_t);
template void launch_gram_upper<double>(const double*, long long, double*, cudaStream_t);

}  // namespace ocwg
