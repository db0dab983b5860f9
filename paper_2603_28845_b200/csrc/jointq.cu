// JointQ refiner on the GPU (replaces jointq.cpp:60-255): a
// local search over integer codes, group scales and (asymmetric) zero points
// against the regularised activation objective
//   J = ||X What - X W||_F^2 + n lambda ||What - W||_F^2 = sum_j e_j^T H e_j,
//   H = X^T X + n lambda I,  E = What - W  (n = calibration rows of X).
//
// Structure of the search (jointq.cpp:187-252): per pass, (A) a scale refit of
// every group, (B) +-1..+-radius code moves in row-major order, (C) +-1
// zero-point moves (asymmetric); a move is accepted on strict improvement and
// applied at once (E and G = H E updated), so proposals are sequential.  Two
// groups only interact through the columns they share: with per-group
// granularity (groups along a row's columns) every 'column block' of
// group_size columns is an independent search -- its proposals read and its
// moves write only its own columns of E and G.  One CTA runs one block
// (per-channel / per-tensor grids couple all columns: one CTA runs all):
//   * warp 0 evaluates proposals (optimal scale = -num/den over the group's
//     cells, fp16 rounding, objective change) with per-lane partial sums and
//     butterfly reductions -- ~0.2 us per proposal;
//   * an accepted move wakes the whole CTA (named barriers) to apply it: the
//     cells' new residuals, then G[:, j] += H[:, i] d_ij over all n rows
//     (coalesced row segments, fp64 multiply-then-add as the reference's
//     Eigen column update, no FMA contraction).
// Each accepted move is logged with its key (pass, phase, index in the
// reference's global order); the host sorts the logs of all blocks into the
// reference's objective trace.  Deviation, documented: the acceptance
// threshold 1e-10 (1 + |J|) uses the block's own running J (J at entry plus
// the block's accepted changes) instead of the global running J, and sums run
// in a different order than the reference's sequential loops (fp64 rounding).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace ocwg {
namespace {

struct JqArgs {
  const double* h;  // n x n H_eff, row-major; column i read as h[k n + i] (jointq.cpp:163)
  double* e;        // n x m: dequantized - w
  double* g;        // n x m: H_eff e
  const float* w;   // n x m
  int16_t* codes;   // n x m
  float* scales;    // per group
  int32_t* zeros;   // per group
  double* dbuf;     // per unit: max_cells residual changes of the move being applied
  long long n, m, max_cells;
  QCfg c;
  int max_passes, radius;
  double tol;       // jointq.cpp:183
  double obj0;      // J at entry
  unsigned long long* log_key;  // per unit: log_cap entries
  double* log_delta;
  int* log_count;   // per unit accepted moves (the log keeps the first log_cap)
  int* first_zero;  // per unit: first pass without an accepted move (max_passes: none)
  long long log_cap;
  unsigned long long* prof;  // debug: unit 0's cycles per phase (null: off)
};

struct Cells {  // rows [r0, r1) x columns [j0, j1) (jointq.cpp:18-40)
  long long r0, r1, j0, j1;
};
__device__ __forceinline__ Cells cells_of(const JqArgs& a, long long group) {
  Cells x;
  if (a.c.gran == 0) {
    x.r0 = 0, x.r1 = a.n, x.j0 = 0, x.j1 = a.m;
  } else if (a.c.gran == 1) {
    x.r0 = group, x.r1 = group + 1, x.j0 = 0, x.j1 = a.m;
  } else {
    x.r0 = group / a.c.gpr, x.r1 = x.r0 + 1;
    x.j0 = (group % a.c.gpr) * a.c.group, x.j1 = min(a.m, x.j0 + a.c.group);
  }
  return x;
}

struct Prop {  // the code function of a proposal: the current codes, one cell replaced
  long long mi, mj;
  int mc;
};
__device__ __forceinline__ int code_at(const JqArgs& a, const Prop& p, long long i, long long j) {
  return (i == p.mi && j == p.mj) ? p.mc : int(a.codes[i * a.m + j]);
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// residual of cell (i, j) under (s, code function, z): s (code - z) - w (jointq.cpp:134)
__device__ __forceinline__ double fresh_at(const JqArgs& a, const Prop& p, long long i, long long j,
                                           float s, int z) {
  return __dsub_rn(__dmul_rn(double(s), double(code_at(a, p, i, j) - z)), double(a.w[i * a.m + j]));
}

// optimal group scale for fixed codes (jointq.cpp:92-118); warp-wide
__device__ double opt_scale(const JqArgs& a, const Cells& cl, const Prop& p, int z) {
  const int lane = threadIdx.x & 31;
  const long long nr = cl.r1 - cl.r0, ncell = nr * (cl.j1 - cl.j0);
  double num = 0.0, den = 0.0;
  for (long long q = lane; q < ncell; q += 32) {
    const long long j = cl.j0 + q / nr, i = cl.r0 + q % nr;
    const double cc = double(code_at(a, p, i, j) - z);
    if (cc == 0.0) continue;
    double hf = a.g[i * a.m + j];
    double dn = 0.0;
    for (long long k = cl.r0; k < cl.r1; ++k) {
      const double hik = a.h[i * a.n + k];
      const double what = __dadd_rn(a.e[k * a.m + j], double(a.w[k * a.m + j]));
      hf = __dsub_rn(hf, __dmul_rn(hik, what));
      dn = __dadd_rn(dn, __dmul_rn(__dmul_rn(cc, hik), double(code_at(a, p, k, j) - z)));
    }
    num = __dadd_rn(num, __dmul_rn(cc, hf));
    den = __dadd_rn(den, dn);
  }
  num = warp_sum(num);
  den = warp_sum(den);
  if (den <= 0.0) return 0.0;
  return -num / den;
}

// objective change for the group's cells at (s, codes, z) (jointq.cpp:122-141); warp-wide
__device__ double delta_for(const JqArgs& a, const Cells& cl, const Prop& p, float s, int z) {
  const int lane = threadIdx.x & 31;
  const long long nr = cl.r1 - cl.r0, ncell = nr * (cl.j1 - cl.j0);
  double delta = 0.0;
  for (long long q = lane; q < ncell; q += 32) {
    const long long j = cl.j0 + q / nr, i = cl.r0 + q % nr;
    const double d = __dsub_rn(fresh_at(a, p, i, j, s, z), a.e[i * a.m + j]);
    if (d == 0.0) continue;
    double t = __dmul_rn(__dmul_rn(2.0, d), a.g[i * a.m + j]);
    for (long long k = cl.r0; k < cl.r1; ++k) {
      const double dk = __dsub_rn(fresh_at(a, p, k, j, s, z), a.e[k * a.m + j]);
      if (dk != 0.0) t = __dadd_rn(t, __dmul_rn(__dmul_rn(d, a.h[i * a.n + k]), dk));
    }
    delta = __dadd_rn(delta, t);
  }
  return warp_sum(delta);
}

struct JqShared {
  int op;  // 1: apply the move below, 2: exit
  long long group;
  Prop p;
  float s;
  int z;
};

// apply the accepted move (jointq.cpp:144-158); all threads of the CTA
__device__ void apply_move(const JqArgs& a, const JqShared& sh, double* dbuf) {
  const Cells cl = cells_of(a, sh.group);
  const long long nr = cl.r1 - cl.r0, ncol = cl.j1 - cl.j0, ncell = nr * ncol;
  for (long long q = threadIdx.x; q < ncell; q += blockDim.x) {  // d of cell (row-major in j)
    const long long j = cl.j0 + q / nr, i = cl.r0 + q % nr;
    dbuf[q] = __dsub_rn(fresh_at(a, sh.p, i, j, sh.s, sh.z), a.e[i * a.m + j]);
  }
  __syncthreads();
  // G[k, j] += H[k, i] d_ij for the cells' rows i in order (the reference's
  // g.col(j) += h.col(i) * d, column by column)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (long long k = warp; k < a.n; k += nw) {
    double* gk = a.g + k * a.m;
    const double* hk = a.h + k * a.n;
    for (long long jj = lane; jj < ncol; jj += 32) {
      double acc = gk[cl.j0 + jj];
      for (long long r = 0; r < nr; ++r) {
        const double d = dbuf[jj * nr + r];
        if (d != 0.0) acc = __dadd_rn(acc, __dmul_rn(hk[cl.r0 + r], d));
      }
      gk[cl.j0 + jj] = acc;
    }
  }
  __syncthreads();
  for (long long q = threadIdx.x; q < ncell; q += blockDim.x) {
    const long long j = cl.j0 + q / nr, i = cl.r0 + q % nr;
    if (dbuf[q] != 0.0) a.e[i * a.m + j] = fresh_at(a, sh.p, i, j, sh.s, sh.z);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sh.p.mi >= 0) a.codes[sh.p.mi * a.m + sh.p.mj] = int16_t(sh.p.mc);
    a.scales[sh.group] = sh.s;
    a.zeros[sh.group] = sh.z;
  }
  __syncthreads();
}

__device__ __forceinline__ void bar_named(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(int(blockDim.x)) : "memory");
}

__global__ void __launch_bounds__(256) jq_search_kernel(JqArgs a) {
  __shared__ JqShared sh;
  const int unit = blockIdx.x;
  double* dbuf = a.dbuf + (long long)unit * a.max_cells;
  if (threadIdx.x >= 32) {  // helpers: apply each accepted move with warp 0
    while (true) {
      bar_named(1);
      if (sh.op == 2) return;
      apply_move(a, sh, dbuf);
      bar_named(2);
    }
  }
  const int lane = threadIdx.x;
  // the unit's groups and columns
  long long g_first, g_step, g_count, uj0, uj1;
  if (a.c.gran == 2) {
    g_first = unit, g_step = a.c.gpr, g_count = a.n;
    uj0 = (long long)unit * a.c.group, uj1 = min(a.m, uj0 + a.c.group);
  } else {
    g_first = 0, g_step = 1, g_count = a.c.gran == 1 ? a.n : 1;
    uj0 = 0, uj1 = a.m;
  }
  double obj = a.obj0;
  int accepted = 0;
  int fz = a.max_passes;
  auto try_move = [&](long long group, const Prop& p, int z, unsigned long long key) -> bool {
    const Cells cl = cells_of(a, group);
    const double raw = opt_scale(a, cl, p, z);
    float s_new = fp16_round(float(raw));
    if (!(s_new > 0.0f)) {
      if (raw > 0.0) s_new = kFp16MinPositive;
      else return false;
    }
    const double delta = delta_for(a, cl, p, s_new, z);
    if (delta >= -a.tol * (1.0 + fabs(obj))) return false;
    if (lane == 0) {
      sh.op = 1, sh.group = group, sh.p = p, sh.s = s_new, sh.z = z;
    }
    __syncwarp();
    bar_named(1);
    apply_move(a, sh, dbuf);
    bar_named(2);
    obj += delta;
    if (lane == 0) {
      if (accepted < a.log_cap) {
        a.log_key[(long long)unit * a.log_cap + accepted] = key;
        a.log_delta[(long long)unit * a.log_cap + accepted] = delta;
      }
    }
    ++accepted;
    return true;
  };
  const Prop none{-1, -1, 0};
  for (int pass = 0; pass < a.max_passes; ++pass) {
    const unsigned long long pk = (unsigned long long)pass << 58;
    int in_pass = 0;
    // (A) scale refits with the current codes (jointq.cpp:205-210)
    for (long long t = 0; t < g_count; ++t) {
      const long long group = g_first + t * g_step;
      if (try_move(group, none, a.zeros[group], pk | group)) ++in_pass;
    }
    // (B) code moves, row-major; deltas -1, +1, -2, +2, ... (jointq.cpp:211-230)
    for (long long i = 0; i < a.n; ++i) {
      for (long long j = uj0; j < uj1; ++j) {
        const long long group = group_of(a.c, i, j);
        const int cur = int(a.codes[i * a.m + j]);
        for (int r = 1; r <= a.radius; ++r) {
          bool done = false;
          for (int sg = -1; sg <= 1; sg += 2) {
            const int c_new = cur + sg * r;
            if (c_new < a.c.qmin || c_new > a.c.qmax) continue;
            if (try_move(group, Prop{i, j, c_new}, a.zeros[group],
                         pk | (1ull << 56) | (unsigned long long)(i * a.m + j))) {
              ++in_pass;
              done = true;
              break;
            }
          }
          if (done) break;
        }
      }
    }
    // (C) zero-point moves (asymmetric; jointq.cpp:232-246)
    if (a.c.scheme == 1) {
      for (long long t = 0; t < g_count; ++t) {
        const long long group = g_first + t * g_step;
        for (int dz = -1; dz <= 1; dz += 2) {
          const int z_new = a.zeros[group] + dz;
          if (z_new < a.c.qmin || z_new > a.c.qmax) continue;
          if (try_move(group, none, z_new, pk | (2ull << 56) | group)) {
            ++in_pass;
            break;
          }
        }
      }
    }
    if (in_pass == 0) {
      fz = pass;
      break;
    }
  }
  if (lane == 0) {
    a.log_count[unit] = accepted;
    a.first_zero[unit] = fz;
    sh.op = 2;
  }
  __syncwarp();
  bar_named(1);
}

// ---- per-group grids (one row per group, group_size <= 256): speculative
// parallel proposals.  A row's cells (g, e, w, codes, h_ii) sit in shared
// memory; every thread evaluates one proposal of the row against the current
// state, in the reference's own sequential order over the cells (the sums of
// jointq.cpp:92-141, so each proposal's numbers are those of the reference);
// the first accepted proposal in the reference's order (cell, then delta
// -1, +1, -2, ...) is applied, and the row's remaining proposals are
// re-evaluated against the new state.  Proposals before the first accepted
// one were rejected, so they saw exactly the state the sequential search
// would have shown them: the result equals the sequential search.
constexpr int kRowMax = 256;
struct RowSm {
  double g[kRowMax], e[kRowMax], d[kRowMax];
  float w[kRowMax];
  int c[kRowMax];
  double hii;
  int best;
  float s;
  double delta;
  int jp, cp, z;
};

// one proposal: code cp at column jp (jp < 0: none), zero point z
struct RowView {  // a row's cells in shared memory
  const double *g, *e;
  const float* w;
  const int* c;
  double hii;
};
__device__ bool eval_row_prop(const RowView& r, int ncol, int jp, int cp, int z, double thr, float& s_out,
                              double& delta_out) {
  // (branch-free: a skipped cell keeps the running sums by selection, so the
  // loads and products of the next cells issue ahead of the add chains)
  double num = 0.0, den = 0.0;  // jointq.cpp:95-118
#pragma unroll 8
  for (int j = 0; j < ncol; ++j) {
    const double cc = double((j == jp ? cp : r.c[j]) - z);
    const double what = __dadd_rn(r.e[j], double(r.w[j]));
    const double hf = __dsub_rn(r.g[j], __dmul_rn(r.hii, what));
    const double nn = __dadd_rn(num, __dmul_rn(cc, hf));
    const double dn = __dadd_rn(den, __dmul_rn(__dmul_rn(cc, r.hii), cc));
    num = cc != 0.0 ? nn : num;
    den = cc != 0.0 ? dn : den;
  }
  const double raw = den <= 0.0 ? 0.0 : -num / den;
  float s = fp16_round(float(raw));  // jointq.cpp:178-183
  if (!(s > 0.0f)) {
    if (raw > 0.0) s = kFp16MinPositive;
    else return false;
  }
  double delta = 0.0;  // jointq.cpp:122-141
#pragma unroll 8
  for (int j = 0; j < ncol; ++j) {
    const double fresh =
        __dsub_rn(__dmul_rn(double(s), double((j == jp ? cp : r.c[j]) - z)), double(r.w[j]));
    const double d = __dsub_rn(fresh, r.e[j]);
    const double t1 = __dadd_rn(delta, __dmul_rn(__dmul_rn(2.0, d), r.g[j]));
    const double t2 = __dadd_rn(t1, __dmul_rn(__dmul_rn(d, r.hii), d));
    delta = d != 0.0 ? t2 : delta;
  }
  s_out = s;
  delta_out = delta;
  return delta < thr;
}

// G is updated lazily: an accepted move's residual changes d (one row i_m)
// join a pending list; a row is materialised when loaded, and the whole
// column block is rewritten once per kPend moves.  Every element still gets
// its additions g += h(k, i_m) d_m(j) one at a time in move order (multiply,
// then add), so the values are those of the per-move update (jointq.cpp:142)
// with 1 / kPend of its memory traffic.
constexpr int kPend = 48;
constexpr int kSpec = 16;  // rows per speculative refit round (phases A and C)
__global__ void __launch_bounds__(256) jq_search_rows_kernel(JqArgs a) {
  __shared__ RowSm r;
  __shared__ int pend_i[kPend];
  __shared__ double pend_h[kPend];  // h(i, i_p) of the row being loaded
  __shared__ int npend;
  extern __shared__ double pend_d[];  // [kPend][ncol], then the speculative rows below
  const int unit = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const long long j0 = (long long)unit * a.c.group, j1 = min(a.m, j0 + a.c.group);
  const int ncol = int(j1 - j0);
  const int nd = 2 * a.radius;  // code deltas per cell: -1, +1, -2, +2, ...
  double obj = a.obj0;
  int accepted = 0, fz = a.max_passes;
  // kSpec rows for the speculative refits (phases A and C): g, e, w, codes, h_ii,
  // h(i, i_p) of the pending moves
  double* sp_g = pend_d + kPend * ncol;
  double* sp_e = sp_g + kSpec * ncol;
  double* sp_ph = sp_e + kSpec * ncol;  // [kSpec][kPend]
  double* sp_h = sp_ph + kSpec * kPend;
  float* sp_w = reinterpret_cast<float*>(sp_h + kSpec);
  int* sp_c = reinterpret_cast<int*>(sp_w + kSpec * ncol);
  if (tid == 0) npend = 0;
  __syncthreads();
  unsigned long long tph[6] = {0, 0, 0, 0, 0, 0};  // debug timers: A, B evals, B, C, rounds, flush
  auto clk = [] { return (unsigned long long)clock64(); };
  auto load = [&](long long i) {
    const int np = npend;
    if (tid < np) pend_h[tid] = a.h[i * a.n + pend_i[tid]];
    __syncthreads();
    for (int j = tid; j < ncol; j += nt) {
      const long long o = i * a.m + j0 + j;
      double gv = a.g[o];
      for (int p = 0; p < np; ++p) {
        const double dv = pend_d[p * ncol + j];
        if (dv != 0.0) gv = __dadd_rn(gv, __dmul_rn(pend_h[p], dv));
      }
      r.g[j] = gv;
      r.e[j] = a.e[o];
      r.w[j] = a.w[o];
      r.c[j] = a.codes[o];
    }
    if (tid == 0) r.hii = a.h[i * a.n + i];
    __syncthreads();
  };
  // rows i0 .. i0+R-1 into the speculative buffers (G materialised like load())
  auto load_spec = [&](long long i0, int R) {
    const int np = npend;
    for (int e = tid; e < R * kPend; e += nt) {
      const int q = e / kPend, p = e % kPend;
      if (p < np) sp_ph[q * kPend + p] = a.h[(i0 + q) * a.n + pend_i[p]];
    }
    if (tid < R) sp_h[tid] = a.h[(i0 + tid) * a.n + i0 + tid];
    __syncthreads();
    for (int e = tid; e < R * ncol; e += nt) {
      const int q = e / ncol, j = e % ncol;
      const long long o = (i0 + q) * a.m + j0 + j;
      double gv = a.g[o];
      for (int p = 0; p < np; ++p) {
        const double dv = pend_d[p * ncol + j];
        if (dv != 0.0) gv = __dadd_rn(gv, __dmul_rn(sp_ph[q * kPend + p], dv));
      }
      sp_g[q * ncol + j] = gv;
      sp_e[q * ncol + j] = a.e[o];
      sp_w[q * ncol + j] = a.w[o];
      sp_c[q * ncol + j] = a.codes[o];
    }
    __syncthreads();
  };
  auto spec_view = [&](int q) {
    return RowView{sp_g + q * ncol, sp_e + q * ncol, sp_w + q * ncol, sp_c + q * ncol, sp_h[q]};
  };
  auto flush = [&] {  // G[:, block] += the pending moves, in order
    // a warp takes kFR rows at a time: 4 kFR independent add chains per lane
    // (each element still adds its moves one at a time, in order), and every
    // pending d read from shared memory serves kFR rows
    constexpr int kFR = 8;
    const int np = npend;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (long long k0 = (long long)warp * kFR; k0 < a.n; k0 += (long long)nw * kFR) {
      for (int jb = 0; jb < ncol; jb += 128) {
        double gv[kFR][4], hl0[kFR], hl1[kFR];
#pragma unroll
        for (int q = 0; q < kFR; ++q) {
          const long long k = k0 + q;
          const bool kok = k < a.n;
          const double* hk = a.h + (kok ? k : 0) * a.n;
          hl0[q] = kok && lane < np ? hk[pend_i[lane]] : 0.0;
          hl1[q] = kok && lane + 32 < np ? hk[pend_i[lane + 32]] : 0.0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int j = jb + lane + 32 * t;
            gv[q][t] = (kok && j < ncol) ? a.g[k * a.m + j0 + j] : 0.0;
          }
        }
        for (int p = 0; p < np; ++p) {
          double dv[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int j = jb + lane + 32 * t;
            dv[t] = j < ncol ? pend_d[p * ncol + j] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < kFR; ++q) {
            const double hv = __shfl_sync(0xffffffffu, p < 32 ? hl0[q] : hl1[q], p & 31);
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (dv[t] != 0.0) gv[q][t] = __dadd_rn(gv[q][t], __dmul_rn(hv, dv[t]));
          }
        }
#pragma unroll
        for (int q = 0; q < kFR; ++q) {
          const long long k = k0 + q;
          if (k >= a.n) continue;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int j = jb + lane + 32 * t;
            if (j < ncol) a.g[k * a.m + j0 + j] = gv[q][t];
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) npend = 0;
    __syncthreads();
  };
  // apply the move in r (jointq.cpp:144-158): E now, G through the pending list
  auto apply = [&](long long i, long long group, unsigned long long key) {
    const int slot = npend;
    __syncthreads();  // (every thread has its slot before thread 0 advances npend)
    for (int j = tid; j < ncol; j += nt) {
      const double fresh = __dsub_rn(__dmul_rn(double(r.s), double((j == r.jp ? r.cp : r.c[j]) - r.z)),
                                     double(r.w[j]));
      const double d = __dsub_rn(fresh, r.e[j]);
      pend_d[slot * ncol + j] = d;
      if (d != 0.0) a.e[i * a.m + j0 + j] = fresh;
    }
    if (tid == 0) {
      pend_i[slot] = int(i);
      npend = slot + 1;
      if (r.jp >= 0) a.codes[i * a.m + j0 + r.jp] = int16_t(r.cp);
      a.scales[group] = r.s;
      a.zeros[group] = r.z;
      if (accepted < a.log_cap) {
        a.log_key[(long long)unit * a.log_cap + accepted] = key;
        a.log_delta[(long long)unit * a.log_cap + accepted] = r.delta;
      }
    }
    obj = __dadd_rn(obj, r.delta);
    ++accepted;
    __syncthreads();
    const unsigned long long tf = clk();
    if (npend == kPend) flush();
    tph[5] += clk() - tf;
    load(i);
  };
  auto thr_of = [&] { return __dmul_rn(-a.tol, __dadd_rn(1.0, fabs(obj))); };  // jointq.cpp:183
  auto rowv = [&] { return RowView{r.g, r.e, r.w, r.c, r.hii}; };
  for (int pass = 0; pass < a.max_passes; ++pass) {
    const unsigned long long pk = (unsigned long long)pass << 58;
    int in_pass = 0;
    unsigned long long tc0 = clk();
    // (A) scale refit of each row's group (jointq.cpp:205-210), one row at a time:
    // refits are accepted often, so evaluating rows ahead mostly repeats work
    // (measured: kSpec-row rounds took phase A from 1.5 to 2.5 G cycles at C2)
    for (long long i = 0; i < a.n; ++i) {
      const long long group = i * a.c.gpr + unit;
      load(i);
      if (tid == 0) {
        float s;
        double dl;
        r.best = eval_row_prop(rowv(), ncol, -1, 0, a.zeros[group], thr_of(), s, dl) ? 0 : -1;
        r.s = s, r.delta = dl, r.jp = -1, r.cp = 0, r.z = a.zeros[group];
      }
      __syncthreads();
      if (r.best == 0) {
        apply(i, group, pk | (unsigned long long)group);
        ++in_pass;
      }
      __syncthreads();
    }
    tph[0] += clk() - tc0;
    tc0 = clk();
    // (B) code moves in row-major order, speculatively in parallel (jointq.cpp:211-230)
    for (long long i = 0; i < a.n; ++i) {
      const long long group = i * a.c.gpr + unit;
      load(i);
      int start = 0;  // first cell still to try
      while (start < ncol) {
        const unsigned long long te = clk();
        if (tid == 0) r.best = 0x7fffffff;
        __syncthreads();
        const int z = a.zeros[group];
        const double thr = thr_of();
        for (int k = tid; k < (ncol - start) * nd; k += nt) {
          const int jp = start + k / nd, di = k % nd;
          const int cp = r.c[jp] + ((di & 1) ? 1 : -1) * (di / 2 + 1);
          if (cp < a.c.qmin || cp > a.c.qmax) continue;
          float s;
          double dl;
          if (eval_row_prop(rowv(), ncol, jp, cp, z, thr, s, dl)) atomicMin(&r.best, k);
        }
        __syncthreads();
        const int best = r.best;
        tph[1] += clk() - te;
        tph[4] += 1;
        if (best == 0x7fffffff) break;
        __syncthreads();
        if (tid == 0) {  // re-evaluate the winner for its (s, delta) (deterministic)
          const int jp = start + best / nd, di = best % nd;
          const int cp = r.c[jp] + ((di & 1) ? 1 : -1) * (di / 2 + 1);
          float s;
          double dl;
          eval_row_prop(rowv(), ncol, jp, cp, z, thr, s, dl);
          r.s = s, r.delta = dl, r.jp = jp, r.cp = cp, r.z = z;
        }
        __syncthreads();
        const int jp = r.jp;
        apply(i, group, pk | (1ull << 56) | (unsigned long long)(i * a.m + j0 + jp));
        ++in_pass;
        start = jp + 1;
      }
      __syncthreads();
    }
    tph[2] += clk() - tc0;
    tc0 = clk();
    // (C) zero-point moves (asymmetric; jointq.cpp:232-246)
    if (a.c.scheme == 1) {
      // kSpec rows x (z - 1, z + 1) at a time, first accepted in the reference's order
      // (zero moves are rarely accepted: C2 phase C 0.86 -> 0.13 G cycles)
      for (long long i0 = 0; i0 < a.n;) {
        const int R = int(min((long long)kSpec, a.n - i0));
        load_spec(i0, R);
        if (tid == 0) r.best = 0x7fffffff;
        __syncthreads();
        const double thr = thr_of();
        if (tid < 2 * R) {
          const int q = tid >> 1, dz = (tid & 1) ? 1 : -1;
          const long long group = (i0 + q) * a.c.gpr + unit;
          const int z_new = a.zeros[group] + dz;
          float s;
          double dl;
          if (z_new >= a.c.qmin && z_new <= a.c.qmax &&
              eval_row_prop(spec_view(q), ncol, -1, 0, z_new, thr, s, dl))
            atomicMin(&r.best, tid);
        }
        __syncthreads();
        const int best = r.best;
        if (best == 0x7fffffff) {
          i0 += R;
          continue;
        }
        const long long i = i0 + (best >> 1), group = i * a.c.gpr + unit;
        const int z_new = a.zeros[group] + ((best & 1) ? 1 : -1);
        load(i);
        if (tid == 0) {
          float s;
          double dl;
          eval_row_prop(rowv(), ncol, -1, 0, z_new, thr, s, dl);
          r.s = s, r.delta = dl, r.jp = -1, r.cp = 0, r.z = z_new;
        }
        __syncthreads();
        apply(i, group, pk | (2ull << 56) | (unsigned long long)group);
        ++in_pass;
        i0 = i + 1;
      }
    }
    tph[3] += clk() - tc0;
    if (in_pass == 0) {
      fz = pass;
      break;
    }
  }
  if (tid == 0) {
    a.log_count[unit] = accepted;
    a.first_zero[unit] = fz;
    if (a.prof && unit == 0)
      for (int q = 0; q < 6; ++q) a.prof[q] = tph[q];
  }
}

// e = double(s (code - z)) - double(w): the reference's to_eigen_d(dequantize(q)) - to_eigen_d(w)
__global__ void jq_residual_kernel(const int16_t* codes, const float* scales, const int32_t* zeros,
                                   const float* w, long long n, long long m, QCfg c, double* e) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n * m;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / m, j = t % m, gi = group_of(c, i, j);
    const float wh = __fmul_rn(scales[gi], float(int(codes[t]) - zeros[gi]));  // quant.cpp:33-35
    e[t] = double(wh) - double(w[t]);
  }
}
__global__ void jq_add_diag_kernel(double* h, long long n, double v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    h[i * n + i] += v;
}
// per-block partial sums of a[t] * b[t] (b null: a[t]^2), fixed order
__global__ void jq_dot_kernel(const double* a, const double* b, long long len, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < len;
       t += (long long)gridDim.x * blockDim.x)
    s += a[t] * (b ? b[t] : a[t]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void jq_opt_scale_kernel(JqArgs a, long long group, double* out) {
  const Prop none{-1, -1, 0};
  const double v = opt_scale(a, cells_of(a, group), none, a.zeros[group]);
  if (threadIdx.x == 0) *out = v;
}

constexpr int kDotBlocks = 256;
double dot(const double* x, const double* y, long long len, double* part, cudaStream_t st) {
  jq_dot_kernel<<<kDotBlocks, 256, 0, st>>>(x, y, len, part);
  count_launches(1);
  std::vector<double> h(kDotBlocks);
  cudaMemcpyAsync(h.data(), part, sizeof(double) * kDotBlocks, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}

}  // namespace

size_t jointq_units(const QCfg& c, long long m) { return c.gran == 2 ? size_t(c.gpr) : 1; }

void jointq_residual(const int16_t* codes, const float* scales, const int32_t* zeros,
                     const float* w, long long n, long long m, const QCfg& c, double* e,
                     cudaStream_t st) {
  jq_residual_kernel<<<592, 256, 0, st>>>(codes, scales, zeros, w, n, m, c, e);
  count_launches(1);
}

// H_eff, E, G on the device (jointq.cpp:64-73); returns J at entry.
double jointq_setup(const float* x, long long tokens, const float* w, long long n, long long m,
                    const QCfg& c, const int16_t* codes, const float* scales, const int32_t* zeros,
                    double lambda, double* h, double* e, double* g, double* part, cudaStream_t st) {
  if (tokens > 0)
    gemm<double, float, float>(n, n, tokens, 1.0, x, n, true, x, n, false, 0.0, h, n, false, st);
  else
    cudaMemsetAsync(h, 0, size_t(n) * size_t(n) * sizeof(double), st);
  jq_add_diag_kernel<<<64, 256, 0, st>>>(h, n, double(tokens) * lambda);
  count_launches(1);
  jointq_residual(codes, scales, zeros, w, n, m, c, e, st);
  gemm<double, double, double>(n, m, n, 1.0, h, n, false, e, m, false, 0.0, g, m, false, st);
  return dot(e, g, n * m, part, st);
}

int jointq_search(const float* w, long long n, long long m, const QCfg& c, int16_t* codes,
                  float* scales, int32_t* zeros, const double* h, double* e, double* g,
                  double* dbuf, long long max_cells, double obj0, int max_passes, int radius,
                  unsigned long long* log_key, double* log_delta, int* log_count, int* first_zero,
                  long long log_cap, cudaStream_t st) {
  JqArgs a{};
  a.h = h, a.e = e, a.g = g, a.w = w, a.codes = codes, a.scales = scales, a.zeros = zeros;
  a.dbuf = dbuf, a.n = n, a.m = m, a.max_cells = max_cells, a.c = c;
  a.max_passes = max_passes, a.radius = radius, a.tol = 1e-10, a.obj0 = obj0;
  a.log_key = log_key, a.log_delta = log_delta, a.log_count = log_count, a.first_zero = first_zero;
  a.log_cap = log_cap;
  static unsigned long long* prof = nullptr;
  if (getenv("OCWG_DEBUG_JQ")) {
    if (!prof) cudaMalloc(&prof, 6 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 6 * sizeof(unsigned long long), st);
    a.prof = prof;
  }
  const int units = int(jointq_units(c, m));
  if (c.gran == 2 && c.group <= kRowMax) {
    const int ncol = int(std::min<long long>(c.group, m));
    const size_t dyn = size_t(kPend) * ncol * sizeof(double) +                 // pending d
                       size_t(kSpec) * ncol * (2 * sizeof(double) + sizeof(float) + sizeof(int)) +
                       size_t(kSpec) * (kPend + 1) * sizeof(double);            // h(i, i_p), h_ii
    cudaFuncSetAttribute(jq_search_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
    jq_search_rows_kernel<<<units, 256, dyn, st>>>(a);
    if (a.prof) {
      unsigned long long h[6];
      cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      fprintf(stderr, "jointq unit 0 Mcycles: A %.1f, B %.1f (evals %.1f in %llu rounds), C %.1f, flush %.1f\n",
              h[0] / 1e6, h[2] / 1e6, h[1] / 1e6, h[4], h[3] / 1e6, h[5] / 1e6);
    }
  } else {
    jq_search_kernel<<<units, 256, 0, st>>>(a);
  }
  count_launches(1);
  return int(cudaGetLastError());
}

double jointq_optimal_scale(const float* w, long long n, long long m, const QCfg& c,
                            const int16_t* codes, const float* scales, const int32_t* zeros,
                            const double* h, double* e, double* g, long long group, double* out,
                            cudaStream_t st) {
  JqArgs a{};
  a.h = h, a.e = e, a.g = g, a.w = w, a.codes = const_cast<int16_t*>(codes);
  a.scales = const_cast<float*>(scales), a.zeros = const_cast<int32_t*>(zeros);
  a.n = n, a.m = m, a.c = c;
  jq_opt_scale_kernel<<<1, 32, 0, st>>>(a, group, out);
  count_launches(1);
  double v = 0.0;
  cudaMemcpyAsync(&v, out, sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return v;
}

// ||X D||^2 + tokens lambda ||D||^2, D = What - W (jointq.cpp:160-167), X in token chunks
double jointq_objective_dev(const float* x, long long tokens, long long n, long long m,
                            const double* e, double lambda, double* y, long long chunk, double* part,
                            cudaStream_t st) {
  double s = 0.0;
  for (long long t0 = 0; t0 < tokens; t0 += chunk) {
    const long long tl = std::min(chunk, tokens - t0);
    gemm<double, float, double>(tl, m, n, 1.0, x + t0 * n, n, false, e, m, false, 0.0, y, m, false,
                                st);
    s += dot(y, nullptr, tl * m, part, st);
  }
  return s + double(tokens) * lambda * dot(e, nullptr, n * m, part, st);
}

}  // namespace ocwg
