// Internal launch interface between the C-ABI host layer (capi.cu) and the
// kernels.  All pointers are device pointers; all launches are async on
// `st`.  Nothing here is exported from libocwg.so.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ocwg {

// SM count of the CURRENT device (cached per device ordinal).
int device_sms();

// Kernel launches issued by this library (for the bench's gpu_launches claim).
void count_launches(unsigned long long n);
unsigned long long launches_issued();

// Device-side status word written by kernels (0 = ok).  Bits:
enum DevFlag : unsigned {
  kFlagNonFinite = 1u,     // calibrate_grids saw NaN/Inf   -> invalid_input
  kFlagNotPD = 2u,         // Cholesky pivot <= 0 / NaN     -> numeric_error
  kFlagEmptyGroup = 4u,    // never expected
};

// ---- grids / RTN / pack (quant.cu) -------------------------------------
// Per-group min/max -> (scale, zero), minmax or 100-candidate MSE search
// (quant.cpp:51-74, 96-140, 168-196).  W is rows x cols row-major fp32.
void launch_calibrate_grids(const float* w, long long rows, long long cols, long long ld,
                            const QCfg& c, int mse, float* scales, int32_t* zeros, unsigned* flag,
                            float* ws_minmax, cudaStream_t st);
// codes[i*cols+j] = quantize(w[i,j], grid(i,j)); optional w_hat (quant.cpp:198-210, 212-218)
void launch_quantize_rtn(const float* w, long long rows, long long cols, long long ld,
                         const QCfg& c,
                         const float* scales, const int32_t* zeros, int16_t* codes,
                         float* w_hat, cudaStream_t st);
void launch_dequantize(const int16_t* codes, long long rows, long long cols, const QCfg& c,
                       const float* scales, const int32_t* zeros, float* out, cudaStream_t st);
// OCW1 uniform payload (container.cpp:15-35, 66-70, 129-139)
void launch_pack(const int16_t* codes, long long n_codes, long long n_groups, const QCfg& c,
                 const float* scales, const int32_t* zeros, uint8_t* out, cudaStream_t st);
void launch_unpack(const uint8_t* payload, long long n_codes, long long n_groups, const QCfg& c,
                   int16_t* codes, float* scales, int32_t* zeros, cudaStream_t st);
// act-order: stable descending sort of diag(H) (layerwise.cpp:11-18); `diag`
// is a contiguous copy of diag(H) (launch_damp writes one; unused without act-order)
void launch_order(const float* diag, long long n, int actorder, int32_t* order, cudaStream_t st);
// AutoBit candidate grid (autobit.cpp:45-61): out[14] = RTN errors of bits
// {2..8} x {per_group 128, per_channel}, symmetric; partial: rows x 14 doubles
void launch_candidate_grid(const float* w, long long rows, long long cols, long long ld, int act,
                           const double* in_diag, double* partial, double* out, unsigned* flag,
                           cudaStream_t st);

// ---- factorisation (factor.cu), T = float (default) or double ---------------
// A = reversed-permuted, dampened copy of H (layerwise.cpp:31-41):
//   A[i][j] = T(double(H[o(i)][o(j)]) + (i==j) * damp),  o(i) = order[n-1-i]
// damp = percdamp * mean(diag(double(H))) computed on device into *damp
// (layerwise.cpp:32-33); with diag != nullptr the kernel also stores diag(H)
// there contiguously (n floats) for launch_order.
void launch_damp(const float* h, long long n, double percdamp, double* damp, float* diag,
                 cudaStream_t st);
// damp_ready: *damp was already written by launch_damp on the same stream.
template <typename T>
void launch_build_factor_input(const float* h, long long n, const int32_t* order,
                               double percdamp, T* a, double* damp, cudaStream_t st,
                               bool damp_ready = false);
// In-place lower Cholesky A = L L^T (n x n row-major, lower used) by the
// persistent tile-dataflow kernel, over macro panels of `macro_cols` columns
// (<= 0: one panel) with a trailing SYRK (mm<T>) between panels.  Emits
// G[k][i] = L[n-1-i][n-1-k] / L[n-1-k][n-1-k] (i < k) for the sweep into ghi
// (+ glo: tf32 hi/lo split when non-null, T = float, with the plain value in
// gpl; gtt (optional): the diagonal 128 x 128 blocks of G^T, n x 128 fp32, in
// the in-block kernel's lane order (gp_pos in factor.cu)).  flags: ints
// from cholesky_flag_ints(n).  Sets kFlagNotPD in *status on breakdown.
size_t cholesky_flag_ints(long long n);
template <typename T>
void cholesky_g(T* a, long long n, T* ghi, float* glo, float* gpl, float* gtt, int* flags,
                unsigned* status, long long macro_cols, cudaStream_t st, float* lhi = nullptr,
                float* llo = nullptr);
// (fp32, n % 4 == 0: lhi / llo, n x n each, receive the tf32 hi / lo split of
// every published L tile, and the workers' tile products run on tcgen05)
// X = L^-1 (n x n lower) from the Cholesky factor; ws as upper_from_cholesky.
template <typename T>
void lower_inverse(const T* a, long long n, T* x, T* ws, cudaStream_t st);
// U = (J L J)^-1 (n x n upper, processing order) from the Cholesky factor:
// parity artefacts only.  ws: ceil(n/64)*64*64 + n*n elements.
template <typename T>
void upper_from_cholesky(const T* a, long long n, T* u, T* ws, cudaStream_t st);
// hinv = U^T U in fp64 (parity artefact: (H_p + damp I)^-1 in processing order)
template <typename T>
void launch_gram_upper(const T* u, long long n, double* hinv, cudaStream_t st);

// ---- SIMT GEMM (gemm.cu) ---------------------------------------------------
// C[m x n] = beta*C + alpha * op(A) * op(B); op(A)[i][k] = A[i*lda + k] or
// (transA) A[k*lda + i]; same for B.  lower_only: skip output tiles strictly
// above the diagonal.  Compute type T; A/B element types TA/TB.  Batched
// form: batch b uses A + b*sa, B + b*sb, C + b*sc.
template <typename T, typename TA, typename TB>
void gemm(long long m, long long n, long long k, double alpha, const TA* a, long long lda,
          bool ta, const TB* b, long long ldb, bool tb, double beta, T* c, long long ldc,
          bool lower_only, cudaStream_t st, int batch = 1, long long sa = 0, long long sb = 0,
          long long sc = 0, int tri = 0);
// (tri, fp64 tensor-core path: op(A) is lower (1) / upper (2) triangular and the
// k range that multiplies its zeros is skipped)

// ---- tensor-core fp32-accurate GEMM (tc_gemm.cu): 3xTF32 on tcgen05 ---------
size_t tc_gemm_workspace_floats(long long m, long long n, long long k, int batch = 1);
bool tc_gemm_tf32x3(int batch, long long m, long long n, long long k, float alpha, const float* a,
                    long long lda, long long sa, bool ta, const float* b, long long ldb,
                    long long sb, bool tb, float beta, float* c, long long ldc, long long sc,
                    bool lower_only, float* ws, size_t ws_floats, cudaStream_t st);
// Workspace for the fp32 GEMMs of the factorisation / sweep (set by the C ABI
// per call).  With a workspace set, fp32 GEMMs run on the tensor cores.
void set_tc_workspace(float* ws, size_t floats);
// Pre-split K-major operands: C = beta C + alpha (a_hi+a_lo)(b_hi+b_lo)^T, A m x k,
// B n x k.  Returns false when the shape/alignment needs another path.
bool tc_gemm_presplit(long long m, long long n, long long k, float alpha, const float* a_hi,
                      const float* a_lo, long long lda, const float* b_hi, const float* b_lo,
                      long long ldb, float beta, float* c, long long ldc, cudaStream_t st,
                      int max_ctas = 0, bool pdl = false);
// The same product on 2-SM pairs (cta_group::2, 256 x 256 tiles, tc_gemm2.cu):
// half the per-SM operand traffic; false if unsupported (caller falls back).
bool tc_gemm2_presplit(long long m, long long n, long long k, float alpha, const float* a_hi,
                       const float* a_lo, long long lda, const float* b_hi, const float* b_lo,
                       long long ldb, float beta, float* c, long long ldc, cudaStream_t st,
                       bool pdl = false, int ksplit = 1, int* kflag = nullptr, int epoch = 0);
// (ksplit <= 4: K parts of a tile on different pairs, each adding to the previous
// part's store in order; kflag: 2 ints per 256 x 256 tile, below 4 epoch + 1
// before the launch -- zero them once, then pass increasing epochs >= 1)
// pdl: launched as a programmatic dependent of the previous kernel on st (the
// kernel's setup overlaps that kernel's tail; its loads wait in griddepcontrol)
// Dispatch: T = float -> tcgen05 3xTF32 (when a workspace is set and the
// problem is big enough to fill tiles), else SIMT.
template <typename T>
void mm(long long m, long long n, long long k, double alpha, const T* a, long long lda, bool ta,
        const T* b, long long ldb, bool tb, double beta, T* c, long long ldc, bool lower_only,
        cudaStream_t st, int batch = 1, long long sa = 0, long long sb = 0, long long sc = 0);

// ---- GPTQ sweep (sweep.cu) ---------------------------------------------
constexpr long long kMaxSweepBlock = 128;
// D buffer elements per block parity (m x 128, K-major)
size_t sweep_delta_elems(long long m);
// Closed-form sweep over G (factor.cu).  w: original W (row stride ldw);
// gpl: plain G (in-block staging), ghi/glo: the GEMM operand (glo null =
// plain, SIMT GEMM); codes / w_hat written with row stride ldo in original row
// order; acc: n x m scratch; dpl/dhi/dlo: two D buffers each (plain; tf32
// hi/lo when glo != null); aux: second stream for the trailing GEMMs;
// ev: 5 events (fork, in-block, trailing x2, join).
template <typename T>
void gptq_sweep_g(const float* w, long long ldw, long long n, long long m, const T* gpl,
                  const float* gtt, const T* ghi, const float* glo, const int32_t* order, const QCfg& c,
                  const float* scales, const int32_t* zeros, long long block, int16_t* codes,
                  float* w_hat, long long ldo, T* acc, T* const dpl[2], float* const dhi[2],
                  float* const dlo[2], int* kflag, cudaStream_t st, void* tab = nullptr,
                  cudaStream_t aux = nullptr, cudaEvent_t* ev = nullptr);
// (tab: sweep_table_bytes(m), one super-block's {w, s, 1/s, z} table, built on
// `aux` beside each trailing GEMM with the two events ev[0..1])
size_t sweep_table_bytes(long long m);
// fp32 pre-split path (kflag != null): left-looking sweep, D of every row kept:
// dpl[0] / dhi[0] / dlo[0] are m x n K-major (ld n); kflag: sweep_kflag_ints.
size_t sweep_kflag_ints(long long n, long long m);

// ---- statistics (gram_tc.cu, stats.cu) ------------------------------------
// Tensor-core statistics: gram (+)= sum_s ops[gA[s]]^T ops[gB[s]] (symmetric
// operand set; upper tiles computed, mirrored) and cross (+)= sum_s
// ops[cA[s]]^T ops[cB[s]] (full).  Operands: tokens x dim bf16, row stride ld
// (ld % 8 == 0, >= dim).  Outputs dim x dim row-major, fp32 or (f64) fp64.
struct GramSpec {
  long long tokens = 0, dim = 0, ld = 0;
  const uint16_t* ops[4] = {};
  int nops = 0;
  int gseg = 0, gA[3] = {}, gB[3] = {};
  int cseg = 0, cA[3] = {}, cB[3] = {};
  void* gram = nullptr;
  void* cross = nullptr;
  bool f64 = false, accumulate = false;
  long long window_tokens = 0;  // max tokens per TMEM accumulation (0: 16384)
};
size_t gram_tc_workspace_bytes(long long dim);
// 0 ok, -1 unsupported shape, -2 workspace too small, > 0 CUDA error
int gram_tc(const GramSpec& s, void* ws, size_t ws_bytes, cudaStream_t st);
// bf16 X (tokens x dim, row-major, dim % 8 == 0) -> H (dim x dim fp32,
// symmetric, full); accumulate: H += X^T X else H = X^T X.
size_t hessian_tc_workspace_bytes(long long tokens, long long dim);
int hessian_tc(const uint16_t* x, long long tokens, long long dim, float* h, int accumulate,
               void* ws, size_t ws_bytes, cudaStream_t st);
// SIMT cross-check kernel (same contract as hessian_tc), used by tests only.
void hessian_simt(const uint16_t* x, long long tokens, long long dim, float* h, int accumulate,
                  cudaStream_t st);
// bf16 rows (rows x dim) -> rows x ld with zero pad columns (TMA needs ld % 8 == 0)
void launch_pad_bf16(const uint16_t* x, long long rows, long long dim, long long ld, uint16_t* out,
                     cudaStream_t st);
// fp32 -> bf16 parts for the tensor-core statistics (rows x ld, pad columns 0):
//   p1 = bf16(xp), p2 = bf16(xp - p1);  (xf != null) d = fp64(xf) - fp64(xp),
//   d1 = bf16(d), d2 = bf16(d - d1).  *flags |= 1 when some p2 != 0 (xp not
//   bf16-exact), 2 when some d != 0.
void launch_split_bf16(const float* xp, const float* xf, long long rows, long long dim, long long ld,
                       uint16_t* p1, uint16_t* p2, uint16_t* d1, uint16_t* d2, unsigned* flags,
                       cudaStream_t st);
// fp64 accumulate_stats for fp32 inputs on the FP64 pipe (OCWG_FP64 precision):
// gram += Xp^T Xp, cross += Xp^T (Xf - Xp).  diff_ws: rows*dim doubles.
void accumulate_stats_f64(const float* x_fp, const float* x_pert, long long rows, long long dim,
                          double* gram, double* cross, double* diff_ws, cudaStream_t st);
// out[i] += in[i] (fp32 -> fp64), n elements
void launch_add_f32_to_f64(const float* in, long long n, double* out, cudaStream_t st);

// ---- QEP target correction (qep.cu), fp64 -----------------------------------
size_t qep_workspace_doubles(long long n, long long m);
// out = W + alpha (gram + eta*mean(diag gram) I)^-1 (cross W); flags: Cholesky flags
void qep_target_f64(const float* w, const double* gram, const double* cross, long long n,
                    long long m, double alpha, double eta, float* out, double* ws, int* flags,
                    unsigned* status, cudaStream_t st);

// ---- seeded synthetic inputs (synth.cu) ------------------------
// kind 0: bf16(g * col_scale[c]) (col_scale may be null: 1); kind 1: bf16(silu(a) * b);
// kind 2: fp32 value of bf16(g * stddev).  g: Philox4x32-10 + Box-Muller normals.
void launch_synth(int kind, unsigned long long seed, long long rows, long long cols, float stddev,
                  const float* col_scale, void* out, int max_ctas, cudaStream_t st);

// ---- debug micro-benchmarks -------------------------------------------------
void debug_factor_bench(int iters, long long* cycles, float* out, cudaStream_t st);
int debug_sweep_trace(unsigned long long* out, int cap);

// ---- misc ----------------------------------------------------------------
void launch_f64_to_f32(const double* in, long long n, float* out, cudaStream_t st);
void launch_f32_to_f64(const float* in, long long n, double* out, cudaStream_t st);
// objective: sum_ij D[i][j] * (H D)[i][j], D = w_hat - w (quant.cpp:230-236)
void activation_objective(const float* w, const float* w_hat, const float* h, long long n,
                          long long m, double* out_dev, double* ws, cudaStream_t st);


// ---- JointQ refiner (jointq.cu; jointq.cpp:60-255) -------------------------
// independent search units: column blocks (per_group) or one (per_channel / per_tensor)
size_t jointq_units(const QCfg& c, long long m);
// E = double(s (code - z)) - double(W)
void jointq_residual(const int16_t* codes, const float* scales, const int32_t* zeros,
                     const float* w, long long n, long long m, const QCfg& c, double* e,
                     cudaStream_t st);
// H_eff = X^T X + tokens lambda I, E = What - W, G = H_eff E (fp64, device); returns J at
// entry.  part: 256 doubles of scratch.
double jointq_setup(const float* x, long long tokens, const float* w, long long n, long long m,
                    const QCfg& c, const int16_t* codes, const float* scales, const int32_t* zeros,
                    double lambda, double* h, double* e, double* g, double* part, cudaStream_t st);
// the local search (codes / scales / zeros refined in place); per unit: log of
// (key, objective change) of the first log_cap accepted moves, the count, and the
// first pass without a move.  dbuf: units * max_cells doubles.
int jointq_search(const float* w, long long n, long long m, const QCfg& c, int16_t* codes,
                  float* scales, int32_t* zeros, const double* h, double* e, double* g,
                  double* dbuf, long long max_cells, double obj0, int max_passes, int radius,
                  unsigned long long* log_key, double* log_delta, int* log_count, int* first_zero,
                  long long log_cap, cudaStream_t st);
double jointq_optimal_scale(const float* w, long long n, long long m, const QCfg& c,
                            const int16_t* codes, const float* scales, const int32_t* zeros,
                            const double* h, double* e, double* g, long long group, double* out,
                            cudaStream_t st);
// ||X E||^2 + tokens lambda ||E||^2 (X in token chunks; y: chunk * m doubles)
double jointq_objective_dev(const float* x, long long tokens, long long n, long long m,
                            const double* e, double lambda, double* y, long long chunk, double* part,
                            cudaStream_t st);

// in-place transpose of an n x n fp64 matrix (column-major caller statistics)
void transpose_sq_f64(double* a, long long n, cudaStream_t st);

}  // namespace ocwg
