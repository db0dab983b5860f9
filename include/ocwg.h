/*
 * ocwg.h -- C ABI of the B200 (sm_100a) GPTQ layer-quantize library
 * (libocwg.so).  Drop-in boundary for the OneComp "ocw" reference's hot path.
 *
 * Every entry point replaces one reference C++ function of the layer-wise PTQ
 * path (citations are /root/reference/proj/...); the C++ drop-in
 * (paper_2603_28845_b200/cpp/ocw_dropin.cpp) re-exposes them under the
 * reference's own `ocw::` signatures, and the Python host mirror
 * (paper_2603_28845_b200/__init__.py) binds them with ctypes.
 *
 * Conventions
 *   - Orientation is the reference's: W is N x M with N = INPUT rows and
 *     M = OUTPUT columns (model.hpp:14); H is N x N; X is T x N (tokens x in).
 *     All matrices are dense row-major.
 *   - Status codes mirror the reference's exception classes and CLI exit codes
 *     (errors.hpp:9-21, ocw_cli.cpp:9-12): OCWG_INVALID_INPUT == invalid_input,
 *     OCWG_NUMERIC_ERROR == numeric_error; CUDA failures are >= 16.  No C++
 *     exception crosses the ABI; ocwg_last_error() holds the message
 *     (thread-local).
 *   - Host-pointer entry points are synchronous (value semantics, like the
 *     reference).  *_dev entry points take DEVICE pointers, run on the
 *     context's stream and return after the stream has drained (or, with
 *     ocwg_set_async, right after enqueueing).
 *   - Grids are passed structure-of-arrays: scales (fp32 value of the
 *     reference-fp16-rounded scale) and int32 zero points, in group-index order
 *     (QuantizedMatrix::grids, quant.hpp:54-63).  qmin/qmax follow from the config.
 *   - No CPU fallback: every compute entry point runs CUDA kernels; a missing
 *     or unusable GPU is reported as OCWG_CUDA_ERROR.
 */
#ifndef OCWG_H
#define OCWG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCWG_OK 0
#define OCWG_INVALID_INPUT 1 /* ocw::invalid_input */
#define OCWG_IO_ERROR 2      /* ocw::io_error      */
#define OCWG_NUMERIC_ERROR 3 /* ocw::numeric_error */
#define OCWG_CUDA_ERROR 16
#define OCWG_UNSUPPORTED 17

/* quant.hpp:12-14 */
#define OCWG_SYMMETRIC 0
#define OCWG_ASYMMETRIC 1
#define OCWG_PER_TENSOR 0
#define OCWG_PER_CHANNEL 1
#define OCWG_PER_GROUP 2
#define OCWG_MINMAX 0
#define OCWG_MSE_GRID 1

/* arithmetic of the factorisation + GPTQ sweep (the reference uses fp64,
 * layerwise.cpp:31-90; fp32 keeps >= 99.9 % identical codes -- 99.94-99.9997 % at the
 * BASELINE configs) */
#define OCWG_FP32 0
#define OCWG_FP64 1

/* layout of the fp64 statistics (gram / cross) host matrices taken and returned
 * by ocwg_accumulate_stats, ocwg_quantize_layer and ocwg_qep_target: row-major
 * (default) or column-major (an Eigen::MatrixXd's storage, CalibStats
 * stats.hpp:15-24 -- the C++ drop-in passes them without host-side copies) */
#define OCWG_ROW_MAJOR 0
#define OCWG_COL_MAJOR 1

/* QuantConfig (quant.hpp:21-28) */
typedef struct ocwg_quant_config {
  int32_t bits;        /* [1, 8] */
  int32_t scheme;      /* OCWG_SYMMETRIC / OCWG_ASYMMETRIC */
  int32_t granularity; /* OCWG_PER_TENSOR / _CHANNEL / _GROUP */
  int32_t reserved;
  uint64_t group_size; /* per_group only; short final group allowed */
} ocwg_quant_config;

/* GptqOptions (layerwise.hpp:11-15) */
typedef struct ocwg_gptq_options {
  int32_t actorder;    /* stable sort by descending diag(H) */
  int32_t reserved;
  double percdamp;     /* (0, 1] */
  uint64_t block_cols; /* lazy-update block (reference default 32) */
} ocwg_gptq_options;

typedef struct ocwg_ctx ocwg_ctx;

/* ---- library / context ------------------------------------------------ */
const char* ocwg_last_error(void);
int ocwg_version(void);
/* Context on one CUDA device: stream, workspace pool, device status word. */
int ocwg_create(int device, ocwg_ctx** out);
int ocwg_destroy(ocwg_ctx* ctx);
/* OCWG_FP32 (default, fast: tensor-core statistics, fp32 factorisation +
 * 3xTF32 sweep) or OCWG_FP64 (the reference's arithmetic class throughout). */
int ocwg_set_precision(ocwg_ctx* ctx, int precision);
int ocwg_set_stats_layout(ocwg_ctx* ctx, int layout);
/* Run subsequent work on an external cudaStream_t (NULL = the CUDA legacy
 * default stream).  A new context uses its own non-blocking stream. */
int ocwg_set_stream(ocwg_ctx* ctx, void* cuda_stream);
/* on != 0: *_dev entry points return as soon as their work is enqueued;
 * device-side errors (not positive definite, non-finite W) stay latched in the
 * context and are reported by the next ocwg_synchronize. */
int ocwg_set_async(ocwg_ctx* ctx, int on);
/* Drain the context's stream; returns the latched status of async calls. */
int ocwg_synchronize(ocwg_ctx* ctx);

/* ---- quant.hpp --------------------------------------------------------- */
/* QuantConfig::validate (quant.cpp:19-25) */
int ocwg_validate_config(const ocwg_quant_config* cfg);
/* quant_group_count (quant.cpp:151-154) */
uint64_t ocwg_group_count(const ocwg_quant_config* cfg, uint64_t rows, uint64_t cols);
/* uniform_storage_bytes (quant.cpp:220-224) */
uint64_t ocwg_storage_bytes(const ocwg_quant_config* cfg, uint64_t rows, uint64_t cols);
/* calibrate_grids (quant.cpp:168-196) */
int ocwg_calibrate_grids(ocwg_ctx* ctx, const float* w, uint64_t rows, uint64_t cols,
                         const ocwg_quant_config* cfg, int scale_mode, float* scales,
                         int32_t* zeros);
/* quantize_matrix (quant.cpp:198-210): codes int16 row-major */
/* AutoBit's default candidate grid (autobit.cpp:45-61 candidate_grid with
 * estimate_error :16-34): RTN error of W (rows x cols, host) under bits 2..8 x
 * {per_group 128, per_channel}, symmetric -- errors[14] / cost_bytes[14] in
 * the reference's order (bits ascending, grouped first), one pass over W on
 * the GPU.  mode 0 naive ||dW||^2; 1 act-aware 1/2 sum_ij in_diag[i] dW_ij^2
 * (in_diag: rows doubles, NULL = ones).  SURVEY §8 f3. */
int ocwg_candidate_grid(ocwg_ctx* ctx, const float* w, uint64_t rows, uint64_t cols, int mode,
                        const double* in_diag, double* errors, uint64_t* cost_bytes);
int ocwg_quantize_matrix(ocwg_ctx* ctx, const float* w, uint64_t rows, uint64_t cols,
                         const ocwg_quant_config* cfg, int scale_mode, int16_t* codes,
                         float* scales, int32_t* zeros);
/* dequantize (quant.cpp:212-218) */
int ocwg_dequantize(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                    const int32_t* zeros, uint64_t rows, uint64_t cols,
                    const ocwg_quant_config* cfg, float* out);
/* activation_objective (quant.cpp:230-236): tr((W_hat - W)^T H (W_hat - W)) */
int ocwg_activation_objective(ocwg_ctx* ctx, const float* w, const float* w_hat, const float* h,
                              uint64_t n, uint64_t m, double* out);

/* ---- OCW1 uniform payload (container.cpp:15-35, 66-70, 129-139, 168-199) */
/* out_len must be >= ocwg_storage_bytes(); exactly that many bytes are written */
int ocwg_pack_uniform(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                      const int32_t* zeros, uint64_t rows, uint64_t cols,
                      const ocwg_quant_config* cfg, uint8_t* out, uint64_t out_len);
int ocwg_unpack_uniform(ocwg_ctx* ctx, const uint8_t* payload, uint64_t len, uint64_t rows,
                        uint64_t cols, const ocwg_quant_config* cfg, int16_t* codes,
                        float* scales, int32_t* zeros);

/* ---- stats.hpp --------------------------------------------------------- */
/* accumulate_stats (stats.cpp:10-19): gram += Xp^T Xp; cross += Xp^T (X - Xp),
 * fp64 n x n row-major, updated in place; cross may be NULL when
 * x_fp == x_pert (then cross is identically 0, test_core.cpp:273-279).
 * OCWG_FP32 precision (default): tcgen05 tensor cores on bf16 parts of the
 * inputs (Xp = P1 + P2, X - Xp = D1 + D2; gram = P1'P1 + P1'P2 + P2'P1,
 * cross = P1'D1 + P1'D2 + P2'D1; fp32 accumulation per 8192 tokens, fp64
 * across), |dH_ij| <~ 1e-5 sqrt(H_ii H_jj).  OCWG_FP64: fp64 GEMMs (DMMA tensor cores). */
int ocwg_accumulate_stats(ocwg_ctx* ctx, const float* x_fp, const float* x_pert, uint64_t rows,
                          uint64_t dim, double* gram, double* cross, uint64_t* token_count);
/* Hessian of bf16 calibration tokens on the tensor cores: H (+)= X^T X.
 * x: T x N bf16 bits (uint16), h: N x N fp32.  (stats.cpp:16 for bf16 X) */
int ocwg_hessian_bf16(ocwg_ctx* ctx, const uint16_t* x, uint64_t tokens, uint64_t dim, float* h,
                      int accumulate);

/* ---- layerwise.hpp ----------------------------------------------------- */
/* gptq_order (layerwise.cpp:11-18) */
int ocwg_gptq_order(ocwg_ctx* ctx, const float* h, uint64_t n, int actorder, int64_t* order);
/* gptq_quantize (layerwise.cpp:20-93).  w_hat (N x M dequantized) may be NULL. */
int ocwg_gptq_quantize(ocwg_ctx* ctx, const float* w, const float* h, uint64_t n, uint64_t m,
                       const ocwg_quant_config* cfg, const ocwg_gptq_options* opts,
                       int scale_mode, int16_t* codes, float* scales, int32_t* zeros,
                       float* w_hat);
/* Parity artefacts of layerwise.cpp:29-51: processing order, damp, the
 * dampened permuted inverse hinv = H_p^-1 and its upper factor U (each
 * output may be NULL; hinv/u are N x N fp64 row-major, processing order). */
int ocwg_gptq_factor(ocwg_ctx* ctx, const float* h, uint64_t n, int actorder, double percdamp,
                     int64_t* order, double* hinv, double* u, double* damp);
/* qep_target (layerwise.cpp:95-112): out = W + alpha (gram + lambda I)^-1 (cross W),
 * lambda = eta * mean(diag(gram)); fp64 like the reference.  gram / cross:
 * N x N fp64 (CalibStats), W / out: N x M fp32 (out may alias W). */
int ocwg_qep_target(ocwg_ctx* ctx, const float* w, const double* gram, const double* cross,
                    uint64_t n, uint64_t m, double alpha, double eta, float* out);
/* QepOptions (layerwise.hpp:33-36) */
typedef struct ocwg_qep_options {
  double alpha; /* [0, 1] */
  double eta;   /* > 0 */
} ocwg_qep_options;
/* quantize_layer (layerwise.cpp:120-126) over fp64 CalibStats (gram, cross:
 * N x N), in one device round trip: [qep_target when qep != NULL] -> RTN
 * (method 0) or GPTQ (method 1) on fp32(gram).  cross may be NULL without
 * QEP.  w_hat (N x M dequantized) may be NULL. */
int ocwg_quantize_layer(ocwg_ctx* ctx, const float* w, const double* gram, const double* cross,
                        uint64_t n, uint64_t m, int method, const ocwg_quant_config* cfg,
                        const ocwg_gptq_options* opts, int scale_mode,
                        const ocwg_qep_options* qep, int16_t* codes, float* scales,
                        int32_t* zeros, float* w_hat);

/* ---- jointq.hpp (the format-preserving refiner of GPTQ output)
 * W is N x M (rows x cols, the QuantizedMatrix orientation), X is T x N fp32
 * (T calibration rows; X cols == W rows).  Objective (jointq.hpp:18-20):
 *   ||X What - X W||_F^2 + T lambda ||What - W||_F^2.
 * jointq_refine (jointq.cpp:169-255): codes / scales / zeros are read and
 * overwritten with the refined matrix (same format).  trace receives the
 * objective at entry and after each accepted move in the reference's move
 * order (first trace_cap entries; *trace_len = total entries, 0 if the move log
 * overflowed); *accepted_moves and *passes as JointqResult.  Searches of
 * independent column blocks (per-group grids) run concurrently, one CTA each;
 * the acceptance threshold uses the block's own running objective. */
int ocwg_jointq_refine(ocwg_ctx* ctx, const float* w, uint64_t n, uint64_t m, const float* x,
                       uint64_t tokens, const ocwg_quant_config* cfg, int16_t* codes,
                       float* scales, int32_t* zeros, double lambda, int max_passes,
                       int move_radius, double* trace, uint64_t trace_cap, uint64_t* trace_len,
                       uint64_t* accepted_moves, int* passes);
/* jointq_objective (jointq.cpp:160-167), fp64 */
int ocwg_jointq_objective(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                          const int32_t* zeros, const float* w, uint64_t n, uint64_t m,
                          const float* x, uint64_t tokens, const ocwg_quant_config* cfg,
                          double lambda, double* out);
/* jointq_optimal_group_scale (jointq.cpp:169-175): the 1-D optimum of one group's scale */
int ocwg_jointq_optimal_group_scale(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                                    const int32_t* zeros, const float* w, uint64_t n, uint64_t m,
                                    const float* x, uint64_t tokens, const ocwg_quant_config* cfg,
                                    double lambda, uint64_t group, double* out);

/* ---- end-to-end layer quantize from calibration tokens (north_star call) --
 * W (N x M fp32) + X (T x N bf16) -> codes, grids, dequantized W and the
 * packed OCW1 payload.  Any output may be NULL.  h_out (N x N fp32) returns
 * the Hessian X^T X (unnormalised, as stats.cpp:16). */
int ocwg_quantize_layer_x(ocwg_ctx* ctx, const float* w, const uint16_t* x, uint64_t tokens,
                          uint64_t n, uint64_t m, const ocwg_quant_config* cfg,
                          const ocwg_gptq_options* opts, int scale_mode, int16_t* codes,
                          float* scales, int32_t* zeros, float* w_hat, uint8_t* payload,
                          uint64_t payload_len, float* h_out);
/* ---- layers sharing one calibration input (the sweep
 * driver's q/k/v and gate/up groups, run_layerwise_sweep pipeline.cpp:215-226
 * and model.cpp:301-307) -- `count` weights W_i (N x M_i fp32, host) that see
 * the same X (T x N bf16, host): ONE Hessian, one order + factorisation (they
 * depend on H only, layerwise.cpp:31-51), then one grid + sweep + pack per W.
 * Results equal `count` separate ocwg_quantize_layer_x calls bit for bit.
 * Per-layer outputs codes[i] (N x M_i), scales[i], zeros[i], payload[i]
 * (payload_len[i] bytes); any output pointer may be NULL. */
int ocwg_quantize_layers_x(ocwg_ctx* ctx, int count, const float* const* w, const uint64_t* m,
                           const uint16_t* x, uint64_t tokens, uint64_t n,
                           const ocwg_quant_config* cfg, const ocwg_gptq_options* opts,
                           int scale_mode, int16_t* const* codes, float* const* scales,
                           int32_t* const* zeros, uint8_t* const* payload,
                           const uint64_t* payload_len);
/* ocwg_quantize_layers_x with every pointer in device memory (w, m and the
 * output pointer arrays themselves are host arrays of device pointers);
 * codes / scales / zeros required, payload[i] optional.  Async-capable. */
int ocwg_quantize_layers_x_dev(ocwg_ctx* ctx, int count, const float* const* w, const uint64_t* m,
                               const uint16_t* x, uint64_t tokens, uint64_t n,
                               const ocwg_quant_config* cfg, const ocwg_gptq_options* opts,
                               int scale_mode, int16_t* const* codes, float* const* scales,
                               int32_t* const* zeros, uint8_t* const* payload);
/* Seeded synthetic inputs on the device (counter-based
 * Philox4x32-10 + Box-Muller normals g, independent of launch shape):
 *   kind 0: out (bf16 bits, rows x cols) = bf16(g * col_scale[c]) (col_scale
 *           device fp32[cols], NULL = 1) -- calibration X with outlier channels;
 *   kind 1: out (bf16 bits) = bf16(silu(a) * b) -- down_proj calibration X;
 *   kind 2: out (fp32) = float(bf16(g * stddev)) -- bf16-valued W. */
int ocwg_synth_dev(ocwg_ctx* ctx, int kind, uint64_t seed, uint64_t rows, uint64_t cols,
                   double stddev, const float* col_scale, void* out);
/* Same with every pointer in device memory (inputs resident in HBM). */
int ocwg_quantize_layer_x_dev(ocwg_ctx* ctx, const float* w, const uint16_t* x, uint64_t tokens,
                              uint64_t n, uint64_t m, const ocwg_quant_config* cfg,
                              const ocwg_gptq_options* opts, int scale_mode, int16_t* codes,
                              float* scales, int32_t* zeros, float* w_hat, uint8_t* payload,
                              float* h_out);
/* Device-pointer pieces, for sharded use (Hessian token shards + all-reduce,
 * then GPTQ on a column slab of W).  w is N x M with row stride ldw (>= M),
 * so a column slab of a larger W is passed as (w + j0, m = slab, ldw = M);
 * codes / w_hat use the same row stride ldw; scales / zeros are the slab's own
 * grids (N x ceil(m/G) for per-group). */
int ocwg_hessian_bf16_dev(ocwg_ctx* ctx, const uint16_t* x, uint64_t tokens, uint64_t dim,
                          float* h, int accumulate);
int ocwg_gptq_quantize_dev(ocwg_ctx* ctx, const float* w, uint64_t ldw, const float* h,
                           uint64_t n, uint64_t m, const ocwg_quant_config* cfg,
                           const ocwg_gptq_options* opts, int scale_mode, int16_t* codes,
                           float* scales, int32_t* zeros, float* w_hat);
int ocwg_pack_uniform_dev(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                          const int32_t* zeros, uint64_t rows, uint64_t cols,
                          const ocwg_quant_config* cfg, uint8_t* out);

/* ---- test / profiling hooks -------------------------------------------- */
/* impl: 0 = tcgen05 kernel (product), 1 = SIMT fp64-accumulate cross-check */
int ocwg_debug_hessian_dev(ocwg_ctx* ctx, const uint16_t* x, uint64_t tokens, uint64_t dim,
                           float* h, int accumulate, int impl);
/* bf16 parts of fp32 statistics inputs (stats.cu split_bf16), device pointers */
int ocwg_debug_split_dev(ocwg_ctx* ctx, const float* xp, const float* xf, uint64_t rows,
                         uint64_t dim, uint64_t ld, uint16_t* p1, uint16_t* p2, uint16_t* d1,
                         uint16_t* d2, unsigned* flags);
/* The general tensor-core statistics kernel (gram_tc.cu), device pointers:
 * gram (+)= sum_s ops[ga[s]]^T ops[gb[s]] (s < gseg; symmetric operand set)
 * and cross (+)= sum_s ops[ca[s]]^T ops[cb[s]] (s < cseg); ops: tokens x dim
 * bf16 with row stride ld (% 8 == 0); outputs dim x dim fp32 (f64 = 0) or
 * fp64; window: tokens per TMEM accumulation (0 = default). */
int ocwg_debug_gram_dev(ocwg_ctx* ctx, const uint16_t* const* ops, int nops, uint64_t tokens,
                        uint64_t dim, uint64_t ld, int gseg, const int* ga, const int* gb, int cseg,
                        const int* ca, const int* cb, void* gram, void* cross, int f64,
                        int accumulate, int64_t window);
/* Phase timing of gptq (CUDA events): on != 0 enables recording; phase_ms
 * (may be NULL) receives the last run's [order+damp+permute-H, Cholesky,
 * triangular inverse, grids, sweep] in milliseconds. */
int ocwg_debug_profile(ocwg_ctx* ctx, int on, double* phase_ms);
/* GEMM micro-benchmark hook (device pointers): C = beta C + alpha op(A) op(B). */
int ocwg_debug_gemm(ocwg_ctx* ctx, int precision, uint64_t m, uint64_t n, uint64_t k, double alpha,
                    const void* a, uint64_t lda, int ta, const void* b, uint64_t ldb, int tb,
                    double beta, void* c, uint64_t ldc, int lower_only, int reps, double* ms);
/* Micro-benchmark of the 64 x 64 diagonal-tile factorisation (one CTA):
 * cycles[0] = total clocks over `iters` runs, cycles[1] = clocks of the last;
 * l_out (64 x 64 fp32) = the factor, for a check. */
int ocwg_debug_factor_bench(ocwg_ctx* ctx, int iters, long long* cycles, float* l_out);
/* Phase timestamps (globaltimer ns, 8 per CTA) of the in-block sweep launch
 * whose first row equals $OCWG_SWEEP_TRACE_IB; returns the count copied. */
int ocwg_debug_sweep_trace(ocwg_ctx* ctx, unsigned long long* out, int cap);
/* Number of kernels this library launched on the context so far. */
uint64_t ocwg_launch_count(ocwg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* OCWG_H */
