// C++ drop-in for the reference's hot path: the `ocw::` functions declared in
// /root/reference/proj/include/ocw/{quant,stats,layerwise}.hpp (used verbatim
// from the reference tree, never copied), implemented over the C ABI of
// libocwg.so (include/ocwg.h).  A maintainer links this file instead of
// proj/src/{quant,stats,layerwise}.cpp; callers (run_layerwise_sweep, the CLI,
// the tests) are unchanged.  Every function with numerical work runs on the
// GPU; the remaining ones are integer bookkeeping of the interface (code
// ranges, group topology, byte counts) and the scalar quantiser itself.
//
// Error contract (errors.hpp:9-21): OCWG_INVALID_INPUT -> ocw::invalid_input,
// OCWG_IO_ERROR -> ocw::io_error, OCWG_NUMERIC_ERROR -> ocw::numeric_error,
// CUDA failures -> std::runtime_error.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ocw/errors.hpp"
#include "ocw/jointq.hpp"
#include "ocw/layerwise.hpp"
#include "ocw/quant.hpp"
#include "ocw/stats.hpp"
#include "ocwg.h"

namespace ocw {
namespace {

// One context per host thread (concurrent calls).
// Arithmetic: OCWG_FP32 by default -- tensor-core statistics (bf16 parts, fp32
// per 8192-token window, fp64 across), fp32 Cholesky and 3xTF32 sweep: codes
// >= 99.9 % identical to the reference's fp64 path, H within 1e-5 of it.
// OCW_GPU_PRECISION=fp64 selects the reference's arithmetic class (fp64
// factorisation, sweep and statistics) for bit-level comparisons.
ocwg_ctx* ctx() {
  thread_local struct Holder {
    ocwg_ctx* c = nullptr;
    Holder() {
      const char* d = std::getenv("OCWG_DEVICE");
      if (ocwg_create(d ? std::atoi(d) : 0, &c) != OCWG_OK)
        throw std::runtime_error(std::string("ocwg_create: ") + ocwg_last_error());
      const char* p = std::getenv("OCW_GPU_PRECISION");
      if (p && std::strcmp(p, "fp64") == 0) ocwg_set_precision(c, OCWG_FP64);
      // CalibStats keeps gram / cross as Eigen (column-major) matrices: hand the
      // storage over as is, the device transposes (no host-side copies)
      ocwg_set_stats_layout(c, OCWG_COL_MAJOR);
    }
    ~Holder() { ocwg_destroy(c); }
  } h;
  return h.c;
}

void check(int s) {
  if (s == OCWG_OK) return;
  const std::string msg = ocwg_last_error();
  if (s == OCWG_INVALID_INPUT) throw invalid_input(msg);
  if (s == OCWG_IO_ERROR) throw io_error(msg);
  if (s == OCWG_NUMERIC_ERROR) throw numeric_error(msg);
  throw std::runtime_error(msg);
}

ocwg_quant_config cc(const QuantConfig& c) {
  ocwg_quant_config o{};
  o.bits = c.bits;
  o.scheme = c.scheme == Scheme::asymmetric ? OCWG_ASYMMETRIC : OCWG_SYMMETRIC;
  o.granularity = c.granularity == Granularity::per_tensor    ? OCWG_PER_TENSOR
                  : c.granularity == Granularity::per_channel ? OCWG_PER_CHANNEL
                                                              : OCWG_PER_GROUP;
  o.group_size = c.group_size;
  return o;
}

int mode_of(ScaleMode m) { return m == ScaleMode::mse_grid ? OCWG_MSE_GRID : OCWG_MINMAX; }

std::vector<QuantGrid> grids_of(const std::vector<float>& s, const std::vector<int32_t>& z,
                                const QuantConfig& cfg) {
  std::vector<QuantGrid> g(s.size());
  const int lo = scheme_qmin(cfg.bits, cfg.scheme), hi = scheme_qmax(cfg.bits, cfg.scheme);
  for (size_t i = 0; i < s.size(); ++i) g[i] = QuantGrid{s[i], z[i], lo, hi};
  return g;
}

void split_grids(const QuantizedMatrix& q, std::vector<float>& s, std::vector<int32_t>& z) {
  s.resize(q.grids.size());
  z.resize(q.grids.size());
  for (size_t i = 0; i < q.grids.size(); ++i) {
    s[i] = q.grids[i].scale;
    z[i] = q.grids[i].zero_point;
  }
}

// one grid over a span (per-tensor calibration of a 1 x n matrix on the GPU)
QuantGrid span_grid(std::span<const float> values, int bits, Scheme scheme, ScaleMode mode) {
  if (values.empty()) throw invalid_input("calibrate: empty input");
  QuantConfig cfg;
  cfg.bits = bits;
  cfg.scheme = scheme;
  cfg.granularity = Granularity::per_tensor;
  const ocwg_quant_config c = cc(cfg);
  float s = 0.f;
  int32_t z = 0;
  check(ocwg_calibrate_grids(ctx(), values.data(), 1, values.size(), &c, mode_of(mode), &s, &z));
  return grids_of({s}, {z}, cfg)[0];
}

}  // namespace

// ------------------------------------------------------------------ quant.hpp
int scheme_qmin(int bits, Scheme scheme) {
  return scheme == Scheme::asymmetric ? 0 : -((1 << (bits - 1)) - 1);
}
int scheme_qmax(int bits, Scheme scheme) {
  return scheme == Scheme::asymmetric ? (1 << bits) - 1 : (1 << (bits - 1)) - 1;
}

void QuantConfig::validate() const {
  const ocwg_quant_config c = cc(*this);
  check(ocwg_validate_config(&c));
}

std::pair<int, float> quantize_scalar(float w, const QuantGrid& g) {
  // code = clamp(int(nearbyint(w / s)) + z, qmin, qmax); ties-to-even
  const long long r = (long long)(int)std::nearbyint(w / g.scale) + g.zero_point;
  const int code = int(r < g.qmin ? g.qmin : (r > g.qmax ? g.qmax : r));
  return {code, dequantize_scalar(code, g)};
}
float dequantize_scalar(int code, const QuantGrid& g) {
  return g.scale * float(code - g.zero_point);
}

QuantGrid calibrate_asymmetric(std::span<const float> values, int bits) {
  return span_grid(values, bits, Scheme::asymmetric, ScaleMode::minmax);
}
QuantGrid calibrate_symmetric(std::span<const float> values, int bits) {
  if (bits < 2) throw invalid_input("calibrate_symmetric: bits must be >= 2");
  return span_grid(values, bits, Scheme::symmetric, ScaleMode::minmax);
}
QuantGrid calibrate_grid(std::span<const float> values, int bits, Scheme scheme) {
  return span_grid(values, bits, scheme, ScaleMode::minmax);
}
QuantGrid calibrate_grid_mse(std::span<const float> values, int bits, Scheme scheme) {
  return span_grid(values, bits, scheme, ScaleMode::mse_grid);
}

size_t quant_groups_per_row(const QuantConfig& cfg, size_t cols) {
  if (cfg.granularity == Granularity::per_tensor) return 0;
  if (cfg.granularity == Granularity::per_channel) return 1;
  return (cols + cfg.group_size - 1) / cfg.group_size;
}
size_t quant_group_count(const QuantConfig& cfg, size_t rows, size_t cols) {
  const ocwg_quant_config c = cc(cfg);
  return size_t(ocwg_group_count(&c, rows, cols));
}
size_t QuantizedMatrix::group_count() const { return quant_group_count(config, rows, cols); }
size_t QuantizedMatrix::group_index(size_t i, size_t j) const {
  if (config.granularity == Granularity::per_tensor) return 0;
  if (config.granularity == Granularity::per_channel) return i;
  return i * quant_groups_per_row(config, cols) + j / config.group_size;
}

std::vector<QuantGrid> calibrate_grids(const Matrix& w, const QuantConfig& cfg, ScaleMode mode) {
  cfg.validate();
  const ocwg_quant_config c = cc(cfg);
  const size_t ng = quant_group_count(cfg, w.rows, w.cols);
  std::vector<float> s(ng);
  std::vector<int32_t> z(ng);
  check(ocwg_calibrate_grids(ctx(), w.data.data(), w.rows, w.cols, &c, mode_of(mode), s.data(),
                             z.data()));
  return grids_of(s, z, cfg);
}

QuantizedMatrix quantize_matrix(const Matrix& w, const QuantConfig& cfg, ScaleMode mode) {
  cfg.validate();
  const ocwg_quant_config c = cc(cfg);
  const size_t ng = quant_group_count(cfg, w.rows, w.cols);
  std::vector<float> s(ng);
  std::vector<int32_t> z(ng);
  QuantizedMatrix q{w.rows, w.cols, cfg, std::vector<int16_t>(w.rows * w.cols), {}};
  check(ocwg_quantize_matrix(ctx(), w.data.data(), w.rows, w.cols, &c, mode_of(mode),
                             q.codes.data(), s.data(), z.data()));
  q.grids = grids_of(s, z, cfg);
  return q;
}

Matrix dequantize(const QuantizedMatrix& q) {
  const ocwg_quant_config c = cc(q.config);
  std::vector<float> s;
  std::vector<int32_t> z;
  split_grids(q, s, z);
  Matrix out(q.rows, q.cols);
  if (q.rows * q.cols == 0) return out;
  check(ocwg_dequantize(ctx(), q.codes.data(), s.data(), z.data(), q.rows, q.cols, &c,
                        out.data.data()));
  return out;
}

size_t uniform_storage_bytes(const QuantConfig& cfg, size_t rows, size_t cols) {
  const ocwg_quant_config c = cc(cfg);
  return size_t(ocwg_storage_bytes(&c, rows, cols));
}
size_t storage_bytes(const QuantizedMatrix& q) {
  return uniform_storage_bytes(q.config, q.rows, q.cols);
}

double activation_objective(const Matrix& w, const Matrix& w_hat, const Matrix& h) {
  require_same_shape(w, w_hat, "activation_objective");
  if (h.rows != w.rows || h.cols != w.rows)
    throw invalid_input("activation_objective: H must be N x N with N = rows of W");
  double out = 0.0;
  check(ocwg_activation_objective(ctx(), w.data.data(), w_hat.data.data(), h.data.data(), w.rows,
                                  w.cols, &out));
  return out;
}

// ------------------------------------------------------------------ stats.hpp
Matrix CalibStats::gram_matrix() const {  // fp64 -> fp32 (stats.cpp:7)
  Matrix m(dim(), dim());
  for (size_t i = 0; i < m.rows; ++i)
    for (size_t j = 0; j < m.cols; ++j)
      m.data[i * m.cols + j] = float(gram(Eigen::Index(i), Eigen::Index(j)));
  return m;
}
Matrix CalibStats::cross_matrix() const {
  Matrix m(dim(), dim());
  for (size_t i = 0; i < m.rows; ++i)
    for (size_t j = 0; j < m.cols; ++j)
      m.data[i * m.cols + j] = float(cross(Eigen::Index(i), Eigen::Index(j)));
  return m;
}


void accumulate_stats(CalibStats& stats, const Matrix& x_fp, const Matrix& x_pert) {
  require_same_shape(x_fp, x_pert, "accumulate_stats");
  if (x_fp.cols != stats.dim())
    throw invalid_input("accumulate_stats: stats dimension " + std::to_string(stats.dim()) +
                        " does not match inputs with " + std::to_string(x_fp.cols) + " columns");
  uint64_t tokens = stats.token_count;
  // identical inputs: cross += Xp^T (X - Xp) is identically zero (stats.cpp:17)
  const bool same = x_fp.data == x_pert.data;
  const float* xf = same ? x_pert.data.data() : x_fp.data.data();
  check(ocwg_accumulate_stats(ctx(), xf, x_pert.data.data(), x_fp.rows, x_fp.cols,
                              stats.gram.data(), same ? nullptr : stats.cross.data(), &tokens));
  stats.token_count = size_t(tokens);
}

// ------------------------------------------------------------------ layerwise.hpp
std::vector<size_t> gptq_order(const Matrix& h, bool actorder) {
  if (h.rows != h.cols) throw invalid_input("gptq_order: H must be square");
  std::vector<int64_t> o(h.rows);
  check(ocwg_gptq_order(ctx(), h.data.data(), h.rows, actorder ? 1 : 0, o.data()));
  return std::vector<size_t>(o.begin(), o.end());
}

QuantizedMatrix gptq_quantize(const Matrix& w, const Matrix& h, const QuantConfig& cfg,
                              const GptqOptions& opts, ScaleMode mode) {
  cfg.validate();  // layerwise.cpp:22
  if (h.rows != w.rows || h.cols != w.rows)
    throw invalid_input("gptq_quantize: H must be N x N with N = rows of W");
  const ocwg_quant_config c = cc(cfg);
  const ocwg_gptq_options o{opts.actorder ? 1 : 0, 0, opts.percdamp, uint64_t(opts.block_cols)};
  const size_t ng = quant_group_count(cfg, w.rows, w.cols);
  std::vector<float> s(ng);
  std::vector<int32_t> z(ng);
  QuantizedMatrix q{w.rows, w.cols, cfg, std::vector<int16_t>(w.rows * w.cols), {}};
  check(ocwg_gptq_quantize(ctx(), w.data.data(), h.data.data(), w.rows, w.cols, &c, &o,
                           mode_of(mode), q.codes.data(), s.data(), z.data(), nullptr));
  q.grids = grids_of(s, z, cfg);
  return q;
}

Matrix qep_target(const Matrix& w, const CalibStats& stats, const QepOptions& opts) {
  if (stats.dim() != w.rows)
    throw invalid_input("qep_target: stats dimension does not match W rows");
  Matrix out(w.rows, w.cols);
  check(ocwg_qep_target(ctx(), w.data.data(), stats.gram.data(), stats.cross.data(), w.rows, w.cols,
                        opts.alpha, opts.eta, out.data.data()));
  return out;
}

BaseQuantMethod base_method_from_name(const std::string& name) {
  if (name == "rtn") return BaseQuantMethod::rtn;
  if (name == "gptq") return BaseQuantMethod::gptq;
  throw invalid_input("unknown quantization method: " + name);
}

// [qep_target] -> RTN / GPTQ on stats.gram_matrix() (layerwise.cpp:120-126) in
// one device round trip: W and the fp64 statistics go in once, the QEP target
// and fp32(gram) stay on the device.
QuantizedMatrix quantize_layer(const Matrix& w, const CalibStats& stats,
                               const LayerQuantOptions& opts) {
  if (opts.method == BaseQuantMethod::rtn && !opts.qep)
    return quantize_matrix(w, opts.config, opts.scale_mode);
  if (stats.dim() != w.rows)
    throw invalid_input(opts.qep ? "qep_target: stats dimension does not match W rows"
                                 : "gptq_quantize: H must be N x N with N = rows of W");
  const QuantConfig& cfg = opts.config;
  const ocwg_quant_config c = cc(cfg);
  const ocwg_gptq_options o{opts.gptq.actorder ? 1 : 0, 0, opts.gptq.percdamp,
                            uint64_t(opts.gptq.block_cols)};
  ocwg_qep_options qo{};
  if (opts.qep) qo = ocwg_qep_options{opts.qep->alpha, opts.qep->eta};
  const size_t ng = quant_group_count(cfg, w.rows, w.cols);
  std::vector<float> s(ng);
  std::vector<int32_t> z(ng);
  QuantizedMatrix q{w.rows, w.cols, cfg, std::vector<int16_t>(w.rows * w.cols), {}};
  check(ocwg_quantize_layer(ctx(), w.data.data(), stats.gram.data(),
                            opts.qep ? stats.cross.data() : nullptr, w.rows,
                            w.cols, opts.method == BaseQuantMethod::gptq ? 1 : 0, &c, &o,
                            mode_of(opts.scale_mode), opts.qep ? &qo : nullptr, q.codes.data(),
                            s.data(), z.data(), nullptr));
  q.grids = grids_of(s, z, cfg);
  return q;
}


// ------------------------------------------------------------------ jointq.hpp
namespace {
void jq_validate(const QuantizedMatrix& q, const Matrix& w, const Matrix& x) {  // jointq.cpp:42-58
  q.config.validate();
  if (q.rows != w.rows || q.cols != w.cols)
    throw invalid_input("jointq: quantized shape does not match W");
  if (x.cols != w.rows) throw invalid_input("jointq: X cols must equal W rows");
  if (q.codes.size() != q.rows * q.cols || q.grids.size() != q.group_count())
    throw invalid_input("jointq: malformed quantized matrix (expect the uniform GPTQ format)");
  for (size_t i = 0; i < q.rows; ++i)
    for (size_t j = 0; j < q.cols; ++j) {
      const QuantGrid& g = q.grids[q.group_index(i, j)];
      const int code = q.codes[i * q.cols + j];
      if (code < g.qmin || code > g.qmax) throw invalid_input("jointq: code outside the codebook range");
    }
}
}  // namespace

double jointq_objective(const QuantizedMatrix& q, const Matrix& w, const Matrix& x, double lambda) {
  if (lambda < 0.0) throw invalid_input("jointq_objective: lambda must be >= 0");
  if (q.rows != w.rows || q.cols != w.cols || x.cols != w.rows)
    throw invalid_input("jointq_objective: shape mismatch");
  const ocwg_quant_config c = cc(q.config);
  std::vector<float> s;
  std::vector<int32_t> z;
  split_grids(q, s, z);
  double out = 0.0;
  check(ocwg_jointq_objective(ctx(), q.codes.data(), s.data(), z.data(), w.data.data(), w.rows,
                              w.cols, x.data.data(), x.rows, &c, lambda, &out));
  return out;
}

double jointq_optimal_group_scale(const QuantizedMatrix& q, const Matrix& w, const Matrix& x,
                                  double lambda, size_t group) {
  jq_validate(q, w, x);
  const ocwg_quant_config c = cc(q.config);
  std::vector<float> s;
  std::vector<int32_t> z;
  split_grids(q, s, z);
  double out = 0.0;
  check(ocwg_jointq_optimal_group_scale(ctx(), q.codes.data(), s.data(), z.data(), w.data.data(),
                                        w.rows, w.cols, x.data.data(), x.rows, &c, lambda, group,
                                        &out));
  return out;
}

JointqResult jointq_refine(const QuantizedMatrix& q0, const Matrix& w, const Matrix& x,
                           const JointqOptions& opts) {
  jq_validate(q0, w, x);
  if (opts.lambda < 0.0) throw invalid_input("jointq_refine: lambda must be >= 0");
  if (opts.move_radius < 1) throw invalid_input("jointq_refine: move_radius must be >= 1");
  const ocwg_quant_config c = cc(q0.config);
  std::vector<float> s;
  std::vector<int32_t> z;
  split_grids(q0, s, z);
  JointqResult res;
  res.refined = q0;
  // at most one accepted move per group refit, cell and zero step per pass
  const uint64_t bound =
      uint64_t(std::max(0, opts.max_passes)) * (q0.rows * q0.cols + 2 * q0.grids.size()) + 1;
  std::vector<double> trace(std::min<uint64_t>(bound, uint64_t(1) << 24));
  uint64_t len = 0, acc = 0;
  int passes = 0;
  check(ocwg_jointq_refine(ctx(), w.data.data(), w.rows, w.cols, x.data.data(), x.rows, &c,
                           res.refined.codes.data(), s.data(), z.data(), opts.lambda,
                           opts.max_passes, opts.move_radius, trace.data(), trace.size(), &len,
                           &acc, &passes));
  if (len == 0 || len > trace.size())
    throw std::runtime_error("jointq_refine: objective trace overflow");
  for (size_t g = 0; g < res.refined.grids.size(); ++g) {
    res.refined.grids[g].scale = s[g];
    res.refined.grids[g].zero_point = z[g];
  }
  trace.resize(len);
  res.objective_trace = std::move(trace);
  res.accepted_moves = size_t(acc);
  res.passes = passes;
  return res;
}

}  // namespace ocw
