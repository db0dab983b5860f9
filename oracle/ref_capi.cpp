// C entry points over the reference's OWN hot-path sources (proj/src/quant.cpp,
// stats.cpp, layerwise.cpp, matrix.cpp compiled unmodified from
// /root/reference by oracle/build_ref.sh against our Eigen-API shim).
//
// TEST INFRASTRUCTURE ONLY: loaded with ctypes by tests/ (as the parity
// checker), by tests/golden/make_golden.py (fixture generation) and by
// bench.py's cpu_baseline / --impl reference arm (the CPU baseline).  Never
// linked into the product library.
//
// Status codes mirror include/ocwg.h: 0 ok, 1 invalid_input, 2 io_error,
// 3 numeric_error, 4 other.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "ocw/errors.hpp"
#include "ocw/eigen_map.hpp"
#include "ocw/jointq.hpp"
#include "ocw/layerwise.hpp"
#include "ocw/autobit.hpp"
#include "ocw/quant.hpp"
#include "ocw/stats.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ocw::invalid_input& e) {
    g_err = e.what();
    return 1;
  } catch (const ocw::io_error& e) {
    g_err = e.what();
    return 2;
  } catch (const ocw::numeric_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

ocw::Matrix to_matrix(const float* p, size_t rows, size_t cols) {
  ocw::Matrix m(rows, cols);
  if (rows * cols != 0) std::memcpy(m.data.data(), p, rows * cols * sizeof(float));
  return m;
}

ocw::QuantConfig make_cfg(int bits, int scheme, int gran, size_t group) {
  ocw::QuantConfig c;
  c.bits = bits;
  c.scheme = scheme == 1 ? ocw::Scheme::asymmetric : ocw::Scheme::symmetric;
  c.granularity = gran == 0   ? ocw::Granularity::per_tensor
                  : gran == 1 ? ocw::Granularity::per_channel
                              : ocw::Granularity::per_group;
  c.group_size = group;
  return c;
}

void export_q(const ocw::QuantizedMatrix& q, int16_t* codes, float* scales, int32_t* zeros) {
  if (codes) std::memcpy(codes, q.codes.data(), q.codes.size() * sizeof(int16_t));
  for (size_t g = 0; g < q.grids.size(); ++g) {
    if (scales) scales[g] = q.grids[g].scale;
    if (zeros) zeros[g] = q.grids[g].zero_point;
  }
}

ocw::QuantizedMatrix import_q(const int16_t* codes, const float* scales, const int32_t* zeros,
                              size_t rows, size_t cols, const ocw::QuantConfig& cfg) {
  ocw::QuantizedMatrix q;
  q.rows = rows;
  q.cols = cols;
  q.config = cfg;
  q.codes.assign(codes, codes + rows * cols);
  const size_t ng = ocw::quant_group_count(cfg, rows, cols);
  q.grids.resize(ng);
  for (size_t g = 0; g < ng; ++g) {
    q.grids[g].scale = scales[g];
    q.grids[g].zero_point = zeros[g];
    q.grids[g].qmin = ocw::scheme_qmin(cfg.bits, cfg.scheme);
    q.grids[g].qmax = ocw::scheme_qmax(cfg.bits, cfg.scheme);
  }
  return q;
}

}  // namespace

extern "C" {

const char* ocwref_last_error() { return g_err.c_str(); }
const char* ocwref_blas_name() { return Eigen::shim::blas_name(); }
void ocwref_use_blas(int on) { Eigen::shim::blas_enabled() = on != 0; }
void ocwref_set_threads(int n) {
  if (Eigen::shim::blas().set_threads) Eigen::shim::blas().set_threads(n);
}

size_t ocwref_group_count(int bits, int scheme, int gran, size_t group, size_t rows, size_t cols) {
  return ocw::quant_group_count(make_cfg(bits, scheme, gran, group), rows, cols);
}
size_t ocwref_storage_bytes(int bits, int scheme, int gran, size_t group, size_t rows,
                            size_t cols) {
  return ocw::uniform_storage_bytes(make_cfg(bits, scheme, gran, group), rows, cols);
}

// matrix.cpp:57-62 seeded fixture generator
int ocwref_random_gaussian(size_t rows, size_t cols, uint64_t seed, float stddev, float* out) {
  return guard([&] {
    ocw::Matrix m = ocw::random_gaussian(rows, cols, seed, stddev);
    std::memcpy(out, m.data.data(), m.size() * sizeof(float));
  });
}

// quant.cpp:168-196
int ocwref_calibrate_grids(const float* w, size_t rows, size_t cols, int bits, int scheme,
                           int gran, size_t group, int mse, float* scales, int32_t* zeros) {
  return guard([&] {
    auto grids = ocw::calibrate_grids(to_matrix(w, rows, cols), make_cfg(bits, scheme, gran, group),
                                      mse ? ocw::ScaleMode::mse_grid : ocw::ScaleMode::minmax);
    for (size_t g = 0; g < grids.size(); ++g) {
      scales[g] = grids[g].scale;
      zeros[g] = grids[g].zero_point;
    }
  });
}

// quant.cpp:198-210
int ocwref_quantize_matrix(const float* w, size_t rows, size_t cols, int bits, int scheme,
                           int gran, size_t group, int mse, int16_t* codes, float* scales,
                           int32_t* zeros) {
  return guard([&] {
    auto q = ocw::quantize_matrix(to_matrix(w, rows, cols), make_cfg(bits, scheme, gran, group),
                                  mse ? ocw::ScaleMode::mse_grid : ocw::ScaleMode::minmax);
    export_q(q, codes, scales, zeros);
  });
}

// autobit.cpp:45-61 (candidate_grid) with estimate_error :16-34: errors and
// storage costs of bits {2..8} x {per_group 128, per_channel}, symmetric
int ocwref_candidate_grid(const float* w, size_t rows, size_t cols, int mode,
                          const double* in_diag, double* errs, size_t* costs) {
  return guard([&] {
    std::vector<double> diag;
    if (in_diag) diag.assign(in_diag, in_diag + rows);
    auto cands = ocw::candidate_grid(to_matrix(w, rows, cols),
                                     mode ? ocw::ErrorMode::act_aware : ocw::ErrorMode::naive,
                                     in_diag ? &diag : nullptr);
    for (size_t k = 0; k < cands.size(); ++k) {
      errs[k] = cands[k].err;
      costs[k] = cands[k].cost_bytes;
    }
  });
}

// quant.cpp:212-218
int ocwref_dequantize(const int16_t* codes, const float* scales, const int32_t* zeros, size_t rows,
                      size_t cols, int bits, int scheme, int gran, size_t group, float* out) {
  return guard([&] {
    auto q = import_q(codes, scales, zeros, rows, cols, make_cfg(bits, scheme, gran, group));
    ocw::Matrix d = ocw::dequantize(q);
    std::memcpy(out, d.data.data(), d.size() * sizeof(float));
  });
}

// quant.cpp:230-236
int ocwref_activation_objective(const float* w, const float* w_hat, const float* h, size_t n,
                                size_t m, double* out) {
  return guard([&] {
    *out = ocw::activation_objective(to_matrix(w, n, m), to_matrix(w_hat, n, m), to_matrix(h, n, n));
  });
}

// layerwise.cpp:11-18
int ocwref_gptq_order(const float* h, size_t n, int actorder, int64_t* order) {
  return guard([&] {
    auto o = ocw::gptq_order(to_matrix(h, n, n), actorder != 0);
    for (size_t i = 0; i < n; ++i) order[i] = int64_t(o[i]);
  });
}

// layerwise.cpp:20-93 (the routine the CUDA path replaces)
int ocwref_gptq_quantize(const float* w, const float* h, size_t n, size_t m, int bits, int scheme,
                         int gran, size_t group, int actorder, double percdamp, size_t block,
                         int mse, int16_t* codes, float* scales, int32_t* zeros, double* seconds) {
  return guard([&] {
    ocw::GptqOptions o;
    o.actorder = actorder != 0;
    o.percdamp = percdamp;
    o.block_cols = block;
    const ocw::Matrix wm = to_matrix(w, n, m), hm = to_matrix(h, n, n);
    const auto t0 = std::chrono::steady_clock::now();
    auto q = ocw::gptq_quantize(wm, hm, make_cfg(bits, scheme, gran, group), o,
                                mse ? ocw::ScaleMode::mse_grid : ocw::ScaleMode::minmax);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    export_q(q, codes, scales, zeros);
  });
}

// Parity artefacts of layerwise.cpp:31-51 that gptq_quantize keeps internal:
// the dampened, permuted inverse hinv = hp^-1 and its upper factor U.  This
// restates exactly those lines (same shim LLT / solve the routine uses).
int ocwref_gptq_factor(const float* h, size_t n, int actorder, double percdamp, double* hinv_out,
                       double* u_out, double* damp_out) {
  return guard([&] {
    const ocw::Matrix hm = to_matrix(h, n, n);
    const auto order = ocw::gptq_order(hm, actorder != 0);
    Eigen::MatrixXd hd = ocw::to_eigen_d(hm);
    const double damp = percdamp * hd.diagonal().mean();
    hd.diagonal().array() += damp;
    Eigen::MatrixXd hp{Eigen::Index(n), Eigen::Index(n)};
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j)
        hp(Eigen::Index(i), Eigen::Index(j)) = hd(Eigen::Index(order[i]), Eigen::Index(order[j]));
    Eigen::LLT<Eigen::MatrixXd> llt(hp);
    if (llt.info() != Eigen::Success)
      throw ocw::numeric_error("gptq_quantize: Gram matrix is not positive definite after dampening");
    Eigen::MatrixXd hinv = llt.solve(Eigen::MatrixXd::Identity(Eigen::Index(n), Eigen::Index(n)));
    Eigen::LLT<Eigen::MatrixXd> llt_inv(hinv);
    if (llt_inv.info() != Eigen::Success)
      throw ocw::numeric_error("gptq_quantize: inverse Gram factorization failed");
    Eigen::MatrixXd u = llt_inv.matrixU();
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) {
        if (hinv_out) hinv_out[i * n + j] = hinv(Eigen::Index(i), Eigen::Index(j));
        if (u_out) u_out[i * n + j] = u(Eigen::Index(i), Eigen::Index(j));
      }
    if (damp_out) *damp_out = damp;
  });
}

// stats.cpp:10-19, streaming: gram/cross (row-major n x n fp64) are read,
// accumulated into, and written back; token_count is updated likewise.
int ocwref_accumulate_stats(const float* x_fp, const float* x_pert, size_t rows, size_t dim,
                            double* gram, double* cross, uint64_t* token_count, double* seconds) {
  return guard([&] {
    ocw::CalibStats s(dim);
    for (size_t i = 0; i < dim; ++i)
      for (size_t j = 0; j < dim; ++j) {
        s.gram(Eigen::Index(i), Eigen::Index(j)) = gram[i * dim + j];
        s.cross(Eigen::Index(i), Eigen::Index(j)) = cross ? cross[i * dim + j] : 0.0;
      }
    s.token_count = token_count ? *token_count : 0;
    const ocw::Matrix xf = to_matrix(x_fp, rows, dim), xp = to_matrix(x_pert, rows, dim);
    const auto t0 = std::chrono::steady_clock::now();
    ocw::accumulate_stats(s, xf, xp);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (size_t i = 0; i < dim; ++i)
      for (size_t j = 0; j < dim; ++j) {
        gram[i * dim + j] = s.gram(Eigen::Index(i), Eigen::Index(j));
        if (cross) cross[i * dim + j] = s.cross(Eigen::Index(i), Eigen::Index(j));
      }
    if (token_count) *token_count = s.token_count;
  });
}

// layerwise.cpp:95-112 (QEP target; next-row f1)
int ocwref_qep_target(const float* w, const double* gram, const double* cross, size_t n, size_t m,
                      double alpha, double eta, float* out) {
  return guard([&] {
    ocw::CalibStats s(n);
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) {
        s.gram(Eigen::Index(i), Eigen::Index(j)) = gram[i * n + j];
        s.cross(Eigen::Index(i), Eigen::Index(j)) = cross[i * n + j];
      }
    ocw::Matrix t = ocw::qep_target(to_matrix(w, n, m), s, {alpha, eta});
    std::memcpy(out, t.data.data(), t.size() * sizeof(float));
  });
}

// layerwise.cpp:120-126: quantize_layer over fp64 statistics
int ocwref_quantize_layer(const float* w, const double* gram, const double* cross, size_t n,
                          size_t m, int method_gptq, int bits, int scheme, int gran, size_t group,
                          int mse, int actorder, double percdamp, size_t block, int qep,
                          double alpha, double eta, int16_t* codes, float* scales, int32_t* zeros) {
  return guard([&] {
    ocw::CalibStats s(n);
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) {
        s.gram(Eigen::Index(i), Eigen::Index(j)) = gram[i * n + j];
        s.cross(Eigen::Index(i), Eigen::Index(j)) = cross ? cross[i * n + j] : 0.0;
      }
    ocw::LayerQuantOptions o;
    o.method = method_gptq ? ocw::BaseQuantMethod::gptq : ocw::BaseQuantMethod::rtn;
    o.config = make_cfg(bits, scheme, gran, group);
    o.scale_mode = mse ? ocw::ScaleMode::mse_grid : ocw::ScaleMode::minmax;
    o.gptq.actorder = actorder != 0;
    o.gptq.percdamp = percdamp;
    o.gptq.block_cols = block;
    if (qep) o.qep = ocw::QepOptions{alpha, eta};
    auto q = ocw::quantize_layer(to_matrix(w, n, m), s, o);
    export_q(q, codes, scales, zeros);
  });
}

// jointq.cpp:160-255: refine in place; trace up to trace_cap entries
int ocwref_jointq_refine(const float* w, size_t rows, size_t cols, const float* x, size_t tokens,
                         int bits, int scheme, int gran, size_t group, int16_t* codes,
                         float* scales, int32_t* zeros, double lambda, int max_passes, int radius,
                         double* trace, size_t trace_cap, size_t* trace_len, size_t* accepted,
                         int* passes) {
  return guard([&] {
    const ocw::QuantConfig cfg = make_cfg(bits, scheme, gran, group);
    const ocw::QuantizedMatrix q0 = import_q(codes, scales, zeros, rows, cols, cfg);
    const ocw::JointqResult r = ocw::jointq_refine(q0, to_matrix(w, rows, cols),
                                                   to_matrix(x, tokens, rows),
                                                   {lambda, max_passes, radius});
    export_q(r.refined, codes, scales, zeros);
    *trace_len = r.objective_trace.size();
    for (size_t t = 0; t < r.objective_trace.size() && t < trace_cap; ++t) trace[t] = r.objective_trace[t];
    *accepted = r.accepted_moves;
    *passes = r.passes;
  });
}
int ocwref_jointq_objective(const int16_t* codes, const float* scales, const int32_t* zeros,
                            const float* w, size_t rows, size_t cols, const float* x, size_t tokens,
                            int bits, int scheme, int gran, size_t group, double lambda, double* out) {
  return guard([&] {
    const ocw::QuantConfig cfg = make_cfg(bits, scheme, gran, group);
    *out = ocw::jointq_objective(import_q(codes, scales, zeros, rows, cols, cfg),
                                 to_matrix(w, rows, cols), to_matrix(x, tokens, rows), lambda);
  });
}
int ocwref_jointq_optimal_group_scale(const int16_t* codes, const float* scales,
                                      const int32_t* zeros, const float* w, size_t rows,
                                      size_t cols, const float* x, size_t tokens, int bits,
                                      int scheme, int gran, size_t group_size, double lambda,
                                      size_t group, double* out) {
  return guard([&] {
    const ocw::QuantConfig cfg = make_cfg(bits, scheme, gran, group_size);
    *out = ocw::jointq_optimal_group_scale(import_q(codes, scales, zeros, rows, cols, cfg),
                                           to_matrix(w, rows, cols), to_matrix(x, tokens, rows),
                                           lambda, group);
  });
}

}  // extern "C"
