// Times the reference's OWN API path through the GPU drop-in at a BASELINE
// config: what run_layerwise_sweep does per layer (pipeline.cpp:215-226) --
//   CalibStats stats(N); accumulate_stats(stats, x_fp, x_hat);
//   quantize_layer(w, stats, {gptq, cfg, minmax, gptq opts, [qep]});
// with fp32 host matrices in and out (ocw::Matrix), X_hat != X.  Built by
// cpp/build_dropin.sh; bench.py runs it and reports the "dropin" key.
//
//   dropin_bench [T N M]   (default C2: 262144 4096 4096)
// Inputs: seeded synthetic (splitmix64 -> Box-Muller), X ~ N(0,1) with 1% of
// channels x20, X_hat = X + 0.02 N(0,1), W = bf16-valued 0.02 N(0,1).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "ocw/layerwise.hpp"
#include "ocw/quant.hpp"
#include "ocw/stats.hpp"

namespace {

uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
float normal_at(uint64_t seed, uint64_t i) {  // counter-based: element i of stream seed
  const uint64_t r = splitmix(seed ^ (i * 0xD1B54A32D192ED03ULL));
  const double u1 = (double((r >> 11) & ((1ULL << 26) - 1)) + 1.0) / double(1ULL << 26);
  const double u2 = double(r >> 38) / double(1ULL << 26);
  return float(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2));
}
float bf16_round(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  std::memcpy(&v, &u, 4);
  return v;
}
template <typename F>
void parallel_for(size_t n, F&& f) {
  const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t i = n * t / nt; i < n * (t + 1) / nt; ++i) f(i);
    });
  for (auto& x : th) x.join();
}
double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

int main(int argc, char** argv) {
  const size_t T = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 262144;
  const size_t N = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4096;
  const size_t M = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 4096;
  using namespace ocw;
  // warm-up: context creation and first-use costs, on a small layer
  {
    Matrix xs = random_gaussian(256, 64, 1), ws = random_gaussian(64, 64, 2, 0.02f);
    CalibStats s(64);
    accumulate_stats(s, xs, xs);
    LayerQuantOptions o;
    o.config.bits = 4;
    o.config.scheme = Scheme::asymmetric;
    o.config.granularity = Granularity::per_group;
    o.config.group_size = 32;
    (void)quantize_layer(ws, s, o);
  }
  const auto tg = std::chrono::steady_clock::now();
  std::vector<float> scale(N, 1.0f);
  for (size_t k = 0; k < (N + 50) / 100; ++k) scale[splitmix(0x5EED2002ULL + k) % N] = 20.0f;
  Matrix x(T, N), xh(T, N), w(N, M);
  parallel_for(T, [&](size_t r) {
    for (size_t c = 0; c < N; ++c) {
      const float v = normal_at(0x5EED1020ULL, r * N + c) * scale[c];
      x.data[r * N + c] = v;
      xh.data[r * N + c] = v + 0.02f * normal_at(0x5EED1021ULL, r * N + c);
    }
  });
  parallel_for(N, [&](size_t r) {
    for (size_t c = 0; c < M; ++c) w.data[r * M + c] = bf16_round(0.02f * normal_at(0x5EED0020ULL, r * M + c));
  });
  const double gen_ms = ms_since(tg);

  LayerQuantOptions opts;  // run_pipeline's defaults: block_cols 32 (layerwise.hpp:14)
  opts.method = BaseQuantMethod::gptq;
  opts.config.bits = 4;
  opts.config.scheme = Scheme::asymmetric;
  opts.config.granularity = Granularity::per_group;
  opts.config.group_size = 128;
  opts.gptq.actorder = true;
  opts.gptq.percdamp = 0.01;
  LayerQuantOptions opts_qep = opts;
  opts_qep.qep = QepOptions{};

  // the first full-size call grows the library's device workspace (one-time);
  // the reference pipeline calls accumulate_stats once per layer, so the
  // steady-state (second) call is the figure reported
  CalibStats stats0(N);
  auto t0 = std::chrono::steady_clock::now();
  accumulate_stats(stats0, x, xh);
  const double stats_first_ms = ms_since(t0);
  CalibStats stats(N);
  t0 = std::chrono::steady_clock::now();
  accumulate_stats(stats, x, xh);
  const double stats_ms = ms_since(t0);
  t0 = std::chrono::steady_clock::now();
  QuantizedMatrix q = quantize_layer(w, stats, opts);
  const double ql_ms = ms_since(t0);
  t0 = std::chrono::steady_clock::now();
  QuantizedMatrix qq = quantize_layer(w, stats, opts_qep);
  const double qlq_ms = ms_since(t0);
  size_t same = 0;
  for (size_t i = 0; i < q.codes.size(); ++i) same += q.codes[i] == qq.codes[i];
  std::printf(
      "{\"tokens\": %zu, \"n\": %zu, \"m\": %zu, \"accumulate_stats_ms\": %.3f, "
      "\"accumulate_stats_first_call_ms\": %.3f, "
      "\"quantize_layer_ms\": %.3f, \"quantize_layer_qep_ms\": %.3f, "
      "\"layer_ms\": %.3f, \"layer_qep_ms\": %.3f, \"input_gen_ms\": %.1f, "
      "\"qep_codes_changed_frac\": %.5f, \"token_count\": %zu}\n",
      T, N, M, stats_ms, stats_first_ms, ql_ms, qlq_ms, stats_ms + ql_ms, stats_ms + qlq_ms, gen_ms,
      1.0 - double(same) / double(q.codes.size()), stats.token_count);
  return 0;
}
