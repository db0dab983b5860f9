// C ABI of libocwg.so (include/ocwg.h): context, workspace, error mapping and
// the orchestration of the kernels into the reference's hot-path functions.
// Validation order and error classes follow the reference exactly
// (quant.cpp:19-25,168-171; layerwise.cpp:22-26,43-49; stats.cpp:11-15).
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ocwg.h"
#include "kernels.h"

namespace ocwg {

static std::atomic<unsigned long long> g_launches{0};
void count_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
unsigned long long launches_issued() { return g_launches.load(std::memory_order_relaxed); }

int device_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v <= 0) {
    v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

}  // namespace ocwg

using namespace ocwg;

struct ocwg_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  void* ws = nullptr;  // device arena
  size_t ws_bytes = 0;
  unsigned* flag = nullptr;  // device status word
  unsigned* flag_host = nullptr;
  int precision = OCWG_FP32;  // factorisation + sweep arithmetic
  bool stats_colmajor = false;  // fp64 gram / cross host matrices column-major (ocwg_set_stats_layout)
  bool profile = false;       // record phase events in run_gptq
  bool tensor_core_gemm = true;  // fp32 GEMMs on tcgen05 (3xTF32) vs SIMT
  bool async_dev = false;        // *_dev calls return without draining the stream
  cudaEvent_t ev[6] = {};
  double phase_ms[5] = {};
  cudaStream_t aux = nullptr;      // second stream: the sweep's trailing GEMMs
  cudaEvent_t sev[5] = {};         // sweep fork / in-block / trailing x2 / join
  cudaStream_t cpy = nullptr;      // host <-> device copies of the host-pointer calls
  void* io = nullptr;              // grow-only device buffers of the host-pointer calls
  size_t io_bytes = 0;
  std::vector<cudaEvent_t> cev;    // per-chunk copy events
  void* stage[2] = {nullptr, nullptr};  // pinned staging for large pageable host copies
  cudaEvent_t stage_ev[2] = {};
  std::mutex mu;
};

namespace {

thread_local std::string g_err;

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(OCWG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return OCWG_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return OCWG_CUDA_ERROR;
  }
}

// ---------------------------------------------------------------- config
void validate(const ocwg_quant_config* c) {  // QuantConfig::validate (quant.cpp:19-25)
  if (!c) fail(OCWG_INVALID_INPUT, "QuantConfig: null");
  if (c->bits < 1 || c->bits > 8) fail(OCWG_INVALID_INPUT, "QuantConfig: bits must be in [1,8]");
  if (c->scheme == OCWG_SYMMETRIC && c->bits < 2)
    fail(OCWG_INVALID_INPUT,
         "QuantConfig: symmetric grids need bits >= 2 (1-bit signed range is empty)");
  if (c->scheme != OCWG_SYMMETRIC && c->scheme != OCWG_ASYMMETRIC)
    fail(OCWG_INVALID_INPUT, "QuantConfig: unknown scheme");
  if (c->granularity < 0 || c->granularity > 2)
    fail(OCWG_INVALID_INPUT, "QuantConfig: unknown granularity");
  if (c->granularity == OCWG_PER_GROUP && c->group_size < 1)
    fail(OCWG_INVALID_INPUT, "QuantConfig: group_size must be >= 1");
}

QCfg qcfg(const ocwg_quant_config* c, uint64_t cols) {
  QCfg q;
  q.bits = c->bits;
  q.scheme = c->scheme;
  q.gran = c->granularity;
  q.group = c->granularity == OCWG_PER_GROUP ? (long long)c->group_size : 1;
  q.qmin = c->scheme == OCWG_ASYMMETRIC ? 0 : -((1 << (c->bits - 1)) - 1);
  q.qmax = c->scheme == OCWG_ASYMMETRIC ? (1 << c->bits) - 1 : (1 << (c->bits - 1)) - 1;
  q.gpr = c->granularity == OCWG_PER_TENSOR ? 0
          : c->granularity == OCWG_PER_CHANNEL ? 1
                                               : (long long)((cols + c->group_size - 1) / c->group_size);
  return q;
}

uint64_t group_count(const ocwg_quant_config* c, uint64_t rows, uint64_t cols) {
  if (c->granularity == OCWG_PER_TENSOR) return 1;
  if (c->granularity == OCWG_PER_CHANNEL) return rows;
  return rows * ((cols + c->group_size - 1) / c->group_size);
}

uint64_t storage_bytes(const ocwg_quant_config* c, uint64_t rows, uint64_t cols) {
  const uint64_t code_bits = rows * cols * uint64_t(c->bits);
  const uint64_t meta = 2 + (c->scheme == OCWG_ASYMMETRIC ? 1 : 0);
  return (code_bits + 7) / 8 + group_count(c, rows, cols) * meta;
}

// ---------------------------------------------------------------- workspace arena
struct Arena {
  ocwg_ctx* ctx;
  size_t off = 0;
  std::vector<std::pair<size_t, size_t>> reqs;
  explicit Arena(ocwg_ctx* c) : ctx(c) {}
  static size_t al(size_t b) { return (b + 255) & ~size_t(255); }
  // two-phase: reserve sizes, then commit (grow once), then take pointers
  size_t reserve(size_t bytes) {
    const size_t o = off;
    off += al(bytes);
    return o;
  }
  void commit() {
    if (off > ctx->ws_bytes) {
      if (ctx->ws) cudaFree(ctx->ws);
      ctx->ws = nullptr;
      ctx->ws_bytes = 0;
      ck(cudaMalloc(&ctx->ws, off), "cudaMalloc(workspace)");
      ctx->ws_bytes = off;
    }
  }
  template <typename T>
  T* at(size_t o) const {
    return reinterpret_cast<T*>(static_cast<char*>(ctx->ws) + o);
  }
};

void begin(ocwg_ctx* ctx, bool dev_call = false) {
  if (!ctx) fail(OCWG_INVALID_INPUT, "null context");
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  // async device calls keep the status word sticky until ocwg_synchronize
  if (!(dev_call && ctx->async_dev))
    ck(cudaMemsetAsync(ctx->flag, 0, sizeof(unsigned), ctx->stream), "reset status");
}

// drain the stream; map device status bits to the reference's error classes
void finish(ocwg_ctx* ctx, bool numeric_first = true) {
  ck(cudaGetLastError(), "kernel launch");
  ck(cudaMemcpyAsync(ctx->flag_host, ctx->flag, sizeof(unsigned), cudaMemcpyDeviceToHost,
                     ctx->stream),
     "status D2H");
  ck(cudaStreamSynchronize(ctx->stream), "stream synchronize");
  const unsigned f = *ctx->flag_host;
  if (numeric_first && (f & kFlagNotPD))
    fail(OCWG_NUMERIC_ERROR, "gptq_quantize: Gram matrix is not positive definite after dampening");
  if (f & kFlagNonFinite) fail(OCWG_INVALID_INPUT, "calibrate_grids: non-finite entry");
  if (f & kFlagNotPD)
    fail(OCWG_NUMERIC_ERROR, "gptq_quantize: Gram matrix is not positive definite after dampening");
}

// device-pointer entry points: drain (and map the status word) unless async
void finish_dev(ocwg_ctx* ctx) {
  if (ctx->async_dev) {
    ck(cudaGetLastError(), "kernel launch");
    return;
  }
  finish(ctx);
}

void h2d(void* d, const void* h, size_t bytes, ocwg_ctx* ctx) {
  if (bytes) ck(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream), "H2D");
}
void d2h(void* h, const void* d, size_t bytes, ocwg_ctx* ctx) {
  if (bytes && h) ck(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
}

// Large copies between PAGEABLE host memory (e.g. the std::vector inside an
// ocw::Matrix) and the device: through two pinned staging buffers, the host
// side memcpy of one chunk (several CPU threads) overlapping the DMA of the
// other, instead of the driver's synchronous pageable path.
constexpr size_t kStageBytes = size_t(64) << 20;
// Host memcpy on a persistent pool of worker threads (spawning 16 threads per
// 64 MiB chunk cost ~0.3 ms against ~1 ms of copying).  One job at a time.
class CopyPool {
 public:
  static CopyPool& get() {  // never destroyed: its detached workers wait on it until exit
    static CopyPool* p = new CopyPool;
    return *p;
  }
  void run(void* dst, const void* src, size_t bytes) {
    std::lock_guard<std::mutex> job(job_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst), src_ = static_cast<const char*>(src), bytes_ = bytes;
      pending_ = nt_;
      ++gen_;
    }
    cv_.notify_all();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }
  unsigned threads() const { return nt_; }

 private:
  CopyPool() : nt_(std::max(1u, std::min(16u, std::thread::hardware_concurrency()))) {
    for (unsigned t = 0; t < nt_; ++t)
      std::thread([this, t] { worker(t); }).detach();  // live for the process
  }
  void worker(unsigned t) {
    unsigned long long seen = 0;
    while (true) {
      char* d;
      const char* sp;
      size_t n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        d = dst_, sp = src_, n = bytes_;
      }
      const size_t a = n * t / nt_, b = n * (t + 1) / nt_;
      if (b > a) std::memcpy(d + a, sp + a, b - a);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  const unsigned nt_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  unsigned long long gen_ = 0;
  unsigned pending_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};
void par_memcpy(void* dst, const void* src, size_t bytes) {
  // (measured on the B200 box's 16 host cores: 49 GB/s with 8 threads, 65 with 16)
  if (bytes < (size_t(4) << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
  CopyPool::get().run(dst, src, bytes);
}
void ensure_stage(ocwg_ctx* ctx) {
  for (int b = 0; b < 2; ++b) {
    if (!ctx->stage[b]) {
      ck(cudaMallocHost(&ctx->stage[b], kStageBytes), "cudaMallocHost(stage)");
      ck(cudaEventCreateWithFlags(&ctx->stage_ev[b], cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventRecord(ctx->stage_ev[b], ctx->cpy), "event");
    }
  }
}
bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
// H2D of a large host buffer, ordered before later work on ctx->stream
void h2d_big(void* d, const void* h, size_t bytes, ocwg_ctx* ctx) {
  if (bytes < kStageBytes || is_pinned(h)) return h2d(d, h, bytes, ctx);
  ensure_stage(ctx);
  ck(cudaEventRecord(ctx->stage_ev[0], ctx->stream), "event");  // after prior work on the stream
  ck(cudaStreamWaitEvent(ctx->cpy, ctx->stage_ev[0], 0), "event");
  ck(cudaEventRecord(ctx->stage_ev[0], ctx->cpy), "event");
  ck(cudaEventRecord(ctx->stage_ev[1], ctx->cpy), "event");
  for (size_t off = 0, k = 0; off < bytes; off += kStageBytes, ++k) {
    const int b = int(k & 1);
    const size_t len = std::min(kStageBytes, bytes - off);
    ck(cudaEventSynchronize(ctx->stage_ev[b]), "event sync");  // its previous DMA is done
    par_memcpy(ctx->stage[b], static_cast<const char*>(h) + off, len);
    ck(cudaMemcpyAsync(static_cast<char*>(d) + off, ctx->stage[b], len, cudaMemcpyHostToDevice,
                       ctx->cpy),
       "H2D(staged)");
    ck(cudaEventRecord(ctx->stage_ev[b], ctx->cpy), "event");
  }
  ck(cudaStreamWaitEvent(ctx->stream, ctx->stage_ev[0], 0), "event");
  ck(cudaStreamWaitEvent(ctx->stream, ctx->stage_ev[1], 0), "event");
}
// Staged H2D of a (pageable) host buffer on ctx->cpy, ordered after `dep` (an
// event on another stream marking the destination free; null: none) and NOT
// joined to ctx->stream -- the caller waits on an event recorded on ctx->cpy.
// Returns once the last staging memcpy is issued (its DMA may be in flight).
void h2d_staged_async(void* d, const void* h, size_t bytes, ocwg_ctx* ctx, cudaEvent_t dep,
                      cudaEvent_t done) {
  ensure_stage(ctx);
  if (dep) ck(cudaStreamWaitEvent(ctx->cpy, dep, 0), "event");
  if (bytes < kStageBytes || is_pinned(h)) {
    if (is_pinned(h)) {
      ck(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->cpy), "H2D");
    } else {  // small pageable: through staging buffer 0
      ck(cudaEventSynchronize(ctx->stage_ev[0]), "event sync");
      std::memcpy(ctx->stage[0], h, bytes);
      ck(cudaMemcpyAsync(d, ctx->stage[0], bytes, cudaMemcpyHostToDevice, ctx->cpy), "H2D(staged)");
      ck(cudaEventRecord(ctx->stage_ev[0], ctx->cpy), "event");
    }
  } else {
    for (size_t off = 0, k = 0; off < bytes; off += kStageBytes, ++k) {
      const int b = int(k & 1);
      const size_t len = std::min(kStageBytes, bytes - off);
      ck(cudaEventSynchronize(ctx->stage_ev[b]), "event sync");  // its previous DMA is done
      par_memcpy(ctx->stage[b], static_cast<const char*>(h) + off, len);
      ck(cudaMemcpyAsync(static_cast<char*>(d) + off, ctx->stage[b], len, cudaMemcpyHostToDevice,
                         ctx->cpy),
         "H2D(staged)");
      ck(cudaEventRecord(ctx->stage_ev[b], ctx->cpy), "event");
    }
  }
  if (done) ck(cudaEventRecord(done, ctx->cpy), "event");
}
// D2H of a large device buffer after the work on ctx->stream; synchronous
void d2h_big(void* h, const void* d, size_t bytes, ocwg_ctx* ctx) {
  if (!h || !bytes) return;
  if (bytes < kStageBytes || is_pinned(h)) {
    d2h(h, d, bytes, ctx);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    return;
  }
  ensure_stage(ctx);
  size_t pend_off[2] = {0, 0}, pend_len[2] = {0, 0};
  for (size_t off = 0, k = 0; off < bytes; off += kStageBytes, ++k) {
    const int b = int(k & 1);
    const size_t len = std::min(kStageBytes, bytes - off);
    if (pend_len[b]) {  // drain what this buffer holds
      ck(cudaEventSynchronize(ctx->stage_ev[b]), "event sync");
      par_memcpy(static_cast<char*>(h) + pend_off[b], ctx->stage[b], pend_len[b]);
    }
    ck(cudaMemcpyAsync(ctx->stage[b], static_cast<const char*>(d) + off, len,
                       cudaMemcpyDeviceToHost, ctx->stream),
       "D2H(staged)");
    ck(cudaEventRecord(ctx->stage_ev[b], ctx->stream), "event");
    pend_off[b] = off;
    pend_len[b] = len;
  }
  for (int b = 0; b < 2; ++b)
    if (pend_len[b]) {
      ck(cudaEventSynchronize(ctx->stage_ev[b]), "event sync");
      par_memcpy(static_cast<char*>(h) + pend_off[b], ctx->stage[b], pend_len[b]);
    }
}

// ---------------------------------------------------------------- GPTQ core (device pointers)
struct GptqBufs {
  int32_t* order;
  double* damp;
  void* a;     // n x n  T: factor input, overwritten by L
  void* ghi;   // n x n  T: G (tf32 hi part when split)
  float* glo;  // n x n  fp32 lo part (null: plain G in ghi)
  void* gpl;   // n x n  T: plain G (== ghi when not split)
  float* gtt;  // n x 128 fp32: diagonal blocks of G^T in in-block lane order
  int* flags;  // Cholesky tile flags
  void* acc;   // n x m  T: sweep partial sums
  void* dpl[2];   // D, K-major: split -- dpl[0] m x n (every row); else m x 512 by parity
  float* dhi[2];  // D tf32 hi / lo (split only: [0] m x n)
  float* dlo[2];
  int* kflag;     // split-K tile flags of the left-looking sweep GEMMs (split only)
  float* lhi;     // n x n: tf32 hi / lo split of L (split only; the Cholesky's tcgen05 products)
  float* llo;
  void* tab;      // one super-block's sweep table (split only)
  float* tcws;
  size_t tcws_floats;
};

long long chol_macro_cols(uint64_t n) {
  if (const char* e = getenv("OCWG_CHOL_MACRO")) return atoll(e);
  return n <= 4608 ? 0 : 2048;
}

// G / D stored as tf32 hi/lo pairs for the tcgen05 3xTF32 trailing GEMM
bool split_g(const ocwg_ctx* ctx, uint64_t n) {
  return ctx->precision == OCWG_FP32 && ctx->tensor_core_gemm && n % 4 == 0;
}

size_t tc_ws_floats(uint64_t n) {
  // largest mm<float> of the factorisation: the macro-panel trailing SYRK
  // (n x n x macro) and the parity-artefact inverse doubling (<= 2 n^2 per level)
  const long long nn = (long long)n;
  const long long mc = std::max<long long>(64, chol_macro_cols(n) > 0 ? chol_macro_cols(n) : 64);
  return std::max(tc_gemm_workspace_floats(nn, nn, mc), size_t(2 * nn * nn + 4 * nn * 4 + 64));
}

void gptq_reserve(Arena& ar, const ocwg_ctx* ctx, uint64_t n, uint64_t m, size_t* o) {
  const size_t es = ctx->precision == OCWG_FP64 ? 8 : 4;
  const bool split = split_g(ctx, n);
  const size_t de = sweep_delta_elems((long long)std::max<uint64_t>(m, 1));
  o[0] = ar.reserve(n * sizeof(int32_t));
  o[1] = ar.reserve(sizeof(double));
  o[2] = ar.reserve(n * n * es);
  o[3] = ar.reserve(n * n * es);
  o[4] = ar.reserve(split ? 2 * n * n * 4 : 0);
  o[5] = ar.reserve(cholesky_flag_ints((long long)n) * sizeof(int));
  o[6] = ar.reserve(n * std::max<uint64_t>(m, 1) * es);
  o[7] = ar.reserve(split ? n * m * 4 : 2 * de * es);
  o[8] = ar.reserve(split ? 2 * n * m * 4 : 0);
  o[9] = ar.reserve(tc_ws_floats(n) * sizeof(float));
  o[10] = ar.reserve(split ? n * 128 * 4 + 1024 : 0);
  o[11] = ar.reserve(split ? sweep_kflag_ints((long long)n, (long long)m) * sizeof(int) : 0);
  o[12] = ar.reserve(split ? 2 * n * n * 4 : 0);
  o[13] = ar.reserve(split ? sweep_table_bytes((long long)std::max<uint64_t>(m, 1)) : 0);
}
GptqBufs gptq_bufs(const Arena& ar, const ocwg_ctx* ctx, const size_t* o, uint64_t n, uint64_t m) {
  const size_t es = ctx->precision == OCWG_FP64 ? 8 : 4;
  const bool split = split_g(ctx, n);
  const size_t de = sweep_delta_elems((long long)std::max<uint64_t>(m, 1));
  GptqBufs b;
  b.order = ar.at<int32_t>(o[0]);
  b.damp = ar.at<double>(o[1]);
  b.a = ar.at<void>(o[2]);
  b.ghi = ar.at<void>(o[3]);
  b.glo = split ? ar.at<float>(o[4]) : nullptr;
  b.gpl = split ? static_cast<void*>(ar.at<float>(o[4]) + n * n) : b.ghi;
  b.flags = ar.at<int>(o[5]);
  b.acc = ar.at<void>(o[6]);
  b.dpl[0] = ar.at<char>(o[7]);
  b.dpl[1] = split ? nullptr : ar.at<char>(o[7]) + de * es;
  b.dhi[0] = split ? ar.at<float>(o[8]) : nullptr;
  b.dlo[0] = split ? ar.at<float>(o[8]) + n * m : nullptr;
  b.dhi[1] = b.dlo[1] = nullptr;
  b.kflag = split ? ar.at<int>(o[11]) : nullptr;
  b.lhi = split ? ar.at<float>(o[12]) : nullptr;
  b.llo = split ? ar.at<float>(o[12]) + n * n : nullptr;
  b.tab = split ? ar.at<void>(o[13]) : nullptr;
  b.tcws = ar.at<float>(o[9]);
  b.tcws_floats = tc_ws_floats(n);
  b.gtt = split ? ar.at<float>(o[10]) : nullptr;
  return b;
}

template <typename T>
void run_factor_t(ocwg_ctx* ctx, const float* h_dev, uint64_t n, int actorder, double percdamp,
                  const GptqBufs& b) {
  cudaStream_t st = ctx->stream;
  set_tc_workspace(ctx->tensor_core_gemm ? b.tcws : nullptr, b.tcws_floats);
  // damp first, leaving a contiguous diag(H) in the factor-input buffer (the
  // build below overwrites it) so the act-order rank count reads it coalesced
  float* diag = actorder ? static_cast<float*>(b.a) : nullptr;
  launch_damp(h_dev, (long long)n, percdamp, b.damp, diag, st);
  launch_order(diag, (long long)n, actorder, b.order, st);
  launch_build_factor_input<T>(h_dev, (long long)n, b.order, percdamp, static_cast<T*>(b.a), b.damp,
                               st, /*damp_ready=*/true);
  if (ctx->profile) cudaEventRecord(ctx->ev[1], st);
  cholesky_g<T>(static_cast<T*>(b.a), (long long)n, static_cast<T*>(b.ghi), b.glo,
                b.glo ? static_cast<float*>(b.gpl) : nullptr, b.gtt, b.flags, ctx->flag,
                chol_macro_cols(n), st, b.lhi, b.llo);
  if (ctx->profile) {
    cudaEventRecord(ctx->ev[2], st);
    cudaEventRecord(ctx->ev[3], st);  // (no triangular inverse on the hot path)
  }
}

// order + damp + Cholesky (L, G) on device; the reference's :29-51
void run_factor(ocwg_ctx* ctx, const float* h_dev, uint64_t n, int actorder, double percdamp,
                const GptqBufs& b) {
  if (ctx->precision == OCWG_FP64)
    run_factor_t<double>(ctx, h_dev, n, actorder, percdamp, b);
  else
    run_factor_t<float>(ctx, h_dev, n, actorder, percdamp, b);
}

template <typename T>
void run_sweep_t(ocwg_ctx* ctx, const float* w, uint64_t ldw, uint64_t n, uint64_t m, const QCfg& c,
                 const ocwg_gptq_options* opts, int16_t* codes, const float* scales,
                 const int32_t* zeros, float* w_hat, const GptqBufs& b) {
  T* const dp[2] = {static_cast<T*>(b.dpl[0]), static_cast<T*>(b.dpl[1])};
  float* const dh[2] = {b.dhi[0], b.dhi[1]};
  float* const dl[2] = {b.dlo[0], b.dlo[1]};
  gptq_sweep_g<T>(w, (long long)ldw, (long long)n, (long long)m, static_cast<const T*>(b.gpl),
                  b.gtt, static_cast<const T*>(b.ghi), b.glo, b.order, c, scales, zeros,
                  (long long)opts->block_cols, codes, w_hat, (long long)ldw, static_cast<T*>(b.acc),
                  dp, dh, dl, b.kflag, ctx->stream, b.tab, ctx->aux, ctx->sev + 3);
}

// gptq_quantize on device buffers (w row stride ldw; codes/w_hat stride ldw)
// w_ready (optional): event after which W is resident -- only the grids and
// the sweep wait for it, the factorisation (H only) does not.
void run_gptq(ocwg_ctx* ctx, const float* w, uint64_t ldw, const float* h_dev, uint64_t n,
              uint64_t m, const ocwg_quant_config* cfg, const ocwg_gptq_options* opts, int mode,
              int16_t* codes, float* scales, int32_t* zeros, float* w_hat, const GptqBufs& b,
              float* mm_ws, cudaEvent_t w_ready = nullptr) {
  const QCfg c = qcfg(cfg, m);
  if (ctx->profile) cudaEventRecord(ctx->ev[0], ctx->stream);
  // the grids depend on W only (quant.cpp:168-196): they are calibrated on the
  // auxiliary stream while the latency-bound factorisation runs
  const bool overlap = !ctx->profile;
  if (!overlap && w_ready) ck(cudaStreamWaitEvent(ctx->stream, w_ready, 0), "event");
  if (overlap) {
    ck(cudaEventRecord(ctx->sev[0], ctx->stream), "event");
    ck(cudaStreamWaitEvent(ctx->aux, ctx->sev[0], 0), "event");
    if (w_ready) ck(cudaStreamWaitEvent(ctx->aux, w_ready, 0), "event");
    launch_calibrate_grids(w, (long long)n, (long long)m, (long long)ldw, c, mode, scales, zeros,
                           ctx->flag, mm_ws, ctx->aux);
    ck(cudaEventRecord(ctx->sev[1], ctx->aux), "event");
  }
  run_factor(ctx, h_dev, n, opts->actorder, opts->percdamp, b);
  if (overlap) {
    ck(cudaStreamWaitEvent(ctx->stream, ctx->sev[1], 0), "event");
  } else {
    launch_calibrate_grids(w, (long long)n, (long long)m, (long long)ldw, c, mode, scales, zeros,
                           ctx->flag, mm_ws, ctx->stream);
  }
  if (ctx->profile) cudaEventRecord(ctx->ev[4], ctx->stream);
  if (ctx->precision == OCWG_FP64)
    run_sweep_t<double>(ctx, w, ldw, n, m, c, opts, codes, scales, zeros, w_hat, b);
  else
    run_sweep_t<float>(ctx, w, ldw, n, m, c, opts, codes, scales, zeros, w_hat, b);
  if (ctx->profile) {
    cudaEventRecord(ctx->ev[5], ctx->stream);
    cudaEventSynchronize(ctx->ev[5]);
    for (int k = 0; k < 5; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev[k], ctx->ev[k + 1]);
      ctx->phase_ms[k] = ms;
    }
  }
}

void check_gptq_args(const ocwg_quant_config* cfg, const ocwg_gptq_options* opts, uint64_t n,
                     uint64_t m) {
  validate(cfg);  // layerwise.cpp:22
  if (!opts) fail(OCWG_INVALID_INPUT, "gptq_quantize: null options");
  if (!(opts->percdamp > 0.0) || opts->percdamp > 1.0)  // :25-26
    fail(OCWG_INVALID_INPUT, "gptq_quantize: percdamp must be in (0, 1]");
  (void)n;
  (void)m;
}

// H (+)= X^T X of bf16 X (device, tokens x n) on the tensor cores, any n:
// rows are re-strided to a multiple of 8 elements (TMA's 16-byte row pitch)
// into `pad` (hessian_pad_bytes) when n % 8 != 0.
size_t hessian_pad_bytes(uint64_t tokens, uint64_t n) {
  return n % 8 ? size_t(tokens) * size_t((n + 7) / 8 * 8) * 2 : 0;
}
void run_hessian(const uint16_t* x, uint64_t tokens, uint64_t n, float* h, bool accumulate,
                 void* gws, size_t gws_bytes, uint16_t* pad, cudaStream_t st) {
  if (tokens == 0) {
    if (!accumulate) ck(cudaMemsetAsync(h, 0, n * n * 4, st), "memset");
    return;
  }
  GramSpec s;
  s.tokens = (long long)tokens;
  s.dim = (long long)n;
  s.ld = (long long)n;
  s.ops[0] = x;
  if (n % 8) {
    s.ld = (long long)((n + 7) / 8 * 8);
    launch_pad_bf16(x, (long long)tokens, (long long)n, s.ld, pad, st);
    s.ops[0] = pad;
  }
  s.nops = 1;
  s.gseg = 1;
  s.gram = h;
  s.accumulate = accumulate;
  static const long long window = [] {  // tuning switch: OCWG_HESSIAN_WINDOW tokens
    const char* e = getenv("OCWG_HESSIAN_WINDOW");
    return e ? atoll(e) : 0LL;
  }();
  s.window_tokens = window;
  const int r = gram_tc(s, gws, gws_bytes, st);
  if (r == -1) fail(OCWG_INVALID_INPUT, "hessian: shape outside the tensor-core kernel's range");
  if (r != 0) fail(OCWG_CUDA_ERROR, "hessian: tensor-core kernel launch failed");
}

}  // namespace

extern "C" {

const char* ocwg_last_error(void) { return g_err.c_str(); }
int ocwg_version(void) { return 1; }

int ocwg_create(int device, ocwg_ctx** out) {
  return guard([&] {
    if (!out) fail(OCWG_INVALID_INPUT, "null out");
    int n = 0;
    ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) fail(OCWG_CUDA_ERROR, "no such CUDA device");
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new ocwg_ctx;
    c->device = device;
    ck(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own;
    ck(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking), "cudaStreamCreate(aux)");
    ck(cudaStreamCreateWithFlags(&c->cpy, cudaStreamNonBlocking), "cudaStreamCreate(cpy)");
    for (auto& e : c->sev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaMalloc(&c->flag, sizeof(unsigned)), "cudaMalloc(flag)");
    ck(cudaMallocHost(&c->flag_host, sizeof(unsigned)), "cudaMallocHost(flag)");
    *out = c;
  });
}

int ocwg_destroy(ocwg_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->ws) cudaFree(ctx->ws);
    cudaFree(ctx->flag);
    cudaFreeHost(ctx->flag_host);
    cudaStreamSynchronize(ctx->aux);
    for (auto& e : ctx->sev) cudaEventDestroy(e);
    for (auto& e : ctx->ev)
      if (e) cudaEventDestroy(e);
    cudaStreamSynchronize(ctx->cpy);
    for (auto& e : ctx->cev) cudaEventDestroy(e);
    if (ctx->io) cudaFree(ctx->io);
    for (int b = 0; b < 2; ++b) {
      if (ctx->stage[b]) cudaFreeHost(ctx->stage[b]);
      if (ctx->stage_ev[b]) cudaEventDestroy(ctx->stage_ev[b]);
    }
    cudaStreamDestroy(ctx->cpy);
    cudaStreamDestroy(ctx->aux);
    cudaStreamDestroy(ctx->own);
    delete ctx;
  });
}

int ocwg_set_stats_layout(ocwg_ctx* ctx, int layout) {
  return guard([&] {
    if (!ctx) fail(OCWG_INVALID_INPUT, "null context");
    if (layout != OCWG_ROW_MAJOR && layout != OCWG_COL_MAJOR)
      fail(OCWG_INVALID_INPUT, "layout must be OCWG_ROW_MAJOR or OCWG_COL_MAJOR");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->stats_colmajor = layout == OCWG_COL_MAJOR;
  });
}

int ocwg_set_precision(ocwg_ctx* ctx, int precision) {
  return guard([&] {
    if (!ctx) fail(OCWG_INVALID_INPUT, "null context");
    if (precision != OCWG_FP32 && precision != OCWG_FP64)
      fail(OCWG_INVALID_INPUT, "precision must be OCWG_FP32 or OCWG_FP64");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->precision = precision;
  });
}

int ocwg_debug_profile(ocwg_ctx* ctx, int on, double* phase_ms) {
  return guard([&] {
    if (!ctx) fail(OCWG_INVALID_INPUT, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (on && !ctx->ev[0])
      for (auto& e : ctx->ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    ctx->profile = on != 0;
    if (phase_ms)
      for (int k = 0; k < 5; ++k) phase_ms[k] = ctx->phase_ms[k];
  });
}

int ocwg_set_stream(ocwg_ctx* ctx, void* s) {
  return guard([&] {
    if (!ctx) fail(OCWG_INVALID_INPUT, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->stream = static_cast<cudaStream_t>(s);  // NULL = the legacy default stream
  });
}

int ocwg_set_async(ocwg_ctx* ctx, int on) {
  return guard([&] {
    if (!ctx) fail(OCWG_INVALID_INPUT, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->async_dev = on != 0;
  });
}

int ocwg_synchronize(ocwg_ctx* ctx) {
  return guard([&] {
    if (!ctx) fail(OCWG_INVALID_INPUT, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    // drain, read and clear the (sticky) status word of async device calls
    ck(cudaGetLastError(), "kernel launch");
    ck(cudaMemcpyAsync(ctx->flag_host, ctx->flag, sizeof(unsigned), cudaMemcpyDeviceToHost,
                       ctx->stream),
       "status D2H");
    ck(cudaMemsetAsync(ctx->flag, 0, sizeof(unsigned), ctx->stream), "reset status");
    ck(cudaStreamSynchronize(ctx->stream), "stream synchronize");
    const unsigned f = *ctx->flag_host;
    if (f & kFlagNotPD)
      fail(OCWG_NUMERIC_ERROR, "gptq_quantize: Gram matrix is not positive definite after dampening");
    if (f & kFlagNonFinite) fail(OCWG_INVALID_INPUT, "calibrate_grids: non-finite entry");
  });
}

uint64_t ocwg_launch_count(ocwg_ctx*) { return launches_issued(); }

int ocwg_debug_factor_bench(ocwg_ctx* ctx, int iters, long long* cycles, float* l_out) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    Arena ar(ctx);
    const size_t oc = ar.reserve(64), oo = ar.reserve(64 * 64 * 4);
    ar.commit();
    debug_factor_bench(iters, ar.at<long long>(oc), ar.at<float>(oo), ctx->stream);
    d2h(cycles, ar.at<long long>(oc), 8 * 8, ctx);
    d2h(l_out, ar.at<float>(oo), 64 * 64 * 4, ctx);
    finish(ctx);
  });
}

int ocwg_debug_sweep_trace(ocwg_ctx* ctx, unsigned long long* out, int cap) {
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaDeviceSynchronize();
  return debug_sweep_trace(out, cap);
}

int ocwg_debug_gemm(ocwg_ctx* ctx, int precision, uint64_t m, uint64_t n, uint64_t k, double alpha,
                    const void* a, uint64_t lda, int ta, const void* b, uint64_t ldb, int tb,
                    double beta, void* c, uint64_t ldc, int lower_only, int reps, double* ms) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventRecord(e0, ctx->stream), "event");
    float* tcws = nullptr;
    size_t tcf = 0;
    if (precision == 2) {  // tcgen05 3xTF32 path
      tcf = tc_gemm_workspace_floats((long long)m, (long long)n, (long long)k);
      Arena ar(ctx);
      const size_t o = ar.reserve(tcf * 4);
      ar.commit();
      tcws = ar.at<float>(o);
    }
    for (int r = 0; r < reps; ++r) {
      if (precision == 2) {
        if (!tc_gemm_tf32x3(1, (long long)m, (long long)n, (long long)k, float(alpha),
                            static_cast<const float*>(a), (long long)lda, 0, ta != 0,
                            static_cast<const float*>(b), (long long)ldb, 0, tb != 0, float(beta),
                            static_cast<float*>(c), (long long)ldc, 0, lower_only != 0, tcws, tcf,
                            ctx->stream))
          fail(OCWG_UNSUPPORTED, "tc_gemm_tf32x3 rejected the shape");
      } else if (precision == OCWG_FP64)
        gemm<double, double, double>((long long)m, (long long)n, (long long)k, alpha,
                                     static_cast<const double*>(a), (long long)lda, ta != 0,
                                     static_cast<const double*>(b), (long long)ldb, tb != 0, beta,
                                     static_cast<double*>(c), (long long)ldc, lower_only != 0,
                                     ctx->stream);
      else
        gemm<float, float, float>((long long)m, (long long)n, (long long)k, alpha,
                                  static_cast<const float*>(a), (long long)lda, ta != 0,
                                  static_cast<const float*>(b), (long long)ldb, tb != 0, beta,
                                  static_cast<float*>(c), (long long)ldc, lower_only != 0,
                                  ctx->stream);
    }
    ck(cudaEventRecord(e1, ctx->stream), "event");
    finish(ctx);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    if (ms) *ms = t / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int ocwg_validate_config(const ocwg_quant_config* cfg) {
  return guard([&] { validate(cfg); });
}
uint64_t ocwg_group_count(const ocwg_quant_config* cfg, uint64_t rows, uint64_t cols) {
  return group_count(cfg, rows, cols);
}
uint64_t ocwg_storage_bytes(const ocwg_quant_config* cfg, uint64_t rows, uint64_t cols) {
  return storage_bytes(cfg, rows, cols);
}

// ------------------------------------------------------------------ quant.hpp
int ocwg_calibrate_grids(ocwg_ctx* ctx, const float* w, uint64_t rows, uint64_t cols,
                         const ocwg_quant_config* cfg, int mode, float* scales, int32_t* zeros) {
  return guard([&] {
    validate(cfg);
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const uint64_t ng = group_count(cfg, rows, cols);
    Arena ar(ctx);
    const size_t ow = ar.reserve(rows * cols * 4), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                 om = ar.reserve(4096 * 4);
    ar.commit();
    h2d(ar.at<float>(ow), w, rows * cols * 4, ctx);
    if (rows * cols > 0)
      launch_calibrate_grids(ar.at<float>(ow), (long long)rows, (long long)cols, (long long)cols,
                             qcfg(cfg, cols), mode, ar.at<float>(os), ar.at<int32_t>(oz),
                             ctx->flag, ar.at<float>(om), ctx->stream);
    finish(ctx);
    if (rows == 0 || cols == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
    d2h(scales, ar.at<float>(os), ng * 4, ctx);
    d2h(zeros, ar.at<int32_t>(oz), ng * 4, ctx);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int ocwg_candidate_grid(ocwg_ctx* ctx, const float* w, uint64_t rows, uint64_t cols, int mode,
                        const double* in_diag, double* errors, uint64_t* cost_bytes) {
  return guard([&] {
    if (mode != 0 && mode != 1) fail(OCWG_INVALID_INPUT, "unknown error mode");
    if (rows == 0 || cols == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
    for (int k = 0; k < 14; ++k) {  // autobit.cpp:47-58
      ocwg_quant_config c{};
      c.bits = 2 + k / 2;
      c.scheme = 0;                       // symmetric
      c.granularity = (k & 1) ? 1 : 2;    // grouped first, then per-channel
      c.group_size = 128;
      if (cost_bytes) cost_bytes[k] = storage_bytes(&c, rows, cols);
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    Arena ar(ctx);
    const size_t ow = ar.reserve(rows * cols * 4), od = ar.reserve(rows * 8),
                 op = ar.reserve(rows * 14 * 8), oe = ar.reserve(14 * 8);
    ar.commit();
    h2d(ar.at<float>(ow), w, rows * cols * 4, ctx);
    if (in_diag) h2d(ar.at<double>(od), in_diag, rows * 8, ctx);
    launch_candidate_grid(ar.at<float>(ow), (long long)rows, (long long)cols, (long long)cols, mode,
                          in_diag ? ar.at<double>(od) : nullptr, ar.at<double>(op),
                          ar.at<double>(oe), ctx->flag, ctx->stream);
    finish(ctx);
    d2h(errors, ar.at<double>(oe), 14 * 8, ctx);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int ocwg_quantize_matrix(ocwg_ctx* ctx, const float* w, uint64_t rows, uint64_t cols,
                         const ocwg_quant_config* cfg, int mode, int16_t* codes, float* scales,
                         int32_t* zeros) {
  return guard([&] {
    validate(cfg);
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const uint64_t ng = group_count(cfg, rows, cols);
    Arena ar(ctx);
    const size_t ow = ar.reserve(rows * cols * 4), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                 oc = ar.reserve(rows * cols * 2), om = ar.reserve(4096 * 4);
    ar.commit();
    const QCfg c = qcfg(cfg, cols);
    h2d(ar.at<float>(ow), w, rows * cols * 4, ctx);
    if (rows * cols > 0) {
      launch_calibrate_grids(ar.at<float>(ow), (long long)rows, (long long)cols, (long long)cols, c,
                             mode, ar.at<float>(os), ar.at<int32_t>(oz), ctx->flag,
                             ar.at<float>(om), ctx->stream);
      launch_quantize_rtn(ar.at<float>(ow), (long long)rows, (long long)cols, (long long)cols, c,
                          ar.at<float>(os), ar.at<int32_t>(oz), ar.at<int16_t>(oc), nullptr,
                          ctx->stream);
    }
    finish(ctx);
    if (rows == 0 || cols == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
    d2h(codes, ar.at<int16_t>(oc), rows * cols * 2, ctx);
    d2h(scales, ar.at<float>(os), ng * 4, ctx);
    d2h(zeros, ar.at<int32_t>(oz), ng * 4, ctx);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int ocwg_dequantize(ocwg_ctx* ctx, const int16_t* codes, const float* scales, const int32_t* zeros,
                    uint64_t rows, uint64_t cols, const ocwg_quant_config* cfg, float* out) {
  return guard([&] {
    validate(cfg);
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const uint64_t ng = group_count(cfg, rows, cols);
    Arena ar(ctx);
    const size_t oc = ar.reserve(rows * cols * 2), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                 oo = ar.reserve(rows * cols * 4);
    ar.commit();
    h2d(ar.at<int16_t>(oc), codes, rows * cols * 2, ctx);
    h2d(ar.at<float>(os), scales, ng * 4, ctx);
    h2d(ar.at<int32_t>(oz), zeros, ng * 4, ctx);
    if (rows * cols != 0)
      launch_dequantize(ar.at<int16_t>(oc), (long long)rows, (long long)cols, qcfg(cfg, cols),
                        ar.at<float>(os), ar.at<int32_t>(oz), ar.at<float>(oo), ctx->stream);
    d2h(out, ar.at<float>(oo), rows * cols * 4, ctx);
    finish(ctx);
  });
}

int ocwg_activation_objective(ocwg_ctx* ctx, const float* w, const float* w_hat, const float* h,
                              uint64_t n, uint64_t m, double* out) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    Arena ar(ctx);
    const size_t ow = ar.reserve(n * m * 4), owh = ar.reserve(n * m * 4), oh = ar.reserve(n * n * 4),
                 ows = ar.reserve(2 * n * m * 8), oo = ar.reserve(8);
    ar.commit();
    h2d(ar.at<float>(ow), w, n * m * 4, ctx);
    h2d(ar.at<float>(owh), w_hat, n * m * 4, ctx);
    h2d(ar.at<float>(oh), h, n * n * 4, ctx);
    activation_objective(ar.at<float>(ow), ar.at<float>(owh), ar.at<float>(oh), (long long)n,
                         (long long)m, ar.at<double>(oo), ar.at<double>(ows), ctx->stream);
    d2h(out, ar.at<double>(oo), 8, ctx);
    finish(ctx);
  });
}

// ------------------------------------------------------------------ jointq.hpp
namespace {
void jq_check_codes(const ocwg_quant_config* cfg, const int16_t* codes, uint64_t n, uint64_t m) {
  const QCfg c = qcfg(cfg, m);  // jointq.cpp:50-56
  for (uint64_t t = 0; t < n * m; ++t)
    if (codes[t] < c.qmin || codes[t] > c.qmax)
      fail(OCWG_INVALID_INPUT, "jointq: code outside the codebook range");
}
}  // namespace

int ocwg_jointq_refine(ocwg_ctx* ctx, const float* w, uint64_t n, uint64_t m, const float* x,
                       uint64_t tokens, const ocwg_quant_config* cfg, int16_t* codes,
                       float* scales, int32_t* zeros, double lambda, int max_passes,
                       int move_radius, double* trace, uint64_t trace_cap, uint64_t* trace_len,
                       uint64_t* accepted_moves, int* passes) {
  return guard([&] {
    validate(cfg);
    jq_check_codes(cfg, codes, n, m);
    if (!(lambda >= 0.0)) fail(OCWG_INVALID_INPUT, "jointq_refine: lambda must be >= 0");
    if (move_radius < 1) fail(OCWG_INVALID_INPUT, "jointq_refine: move_radius must be >= 1");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const uint64_t ng = group_count(cfg, n, m);
    const QCfg c = qcfg(cfg, m);
    const long long units = (long long)jointq_units(c, (long long)m);
    const long long max_cells = std::max<long long>(
        1, c.gran == 0 ? (long long)(n * m) : c.gran == 1 ? (long long)m : c.group);
    const long long log_cap = std::max<long long>(4096, (1LL << 24) / units);
    double obj0 = 0.0;
    std::vector<int> cnt(units, 0), fz(units, 0);
    std::vector<std::pair<unsigned long long, double>> moves;
    bool truncated = false;
    if (n * m > 0) {
      Arena ar(ctx);
      const size_t ox = ar.reserve(std::max<uint64_t>(1, tokens * n) * 4), ow = ar.reserve(n * m * 4),
                   oc = ar.reserve(n * m * 2), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                   oh = ar.reserve(n * n * 8), oe = ar.reserve(n * m * 8), og = ar.reserve(n * m * 8),
                   op = ar.reserve(256 * 8), odb = ar.reserve(size_t(units * max_cells) * 8),
                   olk = ar.reserve(size_t(units * log_cap) * 8),
                   old = ar.reserve(size_t(units * log_cap) * 8), olc = ar.reserve(units * 4),
                   ofz = ar.reserve(units * 4);
      const auto ta = std::chrono::steady_clock::now();
      ar.commit();
      if (tokens) h2d(ar.at<float>(ox), x, tokens * n * 4, ctx);
      else ck(cudaMemsetAsync(ar.at<float>(ox), 0, 4, ctx->stream), "memset");
      h2d(ar.at<float>(ow), w, n * m * 4, ctx);
      h2d(ar.at<int16_t>(oc), codes, n * m * 2, ctx);
      h2d(ar.at<float>(os), scales, ng * 4, ctx);
      h2d(ar.at<int32_t>(oz), zeros, ng * 4, ctx);
      const bool dbg = getenv("OCWG_DEBUG_JQ") != nullptr;
      auto tnow = [&] {
        if (dbg) cudaStreamSynchronize(ctx->stream);
        return std::chrono::steady_clock::now();
      };
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      const auto t0 = tnow();
      if (dbg) fprintf(stderr, "jointq: alloc + H2D %.1f ms\n", ms(ta, t0));
      obj0 = jointq_setup(ar.at<float>(ox), (long long)tokens, ar.at<float>(ow), (long long)n,
                          (long long)m, c, ar.at<int16_t>(oc), ar.at<float>(os), ar.at<int32_t>(oz),
                          lambda, ar.at<double>(oh), ar.at<double>(oe), ar.at<double>(og),
                          ar.at<double>(op), ctx->stream);
      if (max_passes > 0) {
        const int r = jointq_search(ar.at<float>(ow), (long long)n, (long long)m, c,
                                    ar.at<int16_t>(oc), ar.at<float>(os), ar.at<int32_t>(oz),
                                    ar.at<double>(oh), ar.at<double>(oe), ar.at<double>(og),
                                    ar.at<double>(odb), max_cells, obj0, max_passes, move_radius,
                                    ar.at<unsigned long long>(olk), ar.at<double>(old),
                                    ar.at<int>(olc), ar.at<int>(ofz), log_cap, ctx->stream);
        if (r != 0) fail(OCWG_CUDA_ERROR, "jointq_refine: search kernel launch failed");
      } else {
        ck(cudaMemsetAsync(ar.at<int>(olc), 0, units * 4, ctx->stream), "memset");
        ck(cudaMemsetAsync(ar.at<int>(ofz), 0, units * 4, ctx->stream), "memset");
      }
      const auto t2 = tnow();
      if (dbg) fprintf(stderr, "jointq: setup + search %.1f ms\n", ms(t0, t2));
      d2h(codes, ar.at<int16_t>(oc), n * m * 2, ctx);
      d2h(scales, ar.at<float>(os), ng * 4, ctx);
      d2h(zeros, ar.at<int32_t>(oz), ng * 4, ctx);
      d2h(cnt.data(), ar.at<int>(olc), units * 4, ctx);
      d2h(fz.data(), ar.at<int>(ofz), units * 4, ctx);
      ck(cudaStreamSynchronize(ctx->stream), "sync");
      // the reference's move order: keys (pass, phase, index) across the units
      std::vector<unsigned long long> kbuf;
      std::vector<double> dbuf;
      for (long long u = 0; u < units; ++u) {
        const long long k = std::min<long long>(cnt[u], log_cap);
        truncated |= cnt[u] > log_cap;
        if (k == 0) continue;
        kbuf.resize(k);
        dbuf.resize(k);
        ck(cudaMemcpy(kbuf.data(), ar.at<unsigned long long>(olk) + u * log_cap, k * 8,
                      cudaMemcpyDeviceToHost),
           "D2H");
        ck(cudaMemcpy(dbuf.data(), ar.at<double>(old) + u * log_cap, k * 8, cudaMemcpyDeviceToHost),
           "D2H");
        for (long long t = 0; t < k; ++t) moves.emplace_back(kbuf[t], dbuf[t]);
      }
      finish(ctx);
      if (dbg) fprintf(stderr, "jointq: results + logs %.1f ms\n", ms(t2, tnow()));
    }
    std::sort(moves.begin(), moves.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    uint64_t total = 0;
    int fzmax = 0;
    for (long long u = 0; u < (long long)cnt.size(); ++u) {
      total += uint64_t(cnt[u]);
      fzmax = std::max(fzmax, fz[u]);
    }
    if (accepted_moves) *accepted_moves = total;
    // jointq.cpp:248-250: a pass without an accepted move ends the search
    if (passes) *passes = max_passes <= 0 ? 0
                          : n * m == 0 ? 1
                                       : (fzmax < max_passes ? fzmax + 1 : max_passes);
    // trace: J at entry, then after each accepted move (0 entries: move log overflowed)
    const uint64_t len = truncated ? 0 : total + 1;
    if (trace_len) *trace_len = len;
    if (trace && len) {
      double j = obj0;
      if (trace_cap > 0) trace[0] = j;
      for (uint64_t t = 0; t < moves.size(); ++t) {
        j += moves[t].second;
        if (t + 1 < trace_cap) trace[t + 1] = j;
      }
    }
  });
}

int ocwg_jointq_objective(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                          const int32_t* zeros, const float* w, uint64_t n, uint64_t m,
                          const float* x, uint64_t tokens, const ocwg_quant_config* cfg,
                          double lambda, double* out) {
  return guard([&] {
    validate(cfg);
    if (!(lambda >= 0.0)) fail(OCWG_INVALID_INPUT, "jointq_objective: lambda must be >= 0");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    *out = 0.0;
    if (n * m == 0) return;
    const uint64_t ng = group_count(cfg, n, m);
    const QCfg c = qcfg(cfg, m);
    const long long chunk = std::max<long long>(1, std::min<long long>((long long)tokens,
                                                                       (1LL << 26) / (long long)m));
    Arena ar(ctx);
    const size_t ox = ar.reserve(std::max<uint64_t>(1, tokens * n) * 4), ow = ar.reserve(n * m * 4),
                 oc = ar.reserve(n * m * 2), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                 oe = ar.reserve(n * m * 8), oy = ar.reserve(size_t(chunk) * m * 8),
                 op = ar.reserve(256 * 8);
    ar.commit();
    if (tokens) h2d(ar.at<float>(ox), x, tokens * n * 4, ctx);
    h2d(ar.at<float>(ow), w, n * m * 4, ctx);
    h2d(ar.at<int16_t>(oc), codes, n * m * 2, ctx);
    h2d(ar.at<float>(os), scales, ng * 4, ctx);
    h2d(ar.at<int32_t>(oz), zeros, ng * 4, ctx);
    jointq_residual(ar.at<int16_t>(oc), ar.at<float>(os), ar.at<int32_t>(oz), ar.at<float>(ow),
                    (long long)n, (long long)m, c, ar.at<double>(oe), ctx->stream);
    *out = jointq_objective_dev(ar.at<float>(ox), (long long)tokens, (long long)n, (long long)m,
                                ar.at<double>(oe), lambda, ar.at<double>(oy), chunk,
                                ar.at<double>(op), ctx->stream);
    finish(ctx);
  });
}

int ocwg_jointq_optimal_group_scale(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                                    const int32_t* zeros, const float* w, uint64_t n, uint64_t m,
                                    const float* x, uint64_t tokens, const ocwg_quant_config* cfg,
                                    double lambda, uint64_t group, double* out) {
  return guard([&] {
    validate(cfg);
    jq_check_codes(cfg, codes, n, m);
    const uint64_t ng = group_count(cfg, n, m);
    if (group >= ng) fail(OCWG_INVALID_INPUT, "jointq: group index out of range");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const QCfg c = qcfg(cfg, m);
    Arena ar(ctx);
    const size_t ox = ar.reserve(std::max<uint64_t>(1, tokens * n) * 4), ow = ar.reserve(n * m * 4),
                 oc = ar.reserve(n * m * 2), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                 oh = ar.reserve(n * n * 8), oe = ar.reserve(n * m * 8), og = ar.reserve(n * m * 8),
                 op = ar.reserve(256 * 8);
    ar.commit();
    if (tokens) h2d(ar.at<float>(ox), x, tokens * n * 4, ctx);
    else ck(cudaMemsetAsync(ar.at<float>(ox), 0, 4, ctx->stream), "memset");
    h2d(ar.at<float>(ow), w, n * m * 4, ctx);
    h2d(ar.at<int16_t>(oc), codes, n * m * 2, ctx);
    h2d(ar.at<float>(os), scales, ng * 4, ctx);
    h2d(ar.at<int32_t>(oz), zeros, ng * 4, ctx);
    jointq_setup(ar.at<float>(ox), (long long)tokens, ar.at<float>(ow), (long long)n, (long long)m,
                 c, ar.at<int16_t>(oc), ar.at<float>(os), ar.at<int32_t>(oz), lambda,
                 ar.at<double>(oh), ar.at<double>(oe), ar.at<double>(og), ar.at<double>(op),
                 ctx->stream);
    *out = jointq_optimal_scale(ar.at<float>(ow), (long long)n, (long long)m, c, ar.at<int16_t>(oc),
                                ar.at<float>(os), ar.at<int32_t>(oz), ar.at<double>(oh),
                                ar.at<double>(oe), ar.at<double>(og), (long long)group,
                                ar.at<double>(op), ctx->stream);
    finish(ctx);
  });
}

// ------------------------------------------------------------------ packing
int ocwg_pack_uniform_dev(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                          const int32_t* zeros, uint64_t rows, uint64_t cols,
                          const ocwg_quant_config* cfg, uint8_t* out) {
  return guard([&] {
    validate(cfg);
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    launch_pack(codes, (long long)(rows * cols), (long long)group_count(cfg, rows, cols),
                qcfg(cfg, cols), scales, zeros, out, ctx->stream);
    finish_dev(ctx);
  });
}

int ocwg_pack_uniform(ocwg_ctx* ctx, const int16_t* codes, const float* scales,
                      const int32_t* zeros, uint64_t rows, uint64_t cols,
                      const ocwg_quant_config* cfg, uint8_t* out, uint64_t out_len) {
  return guard([&] {
    validate(cfg);
    const uint64_t need = storage_bytes(cfg, rows, cols);
    if (out_len < need) fail(OCWG_INVALID_INPUT, "pack_uniform: output buffer too small");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const uint64_t ng = group_count(cfg, rows, cols);
    Arena ar(ctx);
    const size_t oc = ar.reserve(rows * cols * 2), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                 oo = ar.reserve(need);
    ar.commit();
    h2d(ar.at<int16_t>(oc), codes, rows * cols * 2, ctx);
    h2d(ar.at<float>(os), scales, ng * 4, ctx);
    h2d(ar.at<int32_t>(oz), zeros, ng * 4, ctx);
    launch_pack(ar.at<int16_t>(oc), (long long)(rows * cols), (long long)ng, qcfg(cfg, cols),
                ar.at<float>(os), ar.at<int32_t>(oz), ar.at<uint8_t>(oo), ctx->stream);
    d2h(out, ar.at<uint8_t>(oo), need, ctx);
    finish(ctx);
  });
}

int ocwg_unpack_uniform(ocwg_ctx* ctx, const uint8_t* payload, uint64_t len, uint64_t rows,
                        uint64_t cols, const ocwg_quant_config* cfg, int16_t* codes, float* scales,
                        int32_t* zeros) {
  return guard([&] {
    validate(cfg);
    if (len != storage_bytes(cfg, rows, cols))  // container.cpp:197
      fail(OCWG_IO_ERROR, "container: uniform payload size mismatch");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const uint64_t ng = group_count(cfg, rows, cols);
    Arena ar(ctx);
    const size_t op = ar.reserve(len), oc = ar.reserve(rows * cols * 2), os = ar.reserve(ng * 4),
                 oz = ar.reserve(ng * 4);
    ar.commit();
    h2d(ar.at<uint8_t>(op), payload, len, ctx);
    launch_unpack(ar.at<uint8_t>(op), (long long)(rows * cols), (long long)ng, qcfg(cfg, cols),
                  ar.at<int16_t>(oc), ar.at<float>(os), ar.at<int32_t>(oz), ctx->stream);
    d2h(codes, ar.at<int16_t>(oc), rows * cols * 2, ctx);
    d2h(scales, ar.at<float>(os), ng * 4, ctx);
    d2h(zeros, ar.at<int32_t>(oz), ng * 4, ctx);
    finish(ctx);
  });
}

// ------------------------------------------------------------------ stats.hpp
int ocwg_accumulate_stats(ocwg_ctx* ctx, const float* x_fp, const float* x_pert, uint64_t rows,
                          uint64_t dim, double* gram, double* cross, uint64_t* token_count) {
  return guard([&] {
    if (!gram) fail(OCWG_INVALID_INPUT, "accumulate_stats: null gram");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    // cross += Xp^T (X - Xp) is identically zero when X == Xp: skip it
    const bool same = (x_fp == x_pert), want_cross = cross && !same;
    if (rows == 0 || dim == 0) {
      if (token_count) *token_count += rows;
      return;
    }
    cudaStream_t st = ctx->stream;
    if (ctx->precision == OCWG_FP64) {  // the reference's arithmetic class: fp64 SIMT GEMMs
      Arena ar(ctx);
      const size_t of = ar.reserve(rows * dim * 4), op = ar.reserve(rows * dim * 4),
                   og = ar.reserve(dim * dim * 8), oc = ar.reserve(dim * dim * 8),
                   od = ar.reserve(want_cross ? rows * dim * 8 : 8);
      ar.commit();
      h2d(ar.at<float>(op), x_pert, rows * dim * 4, ctx);
      if (!same) h2d(ar.at<float>(of), x_fp, rows * dim * 4, ctx);
      h2d(ar.at<double>(og), gram, dim * dim * 8, ctx);
      if (want_cross) h2d(ar.at<double>(oc), cross, dim * dim * 8, ctx);
      if (ctx->stats_colmajor) {
        transpose_sq_f64(ar.at<double>(og), (long long)dim, st);
        if (want_cross) transpose_sq_f64(ar.at<double>(oc), (long long)dim, st);
      }
      const float* xf = same ? ar.at<float>(op) : ar.at<float>(of);
      accumulate_stats_f64(xf, ar.at<float>(op), (long long)rows, (long long)dim, ar.at<double>(og),
                           want_cross ? ar.at<double>(oc) : nullptr, ar.at<double>(od), st);
      if (ctx->stats_colmajor) {
        transpose_sq_f64(ar.at<double>(og), (long long)dim, st);
        if (want_cross) transpose_sq_f64(ar.at<double>(oc), (long long)dim, st);
      }
      d2h(gram, ar.at<double>(og), dim * dim * 8, ctx);
      if (want_cross) d2h(cross, ar.at<double>(oc), dim * dim * 8, ctx);
      finish(ctx);
    } else {
      // tensor cores: X_hat = P1 + P2, X - X_hat = D1 + D2 (bf16 parts), fp64 outputs.
      // Token chunks are pipelined: the staged copy of chunk k+1 (host memcpy into
      // pinned staging + DMA on ctx->cpy) runs while chunk k is split and
      // accumulated on ctx->stream; the fp32 chunk buffers are double-buffered.
      const uint64_t ld = (dim + 7) / 8 * 8;
      const uint64_t chunk = std::min<uint64_t>(rows, 32768);  // a multiple of the 8192-token window
      const uint64_t nch = (rows + chunk - 1) / chunk;
      Arena ar(ctx);
      size_t op[2], of[2];
      for (int b = 0; b < 2; ++b) {
        op[b] = ar.reserve(chunk * dim * 4);
        of[b] = ar.reserve(want_cross ? chunk * dim * 4 : 4);
      }
      const size_t o1 = ar.reserve(chunk * ld * 2), o2 = ar.reserve(chunk * ld * 2),
                   o3 = ar.reserve(want_cross ? chunk * ld * 2 : 16),
                   o4 = ar.reserve(want_cross ? chunk * ld * 2 : 16), og = ar.reserve(dim * dim * 8),
                   oc = ar.reserve(want_cross ? dim * dim * 8 : 8), ofl = ar.reserve(16),
                   ows = ar.reserve(gram_tc_workspace_bytes((long long)dim));
      ar.commit();
      const bool dbg = getenv("OCWG_DEBUG_STATS") != nullptr;
      const auto t0 = std::chrono::steady_clock::now();
      h2d_big(ar.at<double>(og), gram, dim * dim * 8, ctx);
      if (want_cross) h2d_big(ar.at<double>(oc), cross, dim * dim * 8, ctx);
      if (ctx->stats_colmajor) {
        transpose_sq_f64(ar.at<double>(og), (long long)dim, st);
        if (want_cross) transpose_sq_f64(ar.at<double>(oc), (long long)dim, st);
      }
      cudaEvent_t ev_free[2], ev_copied[2];
      for (int b = 0; b < 2; ++b) {
        ck(cudaEventCreateWithFlags(&ev_free[b], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&ev_copied[b], cudaEventDisableTiming), "cudaEventCreate");
      }
      struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
          for (int b = 0; b < 4; ++b) cudaEventDestroy(e[b]);
        }
      };
      cudaEvent_t evs[4] = {ev_free[0], ev_free[1], ev_copied[0], ev_copied[1]};
      EvGuard guard_ev{evs};
      bool freed[2] = {false, false};
      auto copy_chunk = [&](uint64_t k) {  // tokens of chunk k -> slot k & 1
        const int b = int(k & 1);
        const uint64_t t0k = k * chunk, len = std::min(chunk, rows - t0k);
        h2d_staged_async(ar.at<float>(op[b]), x_pert + t0k * dim, len * dim * 4, ctx,
                         freed[b] ? ev_free[b] : nullptr, nullptr);
        if (want_cross)
          h2d_staged_async(ar.at<float>(of[b]), x_fp + t0k * dim, len * dim * 4, ctx, nullptr,
                           nullptr);
        ck(cudaEventRecord(ev_copied[b], ctx->cpy), "event");
      };
      uint16_t *p1 = ar.at<uint16_t>(o1), *p2 = ar.at<uint16_t>(o2), *d1 = ar.at<uint16_t>(o3),
               *d2 = ar.at<uint16_t>(o4);
      unsigned* fl = ar.at<unsigned>(ofl);
      copy_chunk(0);
      for (uint64_t k = 0; k < nch; ++k) {
        const int b = int(k & 1);
        const uint64_t len = std::min(chunk, rows - k * chunk);
        ck(cudaStreamWaitEvent(st, ev_copied[b], 0), "event");
        ck(cudaMemsetAsync(fl, 0, 4, st), "memset");
        launch_split_bf16(ar.at<float>(op[b]), want_cross ? ar.at<float>(of[b]) : nullptr,
                          (long long)len, (long long)dim, (long long)ld, p1, p2, d1, d2, fl, st);
        ck(cudaEventRecord(ev_free[b], st), "event");  // the split has read slot b
        freed[b] = true;
        if (k + 1 < nch) copy_chunk(k + 1);  // (host staging overlaps the split / gram on st)
        unsigned f = 0;
        d2h(&f, fl, 4, ctx);
        ck(cudaStreamSynchronize(st), "sync");
        if (dbg) fprintf(stderr, "accumulate_stats: chunk %llu split flags %u\n", (unsigned long long)k, f);
        GramSpec s;
        s.tokens = (long long)len;
        s.dim = (long long)dim;
        s.ld = (long long)ld;
        s.ops[0] = p1;
        s.ops[1] = p2;
        s.ops[2] = d1;
        s.ops[3] = d2;
        s.nops = 4;
        // gram = P1'P1 (+ P1'P2 + P2'P1 when X_hat is not bf16-exact)
        s.gseg = (f & 1u) ? 3 : 1;
        const int ga[3] = {0, 0, 1}, gb[3] = {0, 1, 0};
        // cross = P1'D1 + P1'D2 + P2'D1
        s.cseg = (want_cross && (f & 2u)) ? 3 : 0;
        const int ca[3] = {0, 0, 1}, cb[3] = {2, 3, 2};
        for (int q = 0; q < 3; ++q) s.gA[q] = ga[q], s.gB[q] = gb[q], s.cA[q] = ca[q], s.cB[q] = cb[q];
        s.gram = ar.at<double>(og);
        s.cross = ar.at<double>(oc);
        s.f64 = true;
        s.accumulate = true;
        // fp32 TMEM accumulations of 8192 tokens, fp64 across windows (measured at
        // C2: 2048 -> 8192-token windows take the kernel from 273 to 75 ms, the
        // error still set by the bf16 split, ~7e-6)
        s.window_tokens = 8192;
        if (s.gseg > 0 || s.cseg > 0) {
          const int r = gram_tc(s, ar.at<void>(ows), gram_tc_workspace_bytes((long long)dim), st);
          if (r != 0) fail(OCWG_CUDA_ERROR, "accumulate_stats: tensor-core kernel launch failed");
        }
      }
      if (ctx->stats_colmajor) {
        transpose_sq_f64(ar.at<double>(og), (long long)dim, st);
        if (want_cross) transpose_sq_f64(ar.at<double>(oc), (long long)dim, st);
      }
      finish(ctx);
      if (dbg)
        fprintf(stderr, "accumulate_stats: pipelined H2D + split + gram %.1f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count());
      d2h_big(gram, ar.at<double>(og), dim * dim * 8, ctx);
      if (want_cross) d2h_big(cross, ar.at<double>(oc), dim * dim * 8, ctx);
    }
    if (token_count) *token_count += rows;
  });
}

int ocwg_hessian_bf16_dev(ocwg_ctx* ctx, const uint16_t* x, uint64_t tokens, uint64_t dim,
                          float* h, int accumulate) {
  return ocwg_debug_hessian_dev(ctx, x, tokens, dim, h, accumulate, 0);
}

int ocwg_debug_hessian_dev(ocwg_ctx* ctx, const uint16_t* x, uint64_t tokens, uint64_t dim,
                           float* h, int accumulate, int impl) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    if (tokens == 0) {
      if (!accumulate) ck(cudaMemsetAsync(h, 0, dim * dim * 4, ctx->stream), "memset");
    } else if (impl == 1) {
      hessian_simt(x, (long long)tokens, (long long)dim, h, accumulate, ctx->stream);
    } else {
      Arena ar(ctx);
      const size_t gb = gram_tc_workspace_bytes((long long)dim);
      const size_t o = ar.reserve(gb), op = ar.reserve(hessian_pad_bytes(tokens, dim));
      ar.commit();
      run_hessian(x, tokens, dim, h, accumulate != 0, ar.at<void>(o), gb, ar.at<uint16_t>(op),
                  ctx->stream);
    }
    finish_dev(ctx);
  });
}

int ocwg_debug_split_dev(ocwg_ctx* ctx, const float* xp, const float* xf, uint64_t rows,
                         uint64_t dim, uint64_t ld, uint16_t* p1, uint16_t* p2, uint16_t* d1,
                         uint16_t* d2, unsigned* flags) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    launch_split_bf16(xp, xf, (long long)rows, (long long)dim, (long long)ld, p1, p2, d1, d2, flags,
                      ctx->stream);
    finish_dev(ctx);
  });
}

int ocwg_debug_gram_dev(ocwg_ctx* ctx, const uint16_t* const* ops, int nops, uint64_t tokens,
                        uint64_t dim, uint64_t ld, int gseg, const int* ga, const int* gb, int cseg,
                        const int* ca, const int* cb, void* gram, void* cross, int f64,
                        int accumulate, int64_t window) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    GramSpec s;
    s.tokens = (long long)tokens;
    s.dim = (long long)dim;
    s.ld = (long long)ld;
    s.nops = nops;
    for (int k = 0; k < nops && k < 4; ++k) s.ops[k] = ops[k];
    s.gseg = gseg;
    s.cseg = cseg;
    for (int k = 0; k < 3; ++k) {
      s.gA[k] = k < gseg ? ga[k] : 0;
      s.gB[k] = k < gseg ? gb[k] : 0;
      s.cA[k] = k < cseg ? ca[k] : 0;
      s.cB[k] = k < cseg ? cb[k] : 0;
    }
    s.gram = gram;
    s.cross = cross;
    s.f64 = f64 != 0;
    s.accumulate = accumulate != 0;
    s.window_tokens = window;
    Arena ar(ctx);
    const size_t gbytes = gram_tc_workspace_bytes((long long)dim);
    const size_t o = ar.reserve(gbytes);
    ar.commit();
    const int r = gram_tc(s, ar.at<void>(o), gbytes, ctx->stream);
    if (r == -1) fail(OCWG_INVALID_INPUT, "gram_tc: unsupported shape / segment set");
    if (r != 0) fail(OCWG_CUDA_ERROR, "gram_tc launch failed");
    finish_dev(ctx);
  });
}

int ocwg_hessian_bf16(ocwg_ctx* ctx, const uint16_t* x, uint64_t tokens, uint64_t dim, float* h,
                      int accumulate) {
  return guard([&] {
    float* hd = nullptr;
    uint16_t* xd = nullptr;
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    ck(cudaMalloc(&hd, dim * dim * 4), "cudaMalloc(H)");
    ck(cudaMalloc(&xd, std::max<uint64_t>(1, tokens * dim * 2)), "cudaMalloc(X)");
    h2d(xd, x, tokens * dim * 2, ctx);
    if (accumulate) h2d(hd, h, dim * dim * 4, ctx);
    int r = ocwg_hessian_bf16_dev(ctx, xd, tokens, dim, hd, accumulate);
    std::string msg = g_err;
    if (r == OCWG_OK) {
      d2h(h, hd, dim * dim * 4, ctx);
      try {
        finish(ctx);  // host entry points always drain and report
      } catch (const Error& e) {
        r = e.code;
        msg = e.msg;
      }
    }
    cudaFree(hd);
    cudaFree(xd);
    if (r != OCWG_OK) fail(r, msg);
  });
}

// ------------------------------------------------------------------ layerwise.hpp
int ocwg_gptq_order(ocwg_ctx* ctx, const float* h, uint64_t n, int actorder, int64_t* order) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    Arena ar(ctx);
    const size_t oh = ar.reserve(n * n * 4), oo = ar.reserve(n * 4), od = ar.reserve(n * 4);
    ar.commit();
    h2d(ar.at<float>(oh), h, n * n * 4, ctx);
    if (n) {
      float* diag = ar.at<float>(od);  // diag(H), contiguous
      ck(cudaMemcpy2DAsync(diag, 4, ar.at<float>(oh), (n + 1) * 4, 4, n, cudaMemcpyDeviceToDevice,
                           ctx->stream), "diag copy");
      launch_order(diag, (long long)n, actorder, ar.at<int32_t>(oo), ctx->stream);
    }
    std::vector<int32_t> o(n);
    d2h(o.data(), ar.at<int32_t>(oo), n * 4, ctx);
    finish(ctx);
    for (uint64_t i = 0; i < n; ++i) order[i] = o[i];
  });
}

int ocwg_gptq_factor(ocwg_ctx* ctx, const float* h, uint64_t n, int actorder, double percdamp,
                     int64_t* order, double* hinv, double* u, double* damp) {
  return guard([&] {
    if (!(percdamp > 0.0) || percdamp > 1.0)
      fail(OCWG_INVALID_INPUT, "gptq_quantize: percdamp must be in (0, 1]");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    const size_t es = ctx->precision == OCWG_FP64 ? 8 : 4;
    const uint64_t nblk = (n + 63) / 64;
    Arena ar(ctx);
    size_t o[14];
    gptq_reserve(ar, ctx, n, 1, o);
    const size_t oh = ar.reserve(n * n * 4), ohi = ar.reserve(n * n * 8),
                 ou64 = ar.reserve(n * n * 8), ou = ar.reserve(n * n * es),
                 ouw = ar.reserve((nblk * 64 * 64 + n * n) * es);
    ar.commit();
    const GptqBufs b = gptq_bufs(ar, ctx, o, n, 1);
    h2d(ar.at<float>(oh), h, n * n * 4, ctx);
    run_factor(ctx, ar.at<float>(oh), n, actorder, percdamp, b);
    if (ctx->precision == OCWG_FP64) {
      double* ud = ar.at<double>(ou);
      upper_from_cholesky<double>(static_cast<double*>(b.a), (long long)n, ud, ar.at<double>(ouw),
                                  ctx->stream);
      if (hinv) launch_gram_upper<double>(ud, (long long)n, ar.at<double>(ohi), ctx->stream);
      d2h(u, ud, n * n * 8, ctx);
    } else {
      float* uf = ar.at<float>(ou);
      upper_from_cholesky<float>(static_cast<float*>(b.a), (long long)n, uf, ar.at<float>(ouw),
                                 ctx->stream);
      if (hinv) launch_gram_upper<float>(uf, (long long)n, ar.at<double>(ohi), ctx->stream);
      // U is fp32 on the fast path: widen for the fp64 ABI
      launch_f32_to_f64(uf, (long long)(n * n), ar.at<double>(ou64), ctx->stream);
      d2h(u, ar.at<double>(ou64), n * n * 8, ctx);
    }
    std::vector<int32_t> ord(n);
    d2h(ord.data(), b.order, n * 4, ctx);
    d2h(hinv, ar.at<double>(ohi), n * n * 8, ctx);
    d2h(damp, b.damp, 8, ctx);
    finish(ctx);
    if (order)
      for (uint64_t i = 0; i < n; ++i) order[i] = ord[i];
  });
}

int ocwg_gptq_quantize_dev(ocwg_ctx* ctx, const float* w, uint64_t ldw, const float* h,
                           uint64_t n, uint64_t m, const ocwg_quant_config* cfg,
                           const ocwg_gptq_options* opts, int mode, int16_t* codes, float* scales,
                           int32_t* zeros, float* w_hat) {
  return guard([&] {
    check_gptq_args(cfg, opts, n, m);
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    Arena ar(ctx);
    size_t o[14];
    gptq_reserve(ar, ctx, n, m, o);
    const size_t om = ar.reserve(4096 * 4);
    ar.commit();
    if (n && m)
      run_gptq(ctx, w, ldw, h, n, m, cfg, opts, mode, codes, scales, zeros, w_hat,
               gptq_bufs(ar, ctx, o, n, m), ar.at<float>(om));
    else if (n)
      run_factor(ctx, h, n, opts->actorder, opts->percdamp, gptq_bufs(ar, ctx, o, n, m));
    finish_dev(ctx);
    if (n == 0 || m == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
  });
}

int ocwg_gptq_quantize(ocwg_ctx* ctx, const float* w, const float* h, uint64_t n, uint64_t m,
                       const ocwg_quant_config* cfg, const ocwg_gptq_options* opts, int mode,
                       int16_t* codes, float* scales, int32_t* zeros, float* w_hat) {
  return guard([&] {
    check_gptq_args(cfg, opts, n, m);
    const uint64_t ng = group_count(cfg, n, m);
    void* blob = nullptr;
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t bytes = n * m * 4 + n * n * 4 + n * m * 2 + ng * 8 + n * m * 4 + 4 * 256;
    ck(cudaMalloc(&blob, bytes), "cudaMalloc(io)");
    char* p = static_cast<char*>(blob);
    auto take = [&](size_t b) {
      char* r = p;
      p += (b + 255) & ~size_t(255);
      return r;
    };
    float* wd = reinterpret_cast<float*>(take(n * m * 4));
    float* hd = reinterpret_cast<float*>(take(n * n * 4));
    int16_t* cd = reinterpret_cast<int16_t*>(take(n * m * 2));
    float* sd = reinterpret_cast<float*>(take(ng * 4));
    int32_t* zd = reinterpret_cast<int32_t*>(take(ng * 4));
    float* whd = reinterpret_cast<float*>(take(n * m * 4));
    h2d(wd, w, n * m * 4, ctx);
    h2d(hd, h, n * n * 4, ctx);
    int r = ocwg_gptq_quantize_dev(ctx, wd, m, hd, n, m, cfg, opts, mode, cd, sd, zd,
                                   w_hat ? whd : nullptr);
    std::string msg = g_err;
    if (r == OCWG_OK) {
      d2h(codes, cd, n * m * 2, ctx);
      d2h(scales, sd, ng * 4, ctx);
      d2h(zeros, zd, ng * 4, ctx);
      if (w_hat) d2h(w_hat, whd, n * m * 4, ctx);
      try {
        finish(ctx);  // host entry points always drain and report
      } catch (const Error& e) {
        r = e.code;
        msg = e.msg;
      }
    }
    cudaFree(blob);
    if (r != OCWG_OK) fail(r, msg);
  });
}

int ocwg_quantize_layer(ocwg_ctx* ctx, const float* w, const double* gram, const double* cross,
                        uint64_t n, uint64_t m, int method, const ocwg_quant_config* cfg,
                        const ocwg_gptq_options* opts, int mode, const ocwg_qep_options* qep,
                        int16_t* codes, float* scales, int32_t* zeros, float* w_hat) {
  return guard([&] {
    if (method != 0 && method != 1) fail(OCWG_INVALID_INPUT, "unknown quantization method");
    if (qep) {  // qep_target's checks come first (layerwise.cpp:96-101, 121)
      if (!(qep->alpha >= 0.0 && qep->alpha <= 1.0))
        fail(OCWG_INVALID_INPUT, "qep_target: alpha must be in [0,1]");
      if (!(qep->eta > 0.0)) fail(OCWG_INVALID_INPUT, "qep_target: eta must be positive");
      if (!cross) fail(OCWG_INVALID_INPUT, "qep_target: null cross statistics");
    }
    const bool corr = qep && qep->alpha != 0.0 && n > 0;
    if (method == 1)
      check_gptq_args(cfg, opts, n, m);
    else
      validate(cfg);
    if (n == 0 || m == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    cudaStream_t st = ctx->stream;
    const uint64_t ng = group_count(cfg, n, m);
    const QCfg c = qcfg(cfg, m);
    Arena ar(ctx);
    size_t o[14];
    if (method == 1) gptq_reserve(ar, ctx, n, m, o);
    const size_t ow = ar.reserve(n * m * 4), og = ar.reserve(n * n * 8),
                 oc = ar.reserve(corr ? n * n * 8 : 8), oh = ar.reserve(method == 1 ? n * n * 4 : 4),
                 ot = ar.reserve(corr ? n * m * 4 : 4),
                 oqf = ar.reserve(corr ? cholesky_flag_ints((long long)n) * sizeof(int) : 4),
                 oqw = ar.reserve(corr ? qep_workspace_doubles((long long)n, (long long)m) * 8 : 8),
                 ocd = ar.reserve(n * m * 2), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4),
                 owh = ar.reserve(w_hat ? n * m * 4 : 4), om = ar.reserve(4096 * 4);
    ar.commit();
    float* wd = ar.at<float>(ow);
    h2d_big(wd, w, n * m * 4, ctx);
    if (corr || method == 1) {
      h2d_big(ar.at<double>(og), gram, n * n * 8, ctx);
      if (ctx->stats_colmajor) transpose_sq_f64(ar.at<double>(og), (long long)n, st);
    }
    const float* target = wd;
    if (corr) {  // W* = W + alpha (gram + lambda I)^-1 (cross W)   (layerwise.cpp:103-111)
      h2d_big(ar.at<double>(oc), cross, n * n * 8, ctx);
      if (ctx->stats_colmajor) transpose_sq_f64(ar.at<double>(oc), (long long)n, st);
      set_tc_workspace(nullptr, 0);
      qep_target_f64(wd, ar.at<double>(og), ar.at<double>(oc), (long long)n, (long long)m,
                     qep->alpha, qep->eta, ar.at<float>(ot), ar.at<double>(oqw), ar.at<int>(oqf),
                     ctx->flag, st);
      try {
        finish(ctx);
      } catch (const Error& e) {
        if (e.code == OCWG_NUMERIC_ERROR)
          fail(OCWG_NUMERIC_ERROR, "qep_target: regularized Gram matrix is singular");
        throw;
      }
      target = ar.at<float>(ot);
    }
    int16_t* cd = ar.at<int16_t>(ocd);
    float* sd = ar.at<float>(os);
    int32_t* zd = ar.at<int32_t>(oz);
    float* whd = w_hat ? ar.at<float>(owh) : nullptr;
    if (method == 0) {  // RTN quantize_matrix (quant.cpp:198-210)
      launch_calibrate_grids(target, (long long)n, (long long)m, (long long)m, c, mode, sd, zd,
                             ctx->flag, ar.at<float>(om), st);
      launch_quantize_rtn(target, (long long)n, (long long)m, (long long)m, c, sd, zd, cd, whd, st);
    } else {  // gptq_quantize(target, stats.gram_matrix(), ...): fp64 -> fp32 H (stats.cpp:7)
      float* hd = ar.at<float>(oh);
      launch_f64_to_f32(ar.at<double>(og), (long long)(n * n), hd, st);
      run_gptq(ctx, target, m, hd, n, m, cfg, opts, mode, cd, sd, zd, whd, gptq_bufs(ar, ctx, o, n, m),
               ar.at<float>(om));
    }
    finish(ctx);
    d2h(codes, cd, n * m * 2, ctx);
    d2h(scales, sd, ng * 4, ctx);
    d2h(zeros, zd, ng * 4, ctx);
    if (w_hat) d2h(w_hat, whd, n * m * 4, ctx);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

int ocwg_qep_target(ocwg_ctx* ctx, const float* w, const double* gram, const double* cross,
                    uint64_t n, uint64_t m, double alpha, double eta, float* out) {
  return guard([&] {
    // validation order of layerwise.cpp:96-101
    if (!(alpha >= 0.0 && alpha <= 1.0)) fail(OCWG_INVALID_INPUT, "qep_target: alpha must be in [0,1]");
    if (!(eta > 0.0)) fail(OCWG_INVALID_INPUT, "qep_target: eta must be positive");
    if (alpha == 0.0) {
      if (out != w) std::memmove(out, w, n * m * sizeof(float));
      return;
    }
    if (n == 0) return;
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    Arena ar(ctx);
    const size_t ow = ar.reserve(n * m * 4), og = ar.reserve(n * n * 8), oc = ar.reserve(n * n * 8),
                 oo = ar.reserve(n * m * 4),
                 of = ar.reserve(cholesky_flag_ints((long long)n) * sizeof(int)),
                 ows = ar.reserve(qep_workspace_doubles((long long)n, (long long)m) * 8);
    ar.commit();
    h2d(ar.at<float>(ow), w, n * m * 4, ctx);
    h2d(ar.at<double>(og), gram, n * n * 8, ctx);
    h2d(ar.at<double>(oc), cross, n * n * 8, ctx);
    if (ctx->stats_colmajor) {
      transpose_sq_f64(ar.at<double>(og), (long long)n, ctx->stream);
      transpose_sq_f64(ar.at<double>(oc), (long long)n, ctx->stream);
    }
    set_tc_workspace(nullptr, 0);
    qep_target_f64(ar.at<float>(ow), ar.at<double>(og), ar.at<double>(oc), (long long)n,
                   (long long)m, alpha, eta, ar.at<float>(oo), ar.at<double>(ows), ar.at<int>(of),
                   ctx->flag, ctx->stream);
    d2h(out, ar.at<float>(oo), n * m * 4, ctx);
    try {
      finish(ctx);
    } catch (const Error& e) {
      if (e.code == OCWG_NUMERIC_ERROR)
        fail(OCWG_NUMERIC_ERROR, "qep_target: regularized Gram matrix is singular");
      throw;
    }
  });
}

// ------------------------------------------------------------------ end to end
int ocwg_quantize_layer_x_dev(ocwg_ctx* ctx, const float* w, const uint16_t* x, uint64_t tokens,
                              uint64_t n, uint64_t m, const ocwg_quant_config* cfg,
                              const ocwg_gptq_options* opts, int mode, int16_t* codes,
                              float* scales, int32_t* zeros, float* w_hat, uint8_t* payload,
                              float* h_out) {
  return guard([&] {
    check_gptq_args(cfg, opts, n, m);
    if (n == 0 || m == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    const uint64_t ng = group_count(cfg, n, m);
    Arena ar(ctx);
    size_t o[14];
    gptq_reserve(ar, ctx, n, m, o);
    const size_t om = ar.reserve(4096 * 4);
    const size_t oh = ar.reserve(n * n * 4);
    const size_t hws = gram_tc_workspace_bytes((long long)n);
    const size_t ohw = ar.reserve(hws), opad = ar.reserve(hessian_pad_bytes(tokens, n));
    const size_t oc = ar.reserve(n * m * 2), os = ar.reserve(ng * 4), oz = ar.reserve(ng * 4);
    ar.commit();
    float* h = h_out ? h_out : ar.at<float>(oh);
    int16_t* cd = codes ? codes : ar.at<int16_t>(oc);
    float* sd = scales ? scales : ar.at<float>(os);
    int32_t* zd = zeros ? zeros : ar.at<int32_t>(oz);
    run_hessian(x, tokens, n, h, false, ar.at<void>(ohw), hws, ar.at<uint16_t>(opad), ctx->stream);
    run_gptq(ctx, w, m, h, n, m, cfg, opts, mode, cd, sd, zd, w_hat, gptq_bufs(ar, ctx, o, n, m),
             ar.at<float>(om));
    if (payload) launch_pack(cd, (long long)(n * m), (long long)ng, qcfg(cfg, m), sd, zd, payload,
                             ctx->stream);
    finish_dev(ctx);
  });
}

// Host buffers in, host buffers out.  X streams to the device in token chunks
// on the copy stream while the tensor cores accumulate H chunk by chunk
// (accumulate_stats' streaming contract, stats.cpp:10-19 / test_core.cpp:280-293),
// so the PCIe transfer overlaps the Hessian; device buffers are context-owned
// and reused across calls.
int ocwg_quantize_layer_x(ocwg_ctx* ctx, const float* w, const uint16_t* x, uint64_t tokens,
                          uint64_t n, uint64_t m, const ocwg_quant_config* cfg,
                          const ocwg_gptq_options* opts, int mode, int16_t* codes, float* scales,
                          int32_t* zeros, float* w_hat, uint8_t* payload, uint64_t payload_len,
                          float* h_out) {
  return guard([&] {
    check_gptq_args(cfg, opts, n, m);
    if (n == 0 || m == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
    const uint64_t ng = group_count(cfg, n, m), pb = storage_bytes(cfg, n, m);
    if (payload && payload_len < pb) fail(OCWG_INVALID_INPUT, "payload buffer too small");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    cudaStream_t st = ctx->stream;
    // ---- context-owned io buffers (grow only)
    size_t off = 0;
    auto take = [&](size_t b) {
      const size_t o = off;
      off += (b + 255) & ~size_t(255);
      return o;
    };
    const size_t ow = take(n * m * 4), ox = take(std::max<uint64_t>(1, tokens) * n * 2),
                 oc = take(n * m * 2), os = take(ng * 4), oz = take(ng * 4),
                 owh = take(n * m * 4), opl = take(pb), oh = take(n * n * 4);
    if (off > ctx->io_bytes) {
      ck(cudaStreamSynchronize(st), "sync");
      if (ctx->io) cudaFree(ctx->io);
      ctx->io = nullptr;
      ctx->io_bytes = 0;
      ck(cudaMalloc(&ctx->io, off), "cudaMalloc(io)");
      ctx->io_bytes = off;
    }
    char* io = static_cast<char*>(ctx->io);
    float* wd = reinterpret_cast<float*>(io + ow);
    uint16_t* xd = reinterpret_cast<uint16_t*>(io + ox);
    int16_t* cd = reinterpret_cast<int16_t*>(io + oc);
    float* sd = reinterpret_cast<float*>(io + os);
    int32_t* zd = reinterpret_cast<int32_t*>(io + oz);
    float* whd = reinterpret_cast<float*>(io + owh);
    uint8_t* pd = reinterpret_cast<uint8_t*>(io + opl);
    float* hd = reinterpret_cast<float*>(io + oh);
    // ---- workspace
    Arena ar(ctx);
    size_t o[14];
    gptq_reserve(ar, ctx, n, m, o);
    const size_t om = ar.reserve(4096 * 4);
    const long long chunk = 32768;  // tokens per H2D chunk (a multiple of the 16384 split)
    const size_t hws = gram_tc_workspace_bytes((long long)n);
    const size_t ohw = ar.reserve(hws),
                 opad = ar.reserve(hessian_pad_bytes(std::min<uint64_t>(chunk, tokens), n));
    ar.commit();
    // ---- pipeline: W and X chunks on the copy stream, H chunk by chunk on st
    const long long nchunks = tokens ? ((long long)tokens + chunk - 1) / chunk : 0;
    while ((long long)ctx->cev.size() < nchunks + 2) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      ctx->cev.push_back(e);
    }
    ck(cudaEventRecord(ctx->cev[0], st), "event");  // copies start after prior work on st
    ck(cudaStreamWaitEvent(ctx->cpy, ctx->cev[0], 0), "event");
    if (tokens == 0) ck(cudaMemsetAsync(hd, 0, n * n * 4, st), "memset");
    for (long long k = 0; k < nchunks; ++k) {
      const long long t0 = k * chunk, tc = std::min<long long>(chunk, (long long)tokens - t0);
      ck(cudaMemcpyAsync(xd + t0 * n, x + t0 * n, size_t(tc) * n * 2, cudaMemcpyHostToDevice,
                         ctx->cpy),
         "H2D(X)");
      ck(cudaEventRecord(ctx->cev[2 + k], ctx->cpy), "event");
      ck(cudaStreamWaitEvent(st, ctx->cev[2 + k], 0), "event");
      run_hessian(xd + t0 * n, uint64_t(tc), n, hd, k > 0, ar.at<void>(ohw), hws,
                  ar.at<uint16_t>(opad), st);
    }
    // W goes over PCIe after X: it is needed only by the grids and the sweep, so
    // its copy overlaps the factorisation instead of delaying the first X chunk
    ck(cudaMemcpyAsync(wd, w, n * m * 4, cudaMemcpyHostToDevice, ctx->cpy), "H2D(W)");
    ck(cudaEventRecord(ctx->cev[1], ctx->cpy), "event");
    run_gptq(ctx, wd, m, hd, n, m, cfg, opts, mode, cd, sd, zd, w_hat ? whd : nullptr,
             gptq_bufs(ar, ctx, o, n, m), ar.at<float>(om), ctx->cev[1]);
    ck(cudaStreamWaitEvent(st, ctx->cev[1], 0), "event");  // (W resident for the D2H order)
    if (payload) launch_pack(cd, (long long)(n * m), (long long)ng, qcfg(cfg, m), sd, zd, pd, st);
    d2h(codes, cd, n * m * 2, ctx);
    d2h(scales, sd, ng * 4, ctx);
    d2h(zeros, zd, ng * 4, ctx);
    if (w_hat) d2h(w_hat, whd, n * m * 4, ctx);
    if (payload) d2h(payload, pd, pb, ctx);
    if (h_out) d2h(h_out, hd, n * n * 4, ctx);
    finish(ctx);
  });
}

int ocwg_synth_dev(ocwg_ctx* ctx, int kind, uint64_t seed, uint64_t rows, uint64_t cols,
                   double stddev, const float* col_scale, void* out) {
  return guard([&] {
    if (kind < 0 || kind > 2) fail(OCWG_INVALID_INPUT, "synth: unknown kind");
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    if (rows > 0 && cols > 0)
      launch_synth(kind, (unsigned long long)seed, (long long)rows, (long long)cols, float(stddev),
                   col_scale, out, 0, ctx->stream);
    finish_dev(ctx);
  });
}

int ocwg_quantize_layers_x_dev(ocwg_ctx* ctx, int count, const float* const* w, const uint64_t* m,
                               const uint16_t* x, uint64_t tokens, uint64_t n,
                               const ocwg_quant_config* cfg, const ocwg_gptq_options* opts,
                               int mode, int16_t* const* codes, float* const* scales,
                               int32_t* const* zeros, uint8_t* const* payload) {
  return guard([&] {
    if (count < 1 || !w || !m) fail(OCWG_INVALID_INPUT, "quantize_layers_x: no layers");
    uint64_t mmax = 0;
    for (int i = 0; i < count; ++i) {
      check_gptq_args(cfg, opts, n, m[i]);
      if (n == 0 || m[i] == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
      if (!codes || !codes[i] || !scales || !scales[i] || !zeros || !zeros[i])
        fail(OCWG_INVALID_INPUT, "quantize_layers_x_dev: codes / scales / zeros are required");
      mmax = std::max(mmax, m[i]);
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx, true);
    cudaStream_t st = ctx->stream;
    Arena ar(ctx);
    size_t o[14];
    gptq_reserve(ar, ctx, n, mmax, o);
    const size_t om = ar.reserve(4096 * 4), oh = ar.reserve(n * n * 4);
    const size_t hws = gram_tc_workspace_bytes((long long)n);
    const size_t ohw = ar.reserve(hws), opad = ar.reserve(hessian_pad_bytes(tokens, n));
    ar.commit();
    const GptqBufs b = gptq_bufs(ar, ctx, o, n, mmax);
    float* hd = ar.at<float>(oh);
    // one Hessian + order + factorisation for every layer that reads X
    run_hessian(x, tokens, n, hd, false, ar.at<void>(ohw), hws, ar.at<uint16_t>(opad), st);
    run_factor(ctx, hd, n, opts->actorder, opts->percdamp, b);
    for (int i = 0; i < count; ++i) {
      const uint64_t mi = m[i];
      const QCfg c = qcfg(cfg, mi);
      launch_calibrate_grids(w[i], (long long)n, (long long)mi, (long long)mi, c, mode, scales[i],
                             zeros[i], ctx->flag, ar.at<float>(om), st);
      if (ctx->precision == OCWG_FP64)
        run_sweep_t<double>(ctx, w[i], mi, n, mi, c, opts, codes[i], scales[i], zeros[i], nullptr, b);
      else
        run_sweep_t<float>(ctx, w[i], mi, n, mi, c, opts, codes[i], scales[i], zeros[i], nullptr, b);
      if (payload && payload[i])
        launch_pack(codes[i], (long long)(n * mi), (long long)group_count(cfg, n, mi), c, scales[i],
                    zeros[i], payload[i], st);
    }
    finish_dev(ctx);
  });
}

int ocwg_quantize_layers_x(ocwg_ctx* ctx, int count, const float* const* w, const uint64_t* m,
                           const uint16_t* x, uint64_t tokens, uint64_t n,
                           const ocwg_quant_config* cfg, const ocwg_gptq_options* opts,
                           int mode, int16_t* const* codes, float* const* scales,
                           int32_t* const* zeros, uint8_t* const* payload,
                           const uint64_t* payload_len) {
  return guard([&] {
    if (count < 1 || !w || !m) fail(OCWG_INVALID_INPUT, "quantize_layers_x: no layers");
    uint64_t mmax = 0;
    for (int i = 0; i < count; ++i) {
      check_gptq_args(cfg, opts, n, m[i]);
      if (n == 0 || m[i] == 0) fail(OCWG_INVALID_INPUT, "calibrate_grids: empty matrix");
      if (payload && payload[i] && (!payload_len || payload_len[i] < storage_bytes(cfg, n, m[i])))
        fail(OCWG_INVALID_INPUT, "payload buffer too small");
      mmax = std::max(mmax, m[i]);
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    begin(ctx);
    cudaStream_t st = ctx->stream;
    const uint64_t ngmax = group_count(cfg, n, mmax), pbmax = storage_bytes(cfg, n, mmax);
    size_t off = 0;
    auto take = [&](size_t b) {
      const size_t o = off;
      off += (b + 255) & ~size_t(255);
      return o;
    };
    const size_t ow = take(n * mmax * 4), ox = take(std::max<uint64_t>(1, tokens) * n * 2),
                 oc = take(n * mmax * 2), os = take(ngmax * 4), oz = take(ngmax * 4),
                 opl = take(pbmax), oh = take(n * n * 4);
    if (off > ctx->io_bytes) {
      ck(cudaStreamSynchronize(st), "sync");
      if (ctx->io) cudaFree(ctx->io);
      ctx->io = nullptr;
      ctx->io_bytes = 0;
      ck(cudaMalloc(&ctx->io, off), "cudaMalloc(io)");
      ctx->io_bytes = off;
    }
    char* io = static_cast<char*>(ctx->io);
    float* wd = reinterpret_cast<float*>(io + ow);
    uint16_t* xd = reinterpret_cast<uint16_t*>(io + ox);
    int16_t* cd = reinterpret_cast<int16_t*>(io + oc);
    float* sd = reinterpret_cast<float*>(io + os);
    int32_t* zd = reinterpret_cast<int32_t*>(io + oz);
    uint8_t* pd = reinterpret_cast<uint8_t*>(io + opl);
    float* hd = reinterpret_cast<float*>(io + oh);
    Arena ar(ctx);
    size_t o[14];
    gptq_reserve(ar, ctx, n, mmax, o);
    const size_t om = ar.reserve(4096 * 4);
    const long long chunk = 32768;
    const size_t hws = gram_tc_workspace_bytes((long long)n);
    const size_t ohw = ar.reserve(hws),
                 opad = ar.reserve(hessian_pad_bytes(std::min<uint64_t>(chunk, tokens), n));
    ar.commit();
    const GptqBufs b = gptq_bufs(ar, ctx, o, n, mmax);
    // ---- H = X^T X, X streamed chunk by chunk under the Hessian (as quantize_layer_x)
    const long long nchunks = tokens ? ((long long)tokens + chunk - 1) / chunk : 0;
    while ((long long)ctx->cev.size() < nchunks + 2) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      ctx->cev.push_back(e);
    }
    ck(cudaEventRecord(ctx->cev[0], st), "event");
    ck(cudaStreamWaitEvent(ctx->cpy, ctx->cev[0], 0), "event");
    if (tokens == 0) ck(cudaMemsetAsync(hd, 0, n * n * 4, st), "memset");
    for (long long k = 0; k < nchunks; ++k) {
      const long long t0 = k * chunk, tc = std::min<long long>(chunk, (long long)tokens - t0);
      ck(cudaMemcpyAsync(xd + t0 * n, x + t0 * n, size_t(tc) * n * 2, cudaMemcpyHostToDevice,
                         ctx->cpy),
         "H2D(X)");
      ck(cudaEventRecord(ctx->cev[2 + k], ctx->cpy), "event");
      ck(cudaStreamWaitEvent(st, ctx->cev[2 + k], 0), "event");
      run_hessian(xd + t0 * n, uint64_t(tc), n, hd, k > 0, ar.at<void>(ohw), hws,
                  ar.at<uint16_t>(opad), st);
    }
    // ---- one order + factorisation for every layer
    run_factor(ctx, hd, n, opts->actorder, opts->percdamp, b);
    // ---- per layer: W in, grids + sweep + pack, results out
    for (int i = 0; i < count; ++i) {
      const uint64_t mi = m[i];
      const QCfg c = qcfg(cfg, mi);
      const uint64_t ng = group_count(cfg, n, mi), pb = storage_bytes(cfg, n, mi);
      ck(cudaMemcpyAsync(wd, w[i], n * mi * 4, cudaMemcpyHostToDevice, st), "H2D(W)");
      launch_calibrate_grids(wd, (long long)n, (long long)mi, (long long)mi, c, mode, sd, zd,
                             ctx->flag, ar.at<float>(om), st);
      if (ctx->precision == OCWG_FP64)
        run_sweep_t<double>(ctx, wd, mi, n, mi, c, opts, cd, sd, zd, nullptr, b);
      else
        run_sweep_t<float>(ctx, wd, mi, n, mi, c, opts, cd, sd, zd, nullptr, b);
      const bool pk = payload && payload[i];
      if (pk) launch_pack(cd, (long long)(n * mi), (long long)ng, c, sd, zd, pd, st);
      if (codes && codes[i]) d2h(codes[i], cd, n * mi * 2, ctx);
      if (scales && scales[i]) d2h(scales[i], sd, ng * 4, ctx);
      if (zeros && zeros[i]) d2h(zeros[i], zd, ng * 4, ctx);
      if (pk) d2h(payload[i], pd, pb, ctx);
    }
    finish(ctx);
  });
}

}  // extern "C"
