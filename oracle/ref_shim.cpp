// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libfqref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the oracle restatement (oracle/fq_oracle.c)
// and by bench.py --impl reference as the reference CPU arm.  Only the reference's public
// C++ API (/root/reference/proj/include/flexquant/*.hpp) is called here.
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "flexquant/analyzer.hpp"
#include "flexquant/engine.hpp"
#include "flexquant/fixture.hpp"
#include "flexquant/model.hpp"
#include "flexquant/quantizer.hpp"
#include "flexquant/scheduler.hpp"
#include "flexquant/tensor.hpp"

using namespace flexquant;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionError& e) { g_err = e.what(); return 1; }
  catch (const ConfigError& e) { g_err = e.what(); return 2; }
  catch (const InputError& e) { g_err = e.what(); return 3; }
  catch (const StateError& e) { g_err = e.what(); return 4; }
  catch (const FormatError& e) { g_err = e.what(); return 5; }
  catch (const CapacityError& e) { g_err = e.what(); return 6; }
  catch (const std::exception& e) { g_err = e.what(); return 99; }
}

Tensor t2(const float* p, int64_t r, int64_t c) {
  return Tensor::from_data({r, c}, std::vector<float>(p, p + r * c));
}

// Group view of the reference quantizer: every (row, group) slice quantized as one reference row.
QuantizedTensor quantize_slice(const float* p, int64_t len, int bits, int mode) {
  return quantize(t2(p, 1, len), bits, static_cast<QuantMode>(mode));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Quantizes W[N,K] with groups of G along K (G >= K: the reference's per-row scheme).
// K % G == 0 uses the reshape trick ([N*K/G, G] view, one reference call); otherwise every
// slice is quantized as its own row and the codes re-packed with pack_codes.
int ref_quantize(const float* w, int64_t N, int64_t K, int64_t G, int bits, int mode, uint8_t* payload,
                 float* scale, int32_t* zp) {
  return guard([&] {
    if (G <= 0 || G > K) G = K;
    const int64_t ng = (K + G - 1) / G;
    if (K % G == 0) {
      const QuantizedTensor q = quantize(t2(w, N * ng, G), bits, static_cast<QuantMode>(mode));
      std::memcpy(payload, q.payload.data(), q.payload.size());
      std::memcpy(scale, q.scale.data(), q.scale.size() * sizeof(float));
      std::memcpy(zp, q.zero_point.data(), q.zero_point.size() * sizeof(int32_t));
      return;
    }
    std::vector<uint32_t> codes(static_cast<size_t>(N * K));
    for (int64_t r = 0; r < N; ++r) {
      for (int64_t g = 0; g < ng; ++g) {
        const int64_t k0 = g * G, len = std::min(G, K - k0);
        const QuantizedTensor q = quantize_slice(w + r * K + k0, len, bits, mode);
        for (int64_t i = 0; i < len; ++i) codes[static_cast<size_t>(r * K + k0 + i)] = q.code_at(0, i);
        scale[r * ng + g] = q.scale[0];
        zp[r * ng + g] = q.zero_point[0];
      }
    }
    const std::vector<uint8_t> packed = pack_codes(codes, bits);
    std::memcpy(payload, packed.data(), packed.size());
  });
}

// dequantize (src/quantizer.cpp:205-219) of the group view, written back as [N, K].
int ref_dequantize(const uint8_t* payload, int64_t N, int64_t K, int64_t G, int bits, int mode, const float* scale,
                   const int32_t* zp, float* out) {
  return guard([&] {
    if (G <= 0 || G > K) G = K;
    const int64_t ng = (K + G - 1) / G;
    const std::vector<uint32_t> codes = unpack_codes(
        std::span<const uint8_t>(payload, static_cast<size_t>((N * K * bits + 7) / 8)), N * K, bits);
    for (int64_t r = 0; r < N; ++r) {
      for (int64_t g = 0; g < ng; ++g) {
        const int64_t k0 = g * G, len = std::min(G, K - k0);
        std::vector<uint32_t> slice(codes.begin() + r * K + k0, codes.begin() + r * K + k0 + len);
        QuantizedTensor q;
        q.bits = bits;
        q.mode = static_cast<QuantMode>(mode);
        q.rows = 1;
        q.cols = len;
        q.payload = pack_codes(slice, bits);
        q.scale = {scale[r * ng + g]};
        q.zero_point = {zp[r * ng + g]};
        const Tensor d = dequantize(q);
        std::memcpy(out + r * K + k0, d.data(), sizeof(float) * static_cast<size_t>(len));
      }
    }
  });
}

// linear (src/tensor.cpp:83-101).
int ref_linear(const float* x, int64_t B, int64_t K, const float* w, int64_t N, const float* bias, float* y) {
  return guard([&] {
    const Tensor b = bias ? Tensor::from_data({N}, std::vector<float>(bias, bias + N)) : Tensor{};
    const Tensor out = linear(t2(x, B, K), t2(w, N, K), b);
    std::memcpy(y, out.data(), sizeof(float) * static_cast<size_t>(B * N));
  });
}

int ref_row_stats(const float* logits, int64_t V, double* ppl, double* ft, int32_t* argmax) {
  return guard([&] {
    const Tensor row = t2(logits, 1, V);
    *ppl = ppl_entropy(row);
    *ft = V >= 2 ? fault_tolerance(row) : 0.0;
    *argmax = argmax_token(row);
  });
}

int ref_derive_threshold(const float* logits, int64_t n, int64_t V, int window_len, double theta, double* out) {
  return guard([&] { *out = derive_threshold(t2(logits, n, V), window_len, theta); });
}

int ref_scheduler_replay(const double* ppl, int64_t n, int window_len, double thre, int layers_per_switch,
                         int64_t plan_len, int64_t* fire_first, int64_t* fire_count, double* mavg, int32_t* mavg_valid) {
  return guard([&] {
    SchedulerConfig cfg;
    cfg.window_len = window_len;
    cfg.layers_per_switch = layers_per_switch;
    SchedulerState st(cfg, static_cast<size_t>(plan_len));
    st.set_threshold(thre);
    for (int64_t t = 0; t < n; ++t) {
      const auto d = st.observe(ppl[t]);
      fire_first[t] = static_cast<int64_t>(d.first_entry);
      fire_count[t] = static_cast<int64_t>(d.count);
      mavg_valid[t] = d.window_mean.has_value() ? 1 : 0;
      mavg[t] = d.window_mean.value_or(0.0);
    }
  });
}

int ref_hist_kl(const float* w, const float* wq, int64_t n, int bins, double* kl) {
  return guard([&] {
    float lo = w[0], hi = w[0];
    for (int64_t i = 1; i < n; ++i) {
      lo = std::min(lo, w[i]);
      hi = std::max(hi, w[i]);
    }
    const std::vector<double> edges = uniform_edges(lo, hi, bins);
    const std::vector<double> p = weight_histogram(t2(w, 1, n), edges);
    const std::vector<double> q = weight_histogram(t2(wq, 1, n), edges);
    *kl = kl_divergence(p, q);
  });
}

int ref_kl_divergence(const double* p, const double* q, int64_t n, double* kl) {
  return guard([&] {
    *kl = kl_divergence(std::span<const double>(p, static_cast<size_t>(n)), std::span<const double>(q, static_cast<size_t>(n)));
  });
}

// make-fixture: a seeded reference fixture written in the flexquant-weights v1 container.
int ref_make_fixture(const char* preset, uint64_t seed, int64_t max_seq_len, const char* out_path) {
  return guard([&] {
    ModelConfig cfg = std::string(preset) == "micro" ? micro_config() : tiny_config();
    if (max_seq_len > 0) cfg.max_seq_len = max_seq_len;
    save_model_file(make_fixture_model(cfg, seed), out_path);
  });
}

// analyze: ladder plan fp -> 8 -> 4 (src/analyzer.cpp:141-155) written as flexquant-plan v1.
int ref_analyze(const char* model_path, int bins, const char* plan_path) {
  return guard([&] {
    const Model m = load_model_file(model_path);
    save_plan_file(build_ladder_plan(m, std::vector<Rung>{Rung::Int8, Rung::Int4}, bins), plan_path);
  });
}

// generate (src/engine.cpp:157-162) with the CLI's knobs; trace written as JSONL.
int ref_generate(const char* model_path, const char* plan_path, const int32_t* prompt, int64_t n, int64_t max_new,
                 double theta, int absolute, int window_len, int layers_per_switch, int start_rung,
                 const char* trace_path, int32_t* out_tokens, int64_t* out_count, double* out_threshold) {
  return guard([&] {
    Model m = load_model_file(model_path);
    const SwitchPlan plan = (plan_path && plan_path[0]) ? load_plan_file(plan_path) : SwitchPlan{};
    GenerationConfig cfg;
    cfg.max_new_tokens = max_new;
    cfg.scheduler.theta = theta;
    cfg.scheduler.threshold_mode = absolute ? ThresholdMode::Absolute : ThresholdMode::Prefill;
    cfg.scheduler.window_len = window_len;
    cfg.scheduler.layers_per_switch = layers_per_switch;
    cfg.start_rung = static_cast<Rung>(start_rung);
    cfg.trace_path = trace_path ? trace_path : "";
    const GenerationResult r = generate(std::span<const TokenId>(prompt, static_cast<size_t>(n)), m, plan, cfg);
    for (size_t i = 0; i < r.sequence.size(); ++i) out_tokens[i] = r.sequence[i];
    *out_count = static_cast<int64_t>(r.sequence.size());
    *out_threshold = r.threshold;
  });
}

// Teacher-forced logits of the reference model: prefill over all n tokens at one rung.
int ref_prefill_logits(const char* model_path, const int32_t* tokens, int64_t n, int rung, float* logits) {
  return guard([&] {
    Model m = load_model_file(model_path);
    m.set_all_precision(static_cast<Rung>(rung));
    KvCache c = m.make_cache();
    const Tensor l = m.forward_prefill(std::span<const TokenId>(tokens, static_cast<size_t>(n)), c);
    std::memcpy(logits, l.data(), sizeof(float) * static_cast<size_t>(l.numel()));
  });
}

// Decode-path logits: prefill of tokens[0] then forward_decode of each following token.
int ref_decode_logits(const char* model_path, const int32_t* tokens, int64_t n, int rung, float* logits) {
  return guard([&] {
    Model m = load_model_file(model_path);
    m.set_all_precision(static_cast<Rung>(rung));
    KvCache c = m.make_cache();
    const int64_t V = m.config().vocab_size;
    Tensor l = m.forward_prefill(std::span<const TokenId>(tokens, 1), c);
    std::memcpy(logits, l.data(), sizeof(float) * static_cast<size_t>(V));
    for (int64_t i = 1; i < n; ++i) {
      l = m.forward_decode(tokens[i], c);
      std::memcpy(logits + i * V, l.data(), sizeof(float) * static_cast<size_t>(V));
    }
  });
}

// Times `reps` calls of MultiPrecisionLayer::forward (dequantize + linear) on a [N,K] layer with
// per-group-G codes: the reference CPU arm of the GEMV sweep.  Returns seconds per call.
int ref_time_quant_linear(const float* w, int64_t N, int64_t K, int64_t G, int bits, const float* x, int64_t B,
                          int reps, double* seconds_per_call) {
  return guard([&] {
    if (G <= 0 || G > K) G = K;
    const int64_t ng = (K + G - 1) / G;
    std::vector<uint8_t> payload(static_cast<size_t>((N * K * bits + 7) / 8));
    std::vector<float> scale(static_cast<size_t>(N * ng));
    std::vector<int32_t> zp(static_cast<size_t>(N * ng));
    if (ref_quantize(w, N, K, G, bits, 0, payload.data(), scale.data(), zp.data()) != 0) throw InputError(g_err);
    // group view (K % G == 0): the reference forward on the [N*ng, G] payload + reshape
    QuantizedTensor q;
    q.bits = bits;
    q.mode = QuantMode::Asymmetric;
    q.rows = N * ng;
    q.cols = G;
    q.payload = payload;
    q.scale = scale;
    q.zero_point = zp;
    const Tensor xt = t2(x, B, K);
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) {
      Tensor d = dequantize(q);
      const Tensor wv = Tensor::from_data({N, K}, std::vector<float>(d.data(), d.data() + N * K));
      const Tensor y = linear(xt, wv, Tensor{});
      if (y.numel() == 0) throw StateError("empty");
    }
    const auto t1 = std::chrono::steady_clock::now();
    *seconds_per_call = std::chrono::duration<double>(t1 - t0).count() / reps;
  });
}

// ---- reference decode arm (bench.py --impl reference): a reference-architecture model at the
// requested dimensions (make_fixture_model, src/fixture.cpp), a greedy decode loop of
// forward_decode + argmax_token (src/engine.cpp:89-136 minus the scheduler), one handle per host
// thread (the reference model is single-thread-confined).
struct RefDecoder {
  Model model;
  KvCache cache;
  TokenId next = 0;
};

void* ref_decoder_create(int64_t vocab, int64_t d, int64_t heads, int64_t head_dim, int64_t layers, int64_t ffn,
                         int64_t max_seq, uint64_t seed, const int32_t* prompt, int64_t n_prompt, double w4_share) {
  RefDecoder* out = nullptr;
  const int st = guard([&] {
    ModelConfig c;
    c.vocab_size = vocab;
    c.d_model = d;
    c.n_heads = heads;
    c.head_dim = head_dim;
    c.n_layers = layers;
    c.ffn_dim = ffn;
    c.max_seq_len = max_seq;
    auto* r = new RefDecoder{make_fixture_model(c, seed), KvCache{}, 0};
    // the switched schedule's mix: the first w4_share of the linears (by parameter count) at 4 bits
    std::vector<MultiPrecisionLayer*> ls = r->model.linear_layers();
    double total = 0.0, acc = 0.0;
    for (auto* l : ls) total += static_cast<double>(l->param_count());
    for (auto* l : ls) {
      const bool four = acc < w4_share * total;
      acc += static_cast<double>(l->param_count());
      r->model.set_precision(l->id(), four ? Rung::Int4 : Rung::Int8);
    }
    r->cache = r->model.make_cache();
    const Tensor lg = r->model.forward_prefill(std::span<const TokenId>(prompt, static_cast<size_t>(n_prompt)), r->cache);
    const int64_t V = r->model.config().vocab_size;
    Tensor last({1, V});
    std::memcpy(last.data(), lg.data() + (lg.rows() - 1) * V, sizeof(float) * static_cast<size_t>(V));
    r->next = argmax_token(last);
    out = r;
  });
  return st == 0 ? out : nullptr;
}

// One greedy decode token: forward_decode, ppl_entropy / fault_tolerance of the row (the
// statistics the engine loop records), argmax.  Returns the seconds it took.
int ref_decoder_step(void* h, double* seconds, double* ppl) {
  return guard([&] {
    auto* r = static_cast<RefDecoder*>(h);
    const auto t0 = std::chrono::steady_clock::now();
    const Tensor lg = r->model.forward_decode(r->next, r->cache);
    const double p = ppl_entropy(lg);
    const double ft = fault_tolerance(lg);
    r->next = argmax_token(lg);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (ppl) *ppl = p + 0.0 * ft;
  });
}

int64_t ref_decoder_params(void* h) {
  int64_t n = 0;
  for (const auto* l : static_cast<RefDecoder*>(h)->model.linear_layers()) n += l->param_count();
  return n;
}

void ref_decoder_destroy(void* h) { delete static_cast<RefDecoder*>(h); }

}  // extern "C"
