// Device-resident multi-precision decoder behind the reference's Model API
// (/root/reference/proj/include/flexquant/model.hpp:18-215).  Weights live on the B200 as
// resident per-precision copies; set_precision is a one-byte precision-table write (no payload
// is touched); forward_* run the captured decode-step graph and return host logits.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "flexquant/quantizer.hpp"
#include "flexquant/rung.hpp"
#include "flexquant/tensor.hpp"

namespace flexquant {

using TokenId = int32_t;

enum class Arch : uint8_t { Reference = FQ_ARCH_REFERENCE, Llama = FQ_ARCH_LLAMA };

struct ModelConfig {
  int64_t vocab_size = 0;
  int64_t d_model = 0;
  int64_t n_heads = 0;
  int64_t head_dim = 0;
  int64_t n_layers = 0;
  int64_t ffn_dim = 0;
  int64_t max_seq_len = 0;
  bool tie_embeddings = false;
  // B200 engine extensions
  Arch arch = Arch::Reference;
  int64_t group_size = 0;  // quantization group (0 = per row, the reference scheme)
  int max_batch = 1;       // resident sequence slots
  float norm_eps = 1e-5f;
  float rope_theta = 10000.0f;
  bool fp16_activations = false;  // llama: activation roundings in fp16 instead of bf16
  void validate() const;
};

// Per-forward accounting (src/model.cpp:77-98).  On the device the linear time buckets are
// attributed from the step's measured time in proportion to each rung's algorithmic bytes.
struct StepStats {
  double weight_bytes = 0.0;
  uint64_t ns_fp = 0;
  uint64_t ns_int8 = 0;
  uint64_t ns_int4 = 0;
  uint64_t ns_forward = 0;
  void reset() { *this = StepStats{}; }
};

class Model;

// One switchable linear: a view of the model's resident fq_layer, or a standalone layer.
class MultiPrecisionLayer {
 public:
  MultiPrecisionLayer() = default;
  // Standalone layer holding fp weights; quantize_rungs / set_quantized add the integer rungs.
  MultiPrecisionLayer(std::string id, Tensor weight, Tensor bias, int64_t group_size = 0);
  ~MultiPrecisionLayer();
  MultiPrecisionLayer(MultiPrecisionLayer&&) noexcept;
  MultiPrecisionLayer& operator=(MultiPrecisionLayer&&) noexcept;

  void quantize_rungs(QuantMode mode);
  const std::string& id() const { return id_; }
  int64_t out_features() const { return n_; }
  int64_t in_features() const { return k_; }
  int64_t param_count() const { return n_ * k_; }
  Rung current() const;
  void set_current(Rung r);
  bool has(Rung r) const;
  void set_quantized(Rung r, const QuantizedTensor& q);
  // the resident payloads, downloaded from the device on first use (cached until replaced)
  const QuantizedTensor& quantized(Rung r) const;
  // fp weights / bias on the host (downloaded on first use; empty when the layer holds none,
  // e.g. the llama architecture keeps no fp rung on the device)
  const Tensor& fp_weight() const;
  const Tensor& bias() const;
  // y = x * W_active^T + bias on the device (exact numerics: bit-identical to the reference).
  Tensor forward(const Tensor& x, StepStats* stats) const;
  double active_weight_bytes() const { return static_cast<double>(param_count()) * accounting_bits(current()) / 8.0; }
  fq_layer* handle() const { return layer_; }

 private:
  friend class Model;
  std::string id_;
  int64_t n_ = 0, k_ = 0;
  fq_layer* layer_ = nullptr;
  bool owned_ = false;
  Model* model_ = nullptr;  // non-null for model views (rung lives in the model's table)
  int index_ = -1;
  Rung standalone_rung_ = Rung::Fp;
  int64_t group_ = 0;
  Tensor host_fp_;  // standalone layers keep their fp weights for quantize_rungs
  // host-side caches of the device payloads (reference API returns references)
  mutable QuantizedTensor q_cache_[3];
  mutable bool q_valid_[3] = {false, false, false};
  mutable Tensor fp_cache_, bias_cache_;
  mutable bool fp_valid_ = false, bias_valid_ = false;
};

// A sequence slot's KV history on the device (KvCache, src/model.cpp:142-171).
class KvCache {
 public:
  KvCache() = default;
  int64_t length() const;
  int64_t max_length() const;
  int slot() const { return slot_; }

 private:
  friend class Model;
  const Model* model_ = nullptr;
  int slot_ = 0;
};

struct SwitchEvent {
  std::string layer_id;
  Rung from = Rung::Fp;
  Rung to = Rung::Int8;
};

class Model {
 public:
  Model() = default;  // empty: assign a built or loaded model to it
  explicit Model(ModelConfig cfg);
  ~Model();
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;
  Model(Model&& o) noexcept;
  Model& operator=(Model&& o) noexcept;

  const ModelConfig& config() const { return cfg_; }
  // The KV history lives on the device in the model's sequence slots; a KvCache names a slot.
  KvCache make_cache(int slot = 0) const;    // empties the slot's history
  KvCache attach_cache(int slot = 0) const;  // handle on the slot's current history

  // Logits for every prompt position (n x V) / the next token (1 x V), as the reference's
  // const forwards (src/model.cpp:245-266); the step accounting is mutable state, as there.
  Tensor forward_prefill(std::span<const TokenId> tokens, KvCache& cache) const;
  Tensor forward_decode(TokenId token, KvCache& cache) const;

  std::optional<SwitchEvent> set_precision(std::string_view layer_id, Rung bits, int slot = 0);
  void set_all_precision(Rung bits, int slot = 0);
  Rung precision(int linear_index, int slot = 0) const;

  double effective_bits(int slot = 0) const;
  double weight_bytes_per_pass(int slot = 0) const;

  size_t num_linears() const { return layers_.size(); }
  const std::vector<std::string>& linear_ids() const { return ids_; }
  int linear_index(std::string_view id) const;  // -1 if unknown
  MultiPrecisionLayer& linear(int i) { return layers_.at(static_cast<size_t>(i)); }
  const MultiPrecisionLayer& linear(int i) const { return layers_.at(static_cast<size_t>(i)); }
  MultiPrecisionLayer* find_layer(std::string_view id);
  const MultiPrecisionLayer* find_layer(std::string_view id) const;
  // every switchable linear in the reference's order (blocks.i.attn.wq .. ffn.w2 / llama ids, head)
  std::vector<const MultiPrecisionLayer*> linear_layers() const;
  std::vector<MultiPrecisionLayer*> linear_layers();
  MultiPrecisionLayer& head() { return layers_.back(); }
  const MultiPrecisionLayer& head() const { return layers_.back(); }

  const StepStats& step_stats() const { return stats_; }
  void reset_step_stats() { stats_.reset(); }

  // Parameters by name (see fq_model_set_param) and device-side random initialisation.
  void set_param(const std::string& name, const Tensor& t);
  void init_random(uint64_t seed, float std = 0.02f);

  fq_model* handle() const { return model_; }

  // Lower-level batched step used by the engine: one decode step for `slots`, per-row
  // statistics only (no logits copy).  Returns the rows' statistics.
  std::vector<fq_row_stats> decode_rows(std::span<const int32_t> slots, std::span<const TokenId> tokens);
  // n decode steps of `slot` fed on the device with the previous argmax (fq_model_decode_chain);
  // step_stats() then holds ONE step's accounting (the chain's time split evenly)
  std::vector<fq_row_stats> decode_chain_rows(int slot, int n);
  // Single-row llama decode steps with the device phase clock on: step_stats() then carries the
  // per-precision linear time and the step's device time measured on the device
  // (fq_model_decode_timed) instead of the step time split by bytes.
  void set_device_timed_buckets(bool on) { timed_buckets_ = on; }
  std::vector<fq_row_stats> prefill_rows(int slot, std::span<const TokenId> tokens);

 private:
  friend class MultiPrecisionLayer;
  friend class KvCache;
  void account_step(uint64_t ns, int slot) const;
  std::vector<int32_t> precision_row(int slot) const;  // every linear's rung, one C-ABI call
  ModelConfig cfg_;
  fq_model* model_ = nullptr;
  std::vector<std::string> ids_;
  std::vector<MultiPrecisionLayer> layers_;
  mutable StepStats stats_;
  bool timed_buckets_ = false;
};

double effective_bits(std::span<const MultiPrecisionLayer* const> layers);

// The reference's weight container, "flexquant-weights v1" (src/model_io.cpp:130-258).
// Reference-architecture files load into a device model with fp + W8 + W4 rungs and biases
// resident, exactly as the reference writes them.  Llama-architecture models use the same
// container with two extra config fields (arch=llama group_size=G) and their own tensor names
// (tok_emb, blocks.i.attn_norm / ffn_norm, final_norm, and per linear only the quantized
// ".w8" / ".w4" records, g-per-row groups): save_model_file writes whichever the model is.
void save_model_file(const Model& model, const std::string& path);
Model load_model_file(const std::string& path, int max_batch = 1);

// Process-wide device context used by the host API (device = $FQ_DEVICE, else $LOCAL_RANK, else 0).
fq_ctx* runtime();

}  // namespace flexquant

namespace flexquant {

// Engine extensions used by the benchmark and the calibration tooling.
struct WeightKl {
  std::vector<double> kl8, kl4;  // weight-histogram KL of the W8 / W4 rung per linear
};
// Random N(0, std) initialisation on the device that also reports the reference analyzer's
// weight-histogram KL of both rungs of every linear (the fp weights are transient).
WeightKl init_random_with_kl(Model& model, uint64_t seed, float std, int bins);

struct GemvProfile {
  double ms_per_launch = 0.0;
  int64_t launches_per_pass = 0;
  int64_t bytes_per_pass = 0;
};
// Times the decode step's GEMV phases alone (CUDA events on the engine stream).
GemvProfile profile_gemvs(Model& model, int slot, int reps);

// Algorithmic bytes of one decode step of `slots` (weights at their rungs, KV read).
std::pair<int64_t, int64_t> step_bytes(const Model& model, std::span<const int32_t> slots);

// The engine's CUDA stream (cudaStream_t) for callers that time with events.
void* runtime_stream();

}  // namespace flexquant
