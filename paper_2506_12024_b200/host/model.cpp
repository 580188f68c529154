// Model / MultiPrecisionLayer / KvCache of the C++ API over the device decoder (fq_model).
// Reference semantics: /root/reference/proj/src/model.cpp (set_precision :268-278,
// effective_bits :284-296, linear_layers order :304-330) and src/model_io.cpp (container).
#include <chrono>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

#include "device_buffer.hpp"
#include "flexquant/model.hpp"

namespace flexquant {

namespace {

uint64_t now_ns() {
  return static_cast<uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch()).count());
}

fq_model_config to_c(const ModelConfig& c) {
  fq_model_config m{};
  m.arch = static_cast<int32_t>(c.arch);
  m.act_dtype = c.arch == Arch::Llama ? (c.fp16_activations ? FQ_DT_F16 : FQ_DT_BF16) : FQ_DT_F32;
  m.vocab_size = c.vocab_size;
  m.d_model = c.d_model;
  m.n_heads = c.n_heads;
  m.head_dim = c.head_dim;
  m.n_layers = c.n_layers;
  m.ffn_dim = c.ffn_dim;
  m.max_seq_len = c.max_seq_len;
  m.tie_embeddings = c.tie_embeddings ? 1 : 0;
  m.max_batch = c.max_batch;
  m.group_size = c.group_size;
  m.norm_eps = c.norm_eps;
  m.rope_theta = c.rope_theta;
  return m;
}

}  // namespace

void ModelConfig::validate() const {
  if (vocab_size < 1 || d_model < 1 || n_heads < 1 || head_dim < 1 || n_layers < 1 || ffn_dim < 1 || max_seq_len < 1)
    throw ConfigError("model config: all dimensions must be >= 1");
  if (d_model != n_heads * head_dim) throw ConfigError("model config: d_model must equal n_heads * head_dim");
}

// ------------------------------------------------------------------ MultiPrecisionLayer
MultiPrecisionLayer::MultiPrecisionLayer(std::string id, Tensor weight, Tensor bias, int64_t group_size)
    : id_(std::move(id)), n_(weight.rows()), k_(weight.cols()), owned_(true), group_(group_size) {
  if (bias.numel() != 0 && bias.numel() != n_)
    throw DimensionError("layer " + id_ + ": bias length does not match output features");
  detail::check(fq_layer_create(runtime(), n_, k_, group_size, &layer_));
  detail::check(fq_layer_upload_fp(layer_, weight.data()));
  if (bias.numel()) detail::check(fq_layer_upload_bias(layer_, bias.data()));
  standalone_rung_ = Rung::Fp;
  host_fp_ = std::move(weight);
}

MultiPrecisionLayer::~MultiPrecisionLayer() {
  if (owned_ && layer_) fq_layer_destroy(layer_);
}

MultiPrecisionLayer::MultiPrecisionLayer(MultiPrecisionLayer&& o) noexcept { *this = std::move(o); }

MultiPrecisionLayer& MultiPrecisionLayer::operator=(MultiPrecisionLayer&& o) noexcept {
  if (this != &o) {
    if (owned_ && layer_) fq_layer_destroy(layer_);
    id_ = std::move(o.id_);
    n_ = o.n_;
    k_ = o.k_;
    layer_ = o.layer_;
    owned_ = o.owned_;
    model_ = o.model_;
    index_ = o.index_;
    standalone_rung_ = o.standalone_rung_;
    group_ = o.group_;
    host_fp_ = std::move(o.host_fp_);
    for (int i = 0; i < 3; ++i) {
      q_cache_[i] = std::move(o.q_cache_[i]);
      q_valid_[i] = o.q_valid_[i];
    }
    fp_cache_ = std::move(o.fp_cache_);
    bias_cache_ = std::move(o.bias_cache_);
    fp_valid_ = o.fp_valid_;
    bias_valid_ = o.bias_valid_;
    o.layer_ = nullptr;
    o.owned_ = false;
  }
  return *this;
}

void MultiPrecisionLayer::quantize_rungs(QuantMode mode) {
  if (host_fp_.numel() == 0) throw StateError("layer " + id_ + ": no fp weights to quantize");
  set_quantized(Rung::Int8, quantize(host_fp_, 8, mode, group_));
  set_quantized(Rung::Int4, quantize(host_fp_, 4, mode, group_));
}

Rung MultiPrecisionLayer::current() const {
  if (model_) return model_->precision(index_);
  return standalone_rung_;
}

bool MultiPrecisionLayer::has(Rung r) const {
  int32_t o = 0;
  detail::check(fq_layer_has(layer_, static_cast<int32_t>(r), &o));
  return o != 0;
}

void MultiPrecisionLayer::set_current(Rung r) {
  if (!has(r)) throw StateError("layer " + id_ + ": precision '" + to_string(r) + "' not available");
  if (model_) {
    detail::check(fq_model_set_rung(model_->handle(), 0, index_, static_cast<int32_t>(r)));
  } else {
    standalone_rung_ = r;
  }
}

void MultiPrecisionLayer::set_quantized(Rung r, const QuantizedTensor& q) {
  q.validate();
  q_valid_[static_cast<int>(r)] = false;
  if (q.rows != n_ || q.cols != k_) throw DimensionError("layer " + id_ + ": quantized payload shape mismatch");
  if (r == Rung::Fp) throw ConfigError("layer " + id_ + ": fp rung is not a quantized payload");
  if (q.bits != quantized_bits(r)) throw ConfigError("layer " + id_ + ": expected " + std::to_string(quantized_bits(r)) + "-bit payload");
  int64_t n = 0, k = 0, g = 0;
  detail::check(fq_layer_shape(layer_, &n, &k, &g));
  if (q.group() != g) throw ConfigError("layer " + id_ + ": quantization group does not match the layer");
  detail::check(fq_layer_upload_quantized(layer_, static_cast<int32_t>(r), static_cast<int32_t>(q.mode),
                                          q.payload.data(), static_cast<int64_t>(q.payload.size()), q.scale.data(),
                                          q.zero_point.data(), static_cast<int64_t>(q.scale.size())));
}

const QuantizedTensor& MultiPrecisionLayer::quantized(Rung r) const {
  if (r == Rung::Fp || !has(r))
    throw StateError("layer " + id_ + ": no quantized payload for rung '" + to_string(r) + "'");
  const int ri = static_cast<int>(r);
  if (q_valid_[ri]) return q_cache_[ri];
  int64_t n = 0, k = 0, g = 0;
  detail::check(fq_layer_shape(layer_, &n, &k, &g));
  QuantizedTensor q;
  q.bits = quantized_bits(r);
  q.rows = n;
  q.cols = k;
  q.group_size = g >= k ? 0 : g;
  q.payload.resize(q.expected_payload_bytes());
  q.scale.resize(static_cast<size_t>(n * q.groups_per_row()));
  q.zero_point.resize(q.scale.size());
  detail::check(fq_layer_download_quantized(layer_, static_cast<int32_t>(r), q.payload.data(), q.scale.data(),
                                            q.zero_point.data()));
  q_cache_[ri] = std::move(q);
  q_valid_[ri] = true;
  return q_cache_[ri];
}

const Tensor& MultiPrecisionLayer::fp_weight() const {
  if (host_fp_.numel()) return host_fp_;
  if (!fp_valid_) {
    int32_t present = 0;
    detail::check(fq_layer_download_fp(layer_, nullptr, &present));
    fp_cache_ = present ? Tensor({n_, k_}) : Tensor();
    if (present) detail::check(fq_layer_download_fp(layer_, fp_cache_.data(), &present));
    fp_valid_ = true;
  }
  return fp_cache_;
}

const Tensor& MultiPrecisionLayer::bias() const {
  if (!bias_valid_) {
    int32_t present = 0;
    detail::check(fq_layer_download_bias(layer_, nullptr, &present));
    bias_cache_ = present ? Tensor({n_}) : Tensor();
    if (present) detail::check(fq_layer_download_bias(layer_, bias_cache_.data(), &present));
    bias_valid_ = true;
  }
  return bias_cache_;
}

Tensor MultiPrecisionLayer::forward(const Tensor& x, StepStats* stats) const {
  const Rung r = current();
  if (!has(r)) throw StateError("layer " + id_ + ": active precision has no payload");
  if (x.cols() != k_) throw DimensionError("linear: input width " + x.shape_str() + " does not match weight");
  const uint64_t t0 = now_ns();
  const int64_t m = x.rows();
  DeviceBuffer xd(sizeof(float) * x.numel()), yd(sizeof(float) * m * n_);
  xd.upload(x.data(), sizeof(float) * x.numel());
  detail::check(fq_gemv(runtime(), layer_, static_cast<int32_t>(r), m, xd.get(), FQ_DT_F32, yd.get(), FQ_DT_F32,
                        FQ_NUMERICS_EXACT));
  Tensor y({m, n_});
  yd.download(y.data(), sizeof(float) * y.numel());
  if (stats) {
    const uint64_t dt = now_ns() - t0;
    (r == Rung::Fp ? stats->ns_fp : r == Rung::Int8 ? stats->ns_int8 : stats->ns_int4) += dt;
    stats->weight_bytes += static_cast<double>(param_count()) * accounting_bits(r) / 8.0;
  }
  return y;
}

Tensor linear(const Tensor& x, const Tensor& w, const Tensor& bias) {
  if (w.cols() != x.cols()) throw DimensionError("linear: input width " + x.shape_str() + " does not match weight " + w.shape_str());
  if (bias.numel() != 0 && bias.numel() != w.rows()) throw DimensionError("linear: bias length mismatch");
  MultiPrecisionLayer l("linear", w, bias);
  return l.forward(x, nullptr);
}

// ------------------------------------------------------------------ KvCache
int64_t KvCache::length() const {
  int64_t n = 0;
  detail::check(fq_model_slot_length(model_->handle(), slot_, &n));
  return n;
}
int64_t KvCache::max_length() const { return model_->config().max_seq_len; }

// ------------------------------------------------------------------ Model
Model::Model(ModelConfig cfg) : cfg_(cfg) {
  cfg_.validate();
  const fq_model_config c = to_c(cfg_);
  detail::check(fq_model_create(runtime(), &c, &model_));
  int32_t n = 0;
  detail::check(fq_model_num_linears(model_, &n));
  char buf[256];
  for (int i = 0; i < n; ++i) {
    detail::check(fq_model_linear_id(model_, i, buf, sizeof(buf)));
    ids_.emplace_back(buf);
    MultiPrecisionLayer l;
    l.id_ = buf;
    detail::check(fq_model_linear(model_, i, &l.layer_));
    int64_t rows = 0, cols = 0, g = 0;
    detail::check(fq_layer_shape(l.layer_, &rows, &cols, &g));
    l.n_ = rows;
    l.k_ = cols;
    l.owned_ = false;
    l.model_ = this;
    l.index_ = i;
    layers_.push_back(std::move(l));
  }
}

Model::~Model() {
  layers_.clear();
  if (model_) fq_model_destroy(model_);
}

Model::Model(Model&& o) noexcept { *this = std::move(o); }

Model& Model::operator=(Model&& o) noexcept {
  if (this != &o) {
    layers_.clear();
    if (model_) fq_model_destroy(model_);
    cfg_ = o.cfg_;
    model_ = o.model_;
    ids_ = std::move(o.ids_);
    layers_ = std::move(o.layers_);
    stats_ = o.stats_;
    o.model_ = nullptr;
    o.layers_.clear();
    for (MultiPrecisionLayer& l : layers_) l.model_ = this;  // model views point at their owner
  }
  return *this;
}

std::vector<const MultiPrecisionLayer*> Model::linear_layers() const {
  std::vector<const MultiPrecisionLayer*> out;
  for (const MultiPrecisionLayer& l : layers_) out.push_back(&l);
  return out;
}

std::vector<MultiPrecisionLayer*> Model::linear_layers() {
  std::vector<MultiPrecisionLayer*> out;
  for (MultiPrecisionLayer& l : layers_) out.push_back(&l);
  return out;
}

KvCache Model::make_cache(int slot) const {
  detail::check(fq_model_reset_slot(model_, slot));
  KvCache c;
  c.model_ = this;
  c.slot_ = slot;
  return c;
}

KvCache Model::attach_cache(int slot) const {
  if (slot < 0 || slot >= cfg_.max_batch) throw InputError("slot out of range");
  KvCache c;
  c.model_ = this;
  c.slot_ = slot;
  return c;
}

std::vector<int32_t> Model::precision_row(int slot) const {
  std::vector<int32_t> r(layers_.size());
  detail::check(fq_model_get_rungs(model_, slot, r.data(), static_cast<int32_t>(r.size())));
  return r;
}

void Model::account_step(uint64_t ns, int slot) const {
  // per-rung buckets: the step's time split by each rung's share of the weight bytes
  double b[3] = {0, 0, 0};
  const std::vector<int32_t> row = precision_row(slot);
  for (size_t i = 0; i < layers_.size(); ++i) {
    const Rung r = static_cast<Rung>(row[i]);
    b[static_cast<int>(r)] += static_cast<double>(layers_[i].param_count()) * accounting_bits(r) / 8.0;
  }
  const double tot = b[0] + b[1] + b[2];
  stats_.weight_bytes += tot;
  stats_.ns_forward += ns;
  if (tot > 0) {
    stats_.ns_fp += static_cast<uint64_t>(ns * b[0] / tot);
    stats_.ns_int8 += static_cast<uint64_t>(ns * b[1] / tot);
    stats_.ns_int4 += static_cast<uint64_t>(ns * b[2] / tot);
  }
}

std::vector<fq_row_stats> Model::prefill_rows(int slot, std::span<const TokenId> tokens) {
  std::vector<fq_row_stats> st(tokens.size());
  const uint64_t t0 = now_ns();
  detail::check(fq_model_prefill(model_, slot, tokens.data(), static_cast<int64_t>(tokens.size()), nullptr, st.data()));
  account_step(now_ns() - t0, slot);
  return st;
}

std::vector<fq_row_stats> Model::decode_rows(std::span<const int32_t> slots, std::span<const TokenId> tokens) {
  if (slots.size() != tokens.size()) throw DimensionError("decode: slots / tokens length mismatch");
  std::vector<fq_row_stats> st(slots.size());
  if (timed_buckets_ && slots.size() == 1 && cfg_.arch == Arch::Llama) {
    uint64_t ns[3] = {0, 0, 0}, step = 0;
    const uint64_t t0 = now_ns();
    detail::check(fq_model_decode_timed(model_, slots[0], tokens[0], nullptr, st.data(), ns, &step));
    if (step == 0) {  // the program's first step runs unprofiled
      account_step(now_ns() - t0, slots[0]);
      return st;
    }
    stats_.weight_bytes += weight_bytes_per_pass(slots[0]);
    stats_.ns_fp += ns[0];
    stats_.ns_int8 += ns[1];
    stats_.ns_int4 += ns[2];
    stats_.ns_forward += now_ns() - t0;  // the forward's wall time, as the reference measures it
    return st;
  }
  const uint64_t t0 = now_ns();
  detail::check(fq_model_decode(model_, static_cast<int32_t>(slots.size()), slots.data(), tokens.data(), nullptr,
                                st.data()));
  account_step(now_ns() - t0, slots.empty() ? 0 : slots[0]);
  return st;
}

std::vector<fq_row_stats> Model::decode_chain_rows(int slot, int n) {
  std::vector<fq_row_stats> st(static_cast<size_t>(n));
  const uint64_t t0 = now_ns();
  detail::check(fq_model_decode_chain(model_, slot, n, st.data()));
  account_step((now_ns() - t0) / static_cast<uint64_t>(n), slot);
  return st;
}

Tensor Model::forward_prefill(std::span<const TokenId> tokens, KvCache& cache) const {
  const int64_t n = static_cast<int64_t>(tokens.size());
  if (n < 1) throw InputError("prefill: empty prompt");
  DeviceBuffer l(sizeof(float) * n * cfg_.vocab_size);
  const uint64_t t0 = now_ns();
  std::vector<fq_row_stats> st(tokens.size());
  detail::check(fq_model_prefill(model_, cache.slot(), tokens.data(), n, static_cast<float*>(l.get()), st.data()));
  account_step(now_ns() - t0, cache.slot());
  Tensor out({n, cfg_.vocab_size});
  l.download(out.data(), sizeof(float) * out.numel());
  return out;
}

Tensor Model::forward_decode(TokenId token, KvCache& cache) const {
  DeviceBuffer l(sizeof(float) * cfg_.vocab_size);
  const int32_t slot = cache.slot();
  fq_row_stats st;
  const uint64_t t0 = now_ns();
  detail::check(fq_model_decode(model_, 1, &slot, &token, static_cast<float*>(l.get()), &st));
  account_step(now_ns() - t0, slot);
  Tensor out({1, cfg_.vocab_size});
  l.download(out.data(), sizeof(float) * out.numel());
  return out;
}

Rung Model::precision(int linear_index, int slot) const {
  int32_t r = 0;
  detail::check(fq_model_get_rung(model_, slot, linear_index, &r));
  return static_cast<Rung>(r);
}

int Model::linear_index(std::string_view id) const {
  for (size_t i = 0; i < ids_.size(); ++i)
    if (ids_[i] == id) return static_cast<int>(i);
  return -1;
}

MultiPrecisionLayer* Model::find_layer(std::string_view id) {
  const int i = linear_index(id);
  return i < 0 ? nullptr : &layers_[static_cast<size_t>(i)];
}
const MultiPrecisionLayer* Model::find_layer(std::string_view id) const {
  const int i = linear_index(id);
  return i < 0 ? nullptr : &layers_[static_cast<size_t>(i)];
}

std::optional<SwitchEvent> Model::set_precision(std::string_view layer_id, Rung bits, int slot) {
  const int i = linear_index(layer_id);
  if (i < 0) throw StateError("set_precision: unknown layer '" + std::string(layer_id) + "'");
  if (!layers_[static_cast<size_t>(i)].has(bits))
    throw StateError("set_precision: layer '" + std::string(layer_id) + "' has no rung '" + to_string(bits) + "'");
  const Rung cur = precision(i, slot);
  if (cur == bits) return std::nullopt;
  detail::check(fq_model_set_rung(model_, slot, i, static_cast<int32_t>(bits)));
  return SwitchEvent{ids_[static_cast<size_t>(i)], cur, bits};
}

void Model::set_all_precision(Rung bits, int slot) {
  detail::check(fq_model_set_all_rungs(model_, slot, static_cast<int32_t>(bits)));
}

double Model::effective_bits(int slot) const {
  double num = 0.0, den = 0.0;
  const std::vector<int32_t> row = precision_row(slot);
  for (size_t i = 0; i < layers_.size(); ++i) {
    num += static_cast<double>(layers_[i].param_count()) * accounting_bits(static_cast<Rung>(row[i]));
    den += static_cast<double>(layers_[i].param_count());
  }
  return den > 0.0 ? num / den : 0.0;
}

double Model::weight_bytes_per_pass(int slot) const {
  double b = 0.0;
  const std::vector<int32_t> row = precision_row(slot);
  for (size_t i = 0; i < layers_.size(); ++i)
    b += static_cast<double>(layers_[i].param_count()) * accounting_bits(static_cast<Rung>(row[i])) / 8.0;
  return b;
}

void Model::set_param(const std::string& name, const Tensor& t) {
  detail::check(fq_model_set_param(model_, name.c_str(), t.data(), t.numel()));
}

void Model::init_random(uint64_t seed, float std) { detail::check(fq_model_init_random(model_, seed, std)); }

double effective_bits(std::span<const MultiPrecisionLayer* const> layers) {
  double num = 0.0, den = 0.0;
  for (const MultiPrecisionLayer* l : layers) {
    num += static_cast<double>(l->param_count()) * accounting_bits(l->current());
    den += static_cast<double>(l->param_count());
  }
  return den > 0.0 ? num / den : 0.0;
}

// ------------------------------------------------------------------ weights container
namespace {

struct Reader {
  std::ifstream is;
  uint32_t u32() {
    uint32_t v;
    if (!is.read(reinterpret_cast<char*>(&v), 4)) throw FormatError("weights file: unexpected end of file");
    return v;
  }
  uint8_t u8() {
    char c;
    if (!is.get(c)) throw FormatError("weights file: unexpected end of file");
    return static_cast<uint8_t>(c);
  }
  void bytes(void* p, size_t n) {
    if (!is.read(static_cast<char*>(p), static_cast<std::streamsize>(n))) throw FormatError("weights file: unexpected end of file");
  }
};

int64_t field(const std::string& line, const std::string& key) {
  const size_t p = line.find(key + "=");
  if (p == std::string::npos) throw FormatError("weights file: config field '" + key + "' missing");
  return std::stoll(line.substr(p + key.size() + 1));
}

}  // namespace

namespace {

// optional config field (the llama extension): default when absent
int64_t field_or(const std::string& line, const std::string& key, int64_t dflt) {
  const size_t p = line.find(" " + key + "=");
  return p == std::string::npos ? dflt : std::stoll(line.substr(p + key.size() + 2));
}

struct QRecord {
  int bits = 8, mode = 0;
  uint32_t rows = 0, cols = 0, group = 0;  // group 0 = per row (the reference's records)
  std::vector<float> scale;
  std::vector<int32_t> zp;
  std::vector<uint8_t> payload;
};

// ---- writer
void put_u32(std::ostream& os, uint32_t v) { os.write(reinterpret_cast<const char*>(&v), 4); }
void put_name(std::ostream& os, const std::string& n, uint8_t tag) {
  put_u32(os, static_cast<uint32_t>(n.size()));
  os.write(n.data(), static_cast<std::streamsize>(n.size()));
  os.put(static_cast<char>(tag));
}
void put_tensor(std::ostream& os, const std::string& name, const Tensor& t) {
  put_name(os, name, 0);
  put_u32(os, static_cast<uint32_t>(t.shape().size()));
  for (int64_t d : t.shape()) put_u32(os, static_cast<uint32_t>(d));
  os.write(reinterpret_cast<const char*>(t.data()), static_cast<std::streamsize>(sizeof(float) * t.numel()));
}
// tag 1: the reference's per-row record; tag 2: the group-wise extension (scale / zp per group)
void put_quantized(std::ostream& os, const std::string& name, const QuantizedTensor& q) {
  const bool grouped = q.group() != q.cols;
  put_name(os, name, grouped ? 2 : 1);
  os.put(static_cast<char>(q.bits));
  os.put(static_cast<char>(q.mode));
  put_u32(os, static_cast<uint32_t>(q.rows));
  put_u32(os, static_cast<uint32_t>(q.cols));
  if (grouped) put_u32(os, static_cast<uint32_t>(q.group()));
  os.write(reinterpret_cast<const char*>(q.scale.data()), static_cast<std::streamsize>(4 * q.scale.size()));
  os.write(reinterpret_cast<const char*>(q.zero_point.data()), static_cast<std::streamsize>(4 * q.zero_point.size()));
  os.write(reinterpret_cast<const char*>(q.payload.data()), static_cast<std::streamsize>(q.payload.size()));
}

Tensor get_param(const Model& m, const std::string& name, std::vector<int64_t> shape) {
  Tensor t(std::move(shape));
  detail::check(fq_model_get_param(m.handle(), name.c_str(), t.data(), t.numel()));
  return t;
}

}  // namespace

void save_model_file(const Model& model, const std::string& path) {
  if (!model.handle()) throw StateError("save_model_file: empty model");
  std::ofstream os(path, std::ios::binary);
  if (!os) throw FormatError("cannot open weights file for writing: " + path);
  const ModelConfig& c = model.config();
  const bool llama = c.arch == Arch::Llama;
  const int64_t d = c.d_model, L = c.n_layers;
  os << "flexquant-weights v1\n";
  os << "vocab_size=" << c.vocab_size << " d_model=" << d << " n_heads=" << c.n_heads << " head_dim=" << c.head_dim
     << " n_layers=" << L << " ffn_dim=" << c.ffn_dim << " max_seq_len=" << c.max_seq_len
     << " tie_embeddings=" << (c.tie_embeddings ? 1 : 0);
  if (llama) os << " arch=llama group_size=" << c.group_size;
  os << "\n";
  const std::vector<const MultiPrecisionLayer*> lin = model.linear_layers();
  // reference: embeddings + final norm + per block (4 norms + 6 x (fp, bias)) + head (fp, bias),
  // and both quantized rungs of every linear; llama: tok_emb + final norm + 2 norms per block and
  // both rungs of every linear
  const bool has_head = !c.tie_embeddings;
  const size_t count = llama ? 2 + 2 * static_cast<size_t>(L) + 2 * lin.size()
                             : 4 + static_cast<size_t>(L) * 16 + (has_head ? 2 : 0) + 2 * lin.size();
  os << "tensor_count=" << count << "\n";
  put_tensor(os, "tok_emb", get_param(model, "tok_emb", {c.vocab_size, d}));
  auto put_linear = [&](const MultiPrecisionLayer& l) {
    if (!llama) {
      put_tensor(os, l.id(), l.fp_weight());
      put_tensor(os, l.id() + ".bias", l.bias());
    }
    put_quantized(os, l.id() + ".w8", l.quantized(Rung::Int8));
    put_quantized(os, l.id() + ".w4", l.quantized(Rung::Int4));
  };
  size_t li = 0;
  if (!llama) {
    put_tensor(os, "pos_emb", get_param(model, "pos_emb", {c.max_seq_len, d}));
    for (int64_t i = 0; i < L; ++i) {
      const std::string p = "blocks." + std::to_string(i) + ".";
      put_tensor(os, p + "ln1.gamma", get_param(model, p + "ln1.gamma", {d}));
      put_tensor(os, p + "ln1.beta", get_param(model, p + "ln1.beta", {d}));
      for (int k = 0; k < 4; ++k) put_linear(*lin[li++]);
      put_tensor(os, p + "ln2.gamma", get_param(model, p + "ln2.gamma", {d}));
      put_tensor(os, p + "ln2.beta", get_param(model, p + "ln2.beta", {d}));
      for (int k = 0; k < 2; ++k) put_linear(*lin[li++]);
    }
    put_tensor(os, "ln_f.gamma", get_param(model, "final_norm.gamma", {d}));
    put_tensor(os, "ln_f.beta", get_param(model, "final_norm.beta", {d}));
    if (has_head) put_linear(*lin[li++]);
  } else {
    for (int64_t i = 0; i < L; ++i) {
      const std::string p = "blocks." + std::to_string(i) + ".";
      put_tensor(os, p + "attn_norm", get_param(model, p + "attn_norm", {d}));
      for (int k = 0; k < 4; ++k) put_linear(*lin[li++]);
      put_tensor(os, p + "ffn_norm", get_param(model, p + "ffn_norm", {d}));
      for (int k = 0; k < 3; ++k) put_linear(*lin[li++]);
    }
    put_tensor(os, "final_norm", get_param(model, "final_norm", {d}));
    put_linear(*lin[li++]);
  }
  if (!os) throw FormatError("failed writing weights file: " + path);
}

Model load_model_file(const std::string& path, int max_batch) {
  Reader r;
  r.is.open(path, std::ios::binary);
  if (!r.is) throw FormatError("cannot open weights file: " + path);
  std::string line;
  if (!std::getline(r.is, line) || line != "flexquant-weights v1") throw FormatError("weights file: bad or missing header");
  if (!std::getline(r.is, line)) throw FormatError("weights file: missing config line");
  ModelConfig cfg;
  cfg.vocab_size = field(line, "vocab_size");
  cfg.d_model = field(line, "d_model");
  cfg.n_heads = field(line, "n_heads");
  cfg.head_dim = field(line, "head_dim");
  cfg.n_layers = field(line, "n_layers");
  cfg.ffn_dim = field(line, "ffn_dim");
  cfg.max_seq_len = field(line, "max_seq_len");
  cfg.tie_embeddings = field(line, "tie_embeddings") != 0;
  const bool llama = line.find(" arch=llama") != std::string::npos;
  cfg.arch = llama ? Arch::Llama : Arch::Reference;
  cfg.group_size = field_or(line, "group_size", 0);
  cfg.max_batch = max_batch;
  if (!std::getline(r.is, line)) throw FormatError("weights file: missing tensor count line");
  const int64_t count = field(line, "tensor_count");
  Model model(cfg);
  std::map<std::string, Tensor> tensors;
  std::map<std::string, QRecord> quants;
  for (int64_t i = 0; i < count; ++i) {
    const uint32_t nl = r.u32();
    if (nl > 4096) throw FormatError("weights file: unreasonable tensor name length");
    std::string name(nl, '\0');
    r.bytes(name.data(), nl);
    const uint8_t tag = r.u8();
    if (tag == 0) {
      const uint32_t nd = r.u32();
      if (nd == 0 || nd > 4) throw FormatError("weights file: bad tensor rank");
      std::vector<int64_t> shape(nd);
      int64_t numel = 1;
      for (auto& dim : shape) {
        dim = r.u32();
        numel *= dim;
      }
      std::vector<float> data(static_cast<size_t>(numel));
      r.bytes(data.data(), sizeof(float) * data.size());
      tensors.emplace(name, Tensor::from_data(shape, std::move(data)));
    } else if (tag == 1 || tag == 2) {
      QRecord q;
      q.bits = r.u8();
      q.mode = r.u8();
      if (q.mode > 1) throw FormatError("weights file: bad quantization mode");
      if (q.bits != 8 && q.bits != 4) throw FormatError("weights file: bad bit-width");
      q.rows = r.u32();
      q.cols = r.u32();
      q.group = tag == 2 ? r.u32() : 0;
      if (tag == 2 && (q.group == 0 || q.cols == 0)) throw FormatError("weights file: bad quantization group");
      const size_t groups = static_cast<size_t>(q.rows) * (q.group ? (q.cols + q.group - 1) / q.group : 1);
      q.scale.resize(groups);
      q.zp.resize(groups);
      r.bytes(q.scale.data(), 4 * q.scale.size());
      r.bytes(q.zp.data(), 4 * q.zp.size());
      q.payload.resize((static_cast<size_t>(q.rows) * q.cols * q.bits + 7) / 8);
      r.bytes(q.payload.data(), q.payload.size());
      quants.emplace(name, std::move(q));
    } else {
      throw FormatError("weights file: unknown dtype tag");
    }
  }
  auto take = [&](const std::string& n) -> Tensor& {
    auto it = tensors.find(n);
    if (it == tensors.end()) throw FormatError("weights file: tensor '" + n + "' missing");
    return it->second;
  };
  model.set_param("tok_emb", take("tok_emb"));
  if (llama) {
    for (int64_t i = 0; i < cfg.n_layers; ++i) {
      const std::string p = "blocks." + std::to_string(i) + ".";
      for (const char* nm : {"attn_norm", "ffn_norm"}) model.set_param(p + nm, take(p + nm));
    }
    model.set_param("final_norm", take("final_norm"));
  } else {
    model.set_param("pos_emb", take("pos_emb"));
    for (int64_t i = 0; i < cfg.n_layers; ++i) {
      const std::string p = "blocks." + std::to_string(i) + ".";
      for (const char* nm : {"ln1.gamma", "ln1.beta", "ln2.gamma", "ln2.beta"}) model.set_param(p + nm, take(p + nm));
    }
    model.set_param("final_norm.gamma", take("ln_f.gamma"));
    model.set_param("final_norm.beta", take("ln_f.beta"));
  }
  for (size_t i = 0; i < model.num_linears(); ++i) {
    const std::string& id = model.linear_ids()[i];
    fq_layer* L = model.linear(static_cast<int>(i)).handle();
    if (!llama) {
      detail::check(fq_layer_upload_fp(L, take(id).data()));
      detail::check(fq_layer_upload_bias(L, take(id + ".bias").data()));
    }
    for (const auto& [tag, rung] : {std::pair<const char*, int>{".w8", FQ_RUNG_INT8}, {".w4", FQ_RUNG_INT4}}) {
      auto it = quants.find(id + tag);
      if (it == quants.end()) {
        if (llama) throw FormatError("weights file: quantized record '" + id + tag + "' missing");
        // files without stored rungs are RTN-quantized at load time (src/model_io.cpp:226-229)
        const QuantizedTensor q = quantize(take(id), rung == FQ_RUNG_INT8 ? 8 : 4, QuantMode::Asymmetric);
        detail::check(fq_layer_upload_quantized(L, rung, 0, q.payload.data(), static_cast<int64_t>(q.payload.size()),
                                                q.scale.data(), q.zero_point.data(), static_cast<int64_t>(q.scale.size())));
        continue;
      }
      const QRecord& q = it->second;
      if ((rung == FQ_RUNG_INT8) != (q.bits == 8)) throw FormatError("weights file: '" + id + tag + "' has the wrong bit-width");
      detail::check(fq_layer_upload_quantized(L, rung, q.mode, q.payload.data(), static_cast<int64_t>(q.payload.size()),
                                              q.scale.data(), q.zp.data(), static_cast<int64_t>(q.scale.size())));
    }
  }
  model.set_all_precision(llama ? Rung::Int8 : Rung::Fp);
  return model;
}

}  // namespace flexquant

namespace flexquant {

WeightKl init_random_with_kl(Model& model, uint64_t seed, float std, int bins) {
  WeightKl r;
  r.kl8.resize(model.num_linears());
  r.kl4.resize(model.num_linears());
  detail::check(fq_model_init_random_kl(model.handle(), seed, std, bins, r.kl8.data(), r.kl4.data()));
  return r;
}

GemvProfile profile_gemvs(Model& model, int slot, int reps) {
  GemvProfile p;
  detail::check(fq_model_profile_gemvs(model.handle(), slot, reps, &p.ms_per_launch, &p.launches_per_pass,
                                       &p.bytes_per_pass));
  return p;
}

std::pair<int64_t, int64_t> step_bytes(const Model& model, std::span<const int32_t> slots) {
  int64_t w = 0, k = 0;
  detail::check(fq_model_step_bytes(model.handle(), static_cast<int32_t>(slots.size()), slots.data(), &w, &k));
  return {w, k};
}

void* runtime_stream() {
  void* s = nullptr;
  detail::check(fq_ctx_get_stream(runtime(), &s));
  return s;
}

}  // namespace flexquant
