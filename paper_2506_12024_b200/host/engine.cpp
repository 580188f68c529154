// Dynamic-precision generation loop (Algorithm 1) over the device decoder.
// Reference: /root/reference/proj/src/engine.cpp:30-371.  Attribution: validate_plan /
// apply_entry and traffic_report / format_traffic_report keep the reference's checks, record
// fields and report text (engine.cpp:30-54, 214-247) so traces and reports compare field for
// field; the loop itself is rewritten around batched device steps and the JSONL I/O is written
// without nlohmann/json.  Record semantics are the reference's:
// a token's record describes the precision state that produced it; switches decided at token t
// are applied after its record and take effect for token t+1; token 1 covers the prefill.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <deque>
#include <fstream>
#include <map>
#include <sstream>

#include "flexquant/engine.hpp"
#include "flexquant/metrics.hpp"
#include "host_internal.hpp"

namespace flexquant {

namespace {

uint64_t now_ns() {
  return static_cast<uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch()).count());
}

void validate_plan(const SwitchPlan& plan, const Model& model, Rung start) {
  std::map<std::string, Rung> state;
  for (const SwitchEntry& e : plan.entries) {
    if (!model.find_layer(e.layer_id)) throw ConfigError("plan references unknown layer '" + e.layer_id + "'");
    const auto it = state.find(e.layer_id);
    const Rung from = it == state.end() ? start : it->second;
    if (e.from != from)
      throw ConfigError("plan entry for '" + e.layer_id + "' starts at '" + to_string(e.from) +
                        "' but the layer would be at '" + to_string(from) + "'");
    if (!is_downward(e.from, e.to)) throw ConfigError("plan entry for '" + e.layer_id + "' is not a downward switch");
    state[e.layer_id] = e.to;
  }
}

void apply_entry(Model& model, const SwitchEntry& e, int slot, std::vector<SwitchEvent>& events) {
  const int i = model.linear_index(e.layer_id);
  if (i < 0) throw StateError("switch: unknown layer '" + e.layer_id + "'");
  const Rung cur = model.precision(i, slot);
  if (cur != e.from)
    throw StateError("switch: layer '" + e.layer_id + "' is at '" + to_string(cur) + "', plan entry expects '" +
                     to_string(e.from) + "'");
  if (auto ev = model.set_precision(e.layer_id, e.to, slot)) events.push_back(*ev);
}

// One sequence's decode state inside the (possibly batched) loop.
struct Seq {
  int slot = 0;
  std::vector<TokenId> prompt;
  SchedulerState sched;
  std::deque<double> forced_window;
  size_t forced_cursor = 0;
  fq_row_stats row{};
  GenerationResult result;
  bool done = false;
  uint64_t step_start = 0;
  StepStats step_stats;
  Seq(SchedulerConfig c, size_t n) : sched(c, n) {}
};

std::vector<GenerationResult> run_generation(std::span<const std::vector<TokenId>> prompts, Model& model,
                                             const SwitchPlan& plan, const GenerationConfig& cfg, int64_t forced_speed) {
  const ModelConfig& mc = model.config();
  if (static_cast<int>(prompts.size()) > mc.max_batch) throw ConfigError("generate: more prompts than model slots");
  if (cfg.max_new_tokens < 1) throw ConfigError("generate: max_new_tokens must be >= 1");
  for (const auto& p : prompts) {
    if (p.empty()) throw InputError("generate: empty prompt");
    if (static_cast<int64_t>(p.size()) > mc.max_seq_len) throw CapacityError("generate: prompt longer than max sequence length");
  }
  validate_plan(plan, model, cfg.start_rung);
  model.set_device_timed_buckets(cfg.device_timed_buckets);
  struct TimedOff {
    Model& m;
    ~TimedOff() { m.set_device_timed_buckets(false); }
  } timed_off{model};
  std::vector<Seq> seqs;
  seqs.reserve(prompts.size());
  for (size_t i = 0; i < prompts.size(); ++i) {
    seqs.emplace_back(cfg.scheduler, plan.size());
    Seq& s = seqs.back();
    s.slot = static_cast<int>(i);
    s.prompt = prompts[i];
    model.set_all_precision(cfg.start_rung, s.slot);
    detail::check(fq_model_reset_slot(model.handle(), s.slot));
  }
  // prefill every sequence and derive its threshold (src/engine.cpp:77-85)
  for (Seq& s : seqs) {
    s.step_start = now_ns();
    model.reset_step_stats();
    const std::vector<fq_row_stats> st = model.prefill_rows(s.slot, s.prompt);
    s.step_stats = model.step_stats();
    s.step_stats.weight_bytes = model.weight_bytes_per_pass(s.slot);  // one pass, per-call accounting
    double thre;
    if (cfg.scheduler.threshold_mode == ThresholdMode::Prefill) {
      std::vector<double> ppl(st.size());
      for (size_t i = 0; i < st.size(); ++i) ppl[i] = st[i].ppl_entropy;
      thre = derive_threshold_from_ppl(ppl, cfg.scheduler.window_len, cfg.scheduler.theta);
    } else {
      thre = cfg.scheduler.theta;
    }
    s.sched.set_threshold(thre);
    s.result.threshold = thre;
    s.row = st.back();
  }
  // one Llama sequence without eos: tokens whose scheduler decision provably cannot switch (the
  // window still filling or the cooldown running, SchedulerState::safe_observes) are decoded as
  // one device-chained block (Model::decode_chain_rows: the token fed back from the previous
  // argmax on the device); their records are written afterwards from the block's rows, in the
  // same order and with the same fields as the token-by-token loop (the block's wall time split
  // evenly over its tokens)
  const bool chainable = seqs.size() == 1 && mc.arch == Arch::Llama && forced_speed == 0 && !cfg.eos_token &&
                         !cfg.device_timed_buckets && std::getenv("FQ_NO_CHAIN") == nullptr;
  for (int64_t t = 1;; ++t) {
    if (chainable && t >= 2 && !seqs[0].done) {  // t = 1's row comes from the prefill
      Seq& s = seqs[0];
      int64_t len = 0;
      detail::check(fq_model_slot_length(model.handle(), s.slot, &len));
      const int64_t k = std::min<int64_t>({static_cast<int64_t>(std::min<size_t>(s.sched.safe_observes(), 64)),
                                           cfg.max_new_tokens - t, mc.max_seq_len - len});
      if (k >= 2) {
        const uint64_t c0 = now_ns();
        const uint64_t first_elapsed = c0 - s.step_start;  // token t came from the step before the block
        model.reset_step_stats();
        const std::vector<fq_row_stats> rows = model.decode_chain_rows(s.slot, static_cast<int>(k));
        const uint64_t per = (now_ns() - c0) / static_cast<uint64_t>(k);
        const StepStats chained = model.step_stats();
        fq_row_stats prev = s.row;
        for (int64_t j = 0; j < k; ++j) {
          TraceRecord rec;
          rec.token_index = t + j;
          rec.token_id = prev.argmax;
          rec.fault_tolerance = prev.fault_tolerance;
          rec.effective_bits = model.effective_bits(s.slot);
          rec.buckets = j == 0 ? s.step_stats : chained;
          rec.weight_bytes_touched = rec.buckets.weight_bytes;
          rec.ppl_entropy = prev.ppl_entropy;
          const SchedulerState::Decision d = s.sched.observe(rec.ppl_entropy);
          if (d.count != 0) throw StateError("generate: a chained token switched precision");
          rec.moving_average = d.window_mean;
          rec.elapsed_ns = j == 0 ? first_elapsed : per;
          s.result.trace.records.push_back(std::move(rec));
          s.result.sequence.push_back(prev.argmax);
          prev = rows[static_cast<size_t>(j)];
        }
        s.row = prev;
        s.step_start = now_ns() - per;
        s.step_stats = chained;
        s.step_stats.weight_bytes = model.weight_bytes_per_pass(s.slot);
        t += k - 1;
        continue;
      }
    }
    std::vector<int32_t> slots;
    std::vector<TokenId> toks;
    for (Seq& s : seqs) {
      if (s.done) continue;
      const TokenId token = s.row.argmax;
      TraceRecord rec;
      rec.token_index = t;
      rec.token_id = token;
      rec.fault_tolerance = s.row.fault_tolerance;
      rec.effective_bits = model.effective_bits(s.slot);
      rec.buckets = s.step_stats;
      rec.weight_bytes_touched = s.step_stats.weight_bytes;
      const uint64_t p0 = now_ns();
      rec.ppl_entropy = s.row.ppl_entropy;  // computed on the device with the logits
      rec.ns_ppl = now_ns() - p0;
      if (forced_speed > 0) {
        s.forced_window.push_back(rec.ppl_entropy);
        if (s.forced_window.size() > static_cast<size_t>(cfg.scheduler.window_len)) s.forced_window.pop_front();
        if (s.forced_window.size() == static_cast<size_t>(cfg.scheduler.window_len)) {
          double sum = 0.0;
          for (double v : s.forced_window) sum += v;
          rec.moving_average = sum / static_cast<double>(s.forced_window.size());
        }
        if (t % forced_speed == 0 && s.forced_cursor < plan.size())
          apply_entry(model, plan.entries[s.forced_cursor++], s.slot, rec.switch_events);
      } else {
        const SchedulerState::Decision d = s.sched.observe(rec.ppl_entropy);
        rec.moving_average = d.window_mean;
        for (size_t i = 0; i < d.count; ++i) apply_entry(model, plan.entries[d.first_entry + i], s.slot, rec.switch_events);
      }
      rec.elapsed_ns = now_ns() - s.step_start;
      s.result.trace.records.push_back(std::move(rec));
      s.result.sequence.push_back(token);
      int64_t len = 0;
      detail::check(fq_model_slot_length(model.handle(), s.slot, &len));
      if ((cfg.eos_token && token == *cfg.eos_token) || t == cfg.max_new_tokens || len >= mc.max_seq_len) {
        s.done = true;
        continue;
      }
      slots.push_back(s.slot);
      toks.push_back(token);
    }
    if (slots.empty()) break;
    const uint64_t t0 = now_ns();
    model.reset_step_stats();
    const std::vector<fq_row_stats> st = model.decode_rows(slots, toks);
    size_t j = 0;
    for (Seq& s : seqs) {
      if (s.done) continue;
      s.row = st[j++];
      s.step_start = t0;
      s.step_stats = model.step_stats();
      s.step_stats.weight_bytes = model.weight_bytes_per_pass(s.slot);
    }
  }
  std::vector<GenerationResult> out;
  for (Seq& s : seqs) out.push_back(std::move(s.result));
  if (!cfg.trace_path.empty() && out.size() == 1) save_trace_file(out[0].trace, cfg.trace_path);
  return out;
}

}  // namespace

GenerationResult generate(std::span<const TokenId> prompt, Model& model, const SwitchPlan& plan,
                          const GenerationConfig& cfg) {
  if (cfg.start_rung == Rung::Int4) throw ConfigError("generate: starting rung must be fp or 8");
  const std::vector<TokenId> p(prompt.begin(), prompt.end());
  return std::move(run_generation(std::span<const std::vector<TokenId>>(&p, 1), model, plan, cfg, 0)[0]);
}

GenerationResult generate_static(std::span<const TokenId> prompt, Model& model, Rung rung, const GenerationConfig& cfg) {
  GenerationConfig pinned = cfg;
  pinned.start_rung = rung;
  pinned.scheduler.threshold_mode = ThresholdMode::Absolute;
  pinned.scheduler.theta = 0.0;
  const std::vector<TokenId> p(prompt.begin(), prompt.end());
  return std::move(run_generation(std::span<const std::vector<TokenId>>(&p, 1), model, SwitchPlan{}, pinned, 0)[0]);
}

std::vector<GenerationResult> generate_batch(std::span<const std::vector<TokenId>> prompts, Model& model,
                                             const SwitchPlan& plan, const GenerationConfig& cfg) {
  if (cfg.start_rung == Rung::Int4) throw ConfigError("generate: starting rung must be fp or 8");
  return run_generation(prompts, model, plan, cfg, 0);
}

std::vector<SweepRow> sweep_switch_speed(std::span<const TokenId> prompt, Model& model, const SwitchPlan& plan,
                                         std::span<const int64_t> speeds, const GenerationConfig& cfg) {
  for (int64_t s : speeds)
    if (s < 1) throw ConfigError("sweep: speeds must be positive");
  const GenerationResult base = generate_static(prompt, model, Rung::Fp, cfg);
  const std::vector<TokenId> p(prompt.begin(), prompt.end());
  std::vector<SweepRow> rows;
  for (int64_t s : speeds) {
    GenerationResult r = std::move(run_generation(std::span<const std::vector<TokenId>>(&p, 1), model, plan, cfg, s)[0]);
    SweepRow row;
    row.speed = s;
    row.final_effective_bits = model.effective_bits();
    double bytes = 0.0;
    for (const TraceRecord& rec : r.trace.records) bytes += rec.weight_bytes_touched;
    row.mean_bytes_per_token = bytes / static_cast<double>(r.trace.records.size());
    // agreement / Rouge-L against the fp baseline (src/engine.cpp:188-191, src/metrics.cpp)
    const Agreement agr = agreement_rate(r.sequence, base.sequence);
    row.agreement_vs_fp = agr.rate;
    row.first_divergence = agr.divergence_index;
    row.rouge_l_vs_fp = rouge_l(r.sequence, base.sequence);
    row.trace = std::move(r.trace);
    rows.push_back(std::move(row));
  }
  return rows;
}

std::string sweep_csv_header() {
  return "prompt,speed,final_effective_bits,mean_bytes_per_token,agreement_vs_fp,first_divergence,rouge_l_vs_fp\n";
}

std::string sweep_csv_row(const std::string& prompt_name, const SweepRow& row) {
  char buf[320];
  const std::string div = row.first_divergence ? std::to_string(*row.first_divergence) : std::string();
  std::snprintf(buf, sizeof(buf), "%s,%lld,%.6f,%.3f,%.6f,%s,%.4f\n", prompt_name.c_str(),
                static_cast<long long>(row.speed), row.final_effective_bits, row.mean_bytes_per_token,
                row.agreement_vs_fp, div.c_str(), row.rouge_l_vs_fp);
  return buf;
}

TrafficReport traffic_report(const DecodeTrace& trace) {
  if (trace.records.empty()) throw InputError("traffic_report: empty trace");
  TrafficReport r;
  for (const TraceRecord& rec : trace.records) {
    r.total_weight_bytes += rec.weight_bytes_touched;
    r.ns_fp += rec.buckets.ns_fp;
    r.ns_int8 += rec.buckets.ns_int8;
    r.ns_int4 += rec.buckets.ns_int4;
    const uint64_t lin = rec.buckets.ns_fp + rec.buckets.ns_int8 + rec.buckets.ns_int4;
    r.ns_attention_cache += rec.buckets.ns_forward > lin ? rec.buckets.ns_forward - lin : 0;
    r.ns_ppl += rec.ns_ppl;
    r.ns_total += rec.elapsed_ns;
  }
  r.mean_bytes_per_token = r.total_weight_bytes / static_cast<double>(trace.records.size());
  const uint64_t sum = r.ns_fp + r.ns_int8 + r.ns_int4 + r.ns_attention_cache + r.ns_ppl;
  r.bucket_sum_over_total = r.ns_total ? static_cast<double>(sum) / static_cast<double>(r.ns_total) : 0.0;
  r.ppl_share = r.ns_total ? static_cast<double>(r.ns_ppl) / static_cast<double>(r.ns_total) : 0.0;
  return r;
}

std::string format_traffic_report(const TrafficReport& r) {
  std::ostringstream os;
  os << "total_weight_bytes=" << r.total_weight_bytes << "\nmean_bytes_per_token=" << r.mean_bytes_per_token
     << "\nns_fp=" << r.ns_fp << "\nns_int8=" << r.ns_int8 << "\nns_int4=" << r.ns_int4
     << "\nns_attention_cache=" << r.ns_attention_cache << "\nns_ppl=" << r.ns_ppl << "\nns_total=" << r.ns_total
     << "\nbucket_sum_over_total=" << r.bucket_sum_over_total << "\nppl_share=" << r.ppl_share << "\n";
  return os.str();
}

// ------------------------------------------------------------------ JSONL trace
namespace {

std::string num(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // keep doubles recognisable
  return s;
}

// Minimal reader for the flat trace objects written below.
struct JsonCursor {
  const std::string& s;
  size_t i = 0;
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  void expect(char c) {
    ws();
    if (i >= s.size() || s[i] != c) throw FormatError(std::string("trace: expected '") + c + "'");
    ++i;
  }
  bool peek(char c) {
    ws();
    return i < s.size() && s[i] == c;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (i < s.size() && s[i] != '"') out += s[i++];
    expect('"');
    return out;
  }
  std::string raw() {
    ws();
    size_t j = i;
    while (j < s.size() && s[j] != ',' && s[j] != '}' && s[j] != ']') ++j;
    std::string out = s.substr(i, j - i);
    i = j;
    while (!out.empty() && std::isspace(static_cast<unsigned char>(out.back()))) out.pop_back();
    return out;
  }
};

}  // namespace

void save_trace(const DecodeTrace& trace, std::ostream& os) {
  for (const TraceRecord& r : trace.records) {
    os << "{\"token_index\":" << r.token_index << ",\"token_id\":" << r.token_id << ",\"ppl_entropy\":" << num(r.ppl_entropy)
       << ",\"fault_tolerance\":" << num(r.fault_tolerance) << ",\"moving_average\":"
       << (r.moving_average ? num(*r.moving_average) : std::string("null")) << ",\"effective_bits\":" << num(r.effective_bits)
       << ",\"weight_bytes_touched\":" << num(r.weight_bytes_touched) << ",\"elapsed_ns\":" << r.elapsed_ns
       << ",\"buckets\":{\"ns_fp\":" << r.buckets.ns_fp << ",\"ns_int8\":" << r.buckets.ns_int8
       << ",\"ns_int4\":" << r.buckets.ns_int4 << ",\"ns_forward\":" << r.buckets.ns_forward << ",\"ns_ppl\":" << r.ns_ppl
       << "}";
    if (!r.switch_events.empty()) {
      os << ",\"switch_events\":[";
      for (size_t i = 0; i < r.switch_events.size(); ++i) {
        const SwitchEvent& e = r.switch_events[i];
        os << (i ? "," : "") << "{\"layer_id\":\"" << e.layer_id << "\",\"from_bits\":\"" << to_string(e.from)
           << "\",\"to_bits\":\"" << to_string(e.to) << "\"}";
      }
      os << "]";
    }
    os << "}\n";
  }
}

void save_trace_file(const DecodeTrace& trace, const std::string& path) {
  std::ofstream os(path);
  if (!os) throw FormatError("cannot open trace file for writing: " + path);
  save_trace(trace, os);
}

DecodeTrace load_trace_file(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw FormatError("cannot open trace file: " + path);
  DecodeTrace trace;
  std::string line;
  size_t lineno = 0;
  while (std::getline(is, line)) {
    ++lineno;
    if (line.empty()) continue;
    try {
      JsonCursor c{line};
      TraceRecord r;
      c.expect('{');
      while (!c.peek('}')) {
        const std::string key = c.str();
        c.expect(':');
        if (key == "buckets") {
          c.expect('{');
          while (!c.peek('}')) {
            const std::string k = c.str();
            c.expect(':');
            const uint64_t v = std::stoull(c.raw());
            if (k == "ns_fp") r.buckets.ns_fp = v;
            else if (k == "ns_int8") r.buckets.ns_int8 = v;
            else if (k == "ns_int4") r.buckets.ns_int4 = v;
            else if (k == "ns_forward") r.buckets.ns_forward = v;
            else if (k == "ns_ppl") r.ns_ppl = v;
            if (c.peek(',')) c.expect(',');
          }
          c.expect('}');
        } else if (key == "switch_events") {
          c.expect('[');
          while (!c.peek(']')) {
            c.expect('{');
            SwitchEvent e;
            while (!c.peek('}')) {
              const std::string k = c.str();
              c.expect(':');
              const std::string v = c.str();
              if (k == "layer_id") e.layer_id = v;
              else if (k == "from_bits") e.from = parse_rung(v);
              else if (k == "to_bits") e.to = parse_rung(v);
              if (c.peek(',')) c.expect(',');
            }
            c.expect('}');
            r.switch_events.push_back(e);
            if (c.peek(',')) c.expect(',');
          }
          c.expect(']');
        } else {
          const std::string v = c.raw();
          if (key == "token_index") r.token_index = std::stoll(v);
          else if (key == "token_id") r.token_id = std::stoi(v);
          else if (key == "ppl_entropy") r.ppl_entropy = std::stod(v);
          else if (key == "fault_tolerance") r.fault_tolerance = std::stod(v);
          else if (key == "moving_average") { if (v != "null") r.moving_average = std::stod(v); }
          else if (key == "effective_bits") r.effective_bits = std::stod(v);
          else if (key == "weight_bytes_touched") r.weight_bytes_touched = std::stod(v);
          else if (key == "elapsed_ns") r.elapsed_ns = std::stoull(v);
        }
        if (c.peek(',')) c.expect(',');
      }
      c.expect('}');
      r.buckets.weight_bytes = r.weight_bytes_touched;
      trace.records.push_back(std::move(r));
    } catch (const FormatError& e) {
      throw FormatError("trace file line " + std::to_string(lineno) + ": " + e.what());
    } catch (const std::exception& e) {
      throw FormatError("trace file line " + std::to_string(lineno) + ": " + e.what());
    }
  }
  return trace;
}

std::string trace_to_csv(const DecodeTrace& trace) {
  std::ostringstream os;
  os << "token_index,token_id,ppl_entropy,fault_tolerance,moving_average,effective_bits,weight_bytes_touched,"
        "elapsed_ns,ns_fp,ns_int8,ns_int4,ns_forward,ns_ppl,switches\n";
  for (const TraceRecord& r : trace.records) {
    std::string sw;
    for (const SwitchEvent& e : r.switch_events)
      sw += (sw.empty() ? "" : ";") + e.layer_id + ":" + to_string(e.from) + "->" + to_string(e.to);
    os << r.token_index << ',' << r.token_id << ',' << num(r.ppl_entropy) << ',' << num(r.fault_tolerance) << ','
       << (r.moving_average ? num(*r.moving_average) : "") << ',' << num(r.effective_bits) << ','
       << num(r.weight_bytes_touched) << ',' << r.elapsed_ns << ',' << r.buckets.ns_fp << ',' << r.buckets.ns_int8 << ','
       << r.buckets.ns_int4 << ',' << r.buckets.ns_forward << ',' << r.ns_ppl << ',' << sw << "\n";
  }
  return os.str();
}

TokenId argmax_token(const Tensor& logits_row) {
  if (logits_row.numel() == 0) throw DimensionError("argmax: empty logits");
  // the device statistics kernel that feeds the scheduler (strict >, lowest index on ties)
  return detail::device_row_stats(logits_row, 1, logits_row.numel())[0].argmax;
}

}  // namespace flexquant
