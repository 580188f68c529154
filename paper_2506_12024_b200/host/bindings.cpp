// pybind11 module `_flexquant`: the C++ host API (include/flexquant/*.hpp) for tests and bench.
// Tensors cross as numpy float32 arrays; errors surface as the flexquant exception classes.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <sstream>

#include "flexquant/analyzer.hpp"
#include "flexquant/engine.hpp"
#include "flexquant/fixture.hpp"
#include "flexquant/metrics.hpp"
#include "flexquant/model.hpp"
#include "flexquant/quantizer.hpp"
#include "flexquant/scheduler.hpp"

namespace py = pybind11;
using namespace flexquant;

namespace {

Tensor to_tensor(const py::array_t<float, py::array::c_style | py::array::forcecast>& a) {
  std::vector<int64_t> shape(a.shape(), a.shape() + a.ndim());
  std::vector<float> data(a.data(), a.data() + a.size());
  return Tensor::from_data(std::move(shape), std::move(data));
}

py::array_t<float> to_numpy(const Tensor& t) {
  py::array_t<float> out(std::vector<py::ssize_t>(t.shape().begin(), t.shape().end()));
  std::copy(t.data(), t.data() + t.numel(), out.mutable_data());
  return out;
}

std::vector<TokenId> to_tokens(const py::array_t<int32_t, py::array::c_style | py::array::forcecast>& a) {
  return std::vector<TokenId>(a.data(), a.data() + a.size());
}

py::dict stats_dict(const fq_row_stats& s) {
  py::dict d;
  d["ppl_entropy"] = s.ppl_entropy;
  d["entropy"] = s.entropy;
  d["p1"] = s.p1;
  d["p2"] = s.p2;
  d["fault_tolerance"] = s.fault_tolerance;
  d["argmax"] = s.argmax;
  return d;
}

}  // namespace

PYBIND11_MODULE(_flexquant, m) {
  m.doc() = "B200 FlexQuant engine: C++ host API over the CUDA C-ABI";

  auto base = py::register_exception<Error>(m, "Error", PyExc_RuntimeError);
  py::register_exception<DimensionError>(m, "DimensionError", base.ptr());
  py::register_exception<ConfigError>(m, "ConfigError", base.ptr());
  py::register_exception<InputError>(m, "InputError", base.ptr());
  py::register_exception<StateError>(m, "StateError", base.ptr());
  py::register_exception<FormatError>(m, "FormatError", base.ptr());
  py::register_exception<CapacityError>(m, "CapacityError", base.ptr());
  py::register_exception<DeviceError>(m, "DeviceError", base.ptr());

  py::enum_<Rung>(m, "Rung").value("Fp", Rung::Fp).value("Int8", Rung::Int8).value("Int4", Rung::Int4);
  py::enum_<QuantMode>(m, "QuantMode").value("Asymmetric", QuantMode::Asymmetric).value("Symmetric", QuantMode::Symmetric);
  py::enum_<ThresholdMode>(m, "ThresholdMode").value("Prefill", ThresholdMode::Prefill).value("Absolute", ThresholdMode::Absolute);
  py::enum_<Arch>(m, "Arch").value("Reference", Arch::Reference).value("Llama", Arch::Llama);
  m.def("accounting_bits", &accounting_bits);
  m.def("parse_rung", [](const std::string& s) { return parse_rung(s); });
  m.def("is_downward", &is_downward);

  // ---------------------------------------------------------------- quantizer
  py::class_<QuantizedTensor>(m, "QuantizedTensor")
      .def(py::init<>())
      .def_readwrite("bits", &QuantizedTensor::bits)
      .def_readwrite("mode", &QuantizedTensor::mode)
      .def_readwrite("rows", &QuantizedTensor::rows)
      .def_readwrite("cols", &QuantizedTensor::cols)
      .def_readwrite("group_size", &QuantizedTensor::group_size)
      .def_property("payload", [](const QuantizedTensor& q) { return py::array_t<uint8_t>(q.payload.size(), q.payload.data()); },
                    [](QuantizedTensor& q, py::array_t<uint8_t> a) { q.payload.assign(a.data(), a.data() + a.size()); })
      .def_property("scale", [](const QuantizedTensor& q) { return py::array_t<float>(q.scale.size(), q.scale.data()); },
                    [](QuantizedTensor& q, py::array_t<float> a) { q.scale.assign(a.data(), a.data() + a.size()); })
      .def_property("zero_point", [](const QuantizedTensor& q) { return py::array_t<int32_t>(q.zero_point.size(), q.zero_point.data()); },
                    [](QuantizedTensor& q, py::array_t<int32_t> a) { q.zero_point.assign(a.data(), a.data() + a.size()); })
      .def("code_at", &QuantizedTensor::code_at)
      .def("validate", &QuantizedTensor::validate)
      .def("stored_offset", &QuantizedTensor::stored_offset)
      .def("expected_payload_bytes", &QuantizedTensor::expected_payload_bytes);
  m.def("quantize", [](py::array_t<float> x, int bits, QuantMode mode, int64_t group) { return quantize(to_tensor(x), bits, mode, group); },
        py::arg("x"), py::arg("bits"), py::arg("mode") = QuantMode::Asymmetric, py::arg("group_size") = 0);
  m.def("quantize_device", [](py::array_t<float> x, int bits, QuantMode mode, int64_t group) { return quantize_device(to_tensor(x), bits, mode, group); },
        py::arg("x"), py::arg("bits"), py::arg("mode") = QuantMode::Asymmetric, py::arg("group_size") = 0);
  m.def("dequantize", [](const QuantizedTensor& q) { return to_numpy(dequantize(q)); });
  m.def("pack_codes", [](std::vector<uint32_t> c, int bits) { return pack_codes(c, bits); });
  m.def("unpack_codes", [](std::vector<uint8_t> p, int64_t n, int bits) { return unpack_codes(p, n, bits); });
  m.def("round_half_even", &round_half_even);
  m.def("linear", [](py::array_t<float> x, py::array_t<float> w, py::array_t<float> b) {
    return to_numpy(linear(to_tensor(x), to_tensor(w), b.size() ? to_tensor(b) : Tensor{}));
  });

  // ---------------------------------------------------------------- scheduler
  m.def("ppl_entropy", [](py::array_t<float> l) { return ppl_entropy(to_tensor(l)); });
  m.def("fault_tolerance", [](py::array_t<float> l) { return fault_tolerance(to_tensor(l)); });
  m.def("argmax_token", [](py::array_t<float> l) { return argmax_token(to_tensor(l)); });
  m.def("derive_threshold", [](py::array_t<float> l, int w, double theta) { return derive_threshold(to_tensor(l), w, theta); });
  py::class_<SchedulerConfig>(m, "SchedulerConfig")
      .def(py::init<>())
      .def_readwrite("window_len", &SchedulerConfig::window_len)
      .def_readwrite("theta", &SchedulerConfig::theta)
      .def_readwrite("threshold_mode", &SchedulerConfig::threshold_mode)
      .def_readwrite("layers_per_switch", &SchedulerConfig::layers_per_switch);
  py::class_<SchedulerState>(m, "SchedulerState")
      .def(py::init<SchedulerConfig, size_t>())
      .def("set_threshold", &SchedulerState::set_threshold)
      .def("threshold", &SchedulerState::threshold)
      .def("moving_average", &SchedulerState::moving_average)
      .def("plan_cursor", &SchedulerState::plan_cursor)
      .def("cooldown_remaining", &SchedulerState::cooldown_remaining)
      .def("observe", [](SchedulerState& s, double v) {
        const auto d = s.observe(v);
        return py::make_tuple(d.window_mean, d.first_entry, d.count);
      });

  // ---------------------------------------------------------------- model
  py::class_<ModelConfig>(m, "ModelConfig")
      .def(py::init<>())
      .def_readwrite("vocab_size", &ModelConfig::vocab_size)
      .def_readwrite("d_model", &ModelConfig::d_model)
      .def_readwrite("n_heads", &ModelConfig::n_heads)
      .def_readwrite("head_dim", &ModelConfig::head_dim)
      .def_readwrite("n_layers", &ModelConfig::n_layers)
      .def_readwrite("ffn_dim", &ModelConfig::ffn_dim)
      .def_readwrite("max_seq_len", &ModelConfig::max_seq_len)
      .def_readwrite("tie_embeddings", &ModelConfig::tie_embeddings)
      .def_readwrite("arch", &ModelConfig::arch)
      .def_readwrite("group_size", &ModelConfig::group_size)
      .def_readwrite("max_batch", &ModelConfig::max_batch)
      .def_readwrite("norm_eps", &ModelConfig::norm_eps)
      .def_readwrite("rope_theta", &ModelConfig::rope_theta)
      .def_readwrite("fp16_activations", &ModelConfig::fp16_activations);
  py::class_<SwitchEvent>(m, "SwitchEvent")
      .def_readonly("layer_id", &SwitchEvent::layer_id)
      .def_readonly("from_", &SwitchEvent::from)
      .def_readonly("to", &SwitchEvent::to);
  py::class_<Model>(m, "Model")
      .def(py::init<ModelConfig>())
      .def("config", &Model::config, py::return_value_policy::reference_internal)
      .def("init_random", &Model::init_random, py::arg("seed"), py::arg("std") = 0.02f)
      .def("set_param", [](Model& md, const std::string& n, py::array_t<float> a) { md.set_param(n, to_tensor(a)); })
      .def("linear_ids", &Model::linear_ids)
      .def("num_linears", &Model::num_linears)
      .def("linear_index", &Model::linear_index)
      .def("set_quantized", [](Model& md, int i, Rung r, const QuantizedTensor& q) { md.linear(i).set_quantized(r, q); })
      .def("quantized", [](Model& md, int i, Rung r) { return md.linear(i).quantized(r); })
      .def("set_precision", &Model::set_precision, py::arg("layer_id"), py::arg("bits"), py::arg("slot") = 0)
      .def("set_all_precision", &Model::set_all_precision, py::arg("bits"), py::arg("slot") = 0)
      .def("precision", &Model::precision, py::arg("index"), py::arg("slot") = 0)
      .def("effective_bits", &Model::effective_bits, py::arg("slot") = 0)
      .def("weight_bytes_per_pass", &Model::weight_bytes_per_pass, py::arg("slot") = 0)
      .def("forward_prefill", [](Model& md, py::array_t<int32_t> t, int slot) {
        KvCache c = md.make_cache(slot);
        return to_numpy(md.forward_prefill(to_tokens(t), c));
      }, py::arg("tokens"), py::arg("slot") = 0)
      .def("forward_decode", [](Model& md, int32_t tok, int slot) {
        KvCache c = md.attach_cache(slot);
        return to_numpy(md.forward_decode(tok, c));
      }, py::arg("token"), py::arg("slot") = 0)
      .def("prefill_rows", [](Model& md, int slot, py::array_t<int32_t> t) {
        py::list out;
        for (const fq_row_stats& s : md.prefill_rows(slot, to_tokens(t))) out.append(stats_dict(s));
        return out;
      })
      .def("reset_slot", [](Model& md, int slot) { md.make_cache(slot); })
      .def("decode_rows", [](Model& md, std::vector<int32_t> slots, std::vector<int32_t> toks) {
        py::list out;
        for (const fq_row_stats& s : md.decode_rows(slots, toks)) out.append(stats_dict(s));
        return out;
      })
      .def("step_stats", [](const Model& md) {
        const StepStats& s = md.step_stats();
        return py::make_tuple(s.weight_bytes, s.ns_fp, s.ns_int8, s.ns_int4, s.ns_forward);
      });
  m.def("init_random_with_kl", [](Model& md, uint64_t seed, float std, int bins) {
    const WeightKl k = init_random_with_kl(md, seed, std, bins);
    return py::make_tuple(k.kl8, k.kl4);
  });
  m.def("profile_gemvs", [](Model& md, int slot, int reps) {
    const GemvProfile p = profile_gemvs(md, slot, reps);
    return py::make_tuple(p.ms_per_launch, p.launches_per_pass, p.bytes_per_pass);
  });
  m.def("step_bytes", [](const Model& md, std::vector<int32_t> slots) { return step_bytes(md, slots); });
  m.def("runtime_stream", []() { return reinterpret_cast<uintptr_t>(runtime_stream()); });
  m.def("load_model_file", [](const std::string& p, int max_batch) { return load_model_file(p, max_batch); },
        py::arg("path"), py::arg("max_batch") = 1);
  m.def("save_model_file", &save_model_file);

  // ---------------------------------------------------------------- analyzer
  py::class_<LayerKlReport>(m, "LayerKlReport")
      .def(py::init<>())
      .def_readwrite("layer_id", &LayerKlReport::layer_id)
      .def_readwrite("bits", &LayerKlReport::bits)
      .def_readwrite("kl", &LayerKlReport::kl)
      .def_readwrite("param_count", &LayerKlReport::param_count);
  py::class_<SwitchEntry>(m, "SwitchEntry")
      .def(py::init<>())
      .def_readwrite("layer_id", &SwitchEntry::layer_id)
      .def_readwrite("from_", &SwitchEntry::from)
      .def_readwrite("to", &SwitchEntry::to)
      .def_readwrite("kl", &SwitchEntry::kl);
  py::class_<SwitchPlan>(m, "SwitchPlan")
      .def(py::init<>())
      .def_readwrite("entries", &SwitchPlan::entries)
      .def("size", &SwitchPlan::size)
      .def("to_text", [](const SwitchPlan& p) {
        std::ostringstream os;
        save_plan(p, os);
        return os.str();
      })
      .def_static("from_text", [](const std::string& s) {
        std::istringstream is(s);
        return load_plan(is);
      });
  m.def("uniform_edges", &uniform_edges);
  m.def("weight_histogram", [](py::array_t<float> w, std::vector<double> e) { return weight_histogram(to_tensor(w), e); });
  m.def("kl_divergence", [](std::vector<double> p, std::vector<double> q) { return kl_divergence(p, q); });
  m.def("analyze_model", &analyze_model);
  m.def("build_switch_plan", [](std::vector<LayerKlReport> r, Rung f, Rung t) { return build_switch_plan(r, f, t); });
  m.def("build_ladder_plan", [](const Model& md, std::vector<Rung> r, int bins) { return build_ladder_plan(md, r, bins); });
  m.def("calibrate_logit_kl", [](Model& md, py::array_t<int32_t> toks, int64_t n, int64_t len, Rung base, Rung flip) {
    const CalibrationResult r = calibrate_logit_kl(md, to_tokens(toks), n, len, base, flip);
    return py::make_tuple(r.block_kl, r.block_entropy, r.reports);
  });
  m.def("save_plan_file", &save_plan_file);
  m.def("load_plan_file", &load_plan_file);

  // ---------------------------------------------------------------- engine
  py::class_<GenerationConfig>(m, "GenerationConfig")
      .def(py::init<>())
      .def_readwrite("max_new_tokens", &GenerationConfig::max_new_tokens)
      .def_readwrite("eos_token", &GenerationConfig::eos_token)
      .def_readwrite("scheduler", &GenerationConfig::scheduler)
      .def_readwrite("start_rung", &GenerationConfig::start_rung)
      .def_readwrite("trace_path", &GenerationConfig::trace_path)
      .def_readwrite("device_timed_buckets", &GenerationConfig::device_timed_buckets);
  py::class_<StepStats>(m, "StepStats")
      .def_readonly("weight_bytes", &StepStats::weight_bytes)
      .def_readonly("ns_fp", &StepStats::ns_fp)
      .def_readonly("ns_int8", &StepStats::ns_int8)
      .def_readonly("ns_int4", &StepStats::ns_int4)
      .def_readonly("ns_forward", &StepStats::ns_forward);
  py::class_<TraceRecord>(m, "TraceRecord")
      .def_readonly("token_index", &TraceRecord::token_index)
      .def_readonly("token_id", &TraceRecord::token_id)
      .def_readonly("ppl_entropy", &TraceRecord::ppl_entropy)
      .def_readonly("fault_tolerance", &TraceRecord::fault_tolerance)
      .def_readonly("moving_average", &TraceRecord::moving_average)
      .def_readonly("effective_bits", &TraceRecord::effective_bits)
      .def_readonly("weight_bytes_touched", &TraceRecord::weight_bytes_touched)
      .def_readonly("elapsed_ns", &TraceRecord::elapsed_ns)
      .def_readonly("switch_events", &TraceRecord::switch_events)
      .def_readonly("buckets", &TraceRecord::buckets);
  py::class_<DecodeTrace>(m, "DecodeTrace")
      .def_readonly("records", &DecodeTrace::records)
      .def("to_jsonl", [](const DecodeTrace& t) {
        std::ostringstream os;
        save_trace(t, os);
        return os.str();
      });
  py::class_<GenerationResult>(m, "GenerationResult")
      .def_readonly("sequence", &GenerationResult::sequence)
      .def_readonly("trace", &GenerationResult::trace)
      .def_readonly("threshold", &GenerationResult::threshold);
  m.def("generate", [](py::array_t<int32_t> p, Model& md, const SwitchPlan& plan, const GenerationConfig& c) {
    const std::vector<TokenId> t = to_tokens(p);
    py::gil_scoped_release nogil;
    return generate(t, md, plan, c);
  });
  m.def("generate_static", [](py::array_t<int32_t> p, Model& md, Rung r, const GenerationConfig& c) {
    const std::vector<TokenId> t = to_tokens(p);
    py::gil_scoped_release nogil;
    return generate_static(t, md, r, c);
  });
  m.def("generate_batch", [](std::vector<std::vector<int32_t>> ps, Model& md, const SwitchPlan& plan, const GenerationConfig& c) {
    py::gil_scoped_release nogil;
    return generate_batch(ps, md, plan, c);
  });
  m.def("traffic_report", [](const DecodeTrace& t) { return format_traffic_report(traffic_report(t)); });
  py::class_<TrafficReport>(m, "TrafficReport")
      .def_readonly("total_weight_bytes", &TrafficReport::total_weight_bytes)
      .def_readonly("mean_bytes_per_token", &TrafficReport::mean_bytes_per_token)
      .def_readonly("bucket_sum_over_total", &TrafficReport::bucket_sum_over_total)
      .def_readonly("ppl_share", &TrafficReport::ppl_share);
  m.def("traffic_report_struct", [](const DecodeTrace& t) { return traffic_report(t); });
  py::class_<SweepRow>(m, "SweepRow")
      .def_readonly("speed", &SweepRow::speed)
      .def_readonly("final_effective_bits", &SweepRow::final_effective_bits)
      .def_readonly("mean_bytes_per_token", &SweepRow::mean_bytes_per_token)
      .def_readonly("agreement_vs_fp", &SweepRow::agreement_vs_fp)
      .def_readonly("first_divergence", &SweepRow::first_divergence)
      .def_readonly("rouge_l_vs_fp", &SweepRow::rouge_l_vs_fp);
  m.def("sweep_switch_speed", [](py::array_t<int32_t> p, Model& md, const SwitchPlan& plan, std::vector<int64_t> speeds,
                                 const GenerationConfig& c) {
    const std::vector<TokenId> t = to_tokens(p);
    py::gil_scoped_release nogil;
    return sweep_switch_speed(t, md, plan, speeds, c);
  });
  m.def("sweep_csv_header", &sweep_csv_header);
  m.def("sweep_csv_row", &sweep_csv_row);
  // fixtures and metrics (include/flexquant/fixture.hpp, metrics.hpp)
  m.def("tiny_config", &tiny_config);
  m.def("micro_config", &micro_config);
  m.def("make_fixture_model", [](const ModelConfig& c, uint64_t seed) { return make_fixture_model(c, seed); });
  m.def("agreement_rate", [](std::vector<int32_t> a, std::vector<int32_t> b) {
    const Agreement g = agreement_rate(a, b);
    return py::make_tuple(g.rate, g.divergence_index ? py::cast(*g.divergence_index) : py::none());
  });
  m.def("rouge_l", [](std::vector<int32_t> a, std::vector<int32_t> b) { return rouge_l(a, b); });
  m.def("load_trace_file", &load_trace_file);
  m.def("save_trace_file", &save_trace_file);
  m.def("trace_to_csv", &trace_to_csv);
}
