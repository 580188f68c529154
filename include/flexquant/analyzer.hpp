// Offline layer-sensitivity analysis and the switch plan (reference:
// include/flexquant/analyzer.hpp, src/analyzer.cpp).  Weight-histogram KL runs on the device
// (counts) with the reference's smoothing / normalisation / KL finished in its sequential
// order; the logit-mode calibration (BASELINE config 4) is new.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <span>
#include <string>
#include <vector>

#include "flexquant/model.hpp"

namespace flexquant {

struct LayerKlReport {
  std::string layer_id;
  Rung bits = Rung::Int8;
  double kl = 0.0;
  int64_t param_count = 0;
};

struct SwitchEntry {
  std::string layer_id;
  Rung from = Rung::Fp;
  Rung to = Rung::Int8;
  double kl = 0.0;
  bool operator==(const SwitchEntry&) const = default;
};

struct SwitchPlan {
  std::vector<SwitchEntry> entries;
  size_t size() const { return entries.size(); }
  bool operator==(const SwitchPlan&) const = default;
};

inline constexpr int kDefaultHistogramBins = 2048;
inline constexpr double kHistogramSmoothing = 1e-10;

std::vector<double> uniform_edges(double lo, double hi, int bins);
std::vector<double> weight_histogram(const Tensor& w, std::span<const double> edges);
double kl_divergence(std::span<const double> p, std::span<const double> q);

// Per-layer weight-histogram KL of `target_bits` against the fp weights (needs fp resident).
std::vector<LayerKlReport> analyze_model(const Model& model, Rung target_bits, int bins);
SwitchPlan build_switch_plan(std::span<const LayerKlReport> reports, Rung from_bits, Rung to_bits);
SwitchPlan build_ladder_plan(const Model& model, std::span<const Rung> rungs, int bins);

// Logit-mode calibration: for every block, KL(softmax(l_flip) || softmax(l_base)) averaged over
// teacher-forced tokens; every linear of a block gets the block's KL (block-granular ranking,
// ties ordered by layer_id as build_switch_plan does).
struct CalibrationResult {
  std::vector<double> block_kl;
  std::vector<double> block_entropy;
  std::vector<LayerKlReport> reports;
};
CalibrationResult calibrate_logit_kl(Model& model, std::span<const TokenId> tokens, int64_t n_seqs, int64_t len,
                                     Rung base, Rung flip);

void save_plan(const SwitchPlan& plan, std::ostream& os);
void save_plan_file(const SwitchPlan& plan, const std::string& path);
SwitchPlan load_plan(std::istream& is);
SwitchPlan load_plan_file(const std::string& path);

}  // namespace flexquant
