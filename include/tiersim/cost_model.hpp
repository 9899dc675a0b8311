// tiersim/cost_model.hpp — the reference cost-estimator interface (core/include/tiersim/cost_model.hpp)
// over libtsb: scalar forms are host arithmetic in libtsb (bit-identical to cost_model.cpp:14-85);
// whole queues go through the GPU scorer (tiersim/scheduler.hpp, BatchScorer).
#pragma once

#include <cctype>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <span>
#include <sstream>
#include <string>
#include <vector>

#include "tiersim/types.hpp"

namespace tiersim {

struct LinearCostModel {
  double slope = 0.0;
  double intercept = 0.0;
};

struct LinearFit {
  LinearCostModel model;
  bool slope_clamped = false;
  bool intercept_clamped = false;
};

struct TokenSample {
  std::int64_t tokens = 0;
  double seconds = 0.0;
};

inline LinearFit fit_linear(std::span<const TokenSample> samples) {
  std::vector<int64_t> t(samples.size());
  std::vector<double> s(samples.size());
  for (std::size_t i = 0; i < samples.size(); ++i) {
    t[i] = samples[i].tokens;
    s[i] = samples[i].seconds;
  }
  LinearFit fit;
  int sc = 0, ic = 0;
  check(tsb_fit_linear(static_cast<int64_t>(samples.size()), t.data(), s.data(), &fit.model.slope,
                       &fit.model.intercept, &sc, &ic));
  fit.slope_clamped = sc != 0;
  fit.intercept_clamped = ic != 0;
  return fit;
}

inline double predict(const LinearCostModel& model, std::int64_t tokens) {
  return tsb_predict(model.slope, model.intercept, tokens);
}

struct ServiceCost {
  double t_load = 0.0;
  double t_comp = 0.0;
  double total() const noexcept { return t_load + t_comp; }
};

struct CostModelPair {
  LinearCostModel load;
  LinearCostModel comp;
  void c_abi(double out[4]) const {
    out[0] = load.slope;
    out[1] = load.intercept;
    out[2] = comp.slope;
    out[3] = comp.intercept;
  }
};

inline ServiceCost estimate_service_cost(const RequestSpec& spec, const LinearCostModel& load_model,
                                         const LinearCostModel& comp_model,
                                         const ClusterConfig& config) {
  detail::SpecView v(spec);
  const tsb_cluster c = config.c_abi();
  double m[4];
  CostModelPair{load_model, comp_model}.c_abi(m);
  ServiceCost cost;
  check(tsb_estimate_service_cost(&v.q, 0, m, &c, &cost.t_load, &cost.t_comp));
  return cost;
}

inline CostModelPair cost_models_from_config(const ClusterConfig& config) {
  const tsb_cluster c = config.c_abi();
  double m[4];
  tsb_cost_models_from_config(&c, m);
  return CostModelPair{{m[0], m[1]}, {m[2], m[3]}};
}

/// Two-column CSV (tokens, seconds), optional header, '#' comments (cost_model.cpp:105-123 contract).
/// Used to calibrate the loading model from measured ingest samples.
inline std::vector<TokenSample> read_samples_csv(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw Error("read_samples_csv: cannot open " + path.string());
  std::vector<TokenSample> out;
  std::string line;
  bool first = true;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    for (char& ch : line)
      if (ch == ',' || ch == ';' || ch == '\t') ch = ' ';
    std::istringstream row(line);
    double tokens = 0.0, seconds = 0.0;
    if (row >> tokens >> seconds) {
      out.push_back({static_cast<std::int64_t>(tokens), seconds});
    } else if (!first) {
      throw Error("read_samples_csv: malformed line in " + path.string() + ": " + line);
    }
    first = false;
  }
  return out;
}

}  // namespace tiersim
