// saber_io.hpp — host-side file formats of the engine's drop-in tools
// (SURVEY §8(f2)): the reference's output files, byte for byte, written from
// the engine's C-ABI results, and the JSON inputs its CLI reads.
//
//   records.csv    metrics.cpp:160-175 (records_to_csv)
//   decisions.csv  scheduler.cpp:148-157 (decisions_to_csv)
//   metrics.json   metrics.cpp:142-158 (to_json(MetricsReport))
//   results.csv    simloop.cpp:279-294 (results_to_csv)
//   summary.json   simloop.cpp:296-314 (summary_to_json)
//   samples.csv    calibration.cpp:170-175 (samples_to_csv)
//   models.json    calibration.cpp:193-212 (to_json(CalibrationReport))
//   model JSON     estimator.cpp:377-400 (to_json(SpeedModel), model_from_json)
//   config JSON    simloop.cpp:328-401 (sim_config_from_json)
// Doubles print as %.17g in CSV (text_io.cpp:9-13); JSON goes through
// nlohmann::json 3.11.3 (the reference's own JSON library, a third-party
// header), so number formatting, key order and NaN -> null are identical.
// Nothing here simulates or fits: every number comes from the engine.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "../../include/saber_cuda.h"

namespace saberb200::io {

extern const char* const kTaskNames[4];    // catalog order (SABER_TASK_*)
extern const char* const kFamilyNames[3];  // ModelFamily order
extern const char* const kKindNames[5];    // DecisionKind order

std::string fmt17(double v);

// --- run (RunOutput) --------------------------------------------------------
struct TaskStats {  // TaskMetrics (metrics.hpp:55-59)
  std::string name;
  int32_t issued = 0;
  int32_t met = 0;
  std::vector<std::pair<double, double>> cdf;
};

struct RunFiles {
  saber_traj_row row{};
  std::vector<saber_request> requests;
  std::vector<std::string> task_names;  // per request
  std::vector<saber_request_state> states;
  std::vector<saber_decision> decisions;
  std::vector<TaskStats> per_task;  // name order
};

std::string records_csv(const RunFiles& r);
std::string decisions_csv(const std::vector<saber_decision>& d);
std::string metrics_json(const RunFiles& r);

// --- sweep (SweepResult) ----------------------------------------------------
struct SweepFiles {
  std::vector<std::string> mixes;  // grid order
  std::vector<double> rps;
  std::vector<int32_t> caps;
  bool with_saber = false;
  int32_t repeats = 1;
  uint64_t seed = 0;
  std::vector<saber_row_stats> rows;        // grid order, repeats innermost
  std::vector<saber_mix_summary> summary;   // per mix
  std::vector<int32_t> best_cap;            // [mix][rps]
};

std::string results_csv(const SweepFiles& s);
std::string summary_json(const SweepFiles& s);

// --- calibrate ----------------------------------------------------------------
struct ModelSpec {
  saber_model m{};
  std::optional<double> fit_r2;
};

std::string samples_csv(const std::vector<int32_t>& loads, const std::vector<double>& speeds);
std::string model_json(const ModelSpec& m);
struct FamilyOutcome {
  int family = 0;
  bool ok = false;
  ModelSpec model;
  std::string error;
};
std::string calibration_json(const ModelSpec& best, const std::vector<FamilyOutcome>& fits);

// --- inputs (throw std::invalid_argument or nlohmann exceptions) ---------------
ModelSpec model_from_json(const std::string& text);
saber_mix mix_from_json(const std::string& text);  // {"task": fraction, ...}
saber_mix preset_mix(const std::string& id);       // w1 / w2 / w3 (types.cpp:27-47)

// SimConfig (simloop.hpp:23-31) with the reference's defaults.
struct SimSettings {
  saber_mix mix{};
  bool has_mix = false;
  double rps = 1.0;
  int32_t num_requests = 100;
  uint64_t workload_seed = 0;
  double length_jitter = 0.2;
  int32_t mode = SABER_MODE_SABER;
  int32_t window_size = 8;
  double tick = 0.01;
  int32_t static_batch_size = 0;
  std::optional<ModelSpec> model;
  ModelSpec ground_truth{saber_model{SABER_USL, {100.0, 0.05, 0.001}}, std::nullopt};
  double prefill_rate = 2000.0;
  std::optional<double> horizon;
  int32_t repeats = 3;
  uint64_t seed = 0;
};
SimSettings sim_settings_from_json(const std::string& text);

}  // namespace saberb200::io
