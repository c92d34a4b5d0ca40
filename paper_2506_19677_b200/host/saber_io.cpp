// saber_io.cpp — see saber_io.hpp.  Each writer cites the reference writer
// whose bytes it reproduces.
#include "saber_io.hpp"

#include <cmath>
#include <cstdio>
#include <map>
#include <stdexcept>

#include "json.hpp"  // nlohmann::json 3.11.3 (third-party; the reference's JSON library)

namespace saberb200::io {

using nlohmann::json;

const char* const kTaskNames[4] = {"code_qna", "code_generation", "code_summary", "code_translation"};
const char* const kFamilyNames[3] = {"usl", "logistic", "linear"};
const char* const kKindNames[5] = {"admit_high", "admit_low", "reject_own", "reject_active", "demote"};

std::string fmt17(double v) {  // text_io.cpp:9-13
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

namespace {

// csv_row (text_io.cpp:15-24): comma-joined, newline-terminated, unquoted.
struct CsvLine {
  std::string* out;
  bool first = true;
  explicit CsvLine(std::string* o) : out(o) {}
  CsvLine(const CsvLine&) = delete;
  CsvLine& operator=(const CsvLine&) = delete;
  CsvLine& operator<<(const std::string& f) {
    if (!first) *out += ',';
    *out += f;
    first = false;
    return *this;
  }
  ~CsvLine() { *out += '\n'; }
};

std::string opt17(double v) { return std::isnan(v) ? std::string() : fmt17(v); }

std::string dump(const json& j) { return j.dump(2) + "\n"; }

json model_value(const ModelSpec& m) {
  json j;
  j["family"] = kFamilyNames[m.m.family];
  const int n = m.m.family == SABER_LINEAR ? 2 : 3;
  j["params"] = std::vector<double>(m.m.params, m.m.params + n);
  if (m.fit_r2) j["fit_r2"] = *m.fit_r2;
  return j;
}

int family_of(const std::string& name) {  // family_from_string (estimator.cpp:409-415)
  for (int f = 0; f < 3; ++f)
    if (name == kFamilyNames[f]) return f;
  throw std::invalid_argument("unknown model family: " + name);
}

}  // namespace

// ---------------------------------------------------------------------- run --
std::string records_csv(const RunFiles& r) {  // metrics.cpp:160-175
  std::string out =
      "request_id,task,arrival_time,admit_time,completion_time,sla,met_sla,final_tier\n";
  for (size_t i = 0; i < r.states.size(); ++i) {
    const saber_request& q = r.requests[i];
    const saber_request_state& s = r.states[i];
    CsvLine(&out) << std::to_string(i) << r.task_names[i] << fmt17(q.arrival_time)
                  << opt17(s.admit_time) << opt17(s.completion_time) << fmt17(q.sla_seconds)
                  << (s.met_sla ? "1" : "0") << (s.demoted ? "low" : "high");
  }
  return out;
}

std::string decisions_csv(const std::vector<saber_decision>& d) {  // scheduler.cpp:148-157
  std::string out = "time,request_id,decision,load_before,pred_speed,req_speed\n";
  for (const saber_decision& x : d)
    CsvLine(&out) << fmt17(x.time) << std::to_string(x.request_id) << kKindNames[x.kind]
                  << std::to_string(x.load_before) << (x.has_pred ? fmt17(x.pred_speed) : "")
                  << (x.has_req ? fmt17(x.req_speed) : "");
  return out;
}

std::string metrics_json(const RunFiles& r) {  // metrics.cpp:142-158
  json j;
  j["goodput"] = r.row.goodput;
  j["ratio_mean"] = r.row.ratio_mean;
  j["ratio_std"] = r.row.ratio_std;
  j["cv"] = r.row.cv;
  json per_task = json::object();
  for (const TaskStats& t : r.per_task) {
    json e;
    e["issued"] = t.issued;
    e["goodput"] = static_cast<double>(t.met) / static_cast<double>(t.issued);
    json pts = json::array();
    for (const auto& [lat, frac] : t.cdf) pts.push_back({lat, frac});
    e["cdf_points"] = pts;
    per_task[t.name] = e;
  }
  j["per_task"] = per_task;
  return dump(j);
}

// -------------------------------------------------------------------- sweep --
std::string results_csv(const SweepFiles& s) {  // simloop.cpp:279-294
  std::string out = "mix,rps,scheduler,static_cap,repeat_seed,goodput,ratio_mean,ratio_std,cv\n";
  size_t k = 0;
  auto row = [&](const std::string& mix, double rps, int cap, int rep) {
    const saber_row_stats& x = s.rows[k++];
    CsvLine(&out) << mix << fmt17(rps) << (cap > 0 ? "static" : "saber")
                  << (cap > 0 ? std::to_string(cap) : std::string())
                  << std::to_string(s.seed + static_cast<uint64_t>(rep)) << fmt17(x.goodput)
                  << opt17(x.ratio_mean) << opt17(x.ratio_std) << opt17(x.cv);
  };
  for (const std::string& mix : s.mixes)
    for (const double rps : s.rps) {
      for (const int32_t cap : s.caps)
        for (int i = 0; i < s.repeats; ++i) row(mix, rps, cap, i);
      if (s.with_saber)
        for (int i = 0; i < s.repeats; ++i) row(mix, rps, 0, i);
    }
  return out;
}

std::string summary_json(const SweepFiles& s) {  // simloop.cpp:296-314
  json j = json::object();
  for (size_t mi = 0; mi < s.mixes.size(); ++mi) {
    const saber_mix_summary& x = s.summary[mi];
    json m;
    m["saber_mean_goodput"] = x.saber_mean_goodput;
    m["best_static_mean_goodput"] = x.best_static_mean_goodput;
    m["delta"] = x.delta;
    m["saber_pooled_cv"] = x.saber_pooled_cv;
    m["best_static_pooled_cv"] = x.best_static_pooled_cv;
    m["saber_rps_mean_cv"] = x.saber_rps_mean_cv;
    m["best_static_rps_mean_cv"] = x.best_static_rps_mean_cv;
    json caps = json::object();
    if (!s.caps.empty())
      for (size_t ri = 0; ri < s.rps.size(); ++ri)
        caps[fmt17(s.rps[ri])] = s.best_cap[mi * s.rps.size() + ri];
    m["best_cap_by_rps"] = caps;
    j[s.mixes[mi]] = m;
  }
  return dump(j);
}

// ---------------------------------------------------------------- calibrate --
std::string samples_csv(const std::vector<int32_t>& loads,
                        const std::vector<double>& speeds) {  // calibration.cpp:170-175
  std::string out = "load,speed\n";
  for (size_t i = 0; i < loads.size(); ++i)
    CsvLine(&out) << std::to_string(loads[i]) << fmt17(speeds[i]);
  return out;
}

std::string model_json(const ModelSpec& m) { return dump(model_value(m)); }  // estimator.cpp:377-385

std::string calibration_json(const ModelSpec& best,
                             const std::vector<FamilyOutcome>& fits) {  // calibration.cpp:193-212
  json j;
  j["best"] = json::parse(model_json(best));
  json arr = json::array();
  for (const FamilyOutcome& f : fits) {
    json e;
    e["family"] = kFamilyNames[f.family];
    e["ok"] = f.ok;
    if (f.ok) {
      e["model"] = json::parse(model_json(f.model));
      e["r2"] = *f.model.fit_r2;
    } else {
      e["error"] = f.error;
    }
    arr.push_back(e);
  }
  j["fits"] = arr;
  return dump(j);
}

// ------------------------------------------------------------------- inputs --
ModelSpec model_from_json(const std::string& text) {  // estimator.cpp:387-400
  const json j = json::parse(text);
  ModelSpec m;
  m.m.family = family_of(j.at("family").get<std::string>());
  const auto p = j.at("params").get<std::vector<double>>();
  const size_t n = m.m.family == SABER_LINEAR ? 2 : 3;
  if (p.size() != n)
    throw std::invalid_argument("model params: expected " + std::to_string(n) + " values");
  for (size_t k = 0; k < n; ++k) m.m.params[k] = p[k];
  if (j.contains("fit_r2")) m.fit_r2 = j["fit_r2"].get<double>();
  return m;
}

saber_mix mix_from_json(const std::string& text) {
  const auto props = json::parse(text).get<std::map<std::string, double>>();
  saber_mix m{};
  for (const auto& [name, frac] : props) {
    int t = -1;
    for (int k = 0; k < 4; ++k)
      if (name == kTaskNames[k]) t = k;
    if (t < 0) throw std::invalid_argument("mix references unknown task: " + name);
    m.frac[t] = frac;
    m.present[t] = 1;
  }
  return m;
}

saber_mix preset_mix(const std::string& id) {  // types.cpp:27-47
  saber_mix m{};
  for (int t = 0; t < 4; ++t) m.present[t] = 1;
  if (id == "w1") {
    m.frac[SABER_TASK_TRANSLATION] = 0.4;
    m.frac[SABER_TASK_GENERATION] = 0.4;
    m.frac[SABER_TASK_QNA] = 0.1;
    m.frac[SABER_TASK_SUMMARY] = 0.1;
  } else if (id == "w2") {
    m.frac[SABER_TASK_QNA] = 0.4;
    m.frac[SABER_TASK_SUMMARY] = 0.4;
    m.frac[SABER_TASK_GENERATION] = 0.1;
    m.frac[SABER_TASK_TRANSLATION] = 0.1;
  } else if (id == "w3") {
    for (int t = 0; t < 4; ++t) m.frac[t] = 0.25;
  } else {
    throw std::invalid_argument("unknown mix preset: " + id);
  }
  return m;
}

SimSettings sim_settings_from_json(const std::string& text) {  // simloop.cpp:328-372
  const json j = json::parse(text);
  SimSettings c;
  if (j.contains("workload")) {
    const json& w = j["workload"];
    if (w.contains("mix")) {
      c.mix = w["mix"].is_string() ? preset_mix(w["mix"].get<std::string>())
                                   : mix_from_json(w["mix"].dump());
      c.has_mix = true;
    }
    if (w.contains("rps")) c.rps = w["rps"].get<double>();
    if (w.contains("num_requests")) c.num_requests = w["num_requests"].get<int>();
    if (w.contains("seed")) c.workload_seed = w["seed"].get<uint64_t>();
    if (w.contains("length_jitter")) c.length_jitter = w["length_jitter"].get<double>();
  }
  if (j.contains("scheduler")) {
    const json& s = j["scheduler"];
    if (s.contains("mode")) {
      const std::string mode = s["mode"].get<std::string>();
      if (mode == "saber") c.mode = SABER_MODE_SABER;
      else if (mode == "static") c.mode = SABER_MODE_STATIC;
      else throw std::invalid_argument("config: unknown scheduler mode " + mode);
    }
    if (s.contains("window_size")) c.window_size = s["window_size"].get<int>();
    if (s.contains("tick")) c.tick = s["tick"].get<double>();
    if (s.contains("static_batch_size")) c.static_batch_size = s["static_batch_size"].get<int>();
  }
  if (j.contains("model") && !j["model"].is_null()) c.model = model_from_json(j["model"].dump());
  if (j.contains("engine")) {
    const json& e = j["engine"];
    if (e.contains("ground_truth")) c.ground_truth = model_from_json(e["ground_truth"].dump());
    if (e.contains("prefill_rate")) c.prefill_rate = e["prefill_rate"].get<double>();
  }
  if (j.contains("horizon") && !j["horizon"].is_null()) c.horizon = j["horizon"].get<double>();
  if (j.contains("repeats")) c.repeats = j["repeats"].get<int>();
  if (j.contains("seed")) c.seed = j["seed"].get<uint64_t>();
  return c;
}

}  // namespace saberb200::io
