// saber_cuda_adapter.hpp — the reference-side binding (header only).
//
// A SaberSim user includes this next to the reference's own headers and links
// libsaber_b200.so; the functions below take and return the reference's types
// (proj/core/include/saber/*.hpp) and throw the reference's exception types,
// so switching a call site is a namespace change:
//
//     saber::sweep(grid, base, jobs)   ->  saber::cuda::sweep(grid, base, jobs)
//     saber::run(cfg)                  ->  saber::cuda::run(cfg)
//     saber::run_with_requests(cfg, r) ->  saber::cuda::run_with_requests(cfg, r)
//     saber::generate(spec)            ->  saber::cuda::generate(spec)
//     saber::fit / calibrate / profile ->  saber::cuda::fit / calibrate / profile
//
// Every value these functions return comes from the engine; the header only
// converts between the reference's types and the C ABI's structs (it calls no
// reference function).
// Only this header depends on the reference; the engine itself (the C ABI in
// saber_cuda.h) does not.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "saber/calibration.hpp"
#include "saber/estimator.hpp"
#include "saber/metrics.hpp"
#include "saber/scheduler.hpp"
#include "saber/simloop.hpp"
#include "saber/types.hpp"
#include "saber/workload.hpp"
#include "saber_cuda.h"

namespace saber::cuda {

namespace detail {

inline const char* kTask[4] = {"code_qna", "code_generation", "code_summary", "code_translation"};
inline const char* kFamily[3] = {"usl", "logistic", "linear"};  // ModelFamily names

// FitError::what() of the engine's reason code (saber_cuda.h SABER_FITERR_*).
inline std::string fit_error_message(int kind, int family) {
  switch (kind) {
    case SABER_FITERR_TOO_FEW:
      return std::string("too few samples or distinct loads to fit ") + kFamily[family];
    case SABER_FITERR_NO_CONVERGENCE:
      return std::string("optimizer did not converge for ") + kFamily[family];
    case SABER_FITERR_INCREASING_LINEAR: return "fitted linear model is increasing in load";
    default: return "fitted model is not non-increasing in load";
  }
}

inline int task_index(const std::string& name) {
  for (int t = 0; t < 4; ++t)
    if (name == kTask[t]) return t;
  return SABER_TASK_CUSTOM;
}

inline void check(saber_status s) {
  if (s == SABER_OK) return;
  const std::string msg = saber_cuda_last_error();
  switch (s) {
    case SABER_EINVAL: throw std::invalid_argument(msg);
    case SABER_EDOMAIN: throw std::domain_error(msg);
    case SABER_EINTERNAL: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline saber_model model_of(const SpeedModel& m) {
  saber_model x{};
  x.family = static_cast<int32_t>(m.family);
  for (int k = 0; k < 3; ++k) x.params[k] = m.params[static_cast<size_t>(k)];
  return x;
}

inline saber_mix mix_of(const WorkloadMix& m) {
  saber_mix x{};
  for (const auto& [name, frac] : m.proportions) {
    const int t = task_index(name);
    if (t < 0) throw std::invalid_argument("mix references unknown task: " + name);
    x.frac[t] = frac;
    x.present[t] = 1;
  }
  return x;
}

inline saber_traj_spec spec_of(const SimConfig& c) {
  saber_traj_spec s{};
  s.mix = mix_of(c.workload.mix);
  s.rps = c.workload.rps;
  s.num_requests = c.workload.num_requests;
  s.workload_seed = c.workload.seed;
  s.length_jitter = c.workload.length_jitter;
  s.mode = c.scheduler.mode == SchedulerMode::Saber ? SABER_MODE_SABER : SABER_MODE_STATIC;
  s.window_size = c.scheduler.window_size;
  s.tick = c.scheduler.tick;
  s.static_batch_size = c.scheduler.static_batch_size;
  s.has_model = c.model.has_value();
  if (c.model) s.model = model_of(*c.model);
  s.ground_truth = model_of(c.engine.ground_truth);
  s.prefill_rate = c.engine.prefill_rate;
  s.has_horizon = c.horizon.has_value();
  s.horizon = c.horizon.value_or(0.0);
  s.seed = c.seed;
  return s;
}

inline const std::string& task_name(int32_t t) {
  static const std::string custom = "custom";
  static const std::string names[4] = {kTask[0], kTask[1], kTask[2], kTask[3]};
  return t >= 0 && t < 4 ? names[t] : custom;
}

inline RequestState state_of(int32_t s) {
  switch (s) {
    case SABER_STATE_QUEUED_LOW: return RequestState::QueuedLow;
    case SABER_STATE_EXECUTING: return RequestState::Executing;
    case SABER_STATE_COMPLETED: return RequestState::Completed;
    default: return RequestState::QueuedHigh;
  }
}

inline std::optional<double> opt(double v) {
  if (std::isnan(v)) return std::nullopt;
  return v;
}

// One trajectory through saber_cuda_run_batch; every field of the RunOutput
// (requests, records, decisions, metrics) is read off the engine's outputs.
// The engine's event trace (Engine::trace) is not produced.
inline RunOutput run_one(const SimConfig& cfg, std::vector<Request> requests, bool replay,
                         int device) {
  saber_traj_spec spec = spec_of(cfg);
  std::vector<saber_request> rq;
  std::vector<std::string> group_name(kTask, kTask + 4);  // generated: name rank
  std::sort(group_name.begin(), group_name.end());
  if (replay) {
    if (requests.empty()) throw std::invalid_argument("run: no requests");
    // per-task metrics group by task name, in name order (std::map)
    std::map<std::string, int32_t> rank;
    for (const Request& r : requests) rank.emplace(r.task, 0);
    group_name.clear();
    for (auto& kv : rank) {
      kv.second = static_cast<int32_t>(group_name.size());
      group_name.push_back(kv.first);
    }
    rq.resize(requests.size());
    for (size_t i = 0; i < requests.size(); ++i) {
      if (requests[i].id != i) throw std::invalid_argument("run: request ids must be 0..n-1");
      rq[i].arrival_time = requests[i].arrival_time;
      rq[i].sla_seconds = requests[i].sla_seconds;
      rq[i].deadline = requests[i].deadline;
      rq[i].input_tokens = requests[i].input_tokens;
      rq[i].max_output_tokens = requests[i].max_output_tokens;
      rq[i].task = task_index(requests[i].task);
      rq[i].group = rank[requests[i].task];
    }
    spec.requests = rq.data();
    spec.num_requests = static_cast<int32_t>(rq.size());
  }
  const int n = spec.num_requests;
  if (n < 1) throw std::invalid_argument("num_requests must be >= 1");
  const int groups = std::max<int>(4, static_cast<int>(group_name.size()));
  saber_run_batch_desc d{&spec, 1, device};
  saber_traj_row row{};
  std::vector<saber_request> req(static_cast<size_t>(n));
  std::vector<saber_request_state> st(static_cast<size_t>(n));
  std::vector<double> cdf_l(static_cast<size_t>(n)), cdf_f(static_cast<size_t>(n));
  std::vector<int32_t> g_issued(static_cast<size_t>(groups)), g_met(static_cast<size_t>(groups));
  int64_t cap = 1 << 16, n_dec = 0;
  std::vector<saber_decision> decs;
  for (;;) {  // grow the decision buffer to the trajectory's count when it overflows
    decs.resize(static_cast<size_t>(cap));
    saber_run_batch_out o{};
    o.rows = &row;
    o.max_n = n;
    o.decisions = decs.data();
    o.decision_cap = cap;
    o.n_decisions = &n_dec;
    o.requests = req.data();
    o.states = st.data();
    o.cdf_latency = cdf_l.data();
    o.cdf_fraction = cdf_f.data();
    o.group_issued = g_issued.data();
    o.group_met = g_met.data();
    o.max_groups = groups;
    const saber_status s = saber_cuda_run_batch(&d, &o);
    if (s == SABER_ECAPACITY && row.decisions > cap) {
      cap = row.decisions;
      continue;
    }
    check(s);
    break;
  }
  RunOutput out;
  if (!replay) requests.resize(static_cast<size_t>(n));
  out.records.reserve(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    Request& r = requests[static_cast<size_t>(i)];
    const saber_request& q = req[static_cast<size_t>(i)];
    const saber_request_state& x = st[static_cast<size_t>(i)];
    if (!replay) {  // the generated workload (generate(), workload.cpp:52-79)
      r.id = static_cast<std::uint64_t>(i);
      r.task = task_name(q.task);
      r.arrival_time = q.arrival_time;
      r.input_tokens = q.input_tokens;
      r.max_output_tokens = q.max_output_tokens;
      r.sla_seconds = q.sla_seconds;
      r.deadline = q.deadline;
    }
    r.generated_tokens = x.generated_tokens;
    r.state = state_of(x.state);
    r.admit_time = opt(x.admit_time);
    r.completion_time = opt(x.completion_time);
    r.recorded_required_speed = opt(x.recorded_required_speed);
    r.demoted = x.demoted != 0;
    RunRecord rec;
    rec.request_id = r.id;
    rec.task = r.task;
    rec.arrival_time = r.arrival_time;
    rec.admit_time = r.admit_time;
    rec.completion_time = r.completion_time;
    rec.sla = r.sla_seconds;
    rec.met_sla = x.met_sla != 0;
    rec.final_tier = x.demoted ? "low" : "high";
    out.records.push_back(std::move(rec));
  }
  for (int64_t k = 0; k < n_dec; ++k) {
    const saber_decision& x = decs[static_cast<size_t>(k)];
    Decision dd;
    dd.time = x.time;
    dd.request_id = x.request_id;
    dd.kind = static_cast<DecisionKind>(x.kind);
    dd.load_before = x.load_before;
    if (x.has_pred) dd.pred_speed = x.pred_speed;
    if (x.has_req) dd.req_speed = x.req_speed;
    out.decisions.push_back(dd);
  }
  // MetricsReport: the row's scalars and, per task group, the engine's
  // issued / met counts and CDF points.
  out.metrics.goodput = row.goodput;
  out.metrics.ratio_mean = row.ratio_mean;
  out.metrics.ratio_std = row.ratio_std;
  out.metrics.cv = row.cv;
  int start = 0;
  for (int g = 0; g < static_cast<int>(group_name.size()); ++g) {
    const int issued = g_issued[static_cast<size_t>(g)];
    if (issued == 0) continue;
    TaskMetrics tm;
    tm.issued = issued;
    tm.goodput = static_cast<double>(g_met[static_cast<size_t>(g)]) / static_cast<double>(issued);
    for (int p = start; p < start + issued; ++p)
      if (!std::isnan(cdf_f[static_cast<size_t>(p)]))
        tm.cdf_points.emplace_back(cdf_l[static_cast<size_t>(p)], cdf_f[static_cast<size_t>(p)]);
    out.metrics.per_task[group_name[static_cast<size_t>(g)]] = std::move(tm);
    start += issued;
  }
  out.requests = std::move(requests);
  return out;
}

}  // namespace detail

// simloop.hpp:49
inline RunOutput run(const SimConfig& config, int device = 0) {
  return detail::run_one(config, {}, false, device);
}

// simloop.hpp:53-54
inline RunOutput run_with_requests(const SimConfig& config, std::vector<Request> requests,
                                   int device = 0) {
  return detail::run_one(config, std::move(requests), true, device);
}

// workload.hpp:31
inline std::vector<Request> generate(const WorkloadSpec& spec, int device = 0) {
  saber_workload_spec w{};
  w.mix = detail::mix_of(spec.mix);
  w.rps = spec.rps;
  w.num_requests = spec.num_requests;
  w.seed = spec.seed;
  w.length_jitter = spec.length_jitter;
  if (w.num_requests < 1) throw std::invalid_argument("num_requests must be >= 1");
  std::vector<saber_request> q(static_cast<size_t>(w.num_requests));
  detail::check(saber_cuda_generate(&w, 1, device, q.data(), w.num_requests));
  std::vector<Request> out(q.size());
  for (size_t i = 0; i < q.size(); ++i) {
    Request& r = out[i];
    r.id = i;
    r.task = detail::task_name(q[i].task);
    r.arrival_time = q[i].arrival_time;
    r.input_tokens = q[i].input_tokens;
    r.max_output_tokens = q[i].max_output_tokens;
    r.sla_seconds = q[i].sla_seconds;
    r.deadline = q[i].deadline;
  }
  return out;
}

// simloop.hpp:96-99.  `jobs` is accepted for signature parity; the device
// decides its own parallelism and the output never depends on it.
inline SweepResult sweep(const SweepGrid& grid, const SimConfig& base, int jobs = 0,
                         int device = 0) {
  (void)jobs;
  std::vector<int32_t> mixes;
  for (const auto& m : grid.mixes) {
    if (m != "w1" && m != "w2" && m != "w3")
      throw std::invalid_argument("unknown mix preset: " + m);
    mixes.push_back(m[1] - '0');
  }
  std::vector<double> rps(grid.rps_list.begin(), grid.rps_list.end());
  std::vector<int32_t> caps(grid.caps.begin(), grid.caps.end());
  saber_sweep_desc d{};
  d.mixes = mixes.data();
  d.n_mixes = static_cast<int32_t>(mixes.size());
  d.rps = rps.data();
  d.n_rps = static_cast<int32_t>(rps.size());
  d.caps = caps.data();
  d.n_caps = static_cast<int32_t>(caps.size());
  d.with_saber = grid.with_saber;
  d.num_requests = base.workload.num_requests;
  d.length_jitter = base.workload.length_jitter;
  d.window_size = base.scheduler.window_size;
  d.tick = base.scheduler.tick;
  d.has_model = base.model.has_value();
  if (base.model) d.model = detail::model_of(*base.model);
  d.ground_truth = detail::model_of(base.engine.ground_truth);
  d.prefill_rate = base.engine.prefill_rate;
  d.has_horizon = base.horizon.has_value();
  d.horizon = base.horizon.value_or(0.0);
  d.repeats = base.repeats;
  d.seed = base.seed;
  d.device = device;
  d.shard_index = 0;
  d.shard_count = 1;
  const int64_t n_rows = saber_cuda_sweep_rows(&d);
  std::vector<saber_row_stats> rows(static_cast<size_t>(n_rows > 0 ? n_rows : 0));
  std::vector<saber_mix_summary> summ(mixes.size());
  std::vector<int32_t> best(mixes.size() * rps.size());
  saber_sweep_out o{};
  o.row_stats = rows.data();
  o.summary = summ.data();
  o.best_cap_by_rps = best.data();
  detail::check(saber_cuda_sweep(&d, &o));
  SweepResult res;
  size_t k = 0;
  for (const auto& m : grid.mixes)
    for (const double r : grid.rps_list) {
      auto push = [&](SchedulerMode mode, int cap, int i) {
        SweepRow row;
        row.mix = m;
        row.rps = r;
        row.scheduler = mode;
        row.static_cap = cap;
        row.repeat_seed = base.seed + static_cast<std::uint64_t>(i);
        row.goodput = rows[k].goodput;
        row.ratio_mean = rows[k].ratio_mean;
        row.ratio_std = rows[k].ratio_std;
        row.cv = rows[k].cv;
        res.rows.push_back(row);
        ++k;
      };
      for (const int cap : grid.caps)
        for (int i = 0; i < base.repeats; ++i) push(SchedulerMode::Static, cap, i);
      if (grid.with_saber)
        for (int i = 0; i < base.repeats; ++i) push(SchedulerMode::Saber, 0, i);
    }
  for (size_t mi = 0; mi < grid.mixes.size(); ++mi) {
    MixSummary s;
    s.saber_mean_goodput = summ[mi].saber_mean_goodput;
    s.best_static_mean_goodput = summ[mi].best_static_mean_goodput;
    s.delta = summ[mi].delta;
    s.saber_pooled_cv = summ[mi].saber_pooled_cv;
    s.best_static_pooled_cv = summ[mi].best_static_pooled_cv;
    s.saber_rps_mean_cv = summ[mi].saber_rps_mean_cv;
    s.best_static_rps_mean_cv = summ[mi].best_static_rps_mean_cv;
    if (!grid.caps.empty())
      for (size_t ri = 0; ri < grid.rps_list.size(); ++ri)
        s.best_cap_by_rps[grid.rps_list[ri]] = best[mi * grid.rps_list.size() + ri];
    res.summary[grid.mixes[mi]] = s;
  }
  return res;
}

// estimator.hpp:61.  Throws FitError with the reference's payload.
inline SpeedModel fit(const std::vector<LoadSpeedSample>& samples, ModelFamily family,
                      int device = 0) {
  std::vector<int32_t> loads(samples.size());
  std::vector<double> speeds(samples.size());
  for (size_t i = 0; i < samples.size(); ++i) {
    loads[i] = samples[i].load;
    speeds[i] = samples[i].speed;
  }
  const int64_t offsets[2] = {0, static_cast<int64_t>(samples.size())};
  const int f = static_cast<int>(family);
  saber_fit_desc d{loads.data(), speeds.data(), offsets, 1, 1 << f, 0, device};
  double params[9] = {}, r2[3] = {};
  int32_t status[3] = {};
  saber_fit_out o{};
  o.params = params;
  o.r2 = r2;
  o.status = status;
  detail::check(saber_cuda_fit_batch(&d, &o));
  const std::array<double, 3> p = {params[3 * f], params[3 * f + 1], params[3 * f + 2]};
  if (status[f] != 0) throw FitError(detail::fit_error_message(status[f], f), family, p, r2[f]);
  SpeedModel m;
  m.family = family;
  m.params = p;
  m.fit_r2 = r2[f];
  return m;
}

// calibration.hpp:54
inline CalibrationReport calibrate(const std::vector<LoadSpeedSample>& samples, int device = 0) {
  std::vector<int32_t> loads(samples.size());
  std::vector<double> speeds(samples.size());
  for (size_t i = 0; i < samples.size(); ++i) {
    loads[i] = samples[i].load;
    speeds[i] = samples[i].speed;
  }
  const int64_t offsets[2] = {0, static_cast<int64_t>(samples.size())};
  saber_fit_desc d{loads.data(), speeds.data(), offsets, 1, 7, 1, device};
  double params[9] = {}, r2[3] = {};
  int32_t status[3] = {}, best = -1;
  saber_fit_out o{};
  o.params = params;
  o.r2 = r2;
  o.status = status;
  o.best_family = &best;
  detail::check(saber_cuda_fit_batch(&d, &o));
  if (best <= -2)
    throw CalibrationError("calibrate: insufficient distinct loads (" + std::to_string(-2 - best) +
                           " < 3)");
  if (best == -1) throw CalibrationError("calibrate: no model family produced a fit");
  CalibrationReport rep;
  for (int f = 0; f < 3; ++f) {
    FamilyFit e;
    e.family = static_cast<ModelFamily>(f);
    e.ok = status[f] == 0;
    if (e.ok) {
      e.model.family = e.family;
      e.model.params = {params[3 * f], params[3 * f + 1], params[3 * f + 2]};
      e.model.fit_r2 = r2[f];
    } else {
      e.error = detail::fit_error_message(status[f], f);
    }
    rep.fits.push_back(e);
  }
  rep.best = rep.fits[static_cast<size_t>(best)].model;
  return rep;
}

// calibration.hpp:29-31
inline std::vector<LoadSpeedSample> profile(const EngineConfig& engine_config,
                                            const WorkloadSpec& profiling_spec, int l_max = 50,
                                            int device = 0) {
  saber_profile_spec s{};
  s.ground_truth = detail::model_of(engine_config.ground_truth);
  s.prefill_rate = engine_config.prefill_rate;
  s.mix = detail::mix_of(profiling_spec.mix);
  s.num_requests = profiling_spec.num_requests;
  s.seed = profiling_spec.seed;
  s.length_jitter = profiling_spec.length_jitter;
  s.l_max = l_max;
  const int64_t n = saber_cuda_profile_samples(&s);
  if (n < 0) throw CalibrationError(saber_cuda_last_error());
  std::vector<int32_t> loads(static_cast<size_t>(n));
  std::vector<double> speeds(static_cast<size_t>(n));
  int64_t offs[2] = {0, 0};
  int32_t status = 0;
  saber_profile_desc d{&s, 1, device};
  saber_profile_out o{offs, loads.data(), speeds.data(), n, &status, 0.0};
  detail::check(saber_cuda_profile_batch(&d, &o));
  if (status != 0) throw CalibrationError("profile: insufficient distinct loads (< 3)");
  std::vector<LoadSpeedSample> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[static_cast<size_t>(i)] = {loads[static_cast<size_t>(i)], speeds[static_cast<size_t>(i)]};
  return out;
}

}  // namespace saber::cuda
