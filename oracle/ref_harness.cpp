// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" harness around the UNMODIFIED reference library.  oracle/Makefile
// compiles this file together with /root/reference/proj/core/src/*.cpp (where
// they lie; nothing is copied) into oracle/_ref/libsaber_ref.so.  It exposes
// the reference's public API (saber::run, run_with_requests, sweep, fit,
// calibrate, profile, predict, generate — proj/core/include/saber/*.hpp) under
// the plain-C signatures of oracle/oracle.h (prefix ref_), so tests and the
// bench's reference arm can drive the real reference on the same inputs as
// the CUDA engine.
#include <atomic>
#include <mutex>
#include <thread>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "oracle.h"
#include "saber/calibration.hpp"
#include "saber/estimator.hpp"
#include "saber/metrics.hpp"
#include "saber/scheduler.hpp"
#include "saber/simloop.hpp"
#include "saber/types.hpp"
#include "saber/workload.hpp"

namespace {

std::string g_err;

const char* kTaskName[4] = {"code_qna", "code_generation", "code_summary",
                            "code_translation"};

int task_index(const std::string& name) {
  for (int t = 0; t < 4; ++t)
    if (name == kTaskName[t]) return t;
  return -1;
}

saber::SpeedModel to_model(const orc_model& m) {
  saber::SpeedModel s;
  s.family = static_cast<saber::ModelFamily>(m.family);
  s.params = {m.p[0], m.p[1], m.p[2]};
  return s;
}

saber::WorkloadMix to_mix(const orc_mix& m) {
  saber::WorkloadMix w;
  for (int t = 0; t < 4; ++t)
    if (m.present[t]) w.proportions[kTaskName[t]] = m.frac[t];
  return w;
}

saber::SimConfig to_config(const orc_sim_config& c) {
  saber::SimConfig s;
  s.workload.mix = to_mix(c.mix);
  s.workload.rps = c.rps;
  s.workload.num_requests = c.num_requests;
  s.workload.seed = c.workload_seed;
  s.workload.length_jitter = c.jitter;
  s.scheduler.mode =
      c.mode == ORC_SABER ? saber::SchedulerMode::Saber : saber::SchedulerMode::Static;
  s.scheduler.window_size = c.window;
  s.scheduler.tick = c.tick;
  s.scheduler.static_batch_size = c.cap;
  if (c.has_model) s.model = to_model(c.model);
  s.engine.ground_truth = to_model(c.ground_truth);
  s.engine.prefill_rate = c.prefill_rate;
  if (c.has_horizon) s.horizon = c.horizon;
  s.seed = c.seed;
  return s;
}

uint64_t dbits(double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  return b;
}

int kind_of(saber::DecisionKind k) { return static_cast<int>(k); }

void fill_out(const saber::RunOutput& o, orc_traj_out* out, orc_record* recs,
              orc_decision* decs, int64_t dec_cap, int64_t* n_dec) {
  std::memset(out, 0, sizeof *out);
  out->goodput = o.metrics.goodput;
  out->ratio_mean = o.metrics.ratio_mean;
  out->ratio_std = o.metrics.ratio_std;
  out->cv = o.metrics.cv;
  uint64_t h = ORC_HASH_SEED;
  for (std::size_t i = 0; i < o.decisions.size(); ++i) {
    const saber::Decision& d = o.decisions[i];
    const uint64_t pb = d.pred_speed ? dbits(*d.pred_speed) : ORC_ABSENT_BITS;
    const uint64_t rb = d.req_speed ? dbits(*d.req_speed) : ORC_ABSENT_BITS;
    const uint64_t w = static_cast<uint64_t>(static_cast<uint32_t>(d.request_id)) |
                       (static_cast<uint64_t>(kind_of(d.kind)) << 32) |
                       (static_cast<uint64_t>(static_cast<uint32_t>(d.load_before)) << 40);
    h += orc_decision_term(static_cast<uint64_t>(i), dbits(d.time), w, pb, rb);
    out->n_kind[kind_of(d.kind)] += 1;
    if (decs && static_cast<int64_t>(i) < dec_cap) {
      orc_decision& x = decs[i];
      x.time = d.time;
      x.request_id = d.request_id;
      x.kind = kind_of(d.kind);
      x.load_before = d.load_before;
      x.has_pred = d.pred_speed.has_value();
      x.has_req = d.req_speed.has_value();
      x.pred_speed = d.pred_speed ? *d.pred_speed : NAN;
      x.req_speed = d.req_speed ? *d.req_speed : NAN;
    }
  }
  out->decisions = static_cast<int64_t>(o.decisions.size());
  out->decision_hash = h;
  if (n_dec) *n_dec = out->decisions;
  int64_t completed = 0, met = 0;
  for (std::size_t i = 0; i < o.records.size(); ++i) {
    const saber::RunRecord& r = o.records[i];
    completed += r.completion_time.has_value();
    met += r.met_sla;
    const int t = task_index(r.task);
    if (t >= 0) {
      out->issued_by_task[t] += 1;
      out->met_by_task[t] += r.met_sla;
    }
    if (recs) {
      orc_record& x = recs[i];
      const saber::Request& q = o.requests[i];
      x.arrival_time = r.arrival_time;
      x.admit_time = r.admit_time ? *r.admit_time : NAN;
      x.completion_time = r.completion_time ? *r.completion_time : NAN;
      x.sla = r.sla;
      x.task = t;
      x.input_tokens = q.input_tokens;
      x.max_output_tokens = q.max_output_tokens;
      x.demoted = q.demoted;
    }
  }
  out->completed = completed;
  out->met = met;
  out->ticks = out->passes = out->decode_updates = out->prefill_updates = -1;
  out->refresh_entries = out->gate_candidates = out->ledger_scanned = -1;
  out->rng_draws = -1;
  out->last_arrival = o.requests.empty() ? 0.0 : o.requests.back().arrival_time;
  out->horizon = NAN;
}

orc_mix to_orc_mix(const saber::WorkloadMix& m) {
  orc_mix x{};
  for (const auto& [name, frac] : m.proportions) {
    const int t = task_index(name);
    x.frac[t] = frac;
    x.present[t] = 1;
  }
  return x;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

std::vector<saber::LoadSpeedSample> to_samples(const int32_t* loads,
                                               const double* speeds, int32_t m) {
  std::vector<saber::LoadSpeedSample> s(static_cast<std::size_t>(m));
  for (int32_t i = 0; i < m; ++i) s[static_cast<std::size_t>(i)] = {loads[i], speeds[i]};
  return s;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_generate(const orc_sim_config* cfg, orc_request* out) {
  return guarded([&] {
    const auto reqs = saber::generate(to_config(*cfg).workload);
    for (std::size_t i = 0; i < reqs.size(); ++i) {
      out[i].arrival_time = reqs[i].arrival_time;
      out[i].sla_seconds = reqs[i].sla_seconds;
      out[i].deadline = reqs[i].deadline;
      out[i].input_tokens = reqs[i].input_tokens;
      out[i].max_output_tokens = reqs[i].max_output_tokens;
      out[i].task = task_index(reqs[i].task);
    }
  });
}

int ref_run(const orc_sim_config* cfg, orc_traj_out* out, orc_record* records,
            orc_decision* decisions, int64_t dec_cap, int64_t* n_dec) {
  return guarded([&] {
    const saber::RunOutput o = saber::run(to_config(*cfg));
    fill_out(o, out, records, decisions, dec_cap, n_dec);
  });
}

// The engine's per-row latency quantiles (p50/p90/p99 over every issued
// request) read off the reference's own cdf (metrics.cpp:61-85): the records
// of saber::run(cfg), relabelled to one task so that cdf() pools them; q[i] =
// the smallest latency whose cumulative fraction reaches p[i] (NaN if none).
int ref_latency_quantiles(const orc_sim_config* cfg, const double* p, int32_t np, double* q) {
  return guarded([&] {
    saber::RunOutput o = saber::run(to_config(*cfg));
    for (auto& r : o.records) r.task = "all";
    const auto pts = saber::cdf(o.records, "all");
    for (int32_t i = 0; i < np; ++i) {
      q[i] = std::nan("");
      for (const auto& [lat, frac] : pts)
        if (frac >= p[i]) {
          q[i] = lat;
          break;
        }
    }
  });
}

int ref_run_with_requests(const orc_sim_config* cfg, const orc_request* rq,
                          int32_t n, orc_traj_out* out, orc_record* records,
                          orc_decision* decisions, int64_t dec_cap,
                          int64_t* n_dec) {
  return guarded([&] {
    std::vector<saber::Request> reqs(static_cast<std::size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
      saber::Request& r = reqs[static_cast<std::size_t>(i)];
      r.id = static_cast<uint64_t>(i);
      r.task = rq[i].task >= 0 && rq[i].task < 4 ? kTaskName[rq[i].task] : "custom";
      r.arrival_time = rq[i].arrival_time;
      r.input_tokens = rq[i].input_tokens;
      r.max_output_tokens = rq[i].max_output_tokens;
      r.sla_seconds = rq[i].sla_seconds;
      r.deadline = rq[i].deadline;
    }
    const saber::RunOutput o =
        saber::run_with_requests(to_config(*cfg), std::move(reqs));
    fill_out(o, out, records, decisions, dec_cap, n_dec);
  });
}

int ref_predict(const orc_model* m, int32_t load, double* out) {
  return guarded([&] { *out = saber::predict(to_model(*m), load); });
}

int ref_fit(const int32_t* loads, const double* speeds, int32_t m,
            int32_t family, double* params, double* r2_or_sse,
            int32_t* fit_error) {
  return guarded([&] {
    try {
      const saber::SpeedModel sm = saber::fit(
          to_samples(loads, speeds, m), static_cast<saber::ModelFamily>(family));
      for (int k = 0; k < 3; ++k) params[k] = sm.params[static_cast<std::size_t>(k)];
      *r2_or_sse = *sm.fit_r2;
      *fit_error = 0;
    } catch (const saber::FitError& e) {
      for (int k = 0; k < 3; ++k) params[k] = e.best_params[static_cast<std::size_t>(k)];
      *r2_or_sse = e.best_sse;
      *fit_error = 1;
    }
  });
}

int ref_calibrate(const int32_t* loads, const double* speeds, int32_t m,
                  int32_t* best_family, double* best_params, double* best_r2,
                  int32_t* ok, double* fam_params, double* fam_r2) {
  return guarded([&] {
    const saber::CalibrationReport rep =
        saber::calibrate(to_samples(loads, speeds, m));
    *best_family = static_cast<int32_t>(rep.best.family);
    for (int k = 0; k < 3; ++k) best_params[k] = rep.best.params[static_cast<std::size_t>(k)];
    *best_r2 = *rep.best.fit_r2;
    for (std::size_t f = 0; f < rep.fits.size(); ++f) {
      ok[f] = rep.fits[f].ok;
      for (int k = 0; k < 3; ++k)
        fam_params[3 * f + static_cast<std::size_t>(k)] =
            rep.fits[f].ok ? rep.fits[f].model.params[static_cast<std::size_t>(k)] : 0.0;
      fam_r2[f] = rep.fits[f].ok ? *rep.fits[f].model.fit_r2 : NAN;
    }
  });
}

int ref_profile(const orc_model* gt, double prefill_rate, const orc_mix* mix,
                int32_t num_requests, uint64_t seed, double jitter,
                int32_t l_max, int32_t* loads, double* speeds, int64_t cap,
                int64_t* n_out) {
  return guarded([&] {
    saber::EngineConfig ec;
    ec.ground_truth = to_model(*gt);
    ec.prefill_rate = prefill_rate;
    saber::WorkloadSpec spec;
    spec.mix = to_mix(*mix);
    spec.num_requests = num_requests;
    spec.seed = seed;
    spec.length_jitter = jitter;
    const auto s = saber::profile(ec, spec, l_max);
    *n_out = static_cast<int64_t>(s.size());
    for (std::size_t i = 0; i < s.size() && static_cast<int64_t>(i) < cap; ++i) {
      loads[i] = s[i].load;
      speeds[i] = s[i].speed;
    }
  });
}

int ref_sweep(const orc_sim_config* base, const int32_t* mix_ids,
              int32_t n_mixes, const double* rps, int32_t n_rps,
              const int32_t* caps, int32_t n_caps, int32_t with_saber,
              int32_t repeats, int32_t jobs, double* row_goodput,
              double* row_ratio_mean, double* row_ratio_std, double* row_cv,
              double* summary, int32_t* best_cap) {
  return guarded([&] {
    saber::SimConfig b = to_config(*base);
    b.repeats = repeats;
    saber::SweepGrid grid;
    for (int32_t i = 0; i < n_mixes; ++i)
      grid.mixes.push_back("w" + std::to_string(mix_ids[i]));
    grid.rps_list.assign(rps, rps + n_rps);
    grid.caps.assign(caps, caps + n_caps);
    grid.with_saber = with_saber != 0;
    const saber::SweepResult r = saber::sweep(grid, b, jobs);
    for (std::size_t i = 0; i < r.rows.size(); ++i) {
      if (row_goodput) row_goodput[i] = r.rows[i].goodput;
      if (row_ratio_mean) row_ratio_mean[i] = r.rows[i].ratio_mean;
      if (row_ratio_std) row_ratio_std[i] = r.rows[i].ratio_std;
      if (row_cv) row_cv[i] = r.rows[i].cv;
    }
    for (int32_t i = 0; i < n_mixes; ++i) {
      const saber::MixSummary& s = r.summary.at(grid.mixes[static_cast<std::size_t>(i)]);
      if (summary) {
        double* o = summary + 7 * i;
        o[0] = s.saber_mean_goodput;
        o[1] = s.best_static_mean_goodput;
        o[2] = s.delta;
        o[3] = s.saber_pooled_cv;
        o[4] = s.best_static_pooled_cv;
        o[5] = s.saber_rps_mean_cv;
        o[6] = s.best_static_rps_mean_cv;
      }
      if (best_cap)
        for (int32_t k = 0; k < n_rps; ++k) {
          const auto it = s.best_cap_by_rps.find(rps[k]);
          best_cap[i * n_rps + k] = it == s.best_cap_by_rps.end() ? 0 : it->second;
        }
    }
  });
}

// The decision logs of a sweep's cells, in the sweep's row order (the cell
// configs simloop.cpp:137-163 builds), each cell through saber::run on a
// pool of `jobs` threads: per row the decision count and the digest of
// oracle.h.  saber::sweep itself returns no decision data.
int ref_sweep_decisions(const orc_sim_config* base, const int32_t* mix_ids, int32_t n_mixes,
                        const double* rps, int32_t n_rps, const int32_t* caps, int32_t n_caps,
                        int32_t with_saber, int32_t repeats, int32_t jobs, int64_t* decisions,
                        uint64_t* hashes) {
  return guarded([&] {
    std::vector<orc_sim_config> cells;
    for (int32_t m = 0; m < n_mixes; ++m)
      for (int32_t r = 0; r < n_rps; ++r) {
        orc_sim_config c = *base;
        c.mix = to_orc_mix(saber::preset_mix("w" + std::to_string(mix_ids[m])));
        c.rps = rps[r];
        for (int32_t k = 0; k <= n_caps; ++k) {
          if (k == n_caps && !with_saber) break;
          for (int32_t i = 0; i < repeats; ++i) {
            orc_sim_config x = c;
            x.workload_seed = x.seed = base->seed + static_cast<uint64_t>(i);
            x.mode = k < n_caps ? ORC_STATIC : ORC_SABER;
            x.cap = k < n_caps ? caps[k] : 0;
            x.has_model = k < n_caps ? 0 : base->has_model;
            cells.push_back(x);
          }
        }
      }
    std::atomic<std::size_t> next{0};
    std::string err;
    std::mutex mu;
    auto worker = [&] {
      for (std::size_t i = next++; i < cells.size(); i = next++) {
        try {
          orc_traj_out o{};
          fill_out(saber::run(to_config(cells[i])), &o, nullptr, nullptr, 0, nullptr);
          decisions[i] = o.decisions;
          hashes[i] = o.decision_hash;
        } catch (const std::exception& e) {
          std::lock_guard<std::mutex> lk(mu);
          err = e.what();
        }
      }
    };
    const int n = jobs > 0 ? jobs : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int t = 0; t < n; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    if (!err.empty()) throw std::runtime_error(err);
  });
}

// trace_from_csv / trace_to_csv (workload.cpp:87-138) for the trace parity
// tests; requests in orc_request form.
int ref_trace_from_csv(const char* text, orc_request* out, int32_t cap, int32_t* n) {
  return guarded([&] {
    const auto reqs = saber::trace_from_csv(text);
    *n = static_cast<int32_t>(reqs.size());
    for (std::size_t i = 0; i < reqs.size() && static_cast<int32_t>(i) < cap; ++i) {
      out[i].arrival_time = reqs[i].arrival_time;
      out[i].sla_seconds = reqs[i].sla_seconds;
      out[i].deadline = reqs[i].deadline;
      out[i].input_tokens = reqs[i].input_tokens;
      out[i].max_output_tokens = reqs[i].max_output_tokens;
      out[i].task = task_index(reqs[i].task);
    }
  });
}

int ref_trace_to_csv(const orc_request* rq, int32_t n, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::vector<saber::Request> reqs(static_cast<std::size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
      saber::Request& r = reqs[static_cast<std::size_t>(i)];
      r.id = static_cast<uint64_t>(i);
      r.task = kTaskName[rq[i].task];
      r.arrival_time = rq[i].arrival_time;
      r.input_tokens = rq[i].input_tokens;
      r.max_output_tokens = rq[i].max_output_tokens;
    }
    const std::string s = saber::trace_to_csv(reqs);
    *len = s.size();
    if (cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

}  // extern "C"
