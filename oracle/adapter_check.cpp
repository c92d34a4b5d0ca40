// adapter_check.cpp — TEST INFRASTRUCTURE ONLY.
//
// Drives the reference's own API and the drop-in adapter
// (include/saber_cuda_adapter.hpp -> libsaber_b200.so) on the same inputs and
// compares the results field by field:
//   saber::sweep(grid, base)      vs saber::cuda::sweep(grid, base)
//   saber::run(cfg)               vs saber::cuda::run(cfg)
//   saber::run_with_requests(...) vs saber::cuda::run_with_requests(...)
// Built by oracle/Makefile into oracle/_ref/adapter_check (it links the
// compiled reference); tests/test_adapter.py runs it.
#include <cmath>
#include <optional>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#include "saber_cuda_adapter.hpp"

namespace {

int failures = 0;

bool same(double a, double b) { return (std::isnan(a) && std::isnan(b)) || a == b; }

void expect(bool ok, const std::string& what) {
  if (!ok) {
    ++failures;
    std::printf("MISMATCH %s\n", what.c_str());
  }
}

saber::SpeedModel calibrated_usl() {
  return {saber::ModelFamily::Usl,
          {99.999999999997357, 0.049999999999992085, 0.0010000000000001078}, {}};
}

bool same_opt(const std::optional<double>& a, const std::optional<double>& b) {
  return a.has_value() == b.has_value() && (!a || same(*a, *b));
}

void compare_requests(const std::vector<saber::Request>& a, const std::vector<saber::Request>& b,
                      const std::string& tag) {
  expect(a.size() == b.size(), tag + " request count");
  for (size_t i = 0; i < a.size() && i < b.size(); ++i) {
    const auto& x = a[i];
    const auto& y = b[i];
    const bool ok = x.id == y.id && x.task == y.task && same(x.arrival_time, y.arrival_time) &&
                    x.input_tokens == y.input_tokens && x.max_output_tokens == y.max_output_tokens &&
                    same(x.sla_seconds, y.sla_seconds) && same(x.deadline, y.deadline) &&
                    same(x.generated_tokens, y.generated_tokens) && x.state == y.state &&
                    same_opt(x.admit_time, y.admit_time) &&
                    same_opt(x.completion_time, y.completion_time) &&
                    same_opt(x.recorded_required_speed, y.recorded_required_speed) &&
                    x.demoted == y.demoted;
    if (!ok) {
      expect(false, tag + " request " + std::to_string(i));
      break;
    }
  }
}

void compare_runs(const saber::RunOutput& a, const saber::RunOutput& b, const std::string& tag) {
  compare_requests(a.requests, b.requests, tag);
  expect(a.decisions.size() == b.decisions.size(), tag + " decision count");
  for (size_t i = 0; i < a.decisions.size() && i < b.decisions.size(); ++i) {
    const auto& x = a.decisions[i];
    const auto& y = b.decisions[i];
    const bool ok = x.time == y.time && x.request_id == y.request_id && x.kind == y.kind &&
                    x.load_before == y.load_before && x.pred_speed == y.pred_speed &&
                    x.req_speed == y.req_speed;
    if (!ok) {
      expect(false, tag + " decision " + std::to_string(i));
      break;
    }
  }
  expect(saber::decisions_to_csv(a.decisions) == saber::decisions_to_csv(b.decisions),
         tag + " decisions.csv");
  expect(saber::records_to_csv(a.records) == saber::records_to_csv(b.records), tag + " records.csv");
  expect(saber::to_json(a.metrics) == saber::to_json(b.metrics), tag + " metrics.json");
}

}  // namespace

int main() {
  try {
    // BASELINE config 1 through run().
    saber::SimConfig cfg;
    cfg.workload.mix = saber::preset_mix("w1");
    cfg.workload.rps = 4.0;
    cfg.workload.num_requests = 100;
    cfg.workload.seed = 42;
    cfg.seed = 42;
    cfg.model = calibrated_usl();
    compare_runs(saber::run(cfg), saber::cuda::run(cfg), "config1");

    // A static trajectory and a replayed workload.
    saber::SimConfig st = cfg;
    st.scheduler.mode = saber::SchedulerMode::Static;
    st.scheduler.static_batch_size = 30;
    st.model.reset();
    st.workload.mix = saber::preset_mix("w3");
    st.workload.rps = 8.0;
    compare_runs(saber::run(st), saber::cuda::run(st), "static");
    auto reqs = saber::generate(cfg.workload);
    compare_requests(reqs, saber::cuda::generate(cfg.workload), "generate");
    compare_runs(saber::run_with_requests(cfg, reqs), saber::cuda::run_with_requests(cfg, reqs),
                 "replay");
    // Horizon cut mid-run: executing requests keep their fluid progress,
    // queued ones stay queued (some demoted) — every Request field compared.
    saber::SimConfig cut = cfg;
    cut.workload.rps = 30.0;
    cut.workload.num_requests = 200;
    cut.horizon = 4.0;
    compare_runs(saber::run(cut), saber::cuda::run(cut), "horizon");
    saber::SimConfig cut_st = st;
    cut_st.horizon = 3.3;
    cut_st.engine.prefill_rate = 400.0;  // slots caught in prefill
    compare_runs(saber::run(cut_st), saber::cuda::run(cut_st), "horizon static");
    // Replay with task names outside the catalog (the per-task metrics are
    // keyed by name) and a heavy rate.
    auto custom = saber::generate(cut.workload);
    for (size_t i = 0; i < custom.size(); i += 3) custom[i].task = i % 2 ? "alpha" : "zeta";
    compare_runs(saber::run_with_requests(cfg, custom),
                 saber::cuda::run_with_requests(cfg, custom), "custom tasks");
    // generate() across mixes, rates, sizes and jitters
    for (const char* mx : {"w1", "w2", "w3"})
      for (double rps : {0.5, 7.0, 1e6}) {
        saber::WorkloadSpec w;
        w.mix = saber::preset_mix(mx);
        w.rps = rps;
        w.num_requests = 333;
        w.seed = 1234567;
        w.length_jitter = rps > 1.0 ? 0.0 : 0.6;
        compare_requests(saber::generate(w), saber::cuda::generate(w),
                         std::string("generate ") + mx);
      }

    // A config-2 shaped sweep.
    saber::SweepGrid grid;
    grid.mixes = {"w1", "w2", "w3"};
    grid.rps_list = {2.0, 9.0, 20.0};
    grid.caps = {10, 40, 70};
    grid.with_saber = true;
    saber::SimConfig base;
    base.workload.num_requests = 60;
    base.model = calibrated_usl();
    base.repeats = 3;
    base.seed = 7;
    const saber::SweepResult a = saber::sweep(grid, base, 0);
    const saber::SweepResult b = saber::cuda::sweep(grid, base, 0);
    expect(saber::results_to_csv(a.rows) == saber::results_to_csv(b.rows), "sweep results.csv");
    expect(saber::summary_to_json(a) == saber::summary_to_json(b), "sweep summary.json");

    // The calibration pipeline: profile -> calibrate (USL and linear are
    // bit-exact; the logistic evaluates exp(), compared by its r^2 only).
    saber::EngineConfig ec;
    saber::WorkloadSpec prof;
    prof.mix = saber::preset_mix("w3");
    prof.num_requests = 1000;
    prof.seed = 20260816;
    const auto sa = saber::profile(ec, prof, 50);
    const auto sb = saber::cuda::profile(ec, prof, 50);
    expect(saber::samples_to_csv(sa) == saber::samples_to_csv(sb), "profile samples.csv");
    const auto ca = saber::calibrate(sa);
    const auto cb = saber::cuda::calibrate(sb);
    expect(saber::to_json(ca.best) == saber::to_json(cb.best), "calibrate best_model.json");
    for (int f : {0, 2})
      expect(saber::to_json(ca.fits[f].model) == saber::to_json(cb.fits[f].model),
             std::string("calibrate family ") + std::to_string(f));
    expect(std::abs(*ca.fits[1].model.fit_r2 - *cb.fits[1].model.fit_r2) < 1e-9, "logistic r2");
    const auto fa = saber::fit(sa, saber::ModelFamily::Usl);
    const auto fb = saber::cuda::fit(sb, saber::ModelFamily::Usl);
    expect(saber::to_json(fa) == saber::to_json(fb), "fit usl");
    // FitError / CalibrationError: same type, family, message and payload
    auto fit_error = [](auto&& call) -> std::string {
      try {
        call();
      } catch (const saber::FitError& e) {
        return std::string("FitError ") + saber::to_string(e.family) + " " + e.what() + " " +
               std::to_string(e.best_sse);
      } catch (const saber::CalibrationError& e) {
        return std::string("CalibrationError ") + e.what();
      }
      return "no error";
    };
    const std::vector<saber::LoadSpeedSample> rising = {{1, 10.0}, {2, 12.0}};
    const std::vector<saber::LoadSpeedSample> two = {{1, 10.0}, {2, 9.0}, {2, 8.5}};
    expect(fit_error([&] { saber::fit(rising, saber::ModelFamily::Linear); }) ==
               fit_error([&] { saber::cuda::fit(rising, saber::ModelFamily::Linear); }),
           "FitError increasing linear");
    expect(fit_error([&] { saber::fit(two, saber::ModelFamily::Usl); }) ==
               fit_error([&] { saber::cuda::fit(two, saber::ModelFamily::Usl); }),
           "FitError too few loads");
    expect(fit_error([&] { saber::calibrate(two); }) ==
               fit_error([&] { saber::cuda::calibrate(two); }),
           "CalibrationError insufficient loads");
    std::printf("%s\n", fit_error([&] { saber::cuda::calibrate(two); }).c_str());
  } catch (const std::exception& e) {
    std::printf("EXCEPTION %s\n", e.what());
    return 2;
  }
  if (failures) return 1;
  std::printf("ADAPTER OK\n");
  return 0;
}
