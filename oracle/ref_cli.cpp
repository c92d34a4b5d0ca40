// ref_cli.cpp — TEST INFRASTRUCTURE ONLY.
//
// The reference's CLI surface (proj/tools/saber_sim.cpp:347-439) rebuilt on the
// UNMODIFIED reference library (oracle/_ref/libsaber_ref.so): the reference
// tool needs CLI11, which is not on this image, so this file supplies an
// argument parser for the CLI11 forms the reference uses (`--flag value`,
// `--flag=value`, the boolean `--with-saber`) around the reference's own
// calibrate / run / sweep calls and writers.  tests/test_cli.py diffs the
// product CLI (paper_2506_19677_b200/bin/saber_sim_b200) against it file by
// file.  Built by oracle/Makefile into oracle/_ref/saber_sim_ref.
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"  // nlohmann 3.11.3, the reference's JSON library
#include "saber/text_io.hpp"
#include "saber/calibration.hpp"
#include "saber/metrics.hpp"
#include "saber/scheduler.hpp"
#include "saber/simloop.hpp"

namespace fs = std::filesystem;

namespace {

constexpr int kExitUsage = 2;    // saber_sim.cpp: usage errors
constexpr int kExitRuntime = 3;  // saber_sim.cpp: runtime errors

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};


std::string slurp(const fs::path& p) {
  std::ifstream in(p, std::ios::binary);
  if (!in) throw UsageError("cannot read " + p.string());
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// Write-then-rename, so a crashed run never leaves a truncated output.
void put_file(const fs::path& p, const std::string& text) {
  fs::create_directories(p.parent_path());
  const fs::path tmp = p.string() + ".part";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot write " + tmp.string());
    out << text;
    if (!out.flush()) throw std::runtime_error("short write on " + tmp.string());
  }
  fs::rename(tmp, p);
}

double to_double(const std::string& s, const std::string& flag) {
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (errno != 0 || end == s.c_str() || *end != '\0')
    throw UsageError(flag + ": malformed number \"" + s + "\"");
  return v;
}

long long to_int(const std::string& s, const std::string& flag) {
  errno = 0;
  char* end = nullptr;
  const long long v = std::strtoll(s.c_str(), &end, 10);
  if (errno != 0 || end == s.c_str() || *end != '\0')
    throw UsageError(flag + ": expected an integer, got \"" + s + "\"");
  return v;
}

std::uint64_t to_u64(const std::string& s, const std::string& what) {
  errno = 0;
  char* end = nullptr;
  const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
  if (errno != 0 || end == s.c_str() || *end != '\0' || s[0] == '-')
    throw UsageError(what + " must be an unsigned integer, got \"" + s + "\"");
  return v;
}

std::uint64_t env_seed() {
  const char* e = std::getenv("SABER_SIM_SEED");
  if (!e || !*e) return 42;
  return to_u64(e, "SABER_SIM_SEED");
}

// "1-10,15,20" / "10-100:10": scalars and inclusive ranges a-b[:step]; the
// range values are lo + step*k (clamped to hi), as the reference tool
// expands them, so grids print identically.
std::vector<double> expand_list(const std::string& text, const std::string& flag) {
  std::vector<double> out;
  size_t pos = 0;
  while (pos <= text.size()) {
    const size_t comma = text.find(',', pos);
    const std::string item = text.substr(pos, comma == std::string::npos ? std::string::npos
                                                                          : comma - pos);
    pos = comma == std::string::npos ? text.size() + 1 : comma + 1;
    const size_t dash = item.size() > 1 ? item.find('-', 1) : std::string::npos;
    if (dash == std::string::npos) {
      out.push_back(to_double(item, flag));
      continue;
    }
    std::string hi_s = item.substr(dash + 1);
    double step = 1.0;
    const size_t colon = hi_s.find(':');
    if (colon != std::string::npos) {
      step = to_double(hi_s.substr(colon + 1), flag);
      hi_s = hi_s.substr(0, colon);
    }
    const double lo = to_double(item.substr(0, dash), flag);
    const double hi = to_double(hi_s, flag);
    if (!(step > 0.0) || hi < lo) throw UsageError(flag + ": empty or backward range \"" + item + "\"");
    for (int k = 0;; ++k) {
      const double v = lo + step * k;
      if (v > hi * (1.0 + 1e-12) && v > hi + 1e-12) break;
      out.push_back(v < hi ? v : hi);
    }
  }
  if (out.empty()) throw UsageError(flag + ": empty list \"" + text + "\"");
  return out;
}

saber::WorkloadMix mix_arg(const std::string& a) {
  if (a == "w1" || a == "w2" || a == "w3") return saber::preset_mix(a);
  saber::WorkloadMix m;
  try {
    m.proportions = nlohmann::json::parse(slurp(a)).get<std::map<std::string, double>>();
  } catch (const std::exception& e) {
    throw UsageError(std::string("--mix: expected w1, w2, w3, or a JSON file of task proportions: ") +
                     e.what());
  }
  saber::validate_mix(m);
  return m;
}

saber::SpeedModel model_arg(const std::string& path) {
  try {
    return saber::model_from_json(slurp(path));
  } catch (const std::exception& e) {
    throw UsageError(std::string("--model: ") + e.what());
  }
}

saber::SimConfig config_arg(const std::string& path) {
  if (path.empty()) return saber::SimConfig{};
  try {
    return saber::sim_config_from_json(slurp(path));
  } catch (const std::exception& e) {
    throw UsageError(std::string("--config: ") + e.what());
  }
}

// ------------------------------------------------------------- arguments --
struct Args {
  std::map<std::string, std::string> opt;
  bool with_saber = false;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  const std::string& get(const std::string& k) const { return opt.at(k); }
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& known) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string tok = argv[i];
    if (tok.rfind("--", 0) != 0) throw UsageError("unexpected argument \"" + tok + "\"");
    std::string val;
    bool inline_val = false;
    const size_t eq = tok.find('=');
    if (eq != std::string::npos) {
      val = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      inline_val = true;
    }
    if (tok == "--with-saber" && !inline_val) {
      a.with_saber = true;
      continue;
    }
    bool ok = false;
    for (const auto& k : known) ok = ok || tok == k;
    if (!ok) throw UsageError("unknown option " + tok);
    if (!inline_val) {
      if (i + 1 >= argc) throw UsageError(tok + " requires a value");
      val = argv[++i];
    }
    a.opt[tok] = val;
  }
  return a;
}

double positive(const Args& a, const std::string& k) {
  const double v = to_double(a.get(k), k);
  if (!(v > 0.0)) throw UsageError(k + ": must be positive");
  return v;
}
int positive_int(const Args& a, const std::string& k) {
  const long long v = to_int(a.get(k), k);
  if (v < 1 || v > 2147483647LL) throw UsageError(k + ": must be a positive integer");
  return static_cast<int>(v);
}
double unit_range(const Args& a, const std::string& k) {
  const double v = to_double(a.get(k), k);
  if (!(v >= 0.0 && v <= 1.0)) throw UsageError(k + ": must be in [0, 1]");
  return v;
}

// ------------------------------------------------------------ subcommands --
int cmd_calibrate(const Args& a) {
  if (!a.has("--out")) throw UsageError("calibrate: --out is required");
  const int l_max = a.has("--lmax") ? positive_int(a, "--lmax") : 50;
  const int samples = a.has("--samples") ? positive_int(a, "--samples") : 1000;
  const std::uint64_t seed = a.has("--seed") ? to_u64(a.get("--seed"), "--seed") : env_seed();
  if (saber::planned_distinct_loads(samples, l_max) < 3)
    throw UsageError("insufficient distinct loads: the sample budget reaches fewer than 3 burst "
                     "sizes; raise --samples or lower --lmax");
  saber::WorkloadSpec spec;
  spec.mix = mix_arg(a.has("--mix") ? a.get("--mix") : "w3");
  spec.num_requests = samples;
  spec.seed = seed;
  spec.length_jitter = a.has("--jitter") ? unit_range(a, "--jitter") : 0.2;
  const saber::EngineConfig engine;
  const auto s = saber::profile(engine, spec, l_max);
  const auto report = saber::calibrate(s);
  const fs::path out(a.get("--out"));
  put_file(out / "samples.csv", saber::samples_to_csv(s));
  put_file(out / "models.json", saber::to_json(report));
  put_file(out / "best_model.json", saber::to_json(report.best));
  std::cout << "calibrated " << s.size() << " samples, best family "
            << saber::to_string(report.best.family) << "\n";
  return 0;
}

int cmd_run(const Args& a) {
  if (!a.has("--out")) throw UsageError("run: --out is required");
  saber::SimConfig cfg = config_arg(a.has("--config") ? a.get("--config") : "");
  if (a.has("--mix")) cfg.workload.mix = mix_arg(a.get("--mix"));
  if (a.has("--rps")) cfg.workload.rps = positive(a, "--rps");
  if (a.has("--requests")) cfg.workload.num_requests = positive_int(a, "--requests");
  if (a.has("--jitter")) cfg.workload.length_jitter = unit_range(a, "--jitter");
  if (a.has("--scheduler")) {
    const std::string& m = a.get("--scheduler");
    if (m == "saber") cfg.scheduler.mode = saber::SchedulerMode::Saber;
    else if (m == "static") cfg.scheduler.mode = saber::SchedulerMode::Static;
    else throw UsageError("--scheduler: expected saber or static, got \"" + m + "\"");
  }
  if (a.has("--cap")) cfg.scheduler.static_batch_size = positive_int(a, "--cap");
  if (a.has("--window")) cfg.scheduler.window_size = positive_int(a, "--window");
  if (a.has("--tick")) cfg.scheduler.tick = positive(a, "--tick");
  if (a.has("--model")) cfg.model = model_arg(a.get("--model"));
  if (a.has("--prefill-rate")) cfg.engine.prefill_rate = to_double(a.get("--prefill-rate"), "--prefill-rate");
  if (a.has("--horizon")) cfg.horizon = positive(a, "--horizon");
  std::optional<std::uint64_t> seed;
  if (a.has("--seed")) seed = to_u64(a.get("--seed"), "--seed");
  else if (!a.has("--config")) seed = env_seed();
  if (seed) {
    cfg.workload.seed = *seed;
    cfg.seed = *seed;
  }
  if (cfg.scheduler.mode == saber::SchedulerMode::Saber && !cfg.model)
    throw UsageError("saber scheduler requires --model");
  if (cfg.scheduler.mode == saber::SchedulerMode::Static && cfg.scheduler.static_batch_size < 1)
    throw UsageError("static scheduler requires --cap");
  const saber::RunOutput r = saber::run(cfg);
  const fs::path out(a.get("--out"));
  put_file(out / "records.csv", saber::records_to_csv(r.records));
  put_file(out / "decisions.csv", saber::decisions_to_csv(r.decisions));
  put_file(out / "metrics.json", saber::to_json(r.metrics));
  std::cout << "ran " << r.records.size() << " requests, goodput "
            << saber::format_double(r.metrics.goodput) << "\n";
  return 0;
}

int cmd_sweep(const Args& a) {
  if (!a.has("--out")) throw UsageError("sweep: --out is required");
  saber::SimConfig base = config_arg(a.has("--config") ? a.get("--config") : "");
  if (a.has("--repeats")) base.repeats = positive_int(a, "--repeats");
  if (a.has("--requests")) base.workload.num_requests = positive_int(a, "--requests");
  if (a.has("--window")) base.scheduler.window_size = positive_int(a, "--window");
  if (a.has("--tick")) base.scheduler.tick = positive(a, "--tick");
  if (a.has("--jitter")) base.workload.length_jitter = unit_range(a, "--jitter");
  if (a.has("--prefill-rate")) base.engine.prefill_rate = to_double(a.get("--prefill-rate"), "--prefill-rate");
  if (a.has("--model")) base.model = model_arg(a.get("--model"));
  if (a.has("--seed")) base.seed = to_u64(a.get("--seed"), "--seed");
  else if (!a.has("--config")) base.seed = env_seed();
  int jobs = 0;
  if (a.has("--jobs")) {
    const long long j = to_int(a.get("--jobs"), "--jobs");
    if (j < 0) throw UsageError("--jobs: must be >= 0");
    jobs = static_cast<int>(j);
  }
  saber::SweepGrid grid;
  const std::string mixes = a.has("--mixes") ? a.get("--mixes") : "w1,w2,w3";
  std::stringstream ss(mixes);
  std::string m;
  while (std::getline(ss, m, ',')) {
    if (m != "w1" && m != "w2" && m != "w3") throw UsageError("--mixes: unknown preset \"" + m + "\"");
    grid.mixes.push_back(m);
  }
  if (grid.mixes.empty()) throw UsageError("--mixes: empty list");
  grid.rps_list = expand_list(a.has("--rps") ? a.get("--rps") : "1-10,15,20", "--rps");
  for (const double c : expand_list(a.has("--caps") ? a.get("--caps") : "10-100:10", "--caps")) {
    const int ci = static_cast<int>(c);
    if (c != static_cast<double>(ci) || ci < 1)
      throw UsageError("--caps: caps must be positive integers, got " + std::to_string(c));
    grid.caps.push_back(ci);
  }
  grid.with_saber = a.with_saber;
  if (grid.with_saber && !base.model) throw UsageError("--with-saber requires --model");
  const saber::SweepResult res = saber::sweep(grid, base, jobs);
  const fs::path out(a.get("--out"));
  put_file(out / "results.csv", saber::results_to_csv(res.rows));
  put_file(out / "summary.json", saber::summary_to_json(res));
  std::cout << "swept " << res.rows.size() << " rows over " << grid.mixes.size() << " mixes\n";
  return 0;
}

const char* kUsage =
    "usage: saber_sim_ref {calibrate|run|sweep} --out DIR [options]\n"
    "  calibrate: --lmax N --samples N --seed S --mix ID|FILE --jitter X\n"
    "  run:       --config FILE --mix ID|FILE --rps X --requests N --scheduler saber|static\n"
    "             --cap N --model FILE --window N --tick X --jitter X --prefill-rate X\n"
    "             --horizon X --seed S\n"
    "  sweep:     --config FILE --mixes LIST --rps LIST --caps LIST --with-saber --model FILE\n"
    "             --repeats N --requests N --window N --tick X --jitter X --prefill-rate X\n"
    "             --jobs N --seed S\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage;
    return kExitUsage;
  }
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    std::cout << kUsage;
    return 0;
  }
  try {
    if (sub == "calibrate")
      return cmd_calibrate(parse_args(argc, argv, 2, {"--out", "--lmax", "--samples", "--seed", "--mix",
                                                      "--jitter"}));
    if (sub == "run")
      return cmd_run(parse_args(argc, argv, 2, {"--out", "--config", "--mix", "--rps", "--requests",
                                                "--scheduler", "--cap", "--model", "--window", "--tick",
                                                "--jitter", "--prefill-rate", "--horizon", "--seed"}));
    if (sub == "sweep")
      return cmd_sweep(parse_args(argc, argv, 2, {"--out", "--config", "--mixes", "--rps", "--caps",
                                                  "--model", "--repeats", "--requests", "--window",
                                                  "--tick", "--jitter", "--prefill-rate", "--jobs",
                                                  "--seed"}));
    throw UsageError("unknown subcommand \"" + sub + "\"");
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitRuntime;
  }
}
