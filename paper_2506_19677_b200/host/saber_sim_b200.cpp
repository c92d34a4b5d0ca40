// saber_sim_b200 — the reference CLI surface (proj/tools/saber_sim.cpp:347-439)
// on the B200 engine.  Same subcommands, flags, defaults, SABER_SIM_SEED rule,
// output files and exit codes (0 ok, 2 usage / config error, 3 runtime
// failure); every number comes from libsaber_b200.so through the C ABI and
// every file is written by saber_io (byte-identical to the reference's
// writers).  It links nothing of the reference.
//
//   calibrate --out DIR [--lmax N] [--samples N] [--seed S] [--mix M] [--jitter J]
//   run       --out DIR [--config F] [--mix M] [--rps R] [--requests N]
//             [--scheduler saber|static] [--cap N] [--model F] [--window N]
//             [--tick T] [--jitter J] [--prefill-rate P] [--horizon H] [--seed S]
//             [--trace F]   (extension: replay a trace CSV, workload.cpp:97-138)
//   sweep     --out DIR [--config F] [--mixes L] [--rps L] [--caps L] [--with-saber]
//             [--model F] [--repeats N] [--requests N] [--window N] [--tick T]
//             [--jitter J] [--prefill-rate P] [--jobs N] [--seed S]
//   --device N (extension) picks the CUDA device.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "saber_io.hpp"

namespace fs = std::filesystem;
using namespace saberb200;

namespace {

constexpr int kOk = 0, kUsage = 2, kRuntime = 3;

// A mistake the caller fixes from the message alone: exit 2.
struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------ engine errors --
void engine(saber_status s) {
  if (s == SABER_OK) return;
  const std::string msg = saber_cuda_last_error();
  if (s == SABER_EINVAL) throw std::invalid_argument(msg);  // exit 2, like the reference
  throw std::runtime_error(msg);                              // exit 3
}

// ------------------------------------------------------------ command line --
enum class Check { None, Positive, NonNegative, Unit };
struct Flag {
  const char* name;
  bool takes_value;
  Check check;
};

const std::map<std::string, std::vector<Flag>>& grammar() {
  static const std::map<std::string, std::vector<Flag>> g = {
      {"calibrate",
       {{"--out", true, Check::None}, {"--lmax", true, Check::Positive},
        {"--samples", true, Check::Positive}, {"--seed", true, Check::None},
        {"--mix", true, Check::None}, {"--jitter", true, Check::Unit},
        {"--device", true, Check::NonNegative}}},
      {"run",
       {{"--out", true, Check::None}, {"--config", true, Check::None}, {"--mix", true, Check::None},
        {"--rps", true, Check::Positive}, {"--requests", true, Check::Positive},
        {"--scheduler", true, Check::None}, {"--cap", true, Check::Positive},
        {"--model", true, Check::None}, {"--window", true, Check::Positive},
        {"--tick", true, Check::Positive}, {"--jitter", true, Check::Unit},
        {"--prefill-rate", true, Check::None}, {"--horizon", true, Check::Positive},
        {"--seed", true, Check::None}, {"--trace", true, Check::None},
        {"--device", true, Check::NonNegative}}},
      {"sweep",
       {{"--out", true, Check::None}, {"--config", true, Check::None},
        {"--mixes", true, Check::None}, {"--rps", true, Check::None}, {"--caps", true, Check::None},
        {"--with-saber", false, Check::None}, {"--model", true, Check::None},
        {"--repeats", true, Check::Positive}, {"--requests", true, Check::Positive},
        {"--window", true, Check::Positive}, {"--tick", true, Check::Positive},
        {"--jitter", true, Check::Unit}, {"--prefill-rate", true, Check::None},
        {"--jobs", true, Check::NonNegative}, {"--seed", true, Check::None},
        {"--device", true, Check::NonNegative}}},
  };
  return g;
}

double number(const std::string& flag, const std::string& text) {
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(text.c_str(), &end);
  if (text.empty() || errno != 0 || *end != '\0')
    throw Usage(flag + ": malformed number \"" + text + "\"");
  return v;
}

struct Args {
  std::string command;
  std::map<std::string, std::string> values;
  std::set<std::string> flags;

  bool has(const std::string& k) const { return values.count(k) || flags.count(k); }
  std::string str(const std::string& k, const std::string& dflt = "") const {
    const auto it = values.find(k);
    return it == values.end() ? dflt : it->second;
  }
  double real(const std::string& k) const { return number(k, values.at(k)); }
  int integer(const std::string& k) const {
    const double v = real(k);
    if (v != std::floor(v) || std::fabs(v) > 2147483647.0)
      throw Usage(k + ": expected an integer, got \"" + values.at(k) + "\"");
    return static_cast<int>(v);
  }
  uint64_t u64(const std::string& k) const {
    const std::string& t = values.at(k);
    errno = 0;
    char* end = nullptr;
    const unsigned long long v = std::strtoull(t.c_str(), &end, 10);
    if (t.empty() || t[0] == '-' || errno != 0 || *end != '\0')
      throw Usage(k + ": expected an unsigned integer, got \"" + t + "\"");
    return v;
  }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw Usage("usage: saber_sim_b200 {calibrate|run|sweep} --out DIR [options]");
  Args a;
  a.command = argv[1];
  const auto g = grammar().find(a.command);
  if (g == grammar().end()) throw Usage("unknown subcommand \"" + a.command + "\"");
  for (int i = 2; i < argc; ++i) {
    std::string tok = argv[i], val;
    bool inline_val = false;
    if (const auto eq = tok.find('='); tok.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      inline_val = true;
    }
    const Flag* f = nullptr;
    for (const Flag& x : g->second)
      if (tok == x.name) f = &x;
    if (!f) throw Usage("unknown option \"" + tok + "\" for " + a.command);
    if (!f->takes_value) {
      if (inline_val) throw Usage(tok + " takes no value");
      a.flags.insert(tok);
      continue;
    }
    if (!inline_val) {
      if (i + 1 >= argc) throw Usage(tok + " needs a value");
      val = argv[++i];
    }
    if (f->check != Check::None) {
      const double v = number(tok, val);
      if (f->check == Check::Positive && !(v > 0.0)) throw Usage(tok + ": value must be positive");
      if (f->check == Check::NonNegative && !(v >= 0.0))
        throw Usage(tok + ": value must be non-negative");
      if (f->check == Check::Unit && !(v >= 0.0 && v <= 1.0))
        throw Usage(tok + ": value must be in [0, 1]");
    }
    a.values[tok] = val;
  }
  if (!a.has("--out")) throw Usage("--out is required");
  return a;
}

// ----------------------------------------------------------------- files ----
std::string slurp(const fs::path& p) {
  std::ifstream in(p, std::ios::binary);
  if (!in) throw std::runtime_error("cannot read " + p.string());
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// Written beside the target, then renamed: a file is complete or absent.
void publish(const fs::path& target, const std::string& bytes) {
  if (!target.parent_path().empty()) fs::create_directories(target.parent_path());
  const fs::path staging = fs::path(target.string() + ".tmp");
  {
    std::ofstream out(staging, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot write " + staging.string());
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    out.flush();
    if (!out) throw std::runtime_error("short write on " + staging.string());
  }
  fs::rename(staging, target);
}

// SABER_SIM_SEED (saber_sim.cpp:71-81): default seed when --seed is absent.
uint64_t env_seed() {
  const char* e = std::getenv("SABER_SIM_SEED");
  if (!e || !*e) return 42;
  errno = 0;
  char* end = nullptr;
  const unsigned long long v = std::strtoull(e, &end, 10);
  if (errno != 0 || end == e || *end != '\0')
    throw Usage("SABER_SIM_SEED must be an unsigned integer, got \"" + std::string(e) + "\"");
  return v;
}

// Range grammar "a-b[:step]" items, comma-separated (saber_sim.cpp:94-128).
std::vector<double> range_list(const std::string& text, const std::string& flag) {
  std::vector<double> out;
  std::stringstream items(text);
  std::string item;
  while (std::getline(items, item, ',')) {
    const size_t dash = item.find('-', 1);  // a leading '-' is a sign
    if (dash == std::string::npos) {
      out.push_back(number(flag, item));
      continue;
    }
    std::string hi_s = item.substr(dash + 1);
    double step = 1.0;
    if (const size_t colon = hi_s.find(':'); colon != std::string::npos) {
      step = number(flag, hi_s.substr(colon + 1));
      hi_s.resize(colon);
    }
    const double lo = number(flag, item.substr(0, dash)), hi = number(flag, hi_s);
    if (!(step > 0.0) || hi < lo) throw Usage(flag + ": empty or backward range \"" + item + "\"");
    for (int k = 0;; ++k) {
      const double v = lo + step * k;
      if (v > hi * (1.0 + 1e-12) && v > hi + 1e-12) break;
      out.push_back(v < hi ? v : hi);
    }
  }
  if (out.empty()) throw Usage(flag + ": empty list \"" + text + "\"");
  return out;
}

saber_mix mix_arg(const std::string& arg) {
  if (arg == "w1" || arg == "w2" || arg == "w3") return io::preset_mix(arg);
  try {
    return io::mix_from_json(slurp(arg));
  } catch (const std::invalid_argument&) {
    throw;  // unknown task: the reference's validate_mix message
  } catch (const std::exception& e) {
    throw Usage("--mix: expected w1, w2, w3, or a JSON file of task proportions: " +
                std::string(e.what()));
  }
}

io::ModelSpec model_arg(const std::string& path) {
  try {
    return io::model_from_json(slurp(path));
  } catch (const std::exception& e) {
    throw Usage("--model: " + std::string(e.what()));
  }
}

io::SimSettings base_settings(const Args& a) {
  if (!a.has("--config")) return io::SimSettings{};
  try {
    return io::sim_settings_from_json(slurp(a.str("--config")));
  } catch (const std::exception& e) {
    throw Usage("--config: " + std::string(e.what()));
  }
}

// Overrides shared by run and sweep (saber_sim.cpp:196-220, 260-270).
void apply_common(const Args& a, io::SimSettings* c) {
  if (a.has("--requests")) c->num_requests = a.integer("--requests");
  if (a.has("--window")) c->window_size = a.integer("--window");
  if (a.has("--tick")) c->tick = a.real("--tick");
  if (a.has("--jitter")) c->length_jitter = a.real("--jitter");
  if (a.has("--prefill-rate")) c->prefill_rate = a.real("--prefill-rate");
  if (a.has("--model")) c->model = model_arg(a.str("--model"));
}

// ------------------------------------------------------------- calibrate ----
int calibrate(const Args& a, uint64_t default_seed) {
  saber_profile_spec ps{};
  ps.ground_truth = io::SimSettings{}.ground_truth.m;  // EngineConfig defaults
  ps.prefill_rate = 2000.0;
  ps.l_max = a.has("--lmax") ? a.integer("--lmax") : 50;
  ps.num_requests = a.has("--samples") ? a.integer("--samples") : 1000;
  ps.seed = a.has("--seed") ? a.u64("--seed") : default_seed;
  ps.length_jitter = a.has("--jitter") ? a.real("--jitter") : 0.2;
  if (saber_cuda_profile_planned_loads(ps.num_requests, ps.l_max) < 3)
    throw Usage(
        "insufficient distinct loads: the sample budget reaches fewer than 3 burst sizes; "
        "raise --samples or lower --lmax");
  ps.mix = mix_arg(a.str("--mix", "w3"));
  const int device = a.has("--device") ? a.integer("--device") : 0;

  const int64_t n = saber_cuda_profile_samples(&ps);
  if (n < 0) engine(SABER_EINVAL);
  std::vector<int32_t> loads(static_cast<size_t>(n));
  std::vector<double> speeds(static_cast<size_t>(n));
  int64_t offs[2] = {0, 0};
  int32_t pstatus = 0;
  saber_profile_desc pd{&ps, 1, device};
  saber_profile_out po{offs, loads.data(), speeds.data(), n, &pstatus, 0.0};
  engine(saber_cuda_profile_batch(&pd, &po));
  if (pstatus != 0) throw std::runtime_error("profile: insufficient distinct loads (< 3)");

  const int64_t curve[2] = {0, n};
  saber_fit_desc fd{loads.data(), speeds.data(), curve, 1, 7, 1, device};
  double params[9] = {}, r2[3] = {};
  int32_t status[3] = {}, best = -1;
  saber_fit_out fo{};
  fo.params = params;
  fo.r2 = r2;
  fo.status = status;
  fo.best_family = &best;
  engine(saber_cuda_fit_batch(&fd, &fo));
  if (best <= -2)
    throw std::runtime_error("calibrate: insufficient distinct loads (" + std::to_string(-2 - best) +
                             " < 3)");
  if (best == -1) throw std::runtime_error("calibrate: no model family produced a fit");
  std::vector<io::FamilyOutcome> fits(3);
  for (int f = 0; f < 3; ++f) {
    io::FamilyOutcome& o = fits[static_cast<size_t>(f)];
    o.family = f;
    o.ok = status[f] == 0;
    o.model.m.family = f;
    for (int k = 0; k < 3; ++k) o.model.m.params[k] = params[3 * f + k];
    if (o.ok) {
      o.model.fit_r2 = r2[f];
    } else {
      o.error = status[f] == SABER_FITERR_TOO_FEW
                    ? std::string("too few samples or distinct loads to fit ") + io::kFamilyNames[f]
                : status[f] == SABER_FITERR_NO_CONVERGENCE
                    ? std::string("optimizer did not converge for ") + io::kFamilyNames[f]
                : status[f] == SABER_FITERR_INCREASING_LINEAR
                    ? "fitted linear model is increasing in load"
                    : "fitted model is not non-increasing in load";
    }
  }
  const io::ModelSpec& chosen = fits[static_cast<size_t>(best)].model;
  const fs::path out(a.str("--out"));
  publish(out / "samples.csv", io::samples_csv(loads, speeds));
  publish(out / "models.json", io::calibration_json(chosen, fits));
  publish(out / "best_model.json", io::model_json(chosen));
  std::cout << "calibrated " << n << " samples, best family " << io::kFamilyNames[best] << "\n";
  return kOk;
}

// ------------------------------------------------------------------- run ----
int run(const Args& a, uint64_t default_seed) {
  io::SimSettings c = base_settings(a);
  if (a.has("--mix")) {
    c.mix = mix_arg(a.str("--mix"));
    c.has_mix = true;
  }
  if (a.has("--rps")) c.rps = a.real("--rps");
  apply_common(a, &c);
  if (a.has("--scheduler")) {
    const std::string s = a.str("--scheduler");
    if (s == "saber") c.mode = SABER_MODE_SABER;
    else if (s == "static") c.mode = SABER_MODE_STATIC;
    else throw Usage("--scheduler: expected saber or static, got \"" + s + "\"");
  }
  if (a.has("--cap")) c.static_batch_size = a.integer("--cap");
  if (a.has("--horizon")) c.horizon = a.real("--horizon");
  std::optional<uint64_t> seed;
  if (a.has("--seed")) seed = a.u64("--seed");
  else if (!a.has("--config")) seed = default_seed;
  if (seed) c.workload_seed = c.seed = *seed;
  if (c.mode == SABER_MODE_SABER && !c.model) throw Usage("saber scheduler requires --model");
  if (c.mode == SABER_MODE_STATIC && c.static_batch_size < 1)
    throw Usage("static scheduler requires --cap");

  saber_traj_spec spec{};
  std::vector<saber_request> replay;
  io::RunFiles r;
  if (a.has("--trace")) {
    const std::string text = slurp(a.str("--trace"));
    int32_t n = 0;
    const saber_status st = saber_cuda_trace_from_csv(text.data(), text.size(), nullptr, 0, &n);
    if (st != SABER_ECAPACITY) engine(st);
    replay.resize(static_cast<size_t>(n));
    engine(saber_cuda_trace_from_csv(text.data(), text.size(), replay.data(), n, &n));
    spec.requests = replay.data();
    spec.num_requests = n;
  } else {
    if (!c.has_mix) throw std::invalid_argument("mix has no tasks");  // validate_mix
    spec.mix = c.mix;
    spec.rps = c.rps;
    spec.num_requests = c.num_requests;
    spec.workload_seed = c.workload_seed;
    spec.length_jitter = c.length_jitter;
  }
  spec.mode = c.mode;
  spec.window_size = c.window_size;
  spec.tick = c.tick;
  spec.static_batch_size = c.static_batch_size;
  spec.has_model = c.model.has_value();
  if (c.model) spec.model = c.model->m;
  spec.ground_truth = c.ground_truth.m;
  spec.prefill_rate = c.prefill_rate;
  spec.has_horizon = c.horizon.has_value();
  spec.horizon = c.horizon.value_or(0.0);
  spec.seed = c.seed;
  const int n = spec.num_requests;
  if (n < 1) throw std::invalid_argument("num_requests must be >= 1");

  saber_run_batch_desc d{&spec, 1, a.has("--device") ? a.integer("--device") : 0};
  r.requests.resize(static_cast<size_t>(n));
  r.states.resize(static_cast<size_t>(n));
  std::vector<double> cdf_l(static_cast<size_t>(n)), cdf_f(static_cast<size_t>(n));
  int32_t issued[4] = {}, met[4] = {};
  int64_t cap = int64_t{1} << 16, n_dec = 0;
  for (;;) {
    r.decisions.resize(static_cast<size_t>(cap));
    saber_run_batch_out o{};
    o.rows = &r.row;
    o.max_n = n;
    o.decisions = r.decisions.data();
    o.decision_cap = cap;
    o.n_decisions = &n_dec;
    o.requests = r.requests.data();
    o.states = r.states.data();
    o.cdf_latency = cdf_l.data();
    o.cdf_fraction = cdf_f.data();
    o.group_issued = issued;
    o.group_met = met;
    o.max_groups = 4;
    const saber_status st = saber_cuda_run_batch(&d, &o);
    if (st == SABER_ECAPACITY && r.row.decisions > cap) {
      cap = r.row.decisions;  // grow to exactly the decision log
      continue;
    }
    engine(st);
    break;
  }
  r.decisions.resize(static_cast<size_t>(n_dec));
  // groups are the catalog tasks in name order (saber_cuda.h saber_request::group)
  static const int kByName[4] = {SABER_TASK_GENERATION, SABER_TASK_QNA, SABER_TASK_SUMMARY,
                                 SABER_TASK_TRANSLATION};
  for (int i = 0; i < n; ++i) r.task_names.push_back(io::kTaskNames[r.requests[static_cast<size_t>(i)].task]);
  int start = 0;
  for (int g = 0; g < 4; ++g) {
    if (issued[g] == 0) continue;
    io::TaskStats t;
    t.name = io::kTaskNames[kByName[g]];
    t.issued = issued[g];
    t.met = met[g];
    for (int p = start; p < start + issued[g]; ++p)
      if (!std::isnan(cdf_f[static_cast<size_t>(p)]))
        t.cdf.emplace_back(cdf_l[static_cast<size_t>(p)], cdf_f[static_cast<size_t>(p)]);
    r.per_task.push_back(std::move(t));
    start += issued[g];
  }
  const fs::path out(a.str("--out"));
  publish(out / "records.csv", io::records_csv(r));
  publish(out / "decisions.csv", io::decisions_csv(r.decisions));
  publish(out / "metrics.json", io::metrics_json(r));
  std::cout << "ran " << n << " requests, goodput " << io::fmt17(r.row.goodput) << "\n";
  return kOk;
}

// ----------------------------------------------------------------- sweep ----
int sweep(const Args& a, uint64_t default_seed) {
  io::SimSettings c = base_settings(a);
  if (a.has("--repeats")) c.repeats = a.integer("--repeats");
  apply_common(a, &c);
  if (a.has("--seed")) c.seed = a.u64("--seed");
  else if (!a.has("--config")) c.seed = default_seed;

  io::SweepFiles s;
  std::vector<int32_t> mix_ids;
  {
    const std::string list = a.str("--mixes", "w1,w2,w3");
    std::stringstream ss(list);
    std::string m;
    while (std::getline(ss, m, ',')) {
      if (m != "w1" && m != "w2" && m != "w3") throw Usage("--mixes: unknown preset \"" + m + "\"");
      s.mixes.push_back(m);
      mix_ids.push_back(m[1] - '0');
    }
    if (s.mixes.empty()) throw Usage("--mixes: empty list");
  }
  s.rps = range_list(a.str("--rps", "1-10,15,20"), "--rps");
  for (const double v : range_list(a.str("--caps", "10-100:10"), "--caps")) {
    const int cap = static_cast<int>(v);
    if (v != static_cast<double>(cap) || cap < 1)
      throw Usage("--caps: caps must be positive integers, got " + std::to_string(v));
    s.caps.push_back(cap);
  }
  s.with_saber = a.flags.count("--with-saber") > 0;
  if (s.with_saber && !c.model) throw Usage("--with-saber requires --model");
  s.repeats = c.repeats;
  s.seed = c.seed;

  saber_sweep_desc d{};
  d.mixes = mix_ids.data();
  d.n_mixes = static_cast<int32_t>(mix_ids.size());
  d.rps = s.rps.data();
  d.n_rps = static_cast<int32_t>(s.rps.size());
  d.caps = s.caps.data();
  d.n_caps = static_cast<int32_t>(s.caps.size());
  d.with_saber = s.with_saber;
  d.num_requests = c.num_requests;
  d.length_jitter = c.length_jitter;
  d.window_size = c.window_size;
  d.tick = c.tick;
  d.has_model = c.model.has_value();
  if (c.model) d.model = c.model->m;
  d.ground_truth = c.ground_truth.m;
  d.prefill_rate = c.prefill_rate;
  d.has_horizon = c.horizon.has_value();
  d.horizon = c.horizon.value_or(0.0);
  d.repeats = c.repeats;
  d.seed = c.seed;
  d.device = a.has("--device") ? a.integer("--device") : 0;
  d.shard_index = 0;
  d.shard_count = 1;
  const int64_t rows = saber_cuda_sweep_rows(&d);
  if (c.repeats < 1) throw std::invalid_argument("repeats must be >= 1");
  s.rows.resize(static_cast<size_t>(rows));
  s.summary.resize(s.mixes.size());
  s.best_cap.resize(s.mixes.size() * s.rps.size());
  saber_sweep_out o{};
  o.row_stats = s.rows.data();
  o.summary = s.summary.data();
  o.best_cap_by_rps = s.best_cap.data();
  engine(saber_cuda_sweep(&d, &o));
  const fs::path out(a.str("--out"));
  publish(out / "results.csv", io::results_csv(s));
  publish(out / "summary.json", io::summary_json(s));
  std::cout << "swept " << rows << " rows over " << s.mixes.size() << " mixes\n";
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && (std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h")) {
    std::cout << "usage: saber_sim_b200 {calibrate|run|sweep} --out DIR [options]\n";
    return kOk;
  }
  try {
    const uint64_t seed = env_seed();  // a bad SABER_SIM_SEED is a usage error for every command
    const Args a = parse(argc, argv);
    if (a.command == "calibrate") return calibrate(a, seed);
    if (a.command == "run") return run(a, seed);
    return sweep(a, seed);
  } catch (const Usage& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kRuntime;
  }
}
