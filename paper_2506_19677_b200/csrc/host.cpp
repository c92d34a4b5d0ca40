// host.cpp — host orchestration behind the C ABI (include/saber_cuda.h).
//
// Responsibilities:
//   * validation with the reference's error semantics (types.cpp:94-100,
//     workload.cpp:41-48, simloop.cpp:38-48, 130-136);
//   * the per-seed workload prologue: std::mt19937_64 draws and glibc log
//      — the only host arithmetic on the path, kept here
//     because glibc's log is not correctly rounded and the device cannot
//     reproduce it bit-for-bit;
//   * predict tables per model (glibc exp for the logistic);
//   * device memory (a grow-only per-device cache), H2D/D2H, kernel launches.
// Compiled with g++ without FMA contraction, like the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "saber_internal.h"

using namespace saberb200;

namespace {

thread_local std::string g_err;

saber_status fail(saber_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

}  // namespace

saber_status saberb200::set_error(saber_status s, const std::string& msg) { return fail(s, msg); }

namespace {

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(SABER_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)

#define LAUNCH_TRY(expr)                                                                    \
  do {                                                                                      \
    if ((expr) != 0)                                                                        \
      return fail(SABER_ECUDA,                                                              \
                  std::string("kernel launch failed: ") + cudaGetErrorString(cudaGetLastError())); \
  } while (0)

// ---------------------------------------------------------------- devices --
saber_status use_device(int device) {
  // Validated once per device (cudaGetDeviceProperties costs milliseconds and
  // would sit inside every one-shot call's timed region).
  static std::mutex mu;
  static std::vector<int> ok;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (device >= 0 && device < static_cast<int>(ok.size()) && ok[static_cast<size_t>(device)]) {
      CUDA_TRY(cudaSetDevice(device));
      return SABER_OK;
    }
  }
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(SABER_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= count)
    return fail(SABER_EINVAL, "device ordinal " + std::to_string(device) + " out of range");
  // The library carries an arch-specific sm_100a cubin and no PTX, so only
  // compute capability 10.0 can run it (sm_103 would fail at every launch).
  int major = 0, minor = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  if (major != 10 || minor != 0) {
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    return fail(SABER_ECUDA, std::string("device is not sm_100 (B200): ") + prop.name);
  }
  CUDA_TRY(cudaSetDevice(device));
  std::lock_guard<std::mutex> lk(mu);
  if (static_cast<int>(ok.size()) < count) ok.resize(static_cast<size_t>(count), 0);
  ok[static_cast<size_t>(device)] = 1;
  return SABER_OK;
}

// Phase timings of the host path (SABER_HOST_TRACE=1 prints them to stderr).
struct HostTrace {
  bool on;
  double t0;
  const char* what;
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  explicit HostTrace(const char* w) : on(std::getenv("SABER_HOST_TRACE") != nullptr), t0(now()), what(w) {}
  void mark(const char* phase) {
    if (!on) return;
    const double t = now();
    std::fprintf(stderr, "[saber host] %s %s %.3f ms\n", what, phase, t - t0);
    t0 = t;
  }
};

// ------------------------------------------------------- device block cache --
// Freed blocks are kept per device for reuse (cudaMalloc/cudaFree would sit in
// every one-shot call's timed region).  A block goes back on the list only
// after the work that used it has finished: every owner synchronises its
// streams before releasing (SyncOnExit, saber_cuda_sweep_plan_destroy).
// saber_cuda_release_cache() returns the cached blocks to the driver.
std::mutex g_pool_mu;
std::map<int, std::multimap<size_t, void*>> g_free;  // device -> size -> ptr

void* pool_alloc(int device, size_t bytes) {
  bytes = (bytes + 255) & ~static_cast<size_t>(255);
  if (bytes == 0) bytes = 256;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto& fl = g_free[device];
    auto it = fl.lower_bound(bytes);
    if (it != fl.end() && it->first <= 2 * bytes + (1 << 20)) {
      void* p = it->second;
      fl.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  return p;
}
void pool_free(int device, void* p, size_t bytes) {
  if (!p) return;
  bytes = (bytes + 255) & ~static_cast<size_t>(255);
  if (bytes == 0) bytes = 256;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_free[device].emplace(bytes, p);
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int device = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    pool_free(device, p, bytes);
    p = nullptr;
    bytes = 0;
  }
  bool alloc(int dev, size_t n) {
    release();
    device = dev;
    bytes = n;
    p = pool_alloc(dev, n);
    return p != nullptr;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Declared after the DevBufs of a call (so destroyed before them): waits for
// the call's stream on every exit path once work was enqueued, so no kernel
// still running can touch a block that went back to the cache.
struct SyncOnExit {
  const cudaStream_t* s[2] = {nullptr, nullptr};
  explicit SyncOnExit(const cudaStream_t* a, const cudaStream_t* b = nullptr) : s{a, b} {}
  SyncOnExit(const SyncOnExit&) = delete;
  SyncOnExit& operator=(const SyncOnExit&) = delete;
  ~SyncOnExit() {
    if (s[0]) cudaStreamSynchronize(*s[0]);
    if (s[1] && *s[1]) cudaStreamSynchronize(*s[1]);
  }
};

#define ALLOC_TRY(buf, dev, n)                                                         \
  do {                                                                                 \
    if (!(buf).alloc((dev), (n)))                                                      \
      return fail(SABER_ECUDA, "device allocation of " + std::to_string(n) + " bytes failed"); \
  } while (0)

// ------------------------------------------------------ reference arithmetic --
const int kAvgInH[4] = {186, 463, 31, 670};
const int kAvgOutH[4] = {43, 387, 30, 617};
const double kSlaH[4] = {1.0, 8.0, 1.0, 12.0};
// std::map<std::string,...> order: code_generation, code_qna, code_summary, code_translation
const int kAlphaH[4] = {SABER_TASK_GENERATION, SABER_TASK_QNA, SABER_TASK_SUMMARY,
                        SABER_TASK_TRANSLATION};
// std::map order of the catalog names (records.cu kNameRank), by catalog id
const int32_t kNameRankH[4] = {1, 0, 2, 3};
constexpr uint64_t kSchedulerSeedSalt = 0x9e3779b97f4a7c15ull;  // scheduler.cpp:14

// estimator.cpp:16-31 (eval), restated with libstdc++'s min/max/clamp.
double eval_model(const saber_model& m, double load) {
  const double* p = m.params;
  switch (m.family) {
    case SABER_USL: {
      const double denom = 1.0 + p[1] * (load - 1.0) + p[2] * load * (load - 1.0);
      return p[0] / denom;
    }
    case SABER_LOGISTIC: {
      double arg = p[1] * (load - p[2]);
      arg = std::min(std::max(arg, -700.0), 700.0);
      return p[0] / (1.0 + std::exp(arg));
    }
    case SABER_LINEAR:
      return std::max(p[0] * load + p[1], 1e-6);
  }
  return 0.0;
}

bool valid_family(int f) { return f == SABER_USL || f == SABER_LOGISTIC || f == SABER_LINEAR; }

saber_status validate_mix(const saber_mix& mix) {
  bool any = false;
  double sum = 0.0;
  for (int a = 0; a < 4; ++a) {
    const int t = kAlphaH[a];
    if (!mix.present[t]) continue;
    any = true;
    if (mix.frac[t] < 0.0 || mix.frac[t] > 1.0)
      return fail(SABER_EINVAL, "mix fraction out of [0,1]");
    sum += mix.frac[t];
  }
  if (!any) return fail(SABER_EINVAL, "mix has no tasks");
  if (std::abs(sum - 1.0) > 1e-9)
    return fail(SABER_EINVAL, "mix fractions sum to " + std::to_string(sum));
  return SABER_OK;
}

saber_mix preset(int id) {
  saber_mix m{};
  for (int t = 0; t < 4; ++t) m.present[t] = 1;
  if (id == 1) {  // types.cpp:28-33
    m.frac[SABER_TASK_TRANSLATION] = 0.4;
    m.frac[SABER_TASK_GENERATION] = 0.4;
    m.frac[SABER_TASK_QNA] = 0.1;
    m.frac[SABER_TASK_SUMMARY] = 0.1;
  } else if (id == 2) {  // types.cpp:35-40
    m.frac[SABER_TASK_QNA] = 0.4;
    m.frac[SABER_TASK_SUMMARY] = 0.4;
    m.frac[SABER_TASK_GENERATION] = 0.1;
    m.frac[SABER_TASK_TRANSLATION] = 0.1;
  } else {  // w3, types.cpp:42-46
    for (int t = 0; t < 4; ++t) m.frac[t] = 0.25;
  }
  return m;
}

// Cumulative thresholds in map order, summed exactly as sample_task does.
void mix_thresholds(const saber_mix& m, double* th, int8_t* task, int8_t* last) {
  double cum = 0.0;
  int k = 0;
  *last = -1;
  for (int a = 0; a < 4; ++a) {
    const int t = kAlphaH[a];
    if (!m.present[t]) continue;
    cum += m.frac[t];
    th[k] = cum;
    task[k] = static_cast<int8_t>(t);
    *last = static_cast<int8_t>(t);
    ++k;
  }
  for (; k < 4; ++k) {
    th[k] = 0.0;
    task[k] = -1;
  }
}

// Per-seed draws of generate() (workload.cpp:52-79): 4 per request in order
// gap, task, input length, output length; the gap kept as glibc -log(1-u).
void seed_draws(uint64_t seed, int n, double* out4, double* neglog_sum) {
  std::mt19937_64 rng(seed);
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    const double nl = -std::log(1.0 - u);
    out4[4 * i + 0] = nl;
    out4[4 * i + 1] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    out4[4 * i + 2] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    out4[4 * i + 3] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    s += nl;
  }
  *neglog_sum = s;
}

// Upper bound on scheduler draws for a trajectory whose horizon is <= hb:
// ticks <= hb/tick + 3 (t = min(t+tick, horizon) accumulation), and each tick
// consumes min(window, |high|) - 1 <= min(window, n) - 1 draws.
// First draw-stream length of a run_batch trajectory (grown x8 on exhaustion).
constexpr int64_t kBatchDrawCap = 1 << 18;

int64_t draw_bound(double hb, double tick, int window, int n) {
  const int per = std::min(window, n) - 1;
  if (per <= 0) return 0;
  const double ticks = hb / tick * (1.0 + 1e-9) + 3.0;
  const double b = ticks * per;
  const double cap = 1ull << 28;
  return static_cast<int64_t>(std::min(b, cap));
}

void fill_table(const saber_model& m, int max_load, double* out) {
  out[0] = std::nan("");
  for (int L = 1; L <= max_load; ++L) out[L] = eval_model(m, static_cast<double>(L));
}

// Picks the register-mask width for n requests.
int nwords_for(int n) {
  if (n <= 64) return 1;
  if (n <= 128) return 2;
  if (n <= 256) return 4;
  return 32;
}

// ---------------------------------------------------------- group scratch --
// Lanes per trajectory.  SABER_GROUP overrides for tuning.
int group_size() {
  const char* e = std::getenv("SABER_GROUP");
  if (e) {
    const int g = std::atoi(e);
    if (g == 1 || g == 2 || g == 4 || g == 8 || g == 16 || g == 32) return g;
  }
  return 32;
}

// The launch needs the wide kernel: more requests than the
// register tier masks hold, or a window the nibble Fisher-Yates cannot shuffle.
bool needs_wide(int nmax, int max_window) {
  return nmax > kMaxRequests || max_window > kMaxWindow;
}

struct Scratch {
  DevBuf ledger, low, wslot_g, wslot_m, wmask, wgate, wneed;
  SimLaunch launch{};
  GroupScratch view{};
  // Kernel configuration: G lanes per trajectory.
  saber_status alloc(int device, int nmax, bool wide = false) {
    const int rc = plan_sim(nmax, group_size(), wide, &launch);
    if (rc != 0)
      return fail(SABER_ECUDA, "trajectory kernel configuration failed (" + std::to_string(rc) +
                                   "): " + cudaGetErrorString(cudaGetLastError()));
    // one ledger / low-FIFO slice per resident group of the LARGEST grid any
    // kernel variant launches with (the mode-specialised grids differ)
    int64_t grid = launch.grid;
    for (int v = 0; v < 3; ++v) grid = std::max<int64_t>(grid, launch.grid_sel[v]);
    const int64_t groups = grid * (kSimBlock / kWarp) * (kWarp / launch.group);
    const size_t per = static_cast<size_t>(nmax);
    ALLOC_TRY(ledger, device, static_cast<size_t>(groups) * per * sizeof(double));
    ALLOC_TRY(low, device, static_cast<size_t>(groups) * per * sizeof(uint16_t));
    view.ledger_need = ledger.as<double>();
    view.low_fifo = low.as<uint16_t>();
    view.groups = groups;
    if (launch.wide) {
      const int nw = (nmax + 63) / 64;
      const size_t g = static_cast<size_t>(groups);
      ALLOC_TRY(wslot_g, device, g * per * 8);
      ALLOC_TRY(wslot_m, device, g * per * 8);
      ALLOC_TRY(wmask, device, g * 2 * static_cast<size_t>(nw) * 8);
      ALLOC_TRY(wgate, device, g * 3 * per * 4);
      ALLOC_TRY(wneed, device, g * per * 8);
      view.wslot_g = wslot_g.as<double>();
      view.wslot_m = wslot_m.as<uint64_t>();
      view.wmask = wmask.as<uint64_t>();
      view.wgate = wgate.as<int32_t>();
      view.wneed = wneed.as<double>();
      view.wmask_nw = nw;
    }
    return SABER_OK;
  }
};

struct Workloads {
  DevBuf arr, dl, sla, mo, in, pf, task, dem, hor, items, seed_base, th, tt, tl;
  DevBuf ka, kd;  // tick-table indices of arrival / demote_after (launch_tick_index)
  WorkloadTables view(int nmax) const {
    WorkloadTables w;
    w.arrival = arr.as<double>();
    w.deadline = dl.as<double>();
    w.sla = sla.as<double>();
    w.max_out = mo.as<double>();
    w.input = in.as<double>();
    w.prefill = pf.as<double>();
    w.task = task.as<int8_t>();
    w.demote_after = dem.as<double>();
    w.horizon = hor.as<double>();
    w.arr_tick = ka.p ? ka.as<int32_t>() : nullptr;
    w.dem_tick = kd.p ? kd.as<int32_t>() : nullptr;
    w.nmax = nmax;
    return w;
  }
  saber_status alloc(int device, int64_t n_work, int nmax) {
    const size_t cells = static_cast<size_t>(n_work) * nmax;
    ALLOC_TRY(arr, device, cells * 8);
    ALLOC_TRY(dl, device, cells * 8);
    ALLOC_TRY(sla, device, cells * 8);
    ALLOC_TRY(mo, device, cells * 8);
    ALLOC_TRY(in, device, cells * 8);
    ALLOC_TRY(pf, device, cells * 8);
    ALLOC_TRY(task, device, cells);
    ALLOC_TRY(dem, device, cells * 8);
    ALLOC_TRY(hor, device, static_cast<size_t>(n_work) * 8);
    return SABER_OK;
  }
};

// Tick table for quiet streaks (saber_internal.h TickTable):
// T[k] = fl(T[k-1] + tick) exactly as simloop.cpp:99-100 accumulates t, up to
// a bound on every horizon of the launch (beyond it streaks simply stop).
struct TickTableBuf {
  DevBuf T, DT;
  TickTable view{};
  int64_t bytes = 0;
  saber_status build(int dev, double tick, double hbound) {
    view = TickTable{};
    bytes = 0;
    if (std::getenv("SABER_NO_STREAK")) return SABER_OK;
    if (!(tick > 0.0) || !(hbound > 0.0)) return SABER_OK;
    double est = hbound / tick * (1.0 + 1e-9) + 8.0;
    if (!(est < static_cast<double>(1 << 22))) est = static_cast<double>(1 << 22);
    const int len = static_cast<int>(est);
    if (len < 4) return SABER_OK;
    std::vector<double> t(static_cast<size_t>(len)), dt(static_cast<size_t>(len - 1));
    t[0] = 0.0;
    double dmax = 0.0;
    for (int k = 1; k < len; ++k) {
      t[static_cast<size_t>(k)] = t[static_cast<size_t>(k - 1)] + tick;
      const double d = t[static_cast<size_t>(k)] - t[static_cast<size_t>(k - 1)];
      dt[static_cast<size_t>(k - 1)] = d;
      dmax = std::max(dmax, d);
    }
    ALLOC_TRY(T, dev, t.size() * 8);
    ALLOC_TRY(DT, dev, dt.size() * 8);
    CUDA_TRY(cudaMemcpy(T.p, t.data(), t.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(DT.p, dt.data(), dt.size() * 8, cudaMemcpyHostToDevice));
    view.T = T.as<double>();
    view.DT = DT.as<double>();
    view.len = len;
    view.tick = tick;
    view.inv_tick = 1.0 / tick;
    view.dt_max = dmax;
    bytes = static_cast<int64_t>((t.size() + dt.size()) * 8);
    return SABER_OK;
  }
};

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  ~Timer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  saber_status init() {
    if (!a) CUDA_TRY(cudaEventCreate(&a));
    if (!b) CUDA_TRY(cudaEventCreate(&b));
    return SABER_OK;
  }
};

saber_status validate_model(const saber_model& m, const char* what) {
  if (!valid_family(m.family))
    return fail(SABER_EINVAL, std::string(what) + ": unknown model family");
  return SABER_OK;
}

}  // namespace

// ============================================================== the sweep ==
struct saber_sweep_plan {
  saber_sweep_desc desc{};
  std::vector<int32_t> mixes, caps;
  std::vector<double> rps;
  int device = 0;
  int n = 0, R = 0, nwords = 1;
  int64_t n_rows = 0, rows_shard = 0;
  int n_items = 0;
  int model_tab = -1, gt_tab = 0;
  double ceiling = 0.0;
  std::vector<int64_t> stream_len;   // generated draws per seed stream (<= stream_full)
  std::vector<int64_t> stream_full;  // the provable bound (draw_bound)
  int64_t stream_cap = 0;            // current cap on stream_len (grows on exhaustion)
  int64_t total_draws = 0;

  Workloads wl;
  DevBuf tables, seeds, s_off, s_len, draws, descs, rows, comp, cursor, err, caps_d;
  DevBuf summary, best_cap, cell_scratch, ratios, order, stats, pool_scratch;
  Scratch scratch;
  TickTableBuf ticktab;
  int32_t n_saber_first = 0;  // SABER rows lead the order: split launch
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // Recorded on the caller's stream at every exit of an enqueueing call
  // (success or error), so destroy can wait for all of the plan's work.
  cudaEvent_t tail_run = nullptr, tail_summ = nullptr;
  // reseed: pinned staging of the per-seed inputs, reusable once `staged` fired
  double* h_base = nullptr;
  uint64_t* h_seeds = nullptr;
  cudaEvent_t staged = nullptr;
  double rmin = 0.0;
  ~saber_sweep_plan() {
    if (staged) {
      cudaEventSynchronize(staged);
      cudaEventDestroy(staged);
    }
    if (h_base) cudaFreeHost(h_base);
    if (h_seeds) cudaFreeHost(h_seeds);
    if (side) cudaStreamDestroy(side);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (tail_run) cudaEventDestroy(tail_run);
    if (tail_summ) cudaEventDestroy(tail_summ);
  }
  Timer all, sim, summ;
  bool run_pending = false, summary_pending = false;
  bool rerun = false;  // the draw streams were grown after an exhaustion
  double last_ms = 0.0, sim_ms = 0.0;
  int launches = 0;
  bool summarized = false;
  int64_t h2d_bytes = 0;
};

namespace {

// Every row of the sweep has the same scheduler mode.
bool desc_all_one_mode(const saber_sweep_desc& d) {
  return (d.with_saber && d.n_caps == 0) || (!d.with_saber && d.n_caps > 0);
}

saber_status validate_sweep(const saber_sweep_desc& d) {
  if (d.n_mixes < 1 || d.n_rps < 1 || (d.n_caps < 1 && !d.with_saber))
    return fail(SABER_EINVAL, "sweep: empty grid");
  if (d.with_saber && !d.has_model)
    return fail(SABER_EINVAL, "sweep: saber variant requires a model");
  for (int i = 0; i < d.n_mixes; ++i)
    if (d.mixes[i] < 1 || d.mixes[i] > 3)
      return fail(SABER_EINVAL, "unknown mix preset: w" + std::to_string(d.mixes[i]));
  for (int i = 0; i < d.n_rps; ++i)
    if (!(d.rps[i] > 0.0)) return fail(SABER_EINVAL, "rps must be > 0");
  // The reference pools grid entries by value (simloop.cpp:206-275: rows are
  // matched on mix name, rps value and cap value); the engine's summary works
  // per grid index, so repeated entries are rejected instead of pooled.
  for (int i = 0; i < d.n_mixes; ++i)
    for (int j = 0; j < i; ++j)
      if (d.mixes[i] == d.mixes[j]) return fail(SABER_EINVAL, "sweep: duplicate mix in the grid");
  for (int i = 0; i < d.n_rps; ++i)
    for (int j = 0; j < i; ++j)
      if (d.rps[i] == d.rps[j]) return fail(SABER_EINVAL, "sweep: duplicate rps in the grid");
  for (int i = 0; i < d.n_caps; ++i)
    for (int j = 0; j < i; ++j)
      if (d.caps[i] == d.caps[j]) return fail(SABER_EINVAL, "sweep: duplicate cap in the grid");
  if (d.num_requests < 1) return fail(SABER_EINVAL, "num_requests must be >= 1");
  if (d.num_requests > kMaxRequestsWide)
    return fail(SABER_EINVAL, "num_requests > " + std::to_string(kMaxRequestsWide) +
                                  " is not supported by the B200 engine");
  if (d.length_jitter < 0.0 || d.length_jitter >= 1.0)
    return fail(SABER_EINVAL, "length_jitter must be in [0, 1)");
  if (d.window_size < 1) return fail(SABER_EINVAL, "window_size must be >= 1");
  if (!(d.tick > 0.0)) return fail(SABER_EINVAL, "tick must be > 0");
  for (int i = 0; i < d.n_caps; ++i)
    if (d.caps[i] < 1) return fail(SABER_EINVAL, "static mode requires a positive batch size");
  if (d.repeats < 1) return fail(SABER_EINVAL, "repeats must be >= 1");
  if (d.has_horizon && !(d.horizon > 0.0)) return fail(SABER_EINVAL, "horizon must be > 0");
  if (saber_status s = validate_model(d.ground_truth, "ground truth")) return s;
  if (d.has_model)
    if (saber_status s = validate_model(d.model, "model")) return s;
  if (!(eval_model(d.ground_truth, 1.0) > 0.0))
    return fail(SABER_EINVAL, "engine ground truth must be positive");
  if (d.shard_count < 1 || d.shard_index < 0 || d.shard_index >= d.shard_count)
    return fail(SABER_EINVAL, "bad shard index/count");
  return SABER_OK;
}

}  // namespace

// K2 (per-row metrics) of the plan's shard on `s` (narrow: few single-warp
// blocks, to run beside another sweep's trajectory kernels).
static saber_status metrics_launch_impl(saber_sweep_plan* P, cudaStream_t s, bool narrow) {
  RowMetricsParams rm{};
  rm.rows = P->rows.as<saber_traj_row>();
  rm.completion = P->comp.as<double>();
  rm.wl = P->wl.view(P->n);
  rm.traj = P->descs.as<TrajDesc>();
  rm.n_traj = static_cast<int32_t>(P->rows_shard);
  rm.narrow = narrow ? 1 : 0;
  LAUNCH_TRY(launch_row_metrics(rm, s));
  ++P->launches;
  return SABER_OK;
}

// (Re)size the per-seed scheduler draw streams to min(bound, cap).
saber_status set_stream_lengths(saber_sweep_plan* P, int dev) {
  const size_t ns = P->stream_full.size();
  if (ns == 0) return SABER_OK;
  std::vector<int64_t> off(ns);
  P->stream_len.assign(ns, 0);
  P->total_draws = 0;
  for (size_t i = 0; i < ns; ++i) {
    P->stream_len[i] = std::min(P->stream_full[i], P->stream_cap);
    off[i] = P->total_draws;
    P->total_draws += P->stream_len[i];
  }
  ALLOC_TRY(P->draws, dev, static_cast<size_t>(std::max<int64_t>(1, P->total_draws)) *
                             (P->scratch.launch.wide ? 8 : 4));
  CUDA_TRY(cudaMemcpy(P->s_off.p, off.data(), ns * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->s_len.p, P->stream_len.data(), ns * 8, cudaMemcpyHostToDevice));
  return SABER_OK;
}

namespace {
// The one-shot saber_cuda_sweep's cached plan (see there).
std::mutex g_oneshot_mu;
saber_sweep_plan* g_oneshot = nullptr;

bool same_model(const saber_model& a, const saber_model& b) {
  return a.family == b.family && std::memcmp(a.params, b.params, sizeof(a.params)) == 0;
}
// Every descriptor field but the base seed.
bool same_grid(const saber_sweep_desc& a, const saber_sweep_desc& b) {
  auto same = [](const auto* x, const auto* y, int n) {
    return n == 0 || std::memcmp(x, y, sizeof(*x) * static_cast<size_t>(n)) == 0;
  };
  return a.n_mixes == b.n_mixes && a.n_rps == b.n_rps && a.n_caps == b.n_caps &&
         same(a.mixes, b.mixes, a.n_mixes) && same(a.rps, b.rps, a.n_rps) &&
         same(a.caps, b.caps, a.n_caps) && a.with_saber == b.with_saber &&
         a.num_requests == b.num_requests &&
         std::memcmp(&a.length_jitter, &b.length_jitter, 8) == 0 && a.window_size == b.window_size &&
         std::memcmp(&a.tick, &b.tick, 8) == 0 && a.has_model == b.has_model &&
         (!a.has_model || same_model(a.model, b.model)) && same_model(a.ground_truth, b.ground_truth) &&
         std::memcmp(&a.prefill_rate, &b.prefill_rate, 8) == 0 && a.has_horizon == b.has_horizon &&
         (!a.has_horizon || std::memcmp(&a.horizon, &b.horizon, 8) == 0) && a.repeats == b.repeats &&
         a.device == b.device && a.shard_index == b.shard_index && a.shard_count == b.shard_count;
}
}  // namespace

extern "C" {

int64_t saber_cuda_sweep_rows(const saber_sweep_desc* d) {
  if (!d) return 0;
  const int64_t per_rps =
      static_cast<int64_t>(d->n_caps) * d->repeats + (d->with_saber ? d->repeats : 0);
  return static_cast<int64_t>(d->n_mixes) * d->n_rps * per_rps;
}

saber_status saber_cuda_sweep_plan_create(const saber_sweep_desc* desc, saber_sweep_plan** out) {
  if (!desc || !out) return fail(SABER_EINVAL, "null argument");
  *out = nullptr;
  if (saber_status s = validate_sweep(*desc)) return s;
  HostTrace tr("sweep_plan_create");
  if (saber_status s = use_device(desc->device)) return s;
  tr.mark("use_device");
  auto* P = new saber_sweep_plan();
  std::unique_ptr<saber_sweep_plan> guard(P);
  P->desc = *desc;
  P->mixes.assign(desc->mixes, desc->mixes + desc->n_mixes);
  P->rps.assign(desc->rps, desc->rps + desc->n_rps);
  P->caps.assign(desc->caps, desc->caps + desc->n_caps);
  P->desc.mixes = P->mixes.data();
  P->desc.rps = P->rps.data();
  P->desc.caps = P->caps.data();
  P->device = desc->device;
  P->n = desc->num_requests;
  P->R = desc->repeats;
  P->nwords = nwords_for(P->n);
  P->n_rows = saber_cuda_sweep_rows(desc);
  P->rows_shard = (P->n_rows - desc->shard_index + desc->shard_count - 1) / desc->shard_count;
  if (P->rows_shard < 0) P->rows_shard = 0;
  const int n = P->n, R = P->R, dev = P->device;
  const int n_mixes = desc->n_mixes, n_rps = desc->n_rps;

  // Host prologue: per-seed generate() draws (glibc log), F5/F8.
  std::vector<double> base(static_cast<size_t>(R) * n * 4);
  std::vector<double> neglog_sum(static_cast<size_t>(R));
  for (int i = 0; i < R; ++i)
    seed_draws(desc->seed + static_cast<uint64_t>(i), n, &base[static_cast<size_t>(i) * n * 4],
               &neglog_sum[static_cast<size_t>(i)]);

  tr.mark("seed_draws");
  // Predict tables: [gt | model], index L in 1..n+1.
  const int tl = n + 2;
  std::vector<double> tab(static_cast<size_t>(2 * tl));
  fill_table(desc->ground_truth, n + 1, &tab[0]);
  P->gt_tab = 0;
  if (desc->has_model) {
    fill_table(desc->model, n + 1, &tab[static_cast<size_t>(tl)]);
    P->model_tab = tl;
    P->ceiling = tab[static_cast<size_t>(tl) + 1];
  } else {
    P->ceiling = std::nan("");
  }

  // Workload items: (mix, rps, repeat) -> generate().
  P->n_items = n_mixes * n_rps * R;
  std::vector<WorkloadItem> items(static_cast<size_t>(P->n_items));
  for (int mi = 0; mi < n_mixes; ++mi)
    for (int ri = 0; ri < n_rps; ++ri)
      for (int r = 0; r < R; ++r) {
        WorkloadItem& it = items[static_cast<size_t>((mi * n_rps + ri) * R + r)];
        it.kind = 0;
        it.n = n;
        it.seed_idx = r;
        it.mix = mi;
        it.rps = P->rps[static_cast<size_t>(ri)];
        it.jitter = desc->length_jitter;
        it.ceiling = desc->with_saber ? P->ceiling : std::nan("");
        it.prefill_rate = desc->prefill_rate;
      }
  std::vector<double> th(static_cast<size_t>(n_mixes) * 4);
  std::vector<int8_t> tt(static_cast<size_t>(n_mixes) * 4), tlast(static_cast<size_t>(n_mixes));
  for (int mi = 0; mi < n_mixes; ++mi)
    mix_thresholds(preset(P->mixes[static_cast<size_t>(mi)]), &th[static_cast<size_t>(mi) * 4],
                   &tt[static_cast<size_t>(mi) * 4], &tlast[static_cast<size_t>(mi)]);

  // Scheduler RNG streams, one per seed, sized by the horizon bound.
  std::vector<uint64_t> seeds;
  P->rmin = P->rps[0];
  for (double r : P->rps) P->rmin = std::min(P->rmin, r);
  if (desc->with_saber) {
    const double rmin = P->rmin;
    for (int i = 0; i < R; ++i) {
      const double last = neglog_sum[static_cast<size_t>(i)] / rmin * (1.0 + 1e-9) + n * 1e-6;
      const double hb = desc->has_horizon ? desc->horizon : last + 10.0 * 12.0 + 1.0;
      const int64_t len = draw_bound(hb, desc->tick, desc->window_size, n);
      seeds.push_back((desc->seed + static_cast<uint64_t>(i)) ^ kSchedulerSeedSalt);
      P->stream_full.push_back(len);
    }
  }

  // Horizon bound over every seed (tick table length).
  double hb_max = 0.0;
  {
    double rmin = P->rps[0];
    for (double r : P->rps) rmin = std::min(rmin, r);
    for (int i = 0; i < R; ++i) {
      const double last = neglog_sum[static_cast<size_t>(i)] / rmin * (1.0 + 1e-9) + n * 1e-6;
      hb_max = std::max(hb_max, desc->has_horizon ? desc->horizon : last + 10.0 * 12.0 + 1.0);
    }
  }
  tr.mark("host tables");
  // Device buffers.
  if (saber_status s = P->wl.alloc(dev, P->n_items, n)) return s;
  ALLOC_TRY(P->wl.items, dev, items.size() * sizeof(WorkloadItem));
  ALLOC_TRY(P->wl.seed_base, dev, base.size() * 8);
  ALLOC_TRY(P->wl.th, dev, th.size() * 8);
  ALLOC_TRY(P->wl.tt, dev, tt.size());
  ALLOC_TRY(P->wl.tl, dev, tlast.size());
  ALLOC_TRY(P->tables, dev, tab.size() * 8);
  ALLOC_TRY(P->caps_d, dev, std::max<size_t>(1, P->caps.size()) * 4);
  ALLOC_TRY(P->descs, dev, static_cast<size_t>(std::max<int64_t>(1, P->rows_shard)) * sizeof(TrajDesc));
  ALLOC_TRY(P->rows, dev, static_cast<size_t>(P->n_rows) * sizeof(saber_traj_row));
  ALLOC_TRY(P->comp, dev, static_cast<size_t>(P->n_rows) * n * 8);
  ALLOC_TRY(P->cursor, dev, 16);
  ALLOC_TRY(P->err, dev, 16);
  ALLOC_TRY(P->summary, dev, static_cast<size_t>(n_mixes) * sizeof(saber_mix_summary));
  ALLOC_TRY(P->best_cap, dev, static_cast<size_t>(n_mixes) * n_rps * 4);
  ALLOC_TRY(P->cell_scratch, dev, static_cast<size_t>(n_mixes) * n_rps * 6 * 8);
  ALLOC_TRY(P->pool_scratch, dev, summary_pool_scratch_bytes(n_mixes, n_rps, R, n));
  ALLOC_TRY(P->ratios, dev, static_cast<size_t>(P->n_rows) * n * 8);
  ALLOC_TRY(P->stats, dev, static_cast<size_t>(std::max<int64_t>(1, P->n_rows)) * sizeof(saber_row_stats));
  if (desc->with_saber) {
    ALLOC_TRY(P->seeds, dev, seeds.size() * 8);
    ALLOC_TRY(P->s_off, dev, P->stream_full.size() * 8);
    ALLOC_TRY(P->s_len, dev, P->stream_full.size() * 8);
  }
  tr.mark("device buffers");
  if (saber_status s = P->scratch.alloc(dev, n, needs_wide(n, desc->window_size))) return s;
  tr.mark("scratch + kernel plan");

  // Execution order: every SABER trajectory first (they are
  // ~4x the work of a static one, and keeping the two code paths apart in
  // time keeps the instruction cache warm: 21.9 vs 25.8 ms on config 2),
  // SABER at high rates first (their gates dominate; low-rate SABER runs are
  // mostly streaks), static rows longest arrival span n / rps first.
  // SABER_ORDER=0 orders by n / rps only, 1 = SABER first by n / rps,
  // 2 = row order (A/B runs).
  {
    const int per_rps = desc->n_caps * R + (desc->with_saber ? R : 0);
    const char* om = std::getenv("SABER_ORDER");
    const int order_mode = om ? std::atoi(om) : 3;
    // The key depends only on (rps index, scheduler class): a stable counting
    // sort over those 2 x n_rps buckets (no comparison sort of the rows).
    auto key_of = [&](int ri, bool sab) {
      double kk = -(n / P->rps[static_cast<size_t>(ri)]) - (sab ? 1.0 : 0.0);
      if (order_mode == 1) kk = (sab ? -1e18 : 0.0) - n / P->rps[static_cast<size_t>(ri)];
      if (order_mode == 2) kk = 0.0;
      if (order_mode == 3)  // SABER first, high rates first (the heavy gates); static longest first
        kk = sab ? -1e18 + n / P->rps[static_cast<size_t>(ri)] : -(n / P->rps[static_cast<size_t>(ri)]);
      return kk;
    };
    std::vector<double> distinct;
    for (int ri = 0; ri < n_rps; ++ri)
      for (int c = 0; c < 2; ++c) distinct.push_back(key_of(ri, c != 0));
    std::sort(distinct.begin(), distinct.end());
    distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
    std::vector<int32_t> bucket_of(static_cast<size_t>(2 * n_rps));
    for (int ri = 0; ri < n_rps; ++ri)
      for (int c = 0; c < 2; ++c)
        bucket_of[static_cast<size_t>(2 * ri + c)] = static_cast<int32_t>(
            std::lower_bound(distinct.begin(), distinct.end(), key_of(ri, c != 0)) -
            distinct.begin());
    std::vector<int32_t> bucket(static_cast<size_t>(P->rows_shard));
    std::vector<int64_t> start(distinct.size() + 1, 0);
    // walk row r = shard_index + k * shard_count incrementally (no divisions):
    // rem = r % per_rps, ri = (r / per_rps) % n_rps
    int64_t rem = desc->shard_index % per_rps;
    int ri = static_cast<int>((desc->shard_index / per_rps) % n_rps);
    for (int64_t k = 0; k < P->rows_shard; ++k) {
      if (k > 0) {
        rem += desc->shard_count;
        while (rem >= per_rps) {
          rem -= per_rps;
          if (++ri == n_rps) ri = 0;
        }
      }
      const bool sab = rem >= static_cast<int64_t>(desc->n_caps) * R;
      const int32_t bk = bucket_of[static_cast<size_t>(2 * ri + (sab ? 1 : 0))];
      bucket[static_cast<size_t>(k)] = bk;
      ++start[static_cast<size_t>(bk) + 1];
      if ((order_mode == 1 || order_mode == 3) && sab) ++P->n_saber_first;
    }
    for (size_t b = 1; b < start.size(); ++b) start[b] += start[b - 1];
    std::vector<int32_t> ord(bucket.size());
    for (size_t k = 0; k < bucket.size(); ++k)
      ord[static_cast<size_t>(start[static_cast<size_t>(bucket[k])]++)] = static_cast<int32_t>(k);
    ALLOC_TRY(P->order, dev, std::max<size_t>(1, ord.size()) * 4);
    if (!ord.empty())
      CUDA_TRY(cudaMemcpy(P->order.p, ord.data(), ord.size() * 4, cudaMemcpyHostToDevice));
    P->h2d_bytes += static_cast<int64_t>(ord.size() * 4);
  }

  tr.mark("order");
  CUDA_TRY(cudaMemcpy(P->wl.items.p, items.data(), items.size() * sizeof(WorkloadItem),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->wl.seed_base.p, base.data(), base.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->wl.th.p, th.data(), th.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->wl.tt.p, tt.data(), tt.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->wl.tl.p, tlast.data(), tlast.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->tables.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
  if (!P->caps.empty())
    CUDA_TRY(cudaMemcpy(P->caps_d.p, P->caps.data(), P->caps.size() * 4, cudaMemcpyHostToDevice));
  if (desc->with_saber) {
    CUDA_TRY(cudaMemcpy(P->seeds.p, seeds.data(), seeds.size() * 8, cudaMemcpyHostToDevice));
    // Scheduler draw streams are generated up to a cap far below the provable
    // bound (config 2 uses <= 19K of ~150K); a trajectory that exhausts its
    // stream raises kErrRngExhausted, and the plan grows the cap (up to the
    // bound) and reruns — never a silent draw (saber_cuda_sweep_plan_wait).
    P->stream_cap = 32768;
    if (const char* e = std::getenv("SABER_DRAW_CAP")) P->stream_cap = std::max(1, std::atoi(e));
    if (saber_status s = set_stream_lengths(P, dev)) return s;
  }
  P->h2d_bytes += static_cast<int64_t>(items.size() * sizeof(WorkloadItem) + base.size() * 8 +
                                      th.size() * 8 + tt.size() + tlast.size() + tab.size() * 8 +
                                      P->caps.size() * 4 + seeds.size() * 8 +
                                      P->stream_full.size() * 16);
  tr.mark("h2d");
  if (saber_status s = P->ticktab.build(dev, desc->tick, hb_max)) return s;
  P->h2d_bytes += P->ticktab.bytes;
  if (P->ticktab.view.len > 0) {
    ALLOC_TRY(P->wl.ka, dev, static_cast<size_t>(P->n_items) * n * 4);
    ALLOC_TRY(P->wl.kd, dev, static_cast<size_t>(P->n_items) * n * 4);
  }
  tr.mark("tick table");
  if (saber_status s = P->all.init()) return s;
  if (saber_status s = P->sim.init()) return s;
  if (saber_status s = P->summ.init()) return s;
  // side stream: the static half of a split launch, and the one-shot
  // summary overlapping the row download
  CUDA_TRY(cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&P->join, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&P->tail_run, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&P->tail_summ, cudaEventDisableTiming));
  tr.mark("events");
  *out = guard.release();
  return SABER_OK;
}

// Records `e` on `s` when the enqueueing call returns, on every path.
struct TailMark {
  cudaEvent_t e;
  cudaStream_t s;
  ~TailMark() { cudaEventRecord(e, s); }
};

static saber_status plan_launch_impl(saber_sweep_plan* P, void* stream, bool with_metrics) {
  if (!P) return fail(SABER_EINVAL, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TailMark tail{P->tail_run, s};
  const saber_sweep_desc& d = P->desc;
  P->rerun = false;
  P->launches = 0;
  P->summarized = false;
  P->summary_pending = false;
  CUDA_TRY(cudaEventRecord(P->all.a, s));
  CUDA_TRY(cudaMemsetAsync(P->rows.p, 0, P->rows.bytes, s));
  CUDA_TRY(cudaMemsetAsync(P->cursor.p, 0, 16, s));
  CUDA_TRY(cudaMemsetAsync(P->err.p, 0, 16, s));
  LAUNCH_TRY(launch_fill_rows(P->comp.as<double>(), P->n_rows, P->n, d.shard_index, d.shard_count, s));
  ++P->launches;

  WorkloadParams wp{};
  wp.items = P->wl.items.as<WorkloadItem>();
  wp.n_items = P->n_items;
  wp.seed_base = P->wl.seed_base.as<double>();
  wp.seed_stride = P->n;
  wp.mix_thresh = P->wl.th.as<double>();
  wp.mix_task = P->wl.tt.as<int8_t>();
  wp.mix_last = P->wl.tl.as<int8_t>();
  wp.arrival = P->wl.arr.as<double>();
  wp.deadline = P->wl.dl.as<double>();
  wp.sla = P->wl.sla.as<double>();
  wp.max_out = P->wl.mo.as<double>();
  wp.input = P->wl.in.as<double>();
  wp.prefill = P->wl.pf.as<double>();
  wp.demote_after = P->wl.dem.as<double>();
  wp.horizon = P->wl.hor.as<double>();
  wp.task = P->wl.task.as<int8_t>();
  wp.nmax = P->n;
  LAUNCH_TRY(launch_workloads(wp, s));
  ++P->launches;
  if (P->wl.ka.p) {
    LAUNCH_TRY(launch_tick_index(P->wl.view(P->n), static_cast<int64_t>(P->n_items) * P->n,
                                 P->ticktab.view, P->wl.ka.as<int32_t>(), P->wl.kd.as<int32_t>(), s));
    ++P->launches;
  }

  if (d.with_saber) {
    RngGenParams rg{};
    rg.seeds = P->seeds.as<uint64_t>();
    rg.draws = P->draws.as<uint32_t>();
    rg.wide = P->scratch.launch.wide;
    rg.off = P->s_off.as<int64_t>();
    rg.len = P->s_len.as<int64_t>();
    rg.n_streams = P->R;
    LAUNCH_TRY(launch_rng_streams(rg, s));
    ++P->launches;
  }

  SweepDescParams dp{};
  dp.n_mixes = d.n_mixes;
  dp.n_rps = d.n_rps;
  dp.n_caps = d.n_caps;
  dp.with_saber = d.with_saber;
  dp.repeats = d.repeats;
  dp.n = P->n;
  dp.caps = P->caps_d.as<int32_t>();
  dp.window = d.window_size;
  dp.tick = d.tick;
  dp.prefill_rate = d.prefill_rate;
  dp.model_tab = P->model_tab;
  dp.gt_tab = P->gt_tab;
  dp.has_horizon = d.has_horizon;
  dp.horizon = d.horizon;
  dp.shard_index = d.shard_index;
  dp.shard_count = d.shard_count;
  dp.out = P->descs.as<TrajDesc>();
  dp.n_rows = P->n_rows;
  LAUNCH_TRY(launch_sweep_descs(dp, s, P->rows_shard));
  ++P->launches;

  SimParams sp{};
  sp.traj = P->descs.as<TrajDesc>();
  sp.n_traj = static_cast<int32_t>(P->rows_shard);
  sp.wl = P->wl.view(P->n);
  sp.tables = P->tables.as<double>();
  sp.rng.draws = P->draws.as<uint32_t>();
  sp.rng.wide = P->scratch.launch.wide;
  sp.rng.off = P->s_off.as<int64_t>();
  sp.rng.len = P->s_len.as<int64_t>();
  sp.scratch = P->scratch.view;
  sp.slot_rows = P->scratch.launch.slot_rows;
  sp.out.rows = P->rows.as<saber_traj_row>();
  sp.out.completion = P->comp.as<double>();
  sp.out.error = P->err.as<int32_t>();
  sp.next_traj = P->cursor.as<int32_t>();
  sp.order = P->order.as<int32_t>();
  sp.ticks = P->ticktab.view;
  CUDA_TRY(cudaEventRecord(P->sim.a, s));
  const bool split = P->n_saber_first > 0 && P->n_saber_first < P->rows_shard &&
                     P->scratch.launch.group == 32 && !P->scratch.launch.wide &&
                     std::getenv("SABER_NO_SPLIT") == nullptr;
  if (split) {
    // SABER rows [0, ns) on the SABER-only kernel, static rows [ns, N) on the
    // static-only kernel, concurrently (the second fills SMs as the first drains).
    SimParams sa = sp, st = sp;
    sa.mode_sel = 2;
    sa.split_saber = 1;
    sa.n_traj = P->n_saber_first;
    st.mode_sel = 1;
    st.first_traj = P->n_saber_first;
    st.next_traj = P->cursor.as<int32_t>() + 1;
    CUDA_TRY(cudaEventRecord(P->fork, s));
    CUDA_TRY(cudaStreamWaitEvent(P->side, P->fork, 0));
    LAUNCH_TRY(launch_sim(sa, P->scratch.launch, s));
    LAUNCH_TRY(launch_sim(st, P->scratch.launch, P->side));
    CUDA_TRY(cudaEventRecord(P->join, P->side));
    CUDA_TRY(cudaStreamWaitEvent(s, P->join, 0));
    P->launches += 2;
  } else {
    // one class only: its specialised kernel (falls back to the generic one
    // off the G = 32 path inside launch_sim)
    if (desc_all_one_mode(d)) sp.mode_sel = d.with_saber ? 2 : 1;
    LAUNCH_TRY(launch_sim(sp, P->scratch.launch, s));
    ++P->launches;
  }
  CUDA_TRY(cudaEventRecord(P->sim.b, s));
  if (with_metrics) {
    if (saber_status st = metrics_launch_impl(P, s, false)) return st;
  }
  CUDA_TRY(cudaEventRecord(P->all.b, s));
  P->run_pending = true;
  return SABER_OK;
}

saber_status saber_cuda_sweep_plan_launch(saber_sweep_plan* P, void* stream) {
  return plan_launch_impl(P, stream, true);
}

saber_status saber_cuda_sweep_plan_launch_sim(saber_sweep_plan* P, void* stream) {
  return plan_launch_impl(P, stream, false);
}

saber_status saber_cuda_sweep_plan_metrics_launch(saber_sweep_plan* P, void* stream) {
  if (!P) return fail(SABER_EINVAL, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  return metrics_launch_impl(P, static_cast<cudaStream_t>(stream), true);
}

saber_status saber_cuda_sweep_plan_wait(saber_sweep_plan* P) {
  if (!P) return fail(SABER_EINVAL, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  if (P->run_pending) {
    CUDA_TRY(cudaEventSynchronize(P->all.b));
    float ms = 0.f, ms2 = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, P->all.a, P->all.b));
    CUDA_TRY(cudaEventElapsedTime(&ms2, P->sim.a, P->sim.b));
    P->last_ms = ms;
    P->sim_ms = ms2;
    P->run_pending = false;
    int32_t err = 0;
    CUDA_TRY(cudaMemcpy(&err, P->err.p, 4, cudaMemcpyDeviceToHost));
    if (err == kErrRngExhausted) {
      int64_t full = 0;
      for (int64_t f : P->stream_full) full = std::max(full, f);
      if (P->stream_cap < full) {
        P->stream_cap = std::min(full, P->stream_cap * 4);
        if (saber_status s = set_stream_lengths(P, P->device)) return s;
        P->rerun = true;
        return fail(SABER_ERETRY, "scheduler RNG streams grown; rerun the sweep");
      }
      return fail(SABER_EINTERNAL, "scheduler RNG stream exhausted (draw bound violated)");
    }
    if (err != 0) return fail(SABER_EINTERNAL, "trajectory kernel error " + std::to_string(err));
  }
  if (P->summary_pending) {
    CUDA_TRY(cudaEventSynchronize(P->summ.b));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, P->summ.a, P->summ.b));
    P->last_ms += ms;
    P->summary_pending = false;
    P->summarized = true;
  }
  return SABER_OK;
}

saber_status saber_cuda_sweep_plan_run(saber_sweep_plan* P, void* stream) {
  for (;;) {
    if (saber_status s = saber_cuda_sweep_plan_launch(P, stream)) return s;
    const saber_status s = saber_cuda_sweep_plan_wait(P);
    if (s != SABER_ERETRY) return s;  // grown draw streams: run again
  }
}

static saber_status summarize_launch_impl(saber_sweep_plan* P, void* stream, bool narrow) {
  if (!P) return fail(SABER_EINVAL, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TailMark tail{P->tail_summ, s};
  const saber_sweep_desc& d = P->desc;
  SummaryParams sp{};
  sp.rows = P->rows.as<saber_traj_row>();
  sp.completion = P->comp.as<double>();
  sp.wl = P->wl.view(P->n);
  sp.n_mixes = d.n_mixes;
  sp.n_rps = d.n_rps;
  sp.n_caps = d.n_caps;
  sp.with_saber = d.with_saber;
  sp.repeats = d.repeats;
  sp.n = P->n;
  sp.caps = P->caps_d.as<int32_t>();
  sp.summary = P->summary.as<saber_mix_summary>();
  sp.best_cap = P->best_cap.as<int32_t>();
  sp.scratch = P->cell_scratch.as<double>();
  sp.pool_scratch = P->pool_scratch.p;
  sp.ratios = P->ratios.as<double>();
  sp.narrow = narrow ? 1 : 0;
  CUDA_TRY(cudaEventRecord(P->summ.a, s));
  LAUNCH_TRY(launch_summary(sp, s));
  CUDA_TRY(cudaEventRecord(P->summ.b, s));
  P->launches += 4;
  P->summary_pending = true;
  return SABER_OK;
}

saber_status saber_cuda_sweep_plan_summarize_launch(saber_sweep_plan* P, void* stream) {
  return summarize_launch_impl(P, stream, true);
}

saber_status saber_cuda_sweep_plan_summarize(saber_sweep_plan* P, void* stream) {
  if (saber_status s = summarize_launch_impl(P, stream, false)) return s;
  return saber_cuda_sweep_plan_wait(P);
}

saber_status saber_cuda_sweep_plan_buffers(saber_sweep_plan* P, saber_sweep_buffers* out) {
  if (!P || !out) return fail(SABER_EINVAL, "null argument");
  out->rows = P->rows.p;
  out->rows_bytes = static_cast<size_t>(P->n_rows) * sizeof(saber_traj_row);
  out->completion_times = P->comp.p;
  out->completion_bytes = static_cast<size_t>(P->n_rows) * P->n * 8;
  out->n_rows = P->n_rows;
  out->rows_this_shard = P->rows_shard;
  return SABER_OK;
}

saber_status saber_cuda_sweep_plan_fetch(saber_sweep_plan* P, saber_sweep_out* out) {
  if (!P || !out) return fail(SABER_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(P->device));
  out->n_rows = P->n_rows;
  out->h2d_bytes = P->h2d_bytes;
  out->d2h_bytes = 0;
  if (out->rows) out->d2h_bytes += static_cast<int64_t>(P->n_rows) * sizeof(saber_traj_row);
  if (out->row_stats) out->d2h_bytes += static_cast<int64_t>(P->n_rows) * sizeof(saber_row_stats);
  if (out->completion_times) out->d2h_bytes += static_cast<int64_t>(P->n_rows) * P->n * 8;
  if (out->summary) out->d2h_bytes += P->desc.n_mixes * static_cast<int64_t>(sizeof(saber_mix_summary));
  if (out->best_cap_by_rps) out->d2h_bytes += static_cast<int64_t>(P->desc.n_mixes) * P->desc.n_rps * 4;
  if (out->rows)
    CUDA_TRY(cudaMemcpy(out->rows, P->rows.p, static_cast<size_t>(P->n_rows) * sizeof(saber_traj_row),
                        cudaMemcpyDeviceToHost));
  if (out->row_stats) {
    const size_t bytes = static_cast<size_t>(P->n_rows) * sizeof(saber_row_stats);
    LAUNCH_TRY(launch_pack_row_stats(P->rows.as<saber_traj_row>(), P->n_rows,
                                     P->stats.as<saber_row_stats>(), nullptr));
    CUDA_TRY(cudaMemcpy(out->row_stats, P->stats.p, bytes, cudaMemcpyDeviceToHost));
  }
  if (out->completion_times)
    CUDA_TRY(cudaMemcpy(out->completion_times, P->comp.p, static_cast<size_t>(P->n_rows) * P->n * 8,
                        cudaMemcpyDeviceToHost));
  if (out->summary || out->best_cap_by_rps) {
    if (!P->summarized) return fail(SABER_EINVAL, "summary requested before summarize");
    if (out->summary)
      CUDA_TRY(cudaMemcpy(out->summary, P->summary.p,
                          static_cast<size_t>(P->desc.n_mixes) * sizeof(saber_mix_summary),
                          cudaMemcpyDeviceToHost));
    if (out->best_cap_by_rps)
      CUDA_TRY(cudaMemcpy(out->best_cap_by_rps, P->best_cap.p,
                          static_cast<size_t>(P->desc.n_mixes) * P->desc.n_rps * 4,
                          cudaMemcpyDeviceToHost));
  }
  out->device_ms = P->last_ms;
  out->kernel_launches = P->launches;
  return SABER_OK;
}

saber_status saber_cuda_sweep_plan_stats(saber_sweep_plan* P, double* device_ms, double* sim_ms,
                                         int32_t* launches) {
  if (!P) return fail(SABER_EINVAL, "null plan");
  if (device_ms) *device_ms = P->last_ms;
  if (sim_ms) *sim_ms = P->sim_ms;
  if (launches) *launches = P->launches;
  return SABER_OK;
}

saber_status saber_cuda_sweep_plan_reseed(saber_sweep_plan* P, uint64_t seed, void* stream) {
  if (!P) return fail(SABER_EINVAL, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = P->n, R = P->R;
  const size_t base_bytes = static_cast<size_t>(R) * n * 4 * 8;
  if (!P->h_base) {
    CUDA_TRY(cudaMallocHost(&P->h_base, base_bytes));
    CUDA_TRY(cudaMallocHost(&P->h_seeds, static_cast<size_t>(R) * 8));
    CUDA_TRY(cudaEventCreateWithFlags(&P->staged, cudaEventDisableTiming));
  } else {
    CUDA_TRY(cudaEventSynchronize(P->staged));  // the previous upload read the staging
  }
  // host prologue: per-seed generate() draws, glibc log
  std::vector<double> neglog(static_cast<size_t>(R));
  for (int i = 0; i < R; ++i)
    seed_draws(seed + static_cast<uint64_t>(i), n, P->h_base + static_cast<size_t>(i) * n * 4,
               &neglog[static_cast<size_t>(i)]);
  P->desc.seed = seed;
  int64_t bytes = static_cast<int64_t>(base_bytes);
  CUDA_TRY(cudaMemcpyAsync(P->wl.seed_base.p, P->h_base, base_bytes, cudaMemcpyHostToDevice, s));
  if (P->desc.with_saber) {
    bool lengths_changed = false;
    for (int i = 0; i < R; ++i) {
      P->h_seeds[i] = (seed + static_cast<uint64_t>(i)) ^ kSchedulerSeedSalt;
      const double last = neglog[static_cast<size_t>(i)] / P->rmin * (1.0 + 1e-9) + n * 1e-6;
      const double hb = P->desc.has_horizon ? P->desc.horizon : last + 10.0 * 12.0 + 1.0;
      const int64_t full = draw_bound(hb, P->desc.tick, P->desc.window_size, n);
      lengths_changed |= std::min(full, P->stream_cap) != P->stream_len[static_cast<size_t>(i)];
      P->stream_full[static_cast<size_t>(i)] = full;
    }
    if (lengths_changed) {  // stream layout changes: re-derive it (synchronous, rare)
      CUDA_TRY(cudaStreamSynchronize(s));
      if (saber_status e = set_stream_lengths(P, P->device)) return e;
    }
    CUDA_TRY(cudaMemcpyAsync(P->seeds.p, P->h_seeds, static_cast<size_t>(R) * 8,
                             cudaMemcpyHostToDevice, s));
    bytes += static_cast<int64_t>(R) * 8;
  }
  CUDA_TRY(cudaEventRecord(P->staged, s));
  P->h2d_bytes = bytes;
  return SABER_OK;
}

saber_status saber_cuda_sweep_plan_fetch_async(saber_sweep_plan* P, saber_sweep_out* out,
                                               void* stream) {
  if (!P || !out) return fail(SABER_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((out->summary || out->best_cap_by_rps) && !P->summary_pending && !P->summarized)
    return fail(SABER_EINVAL, "summary requested before summarize");
  out->n_rows = P->n_rows;
  out->h2d_bytes = P->h2d_bytes;
  out->d2h_bytes = 0;
  const size_t nr = static_cast<size_t>(P->n_rows);
  if (out->rows) {
    CUDA_TRY(cudaMemcpyAsync(out->rows, P->rows.p, nr * sizeof(saber_traj_row), cudaMemcpyDeviceToHost, s));
    out->d2h_bytes += static_cast<int64_t>(nr * sizeof(saber_traj_row));
  }
  if (out->row_stats) {
    LAUNCH_TRY(launch_pack_row_stats(P->rows.as<saber_traj_row>(), P->n_rows,
                                     P->stats.as<saber_row_stats>(), s));
    CUDA_TRY(cudaMemcpyAsync(out->row_stats, P->stats.p, nr * sizeof(saber_row_stats),
                             cudaMemcpyDeviceToHost, s));
    out->d2h_bytes += static_cast<int64_t>(nr * sizeof(saber_row_stats));
  }
  if (out->completion_times) {
    CUDA_TRY(cudaMemcpyAsync(out->completion_times, P->comp.p, nr * P->n * 8, cudaMemcpyDeviceToHost, s));
    out->d2h_bytes += static_cast<int64_t>(nr * P->n * 8);
  }
  if (out->summary) {
    const size_t b = static_cast<size_t>(P->desc.n_mixes) * sizeof(saber_mix_summary);
    CUDA_TRY(cudaMemcpyAsync(out->summary, P->summary.p, b, cudaMemcpyDeviceToHost, s));
    out->d2h_bytes += static_cast<int64_t>(b);
  }
  if (out->best_cap_by_rps) {
    const size_t b = static_cast<size_t>(P->desc.n_mixes) * P->desc.n_rps * 4;
    CUDA_TRY(cudaMemcpyAsync(out->best_cap_by_rps, P->best_cap.p, b, cudaMemcpyDeviceToHost, s));
    out->d2h_bytes += static_cast<int64_t>(b);
  }
  return SABER_OK;
}

void saber_cuda_sweep_plan_destroy(saber_sweep_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  // Wait for everything the plan enqueued (its buffers go back to the cache).
  if (P->tail_run) cudaEventSynchronize(P->tail_run);
  if (P->tail_summ) cudaEventSynchronize(P->tail_summ);
  if (P->side) cudaStreamSynchronize(P->side);
  delete P;
}

saber_status saber_cuda_release_cache(int32_t device) {
  {
    std::lock_guard<std::mutex> lk1(g_oneshot_mu);
    if (g_oneshot && g_oneshot->device == device) {
      saber_cuda_sweep_plan_destroy(g_oneshot);
      g_oneshot = nullptr;
    }
  }
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_free.find(device);
  if (it == g_free.end()) return SABER_OK;
  CUDA_TRY(cudaSetDevice(device));
  for (auto& kv : it->second) cudaFree(kv.second);
  g_free.erase(it);
  return SABER_OK;
}

saber_status saber_cuda_sweep(const saber_sweep_desc* desc, saber_sweep_out* out) {
  if (!desc || !out) return fail(SABER_EINVAL, "null argument");
  if (saber_status s = validate_sweep(*desc)) return s;
  // One-shot calls with the same grid reuse the last call's plan (its device
  // buffers, streams and tick table); the inputs are still staged from the
  // host every call (reseed: host prologue + H2D), so nothing is cached but
  // allocations.  A concurrent caller gets a private plan.
  std::unique_lock<std::mutex> lk(g_oneshot_mu, std::try_to_lock);
  saber_sweep_plan* P = nullptr;
  std::unique_ptr<saber_sweep_plan, void (*)(saber_sweep_plan*)> guard(nullptr,
                                                                        saber_cuda_sweep_plan_destroy);
  if (lk.owns_lock() && g_oneshot && same_grid(g_oneshot->desc, *desc)) {
    P = g_oneshot;
    if (saber_status s = saber_cuda_sweep_plan_reseed(P, desc->seed, nullptr)) return s;
  } else {
    if (saber_status s = saber_cuda_sweep_plan_create(desc, &P)) return s;
    if (lk.owns_lock()) {
      if (g_oneshot) saber_cuda_sweep_plan_destroy(g_oneshot);
      g_oneshot = P;
    } else {
      guard.reset(P);
    }
  }
  if (saber_status s = saber_cuda_sweep_plan_run(P, nullptr)) return s;
  const bool want_summary = out->summary || out->best_cap_by_rps;
  if (want_summary) {
    if (desc->shard_count != 1)
      return fail(SABER_EINVAL, "summary of a sharded sweep needs the rows of every shard "
                                "(all-reduce the plan buffers, then summarize)");
    // the summary runs on the side stream while the rows download
    if (saber_status s = summarize_launch_impl(P, P->side, false)) return s;
  }
  saber_sweep_out rows_part = *out;
  rows_part.summary = nullptr;
  rows_part.best_cap_by_rps = nullptr;
  if (saber_status s = saber_cuda_sweep_plan_fetch(P, &rows_part)) return s;
  int64_t d2h = rows_part.d2h_bytes;
  if (want_summary) {
    if (saber_status s = saber_cuda_sweep_plan_wait(P)) return s;
    saber_sweep_out summ_part{};
    summ_part.summary = out->summary;
    summ_part.best_cap_by_rps = out->best_cap_by_rps;
    if (saber_status s = saber_cuda_sweep_plan_fetch(P, &summ_part)) return s;
    d2h += summ_part.d2h_bytes;
  }
  out->n_rows = P->n_rows;
  out->h2d_bytes = P->h2d_bytes;
  out->d2h_bytes = d2h;
  out->device_ms = P->last_ms;
  out->kernel_launches = P->launches;
  return SABER_OK;
}

const char* saber_cuda_last_error(void) { return g_err.c_str(); }
int32_t saber_cuda_abi_version(void) { return SABER_CUDA_ABI_VERSION; }

int32_t saber_cuda_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return 0;
  int usable = 0;
  for (int i = 0; i < count; ++i) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10 && p.minor == 0) ++usable;
  }
  return usable;
}

saber_status saber_cuda_predict_table(const saber_model* model, int32_t max_load, double* table) {
  if (!model || !table) return fail(SABER_EINVAL, "null argument");
  if (saber_status s = validate_model(*model, "model")) return s;
  if (max_load < 1) return fail(SABER_EDOMAIN, "predict: load must be >= 1");
  for (int L = 1; L <= max_load; ++L) table[L - 1] = eval_model(*model, static_cast<double>(L));
  return SABER_OK;
}

}  // extern "C"

// ============================================================== run batch ==
namespace {

saber_status validate_spec(const saber_traj_spec& s) {
  if (s.window_size < 1) return fail(SABER_EINVAL, "window_size must be >= 1");
  if (!(s.tick > 0.0)) return fail(SABER_EINVAL, "tick must be > 0");
  if (s.mode != SABER_MODE_SABER && s.mode != SABER_MODE_STATIC)
    return fail(SABER_EINVAL, "unknown scheduler mode");
  if (s.mode == SABER_MODE_STATIC && s.static_batch_size < 1)
    return fail(SABER_EINVAL, "static mode requires a positive batch size");
  if (s.mode == SABER_MODE_SABER && !s.has_model)
    return fail(SABER_EINVAL, "saber mode requires a speed model");
  if (s.has_horizon && !(s.horizon > 0.0)) return fail(SABER_EINVAL, "horizon must be > 0");
  if (saber_status e = validate_model(s.ground_truth, "ground truth")) return e;
  if (s.has_model)
    if (saber_status e = validate_model(s.model, "model")) return e;
  if (!(eval_model(s.ground_truth, 1.0) > 0.0))
    return fail(SABER_EINVAL, "engine ground truth must be positive");
  if (s.num_requests < 1)
    return fail(SABER_EINVAL, s.requests ? "run: no requests" : "num_requests must be >= 1");
  if (s.num_requests > kMaxRequestsWide)
    return fail(SABER_EINVAL, "num_requests > " + std::to_string(kMaxRequestsWide) +
                                  " is not supported by the B200 engine");
  if (!s.requests) {
    if (!(s.rps > 0.0)) return fail(SABER_EINVAL, "rps must be > 0");
    if (s.length_jitter < 0.0 || s.length_jitter >= 1.0)
      return fail(SABER_EINVAL, "length_jitter must be in [0, 1)");
    if (saber_status e = validate_mix(s.mix)) return e;
  }
  return SABER_OK;
}

}  // namespace

extern "C" saber_status saber_cuda_run_batch(const saber_run_batch_desc* desc,
                                             saber_run_batch_out* out) {
  if (!desc || !out) return fail(SABER_EINVAL, "null argument");
  const int T = desc->n_traj;
  if (T < 1) return fail(SABER_EINVAL, "run_batch: no trajectories");
  if (!out->rows) return fail(SABER_EINVAL, "run_batch: rows output required");
  int nmax = 1, wmax = 1;
  for (int k = 0; k < T; ++k) {
    if (saber_status s = validate_spec(desc->specs[k])) return s;
    nmax = std::max(nmax, desc->specs[k].num_requests);
    if (desc->specs[k].mode == SABER_MODE_SABER) wmax = std::max(wmax, desc->specs[k].window_size);
  }
  const bool wide = needs_wide(nmax, wmax);
  const bool want_states = out->states || out->cdf_latency || out->cdf_fraction ||
                           out->group_issued || out->group_met;
  if ((out->arrival_times || out->admit_times || out->completion_times || out->demoted ||
       out->requests || want_states) &&
      out->max_n < nmax)
    return fail(SABER_EINVAL, "run_batch: max_n smaller than the largest trajectory");
  if ((out->cdf_latency == nullptr) != (out->cdf_fraction == nullptr) ||
      (out->group_issued == nullptr) != (out->group_met == nullptr))
    return fail(SABER_EINVAL, "run_batch: cdf_latency/cdf_fraction and group_issued/group_met "
                              "come in pairs");
  if (out->group_issued) {
    for (int k = 0; k < T; ++k) {
      const saber_traj_spec& s = desc->specs[k];
      if (!s.requests) {
        if (out->max_groups < 4)
          return fail(SABER_EINVAL, "run_batch: max_groups < 4 with a generated trajectory");
        continue;
      }
      for (int i = 0; i < s.num_requests; ++i)
        if (s.requests[i].group < 0 || s.requests[i].group >= out->max_groups)
          return fail(SABER_EINVAL, "run_batch: request group outside [0, max_groups)");
    }
  }
  if (saber_status s = use_device(desc->device)) return s;
  const int dev = desc->device;

  // Workloads (one per trajectory), tables, streams, descriptors.
  std::vector<WorkloadItem> items(static_cast<size_t>(T));
  std::vector<double> base(static_cast<size_t>(T) * nmax * 4, 0.0);
  std::vector<double> th(static_cast<size_t>(T) * 4);
  std::vector<int8_t> tt(static_cast<size_t>(T) * 4), tlast(static_cast<size_t>(T));
  const size_t cells = static_cast<size_t>(T) * nmax;
  std::vector<double> arr(cells, 0.0), dl(cells, 0.0), sla(cells, 1.0), mo(cells, 1.0), in(cells, 1.0);
  std::vector<int8_t> task(cells, -1);
  std::vector<int32_t> group(cells, -1);  // -1: generated (the task's name rank)
  bool any_replay = false;
  const int tl = nmax + 2;
  std::vector<double> tab(static_cast<size_t>(T) * 2 * tl);
  std::vector<TrajDesc> descs(static_cast<size_t>(T));
  std::vector<std::pair<double, double>> tick_hb;  // (tick, horizon bound) per trajectory
  std::vector<uint64_t> seeds;
  std::vector<int64_t> off, len, stream_full;
  std::vector<int> stream_traj;
  int64_t total_draws = 0;
  for (int k = 0; k < T; ++k) {
    const saber_traj_spec& s = desc->specs[k];
    const int n = s.num_requests;
    double* gt = &tab[static_cast<size_t>(k) * 2 * tl];
    double* mt = gt + tl;
    fill_table(s.ground_truth, nmax + 1, gt);
    double ceiling = std::nan("");
    if (s.mode == SABER_MODE_SABER) {
      fill_table(s.model, nmax + 1, mt);
      ceiling = mt[1];
    }
    WorkloadItem& it = items[static_cast<size_t>(k)];
    it.n = n;
    it.seed_idx = k;
    it.mix = k;
    it.rps = s.rps;
    it.jitter = s.length_jitter;
    it.ceiling = ceiling;
    it.prefill_rate = s.prefill_rate;
    double last_bound = 0.0, max_sla = 12.0;
    if (s.requests) {
      it.kind = 1;
      any_replay = true;
      max_sla = 0.0;
      for (int i = 0; i < n; ++i) {
        const saber_request& q = s.requests[i];
        const size_t o = static_cast<size_t>(k) * nmax + i;
        arr[o] = q.arrival_time;
        dl[o] = q.deadline;
        sla[o] = q.sla_seconds;
        mo[o] = static_cast<double>(q.max_output_tokens);
        in[o] = static_cast<double>(q.input_tokens);
        task[o] = static_cast<int8_t>(q.task >= 0 && q.task < 4 ? q.task : -1);
        group[o] = q.group < 0 ? 0 : q.group;
        max_sla = std::max(max_sla, q.sla_seconds);
      }
      last_bound = s.requests[n - 1].arrival_time;
    } else {
      it.kind = 0;
      double nls = 0.0;
      seed_draws(s.workload_seed, n, &base[static_cast<size_t>(k) * nmax * 4], &nls);
      mix_thresholds(s.mix, &th[static_cast<size_t>(k) * 4], &tt[static_cast<size_t>(k) * 4],
                     &tlast[static_cast<size_t>(k)]);
      last_bound = nls / s.rps * (1.0 + 1e-9) + n * 1e-6;
    }
    TrajDesc& d = descs[static_cast<size_t>(k)];
    d.workload = k;
    d.n = n;
    d.mode = s.mode;
    d.cap = s.static_batch_size;
    d.window = s.window_size;
    d.gt_tab = k * 2 * tl;
    d.model_tab = s.mode == SABER_MODE_SABER ? k * 2 * tl + tl : -1;
    d.tick = s.tick;
    d.horizon = s.has_horizon ? s.horizon : std::nan("");
    d.prefill_rate = s.prefill_rate;
    d.row = k;
    d.stream = -1;
    const double hb = s.has_horizon ? s.horizon : last_bound + 10.0 * max_sla + 1.0;
    tick_hb.emplace_back(s.tick, hb);
    if (s.mode == SABER_MODE_SABER) {
      d.stream = static_cast<int32_t>(seeds.size());
      seeds.push_back(s.seed ^ kSchedulerSeedSalt);
      // Streams start at min(bound, cap) draws and grow x8 (up to the
      // provable bound) for the trajectories that exhaust them, the batch then
      // rerunning — as the sweep plans do.  Long horizons
      // with wide windows bound at 10^8+ draws; a few thousand are used.
      const int64_t full = draw_bound(hb, s.tick, s.window_size, n);
      stream_full.push_back(full);
      stream_traj.push_back(k);
      len.push_back(std::min<int64_t>(full, kBatchDrawCap));
    }
  }
  auto layout_streams = [&]() {
    off.assign(len.size(), 0);
    total_draws = 0;
    for (size_t q = 0; q < len.size(); ++q) {
      off[q] = total_draws;
      total_draws += len[q];
    }
  };
  layout_streams();

  Workloads wl;
  DevBuf tables, seeds_d, off_d, len_d, draws_d, descs_d, rows_d, comp_d, admit_d, demo_d, cursor_d,
      err_d, trace_d, tcount_d, gen_d, group_d, req_d, state_d, cdfl_d, cdff_d, gi_d, gm_d;
  Scratch scratch;
  if (saber_status s = wl.alloc(dev, T, nmax)) return s;
  ALLOC_TRY(wl.items, dev, items.size() * sizeof(WorkloadItem));
  ALLOC_TRY(wl.seed_base, dev, base.size() * 8);
  ALLOC_TRY(wl.th, dev, th.size() * 8);
  ALLOC_TRY(wl.tt, dev, tt.size());
  ALLOC_TRY(wl.tl, dev, tlast.size());
  ALLOC_TRY(tables, dev, tab.size() * 8);
  ALLOC_TRY(descs_d, dev, descs.size() * sizeof(TrajDesc));
  ALLOC_TRY(rows_d, dev, static_cast<size_t>(T) * sizeof(saber_traj_row));
  ALLOC_TRY(comp_d, dev, cells * 8);
  ALLOC_TRY(cursor_d, dev, 16);
  ALLOC_TRY(err_d, dev, 16);
  const bool records = out->admit_times || out->demoted || want_states;
  if (records) {
    ALLOC_TRY(admit_d, dev, cells * 8);
    ALLOC_TRY(demo_d, dev, cells);
  }
  const int max_groups = out->group_issued ? out->max_groups : 0;
  if (want_states) {
    ALLOC_TRY(gen_d, dev, cells * 8);
    ALLOC_TRY(state_d, dev, cells * sizeof(saber_request_state));
    if (any_replay) ALLOC_TRY(group_d, dev, cells * 4);
    if (out->cdf_latency) {
      ALLOC_TRY(cdfl_d, dev, cells * 8);
      ALLOC_TRY(cdff_d, dev, cells * 8);
    }
    if (max_groups > 0) {
      ALLOC_TRY(gi_d, dev, static_cast<size_t>(T) * max_groups * 4);
      ALLOC_TRY(gm_d, dev, static_cast<size_t>(T) * max_groups * 4);
    }
  }
  if (out->requests) ALLOC_TRY(req_d, dev, cells * sizeof(saber_request));
  const bool trace = out->decisions != nullptr;
  if (trace) {
    if (out->decision_cap < 1 || !out->n_decisions)
      return fail(SABER_EINVAL, "run_batch: decision trace needs decision_cap and n_decisions");
    ALLOC_TRY(trace_d, dev, static_cast<size_t>(T) * out->decision_cap * sizeof(saber_decision));
    ALLOC_TRY(tcount_d, dev, static_cast<size_t>(T) * 8);
  }
  if (!seeds.empty()) {
    ALLOC_TRY(seeds_d, dev, seeds.size() * 8);
    ALLOC_TRY(off_d, dev, off.size() * 8);
    ALLOC_TRY(len_d, dev, len.size() * 8);
    ALLOC_TRY(draws_d, dev, static_cast<size_t>(std::max<int64_t>(1, total_draws)) * (wide ? 8 : 4));
  }
  if (saber_status s = scratch.alloc(dev, nmax, wide)) return s;
  // One tick table, for the most common tick of the batch.
  TickTableBuf ticktab;
  {
    std::map<double, std::pair<int, double>> by_tick;
    for (const auto& th_ : tick_hb) {
      auto& e = by_tick[th_.first];
      e.first += 1;
      e.second = std::max(e.second, th_.second);
    }
    double best_tick = 0.0, best_hb = 0.0;
    int best_n = 0;
    for (const auto& e : by_tick)
      if (e.second.first > best_n) {
        best_n = e.second.first;
        best_tick = e.first;
        best_hb = e.second.second;
      }
    if (best_n > 0)
      if (saber_status s = ticktab.build(dev, best_tick, best_hb)) return s;
    if (ticktab.view.len > 0) {
      ALLOC_TRY(wl.ka, dev, cells * 4);
      ALLOC_TRY(wl.kd, dev, cells * 4);
    }
  }

  CUDA_TRY(cudaMemcpy(wl.items.p, items.data(), items.size() * sizeof(WorkloadItem), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.seed_base.p, base.data(), base.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.th.p, th.data(), th.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.tt.p, tt.data(), tt.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.tl.p, tlast.data(), tlast.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.arr.p, arr.data(), cells * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.dl.p, dl.data(), cells * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.sla.p, sla.data(), cells * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.mo.p, mo.data(), cells * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.in.p, in.data(), cells * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(wl.task.p, task.data(), cells, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(tables.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(descs_d.p, descs.data(), descs.size() * sizeof(TrajDesc), cudaMemcpyHostToDevice));
  if (group_d.p) CUDA_TRY(cudaMemcpy(group_d.p, group.data(), cells * 4, cudaMemcpyHostToDevice));
  if (!seeds.empty()) {
    CUDA_TRY(cudaMemcpy(seeds_d.p, seeds.data(), seeds.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(off_d.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(len_d.p, len.data(), len.size() * 8, cudaMemcpyHostToDevice));
  }

  Timer tm;
  if (saber_status s = tm.init()) return s;
  cudaStream_t st = nullptr;
  SyncOnExit sync_guard(&st);
  int launches = 0;
  int32_t err = 0;
  float ms = 0.f;
  for (;;) {  // reruns only after a draw stream grew
  launches = 0;
  CUDA_TRY(cudaEventRecord(tm.a, st));
  CUDA_TRY(cudaMemsetAsync(rows_d.p, 0, rows_d.bytes, st));
  CUDA_TRY(cudaMemsetAsync(cursor_d.p, 0, 16, st));
  CUDA_TRY(cudaMemsetAsync(err_d.p, 0, 16, st));
  LAUNCH_TRY(launch_fill_rows(comp_d.as<double>(), T, nmax, 0, 1, st));
  ++launches;
  if (records) {
    LAUNCH_TRY(launch_fill_rows(admit_d.as<double>(), T, nmax, 0, 1, st));
    ++launches;
    CUDA_TRY(cudaMemsetAsync(demo_d.p, 0, cells, st));
  }
  if (gen_d.p) CUDA_TRY(cudaMemsetAsync(gen_d.p, 0, cells * 8, st));
  if (req_d.p) CUDA_TRY(cudaMemsetAsync(req_d.p, 0, cells * sizeof(saber_request), st));
  WorkloadParams wp{};
  wp.items = wl.items.as<WorkloadItem>();
  wp.n_items = T;
  wp.seed_base = wl.seed_base.as<double>();
  wp.seed_stride = nmax;
  wp.mix_thresh = wl.th.as<double>();
  wp.mix_task = wl.tt.as<int8_t>();
  wp.mix_last = wl.tl.as<int8_t>();
  wp.arrival = wl.arr.as<double>();
  wp.deadline = wl.dl.as<double>();
  wp.sla = wl.sla.as<double>();
  wp.max_out = wl.mo.as<double>();
  wp.input = wl.in.as<double>();
  wp.prefill = wl.pf.as<double>();
  wp.demote_after = wl.dem.as<double>();
  wp.horizon = wl.hor.as<double>();
  wp.task = wl.task.as<int8_t>();
  wp.nmax = nmax;
  LAUNCH_TRY(launch_workloads(wp, st));
  ++launches;
  if (wl.ka.p) {
    LAUNCH_TRY(launch_tick_index(wl.view(nmax), static_cast<int64_t>(cells), ticktab.view,
                                 wl.ka.as<int32_t>(), wl.kd.as<int32_t>(), st));
    ++launches;
  }
  if (!seeds.empty()) {
    RngGenParams rg{};
    rg.seeds = seeds_d.as<uint64_t>();
    rg.draws = draws_d.as<uint32_t>();
    rg.wide = wide;
    rg.off = off_d.as<int64_t>();
    rg.len = len_d.as<int64_t>();
    rg.n_streams = static_cast<int32_t>(seeds.size());
    LAUNCH_TRY(launch_rng_streams(rg, st));
    ++launches;
  }
  SimParams sp{};
  sp.traj = descs_d.as<TrajDesc>();
  sp.n_traj = T;
  sp.wl = wl.view(nmax);
  sp.tables = tables.as<double>();
  sp.rng.draws = draws_d.as<uint32_t>();
  sp.rng.wide = wide;
  sp.rng.off = off_d.as<int64_t>();
  sp.rng.len = len_d.as<int64_t>();
  sp.scratch = scratch.view;
  sp.slot_rows = scratch.launch.slot_rows;
  sp.out.rows = rows_d.as<saber_traj_row>();
  sp.out.completion = comp_d.as<double>();
  sp.out.admit = records ? admit_d.as<double>() : nullptr;
  sp.out.demoted = records ? demo_d.as<uint8_t>() : nullptr;
  sp.out.generated = gen_d.p ? gen_d.as<double>() : nullptr;
  sp.out.trace = trace ? trace_d.as<saber_decision>() : nullptr;
  sp.out.trace_count = trace ? tcount_d.as<int64_t>() : nullptr;
  sp.out.trace_cap = trace ? out->decision_cap : 0;
  sp.out.error = err_d.as<int32_t>();
  sp.next_traj = cursor_d.as<int32_t>();
  sp.ticks = ticktab.view;
  {
    bool any_saber = false, any_static = false;
    for (const TrajDesc& dd : descs) (dd.mode == SABER_MODE_SABER ? any_saber : any_static) = true;
    if (any_saber != any_static) sp.mode_sel = any_saber ? 2 : 1;
  }
  LAUNCH_TRY(launch_sim(sp, scratch.launch, st));
  ++launches;
  RowMetricsParams rm{};
  rm.rows = rows_d.as<saber_traj_row>();
  rm.completion = comp_d.as<double>();
  rm.wl = sp.wl;
  rm.traj = sp.traj;
  rm.n_traj = T;
  LAUNCH_TRY(launch_row_metrics(rm, st));
  ++launches;
  if (want_states || req_d.p) {
    RecordsParams rp{};
    rp.traj = sp.traj;
    rp.n_traj = T;
    rp.wl = sp.wl;
    rp.group = group_d.p ? group_d.as<int32_t>() : nullptr;
    rp.completion = comp_d.as<double>();
    rp.admit = admit_d.as<double>();
    rp.demoted = demo_d.as<uint8_t>();
    rp.generated = gen_d.as<double>();
    rp.requests = req_d.p ? req_d.as<saber_request>() : nullptr;
    rp.states = state_d.p ? state_d.as<saber_request_state>() : nullptr;
    rp.cdf_latency = cdfl_d.p ? cdfl_d.as<double>() : nullptr;
    rp.cdf_fraction = cdff_d.p ? cdff_d.as<double>() : nullptr;
    rp.group_issued = gi_d.p ? gi_d.as<int32_t>() : nullptr;
    rp.group_met = gm_d.p ? gm_d.as<int32_t>() : nullptr;
    rp.max_groups = max_groups;
    if (rp.requests) {
      LAUNCH_TRY(launch_pack_requests(rp, st));
      ++launches;
    }
    if (rp.states) {
      LAUNCH_TRY(launch_records(rp, st));
      ++launches;
    }
  }
  CUDA_TRY(cudaEventRecord(tm.b, st));
  CUDA_TRY(cudaEventSynchronize(tm.b));
  CUDA_TRY(cudaEventElapsedTime(&ms, tm.a, tm.b));
  CUDA_TRY(cudaMemcpy(&err, err_d.p, 4, cudaMemcpyDeviceToHost));
  if (err != kErrRngExhausted) break;
  // grow the streams the failed trajectories ran out of, then rerun
  std::vector<saber_traj_row> rr(static_cast<size_t>(T));
  CUDA_TRY(cudaMemcpy(rr.data(), rows_d.p, rr.size() * sizeof(saber_traj_row), cudaMemcpyDeviceToHost));
  bool grew = false;
  for (size_t q = 0; q < len.size(); ++q) {
    const int k = stream_traj[q];
    const int64_t need_more = static_cast<int64_t>(desc->specs[k].window_size) - 1;
    if (rr[static_cast<size_t>(k)].rng_draws + need_more > len[q] && len[q] < stream_full[q]) {
      len[q] = std::min<int64_t>(stream_full[q], len[q] * 8);
      grew = true;
    }
  }
  if (!grew) break;  // a genuine bound violation: reported below
  layout_streams();
  ALLOC_TRY(draws_d, dev, static_cast<size_t>(std::max<int64_t>(1, total_draws)) * (wide ? 8 : 4));
  CUDA_TRY(cudaMemcpy(off_d.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(len_d.p, len.data(), len.size() * 8, cudaMemcpyHostToDevice));
  }

  CUDA_TRY(cudaMemcpy(out->rows, rows_d.p, static_cast<size_t>(T) * sizeof(saber_traj_row),
                      cudaMemcpyDeviceToHost));
  // [T][nmax] device rows -> the caller's [T][max_n] rows
  auto copy_rows = [&](void* dst, const DevBuf& src, size_t elem) -> saber_status {
    if (!dst) return SABER_OK;
    CUDA_TRY(cudaMemcpy2D(dst, static_cast<size_t>(out->max_n) * elem, src.p,
                          static_cast<size_t>(nmax) * elem, static_cast<size_t>(nmax) * elem,
                          static_cast<size_t>(T), cudaMemcpyDeviceToHost));
    return SABER_OK;
  };
  if (saber_status s = copy_rows(out->completion_times, comp_d, 8)) return s;
  if (saber_status s = copy_rows(out->arrival_times, wl.arr, 8)) return s;
  if (records) {
    if (saber_status s = copy_rows(out->admit_times, admit_d, 8)) return s;
    if (saber_status s = copy_rows(out->demoted, demo_d, 1)) return s;
  }
  if (saber_status s = copy_rows(out->requests, req_d, sizeof(saber_request))) return s;
  if (saber_status s = copy_rows(out->states, state_d, sizeof(saber_request_state))) return s;
  if (saber_status s = copy_rows(out->cdf_latency, cdfl_d, 8)) return s;
  if (saber_status s = copy_rows(out->cdf_fraction, cdff_d, 8)) return s;
  if (max_groups > 0) {
    CUDA_TRY(cudaMemcpy(out->group_issued, gi_d.p, static_cast<size_t>(T) * max_groups * 4,
                        cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(out->group_met, gm_d.p, static_cast<size_t>(T) * max_groups * 4,
                        cudaMemcpyDeviceToHost));
  }
  if (trace) {
    CUDA_TRY(cudaMemcpy(out->n_decisions, tcount_d.p, static_cast<size_t>(T) * 8, cudaMemcpyDeviceToHost));
    // only the records each trajectory wrote
    for (int k = 0; k < T; ++k) {
      const int64_t nk = std::min(out->n_decisions[k], out->decision_cap);
      if (nk > 0)
        CUDA_TRY(cudaMemcpy(out->decisions + static_cast<size_t>(k) * out->decision_cap,
                            trace_d.as<saber_decision>() + static_cast<size_t>(k) * out->decision_cap,
                            static_cast<size_t>(nk) * sizeof(saber_decision), cudaMemcpyDeviceToHost));
    }
  }
  out->device_ms = ms;
  out->kernel_launches = launches;
  if (err == kErrTraceOverflow) return fail(SABER_ECAPACITY, "decision trace capacity exceeded");
  if (err == kErrRngExhausted)
    return fail(SABER_EINTERNAL, "scheduler RNG stream exhausted (draw bound violated)");
  if (err != 0) return fail(SABER_EINTERNAL, "trajectory kernel error " + std::to_string(err));
  return SABER_OK;
}

// generate() (workload.cpp:52-79) for many specs: the host draws (mt19937_64,
// glibc log: SURVEY F1/F5) and the device expansion the trajectory engine uses
// (workloads_kernel), packed as saber_request rows.
extern "C" saber_status saber_cuda_generate(const saber_workload_spec* specs, int32_t n_specs,
                                            int32_t device, saber_request* out, int32_t max_n) {
  if (!specs || !out || n_specs < 1) return fail(SABER_EINVAL, "generate: no specs");
  int nmax = 1;
  for (int k = 0; k < n_specs; ++k) {  // validate(WorkloadSpec) (workload.cpp:41-48)
    const saber_workload_spec& w = specs[k];
    if (!(w.rps > 0.0)) return fail(SABER_EINVAL, "rps must be > 0");
    if (w.num_requests < 1) return fail(SABER_EINVAL, "num_requests must be >= 1");
    if (w.length_jitter < 0.0 || w.length_jitter >= 1.0)
      return fail(SABER_EINVAL, "length_jitter must be in [0, 1)");
    if (saber_status e = validate_mix(w.mix)) return e;
    nmax = std::max(nmax, w.num_requests);
  }
  if (max_n < nmax) return fail(SABER_EINVAL, "generate: max_n smaller than num_requests");
  if (saber_status s = use_device(device)) return s;
  const int dev = device;
  const int T = n_specs;
  const size_t cells = static_cast<size_t>(T) * nmax;
  std::vector<WorkloadItem> items(static_cast<size_t>(T));
  std::vector<double> base(cells * 4, 0.0), th(static_cast<size_t>(T) * 4);
  std::vector<int8_t> tt(static_cast<size_t>(T) * 4), tlast(static_cast<size_t>(T));
  std::vector<TrajDesc> descs(static_cast<size_t>(T));
  for (int k = 0; k < T; ++k) {
    const saber_workload_spec& w = specs[k];
    double nls = 0.0;
    seed_draws(w.seed, w.num_requests, &base[static_cast<size_t>(k) * nmax * 4], &nls);
    mix_thresholds(w.mix, &th[static_cast<size_t>(k) * 4], &tt[static_cast<size_t>(k) * 4],
                   &tlast[static_cast<size_t>(k)]);
    WorkloadItem& it = items[static_cast<size_t>(k)];
    it.kind = 0;
    it.n = w.num_requests;
    it.seed_idx = k;
    it.mix = k;
    it.rps = w.rps;
    it.jitter = w.length_jitter;
    it.ceiling = std::nan("");
    it.prefill_rate = 0.0;
    TrajDesc& d = descs[static_cast<size_t>(k)];
    d = TrajDesc{};
    d.workload = k;
    d.n = w.num_requests;
    d.row = k;
  }
  Workloads wl;
  DevBuf descs_d, req_d;
  if (saber_status s = wl.alloc(dev, T, nmax)) return s;
  ALLOC_TRY(wl.items, dev, items.size() * sizeof(WorkloadItem));
  ALLOC_TRY(wl.seed_base, dev, base.size() * 8);
  ALLOC_TRY(wl.th, dev, th.size() * 8);
  ALLOC_TRY(wl.tt, dev, tt.size());
  ALLOC_TRY(wl.tl, dev, tlast.size());
  ALLOC_TRY(descs_d, dev, descs.size() * sizeof(TrajDesc));
  ALLOC_TRY(req_d, dev, cells * sizeof(saber_request));
  cudaStream_t st = nullptr;
  SyncOnExit sync_guard(&st);
  CUDA_TRY(cudaMemcpyAsync(wl.items.p, items.data(), items.size() * sizeof(WorkloadItem),
                           cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(wl.seed_base.p, base.data(), base.size() * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(wl.th.p, th.data(), th.size() * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(wl.tt.p, tt.data(), tt.size(), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(wl.tl.p, tlast.data(), tlast.size(), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(descs_d.p, descs.data(), descs.size() * sizeof(TrajDesc),
                           cudaMemcpyHostToDevice, st));
  WorkloadParams wp{};
  wp.items = wl.items.as<WorkloadItem>();
  wp.n_items = T;
  wp.seed_base = wl.seed_base.as<double>();
  wp.seed_stride = nmax;
  wp.mix_thresh = wl.th.as<double>();
  wp.mix_task = wl.tt.as<int8_t>();
  wp.mix_last = wl.tl.as<int8_t>();
  wp.arrival = wl.arr.as<double>();
  wp.deadline = wl.dl.as<double>();
  wp.sla = wl.sla.as<double>();
  wp.max_out = wl.mo.as<double>();
  wp.input = wl.in.as<double>();
  wp.prefill = wl.pf.as<double>();
  wp.demote_after = wl.dem.as<double>();
  wp.horizon = wl.hor.as<double>();
  wp.task = wl.task.as<int8_t>();
  wp.nmax = nmax;
  CUDA_TRY(cudaMemsetAsync(req_d.p, 0, cells * sizeof(saber_request), st));
  LAUNCH_TRY(launch_workloads(wp, st));
  RecordsParams rp{};
  rp.traj = descs_d.as<TrajDesc>();
  rp.n_traj = T;
  rp.wl = wl.view(nmax);
  rp.requests = req_d.as<saber_request>();
  LAUNCH_TRY(launch_pack_requests(rp, st));
  CUDA_TRY(cudaMemcpy2DAsync(out, static_cast<size_t>(max_n) * sizeof(saber_request), req_d.p,
                             static_cast<size_t>(nmax) * sizeof(saber_request),
                             static_cast<size_t>(nmax) * sizeof(saber_request), static_cast<size_t>(T),
                             cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return SABER_OK;
}

extern "C" saber_status saber_cuda_fp64_peak(int32_t device, double* tflops) {
  if (!tflops) return fail(SABER_EINVAL, "null argument");
  if (saber_status s = use_device(device)) return s;
  if (fp64_peak(device, tflops) != 0) return fail(SABER_ECUDA, "fp64 microbenchmark failed");
  return SABER_OK;
}

extern "C" saber_status saber_cuda_fit_batch(const saber_fit_desc* desc, saber_fit_out* out) {
  if (!desc || !out) return fail(SABER_EINVAL, "null argument");
  const int N = desc->n_curves;
  if (N < 1) return fail(SABER_EINVAL, "fit_batch: no curves");
  if (!desc->loads || !desc->speeds || !desc->offsets)
    return fail(SABER_EINVAL, "fit_batch: loads, speeds and offsets are required");
  if (!out->params || !out->r2 || !out->status)
    return fail(SABER_EINVAL, "fit_batch: params, r2 and status outputs are required");
  if (desc->calibrate && !out->best_family)
    return fail(SABER_EINVAL, "fit_batch: calibrate needs best_family");
  int mask = desc->family_mask & 7;
  if (desc->calibrate) mask = 7;  // calibrate() fits all three families
  if (mask == 0) return fail(SABER_EINVAL, "fit_batch: empty family mask");
  if (desc->offsets[0] != 0) return fail(SABER_EINVAL, "fit_batch: offsets[0] must be 0");
  for (int c = 0; c < N; ++c)
    if (desc->offsets[c + 1] < desc->offsets[c])
      return fail(SABER_EINVAL, "fit_batch: offsets must be non-decreasing");
  const int64_t M = desc->offsets[N];
  for (int64_t i = 0; i < M; ++i)
    if (desc->loads[i] < 1) return fail(SABER_EDOMAIN, "predict: load must be >= 1");
  if (saber_status s = use_device(desc->device)) return s;
  const int dev = desc->device;
  DevBuf loads, speeds, offs, scratch, conv, iters, trs, params, r2, status, best, itc, trc, cursor;
  ALLOC_TRY(loads, dev, static_cast<size_t>(std::max<int64_t>(1, M)) * 4);
  ALLOC_TRY(speeds, dev, static_cast<size_t>(std::max<int64_t>(1, M)) * 8);
  ALLOC_TRY(offs, dev, static_cast<size_t>(N + 1) * 8);
  ALLOC_TRY(scratch, dev, static_cast<size_t>(2) * N * 5 * 4 * 8);
  ALLOC_TRY(conv, dev, static_cast<size_t>(2) * N * 5 * 4);
  ALLOC_TRY(iters, dev, static_cast<size_t>(2) * N * 5 * 4);
  ALLOC_TRY(trs, dev, static_cast<size_t>(2) * N * 5 * 4);
  ALLOC_TRY(params, dev, static_cast<size_t>(3) * N * 3 * 8);
  ALLOC_TRY(r2, dev, static_cast<size_t>(3) * N * 8);
  ALLOC_TRY(status, dev, static_cast<size_t>(3) * N * 4);
  ALLOC_TRY(best, dev, static_cast<size_t>(N) * 4);
  ALLOC_TRY(itc, dev, static_cast<size_t>(3) * N * 4);
  ALLOC_TRY(trc, dev, static_cast<size_t>(3) * N * 4);
  ALLOC_TRY(cursor, dev, 16);
  Timer tm;
  if (saber_status s = tm.init()) return s;
  cudaStream_t st = nullptr;
  SyncOnExit sync_guard(&st);
  CUDA_TRY(cudaEventRecord(tm.a, st));
  if (M > 0) {
    CUDA_TRY(cudaMemcpyAsync(loads.p, desc->loads, static_cast<size_t>(M) * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(speeds.p, desc->speeds, static_cast<size_t>(M) * 8, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaMemcpyAsync(offs.p, desc->offsets, static_cast<size_t>(N + 1) * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(cursor.p, 0, 16, st));
  FitParams fp{};
  fp.loads = loads.as<int32_t>();
  fp.speeds = speeds.as<double>();
  fp.offsets = offs.as<int64_t>();
  fp.n_curves = N;
  fp.family_mask = mask;
  fp.calibrate = desc->calibrate;
  fp.params = params.as<double>();
  fp.r2 = r2.as<double>();
  fp.status = status.as<int32_t>();
  fp.best_family = best.as<int32_t>();
  fp.iterations = itc.as<int32_t>();
  fp.lm_scratch = scratch.as<double>();
  fp.lm_conv = conv.as<int32_t>();
  fp.lm_iters = iters.as<int32_t>();
  fp.lm_trials = trs.as<int32_t>();
  fp.trials = trc.as<int32_t>();
  fp.cursor = cursor.as<int32_t>();
  {
    // Verification switch (tests/test_gpu_fit.py): the LM passes take the
    // IEEE-division, clamped-exponent path only, which the fast paths must
    // reproduce bit for bit.
    const char* e = std::getenv("SABER_LM_IEEE");
    fp.ieee_only = (e && e[0] == '1') ? 1 : 0;
  }
  int launches = 0;
  LAUNCH_TRY(launch_fit(fp, st, &launches));
  CUDA_TRY(cudaMemcpyAsync(out->params, params.p, static_cast<size_t>(3) * N * 3 * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->r2, r2.p, static_cast<size_t>(3) * N * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(out->status, status.p, static_cast<size_t>(3) * N * 4, cudaMemcpyDeviceToHost, st));
  if (desc->calibrate)
    CUDA_TRY(cudaMemcpyAsync(out->best_family, best.p, static_cast<size_t>(N) * 4, cudaMemcpyDeviceToHost, st));
  if (out->iterations)
    CUDA_TRY(cudaMemcpyAsync(out->iterations, itc.p, static_cast<size_t>(3) * N * 4, cudaMemcpyDeviceToHost, st));
  if (out->trials)
    CUDA_TRY(cudaMemcpyAsync(out->trials, trc.p, static_cast<size_t>(3) * N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaEventRecord(tm.b, st));
  CUDA_TRY(cudaEventSynchronize(tm.b));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, tm.a, tm.b));
  out->device_ms = ms;
  out->kernel_launches = launches;
  return SABER_OK;
}

// ===================================================== bursty Monte-Carlo ==
namespace {

saber_status validate_mc(const saber_mc_desc& d) {
  if (d.n_traj < 0) return fail(SABER_EINVAL, "mc: n_traj must be >= 0");
  if (d.n_mixes < 1 || d.n_rps < 1 || (d.n_caps < 1 && !d.with_saber))
    return fail(SABER_EINVAL, "mc: empty grid");
  if (d.with_saber && !d.has_model) return fail(SABER_EINVAL, "mc: saber variant requires a model");
  for (int i = 0; i < d.n_mixes; ++i)
    if (d.mixes[i] < 1 || d.mixes[i] > 3)
      return fail(SABER_EINVAL, "unknown mix preset: w" + std::to_string(d.mixes[i]));
  for (int i = 0; i < d.n_rps; ++i)
    if (!(d.rps[i] > 0.0)) return fail(SABER_EINVAL, "rps must be > 0");
  for (int i = 0; i < d.n_caps; ++i)
    if (d.caps[i] < 1) return fail(SABER_EINVAL, "static mode requires a positive batch size");
  if (d.num_requests < 1) return fail(SABER_EINVAL, "num_requests must be >= 1");
  if (d.num_requests > kMaxRequestsWide)
    return fail(SABER_EINVAL, "num_requests > " + std::to_string(kMaxRequestsWide) +
                                  " is not supported by the B200 engine");
  if (d.length_jitter < 0.0 || d.length_jitter >= 1.0)
    return fail(SABER_EINVAL, "length_jitter must be in [0, 1)");
  if (d.window_size < 1) return fail(SABER_EINVAL, "window_size must be >= 1");
  if (!(d.tick > 0.0)) return fail(SABER_EINVAL, "tick must be > 0");
  if (saber_status s = validate_model(d.ground_truth, "ground truth")) return s;
  if (d.has_model)
    if (saber_status s = validate_model(d.model, "model")) return s;
  if (!(eval_model(d.ground_truth, 1.0) > 0.0))
    return fail(SABER_EINVAL, "engine ground truth must be positive");
  if (!(d.burst_factor > 0.0) || !(d.mean_calm > 0.0) || !(d.mean_burst > 0.0))
    return fail(SABER_EINVAL, "mc: burst factor and holding-time means must be > 0");
  if (d.scheduler_seeds < 1) return fail(SABER_EINVAL, "mc: scheduler_seeds must be >= 1");
  if (d.shard_count < 1 || d.shard_index < 0 || d.shard_index >= d.shard_count)
    return fail(SABER_EINVAL, "bad shard index/count");
  return SABER_OK;
}

int64_t mc_cells(const saber_mc_desc& d) {
  return static_cast<int64_t>(d.n_mixes) * d.n_rps * (d.n_caps + (d.with_saber ? 1 : 0));
}

bursty::Params mc_params(const saber_mc_desc& d) {
  return bursty::Params{d.seed, d.burst_factor, d.mean_calm, d.mean_burst};
}

}  // namespace

extern "C" int64_t saber_cuda_mc_cells(const saber_mc_desc* d) { return d ? mc_cells(*d) : 0; }

extern "C" saber_status saber_cuda_mc_trace(const saber_mc_desc* desc, int64_t k,
                                            saber_request* requests, saber_traj_spec* spec) {
  if (!desc || !requests || !spec) return fail(SABER_EINVAL, "null argument");
  if (saber_status s = validate_mc(*desc)) return s;
  if (k < 0 || k >= desc->n_traj) return fail(SABER_EINVAL, "mc_trace: trajectory out of range");
  const int per_rps = desc->n_caps + (desc->with_saber ? 1 : 0);
  const int64_t cell = k % mc_cells(*desc);
  const int v = static_cast<int>(cell % per_rps);
  const int ri = static_cast<int>((cell / per_rps) % desc->n_rps);
  const int mi = static_cast<int>((cell / per_rps) / desc->n_rps);
  const saber_mix mix = preset(desc->mixes[mi]);
  double th[4];
  int8_t tt[4], tl;
  mix_thresholds(mix, th, tt, &tl);
  const bursty::Params bp = mc_params(*desc);
  bursty::Gen g;
  bursty::gen_init(g, bp, static_cast<uint64_t>(k));
  const double rps = desc->rps[ri];
  for (int q = 0; q < desc->num_requests; ++q) {
    const double arrival = bursty::gen_arrival(g, bp, rps);
    const double u = bursty::gen_uniform(g);
    int task = tl;  // sample_task (workload.cpp:28-39)
    for (int a = 0; a < 4; ++a)
      if (tt[a] >= 0 && u < th[a]) {
        task = tt[a];
        break;
      }
    auto jl = [&](int avg) {  // jittered_length (workload.cpp:21-26)
      const double lo = avg * (1.0 - desc->length_jitter);
      const double hi = avg * (1.0 + desc->length_jitter);
      return std::max(1, static_cast<int>(std::llround(lo + bursty::gen_uniform(g) * (hi - lo))));
    };
    saber_request& r = requests[q];
    r.arrival_time = arrival;
    r.input_tokens = jl(kAvgInH[task]);
    r.max_output_tokens = jl(kAvgOutH[task]);
    r.sla_seconds = kSlaH[task];
    r.deadline = arrival + kSlaH[task];
    r.task = task;
    r.group = kNameRankH[r.task >= 0 && r.task < 4 ? r.task : 0];
  }
  *spec = saber_traj_spec{};
  spec->mix = mix;
  spec->rps = rps;
  spec->num_requests = desc->num_requests;
  spec->length_jitter = desc->length_jitter;
  spec->requests = nullptr;
  const bool saber = desc->with_saber && v == desc->n_caps;
  spec->mode = saber ? SABER_MODE_SABER : SABER_MODE_STATIC;
  spec->window_size = desc->window_size;
  spec->tick = desc->tick;
  spec->static_batch_size = saber ? 0 : desc->caps[v];
  spec->has_model = saber ? 1 : 0;
  spec->model = desc->model;
  spec->ground_truth = desc->ground_truth;
  spec->prefill_rate = desc->prefill_rate;
  spec->has_horizon = 0;
  spec->seed = desc->scheduler_seed + static_cast<uint64_t>(k % desc->scheduler_seeds);
  return SABER_OK;
}

extern "C" saber_status saber_cuda_mc_sweep(const saber_mc_desc* desc, saber_mc_out* out) {
  if (!desc || !out) return fail(SABER_EINVAL, "null argument");
  if (saber_status s = validate_mc(*desc)) return s;
  if (!out->cell_stats) return fail(SABER_EINVAL, "mc: cell_stats output required");
  if (saber_status s = use_device(desc->device)) return s;
  const saber_mc_desc& d = *desc;
  const int dev = d.device, n = d.num_requests;
  const int64_t cells = mc_cells(d);
  const int64_t mine = d.n_traj > d.shard_index
                           ? (d.n_traj - d.shard_index + d.shard_count - 1) / d.shard_count
                           : 0;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(d.chunk > 0 ? d.chunk : 262144,
                                                               std::max<int64_t>(mine, 1)));
  // tables, mixes, caps, rps
  const int tl = n + 2;
  std::vector<double> tab(static_cast<size_t>(2 * tl));
  fill_table(d.ground_truth, n + 1, &tab[0]);
  double ceiling = std::nan("");
  if (d.has_model) {
    fill_table(d.model, n + 1, &tab[static_cast<size_t>(tl)]);
    ceiling = tab[static_cast<size_t>(tl) + 1];
  }
  std::vector<double> th(static_cast<size_t>(d.n_mixes) * 4);
  std::vector<int8_t> tt(static_cast<size_t>(d.n_mixes) * 4), tlast(static_cast<size_t>(d.n_mixes));
  for (int mi = 0; mi < d.n_mixes; ++mi)
    mix_thresholds(preset(d.mixes[mi]), &th[static_cast<size_t>(mi) * 4],
                   &tt[static_cast<size_t>(mi) * 4], &tlast[static_cast<size_t>(mi)]);
  DevBuf tables, rps_d, caps_d, th_d, tt_d, tl_d, hmax, seeds_d, off_d, len_d, draws_d, descs, rows,
      comp, cursor, err, stats, hist;
  Workloads wl;
  Scratch scratch;
  ALLOC_TRY(tables, dev, tab.size() * 8);
  ALLOC_TRY(rps_d, dev, static_cast<size_t>(d.n_rps) * 8);
  ALLOC_TRY(caps_d, dev, std::max<size_t>(1, static_cast<size_t>(d.n_caps)) * 4);
  ALLOC_TRY(th_d, dev, th.size() * 8);
  ALLOC_TRY(tt_d, dev, tt.size());
  ALLOC_TRY(tl_d, dev, tlast.size());
  ALLOC_TRY(hmax, dev, 16);
  ALLOC_TRY(stats, dev, static_cast<size_t>(cells) * SABER_MC_STATS * 8);
  ALLOC_TRY(hist, dev, static_cast<size_t>(cells) * (SABER_MC_BINS + 1) * 8);
  ALLOC_TRY(descs, dev, static_cast<size_t>(chunk) * sizeof(TrajDesc));
  ALLOC_TRY(rows, dev, static_cast<size_t>(chunk) * sizeof(saber_traj_row));
  ALLOC_TRY(comp, dev, static_cast<size_t>(chunk) * n * 8);
  ALLOC_TRY(cursor, dev, 16);
  ALLOC_TRY(err, dev, 16);
  if (saber_status s = wl.alloc(dev, chunk, n)) return s;
  const bool wide = needs_wide(n, d.with_saber ? d.window_size : 1);
  if (saber_status s = scratch.alloc(dev, n, wide)) return s;
  CUDA_TRY(cudaMemcpy(tables.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(rps_d.p, d.rps, static_cast<size_t>(d.n_rps) * 8, cudaMemcpyHostToDevice));
  if (d.n_caps > 0)
    CUDA_TRY(cudaMemcpy(caps_d.p, d.caps, static_cast<size_t>(d.n_caps) * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(th_d.p, th.data(), th.size() * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(tt_d.p, tt.data(), tt.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(tl_d.p, tlast.data(), tlast.size(), cudaMemcpyHostToDevice));

  McParams mp{};
  mp.n_mixes = d.n_mixes;
  mp.n_rps = d.n_rps;
  mp.n_caps = d.n_caps;
  mp.with_saber = d.with_saber;
  mp.n_cells = static_cast<int32_t>(cells);
  mp.rps = rps_d.as<double>();
  mp.caps = caps_d.as<int32_t>();
  mp.mix_thresh = th_d.as<double>();
  mp.mix_task = tt_d.as<int8_t>();
  mp.mix_last = tl_d.as<int8_t>();
  mp.n = n;
  mp.jitter = d.length_jitter;
  mp.ceiling = d.with_saber ? ceiling : std::nan("");
  mp.bp = mc_params(d);
  mp.shard_index = d.shard_index;
  mp.shard_count = d.shard_count;
  mp.sched_seeds = d.scheduler_seeds;
  mp.window = d.window_size;
  mp.tick = d.tick;
  mp.prefill_rate = d.prefill_rate;
  mp.model_tab = d.has_model ? tl : -1;
  mp.gt_tab = 0;
  mp.arrival = wl.arr.as<double>();
  mp.deadline = wl.dl.as<double>();
  mp.sla = wl.sla.as<double>();
  mp.max_out = wl.mo.as<double>();
  mp.input = wl.in.as<double>();
  mp.prefill = wl.pf.as<double>();
  mp.demote_after = wl.dem.as<double>();
  mp.horizon = wl.hor.as<double>();
  mp.task = wl.task.as<int8_t>();
  mp.descs = descs.as<TrajDesc>();

  Timer all, simt;
  if (saber_status s = all.init()) return s;
  if (saber_status s = simt.init()) return s;
  cudaStream_t st = nullptr;
  int launches = 0;
  float sim_ms_total = 0.f;
  CUDA_TRY(cudaEventRecord(all.a, st));
  CUDA_TRY(cudaMemsetAsync(stats.p, 0, stats.bytes, st));
  CUDA_TRY(cudaMemsetAsync(hist.p, 0, hist.bytes, st));
  CUDA_TRY(cudaMemsetAsync(err.p, 0, 16, st));
  // Scheduler RNG streams sized by the longest default horizon of this shard.
  int32_t pool = 0;
  double hm = 0.0;
  TickTableBuf ticktab;
  if (mine > 0) {
    CUDA_TRY(cudaMemsetAsync(hmax.p, 0, 16, st));
    LAUNCH_TRY(launch_mc_horizon(mp, mine, hmax.as<unsigned long long>(), st));
    ++launches;
    CUDA_TRY(cudaMemcpy(&hm, hmax.p, 8, cudaMemcpyDeviceToHost));
    if (saber_status s = ticktab.build(dev, d.tick, hm + 1.0)) return s;
    if (ticktab.view.len > 0) {
      ALLOC_TRY(wl.ka, dev, static_cast<size_t>(chunk) * n * 4);
      ALLOC_TRY(wl.kd, dev, static_cast<size_t>(chunk) * n * 4);
    }
  }
  if (d.with_saber && mine > 0) {
    pool = static_cast<int32_t>(std::min<int64_t>(d.scheduler_seeds, d.n_traj));
    const int64_t len = draw_bound(hm + 1.0, d.tick, d.window_size, n);
    std::vector<uint64_t> seeds(static_cast<size_t>(pool));
    std::vector<int64_t> off(static_cast<size_t>(pool)), lens(static_cast<size_t>(pool), len);
    for (int32_t s = 0; s < pool; ++s) {
      seeds[static_cast<size_t>(s)] = (d.scheduler_seed + static_cast<uint64_t>(s)) ^ kSchedulerSeedSalt;
      off[static_cast<size_t>(s)] = static_cast<int64_t>(s) * len;
    }
    ALLOC_TRY(seeds_d, dev, seeds.size() * 8);
    ALLOC_TRY(off_d, dev, off.size() * 8);
    ALLOC_TRY(len_d, dev, lens.size() * 8);
    ALLOC_TRY(draws_d, dev, static_cast<size_t>(std::max<int64_t>(1, len * pool)) * (wide ? 8 : 4));
    CUDA_TRY(cudaMemcpy(seeds_d.p, seeds.data(), seeds.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(off_d.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(len_d.p, lens.data(), lens.size() * 8, cudaMemcpyHostToDevice));
    RngGenParams rg{};
    rg.seeds = seeds_d.as<uint64_t>();
    rg.draws = draws_d.as<uint32_t>();
    rg.wide = wide;
    rg.off = off_d.as<int64_t>();
    rg.len = len_d.as<int64_t>();
    rg.n_streams = pool;
    LAUNCH_TRY(launch_rng_streams(rg, st));
    ++launches;
  }
  std::vector<saber_traj_row> host_rows;
  if (out->rows) host_rows.resize(static_cast<size_t>(chunk));
  // split launches (SABER-only + static-only kernels) need both classes
  const bool split_ok = d.with_saber && d.n_caps > 0 && scratch.launch.group == 32 &&
                        !scratch.launch.wide &&
                        std::getenv("SABER_NO_SPLIT") == nullptr;
  std::vector<int32_t> ord_h;
  DevBuf order_d;
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  struct StreamGuard {
    cudaStream_t* s;
    cudaEvent_t* a;
    cudaEvent_t* b;
    ~StreamGuard() {
      if (*s) cudaStreamDestroy(*s);
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
    }
  } sguard{&side, &fork_ev, &join_ev};
  SyncOnExit sync_guard(&st, &side);  // after every DevBuf and the side stream
  if (split_ok) {
    ord_h.resize(static_cast<size_t>(chunk));
    ALLOC_TRY(order_d, dev, static_cast<size_t>(chunk) * 4);
    CUDA_TRY(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming));
  }
  for (int64_t k0 = 0; k0 < mine; k0 += chunk) {
    mp.k0 = k0;
    mp.count = std::min<int64_t>(chunk, mine - k0);
    LAUNCH_TRY(launch_mc_workloads(mp, st));
    if (wl.ka.p)
      LAUNCH_TRY(launch_tick_index(wl.view(n), mp.count * n, ticktab.view, wl.ka.as<int32_t>(),
                                   wl.kd.as<int32_t>(), st));
    // SABER trajectories of the chunk first (their cell is k % cells, the
    // variant (k % cells) % (caps + 1), as mc.cu cell_of), run on the
    // SABER-only kernel while the static ones run on theirs.
    int32_t ns = 0;
    if (split_ok) {
      const int per_rps = d.n_caps + 1;
      int32_t lo = 0, hi = static_cast<int32_t>(mp.count);
      for (int64_t i = 0; i < mp.count; ++i) {
        const int64_t k = d.shard_index + (k0 + i) * d.shard_count;
        const bool sab = (k % cells) % per_rps == d.n_caps;
        if (sab) ord_h[static_cast<size_t>(lo++)] = static_cast<int32_t>(i);
        else ord_h[static_cast<size_t>(--hi)] = static_cast<int32_t>(i);
      }
      ns = lo;
      CUDA_TRY(cudaMemcpyAsync(order_d.p, ord_h.data(), static_cast<size_t>(mp.count) * 4,
                               cudaMemcpyHostToDevice, st));
    }    CUDA_TRY(cudaMemsetAsync(rows.p, 0, static_cast<size_t>(mp.count) * sizeof(saber_traj_row), st));
    CUDA_TRY(cudaMemsetAsync(cursor.p, 0, 16, st));
    LAUNCH_TRY(launch_fill_rows(comp.as<double>(), mp.count, n, 0, 1, st));
    SimParams sp{};
    sp.traj = descs.as<TrajDesc>();
    sp.n_traj = static_cast<int32_t>(mp.count);
    sp.wl = wl.view(n);
    sp.tables = tables.as<double>();
    sp.rng.draws = draws_d.as<uint32_t>();
    sp.rng.wide = wide;
    sp.rng.off = off_d.as<int64_t>();
    sp.rng.len = len_d.as<int64_t>();
    sp.scratch = scratch.view;
    sp.slot_rows = scratch.launch.slot_rows;
    sp.out.rows = rows.as<saber_traj_row>();
    sp.out.completion = comp.as<double>();
    sp.out.error = err.as<int32_t>();
    sp.next_traj = cursor.as<int32_t>();
    sp.ticks = ticktab.view;
    CUDA_TRY(cudaEventRecord(simt.a, st));
    if (split_ok && ns > 0 && ns < mp.count) {
      SimParams sa = sp, sb = sp;
      sa.order = sb.order = order_d.as<int32_t>();
      sa.mode_sel = 2;  // (full SABER grid: the trimmed one measured 2% slower on config 5)
      sa.n_traj = ns;
      sb.mode_sel = 1;
      sb.first_traj = ns;
      sb.next_traj = cursor.as<int32_t>() + 1;
      CUDA_TRY(cudaEventRecord(fork_ev, st));
      CUDA_TRY(cudaStreamWaitEvent(side, fork_ev, 0));
      LAUNCH_TRY(launch_sim(sa, scratch.launch, st));
      LAUNCH_TRY(launch_sim(sb, scratch.launch, side));
      CUDA_TRY(cudaEventRecord(join_ev, side));
      CUDA_TRY(cudaStreamWaitEvent(st, join_ev, 0));
      launches += 1;
    } else {
      LAUNCH_TRY(launch_sim(sp, scratch.launch, st));
    }
    CUDA_TRY(cudaEventRecord(simt.b, st));
    RowMetricsParams rm{};
    rm.rows = rows.as<saber_traj_row>();
    rm.completion = comp.as<double>();
    rm.wl = sp.wl;
    rm.traj = sp.traj;
    rm.n_traj = sp.n_traj;
    LAUNCH_TRY(launch_row_metrics(rm, st));
    LAUNCH_TRY(launch_mc_reduce(mp, rows.as<saber_traj_row>(), comp.as<double>(), stats.as<int64_t>(),
                                out->cell_hist ? hist.as<int64_t>() : nullptr, st));
    launches += 5;
    CUDA_TRY(cudaEventSynchronize(simt.b));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, simt.a, simt.b));
    sim_ms_total += ms;
    if (out->rows) {
      CUDA_TRY(cudaMemcpy(host_rows.data(), rows.p, static_cast<size_t>(mp.count) * sizeof(saber_traj_row),
                          cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < mp.count; ++i)
        out->rows[d.shard_index + (k0 + i) * d.shard_count] = host_rows[static_cast<size_t>(i)];
    }
  }
  CUDA_TRY(cudaEventRecord(all.b, st));
  CUDA_TRY(cudaEventSynchronize(all.b));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, all.a, all.b));
  std::vector<int64_t> hs(static_cast<size_t>(cells) * SABER_MC_STATS);
  CUDA_TRY(cudaMemcpy(hs.data(), stats.p, hs.size() * 8, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < hs.size(); ++i) out->cell_stats[i] += hs[i];
  if (out->cell_hist) {
    std::vector<int64_t> hh(static_cast<size_t>(cells) * (SABER_MC_BINS + 1));
    CUDA_TRY(cudaMemcpy(hh.data(), hist.p, hh.size() * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < hh.size(); ++i) out->cell_hist[i] += hh[i];
  }
  out->device_ms = ms;
  out->sim_kernel_ms = sim_ms_total;
  out->kernel_launches = launches;
  int32_t e = 0;
  CUDA_TRY(cudaMemcpy(&e, err.p, 4, cudaMemcpyDeviceToHost));
  if (e == kErrRngExhausted)
    return fail(SABER_EINTERNAL, "scheduler RNG stream exhausted (draw bound violated)");
  if (e != 0) return fail(SABER_EINTERNAL, "trajectory kernel error " + std::to_string(e));
  return SABER_OK;
}

// ================================================================ profile ==
namespace {

struct BurstPlan {
  std::vector<int32_t> size;
  std::vector<double> in, out;
  int64_t issued = 0;
};

// The burst schedule of profile() (calibration.cpp:72-96): sizes cycle
// 1..l_max; each burst draws one task, one input and one output length.
saber_status plan_bursts(const saber_profile_spec& s, BurstPlan* plan) {
  if (s.l_max < 1) return fail(SABER_EINVAL, "profile: l_max must be >= 1");
  if (saber_status e = validate_mix(s.mix)) return e;
  if (s.num_requests < 1) return fail(SABER_EINVAL, "profile: target sample count must be >= 1");
  if (s.length_jitter < 0.0 || s.length_jitter >= 1.0)
    return fail(SABER_EINVAL, "length_jitter must be in [0, 1)");
  if (saber_status e = validate_model(s.ground_truth, "ground truth")) return e;
  if (!(eval_model(s.ground_truth, 1.0) > 0.0))
    return fail(SABER_EINVAL, "engine ground truth must be positive");
  double th[4];
  int8_t tt[4], tl;
  mix_thresholds(s.mix, th, tt, &tl);
  std::mt19937_64 rng(s.seed);
  auto u01 = [&]() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
  auto jl = [&](int avg) {
    const double lo = avg * (1.0 - s.length_jitter);
    const double hi = avg * (1.0 + s.length_jitter);
    return std::max(1, static_cast<int>(std::llround(lo + u01() * (hi - lo))));
  };
  int size = 0;
  plan->issued = 0;
  while (plan->issued < s.num_requests) {
    size = size % s.l_max + 1;
    const double u = u01();
    int task = tl;
    for (int a = 0; a < 4; ++a)
      if (tt[a] >= 0 && u < th[a]) {
        task = tt[a];
        break;
      }
    const int in = jl(kAvgInH[task]);
    const int outl = jl(kAvgOutH[task]);
    plan->size.push_back(size);
    plan->in.push_back(static_cast<double>(in));
    plan->out.push_back(static_cast<double>(outl));
    plan->issued += size;
  }
  return SABER_OK;
}

}  // namespace

extern "C" int64_t saber_cuda_profile_samples(const saber_profile_spec* spec) {
  if (!spec) return -1;
  BurstPlan plan;
  if (plan_bursts(*spec, &plan) != SABER_OK) return -1;
  return plan.issued;
}

// calibration.cpp:45-56: bursts cycle through sizes 1..l_max until the
// budget is issued; the distinct loads are the distinct sizes reached.
extern "C" int32_t saber_cuda_profile_planned_loads(int32_t num_requests, int32_t l_max) {
  if (l_max < 1 || num_requests < 1) return 0;
  int64_t issued = 0, bursts = 0;
  for (int32_t size = 0; issued < num_requests && bursts < l_max; ++bursts) {
    size = size % l_max + 1;
    issued += size;
  }
  return static_cast<int32_t>(bursts);
}

extern "C" saber_status saber_cuda_profile_batch(const saber_profile_desc* desc,
                                                 saber_profile_out* out) {
  if (!desc || !out || !desc->specs) return fail(SABER_EINVAL, "null argument");
  const int P = desc->n_profiles;
  if (P < 1) return fail(SABER_EINVAL, "profile_batch: no profiles");
  if (!out->sample_offsets || !out->loads || !out->speeds || !out->status)
    return fail(SABER_EINVAL, "profile_batch: outputs required");
  std::vector<int64_t> boff(static_cast<size_t>(P) + 1, 0), soff(static_cast<size_t>(P) + 1, 0);
  std::vector<int32_t> bsize;
  std::vector<double> bin, bout, prate(static_cast<size_t>(P));
  int lmax = 1;
  for (int i = 0; i < P; ++i) lmax = std::max(lmax, desc->specs[i].l_max);
  const int stride = lmax + 2;
  std::vector<double> tab(static_cast<size_t>(P) * stride);
  for (int i = 0; i < P; ++i) {
    const saber_profile_spec& s = desc->specs[i];
    BurstPlan plan;
    if (saber_status e = plan_bursts(s, &plan)) return e;
    bsize.insert(bsize.end(), plan.size.begin(), plan.size.end());
    bin.insert(bin.end(), plan.in.begin(), plan.in.end());
    bout.insert(bout.end(), plan.out.begin(), plan.out.end());
    boff[static_cast<size_t>(i) + 1] = static_cast<int64_t>(bsize.size());
    soff[static_cast<size_t>(i) + 1] = soff[static_cast<size_t>(i)] + plan.issued;
    prate[static_cast<size_t>(i)] = s.prefill_rate;
    fill_table(s.ground_truth, lmax + 1, &tab[static_cast<size_t>(i) * stride]);
  }
  const int64_t S = soff[static_cast<size_t>(P)];
  std::memcpy(out->sample_offsets, soff.data(), soff.size() * 8);
  if (out->capacity < S)
    return fail(SABER_ECAPACITY, "profile_batch: sample buffer too small (" + std::to_string(S) + ")");
  if (saber_status e = use_device(desc->device)) return e;
  const int dev = desc->device;
  DevBuf tables, pr, bo, bs, bi, bt, so, ld, sp;
  ALLOC_TRY(tables, dev, tab.size() * 8);
  ALLOC_TRY(pr, dev, prate.size() * 8);
  ALLOC_TRY(bo, dev, boff.size() * 8);
  ALLOC_TRY(bs, dev, std::max<size_t>(1, bsize.size()) * 4);
  ALLOC_TRY(bi, dev, std::max<size_t>(1, bin.size()) * 8);
  ALLOC_TRY(bt, dev, std::max<size_t>(1, bout.size()) * 8);
  ALLOC_TRY(so, dev, soff.size() * 8);
  ALLOC_TRY(ld, dev, static_cast<size_t>(std::max<int64_t>(1, S)) * 4);
  ALLOC_TRY(sp, dev, static_cast<size_t>(std::max<int64_t>(1, S)) * 8);
  Timer tm;
  if (saber_status e = tm.init()) return e;
  cudaStream_t st = nullptr;
  SyncOnExit sync_guard(&st);
  CUDA_TRY(cudaEventRecord(tm.a, st));
  CUDA_TRY(cudaMemcpyAsync(tables.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(pr.p, prate.data(), prate.size() * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(bo.p, boff.data(), boff.size() * 8, cudaMemcpyHostToDevice, st));
  if (!bsize.empty()) {
    CUDA_TRY(cudaMemcpyAsync(bs.p, bsize.data(), bsize.size() * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(bi.p, bin.data(), bin.size() * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(bt.p, bout.data(), bout.size() * 8, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaMemcpyAsync(so.p, soff.data(), soff.size() * 8, cudaMemcpyHostToDevice, st));
  ProfileParams pp{};
  pp.n_profiles = P;
  pp.tables = tables.as<double>();
  pp.table_stride = stride;
  pp.prefill_rate = pr.as<double>();
  pp.burst_off = bo.as<int64_t>();
  pp.burst_size = bs.as<int32_t>();
  pp.burst_in = bi.as<double>();
  pp.burst_out = bt.as<double>();
  pp.sample_off = so.as<int64_t>();
  pp.loads = ld.as<int32_t>();
  pp.speeds = sp.as<double>();
  LAUNCH_TRY(launch_profile(pp, st));
  if (S > 0) {
    CUDA_TRY(cudaMemcpyAsync(out->loads, ld.p, static_cast<size_t>(S) * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(out->speeds, sp.p, static_cast<size_t>(S) * 8, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaEventRecord(tm.b, st));
  CUDA_TRY(cudaEventSynchronize(tm.b));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, tm.a, tm.b));
  out->device_ms = ms;
  for (int i = 0; i < P; ++i) {  // profile(): < 3 distinct loads -> CalibrationError
    std::vector<int32_t> l(out->loads + soff[static_cast<size_t>(i)],
                           out->loads + soff[static_cast<size_t>(i) + 1]);
    std::sort(l.begin(), l.end());
    const int64_t distinct = std::unique(l.begin(), l.end()) - l.begin();
    out->status[i] = distinct < 3 ? 1 : 0;
  }
  return SABER_OK;
}
