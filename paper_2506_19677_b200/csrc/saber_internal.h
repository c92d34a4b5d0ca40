// saber_internal.h — device data layout shared by the host orchestration
// (host.cpp) and the sm_100a kernels (*.cu).  See DESIGN.md §2 for the HBM map.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/saber_cuda.h"

namespace saberb200 {

// Sets the message saber_cuda_last_error() returns (host.cpp); returns `s`.
saber_status set_error(saber_status s, const std::string& msg);

// Largest request count the register-bitmask trajectory kernel supports
// (8 x 64-bit words of per-request tier masks).  Larger n runs on the wide
// kernel.
constexpr int kMaxRequests = 512;
// Largest admission window the register Fisher-Yates supports (4-bit nibbles
// in one u64).  The reference default is 8 (types.hpp:80); wider windows run
// on the wide kernel.
constexpr int kMaxWindow = 16;
// Request-count limit of the wide kernel: request ids travel in the low 16
// bits of a slot word and in the u16 low-tier FIFO.
constexpr int kMaxRequestsWide = 65536;
// Lanes per warp; per-lane scratch is interleaved with this stride.
constexpr int kWarp = 32;

// One workload = one request list (generate() output or a replayed trace),
// stored SoA with row stride `nmax`.
struct WorkloadTables {
  const double* arrival;   // [W][nmax]
  const double* deadline;  // [W][nmax]
  const double* sla;       // [W][nmax]
  const double* max_out;   // [W][nmax]  (double: compared against fluid progress)
  const double* input;     // [W][nmax]
  const double* prefill;   // [W][nmax] prefill debt input / prefill_rate (Engine::admit), 0 if rate <= 0
  const int8_t* task;      // [W][nmax]  catalog index or -1
  const double* demote_after;  // [W][nmax] safe lower bound on demotion time
  const double* horizon;   // [W]  last arrival + 10 * max sla (simloop.cpp:60-63)
  const int32_t* arr_tick;  // [W][nmax] first tick-table index >= arrival, or null
  const int32_t* dem_tick;  // [W][nmax] first tick-table index >= demote_after, or null
  int32_t nmax;
};

// One trajectory to simulate (a SimConfig bound to a workload).
struct TrajDesc {
  int32_t workload;
  int32_t n;
  int32_t mode;       // SABER_MODE_*
  int32_t cap;        // static_batch_size
  int32_t window;
  int32_t model_tab;  // offset (doubles) of the scheduler model's predict table, -1 none
  int32_t gt_tab;     // offset of the ground-truth table
  int32_t stream;     // scheduler RNG stream index, -1 none
  double tick;
  double horizon;     // NaN => use the workload's default horizon
  double prefill_rate;
  int64_t row;        // output row
};

// Scheduler RNG streams: stream s holds draws [off[s], off[s] + len[s]).
// Each draw is mt19937_64() % 720720 (= lcm(1..16)), exact for every
// `% (i+1)` with i+1 <= 16 the Fisher-Yates needs.
// A wide plan (window > 16) stores the raw 64-bit draws instead
// (`draws` then points at u64 words; off/len count draws either way).
struct RngStreams {
  const uint32_t* draws;
  const int64_t* off;
  const int64_t* len;
  int32_t wide;
};

constexpr uint32_t kDrawModulus = 720720u;  // lcm(1..16)

// Per-group scratch in global memory for the rarely touched queues
// (DESIGN.md §2): the ledger's frozen requirements and the low-tier FIFO.
// The hot per-slot state lives in shared memory (sim_kernel.cu).
// The wide kernel (n > 512 or window > 16) keeps the
// slots, both tier masks and the gate's window in per-group global memory.
struct GroupScratch {
  double* ledger_need;  // [groups][nmax]
  uint16_t* low_fifo;   // [groups][nmax]
  int64_t groups;
  // wide kernel only (null otherwise)
  double* wslot_g;      // [groups][nmax] slot fluid progress
  uint64_t* wslot_m;    // [groups][nmax] slot bits(max_out) | id
  uint64_t* wmask;      // [groups][2][wmask_nw] high tier, ledger
  int32_t* wgate;       // [groups][3][nmax] Fisher-Yates j, window order, candidate id
  double* wneed;        // [groups][nmax] candidate needs
  int32_t wmask_nw;     // ceil(nmax / 64)
};

// Outputs of the trajectory kernel.
struct SimOutputs {
  saber_traj_row* rows;       // [rows]
  double* completion;         // [rows][nmax]   pre-filled NaN by the caller
  double* admit;              // [rows][nmax] or null
  uint8_t* demoted;           // [rows][nmax] or null
  double* generated;          // [rows][nmax] or null: fluid progress of slots still running at the end
  saber_decision* trace;      // [trace_rows][trace_cap] or null
  int64_t* trace_count;       // [rows] or null
  int64_t trace_cap;
  int32_t* error;             // [1] first error code (0 = none)
};

// The tick grid of the reference's run loop (simloop.cpp:99-100): t_0 = 0,
// t_{k+1} = fl(t_k + tick) below the horizon.  It depends only on `tick`, so
// one host-built table serves every trajectory with that tick; DT[k] =
// T[k+1] - T[k] is exact (Sterbenz) and is the dt of a tick's single full pass.
struct TickTable {
  const double* T;    // [len]
  const double* DT;   // [len - 1]
  int32_t len;        // 0 = no table (streaks off)
  double tick;        // trajectories with d.tick == tick use it
  double inv_tick;    // 1 / tick (index estimate only; exactness from T)
  double dt_max;      // max DT
};

struct SimParams {
  const TrajDesc* traj;
  int32_t n_traj;
  WorkloadTables wl;
  const double* tables;       // predict tables, table[L] at model_tab + L
  RngStreams rng;
  GroupScratch scratch;
  int32_t slot_rows;          // ceil(nmax / G): shared-memory slot rows per warp
  SimOutputs out;
  int32_t* next_traj;         // work-queue cursor (device)
  const int32_t* order;       // execution order of the descriptors (longest first), or null
  int32_t no_streak;          // 1 = disable quiet streaks (A/B runs, SABER_NO_STREAK)
  int32_t mode_sel;           // 0 any, 1 static-only, 2 SABER-only kernel (sim_kernel.cu)
  int32_t first_traj;         // this launch simulates order[first_traj .. n_traj)
  int32_t split_saber;        // SABER-only launch beside a static-only one (grid_saber_split)
  TickTable ticks;            // shared tick grid for quiet streaks
};

// Error codes written to SimOutputs::error.
enum : int32_t {
  kErrNone = 0,
  kErrRngExhausted = 1,   // scheduler stream too short (host bound violated)
  kErrTraceOverflow = 2,  // decision trace capacity exceeded
  kErrBadDesc = 3,
  kErrTickTable = 4,      // t != T[k] at a streak (tick-table invariant broken)
};

// Kernel launchers (defined in the .cu files).
// Trajectory kernel configuration: G lanes per trajectory, 4 warps per block.
struct SimLaunch {
  int nwords;     // 64-bit mask words (n <= 64 * nwords)
  int group;      // lanes per trajectory
  int block;      // threads per block
  int grid;       // persistent blocks
  int grid_sel[3];  // persistent blocks per mode-specialised variant (G = 32)
  int grid_saber_split;  // SABER-only blocks when launched beside the static kernel
  int slot_rows;  // ceil(nmax / group)
  size_t smem;    // dynamic shared memory per block
  int wide;       // 1 = the wide kernel (global-memory slots and masks)
};
// One warp (= one trajectory at a time) per block: ptxas allocates the
// single-warp kernels with fewer spills (SABER kernel 8 B vs 44 B at 128
// registers) and the SMs fill block by block (config 2 +1.2%, config 3 +1.2%
// over 128-thread blocks).
#ifndef SABER_SIM_BLOCK
#define SABER_SIM_BLOCK 32
#endif
constexpr int kSimBlock = SABER_SIM_BLOCK;
// `wide`: the launch needs the wide kernel (nmax > kMaxRequests or a window
// > kMaxWindow).
int plan_sim(int nmax, int group, bool wide, SimLaunch* out);
int launch_sim(const SimParams& p, const SimLaunch& l, void* stream);
// Tick-table indices of every request's arrival and demote_after (quiet
// streak bounds without table searches on the trajectory's critical path).
int launch_tick_index(const WorkloadTables& wl, int64_t cells, const TickTable& tt, int32_t* ka,
                      int32_t* kd, void* stream);

struct RngGenParams {
  const uint64_t* seeds;  // [n_streams] already xor-salted
  uint32_t* draws;
  const int64_t* off;
  const int64_t* len;
  int32_t n_streams;
  int32_t wide;           // 1 = store raw u64 draws (window > 16)
};
int launch_rng_streams(const RngGenParams& p, void* stream);

// Workload expansion.  Item kind 0 = generate() from per-seed draws
// (seed_base row seed_idx, mix thresholds `mix`, rate rps); kind 1 = replayed
// requests already written into the tables.  Both get demotion bounds for
// `ceiling` (the SABER model's max_speed; NaN/<=0 disables the bound) and the
// default horizon.
struct WorkloadItem {
  int32_t kind;
  int32_t n;
  int32_t seed_idx;
  int32_t mix;
  double rps;
  double jitter;
  double ceiling;
  double prefill_rate;  // EngineConfig::prefill_rate of every trajectory on this workload
};
struct WorkloadParams {
  const WorkloadItem* items;
  int32_t n_items;
  const double* seed_base;   // [seeds][seed_stride][4]: -log(1-u_gap) (glibc), u_task, u_in, u_out
  int32_t seed_stride;
  const double* mix_thresh;  // [mixes][4] cumulative thresholds, alphabetical order
  const int8_t* mix_task;    // [mixes][4] task at each threshold slot (-1 unused)
  const int8_t* mix_last;    // [mixes] fallback task (last map entry)
  double *arrival, *deadline, *sla, *max_out, *input, *demote_after, *horizon;
  double* prefill;
  int8_t* task;
  int32_t nmax;
};
int launch_workloads(const WorkloadParams& p, void* stream);

// Sweep trajectory descriptors (grid order) for this shard.
struct SweepDescParams {
  int32_t n_mixes, n_rps, n_caps, with_saber, repeats, n;
  const int32_t* caps;
  int32_t window;
  double tick, prefill_rate;
  int32_t model_tab, gt_tab;
  int32_t has_horizon;
  double horizon;
  int32_t shard_index, shard_count;
  TrajDesc* out;          // [rows_this_shard]
  int64_t n_rows;
};
int launch_sweep_descs(const SweepDescParams& p, void* stream, int64_t rows_this_shard);

// Fill completion rows: NaN for rows in this shard, 0 for others.
int launch_fill_rows(double* comp, int64_t n_rows, int32_t nmax, int32_t shard_index,
                     int32_t shard_count, void* stream);

// Per-row metrics epilogue (metrics.cpp:17-140) over rows of this shard.
struct RowMetricsParams {
  saber_traj_row* rows;
  const double* completion;
  WorkloadTables wl;
  const TrajDesc* traj;
  int32_t n_traj;
  int32_t narrow;  // 1 = a few single-warp blocks (beside the trajectory kernels)
  // rows longer than kMaxRequests rank their latencies in global scratch,
  // one [nmax] slice per warp of a fixed grid (kRowMetricsWideWarps)
  double* lat_scratch;
};
constexpr int kRowMetricsWideWarps = 1184;  // 148 SMs x 8 warps
int launch_row_metrics(const RowMetricsParams& p, void* stream);

// run() epilogue (records.cu): the workload as saber_request, the final
// request states / records and the per-group latency CDFs.  All outputs are
// [rows][nmax] (group counts [rows][max_groups]); `group` is [W][nmax] for
// replayed workloads (-1 = generated: the task's name rank), or null.
struct RecordsParams {
  const TrajDesc* traj;
  int32_t n_traj;
  WorkloadTables wl;
  const int32_t* group;
  const double* completion;
  const double* admit;
  const uint8_t* demoted;
  const double* generated;
  saber_request* requests;
  saber_request_state* states;
  double* cdf_latency;
  double* cdf_fraction;
  int32_t* group_issued;
  int32_t* group_met;
  int32_t max_groups;
};
int launch_pack_requests(const RecordsParams& p, void* stream);
int launch_records(const RecordsParams& p, void* stream);

// Sweep summary (simloop.cpp:206-275).
struct SummaryParams {
  const saber_traj_row* rows;
  const double* completion;
  WorkloadTables wl;
  int32_t n_mixes, n_rps, n_caps, with_saber, repeats, n;
  const int32_t* caps;
  saber_mix_summary* summary;   // [n_mixes]
  int32_t* best_cap;            // [n_mixes][n_rps]
  double* scratch;              // [n_mixes][n_rps][6] cell-level means/flags
  double* ratios;               // [n_rows][n] latency/SLA ratios (NaN = never completed)
  int32_t narrow;               // 1 = few small blocks (runs beside the trajectory kernels)
  void* pool_scratch;           // summary_pool_scratch_bytes() bytes (the chunked pooled sums)
};
// Device scratch the chunked pooled sums of a summary need (summary.cu).
size_t summary_pool_scratch_bytes(int n_mixes, int n_rps, int repeats, int n);
int launch_summary(const SummaryParams& p, void* stream);
// The four SweepRow statistics of every row, packed (sweep fetch).
int launch_pack_row_stats(const saber_traj_row* rows, int64_t n_rows, saber_row_stats* out,
                          void* stream);

// Bursty Monte-Carlo sweep (mc.cu, BASELINE config 5).
}  // namespace saberb200
#include "bursty.h"
namespace saberb200 {
struct McParams {
  int32_t n_mixes, n_rps, n_caps, with_saber, n_cells;
  const double* rps;
  const int32_t* caps;
  const double* mix_thresh;
  const int8_t* mix_task;
  const int8_t* mix_last;
  int32_t n;
  double jitter;
  double ceiling;
  bursty::Params bp;
  int64_t k0, count;  // chunk: local i -> trajectory k = shard_index + (k0 + i) * shard_count
  int32_t shard_index, shard_count;
  int32_t sched_seeds;
  int32_t window;
  double tick, prefill_rate;
  int32_t model_tab, gt_tab;
  double *arrival, *deadline, *sla, *max_out, *input, *demote_after, *horizon;
  double* prefill;
  int8_t* task;
  TrajDesc* descs;
};
int launch_mc_horizon(const McParams& p, int64_t count, unsigned long long* hmax, void* stream);
int launch_mc_workloads(const McParams& p, void* stream);
int launch_mc_reduce(const McParams& p, const saber_traj_row* rows, const double* comp,
                     int64_t* stats, int64_t* hist, void* stream);

// Batched profile() (profile_kernel.cu).
struct ProfileParams {
  int32_t n_profiles;
  const double* tables;        // [n_profiles][table_stride] ground-truth predict tables
  int32_t table_stride;
  const double* prefill_rate;  // [n_profiles]
  const int64_t* burst_off;    // [n_profiles + 1]
  const int32_t* burst_size;   // [bursts]
  const double* burst_in;      // [bursts] input tokens
  const double* burst_out;     // [bursts] output tokens
  const int64_t* sample_off;   // [n_profiles + 1]
  int32_t* loads;              // [samples]
  double* speeds;              // [samples]
};
int launch_profile(const ProfileParams& p, void* stream);

// Fitting.
struct FitParams {
  const int32_t* loads;
  const double* speeds;
  const int64_t* offsets;
  int32_t n_curves;
  int32_t family_mask;
  int32_t calibrate;
  double* params;      // [3*n_curves][3]
  double* r2;          // [3*n_curves]
  int32_t* status;     // [3*n_curves]
  int32_t* best_family;// [n_curves]
  int32_t* iterations; // [3*n_curves]
  double* lm_scratch;  // [3*n_curves*5][4]: per-start (p0,p1,p2,sse)
  int32_t* lm_conv;    // [3*n_curves*5]
  int32_t* lm_iters;   // [3*n_curves*5]
  int32_t* lm_trials;  // [3*n_curves*5] damping trials per start
  int32_t* trials;     // [3*n_curves] summed over the starts (or null)
  int32_t* cursor;     // work queue
  int32_t ieee_only;   // SABER_LM_IEEE=1: LM passes skip the fast paths (checks)
};
int launch_fit(const FitParams& p, void* stream, int* launches);

int fp64_peak(int device, double* tflops);

}  // namespace saberb200
