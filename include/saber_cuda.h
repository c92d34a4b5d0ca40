/*
 * saber_cuda.h — the drop-in C ABI of the B200 SABER engine.
 *
 * The reference (SaberSim, /root/reference/proj) has no C ABI: its boundary is
 * the installed C++20 API of sabersim::saber_core.  Every entry point below
 * replaces one call of that API on the hot path; the citation says which
 * (paths relative to proj/core/include/saber/ and proj/core/src/).
 *
 *   saber_cuda_sweep          <- SweepResult sweep(const SweepGrid&, const SimConfig&, int jobs)
 *                                 simloop.hpp:96-99, simloop.cpp:130-277
 *   saber_cuda_run_batch      <- RunOutput run(const SimConfig&)               simloop.hpp:49
 *                                 RunOutput run_with_requests(const SimConfig&, std::vector<Request>)
 *                                 simloop.hpp:53-54, simloop.cpp:50-116
 *                                 (many independent trajectories per call)
 *   saber_cuda_fit_batch      <- SpeedModel fit(const std::vector<LoadSpeedSample>&, ModelFamily)
 *                                 estimator.hpp:61, estimator.cpp:241-346
 *                                 CalibrationReport calibrate(const std::vector<LoadSpeedSample>&)
 *                                 calibration.hpp:54, calibration.cpp:137-168
 *                                 (many independent curves per call)
 *   saber_cuda_profile_batch  <- profile(const EngineConfig&, const WorkloadSpec&, int l_max)
 *                                 calibration.hpp:29-31, calibration.cpp:58-135 (batched)
 *   saber_cuda_predict_table  <- double predict(const SpeedModel&, int)       estimator.hpp:39
 *   saber_cuda_generate       <- std::vector<Request> generate(const WorkloadSpec&)
 *                                 workload.hpp:31, workload.cpp:52-79 (batched)
 *   saber_cuda_trace_from_csv / _to_csv <- trace_from_csv / trace_to_csv
 *                                 workload.hpp:38-39, workload.cpp:87-138
 *
 * Conventions: plain C, POD structs, caller-owned memory, no exceptions.  Every
 * function returns a saber_status; on failure saber_cuda_last_error() holds a
 * one-line message.  Status codes map onto the reference's exception types:
 *   SABER_EINVAL  -> std::invalid_argument   (config / validation errors)
 *   SABER_EDOMAIN -> std::domain_error       (predict with load < 1)
 *   SABER_EFIT    -> saber::FitError         (per curve, see saber_fit_out)
 *   SABER_ECUDA   -> std::runtime_error      (device failure; CLI exit 3)
 * There is no CPU fallback: with no usable sm_100 device every compute call
 * returns SABER_ECUDA.
 */
#ifndef SABER_CUDA_H
#define SABER_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SABER_CUDA_ABI_VERSION 2

typedef enum {
  SABER_OK = 0,
  SABER_EINVAL = 1,
  SABER_EDOMAIN = 2,
  SABER_EFIT = 3,
  SABER_ECUDA = 4,
  SABER_ECAPACITY = 5, /* a caller-sized buffer (e.g. decision trace) is too small */
  SABER_EINTERNAL = 6, /* an invariant the reference would throw logic_error on */
  SABER_ERETRY = 7     /* recoverable: a sweep plan grew its scheduler draw streams
                          (a trajectory exhausted one); the launched results are
                          void — launch the plan again (saber_cuda_sweep_plan_run
                          does this itself) */
} saber_status;

/* Task catalog (types.cpp:10-18), in catalog order. */
enum { SABER_TASK_QNA = 0, SABER_TASK_GENERATION = 1, SABER_TASK_SUMMARY = 2,
       SABER_TASK_TRANSLATION = 3, SABER_TASK_CUSTOM = -1 };
/* ModelFamily (estimator.hpp:21). */
enum { SABER_USL = 0, SABER_LOGISTIC = 1, SABER_LINEAR = 2 };
/* SchedulerMode (types.hpp:76). */
enum { SABER_MODE_SABER = 0, SABER_MODE_STATIC = 1 };
/* RequestState (types.hpp:43). */
enum { SABER_STATE_QUEUED_HIGH = 0, SABER_STATE_QUEUED_LOW = 1, SABER_STATE_EXECUTING = 2,
       SABER_STATE_COMPLETED = 3 };
/* DecisionKind (scheduler.hpp:46). */
enum { SABER_ADMIT_HIGH = 0, SABER_ADMIT_LOW = 1, SABER_REJECT_OWN = 2,
       SABER_REJECT_ACTIVE = 3, SABER_DEMOTE = 4 };

/* SpeedModel (estimator.hpp:29-33). Linear uses params[0..1]. */
typedef struct {
  int32_t family;
  double params[3];
} saber_model;

/* WorkloadMix (types.hpp:31-33): fraction per catalog task; present[t]=0 means
 * the task is absent from the map (a present zero-fraction task is legal). */
typedef struct {
  double frac[4];
  int32_t present[4];
} saber_mix;

/* One trajectory's result row: SweepRow (simloop.hpp:63-73) + MetricsReport
 * (metrics.hpp:63-69) scalars, decision statistics and the reference-algorithm
 * event counts used for the roofline.  All fields are 8 bytes so
 * a row buffer can be all-reduced as uint64 (disjoint shards sum exactly). */
typedef struct {
  double goodput;     /* met / n */
  double ratio_mean;  /* NaN when nothing completed */
  double ratio_std;
  double cv;
  int64_t n;          /* requests in the trajectory; 0 = row not simulated here */
  int64_t completed;
  int64_t met;
  int64_t decisions;
  int64_t n_kind[5];  /* by DecisionKind */
  uint64_t decision_hash; /* hash of the ordered decision log */
  int64_t issued_by_task[4];
  int64_t met_by_task[4];
  int64_t ticks, passes, decode_updates, prefill_updates;
  int64_t refresh_entries, gate_candidates, ledger_scanned, rng_draws;
  double last_arrival;
  double horizon;
  /* Latency percentiles p50, p90, p99 of completion - arrival over the
   * trajectory's issued requests, read off the reference's cdf
   * (metrics.cpp:61-85, all tasks): the smallest latency x whose fraction
   * (#latencies <= x) / issued is >= p; NaN when that fraction is never
   * reached (too few completions).  Exact (an order statistic). */
  double latency_q[3];
} saber_traj_row;

/* Decision record (scheduler.hpp:48-55). Absent speeds: has_* = 0. */
typedef struct {
  double time;
  uint64_t request_id;
  int32_t kind;
  int32_t load_before;
  int32_t has_pred, has_req;
  double pred_speed;
  double req_speed;
} saber_decision;

/* --------------------------------------------------------------------------
 * Sweep (simloop.hpp:56-99).  Rows are in the reference's grid order:
 * mix -> rps -> [caps..., saber] -> repeat (seed = base.seed + repeat).
 * -------------------------------------------------------------------------- */
typedef struct {
  /* SweepGrid */
  const int32_t* mixes; /* preset ids: 1 = "w1", 2 = "w2", 3 = "w3" */
  int32_t n_mixes;
  const double* rps;
  int32_t n_rps;
  const int32_t* caps;
  int32_t n_caps;
  int32_t with_saber;
  /* base SimConfig (simloop.hpp:23-31) */
  int32_t num_requests;
  double length_jitter;
  int32_t window_size;
  double tick;
  int32_t has_model;
  saber_model model;
  saber_model ground_truth;
  double prefill_rate;
  int32_t has_horizon;
  double horizon;
  int32_t repeats;
  uint64_t seed;
  /* execution */
  int32_t device;        /* CUDA ordinal */
  int32_t shard_index;   /* this process simulates rows r with r % shard_count == shard_index */
  int32_t shard_count;   /* 1 = everything */
} saber_sweep_desc;

/* MixSummary (simloop.hpp:80-89), one per mix, in grid order. */
typedef struct {
  double saber_mean_goodput;
  double best_static_mean_goodput;
  double delta;
  double saber_pooled_cv;
  double best_static_pooled_cv;
  double saber_rps_mean_cv;
  double best_static_rps_mean_cv;
} saber_mix_summary;

/* The reference's SweepRow payload (simloop.hpp:63-73): the four statistics
 * of a row; its keys (mix, rps, scheduler, cap, seed) follow from the grid order. */
typedef struct {
  double goodput;
  double ratio_mean;  /* NaN when nothing completed */
  double ratio_std;
  double cv;
} saber_row_stats;

typedef struct {
  saber_traj_row* rows;            /* [n_rows] or NULL */
  double* completion_times;        /* [n_rows][num_requests] or NULL (NaN = never) */
  saber_mix_summary* summary;      /* [n_mixes] or NULL (needs shard_count == 1) */
  int32_t* best_cap_by_rps;        /* [n_mixes][n_rps] or NULL; 0 when no caps */
  /* telemetry, filled by the call */
  int64_t n_rows;
  double device_ms;                /* CUDA-event time of the device work */
  int32_t kernel_launches;
  int64_t h2d_bytes;               /* host->device bytes of the inputs (plan create) */
  int64_t d2h_bytes;               /* device->host bytes of the results (fetch) */
  /* ABI 2: [n_rows] or NULL — just the SweepRow statistics (32 B per row
   * instead of the 280 B saber_traj_row), packed on the device */
  saber_row_stats* row_stats;
} saber_sweep_out;

/* Number of rows a sweep produces (= SweepResult::rows.size()). */
int64_t saber_cuda_sweep_rows(const saber_sweep_desc* desc);

/* One-shot sweep, host buffers in and out (the end-to-end path). */
saber_status saber_cuda_sweep(const saber_sweep_desc* desc, saber_sweep_out* out);

/* Staged sweep for device-resident timing and multi-GPU reduction:
 *   create  : validate, host prologue (per-seed workload draws), device buffers, H2D
 *   run     : all device work on `stream` (workload expansion, scheduler RNG
 *             streams, trajectory simulation, per-row metrics)
 *   summarize: per-cell means, best-cap argmax, pooled CVs from the device rows
 *   fetch   : D2H into an out struct
 * The device row / completion buffers are exposed so a caller can all-reduce
 * them across ranks (rows of other shards are zero, so a uint64 sum gathers). */
typedef struct saber_sweep_plan saber_sweep_plan;
typedef struct {
  void* rows;              /* saber_traj_row[n_rows] on device */
  size_t rows_bytes;
  void* completion_times;  /* double[n_rows][num_requests] on device */
  size_t completion_bytes;
  int64_t n_rows;
  int64_t rows_this_shard;
} saber_sweep_buffers;

saber_status saber_cuda_sweep_plan_create(const saber_sweep_desc* desc, saber_sweep_plan** plan);
saber_status saber_cuda_sweep_plan_run(saber_sweep_plan* plan, void* cuda_stream);
saber_status saber_cuda_sweep_plan_summarize(saber_sweep_plan* plan, void* cuda_stream);
/* Asynchronous halves of run / summarize: enqueue on the stream and return;
 * saber_cuda_sweep_plan_wait synchronises, checks the kernels' error flag and
 * updates the stats.  Lets a caller pipeline sweeps (the summary of one plan
 * overlapping the simulation of another on a second stream). */
saber_status saber_cuda_sweep_plan_launch(saber_sweep_plan* plan, void* cuda_stream);
saber_status saber_cuda_sweep_plan_summarize_launch(saber_sweep_plan* plan, void* cuda_stream);
saber_status saber_cuda_sweep_plan_wait(saber_sweep_plan* plan);
/* launch = launch_sim + metrics_launch on one stream.  Split, the per-row
 * metrics (which feed the summary and the fetched rows) can run on the
 * summary's stream; multi-GPU: before the gather (each rank owns its rows). */
saber_status saber_cuda_sweep_plan_launch_sim(saber_sweep_plan* plan, void* cuda_stream);
saber_status saber_cuda_sweep_plan_metrics_launch(saber_sweep_plan* plan, void* cuda_stream);
saber_status saber_cuda_sweep_plan_buffers(saber_sweep_plan* plan, saber_sweep_buffers* out);
saber_status saber_cuda_sweep_plan_fetch(saber_sweep_plan* plan, saber_sweep_out* out);
/* Pipelined use (several sweeps in flight):
 *   reseed     : the host prologue for base seed `seed` (per-seed generate()
 *                draws, glibc log) into the plan's pinned staging, uploaded
 *                asynchronously on `stream`; the next launch simulates it
 *   fetch_async: the out struct's requested results copied on `stream`
 *                (caller buffers should be pinned; read them after the stream
 *                synchronises).  Enqueue after summarize_launch on the same
 *                stream (or order the streams) when the summary is wanted. */
saber_status saber_cuda_sweep_plan_reseed(saber_sweep_plan* plan, uint64_t seed, void* cuda_stream);
saber_status saber_cuda_sweep_plan_fetch_async(saber_sweep_plan* plan, saber_sweep_out* out,
                                               void* cuda_stream);
/* CUDA-event time and launches of the last plan_run (+ summarize). */
saber_status saber_cuda_sweep_plan_stats(saber_sweep_plan* plan, double* device_ms,
                                         double* sim_kernel_ms, int32_t* launches);
/* Waits for every piece of work the plan enqueued, then frees it. */
void saber_cuda_sweep_plan_destroy(saber_sweep_plan* plan);

/* --------------------------------------------------------------------------
 * Multi-GPU.  A sweep shards its rows over GPUs (desc
 * shard_index / shard_count: rows r with r % count == index) with no exchange
 * during simulation; the final statistics reduce is one NCCL uint64 SUM of the
 * shards' row and completion buffers onto the root (disjoint shards, so an
 * exact gather), after which the root summarizes and fetches.
 *   one process per GPU: saber_cuda_nccl_unique_id on one rank (the caller
 *     broadcasts the 128 bytes), saber_cuda_nccl_init on every rank, and
 *     saber_cuda_sweep_plan_gather after each plan launch/run;
 *   one process, several GPUs: saber_cuda_sweep_multi (a host thread, stream
 *     and plan per device, ncclCommInitAll).
 * NCCL (libnccl.so.2) is loaded on first use.
 * -------------------------------------------------------------------------- */
typedef struct saber_nccl saber_nccl;
saber_status saber_cuda_nccl_unique_id(uint8_t* id /* [128] */);
saber_status saber_cuda_nccl_init(const uint8_t* id /* [128] */, int32_t n_ranks, int32_t rank,
                                  int32_t device, saber_nccl** comm);
void saber_cuda_nccl_destroy(saber_nccl* comm);
/* Enqueues the reduce of this rank's plan buffers onto `root` on `stream`
 * (after the plan's launch on that stream); every rank calls it. */
saber_status saber_cuda_sweep_plan_gather(saber_sweep_plan* plan, saber_nccl* comm, int32_t root,
                                          void* cuda_stream);
/* The whole sweep (desc->shard_count == 1) over n_devices distinct GPUs; the
 * outputs are those of saber_cuda_sweep. */
saber_status saber_cuda_sweep_multi(const saber_sweep_desc* desc, const int32_t* devices,
                                    int32_t n_devices, saber_sweep_out* out);

/* --------------------------------------------------------------------------
 * Trajectory batch (run / run_with_requests).  Each trajectory is either
 * generated (generate(): WorkloadSpec + its seed) or replayed from explicit
 * requests (ids 0..n-1 in arrival order).
 * -------------------------------------------------------------------------- */
/* The static fields of a Request (types.hpp:45-59); its id is its index. */
typedef struct {
  double arrival_time;
  double sla_seconds;
  double deadline;         /* absolute; the reference keeps it independent of sla */
  int32_t input_tokens;
  int32_t max_output_tokens;
  int32_t task;            /* SABER_TASK_* (CUSTOM for non-catalog names) */
  int32_t group;           /* task group of the per-task metrics (MetricsReport::per_task,
                              a std::map keyed by task name): requests with equal group
                              share one CDF, groups ordered by value.  The engine numbers
                              the catalog tasks by name rank (code_generation 0, code_qna 1,
                              code_summary 2, code_translation 3); a replay caller numbers
                              its task names in the same (sorted) order. */
} saber_request;

/* A request's mutable state at the end of a run (Request, types.hpp:45-59) and
 * its RunRecord fields (make_record, metrics.cpp:17-30). */
typedef struct {
  double admit_time;               /* NaN = never admitted */
  double completion_time;          /* NaN = never completed */
  double generated_tokens;         /* fluid progress (max_output_tokens once completed) */
  double recorded_required_speed;  /* required_speed at admission; NaN = never admitted */
  int32_t state;                   /* SABER_STATE_* */
  int32_t met_sla;                 /* completed and completion - arrival <= sla */
  int32_t demoted;                 /* ever in the low tier (final_tier "low") */
  int32_t pad_;
} saber_request_state;

typedef struct {
  /* WorkloadSpec (workload.hpp:15-21); ignored when `requests` is set */
  saber_mix mix;
  double rps;
  int32_t num_requests;
  uint64_t workload_seed;
  double length_jitter;
  /* replay (run_with_requests): num_requests entries, or NULL */
  const saber_request* requests;
  /* SchedulerConfig (types.hpp:78-83) */
  int32_t mode;
  int32_t window_size;
  double tick;
  int32_t static_batch_size;
  /* SimConfig rest */
  int32_t has_model;
  saber_model model;
  saber_model ground_truth;
  double prefill_rate;
  int32_t has_horizon;
  double horizon;
  uint64_t seed;           /* scheduler seed (SimConfig::seed) */
} saber_traj_spec;

typedef struct {
  const saber_traj_spec* specs;
  int32_t n_traj;
  int32_t device;
} saber_run_batch_desc;

typedef struct {
  saber_traj_row* rows;          /* [n_traj] */
  /* per-request outputs, [n_traj][max_n] or NULL (RunRecord, metrics.hpp:20-30) */
  double* arrival_times;
  double* admit_times;           /* NaN = never admitted */
  double* completion_times;      /* NaN = never completed */
  uint8_t* demoted;              /* final_tier == "low" */
  int32_t max_n;                 /* row stride of the per-request arrays */
  /* full decision logs (decisions.csv), optional: trajectory k writes at
   * decisions + k*decision_cap; counts in n_decisions[k] */
  saber_decision* decisions;
  int64_t decision_cap;
  int64_t* n_decisions;
  double device_ms;
  int32_t kernel_launches;
  /* --- ABI 2: the full RunOutput (simloop.hpp:37-43) from the engine, each
   * optional, row stride max_n (group counts: max_groups) --- */
  saber_request* requests;         /* the workload: generate() output or the replay */
  saber_request_state* states;     /* final request states + records */
  /* Per task group g (saber_request::group) of trajectory k, the latency CDF
   * of cdf() (metrics.cpp:61-85): the group's issued requests occupy positions
   * [start_g, start_g + issued_g) of row k, start_g = #requests of smaller
   * groups; the group's CDF points are the positions whose fraction is not
   * NaN, in ascending latency order. */
  double* cdf_latency;
  double* cdf_fraction;
  int32_t* group_issued;           /* [n_traj][max_groups]: TaskMetrics::issued */
  int32_t* group_met;              /* [n_traj][max_groups]: met_sla count (goodput = met / issued) */
  int32_t max_groups;              /* >= 4 when any trajectory is generated; > every replay group */
} saber_run_batch_out;

saber_status saber_cuda_run_batch(const saber_run_batch_desc* desc, saber_run_batch_out* out);

/* --------------------------------------------------------------------------
 * Workload generation <- std::vector<Request> generate(const WorkloadSpec&)
 *   workload.hpp:31, workload.cpp:52-79.  Spec k's requests land at
 *   out + k * max_n (num_requests entries); bit-identical to the reference.
 * -------------------------------------------------------------------------- */
typedef struct {
  saber_mix mix;
  double rps;
  int32_t num_requests;
  uint64_t seed;
  double length_jitter;
} saber_workload_spec;

saber_status saber_cuda_generate(const saber_workload_spec* specs, int32_t n_specs, int32_t device,
                                 saber_request* out, int32_t max_n);

/* --------------------------------------------------------------------------
 * Trace CSV round trip (host-side, no device) <-
 *   std::vector<Request> trace_from_csv(const std::string&)  workload.hpp:39, workload.cpp:97-138
 *   std::string trace_to_csv(const std::vector<Request>&)    workload.hpp:38, workload.cpp:87-95
 * from_csv parses `len` bytes of `text`; *n_out = rows; SABER_ECAPACITY when
 * out is NULL or cap < rows (call again with a larger buffer).  to_csv writes
 * a NUL-terminated text; *len_out = its length without the NUL;
 * SABER_ECAPACITY when cap <= *len_out.
 * -------------------------------------------------------------------------- */
saber_status saber_cuda_trace_from_csv(const char* text, size_t len, saber_request* out,
                                       int32_t cap, int32_t* n_out);
saber_status saber_cuda_trace_to_csv(const saber_request* requests, int32_t n, char* buf,
                                     size_t cap, size_t* len_out);

/* --------------------------------------------------------------------------
 * Monte-Carlo sweep with bursty arrivals (BASELINE config 5; no reference
 * counterpart: the reference generator is Poisson only, workload.cpp:60).
 * Trajectory k (0 <= k < n_traj) simulates cell k % n_cells of the grid
 * mix -> rps -> [caps..., saber] on its own arrival trace: a 2-state MMPP
 * (burst rate = burst_factor * rps, exponential holding times with means
 * mean_calm / mean_burst) drawn from Philox4x32-10 keyed by (seed, k); tasks
 * and lengths follow generate()'s rules.  Its scheduler seed (SimConfig::seed)
 * is scheduler_seed + k % scheduler_seeds.  saber_cuda_mc_trace() rebuilds any
 * trajectory's requests and config on the host, bit-identically, so it can
 * be replayed through run_with_requests().
 * -------------------------------------------------------------------------- */
#define SABER_MC_STATS 8   /* trajectories, requests, met, completed, decisions,
                              admitted, sum of decision-hash low bits, ticks */
#define SABER_MC_BINS 64   /* latency/SLA ratio bins: 4 per octave from 2^-6 */

typedef struct {
  int64_t n_traj;
  const int32_t* mixes;
  int32_t n_mixes;
  const double* rps;
  int32_t n_rps;
  const int32_t* caps;
  int32_t n_caps;
  int32_t with_saber;
  int32_t num_requests;
  double length_jitter;
  int32_t window_size;
  double tick;
  int32_t has_model;
  saber_model model;
  saber_model ground_truth;
  double prefill_rate;
  /* bursty arrivals */
  uint64_t seed;
  double burst_factor;
  double mean_calm;
  double mean_burst;
  uint64_t scheduler_seed;
  int32_t scheduler_seeds;
  /* execution */
  int32_t device;
  int32_t shard_index;   /* this process runs trajectories k with k % shard_count == shard_index */
  int32_t shard_count;
  int64_t chunk;         /* trajectories per device batch (0 = automatic) */
} saber_mc_desc;

typedef struct {
  int64_t* cell_stats;     /* [n_cells][SABER_MC_STATS], accumulated (not cleared) */
  int64_t* cell_hist;      /* [n_cells][SABER_MC_BINS + 1] (+1: never completed), accumulated, or NULL */
  saber_traj_row* rows;    /* [n_traj] rows of this shard's trajectories, or NULL */
  double device_ms;
  double sim_kernel_ms;
  int32_t kernel_launches;
} saber_mc_out;

int64_t saber_cuda_mc_cells(const saber_mc_desc* desc);
saber_status saber_cuda_mc_sweep(const saber_mc_desc* desc, saber_mc_out* out);
/* Host twin: trajectory k's requests (num_requests entries) and its config
 * (spec->requests is left NULL).  Pure host code, no device needed. */
saber_status saber_cuda_mc_trace(const saber_mc_desc* desc, int64_t k, saber_request* requests,
                                 saber_traj_spec* spec);

/* --------------------------------------------------------------------------
 * Batched offline profiling <- std::vector<LoadSpeedSample>
 *   profile(const EngineConfig&, const WorkloadSpec&, int l_max)
 *   calibration.hpp:29-31, calibration.cpp:58-135
 * Each profile's samples land at [sample_offsets[p], sample_offsets[p+1]).
 * -------------------------------------------------------------------------- */
typedef struct {
  saber_model ground_truth;  /* EngineConfig (engine.hpp:16-19) */
  double prefill_rate;
  saber_mix mix;             /* profiling WorkloadSpec (rps unused, calibration.hpp:28) */
  int32_t num_requests;
  uint64_t seed;
  double length_jitter;
  int32_t l_max;
} saber_profile_spec;

typedef struct {
  const saber_profile_spec* specs;
  int32_t n_profiles;
  int32_t device;
} saber_profile_desc;

typedef struct {
  int64_t* sample_offsets;   /* [n_profiles + 1], filled by the call */
  int32_t* loads;            /* [capacity] LoadSpeedSample::load */
  double* speeds;            /* [capacity] LoadSpeedSample::speed */
  int64_t capacity;
  int32_t* status;           /* [n_profiles]: 0 ok, 1 CalibrationError (< 3 distinct loads) */
  double device_ms;
} saber_profile_out;

/* Number of samples profile() yields for one spec (host-side, no device). */
int64_t saber_cuda_profile_samples(const saber_profile_spec* spec);
/* planned_distinct_loads(num_requests, l_max) (calibration.hpp, calibration.cpp:45-56):
 * distinct burst sizes a profiling budget reaches (host-side, no device). */
int32_t saber_cuda_profile_planned_loads(int32_t num_requests, int32_t l_max);
saber_status saber_cuda_profile_batch(const saber_profile_desc* desc, saber_profile_out* out);

/* --------------------------------------------------------------------------
 * Batched fitting (estimator.cpp:33-375, calibration.cpp:137-168).
 * Curve c owns samples [offsets[c], offsets[c+1]).
 * -------------------------------------------------------------------------- */
typedef struct {
  const int32_t* loads;    /* LoadSpeedSample::load */
  const double* speeds;    /* LoadSpeedSample::speed */
  const int64_t* offsets;  /* [n_curves + 1] */
  int32_t n_curves;
  int32_t family_mask;     /* bit f => fit family f; calibrate needs 0x7 */
  int32_t calibrate;       /* 1 => also select best family (calibrate()) */
  int32_t device;
} saber_fit_desc;

typedef struct {
  /* per family f (0..2) and curve c: index [f * n_curves + c] */
  double* params;          /* [3 * n_curves][3]: fitted params or FitError best params */
  double* r2;              /* fit_r2, or FitError best_sse when status != 0 */
  int32_t* status;         /* 0 ok, -1 not fitted, > 0 FitError (estimator.hpp:46-58)
                              with the reason SABER_FITERR_* */
  int32_t* best_family;    /* [n_curves] calibrate(): the selected family; -1 when no
                              family fit; -(2 + d) when only d < 3 distinct loads */
  int32_t* iterations;     /* [3 * n_curves] total LM iterations over the 5 starts (or NULL) */
  double device_ms;
  int32_t kernel_launches;
  int32_t* trials;         /* [3 * n_curves] total LM damping trials (solve + sse) over the
                              5 starts (or NULL): with `iterations`, the in-kernel counts of
                              the algorithmic FP64 work */
} saber_fit_out;

/* FitError reasons (estimator.cpp:208-346), i.e. FitError::what():
 *   TOO_FEW            "too few samples or distinct loads to fit <family>"
 *   NO_CONVERGENCE     "optimizer did not converge for <family>"
 *   INCREASING_LINEAR  "fitted linear model is increasing in load"
 *   NOT_MONOTONE       "fitted model is not non-increasing in load" */
enum { SABER_FITERR_TOO_FEW = 1, SABER_FITERR_NO_CONVERGENCE = 2,
       SABER_FITERR_INCREASING_LINEAR = 3, SABER_FITERR_NOT_MONOTONE = 4 };

saber_status saber_cuda_fit_batch(const saber_fit_desc* desc, saber_fit_out* out);

/* predict(model, L) for L = 1..max_load into table[0..max_load-1], computed
 * exactly as the engine's device tables are (estimator.cpp:16-31). */
saber_status saber_cuda_predict_table(const saber_model* model, int32_t max_load, double* table);

/* --------------------------------------------------------------------------
 * Misc.
 * -------------------------------------------------------------------------- */
const char* saber_cuda_last_error(void);
/* Device blocks freed by finished calls are cached for reuse, and the
 * one-shot saber_cuda_sweep keeps its last plan for calls with the same grid;
 * this destroys that plan and returns the cached blocks of `device` to the
 * driver. */
saber_status saber_cuda_release_cache(int32_t device);
int32_t saber_cuda_abi_version(void);
/* Number of usable sm_100 devices (0 on a CPU-only host). */
int32_t saber_cuda_device_count(void);
/* FP64 FMA throughput microbenchmark on `device` (TFLOP/s, 2 flops per DFMA),
 * used as the roofline denominator for the FP64 path. */
saber_status saber_cuda_fp64_peak(int32_t device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* SABER_CUDA_H */
