/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C interface shared by the two CPU checkers under oracle/:
 *   - saber_oracle.c : a C restatement of the reference algorithm (prefix orc_)
 *   - ref_harness.cpp: a thin extern "C" harness over the reference itself,
 *                      compiled from /root/reference/proj/core/src into
 *                      oracle/_ref/libsaber_ref.so (prefix ref_)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load these libraries.  The product (paper_2506_19677_b200) never
 * links or calls anything declared here.
 *
 * Both libraries export the same functions with their own prefix, so a test
 * can run the same case through either one and compare.
 */
#ifndef SABER_ORACLE_H
#define SABER_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Task catalog order (reference proj/core/src/types.cpp:10-18). */
enum { ORC_QNA = 0, ORC_GENERATION = 1, ORC_SUMMARY = 2, ORC_TRANSLATION = 3 };
/* Model families (reference estimator.hpp:21). */
enum { ORC_USL = 0, ORC_LOGISTIC = 1, ORC_LINEAR = 2 };
/* Scheduler modes (reference types.hpp:76). */
enum { ORC_SABER = 0, ORC_STATIC = 1 };
/* Decision kinds (reference scheduler.hpp:46). */
enum {
  ORC_ADMIT_HIGH = 0,
  ORC_ADMIT_LOW = 1,
  ORC_REJECT_OWN = 2,
  ORC_REJECT_ACTIVE = 3,
  ORC_DEMOTE = 4
};

typedef struct {
  int32_t family;
  double p[3];
} orc_model;

/* WorkloadMix as fractions per catalog task plus a presence flag (the
 * reference's std::map may hold zero-fraction entries, which still matter for
 * its "last entry" fallback, workload.cpp:28-39). */
typedef struct {
  double frac[4];
  int32_t present[4];
} orc_mix;

typedef struct {
  orc_mix mix;
  double rps;
  int32_t num_requests;
  uint64_t workload_seed;
  double jitter;

  int32_t mode;      /* ORC_SABER / ORC_STATIC */
  int32_t window;
  double tick;
  int32_t cap;

  int32_t has_model;
  orc_model model;
  orc_model ground_truth;
  double prefill_rate;

  int32_t has_horizon;
  double horizon;
  uint64_t seed;     /* scheduler seed (SimConfig::seed) */
} orc_sim_config;

/* One explicit request for the replay path (run_with_requests). */
typedef struct {
  double arrival_time;
  double sla_seconds;
  double deadline;
  int32_t input_tokens;
  int32_t max_output_tokens;
  int32_t task; /* catalog index, or -1 for a custom task name */
} orc_request;

typedef struct {
  double time;
  uint64_t request_id;
  int32_t kind;
  int32_t load_before;
  int32_t has_pred, has_req;
  double pred_speed;
  double req_speed;
} orc_decision;

typedef struct {
  /* MetricsReport (metrics.hpp:63-69) */
  double goodput, ratio_mean, ratio_std, cv;
  int64_t completed;
  int64_t met;
  int64_t decisions;
  int64_t n_kind[5];
  uint64_t decision_hash;
  int64_t issued_by_task[4];
  int64_t met_by_task[4];
  /* Event counters of the reference algorithm; the compiled
   * reference harness cannot see engine internals and leaves these at -1. */
  int64_t ticks, passes, decode_updates, prefill_updates;
  int64_t refresh_entries, gate_candidates, ledger_scanned, rng_draws;
  double last_arrival;
  double horizon;
} orc_traj_out;

/* Per-request outputs (NaN where absent). */
typedef struct {
  double arrival_time, admit_time, completion_time, sla;
  int32_t task, input_tokens, max_output_tokens, demoted;
} orc_record;

/* Decision-log digest used by every implementation (oracle restatement,
 * reference harness, CUDA kernel).  For the i-th decision d (0-based, in
 * emission order):
 *   x_i = id | kind<<32 | (u64)(u32)load<<40
 *         ^ rotl(pred_bits,17) ^ rotl(req_bits,43) ^ rotl(bits(d.time),7)
 *   h   = sum_i mix64(x_i + (i+1) * 0x9E3779B97F4A7C15)   (mod 2^64)
 * with absent speeds as ORC_ABSENT_BITS and mix64 the splitmix64 finaliser.
 * Every term carries its position, so the digest is order-sensitive, and the
 * terms are independent, so the device can form them lane-parallel
 * (DESIGN.md §5).  The empty log hashes to ORC_HASH_SEED (0).  */
#define ORC_HASH_SEED 0ULL
#define ORC_ABSENT_BITS 0xFFF8000000000001ULL

static inline uint64_t orc_rotl(uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}
static inline uint64_t orc_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
static inline uint64_t orc_decision_term(uint64_t index, uint64_t time_bits, uint64_t w,
                                         uint64_t pb, uint64_t rb) {
  const uint64_t x = w ^ orc_rotl(pb, 17) ^ orc_rotl(rb, 43) ^ orc_rotl(time_bits, 7);
  return orc_mix64(x + (index + 1) * 0x9E3779B97F4A7C15ULL);
}

/* ---- functions exported by both libraries (prefix orc_ / ref_) ---------- */
/* Each returns 0 on success, nonzero on error (message in *_last_error()). */

#define ORC_DECLARE(P)                                                         \
  const char* P##last_error(void);                                             \
  /* generate(): n requests for a WorkloadSpec. */                             \
  int P##generate(const orc_sim_config* cfg, orc_request* out);                \
  /* run(): one trajectory.  records (n entries) and decisions (capacity       \
   * dec_cap, count in *n_dec) may be NULL. */                                 \
  int P##run(const orc_sim_config* cfg, orc_traj_out* out,                     \
             orc_record* records, orc_decision* decisions, int64_t dec_cap,    \
             int64_t* n_dec);                                                  \
  /* run_with_requests(): replay n explicit requests. */                       \
  int P##run_with_requests(const orc_sim_config* cfg, const orc_request* reqs, \
                           int32_t n, orc_traj_out* out, orc_record* records,  \
                           orc_decision* decisions, int64_t dec_cap,           \
                           int64_t* n_dec);                                    \
  /* predict(model, load) */                                                   \
  int P##predict(const orc_model* m, int32_t load, double* out);               \
  /* fit(samples, family): status 0 ok, 1 FitError. params/r2 filled on ok,  \
   * best params/sse on FitError. */                                           \
  int P##fit(const int32_t* loads, const double* speeds, int32_t m,            \
             int32_t family, double* params, double* r2_or_sse,                \
             int32_t* fit_error);                                              \
  /* calibrate(): best family index, per-family ok flags, params, r2. */      \
  int P##calibrate(const int32_t* loads, const double* speeds, int32_t m,      \
                   int32_t* best_family, double* best_params, double* best_r2, \
                   int32_t* ok, double* fam_params, double* fam_r2);           \
  /* profile(): fills up to cap samples, count in *n_out. */                   \
  int P##profile(const orc_model* gt, double prefill_rate, const orc_mix* mix, \
                 int32_t num_requests, uint64_t seed, double jitter,           \
                 int32_t l_max, int32_t* loads, double* speeds, int64_t cap,   \
                 int64_t* n_out);                                              \
  /* sweep(): rows in the reference's grid order; ratios optional. */          \
  int P##sweep(const orc_sim_config* base, const int32_t* mix_ids,             \
               int32_t n_mixes, const double* rps, int32_t n_rps,              \
               const int32_t* caps, int32_t n_caps, int32_t with_saber,        \
               int32_t repeats, int32_t jobs, double* row_goodput,             \
               double* row_ratio_mean, double* row_ratio_std,                  \
               double* row_cv, double* summary /* n_mixes x 7 */,              \
               int32_t* best_cap /* n_mixes x n_rps */);

ORC_DECLARE(orc_)
ORC_DECLARE(ref_)

/* Extra restatement-only helpers. */
uint64_t orc_mt19937_64_nth(uint64_t seed, int64_t n); /* n-th output, 1-based */

/* Preset mixes w1/w2/w3 as orc_mix (types.cpp:27-47). id = 1, 2, 3. */
int orc_preset_mix(int32_t id, orc_mix* out);

#ifdef __cplusplus
}
#endif
#endif
