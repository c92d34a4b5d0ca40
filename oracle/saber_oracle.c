/*
 * saber_oracle.c — TEST INFRASTRUCTURE ONLY (never linked by the product).
 *
 * A plain-C restatement of the SaberSim reference algorithm on the hot path,
 * used as the parity checker for the CUDA engine.  Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * It is pinned against the compiled reference (oracle/_ref/libsaber_ref.so,
 * built from the reference sources by oracle/Makefile) by tests/test_oracle.py,
 * and against the reference's own known-answer vectors restated in tests/.
 *
 * Arithmetic rules that make it bit-identical to the reference:
 *   - compiled without FMA contraction (-ffp-contract=off, baseline x86-64),
 *     matching the reference objects, which contain no vfmadd;
 *   - the same expression shapes and evaluation order as the reference;
 *   - std::min/std::max/std::clamp semantics restated exactly (stl_algobase.h);
 *   - glibc log/exp, the same functions the reference calls.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* orc_last_error(void) { return g_err; }
#define FAIL(...)                                   \
  do {                                              \
    snprintf(g_err, sizeof g_err, __VA_ARGS__);     \
    return 1;                                       \
  } while (0)

/* std::max / std::min / std::clamp exactly as libstdc++ defines them. */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double sclamp(double v, double lo, double hi) {
  return smin(smax(v, lo), hi);
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 (C++ [rand.eng.mers], parameters of std::mt19937_64).         */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t s[312];
  int i;
} mt64;

static void mt_seed(mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int k = 1; k < 312; ++k)
    m->s[k] = 6364136223846793005ULL * (m->s[k - 1] ^ (m->s[k - 1] >> 62)) +
              (uint64_t)k;
  m->i = 312;
}

static void mt_twist(mt64* m) {
  for (int k = 0; k < 312; ++k) {
    const uint64_t x = (m->s[k] & 0xFFFFFFFF80000000ULL) |
                       (m->s[(k + 1) % 312] & 0x7FFFFFFFULL);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    m->s[k] = m->s[(k + 156) % 312] ^ xa;
  }
  m->i = 0;
}

static uint64_t mt_next(mt64* m) {
  if (m->i >= 312) mt_twist(m);
  uint64_t y = m->s[m->i++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

uint64_t orc_mt19937_64_nth(uint64_t seed, int64_t n) {
  mt64 m;
  mt_seed(&m, seed);
  uint64_t v = 0;
  for (int64_t k = 0; k < n; ++k) v = mt_next(&m);
  return v;
}

/* uniform01: top 53 bits (workload.cpp:17-19). */
static inline double uniform01(mt64* m) {
  return (double)(mt_next(m) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------------ */
/* Domain constants (types.cpp:10-47).                                      */
/* ------------------------------------------------------------------------ */
static const int kAvgIn[4] = {186, 463, 31, 670};
static const int kAvgOut[4] = {43, 387, 30, 617};
static const double kSla[4] = {1.0, 8.0, 1.0, 12.0};
/* std::map<std::string,double> iteration order = alphabetical names:
 * code_generation < code_qna < code_summary < code_translation. */
static const int kAlpha[4] = {ORC_GENERATION, ORC_QNA, ORC_SUMMARY,
                              ORC_TRANSLATION};

int orc_preset_mix(int32_t id, orc_mix* out) {
  memset(out, 0, sizeof *out);
  for (int t = 0; t < 4; ++t) out->present[t] = 1;
  switch (id) {
    case 1: /* w1: heavy-task majority */
      out->frac[ORC_TRANSLATION] = 0.4;
      out->frac[ORC_GENERATION] = 0.4;
      out->frac[ORC_QNA] = 0.1;
      out->frac[ORC_SUMMARY] = 0.1;
      return 0;
    case 2: /* w2: light-task majority */
      out->frac[ORC_QNA] = 0.4;
      out->frac[ORC_SUMMARY] = 0.4;
      out->frac[ORC_GENERATION] = 0.1;
      out->frac[ORC_TRANSLATION] = 0.1;
      return 0;
    case 3: /* w3: uniform */
      for (int t = 0; t < 4; ++t) out->frac[t] = 0.25;
      return 0;
  }
  FAIL("unknown mix preset: w%d", id);
}

/* validate_mix (types.cpp:49-65). */
static int validate_mix(const orc_mix* mix) {
  double sum = 0.0;
  int any = 0;
  for (int a = 0; a < 4; ++a) {
    const int t = kAlpha[a];
    if (!mix->present[t]) continue;
    any = 1;
    if (mix->frac[t] < 0.0 || mix->frac[t] > 1.0)
      FAIL("mix fraction out of [0,1]");
    sum += mix->frac[t];
  }
  if (!any) FAIL("mix has no tasks");
  if (fabs(sum - 1.0) > 1e-9) FAIL("mix fractions sum to %f", sum);
  return 0;
}

/* sample_task (workload.cpp:28-39). */
static int sample_task(mt64* rng, const orc_mix* mix) {
  const double u = uniform01(rng);
  double cum = 0.0;
  int last = -1;
  for (int a = 0; a < 4; ++a) {
    const int t = kAlpha[a];
    if (!mix->present[t]) continue;
    last = t;
    cum += mix->frac[t];
    if (u < cum) return t;
  }
  return last;
}

/* jittered_length (workload.cpp:21-26). */
static int jittered_length(mt64* rng, int avg, double jitter) {
  const double lo = avg * (1.0 - jitter);
  const double hi = avg * (1.0 + jitter);
  const double v = lo + uniform01(rng) * (hi - lo);
  const long long r = llround(v);
  return r < 1 ? 1 : (int)r;
}

/* ------------------------------------------------------------------------ */
/* Speed models (estimator.cpp:16-31, 234-239).                             */
/* ------------------------------------------------------------------------ */
static double eval_model(int family, const double* p, double load) {
  switch (family) {
    case ORC_USL: {
      const double denom = 1.0 + p[1] * (load - 1.0) + p[2] * load * (load - 1.0);
      return p[0] / denom;
    }
    case ORC_LOGISTIC: {
      const double arg = sclamp(p[1] * (load - p[2]), -700.0, 700.0);
      return p[0] / (1.0 + exp(arg));
    }
    case ORC_LINEAR:
      return smax(p[0] * load + p[1], 1e-6);
  }
  return 0.0;
}

int orc_predict(const orc_model* m, int32_t load, double* out) {
  if (load < 1) FAIL("predict: load must be >= 1");
  *out = eval_model(m->family, m->p, (double)load);
  return 0;
}

static double predict_i(const orc_model* m, int load) {
  return eval_model(m->family, m->p, (double)load);
}

/* ------------------------------------------------------------------------ */
/* Workload generator (workload.cpp:52-79).                                 */
/* ------------------------------------------------------------------------ */
int orc_generate(const orc_sim_config* cfg, orc_request* out) {
  if (!(cfg->rps > 0.0)) FAIL("rps must be > 0");
  if (cfg->num_requests < 1) FAIL("num_requests must be >= 1");
  if (cfg->jitter < 0.0 || cfg->jitter >= 1.0)
    FAIL("length_jitter must be in [0, 1)");
  if (validate_mix(&cfg->mix)) return 1;
  mt64 rng;
  mt_seed(&rng, cfg->workload_seed);
  double t = 0.0;
  for (int i = 0; i < cfg->num_requests; ++i) {
    const double gap = -log(1.0 - uniform01(&rng)) / cfg->rps;
    double arrival = t + gap;
    if (!(arrival > t)) arrival = t + 1e-6;
    t = arrival;
    const int task = sample_task(&rng, &cfg->mix);
    orc_request* r = &out[i];
    r->task = task;
    r->arrival_time = arrival;
    r->input_tokens = jittered_length(&rng, kAvgIn[task], cfg->jitter);
    r->max_output_tokens = jittered_length(&rng, kAvgOut[task], cfg->jitter);
    r->sla_seconds = kSla[task];
    r->deadline = arrival + kSla[task]; /* deadline_of, types.cpp:90-92 */
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Simulation state.                                                        */
/* ------------------------------------------------------------------------ */
enum { ST_HIGH = 0, ST_LOW = 1, ST_EXEC = 2, ST_DONE = 3, ST_PENDING = 4 };

typedef struct {
  double arrival, sla, deadline, generated;
  int in_tok, out_tok, task, state, demoted;
  double admit_time, completion_time; /* NaN when absent */
} req_t;

/* required_speed (types.cpp:82-88). */
static double required_speed(const req_t* r, double now) {
  if (now >= r->deadline) return INFINITY;
  const double remaining = (double)r->out_tok - r->generated;
  if (remaining <= 0.0) return 0.0;
  return remaining / (r->deadline - now);
}

typedef struct {
  int id;
  double prefill_left, decode_start, load_time;
} slot_t;

typedef struct {
  orc_model gt;
  double prefill_rate;
  double clock;
  slot_t* slots;
  int n_active;
  /* counters */
  int64_t passes, decode_updates, prefill_updates;
} engine_t;

typedef struct {
  double time;
  int id;
  double decode_start, duration, mean_load;
} completion_t;

/* Engine::admit (engine.cpp:26-49). */
static void engine_admit(engine_t* e, req_t* reqs, int id, double now) {
  req_t* r = &reqs[id];
  r->state = ST_EXEC;
  r->admit_time = now;
  slot_t s;
  s.id = id;
  s.prefill_left = e->prefill_rate > 0.0 ? r->in_tok / e->prefill_rate : 0.0;
  s.decode_start = -1.0;
  s.load_time = 0.0;
  if (s.prefill_left == 0.0) s.decode_start = now;
  e->slots[e->n_active++] = s;
}

/* Engine::advance_to (engine.cpp:51-127).  Completions appended to *out. */
static int engine_advance(engine_t* e, req_t* reqs, double t,
                          completion_t* out) {
  int n_out = 0;
  while (e->clock < t) {
    if (e->n_active == 0) {
      e->clock = t;
      break;
    }
    ++e->passes;
    const int load = e->n_active;
    const double speed = predict_i(&e->gt, load);
    double dt = t - e->clock;
    for (int k = 0; k < e->n_active; ++k) {
      const slot_t* s = &e->slots[k];
      double boundary;
      if (s->prefill_left > 0.0) {
        boundary = s->prefill_left;
      } else {
        const req_t* r = &reqs[s->id];
        const double remaining = r->out_tok - r->generated;
        boundary = remaining / speed;
      }
      dt = smin(dt, boundary);
    }
    const double group = dt * (1.0 + 1e-12);
    for (int k = 0; k < e->n_active; ++k) {
      slot_t* s = &e->slots[k];
      if (s->prefill_left > 0.0) {
        ++e->prefill_updates;
        s->prefill_left = s->prefill_left <= group ? 0.0 : s->prefill_left - dt;
      } else {
        ++e->decode_updates;
        reqs[s->id].generated += speed * dt;
        s->load_time += load * dt;
      }
    }
    e->clock += dt;
    for (int k = 0; k < e->n_active; ++k) {
      slot_t* s = &e->slots[k];
      if (s->prefill_left == 0.0 && s->decode_start < 0.0)
        s->decode_start = e->clock;
    }
    for (int k = 0; k < e->n_active;) {
      slot_t* s = &e->slots[k];
      req_t* r = &reqs[s->id];
      const int done = s->decode_start >= 0.0 &&
                       r->generated + speed * (group - dt) >= r->out_tok;
      if (!done) {
        ++k;
        continue;
      }
      r->generated = r->out_tok;
      r->completion_time = e->clock;
      r->state = ST_DONE;
      completion_t c;
      c.time = e->clock;
      c.id = s->id;
      c.decode_start = s->decode_start;
      c.duration = e->clock - s->decode_start;
      c.mean_load = s->load_time / c.duration;
      out[n_out++] = c;
      memmove(&e->slots[k], &e->slots[k + 1],
              sizeof(slot_t) * (size_t)(e->n_active - k - 1));
      --e->n_active;
    }
  }
  return n_out;
}

/* ------------------------------------------------------------------------ */
/* Decision log + hash.                                                     */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t hash;
  int64_t count;
  int64_t n_kind[5];
  orc_decision* buf;
  int64_t cap;
  int overflow;
} declog_t;

static inline uint64_t dbits(double v) {
  uint64_t b;
  memcpy(&b, &v, 8);
  return b;
}

static void declog_push(declog_t* L, double time, int id, int kind, int load,
                        int has_pred, double pred, int has_req, double req) {
  const uint64_t pb = has_pred ? dbits(pred) : ORC_ABSENT_BITS;
  const uint64_t rb = has_req ? dbits(req) : ORC_ABSENT_BITS;
  const uint64_t w = ((uint64_t)(uint32_t)id) | ((uint64_t)kind << 32) |
                     ((uint64_t)(uint32_t)load << 40);
  L->hash += orc_decision_term((uint64_t)L->count, dbits(time), w, pb, rb);
  if (L->buf) {
    if (L->count < L->cap) {
      orc_decision* d = &L->buf[L->count];
      d->time = time;
      d->request_id = (uint64_t)id;
      d->kind = kind;
      d->load_before = load;
      d->has_pred = has_pred;
      d->has_req = has_req;
      d->pred_speed = has_pred ? pred : NAN;
      d->req_speed = has_req ? req : NAN;
    } else {
      L->overflow = 1;
    }
  }
  ++L->count;
  ++L->n_kind[kind];
}

/* ------------------------------------------------------------------------ */
/* run_with_requests (simloop.cpp:50-111) with both schedulers inlined:     */
/*   SaberScheduler (scheduler.cpp:25-116), StaticScheduler (129-146).     */
/* ------------------------------------------------------------------------ */
static int validate_cfg(const orc_sim_config* c) {
  if (c->window < 1) FAIL("window_size must be >= 1");
  if (!(c->tick > 0.0)) FAIL("tick must be > 0");
  if (c->mode == ORC_STATIC && c->cap < 1)
    FAIL("static mode requires a positive batch size");
  if (c->mode == ORC_SABER && !c->has_model)
    FAIL("saber mode requires a speed model");
  if (c->has_horizon && !(c->horizon > 0.0)) FAIL("horizon must be > 0");
  if (predict_i(&c->ground_truth, 1) <= 0.0)
    FAIL("engine ground truth must be positive");
  return 0;
}

static int simulate(const orc_sim_config* cfg, req_t* reqs, int n,
                    orc_traj_out* out, orc_record* records,
                    orc_decision* decisions, int64_t dec_cap, int64_t* n_dec) {
  double max_sla = 0.0;
  for (int i = 0; i < n; ++i) max_sla = smax(max_sla, reqs[i].sla);
  const double horizon = cfg->has_horizon
                             ? cfg->horizon
                             : reqs[n - 1].arrival + 10.0 * max_sla;

  engine_t eng;
  memset(&eng, 0, sizeof eng);
  eng.gt = cfg->ground_truth;
  eng.prefill_rate = cfg->prefill_rate;
  eng.slots = (slot_t*)malloc(sizeof(slot_t) * (size_t)n);
  completion_t* comps = (completion_t*)malloc(sizeof(completion_t) * (size_t)n);
  int* high = (int*)malloc(sizeof(int) * (size_t)n);
  int* low = (int*)malloc(sizeof(int) * (size_t)n);
  int* keep = (int*)malloc(sizeof(int) * (size_t)n);
  /* ledger: id -> frozen need (std::map; only membership/max matter). */
  double* ledger = (double*)malloc(sizeof(double) * (size_t)n);
  char* in_ledger = (char*)calloc((size_t)n, 1);
  int n_high = 0, low_head = 0, low_tail = 0, ledger_size = 0;

  declog_t L;
  memset(&L, 0, sizeof L);
  L.hash = ORC_HASH_SEED;
  L.buf = decisions;
  L.cap = dec_cap;

  mt64 rng;
  if (cfg->mode == ORC_SABER) mt_seed(&rng, cfg->seed ^ 0x9e3779b97f4a7c15ULL);
  const double ceiling =
      cfg->mode == ORC_SABER ? predict_i(&cfg->model, 1) : 0.0;

  int64_t ticks = 0, refresh_entries = 0, gate_cands = 0, ledger_scanned = 0,
          draws = 0;
  int next_arrival = 0, completed = 0;
  double t = 0.0;
  for (;;) {
    while (next_arrival < n && reqs[next_arrival].arrival <= t) {
      reqs[next_arrival].state = ST_HIGH;
      high[n_high++] = next_arrival;
      ++next_arrival;
    }
    ++ticks;
    const int load = eng.n_active;
    if (cfg->mode == ORC_SABER) {
      /* refresh_tiers (scheduler.cpp:38-55) */
      refresh_entries += n_high;
      int nk = 0;
      for (int q = 0; q < n_high; ++q) {
        const int id = high[q];
        const double need = required_speed(&reqs[id], t);
        if (need > ceiling) {
          reqs[id].state = ST_LOW;
          reqs[id].demoted = 1;
          low[low_tail++] = id;
          declog_push(&L, t, id, ORC_DEMOTE, load, 1, ceiling, 1, need);
        } else {
          keep[nk++] = id;
        }
      }
      memcpy(high, keep, sizeof(int) * (size_t)nk);
      n_high = nk;
      /* admission_step (scheduler.cpp:57-110) */
      if (n_high > 0) {
        const int window = cfg->window < n_high ? cfg->window : n_high;
        int order[1024];
        int* ord = window <= 1024 ? order : (int*)malloc(sizeof(int) * (size_t)window);
        for (int i = 0; i < window; ++i) ord[i] = i;
        for (int i = window - 1; i > 0; --i) {
          const int j = (int)(mt_next(&rng) % (uint64_t)(i + 1));
          ++draws;
          const int tmp = ord[i];
          ord[i] = ord[j];
          ord[j] = tmp;
        }
        const int ld = eng.n_active;
        const double pred = predict_i(&cfg->model, ld + 1);
        ledger_scanned += ledger_size;
        for (int c = 0; c < window; ++c) {
          const int pos = ord[c];
          const int id = high[pos];
          ++gate_cands;
          const double need = required_speed(&reqs[id], t);
          if (pred < need) {
            declog_push(&L, t, id, ORC_REJECT_OWN, ld, 1, pred, 1, need);
            continue;
          }
          int violates = 0;
          for (int k = 0; k < n && !violates; ++k)
            if (in_ledger[k] && pred < ledger[k]) violates = 1;
          if (violates) {
            declog_push(&L, t, id, ORC_REJECT_ACTIVE, ld, 1, pred, 1, need);
            continue;
          }
          engine_admit(&eng, reqs, id, t);
          in_ledger[id] = 1;
          ledger[id] = need;
          ++ledger_size;
          memmove(&high[pos], &high[pos + 1], sizeof(int) * (size_t)(n_high - pos - 1));
          --n_high;
          declog_push(&L, t, id, ORC_ADMIT_HIGH, ld, 1, pred, 1, need);
          break;
        }
        if (ord != order) free(ord);
      } else if (low_head < low_tail) {
        const int id = low[low_head++];
        const int ld = eng.n_active;
        const double need = required_speed(&reqs[id], t);
        engine_admit(&eng, reqs, id, t);
        declog_push(&L, t, id, ORC_ADMIT_LOW, ld, 0, 0.0, 1, need);
      }
    } else {
      /* static_step (scheduler.cpp:129-144) */
      int head = 0;
      while (eng.n_active < cfg->cap && head < n_high) {
        const int id = high[head++];
        const int ld = eng.n_active;
        engine_admit(&eng, reqs, id, t);
        declog_push(&L, t, id, ORC_ADMIT_HIGH, ld, 0, 0.0, 0, 0.0);
      }
      memmove(high, high + head, sizeof(int) * (size_t)(n_high - head));
      n_high -= head;
    }

    if (t >= horizon) break;
    const double next = smin(t + cfg->tick, horizon);
    const int nc = engine_advance(&eng, reqs, next, comps);
    for (int k = 0; k < nc; ++k) {
      ++completed;
      const int id = comps[k].id;
      if (in_ledger[id]) {
        in_ledger[id] = 0;
        --ledger_size;
      }
    }
    t = next;
    if (completed == n) break;
  }

  /* make_record + compute_metrics (metrics.cpp:17-30, 107-140). */
  memset(out, 0, sizeof *out);
  int64_t met = 0, n_ratio = 0, ncomp = 0;
  for (int i = 0; i < n; ++i) {
    const req_t* r = &reqs[i];
    const int has_c = !isnan(r->completion_time);
    const int m = has_c && r->completion_time - r->arrival <= r->sla;
    met += m;
    ncomp += has_c;
    if (r->task >= 0 && r->task < 4) {
      out->issued_by_task[r->task] += 1;
      out->met_by_task[r->task] += m;
    }
    if (records) {
      orc_record* rec = &records[i];
      rec->arrival_time = r->arrival;
      rec->admit_time = r->admit_time;
      rec->completion_time = r->completion_time;
      rec->sla = r->sla;
      rec->task = r->task;
      rec->input_tokens = r->in_tok;
      rec->max_output_tokens = r->out_tok;
      rec->demoted = r->demoted;
    }
  }
  out->goodput = (double)met / (double)n;
  double mean = 0.0;
  for (int i = 0; i < n; ++i) {
    const req_t* r = &reqs[i];
    if (isnan(r->completion_time)) continue;
    mean += (r->completion_time - r->arrival) / r->sla;
    ++n_ratio;
  }
  if (n_ratio == 0) {
    out->ratio_mean = out->ratio_std = out->cv = NAN;
  } else {
    mean /= (double)n_ratio;
    double var = 0.0;
    for (int i = 0; i < n; ++i) {
      const req_t* r = &reqs[i];
      if (isnan(r->completion_time)) continue;
      const double v = (r->completion_time - r->arrival) / r->sla;
      var += (v - mean) * (v - mean);
    }
    var /= (double)n_ratio;
    out->ratio_mean = mean;
    out->ratio_std = sqrt(var);
    out->cv = mean == 0.0 ? NAN : out->ratio_std / mean;
  }
  out->completed = ncomp;
  out->met = met;
  out->decisions = L.count;
  memcpy(out->n_kind, L.n_kind, sizeof L.n_kind);
  out->decision_hash = L.hash;
  out->ticks = ticks;
  out->passes = eng.passes;
  out->decode_updates = eng.decode_updates;
  out->prefill_updates = eng.prefill_updates;
  out->refresh_entries = refresh_entries;
  out->gate_candidates = gate_cands;
  out->ledger_scanned = ledger_scanned;
  out->rng_draws = draws;
  out->last_arrival = reqs[n - 1].arrival;
  out->horizon = horizon;
  if (n_dec) *n_dec = L.count;

  free(eng.slots);
  free(comps);
  free(high);
  free(low);
  free(keep);
  free(ledger);
  free(in_ledger);
  if (L.overflow) FAIL("decision buffer too small (%lld needed)", (long long)L.count);
  return 0;
}

static void init_req(req_t* r, const orc_request* s) {
  r->arrival = s->arrival_time;
  r->sla = s->sla_seconds;
  r->deadline = s->deadline;
  r->generated = 0.0;
  r->in_tok = s->input_tokens;
  r->out_tok = s->max_output_tokens;
  r->task = s->task;
  r->state = ST_PENDING;
  r->demoted = 0;
  r->admit_time = NAN;
  r->completion_time = NAN;
}

int orc_run_with_requests(const orc_sim_config* cfg, const orc_request* rq,
                          int32_t n, orc_traj_out* out, orc_record* records,
                          orc_decision* decisions, int64_t dec_cap,
                          int64_t* n_dec) {
  if (validate_cfg(cfg)) return 1;
  if (n < 1) FAIL("run: no requests");
  req_t* reqs = (req_t*)malloc(sizeof(req_t) * (size_t)n);
  for (int i = 0; i < n; ++i) init_req(&reqs[i], &rq[i]);
  const int rc = simulate(cfg, reqs, n, out, records, decisions, dec_cap, n_dec);
  free(reqs);
  return rc;
}

int orc_run(const orc_sim_config* cfg, orc_traj_out* out, orc_record* records,
            orc_decision* decisions, int64_t dec_cap, int64_t* n_dec) {
  if (validate_cfg(cfg)) return 1;
  const int n = cfg->num_requests;
  if (n < 1) FAIL("num_requests must be >= 1");
  orc_request* rq = (orc_request*)malloc(sizeof(orc_request) * (size_t)n);
  if (orc_generate(cfg, rq)) {
    free(rq);
    return 1;
  }
  const int rc =
      orc_run_with_requests(cfg, rq, n, out, records, decisions, dec_cap, n_dec);
  free(rq);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Fitting (estimator.cpp:33-375) and calibration (calibration.cpp:137-168).*/
/* ------------------------------------------------------------------------ */
typedef struct {
  const int32_t* load;
  const double* speed;
  int m;
} samples_t;

static double sse_of(int family, const double* p, const samples_t* S) {
  double sse = 0.0;
  for (int i = 0; i < S->m; ++i) {
    const double r = eval_model(family, p, S->load[i]) - S->speed[i];
    sse += r * r;
  }
  return sse;
}

static void project(int family, double peak, double* p) {
  if (family == ORC_USL) {
    p[0] = smax(p[0], 1e-9);
    p[1] = smax(p[1], 0.0);
    p[2] = smax(p[2], 0.0);
  } else {
    p[0] = sclamp(p[0], 1e-9, 2.0 * peak);
    p[1] = smax(p[1], 0.0);
    p[2] = sclamp(p[2], -1e4, 1e4);
  }
}

typedef struct {
  double p[3];
  double sse;
  int converged;
} lm_out;

/* levenberg_marquardt (estimator.cpp:54-169). */
static lm_out lm(int family, const double* start, double peak,
                 const samples_t* S) {
  const int np = 3;
  const int m = S->m;
  double th[3] = {start[0], start[1], start[2]};
  project(family, peak, th);
  double sse = sse_of(family, th, S);
  double lambda = 1e-3;
  int converged = 0;
  double* res = (double*)malloc(sizeof(double) * (size_t)m);
  double* jac = (double*)malloc(sizeof(double) * 3 * (size_t)m);
  for (int iter = 0; iter < 400; ++iter) {
    for (int i = 0; i < m; ++i)
      res[i] = eval_model(family, th, S->load[i]) - S->speed[i];
    for (int j = 0; j < np; ++j) {
      const double h = 1e-6 * smax(fabs(th[j]), 1e-3);
      double lo[3] = {th[0], th[1], th[2]}, hi[3] = {th[0], th[1], th[2]};
      lo[j] -= h;
      hi[j] += h;
      for (int i = 0; i < m; ++i)
        jac[i * 3 + j] = (eval_model(family, hi, S->load[i]) -
                          eval_model(family, lo, S->load[i])) /
                         (2.0 * h);
    }
    double a[3][3] = {{0}}, g[3] = {0};
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < np; ++j) {
        g[j] += jac[i * 3 + j] * res[i];
        for (int k = j; k < np; ++k) a[j][k] += jac[i * 3 + j] * jac[i * 3 + k];
      }
    for (int j = 0; j < np; ++j)
      for (int k = 0; k < j; ++k) a[j][k] = a[k][j];

    int stepped = 0;
    while (lambda <= 1e12) {
      double s[3][3], rhs[3];
      for (int j = 0; j < np; ++j) {
        for (int k = 0; k < np; ++k) s[j][k] = a[j][k];
        s[j][j] += lambda * smax(a[j][j], 1e-12);
        rhs[j] = -g[j];
      }
      int perm[3] = {0, 1, 2};
      int singular = 0;
      for (int col = 0; col < np; ++col) {
        int piv = col;
        for (int r = col + 1; r < np; ++r)
          if (fabs(s[perm[r]][col]) > fabs(s[perm[piv]][col])) piv = r;
        const int tp = perm[col];
        perm[col] = perm[piv];
        perm[piv] = tp;
        const double d = s[perm[col]][col];
        if (fabs(d) < 1e-300) {
          singular = 1;
          break;
        }
        for (int r = col + 1; r < np; ++r) {
          const double f = s[perm[r]][col] / d;
          for (int c = col; c < np; ++c) s[perm[r]][c] -= f * s[perm[col]][c];
          rhs[perm[r]] -= f * rhs[perm[col]];
        }
      }
      double delta[3] = {0, 0, 0};
      if (!singular) {
        for (int col = np - 1; col >= 0; --col) {
          double v = rhs[perm[col]];
          for (int c = col + 1; c < np; ++c) v -= s[perm[col]][c] * delta[c];
          delta[col] = v / s[perm[col]][col];
        }
      }
      double trial[3] = {th[0], th[1], th[2]};
      for (int j = 0; j < np; ++j) trial[j] += delta[j];
      project(family, peak, trial);
      const double trial_sse = singular ? INFINITY : sse_of(family, trial, S);
      if (trial_sse < sse) {
        double step = 0.0, scale = 1.0;
        for (int j = 0; j < np; ++j) {
          step = smax(step, fabs(trial[j] - th[j]));
          scale = smax(scale, fabs(trial[j]));
        }
        const double gain = sse - trial_sse;
        th[0] = trial[0];
        th[1] = trial[1];
        th[2] = trial[2];
        sse = trial_sse;
        lambda = smax(lambda / 3.0, 1e-12);
        stepped = 1;
        if (gain <= 1e-8 * (1.0 + sse) || step <= 1e-9 * scale) converged = 1;
        break;
      }
      lambda *= 4.0;
    }
    if (!stepped) converged = 1;
    if (converged) break;
  }
  free(res);
  free(jac);
  lm_out o = {{th[0], th[1], th[2]}, sse, converged};
  return o;
}

/* starting_points (estimator.cpp:171-206). */
static void starting_points(int family, const samples_t* S, double st[5][3]) {
  double vmax = 0.0;
  double lo = S->load[0], hi = S->load[0];
  for (int i = 0; i < S->m; ++i) {
    vmax = smax(vmax, S->speed[i]);
    lo = smin(lo, (double)S->load[i]);
    hi = smax(hi, (double)S->load[i]);
  }
  const double mid = 0.5 * (lo + hi);
  double half_load = mid, half_gap = INFINITY;
  for (int i = 0; i < S->m; ++i) {
    const double gap = fabs(S->speed[i] - 0.5 * vmax);
    if (gap < half_gap) {
      half_gap = gap;
      half_load = S->load[i];
    }
  }
  if (family == ORC_USL) {
    const double u[5][3] = {{vmax, 1e-3, 1e-6},
                            {vmax, 1e-2, 1e-4},
                            {vmax, 5e-2, 1e-3},
                            {vmax, 2e-1, 1e-3},
                            {1.1 * vmax, 5e-1, 1e-2}};
    memcpy(st, u, sizeof u);
  } else {
    const double l[5][3] = {{1.05 * vmax, 0.02, half_load},
                            {1.05 * vmax, 0.05, half_load},
                            {1.05 * vmax, 0.1, half_load},
                            {1.05 * vmax, 0.3, mid},
                            {1.5 * vmax, 1.0, half_load}};
    memcpy(st, l, sizeof l);
  }
}

/* r_squared_from_predictions (estimator.cpp:357-375). */
static double r_squared(int family, const double* p, const samples_t* S) {
  double mean = 0.0;
  for (int i = 0; i < S->m; ++i) mean += S->speed[i];
  mean /= (double)S->m;
  double ss_res = 0.0, ss_tot = 0.0;
  for (int i = 0; i < S->m; ++i) {
    const double pr = eval_model(family, p, S->load[i]);
    ss_res += (pr - S->speed[i]) * (pr - S->speed[i]);
    ss_tot += (S->speed[i] - mean) * (S->speed[i] - mean);
  }
  if (ss_tot == 0.0) return ss_res == 0.0 ? 1.0 : 0.0;
  return 1.0 - ss_res / ss_tot;
}

static int count_distinct(const int32_t* loads, int m) {
  /* loads are small positive ints in practice; sort a copy. */
  int32_t* c = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  memcpy(c, loads, sizeof(int32_t) * (size_t)m);
  for (int i = 1; i < m; ++i) { /* insertion sort: m is small */
    int32_t v = c[i];
    int j = i - 1;
    while (j >= 0 && c[j] > v) {
      c[j + 1] = c[j];
      --j;
    }
    c[j + 1] = v;
  }
  int d = 0;
  for (int i = 0; i < m; ++i)
    if (i == 0 || c[i] != c[i - 1]) ++d;
  free(c);
  return d;
}

/* fit (estimator.cpp:241-346).  Returns 0 ok / 1 FitError (fit_error=1). */
static int fit_impl(const samples_t* S, int family, double* params,
                    double* r2_or_sse) {
  const int need = family == ORC_LINEAR ? 2 : 3;
  if (S->m < need || count_distinct(S->load, S->m) < need) {
    params[0] = params[1] = params[2] = 0.0;
    *r2_or_sse = INFINITY;
    return 1;
  }
  double p[3] = {0, 0, 0};
  if (family == ORC_LINEAR) {
    /* fit_linear (estimator.cpp:208-230) */
    const double n = (double)S->m;
    double mx = 0.0, my = 0.0;
    for (int i = 0; i < S->m; ++i) {
      mx += S->load[i];
      my += S->speed[i];
    }
    mx /= n;
    my /= n;
    double sxx = 0.0, sxy = 0.0;
    for (int i = 0; i < S->m; ++i) {
      sxx += (S->load[i] - mx) * (S->load[i] - mx);
      sxy += (S->load[i] - mx) * (S->speed[i] - my);
    }
    const double a = sxy / sxx;
    const double b = my - a * mx;
    p[0] = a;
    p[1] = b;
    p[2] = 0.0;
    if (a > 0.0) {
      memcpy(params, p, sizeof p);
      *r2_or_sse = sse_of(ORC_LINEAR, p, S);
      return 1;
    }
  } else {
    double peak = 0.0;
    for (int i = 0; i < S->m; ++i) peak = smax(peak, S->speed[i]);
    double st[5][3];
    starting_points(family, S, st);
    lm_out best;
    best.sse = INFINITY;
    best.p[0] = best.p[1] = best.p[2] = 0.0;
    best.converged = 0;
    int any_conv = 0;
    for (int k = 0; k < 5; ++k) {
      const lm_out o = lm(family, st[k], peak, S);
      any_conv = any_conv || o.converged;
      if (o.sse < best.sse) best = o;
    }
    if (!any_conv || !isfinite(best.sse)) {
      memcpy(params, best.p, sizeof best.p);
      *r2_or_sse = best.sse;
      return 1;
    }
    /* polish_amplitude + consider + zero-snap (estimator.cpp:291-331). */
    for (int round = 0; round < 3; ++round) {
      double q[3] = {best.p[0], best.p[1], best.p[2]};
      if (round > 0) {
        const int j = round;
        if (!(best.p[j] != 0.0 && fabs(best.p[j]) <= 1e-7)) continue;
        q[j] = 0.0;
        project(family, peak, q);
      }
      double num = 0.0, den = 0.0;
      for (int i = 0; i < S->m; ++i) {
        const double unit[3] = {1.0, q[1], q[2]};
        const double shape = eval_model(family, unit, S->load[i]);
        num += shape * S->speed[i];
        den += shape * shape;
      }
      if (den > 0.0 && isfinite(num / den)) {
        q[0] = num / den;
        project(family, peak, q);
      }
      const double s2 = sse_of(family, q, S);
      if (s2 <= best.sse) {
        memcpy(best.p, q, sizeof q);
        best.sse = s2;
      }
    }
    memcpy(p, best.p, sizeof p);
  }
  if (family != ORC_USL) {
    double prev = eval_model(family, p, 1.0);
    for (int load = 2; load <= 1000; ++load) {
      const double cur = eval_model(family, p, (double)load);
      if (cur > prev + 1e-9 * smax(1.0, fabs(prev))) {
        memcpy(params, p, sizeof p);
        *r2_or_sse = sse_of(family, p, S);
        return 1;
      }
      prev = cur;
    }
  }
  memcpy(params, p, sizeof p);
  *r2_or_sse = r_squared(family, p, S);
  return 0;
}

int orc_fit(const int32_t* loads, const double* speeds, int32_t m,
            int32_t family, double* params, double* r2_or_sse,
            int32_t* fit_error) {
  samples_t S = {loads, speeds, m};
  *fit_error = fit_impl(&S, family, params, r2_or_sse);
  return 0;
}

int orc_calibrate(const int32_t* loads, const double* speeds, int32_t m,
                  int32_t* best_family, double* best_params, double* best_r2,
                  int32_t* ok, double* fam_params, double* fam_r2) {
  samples_t S = {loads, speeds, m};
  if (count_distinct(loads, m) < 3)
    FAIL("calibrate: insufficient distinct loads");
  int have = 0;
  double br2 = 0.0;
  for (int f = 0; f < 3; ++f) {
    double p[3], v;
    const int err = fit_impl(&S, f, p, &v);
    ok[f] = !err;
    memcpy(&fam_params[3 * f], p, sizeof p);
    fam_r2[f] = err ? NAN : v;
    if (!err && (!have || v > br2)) {
      have = 1;
      br2 = v;
      *best_family = f;
      memcpy(best_params, p, sizeof p);
      *best_r2 = v;
    }
  }
  if (!have) FAIL("calibrate: no model family produced a fit");
  return 0;
}

/* ------------------------------------------------------------------------ */
/* profile (calibration.cpp:58-135).                                        */
/* ------------------------------------------------------------------------ */
int orc_profile(const orc_model* gt, double prefill_rate, const orc_mix* mix,
                int32_t num_requests, uint64_t seed, double jitter,
                int32_t l_max, int32_t* loads, double* speeds, int64_t cap,
                int64_t* n_out) {
  if (l_max < 1) FAIL("profile: l_max must be >= 1");
  if (validate_mix(mix)) return 1;
  if (num_requests < 1) FAIL("profile: target sample count must be >= 1");
  mt64 rng;
  mt_seed(&rng, seed);
  /* plan bursts */
  int nb = 0, nb_cap = 16, issued = 0, size = 0;
  int(*bursts)[4] = malloc(sizeof(int[4]) * (size_t)nb_cap);
  while (issued < num_requests) {
    size = size % l_max + 1;
    const int task = sample_task(&rng, mix);
    const int in = jittered_length(&rng, kAvgIn[task], jitter);
    const int outl = jittered_length(&rng, kAvgOut[task], jitter);
    if (nb == nb_cap) {
      nb_cap *= 2;
      bursts = realloc(bursts, sizeof(int[4]) * (size_t)nb_cap);
    }
    bursts[nb][0] = size;
    bursts[nb][1] = task;
    bursts[nb][2] = in;
    bursts[nb][3] = outl;
    ++nb;
    issued += size;
  }
  req_t* reqs = (req_t*)malloc(sizeof(req_t) * (size_t)issued);
  engine_t eng;
  memset(&eng, 0, sizeof eng);
  eng.gt = *gt;
  eng.prefill_rate = prefill_rate;
  eng.slots = (slot_t*)malloc(sizeof(slot_t) * (size_t)issued);
  completion_t* comps = (completion_t*)malloc(sizeof(completion_t) * (size_t)issued);
  int n_req = 0;
  int64_t ns = 0;
  const int static_cap = 10 * l_max;
  for (int b = 0; b < nb; ++b) {
    const double now = eng.clock;
    const int first = n_req;
    for (int i = 0; i < bursts[b][0]; ++i) {
      req_t* r = &reqs[n_req++];
      memset(r, 0, sizeof *r);
      r->task = bursts[b][1];
      r->arrival = now;
      r->in_tok = bursts[b][2];
      r->out_tok = bursts[b][3];
      r->sla = kSla[r->task];
      r->deadline = now + kSla[r->task];
      r->admit_time = NAN;
      r->completion_time = NAN;
      r->state = ST_HIGH;
    }
    for (int id = first; id < n_req && eng.n_active < static_cap; ++id)
      engine_admit(&eng, reqs, id, now);
    while (eng.n_active > 0) {
      const int nc = engine_advance(&eng, reqs, eng.clock + 60.0, comps);
      for (int k = 0; k < nc; ++k) {
        if (ns < cap) {
          loads[ns] = (int32_t)llround(comps[k].mean_load);
          speeds[ns] = reqs[comps[k].id].out_tok / comps[k].duration;
        }
        ++ns;
      }
    }
  }
  free(bursts);
  free(reqs);
  free(eng.slots);
  free(comps);
  *n_out = ns;
  if (ns > cap) FAIL("profile: sample buffer too small (%lld)", (long long)ns);
  if (count_distinct(loads, (int)ns) < 3)
    FAIL("profile: insufficient distinct loads");
  return 0;
}

/* ------------------------------------------------------------------------ */
/* sweep (simloop.cpp:130-277), sequential.                                 */
/* ------------------------------------------------------------------------ */
static double mean_of(const double* v, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i];
  return s / (double)n;
}

static double cv_or_nan(const double* v, int64_t n) {
  if (n == 0) return NAN;
  double mean = 0.0;
  for (int64_t i = 0; i < n; ++i) mean += v[i];
  mean /= (double)n;
  if (mean == 0.0) return NAN;
  double var = 0.0;
  for (int64_t i = 0; i < n; ++i) var += (v[i] - mean) * (v[i] - mean);
  var /= (double)n;
  return sqrt(var) / mean;
}

int orc_sweep(const orc_sim_config* base, const int32_t* mix_ids,
              int32_t n_mixes, const double* rps, int32_t n_rps,
              const int32_t* caps, int32_t n_caps, int32_t with_saber,
              int32_t repeats, int32_t jobs, double* row_goodput,
              double* row_ratio_mean, double* row_ratio_std, double* row_cv,
              double* summary, int32_t* best_cap) {
  (void)jobs;
  if (n_mixes < 1 || n_rps < 1 || (n_caps < 1 && !with_saber))
    FAIL("sweep: empty grid");
  if (with_saber && !base->has_model)
    FAIL("sweep: saber variant requires a model");
  const int per_rps = n_caps * repeats + (with_saber ? repeats : 0);
  const int64_t n_rows = (int64_t)n_mixes * n_rps * per_rps;
  const int n = base->num_requests;
  double* ratios = (double*)malloc(sizeof(double) * (size_t)(n_rows * n));
  int64_t* n_ratios = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_rows);
  orc_record* rec = (orc_record*)malloc(sizeof(orc_record) * (size_t)n);
  int64_t idx = 0;
  for (int mi = 0; mi < n_mixes; ++mi)
    for (int ri = 0; ri < n_rps; ++ri)
      for (int v = 0; v < n_caps + (with_saber ? 1 : 0); ++v)
        for (int i = 0; i < repeats; ++i, ++idx) {
          orc_sim_config c = *base;
          if (orc_preset_mix(mix_ids[mi], &c.mix)) return 1;
          c.rps = rps[ri];
          c.workload_seed = base->seed + (uint64_t)i;
          c.seed = base->seed + (uint64_t)i;
          if (v < n_caps) {
            c.mode = ORC_STATIC;
            c.cap = caps[v];
            c.has_model = 0;
          } else {
            c.mode = ORC_SABER;
            c.cap = 0;
          }
          orc_traj_out o;
          if (orc_run(&c, &o, rec, NULL, 0, NULL)) return 1;
          row_goodput[idx] = o.goodput;
          row_ratio_mean[idx] = o.ratio_mean;
          row_ratio_std[idx] = o.ratio_std;
          row_cv[idx] = o.cv;
          int64_t k = 0;
          for (int q = 0; q < n; ++q)
            if (!isnan(rec[q].completion_time))
              ratios[idx * n + k++] =
                  (rec[q].completion_time - rec[q].arrival_time) / rec[q].sla;
          n_ratios[idx] = k;
        }
  /* per-mix summary */
  double* pool_s = (double*)malloc(sizeof(double) * (size_t)(n_rows * n + 1));
  double* pool_t = (double*)malloc(sizeof(double) * (size_t)(n_rows * n + 1));
  double* cell = (double*)malloc(sizeof(double) * (size_t)(repeats * n + 1));
  double* sm = (double*)malloc(sizeof(double) * (size_t)n_rps);
  double* tm = (double*)malloc(sizeof(double) * (size_t)n_rps);
  double* srm = (double*)malloc(sizeof(double) * (size_t)n_rps);
  double* trm = (double*)malloc(sizeof(double) * (size_t)n_rps);
  double* gs = (double*)malloc(sizeof(double) * (size_t)((n_caps + 1) * repeats + 1));
  for (int mi = 0; mi < n_mixes; ++mi) {
    int64_t ps = 0, pt = 0;
    int nsm = 0, ntm = 0, nsrm = 0, ntrm = 0;
    for (int ri = 0; ri < n_rps; ++ri) {
      const int64_t base_row = ((int64_t)mi * n_rps + ri) * per_rps;
      if (n_caps > 0) {
        /* std::map<int,...> iterates caps ascending; ties keep the smaller. */
        int order[4096];
        for (int v = 0; v < n_caps; ++v) order[v] = v;
        for (int a = 1; a < n_caps; ++a) {
          int x = order[a], b = a - 1;
          while (b >= 0 && caps[order[b]] > caps[x]) {
            order[b + 1] = order[b];
            --b;
          }
          order[b + 1] = x;
        }
        int bcap = 0, bv = -1;
        double bmean = -1.0;
        for (int a = 0; a < n_caps; ++a) {
          const int v = order[a];
          if (a > 0 && caps[order[a - 1]] == caps[v]) continue; /* merged key */
          int ng = 0;
          for (int w = 0; w < n_caps; ++w)
            if (caps[w] == caps[v])
              for (int i = 0; i < repeats; ++i)
                gs[ng++] = row_goodput[base_row + (int64_t)w * repeats + i];
          const double mval = mean_of(gs, ng);
          if (mval > bmean) {
            bmean = mval;
            bcap = caps[v];
            bv = v;
          }
        }
        best_cap[mi * n_rps + ri] = bcap;
        tm[ntm++] = bmean;
        int64_t nc = 0;
        for (int w = 0; w < n_caps; ++w) {
          if (caps[w] != caps[bv]) continue;
          for (int i = 0; i < repeats; ++i) {
            const int64_t r = base_row + (int64_t)w * repeats + i;
            for (int64_t q = 0; q < n_ratios[r]; ++q) {
              pool_t[pt++] = ratios[r * n + q];
              cell[nc++] = ratios[r * n + q];
            }
          }
        }
        if (nc > 0) trm[ntrm++] = mean_of(cell, nc);
      } else {
        best_cap[mi * n_rps + ri] = 0;
      }
      if (with_saber) {
        int64_t nc = 0;
        for (int i = 0; i < repeats; ++i) {
          const int64_t r = base_row + (int64_t)n_caps * repeats + i;
          gs[i] = row_goodput[r];
          for (int64_t q = 0; q < n_ratios[r]; ++q) {
            pool_s[ps++] = ratios[r * n + q];
            cell[nc++] = ratios[r * n + q];
          }
        }
        sm[nsm++] = mean_of(gs, repeats);
        if (nc > 0) srm[nsrm++] = mean_of(cell, nc);
      }
    }
    double* s = &summary[mi * 7];
    s[0] = nsm ? mean_of(sm, nsm) : NAN;
    s[1] = ntm ? mean_of(tm, ntm) : NAN;
    s[2] = s[0] - s[1];
    s[3] = cv_or_nan(pool_s, ps);
    s[4] = cv_or_nan(pool_t, pt);
    s[5] = cv_or_nan(srm, nsrm);
    s[6] = cv_or_nan(trm, ntrm);
  }
  free(ratios);
  free(n_ratios);
  free(rec);
  free(pool_s);
  free(pool_t);
  free(cell);
  free(sm);
  free(tm);
  free(srm);
  free(trm);
  free(gs);
  return 0;
}
