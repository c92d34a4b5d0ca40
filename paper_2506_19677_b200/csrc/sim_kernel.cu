// sim_kernel.cu — the trajectory engine (K1) and its per-row metrics epilogue
// (K2) for sm_100a.
//
// One LANE owns one trajectory: a persistent grid pulls
// trajectory indices from a warp-aggregated atomic work queue, and each lane
// runs the reference's tick loop (simloop.cpp:78-101) for its trajectory:
//   arrivals -> refresh_tiers -> admission_step | static_step  (scheduler.cpp)
//   -> Engine::advance_to (engine.cpp:51-127) -> completions.
// 32 trajectories share a warp's instruction stream, so per-tick scheduler
// logic costs ~1/32 of an issue slot per trajectory instead of a whole warp.
//
// Bit-exactness with the reference: compiled with --fmad=false
// (the reference has no FMA); every floating-point expression keeps
// the reference's operand order; predict() comes from host-built tables
// (SURVEY F6); the scheduler RNG from precomputed mt19937_64 streams
// (SURVEY F2).  Two exact algebraic rewrites remove per-slot divides:
//   * min_i fl(rem_i / speed) == fl(min_i rem_i / speed), because correctly
//     rounded division by a positive constant is monotone;
//   * a high-tier request cannot demote before demote_after[i], a safe lower
//     bound (prologue.cu), so refresh only scans when one might.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "saber_internal.h"

namespace cg = cooperative_groups;

namespace saberb200 {
namespace {

constexpr double kInf = __builtin_huge_val();
constexpr double kOnePlusTol = 1.0 + 1e-12;  // engine.cpp:17,76 (kGroupTol)
constexpr uint64_t kHashSeed = 0x243F6A8885A308D3ULL;
constexpr uint64_t kAbsent = 0xFFF8000000000001ULL;
constexpr int kBlock = 128;

__device__ __forceinline__ uint64_t hstep(uint64_t h, uint64_t x) {
  h ^= x;
  h *= 0x9E3779B97F4A7C15ULL;
  h ^= h >> 32;
  return h;
}
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}
__device__ __forceinline__ uint64_t dbits(double v) {
  return static_cast<uint64_t>(__double_as_longlong(v));
}

// required_speed (types.cpp:82-88) for a queued request: generated == 0.
__device__ __forceinline__ double queued_need(double max_out, double deadline,
                                              double now) {
  if (now >= deadline) return kInf;
  const double remaining = max_out - 0.0;
  if (remaining <= 0.0) return 0.0;
  return remaining / (deadline - now);
}

// Per-request tier membership as an NW x 64-bit register bitmask.  All word
// indices are resolved through unrolled selects so nothing spills to local
// memory.
template <int NW>
struct Mask {
  uint64_t w[NW];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = 0;
  }
  __device__ __forceinline__ void set(int id) {
#pragma unroll
    for (int i = 0; i < NW; ++i)
      if (i == (id >> 6)) w[i] |= 1ull << (id & 63);
  }
  __device__ __forceinline__ void reset(int id) {
#pragma unroll
    for (int i = 0; i < NW; ++i)
      if (i == (id >> 6)) w[i] &= ~(1ull << (id & 63));
  }
  __device__ __forceinline__ bool test(int id) const {
    bool r = false;
#pragma unroll
    for (int i = 0; i < NW; ++i)
      if (i == (id >> 6)) r = (w[i] >> (id & 63)) & 1ull;
    return r;
  }
  __device__ __forceinline__ bool any() const {
    uint64_t a = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) a |= w[i];
    return a != 0;
  }
  __device__ __forceinline__ int count() const {
    int c = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) c += __popcll(w[i]);
    return c;
  }
  __device__ __forceinline__ int lowest() const {
    int r = -1;
#pragma unroll
    for (int i = NW - 1; i >= 0; --i)
      if (w[i]) r = i * 64 + __ffsll(static_cast<long long>(w[i])) - 1;
    return r;
  }
  // k-th set bit in ascending id order (0-based); k < count().
  __device__ __forceinline__ int select(int k) const {
    int r = -1;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const int c = __popcll(w[i]);
      if (r < 0 && k < c) {
        uint64_t x = w[i];
        for (int j = 0; j < k; ++j) x &= x - 1;
        r = i * 64 + __ffsll(static_cast<long long>(x)) - 1;
      }
      if (r < 0) k -= c;
    }
    return r;
  }
};

struct DecisionLog {
  uint64_t h;
  int32_t n;
  int32_t k0, k1, k2, k3, k4;
};

template <bool kTrace>
__device__ __forceinline__ void push_decision(DecisionLog& L, double t, int id,
                                              int kind, int load, uint64_t pb,
                                              uint64_t rb, saber_decision* tr,
                                              int64_t cap, int32_t* err) {
  const uint64_t w = static_cast<uint64_t>(static_cast<uint32_t>(id)) |
                     (static_cast<uint64_t>(kind) << 32) |
                     (static_cast<uint64_t>(static_cast<uint32_t>(load)) << 40);
  L.h = hstep(L.h, dbits(t));
  L.h = hstep(L.h, w ^ rotl64(pb, 17) ^ rotl64(rb, 43));
  if (kTrace && tr != nullptr) {
    if (L.n < cap) {
      saber_decision& d = tr[L.n];
      d.time = t;
      d.request_id = static_cast<uint64_t>(id);
      d.kind = kind;
      d.load_before = load;
      d.has_pred = pb != kAbsent;
      d.has_req = rb != kAbsent;
      d.pred_speed = pb != kAbsent ? __longlong_as_double(static_cast<long long>(pb)) : nan("");
      d.req_speed = rb != kAbsent ? __longlong_as_double(static_cast<long long>(rb)) : nan("");
    } else {
      atomicCAS(err, kErrNone, kErrTraceOverflow);
    }
  }
  ++L.n;
  L.k0 += kind == 0;
  L.k1 += kind == 1;
  L.k2 += kind == 2;
  L.k3 += kind == 3;
  L.k4 += kind == 4;
}

// Simulates trajectory `ti` on this lane.  G/M/SID are the lane's slot arrays
// (stride 32), LNEED/LOW its ledger and low-tier FIFO (stride 32).
template <int NW, bool kTrace, bool kRecords>
__device__ __forceinline__ void simulate_one(const SimParams& P, int ti,
                                             double* __restrict__ G,
                                             double* __restrict__ M,
                                             uint16_t* __restrict__ SID,
                                             double* __restrict__ LNEED,
                                             uint16_t* __restrict__ LOW) {
  const TrajDesc d = P.traj[ti];
  const int n = d.n;
  const int nmax = P.wl.nmax;
  const int64_t wo = static_cast<int64_t>(d.workload) * nmax;
  const double* __restrict__ ARR = P.wl.arrival + wo;
  const double* __restrict__ DL = P.wl.deadline + wo;
  const double* __restrict__ MO = P.wl.max_out + wo;
  const double* __restrict__ IN = P.wl.input + wo;
  const double* __restrict__ DEM = P.wl.demote_after + wo;
  const double* __restrict__ GT = P.tables + d.gt_tab;
  const bool saber = d.mode == SABER_MODE_SABER;
  const double* __restrict__ MT = P.tables + (saber ? d.model_tab : d.gt_tab);
  const double horizon = isnan(d.horizon) ? P.wl.horizon[d.workload] : d.horizon;
  const double tick = d.tick;
  const double pr = d.prefill_rate;
  const double ceiling = saber ? MT[1] : 0.0;  // max_speed = predict(model, 1)
  const uint32_t* __restrict__ draws =
      saber ? P.rng.draws + P.rng.off[d.stream] : nullptr;
  const int64_t draw_len = saber ? P.rng.len[d.stream] : 0;
  double* __restrict__ COMP = P.out.completion + d.row * nmax;
  double* __restrict__ ADM = kRecords && P.out.admit ? P.out.admit + d.row * nmax : nullptr;
  uint8_t* __restrict__ DEMO =
      kRecords && P.out.demoted ? P.out.demoted + d.row * nmax : nullptr;
  saber_decision* tr = kTrace && P.out.trace ? P.out.trace + d.row * P.out.trace_cap : nullptr;

  Mask<NW> high, ledger;
  high.clear();
  ledger.clear();
  int ledger_size = 0;
  double ledger_max = -kInf;
  double min_td = kInf;  // lower bound on the earliest possible demotion
  int low_head = 0, low_tail = 0;

  int A = 0;  // |active|
  double clock = 0.0;
  double min_pf = kInf, min_rem = kInf;

  int next = 0;
  double na_t = n > 0 ? ARR[0] : kInf;
  int completed = 0;
  int64_t draw_pos = 0;
  bool failed = false;

  DecisionLog L{kHashSeed, 0, 0, 0, 0, 0, 0};
  int32_t ticks = 0, passes = 0, decode_updates = 0, prefill_updates = 0;
  int32_t refresh_entries = 0, cands = 0, ledger_scanned = 0, rng_draws = 0;

  // Engine::admit (engine.cpp:26-49), slot appended in admit order.
  auto admit = [&](int id, double now) {
    const double pl = pr > 0.0 ? IN[id] / pr : 0.0;
    const double m = MO[id];
    if (pl == 0.0) {
      G[A * kWarp] = 0.0;  // decode starts at admission
      min_rem = fmin(min_rem, m - 0.0);
    } else {
      G[A * kWarp] = -pl;
      min_pf = fmin(min_pf, pl);
    }
    M[A * kWarp] = m;
    SID[A * kWarp] = static_cast<uint16_t>(id);
    ++A;
    if (kRecords && ADM) ADM[id] = now;
  };

  double t = 0.0;
  for (;;) {
    // Arrivals due at t (simloop.cpp:79-85): arrival times strictly increase.
    while (na_t <= t) {
      high.set(next);
      if (saber) min_td = fmin(min_td, DEM[next]);
      ++next;
      na_t = next < n ? ARR[next] : kInf;
    }
    ++ticks;
    const int load = A;
    if (saber) {
      const int hc = high.count();
      refresh_entries += hc;
      // refresh_tiers (scheduler.cpp:38-55): scan in queue (= id) order only
      // when some entry may have crossed its demotion bound.
      if (hc > 0 && t >= min_td) {
        double nm = kInf;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          uint64_t b = high.w[i];
          while (b) {
            const int bit = __ffsll(static_cast<long long>(b)) - 1;
            b &= b - 1;
            const int id = i * 64 + bit;
            const double T = DEM[id];
            bool demote = false;
            if (t >= T) {
              const double need = queued_need(MO[id], DL[id], t);
              if (need > ceiling) {
                demote = true;
                high.w[i] &= ~(1ull << bit);
                LOW[low_tail * kWarp] = static_cast<uint16_t>(id);
                ++low_tail;
                push_decision<kTrace>(L, t, id, SABER_DEMOTE, load, dbits(ceiling),
                                      dbits(need), tr, P.out.trace_cap, P.out.error);
                if (kRecords && DEMO) DEMO[id] = 1;
              }
            }
            if (!demote) nm = fmin(nm, T);
          }
        }
        min_td = nm;
      }
      if (high.any()) {
        // admission_step, high tier (scheduler.cpp:58-95).
        const int hcount = high.count();
        const int w = d.window < hcount ? d.window : hcount;
        uint64_t ord = 0xFEDCBA9876543210ull;  // window positions as nibbles
#pragma unroll
        for (int i = kMaxWindow - 1; i >= 1; --i) {
          if (i < w) {
            if (draw_pos >= draw_len) {
              failed = true;
            } else {
              const uint32_t x = draws[draw_pos++];
              const uint32_t j = x % static_cast<uint32_t>(i + 1);  // rng() % (i+1)
              const uint64_t a = (ord >> (4 * i)) & 15ull;
              const uint64_t bb = (ord >> (4 * j)) & 15ull;
              const uint64_t x2 = a ^ bb;
              ord ^= (x2 << (4 * i)) | (x2 << (4 * j));
            }
          }
        }
        if (failed) break;
        rng_draws += w - 1;
        const double pred = MT[load + 1];
        const bool violates = pred < ledger_max;  // ActiveLedger::violates
        ledger_scanned += ledger_size;
        for (int c = 0; c < w; ++c) {
          const int pos = static_cast<int>((ord >> (4 * c)) & 15ull);
          const int id = high.select(pos);
          ++cands;
          const double need = queued_need(MO[id], DL[id], t);
          if (pred < need) {
            push_decision<kTrace>(L, t, id, SABER_REJECT_OWN, load, dbits(pred),
                                  dbits(need), tr, P.out.trace_cap, P.out.error);
            continue;
          }
          if (violates) {
            push_decision<kTrace>(L, t, id, SABER_REJECT_ACTIVE, load, dbits(pred),
                                  dbits(need), tr, P.out.trace_cap, P.out.error);
            continue;
          }
          admit(id, t);
          ledger.set(id);
          ++ledger_size;
          LNEED[id * kWarp] = need;
          ledger_max = (ledger_max < need) ? need : ledger_max;
          high.reset(id);
          push_decision<kTrace>(L, t, id, SABER_ADMIT_HIGH, load, dbits(pred),
                                dbits(need), tr, P.out.trace_cap, P.out.error);
          break;
        }
      } else if (low_head < low_tail) {
        // admission_step, low tier (scheduler.cpp:97-108).
        const int id = LOW[low_head * kWarp];
        ++low_head;
        const double need = queued_need(MO[id], DL[id], t);
        admit(id, t);
        push_decision<kTrace>(L, t, id, SABER_ADMIT_LOW, load, kAbsent, dbits(need),
                              tr, P.out.trace_cap, P.out.error);
      }
    } else {
      // StaticScheduler::static_step (scheduler.cpp:129-144).
      while (A < d.cap && high.any()) {
        const int id = high.lowest();
        high.reset(id);
        const int before = A;
        admit(id, t);
        push_decision<kTrace>(L, t, id, SABER_ADMIT_HIGH, before, kAbsent, kAbsent,
                              tr, P.out.trace_cap, P.out.error);
      }
    }

    if (t >= horizon) break;
    const double nt = (horizon < t + tick) ? horizon : t + tick;

    // Engine::advance_to(nt) (engine.cpp:51-127).
    bool ledger_dirty = false;
    while (clock < nt) {
      if (A == 0) {
        clock = nt;
        break;
      }
      ++passes;
      const double speed = GT[A];
      double dt = nt - clock;
      if (min_pf < dt) dt = min_pf;
      const double bnd = min_rem / speed;
      if (bnd < dt) dt = bnd;
      const double group = dt * kOnePlusTol;
      const double sdt = speed * dt;
      const double sgd = speed * (group - dt);
      const double nclock = clock + dt;
      double npf = kInf, nrem = kInf;
      int j = 0;
      decode_updates += A;
      for (int k = 0; k < A; ++k) {
        double g = G[k * kWarp];
        const double m = M[k * kWarp];
        bool done;
        if (g < 0.0) {  // prefill slot: g = -prefill_left
          ++prefill_updates;
          if (-g <= group) {
            g = 0.0;  // decode starts at nclock
            done = g + sgd >= m;
          } else {
            g = g + dt;  // == -(prefill_left - dt), exactly
            npf = fmin(npf, -g);
            done = false;
          }
        } else {
          g = g + sdt;
          done = g + sgd >= m;
        }
        if (!done) {
          if (g >= 0.0) nrem = fmin(nrem, m - g);
          G[j * kWarp] = g;
          if (j != k) {
            M[j * kWarp] = m;
            SID[j * kWarp] = SID[k * kWarp];
          }
          ++j;
        } else {
          const int id = SID[k * kWarp];
          COMP[id] = nclock;
          ++completed;
          if (saber && ledger.test(id)) {
            ledger.reset(id);
            --ledger_size;
            ledger_dirty = true;
          }
        }
      }
      A = j;
      clock = nclock;
      min_pf = npf;
      min_rem = nrem;
    }
    if (ledger_dirty) {
      double mx = -kInf;
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        uint64_t b = ledger.w[i];
        while (b) {
          const int id = i * 64 + __ffsll(static_cast<long long>(b)) - 1;
          b &= b - 1;
          const double v = LNEED[id * kWarp];
          mx = (mx < v) ? v : mx;
        }
      }
      ledger_max = mx;
    }
    t = nt;
    if (completed == n) break;
  }
  decode_updates -= prefill_updates;

  if (failed) atomicCAS(P.out.error, kErrNone, kErrRngExhausted);
  saber_traj_row* R = P.out.rows + d.row;
  R->n = n;
  R->decisions = L.n;
  R->n_kind[0] = L.k0;
  R->n_kind[1] = L.k1;
  R->n_kind[2] = L.k2;
  R->n_kind[3] = L.k3;
  R->n_kind[4] = L.k4;
  R->decision_hash = L.h;
  R->ticks = ticks;
  R->passes = passes;
  R->decode_updates = decode_updates;
  R->prefill_updates = prefill_updates;
  R->refresh_entries = refresh_entries;
  R->gate_candidates = cands;
  R->ledger_scanned = ledger_scanned;
  R->rng_draws = rng_draws;
  R->last_arrival = n > 0 ? ARR[n - 1] : 0.0;
  R->horizon = horizon;
  if (kTrace && P.out.trace_count) P.out.trace_count[d.row] = L.n;
}

template <int NW, bool kTrace, bool kRecords>
__global__ void __launch_bounds__(kBlock) sim_kernel(const SimParams P) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t S = P.scratch.slots;
  const int64_t sb = warp_global * S * kWarp + lane;
  const int64_t nb = warp_global * static_cast<int64_t>(P.wl.nmax) * kWarp + lane;
  double* G = P.scratch.slot_g + sb;
  double* M = P.scratch.slot_m + sb;
  uint16_t* SID = P.scratch.slot_id + sb;
  double* LNEED = P.scratch.ledger_need + nb;
  uint16_t* LOW = P.scratch.low_fifo + nb;
  for (;;) {
    int ti;
    {
      cg::coalesced_group g = cg::coalesced_threads();
      int base = 0;
      if (g.thread_rank() == 0) base = atomicAdd(P.next_traj, static_cast<int>(g.size()));
      base = g.shfl(base, 0);
      ti = base + static_cast<int>(g.thread_rank());
    }
    if (ti >= P.n_traj) break;
    simulate_one<NW, kTrace, kRecords>(P, ti, G, M, SID, LNEED, LOW);
  }
}

// K2: per-row metrics (make_record + compute_metrics, metrics.cpp:17-140).
// Sequential sums in request-id order, exactly as the reference.
__global__ void __launch_bounds__(128) row_metrics_kernel(const RowMetricsParams p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_traj) return;
  const TrajDesc d = p.traj[i];
  const int nmax = p.wl.nmax;
  const int64_t wo = static_cast<int64_t>(d.workload) * nmax;
  const double* C = p.completion + d.row * nmax;
  const double* ARR = p.wl.arrival + wo;
  const double* SLA = p.wl.sla + wo;
  const int8_t* TASK = p.wl.task + wo;
  int64_t met = 0, comp = 0;
  int64_t issued[4] = {0, 0, 0, 0}, metk[4] = {0, 0, 0, 0};
  double sum = 0.0;
  for (int q = 0; q < d.n; ++q) {
    const double c = C[q];
    const bool has = !isnan(c);
    const bool m = has && c - ARR[q] <= SLA[q];
    met += m;
    comp += has;
    const int tk = TASK[q];
    if (tk >= 0 && tk < 4) {
      issued[tk] += 1;
      metk[tk] += m;
    }
    if (has) sum += (c - ARR[q]) / SLA[q];
  }
  saber_traj_row* R = p.rows + d.row;
  R->goodput = static_cast<double>(met) / static_cast<double>(d.n);
  R->completed = comp;
  R->met = met;
  for (int k = 0; k < 4; ++k) {
    R->issued_by_task[k] = issued[k];
    R->met_by_task[k] = metk[k];
  }
  if (comp == 0) {
    R->ratio_mean = R->ratio_std = R->cv = nan("");
    return;
  }
  const double mean = sum / static_cast<double>(comp);
  double var = 0.0;
  for (int q = 0; q < d.n; ++q) {
    const double c = C[q];
    if (isnan(c)) continue;
    const double v = (c - ARR[q]) / SLA[q];
    var += (v - mean) * (v - mean);
  }
  var /= static_cast<double>(comp);
  R->ratio_mean = mean;
  R->ratio_std = sqrt(var);
  R->cv = mean == 0.0 ? nan("") : R->ratio_std / mean;
}

template <int NW>
int launch_nw(const SimParams& p, bool trace, bool records, int grid, cudaStream_t s) {
  if (trace)
    sim_kernel<NW, true, true><<<grid, kBlock, 0, s>>>(p);
  else if (records)
    sim_kernel<NW, false, true><<<grid, kBlock, 0, s>>>(p);
  else
    sim_kernel<NW, false, false><<<grid, kBlock, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <int NW>
int occ_nw(int* blocks) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, sim_kernel<NW, false, false>,
                                                       kBlock, 0) == cudaSuccess
             ? 0
             : 1;
}

}  // namespace

int sim_occupancy_grid(int nwords, int block, int* grid) {
  (void)block;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
  int rc = 1;
  switch (nwords) {
    case 1: rc = occ_nw<1>(&per_sm); break;
    case 2: rc = occ_nw<2>(&per_sm); break;
    case 4: rc = occ_nw<4>(&per_sm); break;
    case 8: rc = occ_nw<8>(&per_sm); break;
  }
  if (rc) return rc;
  *grid = sms * (per_sm > 0 ? per_sm : 1);
  return 0;
}

int launch_sim(const SimParams& p, int nwords, int grid, int block, void* stream) {
  (void)block;
  const bool trace = p.out.trace != nullptr;
  const bool records = p.out.admit != nullptr || p.out.demoted != nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (nwords) {
    case 1: return launch_nw<1>(p, trace, records, grid, s);
    case 2: return launch_nw<2>(p, trace, records, grid, s);
    case 4: return launch_nw<4>(p, trace, records, grid, s);
    case 8: return launch_nw<8>(p, trace, records, grid, s);
  }
  return 1;
}

int launch_row_metrics(const RowMetricsParams& p, void* stream) {
  if (p.n_traj == 0) return 0;
  const int block = 128;
  const int grid = (p.n_traj + block - 1) / block;
  row_metrics_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
