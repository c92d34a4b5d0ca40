// sim_lane.cu — lane-per-trajectory lockstep variant of the trajectory engine.
//
// Each LANE owns one trajectory; the warp's single loop executes ONE TICK of
// every lane's trajectory per iteration (simloop.cpp:78-101), so the
// scheduler's scalar work — arrivals, refresh_tiers, the Fisher-Yates window,
// the gate, the decision hash — is issued once per 32 trajectories.  When a
// lane's trajectory ends it writes its row and pulls the next index from the
// work queue inside the same loop, so lanes never wait for the warp's slowest
// trajectory (only at the very end of the queue).
//
// The lane's engine slots live in shared memory, [slot][lane] interleaved:
// g (f64: generated tokens, or -prefill_left while prefilling) and
// (max_output_tokens << 9 | id) (u32).  Every pass is the reference's full
// update with completion detection and the exact next-event minima
// (engine.cpp:55-125), with the order-preserving erase done inline by a write
// index; the arithmetic and exactness rules are those of sim_kernel.cu
// (DESIGN.md §3).  Used for n <= 128 and max_output_tokens < 2^23; larger
// trajectories take the group kernel.
#include <cooperative_groups.h>

#include "sim_common.cuh"

namespace cg = cooperative_groups;

namespace saberb200 {
namespace {

using namespace simdev;

constexpr int kLaneBlock = 32;  // one warp per block: shared memory is allotted per warp

template <int NW, bool kTrace, bool kRecords>
__global__ void __launch_bounds__(kLaneBlock) sim_lane_kernel(const SimParams P) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint32_t INV[kMaxWindow + 1];  // ceil(2^32 / d), d = 2..16
  const int lane = threadIdx.x;
  if (lane >= 2 && lane <= kMaxWindow)
    INV[lane] = static_cast<uint32_t>((0x100000000ull + lane - 1) / lane);
  __syncwarp();
  const int S = P.slot_rows;  // slots per lane (= nmax)
  double* SG = reinterpret_cast<double*>(smem_raw) + lane;
  uint32_t* SM = reinterpret_cast<uint32_t*>(smem_raw + static_cast<size_t>(S) * kWarp * 8) + lane;
  const int nmax = P.wl.nmax;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * kLaneBlock + lane;
  double* __restrict__ LNEED = P.scratch.ledger_need + gid * nmax;
  uint16_t* __restrict__ LOW = P.scratch.low_fifo + gid * nmax;

  // ---- trajectory state (registers) ----
  TrajDesc d;
  int n = 0, ti = 0;
  const double* ARR = nullptr;
  const double* DL = nullptr;
  const double* MO = nullptr;
  const double* IN = nullptr;
  const double* DEM = nullptr;
  const double* GT = nullptr;
  const double* MT = nullptr;
  const uint32_t* draws = nullptr;
  double* COMP = nullptr;
  bool saber = false;
  double horizon = 0.0, ceiling = 0.0;
  int64_t draw_len = 0, draw_pos = 0;
  Mask<NW> high, ledger;
  int ledger_size = 0, low_head = 0, low_tail = 0, A = 0, next = 0, completed = 0;
  double ledger_max = -kInf, min_td = kInf, clock = 0.0, min_pf = kInf, min_rem = kInf;
  double na_t = kInf, t = 0.0;
  bool failed = false;
  DecisionLog L{kHashSeed, 0, 0, 0, 0, 0, 0};
  int32_t ticks = 0, passes = 0, decode_updates = 0, prefill_updates = 0;
  int32_t refresh_entries = 0, cands = 0, ledger_scanned = 0, rng_draws = 0;

  auto fetch = [&]() -> bool {
    cg::coalesced_group g = cg::coalesced_threads();
    int base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(P.next_traj, static_cast<int>(g.size()));
    base = g.shfl(base, 0);
    ti = base + static_cast<int>(g.thread_rank());
    if (ti >= P.n_traj) return false;
    d = P.traj[P.order ? P.order[ti] : ti];
    n = d.n;
    const int64_t wo = static_cast<int64_t>(d.workload) * nmax;
    ARR = P.wl.arrival + wo;
    DL = P.wl.deadline + wo;
    MO = P.wl.max_out + wo;
    IN = P.wl.input + wo;
    DEM = P.wl.demote_after + wo;
    GT = P.tables + d.gt_tab;
    saber = d.mode == SABER_MODE_SABER;
    MT = P.tables + (saber ? d.model_tab : d.gt_tab);
    horizon = isnan(d.horizon) ? P.wl.horizon[d.workload] : d.horizon;
    ceiling = saber ? MT[1] : 0.0;
    draws = saber ? P.rng.draws + P.rng.off[d.stream] : nullptr;
    draw_len = saber ? P.rng.len[d.stream] : 0;
    draw_pos = 0;
    COMP = P.out.completion + d.row * nmax;
    high.clear();
    ledger.clear();
    ledger_size = low_head = low_tail = A = next = completed = 0;
    ledger_max = -kInf;
    min_td = kInf;
    clock = 0.0;
    min_pf = min_rem = kInf;
    na_t = n > 0 ? ARR[0] : kInf;
    t = 0.0;
    failed = false;
    L = DecisionLog{kHashSeed, 0, 0, 0, 0, 0, 0};
    ticks = passes = decode_updates = prefill_updates = 0;
    refresh_entries = cands = ledger_scanned = rng_draws = 0;
    return true;
  };

  auto finish = [&]() {
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
  };

  // Engine::admit (engine.cpp:26-49): append slot A.
  auto admit = [&](int id, double now) {
    const double pl = d.prefill_rate > 0.0 ? IN[id] / d.prefill_rate : 0.0;
    const double m = MO[id];
    if (pl == 0.0) {
      SG[A * kWarp] = 0.0;  // decode starts at admission
      min_rem = dmin(min_rem, m - 0.0);
    } else {
      SG[A * kWarp] = -pl;
      min_pf = dmin(min_pf, pl);
    }
    SM[A * kWarp] = (static_cast<uint32_t>(m) << 9) | static_cast<uint32_t>(id);
    ++A;
    if (kRecords && P.out.admit) P.out.admit[d.row * nmax + id] = now;
  };

  if (!fetch()) return;
  for (;;) {
    saber_decision* tr = kTrace && P.out.trace ? P.out.trace + d.row * P.out.trace_cap : nullptr;
    bool ended = false;
    // ---- scheduler step at t ----
    while (na_t <= t) {  // arrivals (simloop.cpp:79-85)
      high.set(next);
      if (saber) min_td = dmin(min_td, DEM[next]);
      ++next;
      na_t = next < n ? ARR[next] : kInf;
    }
    ++ticks;
    const int load = A;
    if (saber) {
      const int hc = high.count();
      refresh_entries += hc;
      if (hc > 0 && t >= min_td) {  // refresh_tiers (scheduler.cpp:38-55)
        double nm = kInf;
        for (int i = 0; i < NW; ++i) {
          uint64_t b = high.word(i);
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
                high.andnot(i, 1ull << bit);
                LOW[low_tail] = static_cast<uint16_t>(id);
                ++low_tail;
                push_decision<kTrace>(L, t, id, SABER_DEMOTE, load, dbits(ceiling), dbits(need),
                                      tr, P.out.trace_cap, P.out.error, true);
                if (kRecords && P.out.demoted) P.out.demoted[d.row * nmax + id] = 1;
              }
            }
            if (!demote) nm = dmin(nm, T);
          }
        }
        min_td = nm;
      }
      if (high.any()) {  // admission_step, high tier (scheduler.cpp:58-95)
        const int hcount = high.count();
        const int w = d.window < hcount ? d.window : hcount;
        if (draw_pos + (w - 1) > draw_len) {
          failed = true;
          ended = true;
        } else {
          uint64_t ord = 0xFEDCBA9876543210ull;
          for (int i = w - 1; i >= 1; --i) {
            const uint32_t x = draws[draw_pos++];
            const uint32_t d1 = static_cast<uint32_t>(i + 1);
            const uint32_t j = x - __umulhi(x, INV[d1]) * d1;
            const uint64_t a = (ord >> (4 * i)) & 15ull;
            const uint64_t bb = (ord >> (4 * j)) & 15ull;
            const uint64_t x2 = a ^ bb;
            ord ^= (x2 << (4 * i)) | (x2 << (4 * j));
          }
          rng_draws += w - 1;
          const double pred = MT[load + 1];
          const bool violates = pred < ledger_max;
          ledger_scanned += ledger_size;
          for (int c = 0; c < w; ++c) {
            const int id = high.select(static_cast<int>((ord >> (4 * c)) & 15ull));
            ++cands;
            const double need = queued_need(MO[id], DL[id], t);
            if (pred < need) {
              push_decision<kTrace>(L, t, id, SABER_REJECT_OWN, load, dbits(pred), dbits(need), tr,
                                    P.out.trace_cap, P.out.error, true);
              continue;
            }
            if (violates) {
              push_decision<kTrace>(L, t, id, SABER_REJECT_ACTIVE, load, dbits(pred), dbits(need),
                                    tr, P.out.trace_cap, P.out.error, true);
              continue;
            }
            admit(id, t);
            ledger.set(id);
            ++ledger_size;
            LNEED[id] = need;
            ledger_max = (ledger_max < need) ? need : ledger_max;
            high.reset(id);
            push_decision<kTrace>(L, t, id, SABER_ADMIT_HIGH, load, dbits(pred), dbits(need), tr,
                                  P.out.trace_cap, P.out.error, true);
            break;
          }
        }
      } else if (low_head < low_tail) {  // admission_step, low tier
        const int id = LOW[low_head];
        ++low_head;
        const double need = queued_need(MO[id], DL[id], t);
        admit(id, t);
        push_decision<kTrace>(L, t, id, SABER_ADMIT_LOW, load, kAbsent, dbits(need), tr,
                              P.out.trace_cap, P.out.error, true);
      }
    } else {  // StaticScheduler::static_step (scheduler.cpp:129-144)
      while (A < d.cap && high.any()) {
        const int id = high.lowest();
        high.reset(id);
        const int before = A;
        admit(id, t);
        push_decision<kTrace>(L, t, id, SABER_ADMIT_HIGH, before, kAbsent, kAbsent, tr,
                              P.out.trace_cap, P.out.error, true);
      }
    }

    if (!ended && t >= horizon) ended = true;
    if (!ended) {
      const double nt = (horizon < t + d.tick) ? horizon : t + d.tick;
      // ---- Engine::advance_to(nt) (engine.cpp:51-127) ----
      bool dirty = false;
      while (clock < nt) {
        if (A == 0) {
          clock = nt;
          break;
        }
        ++passes;
        const double speed = GT[A];
        double dt = nt - clock;
        if (min_pf < dt) dt = min_pf;
        if (min_rem < speed * dt * kOnePlusTol) {
          const double bnd = min_rem / speed;
          if (bnd < dt) dt = bnd;
        }
        const double group = dt * kOnePlusTol;
        const double sdt = speed * dt;
        const double sgd = speed * (group - dt);
        const double nclock = clock + dt;
        double npf = kInf, nrem = kInf;
        int j = 0, pfc = 0;
        const int a0 = A;
        for (int k = 0; k < a0; ++k) {
          double g = SG[k * kWarp];
          const uint32_t mi = SM[k * kWarp];
          const double m = static_cast<double>(mi >> 9);
          bool done;
          if (g < 0.0) {
            ++pfc;
            if (-g <= group) {
              g = 0.0;
              done = g + sgd >= m;
            } else {
              g = g + dt;
              npf = dmin(npf, -g);
              done = false;
            }
          } else {
            g = g + sdt;
            done = g + sgd >= m;
          }
          if (!done) {
            if (g >= 0.0) nrem = dmin(nrem, m - g);
            SG[j * kWarp] = g;
            if (j != k) SM[j * kWarp] = mi;
            ++j;
          } else {
            const int id = static_cast<int>(mi & 511u);
            COMP[id] = nclock;
            ++completed;
            if (saber && ledger.test(id)) {
              ledger.reset(id);
              --ledger_size;
              dirty = true;
            }
          }
        }
        A = j;
        clock = nclock;
        min_pf = npf;
        min_rem = nrem;
        prefill_updates += pfc;
        decode_updates += a0 - pfc;
      }
      if (dirty) {
        double mx = -kInf;
        for (int i = 0; i < NW; ++i) {
          uint64_t b = ledger.word(i);
          while (b) {
            const int id = i * 64 + __ffsll(static_cast<long long>(b)) - 1;
            b &= b - 1;
            const double v = LNEED[id];
            mx = (mx < v) ? v : mx;
          }
        }
        ledger_max = mx;
      }
      t = nt;
      if (completed == n) ended = true;
    }
    if (ended) {
      finish();
      if (!fetch()) break;
    }
  }
}

template <int NW, bool kTrace, bool kRecords>
void* lane_ptr() {
  return reinterpret_cast<void*>(&sim_lane_kernel<NW, kTrace, kRecords>);
}

template <int NW>
void* pick_lane_tr(bool trace, bool records) {
  if (trace) return lane_ptr<NW, true, true>();
  if (records) return lane_ptr<NW, false, true>();
  return lane_ptr<NW, false, false>();
}

void* pick_lane(int nw, bool trace, bool records) {
  switch (nw) {
    case 1: return pick_lane_tr<1>(trace, records);
    case 2: return pick_lane_tr<2>(trace, records);
  }
  return nullptr;
}

}  // namespace

int plan_sim_lane(int nmax, SimLaunch* out) {
  if (nmax > 128) return 4;
  SimLaunch l{};
  l.nwords = nmax <= 64 ? 1 : 2;
  l.group = 1;
  l.lane = 1;
  l.slot_rows = nmax;
  l.smem = static_cast<size_t>(nmax) * kWarp * 12;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
  for (int tr = 0; tr < 2; ++tr)
    for (int rec = 0; rec < 2; ++rec)
      if (cudaFuncSetAttribute(pick_lane(l.nwords, tr != 0, rec != 0),
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(l.smem)) != cudaSuccess)
        return 2;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pick_lane(l.nwords, false, false),
                                                    kLaneBlock, l.smem) != cudaSuccess)
    return 1;
  if (per_sm < 1) return 3;
  l.grid = sms * per_sm;
  l.block = kLaneBlock;
  *out = l;
  return 0;
}

int launch_sim_lane(const SimParams& p, const SimLaunch& l, void* stream) {
  const bool trace = p.out.trace != nullptr;
  const bool records = p.out.admit != nullptr || p.out.demoted != nullptr;
  void* k = pick_lane(l.nwords, trace, records);
  if (!k) return 1;
  void* args[] = {const_cast<SimParams*>(&p)};
  return cudaLaunchKernel(k, dim3(l.grid), dim3(kLaneBlock), args, l.smem,
                          static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? 0
             : 1;
}

}  // namespace saberb200
