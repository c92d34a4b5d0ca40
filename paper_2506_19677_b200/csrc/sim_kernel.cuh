// sim_kernel.cuh — the trajectory engine (K1) for sm_100a: simulate_one and
// the persistent sim_kernel.  Included by the per-mask-width instantiation
// units sim_inst_nw{1,2,4,8}.cu (compiled in parallel) and by sim_kernel.cu.
//
//
// A GROUP of G lanes owns one trajectory.  A persistent grid
// pulls trajectory indices from an atomic work queue; every lane of the group
// carries an identical copy of the trajectory's scalar state (clock, tiers as
// register bitmasks, ledger, RNG cursor, decision hash) and runs the
// reference's tick loop (simloop.cpp:78-101):
//   arrivals -> refresh_tiers -> admission_step | static_step  (scheduler.cpp)
//   -> Engine::advance_to (engine.cpp:51-127) -> completions.
// The engine's per-slot work — the only part that scales with the batch — is
// split across the group: slot k is updated by lane k % G, with the slot
// state (fluid progress / prefill debt, max_out | id) held in shared memory in
// a lane-interleaved layout (conflict-free 64-bit accesses), and the
// next-event minima combined with REDUX.MIN over the group.
//
// Bit-exactness with the reference: compiled with --fmad=false
// (the reference has no FMA); every floating-point expression keeps
// the reference's operand order; predict() comes from host-built tables
// (SURVEY F6); the scheduler RNG from precomputed mt19937_64 streams
// (SURVEY F2).  Three exact rewrites remove work without changing any result:
//   * min_i fl(rem_i / speed) == fl(min_i rem_i / speed), because correctly
//     rounded division by a positive constant is monotone;
//   * that one divide is skipped when min_rem >= speed*dt*(1+1e-12), which
//     proves fl(min_rem / speed) >= dt, i.e. the boundary cannot bind;
//   * a high-tier request cannot demote before demote_after[i], a safe lower
//     bound (prologue.cu), so refresh only scans when one might.
// Slot order inside the engine never affects a result (min is order-free,
// completions of one pass share the clock), so completed slots are removed by
// swap-with-last instead of the reference's order-preserving erase.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "saber_internal.h"
#include "sim_common.cuh"

namespace saberb200 {
namespace {

using namespace simdev;

// Blocks per SM for the register budget (kSimBlock-thread blocks): generic
// and SABER kernels 16 warps (128 registers), static kernel 25 (ptxas: 72
// registers, 28 warps fit).
#ifndef SABER_SIM_MIN_BLOCKS
#define SABER_SIM_MIN_BLOCKS (512 / SABER_SIM_BLOCK)
#endif
#ifndef SABER_STATIC_MIN_BLOCKS
#define SABER_STATIC_MIN_BLOCKS (800 / SABER_SIM_BLOCK)
#endif
#ifndef SABER_SABER_MIN_BLOCKS
#define SABER_SABER_MIN_BLOCKS (512 / SABER_SIM_BLOCK)
#endif

#ifdef SABER_STREAK_STATS
#define SEC_BEGIN() const long long sec_t0_ = clock64()
#define SEC_END(k) st_cyc[k] += clock64() - sec_t0_
#else
#define SEC_BEGIN()
#define SEC_END(k)
#endif

// Scheduler-mode specialisation of the trajectory kernel:
// kSel 0 = any trajectory, 1 = static only, 2 = SABER only.  The specialised
// variants drop the other mode's code (smaller footprint in the instruction
// cache, fewer live registers) and serve the sweep's two row classes.
enum : int { kSelAny = 0, kSelStatic = 1, kSelSaber = 2 };


// Shared-memory slot arrays of one group: slot k lives at row k / G, column
// grp * G + k % G of the warp's [rows][32] tile (so lane k % G of the group
// always touches its own column: 32 lanes hit 32 consecutive 8-byte words).
template <int G>
struct Slots {
  double* g;     // fluid progress (>= 0) or -prefill_left (< 0); kDoneMark when done
  uint64_t* m;   // bits(max_output_tokens) | request id (low 16 bits are free)
  uint32_t* dbuf;  // this group's staging buffer for scheduler draws, G * (kMaxWindow - 1)
  int col0;      // grp * G
  static_assert((G & (G - 1)) == 0, "G must be a power of two");
  __device__ __forceinline__ int idx(int k) const {
    return ((k / G) << 5) + col0 + (k & (G - 1));
  }
};

// An integer q <= a / b (a >= 0 finite, b > 0), capped at 2^30, without a
// DDIV: b is rounded up and a down to float, the approximate reciprocal
// (MUFU, |rel err| < 2^-22) and the product are scaled down by 4e-5, so the
// result is a strict lower bound of the true quotient.
__device__ __forceinline__ int floor_div_lb(double a, double b) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__double2float_ru(b)));
  const float q = __double2float_rd(a) * (r * 0.99996f);
  return static_cast<int>(fminf(q, 1073741824.0f));
}

// min{k : T[k] >= x} over the tick table (len if none; x may be +-inf;
// NaN maps to len).
__device__ __forceinline__ int tick_index(const TickTable& tt, double x) {
  if (isnan(x)) return tt.len;
  int k = static_cast<int>(fmin(fmax(x * tt.inv_tick, 0.0), static_cast<double>(tt.len)));
  while (k > 0 && tt.T[k - 1] >= x) --k;
  while (k < tt.len && tt.T[k] < x) ++k;
  return k;
}

// Quiet streak: K consecutive ticks k0 .. k0+K-1, each one
// full quiet pass of dt = DT[k], applied slot by slot from registers.
// Per pass the reference computes generated += speed*dt (decode) or
// prefill_left -= dt (prefill, stored as g = -prefill_left); here every slot
// adds fl(mult * dt) with mult = speed (decode) or 1.0 (prefill: fl(1*dt) = dt),
// which is that same value.  The caller has proved that no pass of the streak
// ends a prefill, binds the decode boundary or completes a slot.  Returns the
// exact prefill minimum after the streak (the per-pass chain min_pf -= dt).
// kDec: no slot is in prefill (npre == 0, uniform), so every slot adds the
// same fl(speed * dt) and the product is formed once per tick, not per slot.
template <int G, int kC, bool kDec>
__device__ __forceinline__ double streak_chunks(const Slots<G>& S, int sub, int A, double speed,
                                               const double* __restrict__ DT, int K, double pf) {
  // Chunk 0 runs on every lane of the group (it also carries the replicated
  // min_pf chain); later chunks only while the lane still owns slots.
  for (int base = sub, first = 1; first || base < A; base += kC * G, first = 0) {
    double g[kC], mult[kC];
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      const int k = base + i * G;
      g[i] = k < A ? S.g[S.idx(k)] : 0.0;
      mult[i] = g[i] < 0.0 ? 1.0 : speed;
    }
    int j = 0;
#ifndef SABER_DT_VEC
#define SABER_DT_VEC 1
#endif
    // 4-tick blocks of DT as two 16-byte loads: peel one tick first when
    // DT + 0 is not 16-byte aligned (the per-tick update is the same either way)
    if (SABER_DT_VEC && K >= 1 && (reinterpret_cast<uintptr_t>(DT) & 8u)) {
      const double d0 = DT[0];
#pragma unroll
      for (int i = 0; i < kC; ++i) g[i] = g[i] + mult[i] * d0;  // mult == speed when kDec
      if (!kDec && first) pf = pf - d0;
      j = 1;
    }
#pragma unroll 1
    for (; j + 4 <= K; j += 4) {
      double d0, d1, d2, d3;
      if (SABER_DT_VEC) {
        const double2 a = reinterpret_cast<const double2*>(DT + j)[0];
        const double2 b = reinterpret_cast<const double2*>(DT + j)[1];
        d0 = a.x;
        d1 = a.y;
        d2 = b.x;
        d3 = b.y;
      } else {
        d0 = DT[j];
        d1 = DT[j + 1];
        d2 = DT[j + 2];
        d3 = DT[j + 3];
      }
      if (kDec) {
        const double s0 = speed * d0, s1 = speed * d1, s2 = speed * d2, s3 = speed * d3;
#pragma unroll
        for (int i = 0; i < kC; ++i) g[i] = (((g[i] + s0) + s1) + s2) + s3;
      } else {
#pragma unroll
        for (int i = 0; i < kC; ++i) {
          g[i] = g[i] + mult[i] * d0;
          g[i] = g[i] + mult[i] * d1;
          g[i] = g[i] + mult[i] * d2;
          g[i] = g[i] + mult[i] * d3;
        }
        if (first) pf = (((pf - d0) - d1) - d2) - d3;
      }
    }
#pragma unroll 1
    for (; j < K; ++j) {
      const double d0 = DT[j];
#pragma unroll
      for (int i = 0; i < kC; ++i) g[i] = g[i] + mult[i] * d0;  // mult == speed when kDec
      if (!kDec && first) pf = pf - d0;
    }
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      const int k = base + i * G;
      if (k < A) S.g[S.idx(k)] = g[i];
    }
  }
  return pf;
}

// kCompact (the SABER kernel): one chunk width for every slot count — a
// smaller instruction footprint measured faster than the specialised widths
// for that kernel.  SABER keeps the batch small (A <= 32 nearly always), so
// the width is one slot per lane.
#ifndef SABER_COMPACT_KC
#define SABER_COMPACT_KC 1
#endif
#ifndef SABER_COMPACT_DEC
#define SABER_COMPACT_DEC 1
#endif
template <int G, bool kCompact = false>
__device__ __forceinline__ double streak_slots(const Slots<G>& S, int sub, int A, int npre,
                                               double speed, const double* __restrict__ DT, int K,
                                               double pf) {
  if (kCompact) {
    if (SABER_COMPACT_DEC && npre == 0)
      return streak_chunks<G, SABER_COMPACT_KC, true>(S, sub, A, speed, DT, K, pf);
    return streak_chunks<G, SABER_COMPACT_KC, false>(S, sub, A, speed, DT, K, pf);
  }
  if (A <= G) return streak_chunks<G, 1, false>(S, sub, A, speed, DT, K, pf);
  if (npre == 0) {  // min_pf is +inf and stays so
    if (A <= 2 * G) return streak_chunks<G, 2, true>(S, sub, A, speed, DT, K, pf);
    return streak_chunks<G, 4, true>(S, sub, A, speed, DT, K, pf);
  }
  if (A <= 2 * G) return streak_chunks<G, 2, false>(S, sub, A, speed, DT, K, pf);
  return streak_chunks<G, 4, false>(S, sub, A, speed, DT, K, pf);
}

// Gate streak decisions: ticks k0+1 .. k0+K-1 of a streak
// whose tick k0 gate admitted nobody.  Each such tick runs the reference's
// admission_step (scheduler.cpp:57-95) on an unchanged window: w-1 draws for
// the Fisher-Yates, then every candidate is rejected — RejectOwn when
// pred < need(t), else RejectActive (need grows with t, so a candidate that
// could pass its own test at k0 was already blocked by the ledger).  Lane
// `sub` takes ticks k0+1+sub, k0+1+sub+G, ...; the digest terms (oracle.h)
// carry their log index n0 + (j-1) w + c, so they are summed in any order.
template <int G, bool kTrace, int NW>
__device__ __forceinline__ void gate_streak_decisions(
    const SimParams& P, const Slots<G>& S, int sub, unsigned gmask, const Mask<NW>& high,
    const double* __restrict__ MO, const double* __restrict__ DL,
    const uint32_t* __restrict__ draws, int64_t draw_pos, int k0, int K, int w, int load,
    double pred, DecisionLog& L, saber_decision* tr, const uint32_t* __restrict__ INV) {
  // the window (first w queued ids) on lanes 0..w-1
  int wid = 0;
  double wm = 0.0, wdl = 0.0;
  if (sub < w) {
    wid = high.select(sub);
    wm = MO[wid];
    wdl = DL[wid];
  }
  const uint64_t pb = dbits(pred);
  const uint64_t wl = static_cast<uint64_t>(static_cast<uint32_t>(load)) << 40;
  const int64_t n0 = L.n;
  uint64_t hs = 0;
  unsigned own = 0, act = 0;
  for (int jb = 1; jb < K; jb += G) {
    const int j = jb + sub;
    const bool live = j < K;
    const double tj = live ? P.ticks.T[k0 + j] : 0.0;
    const uint64_t tb = dbits(tj);
    // This round's draws (ticks jb .. jb+G-1, w-1 each, consecutive in the
    // stream) are staged through shared memory with coalesced loads, then
    // every lane runs its tick's Fisher-Yates from there (a rolled loop keeps
    // the kernel's instruction footprint small).
    const int nd = min(G, K - jb) * (w - 1);
    const uint32_t* __restrict__ src = draws + draw_pos + static_cast<int64_t>(jb - 1) * (w - 1);
    for (int q = sub; q < nd; q += G) S.dbuf[q] = src[q];
    __syncwarp(gmask);
    const uint32_t* my = S.dbuf + sub * (w - 1);
    uint64_t ord = 0xFEDCBA9876543210ull;
#pragma unroll 1
    for (int q = 0; q < w - 1; ++q) {
      const uint32_t x = live ? my[q] : 0u;
      const uint32_t i = static_cast<uint32_t>(w - 1 - q);
      const uint32_t jj = x - __umulhi(x, INV[i + 1]) * (i + 1);
      const uint64_t a = (ord >> (4 * i)) & 15ull;
      const uint64_t bb = (ord >> (4 * jj)) & 15ull;
      const uint64_t x2 = a ^ bb;
      ord ^= (x2 << (4 * i)) | (x2 << (4 * jj));
    }
    __syncwarp(gmask);  // the buffer is refilled next round
    for (int c = 0; c < w; ++c) {
      const int p = static_cast<int>((ord >> (4 * c)) & 15ull);
      const int id = __shfl_sync(gmask, wid, S.col0 + p);
      const double m = __shfl_sync(gmask, wm, S.col0 + p);
      const double dl = __shfl_sync(gmask, wdl, S.col0 + p);
      if (!live) continue;
      const double need = queued_need(m, dl, tj);
      const int kind = pred < need ? SABER_REJECT_OWN : SABER_REJECT_ACTIVE;
      own += kind == SABER_REJECT_OWN;
      act += kind == SABER_REJECT_ACTIVE;
      const int64_t idx = n0 + static_cast<int64_t>(j - 1) * w + c;
      const uint64_t w64 = static_cast<uint64_t>(static_cast<uint32_t>(id)) |
                           (static_cast<uint64_t>(kind) << 32) | wl;
      hs += decision_term(static_cast<uint64_t>(idx), tb, w64, pb, dbits(need));
      if (kTrace && tr != nullptr) {
        if (idx < P.out.trace_cap) {
          saber_decision& dd = tr[idx];
          dd.time = tj;
          dd.request_id = static_cast<uint64_t>(id);
          dd.kind = kind;
          dd.load_before = load;
          dd.has_pred = 1;
          dd.has_req = 1;
          dd.pred_speed = pred;
          dd.req_speed = need;
        } else {
          atomicCAS(P.out.error, kErrNone, kErrTraceOverflow);
        }
      }
    }
  }
  // group sums (64-bit digest: butterfly over the group's lanes)
#pragma unroll
  for (int o = 1; o < G; o <<= 1) hs += __shfl_xor_sync(gmask, hs, o);
  own = group_sum<G>(own, gmask);
  act = group_sum<G>(act, gmask);
  const int64_t nd = static_cast<int64_t>(K - 1) * w;
  L.h += hs;
  L.n += static_cast<int32_t>(nd);
  L.k2 += static_cast<int32_t>(own);
  L.k3 += static_cast<int32_t>(act);
}

// Whole-warp gate streak (G == 32): the same decisions as
// gate_streak_decisions, in two phases per round of up to 32 ticks.  Phase A,
// lane = tick: the tick's Fisher-Yates permutation of the window as packed
// nibbles, parked in the draw staging buffer.  Phase B, lane = (tick,
// position) pair: the candidate's need, kind and digest term — so the
// per-decision work (a divide and the digest mix) runs on ~all 32 lanes
// instead of one lane per tick.
template <bool kTrace, int NW>
__device__ __forceinline__ void gate_streak_warp(
    const SimParams& P, const Slots<kWarp>& S, int sub, const Mask<NW>& high,
    const double* __restrict__ MO, const double* __restrict__ DL,
    const uint32_t* __restrict__ draws, int64_t draw_pos, int k0, int K, int w, int load,
    double pred, DecisionLog& L, saber_decision* tr, const uint32_t* __restrict__ INV) {
  int wid = 0;
  double wm = 0.0, wdl = 0.0;
  if (sub < w) {
    wid = high.select(sub);
    wm = MO[wid];
    wdl = DL[wid];
  }
  const uint64_t pb = dbits(pred);
  const int64_t n0 = L.n;
  const uint32_t invw = w > 1 ? INV[w] : 0u;
  uint64_t* __restrict__ ords = reinterpret_cast<uint64_t*>(S.dbuf);
  uint64_t hs = 0;
  unsigned own = 0;
  for (int jb = 1; jb < K; jb += kWarp) {
    const int nt = min(kWarp, K - jb);
    const int nd = nt * (w - 1);
    const uint32_t* __restrict__ src = draws + draw_pos + static_cast<int64_t>(jb - 1) * (w - 1);
#pragma unroll 1
    for (int q = sub; q < nd; q += kWarp) S.dbuf[q] = src[q];
    __syncwarp();
    uint64_t ord = 0xFEDCBA9876543210ull;
    if (sub < nt) {
      const uint32_t* my = S.dbuf + sub * (w - 1);
#pragma unroll 1
      for (int q = 0; q < w - 1; ++q) {
        const uint32_t x = my[q];
        const uint32_t i = static_cast<uint32_t>(w - 1 - q);
        const uint32_t jj = x - __umulhi(x, INV[i + 1]) * (i + 1);
        const uint64_t a = (ord >> (4 * i)) & 15ull;
        const uint64_t bb = (ord >> (4 * jj)) & 15ull;
        const uint64_t x2 = a ^ bb;
        ord ^= (x2 << (4 * i)) | (x2 << (4 * jj));
      }
    }
    __syncwarp();  // every lane's draws are consumed before the buffer is reused
    ords[sub] = ord;
    __syncwarp();
    const int np = nt * w;
#pragma unroll 1
    for (int p0 = 0; p0 < np; p0 += kWarp) {
      const int p = p0 + sub;
      const bool live = p < np;
      const int jj = live ? (w > 1 ? static_cast<int>(__umulhi(static_cast<uint32_t>(p), invw)) : p) : 0;
      const int c = p - jj * w;
      const int pos = live ? static_cast<int>((ords[jj] >> (4 * c)) & 15ull) : 0;
      const int id = __shfl_sync(0xFFFFFFFFu, wid, pos);
      const double m = __shfl_sync(0xFFFFFFFFu, wm, pos);
      const double dl = __shfl_sync(0xFFFFFFFFu, wdl, pos);
      if (live) {
        const int j = jb + jj;
        const double tj = P.ticks.T[k0 + j];
        const double need = queued_need(m, dl, tj);
        const int kind = pred < need ? SABER_REJECT_OWN : SABER_REJECT_ACTIVE;
        own += kind == SABER_REJECT_OWN;
        const int64_t idx = n0 + static_cast<int64_t>(j - 1) * w + c;
        const uint64_t tb = dbits(tj), rb = dbits(need);
        hs += decision_term(static_cast<uint64_t>(idx), tb, decision_word(id, kind, load), pb, rb);
        if (kTrace && tr != nullptr)
          write_decision(tr, idx, P.out.trace_cap, P.out.error, tj, id, kind, load, pb, rb);
      }
    }
    __syncwarp();  // the buffer is refilled next round
  }
  hs = warp_sum_u64(hs);
  own = __reduce_add_sync(0xFFFFFFFFu, own);
  const int32_t ndec = static_cast<int32_t>(K - 1) * w;
  L.h += hs;
  L.n += ndec;
  L.k2 += static_cast<int32_t>(own);
  L.k3 += ndec - static_cast<int32_t>(own);
}

// max over the ledger's needs (ActiveLedger, scheduler.hpp:30-44), -inf when
// empty.  Needs are >= +0, so their bit patterns order like the values; with
// a whole warp per trajectory every lane tests two ids of each mask word.
template <int G, int NW, class MaskT>
__device__ __forceinline__ double ledger_max_of(const MaskT& ledger, int size,
                                                const double* __restrict__ LNEED, int sub) {
  if (size == 0) return -kInf;
  if constexpr (MaskT::kGlobal) {  // wide kernel: words [0, hi) in global memory
    uint64_t k = 0;
#pragma unroll 1
    for (int i = 0; i < ledger.word_end(); ++i) {
      const uint64_t wd = ledger.word(i);
      if (wd == 0) continue;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int bit = hh * 32 + sub;
        if ((wd >> bit) & 1ull) {
          const uint64_t v = dbits(LNEED[i * 64 + bit]);
          k = k < v ? v : k;
        }
      }
    }
    return bitsd(warp_max_u64(k));
  } else if constexpr (G == kWarp) {
    uint64_t k = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const uint64_t wd = ledger.word(i);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int bit = hh * 32 + sub;
        if ((wd >> bit) & 1ull) {
          const uint64_t v = dbits(LNEED[i * 64 + bit]);
          k = k < v ? v : k;
        }
      }
    }
    return bitsd(warp_max_u64(k));
  } else {
    double mx = -kInf;
    for (int i = 0; i < NW; ++i) {
      uint64_t b = ledger.word(i);
      while (b) {
        const int q = i * 64 + __ffsll(static_cast<long long>(b)) - 1;
        b &= b - 1;
        const double v = LNEED[q];
        mx = (mx < v) ? v : mx;
      }
    }
    return mx;
  }
}

// Simulates trajectory `ti` on this group.
// Per-group global scratch of the wide kernel.
struct WideScratch {
  uint64_t* masks;   // [2][nw]: high tier, ledger
  int nw;
  int32_t* gate;     // [3][nmax]: Fisher-Yates j, window order, candidate id
  double* need;      // [nmax] candidate needs
};

template <int NW, int G, bool kTrace, bool kRecords, int kSel, bool kWide = false>
__device__ __forceinline__ void simulate_one(const SimParams& P, int ti, const Slots<G>& S,
                                             int sub, unsigned gmask,
                                             double* __restrict__ LNEED,
                                             uint16_t* __restrict__ LOW,
                                             const uint32_t* __restrict__ INV,
                                             const WideScratch& WS = WideScratch{}) {
  static_assert(!kWide || (G == kWarp && kSel == kSelAny), "wide kernel: whole warps, any mode");
  const TrajDesc d = P.traj[P.order ? P.order[ti] : ti];
  const int n = d.n;
  const int nmax = P.wl.nmax;
  const int64_t wo = static_cast<int64_t>(d.workload) * nmax;
  const double* __restrict__ GT = P.tables + d.gt_tab;
  const bool saber = kSel == kSelSaber ? true
                     : kSel == kSelStatic ? false
                                          : d.mode == SABER_MODE_SABER;
  if (kSel != kSelAny && saber != (d.mode == SABER_MODE_SABER)) {
    if (sub == 0) atomicCAS(P.out.error, kErrNone, kErrBadDesc);  // loud: wrong kernel
    return;
  }
  const double* __restrict__ MT = P.tables + (saber ? d.model_tab : d.gt_tab);
  const double horizon = isnan(d.horizon) ? P.wl.horizon[d.workload] : d.horizon;
  const double tick = d.tick;
  const double ceiling = saber ? MT[1] : 0.0;  // max_speed = predict(model, 1)
  const uint32_t* __restrict__ draws =
      saber ? P.rng.draws + P.rng.off[d.stream] : nullptr;
  const int64_t draw_len = saber ? P.rng.len[d.stream] : 0;
  double* __restrict__ COMP = P.out.completion + d.row * nmax;
  double* __restrict__ ADM = kRecords && P.out.admit ? P.out.admit + d.row * nmax : nullptr;
  uint8_t* __restrict__ DEMO =
      kRecords && P.out.demoted ? P.out.demoted + d.row * nmax : nullptr;
  const bool leader = sub == 0;
  saber_decision* tr = kTrace && P.out.trace ? P.out.trace + d.row * P.out.trace_cap : nullptr;

  using MaskT = typename std::conditional<kWide, GMask, Mask<NW>>::type;
  MaskT high, ledger;
  if constexpr (kWide) {
    high.bind(WS.masks, WS.nw, sub);
    ledger.bind(WS.masks + WS.nw, WS.nw, sub);
  }
  high.clear();
  ledger.clear();
  int hn = 0;  // |high tier| (kept beside the mask: no popcount per query)
  // wide kernel: raw 64-bit scheduler draws (window > 16)
  const uint64_t* __restrict__ draws64 =
      kWide && saber ? reinterpret_cast<const uint64_t*>(P.rng.draws) + P.rng.off[d.stream]
                     : nullptr;
  int ledger_size = 0;
  double ledger_max = -kInf;
  double min_td = kInf;  // lower bound on the earliest possible demotion
  int low_head = 0, low_tail = 0;

  int A = 0;         // |active|
  int npre = 0;      // active slots still in prefill
  double clock = 0.0;
  double min_pf = kInf;   // exact min prefill_left over prefill slots
  double rem_lb = kInf;   // lower bound on min (max_out - generated) over decode slots
  bool rem_exact = true;  // rem_lb is the exact minimum
  double m_hi = 0.0;      // >= max_output_tokens of every active slot
  // speed_A caches predict(gt, A); it changes only with A.
  double speed_A = 0.0;
  bool sblock = false;  // quiet-streak bounds exhausted until the next event (§3.5)
  auto retune = [&]() { speed_A = GT[A]; };

  int next = 0;
  double na_t = n > 0 ? P.wl.arrival[wo + 0] : kInf;
  int completed = 0;
  int64_t draw_pos = 0;
  bool failed = false;

  DecisionLog L{kHashSeed, 0, 0, 0, 0, 0, 0};
  int32_t ticks = 0, passes = 0, decode_updates = 0, prefill_updates = 0;
  int32_t refresh_entries = 0, cands = 0, ledger_scanned = 0, rng_draws = 0;

  // Engine::admit (engine.cpp:26-49): append slot A.  Every lane of the group
  // writes the same values, so the owning lane reads back its own write.
  auto admit = [&](int id, double now) {
    const double pl = P.wl.prefill[wo + id];  // input / prefill_rate (prologue)
    const double m = P.wl.max_out[wo + id];
    const int s = S.idx(A);
    if (pl == 0.0) {
      S.g[s] = 0.0;  // decode starts at admission
      rem_lb = dmin(rem_lb, m - 0.0);
    } else {
      S.g[s] = -pl;
      min_pf = dmin(min_pf, pl);
      ++npre;
    }
    m_hi = (m_hi < m) ? m : m_hi;
    S.m[s] = dbits(m) | static_cast<uint64_t>(id);
    ++A;
    sblock = false;
    retune();
    if (kRecords && ADM && leader) ADM[id] = now;
  };

  // Tick table: kh = first tick index at/after the horizon,
  // ka = first tick index at/after the next arrival (lazily, -1 = stale).
  bool use_tab = !P.no_streak && P.ticks.len > 0 && tick == P.ticks.tick && P.wl.arr_tick != nullptr;
  const int kh = use_tab ? tick_index(P.ticks, horizon) : 0;
  // tick index of the next arrival, and of min_td (tick_index is monotone, so
  // it follows min_td's own updates: min at arrival, recomputed at a scan)
  int ka = use_tab ? (n > 0 ? P.wl.arr_tick[wo + 0] : P.ticks.len) : 0;
  int min_kd = 0x7FFFFFFF;
#ifdef SABER_STREAK_STATS
  int st_ticks = 0, st_count = 0, st_quiet = 0, st_exact = 0;
  const long long st_t0 = clock64();
  long long st_cyc[5] = {0, 0, 0, 0, 0};
  int st_scans = 0;
  // streak-end causes (stats build): [0..3] K >= 2 bound by Kb / arrival /
  // demotion or draws / horizon; [4..7] the same for K < 2 attempts;
  // [8..11] streak condition false: sblock / A == 0 / gate admitted / other
  int st_cause[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif

  double t = 0.0;
  for (;;) {
    // Arrivals due at t (simloop.cpp:79-85).
    while (na_t <= t) {
      high.set(next);
      ++hn;
      if (saber) min_td = dmin(min_td, P.wl.demote_after[wo + next]);
      if (saber && use_tab) min_kd = min(min_kd, P.wl.dem_tick[wo + next]);
      ++next;
      na_t = next < n ? P.wl.arrival[wo + next] : kInf;
      if (use_tab) ka = next < n ? P.wl.arr_tick[wo + next] : P.ticks.len;
    }
    ++ticks;
    const int load = A;
    // Gate outcome of this tick, for a gate streak.
    bool gate_idle = false;
    int gate_w = 0;
    double gate_pred = 0.0;
#ifdef SABER_STREAK_STATS
    const long long sched_t0 = clock64();
#endif
    if (saber) {
      const int hc = hn;
      refresh_entries += hc;
      // refresh_tiers (scheduler.cpp:38-55): scan in queue (= id) order only
      // when some entry may have crossed its demotion bound.
      if (hc > 0 && t >= min_td) {
#ifdef SABER_STREAK_STATS
        const long long scan_t0 = clock64();
        st_scans += 1;
#endif
        double nm = kInf;
        int nkd = 0x7FFFFFFF;
        if constexpr (G == kWarp) {
          // Lane-parallel scan: lane l tests ids 64 i + l and 64 i + 32 + l of
          // every tier word; the demotions of one half-word are ranked by
          // lane (= id) order, so each one's log index, FIFO slot and digest
          // term follow from a ballot prefix count.
          uint64_t key = dkey(kInf);
          uint64_t hterm = 0;
          int ndem = 0;
#pragma unroll 1
          for (int q = 2 * high.word_begin(); q < 2 * high.word_end(); ++q) {  // half-words
            const uint32_t hw = static_cast<uint32_t>(high.word(q >> 1) >> ((q & 1) * 32));
            if (hw == 0) continue;
            const int id = q * 32 + sub;
            const bool mem = ((hw >> sub) & 1u) != 0;
            bool demote = false;
            double need = 0.0;
            if (mem) {
              const double T = P.wl.demote_after[wo + id];
              if (t >= T) {
                need = queued_need(P.wl.max_out[wo + id], P.wl.deadline[wo + id], t);
                demote = need > ceiling;
              }
              if (!demote) {
                key = key < dkey(T) ? key : dkey(T);
                if (use_tab) nkd = min(nkd, P.wl.dem_tick[wo + id]);
              }
            }
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, demote);
            if (bal) {
              if (demote) {
                const int rank = ndem + __popc(bal & lanemask_lt());
                LOW[low_tail + rank] = static_cast<uint16_t>(id);
                const uint64_t rb = dbits(need), pb = dbits(ceiling);
                hterm += decision_term(static_cast<uint64_t>(L.n + rank), dbits(t),
                                       decision_word(id, SABER_DEMOTE, load), pb, rb);
                if (kTrace && tr != nullptr)
                  write_decision(tr, L.n + rank, P.out.trace_cap, P.out.error, t, id,
                                 SABER_DEMOTE, load, pb, rb);
                if (kRecords && DEMO) DEMO[id] = 1;
              }
              ndem += __popc(bal);
              high.andnot(q >> 1, static_cast<uint64_t>(bal) << ((q & 1) * 32));
              hn -= __popc(bal);
            }
          }
          if (ndem) {
            L.h += warp_sum_u64(hterm);
            L.n += ndem;
            L.k4 += ndem;
            low_tail += ndem;
            __syncwarp();  // the FIFO entries written by other lanes
          }
          nm = keyd(warp_min_u64(key));
          nkd = __reduce_min_sync(0xFFFFFFFFu, nkd);
        } else {
        for (int i = 0; i < NW; ++i) {
          uint64_t b = high.word(i);
          while (b) {
            const int bit = __ffsll(static_cast<long long>(b)) - 1;
            b &= b - 1;
            const int id = i * 64 + bit;
            const double T = P.wl.demote_after[wo + id];
            bool demote = false;
            if (t >= T) {
              const double need = queued_need(P.wl.max_out[wo + id], P.wl.deadline[wo + id], t);
              if (need > ceiling) {
                demote = true;
                high.andnot(i, 1ull << bit);
                --hn;
                LOW[low_tail] = static_cast<uint16_t>(id);
                ++low_tail;
                push_decision<kTrace>(L, t, id, SABER_DEMOTE, load, dbits(ceiling), dbits(need),
                                      tr, P.out.trace_cap, P.out.error, leader);
                if (kRecords && DEMO && leader) DEMO[id] = 1;
              }
            }
            if (!demote) {
              nm = dmin(nm, T);
              if (use_tab) nkd = min(nkd, P.wl.dem_tick[wo + id]);
            }
          }
        }
        }
        min_td = nm;
        min_kd = nkd;
#ifdef SABER_STREAK_STATS
        st_cyc[4] += clock64() - scan_t0;
#endif
      }
      if (kWide && hn > 0) {
        // admission_step, high tier (scheduler.cpp:58-95), any window: the
        // Fisher-Yates j's lane-parallel (64-bit draws), the swaps by lane 0,
        // then 32 window positions per round with the first passing one found
        // by ballot.
        const int hcount = hn;
        const int w = d.window < hcount ? d.window : hcount;
        if (draw_pos + (w - 1) > draw_len) {
          failed = true;
          break;
        }
        int32_t* __restrict__ WJ = WS.gate;
        int32_t* __restrict__ WO = WS.gate + nmax;
        int32_t* __restrict__ WC = WS.gate + 2 * nmax;
        double* __restrict__ WN = WS.need;
        const double pred = MT[load + 1];
        const bool violates = pred < ledger_max;  // ActiveLedger::violates
        for (int q = sub; q < w - 1; q += kWarp)
          WJ[q] = static_cast<int32_t>(draws64[draw_pos + q] % static_cast<uint64_t>(w - q));
        for (int c = sub; c < w; c += kWarp) WO[c] = c;
        __syncwarp();
        if (leader) {
          for (int q = 0; q < w - 1; ++q) {
            const int i = w - 1 - q, j = WJ[q];
            const int a = WO[i];
            WO[i] = WO[j];
            WO[j] = a;
          }
        }
        __syncwarp();
        int first = w;
        for (int c0 = 0; c0 < w; c0 += kWarp) {
          const int c = c0 + sub;
          bool ok = false;
          if (c < w) {
            const int id = high.select(WO[c]);
            const double need = queued_need(P.wl.max_out[wo + id], P.wl.deadline[wo + id], t);
            WC[c] = id;
            WN[c] = need;
            ok = !(pred < need) && !violates;
          }
          const unsigned b = __ballot_sync(0xFFFFFFFFu, ok);
          if (b) {
            first = c0 + __ffs(b) - 1;
            break;
          }
        }
        __syncwarp();
        draw_pos += w - 1;
        rng_draws += w - 1;
        ledger_scanned += ledger_size;
        const int last = first < w ? first : w - 1;
        uint64_t term = 0;
        unsigned own = 0, act = 0;
        for (int c = sub; c <= last; c += kWarp) {
          const int id = WC[c];
          const double need = WN[c];
          const int kind = c < first ? (pred < need ? SABER_REJECT_OWN : SABER_REJECT_ACTIVE)
                                     : SABER_ADMIT_HIGH;
          const uint64_t pb = dbits(pred), rb = dbits(need);
          term += decision_term(static_cast<uint64_t>(L.n + c), dbits(t),
                                decision_word(id, kind, load), pb, rb);
          if (kTrace && tr != nullptr)
            write_decision(tr, L.n + c, P.out.trace_cap, P.out.error, t, id, kind, load, pb, rb);
          own += kind == SABER_REJECT_OWN;
          act += kind == SABER_REJECT_ACTIVE;
        }
        L.h += warp_sum_u64(term);
        L.k2 += static_cast<int32_t>(__reduce_add_sync(0xFFFFFFFFu, own));
        L.k3 += static_cast<int32_t>(__reduce_add_sync(0xFFFFFFFFu, act));
        L.n += last + 1;
        cands += last + 1;
        if (first < w) {
          const int id = WC[first];
          const double need = WN[first];
          __syncwarp();  // every lane has read the window before it is reused
          admit(id, t);
          ledger.set(id);
          ++ledger_size;
          if (leader) LNEED[id] = need;
          __syncwarp();
          ledger_max = (ledger_max < need) ? need : ledger_max;
          high.reset(id);
          --hn;
          L.k0 += 1;
        }
        __syncwarp();
      } else if (!kWide && hn > 0) {
        // admission_step, high tier (scheduler.cpp:58-95).
        const int hcount = hn;
        const int w = d.window < hcount ? d.window : hcount;
        if (draw_pos + (w - 1) > draw_len) {
          failed = true;
          break;
        }
        // Fisher-Yates over the window: j = rng() % (i+1) for i = w-1..1.
        // Draws are stored mod lcm(1..16); x % d is exact via the reciprocal
        // table (x < 2^20).  All w-1 draws are independent
        // loads, issued before anything consumes them.
        const double pred = MT[load + 1];
        const bool violates = pred < ledger_max;  // ActiveLedger::violates
        unsigned okmask = 0;
        // The gate (scheduler.cpp:71-94), evaluated for the whole window at
        // once.  Candidate c is admitted iff it is the first with pred >= need
        // and no ledger violation; decisions are then emitted in shuffled order.
        constexpr int kQ = G >= kMaxWindow ? 1 : (kMaxWindow + G - 1) / G;
        int cid[kQ];
        double cneed[kQ];
        if constexpr (G >= kMaxWindow) {
          // Lane q holds draw q, which serves swap i = w-1-q.  Lane c owns
          // shuffled position c: the element FY leaves at c is
          // tau_{w-1}(...tau_1(c)) with tau_i = (i j_i), walked over
          // i = 1..w-1 with compares and selects, all lanes at once.
          int jl = 0;
          if (sub < w - 1) {
            const uint32_t x = draws[draw_pos + sub];
            const uint32_t d1 = static_cast<uint32_t>(w - sub);  // i + 1
            jl = static_cast<int>(x - __umulhi(x, INV[d1]) * d1);
          }
          int pos = sub;
#pragma unroll 1
          for (int q = w - 2; q >= 0; --q) {
            const int i = w - 1 - q;
            const int j = __shfl_sync(gmask, jl, S.col0 + q);
            pos = pos == i ? j : (pos == j ? i : pos);
          }
          cid[0] = 0;
          cneed[0] = 0.0;
          if (sub < w) {
            cid[0] = high.select(pos);
            cneed[0] = queued_need(P.wl.max_out[wo + cid[0]], P.wl.deadline[wo + cid[0]], t);
            if (!(pred < cneed[0]) && !violates) okmask = 1u << sub;
          }
        } else {
          uint32_t xq[kMaxWindow - 1];
#pragma unroll
          for (int q = 0; q < kMaxWindow - 1; ++q) xq[q] = q < w - 1 ? draws[draw_pos + q] : 0u;
          uint64_t ord = 0xFEDCBA9876543210ull;  // window positions as nibbles
#pragma unroll
          for (int q = 0; q < kMaxWindow - 1; ++q) {
            if (q < w - 1) {
              const int i = w - 1 - q;
              const uint32_t d1 = static_cast<uint32_t>(i + 1);
              const uint32_t j = xq[q] - __umulhi(xq[q], INV[d1]) * d1;
              const uint64_t a = (ord >> (4 * i)) & 15ull;
              const uint64_t bb = (ord >> (4 * j)) & 15ull;
              const uint64_t x2 = a ^ bb;
              ord ^= (x2 << (4 * i)) | (x2 << (4 * j));
            }
          }
#pragma unroll
          for (int q = 0; q < kQ; ++q) {
            const int c = sub + G * q;
            cid[q] = 0;
            cneed[q] = 0.0;
            if (c < w) {
              cid[q] = high.select(static_cast<int>((ord >> (4 * c)) & 15ull));
              cneed[q] = queued_need(P.wl.max_out[wo + cid[q]], P.wl.deadline[wo + cid[q]], t);
              if (!(pred < cneed[q]) && !violates) okmask |= 1u << c;
            }
          }
        }
        draw_pos += w - 1;
        rng_draws += w - 1;
        ledger_scanned += ledger_size;
        if (G > 1) okmask = __reduce_or_sync(gmask, okmask);
        const int first = okmask ? __ffs(okmask) - 1 : w;  // admitted position, or none
        gate_idle = first == w;
        gate_w = w;
        gate_pred = pred;
        const int last = first < w ? first : w - 1;
        if constexpr (G == kWarp) {
          // Lane-parallel emission: lane c <= last forms decision c of this
          // tick (rejections before the admitted position, then the
          // admission) at log index L.n + c; the digest terms are summed and
          // the kinds counted over the warp.
          uint64_t term = 0;
          int kind = -1;
          if (sub <= last) {
            kind = sub < first ? (pred < cneed[0] ? SABER_REJECT_OWN : SABER_REJECT_ACTIVE)
                               : SABER_ADMIT_HIGH;
            const uint64_t pb = dbits(pred), rb = dbits(cneed[0]);
            term = decision_term(static_cast<uint64_t>(L.n + sub), dbits(t),
                                 decision_word(cid[0], kind, load), pb, rb);
            if (kTrace && tr != nullptr)
              write_decision(tr, L.n + sub, P.out.trace_cap, P.out.error, t, cid[0], kind, load,
                             pb, rb);
          }
          L.h += warp_sum_u64(term);
          L.k2 += __popc(__ballot_sync(0xFFFFFFFFu, kind == SABER_REJECT_OWN));
          L.k3 += __popc(__ballot_sync(0xFFFFFFFFu, kind == SABER_REJECT_ACTIVE));
          L.n += last + 1;
          cands += last + 1;
          if (first < w) {
            const int id = __shfl_sync(0xFFFFFFFFu, cid[0], first);
            const double need = __shfl_sync(0xFFFFFFFFu, cneed[0], first);
            admit(id, t);
            ledger.set(id);
            ++ledger_size;
            LNEED[id] = need;
            ledger_max = (ledger_max < need) ? need : ledger_max;
            high.reset(id);
            --hn;
            L.k0 += 1;
          }
        } else {
        for (int c = 0; c <= last; ++c) {
          int id;
          double need;
          if (G == 1) {
            id = cid[c];
            need = cneed[c];
          } else {
            const int q = c / G;
            int myid = cid[0];
            double myneed = cneed[0];
#pragma unroll
            for (int qq = 1; qq < kQ; ++qq)
              if (qq == q) {
                myid = cid[qq];
                myneed = cneed[qq];
              }
            id = __shfl_sync(gmask, myid, S.col0 + (c % G));
            need = __shfl_sync(gmask, myneed, S.col0 + (c % G));
          }
          ++cands;
          if (c < first) {
            push_decision<kTrace>(L, t, id, pred < need ? SABER_REJECT_OWN : SABER_REJECT_ACTIVE,
                                  load, dbits(pred), dbits(need), tr, P.out.trace_cap, P.out.error,
                                  leader);
          } else {
            admit(id, t);
            ledger.set(id);
            ++ledger_size;
            LNEED[id] = need;
            ledger_max = (ledger_max < need) ? need : ledger_max;
            high.reset(id);
            --hn;
            push_decision<kTrace>(L, t, id, SABER_ADMIT_HIGH, load, dbits(pred), dbits(need), tr,
                                  P.out.trace_cap, P.out.error, leader);
          }
        }
        }
      } else if (low_head < low_tail) {
        // admission_step, low tier (scheduler.cpp:97-108).
        const int id = LOW[low_head];
        ++low_head;
        const double need = queued_need(P.wl.max_out[wo + id], P.wl.deadline[wo + id], t);
        admit(id, t);
        push_decision<kTrace>(L, t, id, SABER_ADMIT_LOW, load, kAbsent, dbits(need), tr,
                              P.out.trace_cap, P.out.error, leader);
      }
    } else {
      // StaticScheduler::static_step (scheduler.cpp:129-144).
      while (A < d.cap && hn > 0) {
        const int id = high.lowest();
        high.reset(id);
        --hn;
        const int before = A;
        admit(id, t);
        push_decision<kTrace>(L, t, id, SABER_ADMIT_HIGH, before, kAbsent, kAbsent, tr,
                              P.out.trace_cap, P.out.error, leader);
      }
    }

#ifdef SABER_STREAK_STATS
    st_cyc[2] += clock64() - sched_t0;
#endif
    if (t >= horizon) break;

    // Quiet streak: from this tick on, consecutive ticks
    // whose scheduler step is provably a no-op (no arrival, nothing
    // admissible) and whose single engine pass is provably quiet run as one
    // register-resident sweep over the slots.  K is bounded by the next
    // arrival's tick, the horizon, and the prefill / decode minima:
    //   * min_pf_j > dt_j (1 + 1e-12) for every pass j (no prefill ends);
    //   * min_rem_j >= sdt_j (1 + 1e-9) + 1e-15 (m_hi + sdt_j + 1), the
    //     quiet-pass test below (decode boundary cannot bind, no completion);
    // both minima shrink by at most dt_max / speed*dt_max (+ rounding) per pass.
    // A SABER tick whose gate admitted nobody starts a gate streak: with the
    // high tier, load and ledger unchanged, every later tick of the streak
    // rejects the same window again (need = m / (dl - t) only grows), so its
    // decisions are generated lane-parallel (gate_streak below).
    const bool gate_streak = saber && hn > 0;
#ifdef SABER_STREAK_STATS
    {
      const bool cond = saber ? (gate_streak ? (!kWide && G >= kMaxWindow && gate_idle) : low_head == low_tail)
                              : !(A < d.cap && hn > 0);
      if (use_tab && !(!sblock && A > 0 && cond))
        st_cause[sblock ? 8 : A == 0 ? 9 : (gate_streak && !gate_idle) ? 10 : 11] += 1;
    }
#endif
    if (use_tab && !sblock && A > 0 &&
        (saber ? (gate_streak ? (!kWide && G >= kMaxWindow && gate_idle) : low_head == low_tail)
               : !(A < d.cap && hn > 0))) {
      const int k0 = ticks - 1;
      const double dtm = P.ticks.dt_max;
      // Kb passes keep both minima provably quiet: for pass j <= Kb - 1 the
      // remaining margin is still >= one full per-pass decrement.
      int Kb = 1 << 30;
      if (npre > 0) Kb = floor_div_lb(min_pf * (1.0 - 2e-7), dtm * (1.0 + 1e-6));
      double delta = 0.0;
      if (A > npre) {
        const double sm = speed_A * dtm * (1.0 + 1e-15);
        delta = sm * (1.0 + 1e-6) + 2e-15 * (m_hi + sm + 1.0);
        Kb = min(Kb, floor_div_lb(rem_lb, delta));
      }
      // The bounds only shrink until the next admission / exact pass.
      if (Kb < 2) sblock = true;
      // Arrivals that cannot change any scheduler step of the streak are
      // absorbed into it: a SABER gate streak whose window
      // is full (a new id enters the high tier behind the window, so every
      // gate of the streak sees the same w candidates).  (Static streaks with
      // a full batch could absorb arrivals too, but they end at the next
      // prefill end / completion long before an arrival: measured no gain.)
      const bool absorb = gate_streak && hn >= d.window;
      int K = 0;
      if (Kb >= 2) {
        K = min(Kb, kh - 1 - k0);
        if (!absorb) K = min(K, ka - k0);
        if (gate_streak) {
          // no refresh scan (t < min_td) and enough scheduler draws
          K = min(K, min_kd - k0);
          // K - 1 further gates of gate_w - 1 draws each must fit the stream;
          // the (64-bit) division only when they might not
          if (gate_w > 1 && static_cast<int64_t>(K - 1) * (gate_w - 1) > draw_len - draw_pos)
            K = static_cast<int>(1 + (draw_len - draw_pos) / (gate_w - 1));
        }
      }
#ifdef SABER_STREAK_STATS
      {
        const int kbv = Kb;
        const int kav = absorb ? 1 << 30 : ka - k0;
        const int kdv = gate_streak ? min(min_kd - k0, gate_w > 1 ? static_cast<int>(min(static_cast<int64_t>(1 << 30), 1 + (draw_len - draw_pos) / (gate_w - 1))) : 1 << 30) : 1 << 30;
        const int base = K >= 2 ? 0 : 4;
        const int Kc = Kb < 2 ? Kb : K;
        st_cause[base + (Kc == kbv ? 0 : Kc == kav ? 1 : Kc == kdv ? 2 : 3)] += 1;
      }
#endif
      const int hc_streak = gate_streak ? hn : 0;
      int64_t arr_extra = 0;  // high-tier entries the absorbed arrivals add to later refreshes
      if (absorb && K >= 2 && next < n && ka < k0 + K) {
        // the streak must also end before any absorbed request's demotion
        // bound tick (its refresh could demote it)
        if (saber) {
          for (int q = next; q < n && P.wl.arr_tick[wo + q] < k0 + K; ++q)
            K = min(K, P.wl.dem_tick[wo + q] - k0);
        }
        if (K >= 2) {
          while (next < n) {
            const int a = P.wl.arr_tick[wo + next];
            if (a >= k0 + K) break;
            high.set(next);
            ++hn;
            if (saber) {
              min_td = dmin(min_td, P.wl.demote_after[wo + next]);
              min_kd = min(min_kd, P.wl.dem_tick[wo + next]);
            }
            arr_extra += k0 + K - a;
            ++next;
          }
          na_t = next < n ? P.wl.arrival[wo + next] : kInf;
          ka = next < n ? P.wl.arr_tick[wo + next] : P.ticks.len;
        }
      }
      if (K >= 2) {
#ifdef SABER_DEBUG_CHECKS
        if (P.ticks.T[k0] != t || clock != t) {  // invariant t_k == T[k] at a tick start
          if (leader) atomicCAS(P.out.error, kErrNone, kErrTickTable);
          use_tab = false;
        } else
#endif
        {
          const double t_after = P.ticks.T[k0 + K];  // issued early, used after the sweep
          const double* __restrict__ DTk = P.ticks.DT + k0;
          // min_pf stays exact: the same per-pass chain min_pf -= dt
          {
            SEC_BEGIN();
            min_pf = streak_slots<G, kSel == kSelSaber>(S, sub, A, npre, speed_A, DTk, K, min_pf);
            SEC_END(1);
          }
          if (A > npre) rem_lb = rem_lb - static_cast<double>(K) * delta;
          rem_exact = false;
          if constexpr (!kWide) if (gate_streak) {
            SEC_BEGIN();
            if constexpr (G == kWarp)
              gate_streak_warp<kTrace, NW>(P, S, sub, high, P.wl.max_out + wo, P.wl.deadline + wo,
                                           draws, draw_pos, k0, K, gate_w, A, gate_pred, L, tr, INV);
            else
              gate_streak_decisions<G, kTrace, NW>(P, S, sub, gmask, high, P.wl.max_out + wo,
                                                   P.wl.deadline + wo, draws, draw_pos, k0, K,
                                                   gate_w, A, gate_pred, L, tr, INV);
            SEC_END(0);
            const int64_t extra = K - 1;
            draw_pos += extra * (gate_w - 1);
            rng_draws += static_cast<int32_t>(extra * (gate_w - 1));
            cands += static_cast<int32_t>(extra * gate_w);
            ledger_scanned += static_cast<int32_t>(extra * ledger_size);
            refresh_entries += static_cast<int32_t>(extra * hc_streak + arr_extra);
          }
#ifdef SABER_STREAK_STATS
          st_ticks += K;
          st_count += 1;
#endif
          // A streak that used up the engine bound leaves < 2 passes of it:
          // the next attempt would fail, so none is made until the next
          // event resets sblock (streaks are an optimisation; skipping one
          // never changes a result).
#ifndef SABER_SBLOCK_AFTER_KB
#define SABER_SBLOCK_AFTER_KB 1
#endif
          if (SABER_SBLOCK_AFTER_KB && K == Kb) sblock = true;
          ticks += K - 1;  // this tick was counted above
          passes += K;
          prefill_updates += K * npre;
          decode_updates += K * (A - npre);
          t = t_after;
          clock = t;
          continue;
        }
      }
    }
    // Idle engine and empty queues: nothing happens before the tick of the
    // next arrival, so those ticks (each: no scheduler action, advance_to
    // with no active request) are skipped on the tick table.
#ifndef SABER_IDLE_SKIP
#define SABER_IDLE_SKIP 1
#endif
    if (SABER_IDLE_SKIP && use_tab && A == 0 && completed < n && hn == 0 &&
        low_head == low_tail) {
      const int k0 = ticks - 1;
      const int kj = min(ka, kh - 1);
      if (kj - k0 >= 2) {
        ticks += kj - k0 - 1;
        t = P.ticks.T[kj];
        clock = t;
        continue;
      }
    }
    const double nt = (horizon < t + tick) ? horizon : t + tick;

    // Engine::advance_to(nt) (engine.cpp:51-127).
#ifdef SABER_STREAK_STATS
    const long long eng_t0 = clock64();
#endif
    while (clock < nt) {
      if (A == 0) {
        clock = nt;
        break;
      }
      ++passes;
      double dt = nt - clock;
      const double speed = speed_A;
      if (min_pf < dt) dt = min_pf;
      // Quiet pass: no prefill ends (min_pf is exact) and the
      // lower bound on min(max_out - generated) proves both that the decode
      // boundary cannot bind and that no slot can satisfy the completion
      // test.  Every slot then just advances, and the new minima follow from
      // the scalars: min fl(pl - dt) == fl(min_pf - dt) (monotone rounding).
      const double sdt0 = speed * dt;
      const bool quiet = !(min_pf <= dt * kOnePlusTol) &&
                         rem_lb >= sdt0 * (1.0 + 1e-9) + 1e-15 * (m_hi + sdt0 + 1.0);
      if (quiet) {
        const double sdt = sdt0;
#pragma unroll 4
        for (int k = sub, s = S.idx(sub); k < A; k += G, s += kWarp) {
          const double g = S.g[s];
          S.g[s] = g < 0.0 ? g + dt : g + sdt;
        }
        min_pf = min_pf - dt;  // == min over prefill slots of fl(pl - dt)
        rem_lb = (rem_lb - sdt) - 1e-15 * (m_hi + sdt + fabs(rem_lb));
        rem_exact = false;
        prefill_updates += npre;
        decode_updates += A - npre;
        clock = clock + dt;
#ifdef SABER_STREAK_STATS
        st_quiet += 1;
#endif
        continue;
      }
      // Exact pass.  First make the decode minimum exact if it is a bound.
      sblock = false;
#ifdef SABER_STREAK_STATS
      st_exact += 1;
#endif
      // (Only needed when the bound cannot already show that the decode
      // boundary does not bind this pass: min_rem >= rem_lb >= speed*dt*(1+1e-12)
      // gives fl(min_rem / speed) > dt.  The pass below recomputes the exact
      // minimum either way.)
      if (!rem_exact && rem_lb < speed * dt * kOnePlusTol) {
        double r = kInf;
#pragma unroll 1
        for (int k = sub, s = S.idx(sub); k < A; k += G, s += kWarp) {
          const double g = S.g[s];
          if (g >= 0.0) r = dmin(r, bitsd(S.m[s] & ~kIdMask) - g);
        }
        rem_lb = group_min_pos<G>(r, gmask);
        rem_exact = true;
      }
      // dt = min(dt, fl(min_rem / speed)); the divide can only bind when
      // min_rem < speed * dt * (1 + 1e-12) (see header).
      if (rem_lb < speed * dt * kOnePlusTol) {
        const double bnd = rem_lb / speed;
        if (bnd < dt) dt = bnd;
      }
      const double group = dt * kOnePlusTol;
      const double sdt = speed * dt;
      const double sgd = speed * (group - dt);
      const double nclock = clock + dt;
      double npf = kInf, nrem = kInf;
      unsigned counts = 0;  // (done << 16) | still-in-prefill
      int done_k = -1, done_id = -1;  // this lane's last completed slot / request
      for (int k = sub, s = S.idx(sub); k < A; k += G, s += kWarp) {
        double g = S.g[s];
        const uint64_t mb = S.m[s];
        const double m = bitsd(mb & ~kIdMask);
        bool done;
        if (g < 0.0) {  // prefill slot: g = -prefill_left
          if (-g <= group) {
            g = 0.0;  // decode starts at nclock
            done = g + sgd >= m;
          } else {
            g = g + dt;  // == -(prefill_left - dt), exactly
            npf = dmin(npf, -g);
            ++counts;
            done = false;
          }
        } else {
          g = g + sdt;
          done = g + sgd >= m;
        }
        if (!done) {
          if (g >= 0.0) nrem = dmin(nrem, m - g);
          S.g[s] = g;
        } else {
          S.g[s] = bitsd(kDoneMark);
          done_id = static_cast<int>(mb & kIdMask);
          done_k = k;
          COMP[done_id] = nclock;
          counts += 1u << 16;
        }
      }
      prefill_updates += npre;
      decode_updates += A - npre;
      min_pf = group_min_pos<G>(npf, gmask);
      rem_lb = group_min_pos<G>(nrem, gmask);
      rem_exact = true;
      const unsigned tot = group_sum<G>(counts, gmask);
      npre = static_cast<int>(tot & 0xFFFFu);
      const unsigned ndone = tot >> 16;
      if (ndone == 1) {
        // One completion (the common event): fetch it from its owner lane,
        // update the replicated ledger, and swap the last slot into its place.
        unsigned owner = 0;
        if (G > 1) owner = __ffs(__ballot_sync(gmask, done_k >= 0)) - 1;
        const int k = G > 1 ? __shfl_sync(gmask, done_k, owner) : done_k;
        const int id = G > 1 ? __shfl_sync(gmask, done_id, owner) : done_id;
        if (saber && ledger.test(id)) {
          ledger.reset(id);
          --ledger_size;
          ledger_max = ledger_max_of<G, NW>(ledger, ledger_size, LNEED, sub);
        }
        if (k != A - 1) {
          const int dst = S.idx(k), src = S.idx(A - 1);
          __syncwarp(gmask);
          if (leader) {
            S.g[dst] = S.g[src];
            S.m[dst] = S.m[src];
          }
          __syncwarp(gmask);
        }
        A -= 1;
        retune();
        completed += 1;
      } else if (ndone) {
        // Several completions in one pass (lockstep bursts): every lane
        // replays them for the replicated scheduler state, then the leader
        // compacts the slot array by swap-with-last.
        __syncwarp(gmask);
        bool dirty = false;
#pragma unroll 1
        for (int k = 0; k < A; ++k) {
          const int s = S.idx(k);
          if (dbits(S.g[s]) != kDoneMark) continue;
          const int id = static_cast<int>(S.m[s] & kIdMask);
          if (saber && ledger.test(id)) {
            ledger.reset(id);
            --ledger_size;
            dirty = true;
          }
        }
        __syncwarp(gmask);
        if (leader) {
          int a = A;
          for (int k = 0; k < a;) {
            const int s = S.idx(k);
            if (dbits(S.g[s]) != kDoneMark) {
              ++k;
              continue;
            }
            const int last = S.idx(a - 1);
            S.g[s] = S.g[last];
            S.m[s] = S.m[last];
            --a;
          }
        }
        __syncwarp(gmask);
        A -= static_cast<int>(ndone);
        retune();
        completed += static_cast<int>(ndone);
        if (dirty) ledger_max = ledger_max_of<G, NW>(ledger, ledger_size, LNEED, sub);
      }
      clock = nclock;
    }
#ifdef SABER_STREAK_STATS
    st_cyc[3] += clock64() - eng_t0;
#endif
    t = nt;
    if (completed == n) break;
  }

  if (failed && leader) atomicCAS(P.out.error, kErrNone, kErrRngExhausted);
  if (kRecords && P.out.generated) {
    // fluid progress of the requests still running (Request::generated_tokens;
    // a slot in prefill has generated nothing yet)
    double* __restrict__ GEN = P.out.generated + d.row * nmax;
    for (int k = sub, s = S.idx(sub); k < A; k += G, s += kWarp) {
      const double g = S.g[s];
      GEN[static_cast<int>(S.m[s] & kIdMask)] = g < 0.0 ? 0.0 : g;
    }
  }
  if (leader) {
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
    R->last_arrival = n > 0 ? P.wl.arrival[wo + n - 1] : 0.0;
    R->horizon = horizon;
#ifdef SABER_STREAK_STATS
    R->last_arrival = st_ticks;
    R->horizon = st_count;
    R->ratio_mean = static_cast<double>(clock64() - st_t0);  // overwritten by row metrics
    R->n_kind[4] = clock64() - st_t0;
    for (int q = 0; q < 4; ++q) R->n_kind[q] = st_cyc[q];
    R->rng_draws = st_cyc[4];
    R->gate_candidates = st_scans;
    R->decision_hash = (static_cast<uint64_t>(st_quiet) << 32) | static_cast<uint32_t>(st_exact);
    R->refresh_entries = 0;
    R->ledger_scanned = 0;
    R->prefill_updates = 0;
    for (int q = 0; q < 4; ++q) {
      R->refresh_entries |= static_cast<int64_t>(min(st_cause[q], 0xFFFF)) << (16 * q);
      R->ledger_scanned |= static_cast<int64_t>(min(st_cause[4 + q], 0xFFFF)) << (16 * q);
      R->prefill_updates |= static_cast<int64_t>(min(st_cause[8 + q], 0xFFFF)) << (16 * q);
    }
#endif
    if (kTrace && P.out.trace_count) P.out.trace_count[d.row] = L.n;
  }
}

template <int NW, int G, bool kTrace, bool kRecords, int kSel>
__global__ void __launch_bounds__(kSimBlock, kSel == kSelStatic  ? SABER_STATIC_MIN_BLOCKS
                                             : kSel == kSelSaber ? SABER_SABER_MIN_BLOCKS
                                                                 : SABER_SIM_MIN_BLOCKS)
    sim_kernel(const SimParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  __shared__ uint32_t inv[kMaxWindow + 1];  // ceil(2^32 / d) for d = 2..16
  if (threadIdx.x >= 2 && threadIdx.x <= kMaxWindow)
    inv[threadIdx.x] = static_cast<uint32_t>((0x100000000ull + threadIdx.x - 1) / threadIdx.x);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = lane / G;
  const int sub = lane % G;
  const unsigned gmask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << (grp * G);
  const int rows = P.slot_rows;
  uint64_t* tile = smem + static_cast<size_t>(warp) * rows * kWarp * 2;
  Slots<G> S;
  S.g = reinterpret_cast<double*>(tile);
  S.m = tile + static_cast<size_t>(rows) * kWarp;
  S.dbuf = reinterpret_cast<uint32_t*>(smem + static_cast<size_t>(kSimBlock / kWarp) * rows * kWarp * 2) +
           static_cast<size_t>(warp) * kWarp * (kMaxWindow - 1) + grp * G * (kMaxWindow - 1);
  S.col0 = grp * G;
  const int64_t group_id =
      (static_cast<int64_t>(blockIdx.x) * (kSimBlock / kWarp) + warp) * (kWarp / G) + grp;
  if (group_id >= P.scratch.groups) {  // scratch sized for a smaller grid: loud, never silent
    if (lane == 0) atomicCAS(P.out.error, kErrNone, kErrBadDesc);
    return;
  }
  double* LNEED = P.scratch.ledger_need + group_id * P.wl.nmax;
  uint16_t* LOW = P.scratch.low_fifo + group_id * P.wl.nmax;
  for (;;) {
    int ti = 0;
    if (sub == 0) ti = P.first_traj + atomicAdd(P.next_traj, 1);
    ti = __shfl_sync(gmask, ti, grp * G);
    if (ti >= P.n_traj) break;
    simulate_one<NW, G, kTrace, kRecords, kSel>(P, ti, S, sub, gmask, LNEED, LOW, inv);
    __syncwarp(gmask);
  }
}

// The wide kernel: one trajectory per warp, slots, tier
// masks and the gate window in the warp's global scratch (L1/L2-resident),
// any n <= kMaxRequestsWide and any window.  No dynamic shared memory.
template <bool kTrace, bool kRecords>
__global__ void __launch_bounds__(kSimBlock) sim_kernel_wide(const SimParams P) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t group_id = static_cast<int64_t>(blockIdx.x) * (kSimBlock / kWarp) + warp;
  if (group_id >= P.scratch.groups) {
    if (lane == 0) atomicCAS(P.out.error, kErrNone, kErrBadDesc);
    return;
  }
  const int64_t nmax = P.wl.nmax;
  const int nw = P.scratch.wmask_nw;
  Slots<kWarp> S;
  S.g = P.scratch.wslot_g + group_id * nmax;
  S.m = P.scratch.wslot_m + group_id * nmax;
  S.dbuf = nullptr;
  S.col0 = 0;
  WideScratch WS;
  WS.masks = P.scratch.wmask + group_id * 2 * nw;
  WS.nw = nw;
  WS.gate = P.scratch.wgate + group_id * 3 * nmax;
  WS.need = P.scratch.wneed + group_id * nmax;
  double* LNEED = P.scratch.ledger_need + group_id * nmax;
  uint16_t* LOW = P.scratch.low_fifo + group_id * nmax;
  for (;;) {
    int ti = 0;
    if (lane == 0) ti = P.first_traj + atomicAdd(P.next_traj, 1);
    ti = __shfl_sync(0xFFFFFFFFu, ti, 0);
    if (ti >= P.n_traj) break;
    simulate_one<1, kWarp, kTrace, kRecords, kSelAny, true>(P, ti, S, lane, 0xFFFFFFFFu, LNEED,
                                                            LOW, nullptr, WS);
    __syncwarp();
  }
}

template <int NW, int G, bool kTrace, bool kRecords, int kSel = kSelAny>
void* kernel_ptr() {
  return reinterpret_cast<void*>(&sim_kernel<NW, G, kTrace, kRecords, kSel>);
}

// Mode-specialised variants exist for the bench path only: G = 32, no trace,
// no per-request records; everything else uses kSelAny.
template <int NW, int G>
void* pick_tr(bool trace, bool records, int sel) {
  if (trace) return kernel_ptr<NW, G, true, true>();
  if (records) return kernel_ptr<NW, G, false, true>();
  if (G == kWarp && sel == kSelStatic) return kernel_ptr<NW, kWarp, false, false, kSelStatic>();
  if (G == kWarp && sel == kSelSaber) return kernel_ptr<NW, kWarp, false, false, kSelSaber>();
  return kernel_ptr<NW, G, false, false>();
}

template <int NW>
void* pick_g(int g, bool trace, bool records, int sel) {
  switch (g) {
    case 1: return pick_tr<NW, 1>(trace, records, sel);
    case 2: return pick_tr<NW, 2>(trace, records, sel);
    case 4: return pick_tr<NW, 4>(trace, records, sel);
    case 8: return pick_tr<NW, 8>(trace, records, sel);
    case 16: return pick_tr<NW, 16>(trace, records, sel);
    case 32: return pick_tr<NW, 32>(trace, records, sel);
  }
  return nullptr;
}

}  // namespace
}  // namespace saberb200
