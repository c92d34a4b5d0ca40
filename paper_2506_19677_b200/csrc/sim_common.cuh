// sim_common.cuh — device helpers of the trajectory kernels (sim_kernel.cu,
// mc.cu).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "saber_internal.h"

namespace saberb200 {
namespace simdev {

constexpr double kInf = __builtin_huge_val();
constexpr double kOnePlusTol = 1.0 + 1e-12;  // engine.cpp:17,76 (kGroupTol)
constexpr uint64_t kHashSeed = 0;  // oracle.h ORC_HASH_SEED: the empty log
constexpr uint64_t kAbsent = 0xFFF8000000000001ULL;
constexpr uint64_t kDoneMark = 0xFFF0DEAD0000DEADULL;  // a NaN the engine never produces
constexpr uint64_t kIdMask = 0xFFFFull;

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
// One decision's term of the log digest (oracle.h orc_decision_term).
__device__ __forceinline__ uint64_t decision_term(uint64_t index, uint64_t tb, uint64_t w,
                                                  uint64_t pb, uint64_t rb) {
  const uint64_t x = w ^ rotl64(pb, 17) ^ rotl64(rb, 43) ^ rotl64(tb, 7);
  return mix64(x + (index + 1) * 0x9E3779B97F4A7C15ULL);
}
__device__ __forceinline__ uint64_t dbits(double v) {
  return static_cast<uint64_t>(__double_as_longlong(v));
}
__device__ __forceinline__ double bitsd(uint64_t b) {
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }

// required_speed (types.cpp:82-88) for a queued request: generated == 0.
__device__ __forceinline__ double queued_need(double max_out, double deadline,
                                              double now) {
  if (now >= deadline) return kInf;
  const double remaining = max_out - 0.0;
  if (remaining <= 0.0) return 0.0;
  return remaining / (deadline - now);
}

// Group minimum of a non-negative double (IEEE order == unsigned bit order).
template <int G>
__device__ __forceinline__ double group_min_pos(double v, unsigned gmask) {
  if (G == 1) return v;
  const uint64_t b = dbits(v);
  const unsigned hi = static_cast<unsigned>(b >> 32);
  const unsigned lo = static_cast<unsigned>(b);
  const unsigned mhi = __reduce_min_sync(gmask, hi);
  const unsigned mlo = __reduce_min_sync(gmask, hi == mhi ? lo : 0xFFFFFFFFu);
  return bitsd((static_cast<uint64_t>(mhi) << 32) | mlo);
}
template <int G>
__device__ __forceinline__ unsigned group_sum(unsigned v, unsigned gmask) {
  if (G == 1) return v;
  return __reduce_add_sync(gmask, v);
}

// Whole-warp reductions (G == 32 paths).  dkey maps a non-NaN double to a
// 64-bit key whose unsigned order is the double order (-0 < +0 is harmless:
// the keys are only compared, and keyd inverts dkey exactly).
__device__ __forceinline__ uint64_t dkey(double v) {
  const uint64_t b = dbits(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double keyd(uint64_t k) {
  return bitsd((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k);
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32);
  const unsigned mhi = __reduce_min_sync(0xFFFFFFFFu, hi);
  const unsigned mlo =
      __reduce_min_sync(0xFFFFFFFFu, hi == mhi ? static_cast<unsigned>(v) : 0xFFFFFFFFu);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32);
  const unsigned mhi = __reduce_max_sync(0xFFFFFFFFu, hi);
  const unsigned mlo = __reduce_max_sync(0xFFFFFFFFu, hi == mhi ? static_cast<unsigned>(v) : 0u);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}
// Sum mod 2^64 over the warp with three 32-bit REDUX.SUMs: the low word in
// two 16-bit halves (each sum < 2^21, exact, so the carry into the high word
// is exact) and the high word mod 2^32.
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
  const unsigned lo = static_cast<unsigned>(v), hi = static_cast<unsigned>(v >> 32);
  const unsigned s0 = __reduce_add_sync(0xFFFFFFFFu, lo & 0xFFFFu);
  const unsigned s1 = __reduce_add_sync(0xFFFFFFFFu, lo >> 16);
  const unsigned sh = __reduce_add_sync(0xFFFFFFFFu, hi);
  return (static_cast<uint64_t>(sh) << 32) + (static_cast<uint64_t>(s1) << 16) + s0;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Position of the k-th set bit of x (0-based, k < popc(x)): branch-free
// binary search on popcounts (no data-dependent loop, so lanes asking for
// different k stay converged).
__device__ __forceinline__ int select64(uint64_t x, int k) {
  uint32_t v = static_cast<uint32_t>(x);
  int pos = 0;
  int c = __popc(v);
  if (k >= c) {
    k -= c;
    pos = 32;
    v = static_cast<uint32_t>(x >> 32);
  }
  c = __popc(v & 0xFFFFu);
  if (k >= c) { k -= c; pos += 16; v >>= 16; }
  c = __popc(v & 0xFFu);
  if (k >= c) { k -= c; pos += 8; v >>= 8; }
  c = __popc(v & 0xFu);
  if (k >= c) { k -= c; pos += 4; v >>= 4; }
  c = __popc(v & 0x3u);
  if (k >= c) { k -= c; pos += 2; v >>= 2; }
  if (k >= static_cast<int>(v & 1u)) pos += 1;
  return pos;
}

// Per-request tier membership as an NW x 64-bit register bitmask.  Built as a
// recursive struct of scalar words (no array), so a runtime word index can
// never turn into a local-memory access.
template <int NW, int B = 0>
struct Mask {
  static constexpr bool kGlobal = false;
  uint64_t w;
  Mask<NW - 1, B + 1> r;
  __device__ __forceinline__ void clear() { w = 0; r.clear(); }
  __device__ __forceinline__ void set(int id) {
    if ((id >> 6) == B) w |= 1ull << (id & 63);
    else r.set(id);
  }
  __device__ __forceinline__ void reset(int id) {
    if ((id >> 6) == B) w &= ~(1ull << (id & 63));
    else r.reset(id);
  }
  __device__ __forceinline__ bool test(int id) const {
    return (id >> 6) == B ? ((w >> (id & 63)) & 1ull) != 0 : r.test(id);
  }
  __device__ __forceinline__ uint64_t word(int i) const { return i == B ? w : r.word(i); }
  __device__ __forceinline__ void andnot(int i, uint64_t m) {
    if (i == B) w &= ~m;
    else r.andnot(i, m);
  }
  __device__ __forceinline__ bool any() const { return w != 0 || r.any(); }
  __device__ __forceinline__ int word_begin() const { return 0; }
  __device__ __forceinline__ int word_end() const { return NW; }
  __device__ __forceinline__ int count() const { return __popcll(w) + r.count(); }
  __device__ __forceinline__ int lowest() const {
    return w ? B * 64 + __ffsll(static_cast<long long>(w)) - 1 : r.lowest();
  }
  // k-th set bit in ascending id order (0-based); k < count().  The word
  // holding it is picked with selects (no per-word copy of select64).
  __device__ __forceinline__ void pick(int& k, uint64_t& word, int& base) const {
    const int c = __popcll(w);
    if (k < c) {
      word = w;
      base = B * 64;
    } else {
      k -= c;
      r.pick(k, word, base);
    }
  }
  __device__ __forceinline__ int select(int k) const {
    uint64_t word = w;
    int base = 0;
    pick(k, word, base);
    return base + select64(word, k);
  }
};
template <int B>
struct Mask<0, B> {
  static constexpr bool kGlobal = false;
  __device__ __forceinline__ void clear() {}
  __device__ __forceinline__ void set(int) {}
  __device__ __forceinline__ void reset(int) {}
  __device__ __forceinline__ bool test(int) const { return false; }
  __device__ __forceinline__ uint64_t word(int) const { return 0; }
  __device__ __forceinline__ void andnot(int, uint64_t) {}
  __device__ __forceinline__ bool any() const { return false; }
  __device__ __forceinline__ int count() const { return 0; }
  __device__ __forceinline__ int lowest() const { return -1; }
  __device__ __forceinline__ int select(int) const { return -1; }
  __device__ __forceinline__ void pick(int&, uint64_t&, int&) const {}
};

// Tier mask of the wide kernel: `nw` 64-bit words in the
// group's global scratch, plus scalar copies (identical on every lane) of
// the member count, a lower bound `lo` on the first non-empty word and an
// upper bound `hi` on the last one.  Every lane reads the words; lane 0
// alone writes them, between two __syncwarp()s, so no lane ever observes a
// half-applied update.  Whole-warp groups only (G = 32).
struct GMask {
  static constexpr bool kGlobal = true;
  uint64_t* p;
  int nw, cnt, lo, hi;
  bool leader;
  __device__ __forceinline__ void bind(uint64_t* words, int n_words, int sub) {
    p = words;
    nw = n_words;
    leader = sub == 0;
  }
  __device__ __forceinline__ void clear() {
    __syncwarp();
    for (int i = static_cast<int>(threadIdx.x & 31); i < nw; i += 32) p[i] = 0;
    __syncwarp();
    cnt = 0;
    lo = 0;
    hi = 0;
  }
  __device__ __forceinline__ void put(int i, uint64_t v) {
    __syncwarp();
    if (leader) p[i] = v;
    __syncwarp();
  }
  __device__ __forceinline__ void set(int id) {
    const int i = id >> 6;
    put(i, p[i] | (1ull << (id & 63)));
    ++cnt;
    hi = hi > i + 1 ? hi : i + 1;
  }
  __device__ __forceinline__ void reset(int id) {
    const int i = id >> 6;
    put(i, p[i] & ~(1ull << (id & 63)));
    --cnt;
  }
  __device__ __forceinline__ bool test(int id) const { return ((p[id >> 6] >> (id & 63)) & 1ull) != 0; }
  __device__ __forceinline__ uint64_t word(int i) const { return p[i]; }
  __device__ __forceinline__ void andnot(int i, uint64_t m) {
    const uint64_t w = p[i];
    cnt -= __popcll(w & m);
    put(i, w & ~m);
  }
  __device__ __forceinline__ bool any() const { return cnt > 0; }
  __device__ __forceinline__ int count() const { return cnt; }
  __device__ __forceinline__ int word_begin() const { return lo; }
  __device__ __forceinline__ int word_end() const { return hi; }
  // lowest member (cnt > 0); advances lo past empty words (uniform call)
  __device__ __forceinline__ int lowest() {
    while (p[lo] == 0) ++lo;
    return lo * 64 + __ffsll(static_cast<long long>(p[lo])) - 1;
  }
  // k-th member in ascending id order (k < cnt); per-lane k may differ
  __device__ __forceinline__ int select(int k) const {
    for (int i = lo;; ++i) {
      const uint64_t w = p[i];
      const int c = __popcll(w);
      if (k < c) return i * 64 + select64(w, k);
      k -= c;
    }
  }
};

struct DecisionLog {
  uint64_t h;
  int32_t n;
  int32_t k0, k1, k2, k3, k4;
};

// One full decision record (trace mode) at log index idx.
__device__ __forceinline__ void write_decision(saber_decision* tr, int64_t idx, int64_t cap,
                                               int32_t* err, double t, int id, int kind, int load,
                                               uint64_t pb, uint64_t rb) {
  if (idx < cap) {
    saber_decision& d = tr[idx];
    d.time = t;
    d.request_id = static_cast<uint64_t>(id);
    d.kind = kind;
    d.load_before = load;
    d.has_pred = pb != kAbsent;
    d.has_req = rb != kAbsent;
    d.pred_speed = pb != kAbsent ? bitsd(pb) : nan("");
    d.req_speed = rb != kAbsent ? bitsd(rb) : nan("");
  } else {
    atomicCAS(err, kErrNone, kErrTraceOverflow);
  }
}

__device__ __forceinline__ uint64_t decision_word(int id, int kind, int load) {
  return static_cast<uint64_t>(static_cast<uint32_t>(id)) | (static_cast<uint64_t>(kind) << 32) |
         (static_cast<uint64_t>(static_cast<uint32_t>(load)) << 40);
}

template <bool kTrace>
__device__ __forceinline__ void push_decision(DecisionLog& L, double t, int id,
                                              int kind, int load, uint64_t pb,
                                              uint64_t rb, saber_decision* tr,
                                              int64_t cap, int32_t* err, bool writer) {
  L.h += decision_term(static_cast<uint64_t>(L.n), dbits(t), decision_word(id, kind, load), pb, rb);
  if (kTrace && tr != nullptr && writer) write_decision(tr, L.n, cap, err, t, id, kind, load, pb, rb);
  ++L.n;
  L.k0 += kind == 0;
  L.k1 += kind == 1;
  L.k2 += kind == 2;
  L.k3 += kind == 3;
  L.k4 += kind == 4;
}


}  // namespace simdev
}  // namespace saberb200
