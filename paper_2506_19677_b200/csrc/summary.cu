// summary.cu — sweep summary on the device (simloop.cpp:206-275).
//
// S0 (grid-parallel): ratio[row][q] = (completion - arrival) / sla, NaN when
//    the request never completed (ratio_to_sla, metrics.cpp:39-47).
// S1 (warp per (mix, rps)): per-cell mean goodput over repeats, the static
//    argmax over caps in ascending order with ties to the smaller cap, and the
//    per-cell latency-ratio means.
// S2 (warp per (mix, variant)): means over the rps grid, pooled CVs over every
//    ratio of the chosen cells, and CVs of the per-rps ratio means.
// The reference's sums are sequential left-to-right double additions, so the
// summary is bit-identical only if the device adds in the same order.  The
// sums therefore stay sequential, but a whole warp streams the contiguous
// ratio blocks (coalesced 256-byte loads) and hands the values to the
// dependent add chain through shuffles, so the chain never waits on memory.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdlib>

#include "exact_sum.cuh"
#include "saber_internal.h"

namespace saberb200 {
namespace {

using exactsum::block_exact_seq_sum;
using exactsum::kExactK;
using exactsum::kExactThreads;

constexpr int kCellScratch = 6;
constexpr int kMaxSegments = 512;  // rps values of one pool the exact-sum kernel indexes
constexpr unsigned kFull = 0xFFFFFFFFu;

__global__ void __launch_bounds__(256) ratios_kernel(const SummaryParams p) {
  const int64_t total = static_cast<int64_t>(p.n_mixes) * p.n_rps *
                        (static_cast<int64_t>(p.n_caps) * p.repeats + (p.with_saber ? p.repeats : 0)) *
                        p.n;
  const int per_rps = p.n_caps * p.repeats + (p.with_saber ? p.repeats : 0);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / p.n;
    const int q = static_cast<int>(i % p.n);
    const int64_t cell = row / per_rps;
    const int rem = static_cast<int>(row % per_rps);
    const int rep = rem < p.n_caps * p.repeats ? rem % p.repeats : rem - p.n_caps * p.repeats;
    const int64_t w = cell * p.repeats + rep;  // workload (mix, rps, seed)
    const double c = p.completion[row * p.wl.nmax + q];
    const int64_t o = w * p.wl.nmax + q;
    p.ratios[i] = isnan(c) ? nan("") : (c - p.wl.arrival[o]) / p.wl.sla[o];
  }
}

// Sequential sums over `len` contiguous values (NaN = absent), in order.  The
// warp loads 8 x 32 values per lane-batch and prefetches the next batch while
// the dependent add chain consumes the current one through shuffles.
constexpr int kBatch = 8;

template <class F>
__device__ __forceinline__ void warp_stream(const double* v, int64_t len, F&& consume) {
  const int lane = threadIdx.x & 31;
  double cur[kBatch], nxt[kBatch];
#pragma unroll
  for (int c = 0; c < kBatch; ++c) {
    const int64_t i = c * 32 + lane;
    cur[c] = i < len ? v[i] : nan("");
  }
  for (int64_t base = 0; base < len; base += 32 * kBatch) {
#pragma unroll
    for (int c = 0; c < kBatch; ++c) {
      const int64_t i = base + 32 * kBatch + c * 32 + lane;
      nxt[c] = i < len ? v[i] : nan("");
    }
#pragma unroll
    for (int c = 0; c < kBatch; ++c) {
#pragma unroll
      for (int j = 0; j < 32; ++j) consume(__shfl_sync(kFull, cur[c], j));
    }
#pragma unroll
    for (int c = 0; c < kBatch; ++c) cur[c] = nxt[c];
  }
}

__device__ __forceinline__ void warp_seq_sum(const double* v, int64_t len, double& sum,
                                             int64_t& cnt) {
  warp_stream(v, len, [&](double y) {
    const bool ok = !isnan(y);
    sum += ok ? y : 0.0;  // sum >= +0 and y >= 0: adding +0.0 is exact
    cnt += ok;
  });
}
__device__ __forceinline__ void warp_seq_sq(const double* v, int64_t len, double mean,
                                            double& acc) {
  warp_stream(v, len, [&](double y) {
    const double d = isnan(y) ? 0.0 : (y - mean) * (y - mean);
    acc += d;  // acc >= +0: adding +0.0 is exact
  });
}

__global__ void summary_cells_kernel(const SummaryParams p) {
  const int cell = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (cell >= p.n_mixes * p.n_rps) return;
  const int lane = threadIdx.x & 31;
  const int R = p.repeats;
  const int per_rps = p.n_caps * R + (p.with_saber ? R : 0);
  const int64_t base = static_cast<int64_t>(cell) * per_rps;
  double out[kCellScratch];
  const double nanv = nan("");
  out[0] = out[1] = out[2] = out[3] = nanv;
  out[4] = out[5] = 0.0;
  int best_cap = 0;
  if (p.n_caps > 0) {
    double best_mean = -1.0;
    long long prev = LLONG_MIN;
    for (;;) {  // unique caps in ascending order (std::map iteration)
      long long cap = LLONG_MAX;
      for (int w = 0; w < p.n_caps; ++w)
        if (p.caps[w] > prev && p.caps[w] < cap) cap = p.caps[w];
      if (cap == LLONG_MAX) break;
      prev = cap;
      double s = 0.0;
      int64_t c = 0;
      for (int w = 0; w < p.n_caps; ++w) {
        if (p.caps[w] != cap) continue;
        for (int i = 0; i < R; ++i) {
          s += p.rows[base + static_cast<int64_t>(w) * R + i].goodput;
          ++c;
        }
      }
      const double m = s / static_cast<double>(c);
      if (m > best_mean) {
        best_mean = m;
        best_cap = static_cast<int>(cap);
      }
    }
    out[1] = best_mean;
    double s = 0.0;
    int64_t c = 0;
    for (int w = 0; w < p.n_caps; ++w) {
      if (p.caps[w] != best_cap) continue;
      warp_seq_sum(p.ratios + (base + static_cast<int64_t>(w) * R) * p.n,
                   static_cast<int64_t>(R) * p.n, s, c);
    }
    if (c > 0) {
      out[3] = s / static_cast<double>(c);
      out[5] = 1.0;
    }
  }
  if (p.with_saber) {
    const int64_t sb = base + static_cast<int64_t>(p.n_caps) * R;
    double g = 0.0;
    for (int i = 0; i < R; ++i) g += p.rows[sb + i].goodput;
    out[0] = g / static_cast<double>(R);
    double s = 0.0;
    int64_t c = 0;
    warp_seq_sum(p.ratios + sb * p.n, static_cast<int64_t>(R) * p.n, s, c);
    if (c > 0) {
      out[2] = s / static_cast<double>(c);
      out[4] = 1.0;
    }
  }
  if (lane == 0) {
    p.best_cap[cell] = best_cap;
    for (int k = 0; k < kCellScratch; ++k) p.scratch[static_cast<int64_t>(cell) * kCellScratch + k] = out[k];
  }
}

// cv_or_nan (simloop.cpp:28-35) over scratch column `col` gated by `flag`.
__device__ double cv_cells(const double* sc, int n_rps, int col, int flag) {
  double mean = 0.0;
  int64_t n = 0;
  for (int ri = 0; ri < n_rps; ++ri)
    if (sc[ri * kCellScratch + flag] != 0.0) {
      mean += sc[ri * kCellScratch + col];
      ++n;
    }
  if (n == 0) return nan("");
  mean /= static_cast<double>(n);
  if (mean == 0.0) return nan("");
  double var = 0.0;
  for (int ri = 0; ri < n_rps; ++ri)
    if (sc[ri * kCellScratch + flag] != 0.0) {
      const double v = sc[ri * kCellScratch + col];
      var += (v - mean) * (v - mean);
    }
  var /= static_cast<double>(n);
  return sqrt(var) / mean;
}

// Pooled sequential sums for one (mix, variant): a 2-warp block.  Warp 1
// streams the pooled ratio blocks (rps in grid order, the chosen cell's rows,
// request ids in order) into a double-buffered shared ring; lane 0 of warp 0
// runs the reference's left-to-right add chain over it, so the chain (8-cycle
// DADD latency) never waits on memory.  Pass 1 sums, pass 2 sums squares of
// deviations from the pass-1 mean (cv(), metrics.cpp:49-59).
constexpr int kChunk = 1024;

// Walks the pooled sequence lazily: segment = the contiguous ratio block
// (R rows x n requests) of the chosen cell at each rps, in grid order.
struct SegmentWalk {
  int ri = 0, wi = -1;
  __device__ bool next(const SummaryParams& p, int mi, int variant, const double** ptr,
                       int64_t* len) {
    const int R = p.repeats;
    const int per_rps = p.n_caps * R + (p.with_saber ? R : 0);
    while (ri < p.n_rps) {
      const int64_t base = (static_cast<int64_t>(mi) * p.n_rps + ri) * per_rps;
      if (variant == 0) {
        if (wi < 0) {
          wi = 0;
          *ptr = p.ratios + (base + static_cast<int64_t>(p.n_caps) * R) * p.n;
          *len = static_cast<int64_t>(R) * p.n;
          return true;
        }
      } else {
        const int bc = p.best_cap[mi * p.n_rps + ri];
        for (++wi; wi < p.n_caps; ++wi)
          if (p.caps[wi] == bc) {
            *ptr = p.ratios + (base + static_cast<int64_t>(wi) * R) * p.n;
            *len = static_cast<int64_t>(R) * p.n;
            return true;
          }
      }
      ++ri;
      wi = -1;
    }
    return false;
  }
};

__device__ int64_t pool_length(const SummaryParams& p, int mi, int variant) {
  SegmentWalk w;
  const double* ptr;
  int64_t len, total = 0;
  while (w.next(p, mi, variant, &ptr, &len)) total += len;
  return total;
}

__global__ void __launch_bounds__(64) summary_mix_kernel(const SummaryParams p) {
  const int mi = blockIdx.x >> 1;
  const int variant = blockIdx.x & 1;  // 0 = saber, 1 = best static
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double ring[2][kChunk];
  __shared__ double s_out[3];
  __shared__ int64_t s_cnt;
  const double* sc = p.scratch + static_cast<int64_t>(mi) * p.n_rps * kCellScratch;
  const bool present = variant == 0 ? p.with_saber != 0 : p.n_caps > 0;
  const int64_t total = present ? pool_length(p, mi, variant) : 0;
  const int chunks = present ? static_cast<int>((total + kChunk - 1) / kChunk) : 0;
  double sum = 0.0, acc = 0.0, mean = 0.0;
  int64_t cnt = 0;  // completed ratios in the pool (counted by the loader warp)
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      if (warp == 1) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
        if (lane == 0) s_cnt = cnt;
      }
      __syncthreads();
      cnt = s_cnt;
      if (threadIdx.x == 0) s_out[0] = cnt > 0 ? sum / static_cast<double>(cnt) : 0.0;
      __syncthreads();
      mean = s_out[0];
      if (!(cnt > 0 && mean != 0.0)) break;
    }
    // Never-completed requests (NaN) are not in the reference's pool; the
    // loader replaces them by a value whose contribution is an exact +0:
    // 0.0 in the sum (sum >= +0) and the mean in the squared deviations.
    const double fill = pass == 0 ? 0.0 : mean;
    // loader state (warp 1): current segment and offset in it
    SegmentWalk walk;
    const double* sp = nullptr;
    int64_t slen = 0, off = 0;
    bool have = walk.next(p, mi, variant, &sp, &slen);
    for (int c = 0; c <= chunks; ++c) {
      if (warp == 1 && c < chunks) {
        double* dst = ring[c & 1];
        int filled = 0;
        while (filled < kChunk && have) {
          const int64_t avail = slen - off;
          const int take = static_cast<int>(avail < kChunk - filled ? avail : kChunk - filled);
          // eight independent loads in flight per lane before any store
          for (int i0 = 0; i0 < take; i0 += 8 * 32) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int i = i0 + u * 32 + lane;
              v[u] = i < take ? sp[off + i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int i = i0 + u * 32 + lane;
              if (i < take) {
                const bool ok = !isnan(v[u]);
                dst[filled + i] = ok ? v[u] : fill;
                if (pass == 0) cnt += ok;
              }
            }
          }
          filled += take;
          off += take;
          if (off == slen) {
            have = walk.next(p, mi, variant, &sp, &slen);
            off = 0;
          }
        }
        for (int i = filled + lane; i < kChunk; i += 32) dst[i] = fill;
      }
      if (warp == 0 && lane == 0 && c > 0) {
        // The dependent add chain, eight values per step with every shared
        // load of the step issued before its first add.
        const double2* src = reinterpret_cast<const double2*>(ring[(c - 1) & 1]);
        // software-pipelined: the next eight values are loaded while the
        // current eight run through the chain
        double2 a0 = src[0], a1 = src[1], a2 = src[2], a3 = src[3];
        if (pass == 0) {
#pragma unroll 1
          for (int i = 4; i <= kChunk / 2; i += 4) {
            const int k = i < kChunk / 2 ? i : 0;
            const double2 b0 = src[k], b1 = src[k + 1], b2 = src[k + 2], b3 = src[k + 3];
            sum += a0.x;
            sum += a0.y;
            sum += a1.x;
            sum += a1.y;
            sum += a2.x;
            sum += a2.y;
            sum += a3.x;
            sum += a3.y;
            a0 = b0;
            a1 = b1;
            a2 = b2;
            a3 = b3;
          }
        } else {
#pragma unroll 1
          for (int i = 4; i <= kChunk / 2; i += 4) {
            const int k = i < kChunk / 2 ? i : 0;
            const double2 b0 = src[k], b1 = src[k + 1], b2 = src[k + 2], b3 = src[k + 3];
            const double e0 = a0.x - mean, e1 = a0.y - mean, e2 = a1.x - mean, e3 = a1.y - mean;
            const double e4 = a2.x - mean, e5 = a2.y - mean, e6 = a3.x - mean, e7 = a3.y - mean;
            acc += e0 * e0;
            acc += e1 * e1;
            acc += e2 * e2;
            acc += e3 * e3;
            acc += e4 * e4;
            acc += e5 * e5;
            acc += e6 * e6;
            acc += e7 * e7;
            a0 = b0;
            a1 = b1;
            a2 = b2;
            a3 = b3;
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x != 0) return;
  const double nanv = nan("");
  double mean_goodput = nanv, pooled = nanv, rps_cv = nanv;
  if (present) {
    double s = 0.0;
    for (int ri = 0; ri < p.n_rps; ++ri) s += sc[ri * kCellScratch + (variant == 0 ? 0 : 1)];
    mean_goodput = s / static_cast<double>(p.n_rps);
    if (cnt > 0 && mean != 0.0) pooled = sqrt(acc / static_cast<double>(cnt)) / mean;
    rps_cv = cv_cells(sc, p.n_rps, variant == 0 ? 2 : 3, variant == 0 ? 4 : 5);
  }
  saber_mix_summary* out = p.summary + mi;
  if (variant == 0) {
    out->saber_mean_goodput = mean_goodput;
    out->saber_pooled_cv = pooled;
    out->saber_rps_mean_cv = rps_cv;
  } else {
    out->best_static_mean_goodput = mean_goodput;
    out->best_static_pooled_cv = pooled;
    out->best_static_rps_mean_cv = rps_cv;
  }
}

// The same pooled sums on ONE warp, no block barrier: every lane loads a
// strided slice of the next 256 pooled values into registers (two batches in
// flight), writes this batch's terms to a warp-private shared buffer, and the
// dependent add chain reads them back in pool order with broadcast 16-byte
// loads (half an LDS per value, in the shadow of the 8-cycle DADD chain;
// shuffles cost 11 cycles per value, profiles/latency_probe_b200.txt).
// Never-completed requests contribute an exact +0 (0 to the sum, a zero term
// to the deviations) and are counted with a ballot.  Every lane carries the
// same chain value.
constexpr int kStream = 8;  // values per lane per batch (a batch = 256 values)

__device__ __forceinline__ double pooled_chain(const SummaryParams& p, int mi, int variant,
                                               int pass, double mean, int64_t* cnt,
                                               double* buf /* [2][32 * kStream] shared */) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int64_t c = 0;
  SegmentWalk walk;
  const double* sp = nullptr;
  int64_t slen = 0;
  const double pad = nan("");  // beyond a segment: skipped like a never-completed request
  int parity = 0;
  while (walk.next(p, mi, variant, &sp, &slen)) {
    double cur[kStream], nxt[kStream];
#pragma unroll
    for (int u = 0; u < kStream; ++u) {
      const int64_t i = static_cast<int64_t>(u) * 32 + lane;
      cur[u] = i < slen ? sp[i] : pad;
    }
    for (int64_t base = 0; base < slen; base += 32 * kStream) {
      const int64_t nb = base + 32 * kStream;
#pragma unroll
      for (int u = 0; u < kStream; ++u) {  // next batch, issued before this one's chain
        const int64_t i = nb + static_cast<int64_t>(u) * 32 + lane;
        nxt[u] = i < slen ? sp[i] : pad;
      }
      // this batch's terms, in pool order, into the shared buffer
      double* bb = buf + parity * (32 * kStream);
#pragma unroll
      for (int u = 0; u < kStream; ++u) {
        const double v = cur[u];
        const bool ok = !isnan(v);
        double term;
        if (pass == 0) {
          term = ok ? v : 0.0;
          c += __popc(__ballot_sync(kFull, ok));
        } else {
          const double e = v - mean;
          term = ok ? e * e : 0.0;
        }
        bb[u * 32 + lane] = term;
      }
      __syncwarp();
      // the chain: every lane reads the same words (broadcast), two per load
      const double2* b2 = reinterpret_cast<const double2*>(bb);
#pragma unroll 8
      for (int k = 0; k < 16 * kStream; ++k) {
        const double2 x = b2[k];
        acc += x.x;
        acc += x.y;
      }
      parity ^= 1;  // the other half is written next; this one is read by then
#pragma unroll
      for (int u = 0; u < kStream; ++u) cur[u] = nxt[u];
    }
  }
  if (cnt) *cnt = c;
  return acc;
}

__global__ void __launch_bounds__(32) summary_mix_warp_kernel(const SummaryParams p) {
  __shared__ __align__(16) double buf[2 * 32 * kStream];
  const int mi = blockIdx.x >> 1;
  const int variant = blockIdx.x & 1;  // 0 = saber, 1 = best static
  const double* sc = p.scratch + static_cast<int64_t>(mi) * p.n_rps * kCellScratch;
  const bool present = variant == 0 ? p.with_saber != 0 : p.n_caps > 0;
  const double nanv = nan("");
  double mean_goodput = nanv, pooled = nanv, rps_cv = nanv;
  if (present) {
    int64_t cnt = 0;
    const double sum = pooled_chain(p, mi, variant, 0, 0.0, &cnt, buf);
    if (cnt > 0) {
      const double mean = sum / static_cast<double>(cnt);
      if (mean != 0.0) {
        __syncwarp();
        const double acc = pooled_chain(p, mi, variant, 1, mean, nullptr, buf);
        pooled = sqrt(acc / static_cast<double>(cnt)) / mean;
      }
    }
    double s = 0.0;
    for (int ri = 0; ri < p.n_rps; ++ri) s += sc[ri * kCellScratch + (variant == 0 ? 0 : 1)];
    mean_goodput = s / static_cast<double>(p.n_rps);
    rps_cv = cv_cells(sc, p.n_rps, variant == 0 ? 2 : 3, variant == 0 ? 4 : 5);
  }
  if (threadIdx.x != 0) return;
  saber_mix_summary* out = p.summary + mi;
  if (variant == 0) {
    out->saber_mean_goodput = mean_goodput;
    out->saber_pooled_cv = pooled;
    out->saber_rps_mean_cv = rps_cv;
  } else {
    out->best_static_mean_goodput = mean_goodput;
    out->best_static_pooled_cv = pooled;
    out->best_static_rps_mean_cv = rps_cv;
  }
}

// Exact parallel sum and count of one contiguous block of ratios (NaN =
// never completed: not in the pool, an exact +0 in the sum).
__device__ void block_ratio_sum(const double* v, int64_t len, double& sum, int64_t& cnt) {
  __shared__ unsigned long long c_sh;
  if (threadIdx.x == 0) c_sh = 0;
  __syncthreads();
  int64_t c = 0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) c += !isnan(v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&c_sh, static_cast<unsigned long long>(c));
  __syncthreads();
  cnt = static_cast<int64_t>(c_sh);
  sum = block_exact_seq_sum(
      len,
      [&](int64_t b, double (&t)[kExactK]) {
#pragma unroll
        for (int j = 0; j < kExactK; ++j) {
          const double x = b + j < len ? v[b + j] : 0.0;
          t[j] = isnan(x) ? 0.0 : x;
        }
      },
      [&](int64_t i) {
        const double x = v[i];
        return isnan(x) ? 0.0 : x;
      });
  __syncthreads();  // c_sh is reused by the next call
}

// S1 with the exact parallel sums: one block per (mix, rps) cell.
__global__ void __launch_bounds__(kExactThreads) summary_cells_exact_kernel(const SummaryParams p) {
  const int cell = blockIdx.x;
  const int R = p.repeats;
  const int per_rps = p.n_caps * R + (p.with_saber ? R : 0);
  const int64_t base = static_cast<int64_t>(cell) * per_rps;
  const int64_t len = static_cast<int64_t>(R) * p.n;
  __shared__ int best_cap_sh;
  __shared__ double best_mean_sh;
  double out[kCellScratch];
  const double nanv = nan("");
  out[0] = out[1] = out[2] = out[3] = nanv;
  out[4] = out[5] = 0.0;
  if (p.n_caps > 0) {
    if (threadIdx.x == 0) {  // unique caps ascending (std::map order), ties to the smaller
      double best_mean = -1.0;
      int best_cap = 0;
      long long prev = LLONG_MIN;
      for (;;) {
        long long cap = LLONG_MAX;
        for (int w = 0; w < p.n_caps; ++w)
          if (p.caps[w] > prev && p.caps[w] < cap) cap = p.caps[w];
        if (cap == LLONG_MAX) break;
        prev = cap;
        double sm = 0.0;
        int64_t c = 0;
        for (int w = 0; w < p.n_caps; ++w) {
          if (p.caps[w] != cap) continue;
          for (int i = 0; i < R; ++i) {
            sm += p.rows[base + static_cast<int64_t>(w) * R + i].goodput;
            ++c;
          }
        }
        const double m = sm / static_cast<double>(c);
        if (m > best_mean) {
          best_mean = m;
          best_cap = static_cast<int>(cap);
        }
      }
      best_cap_sh = best_cap;
      best_mean_sh = best_mean;
    }
    __syncthreads();
    const int best_cap = best_cap_sh;
    out[1] = best_mean_sh;
    int wb = 0;
    while (p.caps[wb] != best_cap) ++wb;  // caps are unique (validate_sweep)
    double sm;
    int64_t c;
    block_ratio_sum(p.ratios + (base + static_cast<int64_t>(wb) * R) * p.n, len, sm, c);
    if (c > 0) {
      out[3] = sm / static_cast<double>(c);
      out[5] = 1.0;
    }
    if (threadIdx.x == 0) p.best_cap[cell] = best_cap;
  } else if (threadIdx.x == 0) {
    p.best_cap[cell] = 0;
  }
  if (p.with_saber) {
    const int64_t sb = base + static_cast<int64_t>(p.n_caps) * R;
    double g = 0.0;
    for (int i = 0; i < R; ++i) g += p.rows[sb + i].goodput;
    out[0] = g / static_cast<double>(R);
    double sm;
    int64_t c;
    block_ratio_sum(p.ratios + sb * p.n, len, sm, c);
    if (c > 0) {
      out[2] = sm / static_cast<double>(c);
      out[4] = 1.0;
    }
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < kCellScratch; ++k) p.scratch[static_cast<int64_t>(cell) * kCellScratch + k] = out[k];
}

// Pooled CV terms of one (mix, variant) with the exact parallel sums: one block.
__global__ void __launch_bounds__(kExactThreads) summary_mix_exact_kernel(const SummaryParams p) {
  __shared__ const double* seg[kMaxSegments];
  const int mi = blockIdx.x >> 1;
  const int variant = blockIdx.x & 1;  // 0 = saber, 1 = best static
  const int lane = threadIdx.x & 31;
  const double* sc = p.scratch + static_cast<int64_t>(mi) * p.n_rps * kCellScratch;
  const bool present = variant == 0 ? p.with_saber != 0 : p.n_caps > 0;
  const double nanv = nan("");
  double mean_goodput = nanv, pooled = nanv, rps_cv = nanv;
  if (present) {
    // the pool: segments of R x n ratios (rps in grid order, the chosen cell)
    __shared__ int nseg_sh;
    if (threadIdx.x == 0) {
      int k = 0;
      SegmentWalk walk;
      const double* sp;
      int64_t slen;
      while (walk.next(p, mi, variant, &sp, &slen) && k < kMaxSegments) seg[k++] = sp;
      nseg_sh = k;
    }
    __syncthreads();
    const int nseg = nseg_sh;
    const int64_t L = static_cast<int64_t>(p.repeats) * p.n;
    const int64_t total = static_cast<int64_t>(nseg) * L;
    const double invL = 1.0 / static_cast<double>(L);
    // segment and offset of pooled index i without a 64-bit division
    auto locate = [&](int64_t i, int64_t& sg, int64_t& off) {
      sg = static_cast<int64_t>(static_cast<double>(i) * invL);
      off = i - sg * L;
      while (off < 0) { --sg; off += L; }
      while (off >= L) { ++sg; off -= L; }
    };
    auto at = [&](int64_t i) {
      int64_t sg, off;
      locate(i, sg, off);
      return seg[sg][off];
    };
    // K consecutive pooled values from b (NaN beyond the pool)
    auto load_run = [&](int64_t b, double (&t)[kExactK]) {
      int64_t sg, off;
      locate(b, sg, off);
#pragma unroll
      for (int j = 0; j < kExactK; ++j) {
        t[j] = b + j < total ? seg[sg][off] : nan("");
        if (++off == L) { ++sg; off = 0; }
      }
    };
    __shared__ unsigned long long cnt_sh;
    if (threadIdx.x == 0) cnt_sh = 0;
    __syncthreads();
    int64_t cnt = 0;
    for (int k = 0; k < nseg; ++k)
      for (int64_t o = threadIdx.x; o < L; o += kExactThreads) cnt += !isnan(seg[k][o]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
    if (lane == 0) atomicAdd(&cnt_sh, static_cast<unsigned long long>(cnt));
    __syncthreads();
    cnt = static_cast<int64_t>(cnt_sh);
    const double sum = block_exact_seq_sum(
        total,
        [&](int64_t b, double (&t)[kExactK]) {
          load_run(b, t);
#pragma unroll
          for (int j = 0; j < kExactK; ++j) t[j] = isnan(t[j]) ? 0.0 : t[j];
        },
        [&](int64_t i) {
          const double v = at(i);
          return isnan(v) ? 0.0 : v;
        });
    if (cnt > 0) {
      const double mean = sum / static_cast<double>(cnt);
      if (mean != 0.0) {
        const double acc = block_exact_seq_sum(
            total,
            [&](int64_t b, double (&t)[kExactK]) {
              load_run(b, t);
#pragma unroll
              for (int j = 0; j < kExactK; ++j)
                t[j] = isnan(t[j]) ? 0.0 : (t[j] - mean) * (t[j] - mean);
            },
            [&](int64_t i) {
              const double v = at(i);
              return isnan(v) ? 0.0 : (v - mean) * (v - mean);
            });
        pooled = sqrt(acc / static_cast<double>(cnt)) / mean;
      }
    }
    double s = 0.0;
    for (int ri = 0; ri < p.n_rps; ++ri) s += sc[ri * kCellScratch + (variant == 0 ? 0 : 1)];
    mean_goodput = s / static_cast<double>(p.n_rps);
    rps_cv = cv_cells(sc, p.n_rps, variant == 0 ? 2 : 3, variant == 0 ? 4 : 5);
  }
  if (threadIdx.x != 0) return;
  saber_mix_summary* out = p.summary + mi;
  if (variant == 0) {
    out->saber_mean_goodput = mean_goodput;
    out->saber_pooled_cv = pooled;
    out->saber_rps_mean_cv = rps_cv;
  } else {
    out->best_static_mean_goodput = mean_goodput;
    out->best_static_pooled_cv = pooled;
    out->best_static_rps_mean_cv = rps_cv;
  }
}

// ---------------------------------------------------------------------------
// The pooled sums over the whole GPU.  One block per (chain, 2,048-term
// chunk) speculates the chunk's binade from approximate prefix sums and
// reduces the chunk to its integer increment R (ties resolved for both
// parities of the starting integer); one block per chain then walks the
// chunks in order, adding R exactly when the true running sum is in the
// predicted binade and the chunk provably stays in it, and re-running the
// chunk with block_exact_seq_sum_range otherwise (binade crossings, a tie
// list over the cap, a mispredicted binade).  Same bits as the chain.
using exactsum::kTieCap;
constexpr int kPoolChunk = kExactThreads * kExactK;

struct ChunkSpec {
  double approx;        // any-order sum of the chunk's terms (speculation only)
  int64_t R;            // integer increment on the predicted grid, ties at q
  int64_t cnt;          // completed ratios in the chunk (pass 0)
  int32_t extra0, extra1;  // ties' rounding for an even / odd starting integer
  int32_t e, valid;     // predicted binade exponent; 0 = walk re-runs the chunk
};

struct PoolChain {
  const double* seg[kMaxSegments];
  int nseg;
  int64_t L, total;
  double invL;
};

__device__ __forceinline__ void pool_build(const SummaryParams& p, int chain, PoolChain& pc) {
  if (threadIdx.x == 0) {
    const int mi = chain >> 1, variant = chain & 1;
    const bool present = variant == 0 ? p.with_saber != 0 : p.n_caps > 0;
    int k = 0;
    if (present) {
      SegmentWalk walk;
      const double* sp;
      int64_t slen;
      while (walk.next(p, mi, variant, &sp, &slen) && k < kMaxSegments) pc.seg[k++] = sp;
    }
    pc.nseg = k;
    pc.L = static_cast<int64_t>(p.repeats) * p.n;
    pc.total = static_cast<int64_t>(k) * pc.L;
    pc.invL = 1.0 / static_cast<double>(pc.L);
  }
  __syncthreads();
}

// pooled value i (NaN = never completed), i < total
__device__ __forceinline__ double pool_at(const PoolChain& pc, int64_t i) {
  int64_t sg = static_cast<int64_t>(static_cast<double>(i) * pc.invL);  // no 64-bit division
  int64_t off = i - sg * pc.L;
  if (off < 0) {
    --sg;
    off += pc.L;
  } else if (off >= pc.L) {
    ++sg;
    off -= pc.L;
  }
  return pc.seg[sg][off];
}
// pass 0: the ratio; pass 1: its squared deviation from the mean; NaN -> +0
__device__ __forceinline__ double pool_term(double x, int pass, double mean) {
  if (isnan(x)) return 0.0;
  return pass == 0 ? x : (x - mean) * (x - mean);
}

__global__ void __launch_bounds__(kExactThreads) pool_approx_kernel(const SummaryParams p, int pass,
                                                                    const double* means,
                                                                    ChunkSpec* spec, int C) {
  __shared__ PoolChain pc;
  __shared__ double red[kExactThreads / 32];
  __shared__ unsigned long long cnt_sh;
  const int chain = blockIdx.x / C, chunk = blockIdx.x % C;
  pool_build(p, chain, pc);
  const double mean = pass == 1 ? means[2 * chain] : 0.0;
  const int64_t lo = static_cast<int64_t>(chunk) * kPoolChunk;
  const int64_t hi = lo + kPoolChunk < pc.total ? lo + kPoolChunk : pc.total;
  if (threadIdx.x == 0) cnt_sh = 0;
  double a = 0.0;
  int64_t c = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kExactThreads) {
    const double x = pool_at(pc, i);
    a += pool_term(x, pass, mean);
    c += !isnan(x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(kFull, a, o);
    c += __shfl_xor_sync(kFull, c, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = a;
    atomicAdd(&cnt_sh, static_cast<unsigned long long>(c));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kExactThreads / 32; ++w) t += red[w];
    ChunkSpec& sp = spec[blockIdx.x];
    sp.approx = t;
    sp.cnt = static_cast<int64_t>(cnt_sh);
  }
}

__global__ void __launch_bounds__(kExactThreads) pool_spec_kernel(const SummaryParams p, int pass,
                                                                  const double* means,
                                                                  ChunkSpec* spec, int C) {
  __shared__ PoolChain pc;
  __shared__ double red[kExactThreads / 32];
  __shared__ int64_t wtot[kExactThreads / 32];
  __shared__ int wtie[kExactThreads / 32];
  __shared__ int64_t tie_rel[kTieCap], tie_q[kTieCap];
  __shared__ double s_pred;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chain = blockIdx.x / C, chunk = blockIdx.x % C;
  pool_build(p, chain, pc);
  const double mean = pass == 1 ? means[2 * chain] : 0.0;
  const int64_t lo = static_cast<int64_t>(chunk) * kPoolChunk;
  // approximate running sum at the chunk start (any order: speculation only)
  double a = 0.0;
  for (int k = tid; k < chunk; k += kExactThreads) a += spec[static_cast<int64_t>(chain) * C + k].approx;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
  if (lane == 0) red[warp] = a;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kExactThreads / 32; ++w) t += red[w];
    s_pred = t;
  }
  __syncthreads();
  const double sp0 = s_pred;
  ChunkSpec& out = spec[blockIdx.x];
  if (!(sp0 > 0.0) || lo >= pc.total) {
    if (tid == 0) out.valid = 0;
    return;
  }
  const int e = ilogb(sp0);
  const double iu = ldexp(1.0, 52 - e);
  constexpr int64_t kTop = 1ll << 53;
  int64_t q[kExactK];
  int fc[kExactK];
  int64_t tot = 0;
  int nties = 0;
  const int64_t b = lo + static_cast<int64_t>(tid) * kExactK;
#pragma unroll
  for (int j = 0; j < kExactK; ++j) {
    const double t = b + j < pc.total ? pool_term(pool_at(pc, b + j), pass, mean) : 0.0;
    const double v = t * iu;
    const double fl = floor(v);
    const double fr = v - fl;
    q[j] = fl < 9.0e15 ? static_cast<int64_t>(fl) : kTop;
    fc[j] = fr > 0.5 ? 2 : (fr == 0.5 ? 1 : 0);
    tot += q[j] + (fc[j] == 2 ? 1 : 0);
    nties += fc[j] == 1;
  }
  int64_t inc = tot;
  int tinc = nties;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, inc, o);
    const int z = __shfl_up_sync(kFull, tinc, o);
    if (lane >= o) {
      inc += y;
      tinc += z;
    }
  }
  if (lane == 31) {
    wtot[warp] = inc;
    wtie[warp] = tinc;
  }
  __syncthreads();
  int64_t wbase = 0, all = 0;
  int tbase = 0, tall = 0;
#pragma unroll
  for (int w = 0; w < kExactThreads / 32; ++w) {
    if (w < warp) {
      wbase += wtot[w];
      tbase += wtie[w];
    }
    all += wtot[w];
    tall += wtie[w];
  }
  if (tall > kTieCap) {
    if (tid == 0) out.valid = 0;
    return;
  }
  if (tall > 0) {
    int k = tbase + tinc - nties;
    int64_t rel = wbase + inc - tot;  // increments before this thread's first term
#pragma unroll
    for (int j = 0; j < kExactK; ++j) {
      if (fc[j] == 1) {
        tie_rel[k] = rel;
        tie_q[k] = q[j];
        ++k;
      }
      rel += q[j] + (fc[j] == 2 ? 1 : 0);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int64_t x0 = 0, x1 = 0;  // starting integer even / odd
    for (int t = 0; t < tall; ++t) {
      x0 += (tie_rel[t] + x0 + tie_q[t]) & 1;
      x1 += (1 + tie_rel[t] + x1 + tie_q[t]) & 1;
    }
    out.R = all;
    out.extra0 = static_cast<int32_t>(x0);
    out.extra1 = static_cast<int32_t>(x1);
    out.e = e;
    out.valid = 1;
  }
}

// The in-order walk over one chain's chunks (one block); pass 0 leaves the
// mean and count in means[2 chain], pass 1 writes the mix summary.
__global__ void __launch_bounds__(kExactThreads) pool_walk_kernel(const SummaryParams p, int pass,
                                                                  double* means,
                                                                  const ChunkSpec* spec, int C) {
  __shared__ PoolChain pc;
  const int chain = blockIdx.x;
  const int mi = chain >> 1, variant = chain & 1;
  pool_build(p, chain, pc);
  const bool present = variant == 0 ? p.with_saber != 0 : p.n_caps > 0;
  double mean = pass == 1 ? means[2 * chain] : 0.0;
  const int64_t cnt_prev = pass == 1 ? static_cast<int64_t>(means[2 * chain + 1]) : 0;
  const bool run = present && (pass == 0 || (cnt_prev > 0 && mean != 0.0));
  double s = 0.0;
  int64_t cnt = 0;
  if (run) {
    constexpr int64_t kTop = 1ll << 53;
    for (int c = 0; c < C; ++c) {
      const int64_t lo = static_cast<int64_t>(c) * kPoolChunk;
      if (lo >= pc.total) break;
      const int64_t hi = lo + kPoolChunk < pc.total ? lo + kPoolChunk : pc.total;
      const ChunkSpec sp = spec[static_cast<int64_t>(chain) * C + c];
      cnt += sp.cnt;
      bool done = false;
      if (sp.valid && s > 0.0 && ilogb(s) == sp.e) {
        const double iu = ldexp(1.0, 52 - sp.e), u = ldexp(1.0, sp.e - 52);
        const int64_t S = static_cast<int64_t>(s * iu);
        const int64_t ex = (S & 1) ? sp.extra1 : sp.extra0;
        if (S + sp.R + ex < kTop - 1) {
          s = static_cast<double>(S + sp.R + ex) * u;
          done = true;
        }
      }
      if (!done) {
        s = exactsum::block_exact_seq_sum_range(
            s, lo, hi,
            [&](int64_t bb, double (&t)[kExactK]) {
#pragma unroll
              for (int j = 0; j < kExactK; ++j)
                t[j] = bb + j < hi ? pool_term(pool_at(pc, bb + j), pass, mean) : 0.0;
            },
            [&](int64_t i) { return pool_term(pool_at(pc, i), pass, mean); });
      }
    }
  }
  if (threadIdx.x != 0) return;
  if (pass == 0) {
    means[2 * chain] = cnt > 0 ? s / static_cast<double>(cnt) : 0.0;
    means[2 * chain + 1] = static_cast<double>(cnt);
    return;
  }
  const double* sc = p.scratch + static_cast<int64_t>(mi) * p.n_rps * kCellScratch;
  const double nanv = nan("");
  double mean_goodput = nanv, pooled = nanv, rps_cv = nanv;
  if (present) {
    if (cnt_prev > 0 && mean != 0.0) pooled = sqrt(s / static_cast<double>(cnt_prev)) / mean;
    double g = 0.0;
    for (int ri = 0; ri < p.n_rps; ++ri) g += sc[ri * kCellScratch + (variant == 0 ? 0 : 1)];
    mean_goodput = g / static_cast<double>(p.n_rps);
    rps_cv = cv_cells(sc, p.n_rps, variant == 0 ? 2 : 3, variant == 0 ? 4 : 5);
  }
  saber_mix_summary* o = p.summary + mi;
  if (variant == 0) {
    o->saber_mean_goodput = mean_goodput;
    o->saber_pooled_cv = pooled;
    o->saber_rps_mean_cv = rps_cv;
  } else {
    o->best_static_mean_goodput = mean_goodput;
    o->best_static_pooled_cv = pooled;
    o->best_static_rps_mean_cv = rps_cv;
  }
}

// delta = saber - best static (simloop.cpp:262), after both variants wrote.
__global__ void summary_delta_kernel(const SummaryParams p) {
  const int mi = blockIdx.x * blockDim.x + threadIdx.x;
  if (mi >= p.n_mixes) return;
  saber_mix_summary* out = p.summary + mi;
  out->delta = out->saber_mean_goodput - out->best_static_mean_goodput;
}

}  // namespace

size_t summary_pool_scratch_bytes(int n_mixes, int n_rps, int repeats, int n) {
  const int64_t total = static_cast<int64_t>(n_rps) * repeats * n;
  const int64_t C = (total + kPoolChunk - 1) / kPoolChunk;
  return static_cast<size_t>(2 * n_mixes) * static_cast<size_t>(C) * sizeof(ChunkSpec) +
         static_cast<size_t>(2 * n_mixes) * 2 * sizeof(double);
}

int launch_summary(const SummaryParams& p, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int cells = p.n_mixes * p.n_rps;
  if (cells == 0) return 0;
  // narrow: the summary of one sweep overlapping the next sweep's trajectory
  // kernels (bench.py pipelining) — small blocks that fit in the register
  // file those kernels leave free (the static kernel leaves 4,096 registers
  // per SM: one warp of the cells kernel or two of the ratios kernel fit)
  // Beside running trajectory kernels (narrow: bench.py's pipelined sweeps)
  // short pools keep the sequential single-warp chains, which fit in the
  // registers those kernels leave free and finish within the next sweep's
  // simulation (config 2: 128K terms, ~1.9 ms); long pools (config 3, the
  // N-GPU root) and stand-alone summaries use the exact parallel sums.
  const int64_t pool = static_cast<int64_t>(p.n_rps) * p.repeats * p.n;
  const bool chain = std::getenv("SABER_SUMMARY_CHAIN") != nullptr ||
                     (p.narrow && pool <= (int64_t{1} << 18) &&
                      std::getenv("SABER_SUMMARY_EXACT") == nullptr);
  if (p.narrow) {
    ratios_kernel<<<148, 64, 0, s>>>(p);
  } else {
    ratios_kernel<<<1184, 256, 0, s>>>(p);
  }
  if (chain && p.narrow)
    summary_cells_kernel<<<cells, 32, 0, s>>>(p);
  else if (chain)
    summary_cells_kernel<<<(cells * 32 + 127) / 128, 128, 0, s>>>(p);
  else
    summary_cells_exact_kernel<<<cells, kExactThreads, 0, s>>>(p);
  if (std::getenv("SABER_SUMMARY_RING"))
    summary_mix_kernel<<<2 * p.n_mixes, 64, 0, s>>>(p);
  else if (chain || p.n_rps > kMaxSegments)
    summary_mix_warp_kernel<<<2 * p.n_mixes, 32, 0, s>>>(p);
  else if (std::getenv("SABER_SUMMARY_BLOCK"))
    summary_mix_exact_kernel<<<2 * p.n_mixes, kExactThreads, 0, s>>>(p);
  else {
    // chunked: approx sums, speculation, walk — per pass (stream-ordered scratch)
    const int chains = 2 * p.n_mixes;
    const int64_t total = static_cast<int64_t>(p.n_rps) * p.repeats * p.n;
    const int C = static_cast<int>((total + kPoolChunk - 1) / kPoolChunk);
    if (!p.pool_scratch) return 1;
    ChunkSpec* spec = static_cast<ChunkSpec*>(p.pool_scratch);
    double* means = reinterpret_cast<double*>(spec + static_cast<size_t>(chains) * C);
    for (int pass = 0; pass < 2; ++pass) {
      pool_approx_kernel<<<chains * C, kExactThreads, 0, s>>>(p, pass, means, spec, C);
      pool_spec_kernel<<<chains * C, kExactThreads, 0, s>>>(p, pass, means, spec, C);
      pool_walk_kernel<<<chains, kExactThreads, 0, s>>>(p, pass, means, spec, C);
    }
  }
  summary_delta_kernel<<<1, 32, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
