// exact_sum.cuh — left-to-right double sums of non-negative terms computed
// in parallel with the sequential chain's exact bits (summary.cu; checked by
// tools/exact_sum_check.cu).
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cmath>
#include <cstdint>

namespace saberb200 {
namespace exactsum {

constexpr unsigned kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// Exact left-to-right sums in parallel.  The pooled sums are sequential by
// definition: s_0 = +0, s_k = RN(s_{k-1} + t_k), every t_k >= +0.  While s
// stays in one binade [2^e, 2^(e+1)) its grid is u = 2^(e-52), s = S u with
// an integer S, and t/u = q + f is exact (a power-of-two scaling), so
//     RN(S u + t) = (S + q + [f > 1/2]) u        unless f = 1/2 (a tie)
// whenever S + q + f < 2^53 - 1/2 (the result stays in the binade).  The
// increments r = q + [f > 1/2] do not depend on s, so a whole tile of terms
// is one integer prefix sum — computed by the block in parallel.  The first
// term of a tile that is a tie or leaves the binade (checked exactly against
// the integer prefix) is added with an ordinary DADD instead, which also
// moves s to its new binade, and the tile restarts after it.  Result: the
// same bits as the sequential chain (ties and binade changes are rare: a few
// dozen per million terms), at a few cycles per term instead of one 8-cycle
// dependent DADD each.
#ifndef SABER_EXACT_K
#define SABER_EXACT_K 4
#endif
#ifndef SABER_EXACT_T
#define SABER_EXACT_T 512
#endif
constexpr int kExactK = SABER_EXACT_K;  // terms per thread per tile
constexpr int kExactThreads = SABER_EXACT_T;
constexpr int kTieCap = 512;  // ties a tile resolves in place (more: term by term)  // a tile = 2,048 terms (4 x 512 measured best)

// `run(b, t)` fills t[0..kExactK) with the terms b, b+1, ... (t_i >= +0,
// +0 beyond n); `term(i)` returns one term.  Called by the whole block;
// every thread returns the sum.
// block_exact_seq_sum_range: the same from a running sum s0 over terms
// [lo, n) (s0 = +0, lo = 0: the whole chain).
template <class Run, class Term>
__device__ double block_exact_seq_sum_range(double s0, int64_t lo, int64_t n, Run&& run_terms,
                                            Term&& term) {
  __shared__ int64_t wtot[kExactThreads / 32];
  __shared__ int wtie[kExactThreads / 32];
  __shared__ int64_t tie_T[kTieCap], tie_q[kTieCap];
  __shared__ int64_t extra_sh;
  __shared__ int cand_min;
  __shared__ int64_t cand_S;
  __shared__ double s_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kExactThreads / 32;
  constexpr int kTile = kExactThreads * kExactK;
  constexpr int64_t kTop = 1ll << 53;
  double s = s0;
  int64_t pos = lo;
  if (!(s0 > 0.0)) {
    // bootstrap: the first terms sequentially (s is small next to them) on
    // warp 0, 32 coalesced loads at a time feeding the add chain by shuffles
    const int64_t boot = n - lo < 512 ? n : lo + 512;
    if (warp == 0) {
      for (int64_t b0 = lo; b0 < boot; b0 += 32) {
        const double t = b0 + lane < boot ? term(b0 + lane) : 0.0;
        for (int j = 0; j < 32; ++j) s += __shfl_sync(kFull, t, j);  // +0 past boot: exact
      }
      if (lane == 0) s_sh = s;
    }
    __syncthreads();
    s = s_sh;
    pos = boot;
  }
  while (pos < n) {
    if (!(s > 0.0)) {  // all terms so far were +0: one more sequential stretch
      __syncthreads();
      const int64_t end = pos + 512 < n ? pos + 512 : n;
      if (warp == 0) {
        for (int64_t b0 = pos; b0 < end; b0 += 32) {
          const double t = b0 + lane < end ? term(b0 + lane) : 0.0;
          for (int j = 0; j < 32; ++j) s += __shfl_sync(kFull, t, j);
        }
        if (lane == 0) s_sh = s;
      }
      __syncthreads();
      s = s_sh;
      pos = end;
      continue;
    }
    const int e = ilogb(s);
    const double iu = ldexp(1.0, 52 - e), u = ldexp(1.0, e - 52);
    const int64_t S = static_cast<int64_t>(s * iu);  // exact: 2^52 <= S < 2^53
    const int64_t b = pos + static_cast<int64_t>(tid) * kExactK;
    int64_t q[kExactK];
    int fc[kExactK];  // the fraction of t/u: 0 below 1/2, 1 exactly 1/2 (a tie), 2 above
    int64_t tot = 0;
    int nties = 0;
    {
      double tv[kExactK];
      run_terms(b, tv);
#pragma unroll
      for (int j = 0; j < kExactK; ++j) {
        const double v = tv[j] * iu;  // exact scaling
        const double fl = floor(v);
        const double fr = v - fl;
        q[j] = fl < 9.0e15 ? static_cast<int64_t>(fl) : kTop;  // >= 2^53 leaves the binade anyway
        fc[j] = fr > 0.5 ? 2 : (fr == 0.5 ? 1 : 0);
        tot += q[j] + (fc[j] == 2 ? 1 : 0);
        nties += fc[j] == 1;
      }
    }
    // block exclusive scans of the threads' increments and tie counts
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
    if (tid == 0) cand_min = INT_MAX;
    __syncthreads();
    int64_t wbase = 0, all = 0;
    int tbase = 0, tall = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const int64_t x = wtot[w];
      const int z = wtie[w];
      if (w < warp) {
        wbase += x;
        tbase += z;
      }
      all += x;
      tall += z;
    }
    const int64_t excl = wbase + inc - tot;
    // Ties resolved in order without leaving the tile: a tie at running
    // integer T (everything before it, earlier ties included) adds q or q + 1
    // so that T + result is even (round half to even); only the parity of
    // the earlier ties' choices matters, so thread 0 walks the tie list.
    // Valid when the whole tile provably stays in the binade: every partial
    // sum is at most S + all + (number of ties) + 1/2.
    if (S + all + tall < kTop - 1 && tall <= kTieCap) {
      if (tall > 0) {
        int k = tbase + tinc - nties;
        int64_t run = S + excl;
#pragma unroll
        for (int j = 0; j < kExactK; ++j) {
          if (fc[j] == 1) {
            tie_T[k] = run;
            tie_q[k] = q[j];
            ++k;
          }
          run += q[j] + (fc[j] == 2 ? 1 : 0);
        }
        __syncthreads();
        if (tid == 0) {
          int64_t extra = 0;
          for (int t = 0; t < tall; ++t) extra += (tie_T[t] + extra + tie_q[t]) & 1;
          extra_sh = extra;
        }
        __syncthreads();
        all += extra_sh;
      }
      s = static_cast<double>(S + all) * u;  // exact: < 2^53 on the grid
      pos = pos + kTile < n ? pos + kTile : n;
      __syncthreads();  // wtot / wtie / tie lists are rewritten next tile
      continue;
    }
    // this thread's first term that is a tie or leaves the binade
    int cj = kExactK;
    int64_t run = S + excl;
#pragma unroll
    for (int j = 0; j < kExactK; ++j) {
      const int64_t I = run + q[j];
      const bool cand = fc[j] == 1 || I >= kTop || (I == kTop - 1 && fc[j] >= 1);
      if (cand && cj == kExactK && b + j < n) cj = j;
      if (cj == kExactK) run = I + (fc[j] == 2 ? 1 : 0);
    }
    if (cj < kExactK) atomicMin(&cand_min, tid * kExactK + cj);
    __syncthreads();
    const int c = cand_min;
    if (c == INT_MAX) {
      s = static_cast<double>(S + all) * u;  // exact: < 2^53 on the grid
      pos = pos + kTile < n ? pos + kTile : n;
      __syncthreads();  // wtot / cand_min are rewritten next tile
      continue;
    }
#ifdef SABER_EXACT_DEBUG
    if (tid == 0) {
      const double tcd = term(pos + c);
      const double vv = tcd * iu;
      printf("cand pos %lld c %d e %d t %.17g v %.17g frac %.17g\n", (long long)pos, c, e, tcd, vv, vv - floor(vv));
    }
#endif
    if (tid * kExactK + cj == c) cand_S = run;  // S before the candidate term
    __syncthreads();
    if (tid == 0) s_sh = static_cast<double>(cand_S) * u + term(pos + c);  // one DADD
    __syncthreads();
    s = s_sh;
    pos += c + 1;
  }
  return s;
}

template <class Run, class Term>
__device__ double block_exact_seq_sum(int64_t n, Run&& run_terms, Term&& term) {
  return block_exact_seq_sum_range(0.0, 0, n, run_terms, term);
}

}  // namespace exactsum
}  // namespace saberb200
