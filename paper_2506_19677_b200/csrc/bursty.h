// bursty.h — the bursty (MMPP) arrival generator of BASELINE config 5, shared
// verbatim by the device (workloads kernel) and the host twin
// (saber_cuda_mc_trace), so both produce bit-identical traces.
//
// The reference only has Poisson arrivals (workload.cpp:60); bursty traffic is
// named as a threat to validity in the paper and SURVEY §8(d)
// specifies this extension: a 2-state Markov-modulated Poisson process whose
// burst-state rate is `burst_factor` x rps, with exponential state holding
// times (mean `mean_calm` s in the calm state, `mean_burst` s in the burst
// state), drawn from Philox4x32-10 keyed by (seed, trajectory).
//
// Determinism across host and device: only IEEE-754 correctly rounded
// +, -, *, / and exact bit manipulation are used (det_log below), and both
// sides compile without FMA contraction (nvcc --fmad=false, g++
// -ffp-contract=off).  Task and length sampling reuse the reference's
// generate() rules (workload.cpp:21-39) on Philox uniforms.
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define SABER_HD __host__ __device__ __forceinline__
#else
#define SABER_HD inline
#endif

namespace saberb200 {
namespace bursty {

struct Params {
  uint64_t seed;        // Philox key
  double burst_factor;  // burst-state rate = burst_factor * rps
  double mean_calm;     // mean calm-state holding time (s)
  double mean_burst;    // mean burst-state holding time (s)
};

// Philox4x32-10 (Salmon et al., SC'11).
SABER_HD void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c[0];
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c[2];
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    const uint32_t n0 = hi1 ^ c[1] ^ k0;
    const uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Uniform in [0, 1) from draw `i` of trajectory `traj` (top 53 bits).
SABER_HD double uniform(uint64_t seed, uint64_t traj, uint64_t i) {
  uint32_t c[4] = {static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32),
                   static_cast<uint32_t>(traj), static_cast<uint32_t>(traj >> 32)};
  philox4x32_10(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const uint64_t x = (static_cast<uint64_t>(c[0]) << 32) | c[1];
  return static_cast<double>(x >> 11) * 0x1.0p-53;
}

SABER_HD uint64_t bits_of(double v) {
  uint64_t b;
  memcpy(&b, &v, 8);
  return b;
}
SABER_HD double from_bits(uint64_t b) {
  double v;
  memcpy(&v, &b, 8);
  return v;
}

// Natural log for x in (0, 1], from +,-,*,/ only: x = m * 2^e with
// m in [sqrt(1/2), sqrt(2)), log m = 2 atanh(s), s = (m-1)/(m+1), |s| < 0.172,
// summed as an odd series to s^23 (truncation < 1e-18 relative).
SABER_HD double det_log(double x) {
  uint64_t b = bits_of(x);
  int e = static_cast<int>((b >> 52) & 0x7FF) - 1023;
  if (((b >> 52) & 0x7FF) == 0) {  // subnormal: scale up exactly
    x = x * 0x1.0p54;
    b = bits_of(x);
    e = static_cast<int>((b >> 52) & 0x7FF) - 1023 - 54;
  }
  double m = from_bits((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);  // [1, 2)
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e = e + 1;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double z = s * s;
  double p = 1.0 / 23.0;
  p = p * z + 1.0 / 21.0;
  p = p * z + 1.0 / 19.0;
  p = p * z + 1.0 / 17.0;
  p = p * z + 1.0 / 15.0;
  p = p * z + 1.0 / 13.0;
  p = p * z + 1.0 / 11.0;
  p = p * z + 1.0 / 9.0;
  p = p * z + 1.0 / 7.0;
  p = p * z + 1.0 / 5.0;
  p = p * z + 1.0 / 3.0;
  p = p * z + 1.0;
  const double lnm = 2.0 * s * p;
  const double ln2_hi = 6.93147180369123816490e-01;  // fdlibm split of ln 2
  const double ln2_lo = 1.90821492927058770002e-10;
  const double de = static_cast<double>(e);
  return de * ln2_hi + (de * ln2_lo + lnm);
}

// Exponential variate with mean `mean` from uniform u in [0, 1).
SABER_HD double exp_variate(double u, double mean) { return -det_log(1.0 - u) * mean; }

// Request i's attributes, produced in arrival order by the generator state.
struct Gen {
  uint64_t seed, traj, draw;
  double t;          // last arrival time
  double switch_at;  // end of the current state
  int burst;         // 0 calm, 1 burst
};

SABER_HD void gen_init(Gen& g, const Params& p, uint64_t traj) {
  g.seed = p.seed;
  g.traj = traj;
  g.draw = 0;
  g.t = 0.0;
  g.burst = 0;
  g.switch_at = exp_variate(uniform(g.seed, g.traj, g.draw++), p.mean_calm);
}

// Next arrival time for rate `rps` (memoryless redraw at state switches),
// strictly increasing as generate() guarantees (workload.cpp:61-63).
SABER_HD double gen_arrival(Gen& g, const Params& p, double rps) {
  double t = g.t;
  for (;;) {
    const double rate = g.burst ? p.burst_factor * rps : rps;
    const double gap = exp_variate(uniform(g.seed, g.traj, g.draw++), 1.0) / rate;
    if (t + gap <= g.switch_at) {
      t = t + gap;
      break;
    }
    t = g.switch_at;
    g.burst = !g.burst;
    g.switch_at = t + exp_variate(uniform(g.seed, g.traj, g.draw++),
                                  g.burst ? p.mean_burst : p.mean_calm);
  }
  double arrival = t;
  if (!(arrival > g.t)) arrival = g.t + 1e-6;
  g.t = arrival;
  return arrival;
}

// Next uniform for task / length sampling.
SABER_HD double gen_uniform(Gen& g) { return uniform(g.seed, g.traj, g.draw++); }

}  // namespace bursty
}  // namespace saberb200
