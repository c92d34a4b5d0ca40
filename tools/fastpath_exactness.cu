// fastpath_exactness.cu — bit-for-bit checks of the branch-free fast paths
// the LM kernel uses (csrc/fast_math.cuh, fit_kernel.cu div_by):
//   exp_bounded(x) == exp(x)            for random x in [-700, 700]
//   div_fast(x, d) == x / d             whenever div_fast reports ok
//   Markstein q' (RN(1/d) reciprocal)   == x / d   (div_by's fast path)
//   div_unchecked(x, d, rcp_unchecked(d)) == x / d   for d in the exponent
//       window [2^-256, 2^256) (window_bits) and x = +0 or any x whose
//       quotient is normal in (2^-900, 2^900) — the LM passes' condition
// Operands: random mantissas incl. all-ones / power-of-two / near-boundary
// patterns, exponents over 2^-100..2^100 (the window case: d over 2^-260..
// 2^260, x over 2^-660..2^660).  Prints mismatches, exit 1 if any.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_2506_19677_b200/csrc/fast_math.cuh"

using namespace saberb200::fastmath;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ double make(uint64_t r, int emin, int erange) {
  uint64_t m = r & 0xFFFFFFFFFFFFFull;
  const int kind = (r >> 52) & 7;
  if (kind == 0) m = 0xFFFFFFFFFFFFFull;
  if (kind == 1) m = 0;
  if (kind == 2) m = (r >> 12) & 0xFull;
  if (kind == 3) m = 0xFFFFFFFFFFFFFull - ((r >> 12) & 0xFull);
  const int e = emin + static_cast<int>((r >> 56) % erange);
  const uint64_t bits = (static_cast<uint64_t>(e + 1023) << 52) | m | ((r >> 63) << 63);
  return __longlong_as_double(static_cast<long long>(bits));
}
// make() with the exponent drawn from a second word (any range width)
__device__ double make_w(uint64_t r, uint64_t re, int emin, int erange) {
  const double v = make(r, 0, 1);
  const int e = emin + static_cast<int>(re % static_cast<uint64_t>(erange));
  const uint64_t bits = (__double_as_longlong(v) & 0x800FFFFFFFFFFFFFull) |
                        (static_cast<uint64_t>(e + 1023) << 52);
  return __longlong_as_double(static_cast<long long>(bits));
}
__global__ void k(uint64_t seed, int64_t n, unsigned long long* bad, unsigned long long* used,
                  double* ex) {
  unsigned long long u = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = mix(seed ^ (3 * i)), b = mix(seed ^ (3 * i + 1)), c = mix(seed ^ (3 * i + 2));
    const double x = make(a, -100, 200), d = make(b, -100, 200);
    // exp on [-700, 700]
    const double xe = (static_cast<double>(c >> 11) * 0x1.0p-53 - 0.5) * 1400.0;
    if (__double_as_longlong(exp_bounded(xe)) != __double_as_longlong(exp(xe))) {
      const unsigned long long q = atomicAdd(bad, 1ull);
      if (q < 8) { ex[3 * q] = 0; ex[3 * q + 1] = xe; ex[3 * q + 2] = 0; }
    }
    // division fast path
    bool ok = true;
    const double q1 = div_fast(x, d, ok);
    if (ok) {
      ++u;
      if (__double_as_longlong(q1) != __double_as_longlong(x / d)) {
        const unsigned long long q = atomicAdd(bad, 1ull);
        if (q < 8) { ex[3 * q] = 1; ex[3 * q + 1] = x; ex[3 * q + 2] = d; }
      }
    }
    // the window-checked unchecked quotient (fit_kernel.cu Div)
    {
      const uint64_t a2 = mix(a ^ 0x5bd1e995ull), b2 = mix(b ^ 0x5bd1e995ull);
      const double dw = make_w(b2, mix(b2), -260, 520);
      const double xw = (mix(a2) & 63) == 0 ? 0.0 : make_w(a2, mix(a2) >> 6, -660, 1320);
      if (window_ok(window_bits(dw))) {
        const double q = xw / dw, aq = fabs(q);
        if (xw == 0.0 || (aq > 0x1.0p-900 && aq < 0x1.0p900)) {
          ++u;
          if (__double_as_longlong(div_unchecked(xw, dw, rcp_unchecked(dw))) != __double_as_longlong(q)) {
            const unsigned long long qq = atomicAdd(bad, 1ull);
            if (qq < 8) { ex[3 * qq] = 3; ex[3 * qq + 1] = xw; ex[3 * qq + 2] = dw; }
          }
        }
      }
    }
    // Markstein with a correctly rounded reciprocal (fit_kernel.cu div_by)
    const double y = __drcp_rn(d);
    const double qm = x * y;
    const double qm2 = fma(fma(-d, qm, x), y, qm);
    if (__double_as_longlong(qm2) != __double_as_longlong(x / d)) {
      const unsigned long long q = atomicAdd(bad, 1ull);
      if (q < 8) { ex[3 * q] = 2; ex[3 * q + 1] = x; ex[3 * q + 2] = d; }
    }
  }
  atomicAdd(used, u);
}
int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1ll << 32);
  unsigned long long *bad, *used;
  double* ex;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&used, 8);
  cudaMallocManaged(&ex, 24 * 8);
  *bad = 0;
  *used = 0;
  for (int s = 0; s < 4; ++s) {
    k<<<148 * 16, 256>>>(0x1234567ull + s * 7919, n / 4, bad, used, ex);
    cudaDeviceSynchronize();
  }
  printf("checked %lld samples (exp, Markstein quotient), %llu fast-path quotients; mismatches %llu\n",
         (long long)n, *used, *bad);
  for (unsigned long long c = 0; c < *bad && c < 8; ++c)
    printf("  kind %g x=%.17g d=%.17g\n", ex[3 * c], ex[3 * c + 1], ex[3 * c + 2]);
  return *bad ? 1 : 0;
}
