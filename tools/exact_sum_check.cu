// exact_sum_check.cu — the parallel left-to-right summation of the sweep
// summary (csrc/exact_sum.cuh) against the sequential DADD chain, bit for bit,
// on random non-negative sequences built to hit its hard cases: exact zeros,
// ties (terms with few significant bits, so t/u often ends in exactly 1/2),
// binade crossings (terms as large as the running sum, powers of two), long
// runs of tiny terms next to a huge sum, and the ratio-like mixture the
// summary sees.  One block per case; prints mismatches, exit 1 if any.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_2506_19677_b200/csrc/exact_sum.cuh"

using namespace saberb200::exactsum;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ double gen(uint64_t seed, int64_t i, int kind) {
  const uint64_t r = mix(seed ^ (static_cast<uint64_t>(i) * 0x9E3779B97F4A7C15ULL));
  const double u = static_cast<double>(r >> 11) * 0x1.0p-53;
  switch (kind) {
    case 0: return (r & 7) == 0 ? 0.0 : u * 10.0;                           // ratios with zeros
    case 1: return ldexp(static_cast<double>((r >> 8) & 7), -static_cast<int>(r & 63));  // few bits: ties
    case 2: return ldexp(1.0, static_cast<int>(r % 40) - 20);               // powers of two
    case 3: return i < 4 ? 1e12 : u * 1e-6;                                 // tiny terms, huge sum
    case 4: return (r & 1) ? ldexp(static_cast<double>(r >> 40), -20) : u;  // mixed grids
    default: return u * u * 100.0;                                          // squared deviations
  }
}
__global__ void __launch_bounds__(kExactThreads) k(uint64_t seed0, int64_t nmax, double* buf,
                                                    unsigned long long* bad, double* ex) {
  const uint64_t seed = mix(seed0 + blockIdx.x);
  const int kind = static_cast<int>(mix(seed) % 6);
  const int64_t n = 1 + static_cast<int64_t>(mix(seed + 1) % nmax);
  double* v = buf + static_cast<int64_t>(blockIdx.x) * nmax;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] = gen(seed, i, kind);
  __syncthreads();
  const double got = block_exact_seq_sum(
      n,
      [&](int64_t b, double (&t)[kExactK]) {
#pragma unroll
        for (int j = 0; j < kExactK; ++j) t[j] = b + j < n ? v[b + j] : 0.0;
      },
      [&](int64_t i) { return v[i]; });
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i];
    if (__double_as_longlong(s) != __double_as_longlong(got)) {
      const unsigned long long c = atomicAdd(bad, 1ull);
      if (c < 8) { ex[3 * c] = kind; ex[3 * c + 1] = s; ex[3 * c + 2] = got; }
    }
  }
}
int main(int argc, char** argv) {
  const int cases = argc > 1 ? atoi(argv[1]) : 4096;
  const int64_t nmax = argc > 2 ? atoll(argv[2]) : 100000;
  const int per = 512;
  double* buf;
  unsigned long long* bad;
  double* ex;
  cudaMalloc(&buf, sizeof(double) * nmax * per);
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&ex, 24 * 8);
  *bad = 0;
  for (int c0 = 0; c0 < cases; c0 += per) {
    k<<<per, kExactThreads>>>(0xC0FFEEull + c0, nmax, buf, bad, ex);
    cudaDeviceSynchronize();
  }
  const cudaError_t e = cudaGetLastError();
  printf("%d sequences (n <= %lld), mismatches %llu%s\n", cases, (long long)nmax, *bad,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  for (unsigned long long c = 0; c < *bad && c < 8; ++c)
    printf("  kind %g sequential %.17g parallel %.17g\n", ex[3 * c], ex[3 * c + 1], ex[3 * c + 2]);
  return (*bad || e != cudaSuccess) ? 1 : 0;
}
