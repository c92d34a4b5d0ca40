// div_exactness.cu — checks the shared-reciprocal quotient used by the LM
// kernel (fit_kernel.cu div_by) against IEEE division on random operands:
//   y = __drcp_rn(d), q = x*y, r = fma(-d, q, x), q' = fma(r, y, q)  ==  x / d ?
// Operands: x, d with random mantissas (incl. all-ones / all-zeros / near-
// boundary patterns) and exponents spanning 2^-200..2^200.  Prints mismatches.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ double make(uint64_t r, int emin, int erange) {
  uint64_t m = r & 0xFFFFFFFFFFFFFull;
  const int kind = (r >> 52) & 7;
  if (kind == 0) m = 0xFFFFFFFFFFFFFull;          // all ones
  if (kind == 1) m = 0;                             // power of two
  if (kind == 2) m = (r >> 12) & 0xFull;            // near a power of two
  if (kind == 3) m = 0xFFFFFFFFFFFFFull - ((r >> 12) & 0xFull);
  const int e = emin + static_cast<int>((r >> 56) % erange);
  const uint64_t bits = (static_cast<uint64_t>(e + 1023) << 52) | m | ((r >> 63) << 63);
  return __longlong_as_double(static_cast<long long>(bits));
}
__global__ void k(uint64_t seed, int64_t n, unsigned long long* bad, double* ex) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = mix(seed ^ (2 * i)), b = mix(seed ^ (2 * i + 1));
    const double x = make(a, -100, 200), d = make(b, -100, 200);
    const double y = __drcp_rn(d);
    const double q = x * y;
    const double r = fma(-d, q, x);
    const double q2 = fma(r, y, q);
    const double want = x / d;
    if (__double_as_longlong(q2) != __double_as_longlong(want)) {
      const unsigned long long c = atomicAdd(bad, 1ull);
      if (c < 8) { ex[2 * c] = x; ex[2 * c + 1] = d; }
    }
  }
}
int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1ll << 32);
  unsigned long long* bad; double* ex;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&ex, 16 * 8);
  *bad = 0;
  for (int s = 0; s < 4; ++s) {
    k<<<148 * 16, 256>>>(0x1234567ull + s * 7919, n / 4, bad, ex);
    cudaDeviceSynchronize();
  }
  printf("checked %lld quotients, mismatches %llu\n", (long long)n, *bad);
  for (unsigned long long c = 0; c < *bad && c < 8; ++c) printf("  x=%.17g d=%.17g\n", ex[2 * c], ex[2 * c + 1]);
  return *bad ? 1 : 0;
}
