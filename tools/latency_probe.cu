// latency_probe.cu — dependent-chain latency of FP64/FP32/SHFL ops on the
// B200 (cycles per op via clock64), to size the ILP the kernels need.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x * 1e-9 + 1.0;
  float f = threadIdx.x * 1e-9f + 1.0f;
  unsigned u = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = x + a;
      if (OP == 1) x = x * b;
      if (OP == 2) x = fma(x, b, a);
      if (OP == 3) f = f + (float)a;
      if (OP == 4) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + a;
      if (OP == 5) x = x / b;
      if (OP == 6) x = (x < b) ? x + a : x - a;
      if (OP == 7) u = u * 2654435761u + 1u;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x + f + u;
}

// The summary's pooled chain (summary.cu pooled_chain): 32 values per step,
// broadcast by shuffles, added in sequence.  Reports cycles per added value.
__global__ void pooled(const double* v, double* out, long long* cyc, int n) {
  double acc = 0.0;
  long long t0 = clock64();
  for (int b = 0; b < n; ++b) {
    const double term = v[(b * 32 + threadIdx.x) & 4095];
    double w[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) w[k] = __shfl_sync(0xffffffffu, term, k);
#pragma unroll
    for (int k = 0; k < 32; ++k) acc += w[k];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = acc;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const char* names[] = {"DADD", "DMUL", "DFMA", "FADD", "SHFL+DADD", "DDIV", "DSETP+SEL+DADD", "IMAD"};
  const int n = 4096;
  for (int op = 0; op < 8; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
        case 1: chain<1><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
        case 2: chain<2><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
        case 3: chain<3><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
        case 4: chain<4><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
        case 5: chain<5><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
        case 6: chain<6><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
        case 7: chain<7><<<1, 32>>>(out, cyc, 1e-9, 0.999, n); break;
      }
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-16s %.2f cycles/op (1 warp, dependent chain)\n", names[op], (double)c / (n * 16));
  }
  {
    double* v;
    cudaMalloc(&v, 4096 * 8);
    cudaMemset(v, 0, 4096 * 8);
    for (int rep = 0; rep < 2; ++rep) {
      pooled<<<1, 32>>>(v, out, cyc, n);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-16s %.2f cycles/value (summary pooled chain)\n", "SHFLx32+DADDx32", (double)c / (n * 32));
  }
  return 0;
}
