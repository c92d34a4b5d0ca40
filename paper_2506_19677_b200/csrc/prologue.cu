// prologue.cu — device-side preparation kernels for the trajectory engine:
//   K0a workloads_kernel : generate() per (seed, rps, mix) from per-seed draws
//                          (workload.cpp:52-79) and the demotion bounds
//   K0b rng_stream_kernel: the scheduler's mt19937_64 stream per seed
//                          (scheduler.cpp:27,67), warp-parallel twist
//   K0c sweep_desc_kernel: sweep grid expansion (simloop.cpp:137-152)
//   fill_rows_kernel     : completion rows NaN (this shard) / 0 (others)
// All compiled with --fmad=false so every a*b+c rounds twice, as in the
// reference.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "saber_internal.h"

namespace saberb200 {
namespace {

constexpr double kInf = __builtin_huge_val();
__constant__ int kAvgIn[4] = {186, 463, 31, 670};   // types.cpp:10-18
__constant__ int kAvgOut[4] = {43, 387, 30, 617};
__constant__ double kSla[4] = {1.0, 8.0, 1.0, 12.0};

// jittered_length (workload.cpp:21-26) given its uniform draw u.
__device__ __forceinline__ int jittered(int avg, double jitter, double u) {
  const double lo = avg * (1.0 - jitter);
  const double hi = avg * (1.0 + jitter);
  const double v = lo + u * (hi - lo);
  const long long r = llround(v);
  return r < 1 ? 1 : static_cast<int>(r);
}

// Safe lower bound on the time a queued request (max_out m, deadline dl) can
// first satisfy required_speed > c.  Demotion needs
// fl(m / fl(dl - t)) > c, hence m / fl(dl - t) > c (c is representable),
// hence dl - t < (m / c) / (1 - 2^-53).  The 1e-9 margins dominate every
// rounding error in evaluating the bound itself.
__device__ __forceinline__ double demote_bound(double m, double dl, double c) {
  if (!(c > 0.0)) return -kInf;
  const double q = m / c;
  if (!isfinite(q)) return -kInf;
  return dl - q * (1.0 + 1e-9) - 1e-9 * (fabs(dl) + 1.0);
}

__global__ void __launch_bounds__(128) workloads_kernel(const WorkloadParams p) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= p.n_items) return;
  const WorkloadItem it = p.items[w];
  const int64_t o = static_cast<int64_t>(w) * p.nmax;
  double t = 0.0, max_sla = 0.0, last = 0.0;
  if (it.kind == 0) {
    const double* sb = p.seed_base + static_cast<int64_t>(it.seed_idx) * p.seed_stride * 4;
    const double* th = p.mix_thresh + it.mix * 4;
    const int8_t* tt = p.mix_task + it.mix * 4;
    const int last_task = p.mix_last[it.mix];
    for (int i = 0; i < it.n; ++i) {
      const double gap = sb[4 * i + 0] / it.rps;  // (-log(1-u)) / rps
      double arrival = t + gap;
      if (!(arrival > t)) arrival = t + 1e-6;  // strict increase
      t = arrival;
      const double u = sb[4 * i + 1];
      int task = last_task;  // sample_task (workload.cpp:28-39)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (tt[k] >= 0 && u < th[k]) {
          task = tt[k];
          break;
        }
      }
      const int in = jittered(kAvgIn[task], it.jitter, sb[4 * i + 2]);
      const int out = jittered(kAvgOut[task], it.jitter, sb[4 * i + 3]);
      const double sla = kSla[task];
      const double dl = arrival + sla;  // deadline_of (types.cpp:90-92)
      p.arrival[o + i] = arrival;
      p.deadline[o + i] = dl;
      p.sla[o + i] = sla;
      p.max_out[o + i] = static_cast<double>(out);
      p.input[o + i] = static_cast<double>(in);
      // Engine::admit's prefill debt (engine.cpp:33-35), hoisted out of the
      // trajectory kernel: every trajectory on this workload has this rate
      p.prefill[o + i] = it.prefill_rate > 0.0 ? static_cast<double>(in) / it.prefill_rate : 0.0;
      p.task[o + i] = static_cast<int8_t>(task);
      p.demote_after[o + i] = demote_bound(static_cast<double>(out), dl, it.ceiling);
      max_sla = (max_sla < sla) ? sla : max_sla;
      last = arrival;
    }
  } else {
    // Replayed requests are already in the tables; add the bounds.
    for (int i = 0; i < it.n; ++i) {
      const double sla = p.sla[o + i];
      p.demote_after[o + i] = demote_bound(p.max_out[o + i], p.deadline[o + i], it.ceiling);
      p.prefill[o + i] = it.prefill_rate > 0.0 ? p.input[o + i] / it.prefill_rate : 0.0;
      max_sla = (max_sla < sla) ? sla : max_sla;
      last = p.arrival[o + i];
    }
  }
  p.horizon[w] = last + 10.0 * max_sla;  // simloop.cpp:60-63
}

// mt19937_64 stream generator: one CTA per stream, state in shared memory.
// The twist runs in two parallel phases of 156 words (words 0..155 read only
// old state; words 156..311 read new[0..155] and old[156..311]).
__global__ void __launch_bounds__(160) rng_stream_kernel(const RngGenParams p) {
  const int s = blockIdx.x;
  if (s >= p.n_streams) return;
  __shared__ uint64_t st[312];
  const int tid = threadIdx.x;
  if (tid == 0) {
    uint64_t x = p.seeds[s];
    st[0] = x;
    for (int k = 1; k < 312; ++k) {
      x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(k);
      st[k] = x;
    }
  }
  __syncthreads();
  const int64_t len = p.len[s];
  uint32_t* out = p.draws + p.off[s];
  uint64_t* out64 = reinterpret_cast<uint64_t*>(p.draws) + p.off[s];  // wide plans
  constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
  constexpr uint64_t kMatrix = 0xB5026F5AA96619E9ULL;
  for (int64_t base = 0; base < len; base += 312) {
    uint64_t v = 0;
    if (tid < 156) {
      const uint64_t x = (st[tid] & kUpper) | (st[tid + 1] & kLower);
      v = st[tid + 156] ^ ((x >> 1) ^ ((x & 1ULL) ? kMatrix : 0ULL));
    }
    __syncthreads();
    if (tid < 156) st[tid] = v;
    __syncthreads();
    if (tid < 156) {
      const int k = tid + 156;
      const uint64_t x = (st[k] & kUpper) | (st[(k + 1) % 312] & kLower);
      v = st[k - 156] ^ ((x >> 1) ^ ((x & 1ULL) ? kMatrix : 0ULL));
    }
    __syncthreads();
    if (tid < 156) st[tid + 156] = v;
    __syncthreads();
    for (int k = tid; k < 312; k += blockDim.x) {
      if (base + k < len) {
        uint64_t y = st[k];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        if (p.wide) out64[base + k] = y;
        else out[base + k] = static_cast<uint32_t>(y % kDrawModulus);
      }
    }
    __syncthreads();
  }
}

// Sweep grid expansion for one shard (simloop.cpp:137-152): rows
// mix -> rps -> [caps..., saber] -> repeat; this shard takes r = shard + k*count.
__global__ void sweep_desc_kernel(const SweepDescParams p) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r = p.shard_index + k * p.shard_count;
  if (r >= p.n_rows) return;
  const int R = p.repeats;
  const int per_rps = p.n_caps * R + (p.with_saber ? R : 0);
  const int64_t cell = r / per_rps;
  const int rem = static_cast<int>(r % per_rps);
  const int mi = static_cast<int>(cell / p.n_rps);
  const int ri = static_cast<int>(cell % p.n_rps);
  TrajDesc d;
  d.n = p.n;
  d.window = p.window;
  d.gt_tab = p.gt_tab;
  d.tick = p.tick;
  d.prefill_rate = p.prefill_rate;
  d.horizon = p.has_horizon ? p.horizon : nan("");
  d.row = r;
  int rep;
  if (rem < p.n_caps * R) {
    d.mode = SABER_MODE_STATIC;
    d.cap = p.caps[rem / R];
    rep = rem % R;
    d.model_tab = -1;
    d.stream = -1;
  } else {
    d.mode = SABER_MODE_SABER;
    d.cap = 0;
    rep = rem - p.n_caps * R;
    d.model_tab = p.model_tab;
    d.stream = rep;
  }
  d.workload = (mi * p.n_rps + ri) * R + rep;
  p.out[k] = d;
}

__global__ void fill_rows_kernel(double* comp, int64_t n_rows, int32_t nmax, int32_t shard_index,
                                 int32_t shard_count) {
  const int64_t total = n_rows * nmax;
  const double nanv = nan("");
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / nmax;
    comp[i] = (r % shard_count == shard_index) ? nanv : 0.0;
  }
}

}  // namespace

int launch_workloads(const WorkloadParams& p, void* stream) {
  if (p.n_items == 0) return 0;
  const int block = 128;
  workloads_kernel<<<(p.n_items + block - 1) / block, block, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_rng_streams(const RngGenParams& p, void* stream) {
  if (p.n_streams == 0) return 0;
  rng_stream_kernel<<<p.n_streams, 160, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_sweep_descs(const SweepDescParams& p, void* stream, int64_t rows_this_shard) {
  if (rows_this_shard == 0) return 0;
  const int block = 128;
  const int64_t grid = (rows_this_shard + block - 1) / block;
  sweep_desc_kernel<<<static_cast<unsigned>(grid), block, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_fill_rows(double* comp, int64_t n_rows, int32_t nmax, int32_t shard_index,
                     int32_t shard_count, void* stream) {
  if (n_rows == 0) return 0;
  fill_rows_kernel<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(comp, n_rows, nmax,
                                                                       shard_index, shard_count);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
