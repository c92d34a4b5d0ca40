// mc.cu — device side of the bursty Monte-Carlo sweep (BASELINE config 5).
//
//   mc_horizon_kernel  : per trajectory, the default horizon of its trace
//                        (last arrival + 10 * max sla, simloop.cpp:60-63),
//                        max-reduced, to size the scheduler RNG streams
//   mc_workloads_kernel: per trajectory of a chunk, its bursty trace
//                        (bursty.h) into the workload tables + its TrajDesc
//   mc_reduce_kernel   : per trajectory, integer cell statistics and the
//                        latency/SLA histogram (atomic adds: exact, order-free)
// The trajectory engine itself is the sweep's (sim_kernel.cu) — the traces
// are just another workload source.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "bursty.h"
#include "saber_internal.h"

namespace saberb200 {
namespace {

constexpr double kInf = __builtin_huge_val();
__constant__ int kMcAvgIn[4] = {186, 463, 31, 670};  // types.cpp:10-18
__constant__ int kMcAvgOut[4] = {43, 387, 30, 617};
__constant__ double kMcSla[4] = {1.0, 8.0, 1.0, 12.0};

__device__ __forceinline__ int jitter_len(int avg, double jitter, double u) {
  const double lo = avg * (1.0 - jitter);
  const double hi = avg * (1.0 + jitter);
  const double v = lo + u * (hi - lo);
  const long long r = llround(v);
  return r < 1 ? 1 : static_cast<int>(r);
}

__device__ __forceinline__ int sample_task(const McParams& p, int mi, double u) {
  const double* th = p.mix_thresh + mi * 4;
  const int8_t* tt = p.mix_task + mi * 4;
  int task = p.mix_last[mi];
  for (int k = 0; k < 4; ++k)
    if (tt[k] >= 0 && u < th[k]) {
      task = tt[k];
      break;
    }
  return task;
}

__device__ __forceinline__ void cell_of(const McParams& p, int64_t k, int* mi, int* ri, int* v) {
  const int per_rps = p.n_caps + (p.with_saber ? 1 : 0);
  const int64_t cell = k % p.n_cells;
  *v = static_cast<int>(cell % per_rps);
  const int64_t mr = cell / per_rps;
  *ri = static_cast<int>(mr % p.n_rps);
  *mi = static_cast<int>(mr / p.n_rps);
}

__global__ void mc_horizon_kernel(const McParams p, int64_t count, unsigned long long* hmax) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int64_t k = p.shard_index + i * p.shard_count;
  int mi, ri, v;
  cell_of(p, k, &mi, &ri, &v);
  const double rps = p.rps[ri];
  bursty::Gen g;
  bursty::gen_init(g, p.bp, static_cast<uint64_t>(k));
  double last = 0.0, max_sla = 0.0;
  for (int q = 0; q < p.n; ++q) {
    last = bursty::gen_arrival(g, p.bp, rps);
    const int task = sample_task(p, mi, bursty::gen_uniform(g));
    g.draw += 2;  // input / output length draws
    const double sla = kMcSla[task];
    max_sla = (max_sla < sla) ? sla : max_sla;
  }
  const double h = last + 10.0 * max_sla;
  atomicMax(hmax, static_cast<unsigned long long>(__double_as_longlong(h)));  // h > 0
}

__global__ void mc_workloads_kernel(const McParams p) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= p.count) return;
  const int64_t k = p.shard_index + (p.k0 + i) * p.shard_count;
  int mi, ri, v;
  cell_of(p, k, &mi, &ri, &v);
  const double rps = p.rps[ri];
  const int64_t o = i * p.n;
  bursty::Gen g;
  bursty::gen_init(g, p.bp, static_cast<uint64_t>(k));
  double max_sla = 0.0, last = 0.0;
  const bool saber = p.with_saber && v == p.n_caps;
  for (int q = 0; q < p.n; ++q) {
    const double arrival = bursty::gen_arrival(g, p.bp, rps);
    const int task = sample_task(p, mi, bursty::gen_uniform(g));
    const int in = jitter_len(kMcAvgIn[task], p.jitter, bursty::gen_uniform(g));
    const int out = jitter_len(kMcAvgOut[task], p.jitter, bursty::gen_uniform(g));
    const double sla = kMcSla[task];
    const double dl = arrival + sla;
    p.arrival[o + q] = arrival;
    p.deadline[o + q] = dl;
    p.sla[o + q] = sla;
    p.max_out[o + q] = static_cast<double>(out);
    p.input[o + q] = static_cast<double>(in);
    p.prefill[o + q] = p.prefill_rate > 0.0 ? static_cast<double>(in) / p.prefill_rate : 0.0;
    p.task[o + q] = static_cast<int8_t>(task);
    double T = -kInf;  // demotion bound, as workloads_kernel (prologue.cu)
    if (saber && p.ceiling > 0.0) {
      const double qq = out / p.ceiling;
      if (isfinite(qq)) T = dl - qq * (1.0 + 1e-9) - 1e-9 * (fabs(dl) + 1.0);
    }
    p.demote_after[o + q] = T;
    max_sla = (max_sla < sla) ? sla : max_sla;
    last = arrival;
  }
  p.horizon[i] = last + 10.0 * max_sla;
  TrajDesc d;
  d.workload = static_cast<int32_t>(i);
  d.n = p.n;
  d.window = p.window;
  d.gt_tab = p.gt_tab;
  d.tick = p.tick;
  d.prefill_rate = p.prefill_rate;
  d.horizon = nan("");
  d.row = i;
  if (saber) {
    d.mode = SABER_MODE_SABER;
    d.cap = 0;
    d.model_tab = p.model_tab;
    d.stream = static_cast<int32_t>(k % p.sched_seeds);
  } else {
    d.mode = SABER_MODE_STATIC;
    d.cap = p.caps[v];
    d.model_tab = -1;
    d.stream = -1;
  }
  p.descs[i] = d;
}

// Ratio bin: 4 bins per octave starting at 2^-6, from the exponent and the
// top two mantissa bits (exact, no transcendental).
__device__ __forceinline__ int ratio_bin(double r) {
  if (!(r > 0.0)) return 0;
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(r));
  const int e = static_cast<int>((b >> 52) & 0x7FF) - 1023;
  const int q = static_cast<int>((b >> 50) & 3);
  const int bin = (e + 6) * 4 + q;
  return bin < 0 ? 0 : (bin >= SABER_MC_BINS ? SABER_MC_BINS - 1 : bin);
}

__global__ void mc_reduce_kernel(const McParams p, const saber_traj_row* rows, const double* comp,
                                 unsigned long long* stats, unsigned long long* hist) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= p.count) return;
  const int64_t k = p.shard_index + (p.k0 + i) * p.shard_count;
  const int64_t cell = k % p.n_cells;
  const saber_traj_row& R = rows[i];
  unsigned long long* s = stats + cell * SABER_MC_STATS;
  atomicAdd(s + 0, 1ULL);
  atomicAdd(s + 1, static_cast<unsigned long long>(R.n));
  atomicAdd(s + 2, static_cast<unsigned long long>(R.met));
  atomicAdd(s + 3, static_cast<unsigned long long>(R.completed));
  atomicAdd(s + 4, static_cast<unsigned long long>(R.decisions));
  atomicAdd(s + 5, static_cast<unsigned long long>(R.n_kind[0] + R.n_kind[1]));
  atomicAdd(s + 6, static_cast<unsigned long long>(R.decision_hash & 0xFFFFull));
  atomicAdd(s + 7, static_cast<unsigned long long>(R.ticks));
  if (hist) {
    unsigned long long* h = hist + cell * (SABER_MC_BINS + 1);
    const double* C = comp + i * p.n;
    for (int q = 0; q < p.n; ++q) {
      const double c = C[q];
      if (isnan(c)) {
        atomicAdd(h + SABER_MC_BINS, 1ULL);
      } else {
        const int64_t o = i * p.n + q;
        atomicAdd(h + ratio_bin((c - p.arrival[o]) / p.sla[o]), 1ULL);
      }
    }
  }
}

}  // namespace

int launch_mc_horizon(const McParams& p, int64_t count, unsigned long long* hmax, void* stream) {
  if (count == 0) return 0;
  mc_horizon_kernel<<<static_cast<unsigned>((count + 127) / 128), 128, 0,
                      static_cast<cudaStream_t>(stream)>>>(p, count, hmax);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_mc_workloads(const McParams& p, void* stream) {
  if (p.count == 0) return 0;
  mc_workloads_kernel<<<static_cast<unsigned>((p.count + 127) / 128), 128, 0,
                        static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_mc_reduce(const McParams& p, const saber_traj_row* rows, const double* comp,
                     int64_t* stats, int64_t* hist, void* stream) {
  if (p.count == 0) return 0;
  mc_reduce_kernel<<<static_cast<unsigned>((p.count + 127) / 128), 128, 0,
                     static_cast<cudaStream_t>(stream)>>>(
      p, rows, comp, reinterpret_cast<unsigned long long*>(stats),
      reinterpret_cast<unsigned long long*>(hist));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
