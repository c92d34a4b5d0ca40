// sim_kernel.cu — host side of the trajectory engine (launch planning,
// kernel selection over the instantiation units) plus the per-row metrics
// epilogue (K2) and the tick-index kernel.  The engine itself (K1) is in
// sim_kernel.cuh.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "saber_internal.h"
#include "sim_common.cuh"
#include "sim_kernel.cuh"

namespace saberb200 {

// Defined by sim_inst_nw{1,2,4,8}.cu: the mask-width-NW instantiations.
void* pick_sim_nw1(int g, bool trace, bool records, int sel);
void* pick_sim_nw2(int g, bool trace, bool records, int sel);
void* pick_sim_nw4(int g, bool trace, bool records, int sel);
void* pick_sim_nw8(int g, bool trace, bool records, int sel);
void* pick_sim_wide(bool trace, bool records);  // sim_inst_wide.cu

namespace {

__global__ void tick_index_kernel(const WorkloadTables wl, int64_t cells, const TickTable tt,
                                  int32_t* ka, int32_t* kd) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cells;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    ka[i] = tick_index(tt, wl.arrival[i]);
    kd[i] = tick_index(tt, wl.demote_after[i]);
  }
}

// K2: per-row metrics (make_record + compute_metrics, metrics.cpp:17-140),
// one warp per row: the per-request tests and counts are lane-parallel
// (ballots), and the two sequential sums of compute_metrics run as one
// dependent chain fed by shuffles, in request-id order; requests that never
// completed contribute an exact +0 (sums of non-negative terms).  Then the
// latency percentiles off the reference's cdf (metrics.cpp:61-85) as exact
// order statistics (rank counting over the row's latencies in shared memory).
constexpr int kQuantiles = 3;
__device__ const double kQuantileP[kQuantiles] = {0.5, 0.9, 0.99};

__device__ __forceinline__ void row_metrics_one(const RowMetricsParams& p, const TrajDesc d,
                                                int lane, double* lat) {
  const int nmax = p.wl.nmax;
  const int64_t wo = static_cast<int64_t>(d.workload) * nmax;
  const double* C = p.completion + d.row * nmax;
  const double* ARR = p.wl.arrival + wo;
  const double* SLA = p.wl.sla + wo;
  const int8_t* TASK = p.wl.task + wo;
  int64_t met = 0, comp = 0;
  int64_t issued[4] = {0, 0, 0, 0}, metk[4] = {0, 0, 0, 0};
  double sum = 0.0;
  for (int base = 0; base < d.n; base += kWarp) {
    const int q = base + lane;
    const bool valid = q < d.n;
    const double c = valid ? C[q] : nan("");
    const bool has = valid && !isnan(c);
    const double a = has ? ARR[q] : 0.0, sl = has ? SLA[q] : 1.0;
    const bool m = has && c - a <= sl;
    const int tk = valid ? TASK[q] : -1;
    met += __popc(__ballot_sync(0xFFFFFFFFu, m));
    comp += __popc(__ballot_sync(0xFFFFFFFFu, has));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      issued[k] += __popc(__ballot_sync(0xFFFFFFFFu, tk == k));
      metk[k] += __popc(__ballot_sync(0xFFFFFFFFu, m && tk == k));
    }
    const double v = has ? (c - a) / sl : 0.0;
#pragma unroll
    for (int k = 0; k < kWarp; ++k) sum += __shfl_sync(0xFFFFFFFFu, v, k);
  }
  saber_traj_row* R = p.rows + d.row;
  // latency percentiles: the k-th smallest latency, k = min{i : (i+1)/n >= p}
  {
    __syncwarp();  // the previous row's reads of lat are done
    for (int q = lane; q < d.n; q += kWarp) {
      const double c = C[q];
      lat[q] = isnan(c) ? kInf : c - ARR[q];
    }
    __syncwarp();
    int kq[kQuantiles];
#pragma unroll
    for (int t = 0; t < kQuantiles; ++t) {
      const double pq = kQuantileP[t];
      int k = static_cast<int>(pq * d.n) - 2;
      if (k < 0) k = 0;
      while (static_cast<double>(k + 1) / static_cast<double>(d.n) < pq) ++k;
      kq[t] = k;
    }
    unsigned hit[kQuantiles] = {0u, 0u, 0u};
    double val[kQuantiles] = {0.0, 0.0, 0.0};
    // four of this lane's latencies ranked per pass over the row (one shared
    // load serves four comparisons)
    constexpr int kR = 4;
    for (int q0 = lane; q0 < d.n; q0 += kR * kWarp) {
      double x[kR];
      int less[kR], le[kR];
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const int q = q0 + u * kWarp;
        x[u] = q < d.n ? lat[q] : kInf;
        less[u] = le[u] = 0;
      }
      for (int r = 0; r < d.n; ++r) {
        const double y = lat[r];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          less[u] += y < x[u];
          le[u] += y <= x[u];
        }
      }
#pragma unroll
      for (int u = 0; u < kR; ++u)
#pragma unroll
        for (int t = 0; t < kQuantiles; ++t)
          if (x[u] < kInf && less[u] <= kq[t] && kq[t] < le[u]) {
            hit[t] = 1u;
            val[t] = x[u];
          }
    }
#pragma unroll
    for (int t = 0; t < kQuantiles; ++t) {
      const unsigned who = __ballot_sync(0xFFFFFFFFu, hit[t] != 0u);
      if (who == 0u) {
        if (lane == 0) R->latency_q[t] = nan("");
      } else if (lane == __ffs(who) - 1) {
        R->latency_q[t] = val[t];
      }
    }
  }
  if (lane == 0) {
    R->goodput = static_cast<double>(met) / static_cast<double>(d.n);
    R->completed = comp;
    R->met = met;
    for (int k = 0; k < 4; ++k) {
      R->issued_by_task[k] = issued[k];
      R->met_by_task[k] = metk[k];
    }
  }
  if (comp == 0) {
    if (lane == 0) R->ratio_mean = R->ratio_std = R->cv = nan("");
    return;
  }
  const double mean = sum / static_cast<double>(comp);
  double var = 0.0;
  for (int base = 0; base < d.n; base += kWarp) {
    const int q = base + lane;
    const double c = q < d.n ? C[q] : nan("");
    double t = 0.0;
    if (!isnan(c)) {
      const double v = (c - ARR[q]) / SLA[q];
      t = (v - mean) * (v - mean);
    }
#pragma unroll
    for (int k = 0; k < kWarp; ++k) var += __shfl_sync(0xFFFFFFFFu, t, k);
  }
  if (lane == 0) {
    var /= static_cast<double>(comp);
    R->ratio_mean = mean;
    R->ratio_std = sqrt(var);
    R->cv = mean == 0.0 ? nan("") : R->ratio_std / mean;
  }
}

// Rows longer than kMaxRequests: the same epilogue with each warp's
// latencies in a global-memory slice (L1/L2-resident) instead of shared memory.
__global__ void __launch_bounds__(128) row_metrics_wide_kernel(const RowMetricsParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double* lat = p.lat_scratch + gw * p.wl.nmax;
  for (int64_t i = gw; i < p.n_traj; i += warps) row_metrics_one(p, p.traj[i], lane, lat);
}

__global__ void __launch_bounds__(128) row_metrics_warp_kernel(const RowMetricsParams p) {
  __shared__ double lat_all[128 / kWarp][kMaxRequests];
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < p.n_traj;
       i += warps) {  // uniform per warp
    row_metrics_one(p, p.traj[i], lane, lat_all[threadIdx.x >> 5]);
  }
}

void* pick_kernel(int nw, int g, bool trace, bool records, int sel = kSelAny) {
  switch (nw) {
    case 1: return pick_sim_nw1(g, trace, records, sel);
    case 2: return pick_sim_nw2(g, trace, records, sel);
    case 4: return pick_sim_nw4(g, trace, records, sel);
    case 8: return pick_sim_nw8(g, trace, records, sel);
  }
  return nullptr;
}

}  // namespace

int plan_sim(int nmax, int group, bool wide, SimLaunch* out) {
  SimLaunch l{};
  if (wide) {  // whole warps, everything in global scratch
    l.wide = 1;
    l.group = kWarp;
    l.slot_rows = (nmax + kWarp - 1) / kWarp;
    l.smem = 0;
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pick_sim_wide(false, false),
                                                      kSimBlock, 0) != cudaSuccess)
      return 1;
    if (per_sm < 1) return 3;
    l.grid = sms * per_sm;
    for (int v = 0; v < 3; ++v) l.grid_sel[v] = l.grid;
    l.block = kSimBlock;
    *out = l;
    return 0;
  }
  l.nwords = nmax <= 64 ? 1 : nmax <= 128 ? 2 : nmax <= 256 ? 4 : 8;
  // Widen the group until two blocks' slot tiles fit in shared memory.
  constexpr size_t kTileBudget = 100 * 1024;
  for (;;) {
    l.group = group;
    l.slot_rows = (nmax + group - 1) / group;
    l.smem = static_cast<size_t>(kSimBlock / kWarp) * l.slot_rows * kWarp * 16;
    if (l.smem <= kTileBudget || group >= 32) break;
    group *= 2;
  }
  // + per-warp staging for scheduler draws (gate streaks)
  l.smem += static_cast<size_t>(kSimBlock / kWarp) * kWarp * (kMaxWindow - 1) * 4;
  void* k = pick_kernel(l.nwords, group, false, false);
  if (!k) return 1;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
  for (int tr = 0; tr < 2; ++tr)
    for (int rec = 0; rec < 2; ++rec)
      for (int sel = 0; sel < 3; ++sel) {
        void* kk = pick_kernel(l.nwords, group, tr != 0, rec != 0, sel);
        if (cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(l.smem)) != cudaSuccess)
          return 2;
      }
  for (int sel = 0; sel < 3; ++sel) {
    void* kk = pick_kernel(l.nwords, group, false, false, sel);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kk, kSimBlock, l.smem) != cudaSuccess)
      return 1;
    if (per_sm < 1) return 3;
    l.grid_sel[sel] = sms * per_sm;
  }
  // The SABER kernel fills the register file of every SM (4 x 128 threads x
  // 128 registers); leave 8 SMs one block short so a concurrent sweep summary
  // (single-warp blocks on a side stream) finds room (bench.py pipelining).
  if (l.grid_sel[kSelSaber] > 16 * kSimBlock / kWarp) l.grid_sel[kSelSaber] -= 8;
  // Beside the static kernel (split sweep launches) the SABER kernel keeps
  // two warps per SM fewer: the static blocks start sooner (config 2 9.76 ->
  // 9.70 ms per sweep, r02i box; 1 warp fewer: 9.75, 4 fewer: 9.81; the
  // Monte-Carlo driver's split launches keep the full grid: 2% slower there).
  int trim = 2 * sms;
  if (const char* e = std::getenv("SABER_SPLIT_SABER_TRIM")) trim = std::atoi(e);
  l.grid_saber_split = l.grid_sel[kSelSaber] > trim + sms ? l.grid_sel[kSelSaber] - trim
                                                          : l.grid_sel[kSelSaber];
  l.grid = l.grid_sel[0];
  l.block = kSimBlock;
  *out = l;
  return 0;
}

int launch_sim(const SimParams& p, const SimLaunch& l, void* stream) {
  const bool trace = p.out.trace != nullptr;
  const bool records = p.out.admit != nullptr || p.out.demoted != nullptr;
  const int sel = p.mode_sel;
  void* k = l.wide ? pick_sim_wide(trace, records) : pick_kernel(l.nwords, l.group, trace, records, sel);
  if (!k) return 1;
  int grid = (!l.wide && l.group == kWarp && !trace && !records) ? l.grid_sel[sel] : l.grid;
  if (p.split_saber && sel == kSelSaber && l.grid_saber_split > 0) grid = l.grid_saber_split;
  SimParams q = p;
  q.no_streak = std::getenv("SABER_NO_STREAK") != nullptr;
  void* args[] = {&q};
  return cudaLaunchKernel(k, dim3(grid), dim3(kSimBlock), args, l.smem,
                          static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? 0
             : 1;
}

int launch_tick_index(const WorkloadTables& wl, int64_t cells, const TickTable& tt, int32_t* ka,
                      int32_t* kd, void* stream) {
  if (cells == 0 || tt.len == 0) return 0;
  const int block = 256;
  const int64_t want = (cells + block - 1) / block;
  const int grid = static_cast<int>(want < 4096 ? want : 4096);
  tick_index_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(wl, cells, tt, ka, kd);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_row_metrics(const RowMetricsParams& p, void* stream) {
  if (p.n_traj == 0) return 0;
  const int block = 128;
  if (p.wl.nmax > kMaxRequests) {
    // stream-ordered scratch: one latency slice per warp of a fixed grid
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    RowMetricsParams q = p;
    void* lat = nullptr;
    const size_t bytes = static_cast<size_t>(kRowMetricsWideWarps) * p.wl.nmax * sizeof(double);
    if (cudaMallocAsync(&lat, bytes, st) != cudaSuccess) return 1;
    q.lat_scratch = static_cast<double*>(lat);
    row_metrics_wide_kernel<<<kRowMetricsWideWarps * kWarp / block, block, 0, st>>>(q);
    const bool ok = cudaGetLastError() == cudaSuccess;
    return cudaFreeAsync(lat, st) == cudaSuccess && ok ? 0 : 1;
  }
  if (p.narrow) {  // one warp per block, so a block fits beside the trajectory kernels
    row_metrics_warp_kernel<<<296, kWarp, 0, static_cast<cudaStream_t>(stream)>>>(p);
  } else {
    const int64_t grid = (static_cast<int64_t>(p.n_traj) * kWarp + block - 1) / block;
    row_metrics_warp_kernel<<<static_cast<unsigned>(grid), block, 0,
                              static_cast<cudaStream_t>(stream)>>>(p);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
