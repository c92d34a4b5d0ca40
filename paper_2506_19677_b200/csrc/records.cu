// records.cu — the per-request epilogue of run() / run_with_requests() on the
// device (RunOutput::requests / records / metrics.per_task):
//   pack_requests_kernel : the workload tables -> saber_request AoS (the
//                          generate() output, workload.cpp:52-79, or the replay)
//   records_kernel       : per request the final state (Request, types.hpp:45-59;
//                          make_record, metrics.cpp:17-30) and, per task group,
//                          the empirical latency CDF of cdf() (metrics.cpp:61-85)
//                          with the group's issued / met counts (compute_metrics,
//                          metrics.cpp:107-140).
// One warp per trajectory.  The CDF is built by rank counting (no sort): the
// completed requests of a group are ordered by (latency, id), request q lands
// at the position of its rank, and it carries a point iff it is the last of
// its latency tie, with fraction (#latencies <= its latency) / issued — the
// reference's `seen / issued` at the last element of a tie.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "saber_internal.h"
#include "sim_common.cuh"

namespace saberb200 {
namespace {

using simdev::kInf;

// std::map<std::string, ...> order of the catalog names: code_generation,
// code_qna, code_summary, code_translation (indexed by catalog id).
__constant__ int32_t kNameRank[4] = {1, 0, 2, 3};

__device__ __forceinline__ int32_t group_of(const RecordsParams& p, int64_t o) {
  if (p.group && p.group[o] >= 0) return p.group[o];
  const int t = p.wl.task[o];
  return t >= 0 && t < 4 ? kNameRank[t] : 4;
}

__global__ void __launch_bounds__(128) pack_requests_kernel(const RecordsParams p) {
  const int64_t cells = static_cast<int64_t>(p.n_traj) * p.wl.nmax;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = c / p.wl.nmax;
    const int i = static_cast<int>(c - k * p.wl.nmax);
    const TrajDesc d = p.traj[k];
    if (i >= d.n) continue;
    const int64_t o = static_cast<int64_t>(d.workload) * p.wl.nmax + i;
    saber_request r;
    r.arrival_time = p.wl.arrival[o];
    r.sla_seconds = p.wl.sla[o];
    r.deadline = p.wl.deadline[o];
    r.input_tokens = static_cast<int32_t>(p.wl.input[o]);
    r.max_output_tokens = static_cast<int32_t>(p.wl.max_out[o]);
    r.task = p.wl.task[o];
    r.group = group_of(p, o);
    p.requests[d.row * p.wl.nmax + i] = r;
  }
}

__global__ void __launch_bounds__(128) records_kernel(const RecordsParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; k < p.n_traj;
       k += warps) {  // uniform per warp
    const TrajDesc d = p.traj[k];
    const int n = d.n;
    const int64_t wo = static_cast<int64_t>(d.workload) * p.wl.nmax;
    const int64_t so = d.row * static_cast<int64_t>(p.wl.nmax);  // [rows][nmax] outputs
    const double* ARR = p.wl.arrival + wo;
    const double* C = p.completion + so;
    // final state and record of every request
    for (int q = lane; q < n; q += kWarp) {
      const double c = C[q], a = ARR[q], sla = p.wl.sla[wo + q];
      const double adm = p.admit[so + q];
      const bool done = !isnan(c), admitted = !isnan(adm);
      const bool demoted = p.demoted[so + q] != 0;
      saber_request_state st;
      st.admit_time = adm;
      st.completion_time = c;
      const double m = p.wl.max_out[wo + q];
      // Engine: generated = max_out at completion (engine.cpp:107); the
      // fluid progress of a slot still running; 0 for a queued request.
      st.generated_tokens = done ? m : p.generated[so + q];
      // Engine::admit records required_speed(r, now) with generated == 0
      st.recorded_required_speed =
          admitted ? simdev::queued_need(m, p.wl.deadline[wo + q], adm) : nan("");
      st.state = done ? SABER_STATE_COMPLETED
                      : admitted ? SABER_STATE_EXECUTING
                                 : demoted ? SABER_STATE_QUEUED_LOW : SABER_STATE_QUEUED_HIGH;
      st.met_sla = done && c - a <= sla;  // make_record
      st.demoted = demoted;
      st.pad_ = 0;
      p.states[so + q] = st;
      if (p.cdf_latency) {
        p.cdf_latency[so + q] = nan("");
        p.cdf_fraction[so + q] = nan("");
      }
    }
    if (p.group_issued)
      for (int g = lane; g < p.max_groups; g += kWarp) {
        p.group_issued[d.row * p.max_groups + g] = 0;
        p.group_met[d.row * p.max_groups + g] = 0;
      }
    __syncwarp();
    if (!p.cdf_latency && !p.group_issued) continue;
    for (int q = lane; q < n; q += kWarp) {
      const int32_t gq = group_of(p, wo + q);
      const double cq = C[q];
      const bool hq = !isnan(cq);
      const double lq = hq ? cq - ARR[q] : kInf;
      int start = 0, issued = 0, pos = 0, le = 0, met = 0;
      bool later_tie = false;
      for (int j = 0; j < n; ++j) {
        const int32_t gj = group_of(p, wo + j);
        start += gj < gq;
        if (gj != gq) continue;
        ++issued;
        const double cj = C[j];
        if (isnan(cj)) continue;
        const double lj = cj - ARR[j];
        met += lj <= p.wl.sla[wo + j];
        if (!hq) continue;
        pos += lj < lq || (lj == lq && j < q);
        le += lj <= lq;
        later_tie |= lj == lq && j > q;
      }
      if (hq && p.cdf_latency) {
        p.cdf_latency[so + start + pos] = lq;
        p.cdf_fraction[so + start + pos] =
            later_tie ? nan("") : static_cast<double>(le) / static_cast<double>(issued);
      }
      if (p.group_issued && gq >= 0 && gq < p.max_groups) {
        // every member of the group computes the same counts
        p.group_issued[d.row * p.max_groups + gq] = issued;
        p.group_met[d.row * p.max_groups + gq] = met;
      }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) pack_row_stats_kernel(const saber_traj_row* rows, int64_t n,
                                                            saber_row_stats* out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const saber_traj_row& r = rows[i];
    out[i] = saber_row_stats{r.goodput, r.ratio_mean, r.ratio_std, r.cv};
  }
}

}  // namespace

int launch_pack_row_stats(const saber_traj_row* rows, int64_t n_rows, saber_row_stats* out,
                          void* stream) {
  if (n_rows == 0) return 0;
  const int64_t want = (n_rows + 255) / 256;
  const int grid = static_cast<int>(want < 1184 ? want : 1184);
  pack_row_stats_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, n_rows, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_pack_requests(const RecordsParams& p, void* stream) {
  const int64_t cells = static_cast<int64_t>(p.n_traj) * p.wl.nmax;
  if (cells == 0 || !p.requests) return 0;
  const int block = 128;
  const int64_t want = (cells + block - 1) / block;
  const int grid = static_cast<int>(want < 4096 ? want : 4096);
  pack_requests_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_records(const RecordsParams& p, void* stream) {
  if (p.n_traj == 0 || !p.states) return 0;
  const int block = 128;
  const int64_t want = (static_cast<int64_t>(p.n_traj) * kWarp + block - 1) / block;
  const int grid = static_cast<int>(want < 4096 ? want : 4096);
  records_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
