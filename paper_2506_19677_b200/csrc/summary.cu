// summary.cu — sweep summary on the device (simloop.cpp:206-275).
//
// S1 (thread per (mix, rps)): per-cell mean goodput over repeats, the static
//    argmax over caps in ascending order with ties to the smaller cap, and the
//    per-cell latency-ratio means.
// S2 (block per mix): means over the rps grid, pooled CVs over every ratio of
//    the chosen cells, and CVs of the per-rps ratio means.
// Every sum runs sequentially in the reference's order (rows in grid order,
// ratios in request-id order), so the summary is bit-identical to
// saber::sweep's.  Ratios are recomputed from completion times exactly like
// ratio_to_sla (metrics.cpp:39-47).
#include <cuda_runtime.h>

#include <climits>
#include <cmath>

#include "saber_internal.h"

namespace saberb200 {
namespace {

constexpr int kCellScratch = 6;

struct RowView {
  const double* comp;
  const double* arr;
  const double* sla;
  int n;
};

__device__ __forceinline__ RowView row_view(const SummaryParams& p, int mi, int ri, int64_t row,
                                            int rep) {
  const int64_t w = (static_cast<int64_t>(mi) * p.n_rps + ri) * p.repeats + rep;
  RowView v;
  v.comp = p.completion + row * p.wl.nmax;
  v.arr = p.wl.arrival + w * p.wl.nmax;
  v.sla = p.wl.sla + w * p.wl.nmax;
  v.n = p.n;
  return v;
}

// Adds this row's ratios (id order) to (sum, count).
__device__ __forceinline__ void add_ratios(const RowView& v, double& sum, int64_t& cnt) {
  for (int q = 0; q < v.n; ++q) {
    const double c = v.comp[q];
    if (isnan(c)) continue;
    sum += (c - v.arr[q]) / v.sla[q];
    ++cnt;
  }
}
__device__ __forceinline__ void add_sq(const RowView& v, double mean, double& acc) {
  for (int q = 0; q < v.n; ++q) {
    const double c = v.comp[q];
    if (isnan(c)) continue;
    const double x = (c - v.arr[q]) / v.sla[q];
    acc += (x - mean) * (x - mean);
  }
}

__global__ void summary_cells_kernel(const SummaryParams p) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= p.n_mixes * p.n_rps) return;
  const int mi = cell / p.n_rps, ri = cell % p.n_rps;
  const int R = p.repeats;
  const int per_rps = p.n_caps * R + (p.with_saber ? R : 0);
  const int64_t base = static_cast<int64_t>(cell) * per_rps;
  double* out = p.scratch + static_cast<int64_t>(cell) * kCellScratch;
  const double nanv = nan("");
  out[0] = out[1] = out[2] = out[3] = nanv;
  out[4] = out[5] = 0.0;
  int best_cap = 0;
  if (p.n_caps > 0) {
    double best_mean = -1.0;
    long long prev = LLONG_MIN;
    for (;;) {  // unique caps in ascending order (std::map iteration)
      long long cap = LLONG_MAX;
      for (int w = 0; w < p.n_caps; ++w)
        if (p.caps[w] > prev && p.caps[w] < cap) cap = p.caps[w];
      if (cap == LLONG_MAX) break;
      prev = cap;
      double s = 0.0;
      int64_t c = 0;
      for (int w = 0; w < p.n_caps; ++w) {
        if (p.caps[w] != cap) continue;
        for (int i = 0; i < R; ++i) {
          s += p.rows[base + static_cast<int64_t>(w) * R + i].goodput;
          ++c;
        }
      }
      const double m = s / static_cast<double>(c);
      if (m > best_mean) {
        best_mean = m;
        best_cap = static_cast<int>(cap);
      }
    }
    out[1] = best_mean;
    double s = 0.0;
    int64_t c = 0;
    for (int w = 0; w < p.n_caps; ++w) {
      if (p.caps[w] != best_cap) continue;
      for (int i = 0; i < R; ++i)
        add_ratios(row_view(p, mi, ri, base + static_cast<int64_t>(w) * R + i, i), s, c);
    }
    if (c > 0) {
      out[3] = s / static_cast<double>(c);
      out[5] = 1.0;
    }
  }
  p.best_cap[cell] = best_cap;
  if (p.with_saber) {
    const int64_t sb = base + static_cast<int64_t>(p.n_caps) * R;
    double g = 0.0;
    for (int i = 0; i < R; ++i) g += p.rows[sb + i].goodput;
    out[0] = g / static_cast<double>(R);
    double s = 0.0;
    int64_t c = 0;
    for (int i = 0; i < R; ++i) add_ratios(row_view(p, mi, ri, sb + i, i), s, c);
    if (c > 0) {
      out[2] = s / static_cast<double>(c);
      out[4] = 1.0;
    }
  }
}

// cv_or_nan (simloop.cpp:28-35) over scratch column `col` gated by `flag`.
__device__ double cv_cells(const double* sc, int n_rps, int col, int flag) {
  double mean = 0.0;
  int64_t n = 0;
  for (int ri = 0; ri < n_rps; ++ri)
    if (sc[ri * kCellScratch + flag] != 0.0) {
      mean += sc[ri * kCellScratch + col];
      ++n;
    }
  if (n == 0) return nan("");
  mean /= static_cast<double>(n);
  if (mean == 0.0) return nan("");
  double var = 0.0;
  for (int ri = 0; ri < n_rps; ++ri)
    if (sc[ri * kCellScratch + flag] != 0.0) {
      const double v = sc[ri * kCellScratch + col];
      var += (v - mean) * (v - mean);
    }
  var /= static_cast<double>(n);
  return sqrt(var) / mean;
}

__global__ void summary_mix_kernel(const SummaryParams p) {
  const int mi = blockIdx.x;
  const int variant = threadIdx.x;  // 0 = saber, 1 = best static
  if (mi >= p.n_mixes || variant > 1) return;
  __shared__ double means[2];
  const double* sc = p.scratch + static_cast<int64_t>(mi) * p.n_rps * kCellScratch;
  const int R = p.repeats;
  const int per_rps = p.n_caps * R + (p.with_saber ? R : 0);
  const bool present = variant == 0 ? p.with_saber != 0 : p.n_caps > 0;
  const double nanv = nan("");
  double mean_goodput = nanv, pooled = nanv, rps_cv = nanv;
  if (present) {
    double s = 0.0;
    for (int ri = 0; ri < p.n_rps; ++ri) s += sc[ri * kCellScratch + (variant == 0 ? 0 : 1)];
    mean_goodput = s / static_cast<double>(p.n_rps);
    // pooled ratios: rps in grid order, the chosen cell's rows, ids in order
    double sum = 0.0;
    int64_t cnt = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const double mean = pass == 0 ? 0.0 : sum / static_cast<double>(cnt);
      if (pass == 1 && (cnt == 0 || mean == 0.0)) break;
      double acc = 0.0;
      for (int ri = 0; ri < p.n_rps; ++ri) {
        const int64_t base = (static_cast<int64_t>(mi) * p.n_rps + ri) * per_rps;
        if (variant == 0) {
          const int64_t sb = base + static_cast<int64_t>(p.n_caps) * R;
          for (int i = 0; i < R; ++i) {
            const RowView v = row_view(p, mi, ri, sb + i, i);
            if (pass == 0) add_ratios(v, sum, cnt);
            else add_sq(v, mean, acc);
          }
        } else {
          const int bc = p.best_cap[mi * p.n_rps + ri];
          for (int w = 0; w < p.n_caps; ++w) {
            if (p.caps[w] != bc) continue;
            for (int i = 0; i < R; ++i) {
              const RowView v = row_view(p, mi, ri, base + static_cast<int64_t>(w) * R + i, i);
              if (pass == 0) add_ratios(v, sum, cnt);
              else add_sq(v, mean, acc);
            }
          }
        }
      }
      if (pass == 1) pooled = sqrt(acc / static_cast<double>(cnt)) / mean;
    }
    rps_cv = cv_cells(sc, p.n_rps, variant == 0 ? 2 : 3, variant == 0 ? 4 : 5);
  }
  means[variant] = mean_goodput;
  __syncthreads();
  saber_mix_summary* out = p.summary + mi;
  if (variant == 0) {
    out->saber_mean_goodput = mean_goodput;
    out->saber_pooled_cv = pooled;
    out->saber_rps_mean_cv = rps_cv;
    out->delta = means[0] - means[1];
  } else {
    out->best_static_mean_goodput = mean_goodput;
    out->best_static_pooled_cv = pooled;
    out->best_static_rps_mean_cv = rps_cv;
  }
}

}  // namespace

int launch_summary(const SummaryParams& p, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int cells = p.n_mixes * p.n_rps;
  if (cells == 0) return 0;
  summary_cells_kernel<<<(cells + 63) / 64, 64, 0, s>>>(p);
  summary_mix_kernel<<<p.n_mixes, 2, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
