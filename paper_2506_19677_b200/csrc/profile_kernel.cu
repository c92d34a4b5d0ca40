// profile_kernel.cu — batched offline load-speed profiling (calibration.cpp:58-135).
//
// One thread per profile.  Bursts of sizes cycling 1..l_max are admitted into a
// drained engine (static cap 10*l_max, so the whole burst) and the engine is
// advanced in 60 s steps until empty (calibration.cpp:102-128).  A burst is
// homogeneous — one task, one input length, one output length — so all its
// slots evolve bit-identically through Engine::advance_to (engine.cpp:51-127):
// the same boundary, the same updates, the same completion pass.  One
// representative slot with load = burst size therefore reproduces the
// reference's per-slot loop exactly, and its completion emits `size` identical
// samples (llround(mean_decode_load), max_out / decode_duration).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "saber_internal.h"

namespace saberb200 {
namespace {

constexpr double kOnePlusTol = 1.0 + 1e-12;

__global__ void profile_kernel(const ProfileParams p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_profiles) return;
  const double* GT = p.tables + static_cast<int64_t>(i) * p.table_stride;
  const double pr = p.prefill_rate[i];
  int64_t s = p.sample_off[i];
  double clock = 0.0;
  for (int64_t b = p.burst_off[i]; b < p.burst_off[i + 1]; ++b) {
    const int size = p.burst_size[b];
    const double in = p.burst_in[b];
    const double m = p.burst_out[b];
    // Engine::admit x size at now = clock (engine.cpp:26-49)
    double pl = pr > 0.0 ? in / pr : 0.0;
    double decode_start = pl == 0.0 ? clock : -1.0;
    double g = 0.0, load_time = 0.0;
    int A = size;
    while (A > 0) {  // drain: advance_to(clock + 60) until empty
      const double t = clock + 60.0;
      while (clock < t) {
        if (A == 0) {
          clock = t;
          break;
        }
        const int load = A;
        const double speed = GT[load];
        double dt = t - clock;
        const double boundary = pl > 0.0 ? pl : (m - g) / speed;
        dt = (boundary < dt) ? boundary : dt;
        const double group = dt * kOnePlusTol;
        if (pl > 0.0) {
          pl = pl <= group ? 0.0 : pl - dt;
        } else {
          g += speed * dt;
          load_time += load * dt;
        }
        clock += dt;
        if (pl == 0.0 && decode_start < 0.0) decode_start = clock;
        if (decode_start >= 0.0 && g + speed * (group - dt) >= m) {
          const double duration = clock - decode_start;
          const double mean_load = load_time / duration;
          const int L = static_cast<int>(llround(mean_load));
          const double speed_sample = m / duration;
          for (int k = 0; k < size; ++k, ++s) {
            p.loads[s] = L;
            p.speeds[s] = speed_sample;
          }
          A = 0;
        }
      }
    }
  }
}

}  // namespace

int launch_profile(const ProfileParams& p, void* stream) {
  if (p.n_profiles == 0) return 0;
  profile_kernel<<<(p.n_profiles + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace saberb200
