// sim_inst_wide.cu — instantiates the wide trajectory kernel (n > 512
// requests or an admission window > 16).
#include "sim_kernel.cuh"

namespace saberb200 {
void* pick_sim_wide(bool trace, bool records) {
  if (trace) return reinterpret_cast<void*>(&sim_kernel_wide<true, true>);
  if (records) return reinterpret_cast<void*>(&sim_kernel_wide<false, true>);
  return reinterpret_cast<void*>(&sim_kernel_wide<false, false>);
}
}  // namespace saberb200
