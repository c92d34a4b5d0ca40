// sim_inst_nw2.cu — instantiates the trajectory kernels for 2 x 64-bit
// tier masks (n <= 128 requests); one unit per mask width so the build
// compiles them in parallel.
#include "sim_kernel.cuh"

namespace saberb200 {
void* pick_sim_nw2(int g, bool trace, bool records, int sel) {
  return pick_g<2>(g, trace, records, sel);
}
}  // namespace saberb200
