// sim_inst_nw1.cu — instantiates the trajectory kernels for 1 x 64-bit
// tier masks (n <= 64 requests); one unit per mask width so the build
// compiles them in parallel.
#include "sim_kernel.cuh"

namespace saberb200 {
void* pick_sim_nw1(int g, bool trace, bool records, int sel) {
  return pick_g<1>(g, trace, records, sel);
}
}  // namespace saberb200
