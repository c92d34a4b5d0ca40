// sim_inst_nw4.cu — instantiates the trajectory kernels for 4 x 64-bit
// tier masks (n <= 256 requests); one unit per mask width so the build
// compiles them in parallel.
#include "sim_kernel.cuh"

namespace saberb200 {
void* pick_sim_nw4(int g, bool trace, bool records, int sel) {
  return pick_g<4>(g, trace, records, sel);
}
}  // namespace saberb200
