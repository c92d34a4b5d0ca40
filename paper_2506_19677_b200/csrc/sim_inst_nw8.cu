// sim_inst_nw8.cu — instantiates the trajectory kernels for 8 x 64-bit
// tier masks (n <= 512 requests); one unit per mask width so the build
// compiles them in parallel.
#include "sim_kernel.cuh"

namespace saberb200 {
void* pick_sim_nw8(int g, bool trace, bool records, int sel) {
  return pick_g<8>(g, trace, records, sel);
}
}  // namespace saberb200
