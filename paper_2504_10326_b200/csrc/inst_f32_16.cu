// Kernel instantiations for dtype=f32, dim=16, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_f32_16(int G) { return pick_g<float, 16>(G); }
}  // namespace alaya
