// Kernel instantiations for dtype=f32, dim=32, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_f32_32(int G) { return pick_g<float, 32>(G); }
}  // namespace alaya
