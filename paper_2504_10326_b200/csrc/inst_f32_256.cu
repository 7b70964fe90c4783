// Kernel instantiations for dtype=f32, dim=256, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_f32_256(int G) { return pick_g<float, 256>(G); }
}  // namespace alaya
