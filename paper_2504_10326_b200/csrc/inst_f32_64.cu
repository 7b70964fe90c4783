// Kernel instantiations for dtype=f32, dim=64, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_f32_64(int G) { return pick_g<float, 64>(G); }
}  // namespace alaya
