// Kernel instantiations for dtype=f32, dim=128, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_f32_128(int G) { return pick_g<float, 128>(G); }
}  // namespace alaya
