// Kernel instantiations for dtype=bf16, dim=64, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_bf16_64(int G) { return pick_g<__nv_bfloat16, 64>(G); }
}  // namespace alaya
