// Kernel instantiations for dtype=bf16, dim=16, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_bf16_16(int G) { return pick_g<__nv_bfloat16, 16>(G); }
}  // namespace alaya
