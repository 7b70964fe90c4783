// Kernel instantiations for dtype=bf16, dim=32, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_bf16_32(int G) { return pick_g<__nv_bfloat16, 32>(G); }
}  // namespace alaya
