// Kernel instantiations for dtype=bf16, dim=128, group sizes 1..8.
#include "alaya_dispatch.cuh"

namespace alaya {
StageSet pick_bf16_128(int G) { return pick_g<__nv_bfloat16, 128>(G); }
}  // namespace alaya
