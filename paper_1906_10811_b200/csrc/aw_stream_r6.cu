// aw_stream_r6.cu -- instantiations of the streaming kernel for R = 6 (space order 12); dev builds
// also hold the split high-order kernel (aw_hstream.cuh) on the same plan geometry, for A/B runs.
#include "aw_hstream.cuh"

namespace aw {
#ifdef AW_DEV_VARIANTS
const StreamOps* stream_ops_r6_variant(int v);  // aw_stream_r6v.cu (measurement variants, dev builds only)
#endif

const StreamOps* stream_ops_r6() {
#ifdef AW_DEV_VARIANTS
    // AW_STREAM_VARIANT=8: the split high-order kernel (aw_hstream.cuh); 1..5: measurement variants
    // (the split kernel pairs with the round-1 geometry, 16-row tiles: C6v0)
    if (const int v = variant()) return v == 8 ? ops_of_h<H6, C6v0>() : stream_ops_r6_variant(v);
#endif
    return ops_of<C6>();
}
}  // namespace aw
