// aw_stream_r8.cu -- instantiations of the streaming kernel for R = 8 (space order 16); dev builds
// also hold the split high-order kernel (aw_hstream.cuh) on the same plan geometry, for A/B runs.
#include "aw_hstream.cuh"

namespace aw {
#ifdef AW_DEV_VARIANTS
const StreamOps* stream_ops_r8_variant(int v);  // aw_stream_r8v.cu (measurement variants, dev builds only)
#endif

const StreamOps* stream_ops_r8() {
#ifdef AW_DEV_VARIANTS
    // AW_STREAM_VARIANT=8: the split high-order kernel (aw_hstream.cuh); 1..5: measurement variants
    if (const int v = variant()) return v == 8 ? ops_of_h<H8, C8v0>() : stream_ops_r8_variant(v);
#endif
    return ops_of<C8>();
}
}  // namespace aw
