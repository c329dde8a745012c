// aw_stream_r7.cu -- instantiations of the streaming kernel for R = 7 (space order 14); dev builds
// also hold the split high-order kernel (aw_hstream.cuh) on the same plan geometry, for A/B runs.
#include "aw_hstream.cuh"

namespace aw {
const StreamOps* stream_ops_r7() {
#ifdef AW_DEV_VARIANTS
    if (variant() == 8) return ops_of_h<H7, C7v0>();  // AW_STREAM_VARIANT=8: the split high-order kernel (A/B)
    if (variant() == 6) return ops_of<C7v6>();      // half register queue, 12 consumer warps
    if (variant() == 9) return ops_of<C7v9>();      // partial queue (QJ = 2), 12 consumer warps
    if (variant() == 12) return ops_of<C7v12>();    // half queue, 4 rows per thread
    if (variant() == 10) return ops_of<C7v0>();     // the previous product configuration
    if (variant() == 13) return ops_of<C7v13>();
#endif
    return ops_of<C7>();
}
}  // namespace aw
