// aw_stream_r5.cu -- instantiations of the streaming kernel for R = 5 (space order 10).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r5() {
#ifdef AW_DEV_VARIANTS
    if (const int v = variant()) return v == 6 ? ops_of<C5v6>() : v == 8 ? ops_of<C5v8>() : ops_of<C5v7>();  // A/B
#endif
    return ops_of<C5>();
}
}  // namespace aw
