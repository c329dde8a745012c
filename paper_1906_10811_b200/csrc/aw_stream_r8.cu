// aw_stream_r8.cu -- instantiations of the streaming kernel for R = 8 (space order 16).
#include "aw_stream.cuh"

namespace aw {
#ifdef AW_DEV_VARIANTS
const StreamOps* stream_ops_r8_variant(int v);  // aw_stream_r8v.cu (measurement variants, dev builds only)
#endif

const StreamOps* stream_ops_r8() {
#ifdef AW_DEV_VARIANTS
    if (const int v = variant()) return stream_ops_r8_variant(v);  // AW_STREAM_VARIANT=1/2/3 (A/B measurements)
#endif
    return ops_of<C8>();
}
}  // namespace aw
