// aw_stream_r6.cu -- instantiations of the streaming kernel for R = 6 (space order 12).
#include "aw_stream.cuh"

namespace aw {
#ifdef AW_DEV_VARIANTS
const StreamOps* stream_ops_r6_variant(int v);  // aw_stream_r6v.cu (measurement variants, dev builds only)
#endif

const StreamOps* stream_ops_r6() {
#ifdef AW_DEV_VARIANTS
    if (const int v = variant()) return stream_ops_r6_variant(v);  // AW_STREAM_VARIANT=1/2/3 (A/B measurements)
#endif
    return ops_of<C6>();
}
}  // namespace aw
