// aw_stream_r4.cu -- instantiations of the streaming kernel for R = 4 (space order 8).
#include "aw_stream.cuh"

namespace aw {
#ifdef AW_DEV_VARIANTS
const StreamOps* stream_ops_r4_variant(int v);  // aw_stream_r4v.cu (development variants, dev builds only)
#endif

const StreamOps* stream_ops_r4() {
#ifdef AW_DEV_VARIANTS
    if (const int v = variant()) return stream_ops_r4_variant(v);  // AW_STREAM_VARIANT=1/2/3 (A/B measurements)
#endif
    return ops_of<C4>();
}
}  // namespace aw
