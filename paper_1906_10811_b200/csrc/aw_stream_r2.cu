// aw_stream_r2.cu -- instantiations of the streaming kernel for R = 2 (space order 4).
#include "aw_stream.cuh"

namespace aw {
#ifdef AW_DEV_VARIANTS
const StreamOps* stream_ops_r2_variant(int v);  // aw_stream_r2v.cu (development variants, dev builds only)
#endif

const StreamOps* stream_ops_r2() {
#ifdef AW_DEV_VARIANTS
    if (const int v = variant()) return stream_ops_r2_variant(v);  // AW_STREAM_VARIANT=1/2/3 (A/B measurements)
#endif
    return ops_of<C2>();
}
}  // namespace aw
