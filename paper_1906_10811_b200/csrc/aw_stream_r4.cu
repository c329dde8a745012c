// aw_stream_r4.cu -- instantiations of the streaming kernel for R = 4 (space order 8).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r4_variant(int v);  // aw_stream_r4v.cu (development variants)

const StreamOps* stream_ops_r4() {
    const int v = variant();  // AW_STREAM_VARIANT=1/2/3: measurement variants of the R=4 configuration
    return v ? stream_ops_r4_variant(v) : ops_of<C4>();
}
}  // namespace aw
