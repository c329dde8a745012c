// aw_stream_r6.cu -- instantiations of the streaming kernel for R = 6 (space order 12).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r6_variant(int v);  // aw_stream_r6v.cu (measurement variants)

const StreamOps* stream_ops_r6() {
    const int v = variant();
    return v ? stream_ops_r6_variant(v) : ops_of<C6>();
}
}  // namespace aw
