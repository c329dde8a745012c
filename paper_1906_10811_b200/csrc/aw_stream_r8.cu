// aw_stream_r8.cu -- instantiations of the streaming kernel for R = 8 (space order 16).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r8_variant(int v);  // aw_stream_r8v.cu (measurement variants)

const StreamOps* stream_ops_r8() {
    const int v = variant();
    return v ? stream_ops_r8_variant(v) : ops_of<C8>();
}
}  // namespace aw
