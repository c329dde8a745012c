// aw_stream_r7.cu -- instantiations of the streaming kernel for R = 7 (space order 14).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r7() {
    return ops_of<C7>();
}
}  // namespace aw
