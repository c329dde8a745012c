// aw_stream_r8.cu -- instantiations of the streaming kernel for R = 8 (space order 16).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r8() {
    return ops_of<C8>();
}
}  // namespace aw
