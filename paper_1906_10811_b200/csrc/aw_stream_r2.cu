// aw_stream_r2.cu -- instantiations of the streaming kernel for R = 2 (space order 4).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r2() {
    return ops_of<C2>();
}
}  // namespace aw
