// aw_stream_r1.cu -- instantiations of the streaming kernel for R = 1 (space order 2).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r1() {
    return ops_of<C1>();
}
}  // namespace aw
