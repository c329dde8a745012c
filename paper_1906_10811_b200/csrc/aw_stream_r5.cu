// aw_stream_r5.cu -- instantiations of the streaming kernel for R = 5 (space order 10).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r5() {
    return ops_of<C5>();
}
}  // namespace aw
