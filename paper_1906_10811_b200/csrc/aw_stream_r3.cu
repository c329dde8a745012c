// aw_stream_r3.cu -- instantiations of the streaming kernel for R = 3 (space order 6).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r3() {
    return ops_of<C3>();
}
}  // namespace aw
