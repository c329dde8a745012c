// aw_stream_r6v.cu -- measurement variants of the R = 6 configuration (AW_STREAM_VARIANT=1/2/3):
// tile height, rows per thread and ring depths for the high space orders (profiles/r1).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r6_variant(int v) {
    switch (v) {
        case 1: return ops_of<C6v1>();
        case 2: return ops_of<C6v2>();
        case 4: return ops_of<C6v4>();
        case 5: return ops_of<C6v5>();
        case 6: return ops_of<C6v6>();
        case 7: return ops_of<C6v7>();
        case 9: return ops_of<C6v8>();
        case 10: return ops_of<C6v0>();
        default: return ops_of<C6v3>();
    }
}
}  // namespace aw
