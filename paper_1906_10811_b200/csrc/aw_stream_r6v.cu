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
        case 11: return ops_of<C6v11>();
        case 12: return ops_of<C6v12>();
        case 13: return ops_of<C6v13>();
        case 14: return ops_of<C6v14>();
        case 15: return ops_of<C6v15>();
        case 16: return ops_of<C6v16>();
        default: return ops_of<C6v3>();
    }
}
}  // namespace aw
