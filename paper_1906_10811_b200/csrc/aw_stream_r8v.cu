// aw_stream_r8v.cu -- measurement variants of the R = 8 configuration (AW_STREAM_VARIANT=1/2/3):
// tile height, rows per thread and ring depths for the high space orders (profiles/r1).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r8_variant(int v) {
    switch (v) {
        case 1: return ops_of<C8v1>();
        case 2: return ops_of<C8v2>();
        case 4: return ops_of<C8v4>();
        case 5: return ops_of<C8v5>();
        case 6: return ops_of<C8v6>();
        case 7: return ops_of<C8v7>();
        case 9: return ops_of<C8v9>();
        case 10: return ops_of<C8v10>();
        case 11: return ops_of<C8v11>();
        case 12: return ops_of<C8v12>();
        case 13: return ops_of<C8v13>();
        case 14: return ops_of<C8v0>();
        case 15: return ops_of<C8v15>();
        case 16: return ops_of<C8v16>();
        default: return ops_of<C8v3>();
    }
}
}  // namespace aw
