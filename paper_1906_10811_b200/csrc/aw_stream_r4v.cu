// aw_stream_r4v.cu -- development variants of the R = 4 configuration (AW_STREAM_VARIANT=1/2/3),
// kept for A/B measurements of the ring depths and tile height (profiles/README.md).
#include "aw_stream.cuh"

namespace aw {
const StreamOps* stream_ops_r4_variant(int v) {
    switch (v) {
        case 1: return ops_of<C4v1>();
        case 2: return ops_of<C4v2>();
        case 4: return ops_of<C4v4>();
        case 5: return ops_of<C4v5>();
        case 6: return ops_of<C4v6>();
        case 7: return ops_of<C4v7>();
        default: return ops_of<C4v3>();
    }
}
}  // namespace aw
