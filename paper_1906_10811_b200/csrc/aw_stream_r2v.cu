// aw_stream_r2v.cu -- development variants of the R = 2 configuration (AW_STREAM_VARIANT=1/2/3), for
// A/B measurements of the ring depths and tile height on the L2-resident C2 grid (resident kernel).
#include "aw_stream.cuh"

namespace aw {
namespace {
using C2v1 = Cfg<2, 32, 2, 8, 3, 0, 1>;   // deeper u^n ring, shallower streams ring
using C2v2 = Cfg<2, 32, 2, 6, 2, 0, 1>;
using C2v3 = Cfg<2, 16, 2, 8, 8, 0, 1>;   // 64 x 16 tiles (8 consumer warps), deep rings
using C2v4 = Cfg<2, 32, 4, 4, 4, 0, 1, true, 0, 40, 0>;   // half queue, 4 rows per thread (8 consumer warps)
using C2v5 = Cfg<2, 32, 2, 4, 4, 0, 1, true, 0, 40, 0>;   // half queue, 16 consumer warps
}  // namespace
const StreamOps* stream_ops_r2_variant(int v) {
    switch (v) {
        case 1: return ops_of<C2v1>();
        case 2: return ops_of<C2v2>();
        case 4: return ops_of<C2v4>();
        case 5: return ops_of<C2v5>();
        default: return ops_of<C2v3>();
    }
}
}  // namespace aw
