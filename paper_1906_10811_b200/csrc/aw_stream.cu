// aw_stream.cu -- 2.5D z-streaming stencil kernel (placeholder until the TMA kernel lands).
#include "aw_internal.h"

namespace aw {
struct StreamPlan {
    int dummy;
};
cudaError_t stream_prepare(const Geom&, const float* const*, const float*, StreamPlan** plan, int*, cudaStream_t) {
    *plan = nullptr;
    return cudaErrorNotSupported;
}
void stream_release(StreamPlan* p) { delete p; }
cudaError_t launch_stencil_stream(StreamPlan*, const Geom&, const Coefs&, int, const float*, float*, const float*,
                                  const float*, const Halo&, int, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace aw
