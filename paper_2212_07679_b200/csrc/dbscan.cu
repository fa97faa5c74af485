// dbscan.cu -- K12 (placeholder until the GPU DBSCAN lands).
#include "index.h"

namespace snn {
snn_status dbscan_impl(snn_index, double, int32_t, int32_t *, int32_t *, cudaStream_t) {
    return fail(SNN_ERR_UNSUPPORTED, "snn_dbscan: not implemented yet");
}
}  // namespace snn
