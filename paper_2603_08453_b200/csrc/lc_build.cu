// GPU prefill helpers: synthetic workload generation
// and build_index on the device.  (Implemented in a later milestone.)
#include "../../include/lychee_b200.h"
#include "lc_common.cuh"

extern "C" {
int lc_index_build(lc_index_t, const uint32_t*, const uint32_t*, const uint64_t*, double, uint32_t,
                   uint32_t, const uint64_t*) {
    return LC_ERUNTIME;
}
int lc_gen_workload(lc_index_t, uint32_t, uint32_t, double, uint32_t, double, const uint64_t*, uint8_t*,
                    float*) {
    return LC_ERUNTIME;
}
}
