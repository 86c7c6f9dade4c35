// K1 tensor-core path (tcgen05 / TMEM): placeholder until the kernel lands.
#include "common.cuh"

namespace cmf {

int gram_tc_launch(const int64_t *, const int32_t *, const float *, const float *, int64_t,
                   const float *, int, double, int, const float *, bool, void *, int64_t, float *,
                   int64_t *, int32_t *, cudaStream_t) {
    return set_error(CMF_EINVAL, "tensor-core Gram kernel not available in this build");
}

}  // namespace cmf
