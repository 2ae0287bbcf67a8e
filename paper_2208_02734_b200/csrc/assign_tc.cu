// assign_tc.cu -- K1: tcgen05 3xTF32 dense assignment (placeholder until the kernel lands).
#include "common.cuh"

namespace mask {

bool tc_supported(int64_t, int, int64_t) { return false; }

void launch_assign_tc(const float*, int64_t, int, const float*, const float*, const float*,
                      int64_t, const float*, int32_t*, float*, int32_t*, int32_t*, float,
                      cudaStream_t) {
  fail(MASK_ERR_UNSUPPORTED, "tensor-core assignment not built");
}

}  // namespace mask
