// gemm_tc.cu -- tcgen05 kind::i8 variant (placeholder until the kernel lands).
#include "common.cuh"

namespace apnn {

bool tc_i8_supports(const Geom&) { return false; }

cudaError_t launch_tc_i8(const uint32_t*, const uint32_t*, const Geom&, const Epi&, void*, int,
                         cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace apnn
