// nb_train_tc.cu — bf16 training step on tcgen05 (hot-path rows a7-a9).
// Placeholder until the tensor-core backward lands: reports unsupported.
#include "nb_internal.cuh"

namespace nb {

bool train_tc_supported(const nb_desc&) { return false; }
size_t train_tc_scratch_bytes(const nb_model*, int64_t) { return 0; }
cudaError_t launch_train_tc(nb_model*, const float*, const uint8_t*, int64_t, int64_t, float,
                            float, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace nb
