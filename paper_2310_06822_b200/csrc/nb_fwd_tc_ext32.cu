// nb_fwd_tc_ext32.cu — k_fwd_tc instantiations for sine / positional-encoding
// nets of width 32 (EXT kernels, nb_fwd_tc.cuh; R41, R42).
#include "nb_fwd_tc.cuh"

namespace nb {

cudaError_t launch_tc_ext32(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (m->d.pe_depth > 0) return cudaErrorInvalidValue;  // the PE operand needs A >= 32 columns
  return launch_tc_ext_d<32, 0>(m, mode, a, st);
}

}  // namespace nb
