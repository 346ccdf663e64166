// nb_fwd_tc_ext64.cu — k_fwd_tc instantiations for sine / positional-encoding
// nets of width 64 (EXT kernels, nb_fwd_tc.cuh; R41, R42).
#include "nb_fwd_tc.cuh"

namespace nb {

cudaError_t launch_tc_ext64(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (m->d.pe_depth == 0) return launch_tc_ext_d<64, 0>(m, mode, a, st);
  switch (m->d0) {
    case 2: return launch_tc_ext_d<64, 2>(m, mode, a, st);
    case 3: return launch_tc_ext_d<64, 3>(m, mode, a, st);
    case 4: return launch_tc_ext_d<64, 4>(m, mode, a, st);
    case 6: return launch_tc_ext_d<64, 6>(m, mode, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nb
