// nb_fwd_tc_gen64.cu — generic (run-time d0 / L / heads) instantiation of
// k_fwd_tc (nb_fwd_tc.cuh) for width 64, in its own translation unit.
#include "nb_fwd_tc.cuh"

namespace nb {

cudaError_t launch_tc_gen64(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold) {
  if (m->d.activation != NB_RELU || m->d.pe_depth > 0) return launch_tc_ext64(m, mode, a, st);
  return fold ? launch_tc_modes<64, 0, 0, 0, 0, true>(m, mode, a, st)
              : launch_tc_modes<64, 0, 0, 0, 0, false>(m, mode, a, st);
}

}  // namespace nb
