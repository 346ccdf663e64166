// nb_fwd_tc_w128l4_d6.cu — specialised instantiation of k_fwd_tc (nb_fwd_tc.cuh)
// for one BASELINE.json architecture, in its own translation unit.
#include "nb_fwd_tc.cuh"

namespace nb {

cudaError_t launch_tc_w128l4_d6(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold) {
  return fold ? launch_tc_modes<128, 4, 0, 0, 6, true>(m, mode, a, st)
              : launch_tc_modes<128, 4, 0, 0, 6, false>(m, mode, a, st);
}

}  // namespace nb
