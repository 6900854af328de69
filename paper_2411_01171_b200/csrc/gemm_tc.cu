// tcgen05 / TMEM / TMA implicit GEMM (sm_100a).  Placeholder until the
// kernel lands: reports every shape unsupported so sf_gemm uses mma.sync.
#include "common.cuh"

namespace sf {
bool gemm_tc_supported(const sf_gemm_args&) { return false; }
sf_status gemm_tc_launch(const sf_gemm_args&, cudaStream_t) {
  set_error("tcgen05 backend not built");
  return SF_ERR_UNSUPPORTED;
}
}  // namespace sf
