// pass_c2 instantiations for padded channel width CP = 8 (all (LZ, LT) pairs)
#include "pass_c2.cuh"

namespace fno {

cudaError_t launch_pass_c2_cp8(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem, cudaStream_t st) {
#define FNO_C2_CASE(a, b) \
  if (LZ == a && LT == b) return launch_c2_cp<a, b, 8>(maps, p, mode, grid, smem, st);
  FNO_AC_PAIRS(FNO_C2_CASE)
#undef FNO_C2_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fno
