// pass_c3 instantiations for padded channel width CP = 12 (LZ in {8, 16, 32})
#include "pass_c3.cuh"

namespace fno {

cudaError_t launch_pass_c3_cp12(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int grid, size_t smem,
                                 cudaStream_t st) {
#define FNO_C3_CASE(a, b) \
  if (LZ == a && LT == b) return launch_c3_case<a, b, 12>(maps, p, grid, smem, st);
  FNO_AC_PAIRS(FNO_C3_CASE)
#undef FNO_C3_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fno
