// Host side of the tensor-core pass C (kernel: pass_c3.cuh; one translation
// unit per padded width CP): eligibility, shared-memory size, tensor map.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "pass_c3.cuh"

namespace fno {

cudaError_t launch_pass_c3_cp4(const C2Maps&, const PassCParams&, int LZ, int LT, int grid, size_t smem, cudaStream_t);
cudaError_t launch_pass_c3_cp8(const C2Maps&, const PassCParams&, int LZ, int LT, int grid, size_t smem, cudaStream_t);
cudaError_t launch_pass_c3_cp12(const C2Maps&, const PassCParams&, int LZ, int LT, int grid, size_t smem, cudaStream_t);
cudaError_t launch_pass_c3_cp16(const C2Maps&, const PassCParams&, int LZ, int LT, int grid, size_t smem, cudaStream_t);
cudaError_t launch_pass_c3_cp20(const C2Maps&, const PassCParams&, int LZ, int LT, int grid, size_t smem, cudaStream_t);

// layer forward only; tiles of exactly 128 points (LZ * TCH = 128), T a
// multiple of TCH and of 4 (TMA tile loads); FNO_PASS_C3=0 disables
bool pass_c3_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* CPo, int* TCH, size_t* smem) {
  if (mode != EPI_FWD) return false;
#ifdef FNO_DEV_KNOBS   // development builds only: FNO_PASS_C3=0 selects the FFMA pass_c2
  const char* e = std::getenv("FNO_PASS_C3");
  if (e && e[0] == '0') return false;
#endif
  const int CP = (C + 3) & ~3;
  if (CP > 20) return false;
  if (LZ != 8 && LZ != 16 && LZ != 32) return false;
  const int tch = C3T / LZ;
  if (tch > T) return false;   // T % 4 != 0: cp.async tiles (TMA rows would be misaligned)
  // long t codelets (LT >= 30) spill under the two-CTA register cap of the
  // transform warps: measured slower than pass_c2 at c4 (LT = 32, TMA tiles);
  // kept where pass_c2 has no TMA either (T % 4 != 0, c3: faster)
  const int lt_needed = std::min(2 * mt - 1, T);
  if (lt_needed > 16 && T % 4 == 0) return false;
  const size_t s = c3_layout(CP, C, Z, T, mz, mt, LZ).total;
  if (s > 227 * 1024) return false;
  *CPo = CP;
  *TCH = tch;
  *smem = s;
  return true;
}

cudaError_t launch_pass_c3(const PassCParams& p0, int LZ, int LT, int CP, int grid, size_t smem, cudaStream_t st) {
  PassCParams p = p0;
  p.TCH = C3T / LZ;
  C2Maps maps;
  std::memset(&maps, 0, sizeof maps);
  // the TMA kernel assumes full t chunks; a ragged last chunk takes the cp.async kernel
  p.tma_g = c2_tile_group(p, LZ, p.v);
  p.use_tma = (p.tma_g > 0 && c2_encode_tile_map(&maps.m[0], p.v, p, LZ)) ? 1 : 0;
  p.VW = (p.T % 2 == 0) ? 2 : 1;   // cp.async piece (floats) of the non-TMA path
  switch (CP) {
    case 4: return launch_pass_c3_cp4(maps, p, LZ, LT, grid, smem, st);
    case 8: return launch_pass_c3_cp8(maps, p, LZ, LT, grid, smem, st);
    case 12: return launch_pass_c3_cp12(maps, p, LZ, LT, grid, smem, st);
    case 16: return launch_pass_c3_cp16(maps, p, LZ, LT, grid, smem, st);
    case 20: return launch_pass_c3_cp20(maps, p, LZ, LT, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fno
