// Host side of pass C generation 4 (kernel: pass_c4.cuh; one translation unit
// per padded width CP so the instantiations compile in parallel): eligibility,
// ring depth, shared-memory size and the TMA tensor maps of the tile inputs.
#include <cudaTypedefs.h>

#include <cstring>

#include "pass_c4.cuh"

namespace fno {

// padded channel width of the pass_c4 instantiations: 4, 8 and the paper's
// width 20 (C = 9..20 pads to 20: padded channels carry zeros); C > 20 keeps
// the generic pass_c
static int c4_cp_of(int C) {
  if (C <= 4) return 4;
  if (C <= 8) return 8;
  if (C <= 20) return 20;
  return 0;
}

// Tiles of exactly 128 points (LZ in {8, 16, 32}, TCH = 128 / LZ <= T); the
// deepest input ring that fits 227 KB (forward up to 6 stages, backward up to
// 4; at least 2, else the plan keeps pass_c2 / pass_c3)
bool pass_c4_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* CPo, int* NS, size_t* smem) {
  const int CP = c4_cp_of(C);
  if (!CP) return false;
  if (LZ != 8 && LZ != 16 && LZ != 32) return false;
  if (128 / LZ > T) return false;
  const size_t cap = 227 * 1024;
  if (mode == EPI_U) {   // no input tiles; the slab staged when it fits
    for (int sl = (C * mt) % 2 == 0 ? 1 : 0; sl >= 0; --sl) {
      const size_t s = c4_layout(CP, mode, C, Z, T, mz, LZ, 1, 2, sl, mt).total;
      if (s <= cap) {
        *CPo = CP; *NS = 1 | (2 << 8) | (sl << 16); *smem = s;
        return true;
      }
    }
    return false;
  }
  // preference: the column slab staged by TMA (phase 1 off L2) with four U
  // buffers and >= 3 ring stages, staged with two U buffers, then unstaged with
  // four / two U buffers and the deepest ring.  Staging needs 16-byte bulk
  // copies: C mt even (every chunk size and offset a multiple of 16 bytes).
  const bool sl_ok = (C * mt) % 2 == 0;
  struct Pref { int sl, nub, nsmin; };
  const Pref prefs[] = {{1, 4, 3}, {1, 4, 2}, {1, 2, 3}, {0, 4, 3}, {0, 2, 2}};
  for (const Pref& pr : prefs) {
    if (pr.sl && (!sl_ok || mode == EPI_BWD)) continue;   // (the backward kernels are built without the staged slab)
    for (int ns = mode == EPI_FWD ? C4_MAXNS : 4; ns >= pr.nsmin; --ns) {
      const size_t s = c4_layout(CP, mode, C, Z, T, mz, LZ, ns, pr.nub, pr.sl, mt).total;
      if (s <= cap) {
        *CPo = CP; *NS = ns | (pr.nub << 8) | (pr.sl << 16); *smem = s;
        return true;
      }
    }
  }
  return false;
}

cudaError_t launch_pass_c4(const PassCParams& p0, int LZ, int LT, int CP, int mode, int grid, size_t smem,
                           cudaStream_t st) {
  PassCParams p = p0;
  p.TCH = 128 / LZ;
  C2Maps maps;
  std::memset(&maps, 0, sizeof maps);
  // one tile geometry for inputs and outputs (16-byte aligned TMA boxes and
  // float4 stores; the row-group view when T % 4 != 0)
  p.tma_g = c2_tile_group(p, LZ, p.out);
  if (p.tma_g <= 0) return cudaErrorNotSupported;
  if (mode != EPI_U) {
    const float* src0 = mode == EPI_FWD ? p.v : p.dy;
    if (c2_tile_group(p, LZ, src0) != p.tma_g || !c2_encode_tile_map(&maps.m[0], src0, p, LZ))
      return cudaErrorNotSupported;
    if (mode == EPI_BWD && (c2_tile_group(p, LZ, p.v) != p.tma_g || !c2_encode_tile_map(&maps.m[1], p.v, p, LZ)))
      return cudaErrorNotSupported;
    if (p.zsave && c2_tile_group(p, LZ, p.zsave) != p.tma_g) return cudaErrorNotSupported;
  }
#define FNO_C4_CP(cp)                                                                        \
  case cp:                                                                                   \
    return mode == EPI_FWD   ? launch_pass_c4_cp##cp##_fwd(maps, p, LZ, LT, grid, smem, st)  \
           : mode == EPI_BWD ? launch_pass_c4_cp##cp##_bwd(maps, p, LZ, LT, grid, smem, st)  \
                             : launch_pass_c4_cp##cp##_u(maps, p, LZ, LT, grid, smem, st);
  switch (CP) {
    FNO_C4_CP(4)
    FNO_C4_CP(8)
    FNO_C4_CP(20)
    default: return cudaErrorInvalidValue;
  }
#undef FNO_C4_CP
}

}  // namespace fno
