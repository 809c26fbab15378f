// Host side of the channel-width-specialised pass C (kernel: pass_c2.cuh;
// one translation unit per padded width CP so the instantiations compile in
// parallel): tile configuration and the TMA tensor maps of the tile inputs.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "pass_c2.cuh"

namespace fno {

bool pass_c2_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* CPo, int* TCH, int* VW, size_t* smem,
                    int* NX) {
  if (mode == EPI_U) return false;
  const int CP = (C + 3) & ~3;
  if (CP > 20) return false;
  // t chunk: a multiple of 4 with LZ * TCH <= 128 (one 1x1 quad item per
  // thread) and at most T rounded up to 4.  Preference: three CTAs per SM with
  // one X buffer (forward: the epilogue hides the next tile's load), two CTAs
  // with two buffers, then the largest that fits one CTA
  int tmax = (T + 3) & ~3;
  if (tmax * LZ > C2T) tmax = (C2T / LZ) & ~3;
#ifdef FNO_DEV_KNOBS   // development builds only (scripts/variant_lib.sh): force the X buffer count
  const char* nxe = std::getenv("FNO_PASS_C_NX");
  const int force_nx = nxe ? std::atoi(nxe) : 0;
#else
  const int force_nx = 0;
#endif
  // full: only the largest t chunk (a whole 128-point tile).  The backward keeps
  // two buffers while two CTAs per SM fit at full tiles, else takes one buffer at
  // full tiles (c4: 3.49 vs 5.03 ms/launch with two buffers at half tiles)
  struct Opt { size_t budget; int nx; bool full; };
  const Opt opts[] = {{75 * 1024, 1, false}, {113 * 1024, 2, true}, {113 * 1024, 1, true}, {113 * 1024, 2, false},
                      {227 * 1024, 2, false}, {227 * 1024, 1, false}};
  for (const Opt& o : opts) {
    if (force_nx && o.nx != force_nx) continue;
    if (o.nx == 1 && mode != EPI_FWD && !force_nx && !o.full) continue;   // bwd: one buffer only at full tiles
    for (int cand = tmax; cand >= 4 && (!o.full || cand == tmax); cand -= 4) {
      const size_t s = c2_layout(CP, C, Z, T, mz, mt, LZ, cand, mode, o.nx).total;
      if (s <= o.budget) {
        *CPo = CP;
        *TCH = cand;
        *VW = (T % 4 == 0) ? 4 : (T % 2 == 0) ? 2 : 1;
        *smem = s;
        *NX = o.nx;
        return true;
      }
    }
  }
  return false;
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
}  // namespace

// (T, Qz, LZ, Xl*Yl, B*C) view of an NCXYZT field; box [C][1][LZ][1][TCH]
// rows per TMA row group: G consecutive z rows of T floats make one row of the
// view, so that every global stride is a multiple of 16 bytes even when
// T % 4 != 0 (element (z = rz + Qz s, t) with rz = G a + r sits at inner
// coordinate r T + t, group a, s).  A box must also start 16-byte aligned, so
// the t chunks of a z row with (r T) % 4 = sh start sh points early: chunk tc
// covers t in [tc TCH - sh, (tc + 1) TCH - sh), and the ceil(T / TCH) chunks
// must still cover [0, T).  0: no TMA view exists (Qz % G != 0, chunks would
// not cover, or a stride / the base is not 16-byte aligned).
int c2_tile_group(const PassCParams& p, int LZ, const float* base) {
  const int G = (p.T % 4 == 0) ? 1 : (p.T % 2 == 0 ? 2 : 4);
  const long long ZT = (long long)p.Z * p.T;
  if (p.Qz % G != 0 || p.TCH % 4 != 0 || p.TCH > 256 || LZ > 256 || p.C > 256) return 0;
  if ((ZT * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return 0;
  const int nch = (p.T + p.TCH - 1) / p.TCH;
  for (int r = 0; r < G; ++r)
    if (((r * p.T) & 3) + p.T > nch * p.TCH) return 0;
  return G;
}

bool c2_encode_tile_map(CUtensorMap* m, const float* base, const PassCParams& p, int LZ) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return false;
  const int G = c2_tile_group(p, LZ, base);
  if (G == 0) return false;
  const cuuint64_t dims[5] = {cuuint64_t(G) * p.T, cuuint64_t(p.Qz / G), cuuint64_t(LZ), cuuint64_t(p.Xl) * p.Yl,
                              cuuint64_t(p.B) * p.C};
  const cuuint64_t ZT = cuuint64_t(p.Z) * p.T;
  const cuuint64_t strides[4] = {cuuint64_t(G) * p.T * 4, cuuint64_t(p.Qz) * p.T * 4, ZT * 4,
                                 cuuint64_t(p.Xl) * p.Yl * ZT * 4};
  const cuuint32_t box[5] = {cuuint32_t(p.TCH), 1, cuuint32_t(LZ), 1, cuuint32_t(p.C)};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t launch_pass_c2(const PassCParams& p0, int LZ, int LT, int CP, int mode, int grid, size_t smem,
                           cudaStream_t st) {
  PassCParams p = p0;
  C2Maps maps;
  std::memset(&maps, 0, sizeof maps);
  p.use_tma = 0;
  const float* src0 = mode == EPI_FWD ? p.v : p.dy;
  p.tma_g = c2_tile_group(p, LZ, src0);
  if (p.tma_g > 0 && (mode == EPI_FWD || c2_tile_group(p, LZ, p.v) == p.tma_g)) {
    bool ok = c2_encode_tile_map(&maps.m[0], src0, p, LZ);
    if (ok && mode == EPI_BWD) ok = c2_encode_tile_map(&maps.m[1], p.v, p, LZ);
    p.use_tma = ok ? 1 : 0;
  }
  switch (CP) {
    case 4: return launch_pass_c2_cp4(maps, p, LZ, LT, mode, grid, smem, st);
    case 8: return launch_pass_c2_cp8(maps, p, LZ, LT, mode, grid, smem, st);
    case 12: return launch_pass_c2_cp12(maps, p, LZ, LT, mode, grid, smem, st);
    case 16: return launch_pass_c2_cp16(maps, p, LZ, LT, mode, grid, smem, st);
    case 20: return launch_pass_c2_cp20(maps, p, LZ, LT, mode, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fno
