// dW / db of the layer backward as one streaming contraction over the local box
// (the 1x1 of Eq. dist_block, and the adjoint of
// W's and b's broadcast over the points):
//   dW[o][i] = sum_b sum_n dz[b][o][n] v[b][i][n],   db[o] = sum_b sum_n dz[b][o][n]
// n runs over the Xl Yl Z T points of one channel (NCXYZT: contiguous per
// (b, c)).  Used by the split backward (pass C family 5, api.cu): dv comes from
// the forward pass C kernel run with W^T and no bias / activation, and this
// kernel forms dW and db from dz and v, so no pass C kernel carries the
// C x C dW register block (the FFMA pass_c2 backward: 255 registers, 8 warps
// per SM).
//
// HBM-bound by design: 8 B per point-channel read (dz, v), C FMA per
// point-channel.  One CTA per SM, 256 threads; tiles of DWP points x C
// channels of each input arrive by one 2-D TMA each (tensor map: rows (b, c)
// of N floats, box [C][DWP], the tail tile zero-filled out of bounds) into a
// DWNS-stage ring; thread (block bk, quad q) accumulates a DB x DB
// block of dW (DB = CP / 2, the 2 x 2 blocks of the padded C x C) over its
// 4-point quad of every tile.  Per-CTA partials in a fixed order, then the
// caller's fixed-order row sum (launch_rowsum): deterministic.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "kernels.cuh"
#include "launch.h"

namespace fno {

constexpr int DWT = 256;   // threads: 4 dW blocks x 64 quads
constexpr int DWP = 256;   // points per tile (64 quads)
constexpr int DWNS = 5;    // TMA ring stages (5 x 40 KB at C = 20)

struct DwMaps {
  CUtensorMap m[2];   // dz, v: (N, B C) views, box [C][DWP]
};

template <int CP>
__global__ void __launch_bounds__(DWT, 1) dw_partial_kernel(const __grid_constant__ DwMaps maps, const DwParams p) {
  constexpr int DB = CP / 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw);   // [DWNS][2][CP][DWP]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + size_t(DWNS) * 2 * CP * DWP * sizeof(float));
  float* red = reinterpret_cast<float*>(full + DWNS);   // [8 warps][DB * DB + DB]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = p.C;
  const long long N = p.N;
  const long long ntb = (N + DWP - 1) / DWP;   // tiles per batch
  const long long ntiles = (long long)p.B * ntb;
  const bool bulk = p.bulk != 0;

  // padded channel rows are never written by the copies: zero them once
  for (int e = tid; e < DWNS * 2 * (CP - C) * DWP; e += DWT) {
    const int s = e / (2 * (CP - C) * DWP), r = e - s * 2 * (CP - C) * DWP;
    const int a = r / ((CP - C) * DWP), rr = r - a * (CP - C) * DWP;
    ring[((s * 2 + a) * CP + C) * DWP + rr] = 0.f;
  }
  if (tid == 0) {
    for (int s = 0; s < DWNS; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  fence_proxy_async();
  __syncthreads();

  auto tile_of = [&](long long t, int* b, long long* n0) {
    *b = int(t / ntb);
    *n0 = (t - (long long)*b * ntb) * DWP;
  };
  // tile t into stage s: one 2-D TMA per input (thread 0); out-of-bounds
  // points of the tail tile arrive as zeros and still count in the box bytes
  auto issue = [&](long long t, int s) {
    int b;
    long long n0;
    tile_of(t, &b, &n0);
    mbar_expect_tx(&full[s], 2u * unsigned(C) * DWP * 4u);
#pragma unroll
    for (int a = 0; a < 2; ++a)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
              smem_u32(ring + (s * 2 + a) * CP * DWP)),
          "l"(&maps.m[a]), "r"(int(n0)), "r"(b * C), "r"(smem_u32(&full[s]))
          : "memory");
  };

  const int bk = tid >> 6, q = tid & 63;   // dW block (o-half ob, i-half ib), quad
  const int ob = bk >> 1, ib = bk & 1;
  float acc[DB][DB], dba[DB];
#pragma unroll
  for (int j = 0; j < DB; ++j) {
    dba[j] = 0.f;
#pragma unroll
    for (int i = 0; i < DB; ++i) acc[j][i] = 0.f;
  }

  long long t = blockIdx.x;
  if (bulk && tid == 0)
    for (int s = 0; s < DWNS; ++s)
      if (t + (long long)s * gridDim.x < ntiles) issue(t + (long long)s * gridDim.x, s);
  unsigned phases = 0u;
  for (int k = 0; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % DWNS;
    int b;
    long long n0;
    tile_of(t, &b, &n0);
    const int np = int((N - n0 < DWP ? N - n0 : (long long)DWP));
    float* st = ring + s * 2 * CP * DWP;
    if (bulk) {
      mbar_wait(&full[s], (phases >> s) & 1u);
      phases ^= 1u << s;
    } else {   // unaligned rows: plain loads, zeros past the last point of a partial quad
      for (int e = tid; e < 2 * C * DWP; e += DWT) {
        const int a = e / (C * DWP), r = e - a * C * DWP;
        const int c = r / DWP, n = r - c * DWP;
        const float* src = (a == 0 ? p.dz : p.v) + ((long long)b * C + c) * N + n0;
        st[(a * CP + c) * DWP + n] = n < np ? __ldg(src + n) : 0.f;
      }
      __syncthreads();
    }
    if (4 * q < np) {
      const float* Dz = st + (ob * DB) * DWP + 4 * q;
      const float* V = st + (CP + ib * DB) * DWP + 4 * q;
      float4 d4[DB];
#pragma unroll
      for (int j = 0; j < DB; ++j) d4[j] = *reinterpret_cast<const float4*>(Dz + j * DWP);
      if (ib == 0) {
#pragma unroll
        for (int j = 0; j < DB; ++j) dba[j] += (d4[j].x + d4[j].y) + (d4[j].z + d4[j].w);
      }
#pragma unroll
      for (int i = 0; i < DB; ++i) {
        const float4 v4 = *reinterpret_cast<const float4*>(V + i * DWP);
#pragma unroll
        for (int j = 0; j < DB; ++j) {
          float a = acc[j][i];
          a = fmaf(d4[j].x, v4.x, a);
          a = fmaf(d4[j].y, v4.y, a);
          a = fmaf(d4[j].z, v4.z, a);
          a = fmaf(d4[j].w, v4.w, a);
          acc[j][i] = a;
        }
      }
    }
    __syncthreads();   // stage s consumed by every thread
    if (bulk && tid == 0 && t + (long long)DWNS * gridDim.x < ntiles) issue(t + (long long)DWNS * gridDim.x, s);
  }

  // fixed-order reduction: lanes (butterfly), then the two warps of a block
  constexpr int RL = DB * DB + DB;
#pragma unroll
  for (int j = 0; j < DB; ++j) {
#pragma unroll
    for (int i = 0; i < DB; ++i) {
      float v = acc[j][i];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[warp * RL + j * DB + i] = v;
    }
    float v = dba[j];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp * RL + DB * DB + j] = v;
  }
  __syncthreads();
  float* outp = p.part + (long long)blockIdx.x * (C * C + C);
  for (int e = tid; e < 4 * RL; e += DWT) {
    const int blk = e / RL, r = e - blk * RL;
    const float v = red[(2 * blk) * RL + r] + red[(2 * blk + 1) * RL + r];
    const int o0 = (blk >> 1) * DB, i0 = (blk & 1) * DB;
    if (r < DB * DB) {
      const int o = o0 + r / DB, i = i0 + r % DB;
      if (o < C && i < C) outp[o * C + i] = v;
    } else if ((blk & 1) == 0) {
      const int o = o0 + (r - DB * DB);
      if (o < C) outp[C * C + o] = v;
    }
  }
}

size_t dw_partial_smem(int C) {
  const int CP = (C + 3) & ~3;
  const int DB = CP / 2;
  return size_t(DWNS) * 2 * CP * DWP * sizeof(float) + DWNS * sizeof(uint64_t) + 8 * (DB * DB + DB) * sizeof(float);
}

int dw_partial_grid(int B, long long N, int num_sms) {
  const long long nt = (long long)B * ((N + DWP - 1) / DWP);
  return int(std::max<long long>(1, std::min<long long>(nt, num_sms)));
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode_dw = nullptr;
std::once_flag g_encode_dw_once;

// (N, rows) view of an NCXYZT field, rows = (b, c) of N floats; box [C][DWP]
bool encode_rows(CUtensorMap* m, const float* base, long long N, int rows, int C) {
  std::call_once(g_encode_dw_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_dw = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode_dw || N > (1LL << 31) - 1) return false;
  const cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(N) * 4};
  const cuuint32_t box[2] = {cuuint32_t(DWP), cuuint32_t(C)};
  const cuuint32_t estr[2] = {1, 1};
  return g_encode_dw(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t launch_dw_partial(const DwParams& p0, int grid, cudaStream_t st) {
  DwParams p = p0;
  DwMaps maps;
  std::memset(&maps, 0, sizeof maps);
  // TMA rows need 16-byte strides and bases; otherwise plain loads
  p.bulk = (p.N % 4 == 0 && ((reinterpret_cast<uintptr_t>(p.dz) | reinterpret_cast<uintptr_t>(p.v)) & 15) == 0 &&
            encode_rows(&maps.m[0], p.dz, p.N, p.B * p.C, p.C) && encode_rows(&maps.m[1], p.v, p.N, p.B * p.C, p.C))
               ? 1 : 0;
  const size_t smem = dw_partial_smem(p.C);
  const int CP = (p.C + 3) & ~3;
  void (*k)(DwMaps, DwParams) = nullptr;
  switch (CP) {
    case 4: k = dw_partial_kernel<4>; break;
    case 8: k = dw_partial_kernel<8>; break;
    case 12: k = dw_partial_kernel<12>; break;
    case 16: k = dw_partial_kernel<16>; break;
    case 20: k = dw_partial_kernel<20>; break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, DWT, smem, st>>>(maps, p);
  return cudaGetLastError();
}

}  // namespace fno
