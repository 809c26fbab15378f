// Pass A, warp-per-plane form (bwd a9/a10 input side): the
// local index set I_1 = {z, t} of the distributed FFT (Eq. DFFT),
// truncated to the retained modes and written straight into the send-ready
// exchange slab.  Same arithmetic as pass_a.cu; different mapping, for T <= 32:
//
//   * a warp owns PPW = 32 / T planes (b, c, x, y); lane (pw, t) reads column t
//     of its plane straight from HBM (a warp-wide load per z is one contiguous
//     row run: coalesced, no staging), optionally forms dz = dy * GELU'(z) and
//     writes it back (bwd), and evaluates the real z-DFT of the column for
//     kz' = 0..mz (residue decomposition, register FFT codelets);
//   * the kz' x t block goes through a per-warp shared-memory tile to the
//     t-DFT (items (pw, kz')), which writes kt < mt for +kz' and the
//     conjugates for -kz' (v real) into the slab.
// No CTA-wide barrier after the tables: warps run independently, so memory
// latency is hidden by the other warps' transforms.
#include <algorithm>

#include "kernels.cuh"
#include "launch.h"

namespace fno {

static constexpr int A2W = 4;            // warps per CTA
static constexpr int A2T = 32 * A2W;

template <int LZ, int LT, int MODE>
__global__ void __launch_bounds__(A2T) pass_a2_kernel(PassAParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const int nk = mz + 1;
  const int TP = T + 1;
  const int PPW = 32 / T;                 // planes per warp
  const int ZT = Z * T;
  float2* twZ = reinterpret_cast<float2*>(smem_raw);
  float2* twT = twZ + Z;
  short2* dmap = reinterpret_cast<short2*>(twT + T);
  float2* Bw = reinterpret_cast<float2*>(smem_raw + ((size_t(Z + T) * sizeof(float2) + 2 * mz * sizeof(short2) + 15) & ~size_t(15)));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float2* Bb = Bw + size_t(warp) * PPW * nk * TP;   // this warp's [pw][kz'][t] tile

  fill_combine_table(twZ, LZ, p.Qz, Z, 0, -1, tid, A2T);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, -1, tid, A2T);
  for (int j = tid; j < 2 * mz; j += A2T) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  __syncthreads();

  const int pw = lane / T, t = lane - pw * T;
  const bool active = pw < PPW;
  const long long n_groups = (p.n_planes + PPW - 1) / PPW;
  for (long long g = (long long)blockIdx.x * A2W + warp; g < n_groups; g += (long long)gridDim.x * A2W) {
    const long long plane = g * PPW + pw;
    const bool live = active && plane < p.n_planes;
    // ---- phase 1: z-DFT of the real column t, kz' = 0..mz -----------------
    if (live) {
      const long long base = plane * ZT + t;
      const float* __restrict__ in0 = p.in0 + base;
      const float* __restrict__ in1 = p.in1 + base;   // z_saved (MODE_DZ_GELU)
      float* __restrict__ dzo = p.dz_out + base;
      const int Qz = p.Qz;
      // residue classes z = q + Qz s; the loads of class q + 1 are issued
      // before class q is transformed (software prefetch in registers)
      float cur0[LZ], cur1[LZ];
#pragma unroll
      for (int s = 0; s < LZ; ++s) {
        cur0[s] = __ldcs(in0 + (Qz * s) * T);
        if (MODE == MODE_DZ_GELU) cur1[s] = __ldcs(in1 + (Qz * s) * T);
      }
      float2 acc[LZ];
      for (int q = 0; q < Qz; ++q) {
        float nxt0[LZ], nxt1[LZ];
        if (q + 1 < Qz) {
#pragma unroll
          for (int s = 0; s < LZ; ++s) {
            nxt0[s] = __ldcs(in0 + (q + 1 + Qz * s) * T);
            if (MODE == MODE_DZ_GELU) nxt1[s] = __ldcs(in1 + (q + 1 + Qz * s) * T);
          }
        }
        float2 x[LZ];
#pragma unroll
        for (int s = 0; s < LZ; ++s) {
          float d = cur0[s];
          if (MODE == MODE_DZ_GELU) {   // dz = dy * GELU'(z), kept for pass C
            d *= gelu_prime_f(cur1[s]);
            __stcs(dzo + (q + Qz * s) * T, d);
          }
          x[s] = make_float2(d, 0.0f);
        }
        fft<LZ, -1>(x);
        if (q == 0) {
#pragma unroll
          for (int j = 0; j < LZ; ++j) acc[j] = x[j];
        } else {
          const float2* tw = twZ + q * LZ;
#pragma unroll
          for (int j = 0; j < LZ; ++j)
            if (j < nk) acc[j] = cfma(x[j], tw[j], acc[j]);
        }
#pragma unroll
        for (int s = 0; s < LZ; ++s) {
          cur0[s] = nxt0[s];
          if (MODE == MODE_DZ_GELU) cur1[s] = nxt1[s];
        }
      }
      float2* bo = Bb + (pw * nk) * TP + t;
#pragma unroll
      for (int j = 0; j < LZ; ++j)
        if (j < nk) bo[j * TP] = acc[j];
    }
    __syncwarp();
    // ---- phase 2: t-DFT of the complex rows, items (pw, kz') ----------------
    for (int it = lane; it < PPW * nk; it += 32) {
      const int q = it / nk, kzp = it - q * nk;
      const long long pl = g * PPW + q;
      if (pl >= p.n_planes) continue;
      const float2* row = Bb + (q * nk + kzp) * TP;
      float2 acc[LT];
      trunc_fwd<LT>(acc, p.Qt, twT, [&](int tt) { return row[tt]; }, mt, mt - 1);
      const int yl = int(pl % p.Yl);
      long long r1 = pl / p.Yl;
      const int xl = int(r1 % p.Xl);
      r1 /= p.Xl;
      const int c = int(r1 % p.C);
      const int b = int(r1 / p.C);
      const long long pt = ((long long)(b * p.Xl + xl) * p.Yl + yl) * p.C + c;
      if (kzp < mz) {   // kz = +kz' -> retained index jz = kz'
        const short2 dm = dmap[kzp];
        const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
        float2* o = p.out + p.slab.off[dm.x] + (pt * nkz + dm.y) * mt;
#pragma unroll
        for (int i = 0; i < LT; ++i)
          if (i < mt) o[i] = acc[i];
      }
      if (kzp >= 1) {   // kz = -kz' -> retained index jz = 2mz - kz'
        const short2 dm = dmap[2 * mz - kzp];
        const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
        float2* o = p.out + p.slab.off[dm.x] + (pt * nkz + dm.y) * mt;
#pragma unroll
        for (int i = 0; i < LT; ++i) {
          const int kt = (LT - i) % LT;   // residue i holds frequency -kt
          if (kt < mt && (i == 0 || i > LT - mt)) o[kt] = cconj(acc[i]);
        }
      }
    }
    __syncwarp();   // Bb reused by the next group
  }
}

bool pass_a2_config(int Z, int T, int mz, size_t* smem) {
  if (T > 32) return false;
  const int PPW = 32 / T;
  const size_t head = (size_t(Z + T) * sizeof(float2) + 2 * mz * sizeof(short2) + 15) & ~size_t(15);
  *smem = head + size_t(A2W) * PPW * (mz + 1) * (T + 1) * sizeof(float2);
  return *smem <= 48 * 1024;
}

int pass_a2_grid(long long n_planes, int T, int num_sms) {
  const long long groups = (n_planes + (32 / T) - 1) / (32 / T);
  const long long ctas = (groups + A2W - 1) / A2W;
  return int(std::min<long long>(ctas, (long long)num_sms * 6));
}

template <int LZ, int LT>
static cudaError_t launch_a2(const PassAParams& p, int mode, int grid, size_t smem, cudaStream_t st) {
  void (*k)(PassAParams) = mode == MODE_V ? pass_a2_kernel<LZ, LT, MODE_V>
                         : mode == MODE_DZ_GELU ? pass_a2_kernel<LZ, LT, MODE_DZ_GELU>
                                                : pass_a2_kernel<LZ, LT, MODE_DZ_NONE>;
  k<<<grid, A2T, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_pass_a2(const PassAParams& p, int LZ, int LT, int mode, int grid, size_t smem, cudaStream_t st) {
#define FNO_A2_CASE(a, b) \
  if (LZ == a && LT == b) return launch_a2<a, b>(p, mode, grid, smem, st);
  FNO_AC_PAIRS(FNO_A2_CASE)
#undef FNO_A2_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fno
