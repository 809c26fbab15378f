// Pass A (bwd a9/a10 input side): the local index set
// I_1 = {z, t} of the distributed FFT (Eq. DFFT), truncated to the
// retained modes, written straight into the send-ready exchange layout.
//
// Per plane (b, c, x, y) of Z*T reals (contiguous in NCXYZT):
//   phase 1 (z, real input): B[kz'][t] = sum_z v[z][t] w_Z^{-kz' z}, kz' = 0..mz
//            (the negative retained kz are the conjugates, since v is real)
//   phase 2 (t, complex):   V[kz][kt] for kt < mt, kz in K_z, from the DFT of
//            B[kz'] at kt and -kt:  V[kz'][kt] = DFT(B[kz'])[kt],
//            V[-kz'][kt] = conj(DFT(B[kz'])[-kt]).
// This is the real FFT along t of P:144 ("first taking an FFT along time")
// evaluated in the cheaper z-first order (same result by separability).
// Output: kz-owner-ordered slab [d][B][Xl][Yl][C][nkz_d][mt] (complex).
#include "kernels.cuh"
#include "launch.h"

namespace fno {

template <int LZ, int LT, int MODE>
__global__ void __launch_bounds__(256) pass_a_kernel(PassAParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const int ZT = Z * T;
  const int NP = p.NP;
  const int nk = mz + 1;        // kz' = 0..mz
  const int TP = T + 1;         // padded row of B
  float* stage = reinterpret_cast<float*>(smem_raw);                       // NP*Z*T
  float2* Bb = reinterpret_cast<float2*>(stage + ((NP * ZT + 3) & ~3));    // NP*nk*TP
  float2* twZ = Bb + NP * nk * TP;                                         // Z
  float2* twT = twZ + Z;                                                   // T
  short2* dmap = reinterpret_cast<short2*>(twT + T);                       // 2mz: (owner d, local kz)

  const int tid = threadIdx.x, nt = blockDim.x;
  fill_twiddles(twZ, Z, tid, nt);
  fill_twiddles(twT, T, tid, nt);
  for (int j = tid; j < 2 * mz; j += nt) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }

  const long long n_batches = (p.n_planes + NP - 1) / NP;
  for (long long batch = blockIdx.x; batch < n_batches; batch += gridDim.x) {
    const long long plane0 = batch * NP;
    const long long left = p.n_planes - plane0;
    const int np = left < NP ? int(left) : NP;
    __syncthreads();  // previous batch fully consumed; tables visible
    // ---- stage np contiguous planes -------------------------------------
    {
      const long long base = plane0 * ZT;
      const int nel = np * ZT;
      if (MODE == MODE_V || MODE == MODE_DZ_NONE) {
        const float* src = p.in0 + base;
        if ((nel & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          const float4* s4 = reinterpret_cast<const float4*>(src);
          float4* d4 = reinterpret_cast<float4*>(stage);
          for (int i = tid; i < nel / 4; i += nt) d4[i] = __ldcs(s4 + i);
        } else {
          for (int i = tid; i < nel; i += nt) stage[i] = src[i];
        }
      } else {  // dz = dy * gelu'(z_saved)
        const float* dy = p.in0 + base;
        const float* zs = p.in1 + base;
        for (int i = tid; i < nel; i += nt) stage[i] = dy[i] * gelu_prime_f(zs[i]);
      }
    }
    __syncthreads();
    // ---- phase 1: z-DFT of real columns (pencils (plane, t)) --------------
    for (int pid = tid; pid < np * T; pid += nt) {
      const int pl = pid / T, t = pid - pl * T;
      const float* col = stage + pl * ZT + t;
      float2 acc[LZ];
      trunc_fwd<LZ>(acc, Z, p.Qz, 0, twZ, [&](int z) { return make_float2(col[z * T], 0.0f); });
      float2* bo = Bb + (pl * nk) * TP + t;
#pragma unroll
      for (int j = 0; j < LZ; ++j)
        if (j < nk) bo[j * TP] = acc[j];
    }
    __syncthreads();
    // ---- phase 2: t-DFT of complex rows (pencils (plane, kz')) ------------
    for (int pid = tid; pid < np * nk; pid += nt) {
      const int pl = pid / nk, kzp = pid - pl * nk;
      const float2* row = Bb + (pl * nk + kzp) * TP;
      float2 acc[LT];
      trunc_fwd<LT>(acc, T, p.Qt, mt - 1, twT, [&](int t) { return row[t]; });
      // plane -> (b, c, xl, yl)
      const long long plane = plane0 + pl;
      const int yl = int(plane % p.Yl);
      long long r1 = plane / p.Yl;
      const int xl = int(r1 % p.Xl);
      r1 /= p.Xl;
      const int c = int(r1 % p.C);
      const int b = int(r1 / p.C);
      const long long pt = ((long long)(b * p.Xl + xl) * p.Yl + yl) * p.C + c;  // point-channel index in chunk
      if (kzp < mz) {  // kz = +kz' -> retained index jz = kz'
        const short2 dm = dmap[kzp];
        const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
        float2* o = p.out + p.slab.off[dm.x] + (pt * nkz + dm.y) * mt;
#pragma unroll
        for (int i = 0; i < LT; ++i)
          if (i < mt) o[i] = acc[i];
      }
      if (kzp >= 1) {  // kz = -kz' -> retained index jz = 2mz - kz'
        const short2 dm = dmap[2 * mz - kzp];
        const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
        float2* o = p.out + p.slab.off[dm.x] + (pt * nkz + dm.y) * mt;
#pragma unroll
        for (int i = 0; i < LT; ++i) {
          const int kt = (LT - i) % LT;             // residue i holds frequency -kt
          if (kt < mt && (i == 0 || i > LT - mt)) o[kt] = cconj(acc[i]);
        }
      }
    }
  }
}

size_t pass_a_smem(int Z, int T, int mz, int NP) {
  size_t s = (size_t(NP) * Z * T + 3) / 4 * 4 * sizeof(float);
  s += size_t(NP) * (mz + 1) * (T + 1) * sizeof(float2);
  s += size_t(Z + T) * sizeof(float2);
  s += size_t(2 * mz) * sizeof(short2);
  return s;
}

template <int LZ, int LT>
static cudaError_t launch_a(const PassAParams& p, int mode, int grid, size_t smem, cudaStream_t st) {
  void (*k)(PassAParams) = mode == MODE_V ? pass_a_kernel<LZ, LT, MODE_V>
                         : mode == MODE_DZ_GELU ? pass_a_kernel<LZ, LT, MODE_DZ_GELU>
                                                : pass_a_kernel<LZ, LT, MODE_DZ_NONE>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, 256, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_pass_a(const PassAParams& p, int LZ, int LT, int mode, int grid, size_t smem, cudaStream_t st) {
#define FNO_A_CASE(a, b) \
  if (LZ == a && LT == b) return launch_a<a, b>(p, mode, grid, smem, st);
  FNO_AC_PAIRS(FNO_A_CASE)
#undef FNO_A_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fno
