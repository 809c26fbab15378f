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
//
// Streaming: a persistent CTA processes batches of NP consecutive planes (one
// contiguous run of HBM).  Each batch is fetched by one TMA bulk copy
// (cp.async.bulk, completion on an mbarrier) into one of two stage buffers; the
// copy of batch k+2 is issued as soon as phase 1 of batch k has drained its
// buffer, so HBM stays busy while the CTA transforms.
#include <algorithm>

#include "kernels.cuh"
#include "launch.h"

namespace fno {

static constexpr int AT = 128;   // threads per CTA; several CTAs per SM overlap their phases
static constexpr int AT5 = 160;  // forward, 128 % T != 0: floor(160 / T) planes make one phase-1 round (c3: 150 pencils)

// threads per CTA and resident CTAs per SM (the launch bounds) of a mode's kernel
int pass_a_threads(int mode, int T) { return (mode == MODE_V && 128 % T != 0 && T <= AT5) ? AT5 : AT; }
int pass_a_max_blocks(int mode, int T) { return mode == MODE_V ? (pass_a_threads(mode, T) == AT ? 4 : 3) : 3; }

struct ALayout {
  size_t stage[2], bb, twz, twt, dmap, jbase, jnk, bar, total;
  int NA;
};

// NS stage buffers (2: the batch after next streams in while one is transformed;
// 1: the next batch streams in during phase 2 only)
__host__ __device__ inline ALayout a_layout(int Z, int T, int mz, int NP, int mode, int NS) {
  ALayout L{};
  L.NA = (mode == MODE_DZ_GELU) ? 2 : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 127) & ~size_t(127); return o; };
  const size_t sb = size_t(L.NA) * NP * Z * T * sizeof(float);
  L.stage[0] = take(sb);
  L.stage[1] = NS == 2 ? take(sb) : L.stage[0];
  L.bb = take(size_t(NP) * (mz + 1) * (T + 1) * sizeof(float2));
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  L.jbase = take(size_t(2 * mz) * sizeof(float2*));
  L.jnk = take(size_t(2 * mz) * sizeof(int));
  L.bar = take(2 * sizeof(uint64_t));
  L.total = off;
  return L;
}

// HALF: mz = LZ / 2 (nk = LZ / 2 + 1 at compile time: the unused outputs of
// the z codelet are dead code)
template <int LZ, int LT, int MODE, bool HALF, int NT = AT>
__global__ void __launch_bounds__(NT, MODE == MODE_V ? (NT == AT ? 4 : 3) : 3) pass_a_kernel(PassAParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const int ZT = Z * T;
  const int NP = p.NP;
  const int nk = mz + 1;        // kz' = 0..mz
  const int TP = T + 1;         // padded row of B
  const int NS = p.NS;
  const ALayout L = a_layout(Z, T, mz, NP, MODE, NS);
  constexpr int NA = (MODE == MODE_DZ_GELU) ? 2 : 1;
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  float2** jbase = reinterpret_cast<float2**>(smem_raw + L.jbase);   // retained jz -> owner chunk + jl*mt
  int* jnk = reinterpret_cast<int*>(smem_raw + L.jnk);               // retained jz -> owner's nkz
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long n_batches = (p.n_planes + NP - 1) / NP;
  if ((long long)blockIdx.x >= n_batches) return;

  fill_combine_table(twZ, LZ, p.Qz, Z, 0, -1, tid, nt);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, -1, tid, nt);
  for (int j = tid; j < 2 * mz; j += nt) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
    jbase[j] = p.slab.dst[d] + (long long)(j - p.slab.kz_lo[d]) * mt;
    jnk[j] = p.slab.kz_lo[d + 1] - p.slab.kz_lo[d];
  }
  const bool tma = p.use_tma != 0;
  if (tid == 0 && tma) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // fetch batch index kb into stage buffer sb
  auto issue = [&](long long kb, int sb) {
    const long long plane0 = kb * NP;
    const long long left = p.n_planes - plane0;
    const int np = left < NP ? int(left) : NP;
    float* dst = reinterpret_cast<float*>(smem_raw + L.stage[sb]);
    const long long base = plane0 * ZT;
    const unsigned bytes = unsigned(np) * ZT * sizeof(float);
    if (tma) {
      if (tid == 0) {
        fence_proxy_async();
        mbar_expect_tx(&bar[sb], bytes * NA);
        tma_load_1d(dst, p.in0 + base, bytes, &bar[sb]);
        if (NA == 2) tma_load_1d(dst + NP * ZT, p.in1 + base, bytes, &bar[sb]);
      }
    } else {
      for (int i = tid; i < np * ZT; i += nt) {
        cp_async4(dst + i, p.in0 + base + i);
        if (NA == 2) cp_async4(dst + NP * ZT + i, p.in1 + base + i);
      }
      cp_commit();
    }
  };

  long long kb = blockIdx.x;
  issue(kb, 0);
  if (NS == 2 && kb + gridDim.x < n_batches) issue(kb + gridDim.x, 1);
  else if (!tma) cp_commit();
  unsigned phase_bits = 0u;   // mbarrier parity of stage b in bit b
  int sb = 0;
  for (; kb < n_batches; kb += gridDim.x) {
    const long long plane0 = kb * NP;
    const long long left = p.n_planes - plane0;
    const int np = left < NP ? int(left) : NP;
    float* stage = reinterpret_cast<float*>(smem_raw + L.stage[sb]);
    if (tma) {
      mbar_wait(&bar[sb], (phase_bits >> sb) & 1u);
      phase_bits ^= 1u << sb;
    } else {
      if (NS == 2) cp_wait<1>();
      else cp_wait<0>();
      __syncthreads();
    }
    if (MODE == MODE_DZ_GELU) {  // dz = dy * gelu'(z_saved), in place; also kept for pass C
      const float* zs = stage + NP * ZT;
      float* dzo = p.dz_out + plane0 * ZT;
      if ((ZT & 3) == 0) {
        float4* s4 = reinterpret_cast<float4*>(stage);
        const float4* z4 = reinterpret_cast<const float4*>(zs);
        float4* o4 = reinterpret_cast<float4*>(dzo);
        for (int i = tid; i < np * ZT / 4; i += nt) {
          float4 d = s4[i];
          const float4 zz = z4[i];
          d.x *= gelu_prime_f(zz.x);
          d.y *= gelu_prime_f(zz.y);
          d.z *= gelu_prime_f(zz.z);
          d.w *= gelu_prime_f(zz.w);
          s4[i] = d;
          __stcs(o4 + i, d);
        }
      } else {
        for (int i = tid; i < np * ZT; i += nt) {
          const float d = stage[i] * gelu_prime_f(zs[i]);
          stage[i] = d;
          dzo[i] = d;
        }
      }
      fence_proxy_async();  // generic writes before the buffer is refilled by TMA
      __syncthreads();
    }
    // ---- phase 1: z-DFT of real columns (pencils (plane, t)) --------------
    for (int pid = tid; pid < np * T; pid += nt) {
      const int pl = pid / T, t = pid - pl * T;
      const float* col = stage + pl * ZT + t;
      float2 acc[LZ];
      constexpr int NKH = LZ / 2 + 1;
      trunc_fwd<LZ>(acc, p.Qz, twZ, [&](int z) { return make_float2(col[z * T], 0.0f); }, HALF ? NKH : nk, 0);
      float2* bo = Bb + (pl * nk) * TP + t;
#pragma unroll
      for (int j = 0; j < LZ; ++j)
        if (j < (HALF ? NKH : nk)) bo[j * TP] = acc[j];
    }
    __syncthreads();
    // stage buffer drained: prefetch the batch after next (NS = 2) or the
    // next batch (NS = 1) into it
    const long long kn = kb + (long long)NS * gridDim.x;
    if (kn < n_batches) issue(kn, sb);
    else if (!tma) cp_commit();
    // ---- phase 2: t-DFT of complex rows (pencils (plane, kz')) ------------
    for (int pid = tid; pid < np * nk; pid += nt) {
      const int pl = pid / nk, kzp = pid - pl * nk;
      const float2* row = Bb + (pl * nk + kzp) * TP;
      float2 acc[LT];
      trunc_fwd<LT>(acc, p.Qt, twT, [&](int t) { return row[t]; }, mt, mt - 1);
      // plane -> (b, c, xl, yl)
      const long long plane = plane0 + pl;
      const int yl = int(plane % p.Yl);
      long long r1 = plane / p.Yl;
      const int xl = int(r1 % p.Xl);
      r1 /= p.Xl;
      const int c = int(r1 % p.C);
      const int b = int(r1 / p.C);
      const long long pt = ((long long)(b * p.Xl + xl) * p.Yl + yl) * p.C + c;  // point-channel index in chunk
      // rows of mt complex: 16-byte pair stores when mt is even (fewer, wider
      // stores -- over NVLink when the peer exchange writes the owners' slabs)
      const bool pairs = (mt & 1) == 0;
      if (kzp < mz) {  // kz = +kz' -> retained index jz = kz'
        float2* o = jbase[kzp] + pt * jnk[kzp] * mt;
        if (pairs) {
#pragma unroll
          for (int i = 0; i < LT; i += 2)
            if (i < mt) *reinterpret_cast<float4*>(o + i) = make_float4(acc[i].x, acc[i].y, acc[i + 1].x, acc[i + 1].y);
        } else {
#pragma unroll
          for (int i = 0; i < LT; ++i)
            if (i < mt) o[i] = acc[i];
        }
      }
      if (kzp >= 1) {  // kz = -kz' -> retained index jz = 2mz - kz'; frequency -kt sits in residue (LT - kt) % LT
        const int jz = 2 * mz - kzp;
        float2* o = jbase[jz] + pt * jnk[jz] * mt;
        if (pairs) {
#pragma unroll
          for (int kt = 0; kt < LT; kt += 2) {
            if (kt < mt) {
              const float2 a0 = cconj(acc[(LT - kt) % LT]), a1 = cconj(acc[(LT - kt - 1) % LT]);
              *reinterpret_cast<float4*>(o + kt) = make_float4(a0.x, a0.y, a1.x, a1.y);
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < LT; ++i) {
            const int kt = (LT - i) % LT;
            if (kt < mt && (i == 0 || i > LT - mt)) o[kt] = cconj(acc[i]);
          }
        }
      }
    }
    __syncthreads();  // Bb reused by the next batch
    if (NS == 2) sb ^= 1;
  }
  if (!tma) cp_wait<0>();
  if (p.peer) {   // slab stores went to peers over NVLink: publish them before the exchange barrier
    __syncthreads();
    if (tid == 0) __threadfence_system();
  }
}

void pass_a_config(int Z, int T, int mz, int mode, int* NP, int* NS, size_t* smem, int* use_tma) {
  // one z-pencil per thread in phase 1: NP = floor(AT / T) planes per batch.  In order
  // of preference (measured at c2 / c4): two stage buffers at three CTAs per SM
  // (3 x (75 + 1 reserved) KB <= 228 KB), one buffer at two or more CTAs per SM,
  // then half the planes per batch at three CTAs per SM (large Z*T planes such
  // as c4's 128 x 32 backward, two input arrays, would otherwise leave one CTA
  // per SM)
  // (backward, two input arrays: floor, np0 T <= 128 pencils = one per thread,
  // e.g. T = 30 -> 4 planes, 120 pencils in one round instead of 150 in two:
  // c3 backward 0.53 -> 0.39 ms; the forward keeps ceil, measured 0.25 vs 0.275 ms)
  // (forward with 128 % T != 0: 160 threads and floor(160 / T) planes, one
  // phase-1 round, three CTAs per SM; c3 0.249 -> 0.242 ms, bench_c3_a160.json)
  const int at = pass_a_threads(mode, T);
  const int np0 = std::max(1, mode == MODE_DZ_GELU || at != AT ? at / T : (AT + T - 1) / T);
  const size_t per3 = 75 * 1024, per2 = 113 * 1024;
  const int cand[4][2] = {{np0, 2}, {np0, 1}, {std::max(1, np0 / 2), 2}, {std::max(1, np0 / 2), 1}};
  const size_t lim[4] = {per3, per2, per3, per3};
  int np = np0, ns = 1;
  ALayout L{};
  bool found = false;
  for (int i = 0; i < 4; ++i) {
    const auto& c = cand[i];
    L = a_layout(Z, T, mz, c[0], mode, c[1]);
    if (L.total <= lim[i]) {
      np = c[0];
      ns = c[1];
      found = true;
      break;
    }
  }
  if (!found) {   // fall back to one buffer, as many planes as fit one CTA
    ns = 1;
    L = a_layout(Z, T, mz, np, mode, ns);
    while (np > 1 && L.total > 200 * 1024) {
      --np;
      L = a_layout(Z, T, mz, np, mode, ns);
    }
  }
  *NP = np;
  *NS = ns;
  *smem = L.total;
  *use_tma = ((size_t(Z) * T) % 4 == 0) ? 1 : 0;
}

template <int LZ, int LT>
static cudaError_t launch_a(const PassAParams& p, int mode, int grid, size_t smem, cudaStream_t st) {
  const bool half = 2 * p.mz == LZ;
  const int nt = pass_a_threads(mode, p.T);
  void (*k)(PassAParams) =
      mode == MODE_V ? (nt == AT5 ? (half ? pass_a_kernel<LZ, LT, MODE_V, true, AT5> : pass_a_kernel<LZ, LT, MODE_V, false, AT5>)
                                  : (half ? pass_a_kernel<LZ, LT, MODE_V, true> : pass_a_kernel<LZ, LT, MODE_V, false>))
      : mode == MODE_DZ_GELU ? (half ? pass_a_kernel<LZ, LT, MODE_DZ_GELU, true> : pass_a_kernel<LZ, LT, MODE_DZ_GELU, false>)
                             : (half ? pass_a_kernel<LZ, LT, MODE_DZ_NONE, true> : pass_a_kernel<LZ, LT, MODE_DZ_NONE, false>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, nt, smem, st>>>(p);
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
