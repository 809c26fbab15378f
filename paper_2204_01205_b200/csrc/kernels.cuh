// Shared device-side building blocks and kernel parameter blocks of libfno.
//
// Truncated DFTs by residue decomposition.  For an axis of length n with a set
// of needed frequencies that maps injectively onto the residues mod L (L | n),
//   forward:  X[k] = sum_{q<Q} w_n^{-k q} FFT_L(x[q + Q s])[k mod L]
//   inverse:  x[r + Q s] = IFFT_L( X~[j] w_n^{+k_j r} )[s]
// with Q = n / L.  Only the retained modes are ever formed (R_phi
// is non-zero only at the low modes), and the FFT_L codelets (fft.cuh) keep
// every inner twiddle a compile-time immediate; only the Q-way combine uses a
// runtime twiddle table held in shared memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#ifdef FNO_MBAR_DEBUG
#include <cstdio>
#endif

#include "fft.cuh"

#define FNO_MAXP 64

// Profiling-only ablation switches (PassCParams::ablate), compiled in only by
// the scripts/ablate*.sh builds (-DFNO_ABLATE_BUILD); in the product library
// every ablation branch folds away at compile time.
#ifdef FNO_ABLATE_BUILD
#define FNO_ABL(p, bit) (((p).ablate & (bit)) != 0)
#else
#define FNO_ABL(p, bit) false
#endif

namespace fno {

// ---------------------------------------------------------------------------
// parameter blocks (passed by value)
// ---------------------------------------------------------------------------

// Exchange buffer ordered by kz owner: chunk d = [B][Xl][Yl][C][nkz_d][mt]
// (written by pass A, read by pass C).
struct KzSlab {
  int P;
  int kz_lo[FNO_MAXP + 1];   // owner d holds retained kz [kz_lo[d], kz_lo[d+1])
  long long off[FNO_MAXP];   // complex-element offset of chunk d
  float2* dst[FNO_MAXP];     // pass A: where owner d's chunk is written: the local send
                             // buffer + off[d], or (peer exchange) this rank's block of
                             // owner d's receive buffer, mapped over NVLink
};

enum { MODE_V = 0, MODE_DZ_GELU = 1, MODE_DZ_NONE = 2 };  // pass A input
enum { EPI_U = 0, EPI_FWD = 1, EPI_BWD = 2 };            // pass C epilogue

struct PassAParams {
  const float* in0;     // v (MODE_V) or dy
  const float* in1;     // z_saved (MODE_DZ_GELU)
  float2* out;          // kz-ordered slab
  long long n_planes;   // B*C*Xl*Yl
  int Z, T, mz, mt, Qz, Qt, NP;
  int NS;               // pass A stage buffers (1 or 2)
  int C, Xl, Yl;
  int use_tma;          // 1: TMA bulk copies of plane batches (Z*T % 4 == 0)
  float* dz_out;        // MODE_DZ_GELU: dz = dy * gelu'(z) is also written here (read by pass C)
  int peer;             // 1: slab stores go straight to the peers (then a system fence per CTA)
  KzSlab slab;
};

struct PassCParams {
  const float2* in;     // kz-ordered slab (after exchange 2)
  const float* v;       // EPI_FWD: v; EPI_BWD: v (for dW)
  const float* dy;      // EPI_BWD: dz (= dy * sigma'(z), formed by pass A)
  const float* zs;      // unused
  const float* W;       // [C][C] (C_out, C_in)
  const float* bias;    // nullable
  float* out;           // u / y / dv
  float* zsave;         // EPI_FWD, nullable
  float* dWpart;        // EPI_BWD: [gridDim.x][C*C + C] per-CTA partial dW, db
  long long n_cols;     // B*Xl*Yl
  int B, C, Xl, Yl, Z, T, mz, mt, Qz, Qt;
  int TCH, VW;          // t-chunk of a tile, cp.async vector width (floats)
  int use_tma;          // pass_c2/c3: tile inputs by TMA tensor maps (c2_tile_group > 0)
  int tma_g;            // z rows per TMA row group (1: T % 4 == 0; 2: T % 4 == 2; 4: T odd)
  int NX;               // pass_c2: X tile buffers (1 or 2)
  unsigned long long* prof;   // development builds (FNO_C4_PROFILE): pass_c4 role timers, [grid][16]
  int ablate;           // profiling only (FNO_ABLATE): bit 0 skip phase 2, bit 1 skip 1x1, bit 2 skip stores, bit 3 skip dW, bit 4 skip phase 1
  int act_gelu;         // 1: sigma = GELU, 0: identity
  int w_t;              // EPI_FWD kernels: contract with W^T (the dv = W^T dz leg of the split backward)
  float inv_n;          // 1 / (X Y Z T)
  KzSlab slab;
};

// Pass B pencil kernels (x/y transforms on the kz-block after exchange 1).
// Exchange buffer ordered by x/y source: chunk s = [B][Xl][Yl][C][nkz][mt].
struct PassBParams {
  const float2* in;
  float2* out;
  int B, C, X, Y, Xl, Yl, py, nkz, mt, mx, my, Q;
  long long chunk;      // B*Xl*Yl*C*nkz*mt
  int P;                // ranks
  int peer;             // 1: y-inverse stores go straight to the peers (then a system fence per CTA)
  float2* dst[FNO_MAXP];  // y-inverse: base of destination rank d's chunk (local send buffer
                          // + d*chunk, or this rank's block of d's receive buffer over NVLink)
};

struct MixParams {
  const float2* vhat;   // [B][C][M]
  const float2* R;      // [C][C][M]
  const float2* ghat;   // bwd: [B][C][M] = F dz
  float2* what;         // fwd: [B][C][M] mixed; bwd: [B][C][M] = R^H G^
  float2* dR;           // bwd, nullable
  long long M;          // 4 mx my nkz mt
  int B, C, mt, T;
  int accumulate;
  float inv_n;
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// Ampere-style cp.async (LDGSTS): any 4/8/16-byte aligned element
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// TMA bulk copy (cp.async.bulk, UBLKCP) global -> shared, completion counted in
// bytes on an mbarrier (16-byte aligned addresses, size multiple of 16)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "r"(10000000u)
      : "memory");
  return ok != 0;
}
// bounded wait: a barrier that never completes (a malformed async copy or MMA,
// a protocol bug) traps the kernel after ~4 s instead of hanging the GPU.  Each
// try_wait may suspend the warp in hardware (time hint 10 ms) until the phase
// completes, so waiting warps do not spin on the issue slots the working
// warps need; the deadline is checked on the global nanosecond timer.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  if (mbar_test(bar, phase)) return;
  unsigned n = 0;
  unsigned long long t0 = 0;
#ifdef FNO_MBAR_SUSPEND
  while (!mbar_try_wait(bar, phase)) {
#else
  // plain polling: the suspend-hint form (NANOSLEEP.SYNCS) was measured to
  // add wake-up latency to every producer -> consumer hand-off
  while (!mbar_test(bar, phase)) {
#endif
    if ((++n & 1023u) == 0) {   // the deadline is checked rarely: the timer read is not free
      const unsigned long long t = global_ns();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) {
#ifdef FNO_MBAR_DEBUG   // development builds: report the stuck barrier instead of trapping
        printf("mbar timeout: block %d thread %d bar smem+%u parity %u\n", blockIdx.x, threadIdx.x,
               smem_u32(bar), phase);
        return;
#else
        __trap();
#endif
      }
    }
  }
}

// w[j] = exp(-2 pi i j / n), j < n, computed in double and rounded once.
__device__ __forceinline__ void fill_twiddles(float2* w, int n, int tid, int nthreads) {
  for (int j = tid; j < n; j += nthreads) {
    double s, c;
    sincospi(-2.0 * double(j) / double(n), &s, &c);
    w[j] = make_float2(float(c), float(s));
  }
}

// frequency (mod n) represented by residue j of an L-point transform when the
// needed frequencies are {0..L-1-mneg} ∪ {-mneg..-1}
__device__ __forceinline__ int kmod_of(int j, int L, int n, int mneg) {
  return (j >= L - mneg) ? (n - L + j) : j;
}

// Standard normal CDF Phi(z) from the Abramowitz-Stegun 7.1.26 form of erfc
// (|error| <= 1.5e-7 in erf; measured max |Phi error| 2.4e-7, |GELU error|
// 3.1e-7, |GELU' error| 2.4e-7 over [-20, 20]), which shares exp(-z^2/2) with
// the density: one MUFU.EX2 and one MUFU.RCP instead of erff + expf.
__device__ __forceinline__ float rcp_approx_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx_ftz(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float normal_cdf_pdf(float z, float* pdf) {
  const float x = fabsf(z) * 0.70710678118654752440f;
  const float t = rcp_approx_ftz(fmaf(0.3275911f, x, 1.0f));   // argument >= 1: no denormal path
  // 0.5 * t * (a1 + t (a2 + t (a3 + t (a4 + t a5)))), the 1/2 folded into the coefficients
  float poly = fmaf(t, 0.5307027145f, -0.7265760135f);
  poly = fmaf(t, poly, 0.7107068705f);
  poly = fmaf(t, poly, -0.142248368f);
  poly = fmaf(t, poly, 0.127414796f);
  poly *= t;
  const float e = ex2_approx_ftz((z * z) * -0.72134752044448170368f);   // exp(-z^2 / 2)
  const float h = poly * e;                     // Phi(-|z|)
  *pdf = 0.39894228040143267794f * e;
  return z >= 0.f ? 1.0f - h : h;
}
// sigma = GELU(z) = z Phi(z) (exact-erf form, reading Q6) and its derivative.
// Forward: Phi(z) = 1 / (1 + 2^(z P(min(z^2, 30.25)))) with a degree-6 P fitted
// by scripts/fit_gelu.py (max |GELU error| 8.7e-7 in fp32 over [-10, 10],
// relative 6.5e-7 where |GELU| > 0.05 -- as accurate as the A&S form, in 12
// instructions instead of 17: one EX2, one RCP, no select).
__device__ __forceinline__ float gelu_f(float z) {
  const float u = fminf(z * z, 30.25f);
  float q = fmaf(u, -4.677764398053341e-09f, 3.6614977716453723e-07f);
  q = fmaf(u, q, -1.1269662536506075e-05f);
  q = fmaf(u, q, 0.00015897156845312566f);
  q = fmaf(u, q, 9.451490041101351e-05f);
  q = fmaf(u, q, -0.10483447462320328f);
  q = fmaf(u, q, -2.3022098541259766f);
  return z * rcp_approx_ftz(1.0f + ex2_approx_ftz(z * q));
}
__device__ __forceinline__ float gelu_prime_f(float z) {
  float pdf;
  const float cdf = normal_cdf_pdf(z, &pdf);
  return fmaf(z, pdf, cdf);
}

// Q-way combine twiddles of a truncated DFT, one row per residue class:
//   tab[q*L + j] = exp(sign * 2 pi i * kmod_j * q / n),  q < Q, j < L
// (n = Q*L entries).  Computed once per CTA in double, rounded once.
__device__ __forceinline__ void fill_combine_table(float2* tab, int L, int Q, int n, int mneg, int sign, int tid,
                                                   int nthreads) {
  for (int e = tid; e < L * Q; e += nthreads) {
    const int q = e / L, j = e - q * L;
    const long long k = kmod_of(j, L, n, mneg);
    const long long r = (k * q) % n;
    double sn, cs;
    sincospi(2.0 * double(sign) * double(r) / double(n), &sn, &cs);
    tab[e] = make_float2(float(cs), float(sn));
  }
}

// forward truncated DFT of one pencil: acc[j] for every residue j (see header).
// ctab: combine table with sign -1 (fill_combine_table(..., -1, ...)).
// Only residues j < jpos or j >= L - jneg are combined (the others are never
// stored by the callers).
template <int L, class Load>
__device__ __forceinline__ void trunc_fwd(float2 (&acc)[L], int Q, const float2* __restrict__ ctab, Load load,
                                          int jpos = L, int jneg = 0) {
  {
    float2 x[L];
#pragma unroll
    for (int s = 0; s < L; ++s) x[s] = load(Q * s);
    fft<L, -1>(x);
#pragma unroll
    for (int j = 0; j < L; ++j) acc[j] = x[j];
  }
  for (int q = 1; q < Q; ++q) {
    float2 x[L];
#pragma unroll
    for (int s = 0; s < L; ++s) x[s] = load(q + Q * s);
    fft<L, -1>(x);
    const float2* tw = ctab + q * L;
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (j < jpos || j >= L - jneg) acc[j] = cfma(x[j], tw[j], acc[j]);
  }
}

// inverse truncated DFT for residue class r: y[s] = x[r + Q s].
// ctab: combine table with sign +1.
template <int L>
__device__ __forceinline__ void trunc_inv(float2 (&y)[L], const float2 (&e)[L], int r, const float2* __restrict__ ctab) {
  if (r == 0) {
#pragma unroll
    for (int j = 0; j < L; ++j) y[j] = e[j];
  } else {
    const float2* tw = ctab + r * L;
#pragma unroll
    for (int j = 0; j < L; ++j) y[j] = cmul(e[j], tw[j]);
  }
  fft<L, +1>(y);
}

}  // namespace fno
