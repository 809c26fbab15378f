// Pass B: the second index set I_2 = {y, x} of the distributed FFT on the
// rank's block of retained kz planes ("then taking an FFT over the last
// n/2 dimensions"; "2D FFT along the x and y dimensions"), the per-mode
// channel mixing with R_phi on the owner, and the adjoint chain
// back (F_dist^T).  SURVEY §8 rows a3 (fwd x,y), a4 (mixing), a5
// (inverse x,y), a11 (dR).
//
// Layouts:  exchange buffer by x/y source / destination:
//             [s][B][Xl][Yl][C][nkz][mt]  (s = ix*py + iy, chunk = B Xl Yl C nkz mt)
//           H  (after the y transform)   [B][nkz][C][X][2my][mt]
//           V^, W^, G^ (mode cube)       [B][C][2mx][2my][nkz][mt]
//           R, dR                        [C][C][2mx][2my][nkz][mt]
#include "kernels.cuh"
#include "launch.h"

namespace fno {

static constexpr int BT = 128;  // threads per CTA of the pencil kernels
// The forward pencils of length >= 30 run at <= 128 registers (four CTAs per
// SM, a few spilled registers): c3 (L = 32) y forward 0.067 -> 0.065, x forward
// 0.032 -> 0.028 ms/launch; at c2 (L = 16) the y forward lost with it (0.027 ->
// 0.031), as did the inverse pencils: they keep the compiler's allocation

// y forward: slab (x/y-source ordered) -> H.  pencil = (b, kzl, c, x, kt)
template <int L>
__global__ void __launch_bounds__(BT, L >= 30 ? 4 : 1) b_yfwd_kernel(PassBParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);               // Y
  long long* ypart = reinterpret_cast<long long*>(tw + p.Y);      // Y
  const int cm = p.C * p.nkz * p.mt;
  for (int y = threadIdx.x; y < p.Y; y += blockDim.x) ypart[y] = (long long)(y / p.Yl) * p.chunk + (long long)(y % p.Yl) * cm;
  fill_combine_table(tw, L, p.Q, p.Y, p.my, -1, threadIdx.x, blockDim.x);
  __syncthreads();
  const long long total = (long long)p.B * p.nkz * p.C * p.X * p.mt;
  const long long pid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pid >= total) return;
  const int kt = int(pid % p.mt);
  long long r = pid / p.mt;
  const int x = int(r % p.X);
  r /= p.X;
  const int c = int(r % p.C);
  r /= p.C;
  const int kzl = int(r % p.nkz);
  const int b = int(r / p.nkz);
  const int sx = x / p.Xl, xl = x - sx * p.Xl;
  const long long xpart = (long long)sx * p.py * p.chunk + ((long long)b * p.Xl + xl) * p.Yl * cm +
                          (long long)(c * p.nkz + kzl) * p.mt + kt;
  const float2* __restrict__ in = p.in;
  float2 acc[L];
  trunc_fwd<L>(acc, p.Q, tw, [&](int y) { return __ldg(in + xpart + ypart[y]); });
  float2* o = p.out + (((long long)(b * p.nkz + kzl) * p.C + c) * p.X + x) * (2 * p.my) * p.mt + kt;
#pragma unroll
  for (int j = 0; j < L; ++j) {
    if (j < p.my) o[(long long)j * p.mt] = acc[j];
    else if (j >= L - p.my) o[(long long)(j - L + 2 * p.my) * p.mt] = acc[j];
  }
}

// x forward: H -> V^.  pencil = (b, kzl, c, jy, kt)
template <int L>
__global__ void __launch_bounds__(BT, L >= 30 ? 4 : 1) b_xfwd_kernel(PassBParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  fill_combine_table(tw, L, p.Q, p.X, p.mx, -1, threadIdx.x, blockDim.x);
  __syncthreads();
  const int my2 = 2 * p.my;
  const long long total = (long long)p.B * p.nkz * p.C * my2 * p.mt;
  const long long pid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pid >= total) return;
  const int kt = int(pid % p.mt);
  long long r = pid / p.mt;
  const int jy = int(r % my2);
  r /= my2;
  const int c = int(r % p.C);
  r /= p.C;
  const int kzl = int(r % p.nkz);
  const int b = int(r / p.nkz);
  const float2* __restrict__ in = p.in + ((long long)(b * p.nkz + kzl) * p.C + c) * p.X * my2 * p.mt + jy * p.mt + kt;
  const long long xs = (long long)my2 * p.mt;
  float2 acc[L];
  trunc_fwd<L>(acc, p.Q, tw, [&](int x) { return __ldg(in + x * xs); });
  const int mx2 = 2 * p.mx;
  float2* o = p.out + ((((long long)b * p.C + c) * mx2) * my2 + jy) * p.nkz * p.mt + (long long)kzl * p.mt + kt;
  const long long js = (long long)my2 * p.nkz * p.mt;
#pragma unroll
  for (int j = 0; j < L; ++j) {
    if (j < p.mx) o[j * js] = acc[j];
    else if (j >= L - p.mx) o[(j - L + mx2) * js] = acc[j];
  }
}

// x inverse: W^ -> H'.  pencil = (b, kzl, o, jy, kt); loops over residue classes
template <int L>
__global__ void __launch_bounds__(BT) b_xinv_kernel(PassBParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);
  fill_combine_table(tw, L, p.Q, p.X, p.mx, +1, threadIdx.x, blockDim.x);
  __syncthreads();
  const int my2 = 2 * p.my, mx2 = 2 * p.mx;
  const long long total = (long long)p.B * p.nkz * p.C * my2 * p.mt;
  const long long pid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pid >= total) return;
  const int kt = int(pid % p.mt);
  long long r = pid / p.mt;
  const int jy = int(r % my2);
  r /= my2;
  const int oc = int(r % p.C);
  r /= p.C;
  const int kzl = int(r % p.nkz);
  const int b = int(r / p.nkz);
  const float2* __restrict__ in = p.in + ((((long long)b * p.C + oc) * mx2) * my2 + jy) * p.nkz * p.mt + (long long)kzl * p.mt + kt;
  const long long js = (long long)my2 * p.nkz * p.mt;
  float2 e[L];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    if (j < p.mx) e[j] = __ldg(in + j * js);
    else if (j >= L - p.mx) e[j] = __ldg(in + (j - L + mx2) * js);
    else e[j] = make_float2(0.f, 0.f);
  }
  float2* o = p.out + ((long long)(b * p.nkz + kzl) * p.C + oc) * p.X * my2 * p.mt + jy * p.mt + kt;
  const long long xs = (long long)my2 * p.mt;
  for (int rc = 0; rc < p.Q; ++rc) {
    float2 y[L];
    trunc_inv<L>(y, e, rc, tw);
#pragma unroll
    for (int s = 0; s < L; ++s) o[(rc + p.Q * s) * xs] = y[s];
  }
}

// y inverse: H' -> slab (x/y-destination ordered).  pencil = (b, kzl, o, x, kt)
// Destination rank (sx, y / Yl) gets its chunk through dst[]: the local send
// buffer for the NCCL exchange, or (peer exchange) its own receive buffer,
// written over NVLink so exchange 2 needs no data movement of its own.
template <int L>
__global__ void __launch_bounds__(BT) b_yinv_kernel(PassBParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2** dtab = reinterpret_cast<float2**>(smem_raw);                       // [P]
  float2* tw = reinterpret_cast<float2*>(smem_raw + FNO_MAXP * sizeof(float2*));
  long long* ypart = reinterpret_cast<long long*>(tw + p.Y);                  // (y % Yl) * cm
  int* ydst = reinterpret_cast<int*>(ypart + p.Y);                            // y / Yl
  const int cm = p.C * p.nkz * p.mt;
  for (int y = threadIdx.x; y < p.Y; y += blockDim.x) {
    ypart[y] = (long long)(y % p.Yl) * cm;
    ydst[y] = y / p.Yl;
  }
  for (int d = threadIdx.x; d < p.P; d += blockDim.x) dtab[d] = p.dst[d];
  fill_combine_table(tw, L, p.Q, p.Y, p.my, +1, threadIdx.x, blockDim.x);
  __syncthreads();
  const int my2 = 2 * p.my;
  const long long total = (long long)p.B * p.nkz * p.C * p.X * p.mt;
  const long long pid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pid < total) {
    // thread order (kt, kzl, oc) fastest, then x: for a fixed (x, y) the outputs
    // of consecutive threads are contiguous in the destination chunk
    // [B][Xl][Yl][C][nkz][mt], so each warp store is one long run -- these are
    // the remote NVLink stores of the peer exchange (the reads of the
    // L2-resident H buffer are the ones that scatter)
    const int kt = int(pid % p.mt);
    long long r = pid / p.mt;
    const int kzl = int(r % p.nkz);
    r /= p.nkz;
    const int oc = int(r % p.C);
    r /= p.C;
    const int x = int(r % p.X);
    const int b = int(r / p.X);
    const float2* __restrict__ in = p.in + (((long long)(b * p.nkz + kzl) * p.C + oc) * p.X + x) * my2 * p.mt + kt;
    float2 e[L];
#pragma unroll
    for (int j = 0; j < L; ++j) {
      if (j < p.my) e[j] = __ldg(in + (long long)j * p.mt);
      else if (j >= L - p.my) e[j] = __ldg(in + (long long)(j - L + my2) * p.mt);
      else e[j] = make_float2(0.f, 0.f);
    }
    const int sx = x / p.Xl, xl = x - sx * p.Xl;
    const long long o = ((long long)b * p.Xl + xl) * p.Yl * cm + (long long)(oc * p.nkz + kzl) * p.mt + kt;
    float2* const* drow = dtab + sx * p.py;
    for (int rc = 0; rc < p.Q; ++rc) {
      float2 y[L];
      trunc_inv<L>(y, e, rc, tw);
#pragma unroll
      for (int s = 0; s < L; ++s) {
        const int yy = rc + p.Q * s;
        drow[ydst[yy]][o + ypart[yy]] = y[s];
      }
    }
  }
  if (p.peer) {   // stores went to peers over NVLink: publish them before the exchange barrier
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
}

// ---------------------------------------------------------------------------
// per-mode channel mixing (R_phi . F v on owned modes)
// thread per retained mode m; complex fp32 accumulation
// ---------------------------------------------------------------------------
// Mixing is a weight stream at batch 1: each R element is read
// once, coalesced across the mode-minor threads.  A thread owns one mode m and
// a chunk of MCH outputs (fwd: o; bwd: i), so the grid has ceil(C / MCH) times
// more warps in flight than a thread-per-mode kernel.
#ifndef FNO_MCH
#define FNO_MCH 2
#endif
constexpr int MCH = FNO_MCH;

// forward mixing: W^[b,o,m] = sum_i V^[b,i,m] R[i,o,m]
template <int CMAX>
__global__ void __launch_bounds__(256) mix_fwd_kernel(MixParams p) {
  const long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= p.M) return;
  const int C = p.C;
  const int o0 = blockIdx.y * MCH;
  for (int b = 0; b < p.B; ++b) {
    float2 vh[CMAX];
#pragma unroll
    for (int i = 0; i < CMAX; ++i)
      if (i < C) vh[i] = __ldg(p.vhat + ((long long)b * C + i) * p.M + m);
#pragma unroll 1
    for (int oo = 0; oo < MCH; ++oo) {
      const int o = o0 + oo;
      if (o >= C) break;
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < CMAX; ++i)
        if (i < C) acc = cfma(vh[i], __ldcs(p.R + ((long long)i * C + o) * p.M + m), acc);
      p.what[((long long)b * C + o) * p.M + m] = acc;
    }
  }
}

// backward mixing: W'^[b,i,m] = sum_o G^[b,o,m] conj(R[i,o,m]);
// dR[i,o,m] (+)= (c(kt)/N) sum_b conj(V^[b,i,m]) G^[b,o,m]
// Batch 1 (every BASELINE config): two rows i per thread, fully unrolled so
// the R loads of the second row issue before the first row's dR stores -- the
// R read stream and the dR write stream are in flight together.
template <int CMAX>
__global__ void __launch_bounds__(256, 2) mix_bwd_kernel(MixParams p) {
  const long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= p.M) return;
  const int C = p.C;
  const int i0 = blockIdx.y * MCH;
  const int kt = int(m % p.mt);
  const float cw = (kt == 0 || ((p.T & 1) == 0 && 2 * kt == p.T)) ? 1.0f : 2.0f;
  const float scale = cw * p.inv_n;
  float2 g[CMAX];
  if (p.B == 1) {
#pragma unroll
    for (int o = 0; o < CMAX; ++o)
      if (o < C) g[o] = __ldg(p.ghat + (long long)o * p.M + m);
    float2 r[MCH][CMAX];
#pragma unroll
    for (int ii = 0; ii < MCH; ++ii) {
      const int i = i0 + ii;
#pragma unroll
      for (int o = 0; o < CMAX; ++o)
        if (o < C && i < C) r[ii][o] = __ldcs(p.R + ((long long)i * C + o) * p.M + m);
    }
#pragma unroll
    for (int ii = 0; ii < MCH; ++ii) {
      const int i = i0 + ii;
      if (i >= C) continue;
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int o = 0; o < CMAX; ++o)
        if (o < C) acc = cfma_conj_a(r[ii][o], g[o], acc);
      p.what[(long long)i * p.M + m] = acc;
      if (p.dR == nullptr) continue;
      const float2 vs = cscale(cconj(__ldg(p.vhat + (long long)i * p.M + m)), scale);
#pragma unroll
      for (int o = 0; o < CMAX; ++o) {
        if (o < C) {
          float2* d = p.dR + ((long long)i * C + o) * p.M + m;
          float2 val = cmul(vs, g[o]);
          if (p.accumulate) val = cadd(*d, val);
          __stcs(d, val);
        }
      }
    }
    return;
  }
  for (int b = 0; b < p.B; ++b) {
#pragma unroll
    for (int o = 0; o < CMAX; ++o)
      if (o < C) g[o] = __ldg(p.ghat + ((long long)b * C + o) * p.M + m);
#pragma unroll 1
    for (int ii = 0; ii < MCH; ++ii) {
      const int i = i0 + ii;
      if (i >= C) break;
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int o = 0; o < CMAX; ++o)
        if (o < C) acc = cfma_conj_a(__ldcs(p.R + ((long long)i * C + o) * p.M + m), g[o], acc);
      p.what[((long long)b * C + i) * p.M + m] = acc;
    }
  }
  if (p.dR == nullptr) return;
  for (int ii = 0; ii < MCH; ++ii) {
    const int i = i0 + ii;
    if (i >= C) break;
    for (int o = 0; o < C; ++o) {
      float2 acc = make_float2(0.f, 0.f);
      for (int b = 0; b < p.B; ++b)
        acc = cfma_conj_a(__ldg(p.vhat + ((long long)b * C + i) * p.M + m), __ldg(p.ghat + ((long long)b * C + o) * p.M + m), acc);
      float2* d = p.dR + ((long long)i * C + o) * p.M + m;
      float2 val = cscale(acc, scale);
      if (p.accumulate) val = cadd(*d, val);
      *d = val;
    }
  }
}

// ---------------------------------------------------------------------------
// batched mixing (B > 1): per mode the (B x C).(C x C) complex
// product, R read ONCE for all B batch rows.  CTA = 32 consecutive modes x 8
// channel rows (one warp per row: 256-byte coalesced R / V^ / G^ rows); the
// batch rows of V^ (fwd) or G^ (bwd) are re-read by the 8 warps through L1.
// Per R element: B complex MACs (fwd), 2B (bwd: W'^ and dR) -- FFMA keeps up
// with the R stream up to B ~ 16 at C = 20; batches beyond
// BMAX run in chunks of BMAX, re-streaming R per chunk.
// ---------------------------------------------------------------------------
template <int BMAX>
__global__ void __launch_bounds__(256) mix_fwd_batched_kernel(MixParams p, int b0, int nb) {
  const long long m = (long long)blockIdx.x * 32 + (threadIdx.x & 31);
  const int o = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (m >= p.M || o >= p.C) return;
  const int C = p.C;
  float2 acc[BMAX];
#pragma unroll
  for (int b = 0; b < BMAX; ++b) acc[b] = make_float2(0.f, 0.f);
  for (int i = 0; i < C; ++i) {
    const float2 r = __ldcs(p.R + ((long long)i * C + o) * p.M + m);
#pragma unroll
    for (int b = 0; b < BMAX; ++b)
      if (b < nb) acc[b] = cfma(__ldg(p.vhat + ((long long)(b0 + b) * C + i) * p.M + m), r, acc[b]);
  }
#pragma unroll
  for (int b = 0; b < BMAX; ++b)
    if (b < nb) p.what[((long long)(b0 + b) * C + o) * p.M + m] = acc[b];
}

// W'^[b,i] = sum_o G^[b,o] conj(R[i,o]);  dR[i,o] (+)= (c/N) sum_b conj(V^[b,i]) G^[b,o]
// (first chunk b0 == 0 writes or accumulates dR, later chunks add)
template <int BMAX>
__global__ void __launch_bounds__(256) mix_bwd_batched_kernel(MixParams p, int b0, int nb) {
  const long long m = (long long)blockIdx.x * 32 + (threadIdx.x & 31);
  const int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (m >= p.M || i >= p.C) return;
  const int C = p.C;
  const int kt = int(m % p.mt);
  const float cw = (kt == 0 || ((p.T & 1) == 0 && 2 * kt == p.T)) ? 1.0f : 2.0f;
  const float scale = cw * p.inv_n;
  float2 vs[BMAX], acc[BMAX];
#pragma unroll
  for (int b = 0; b < BMAX; ++b) {
    acc[b] = make_float2(0.f, 0.f);
    vs[b] = (b < nb && p.dR) ? cconj(__ldg(p.vhat + ((long long)(b0 + b) * C + i) * p.M + m)) : make_float2(0.f, 0.f);
  }
  for (int o = 0; o < C; ++o) {
    const float2 r = __ldcs(p.R + ((long long)i * C + o) * p.M + m);
    float2 d = make_float2(0.f, 0.f);
#pragma unroll
    for (int b = 0; b < BMAX; ++b) {
      if (b < nb) {
        const float2 g = __ldg(p.ghat + ((long long)(b0 + b) * C + o) * p.M + m);
        acc[b] = cfma_conj_a(r, g, acc[b]);
        d = cfma(vs[b], g, d);
      }
    }
    if (p.dR) {
      float2* dp = p.dR + ((long long)i * C + o) * p.M + m;
      float2 val = cscale(d, scale);
      if (p.accumulate || b0 > 0) val = cadd(*dp, val);
      __stcs(dp, val);
    }
  }
#pragma unroll
  for (int b = 0; b < BMAX; ++b)
    if (b < nb) p.what[((long long)(b0 + b) * C + i) * p.M + m] = acc[b];
}

template <int BMAX>
static cudaError_t launch_mix_batched(const MixParams& p, bool bwd, cudaStream_t st) {
  const dim3 grid(unsigned((p.M + 31) / 32), unsigned((p.C + 7) / 8));
  for (int b0 = 0; b0 < p.B; b0 += BMAX) {
    const int nb = p.B - b0 < BMAX ? p.B - b0 : BMAX;
    if (bwd) mix_bwd_batched_kernel<BMAX><<<grid, 256, 0, st>>>(p, b0, nb);
    else mix_fwd_batched_kernel<BMAX><<<grid, 256, 0, st>>>(p, b0, nb);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

static cudaError_t launch_mix_b(const MixParams& p, bool bwd, cudaStream_t st) {
  if (p.M <= 0) return cudaSuccess;
  if (p.B <= 2) return launch_mix_batched<2>(p, bwd, st);
  if (p.B <= 4) return launch_mix_batched<4>(p, bwd, st);
  if (p.B <= 8) return launch_mix_batched<8>(p, bwd, st);
  return launch_mix_batched<16>(p, bwd, st);
}

// deterministic fixed-order column sums; columns [0, split) go to out0,
// [split, len) to out1 (nullable)
// (one warp per column: lane i sums rows i, i + 32, ... in ascending order, then
// a fixed butterfly -- the same order on every run and every rank)
__global__ void rowsum_kernel(const float* __restrict__ parts, int nparts, int len, int split, float* out0, float* out1,
                              int accumulate) {
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (l >= len) return;
  float s = 0.f;
  for (int p = lane; p < nparts; p += 32) s += parts[(long long)p * len + l];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane != 0) return;
  float* o = (l < split) ? out0 + l : (out1 ? out1 + (l - split) : nullptr);
  if (o) *o = accumulate ? *o + s : s;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <class K>
static cudaError_t launch_pencils(K k, const PassBParams& p, long long total, size_t smem, cudaStream_t st) {
  if (total <= 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const long long grid = (total + BT - 1) / BT;
  k<<<unsigned(grid), BT, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_b_yfwd(const PassBParams& p, int L, cudaStream_t st) {
  const long long total = (long long)p.B * p.nkz * p.C * p.X * p.mt;
  const size_t smem = size_t(p.Y) * (sizeof(float2) + sizeof(long long));
#define FNO_CASE(l) if (L == l) return launch_pencils(b_yfwd_kernel<l>, p, total, smem, st);
  FNO_B_SIZES(FNO_CASE)
#undef FNO_CASE
  return cudaErrorInvalidValue;
}
cudaError_t launch_b_xfwd(const PassBParams& p, int L, cudaStream_t st) {
  const long long total = (long long)p.B * p.nkz * p.C * 2 * p.my * p.mt;
  const size_t smem = size_t(p.X) * sizeof(float2);
#define FNO_CASE(l) if (L == l) return launch_pencils(b_xfwd_kernel<l>, p, total, smem, st);
  FNO_B_SIZES(FNO_CASE)
#undef FNO_CASE
  return cudaErrorInvalidValue;
}
cudaError_t launch_b_xinv(const PassBParams& p, int L, cudaStream_t st) {
  const long long total = (long long)p.B * p.nkz * p.C * 2 * p.my * p.mt;
  const size_t smem = size_t(p.X) * sizeof(float2);
#define FNO_CASE(l) if (L == l) return launch_pencils(b_xinv_kernel<l>, p, total, smem, st);
  FNO_B_SIZES(FNO_CASE)
#undef FNO_CASE
  return cudaErrorInvalidValue;
}
cudaError_t launch_b_yinv(const PassBParams& p, int L, cudaStream_t st) {
  const long long total = (long long)p.B * p.nkz * p.C * p.X * p.mt;
  const size_t smem = FNO_MAXP * sizeof(float2*) + size_t(p.Y) * (sizeof(float2) + sizeof(long long) + sizeof(int));
#define FNO_CASE(l) if (L == l) return launch_pencils(b_yinv_kernel<l>, p, total, smem, st);
  FNO_B_SIZES(FNO_CASE)
#undef FNO_CASE
  return cudaErrorInvalidValue;
}

template <class K>
static cudaError_t launch_mix(K k, const MixParams& p, cudaStream_t st) {
  if (p.M <= 0) return cudaSuccess;
  const dim3 grid(unsigned((p.M + 255) / 256), unsigned((p.C + MCH - 1) / MCH));
  k<<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_mix_fwd(const MixParams& p, cudaStream_t st) {
  if (p.B > 1) return launch_mix_b(p, false, st);
  if (p.C <= 4) return launch_mix(mix_fwd_kernel<4>, p, st);
  if (p.C <= 8) return launch_mix(mix_fwd_kernel<8>, p, st);
  if (p.C <= 12) return launch_mix(mix_fwd_kernel<12>, p, st);
  if (p.C <= 16) return launch_mix(mix_fwd_kernel<16>, p, st);
  if (p.C <= 20) return launch_mix(mix_fwd_kernel<20>, p, st);
  if (p.C <= 24) return launch_mix(mix_fwd_kernel<24>, p, st);
  if (p.C <= 32) return launch_mix(mix_fwd_kernel<32>, p, st);
  if (p.C <= 64) return launch_mix(mix_fwd_kernel<64>, p, st);
  return cudaErrorInvalidValue;
}
cudaError_t launch_mix_bwd(const MixParams& p, cudaStream_t st) {
  if (p.B > 1) return launch_mix_b(p, true, st);
  if (p.C <= 4) return launch_mix(mix_bwd_kernel<4>, p, st);
  if (p.C <= 8) return launch_mix(mix_bwd_kernel<8>, p, st);
  if (p.C <= 12) return launch_mix(mix_bwd_kernel<12>, p, st);
  if (p.C <= 16) return launch_mix(mix_bwd_kernel<16>, p, st);
  if (p.C <= 20) return launch_mix(mix_bwd_kernel<20>, p, st);
  if (p.C <= 24) return launch_mix(mix_bwd_kernel<24>, p, st);
  if (p.C <= 32) return launch_mix(mix_bwd_kernel<32>, p, st);
  if (p.C <= 64) return launch_mix(mix_bwd_kernel<64>, p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_rowsum(const float* parts, int nparts, int len, int split, float* out0, float* out1, int accumulate,
                          cudaStream_t st) {
  rowsum_kernel<<<(len + 7) / 8, 256, 0, st>>>(parts, nparts, len, split, out0, out1, accumulate);
  return cudaGetLastError();
}

bool b_size_supported(int L) {
#define FNO_CASE(l) if (L == l) return true;
  FNO_B_SIZES(FNO_CASE)
#undef FNO_CASE
  return false;
}

}  // namespace fno
