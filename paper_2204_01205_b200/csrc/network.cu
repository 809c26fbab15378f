// Kernels of the whole DFNO network around the blocks (SURVEY §8.f N1,
// PAPER.md §"Full Network" P:135-183): the lift (time affine on an input with
// a time axis of size 1, then channel affine), the
// projection C -> 1, the relative L2 misfit, their
// adjoints, and the Adam update.  All are pointwise along the
// distributed x/y/z/t axes, so they run on the local box with no exchange; the
// replicated parameters' gradients are per-CTA partial sums reduced in a fixed
// order (deterministic), then summed over ranks by the caller (broadcast
// adjoint).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "launch.h"

namespace fno {

// Index math: every kernel runs over (batch b = blockIdx.y) x (an in-plane
// range strided over blockIdx.x) with 32-bit in-plane offsets (local boxes are
// far below 2^31 elements per channel), so no 64-bit division by a runtime
// extent sits on a per-element path.

// ---------------------------------------------------------------------------
// lift: nu0[b][o][sp][t] = s_o Wt[t] + wsum_o bt[t] + bc[o],
//       s_o = sum_c Wc[o][c] a[b][c][sp], wsum_o = sum_c Wc[o][c]
// thread per (b, sp): Cin loads, then C x T outputs (float4 along t)
// ---------------------------------------------------------------------------
template <int VW>
__global__ void __launch_bounds__(512) net_lift_fwd_kernel(NetParams q) {
  extern __shared__ float sh[];
  float* Wc = sh;                       // [C][Cin]
  float* ws = Wc + q.C * q.Cin;         // [C]
  float* bc = ws + q.C;                 // [C]
  for (int e = threadIdx.x; e < q.C * q.Cin; e += blockDim.x) Wc[e] = q.Wc[e];
  for (int o = threadIdx.x; o < q.C; o += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < q.Cin; ++c) s += q.Wc[o * q.Cin + c];
    ws[o] = s;
    bc[o] = q.bc[o];
  }
  __syncthreads();
  // thread per (point, t group of VW); its t group is fixed along the grid
  // stride (a multiple of T / VW), so consecutive lanes store consecutive t
  const int b = blockIdx.y, NS = int(q.NS), T = q.T, TV = T / VW;
  const int g0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int t0 = (g0 % TV) * VW;
  float wt[VW], bt[VW];
#pragma unroll
  for (int k = 0; k < VW; ++k) {
    wt[k] = q.Wt[t0 + k];
    bt[k] = q.bt[t0 + k];
  }
  const int spstride = (gridDim.x * blockDim.x) / TV;
  const float* ab = q.a + (size_t)b * q.Cin * NS;
  for (int sp = g0 / TV; sp < NS; sp += spstride) {
    float av[4];
    for (int c = 0; c < q.Cin; ++c) av[c] = __ldg(ab + (size_t)c * NS + sp);
    float* out = q.nu + ((size_t)b * q.C * NS + sp) * T + t0;
    for (int o = 0; o < q.C; ++o) {
      float s = 0.f;
      for (int c = 0; c < q.Cin; ++c) s = fmaf(Wc[o * q.Cin + c], av[c], s);
      const float w = ws[o], bo = bc[o];
      float* dst = out + (size_t)o * NS * T;
      if (VW == 4) {
        float4 v;
        v.x = fmaf(s, wt[0], fmaf(w, bt[0], bo));
        v.y = fmaf(s, wt[VW > 1 ? 1 : 0], fmaf(w, bt[VW > 1 ? 1 : 0], bo));
        v.z = fmaf(s, wt[VW > 2 ? 2 : 0], fmaf(w, bt[VW > 2 ? 2 : 0], bo));
        v.w = fmaf(s, wt[VW > 3 ? 3 : 0], fmaf(w, bt[VW > 3 ? 3 : 0], bo));
        __stcs(reinterpret_cast<float4*>(dst), v);
      } else {
        dst[0] = fmaf(s, wt[0], fmaf(w, bt[0], bo));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// projection: u[b][i] = sum_o Wp[o] nu[b][o][i] + bp   (thread per float4 / float)
// ---------------------------------------------------------------------------
template <int VW>
__global__ void __launch_bounds__(256) net_proj_fwd_kernel(NetParams q) {
  const int b = blockIdx.y;
  const unsigned NL = unsigned(q.NS * q.T);
  const float bp = q.bp ? q.bp[0] : 0.f;
  const float* src = q.nu + (size_t)b * q.C * NL;
  float* dst = q.u + (size_t)b * NL;
  for (unsigned i = (blockIdx.x * blockDim.x + threadIdx.x) * VW; i < NL; i += gridDim.x * blockDim.x * VW) {
    if (VW == 4) {
      float4 acc = make_float4(bp, bp, bp, bp);
      for (int o = 0; o < q.C; ++o) {
        const float w = __ldg(q.Wp + o);
        const float4 x = __ldcs(reinterpret_cast<const float4*>(src + (size_t)o * NL + i));
        acc.x = fmaf(w, x.x, acc.x); acc.y = fmaf(w, x.y, acc.y); acc.z = fmaf(w, x.z, acc.z); acc.w = fmaf(w, x.w, acc.w);
      }
      *reinterpret_cast<float4*>(dst + i) = acc;
    } else {
      float acc = bp;
      for (int o = 0; o < q.C; ++o) acc = fmaf(__ldg(q.Wp + o), src[(size_t)o * NL + i], acc);
      dst[i] = acc;
    }
  }
}

// fixed-order block reduction of one double per thread (blockDim a multiple of 32)
__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
  return s;   // valid in thread 0
}

// NACC per-thread float accumulators -> one row of per-CTA sums, in a fixed
// order: butterfly within each warp, then the warps in ascending order.
// wsum: shared [nwarps][NACC]; row[j] = sum (j < NACC, skipped where keep(j) is false)
template <int NACC>
__device__ __forceinline__ void block_rows(const float (&acc)[NACC], float* wsum, float* row) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NACC; ++j) {
    float v = acc[j];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (l == 0) wsum[w * NACC + j] = v;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < NACC; j += blockDim.x) {
    float s = 0.f;
    for (int i = 0; i < nw; ++i) s += wsum[i * NACC + j];
    row[j] = s;
  }
}

// ---------------------------------------------------------------------------
// relative L2: per-CTA partial sums of (u - y)^2 and y^2 in fp64
// ---------------------------------------------------------------------------
__global__ void net_loss_partial_kernel(NetParams q) {
  __shared__ double red[32];
  const long long n = (long long)q.B * q.NS * q.T;
  double sd = 0.0, sy = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const double u = q.u[e], y = q.y[e];
    sd += (u - y) * (u - y);
    sy += y * y;
  }
  const double a = block_sum_d(sd, red);
  const double b = block_sum_d(sy, red);
  if (threadIdx.x == 0) {
    q.dparts[2 * blockIdx.x] = a;
    q.dparts[2 * blockIdx.x + 1] = b;
  }
}

// sums nrows rows of 2 doubles (the CTA partials of one rank, or the per-rank
// sums in rank order) in a fixed order: lane l takes rows l, l + 32, ...,
// then a butterfly; writes the sums and, if out != NULL, out = {L, ||u - y||^2, ||y||^2}
__global__ void net_loss_finalize_kernel(const double* parts, int nrows, double* sums, float* out) {
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nrows; i += 32) {
    a += parts[2 * i];
    b += parts[2 * i + 1];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
  }
  if (threadIdx.x == 0) {
    sums[0] = a;
    sums[1] = b;
    if (out) {
      out[0] = float(sqrt(a) / sqrt(b));
      out[1] = float(a);
      out[2] = float(b);
    }
  }
}

// ---------------------------------------------------------------------------
// projection + loss adjoint: du = (u - y) / (||u - y|| ||y||);
// dnu[b][o][i] = Wp[o] du; partials of dWp[o] = sum du nu[o], dbp = sum du
// (thread per float4; row per CTA (b, x): [dWp (C)][dbp])
// ---------------------------------------------------------------------------
template <int CP>
__global__ void __launch_bounds__(256) net_proj_bwd_kernel(NetParams q) {
  extern __shared__ float wsum[];
  const int b = blockIdx.y;
  const unsigned NL = unsigned(q.NS * q.T);
  const float scale = float(1.0 / (sqrt(q.stats[0]) * sqrt(q.stats[1])));
  const float* src = q.nu + (size_t)b * q.C * NL;
  float* dst = q.dnu + (size_t)b * q.C * NL;
  float acc[CP + 1];
#pragma unroll
  for (int j = 0; j <= CP; ++j) acc[j] = 0.f;
  for (unsigned i = (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < NL; i += gridDim.x * blockDim.x * 4) {
    const float4 u4 = *reinterpret_cast<const float4*>(q.u + (size_t)b * NL + i);
    const float4 y4 = *reinterpret_cast<const float4*>(q.y + (size_t)b * NL + i);
    const float4 d = make_float4((u4.x - y4.x) * scale, (u4.y - y4.y) * scale, (u4.z - y4.z) * scale,
                                 (u4.w - y4.w) * scale);
#pragma unroll
    for (int o = 0; o < CP; ++o) {
      if (o < q.C) {
        const float4 x = __ldcs(reinterpret_cast<const float4*>(src + (size_t)o * NL + i));
        acc[o] = fmaf(d.x, x.x, fmaf(d.y, x.y, fmaf(d.z, x.z, fmaf(d.w, x.w, acc[o]))));
        const float w = __ldg(q.Wp + o);
        __stcs(reinterpret_cast<float4*>(dst + (size_t)o * NL + i), make_float4(w * d.x, w * d.y, w * d.z, w * d.w));
      }
    }
    acc[CP] += (d.x + d.y) + (d.z + d.w);
  }
  // row [dWp (C)][dbp], C + 1 floats
  float* row = q.parts + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * (q.C + 1);
  float* tmp = wsum + (blockDim.x >> 5) * (CP + 1);
  block_rows<CP + 1>(acc, wsum, tmp);
  __syncthreads();
  for (int j = threadIdx.x; j <= CP; j += blockDim.x) {
    if (j < q.C) row[j] = tmp[j];
    else if (j == CP) row[q.C] = tmp[j];
  }
}

// ---------------------------------------------------------------------------
// lift adjoint.  With a1_c(t) = Wt[t] a_c + bt[t], s_o = sum_c Wc[o][c] a_c,
// ws_o = sum_c Wc[o][c], and g = dnu0[o][t] at one point:
//   dWc[o][c] += sum_t g a1_c(t) = a_c G1_o + G2_o,  G1 = sum_t g Wt[t], G2 = sum_t g bt[t]
//   dbc[o]    += G0_o = sum_t g
//   dWt[t]    += sum_c da1_c(t) a_c = sum_o s_o g      (da1_c = sum_o Wc[o][c] g)
//   dbt[t]    += sum_c da1_c(t)     = sum_o ws_o g
// Thread per (point, t-quad); each thread keeps its t-quad (the grid stride is
// a multiple of T/4).  Row per CTA: [dWc (CP*CIN)][dbc (CP)][dWt (T)][dbt (T)].
// ---------------------------------------------------------------------------
template <int CP, int CIN, int VW>
__global__ void __launch_bounds__(512) net_lift_bwd_kernel(NetParams q) {
  extern __shared__ float lsh[];
  constexpr int NACC = CP * CIN + CP;
  const int b = blockIdx.y, NS = int(q.NS), T = q.T, TV = T / VW;
  float* Wc = lsh;                         // [CP][CIN] (zero-padded)
  float* ws = Wc + CP * CIN;               // [CP]
  float* tq = ws + CP;                     // [2][blockDim][VW]: per-thread dWt, dbt groups
  float* wsum = tq + 2 * VW * blockDim.x;  // [nwarps][NACC]
  for (int e = threadIdx.x; e < CP * CIN; e += blockDim.x) Wc[e] = (e / CIN < q.C) ? q.Wc[e] : 0.f;
  for (int o = threadIdx.x; o < CP; o += blockDim.x) {
    float s = 0.f;
    if (o < q.C)
      for (int c = 0; c < CIN; ++c) s += q.Wc[o * CIN + c];
    ws[o] = s;
  }
  __syncthreads();
  float acc[NACC];
#pragma unroll
  for (int j = 0; j < NACC; ++j) acc[j] = 0.f;
  float awt[VW], abt[VW], wt[VW], bt[VW];
  const int g0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int t4 = (g0 % TV) * VW;
#pragma unroll
  for (int k = 0; k < VW; ++k) {
    awt[k] = abt[k] = 0.f;
    wt[k] = q.Wt[t4 + k];
    bt[k] = q.bt[t4 + k];
  }
  const int spstride = (gridDim.x * blockDim.x) / TV;
  const float* ab = q.a + (size_t)b * CIN * NS;
  const float* gb = q.dnu + (size_t)b * q.C * NS * T;
  for (int sp = g0 / TV; sp < NS; sp += spstride) {
    float av[CIN];
#pragma unroll
    for (int c = 0; c < CIN; ++c) av[c] = __ldg(ab + (size_t)c * NS + sp);
    const float* gp = gb + (size_t)sp * T + t4;
#pragma unroll
    for (int o = 0; o < CP; ++o) {
      if (o < q.C) {
        float g[VW];
        if (VW == 4) {
          const float4 g4 = __ldcs(reinterpret_cast<const float4*>(gp + (size_t)o * NS * T));
          g[0] = g4.x; g[VW > 1 ? 1 : 0] = g4.y; g[VW > 2 ? 2 : 0] = g4.z; g[VW > 3 ? 3 : 0] = g4.w;
        } else {
          g[0] = __ldcs(gp + (size_t)o * NS * T);
        }
        float G1 = 0.f, G2 = 0.f, G0 = 0.f;
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          G1 = fmaf(g[k], wt[k], G1);
          G2 = fmaf(g[k], bt[k], G2);
          G0 += g[k];
        }
        float so = 0.f;
#pragma unroll
        for (int c = 0; c < CIN; ++c) {
          acc[o * CIN + c] = fmaf(av[c], G1, acc[o * CIN + c] + G2);
          so = fmaf(Wc[o * CIN + c], av[c], so);
        }
        acc[CP * CIN + o] += G0;
        const float wo = ws[o];
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          awt[k] = fmaf(so, g[k], awt[k]);
          abt[k] = fmaf(wo, g[k], abt[k]);
        }
      }
    }
  }
  float* row = q.parts + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * q.plen;
  // dWc, dbc (compacted to C rows when written)
  float* tmp = wsum + (blockDim.x >> 5) * NACC;   // [NACC] block sums
  block_rows<NACC>(acc, wsum, tmp);
  __syncthreads();
  for (int j = threadIdx.x; j < NACC; j += blockDim.x) {
    if (j < CP * CIN) {
      if (j / CIN < q.C) row[j] = tmp[j];
    } else if (j - CP * CIN < q.C) {
      row[q.C * CIN + (j - CP * CIN)] = tmp[j];
    }
  }
  // dWt, dbt: threads with the same t group (tid = group + TV j) summed in ascending j
#pragma unroll
  for (int k = 0; k < VW; ++k) {
    tq[VW * threadIdx.x + k] = awt[k];
    tq[VW * (blockDim.x + threadIdx.x) + k] = abt[k];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int qd = t / VW, k = t % VW;
    float s0 = 0.f, s1 = 0.f;
    for (int j = qd; j < int(blockDim.x); j += TV) {
      s0 += tq[VW * j + k];
      s1 += tq[VW * (blockDim.x + j) + k];
    }
    row[q.C * CIN + q.C + t] = s0;
    row[q.C * CIN + q.C + T + t] = s1;
  }
}

// out[j] (+)= sum_{i < nrows} rows[i * stride + j], j < len, in a fixed order:
// one warp per j, lane l takes rows l, l + 32, ..., then a butterfly
__global__ void rowsum_strided_kernel(const float* rows, int nrows, long long stride, int len, float* out, int acc) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), l = threadIdx.x & 31;
  if (j >= len) return;
  float s = 0.f;
  for (int i = l; i < nrows; i += 32) s += rows[i * stride + j];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (l == 0) out[j] = acc ? out[j] + s : s;
}

// ---------------------------------------------------------------------------
// Adam (Kingma & Ba, Alg. 1, bias-corrected), elementwise, float4 when aligned
// ---------------------------------------------------------------------------
__device__ __forceinline__ void adam1(float& p, float g, float& m, float& v, float lr, float b1, float b2, float eps,
                                      float c1, float c2) {
  m = fmaf(b1, m, (1.f - b1) * g);
  v = fmaf(b2, v, (1.f - b2) * g * g);
  p -= lr * (m / c1) / (sqrtf(v / c2) + eps);
}
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, long long n, float lr, float b1, float b2, float eps, float c1,
                            float c2) {
  const long long n4 = (n % 4 == 0 && ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                                        reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0)
                           ? n / 4 : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 pp = reinterpret_cast<float4*>(p)[i], mm = reinterpret_cast<float4*>(m)[i], vv = reinterpret_cast<float4*>(v)[i];
    const float4 gg = __ldcs(reinterpret_cast<const float4*>(g) + i);
    adam1(pp.x, gg.x, mm.x, vv.x, lr, b1, b2, eps, c1, c2);
    adam1(pp.y, gg.y, mm.y, vv.y, lr, b1, b2, eps, c1, c2);
    adam1(pp.z, gg.z, mm.z, vv.z, lr, b1, b2, eps, c1, c2);
    adam1(pp.w, gg.w, mm.w, vv.w, lr, b1, b2, eps, c1, c2);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    adam1(p[i], g[i], m[i], v[i], lr, b1, b2, eps, c1, c2);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {
// CTAs along x per batch row: enough to fill the GPU about 4 times over
int net_gx(long long units, int block, int B, int num_sms) {
  const long long need = (units + block - 1) / block;
  const long long cap = std::max<long long>(1, (long long)num_sms * 4 / std::max(1, B));
  return int(std::max<long long>(1, std::min(need, cap)));
}
}  // namespace

namespace {
int lift_vw(int T) { return (T % 4 == 0 && T / 4 <= 256) ? 4 : 1; }
int lift_block(int T) {   // a multiple of lcm(32, T / VW), about 256 threads, at most 512
  const int tv = T / lift_vw(T);
  int a = tv, b = 32;
  while (b) { const int r = a % b; a = b; b = r; }
  const int l = tv / a * 32;
  return l >= 256 ? l : (256 / l) * l;
}
}  // namespace

cudaError_t launch_net_lift_fwd(const NetParams& q, int num_sms, cudaStream_t st) {
  const int VW = lift_vw(q.T), block = lift_block(q.T);
  if (block > 512) return cudaErrorInvalidValue;
  const size_t smem = size_t(q.C * q.Cin + 2 * q.C) * sizeof(float);
  const dim3 grid(net_gx(q.NS * (q.T / VW), block, q.B, num_sms), q.B);
  if (VW == 4) net_lift_fwd_kernel<4><<<grid, block, smem, st>>>(q);
  else net_lift_fwd_kernel<1><<<grid, block, smem, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_net_proj_fwd(const NetParams& q, int num_sms, cudaStream_t st) {
  const long long NL = q.NS * q.T;
  if (NL % 4 == 0) net_proj_fwd_kernel<4><<<dim3(net_gx(NL / 4, 256, q.B, num_sms), q.B), 256, 0, st>>>(q);
  else net_proj_fwd_kernel<1><<<dim3(net_gx(NL, 256, q.B, num_sms), q.B), 256, 0, st>>>(q);
  return cudaGetLastError();
}

int net_loss_grid(const NetParams& q, int num_sms) {
  return std::max(1, std::min(num_sms * 8, int(((long long)q.B * q.NS * q.T + 255) / 256)));
}

cudaError_t launch_net_loss_partial(const NetParams& q, int grid, cudaStream_t st) {
  net_loss_partial_kernel<<<grid, 256, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_net_loss_finalize(const double* parts, int nrows, double* sums, float* out, cudaStream_t st) {
  net_loss_finalize_kernel<<<1, 32, 0, st>>>(parts, nrows, sums, out);
  return cudaGetLastError();
}

// rows of partials: B * gx (the projection adjoint needs NL % 4 == 0)
int net_proj_bwd_grid(const NetParams& q, int num_sms) {
  return q.B * net_gx(q.NS * q.T / 4, 256, q.B, num_sms);
}

cudaError_t launch_net_proj_bwd(const NetParams& q, int rows, cudaStream_t st) {
  if ((q.NS * q.T) % 4 != 0) return cudaErrorInvalidValue;
  const int CP = (q.C + 3) & ~3;
  const dim3 grid(rows / q.B, q.B);
  const size_t smem = size_t(9 * (CP + 1)) * sizeof(float);
  switch (CP) {
#define FNO_PB(cp) case cp: net_proj_bwd_kernel<cp><<<grid, 256, smem, st>>>(q); break;
    FNO_PB(4) FNO_PB(8) FNO_PB(12) FNO_PB(16) FNO_PB(20) FNO_PB(24) FNO_PB(28) FNO_PB(32)
#undef FNO_PB
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// rows of partials: B * gx (block rule as the lift forward)
int net_lift_bwd_grid(const NetParams& q, int num_sms) {
  return q.B * net_gx(q.NS * (q.T / lift_vw(q.T)), lift_block(q.T), q.B, num_sms);
}

cudaError_t launch_net_lift_bwd(const NetParams& q, int rows, cudaStream_t st) {
  const int VW = lift_vw(q.T), block = lift_block(q.T);
  if (block > 512) return cudaErrorInvalidValue;
  const int CP = (q.C + 3) & ~3;
  const dim3 grid(rows / q.B, q.B);
  const int NACC = CP * q.Cin + CP;
  const int nw = (block + 31) / 32;
  const size_t smem = size_t(CP * q.Cin + CP + 2 * VW * block + nw * NACC + NACC) * sizeof(float);
#define FNO_LB(cp, cin)                                                                               \
  if (CP == cp && q.Cin == cin) {                                                                     \
    if (VW == 4) net_lift_bwd_kernel<cp, cin, 4><<<grid, block, smem, st>>>(q);                      \
    else net_lift_bwd_kernel<cp, cin, 1><<<grid, block, smem, st>>>(q);                              \
    return cudaGetLastError();                                                                        \
  }
#define FNO_LB_C(cp) FNO_LB(cp, 1) FNO_LB(cp, 2) FNO_LB(cp, 3) FNO_LB(cp, 4)
  FNO_LB_C(4) FNO_LB_C(8) FNO_LB_C(12) FNO_LB_C(16) FNO_LB_C(20) FNO_LB_C(24) FNO_LB_C(28) FNO_LB_C(32)
#undef FNO_LB_C
#undef FNO_LB
  return cudaErrorInvalidValue;
}

cudaError_t launch_rowsum_strided(const float* rows, int nrows, long long stride, int len, float* out, int acc,
                                  cudaStream_t st) {
  if (len <= 0) return cudaSuccess;
  rowsum_strided_kernel<<<(len + 7) / 8, 256, 0, st>>>(rows, nrows, stride, len, out, acc);
  return cudaGetLastError();
}

cudaError_t launch_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
                        float eps, int step, int num_sms, cudaStream_t st) {
  const float c1 = 1.f - powf(b1, float(step)), c2 = 1.f - powf(b2, float(step));
  const long long need = (n / 4 + 255) / 256 + 1;
  const int grid = int(std::max<long long>(1, std::min<long long>(need, (long long)num_sms * 8)));
  adam_kernel<<<grid, 256, 0, st>>>(p, g, m, v, n, lr, b1, b2, eps, c1, c2);
  return cudaGetLastError();
}

}  // namespace fno
