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

#include "launch.h"

namespace fno {

// ---------------------------------------------------------------------------
// lift: nu0[b][o][sp][t] = s_o Wt[t] + wsum_o bt[t] + bc[o],
//       s_o = sum_c Wc[o][c] a[b][c][sp], wsum_o = sum_c Wc[o][c]
// ---------------------------------------------------------------------------
template <int VW>
__global__ void net_lift_fwd_kernel(NetParams q) {
  extern __shared__ float sh[];
  float* Wc = sh;                       // [C][Cin]
  float* ws = Wc + q.C * q.Cin;         // [C]
  float* bc = ws + q.C;                 // [C]
  float* Wt = bc + q.C;                 // [T]
  float* bt = Wt + q.T;                 // [T]
  for (int e = threadIdx.x; e < q.C * q.Cin; e += blockDim.x) Wc[e] = q.Wc[e];
  for (int o = threadIdx.x; o < q.C; o += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < q.Cin; ++c) s += q.Wc[o * q.Cin + c];
    ws[o] = s;
    bc[o] = q.bc[o];
  }
  for (int t = threadIdx.x; t < q.T; t += blockDim.x) {
    Wt[t] = q.Wt[t];
    bt[t] = q.bt[t];
  }
  __syncthreads();
  const int TV = q.T / VW;
  const long long n = (long long)q.B * q.C * q.NS * TV;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int tv = int(e % TV);
    const long long r = e / TV;
    const long long sp = r % q.NS;
    const long long bo = r / q.NS;
    const int o = int(bo % q.C), b = int(bo / q.C);
    float s = 0.f;
    for (int c = 0; c < q.Cin; ++c) s = fmaf(Wc[o * q.Cin + c], __ldg(q.a + ((long long)b * q.Cin + c) * q.NS + sp), s);
    float* out = q.nu + (bo * q.NS + sp) * q.T + tv * VW;
    if (VW == 4) {
      const int t = tv * 4;
      float4 v;
      v.x = fmaf(s, Wt[t + 0], fmaf(ws[o], bt[t + 0], bc[o]));
      v.y = fmaf(s, Wt[t + 1], fmaf(ws[o], bt[t + 1], bc[o]));
      v.z = fmaf(s, Wt[t + 2], fmaf(ws[o], bt[t + 2], bc[o]));
      v.w = fmaf(s, Wt[t + 3], fmaf(ws[o], bt[t + 3], bc[o]));
      __stcs(reinterpret_cast<float4*>(out), v);
    } else {
      out[0] = fmaf(s, Wt[tv], fmaf(ws[o], bt[tv], bc[o]));
    }
  }
}

// ---------------------------------------------------------------------------
// projection: u[b][q] = sum_o Wp[o] nu[b][o][q] + bp
// ---------------------------------------------------------------------------
template <int VW>
__global__ void net_proj_fwd_kernel(NetParams q) {
  const long long NL = q.NS * q.T;
  const long long n = (long long)q.B * NL / VW;
  const float bp = q.bp ? q.bp[0] : 0.f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long b = (e * VW) / NL, i = e * VW - b * NL;
    const float* src = q.nu + b * q.C * NL + i;
    if (VW == 4) {
      float4 acc = make_float4(bp, bp, bp, bp);
      for (int o = 0; o < q.C; ++o) {
        const float w = __ldg(q.Wp + o);
        const float4 x = __ldcs(reinterpret_cast<const float4*>(src + o * NL));
        acc.x = fmaf(w, x.x, acc.x); acc.y = fmaf(w, x.y, acc.y); acc.z = fmaf(w, x.z, acc.z); acc.w = fmaf(w, x.w, acc.w);
      }
      *reinterpret_cast<float4*>(q.u + b * NL + i) = acc;
    } else {
      float acc = bp;
      for (int o = 0; o < q.C; ++o) acc = fmaf(__ldg(q.Wp + o), src[o * NL], acc);
      q.u[b * NL + i] = acc;
    }
  }
}

// fixed-order block reduction of one double per thread (blockDim = 256)
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

// sums nrows rows of 2 doubles in ascending order (the CTA partials of one rank,
// or the per-rank sums in rank order); writes the sums and, if out != NULL,
// out = {L, ||u - y||^2, ||y||^2} as floats
__global__ void net_loss_finalize_kernel(const double* parts, int nrows, double* sums, float* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < nrows; ++i) {
      a += parts[2 * i];
      b += parts[2 * i + 1];
    }
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
// dnu[b][o][q] = Wp[o] du; partials of dWp[o] = sum du nu[o], dbp = sum du
// ---------------------------------------------------------------------------
template <int CP>
__global__ void __launch_bounds__(256) net_proj_bwd_kernel(NetParams q) {
  __shared__ double red[32];
  const long long NL = q.NS * q.T;
  const long long n = (long long)q.B * NL;
  const float scale = float(1.0 / (sqrt(q.stats[0]) * sqrt(q.stats[1])));
  float acc[CP + 1];
#pragma unroll
  for (int j = 0; j <= CP; ++j) acc[j] = 0.f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / NL, i = e - b * NL;
    const float du = (q.u[e] - q.y[e]) * scale;
    const float* src = q.nu + b * q.C * NL + i;
    float* dst = q.dnu + b * q.C * NL + i;
#pragma unroll
    for (int o = 0; o < CP; ++o) {
      if (o < q.C) {
        acc[o] = fmaf(du, src[o * NL], acc[o]);
        dst[o * NL] = __ldg(q.Wp + o) * du;
      }
    }
    acc[CP] += du;
  }
  // fixed-order reduction per accumulator (partials in float, summed in fp64)
#pragma unroll
  for (int j = 0; j <= CP; ++j) {
    if (j < q.C || j == CP) {
      const double s = block_sum_d(double(acc[j]), red);
      if (threadIdx.x == 0) q.parts[(long long)blockIdx.x * (q.C + 1) + (j == CP ? q.C : j)] = float(s);
    }
  }
}

// ---------------------------------------------------------------------------
// lift adjoint: per point (b, sp) and t, with a1_c = Wt[t] a_c + bt[t]:
//   dWc[o][c] += dnu0[o][t] a1_c;   dbc[o] += dnu0[o][t]
//   da1_c = sum_o Wc[o][c] dnu0[o][t];  dWt[t] += sum_c da1_c a_c;  dbt[t] += sum_c da1_c
// Each thread keeps one t (blockDim and the grid stride are multiples of T).
// Partials row per CTA: [dWc (C*Cin)][dbc (C)][dWt (T)][dbt (T)].
// ---------------------------------------------------------------------------
template <int CP, int CIN>
__global__ void __launch_bounds__(256) net_lift_bwd_kernel(NetParams q) {
  extern __shared__ float tsh[];          // [2][blockDim] per-thread dWt, dbt; [nwarps][NACC] warp sums
  const long long n = (long long)q.B * q.NS * q.T;   // items (b, sp, t)
  float aw[CP][CIN], ab[CP];
#pragma unroll
  for (int o = 0; o < CP; ++o) {
    ab[o] = 0.f;
#pragma unroll
    for (int c = 0; c < CIN; ++c) aw[o][c] = 0.f;
  }
  float awt = 0.f, abt = 0.f;
  const int t = int((blockIdx.x * (long long)blockDim.x + threadIdx.x) % q.T);
  const float wt = q.Wt[t], btv = q.bt[t];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / q.T;               // (b, sp)
    const long long sp = r % q.NS, b = r / q.NS;
    float av[CIN], a1[CIN], da1[CIN];
#pragma unroll
    for (int c = 0; c < CIN; ++c) {
      av[c] = __ldg(q.a + (b * CIN + c) * q.NS + sp);
      a1[c] = fmaf(wt, av[c], btv);
      da1[c] = 0.f;
    }
    const float* g = q.dnu + (b * q.C * q.NS + sp) * q.T + t;
#pragma unroll
    for (int o = 0; o < CP; ++o) {
      if (o < q.C) {
        const float gv = __ldcs(g + (long long)o * q.NS * q.T);
        ab[o] += gv;
#pragma unroll
        for (int c = 0; c < CIN; ++c) {
          aw[o][c] = fmaf(gv, a1[c], aw[o][c]);
          da1[c] = fmaf(__ldg(q.Wc + o * CIN + c), gv, da1[c]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CIN; ++c) {
      awt = fmaf(da1[c], av[c], awt);
      abt += da1[c];
    }
  }
  float* row = q.parts + (long long)blockIdx.x * q.plen;
  // fixed-order reduction: butterfly within each warp (constant register
  // indices, fully unrolled), then the warps in ascending order
  constexpr int NACC = CP * CIN + CP;
  float* wsum = tsh + 2 * blockDim.x;     // [nwarps][NACC]
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 0; o < CP; ++o) {
#pragma unroll
    for (int c = 0; c <= CIN; ++c) {
      float v = c < CIN ? aw[o][c < CIN ? c : 0] : ab[o];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (l == 0) wsum[w * NACC + (c < CIN ? o * CIN + c : CP * CIN + o)] = v;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < NACC; j += blockDim.x) {
    const bool isw = j < CP * CIN;
    const int o = isw ? j / CIN : j - CP * CIN;
    if (o >= q.C) continue;
    float s = 0.f;
    for (int i = 0; i < nw; ++i) s += wsum[i * NACC + j];
    row[isw ? o * CIN + (j - o * CIN) : q.C * CIN + o] = s;
  }
  // dWt, dbt: threads with the same t (tid = t + T j) summed in ascending j
  tsh[threadIdx.x] = awt;
  tsh[blockDim.x + threadIdx.x] = abt;
  __syncthreads();
  if (threadIdx.x < q.T) {
    float s0 = 0.f, s1 = 0.f;
    for (int j = threadIdx.x; j < int(blockDim.x); j += q.T) {
      s0 += tsh[j];
      s1 += tsh[blockDim.x + j];
    }
    row[q.C * CIN + q.C + threadIdx.x] = s0;
    row[q.C * CIN + q.C + q.T + threadIdx.x] = s1;
  }
}

// ---------------------------------------------------------------------------
// Adam (Kingma & Ba, Alg. 1, bias-corrected), elementwise over floats
// ---------------------------------------------------------------------------
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, long long n, float lr, float b1, float b2, float eps, float c1,
                            float c2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = fmaf(b1, m[i], (1.f - b1) * gi);
    const float vi = fmaf(b2, v[i], (1.f - b2) * gi * gi);
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {
int net_grid(long long n, int block, int num_sms) {
  const long long need = (n + block - 1) / block;
  return int(need < (long long)num_sms * 8 ? (need > 0 ? need : 1) : (long long)num_sms * 8);
}
}  // namespace

cudaError_t launch_net_lift_fwd(const NetParams& q, int num_sms, cudaStream_t st) {
  const size_t smem = size_t(q.C * q.Cin + 2 * q.C + 2 * q.T) * sizeof(float);
  if (q.T % 4 == 0) {
    net_lift_fwd_kernel<4><<<net_grid((long long)q.B * q.C * q.NS * (q.T / 4), 256, num_sms), 256, smem, st>>>(q);
  } else {
    net_lift_fwd_kernel<1><<<net_grid((long long)q.B * q.C * q.NS * q.T, 256, num_sms), 256, smem, st>>>(q);
  }
  return cudaGetLastError();
}

cudaError_t launch_net_proj_fwd(const NetParams& q, int num_sms, cudaStream_t st) {
  const long long NL = q.NS * q.T;
  if (NL % 4 == 0) net_proj_fwd_kernel<4><<<net_grid((long long)q.B * NL / 4, 256, num_sms), 256, 0, st>>>(q);
  else net_proj_fwd_kernel<1><<<net_grid((long long)q.B * NL, 256, num_sms), 256, 0, st>>>(q);
  return cudaGetLastError();
}

int net_loss_grid(const NetParams& q, int num_sms) { return net_grid((long long)q.B * q.NS * q.T, 256, num_sms); }

cudaError_t launch_net_loss_partial(const NetParams& q, int grid, cudaStream_t st) {
  net_loss_partial_kernel<<<grid, 256, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_net_loss_finalize(const double* parts, int nrows, double* sums, float* out, cudaStream_t st) {
  net_loss_finalize_kernel<<<1, 32, 0, st>>>(parts, nrows, sums, out);
  return cudaGetLastError();
}

int net_proj_bwd_grid(const NetParams& q, int num_sms) { return net_grid((long long)q.B * q.NS * q.T, 256, num_sms); }

cudaError_t launch_net_proj_bwd(const NetParams& q, int grid, cudaStream_t st) {
  const int CP = (q.C + 3) & ~3;
  switch (CP) {
#define FNO_PB(cp) case cp: net_proj_bwd_kernel<cp><<<grid, 256, 0, st>>>(q); break;
    FNO_PB(4) FNO_PB(8) FNO_PB(12) FNO_PB(16) FNO_PB(20) FNO_PB(24) FNO_PB(28) FNO_PB(32)
#undef FNO_PB
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// block size: a multiple of T (each thread keeps one t), about 256
int net_lift_bwd_block(int T) { return T >= 256 ? T : (256 / T) * T; }
int net_lift_bwd_grid(const NetParams& q, int num_sms) {
  return net_grid((long long)q.B * q.NS * q.T, net_lift_bwd_block(q.T), num_sms);
}

cudaError_t launch_net_lift_bwd(const NetParams& q, int grid, cudaStream_t st) {
  const int CP = (q.C + 3) & ~3;
  const int block = net_lift_bwd_block(q.T);
  const size_t smem = size_t(2 * block + (block / 32) * (CP * q.Cin + CP)) * sizeof(float);
#define FNO_LB(cp, cin) \
  if (CP == cp && q.Cin == cin) { net_lift_bwd_kernel<cp, cin><<<grid, block, smem, st>>>(q); return cudaGetLastError(); }
#define FNO_LB_C(cp) FNO_LB(cp, 1) FNO_LB(cp, 2) FNO_LB(cp, 3) FNO_LB(cp, 4)
  FNO_LB_C(4) FNO_LB_C(8) FNO_LB_C(12) FNO_LB_C(16) FNO_LB_C(20) FNO_LB_C(24) FNO_LB_C(28) FNO_LB_C(32)
#undef FNO_LB_C
#undef FNO_LB
  return cudaErrorInvalidValue;
}

// out[j] (+)= sum_{i < nrows} rows[i * stride + j], j < len, ascending i
__global__ void rowsum_strided_kernel(const float* rows, int nrows, long long stride, int len, float* out, int acc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= len) return;
  float s = 0.f;
  for (int i = 0; i < nrows; ++i) s += rows[i * stride + j];
  out[j] = acc ? out[j] + s : s;
}
cudaError_t launch_rowsum_strided(const float* rows, int nrows, long long stride, int len, float* out, int acc,
                                  cudaStream_t st) {
  if (len <= 0) return cudaSuccess;
  rowsum_strided_kernel<<<(len + 127) / 128, 128, 0, st>>>(rows, nrows, stride, len, out, acc);
  return cudaGetLastError();
}

cudaError_t launch_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
                        float eps, int step, int num_sms, cudaStream_t st) {
  const float c1 = 1.f - powf(b1, float(step)), c2 = 1.f - powf(b2, float(step));
  adam_kernel<<<net_grid(n, 256, num_sms), 256, 0, st>>>(p, g, m, v, n, lr, b1, b2, eps, c1, c2);
  return cudaGetLastError();
}

}  // namespace fno
