// Pass C (bwd a9, a12): the adjoint chain of I_1 =
// {z, t} (zero-padded inverse z, C2R along t with real-part semantics,
// P:119-123 "F_dist^T"), fused with the DFNO block epilogue
//   z = W v + b + u ; y = GELU(z)                      (Eq. dist_block)
// or, backward, dv = W^T dz + S^T dz plus the dW, db partial sums
// (broadcast adjoint = sum-reduce).
//
// One CTA per (b, x, y) column (all channels).  The z outputs are produced by
// residue class r (z = r + Qz*s, s < LZ), so a tile holds C x LZ x T values of
// u for the 1x1 channel linear, which needs every channel at a point.
#include "kernels.cuh"
#include "launch.h"

namespace fno {

static constexpr int CT = 256;  // threads per CTA

struct CLayout {
  int Cp, np, nk, TP;
  size_t ws, bias, su, bb, vt, vt2, twz, twt, dmap, total;
};

__host__ __device__ inline CLayout c_layout(int C, int Z, int T, int mz, int mt, int LZ, int mode) {
  CLayout L{};
  L.Cp = (C + 3) & ~3;
  L.np = LZ * T;
  L.nk = mz + 1;
  L.TP = T + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
  L.ws = take(size_t(C) * L.Cp * sizeof(float));
  L.bias = take(size_t(C) * sizeof(float));
  size_t s_bytes = size_t(C) * 2 * mz * mt * sizeof(float2);
  size_t u_bytes = size_t(C) * L.np * sizeof(float);
  L.su = take(s_bytes > u_bytes ? s_bytes : u_bytes);
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.vt = take(mode == EPI_U ? 0 : size_t(C) * L.np * sizeof(float));
  L.vt2 = take(mode == EPI_BWD ? size_t(C) * L.np * sizeof(float) : 0);
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  L.total = off;
  return L;
}

template <int LZ, int LT, int EPI>
__global__ void __launch_bounds__(CT) pass_c_kernel(PassCParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const CLayout L = c_layout(C, Z, T, mz, mt, LZ, EPI);
  float* Ws = reinterpret_cast<float*>(smem_raw + L.ws);
  float* bs = reinterpret_cast<float*>(smem_raw + L.bias);
  float2* S = reinterpret_cast<float2*>(smem_raw + L.su);
  float* U = reinterpret_cast<float*>(smem_raw + L.su);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float* Vt = reinterpret_cast<float*>(smem_raw + L.vt);
  float* Vt2 = reinterpret_cast<float*>(smem_raw + L.vt2);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int np = L.np, nk = L.nk, TP = L.TP, Cp = L.Cp;
  const int ZT = Z * T;
  const int G = (C + 3) / 4;

  fill_twiddles(twZ, Z, tid, nt);
  fill_twiddles(twT, T, tid, nt);
  for (int j = tid; j < 2 * mz; j += nt) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  if (EPI != EPI_U) {
    // Ws[k*Cp + out]: fwd k = input channel (W^T), bwd k = output channel (W)
    for (int e = tid; e < C * Cp; e += nt) {
      const int k = e / Cp, o = e - k * Cp;
      float w = 0.f;
      if (o < C) w = (EPI == EPI_FWD) ? p.W[o * C + k] : p.W[k * C + o];
      Ws[e] = w;
    }
    for (int o = tid; o < C; o += nt) bs[o] = (EPI == EPI_FWD && p.bias) ? p.bias[o] : 0.f;
  }

  // dW / db accumulators (EPI_BWD): thread -> 4x4 block (og, ig) + point group
  const int NB = G * G;
  const int NPG = (EPI == EPI_BWD) ? max(1, nt / NB) : 1;
  const bool dw_thread = (EPI == EPI_BWD) && tid < NB * NPG;
  const int blk = tid % NB, pgrp = tid / NB;
  const int og = blk / G, ig = blk % G;
  float dwacc[4][4];
  float dbacc[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    dbacc[a] = 0.f;
#pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) dwacc[a][c2] = 0.f;
  }

  for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
    const int yl = int(col % p.Yl);
    const long long r1 = col / p.Yl;
    const int xl = int(r1 % p.Xl);
    const int b = int(r1 / p.Xl);
    const long long colpt = ((long long)b * p.Xl + xl) * p.Yl + yl;
    __syncthreads();  // previous column done with S/U/Bb/Vt; tables ready
    // ---- phase 0: this column's retained (kz, kt) spectrum, all channels --
    {
      const int per_c = 2 * mz * mt;
      for (int e = tid; e < C * per_c; e += nt) {
        const int c = e / per_c, rem = e - c * per_c;
        const int jz = rem / mt, kt = rem - jz * mt;
        const short2 dm = dmap[jz];
        const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
        S[e] = __ldcs(p.in + p.slab.off[dm.x] + ((colpt * C + c) * nkz + dm.y) * mt + kt);
      }
    }
    __syncthreads();
    // ---- phase 1: inverse t (C2R weights folded in), pencils (c, kz') ------
    for (int pid = tid; pid < C * nk; pid += nt) {
      const int c = pid / nk, kzp = pid - c * nk;
      const float2* Sp = S + (c * 2 * mz + kzp) * mt;              // kz = +kz'
      const float2* Sn = S + (c * 2 * mz + (2 * mz - kzp)) * mt;   // kz = -kz'
      float2 e[LT];
#pragma unroll
      for (int i = 0; i < LT; ++i) {
        float2 acc = make_float2(0.f, 0.f);
        if (i < mt && kzp < mz) {
          const float cw = (i == 0 || 2 * i == T) ? 1.f : 2.f;
          acc = cscale(Sp[i], cw);
        }
        const int kt = (LT - i) % LT;
        if (kzp >= 1 && kt < mt && (i == 0 || i > LT - mt)) {
          const float cw = (kt == 0 || 2 * kt == T) ? 1.f : 2.f;
          acc = cadd(acc, cscale(cconj(Sn[kt]), cw));
        }
        e[i] = acc;
      }
      float2* bo = Bb + (c * nk + kzp) * TP;
      for (int rt = 0; rt < p.Qt; ++rt) {
        float2 y[LT];
        trunc_inv<LT>(y, e, T, p.Qt, rt, mt - 1, twT);
#pragma unroll
        for (int s = 0; s < LT; ++s) bo[rt + p.Qt * s] = y[s];
      }
    }
    __syncthreads();
    // ---- per residue class of z ------------------------------------------
    for (int rz = 0; rz < p.Qz; ++rz) {
      // stage the epilogue inputs for this tile (EPI_FWD: v; EPI_BWD: dz, v)
      if (EPI != EPI_U) {
        for (int e = tid; e < C * np; e += nt) {
          const int c = e / np, pt = e - c * np;
          const int s = pt / T, t = pt - s * T;
          const long long g = ((long long)b * C + c) * ((long long)p.Xl * p.Yl * ZT) +
                              ((long long)xl * p.Yl + yl) * ZT + (rz + p.Qz * s) * T + t;
          if (EPI == EPI_FWD) {
            Vt[e] = __ldcs(p.v + g);
          } else {
            const float dyv = __ldcs(p.dy + g);
            Vt[e] = p.act_gelu ? dyv * gelu_prime_f(__ldcs(p.zs + g)) : dyv;
            Vt2[e] = __ldcs(p.v + g);
          }
        }
      }
      // phase 2: inverse z (real output), pencils (c, t)
      for (int pid = tid; pid < C * T; pid += nt) {
        const int c = pid / T, t = pid - c * T;
        float2 e[LZ];
#pragma unroll
        for (int i = 0; i < LZ; ++i) e[i] = (i < nk) ? Bb[(c * nk + i) * TP + t] : make_float2(0.f, 0.f);
        float2 y[LZ];
        trunc_inv<LZ>(y, e, Z, p.Qz, rz, 0, twZ);
        if (EPI == EPI_U) {
          float* o = p.out + ((long long)b * C + c) * ((long long)p.Xl * p.Yl * ZT) + ((long long)xl * p.Yl + yl) * ZT + rz * T + t;
#pragma unroll
          for (int s = 0; s < LZ; ++s) __stcs(o + (long long)p.Qz * s * T, y[s].x * p.inv_n);
        } else {
#pragma unroll
          for (int s = 0; s < LZ; ++s) U[(c * LZ + s) * T + t] = y[s].x * p.inv_n;
        }
      }
      if (EPI == EPI_U) continue;
      __syncthreads();
      // phase 3: 1x1 channel linear + epilogue, items (o-group g, point pt)
      for (int it = tid; it < G * np; it += nt) {
        const int g = it / np, pt = it - g * np;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int k = 0; k < C; ++k) {
          const float val = Vt[k * np + pt];
          const float4 w4 = *reinterpret_cast<const float4*>(Ws + k * Cp + 4 * g);
          acc[0] = fmaf(w4.x, val, acc[0]);
          acc[1] = fmaf(w4.y, val, acc[1]);
          acc[2] = fmaf(w4.z, val, acc[2]);
          acc[3] = fmaf(w4.w, val, acc[3]);
        }
        const int s = pt / T, t = pt - s * T;
        const long long gbase = ((long long)xl * p.Yl + yl) * ZT + (rz + p.Qz * s) * T + t;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int o = 4 * g + a;
          if (o < C) {
            const long long gi = ((long long)b * C + o) * ((long long)p.Xl * p.Yl * ZT) + gbase;
            float val = acc[a] + U[o * np + pt];
            if (EPI == EPI_FWD) {
              val += bs[o];
              if (p.zsave) __stcs(p.zsave + gi, val);
              __stcs(p.out + gi, p.act_gelu ? gelu_f(val) : val);
            } else {
              __stcs(p.out + gi, val);
            }
          }
        }
      }
      if (EPI == EPI_BWD && dw_thread) {
        for (int pt = pgrp; pt < np; pt += NPG) {
          float dz4[4], v4[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int o = 4 * og + a, i = 4 * ig + a;
            dz4[a] = (o < C) ? Vt[o * np + pt] : 0.f;
            v4[a] = (i < C) ? Vt2[i * np + pt] : 0.f;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            if (ig == 0) dbacc[a] += dz4[a];
#pragma unroll
            for (int c2 = 0; c2 < 4; ++c2) dwacc[a][c2] = fmaf(dz4[a], v4[c2], dwacc[a][c2]);
          }
        }
      }
      __syncthreads();
    }
  }
  if (EPI == EPI_BWD) {
    // fixed-order CTA reduction of the per-thread partials into dWpart[blockIdx.x]
    __syncthreads();
    float* red = Vt;  // reuse: NB*NPG*20 floats fit in the C*np tile for C >= 2
    const int stride = 20;
    if (dw_thread) {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) red[tid * stride + a * 4 + c2] = dwacc[a][c2];
        red[tid * stride + 16 + a] = dbacc[a];
      }
    }
    __syncthreads();
    float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
    for (int e = tid; e < C * C + C; e += nt) {
      int o, i, slot;
      if (e < C * C) { o = e / C; i = e - o * C; slot = (o % 4) * 4 + (i % 4); }
      else { o = e - C * C; i = 0; slot = 16 + (o % 4); }
      const int bk = (o / 4) * G + (i / 4);
      float s = 0.f;
      for (int g2 = 0; g2 < NPG; ++g2) s += red[(g2 * NB + bk) * stride + slot];
      outp[e] = s;
    }
  }
}

size_t pass_c_smem(int C, int Z, int T, int mz, int mt, int LZ, int mode) {
  CLayout L = c_layout(C, Z, T, mz, mt, LZ, mode);
  size_t t = L.total;
  if (mode == EPI_BWD) {
    // the final reduction reuses the Vt tile: needs 20 floats per thread
    size_t need = size_t(CT) * 20 * sizeof(float);
    size_t have = size_t(C) * L.np * sizeof(float);
    if (need > have) t += need - have;
  }
  return t;
}

template <int LZ, int LT>
static cudaError_t launch_c(const PassCParams& p, int mode, int grid, size_t smem, cudaStream_t st) {
  void (*k)(PassCParams) = mode == EPI_U ? pass_c_kernel<LZ, LT, EPI_U>
                         : mode == EPI_FWD ? pass_c_kernel<LZ, LT, EPI_FWD>
                                           : pass_c_kernel<LZ, LT, EPI_BWD>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, CT, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_pass_c(const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem, cudaStream_t st) {
#define FNO_C_CASE(a, b) \
  if (LZ == a && LT == b) return launch_c<a, b>(p, mode, grid, smem, st);
  FNO_AC_PAIRS(FNO_C_CASE)
#undef FNO_C_CASE
  return cudaErrorInvalidValue;
}

bool ac_pair_supported(int LZ, int LT) {
#define FNO_C_CASE(a, b) \
  if (LZ == a && LT == b) return true;
  FNO_AC_PAIRS(FNO_C_CASE)
#undef FNO_C_CASE
  return false;
}

}  // namespace fno
