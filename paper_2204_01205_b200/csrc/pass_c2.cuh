// Pass C, channel-width-specialised (bwd a9, a12):
// the same adjoint chain of I_1 = {z, t} as pass_c.cu (zero-padded inverse z,
// C2R along t with real-part semantics) fused with the DFNO block
// epilogue (Eq. dist_block)
//   fwd: z = W v + b + u, y = GELU(z)
//   bwd: dv = W^T dz + S^T dz, dW += dz v^T, db += dz    (broadcast adjoint)
// but with the channel count a compile-time constant CP (C rounded up to a
// multiple of 4; padded channels carry zeros), so every channel loop unrolls
// and the 1x1 and dW contractions run as register-blocked FFMA with
// shared-memory broadcasts and no predication.
//
// Structure (one persistent 256-thread CTA per SM, columns (b, x, y) strided
// over the grid):
//   per column: phase 1 inverse t, items (c, kz', t-residue)   -> Bb
//   per tile (z residue rz, t chunk):
//     cp.async of the next tile's inputs          (double-buffered X)
//     phase 2 inverse z, items (c, t) -> U          ┐ no barrier in between:
//     bwd: dW / db on the tile (X only)            ┘ idle phase-2 threads start dW
//     1x1 + epilogue, items (4-point quad, output quarter)
// dW / db accumulators stay in registers for the whole kernel (one 4-row x
// CP/2-column block per warp, lanes over the tile's quads) and are reduced
// across lanes once at the end, in a fixed order (deterministic).
#pragma once

#include <cuda.h>

#include "kernels.cuh"
#include "launch.h"

namespace fno {

constexpr int C2T = 256;   // threads per CTA (8 warps)

// the two TMA tensor maps of the tile inputs (fwd: v; bwd: dz, v)
struct C2Maps {
  CUtensorMap m[2];
};

struct C2Layout {
  int XPS, UPS, TP, nk, QW, WROW;
  size_t ws, bias, s, bb, u, x0, x1, twz, twt, dmap, bar, total;
};

__host__ __device__ inline int c2_num_arrays(int mode) { return mode == EPI_FWD ? 1 : 2; }

// X tiles are dense [CP][LZ][TCH] (the TMA box layout); U rows are padded so
// the phase-2 stores of lanes (c, t) fall on distinct banks
// XR: channel rows of the X tiles (CP, or CP rounded up to 8 for the tensor-core
// 1x1 whose k-steps are 8 channels wide)
__host__ __device__ inline C2Layout c2_layout(int CP, int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode,
                                              int XR) {
  C2Layout L{};
  L.nk = mz + 1;
  L.TP = T + 1;
  L.XPS = LZ * TCH;
  // mma epilogue reads U rows g (+8) at 2t: conflict-free when UPS = 8 mod 32;
  // the FFMA epilogue wants the phase-2 stores conflict-free (UPS = TCH mod 32)
  const int want = XR != CP ? 8 : (TCH < 32 ? TCH : 0);
  L.UPS = L.XPS + ((want - L.XPS % 32) % 32 + 32) % 32;
  L.QW = ((CP / 4) + 3) & ~3;              // one output quarter, padded to a 16-byte multiple
  L.WROW = 4 * L.QW;
  const int NA = c2_num_arrays(mode);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 127) & ~size_t(127); return o; };
  L.x0 = take(size_t(NA) * XR * L.XPS * sizeof(float));
  L.x1 = take(size_t(NA) * XR * L.XPS * sizeof(float));
  L.ws = take(size_t(CP) * L.WROW * sizeof(float));
  L.bias = take(size_t(CP) * sizeof(float));
  L.s = take(size_t(C) * 2 * mz * mt * sizeof(float2));
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.u = take(size_t(CP) * L.UPS * sizeof(float));
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  L.bar = take(2 * sizeof(uint64_t));
  L.total = off;
  return L;
}

__device__ __forceinline__ float4 f4fma(float w, float4 x, float4 a) {
  a.x = fmaf(w, x.x, a.x); a.y = fmaf(w, x.y, a.y); a.z = fmaf(w, x.z, a.z); a.w = fmaf(w, x.w, a.w);
  return a;
}

// 5-D TMA tile load (box [C][1][LZ][1][TCH] of the (T, Qz, LZ, Xl*Yl, B*C) view)
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

// ---- legacy warp-level tensor-core MMA (HMMA) helpers ----------------------
// fp32-accurate products from a tf32 hi*hi MMA plus one bf16 MMA carrying both
// cross terms hi*lo and lo*hi (K-concatenated): x = hi + lo with hi = tf32(x)
// exact and |lo| <= 2^-11 |x|, so the bf16 rounding of the cross terms costs
// ~2^-19 relative and the dropped lo*lo term 2^-22.
__device__ __forceinline__ uint32_t tf32_of(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// two bf16 in one register: k-order element k0 in the low half
__device__ __forceinline__ uint32_t bf16x2_of(float k0, float k1) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(k1), "f"(k0));
  return r;
}
__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16_16x8x16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int LZ, int LT, int CP, int EPI, bool MMA>
__global__ void __launch_bounds__(C2T, 1) pass_c2_kernel(const __grid_constant__ C2Maps maps, const PassCParams p) {
  static_assert(CP % 4 == 0, "CP must be a multiple of 4");
  constexpr int NA = (EPI == EPI_FWD) ? 1 : 2;
  constexpr int Q4 = CP / 4;       // outputs per quarter (1x1) and o-rows per dW block
  constexpr int IB = CP / 2;       // i-columns per dW block
  constexpr int XR = MMA ? ((CP + 7) & ~7) : CP;   // X tile rows (zero beyond C)
  constexpr int KS = XR / 8;       // mma k-steps
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt, TCH = p.TCH;
  const C2Layout L = c2_layout(CP, C, Z, T, mz, mt, LZ, TCH, EPI, XR);
  float* Ws = reinterpret_cast<float*>(smem_raw + L.ws);
  float* bs = reinterpret_cast<float*>(smem_raw + L.bias);
  float2* S = reinterpret_cast<float2*>(smem_raw + L.s);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float* U = reinterpret_cast<float*>(smem_raw + L.u);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  const int tid = threadIdx.x;
  const int nk = L.nk, TP = L.TP, XPS = L.XPS, UPS = L.UPS, QW = L.QW, WROW = L.WROW;
  const long long ZT = (long long)Z * T;
  const long long chan_stride = (long long)p.Xl * p.Yl * ZT;
  const int nch = (T + TCH - 1) / TCH;
  const int tpc = p.Qz * nch;        // tiles per column
  const int QPR = TCH / 4;           // quads per tile row
  const int NQ = LZ * QPR;           // quads per tile (4 * NQ <= C2T by construction)
  const bool vec_out = (T % 4) == 0; // 16-byte aligned output quads
  const bool tma = p.use_tma != 0;
  const unsigned tile_bytes = unsigned(C) * LZ * TCH * sizeof(float);

  long long col = blockIdx.x;
  if (col >= p.n_cols) return;

  fill_combine_table(twZ, LZ, p.Qz, Z, 0, +1, tid, C2T);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, +1, tid, C2T);
  for (int j = tid; j < 2 * mz; j += C2T) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  // Ws[k][q*QW + j] = weight of contraction index k for output q*Q4 + j:
  // fwd k = input channel (W^T), bwd k = output channel of the layer (W)
  for (int e = tid; e < CP * WROW; e += C2T) {
    const int k = e / WROW, r = e - k * WROW;
    const int q = r / QW, j = r - q * QW;
    const int o = q * Q4 + j;
    float w = 0.f;
    if (j < Q4 && o < C && k < C) w = (EPI == EPI_FWD) ? p.W[o * C + k] : p.W[k * C + o];
    Ws[e] = w;
  }
  for (int o = tid; o < CP; o += C2T) bs[o] = (EPI == EPI_FWD && p.bias && o < C) ? p.bias[o] : 0.f;
  // padded channel rows of both tile buffers are never loaded: zero them once
  for (int e = tid; e < NA * (XR - C) * XPS; e += C2T) {
    const int a = e / ((XR - C) * XPS), r = e - a * (XR - C) * XPS;
    reinterpret_cast<float*>(smem_raw + L.x0)[a * XR * XPS + C * XPS + r] = 0.f;
    reinterpret_cast<float*>(smem_raw + L.x1)[a * XR * XPS + C * XPS + r] = 0.f;
  }
  if (tid == 0 && tma) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto col_split = [&](long long c_, int* b_out) {   // column -> (batch, xl*Yl + yl)
    const unsigned cu = unsigned(c_);
    const unsigned per_b = unsigned(p.Xl) * unsigned(p.Yl);
    *b_out = int(cu / per_b);
    return int(cu - unsigned(*b_out) * per_b);
  };
  auto col_base = [&](long long c_) {
    int b;
    const int xy = col_split(c_, &b);
    return (long long)b * C * chan_stride + (long long)xy * ZT;
  };
  auto issue_slab = [&](long long c_) {
    const int per_c = 2 * mz * mt;
    if (p.slab.P == 1 && (per_c & 1) == 0) {
      const float2* src = p.in + c_ * C * per_c;
      for (int e = tid; e < C * per_c / 2; e += C2T) cp_async16(S + 2 * e, src + 2 * e);
      return;
    }
    for (int e = tid; e < C * per_c; e += C2T) {
      const int c = e / per_c, rem = e - c * per_c;
      const int jz = rem / mt, kt = rem - jz * mt;
      const short2 dm = dmap[jz];
      const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
      cp_async8(S + e, p.in + p.slab.off[dm.x] + ((c_ * C + c) * nkz + dm.y) * mt + kt);
    }
  };
  // tile ti of column c_ into buffer `which`: one TMA per input (thread 0), or
  // cp.async by all threads
  auto issue_tile = [&](long long c_, int ti, int which) {
    float* dst = reinterpret_cast<float*>(smem_raw + (which ? L.x1 : L.x0));
    const int rz = ti / nch, tc = ti - rz * nch;
    const int t0 = tc * TCH;
    if (tma) {
      if (tid == 0) {
        int b;
        const int xy = col_split(c_, &b);
        mbar_expect_tx(&bar[which], tile_bytes * NA);
#pragma unroll
        for (int a = 0; a < NA; ++a) tma_load_5d(dst + a * XR * XPS, &maps.m[a], t0, rz, 0, xy, b * C, &bar[which]);
      }
      return;
    }
    const long long base = col_base(c_) + rz * T + t0;
    const int tcw = min(TCH, T - t0);
    const int VW = p.VW;
    const int nvec = (tcw + VW - 1) / VW;
    const int rows = C * LZ;
    for (int e = tid; e < rows * nvec; e += C2T) {
      const int row = e / nvec, vv = e - row * nvec;
      const int c = row / LZ, s = row - c * LZ;
      const long long g = base + c * chan_stride + (long long)p.Qz * s * T + vv * VW;
      const int so = c * XPS + s * TCH + vv * VW;   // + a * XR * XPS per input
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        const float* src = (EPI == EPI_FWD) ? p.v : (a == 0 ? p.dy : p.v);
        float* d = dst + a * XR * XPS + so;
        if (VW == 4) cp_async16(d, src + g);
        else if (VW == 2) cp_async8(d, src + g);
        else cp_async4(d, src + g);
      }
    }
  };

  // dW / db register accumulators (bwd): warp w owns o-rows [ob*Q4, ob*Q4+Q4)
  // and i-columns [ib*IB, ib*IB+IB)
  const int warp = tid >> 5, lane = tid & 31;
  const int ob = warp >> 1, ib = warp & 1;
  float dwa[EPI == EPI_BWD ? Q4 : 1][EPI == EPI_BWD ? IB : 1];
  float dba[EPI == EPI_BWD ? Q4 : 1];
  if (EPI == EPI_BWD) {
#pragma unroll
    for (int j = 0; j < Q4; ++j) {
      dba[j] = 0.f;
#pragma unroll
      for (int i = 0; i < IB; ++i) dwa[j][i] = 0.f;
    }
  }
  // 1x1 item of this thread: quad q1, output quarter qtr1 (one item per thread)
  const int qtr1 = tid & 3, q1 = tid >> 2;
  const int s1 = q1 / QPR, tq1 = (q1 - s1 * QPR) * 4;
  const int po1 = s1 * TCH + tq1;
  const bool item1 = q1 < NQ;
  // tensor-core 1x1: A[m][k] = Ws[k][m] (fwd m = o, k = i; bwd m = i, k = o),
  // 2 m-tiles x KS k-steps, tf32 hi fragments + bf16 (hi | lo) cross fragments
  const int g = lane >> 2, t4 = lane & 3;
  uint32_t ahi[MMA ? 2 : 1][MMA ? KS : 1][4], acr[MMA ? 2 : 1][MMA ? KS : 1][4];
  const int NJ8 = (LZ * TCH / 8 + 7) / 8;   // n8 point tiles per warp
  // per-thread epilogue points of the mma path (fixed across tiles): tile point
  // pp = 8 (warp NJ8 + jj) + 2 t4 = (s, tt) and its offset Qz s T + tt in a column
  int epp[4], eoff[4], ett[4];
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    epp[jj] = 8 * (warp * NJ8 + jj) + 2 * t4;
    const int s = epp[jj] / TCH;
    ett[jj] = epp[jj] - s * TCH;
    eoff[jj] = p.Qz * s * T + ett[jj];
  }
  if constexpr (MMA) {
#pragma unroll
    for (int mt2 = 0; mt2 < 2; ++mt2)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        float av[2][2];   // [row +0/+8][col +0/+4]
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c4 = 0; c4 < 2; ++c4) {
            const int m = 16 * mt2 + g + 8 * h, k = 8 * ks + t4 + 4 * c4;
            av[h][c4] = (m < CP && k < CP) ? Ws[k * WROW + (m / Q4) * QW + (m % Q4)] : 0.f;
          }
        ahi[mt2][ks][0] = tf32_of(av[0][0]);
        ahi[mt2][ks][1] = tf32_of(av[1][0]);
        ahi[mt2][ks][2] = tf32_of(av[0][1]);
        ahi[mt2][ks][3] = tf32_of(av[1][1]);
        float lo[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c4 = 0; c4 < 2; ++c4) lo[h][c4] = av[h][c4] - __uint_as_float(tf32_of(av[h][c4]));
        acr[mt2][ks][0] = bf16x2_of(av[0][0], av[0][1]);
        acr[mt2][ks][1] = bf16x2_of(av[1][0], av[1][1]);
        acr[mt2][ks][2] = bf16x2_of(lo[0][0], lo[0][1]);
        acr[mt2][ks][3] = bf16x2_of(lo[1][0], lo[1][1]);
      }
  }

  issue_slab(col);
  cp_commit();
  issue_tile(col, 0, 0);
  if (!tma) cp_commit();
  unsigned phase_bits = 0u;   // mbarrier parity of buffer b in bit b
  int buf = 0;

  for (; col < p.n_cols; col += gridDim.x) {
    const long long cbase = col_base(col);
    if (tma) cp_wait<0>();
    else cp_wait<1>();   // this column's spectrum (its first tile may still fly)
    __syncthreads();
    // ---- phase 1: inverse t (C2R weights folded in), items (c, kz', rt) ----
    for (int it = (p.ablate & 16) ? C * nk * p.Qt : tid; it < C * nk * p.Qt; it += C2T) {
      const int rt = it % p.Qt;
      const int pid = it / p.Qt;
      const int c = pid / nk, kzp = pid - c * nk;
      const float2* Sp = S + (c * 2 * mz + kzp) * mt;
      const float2* Sn = S + (c * 2 * mz + (2 * mz - kzp)) * mt;
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
      float2 y[LT];
      trunc_inv<LT>(y, e, rt, twT);
      float2* bo = Bb + (c * nk + kzp) * TP + rt;
#pragma unroll
      for (int s = 0; s < LT; ++s) bo[p.Qt * s] = y[s];
    }
    __syncthreads();
    const long long col_next = col + gridDim.x;
    if (col_next < p.n_cols) issue_slab(col_next);   // S is free now
    cp_commit();

    for (int ti = 0; ti < tpc; ++ti) {
      const int rz = ti / nch, tc = ti - rz * nch;
      const int t0 = tc * TCH;
      const int tcw = min(TCH, T - t0);
      if (ti + 1 < tpc) issue_tile(col, ti + 1, buf ^ 1);
      else if (col_next < p.n_cols) issue_tile(col_next, 0, buf ^ 1);
      float* X = reinterpret_cast<float*>(smem_raw + (buf ? L.x1 : L.x0));
      if (tma) {
        mbar_wait(&bar[buf], (phase_bits >> buf) & 1u);   // this tile's inputs (OOB t zero-filled)
        phase_bits ^= 1u << buf;
      } else {
        cp_commit();
        if (ti == 0) cp_wait<2>();          // the next spectrum was committed after this tile
        else cp_wait<1>();
        __syncthreads();
        if (EPI == EPI_BWD && tcw < TCH) {   // ragged t chunk: exact zeros for dW / db
          const int w = TCH - tcw;
          for (int e = tid; e < 2 * C * LZ * w; e += C2T) {
            const int a = e / (C * LZ * w), r = e - a * (C * LZ * w);
            const int row = r / w, tt = tcw + (r - row * w);
            X[a * XR * XPS + row * TCH + tt] = 0.f;
          }
          __syncthreads();
        }
      }
      // ---- phase 2: inverse z (real output), items (c, tt) -> U ----------
      for (int it = (p.ablate & 1) ? C * tcw : tid; it < C * tcw; it += C2T) {
        const int c = it / tcw, tt = it - c * tcw;
        float2 e[LZ];
#pragma unroll
        for (int i = 0; i < LZ; ++i) e[i] = (i < nk) ? Bb[(c * nk + i) * TP + t0 + tt] : make_float2(0.f, 0.f);
        float2 y[LZ];
        trunc_inv<LZ>(y, e, rz, twZ);
        float* uo = U + c * UPS + tt;
#pragma unroll
        for (int s = 0; s < LZ; ++s) uo[s * TCH] = y[s].x * p.inv_n;
      }
      // ---- bwd: dW / db on this tile (X only; no barrier after phase 2) ----
      if (EPI == EPI_BWD && !(p.ablate & 8)) {
        const float* Dz = X;
        const float* Vv = X + XR * XPS;
        for (int q = lane; q < NQ; q += 32) {
          const int po = q * 4;   // quads are contiguous in the dense tile
          float4 dz4[Q4];
#pragma unroll
          for (int j = 0; j < Q4; ++j) dz4[j] = *reinterpret_cast<const float4*>(Dz + (ob * Q4 + j) * XPS + po);
          if (ib == 0) {
#pragma unroll
            for (int j = 0; j < Q4; ++j) dba[j] += (dz4[j].x + dz4[j].y) + (dz4[j].z + dz4[j].w);
          }
#pragma unroll
          for (int i = 0; i < IB; ++i) {
            const float4 v4 = *reinterpret_cast<const float4*>(Vv + (ib * IB + i) * XPS + po);
#pragma unroll
            for (int j = 0; j < Q4; ++j) {
              float a = dwa[j][i];
              a = fmaf(dz4[j].x, v4.x, a);
              a = fmaf(dz4[j].y, v4.y, a);
              a = fmaf(dz4[j].z, v4.z, a);
              a = fmaf(dz4[j].w, v4.w, a);
              dwa[j][i] = a;
            }
          }
        }
      }
      // ---- 1x1 channel linear (X only) ------------------------------------
      float macc[MMA ? 4 : 1][2][4];   // [n8 tile of this warp][m-tile][frag]
      if constexpr (MMA) {
        // 4 n8 point tiles x 2 m-tiles = 8 independent accumulators per warp;
        // per k-step all B fragments are loaded first, then 8 tf32 + 8 bf16 MMAs
        const int jb = warp * NJ8;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int mt2 = 0; mt2 < 2; ++mt2)
#pragma unroll
            for (int e = 0; e < 4; ++e) macc[jj][mt2][e] = 0.f;
        if (NJ8 == 4 && 8 * (jb + 3) < LZ * TCH) {
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            uint32_t bh[4][2], bc[4][2];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const float* xb = X + 8 * (jb + jj) + g;
              const float x0 = xb[(8 * ks + t4) * XPS], x1 = xb[(8 * ks + t4 + 4) * XPS];
              bh[jj][0] = tf32_of(x0);
              bh[jj][1] = tf32_of(x1);
              bc[jj][0] = bf16x2_of(x0 - __uint_as_float(bh[jj][0]), x1 - __uint_as_float(bh[jj][1]));
              bc[jj][1] = bf16x2_of(x0, x1);
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int mt2 = 0; mt2 < 2; ++mt2) mma_tf32_16x8x8(macc[jj][mt2], ahi[mt2][ks], bh[jj][0], bh[jj][1]);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int mt2 = 0; mt2 < 2; ++mt2) mma_bf16_16x8x16(macc[jj][mt2], acr[mt2][ks], bc[jj][0], bc[jj][1]);
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            if (jj >= NJ8 || 8 * (jb + jj) >= LZ * TCH) continue;
            const float* xb = X + 8 * (jb + jj) + g;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              const float x0 = xb[(8 * ks + t4) * XPS], x1 = xb[(8 * ks + t4 + 4) * XPS];
              const uint32_t h0 = tf32_of(x0), h1 = tf32_of(x1);
              const uint32_t c0 = bf16x2_of(x0 - __uint_as_float(h0), x1 - __uint_as_float(h1)), c1 = bf16x2_of(x0, x1);
#pragma unroll
              for (int mt2 = 0; mt2 < 2; ++mt2) {
                mma_tf32_16x8x8(macc[jj][mt2], ahi[mt2][ks], h0, h1);
                mma_bf16_16x8x16(macc[jj][mt2], acr[mt2][ks], c0, c1);
              }
            }
          }
        }
      }
      float4 acc[Q4];
#pragma unroll
      for (int j = 0; j < Q4; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!MMA && item1 && !(p.ablate & 2)) {
        const float* wq = Ws + qtr1 * QW;
#pragma unroll
        for (int k = 0; k < CP; ++k) {
          const float4 x4 = *reinterpret_cast<const float4*>(X + k * XPS + po1);
          float w[Q4 + 4];
#pragma unroll
          for (int j4 = 0; j4 < Q4; j4 += 4) {
            const float4 ww = *reinterpret_cast<const float4*>(wq + k * WROW + j4);
            w[j4] = ww.x; w[j4 + 1] = ww.y; w[j4 + 2] = ww.z; w[j4 + 3] = ww.w;
          }
#pragma unroll
          for (int j = 0; j < Q4; ++j) acc[j] = f4fma(w[j], x4, acc[j]);
        }
      }
      __syncthreads();   // U complete
      // ---- epilogue: + u (+ b, GELU), stores -------------------------------
      if constexpr (MMA) {
        // fast path: full t chunk, even T (8-byte stores), all 4 n8 tiles live
        const bool fast = tcw == TCH && (T % 2) == 0 && NJ8 == 4 && 8 * (warp * 4 + 3) < LZ * TCH;
        const long long tb = cbase + rz * T + t0;
        const bool zs = EPI == EPI_FWD && p.zsave != nullptr;
        const bool act = EPI == EPI_FWD && p.act_gelu;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j8 = warp * NJ8 + jj;
          if (!fast && (jj >= NJ8 || 8 * j8 >= LZ * TCH)) continue;
          const int pp = epp[jj], tt = ett[jj];    // tile point (s, tt), tt even
          if (!fast && tt >= tcw) continue;
          const bool two = fast || tt + 1 < tcw;
          const long long gs = tb + eoff[jj];
#pragma unroll
          for (int mt2 = 0; mt2 < 2; ++mt2)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int o = 16 * mt2 + g + 8 * h;
              if (16 * mt2 + 8 * h >= CP) continue;   // whole row group beyond the padded width
              if (o >= C) continue;
              const float2 u2 = *reinterpret_cast<const float2*>(U + o * UPS + pp);
              float r0 = macc[jj][mt2][2 * h] + u2.x, r1 = macc[jj][mt2][2 * h + 1] + u2.y;
              float* out = p.out + gs + o * chan_stride;
              if (EPI == EPI_FWD) {
                const float bo = bs[o];
                r0 += bo; r1 += bo;
                if (zs) {
                  float* zo = p.zsave + gs + o * chan_stride;
                  if (fast) __stcs(reinterpret_cast<float2*>(zo), make_float2(r0, r1));
                  else { zo[0] = r0; if (two) zo[1] = r1; }
                }
                if (act) { r0 = gelu_f(r0); r1 = gelu_f(r1); }
              }
              if (fast) __stcs(reinterpret_cast<float2*>(out), make_float2(r0, r1));
              else { out[0] = r0; if (two) out[1] = r1; }
            }
        }
      }
      if (!MMA && item1 && tq1 < tcw && !(p.ablate & 4)) {
        const long long gs = cbase + rz * T + t0 + (long long)p.Qz * s1 * T + tq1;
        const int nv = min(4, tcw - tq1);
#pragma unroll
        for (int j = 0; j < Q4; ++j) {
          const int o = qtr1 * Q4 + j;
          if (o >= C) break;
          const float4 u4 = *reinterpret_cast<const float4*>(U + o * UPS + po1);
          float4 r = make_float4(acc[j].x + u4.x, acc[j].y + u4.y, acc[j].z + u4.z, acc[j].w + u4.w);
          float* out = p.out + gs + o * chan_stride;
          if (EPI == EPI_FWD) {
            const float bo = bs[o];
            r.x += bo; r.y += bo; r.z += bo; r.w += bo;
            if (p.zsave) {
              float* zo = p.zsave + gs + o * chan_stride;
              if (vec_out && nv == 4) __stcs(reinterpret_cast<float4*>(zo), r);
              else {
                zo[0] = r.x;
                if (nv > 1) zo[1] = r.y;
                if (nv > 2) zo[2] = r.z;
                if (nv > 3) zo[3] = r.w;
              }
            }
            if (p.act_gelu) {
              r.x = gelu_f(r.x); r.y = gelu_f(r.y); r.z = gelu_f(r.z); r.w = gelu_f(r.w);
            }
          }
          if (vec_out && nv == 4) __stcs(reinterpret_cast<float4*>(out), r);
          else {
            out[0] = r.x;
            if (nv > 1) out[1] = r.y;
            if (nv > 2) out[2] = r.z;
            if (nv > 3) out[3] = r.w;
          }
        }
      }
      __syncthreads();   // U and X[buf] free for reuse
      buf ^= 1;
    }
  }
  cp_wait<0>();
  if (EPI == EPI_BWD) {
    // fixed-order butterfly reduction over the 32 lanes, then one row per CTA
    float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
#pragma unroll
    for (int j = 0; j < Q4; ++j) {
#pragma unroll
      for (int i = 0; i < IB; ++i) {
        float v = dwa[j][i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        const int o = ob * Q4 + j, ii = ib * IB + i;
        if (lane == 0 && o < C && ii < C) outp[o * C + ii] = v;
      }
      if (ib == 0) {
        float v = dba[j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        const int o = ob * Q4 + j;
        if (lane == 0 && o < C) outp[C * C + o] = v;
      }
    }
  }
}

template <int LZ, int LT, int CP>
cudaError_t launch_c2_cp(const C2Maps& maps, const PassCParams& p, int mode, int grid, size_t smem, cudaStream_t st) {
  // tensor-core 1x1 when the tile rows split into n8 point tiles (TCH % 8 == 0)
  const bool mma = CP >= 8 && p.TCH % 8 == 0 && p.use_mma;
  void (*k)(C2Maps, PassCParams) =
      mode == EPI_FWD ? (mma ? pass_c2_kernel<LZ, LT, CP, EPI_FWD, (CP >= 8)> : pass_c2_kernel<LZ, LT, CP, EPI_FWD, false>)
                      : (mma ? pass_c2_kernel<LZ, LT, CP, EPI_BWD, (CP >= 8)> : pass_c2_kernel<LZ, LT, CP, EPI_BWD, false>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, C2T, smem, st>>>(maps, p);
  return cudaGetLastError();
}

// per-width entry points (one translation unit per CP: pass_c2_cp<CP>.cu)
cudaError_t launch_pass_c2_cp4(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                                cudaStream_t st);
cudaError_t launch_pass_c2_cp8(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                                cudaStream_t st);
cudaError_t launch_pass_c2_cp12(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                                cudaStream_t st);
cudaError_t launch_pass_c2_cp16(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                                cudaStream_t st);
cudaError_t launch_pass_c2_cp20(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                                cudaStream_t st);
cudaError_t launch_pass_c2_cp24(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                                cudaStream_t st);

}  // namespace fno
