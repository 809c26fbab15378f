// Pass C, channel-width-specialised (bwd a9, a12):
// the same adjoint chain of I_1 = {z, t} as pass_c.cu (zero-padded inverse z,
// C2R along t with real-part semantics) fused with the DFNO block
// epilogue (Eq. dist_block)
//   fwd: z = W v + b + u, y = GELU(z)
//   bwd: dv = W^T dz + S^T dz, dW += dz v^T, db += dz    (broadcast adjoint)
// with the channel count a compile-time constant CP (C rounded up to a
// multiple of 4; padded channels carry zeros), so every channel loop unrolls
// and the 1x1 and dW contractions run as register-blocked FFMA with
// shared-memory broadcasts and no predication.
//
// Structure: small persistent CTAs (128 threads, ~100 KB of shared memory),
// two resident per SM, so one CTA's transform phases overlap the other's
// epilogue stores and TMA loads (within a CTA the phases are barrier-separated
// and were measured to add up).  Columns (b, x, y) are strided over the grid:
//   per column: phase 1 inverse t, items (c, kz', t-residue), spectrum read
//               from the slab (L2)                                  -> Bb
//   per tile (z residue rz, t chunk of TCH = 128 / LZ):
//     TMA 5-D tensor-map load of the next tile's inputs (double-buffered X)
//     phase 2 inverse z, items (c, t) -> U          ┐ no barrier in between:
//     bwd: dW / db on the tile (X only)            ┘ idle phase-2 threads start dW
//     1x1 + epilogue, items (4-point quad, output quarter)
// dW / db accumulators stay in registers for the whole kernel (a CP/2 x CP/2
// block per warp, one quad per lane per tile) and are reduced across lanes
// once at the end, in a fixed order (deterministic).
#pragma once

#include <cuda.h>

#include "kernels.cuh"
#include "launch.h"

namespace fno {

constexpr int C2T = 128;   // threads per CTA (4 warps); two CTAs per SM

// the two TMA tensor maps of the tile inputs (fwd: v; bwd: dz, v)
struct C2Maps {
  CUtensorMap m[2];
};

struct C2Layout {
  int XPS, UPS, TP, nk, QW, WROW;
  size_t ws, bias, bb, u, x0, x1, twz, twt, dmap, bar, total;
};

__host__ __device__ inline int c2_num_arrays(int mode) { return mode == EPI_FWD ? 1 : 2; }

// X tiles are dense [CP][LZ][TCH] (the TMA box layout); U rows are padded so
// the phase-2 stores of lanes (c, t) fall on distinct banks
// NX: X tile buffers (2: the next tile streams in during the whole tile; 1: it
// streams in during the epilogue, leaving room for a third CTA per SM)
__host__ __device__ inline C2Layout c2_layout(int CP, int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode,
                                              int NX) {
  C2Layout L{};
  L.nk = mz + 1;
  L.TP = T + 1;
  L.XPS = LZ * TCH;
  const int want = TCH < 32 ? TCH : 0;
  L.UPS = L.XPS + ((want - L.XPS % 32) % 32 + 32) % 32;
  L.QW = ((CP / 4) + 3) & ~3;              // one output quarter, padded to a 16-byte multiple
  L.WROW = 4 * L.QW;
  const int NA = c2_num_arrays(mode);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 127) & ~size_t(127); return o; };
  L.x0 = take(size_t(NA) * CP * L.XPS * sizeof(float));
  L.x1 = NX == 2 ? take(size_t(NA) * CP * L.XPS * sizeof(float)) : L.x0;
  L.ws = take(size_t(CP) * L.WROW * sizeof(float));
  L.bias = take(size_t(CP) * sizeof(float));
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.u = take(size_t(CP) * L.UPS * sizeof(float));
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  L.bar = take(2 * sizeof(uint64_t));
  L.total = off;
  return L;
}

// points [k0, k1) of a quad, one scalar store each
__device__ __forceinline__ void store_quad_part(float* dst, float4 r, int k0, int k1) {
  if (k0 <= 0 && k1 > 0) dst[0] = r.x;
  if (k0 <= 1 && k1 > 1) dst[1] = r.y;
  if (k0 <= 2 && k1 > 2) dst[2] = r.z;
  if (k0 <= 3 && k1 > 3) dst[3] = r.w;
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

// HALF: mz = LZ / 2 (nk = LZ / 2 + 1 at compile time: the zero z-spectrum
// inputs of the inverse z codelet fold away)
// RAG: t chunks may be ragged or phase-shifted (T % TCH != 0, row-group TMA
// view, or cp.async tiles); false compiles the full-chunk, aligned-quad case
template <int LZ, int LT, int CP, int EPI, bool HALF, bool RAG>
__global__ void __launch_bounds__(C2T, EPI == EPI_FWD ? 3 : 2) pass_c2_kernel(const __grid_constant__ C2Maps maps, const PassCParams p) {
  static_assert(CP % 4 == 0, "CP must be a multiple of 4");
  constexpr int NA = (EPI == EPI_FWD) ? 1 : 2;
  constexpr int Q4 = CP / 4;       // outputs per 1x1 item (output quarter)
  constexpr int DB = CP / 2;       // dW block: DB o-rows x DB i-columns per warp (2 x 2 warps)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt, TCH = p.TCH;
  const int NX = p.NX;
  const C2Layout L = c2_layout(CP, C, Z, T, mz, mt, LZ, TCH, EPI, NX);
  float* Ws = reinterpret_cast<float*>(smem_raw + L.ws);
  float* bs = reinterpret_cast<float*>(smem_raw + L.bias);
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
  const int per_c = 2 * mz * mt;     // slab complex per (point, channel)

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
    if (j < Q4 && o < C && k < C) w = (EPI == EPI_FWD && !p.w_t) ? p.W[o * C + k] : p.W[k * C + o];
    Ws[e] = w;
  }
  for (int o = tid; o < CP; o += C2T) bs[o] = (EPI == EPI_FWD && p.bias && o < C) ? p.bias[o] : 0.f;
  // padded channel rows of both tile buffers are never loaded: zero them once
  for (int e = tid; e < NA * (CP - C) * XPS; e += C2T) {
    const int a = e / ((CP - C) * XPS), r = e - a * (CP - C) * XPS;
    reinterpret_cast<float*>(smem_raw + L.x0)[a * CP * XPS + C * XPS + r] = 0.f;
    reinterpret_cast<float*>(smem_raw + L.x1)[a * CP * XPS + C * XPS + r] = 0.f;
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
  // retained (c, jz, kt = 0) of column c_ in the kz-owner-ordered slab
  auto slab_at = [&](long long c_, int c, int jz) -> const float2* {
    if (p.slab.P == 1) return p.in + (c_ * C + c) * per_c + jz * mt;
    const short2 dm = dmap[jz];
    const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
    return p.in + p.slab.off[dm.x] + ((c_ * C + c) * nkz + dm.y) * mt;
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
        for (int a = 0; a < NA; ++a)
          tma_load_5d(dst + a * CP * XPS, &maps.m[a], (rz % p.tma_g) * T + t0 - (((rz % p.tma_g) * T) & 3),
                      rz / p.tma_g, 0, xy, b * C, &bar[which]);
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
      const int so = c * XPS + s * TCH + vv * VW;
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        const float* src = (EPI == EPI_FWD) ? p.v : (a == 0 ? p.dy : p.v);
        float* d = dst + a * CP * XPS + so;
        if (VW == 4) cp_async16(d, src + g);
        else if (VW == 2) cp_async8(d, src + g);
        else cp_async4(d, src + g);
      }
    }
  };

  // dW / db register accumulators (bwd): warp w owns o-rows [ob*DB, ob*DB+DB)
  // and i-columns [ib*DB, ib*DB+DB)
  const int warp = tid >> 5, lane = tid & 31;
  const int ob = warp >> 1, ib = warp & 1;
  float dwa[EPI == EPI_BWD ? DB : 1][EPI == EPI_BWD ? DB : 1];
  float dba[EPI == EPI_BWD ? DB : 1];
  if (EPI == EPI_BWD) {
#pragma unroll
    for (int j = 0; j < DB; ++j) {
      dba[j] = 0.f;
#pragma unroll
      for (int i = 0; i < DB; ++i) dwa[j][i] = 0.f;
    }
  }
  // 1x1 item of this thread: quad q1, output quarter qtr1 (one item per thread)
  const int qtr1 = tid & 3, q1 = tid >> 2;
  const int s1 = q1 / QPR, tq1 = (q1 - s1 * QPR) * 4;
  const int po1 = s1 * TCH + tq1;
  const long long go1 = (long long)p.Qz * s1 * T + tq1;   // offset of the quad in a (column, rz, t0) tile
  const bool item1 = q1 < NQ;

  issue_tile(col, 0, 0);
  if (!tma) cp_commit();
  unsigned phase_bits = 0u;   // mbarrier parity of buffer b in bit b
  int buf = 0;

  for (; col < p.n_cols; col += gridDim.x) {
    const long long cbase = col_base(col);
    // ---- phase 1: inverse t (C2R weights folded in), items (c, kz', rt) ----
    // The +kz' and -kz' rows of the slab (L2-resident) are folded into one
    // complex row whose inverse t-DFT is the real z-transform's input.
    for (int it = FNO_ABL(p, 16) ? C * nk * p.Qt : tid; it < C * nk * p.Qt; it += C2T) {
      const int rt = it % p.Qt;
      const int pid = it / p.Qt;
      const int c = pid / nk, kzp = pid - c * nk;
      const float2* Sp = slab_at(col, c, kzp < mz ? kzp : 0);
      const float2* Sn = slab_at(col, c, kzp >= 1 ? 2 * mz - kzp : 0);
      float2 e[LT];
#pragma unroll
      for (int i = 0; i < LT; ++i) {
        float2 acc = make_float2(0.f, 0.f);
        if (i < mt && kzp < mz) {
          const float cw = (i == 0 || 2 * i == T) ? 1.f : 2.f;
          acc = cscale(__ldg(Sp + i), cw);
        }
        const int kt = (LT - i) % LT;
        if (kzp >= 1 && kt < mt && (i == 0 || i > LT - mt)) {
          const float cw = (kt == 0 || 2 * kt == T) ? 1.f : 2.f;
          acc = cadd(acc, cscale(cconj(__ldg(Sn + kt)), cw));
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

    for (int ti = 0; ti < tpc; ++ti) {
      const int rz = ti / nch, tc = ti - rz * nch;
      // TMA tiles of z rows with (z T) % 4 != 0 start sh points early (16-byte
      // aligned rows, c2_tile_group); the tile's valid columns are [ta, tb)
      const int sh = (RAG && tma && p.tma_g > 1) ? ((rz & (p.tma_g - 1)) * T) & 3 : 0;
      const int t0 = tc * TCH - sh;
      const int ta = RAG ? max(0, -t0) : 0, tb = RAG ? min(TCH, T - t0) : TCH, tcw = tb - ta;
      if (NX == 2) {
        if (ti + 1 < tpc) issue_tile(col, ti + 1, buf ^ 1);
        else if (col_next < p.n_cols) issue_tile(col_next, 0, buf ^ 1);
      }
      float* X = reinterpret_cast<float*>(smem_raw + (buf ? L.x1 : L.x0));
      if (tma) {
        mbar_wait(&bar[buf], (phase_bits >> buf) & 1u);   // this tile's inputs
        phase_bits ^= 1u << buf;
        if (EPI == EPI_BWD && RAG && tcw < TCH) {   // ragged t chunk (t outside [0, T): other rows or OOB): exact zeros for dW / db
          const int w = TCH - tcw;
          for (int e = tid; e < 2 * C * LZ * w; e += C2T) {
            const int a = e / (C * LZ * w), r = e - a * (C * LZ * w);
            const int row = r / w, j = r - row * w;
            const int tt = j < ta ? j : tcw + j;
            X[a * CP * XPS + row * TCH + tt] = 0.f;
          }
          fence_proxy_async();   // generic stores before the next TMA write of this buffer
          __syncthreads();
        }
      } else {
        if (NX == 2) {
          cp_commit();
          cp_wait<1>();
        } else {
          cp_wait<0>();
        }
        __syncthreads();
        if (EPI == EPI_BWD && RAG && tcw < TCH) {   // ragged t chunk: exact zeros for dW / db
          const int w = TCH - tcw;
          for (int e = tid; e < 2 * C * LZ * w; e += C2T) {
            const int a = e / (C * LZ * w), r = e - a * (C * LZ * w);
            const int row = r / w, tt = tcw + (r - row * w);
            X[a * CP * XPS + row * TCH + tt] = 0.f;
          }
          __syncthreads();
        }
      }
      // ---- phase 2: inverse z (real output), items (c, tt) -> U ----------
      for (int it = FNO_ABL(p, 1) ? C * tcw : tid; it < C * tcw; it += C2T) {
        const int c = it / tcw, tt = ta + (it - c * tcw);
        float2 e[LZ];
#pragma unroll
        for (int i = 0; i < LZ; ++i)
          e[i] = (i < (HALF ? LZ / 2 + 1 : nk)) ? Bb[(c * nk + i) * TP + t0 + tt] : make_float2(0.f, 0.f);
        float2 y[LZ];
        trunc_inv<LZ>(y, e, rz, twZ);
        float* uo = U + c * UPS + tt;
#pragma unroll
        for (int s = 0; s < LZ; ++s) uo[s * TCH] = y[s].x * p.inv_n;
      }
      // ---- bwd: dW / db on this tile (X only; no barrier after phase 2) ----
      if (EPI == EPI_BWD && !FNO_ABL(p, 8)) {
        const float* Dz = X + ob * DB * XPS;
        const float* Vv = X + CP * XPS + ib * DB * XPS;
        for (int q = lane; q < NQ; q += 32) {
          const int po = q * 4;   // quads are contiguous in the dense tile
          float4 dz4[DB];
#pragma unroll
          for (int j = 0; j < DB; ++j) dz4[j] = *reinterpret_cast<const float4*>(Dz + j * XPS + po);
          if (ib == 0) {
#pragma unroll
            for (int j = 0; j < DB; ++j) dba[j] += (dz4[j].x + dz4[j].y) + (dz4[j].z + dz4[j].w);
          }
#pragma unroll
          for (int i = 0; i < DB; ++i) {
            const float4 v4 = *reinterpret_cast<const float4*>(Vv + i * XPS + po);
#pragma unroll
            for (int j = 0; j < DB; ++j) {
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
      float4 acc[Q4];
#pragma unroll
      for (int j = 0; j < Q4; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (item1 && !FNO_ABL(p, 2)) {
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
      __syncthreads();   // U complete; X no longer read by this tile
      if (NX == 1) {       // single X buffer: the next tile streams in during the epilogue
        if (ti + 1 < tpc) issue_tile(col, ti + 1, 0);
        else if (col_next < p.n_cols) issue_tile(col_next, 0, 0);
        if (!tma) cp_commit();
      }
      // ---- epilogue: + u (+ b, GELU), stores -------------------------------
      const int k0 = RAG ? max(0, ta - tq1) : 0, k1 = RAG ? min(4, tb - tq1) : 4;   // valid points of this thread's quad
      if (item1 && k0 < k1 && !FNO_ABL(p, 4)) {
        const long long gs = cbase + rz * T + t0 + go1;
        // TMA tiles start 16-byte aligned in memory (c2_tile_group), so do their full quads
        const bool full4 = !RAG || ((vec_out || tma) && k0 == 0 && k1 == 4);
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
              if (full4) __stcs(reinterpret_cast<float4*>(zo), r);
              else store_quad_part(zo, r, k0, k1);
            }
            if (p.act_gelu) {
              r.x = gelu_f(r.x); r.y = gelu_f(r.y); r.z = gelu_f(r.z); r.w = gelu_f(r.w);
            }
          }
          if (full4) __stcs(reinterpret_cast<float4*>(out), r);
          else store_quad_part(out, r, k0, k1);
        }
      }
      __syncthreads();   // U and X[buf] free for reuse (and Bb after the last tile)
      if (NX == 2) buf ^= 1;
    }
  }
  cp_wait<0>();
  if (EPI == EPI_BWD) {
    // fixed-order butterfly reduction over the 32 lanes, then one row per CTA
    float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
#pragma unroll
    for (int j = 0; j < DB; ++j) {
#pragma unroll
      for (int i = 0; i < DB; ++i) {
        float v = dwa[j][i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        const int o = ob * DB + j, ii = ib * DB + i;
        if (lane == 0 && o < C && ii < C) outp[o * C + ii] = v;
      }
      if (ib == 0) {
        float v = dba[j];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        const int o = ob * DB + j;
        if (lane == 0 && o < C) outp[C * C + o] = v;
      }
    }
  }
}

template <int LZ, int LT, int CP>
cudaError_t launch_c2_cp(const C2Maps& maps, const PassCParams& p, int mode, int grid, size_t smem, cudaStream_t st) {
  const bool half = 2 * p.mz == LZ;
  const bool rag = !p.use_tma || p.tma_g != 1 || p.T % p.TCH != 0 || p.T % 4 != 0;
  void (*k)(C2Maps, PassCParams) =
      rag ? (mode == EPI_FWD ? (half ? pass_c2_kernel<LZ, LT, CP, EPI_FWD, true, true> : pass_c2_kernel<LZ, LT, CP, EPI_FWD, false, true>)
                             : (half ? pass_c2_kernel<LZ, LT, CP, EPI_BWD, true, true> : pass_c2_kernel<LZ, LT, CP, EPI_BWD, false, true>))
          : (mode == EPI_FWD ? (half ? pass_c2_kernel<LZ, LT, CP, EPI_FWD, true, false> : pass_c2_kernel<LZ, LT, CP, EPI_FWD, false, false>)
                             : (half ? pass_c2_kernel<LZ, LT, CP, EPI_BWD, true, false> : pass_c2_kernel<LZ, LT, CP, EPI_BWD, false, false>));
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, C2T, smem, st>>>(maps, p);
  return cudaGetLastError();
}

// TMA tensor map of a tile input: (T, Qz, LZ, Xl*Yl, B*C) view of an NCXYZT
// field, box [C][1][LZ][1][p.TCH] (pass_c2.cu)
bool c2_encode_tile_map(CUtensorMap* m, const float* base, const PassCParams& p, int LZ);
int c2_tile_group(const PassCParams& p, int LZ, const float* base);

// per-width entry points (one translation unit per CP: pass_c2_cp<CP>.cu)
cudaError_t launch_pass_c2_cp4(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                               cudaStream_t st);
cudaError_t launch_pass_c2_cp8(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem,
                               cudaStream_t st);
cudaError_t launch_pass_c2_cp12(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid,
                                size_t smem, cudaStream_t st);
cudaError_t launch_pass_c2_cp16(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid,
                                size_t smem, cudaStream_t st);
cudaError_t launch_pass_c2_cp20(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int mode, int grid,
                                size_t smem, cudaStream_t st);

}  // namespace fno
