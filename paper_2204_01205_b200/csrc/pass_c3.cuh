// Pass C with the 1x1 channel linear on the 5th-generation tensor cores
// (the north star's "tensor cores ... for the 1x1
// channel linear").  Same adjoint chain of I_1 = {z, t} as pass_c2.cuh
// (zero-padded inverse z, C2R along t with real-part semantics),
// fused with the DFNO block epilogue (Eq. dist_block)
//   z = W v + b + u,   y = GELU(z)
// but the contraction W v (+ b) runs as tcgen05.mma kind::tf32 with the fp32
// accumulator in TMEM instead of 20 FFMA per element on the FP32 pipe, which
// the pass_c2 profile showed to be issue-bound (SURVEY Appendix B budget).
//
// fp32 accuracy from tf32 operands (3xTF32): every operand is split x = hi + lo
// with hi exactly representable in tf32 (low 13 mantissa bits cleared) and
// lo = x - hi (exact in fp32), and D = A_hi B_hi + A_lo B_hi + A_hi B_lo; the
// dropped lo*lo term is below 2^-22 relative.  The bias rides along as an extra
// K column: A[p][CP] = 1, B[o][CP] = b[o].
//
// Tile = one z residue class rz (LZ points s) x TCH = 128 / LZ consecutive t,
// i.e. exactly M = 128 points = the 128 TMEM lanes.  The CTA is
// warp-specialised so the transform and the epilogue of consecutive tiles
// overlap (pass_c2 runs them back to back between CTA-wide barriers):
//   transform warps (4..):  per column phase 1 (inverse t of the slab, -> Bb);
//                           per tile phase 2 (inverse z, -> U[k & 1])
//   epilogue warps (0-3):   per tile: wait the TMA'd v tile X, split it into
//                           the K-major tf32 hi / lo operands, one thread
//                           issues the next tile's TMA and 3 x KP/8 UMMAs
//                           (M128 x NP x K8) into TMEM; then, per TMEM lane
//                           (= point), z = D row + U, GELU, float4 stores
// v tiles arrive by one TMA 5-D tensor-map load (kernel TMA = true; when
// T % 4 != 0 the view's rows are groups of G = 2 or 4 z rows, so its strides
// stay 16-byte multiples -- c2_tile_group), else by cp.async row pieces issued
// by the transform warps.  The columns t >= T of a ragged last t chunk (the
// next row of the group, or TMA zero fill) are computed but never stored.
// U and the TMEM accumulator are double-buffered with full / empty mbarriers
// between the two groups.  (Measured alternatives, slower at c2: more v-tile
// stages paid for by holding Bb for half the t range at a time -- DRAM line
// locality and register spills cost more than the deeper TMA pipeline won.)
#pragma once

#include <cuda.h>

#include "kernels.cuh"
#include "launch.h"
#include "pass_c2.cuh"
#include "umma.cuh"

namespace fno {

constexpr int C3T = 128;   // tile points = M = TMEM lanes = epilogue threads (warps 0-3)

// transform threads: one phase-2 item (c, t) each when that fits in 4-5 warps
#ifndef FNO_C3_EXTRA
#define FNO_C3_EXTRA 32   // one more transform warp: the operand split and phase 1 spread wider (c2 fwd 0.664 -> 0.627 ms)
#endif
__host__ __device__ constexpr int c3_transform_threads(int CP, int LZ) {
#ifdef FNO_C3_NTT
  return FNO_C3_NTT;
#endif
  return FNO_C3_EXTRA + ((CP * (C3T / LZ) + 31) / 32 * 32 > 160 ? 128
         : ((CP * (C3T / LZ) + 31) / 32 * 32 < 128 ? 128 : (CP * (C3T / LZ) + 31) / 32 * 32));
}
__host__ __device__ constexpr int c3_threads(int CP, int LZ) { return C3T + c3_transform_threads(CP, LZ); }



struct C3Layout {
  int KP, NP, UPS, TP, nk, TCH;
  size_t x, ahi, alo, bhi, blo, bb, u0, u1, twz, twt, dmap, bar, slot, total;
};

// KP: K = CP channels + the bias column, rounded up to the UMMA K step (8 tf32)
// NP: N = output channels rounded up to 16 (M = 128 needs N % 16 == 0)
__host__ __device__ inline C3Layout c3_layout(int CP, int C, int Z, int T, int mz, int mt, int LZ) {
  C3Layout L{};
  L.KP = (CP + 1 + 7) & ~7;
  L.NP = (CP + 15) & ~15;
  L.TCH = C3T / LZ;
  L.nk = mz + 1;
  L.TP = T + 1;
  L.UPS = C3T + (L.TCH < 32 ? L.TCH : 0);   // phase-2 stores of lanes (c, t) on distinct banks
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 127) & ~size_t(127); return o; };
  L.x = take(size_t(CP) * C3T * sizeof(float));
  L.ahi = take(size_t(C3T) * L.KP * sizeof(float));
  L.alo = take(size_t(C3T) * L.KP * sizeof(float));
  L.bhi = take(size_t(L.NP) * L.KP * sizeof(float));
  L.blo = take(size_t(L.NP) * L.KP * sizeof(float));
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.u0 = take(size_t(CP) * L.UPS * sizeof(float));
  L.u1 = take(size_t(CP) * L.UPS * sizeof(float));
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  L.bar = take(7 * sizeof(uint64_t));
  L.slot = take(sizeof(uint32_t));
  L.total = off;
  return L;
}

// K-major core-matrix layout (SWIZZLE_NONE): 8 rows x 4 tf32 (16 B) per core
// matrix, core matrices ordered [k / 4][row / 8]; ROWS rows in total
template <int ROWS>
__device__ __forceinline__ int kmaj_off(int row, int k) {
  return ((k >> 2) * (ROWS / 8) + (row >> 3)) * 32 + (row & 7) * 4 + (k & 3);
}

__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// barrier among the `n` threads of one warp group (ids 1, 2; 0 is __syncthreads)
__device__ __forceinline__ void group_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// RAG: t chunks may be ragged or phase-shifted (T % TCH != 0, row-group TMA
// view, or cp.async tiles); false compiles the full-chunk, aligned-quad case
template <int LZ, int LT, int CP, bool HALF, bool TMA, bool RAG>
__global__ void __launch_bounds__(c3_threads(CP, LZ), 2) pass_c3_fwd_kernel(const __grid_constant__ C2Maps maps, const PassCParams p) {
  static_assert(CP % 4 == 0 && CP <= 32 && (CP + 15) / 16 * 16 <= 32, "CP must be a multiple of 4, at most 32");
  static_assert(C3T % LZ == 0 && C3T / LZ >= 4, "LZ must divide the 128 tile points, TCH >= 4");
  constexpr int TCH = C3T / LZ;
  constexpr int KP = (CP + 1 + 7) & ~7;
  constexpr int NP = (CP + 15) & ~15;
  constexpr int NCH = (CP + 7) / 8;          // 8-column TMEM loads covering the outputs
  constexpr int NTT = c3_transform_threads(CP, LZ);
  constexpr int NT = C3T + NTT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const C3Layout L = c3_layout(CP, C, Z, T, mz, mt, LZ);
  float* X = reinterpret_cast<float*>(smem_raw + L.x);
  float* Ahi = reinterpret_cast<float*>(smem_raw + L.ahi);
  float* Alo = reinterpret_cast<float*>(smem_raw + L.alo);
  float* Bhi = reinterpret_cast<float*>(smem_raw + L.bhi);
  float* Blo = reinterpret_cast<float*>(smem_raw + L.blo);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  // bar: [0] v tile landed, [1 + b] MMA into D[b] done, [3 + b] U[b] full,
  // [5 + b] U[b] / D[b] empty (one barrier per buffer: no waiter can fall two
  // phases behind, which parity waits could not tell apart)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  uint64_t* bmma = bar + 1;
  uint64_t* bfull = bar + 3;
  uint64_t* bempty = bar + 5;
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem_raw + L.slot);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = L.nk, TP = L.TP, UPS = L.UPS;
  const long long ZT = (long long)Z * T;
  const long long chan_stride = (long long)p.Xl * p.Yl * ZT;
  const int nch = (T + TCH - 1) / TCH;   // the last t chunk is ragged when T % TCH != 0
  const int tpc = p.Qz * nch;        // tiles per column: ti = rz * nch + t chunk
  const unsigned tile_bytes = unsigned(C) * C3T * sizeof(float);
  const int per_c = 2 * mz * mt;

  if ((long long)blockIdx.x >= p.n_cols) return;

  if (warp == 0) tmem_alloc(slot, 64);   // D double buffer: columns [32 b, 32 b + NP)
  fill_combine_table(twZ, LZ, p.Qz, Z, 0, +1, tid, NT);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, +1, tid, NT);
  for (int j = tid; j < 2 * mz; j += NT) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  // B[o][k] = W[o][k] (k < C), b[o] (k = CP), 0 otherwise; split hi / lo
  for (int e = tid; e < NP * KP; e += NT) {
    const int o = e / KP, k = e - o * KP;
    float w = 0.f;
    if (o < C) {
      if (k < C) w = p.w_t ? p.W[k * C + o] : p.W[o * C + k];
      else if (k == CP && p.bias) w = p.bias[o];
    }
    const float hi = tf32_hi(w);
    Bhi[kmaj_off<NP>(o, k)] = hi;
    Blo[kmaj_off<NP>(o, k)] = w - hi;
  }
  // constant A columns [CP, KP): the bias column is 1, the rest 0 (never rewritten)
  for (int e = tid; e < C3T * (KP - CP); e += NT) {
    const int pp = e / (KP - CP), k = CP + (e - pp * (KP - CP));
    Ahi[kmaj_off<C3T>(pp, k)] = (k == CP) ? 1.f : 0.f;
    Alo[kmaj_off<C3T>(pp, k)] = 0.f;
  }
  // padded channel rows of X are never loaded: zero them once
  for (int e = tid; e < (CP - C) * C3T; e += NT) X[C * C3T + e] = 0.f;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bmma[0], 1);
    mbar_init(&bmma[1], 1);
    mbar_init(&bfull[0], NTT);
    mbar_init(&bfull[1], NTT);
    mbar_init(&bempty[0], C3T);
    mbar_init(&bempty[1], C3T);
    mbar_fence_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;

  auto col_split = [&](long long c_, int* b_out) {   // column -> (batch, xl*Yl + yl)
    const unsigned cu = unsigned(c_);
    const unsigned per_b = unsigned(p.Xl) * unsigned(p.Yl);
    *b_out = int(cu / per_b);
    return int(cu - unsigned(*b_out) * per_b);
  };

  if (warp >= 4) {
    // ============ transform warps: phases 1-2, operand split, MMA issue ==========
    const int ttid = tid - C3T;
    auto slab_at = [&](long long c_, int c, int jz) -> const float2* {
      if (p.slab.P == 1) return p.in + (c_ * C + c) * per_c + jz * mt;
      const short2 dm = dmap[jz];
      const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
      return p.in + p.slab.off[dm.x] + ((c_ * C + c) * nkz + dm.y) * mt;
    };
    // v tile (rz, t chunk tc) of column c_ into X: one TMA (thread 0) on the
    // row-group view (rz = G a + r -> inner coordinate r T + t0, group a), else
    // cp.async row pieces by all transform threads; the ragged chunk leaves
    // stale columns that are never stored
    auto issue_tile = [&](long long c_, int ti) {   // all transform threads
      const int rz = ti / nch, tc = ti - rz * nch;
      int bb;
      const int xy = col_split(c_, &bb);
      if (TMA) {
        if (ttid == 0) {
          mbar_expect_tx(&bar[0], tile_bytes);
          const int r = (rz % p.tma_g) * T;   // 16-byte aligned start: the chunk begins (r & 3) points early
          tma_load_5d(X, &maps.m[0], r + tc * TCH - (r & 3), rz / p.tma_g, 0, xy, bb * C, &bar[0]);
        }
        return;
      }
      const int t0 = tc * TCH, tcw = min(TCH, T - t0), VW = p.VW;
      const int nvec = (tcw + VW - 1) / VW;
      const float* src = p.v + (long long)bb * C * chan_stride + (long long)xy * ZT + rz * T + t0;
      for (int e = ttid; e < C * LZ * nvec; e += NTT) {
        const int row = e / nvec, vv = e - row * nvec;
        const int c = row / LZ, s = row - c * LZ;
        const float* g = src + c * chan_stride + (long long)p.Qz * s * T + vv * VW;
        float* d = X + c * C3T + s * TCH + vv * VW;
        if (VW == 2) cp_async8(d, g);
        else cp_async4(d, g);
      }
      cp_commit();
    };
    const uint32_t idesc = umma_idesc_tf32(C3T, NP, 0, 0);
    constexpr uint32_t A_LBO = (C3T / 8) * 128, B_LBO = (NP / 8) * 128;
    issue_tile(blockIdx.x, 0);
    unsigned k = 0, tphase = 0u;   // tile counter of this CTA, v-tile barrier parity
    for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
      const long long col_next = col + gridDim.x;
      group_sync(1, NTT);   // previous column's phase 2 done with Bb
      // ---- phase 1: inverse t (C2R weights and 1/N folded in), items (c, kz', rt)
      for (int it = FNO_ABL(p, 16) ? C * nk * p.Qt : ttid; it < C * nk * p.Qt; it += NTT) {
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
        for (int s = 0; s < LT; ++s) bo[p.Qt * s] = cscale(y[s], p.inv_n);   // the 1/N of the inverse
      }
      group_sync(1, NTT);   // Bb complete
      // the next column's slab rows into L1 (the only L1-allocating loads of the
      // kernel), so its phase 1 does not stall on L2 / HBM latency
      if (col_next < p.n_cols)
        for (int r = ttid; r < C * 2 * mz; r += NTT)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(slab_at(col_next, r / (2 * mz), r % (2 * mz))));
      for (int ti = 0; ti < tpc; ++ti, ++k) {
        const int rz = ti / nch, tc = ti - rz * nch;
        const int t0 = tc * TCH - ((RAG && TMA && p.tma_g > 1) ? ((rz & (p.tma_g - 1)) * T) & 3 : 0);   // first t of the tile
        const int b = k & 1;
        const unsigned use = k >> 1;
        // U[b] and TMEM D[b] drained by the epilogue (tile k - 2)
        mbar_wait(&bempty[b], (use & 1u) ^ 1u);
        // ---- split the v tile into the K-major tf32 hi / lo operands --------
        if (k > 0) mbar_wait(&bmma[(k - 1) & 1], ((k - 1) >> 1) & 1u);   // MMA k-1 done reading A
        if (TMA) {
          mbar_wait(&bar[0], tphase);
          tphase ^= 1u;
        } else {
          cp_wait<0>();
          group_sync(1, NTT);
        }
        for (int e = FNO_ABL(p, 2) ? C3T * (CP / 4) : ttid; e < C3T * (CP / 4); e += NTT) {
          const int g = e / C3T, pp = e - g * C3T;
          float4 hi, lo;
          const float x0 = X[(4 * g + 0) * C3T + pp], x1 = X[(4 * g + 1) * C3T + pp];
          const float x2 = X[(4 * g + 2) * C3T + pp], x3 = X[(4 * g + 3) * C3T + pp];
          hi.x = tf32_hi(x0); lo.x = x0 - hi.x;
          hi.y = tf32_hi(x1); lo.y = x1 - hi.y;
          hi.z = tf32_hi(x2); lo.z = x2 - hi.z;
          hi.w = tf32_hi(x3); lo.w = x3 - hi.w;
          *reinterpret_cast<float4*>(Ahi + kmaj_off<C3T>(pp, 4 * g)) = hi;
          *reinterpret_cast<float4*>(Alo + kmaj_off<C3T>(pp, 4 * g)) = lo;
        }
        fence_proxy_async();   // generic-proxy operand stores -> visible to the tensor core
        group_sync(1, NTT);    // A complete, X free
        if (ti + 1 < tpc) issue_tile(col, ti + 1);
        else if (col_next < p.n_cols) issue_tile(col_next, 0);
        if (ttid == 0) {
          tc_fence_after();
          const uint32_t dt = tmem + 32u * b;
#pragma unroll
          for (int j = 0; j < KP / 8; ++j) {
            const uint64_t ah = umma_sdesc(Ahi + j * 2 * (A_LBO / 4), A_LBO, 128);
            const uint64_t al = umma_sdesc(Alo + j * 2 * (A_LBO / 4), A_LBO, 128);
            const uint64_t bh = umma_sdesc(Bhi + j * 2 * (B_LBO / 4), B_LBO, 128);
            const uint64_t bl = umma_sdesc(Blo + j * 2 * (B_LBO / 4), B_LBO, 128);
            umma_tf32(dt, ah, bh, idesc, j > 0 ? 1u : 0u);
            umma_tf32(dt, al, bh, idesc, 1u);
            umma_tf32(dt, ah, bl, idesc, 1u);
          }
          umma_commit(&bmma[b]);
        }
        float* U = reinterpret_cast<float*>(smem_raw + (b ? L.u1 : L.u0));
        // ---- phase 2: inverse z (real output), items (c, tt) -> U[b] --------
        const int ta = RAG ? max(0, -t0) : 0, tb = RAG ? min(TCH, T - t0) : TCH;   // valid columns; the others are never stored
        for (int it = FNO_ABL(p, 1) ? C * TCH : ttid; it < C * TCH; it += NTT) {
          const int c = it / TCH, tt = it - c * TCH;
          if (tt < ta || tt >= tb) continue;
          float2 e[LZ];
#pragma unroll
          for (int i = 0; i < LZ; ++i)
            e[i] = (i < (HALF ? LZ / 2 + 1 : nk)) ? Bb[(c * nk + i) * TP + t0 + tt] : make_float2(0.f, 0.f);
          float2 y[LZ];
          trunc_inv<LZ>(y, e, rz, twZ);
          float* uo = U + c * UPS + tt;
#pragma unroll
          for (int s = 0; s < LZ; ++s) uo[s * TCH] = y[s].x;
        }
        mbar_arrive(&bfull[b]);
      }
    }
  } else {
    // ============ epilogue warps (TMEM lanes): z = D + u, GELU, stores ============
    const uint32_t t_row = tmem + ((uint32_t)(32 * warp) << 16);
    unsigned k = 0;
    for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
      int bcol;
      const int xycol = col_split(col, &bcol);
      const long long cbase = (long long)bcol * C * chan_stride + (long long)xycol * ZT;
      for (int ti = 0; ti < tpc; ++ti, ++k) {
        const int rz = ti / nch, tc = ti - rz * nch;
        const int t0 = tc * TCH - ((RAG && TMA && p.tma_g > 1) ? ((rz & (p.tma_g - 1)) * T) & 3 : 0);
        const int b = k & 1;
        const unsigned use = k >> 1;
        float* U = reinterpret_cast<float*>(smem_raw + (b ? L.u1 : L.u0));
        mbar_wait(&bfull[b], use & 1u);   // phase 2 of this tile done
        mbar_wait(&bmma[b], use & 1u);    // MMA of this tile done
        tc_fence_after();
        uint32_t d[NCH][8];
#pragma unroll
        for (int q = 0; q < NCH; ++q) tmem_ld8_nowait(t_row + 32u * b + 8 * q, d[q]);
        tmem_wait_ld();
        tc_fence_before();
#pragma unroll
        for (int o = 0; o < CP; ++o) {
          if (o >= C || FNO_ABL(p, 4)) break;
          U[o * UPS + tid] += __uint_as_float(d[o >> 3][o & 7]);
        }
        __syncwarp();
        // float4 f of the warp: channel o, points 32 warp + 4 (lane % 8) + [0, 4)
        const int pq = 32 * warp + 4 * (lane & 7);
        const int sq = pq / TCH, tq = pq - sq * TCH;
        const long long gq = cbase + (long long)(rz + p.Qz * sq) * T + t0 + tq;
        // valid points [k0, k1) of this quad (ragged chunks); TMA tiles are 16-byte aligned
        const int k0 = RAG ? max(0, -(t0 + tq)) : 0, k1 = RAG ? min(4, T - t0 - tq) : 4;
        const bool v4 = !RAG || ((TMA || T % 4 == 0) && k0 == 0 && k1 == 4);
#pragma unroll
        for (int j = 0; j < (CP + 3) / 4; ++j) {
          const int o = (lane >> 3) + 4 * j;
          if (o >= C || FNO_ABL(p, 4) || k0 >= k1) break;
          float4 r = *reinterpret_cast<const float4*>(U + o * UPS + pq);
          const long long g = gq + o * chan_stride;
          // one copy of the GELU for the full-quad and the ragged stores (code size)
          if (p.zsave) {
            if (v4) __stcs(reinterpret_cast<float4*>(p.zsave + g), r);
            else store_quad_part(p.zsave + g, r, k0, k1);
          }
          if (p.act_gelu) {
            r.x = gelu_f(r.x); r.y = gelu_f(r.y); r.z = gelu_f(r.z); r.w = gelu_f(r.w);
          }
          if (v4) __stcs(reinterpret_cast<float4*>(p.out + g), r);
          else store_quad_part(p.out + g, r, k0, k1);
        }
        mbar_arrive(&bempty[b]);   // U[b], D[b] free
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

template <int LZ, int LT, int CP>
cudaError_t launch_c3_cp(const C2Maps& maps, const PassCParams& p, int grid, size_t smem, cudaStream_t st) {
  const bool half = 2 * p.mz == LZ;
  const bool rag = p.tma_g != 1 || p.T % (C3T / LZ) != 0 || p.T % 4 != 0;
  // TMA tiles (any row-group view, c2_tile_group) or cp.async tiles
  void (*k)(C2Maps, PassCParams) =
      !p.use_tma ? (half ? pass_c3_fwd_kernel<LZ, LT, CP, true, false, true> : pass_c3_fwd_kernel<LZ, LT, CP, false, false, true>)
      : rag      ? (half ? pass_c3_fwd_kernel<LZ, LT, CP, true, true, true> : pass_c3_fwd_kernel<LZ, LT, CP, false, true, true>)
                 : (half ? pass_c3_fwd_kernel<LZ, LT, CP, true, true, false> : pass_c3_fwd_kernel<LZ, LT, CP, false, true, false>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, c3_threads(CP, LZ), smem, st>>>(maps, p);
  return cudaGetLastError();
}

// only tile shapes with LZ in {8, 16, 32} are instantiated
template <int LZ, int LT, int CP>
cudaError_t launch_c3_case(const C2Maps& maps, const PassCParams& p, int grid, size_t smem, cudaStream_t st) {
  if constexpr (LZ >= 8 && LZ <= 32) return launch_c3_cp<LZ, LT, CP>(maps, p, grid, smem, st);
  else return cudaErrorInvalidValue;
}

}  // namespace fno
