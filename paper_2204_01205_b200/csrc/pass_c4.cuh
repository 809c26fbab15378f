// Pass C, generation 4: one warp-specialised sm_100a kernel for the layer
// forward, the layer backward and the plain spectral output (SURVEY §8 rows
// a7, a8; backward a9, a12).  The adjoint chain of I_1 = {z, t} (zero-padded
// inverse z, C2R along t with real-part semantics) fused with the
// DFNO block epilogue (Eq. dist_block):
//   EPI_FWD: z = W v + b + u,  y = sigma(z)             (1x1 + bias on tcgen05)
//   EPI_BWD: dv = W^T dz + u,  dW += dz v^T, db += dz   (both contractions on tcgen05;
//            u = S^T dz, broadcast adjoint = sum)
//   EPI_U:   u = S v (or S^T g)                          (no contraction)
//
// Why a new kernel (pass_c2 / pass_c3 measured 0.24-0.50 of HBM peak): their
// per-column phases run back to back inside a CTA with one v tile in flight,
// so load latency and transform latency add up.  Here each role has its own
// warps and the hand-offs are mbarriers, so the load of tile k+NS, the operand
// split of tile k, the MMAs of tile k, phase 2 of tile k+1 and the epilogue of
// tile k-1 all proceed at once on one SM:
//
//   warp  4      TMA producer: NS-stage ring of input tiles X (v, or dz and v),
//                one 5-D tensor-map box per input (c2_encode_tile_map)
//   warp  5      TMEM owner and MMA issuer (one thread): kind::tf32 3xTF32
//                  D1[p][n]  = sum_k A1[p][k] B1[n][k]   (M128 x N NP x K KP)
//                    fwd: A1 = v^T | 1, B1 = W | b;  bwd: A1 = dz^T, B1 = W^T
//                  D2[o][i]  = sum_p dz[o][p] v'[i][p]   (bwd, M128 x N NW x K128)
//                    v' = v rows and a ones row (-> db); A2 stores only the
//                    ceil(C/8) real row groups, the M = 128 over-read lands in
//                    the following K groups (rows >= C of D2 are never read)
//   warps 0-3    split + epilogue (thread = tile point = TMEM lane): splits
//                tile k into the K-major tf32 hi / lo operands, then finishes
//                tile k-1: D1 row + U column (fwd: GELU, z) -> float4 stores;
//                bwd: warp 0 adds the D2 rows (dW, db) of every tile into fp32
//                registers (a per-tile flush keeps the tensor-core sums short)
//   warps 6-11   transforms: per column phase 1 (inverse t of the slab, C2R
//                weights and 1/N folded in -> Bb), per tile phase 2 (inverse z
//                of residue class rz -> U[k & 1])
//
// fp32 accuracy from tf32 operands (3xTF32): x = hi + lo with hi the tf32
// truncation of x and lo = x - hi; D = A_hi B_hi + A_lo B_hi + A_hi B_lo.
// Tile = one z residue class rz (LZ points) x TCH = 128 / LZ consecutive t:
// M = 128 points; T % 4 != 0 uses the row-group TMA view (c2_tile_group) with
// phase-shifted / ragged t chunks whose out-of-range points are never stored
// and are zeroed in the dW operand.
#pragma once

#include <cuda.h>

#include "kernels.cuh"
#include "launch.h"
#include "pass_c2.cuh"
#include "pass_c3.cuh"
#include "umma.cuh"

namespace fno {

constexpr int C4T = 384;            // 12 warps
constexpr int C4_NTT = 192;         // transform threads (warps 6-11)
constexpr int C4_PROD = 4, C4_MMA = 5, C4_TR0 = 6;
constexpr int C4_MAXNS = 6;

__host__ __device__ constexpr int c4_kp(int CP, int mode) {
  return mode == EPI_FWD ? ((CP + 1 + 7) & ~7) : ((CP + 7) & ~7);
}
__host__ __device__ constexpr int c4_np(int CP) { return (CP + 15) & ~15; }
__host__ __device__ constexpr int c4_nw(int CP) { return (CP + 1 + 15) & ~15; }
__host__ __device__ constexpr int c4_rg(int CP) { return (CP + 7) / 8; }
__host__ __device__ constexpr int c4_tmem_cols(int CP, int mode) {
  return mode == EPI_U ? 0 : (mode == EPI_FWD ? 64 : (64 + 2 * c4_nw(CP) <= 128 ? 128 : 256));
}

struct C4Layout {
  int NS, NOB, KP, NP, NW, RG, nk, TP, UPS;
  size_t x, xstage, op, opstage, a1hi, a1lo, a2hi, a2lo, b2hi, b2lo, b1hi, b1lo, bb, u0, u1, twz, twt, dmap, bar, slot,
      total;
};

// NS: input-tile ring stages; operand buffers: 2 (fwd), 1 (bwd)
__host__ __device__ inline C4Layout c4_layout(int CP, int mode, int C, int Z, int T, int mz, int LZ, int NS) {
  C4Layout L{};
  const bool bwd = mode == EPI_BWD, mma = mode != EPI_U;
  L.NS = mma ? NS : 0;
  L.NOB = mode == EPI_FWD ? 2 : (bwd ? 1 : 0);
  L.KP = c4_kp(CP, mode);
  L.NP = c4_np(CP);
  L.NW = c4_nw(CP);
  L.RG = c4_rg(CP);
  L.nk = mz + 1;
  L.TP = T + 1;
  const int TCH = 128 / LZ;
  L.UPS = 128 + (TCH < 32 ? TCH : 0);   // phase-2 stores of lanes (c, t) on distinct banks
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 1023) & ~size_t(1023); return o; };
  const int NA = bwd ? 2 : 1;
  L.xstage = (size_t(NA) * C * 128 * sizeof(float) + 1023) & ~size_t(1023);
  L.x = take(L.xstage * L.NS);
  // one operand buffer: A1 hi/lo [128][KP]; bwd adds A2 hi/lo (RG row groups,
  // + 2 KB over-read pad each) and B2 hi/lo [NW][128]
  const size_t a1 = size_t(128) * L.KP * sizeof(float);
  const size_t a2 = bwd ? size_t(32) * L.RG * 32 * sizeof(float) + 2048 : 0;
  const size_t b2 = bwd ? size_t(32) * (L.NW / 8) * 32 * sizeof(float) : 0;
  L.a1hi = 0;
  L.a1lo = L.a1hi + a1;
  L.a2hi = L.a1lo + a1;
  L.a2lo = L.a2hi + a2;
  L.b2hi = L.a2lo + a2;
  L.b2lo = L.b2hi + b2;
  L.opstage = ((L.b2lo + b2) + 1023) & ~size_t(1023);
  L.op = take(L.opstage * L.NOB);
  L.b1hi = take(size_t(L.NP) * L.KP * sizeof(float));
  L.b1lo = take(size_t(L.NP) * L.KP * sizeof(float));
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.u0 = take(size_t(C) * L.UPS * sizeof(float));
  L.u1 = take(size_t(C) * L.UPS * sizeof(float));
  auto take16 = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
  L.twz = take16(size_t(Z) * sizeof(float2));
  L.twt = take16(size_t(T) * sizeof(float2));
  L.dmap = take16(size_t(2 * mz) * sizeof(short2));
  L.bar = take16(32 * sizeof(uint64_t));
  L.slot = take16(sizeof(uint32_t));
  L.total = off + 1024;   // + alignment slack of the dynamic shared memory base
  return L;
}

// K-major (SWIZZLE_NONE) element offset, RGS row groups of 8 rows per K group of 4
__device__ __forceinline__ int kmaj_rows(int row, int k, int RGS) {
  return ((k >> 2) * RGS + (row >> 3)) * 32 + (row & 7) * 4 + (k & 3);
}

template <int LZ, int LT, int CP, int EPI, bool HALF, bool RAG>
__global__ void __launch_bounds__(C4T, 1) pass_c4_kernel(const __grid_constant__ C2Maps maps, const PassCParams p) {
  static_assert(CP % 4 == 0 && CP <= 32, "CP must be a multiple of 4, at most 32");
  static_assert(128 % LZ == 0 && 128 / LZ >= 4, "LZ must divide the 128 tile points, TCH >= 4");
  constexpr int TCH = 128 / LZ;
  constexpr bool BWD = EPI == EPI_BWD;
  constexpr bool MMA = EPI != EPI_U;
  constexpr int NA = BWD ? 2 : 1;
  constexpr int KP = c4_kp(CP, EPI), NP = c4_np(CP), NW = c4_nw(CP), RG = c4_rg(CP);
  constexpr int NCH1 = (CP + 7) / 8;
  constexpr int NOB = EPI == EPI_FWD ? 2 : 1;
  constexpr uint32_t TMEM_COLS = c4_tmem_cols(CP, EPI);
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem_raw =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const int NS = MMA ? p.NX : 1;
  const C4Layout L = c4_layout(CP, EPI, C, Z, T, mz, LZ, NS);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  uint64_t* xfull = bars;          // [NS]  TMA bytes landed
  uint64_t* xempty = bars + 8;     // [NS]  128 split threads done reading
  uint64_t* opfull = bars + 16;    // [2]   128 split threads wrote the operands
  uint64_t* opempty = bars + 18;   // [2]   MMAs done reading them (tcgen05.commit)
  uint64_t* dfull = bars + 20;     // [2]   MMAs done writing D[b] (tcgen05.commit)
  uint64_t* dempty = bars + 22;    // [2]   128 epilogue threads read D[b]
  uint64_t* ufull = bars + 24;     // [2]   192 transform threads wrote U[b]
  uint64_t* uempty = bars + 26;    // [2]   128 epilogue threads read U[b]
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem_raw + L.slot);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = L.nk, TP = L.TP, UPS = L.UPS;
  const long long ZT = (long long)Z * T;
  const long long chan_stride = (long long)p.Xl * p.Yl * ZT;
  const int nch = (T + TCH - 1) / TCH;
  const int tpc = p.Qz * nch;
  const unsigned tile_bytes = unsigned(C) * 128 * sizeof(float);
  const int per_c = 2 * mz * mt;

  if ((long long)blockIdx.x >= p.n_cols) return;

  if (MMA && warp == C4_MMA) tmem_alloc(slot, TMEM_COLS);
  fill_combine_table(twZ, LZ, p.Qz, Z, 0, +1, tid, C4T);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, +1, tid, C4T);
  for (int j = tid; j < 2 * mz; j += C4T) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  if (MMA) {
    float* B1hi = reinterpret_cast<float*>(smem_raw + L.b1hi);
    float* B1lo = reinterpret_cast<float*>(smem_raw + L.b1lo);
    // fwd B1[o][k] = W[o][k] (k < C), b[o] (k = CP); bwd B1[i][o] = W[o][i]
    for (int e = tid; e < NP * KP; e += C4T) {
      const int n = e / KP, k = e - n * KP;
      float w = 0.f;
      if (n < C) {
        if (k < C) w = BWD ? p.W[k * C + n] : p.W[n * C + k];
        else if (!BWD && k == CP && p.bias) w = p.bias[n];
      }
      const float hi = tf32_hi(w);
      B1hi[kmaj_off<NP>(n, k)] = hi;
      B1lo[kmaj_off<NP>(n, k)] = w - hi;
    }
    // constant parts of every operand buffer (never rewritten by the split)
    for (int ob = 0; ob < NOB; ++ob) {
      unsigned char* base = smem_raw + L.op + ob * L.opstage;
      float* A1hi = reinterpret_cast<float*>(base + L.a1hi);
      float* A1lo = reinterpret_cast<float*>(base + L.a1lo);
      // A1 columns [CP, KP): bias column 1 (fwd), the rest 0
      for (int e = tid; e < 128 * (KP - CP); e += C4T) {
        const int pp = e / (KP - CP), k = CP + (e - pp * (KP - CP));
        A1hi[kmaj_off<128>(pp, k)] = (!BWD && k == CP) ? 1.f : 0.f;
        A1lo[kmaj_off<128>(pp, k)] = 0.f;
      }
      if (BWD) {
        float* A2hi = reinterpret_cast<float*>(base + L.a2hi);
        float* B2hi = reinterpret_cast<float*>(base + L.b2hi);
        float* A2lo = reinterpret_cast<float*>(base + L.a2lo);
        float* B2lo = reinterpret_cast<float*>(base + L.b2lo);
        // A2 rows [C, 8 RG) and the over-read pad: 0; B2 row C: ones (-> db), rows > C: 0
        for (int e = tid; e < 32 * RG * 32 + 512; e += C4T) {
          if (e >= 32 * RG * 32) { A2hi[e] = 0.f; A2lo[e] = 0.f; continue; }
          const int row = ((e >> 5) % RG) * 8 + ((e & 31) >> 2);
          if (row >= C) { A2hi[e] = 0.f; A2lo[e] = 0.f; }
        }
        for (int e = tid; e < 32 * (NW / 8) * 32; e += C4T) {
          const int row = ((e >> 5) % (NW / 8)) * 8 + ((e & 31) >> 2);
          if (row >= C) { B2hi[e] = (row == C) ? 1.f : 0.f; B2lo[e] = 0.f; }
        }
      }
    }
  }
  if (tid == 0) {
    for (int s = 0; s < NS && MMA; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 128);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&opfull[b], 128);
      mbar_init(&opempty[b], 1);
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], 128);
      mbar_init(&ufull[b], C4_NTT);
      mbar_init(&uempty[b], 128);
    }
    mbar_fence_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = MMA ? *slot : 0u;

  auto col_split = [&](long long c_, int* b_out) {   // column -> (batch, xl*Yl + yl)
    const unsigned cu = unsigned(c_);
    const unsigned per_b = unsigned(p.Xl) * unsigned(p.Yl);
    *b_out = int(cu / per_b);
    return int(cu - unsigned(*b_out) * per_b);
  };
  // first t of tile ti (TMA row groups with (z T) % 4 != 0 start early, c2_tile_group)
  auto tile_t0 = [&](int ti) {
    const int rz = ti / nch, tc = ti - rz * nch;
    return tc * TCH - ((RAG && p.tma_g > 1) ? ((rz & (p.tma_g - 1)) * T) & 3 : 0);
  };
  auto xstage = [&](int s) { return reinterpret_cast<float*>(smem_raw + L.x + s * L.xstage); };
  auto opbuf = [&](int ob) { return smem_raw + L.op + ob * L.opstage; };

  if (warp == C4_PROD) {
    // ======================= TMA producer ========================================
    if (MMA && lane == 0) {
      unsigned k = 0;
      for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
        int bb;
        const int xy = col_split(col, &bb);
        for (int ti = 0; ti < tpc; ++ti, ++k) {
          const int s = int(k % unsigned(NS));
          const unsigned u = k / unsigned(NS);
          mbar_wait(&xempty[s], (u & 1u) ^ 1u);
          mbar_expect_tx(&xfull[s], tile_bytes * NA);
          const int rz = ti / nch, tc = ti - rz * nch;
          const int r = (rz % p.tma_g) * T;
#pragma unroll
          for (int a = 0; a < NA; ++a)
            tma_load_5d(xstage(s) + a * C * 128, &maps.m[a], r + tc * TCH - (r & 3), rz / p.tma_g, 0, xy, bb * C,
                        &xfull[s]);
        }
      }
    }
  } else if (warp == C4_MMA) {
    // ======================= MMA issuer ==========================================
    if (MMA && lane == 0) {
      const uint32_t idesc1 = umma_idesc_tf32(128, NP, 0, 0);
      const uint32_t idesc2 = umma_idesc_tf32(128, NW, 0, 0);
      constexpr uint32_t A1_LBO = (128 / 8) * 128, B1_LBO = (NP / 8) * 128;
      constexpr uint32_t A2_LBO = RG * 128, B2_LBO = (NW / 8) * 128;
      const float* B1hi = reinterpret_cast<const float*>(smem_raw + L.b1hi);
      const float* B1lo = reinterpret_cast<const float*>(smem_raw + L.b1lo);
      unsigned k = 0;
      for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
        for (int ti = 0; ti < tpc; ++ti, ++k) {
          const int b = k & 1;
          const unsigned u = k >> 1;
          const int ob = NOB == 2 ? b : 0;
          const unsigned ou = NOB == 2 ? u : k;
          mbar_wait(&opfull[ob], ou & 1u);
          mbar_wait(&dempty[b], (u & 1u) ^ 1u);
          tc_fence_after();
          const unsigned char* base = opbuf(ob);
          const float* A1hi = reinterpret_cast<const float*>(base + L.a1hi);
          const float* A1lo = reinterpret_cast<const float*>(base + L.a1lo);
          const uint32_t d1 = tmem + 32u * b;
#pragma unroll
          for (int j = 0; j < KP / 8; ++j) {
            const uint64_t ah = umma_sdesc(A1hi + j * 2 * (A1_LBO / 4), A1_LBO, 128);
            const uint64_t al = umma_sdesc(A1lo + j * 2 * (A1_LBO / 4), A1_LBO, 128);
            const uint64_t bh = umma_sdesc(B1hi + j * 2 * (B1_LBO / 4), B1_LBO, 128);
            const uint64_t bl = umma_sdesc(B1lo + j * 2 * (B1_LBO / 4), B1_LBO, 128);
            umma_tf32(d1, ah, bh, idesc1, j > 0 ? 1u : 0u);
            umma_tf32(d1, al, bh, idesc1, 1u);
            umma_tf32(d1, ah, bl, idesc1, 1u);
          }
          if (BWD) {
            const float* A2hi = reinterpret_cast<const float*>(base + L.a2hi);
            const float* A2lo = reinterpret_cast<const float*>(base + L.a2lo);
            const float* B2hi = reinterpret_cast<const float*>(base + L.b2hi);
            const float* B2lo = reinterpret_cast<const float*>(base + L.b2lo);
            const uint32_t d2 = tmem + 64u + uint32_t(NW) * b;
#pragma unroll 4
            for (int j = 0; j < 128 / 8; ++j) {
              const uint64_t ah = umma_sdesc(A2hi + j * 2 * (A2_LBO / 4), A2_LBO, 128);
              const uint64_t al = umma_sdesc(A2lo + j * 2 * (A2_LBO / 4), A2_LBO, 128);
              const uint64_t bh = umma_sdesc(B2hi + j * 2 * (B2_LBO / 4), B2_LBO, 128);
              const uint64_t bl = umma_sdesc(B2lo + j * 2 * (B2_LBO / 4), B2_LBO, 128);
              umma_tf32(d2, ah, bh, idesc2, j > 0 ? 1u : 0u);
              umma_tf32(d2, al, bh, idesc2, 1u);
              umma_tf32(d2, ah, bl, idesc2, 1u);
            }
          }
          umma_commit(&opempty[ob]);
          umma_commit(&dfull[b]);
        }
      }
    }
  } else if (warp >= C4_TR0) {
    // ======================= transforms (phases 1-2) ===============================
    const int ttid = tid - C4_TR0 * 32;
    auto slab_at = [&](long long c_, int c, int jz) -> const float2* {
      if (p.slab.P == 1) return p.in + (c_ * C + c) * per_c + jz * mt;
      const short2 dm = dmap[jz];
      const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
      return p.in + p.slab.off[dm.x] + ((c_ * C + c) * nkz + dm.y) * mt;
    };
    unsigned k = 0;
    for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
      const long long col_next = col + gridDim.x;
      group_sync(2, C4_NTT);   // the previous column's phase 2 is done with Bb
      // ---- phase 1: inverse t (C2R weights and 1/N folded in), items (c, kz', rt)
      for (int it = ttid; it < C * nk * p.Qt; it += C4_NTT) {
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
      group_sync(2, C4_NTT);   // Bb complete
      if (col_next < p.n_cols)   // next column's slab rows into L1 (phase 1 then hits L1)
        for (int r = ttid; r < C * 2 * mz; r += C4_NTT)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(slab_at(col_next, r / (2 * mz), r % (2 * mz))));
      for (int ti = 0; ti < tpc; ++ti, ++k) {
        const int rz = ti / nch;
        const int t0 = tile_t0(ti);
        const int b = k & 1;
        const unsigned u = k >> 1;
        mbar_wait(&uempty[b], (u & 1u) ^ 1u);
        float* U = reinterpret_cast<float*>(smem_raw + (b ? L.u1 : L.u0));
        // ---- phase 2: inverse z (real output), items (c, tt) -> U[b] -----------
        const int ta = RAG ? max(0, -t0) : 0, tb = RAG ? min(TCH, T - t0) : TCH;
        for (int it = ttid; it < C * TCH; it += C4_NTT) {
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
        mbar_arrive(&ufull[b]);
      }
    }
  } else if (warp < 4) {
    // ======================= split + epilogue (TMEM lanes) =========================
    const int et = tid;   // tile point of the epilogue, operand row of the split
    const uint32_t t_row = tmem + ((uint32_t)(32 * warp) << 16);
    float dwacc[BWD ? NW : 1];
#pragma unroll
    for (int i = 0; i < (BWD ? NW : 1); ++i) dwacc[i] = 0.f;

    // operands of tile k (col, ti) from its X stage
    auto split = [&](unsigned k, int ti) {
      const int s = int(k % unsigned(NS));
      const unsigned u = k / unsigned(NS);
      const int ob = NOB == 2 ? int(k & 1) : 0;
      const unsigned ou = NOB == 2 ? (k >> 1) : k;
      mbar_wait(&xfull[s], u & 1u);
      mbar_wait(&opempty[ob], (ou & 1u) ^ 1u);
      const float* X0 = xstage(s);   // v (fwd) or dz (bwd): [C][128]
      unsigned char* base = opbuf(ob);
      float* A1hi = reinterpret_cast<float*>(base + L.a1hi);
      float* A1lo = reinterpret_cast<float*>(base + L.a1lo);
      // A1[p][k] = X0[k][p] (K-major, 4 channels per float4)
      for (int e = et; e < (CP / 4) * 128; e += 128) {
        const int g = e >> 7, pp = e & 127;
        float x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = (4 * g + j < C) ? X0[(4 * g + j) * 128 + pp] : 0.f;
        float4 hi, lo;
        hi.x = tf32_hi(x[0]); lo.x = x[0] - hi.x;
        hi.y = tf32_hi(x[1]); lo.y = x[1] - hi.y;
        hi.z = tf32_hi(x[2]); lo.z = x[2] - hi.z;
        hi.w = tf32_hi(x[3]); lo.w = x[3] - hi.w;
        *reinterpret_cast<float4*>(A1hi + kmaj_off<128>(pp, 4 * g)) = hi;
        *reinterpret_cast<float4*>(A1lo + kmaj_off<128>(pp, 4 * g)) = lo;
      }
      if (BWD) {
        // A2[o][p] = dz (rows = channels, K = points): a 16-byte-chunk transpose
        // of X0; B2[i][p] = v.  Diagonal lane order: each 8-lane phase reads 8
        // distinct chunk columns q and writes 8 distinct rows (bank-conflict free).
        // Points outside [0, T) of a ragged tile are zeroed in A2 (exact dW, db).
        const int t0 = tile_t0(ti);
        const int ta = RAG ? max(0, -t0) : 0, tb = RAG ? min(TCH, T - t0) : TCH;
        const float* V0 = X0 + C * 128;
        float* A2hi = reinterpret_cast<float*>(base + L.a2hi);
        float* A2lo = reinterpret_cast<float*>(base + L.a2lo);
        float* B2hi = reinterpret_cast<float*>(base + L.b2hi);
        float* B2lo = reinterpret_cast<float*>(base + L.b2lo);
        const int w = warp, j8 = lane & 7, ph = lane >> 3;
        // blocks of 8 rows x 8 chunk columns: RG x 4 per operand, 2 operands
        for (int blk = w; blk < 2 * RG * 4; blk += 4) {
          const int opnd = blk / (RG * 4), r = blk - opnd * (RG * 4);
          const int ob8 = r >> 2, qb = r & 3;
          const float* src = opnd == 0 ? X0 : V0;
#pragma unroll
          for (int it = 0; it < 2; ++it) {
            const int o = ob8 * 8 + j8;
            const int q = qb * 8 + ((j8 + ph + 4 * it) & 7);
            if (o < C) {
              float4 x = *reinterpret_cast<const float4*>(src + o * 128 + 4 * q);
              if (RAG && opnd == 0) {
                const int tq = (4 * q) % TCH;   // t within the tile of the chunk's first point
                if (tq + 0 < ta || tq + 0 >= tb) x.x = 0.f;
                if (tq + 1 < ta || tq + 1 >= tb) x.y = 0.f;
                if (tq + 2 < ta || tq + 2 >= tb) x.z = 0.f;
                if (tq + 3 < ta || tq + 3 >= tb) x.w = 0.f;
              }
              float4 hi, lo;
              hi.x = tf32_hi(x.x); lo.x = x.x - hi.x;
              hi.y = tf32_hi(x.y); lo.y = x.y - hi.y;
              hi.z = tf32_hi(x.z); lo.z = x.z - hi.z;
              hi.w = tf32_hi(x.w); lo.w = x.w - hi.w;
              if (opnd == 0) {
                const int off = (q * RG + (o >> 3)) * 32 + (o & 7) * 4;
                *reinterpret_cast<float4*>(A2hi + off) = hi;
                *reinterpret_cast<float4*>(A2lo + off) = lo;
              } else {
                const int off = (q * (NW / 8) + (o >> 3)) * 32 + (o & 7) * 4;
                *reinterpret_cast<float4*>(B2hi + off) = hi;
                *reinterpret_cast<float4*>(B2lo + off) = lo;
              }
            }
          }
        }
      }
      mbar_arrive(&xempty[s]);   // this thread's reads of the X stage are done
      fence_proxy_async();       // generic-proxy operand stores -> visible to the tensor core
      mbar_arrive(&opfull[ob]);
    };

    // results of tile k (col, ti): D1 row + U column -> stores; bwd: D2 -> dW, db
    auto epilogue = [&](unsigned k, long long col, int ti) {
      const int b = k & 1;
      const unsigned u = k >> 1;
      float* U = reinterpret_cast<float*>(smem_raw + (b ? L.u1 : L.u0));
      const int rz = ti / nch;
      const int t0 = tile_t0(ti);
      mbar_wait(&ufull[b], u & 1u);
      if (MMA) {
        mbar_wait(&dfull[b], u & 1u);
        tc_fence_after();
        uint32_t d[NCH1][8];
#pragma unroll
        for (int q = 0; q < NCH1; ++q) tmem_ld8_nowait(t_row + 32u * b + 8 * q, d[q]);
        uint32_t d2[BWD ? NW / 8 : 1][8];
        if (BWD && warp == 0) {
#pragma unroll
          for (int q = 0; q < (BWD ? NW / 8 : 0); ++q) tmem_ld8_nowait(t_row + 64u + uint32_t(NW) * b + 8 * q, d2[q]);
        }
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&dempty[b]);
#pragma unroll
        for (int o = 0; o < CP; ++o) {
          if (o >= C) break;
          U[o * UPS + et] += __uint_as_float(d[o >> 3][o & 7]);
        }
        if (BWD && warp == 0) {
#pragma unroll
          for (int q = 0; q < (BWD ? NW / 8 : 0); ++q)
#pragma unroll
            for (int j = 0; j < 8; ++j) dwacc[8 * q + j] += __uint_as_float(d2[q][j]);
        }
      }
      __syncwarp();
      int bcol;
      const int xycol = col_split(col, &bcol);
      const long long cbase = (long long)bcol * C * chan_stride + (long long)xycol * ZT;
      // float4 f of the warp: channel o, points 32 warp + 4 (lane % 8) + [0, 4)
      const int pq = 32 * warp + 4 * (lane & 7);
      const int sq = pq / TCH, tq = pq - sq * TCH;
      const long long gq = cbase + (long long)(rz + p.Qz * sq) * T + t0 + tq;
      const int k0 = RAG ? max(0, -(t0 + tq)) : 0, k1 = RAG ? min(4, T - t0 - tq) : 4;
      const bool v4 = !RAG || (k0 == 0 && k1 == 4);   // TMA tiles start 16-byte aligned
#pragma unroll
      for (int j = 0; j < (CP + 3) / 4; ++j) {
        const int o = (lane >> 3) + 4 * j;
        if (o >= C || k0 >= k1) break;
        float4 r = *reinterpret_cast<const float4*>(U + o * UPS + pq);
        const long long g = gq + o * chan_stride;
        if (v4) {
          if (EPI == EPI_FWD) {
            if (p.zsave) __stcs(reinterpret_cast<float4*>(p.zsave + g), r);
            if (p.act_gelu) {
              r.x = gelu_f(r.x); r.y = gelu_f(r.y); r.z = gelu_f(r.z); r.w = gelu_f(r.w);
            }
          }
          __stcs(reinterpret_cast<float4*>(p.out + g), r);
        } else {
          const float rv[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (kk >= k0 && kk < k1) {
              float val = rv[kk];
              if (EPI == EPI_FWD) {
                if (p.zsave) p.zsave[g + kk] = val;
                if (p.act_gelu) val = gelu_f(val);
              }
              p.out[g + kk] = val;
            }
          }
        }
      }
      __syncwarp();
      mbar_arrive(&uempty[b]);   // U[b] free
    };

    unsigned k = 0;
    long long pcol = -1;
    int pti = 0;
    for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
      for (int ti = 0; ti < tpc; ++ti, ++k) {
        if (MMA) split(k, ti);
        if (pcol >= 0) epilogue(k - 1, pcol, pti);
        pcol = col;
        pti = ti;
      }
    }
    if (pcol >= 0) epilogue(k - 1, pcol, pti);
    if (BWD && warp == 0) {
      // this CTA's dW / db partial row (fixed order: per tile, in tile order)
      float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
      if (lane < C) {
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          if (i < C) outp[lane * C + i] = dwacc[i];
          else if (i == C) outp[C * C + lane] = dwacc[i];
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (MMA && warp == C4_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

template <int LZ, int LT, int CP, int EPI>
cudaError_t launch_c4_case(const C2Maps& maps, const PassCParams& p, int grid, size_t smem, cudaStream_t st) {
  if constexpr (LZ >= 8 && LZ <= 32) {
    const bool half = 2 * p.mz == LZ;
    const bool rag = p.tma_g != 1 || p.T % (128 / LZ) != 0;
    void (*k)(C2Maps, PassCParams) =
        rag ? (half ? pass_c4_kernel<LZ, LT, CP, EPI, true, true> : pass_c4_kernel<LZ, LT, CP, EPI, false, true>)
            : (half ? pass_c4_kernel<LZ, LT, CP, EPI, true, false> : pass_c4_kernel<LZ, LT, CP, EPI, false, false>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<grid, C4T, smem, st>>>(maps, p);
    return cudaGetLastError();
  } else {
    return cudaErrorInvalidValue;
  }
}

// per-(width, epilogue) entry points: one translation unit each
// (pass_c4_cp<CP>_<mode>.cu, generated by scripts/gen_pass_c4_tus.py)
#define FNO_C4_DECL(cp, e)                                                                                       \
  cudaError_t launch_pass_c4_cp##cp##_##e(const C2Maps& maps, const PassCParams& p, int LZ, int LT, int grid, \
                                          size_t smem, cudaStream_t st);
#define FNO_C4_DECL3(cp) FNO_C4_DECL(cp, u) FNO_C4_DECL(cp, fwd) FNO_C4_DECL(cp, bwd)
FNO_C4_DECL3(4)
FNO_C4_DECL3(8)
FNO_C4_DECL3(12)
FNO_C4_DECL3(16)
FNO_C4_DECL3(20)
FNO_C4_DECL3(24)
FNO_C4_DECL3(32)
#undef FNO_C4_DECL3
#undef FNO_C4_DECL

}  // namespace fno
