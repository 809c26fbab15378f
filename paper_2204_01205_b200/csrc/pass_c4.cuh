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
//                one 5-D tensor-map box per input (c2_encode_tile_map), and
//                (when it fits) the next column's retained-mode slab by 1-D
//                bulk copies, so phase 1 reads shared memory instead of L2
//   warp  5      TMEM owner and MMA issuer (one thread): kind::tf32 3xTF32
//                  D1[p][n]  = sum_k A1[p][k] B1[n][k]   (M128 x N NP x K KP)
//                    fwd: A1 = v^T | 1, B1 = W | b;  bwd: A1 = dz^T, B1 = W^T
//                  D2[o][i]  = sum_p dz[o][p] v'[i][p]   (bwd, M128 x N NW x K128)
//                    v' = v rows and a ones row (-> db); A2 stores only the
//                    ceil(C/8) real row groups, the M = 128 over-read lands in
//                    the following K groups (rows >= C of D2 are never read)
//   warps 0-3,   two split + epilogue warpgroups, even and odd tiles (thread =
//   8-11         tile point = TMEM lane; warps w and w + 8 share the lane
//                quarter w): each splits its tile k into the K-major tf32 hi /
//                lo operands, then finishes its previous tile k-2: D1 row + U
//                column (fwd: GELU, z) -> float4 stores; bwd: warps 0 and 8 add
//                the D2 rows (dW, db) of every tile into fp32 registers (a
//                per-tile flush keeps the tensor-core sums short)
//   warps 6, 7,  transforms: per column phase 1 (inverse t of the slab, C2R
//   12-15        weights and 1/N folded in -> Bb), per tile phase 2 (inverse z
//                of residue class rz -> U[k & 1])
// 16 warps at <= 128 registers; the two epilogue warpgroups give the
// latency-bound epilogue (TMEM load, U, GELU, float4 stores) two tiles in flight.
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

constexpr int C4T = 512;            // 16 warps
constexpr int C4_NTT = 192;         // transform threads (warps 6, 7, 12-15)
constexpr int C4_PROD = 4, C4_MMA = 5;
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
  int NS, NUB, NOB, SL, KP, NP, NW, RG, nk, TP, UPS;
  size_t x, xstage, op, opstage, a1hi, a1lo, a2hi, a2lo, b2hi, b2lo, b1hi, b1lo, bb, u0, ustride, sl, twz, twt, dmap, bar, slot,
      red, total;
};

// NS: input-tile ring stages; NUB: U buffers (2, or 4 = two per epilogue
// warpgroup, so the transforms run a tile further ahead); operand buffers: 2
// (fwd), 1 (bwd)
// SL: the column's slab staged in shared memory by a TMA bulk copy (issued by
// the producer one column ahead), so phase 1 reads shared memory, not L2
__host__ __device__ inline C4Layout c4_layout(int CP, int mode, int C, int Z, int T, int mz, int LZ, int NS,
                                              int NUB = 2, int SL = 0, int mt = 0) {
  C4Layout L{};
  L.NUB = NUB;
  L.SL = SL;
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
  // U buffers only need 16-byte rows: 128-byte granules (c3 forward: four U
  // buffers next to the staged slab then fit 227 KB)
  L.ustride = (size_t(C) * L.UPS * sizeof(float) + 127) & ~size_t(127);
  L.u0 = take(L.ustride * NUB);
  L.sl = take(SL ? size_t(C) * 2 * mz * mt * sizeof(float2) : 0);
  auto take16 = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
  L.twz = take16(size_t(Z) * sizeof(float2));
  L.twt = take16(size_t(T) * sizeof(float2));
  L.dmap = take16(size_t(2 * mz) * sizeof(short2));
  L.bar = take16(40 * sizeof(uint64_t));
  L.slot = take16(sizeof(uint32_t));
  L.red = take16(bwd ? size_t(2) * 32 * L.NW * sizeof(float) : 16);   // dW / db sums of the two warpgroups
  L.total = off;
  return L;
}

// Development builds (-DFNO_C4_PROFILE, scripts/variant_libs.sh): per-CTA
// clock64 timers of each role's waits and work: slot i of CTA b at p.prof[16 b + i]
// (the pass B scratch H, unused during pass C).
#ifdef FNO_C4_PROFILE
#define C4P_DECL unsigned long long c4p[16] = {0};
#define C4P_T(v) const long long v = clock64();
#define C4P_ADD(slot, v) c4p[slot] += (unsigned long long)(clock64() - (v));
#define C4P_DUMP(cond, first, n)                                                               \
  if ((cond) && p.prof)                                                                        \
    for (int i_ = 0; i_ < (n); ++i_) p.prof[16ll * blockIdx.x + (first) + i_] = c4p[(first) + i_];
#else
#define C4P_DECL
#define C4P_T(v)
#define C4P_ADD(slot, v)
#define C4P_DUMP(cond, first, n)
#endif

// SLT: the staged-slab configuration (NX bit 16) at compile time -- one phase-1
// path per instantiation; the smaller kernel measured faster (instruction-cache
// stalls: c3 forward 1.064 -> 1.023, dv leg 0.809 -> 0.729 ms/launch)
template <int LZ, int LT, int CP, int EPI, bool HALF, bool RAG, bool SLT>
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
  // (no run-time realignment of the base: pointer arithmetic through an
  // integer cast loses the shared state space and turns every operand access
  // into a generic LD / ST; SWIZZLE_NONE operands and TMA boxes need 128 B)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const int NS = MMA ? (p.NX & 255) : 1;
  const int NUB = ((p.NX >> 8) & 255) == 4 ? 4 : 2;
  constexpr bool SL = SLT;
  const C4Layout L = c4_layout(CP, EPI, C, Z, T, mz, LZ, NS, NUB, SL ? 1 : 0, mt);
  const float2* sl = reinterpret_cast<const float2*>(smem_raw + L.sl);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  uint64_t* xfull = bars;          // [NS]  TMA bytes landed
  uint64_t* xempty = bars + 8;     // [NS]  4 split warps done reading
  uint64_t* opfull = bars + 16;    // [2]   4 split warps wrote the operands
  uint64_t* opempty = bars + 18;   // [2]   MMAs done reading them (tcgen05.commit)
  uint64_t* dfull = bars + 20;     // [2]   MMAs done writing D[b] (tcgen05.commit)
  uint64_t* dempty = bars + 22;    // [2]   4 epilogue warps read D[b]
  uint64_t* ufull = bars + 24;     // [NUB] 6 transform warps wrote U[k % NUB]
  uint64_t* uempty = bars + 28;    // [NUB] 4 epilogue warps read U[k % NUB]
  uint64_t* slfull = bars + 32;    // [1]   the column's slab landed (SL)
  uint64_t* slempty = bars + 33;   // [1]   6 transform warps finished phase 1 (SL)
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
        if (k < C) w = (BWD || p.w_t) ? p.W[k * C + n] : p.W[n * C + k];
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
    // consumer / producer groups arrive once per warp (lane 0 after a
    // __syncwarp): every mbarrier event wakes the warps sleeping in try_wait,
    // so per-thread arrivals would keep the waiting roles spinning
    for (int s = 0; s < NS && MMA; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&opfull[b], 4);
      mbar_init(&opempty[b], 1);
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], 4);
    }
    mbar_init(slfull, 1);
    mbar_init(slempty, C4_NTT / 32);
    for (int b = 0; b < NUB; ++b) {
      mbar_init(&ufull[b], C4_NTT / 32);
      mbar_init(&uempty[b], 4);
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
  auto tile_t0 = [&](int rz, int tc) {
    return tc * TCH - ((RAG && p.tma_g > 1) ? ((rz & (p.tma_g - 1)) * T) & 3 : 0);
  };
  // (rz, tc) of the next tile: t chunks innermost (ti = rz * nch + tc)
  auto next_tile = [&](int& rz, int& tc) {
    if (++tc == nch) { tc = 0; ++rz; }
  };
  auto xstage = [&](int s) { return reinterpret_cast<float*>(smem_raw + L.x + s * L.xstage); };
  auto opbuf = [&](int ob) { return smem_raw + L.op + ob * L.opstage; };

  if (warp == C4_PROD) {
    // ======================= TMA producer ========================================
    if ((MMA || SL) && lane == 0) {
      C4P_DECL
      int s = 0;
      unsigned xph = 0;   // parity of the ring's current pass
      unsigned ci = 0;    // column count (slab parity)
      for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x, ++ci) {
        int bb;
        const int xy = col_split(col, &bb);
        if (SL) {   // the column's slab, one bulk copy per kz owner chunk (stacked in owner order)
          mbar_wait(slempty, (ci & 1u) ^ 1u);
          mbar_expect_tx(slfull, unsigned(C) * 2 * mz * mt * sizeof(float2));
          for (int d = 0; d < p.slab.P; ++d) {
            const int nkz_d = p.slab.kz_lo[d + 1] - p.slab.kz_lo[d];
            if (nkz_d == 0) continue;
            const unsigned bytes = unsigned(C) * nkz_d * mt * sizeof(float2);
            tma_load_1d(const_cast<float2*>(sl) + (long long)C * mt * p.slab.kz_lo[d],
                        p.in + p.slab.off[d] + col * C * nkz_d * mt, bytes, slfull);
          }
        }
        if (!MMA) continue;
        int rz = 0, tc = 0;
        for (int ti = 0; ti < tpc; ++ti, next_tile(rz, tc)) {
          C4P_T(tw0)
          mbar_wait(&xempty[s], xph ^ 1u);
          C4P_ADD(0, tw0)
          mbar_expect_tx(&xfull[s], tile_bytes * NA);
          const int r = (rz & (p.tma_g - 1)) * T;
#pragma unroll
          for (int a = 0; a < NA; ++a)
            tma_load_5d(xstage(s) + a * C * 128, &maps.m[a], r + tc * TCH - (r & 3), rz / p.tma_g, 0, xy, bb * C,
                        &xfull[s]);
          if (++s == NS) { s = 0; xph ^= 1u; }
        }
      }
      C4P_DUMP(true, 0, 1)
    }
  } else if (warp == C4_MMA) {
    // ======================= MMA issuer ==========================================
    if (MMA && lane == 0) {
      const uint32_t idesc1 = umma_idesc_tf32(128, NP, 0, 0);
      const uint32_t idesc2 = umma_idesc_tf32(128, NW, 0, 0);
      constexpr uint32_t A1_LBO = (128 / 8) * 128, B1_LBO = (NP / 8) * 128;
      constexpr uint32_t A2_LBO = RG * 128, B2_LBO = (NW / 8) * 128;
      // descriptors of operand buffer 0 and K step 0; the start address field
      // (bits 0-13, 16-byte units) advances by plain 64-bit adds
      const uint64_t a1hi0 = umma_sdesc(opbuf(0) + L.a1hi, A1_LBO, 128);
      const uint64_t a1lo0 = umma_sdesc(opbuf(0) + L.a1lo, A1_LBO, 128);
      const uint64_t b1hi0 = umma_sdesc(smem_raw + L.b1hi, B1_LBO, 128);
      const uint64_t b1lo0 = umma_sdesc(smem_raw + L.b1lo, B1_LBO, 128);
      const uint64_t a2hi0 = umma_sdesc(opbuf(0) + L.a2hi, A2_LBO, 128);
      const uint64_t a2lo0 = umma_sdesc(opbuf(0) + L.a2lo, A2_LBO, 128);
      const uint64_t b2hi0 = umma_sdesc(opbuf(0) + L.b2hi, B2_LBO, 128);
      const uint64_t b2lo0 = umma_sdesc(opbuf(0) + L.b2lo, B2_LBO, 128);
      const uint64_t obstep = uint64_t(L.opstage >> 4);
      C4P_DECL
      unsigned k = 0;
      for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
        for (int ti = 0; ti < tpc; ++ti, ++k) {
          const int b = k & 1;
          const unsigned u = k >> 1;
          const int ob = NOB == 2 ? b : 0;
          C4P_T(tm0)
          mbar_wait(&opfull[b], u & 1u);   // tile k's operands (per-parity barrier: no phase aliasing)
          C4P_ADD(1, tm0)
          C4P_T(tm1)
          mbar_wait(&dempty[b], (u & 1u) ^ 1u);
          C4P_ADD(2, tm1)
          tc_fence_after();
          const uint64_t oo = uint64_t(ob) * obstep;
          const uint32_t d1 = tmem + 32u * b;
#pragma unroll
          for (int j = 0; j < KP / 8; ++j) {
            const uint64_t ja = uint64_t(j) * ((2 * A1_LBO) >> 4), jb = uint64_t(j) * ((2 * B1_LBO) >> 4);
            umma_tf32(d1, a1hi0 + oo + ja, b1hi0 + jb, idesc1, j > 0 ? 1u : 0u);
            umma_tf32(d1, a1lo0 + oo + ja, b1hi0 + jb, idesc1, 1u);
            umma_tf32(d1, a1hi0 + oo + ja, b1lo0 + jb, idesc1, 1u);
          }
          if (BWD) {
            const uint32_t d2 = tmem + 64u + uint32_t(NW) * b;
            uint64_t ah = a2hi0 + oo, al = a2lo0 + oo, bh = b2hi0 + oo, bl = b2lo0 + oo;
#pragma unroll 2
            for (int j = 0; j < 128 / 8; ++j) {   // loop-carried descriptors (few registers)
              umma_tf32(d2, ah, bh, idesc2, j > 0 ? 1u : 0u);
              umma_tf32(d2, al, bh, idesc2, 1u);
              umma_tf32(d2, ah, bl, idesc2, 1u);
              ah += (2 * A2_LBO) >> 4; al += (2 * A2_LBO) >> 4;
              bh += (2 * B2_LBO) >> 4; bl += (2 * B2_LBO) >> 4;
            }
          }
          umma_commit(&opempty[b]);
          umma_commit(&dfull[b]);
        }
      }
      C4P_DUMP(true, 1, 2)
    }
  } else if (warp == 6 || warp == 7 || warp >= 12) {
    // ======================= transforms (phases 1-2) ===============================
    const int ttid = (warp < 8 ? warp - 6 : warp - 10) * 32 + lane;
    // staged slab (SL): chunk d at C mt kz_lo[d], rows (c, jz - kz_lo[d]) of that chunk
    // (an offset into the shared array, so the loads stay LDS)
    auto sl_off = [&](int c, int jz) -> int {
      if (p.slab.P == 1) return (c * 2 * mz + jz) * mt;
      const short2 dm = dmap[jz];
      const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
      return C * mt * p.slab.kz_lo[dm.x] + (c * nkz + dm.y) * mt;
    };
    auto slab_at = [&](long long c_, int c, int jz) -> const float2* {
      if (p.slab.P == 1) return p.in + (c_ * C + c) * per_c + jz * mt;
      const short2 dm = dmap[jz];
      const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
      return p.in + p.slab.off[dm.x] + ((c_ * C + c) * nkz + dm.y) * mt;
    };
    C4P_DECL
    unsigned k = 0, ci = 0;
    for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x, ++ci) {
      const long long col_next = col + gridDim.x;
      C4P_T(tp1)
      group_sync(2, C4_NTT);   // the previous column's phase 2 is done with Bb
      if (SL) mbar_wait(slfull, ci & 1u);   // this column's slab in shared memory
      // ---- phase 1: inverse t (C2R weights and 1/N folded in), items (c, kz', rt)
      for (int it = ttid; it < C * nk * p.Qt; it += C4_NTT) {
        const int rt = it % p.Qt;
        const int pid = it / p.Qt;
        const int c = pid / nk, kzp = pid - c * nk;
        const int jzp = kzp < mz ? kzp : 0, jzn = kzp >= 1 ? 2 * mz - kzp : 0;
        const float2* Sp = SL ? nullptr : slab_at(col, c, jzp);
        const float2* Sn = SL ? nullptr : slab_at(col, c, jzn);
        const int op = SL ? sl_off(c, jzp) : 0, on = SL ? sl_off(c, jzn) : 0;
        float2 e[LT];
#pragma unroll
        for (int i = 0; i < LT; ++i) {
          float2 acc = make_float2(0.f, 0.f);
          if (i < mt && kzp < mz) {
            const float cw = (i == 0 || 2 * i == T) ? 1.f : 2.f;
            acc = cscale(SL ? sl[op + i] : __ldg(Sp + i), cw);
          }
          const int kt = (LT - i) % LT;
          if (kzp >= 1 && kt < mt && (i == 0 || i > LT - mt)) {
            const float cw = (kt == 0 || 2 * kt == T) ? 1.f : 2.f;
            acc = cadd(acc, cscale(cconj(SL ? sl[on + kt] : __ldg(Sn + kt)), cw));
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
      if (SL && lane == 0) mbar_arrive(slempty);   // the staged slab may be refilled
      C4P_ADD(8, tp1)
      if (!SL && col_next < p.n_cols)   // next column's slab rows into L1 (phase 1 then hits L1)
        for (int r = ttid; r < C * 2 * mz; r += C4_NTT)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(slab_at(col_next, r / (2 * mz), r % (2 * mz))));
      int rz = 0, tc = 0;
      for (int ti = 0; ti < tpc; ++ti, ++k, next_tile(rz, tc)) {
        const int t0 = tile_t0(rz, tc);
        const int b = NUB == 4 ? int(k & 3u) : int(k & 1u);
        const unsigned u = NUB == 4 ? (k >> 2) : (k >> 1);
        C4P_T(tp2)
        // one waiter, the other transform warps park on the named barrier (no
        // issue slots spent polling)
        if (ttid == 0) mbar_wait(&uempty[b], (u & 1u) ^ 1u);
        group_sync(2, C4_NTT);
        mbar_wait(&uempty[b], (u & 1u) ^ 1u);
        C4P_ADD(9, tp2)
        C4P_T(tp3)
        float* U = reinterpret_cast<float*>(smem_raw + L.u0 + b * L.ustride);
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
        __syncwarp();
        if (lane == 0) mbar_arrive(&ufull[b]);
        C4P_ADD(10, tp3)
      }
    }
    C4P_DUMP(ttid == 0, 8, 3)
  } else {
    // ======================= split + epilogue (TMEM lanes), warps 0-3 | 8-11 ========
    const int ew = warp & 3, wg = warp >> 3;   // lane quarter, warpgroup (even / odd tiles)
    const int et = ew * 32 + lane;             // tile point of the epilogue, operand row of the split
    const int gbar = 1 + 2 * wg;               // this warpgroup's named barrier
    C4P_DECL
    const uint32_t t_row = tmem + ((uint32_t)(32 * ew) << 16);
    // bwd: this warpgroup's dW / db running sums (rows o = lane of warp ew == 0)
    float* dwsum = reinterpret_cast<float*>(smem_raw + L.red) + wg * 32 * NW;
    if (BWD && ew == 0)
      for (int i = 0; i < NW; ++i) dwsum[lane * NW + i] = 0.f;

    // operands of tile k (col, ti) from its X stage
    int xs = wg;
    unsigned xph = 0;   // X ring position of this warpgroup's next split (tiles wg, wg + 2, ...)
    auto split = [&](unsigned k, int rz, int tc) {
      const int s = xs;
      const int ob = NOB == 2 ? int(k & 1) : 0;

      C4P_T(ts0)
      if (et == 0) {   // one waiter; the other split threads park on the named barrier
        mbar_wait(&xfull[s], xph);
        // operand buffer free: fwd (two buffers) after MMA(k-2), bwd (one buffer,
        // shared by the two warpgroups) after MMA(k-1) -- each waited on the
        // per-parity barrier it committed to, so no waiter can be two phases behind
        if (NOB == 2) mbar_wait(&opempty[k & 1], ((k >> 1) & 1u) ^ 1u);
        else if (k > 0) mbar_wait(&opempty[(k - 1) & 1], ((k - 1) >> 1) & 1u);
      }
      group_sync(gbar, 128);
      mbar_wait(&xfull[s], xph);   // completed: one test, the acquire of the TMA bytes for this thread
      xs += 2;
      if (xs >= NS) { xs -= NS; xph ^= 1u; }
      C4P_ADD(3, ts0)
      C4P_T(ts1)
      const float* X0 = xstage(s);   // v (fwd) or dz (bwd): [C][128]
      unsigned char* base = opbuf(ob);
      float* A1hi = reinterpret_cast<float*>(base + L.a1hi);
      float* A1lo = reinterpret_cast<float*>(base + L.a1lo);
      // A1[p][k] = X0[k][p] (K-major, 4 channels per float4)
      // (fully unrolled, loads first: the warps of this role are few, so every
      // hand-off must expose instruction-level parallelism)
      float xa[CP];
#pragma unroll
      for (int k = 0; k < CP; ++k) xa[k] = (k < C) ? X0[k * 128 + et] : 0.f;
#pragma unroll
      for (int g = 0; g < CP / 4; ++g) {
        const int pp = et;
        const float x[4] = {xa[4 * g], xa[4 * g + 1], xa[4 * g + 2], xa[4 * g + 3]};
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
        const int t0 = tile_t0(rz, tc);
        const int ta = RAG ? max(0, -t0) : 0, tb = RAG ? min(TCH, T - t0) : TCH;
        const float* V0 = X0 + C * 128;
        float* A2hi = reinterpret_cast<float*>(base + L.a2hi);
        float* A2lo = reinterpret_cast<float*>(base + L.a2lo);
        float* B2hi = reinterpret_cast<float*>(base + L.b2hi);
        float* B2lo = reinterpret_cast<float*>(base + L.b2lo);
        const int w = ew, j8 = lane & 7, ph = lane >> 3;
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
      fence_proxy_async();       // generic-proxy operand stores -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&xempty[s]);   // the warp's reads of the X stage are done
        mbar_arrive(&opfull[k & 1]);
      }
      C4P_ADD(4, ts1)
    };

    // results of tile k (col, ti): D1 row + U column -> stores; bwd: D2 -> dW, db
    auto epilogue = [&](unsigned k, long long col, int rz, int tc) {
      const int b = k & 1;                      // TMEM D buffer = this warpgroup's
      const unsigned u = k >> 1;
      const int ub = NUB == 4 ? int(k & 3u) : b;  // U buffer
      const unsigned uu = NUB == 4 ? (k >> 2) : u;
      float* U = reinterpret_cast<float*>(smem_raw + L.u0 + ub * L.ustride);
      const int t0 = tile_t0(rz, tc);
      C4P_T(te0)
      if (et == 0) {   // one waiter; the other epilogue threads park on the named barrier
        mbar_wait(&ufull[ub], uu & 1u);
        if (MMA) mbar_wait(&dfull[b], u & 1u);
      }
      group_sync(gbar, 128);
      mbar_wait(&ufull[ub], uu & 1u);             // completed: one test each (acquire)
      if (MMA) mbar_wait(&dfull[b], u & 1u);
      C4P_ADD(5, te0)
      C4P_T(te2)
      if (MMA) {
        tc_fence_after();
        uint32_t d[NCH1][8];
#pragma unroll
        for (int q = 0; q < NCH1; ++q) tmem_ld8_nowait(t_row + 32u * b + 8 * q, d[q]);
        if (BWD && ew == 0) {   // D2 rows (dW, db) first, 8 columns at a time: few live registers
#pragma unroll 1
          for (int q = 0; q < (BWD ? NW / 8 : 0); ++q) {
            uint32_t d2[8];
            tmem_ld8_nowait(t_row + 64u + uint32_t(NW) * b + 8 * q, d2);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) dwsum[lane * NW + 8 * q + j] += __uint_as_float(d2[j]);
          }
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[b]);
        float uv[CP];
#pragma unroll
        for (int o = 0; o < CP; ++o) uv[o] = (o < C) ? U[o * UPS + et] : 0.f;
#pragma unroll
        for (int o = 0; o < CP; ++o)
          if (o < C) U[o * UPS + et] = uv[o] + __uint_as_float(d[o >> 3][o & 7]);

      }
      __syncwarp();
      int bcol;
      const int xycol = col_split(col, &bcol);
      const long long cbase = (long long)bcol * C * chan_stride + (long long)xycol * ZT;
      // float4 f of the warp: channel o, points 32 warp + 4 (lane % 8) + [0, 4)
      const int pq = 32 * ew + 4 * (lane & 7);
      const int sq = pq / TCH, tq = pq - sq * TCH;
      const long long gq = cbase + (long long)(rz + p.Qz * sq) * T + t0 + tq;
      const int k0 = RAG ? max(0, -(t0 + tq)) : 0, k1 = RAG ? min(4, T - t0 - tq) : 4;
      const bool v4 = !RAG || (k0 == 0 && k1 == 4);   // TMA tiles start 16-byte aligned
      constexpr int NJ = (CP + 3) / 4;
      float4 rq[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int o = (lane >> 3) + 4 * j;
        rq[j] = (o < C) ? *reinterpret_cast<const float4*>(U + o * UPS + pq) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int o = (lane >> 3) + 4 * j;
        if (o >= C || k0 >= k1) continue;
        float4 r = rq[j];
        const long long g = gq + o * chan_stride;
        // one copy of the GELU for the full-quad and the ragged stores (code size:
        // the kernel is instruction-cache bound)
        if (EPI == EPI_FWD) {
          if (p.zsave) {
            if (v4) __stcs(reinterpret_cast<float4*>(p.zsave + g), r);
            else store_quad_part(p.zsave + g, r, k0, k1);
          }
          if (p.act_gelu) {
            r.x = gelu_f(r.x); r.y = gelu_f(r.y); r.z = gelu_f(r.z); r.w = gelu_f(r.w);
          }
        }
        if (v4) __stcs(reinterpret_cast<float4*>(p.out + g), r);
        else store_quad_part(p.out + g, r, k0, k1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&uempty[ub]);   // U[ub] free
      C4P_ADD(7, te2)
    };

    C4P_T(tall)
    unsigned k = 0, pk = 0;
    long long pcol = -1;
    int prz = 0, ptc = 0;
    for (long long col = blockIdx.x; col < p.n_cols; col += gridDim.x) {
      int rz = 0, tc = 0;
      for (int ti = 0; ti < tpc; ++ti, ++k, next_tile(rz, tc)) {
        if (int(k & 1u) != wg) continue;   // the other warpgroup's tile
        if (MMA) split(k, rz, tc);
        if (pcol >= 0) epilogue(pk, pcol, prz, ptc);
        pcol = col;
        prz = rz;
        ptc = tc;
        pk = k;
      }
    }
    if (pcol >= 0) epilogue(pk, pcol, prz, ptc);
    C4P_ADD(11, tall)
    C4P_DUMP(tid == 0, 3, 5)
    C4P_DUMP(tid == 0, 11, 1)
    tc_fence_before();
    if (BWD) {
      // the even (warp 0) and odd (warp 8) tiles' dW / db partials, in a fixed order
      const float* red = reinterpret_cast<const float*>(smem_raw + L.red);
      if (warp == 0 || warp == 8) group_sync(4, 64);
      if (warp == 0 && lane < C) {
        float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
        for (int i = 0; i <= C; ++i) {
          const float v = red[lane * NW + i] + red[32 * NW + lane * NW + i];
          if (i < C) outp[lane * C + i] = v;
          else outp[C * C + lane] = v;
        }
      }
    }
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
    const bool sl = (p.NX >> 16) & 1;
    if (EPI == EPI_BWD && sl) return cudaErrorNotSupported;   // the backward is not configured with a staged slab
    constexpr bool SLOK = EPI != EPI_BWD;
    void (*k)(C2Maps, PassCParams) =
        sl ? (rag ? (half ? pass_c4_kernel<LZ, LT, CP, EPI, true, true, SLOK> : pass_c4_kernel<LZ, LT, CP, EPI, false, true, SLOK>)
                  : (half ? pass_c4_kernel<LZ, LT, CP, EPI, true, false, SLOK> : pass_c4_kernel<LZ, LT, CP, EPI, false, false, SLOK>))
           : (rag ? (half ? pass_c4_kernel<LZ, LT, CP, EPI, true, true, false> : pass_c4_kernel<LZ, LT, CP, EPI, false, true, false>)
                  : (half ? pass_c4_kernel<LZ, LT, CP, EPI, true, false, false> : pass_c4_kernel<LZ, LT, CP, EPI, false, false, false>));
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
FNO_C4_DECL3(20)
#undef FNO_C4_DECL3
#undef FNO_C4_DECL

}  // namespace fno
