// Pass C (bwd a9, a12): the adjoint chain of I_1 =
// {z, t} (zero-padded inverse z, C2R along t with real-part semantics,
// P:119-123 "F_dist^T"), fused with the DFNO block epilogue
//   z = W v + b + u ; y = GELU(z)                      (Eq. dist_block)
// or, backward, dv = W^T dz + S^T dz plus the dW, db sums (broadcast adjoint =
// sum-reduce).
//
// One persistent CTA loops over (b, x, y) columns (all channels at once: the
// 1x1 channel linear needs every channel at a point).  The z outputs are
// produced by residue class r (z = r + Qz*s, s < LZ) and t-chunk, so a tile is
// LZ x TCH points x C channels.
//
// Warp specialisation (layer fwd / bwd):
//   producer warps 0-7: per column the inverse t transform; per tile the
//     cp.async prefetch of the next tile's inputs, the inverse z transform
//     (-> U, the spectral part), the tf32 hi/lo split into the tensor-core
//     operand layouts and, from one elected lane, the tcgen05.mma issue;
//   epilogue warps 8-15: TMEM -> registers, + U + bias, GELU, stores (fwd) or
//     dv stores and the dW/db accumulation (bwd).
// U and the TMEM accumulators are double-buffered, so the producers transform
// tile n+1 while the epilogue drains tile n; mbarriers (full / empty /
// mma-done) order the two roles.
//
// The channel contractions are dense GEMMs on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), in 3xTF32 form
// (a_hi b_hi + a_hi b_lo + a_lo b_hi) so the result keeps fp32 accuracy:
//   fwd:  D[point][o] = sum_i V[point][i] W[o][i]          M=128 points, N=o, K=i
//   bwd:  D[point][i] = sum_o dz[point][o] W[o][i]         (W^T dz)
//         D2[o][i]    = sum_points dz[point][o] v[point][i] (dW; column i=C is a
//                       ones channel, giving db)           M=128 (o), N=i, K=points
// Operands are K-major "interleaved" core matrices (8 rows x 16 bytes,
// SWIZZLE_NONE), float offsets:
//   KM  (rows = points, K = channels): ((c/4)*NBm + m/8)*32 + (m%8)*4 + (c%4)
//   CM  (rows = channels, K = points): ((m/4)*C8 + c/8)*32 + (c%8)*4 + (m%4)
// with NBm = points/8 and C8 = channel blocks of 8.
#include "kernels.cuh"
#include "launch.h"
#include "umma.cuh"

namespace fno {

static constexpr int CT = 512;  // threads per CTA (16 warps)
static constexpr int FT = 256;  // producer threads (warps 0-7)

__device__ __forceinline__ void f_bar() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

struct CLayout {
  int Cp, nk, TP, RS, NPS, npad, NAR, KP, C8, N1, N2, MT, dcols, tcols;
  size_t wb, bias, s, bb, u0, u1, r0, r1, cmv0, cmv1, kmh, kml, cmdh, cmdl, cmvl, dwacc, twz, twt, dmap, bars, tmem,
      total;
};

__host__ __device__ inline CLayout c_layout(int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode) {
  CLayout L{};
  const bool tc = mode != EPI_U, bwd = mode == EPI_BWD;
  L.Cp = (C + 3) & ~3;
  L.nk = mz + 1;
  L.TP = T + 1;
  L.RS = (TCH + 3) & ~3;                      // point-groups of 4 never straddle a z row
  L.NPS = LZ * L.RS;                          // points per tile (incl. padding)
  L.npad = (L.NPS + 127) & ~127;              // whole 128-row MMA tiles
  L.MT = L.npad / 128;
  L.NAR = mode == EPI_FWD ? 1 : (bwd ? 2 : 0);  // raw [c][point] staging arrays: v | dy, z
  L.KP = ((C + 7) / 8) * 8;                   // K of the W GEMMs (channels, padded to 8)
  L.C8 = (C + 1 + 7) / 8;                     // channel blocks of the CM layout (+ ones channel)
  L.N1 = ((C + 15) / 16) * 16;                // MMA N of the W GEMMs
  L.N2 = ((C + 1 + 15) / 16) * 16;            // MMA N of dW (incl. the ones column)
  L.dcols = tc ? L.MT * L.N1 + (bwd ? L.N2 : 0) : 0;
  int alloc = 32;
  while (alloc < 2 * L.dcols) alloc *= 2;
  L.tcols = alloc;
  const size_t raw = size_t(C) * L.npad * sizeof(float);
  const size_t km = size_t(L.npad) * L.KP * sizeof(float);
  const size_t cm = size_t(L.npad) * L.C8 * 8 * sizeof(float);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 127) & ~size_t(127); return o; };
  L.wb = take(tc ? 2 * size_t(L.N1) * L.KP * sizeof(float) : 0);   // B hi, lo (K-major)
  L.bias = take(size_t(C) * sizeof(float));
  L.s = take(size_t(C) * 2 * mz * mt * sizeof(float2));
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.kmh = take(tc ? km : 0);
  L.kml = take(tc ? km : 0);
  L.cmdh = take(bwd ? cm : 0);
  L.cmdl = take(bwd ? cm : 0);
  L.cmvl = take(bwd ? cm : 0);
  L.cmv0 = take(bwd ? cm : 0);
  L.cmv1 = take(bwd ? cm : 0);
  L.u0 = take(tc ? size_t(C) * L.npad * sizeof(float) : 0);   // after the CM buffers: dW descriptors
  L.u1 = take(tc ? size_t(C) * L.npad * sizeof(float) : 0);   // may read a little past them
  L.r0 = take(size_t(L.NAR) * raw);
  L.r1 = take(size_t(L.NAR) * raw);
  L.dwacc = take(bwd ? size_t(C) * L.N2 * sizeof(float) : 0);
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  L.bars = take(6 * sizeof(uint64_t));
  L.tmem = take(sizeof(uint32_t));
  L.total = off;
  return L;
}

// per-column phase 1: inverse t with the C2R weights folded in, pencils (c, kz')
template <int LT>
__device__ __forceinline__ void phase1(const float2* S, float2* Bb, const float2* twT, int C, int T, int mz, int mt,
                                       int nk, int TP, int Qt, int tid, int nthr) {
  for (int pid = tid; pid < C * nk; pid += nthr) {
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
    for (int rt = 0; rt < Qt; ++rt) {
      float2 y[LT];
      trunc_inv<LT>(y, e, rt, twT);
#pragma unroll
      for (int s = 0; s < LT; ++s) bo[rt + Qt * s] = y[s];
    }
  }
}

// column index -> NCXYZT offset of (b, c=0, xl, yl, z=0, t=0)
__device__ __forceinline__ long long col_base_of(const PassCParams& p, long long c_, long long ZT, long long chan_stride) {
  const unsigned cu = unsigned(c_);            // n_cols < 2^31 (checked by the plan)
  const unsigned yl = cu % unsigned(p.Yl);
  const unsigned r1 = cu / unsigned(p.Yl);
  const unsigned xl = r1 % unsigned(p.Xl);
  const unsigned b = r1 / unsigned(p.Xl);
  return (long long)b * p.C * chan_stride + ((long long)xl * p.Yl + yl) * ZT;
}

__device__ __forceinline__ void issue_slab(const PassCParams& p, float2* S, const short2* dmap, long long colpt, int C,
                                           int mz, int mt, int tid, int nthr) {
  const int per_c = 2 * mz * mt;
  if (p.slab.P == 1 && (per_c & 1) == 0) {   // one owner: a contiguous run of C*2mz*mt complex
    const float2* src = p.in + colpt * C * per_c;
    for (int e = tid; e < C * per_c / 2; e += nthr) cp_async16(S + 2 * e, src + 2 * e);
    return;
  }
  for (int e = tid; e < C * per_c; e += nthr) {
    const int c = e / per_c, rem = e - c * per_c;
    const int jz = rem / mt, kt = rem - jz * mt;
    const short2 dm = dmap[jz];
    const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
    cp_async8(S + e, p.in + p.slab.off[dm.x] + ((colpt * C + c) * nkz + dm.y) * mt + kt);
  }
}

// ---------------------------------------------------------------------------
// spectral convolution only (u = S v): no channel contraction, all warps
// ---------------------------------------------------------------------------
template <int LZ, int LT>
__global__ void __launch_bounds__(CT, 1) pass_c_u_kernel(PassCParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt;
  const CLayout L = c_layout(C, Z, T, mz, mt, LZ, T, EPI_U);
  float2* S = reinterpret_cast<float2*>(smem_raw + L.s);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nk = L.nk, TP = L.TP;
  const long long ZT = (long long)Z * T;
  const long long chan_stride = (long long)p.Xl * p.Yl * ZT;
  long long col = blockIdx.x;
  if (col >= p.n_cols) return;
  fill_combine_table(twZ, LZ, p.Qz, Z, 0, +1, tid, nt);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, +1, tid, nt);
  for (int j = tid; j < 2 * mz; j += nt) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  __syncthreads();
  issue_slab(p, S, dmap, col, C, mz, mt, tid, nt);
  cp_commit();
  for (; col < p.n_cols; col += gridDim.x) {
    cp_wait<0>();
    __syncthreads();
    phase1<LT>(S, Bb, twT, C, T, mz, mt, nk, TP, p.Qt, tid, nt);
    __syncthreads();
    const long long col_next = col + gridDim.x;
    if (col_next < p.n_cols) issue_slab(p, S, dmap, col_next, C, mz, mt, tid, nt);
    cp_commit();
    const long long cbase = col_base_of(p, col, ZT, chan_stride);
    for (int rz = 0; rz < p.Qz; ++rz) {
      for (int pid = tid; pid < C * T; pid += nt) {
        const int c = pid / T, t = pid - c * T;
        float2 e[LZ];
#pragma unroll
        for (int i = 0; i < LZ; ++i) e[i] = (i < nk) ? Bb[(c * nk + i) * TP + t] : make_float2(0.f, 0.f);
        float2 y[LZ];
        trunc_inv<LZ>(y, e, rz, twZ);
        float* o = p.out + cbase + c * chan_stride + rz * T + t;
#pragma unroll
        for (int s = 0; s < LZ; ++s) __stcs(o + (long long)p.Qz * s * T, y[s].x * p.inv_n);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// DFNO block forward / backward with tensor-core channel contractions
// ---------------------------------------------------------------------------
template <int LZ, int LT, int EPI>
__global__ void __launch_bounds__(CT, 1) pass_c_kernel(PassCParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt, TCH = p.TCH;
  const CLayout L = c_layout(C, Z, T, mz, mt, LZ, TCH, EPI);
  constexpr bool BWD = (EPI == EPI_BWD);
  float* WB = reinterpret_cast<float*>(smem_raw + L.wb);
  float* bs = reinterpret_cast<float*>(smem_raw + L.bias);
  float2* S = reinterpret_cast<float2*>(smem_raw + L.s);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float* KMH = reinterpret_cast<float*>(smem_raw + L.kmh);
  float* KML = reinterpret_cast<float*>(smem_raw + L.kml);
  float* CMDH = reinterpret_cast<float*>(smem_raw + L.cmdh);
  float* CMDL = reinterpret_cast<float*>(smem_raw + L.cmdl);
  float* CMVL = reinterpret_cast<float*>(smem_raw + L.cmvl);
  float* DWA = reinterpret_cast<float*>(smem_raw + L.dwacc);   // [C][N2] fp32 dW/db accumulator
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L.bars);   // full[2], empty[2], mma[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + L.tmem);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nk = L.nk, TP = L.TP, RS = L.RS, NPS = L.NPS, C8 = L.C8, KP = L.KP, npad = L.npad, MT = L.MT;
  const int NBm = npad / 8;
  const long long ZT = (long long)Z * T;
  const long long chan_stride = (long long)p.Xl * p.Yl * ZT;
  const int nch = (T + TCH - 1) / TCH;
  const int tpc = p.Qz * nch;  // tiles per column

  const long long col0 = blockIdx.x;
  if (col0 >= p.n_cols) return;

  // ---- setup (all warps) -------------------------------------------------------
  fill_combine_table(twZ, LZ, p.Qz, Z, 0, +1, tid, CT);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, +1, tid, CT);
  for (int j = tid; j < 2 * mz; j += CT) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  for (int o = tid; o < C; o += CT) bs[o] = (EPI == EPI_FWD && p.bias) ? p.bias[o] : 0.f;
  {
    // B operand of the W GEMM, K-major interleaved: element (n, k) at
    // ((k/4)*(N1/8) + n/8)*32 + (n%8)*4 + (k%4); fwd B[n=o][k=i] = W[o][i],
    // bwd B[n=i][k=o] = W[o][i]; hi and lo parts for 3xTF32
    const int nb8 = L.N1 / 8;
    const int bfl = L.N1 * KP;
    for (int e = tid; e < bfl; e += CT) {
      const int kc = e / (nb8 * 32), r = e - kc * nb8 * 32;
      const int nb = r / 32, r2 = r - nb * 32;
      const int n = nb * 8 + r2 / 4, k = kc * 4 + (r2 & 3);
      float w = 0.f;
      if (n < C && k < C) w = (EPI == EPI_FWD) ? p.W[n * C + k] : p.W[k * C + n];
      const float hi = tf32_hi(w);
      WB[e] = hi;
      WB[bfl + e] = w - hi;
    }
  }
  {
    // zero the operand and staging buffers once: padded channels stay zero
    float* z0 = reinterpret_cast<float*>(smem_raw + L.kmh);
    const size_t nz = (L.twz - L.kmh) / sizeof(float);
    for (size_t e = tid; e < nz; e += CT) z0[e] = 0.f;
  }
  if (warp == 0) tmem_alloc(tmem_slot, L.tcols);
  if (tid == 0) {
    mbar_init(&bars[0], FT);  // full[0]
    mbar_init(&bars[1], FT);  // full[1]
    mbar_init(&bars[2], FT);  // empty[0]
    mbar_init(&bars[3], FT);  // empty[1]
    mbar_init(&bars[4], 1);   // mma[0]
    mbar_init(&bars[5], 1);   // mma[1]
    mbar_fence_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // =========================== producer warps ===============================
    const int ft = tid;
    // tile inputs: part 0 = the raw [c][point] staging arrays (v | dy, z);
    // part 1 = v in the CM operand layout (bwd; read by the dW MMA, so it is
    // only refilled after that MMA has completed)
    auto issue_tile = [&](long long cb, int ti, int b, int part) {
      if (part == 1 && !BWD) return;
      float* raw = reinterpret_cast<float*>(smem_raw + (b ? L.r1 : L.r0));
      float* cmv = reinterpret_cast<float*>(smem_raw + (b ? L.cmv1 : L.cmv0));
      const int rz = ti / nch, tc = ti - rz * nch;
      const int t0 = tc * TCH;
      const int tcw = min(TCH, T - t0);
      const long long base = cb + rz * T + t0;
      const int VW = p.VW;
      const int nvec = tcw / VW;                 // vectors per row (tcw % VW == 0 by construction)
      const int vv = ft % nvec, rstep = FT / nvec;
      for (int row = ft / nvec; row < C * LZ; row += rstep) {
        const int c = row / LZ, s = row - c * LZ;
        const long long g = base + c * chan_stride + (long long)p.Qz * s * T + vv * VW;
        const int m = s * RS + vv * VW;
        if (part == 0) {
          float* d0 = raw + c * npad + m;
          const float* s0 = BWD ? p.dy : p.v;
          if (VW == 4) cp_async16(d0, s0 + g);
          else if (VW == 2) cp_async8(d0, s0 + g);
          else cp_async4(d0, s0 + g);
          if (BWD) {
            float* d1 = raw + C * npad + c * npad + m;
            if (VW == 4) cp_async16(d1, p.zs + g);
            else if (VW == 2) cp_async8(d1, p.zs + g);
            else cp_async4(d1, p.zs + g);
          }
        } else {
          float* d2 = cmv + ((m >> 2) * C8 + (c >> 3)) * 32 + (c & 7) * 4 + (m & 3);
          if (VW == 4) cp_async16(d2, p.v + g);
          else if (VW == 2) cp_async8(d2, p.v + g);
          else cp_async4(d2, p.v + g);
        }
      }
    };

    issue_slab(p, S, dmap, col0, C, mz, mt, ft, FT);
    cp_commit();
    issue_tile(col_base_of(p, col0, ZT, chan_stride), 0, 0, 0);
    issue_tile(col_base_of(p, col0, ZT, chan_stride), 0, 0, 1);
    cp_commit();
    cp_wait<1>();  // S(col0)
    f_bar();
    int n = 0;     // tile sequence number of this CTA
    for (long long col = col0; col < p.n_cols; col += gridDim.x) {
      phase1<LT>(S, Bb, twT, C, T, mz, mt, nk, TP, p.Qt, ft, FT);
      f_bar();
      const long long cbase = col_base_of(p, col, ZT, chan_stride);
      const long long col_next = col + gridDim.x;
      const long long cbase_next = col_next < p.n_cols ? col_base_of(p, col_next, ZT, chan_stride) : 0;
      if (col_next < p.n_cols) issue_slab(p, S, dmap, col_next, C, mz, mt, ft, FT);  // S is free now
      cp_commit();
      for (int ti = 0; ti < tpc; ++ti, ++n) {
        const int b = n & 1;
        const int rz = ti / nch, tc = ti - rz * nch;
        const int t0 = tc * TCH;
        const int tcw = min(TCH, T - t0);
        const bool has_next = (ti + 1 < tpc) || (col_next < p.n_cols);
        const long long nb_base = (ti + 1 < tpc) ? cbase : cbase_next;
        const int nb_ti = (ti + 1 < tpc) ? ti + 1 : 0;
        if (has_next) issue_tile(nb_base, nb_ti, b ^ 1, 0);
        cp_commit();
        if (n >= 2) mbar_wait(&bars[2 + b], ((n - 2) >> 1) & 1);   // epilogue done with U[b], D[b]
        // ---- inverse z (real output) -> U[b], pencils (c, tt) ----------------
        float* U = reinterpret_cast<float*>(smem_raw + (b ? L.u1 : L.u0));
        for (int pid = ft; pid < C * tcw; pid += FT) {
          const int c = pid / tcw, tt = pid - c * tcw;
          const int t = t0 + tt;
          float2 e[LZ];
#pragma unroll
          for (int i = 0; i < LZ; ++i) e[i] = (i < nk) ? Bb[(c * nk + i) * TP + t] : make_float2(0.f, 0.f);
          float2 y[LZ];
          trunc_inv<LZ>(y, e, rz, twZ);
          float* uo = U + c * npad + tt;
#pragma unroll
          for (int s = 0; s < LZ; ++s) uo[s * RS] = y[s].x * p.inv_n;
        }
        cp_wait<1>();                       // this tile's inputs (and the next spectrum) landed
        if (n >= 1) mbar_wait(&bars[4 + (b ^ 1)], ((n - 1) >> 1) & 1);   // MMAs of tile n-1 done
        if (has_next) issue_tile(nb_base, nb_ti, b ^ 1, 1);             // v of tile n+1 -> CM[b^1]
        cp_commit();
        f_bar();
        // ---- tf32 hi/lo split + layout change (bwd: dz, invalid points, ones) --
        const float* R0 = reinterpret_cast<const float*>(smem_raw + (b ? L.r1 : L.r0));
        float* CMV = reinterpret_cast<float*>(smem_raw + (b ? L.cmv1 : L.cmv0));
        const int nc4 = BWD ? (C + 1 + 3) / 4 : (C + 3) / 4;
        for (int it = ft; it < (npad / 4) * nc4; it += FT) {
          const int g = it / nc4, cc = it - g * nc4;
          const int m0 = 4 * g;
          bool ok[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int m = m0 + j;
            const int s = m / RS, tt = m - s * RS;
            ok[j] = (m < NPS) && (tt < tcw);
          }
          float a[4][4];   // [channel j][point i]: v (fwd) or dz (bwd)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = 4 * cc + j;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f), zz = x;
            if (c < C) {
              x = *reinterpret_cast<const float4*>(R0 + c * npad + m0);
              if (BWD) zz = *reinterpret_cast<const float4*>(R0 + C * npad + c * npad + m0);
            }
            const float xs[4] = {x.x, x.y, x.z, x.w}, zs4[4] = {zz.x, zz.y, zz.z, zz.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (!BWD) a[j][i] = xs[i];
              else a[j][i] = (c < C && ok[i]) ? (p.act_gelu ? xs[i] * gelu_prime_f(zs4[i]) : xs[i]) : 0.f;
            }
          }
          if (4 * cc < KP) {   // KM (rows = points): A of the W GEMM
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int m = m0 + i;
              const int off = (cc * NBm + (m >> 3)) * 32 + (m & 7) * 4;
              float h[4], l[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                h[j] = tf32_hi(a[j][i]);
                l[j] = a[j][i] - h[j];
              }
              *reinterpret_cast<float4*>(KMH + off) = make_float4(h[0], h[1], h[2], h[3]);
              *reinterpret_cast<float4*>(KML + off) = make_float4(l[0], l[1], l[2], l[3]);
            }
          }
          if (BWD) {  // CM (rows = channels): dW GEMM operands dz (A) and v (B, hi in place)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int c = 4 * cc + j;
              if (c >= 8 * C8) continue;
              const int off = (g * C8 + (c >> 3)) * 32 + (c & 7) * 4;
              float4 v4 = *reinterpret_cast<const float4*>(CMV + off);
              const float vin[4] = {v4.x, v4.y, v4.z, v4.w};
              float dh[4], dl[4], vh[4], vl[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                dh[i] = tf32_hi(a[j][i]);
                dl[i] = a[j][i] - dh[i];
                const float vv = (c < C) ? (ok[i] ? vin[i] : 0.f) : ((c == C && ok[i]) ? 1.f : 0.f);
                vh[i] = tf32_hi(vv);
                vl[i] = vv - vh[i];
              }
              *reinterpret_cast<float4*>(CMDH + off) = make_float4(dh[0], dh[1], dh[2], dh[3]);
              *reinterpret_cast<float4*>(CMDL + off) = make_float4(dl[0], dl[1], dl[2], dl[3]);
              *reinterpret_cast<float4*>(CMV + off) = make_float4(vh[0], vh[1], vh[2], vh[3]);
              *reinterpret_cast<float4*>(CMVL + off) = make_float4(vl[0], vl[1], vl[2], vl[3]);
            }
          }
        }
        fence_proxy_async();   // generic smem writes -> visible to the tensor core (async proxy)
        mbar_arrive(&bars[b]); // full[b]: U[b] is written
        f_bar();
        // ---- tcgen05.mma from one elected lane of warp 0 --------------------
        if (warp == 0) {
          tc_fence_after();
          const bool leader = elect_one();
          const uint32_t dbase = tmem + b * L.dcols;
          const uint32_t idesc1 = umma_idesc_tf32(128, L.N1, 0, 0);
          const uint32_t lboA = NBm * 128;            // K-major A: 4-channel chunk stride
          const uint32_t lboB = (L.N1 / 8) * 128;     // K-major B: 4-channel chunk stride
          for (int m4 = 0; m4 < MT; ++m4) {
            for (int ks = 0; ks < KP / 8; ++ks) {
              const int ao = m4 * 16 * 32 + ks * 2 * NBm * 32;            // floats
              const uint64_t ah = umma_sdesc(KMH + ao, lboA, 128);
              const uint64_t al = umma_sdesc(KML + ao, lboA, 128);
              const uint64_t bh = umma_sdesc(WB + ks * 2 * (lboB / 4), lboB, 128);
              const uint64_t bl = umma_sdesc(WB + L.N1 * KP + ks * 2 * (lboB / 4), lboB, 128);
              if (leader) {
                umma_tf32(dbase + m4 * L.N1, ah, bh, idesc1, ks > 0 ? 1u : 0u);
                umma_tf32(dbase + m4 * L.N1, ah, bl, idesc1, 1u);
                umma_tf32(dbase + m4 * L.N1, al, bh, idesc1, 1u);
              }
            }
          }
          if (BWD) {
            const uint32_t idesc2 = umma_idesc_tf32(128, L.N2, 0, 0);
            const uint32_t d2 = dbase + MT * L.N1;
            for (int ks = 0; ks < npad / 8; ++ks) {
              const int ko = ks * 2 * C8 * 32;                              // 8 points = 2 groups
              const uint64_t ah = umma_sdesc(CMDH + ko, C8 * 128, 128);
              const uint64_t al = umma_sdesc(CMDL + ko, C8 * 128, 128);
              const uint64_t bh = umma_sdesc(CMV + ko, C8 * 128, 128);
              const uint64_t bl = umma_sdesc(CMVL + ko, C8 * 128, 128);
              if (leader) {
                umma_tf32(d2, ah, bh, idesc2, ks > 0 ? 1u : 0u);   // fresh per tile
                umma_tf32(d2, ah, bl, idesc2, 1u);
                umma_tf32(d2, al, bh, idesc2, 1u);
              }
            }
          }
          __syncwarp();
          if (leader) umma_commit(&bars[4 + b]);
        }
      }
    }
    cp_wait<0>();
  } else {
    // =========================== epilogue warps ===============================
    const int q = warp & 3;          // TMEM lane quadrant (== warp % 4)
    const int h = (warp - 8) >> 2;   // two epilogue warps per quadrant split the output columns
    int n = 0;
    for (long long col = col0; col < p.n_cols; col += gridDim.x) {
      const long long cbase = col_base_of(p, col, ZT, chan_stride);
      for (int ti = 0; ti < tpc; ++ti, ++n) {
        const int b = n & 1;
        const int rz = ti / nch, tc = ti - rz * nch;
        const int t0 = tc * TCH;
        const int tcw = min(TCH, T - t0);
        const long long tbase = cbase + rz * T + t0;
        mbar_wait(&bars[b], (n >> 1) & 1);       // U[b] written
        mbar_wait(&bars[4 + b], (n >> 1) & 1);   // MMAs of tile n done
        tc_fence_after();
        const float* U = reinterpret_cast<const float*>(smem_raw + (b ? L.u1 : L.u0));
        const uint32_t dbase = tmem + b * L.dcols + ((uint32_t)(32 * q) << 16);
        for (int m4 = 0; m4 < MT; ++m4) {
          const int m = m4 * 128 + 32 * q + lane;
          const int s = m / RS, tt = m - s * RS;
          const bool okp = (m < NPS) && (tt < tcw);
          const long long gs = tbase + (long long)p.Qz * s * T + tt;
          for (int c0 = 8 * h; c0 < C; c0 += 16) {
            float d8[8];
            tmem_ld8(dbase + m4 * L.N1 + c0, d8);
            if (!okp) continue;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int o = c0 + j;
              if (o < C) {
                float val = d8[j] + U[o * npad + m];
                const long long gi = gs + o * chan_stride;
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
        }
        if (BWD && h == 0 && 32 * q < C) {
          // this tile's dW/db (TMEM rows o, columns i; i = C is db) -> fp32 smem
          // accumulator, keeping the tensor-core accumulation depth to one tile
          const int o = 32 * q + lane;
          for (int c0 = 0; c0 <= C; c0 += 8) {
            float d8[8];
            tmem_ld8(dbase + MT * L.N1 + c0, d8);
            if (o < C) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (c0 + j <= C) DWA[o * L.N2 + c0 + j] += d8[j];
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&bars[2 + b]);   // empty[b]
      }
    }
  }
  __syncthreads();
  if (BWD) {
    float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
    for (int e = tid; e < C * C + C; e += CT) {
      if (e < C * C) {
        const int o = e / C, i = e - o * C;
        outp[e] = DWA[o * L.N2 + i];
      } else {
        outp[e] = DWA[(e - C * C) * L.N2 + C];
      }
    }
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, L.tcols);
  }
}

static size_t c_smem_for(int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode) {
  return c_layout(C, Z, T, mz, mt, LZ, TCH, mode).total;
}

void pass_c_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* TCH, int* VW, size_t* smem) {
  const size_t budget = 227 * 1024;
  // candidate chunks: T, then divisors of T that are multiples of 4, then any
  // multiple of 4 (descending) -- the first that fits
  int tch = T;
  size_t s = c_smem_for(C, Z, T, mz, mt, LZ, tch, mode);
  for (int pass = 0; pass < 2 && s > budget && mode != EPI_U; ++pass) {
    for (int cand = (T - 1) & ~3; cand >= 4; cand -= 4) {
      if (pass == 0 && T % cand) continue;
      tch = cand;
      s = c_smem_for(C, Z, T, mz, mt, LZ, tch, mode);
      if (s <= budget) break;
    }
  }
  int vw = 1;
  if (T % 4 == 0 && tch % 4 == 0) vw = 4;
  else if (T % 2 == 0 && tch % 2 == 0) vw = 2;
  if (vw > 1 && (T % tch) % vw != 0) vw = 1;   // ragged last chunk
  *TCH = tch;
  *VW = vw;
  *smem = s;
}

template <int LZ, int LT>
static cudaError_t launch_c(const PassCParams& p, int mode, int grid, size_t smem, cudaStream_t st) {
  void (*k)(PassCParams) = mode == EPI_U ? pass_c_u_kernel<LZ, LT>
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
