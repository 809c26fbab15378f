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
// LZ x TCH points x C channels.  Streaming is software-pipelined with cp.async:
// the next tile's inputs (v; or dy, z, v) and the next column's spectrum are in
// flight while the current tile is transformed and consumed.
//
// The channel contractions are dense GEMMs on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), in 3xTF32 form
// (a_hi b_hi + a_hi b_lo + a_lo b_hi) so the result keeps fp32 accuracy:
//   fwd:  D[point][o] = sum_i V[point][i] W[o][i]          M=128 points, N=o, K=i
//   bwd:  D[point][i] = sum_o dz[point][o] W[o][i]         (W^T dz)
//         D2[o][i]   += sum_points dz[point][o] v[point][i] (dW; column i=C is a
//                       ones channel, giving db)           M=128 (o), N=i, K=points
// All tensor-core operands are K-major "interleaved" core matrices (8 rows x 16
// bytes, SWIZZLE_NONE): the tile inputs land by 16-byte cp.async in a
// channel-major staging layout [c][point], and the tf32 hi/lo split pass writes
//   KM  (rows = points, K = channels): ((c/4)*NBm + m/8)*32 + (m%8)*4 + (c%4)
//   CM  (rows = channels, K = points): ((m/4)*C8 + c/8)*32 + (c%8)*4 + (m%4)
// (float offsets; NBm = points/8, C8 = channel blocks of 8).  KM feeds the W
// GEMMs (A), CM the dW GEMM (A = dz, B = v).
#include "kernels.cuh"
#include "launch.h"
#include "umma.cuh"

namespace fno {

static constexpr int CT = 256;  // threads per CTA (8 warps)

struct CLayout {
  int Cp, nk, TP, RS, NPS, NA, KP, C8, N1, N2, npad, tcols;
  size_t ws, bias, wb, s, bb, u, r0, r1, kmh, kml, cmdh, cmdl, cmvh, cmvl, twz, twt, dmap, dwacc, bar, tmem, total;
};

__host__ __device__ inline int c_num_arrays(int mode) { return mode == EPI_U ? 0 : (mode == EPI_FWD ? 1 : 3); }

__host__ __device__ inline CLayout c_layout(int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode) {
  CLayout L{};
  L.Cp = (C + 3) & ~3;
  L.nk = mz + 1;
  L.TP = T + 1;
  L.RS = (TCH + 3) & ~3;                      // point-groups of 4 never straddle a z row
  L.NPS = LZ * L.RS;                          // points per tile (incl. padding)
  L.npad = (L.NPS + 127) & ~127;              // rounded up to whole 128-row MMA tiles
  L.NA = c_num_arrays(mode);
  L.KP = ((C + 7) / 8) * 8;                   // K of the W GEMMs (channels, padded to 8)
  L.C8 = (C + 1 + 7) / 8;                     // channel blocks of the CM layout (+ ones channel)
  L.N1 = ((C + 15) / 16) * 16;                // MMA N for the W GEMMs
  L.N2 = ((C + 1 + 15) / 16) * 16;            // MMA N for dW (incl. the ones column)
  const int mtiles = L.npad / 128;
  int cols = (mode == EPI_U) ? 0 : mtiles * L.N1 + (mode == EPI_BWD ? L.N2 : 0);
  int alloc = 32;
  while (alloc < cols) alloc *= 2;
  L.tcols = alloc;
  const size_t raw = size_t(C) * L.npad * sizeof(float);            // one staging array [c][point]
  const size_t km = size_t(L.npad) * L.KP * sizeof(float);
  const size_t cm = size_t(L.npad) * L.C8 * 8 * sizeof(float);
  const bool bwd = mode == EPI_BWD, tc = mode != EPI_U;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 127) & ~size_t(127); return o; };
  L.ws = take(size_t(C) * L.Cp * sizeof(float));
  L.bias = take(size_t(C) * sizeof(float));
  L.wb = take(tc ? 2 * size_t(L.N1) * L.KP * sizeof(float) : 0);   // B hi, lo (K-major)
  L.s = take(size_t(C) * 2 * mz * mt * sizeof(float2));
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.u = take(tc ? size_t(C) * L.npad * sizeof(float) : 0);
  L.r0 = take(size_t(L.NA) * raw);
  L.r1 = take(size_t(L.NA) * raw);
  L.kmh = take(tc ? km : 0);
  L.kml = take(tc ? km : 0);
  L.cmdh = take(bwd ? cm : 0);
  L.cmdl = take(bwd ? cm : 0);
  L.cmvh = take(bwd ? cm : 0);
  L.cmvl = take(bwd ? cm : 0);
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  L.dwacc = take(bwd ? size_t(C) * L.N2 * sizeof(float) : 0);
  L.bar = take(sizeof(uint64_t));
  L.tmem = take(sizeof(uint32_t));
  L.total = off + 2048;                          // guard: dW descriptors read up to 16 channel blocks
  return L;
}

template <int LZ, int LT, int EPI>
__global__ void __launch_bounds__(CT, 1) pass_c_kernel(PassCParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt, TCH = p.TCH;
  const CLayout L = c_layout(C, Z, T, mz, mt, LZ, TCH, EPI);
  float* Ws = reinterpret_cast<float*>(smem_raw + L.ws);
  float* bs = reinterpret_cast<float*>(smem_raw + L.bias);
  float* WB = reinterpret_cast<float*>(smem_raw + L.wb);
  float2* S = reinterpret_cast<float2*>(smem_raw + L.s);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float* U = reinterpret_cast<float*>(smem_raw + L.u);
  float* KMH = reinterpret_cast<float*>(smem_raw + L.kmh);
  float* KML = reinterpret_cast<float*>(smem_raw + L.kml);
  float* CMDH = reinterpret_cast<float*>(smem_raw + L.cmdh);
  float* CMDL = reinterpret_cast<float*>(smem_raw + L.cmdl);
  float* CMVH = reinterpret_cast<float*>(smem_raw + L.cmvh);
  float* CMVL = reinterpret_cast<float*>(smem_raw + L.cmvl);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  float* DWA = reinterpret_cast<float*>(smem_raw + L.dwacc);   // [C][N2] fp32 dW/db accumulator
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + L.tmem);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nk = L.nk, TP = L.TP, RS = L.RS, NPS = L.NPS, C8 = L.C8, KP = L.KP, npad = L.npad;
  constexpr int NA = (EPI == EPI_U) ? 0 : (EPI == EPI_FWD ? 1 : 3);
  const int raw_floats = C * npad;
  const int NBm = npad / 8;
  const long long ZT = (long long)Z * T;
  const long long chan_stride = (long long)p.Xl * p.Yl * ZT;
  const int nch = (T + TCH - 1) / TCH;
  const int tpc = p.Qz * nch;  // tiles per column
  const int MT = npad / 128;

  long long col = blockIdx.x;
  if (col >= p.n_cols) return;

  fill_combine_table(twZ, LZ, p.Qz, Z, 0, +1, tid, nt);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, +1, tid, nt);
  for (int j = tid; j < 2 * mz; j += nt) {
    int d = 0;
    while (j >= p.slab.kz_lo[d + 1]) ++d;
    dmap[j] = make_short2(short(d), short(j - p.slab.kz_lo[d]));
  }
  uint32_t tmem = 0;
  if (EPI != EPI_U) {
    for (int o = tid; o < C; o += nt) bs[o] = (EPI == EPI_FWD && p.bias) ? p.bias[o] : 0.f;
    if (EPI == EPI_BWD)
      for (int e = tid; e < C * L.N2; e += nt) DWA[e] = 0.f;
    // B operand of the W GEMM, K-major interleaved: element (n, k) at
    // ((k/4)*(N1/8) + n/8)*32 + (n%8)*4 + (k%4); fwd B[n=o][k=i] = W[o][i],
    // bwd B[n=i][k=o] = W[o][i]; hi and lo parts for 3xTF32
    const int nb8 = L.N1 / 8;
    const int bfl = L.N1 * KP;
    for (int e = tid; e < bfl; e += nt) {
      const int kc = e / (nb8 * 32), r = e - kc * nb8 * 32;
      const int nb = r / 32, r2 = r - nb * 32;
      const int n = nb * 8 + r2 / 4, k = kc * 4 + (r2 & 3);
      float w = 0.f;
      if (n < C && k < C) w = (EPI == EPI_FWD) ? p.W[n * C + k] : p.W[k * C + n];
      const float hi = tf32_hi(w);
      WB[e] = hi;
      WB[bfl + e] = w - hi;
    }
    // zero the operand buffers once: padded channels stay zero
    float* z0 = reinterpret_cast<float*>(smem_raw + L.kmh);
    const size_t nz = (L.twz - L.kmh) / sizeof(float);
    for (size_t e = tid; e < nz; e += nt) z0[e] = 0.f;
    if (warp == 0) tmem_alloc(tmem_slot, L.tcols);
    if (tid == 0) {
      mbar_init(mbar, 1);
      mbar_fence_init();
    }
    fence_proxy_async();
    tc_fence_before();
  }
  __syncthreads();
  if (EPI != EPI_U) {
    tc_fence_after();
    tmem = *tmem_slot;
  }

  // ---- async loaders ---------------------------------------------------------
  auto col_base = [&](long long c_) {
    const int yl = int(c_ % p.Yl);
    const long long r1 = c_ / p.Yl;
    const int xl = int(r1 % p.Xl);
    const int b = int(r1 / p.Xl);
    return (long long)b * C * chan_stride + ((long long)xl * p.Yl + yl) * ZT;
  };
  auto issue_slab = [&](long long c_) {
    const long long colpt = c_;  // ((b*Xl + xl)*Yl + yl) == column index
    const int per_c = 2 * mz * mt;
    for (int e = tid; e < C * per_c; e += nt) {
      const int c = e / per_c, rem = e - c * per_c;
      const int jz = rem / mt, kt = rem - jz * mt;
      const short2 dm = dmap[jz];
      const int nkz = p.slab.kz_lo[dm.x + 1] - p.slab.kz_lo[dm.x];
      cp_async8(S + e, p.in + p.slab.off[dm.x] + ((colpt * C + c) * nkz + dm.y) * mt + kt);
    }
  };
  auto issue_tile = [&](long long cb, int ti, int which) {
    if (NA == 0) return;
    float* dst = reinterpret_cast<float*>(smem_raw + (which ? L.r1 : L.r0));
    const int rz = ti / nch, tc = ti - rz * nch;
    const int t0 = tc * TCH;
    const int tcw = min(TCH, T - t0);
    const long long base = cb + rz * T + t0;
    const int VW = p.VW;
    const int nvec = tcw / VW;                 // vectors per row (tcw % VW == 0 by construction)
    const int rows = C * LZ;
    // thread -> (vector vv, first row); rows advance by nt / nvec
    const int vv = tid % nvec, r0 = tid / nvec, rstep = nt / nvec;
    if (r0 >= rstep) return;
    for (int row = r0; row < rows; row += rstep) {
      const int c = row / LZ, s = row - c * LZ;
      const long long g = base + c * chan_stride + (long long)p.Qz * s * T + vv * VW;
      const int so = c * npad + s * RS + vv * VW;
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        const float* src = (EPI == EPI_FWD) ? p.v : (a == 0 ? p.dy : (a == 1 ? p.zs : p.v));
        float* d = dst + a * raw_floats + so;
        if (VW == 4) cp_async16(d, src + g);
        else if (VW == 2) cp_async8(d, src + g);
        else cp_async4(d, src + g);
      }
    }
  };

  issue_slab(col);
  cp_commit();
  issue_tile(col_base(col), 0, 0);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  int buf = 0;
  unsigned mphase = 0;

  for (; col < p.n_cols; col += gridDim.x) {
    const long long cbase = col_base(col);
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
        trunc_inv<LT>(y, e, rt, twT);
#pragma unroll
        for (int s = 0; s < LT; ++s) bo[rt + p.Qt * s] = y[s];
      }
    }
    __syncthreads();
    const long long col_next = col + gridDim.x;
    const long long cbase_next = col_next < p.n_cols ? col_base(col_next) : 0;
    if (col_next < p.n_cols) issue_slab(col_next);  // S is free now
    cp_commit();

    for (int ti = 0; ti < tpc; ++ti) {
      const int rz = ti / nch, tc = ti - rz * nch;
      const int t0 = tc * TCH;
      const int tcw = min(TCH, T - t0);
      if (ti + 1 < tpc) issue_tile(cbase, ti + 1, buf ^ 1);
      else if (col_next < p.n_cols) issue_tile(cbase_next, 0, buf ^ 1);
      cp_commit();
      const long long tbase = cbase + rz * T + t0;   // + o*chan_stride + Qz*s*T + tt
      // ---- phase 2: inverse z (real output) for this tile, pencils (c, tt) --
      for (int pid = tid; pid < C * tcw; pid += nt) {
        const int c = pid / tcw, tt = pid - c * tcw;
        const int t = t0 + tt;
        float2 e[LZ];
#pragma unroll
        for (int i = 0; i < LZ; ++i) e[i] = (i < nk) ? Bb[(c * nk + i) * TP + t] : make_float2(0.f, 0.f);
        float2 y[LZ];
        trunc_inv<LZ>(y, e, rz, twZ);
        if (EPI == EPI_U) {
          float* o = p.out + tbase + c * chan_stride + tt;
#pragma unroll
          for (int s = 0; s < LZ; ++s) __stcs(o + (long long)p.Qz * s * T, y[s].x * p.inv_n);
        } else {
          float* uo = U + c * npad + tt;
#pragma unroll
          for (int s = 0; s < LZ; ++s) uo[s * RS] = y[s].x * p.inv_n;
        }
      }
      cp_wait<1>();      // this tile's inputs (and the next column's spectrum) have landed
      __syncthreads();
      if (EPI != EPI_U) {
        const float* R0 = reinterpret_cast<const float*>(smem_raw + (buf ? L.r1 : L.r0));
        // ---- tf32 hi/lo split + layout change (bwd: form dz, zero invalid points,
        //      ones channel); a thread handles 4 points x 4 channels
        const int nc4 = (EPI == EPI_BWD) ? (C + 1 + 3) / 4 : (C + 3) / 4;
        for (int it = tid; it < (npad / 4) * nc4; it += nt) {
          const int g = it / nc4, cc = it - g * nc4;
          const int m0 = 4 * g;
          bool ok[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int m = m0 + j;
            const int s = m / RS, tt = m - s * RS;
            ok[j] = (m < NPS) && (tt < tcw);
          }
          float a[4][4], vb[4][4];   // [channel j][point i]
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = 4 * cc + j;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f), zz = x, v4 = x;
            if (c < C) {
              x = *reinterpret_cast<const float4*>(R0 + c * npad + m0);
              if (EPI == EPI_BWD) {
                zz = *reinterpret_cast<const float4*>(R0 + raw_floats + c * npad + m0);
                v4 = *reinterpret_cast<const float4*>(R0 + 2 * raw_floats + c * npad + m0);
              }
            }
            const float xs[4] = {x.x, x.y, x.z, x.w}, zs4[4] = {zz.x, zz.y, zz.z, zz.w},
                        vs[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (EPI == EPI_FWD) {
                a[j][i] = xs[i];
              } else {
                a[j][i] = (c < C && ok[i]) ? (p.act_gelu ? xs[i] * gelu_prime_f(zs4[i]) : xs[i]) : 0.f;
                vb[j][i] = (c < C) ? (ok[i] ? vs[i] : 0.f) : ((c == C && ok[i]) ? 1.f : 0.f);
              }
            }
          }
          // KM (rows = points): the W-GEMM A operand (input v fwd, dz bwd)
          if (4 * cc < KP) {
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
          if (EPI == EPI_BWD) {  // CM (rows = channels): dW GEMM operands dz (A) and v (B)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int c = 4 * cc + j;
              if (c >= 8 * C8) continue;
              const int off = (g * C8 + (c >> 3)) * 32 + (c & 7) * 4;
              float dh[4], dl[4], vh[4], vl[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                dh[i] = tf32_hi(a[j][i]);
                dl[i] = a[j][i] - dh[i];
                vh[i] = tf32_hi(vb[j][i]);
                vl[i] = vb[j][i] - vh[i];
              }
              *reinterpret_cast<float4*>(CMDH + off) = make_float4(dh[0], dh[1], dh[2], dh[3]);
              *reinterpret_cast<float4*>(CMDL + off) = make_float4(dl[0], dl[1], dl[2], dl[3]);
              *reinterpret_cast<float4*>(CMVH + off) = make_float4(vh[0], vh[1], vh[2], vh[3]);
              *reinterpret_cast<float4*>(CMVL + off) = make_float4(vl[0], vl[1], vl[2], vl[3]);
            }
          }
        }
        fence_proxy_async();   // generic smem writes -> visible to the tensor core (async proxy)
        __syncthreads();
        // ---- tcgen05.mma, issued by one thread ------------------------------
        if (warp == 0) {
          tc_fence_after();
          const bool leader = elect_one();
          const uint32_t idesc1 = umma_idesc_tf32(128, L.N1, 0, 0);
          const uint32_t lboA = NBm * 128;            // K-major A: 4-channel chunk stride
          const uint32_t lboB = (L.N1 / 8) * 128;     // K-major B: 4-channel chunk stride
          for (int m4 = 0; m4 < MT; ++m4) {
            const uint32_t d = tmem + m4 * L.N1;
            for (int ks = 0; ks < KP / 8; ++ks) {
              const int ao = m4 * 16 * 32 + ks * 2 * NBm * 32;            // floats
              const uint64_t ah = umma_sdesc(KMH + ao, lboA, 128);
              const uint64_t al = umma_sdesc(KML + ao, lboA, 128);
              const uint64_t bh = umma_sdesc(WB + ks * 2 * (lboB / 4), lboB, 128);
              const uint64_t bl = umma_sdesc(WB + L.N1 * KP + ks * 2 * (lboB / 4), lboB, 128);
              if (leader) {
                umma_tf32(d, ah, bh, idesc1, ks > 0 ? 1u : 0u);
                umma_tf32(d, ah, bl, idesc1, 1u);
                umma_tf32(d, al, bh, idesc1, 1u);
              }
            }
          }
          if (EPI == EPI_BWD) {
            const uint32_t idesc2 = umma_idesc_tf32(128, L.N2, 0, 0);
            const uint32_t d2 = tmem + MT * L.N1;
            for (int ks = 0; ks < npad / 8; ++ks) {
              const int ko = ks * 2 * C8 * 32;                              // 8 points = 2 groups
              const uint64_t ah = umma_sdesc(CMDH + ko, C8 * 128, 128);
              const uint64_t al = umma_sdesc(CMDL + ko, C8 * 128, 128);
              const uint64_t bh = umma_sdesc(CMVH + ko, C8 * 128, 128);
              const uint64_t bl = umma_sdesc(CMVL + ko, C8 * 128, 128);
              if (leader) {
                umma_tf32(d2, ah, bh, idesc2, ks > 0 ? 1u : 0u);   // fresh per tile
                umma_tf32(d2, ah, bl, idesc2, 1u);
                umma_tf32(d2, al, bh, idesc2, 1u);
              }
            }
          }
          __syncwarp();
          if (leader) umma_commit(mbar);
        }
        mbar_wait(mbar, mphase);
        mphase ^= 1u;
        tc_fence_after();
        // ---- epilogue: TMEM -> registers, + S-part (U) + bias, GELU, stores ---
        {
          const int q = warp & 3, h = warp >> 2;   // TMEM lane quadrant, column half
          const int hw = L.N1 / 2;
          for (int m4 = 0; m4 < MT; ++m4) {
            const int m = m4 * 128 + 32 * q + lane;
            const int s = m / RS, tt = m - s * RS;
            const bool okp = (m < NPS) && (tt < tcw);
            const long long gs = tbase + (long long)p.Qz * s * T + tt;
            for (int c0 = 0; c0 < hw; c0 += 8) {
              float d8[8];
              tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + m4 * L.N1 + h * hw + c0, d8);
              if (!okp) continue;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int o = h * hw + c0 + j;
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
        }
        if (EPI == EPI_BWD && warp < 4) {
          // this tile's dW/db partial (TMEM rows o, columns i) -> fp32 smem accumulator;
          // keeps the tensor-core accumulation depth to one tile
          const int o = 32 * warp + lane;
          for (int c0 = 0; c0 < L.N2; c0 += 8) {
            float d8[8];
            tmem_ld8(tmem + ((uint32_t)(32 * warp) << 16) + MT * L.N1 + c0, d8);
            if (o < C) {
#pragma unroll
              for (int j = 0; j < 8; ++j) DWA[o * L.N2 + c0 + j] += d8[j];
            }
          }
        }
        tc_fence_before();
      }
      __syncthreads();
      buf ^= 1;
    }
  }
  cp_wait<0>();
  if (EPI == EPI_BWD) {
    // dW, db of this CTA (column i = C of the accumulator is db)
    __syncthreads();
    float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
    for (int e = tid; e < C * C + C; e += nt) {
      if (e < C * C) {
        const int o = e / C, i = e - o * C;
        outp[e] = DWA[o * L.N2 + i];
      } else {
        outp[e] = DWA[(e - C * C) * L.N2 + C];
      }
    }
    tc_fence_before();
  }
  if (EPI != EPI_U) {
    __syncthreads();
    if (warp == 0) {
      tc_fence_after();
      tmem_dealloc(tmem, L.tcols);
    }
  }
}

// smem bytes for a given chunk width
static size_t c_smem_for(int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode) {
  return c_layout(C, Z, T, mz, mt, LZ, TCH, mode).total;
}

void pass_c_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* TCH, int* VW, size_t* smem) {
  const size_t budget = 227 * 1024;
  // candidate chunks: T, then divisors of T that are multiples of 4, then any
  // multiple of 4 (descending) -- the first that fits
  int tch = T;
  size_t s = c_smem_for(C, Z, T, mz, mt, LZ, tch, mode);
  for (int pass = 0; pass < 2 && s > budget; ++pass) {
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
