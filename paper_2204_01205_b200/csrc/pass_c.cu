// Pass C (bwd a9, a12): the adjoint chain of I_1 =
// {z, t} (zero-padded inverse z, C2R along t with real-part semantics,
// P:119-123 "F_dist^T"), fused with the DFNO block epilogue
//   z = W v + b + u ; y = GELU(z)                      (Eq. dist_block)
// or, backward, dv = W^T dz + S^T dz plus the dW, db partial sums
// (broadcast adjoint = sum-reduce).
//
// One persistent CTA loops over (b, x, y) columns (all channels at once: the
// 1x1 channel linear needs every channel at a point).  The z outputs are
// produced by residue class r (z = r + Qz*s, s < LZ) and t-chunk, so a tile is
// C x LZ x TCH values.  Streaming is software-pipelined with cp.async: the next
// tile's inputs (v; or dy, z, v) and the next column's spectrum are in flight
// while the current tile is transformed and consumed.
#include "kernels.cuh"
#include "launch.h"

namespace fno {

static constexpr int CT = 512;  // threads per CTA (16 warps)

struct CLayout {
  int Cp, nk, TP, RS, NPS, NA;
  size_t ws, bias, s, bb, u, v0, v1, twz, twt, dmap, dws, total;
};

__host__ __device__ inline int c_num_arrays(int mode) { return mode == EPI_U ? 0 : (mode == EPI_FWD ? 1 : 2); }

// tile rows have stride RS (even, and a multiple of 4 when TCH is) so point
// pairs and 16-byte async copies stay aligned
__host__ __device__ inline CLayout c_layout(int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode) {
  CLayout L{};
  L.Cp = (C + 3) & ~3;
  L.nk = mz + 1;
  L.TP = T + 1;
  L.RS = TCH + (TCH & 1);
  L.NPS = LZ * L.RS;
  L.NA = c_num_arrays(mode);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
  L.ws = take(size_t(C) * L.Cp * sizeof(float));
  L.bias = take(size_t(C) * sizeof(float));
  L.s = take(size_t(C) * 2 * mz * mt * sizeof(float2));
  L.bb = take(size_t(C) * L.nk * L.TP * sizeof(float2));
  L.u = take(mode == EPI_U ? 0 : size_t(C) * L.NPS * sizeof(float));
  L.v0 = take(size_t(L.NA) * C * L.NPS * sizeof(float));
  L.v1 = take(size_t(L.NA) * C * L.NPS * sizeof(float));
  L.twz = take(size_t(Z) * sizeof(float2));
  L.twt = take(size_t(T) * sizeof(float2));
  L.dmap = take(size_t(2 * mz) * sizeof(short2));
  const int G = (C + 3) / 4, G8 = (C + 7) / 8;
  L.dws = take(mode == EPI_BWD ? size_t(G) * G8 * 36 * sizeof(float) : 0);   // per-CTA dW/db, 4x8 blocks
  L.total = off;
  return L;
}

template <int LZ, int LT, int EPI>
__global__ void __launch_bounds__(CT, 1) pass_c_kernel(PassCParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int C = p.C, Z = p.Z, T = p.T, mz = p.mz, mt = p.mt, TCH = p.TCH;
  const CLayout L = c_layout(C, Z, T, mz, mt, LZ, TCH, EPI);
  float* Ws = reinterpret_cast<float*>(smem_raw + L.ws);
  float* bs = reinterpret_cast<float*>(smem_raw + L.bias);
  float2* S = reinterpret_cast<float2*>(smem_raw + L.s);
  float2* Bb = reinterpret_cast<float2*>(smem_raw + L.bb);
  float* U = reinterpret_cast<float*>(smem_raw + L.u);
  float2* twZ = reinterpret_cast<float2*>(smem_raw + L.twz);
  float2* twT = reinterpret_cast<float2*>(smem_raw + L.twt);
  short2* dmap = reinterpret_cast<short2*>(smem_raw + L.dmap);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nk = L.nk, TP = L.TP, Cp = L.Cp, NPS = L.NPS, RS = L.RS;
  constexpr int NA = (EPI == EPI_U) ? 0 : (EPI == EPI_FWD ? 1 : 2);
  const long long ZT = (long long)Z * T;
  const long long chan_stride = (long long)p.Xl * p.Yl * ZT;
  const int G = (C + 3) / 4;
  const int nch = (T + TCH - 1) / TCH;
  const int tpc = p.Qz * nch;  // tiles per column
  const int HP = RS / 2;       // point pairs per tile row
  const int tx = tid % HP, ty = tid / HP, TY = nt / HP;

  long long col = blockIdx.x;
  if (col >= p.n_cols) return;

  fill_combine_table(twZ, LZ, p.Qz, Z, 0, +1, tid, nt);
  fill_combine_table(twT, LT, p.Qt, T, mt - 1, +1, tid, nt);
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
      if (o < C) w = (EPI == EPI_FWD && !p.w_t) ? p.W[o * C + k] : p.W[k * C + o];
      Ws[e] = w;
    }
    for (int o = tid; o < C; o += nt) bs[o] = (EPI == EPI_FWD && p.bias) ? p.bias[o] : 0.f;
  }
  __syncthreads();  // dmap ready for the slab loader

  // ---- async loaders ---------------------------------------------------------
  auto col_base = [&](long long c_, int* b_out) {
    const unsigned cu = unsigned(c_);          // n_cols < 2^31 (checked by the plan)
    const unsigned yl = cu % unsigned(p.Yl);
    const unsigned r1 = cu / unsigned(p.Yl);
    const unsigned xl = r1 % unsigned(p.Xl);
    const int b = int(r1 / unsigned(p.Xl));
    *b_out = b;
    return (long long)b * C * chan_stride + ((long long)xl * p.Yl + yl) * ZT;
  };
  auto issue_slab = [&](long long c_) {
    const long long colpt = c_;  // ((b*Xl + xl)*Yl + yl) == column index
    const int per_c = 2 * mz * mt;
    if (p.slab.P == 1 && (per_c & 1) == 0) {   // one owner: a contiguous run of C*2mz*mt complex
      const float2* src = p.in + colpt * C * per_c;
      for (int e = tid; e < C * per_c / 2; e += nt) cp_async16(S + 2 * e, src + 2 * e);
      return;
    }
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
    float* dst = reinterpret_cast<float*>(smem_raw + (which ? L.v1 : L.v0));
    const int rz = ti / nch, tc = ti - rz * nch;
    const int t0 = tc * TCH;
    const int tcw = min(TCH, T - t0);
    const long long base = cb + rz * T + t0;
    const int VW = p.VW;
    const int nvec = tcw / VW;                 // vectors per row (tcw % VW == 0 by construction)
    const int rows = C * LZ;
    const int vv = tid % nvec, rstep = nt / nvec;
    for (int row = tid / nvec; row < rows; row += rstep) {
      const int c = row / LZ, s = row - c * LZ;
      const long long g = base + c * chan_stride + (long long)p.Qz * s * T + vv * VW;
      const int so = c * NPS + s * RS + vv * VW;
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        const float* src = (EPI == EPI_FWD) ? p.v : (a == 0 ? p.dy : p.v);   // bwd: dz (pass A), v
        float* d = dst + a * C * NPS + so;
        if (VW == 4) cp_async16(d, src + g);
        else if (VW == 2) cp_async8(d, src + g);
        else cp_async4(d, src + g);
      }
    }
  };

  // dW / db (EPI_BWD): 4 (o) x 8 (i) blocks; a warp owns a block, its lanes
  // stride over each tile's point pairs (conflict-free row reads) and reduce
  // their partial sums per tile, in a fixed order, into a per-CTA fp32
  // accumulator in shared memory.  (Keeping the partials in registers across
  // tiles measured slower: 36 more live registers under the 128-register cap.)
  const int G8 = (C + 7) / 8;
  const int NB = G * G8;
  float* DWS = reinterpret_cast<float*>(smem_raw + L.dws);   // [NB][32 dW + 4 db]
  const int warp = tid >> 5, lane = tid & 31, nwarps = nt >> 5;
  if (EPI == EPI_BWD) {
    for (int e = tid; e < NB * 36; e += nt) DWS[e] = 0.f;
  }

  issue_slab(col);
  cp_commit();
  {
    int b0;
    issue_tile(col_base(col, &b0), 0, 0);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  int buf = 0;

  for (; col < p.n_cols; col += gridDim.x) {
    int b;
    const long long cbase = col_base(col, &b);
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
    int bnext = 0;
    const long long cbase_next = col_next < p.n_cols ? col_base(col_next, &bnext) : 0;
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
          float* uo = U + c * NPS + tt;
#pragma unroll
          for (int s = 0; s < LZ; ++s) uo[s * RS] = y[s].x * p.inv_n;
        }
      }
      cp_wait<1>();      // this tile's inputs (and the next column's spectrum) have landed
      __syncthreads();
      if (EPI != EPI_U) {
        float* V = reinterpret_cast<float*>(smem_raw + (buf ? L.v1 : L.v0));
        const bool ok0 = 2 * tx < tcw, ok1 = 2 * tx + 1 < tcw;
        if (EPI == EPI_BWD) {
          // zero the invalid slots (ragged t chunk) so dW sees exact zeros
          if (tcw < RS) {
            for (int r = ty; ty < TY && r < C * LZ; r += TY) {
              float* dzr = V + r * RS + 2 * tx;
              float* vr = V + C * NPS + r * RS + 2 * tx;
              if (!ok0) { dzr[0] = 0.f; vr[0] = 0.f; }
              if (!ok1) { dzr[1] = 0.f; vr[1] = 0.f; }
            }
            __syncthreads();
          }
        }
        // ---- phase 3: 1x1 channel linear + epilogue; rows (o-group, s) x pairs
        if (ty < TY) {
          for (int r = ty; r < G * LZ; r += TY) {
            const int g = r / LZ, s = r - g * LZ;
            const int p0 = s * RS + 2 * tx;
            float acc[4][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
            const float* vp = V + p0;
            const float* wp = Ws + 4 * g;
            for (int k = 0; k < C; ++k) {
              const float2 v2 = *reinterpret_cast<const float2*>(vp + k * NPS);
              const float4 w4 = *reinterpret_cast<const float4*>(wp + k * Cp);
              acc[0][0] = fmaf(w4.x, v2.x, acc[0][0]); acc[0][1] = fmaf(w4.x, v2.y, acc[0][1]);
              acc[1][0] = fmaf(w4.y, v2.x, acc[1][0]); acc[1][1] = fmaf(w4.y, v2.y, acc[1][1]);
              acc[2][0] = fmaf(w4.z, v2.x, acc[2][0]); acc[2][1] = fmaf(w4.z, v2.y, acc[2][1]);
              acc[3][0] = fmaf(w4.w, v2.x, acc[3][0]); acc[3][1] = fmaf(w4.w, v2.y, acc[3][1]);
            }
            const long long gs = tbase + (long long)p.Qz * s * T + 2 * tx;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const int o = 4 * g + a;
              if (o >= C) break;
              const float2 u2 = *reinterpret_cast<const float2*>(U + o * NPS + p0);
              float* out = p.out + gs + o * chan_stride;
              float v0 = acc[a][0] + u2.x, v1 = acc[a][1] + u2.y;
              if (EPI == EPI_FWD) {
                v0 += bs[o];
                v1 += bs[o];
                if (p.zsave) {
                  float* zo = p.zsave + gs + o * chan_stride;
                  if (ok0) __stcs(zo, v0);
                  if (ok1) __stcs(zo + 1, v1);
                }
                if (p.act_gelu) {
                  v0 = gelu_f(v0);
                  v1 = gelu_f(v1);
                }
              }
              if (ok0) __stcs(out, v0);
              if (ok1) __stcs(out + 1, v1);
            }
          }
        }
        if (EPI == EPI_BWD) {
          const float* Dz = V;
          const float* Vv = V + C * NPS;
          for (int bk = warp; bk < NB; bk += nwarps) {
            const int og = bk / G8, ig = bk - og * G8;
            float acc[4][8], dsum[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              dsum[a] = 0.f;
#pragma unroll
              for (int c2 = 0; c2 < 8; ++c2) acc[a][c2] = 0.f;
            }
            for (int q = lane; q < NPS / 2; q += 32) {
              const int p0 = 2 * q;
              float2 dz2[4], v2[8];
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                const int o = 4 * og + a;
                dz2[a] = (o < C) ? *reinterpret_cast<const float2*>(Dz + o * NPS + p0) : make_float2(0.f, 0.f);
              }
#pragma unroll
              for (int c2 = 0; c2 < 8; ++c2) {
                const int i = 8 * ig + c2;
                v2[c2] = (i < C) ? *reinterpret_cast<const float2*>(Vv + i * NPS + p0) : make_float2(0.f, 0.f);
              }
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                dsum[a] += dz2[a].x + dz2[a].y;
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2) {
                  acc[a][c2] = fmaf(dz2[a].x, v2[c2].x, acc[a][c2]);
                  acc[a][c2] = fmaf(dz2[a].y, v2[c2].y, acc[a][c2]);
                }
              }
            }
            // fixed-order transpose-reduction of the 32 dW partials over the 32
            // lanes (31 shuffles instead of 160): at each level a lane keeps the
            // half of its values selected by its lane bit and adds the partner's
            // copy of that half; lane l ends with the total of value l = (a, c2)
            {
              float* v = &acc[0][0];
#pragma unroll
              for (int n = 16; n > 0; n >>= 1) {
                const bool up = (lane & n) != 0;
#pragma unroll
                for (int j = 0; j < n; ++j) {
                  const float send = up ? v[j] : v[j + n];
                  const float keep = up ? v[j + n] : v[j];
                  v[j] = keep + __shfl_xor_sync(0xffffffffu, send, n);
                }
              }
              float* dst = DWS + bk * 36;
              dst[lane] += v[0];
              if (ig == 0) {
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                  for (int off = 16; off > 0; off >>= 1) dsum[a] += __shfl_xor_sync(0xffffffffu, dsum[a], off);
                if (lane == 0) {
#pragma unroll
                  for (int a = 0; a < 4; ++a) dst[32 + a] += dsum[a];
                }
              }
            }
          }
        }
      }
      __syncthreads();
      buf ^= 1;
    }
  }
  cp_wait<0>();
  if (EPI == EPI_BWD) {
    __syncthreads();
    float* outp = p.dWpart + (long long)blockIdx.x * (C * C + C);
    for (int e = tid; e < C * C + C; e += nt) {
      int o, i, slot;
      if (e < C * C) { o = e / C; i = e - o * C; slot = (o % 4) * 8 + (i % 8); }
      else { o = e - C * C; i = 0; slot = 32 + (o % 4); }
      outp[e] = DWS[((o / 4) * G8 + (i / 8)) * 36 + slot];
    }
  }
}

// smem bytes for a given chunk width
static size_t c_smem_for(int C, int Z, int T, int mz, int mt, int LZ, int TCH, int mode) {
  return c_layout(C, Z, T, mz, mt, LZ, TCH, mode).total;
}

void pass_c_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* TCH, int* VW, size_t* smem) {
  const size_t budget = 227 * 1024;
  // candidate chunks: T, then multiples of 4 (descending), then 2, 1
  int tch = T;
  size_t s = c_smem_for(C, Z, T, mz, mt, LZ, tch, mode);
  for (int cand = (T - 1) & ~3; s > budget && cand >= 4; cand -= 4) {
    tch = cand;
    s = c_smem_for(C, Z, T, mz, mt, LZ, tch, mode);
  }
  for (int cand : {2, 1}) {
    if (s <= budget) break;
    tch = cand;
    s = c_smem_for(C, Z, T, mz, mt, LZ, tch, mode);
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
