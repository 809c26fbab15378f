// Host-side launchers of the libfno kernels and the supported transform sizes.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

// (LZ, LT) register-FFT pairs instantiated for passes A and C.  LZ covers the
// real z-axis transform (needs mz+1 residues), LT the t-axis (needs
// min(2mt-1, T) residues).  Chosen by the plan as the smallest supported
// divisor of Z / T that is large enough; see fno_plan_create.
#define FNO_AC_PAIRS(X) \
  X(2, 4)               \
  X(4, 5)               \
  X(8, 8)               \
  X(8, 16)              \
  X(16, 15)             \
  X(16, 16)             \
  X(16, 30)             \
  X(16, 32)             \
  X(32, 32)

// L values instantiated for the pass-B pencil kernels (x and y transforms,
// need 2m residues).
#define FNO_B_SIZES(X) X(2) X(4) X(5) X(6) X(8) X(16) X(30) X(32)

namespace fno {

// planes per batch NP, dynamic shared memory and TMA eligibility for a pass-A mode
void pass_a_config(int Z, int T, int mz, int mode, int* NP, int* NS, size_t* smem, int* use_tma);
int pass_a_threads(int mode, int T);      // threads per CTA of the mode's pass A kernel
int pass_a_max_blocks(int mode, int T);   // its resident CTAs per SM (launch bounds)
cudaError_t launch_pass_a(const PassAParams& p, int LZ, int LT, int mode, int grid, size_t smem, cudaStream_t st);


// chooses the t-chunk TCH (largest that fits shared memory), the cp.async
// vector width VW and the dynamic shared memory size for a pass-C mode
void pass_c_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* TCH, int* VW, size_t* smem);
cudaError_t launch_pass_c(const PassCParams& p, int LZ, int LT, int mode, int grid, size_t smem, cudaStream_t st);

// channel-width-specialised pass C (pass_c2.cu) for the layer epilogues
// (EPI_FWD / EPI_BWD) when C <= 20: false if the configuration is not covered
bool pass_c2_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* CP, int* TCH, int* VW, size_t* smem,
                    int* NX);
cudaError_t launch_pass_c2(const PassCParams& p, int LZ, int LT, int CP, int mode, int grid, size_t smem,
                           cudaStream_t st);

// tensor-core pass C (pass_c3.cu): layer forward with the 1x1 + bias on
// tcgen05 (3xTF32, TMEM accumulator); false if the configuration is not covered
bool pass_c3_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* CP, int* TCH, size_t* smem);
cudaError_t launch_pass_c3(const PassCParams& p, int LZ, int LT, int CP, int grid, size_t smem, cudaStream_t st);

// pass C generation 4 (pass_c4.cu): warp-specialised, TMA input ring, tcgen05
// 1x1 (fwd), W^T dz and dW / db (bwd); every epilogue mode.  false if the
// configuration is not covered; launch returns cudaErrorNotSupported when the
// tensors' alignment rules out the TMA tile view (the caller falls back)
bool pass_c4_config(int C, int Z, int T, int mz, int mt, int LZ, int mode, int* CP, int* NS, size_t* smem);
cudaError_t launch_pass_c4(const PassCParams& p, int LZ, int LT, int CP, int mode, int grid, size_t smem,
                           cudaStream_t st);

// pass B: y forward (slab -> H), x forward (H -> V^), x inverse (W^ -> H'),
// y inverse (H' -> slab)
cudaError_t launch_b_yfwd(const PassBParams& p, int L, cudaStream_t st);
cudaError_t launch_b_xfwd(const PassBParams& p, int L, cudaStream_t st);
cudaError_t launch_b_xinv(const PassBParams& p, int L, cudaStream_t st);
cudaError_t launch_b_yinv(const PassBParams& p, int L, cudaStream_t st);

cudaError_t launch_mix_fwd(const MixParams& p, cudaStream_t st);
cudaError_t launch_mix_bwd(const MixParams& p, cudaStream_t st);

// dW / db partials of the split backward (dw.cu): per CTA one row
// [C * C + C] of sum_b sum_n dz[b][o][n] v[b][i][n] and sum dz[b][o][n], n over the
// N = Xl Yl Z T points of a channel (NCXYZT fields); C <= 20
struct DwParams {
  const float* dz;
  const float* v;
  float* part;          // [grid][C * C + C]
  long long N;
  int B, C;
  int bulk;             // set by launch_dw_partial: rows 16-byte aligned (2-D TMA tiles), else plain loads
};
size_t dw_partial_smem(int C);
int dw_partial_grid(int B, long long N, int num_sms);
cudaError_t launch_dw_partial(const DwParams& p, int grid, cudaStream_t st);

// deterministic fixed-order sum of nparts rows of `len` floats; columns
// [0, split) go to out0, the rest to out1 (nullable); out = sum or out += sum
cudaError_t launch_rowsum(const float* parts, int nparts, int len, int split, float* out0, float* out1, int accumulate,
                          cudaStream_t st);

// whole-network kernels (network.cu)
struct NetParams {
  int B, C, Cin, T;
  long long NS;                          // local spatial points Xl*Yl*Z
  const float* a;                        // input [B][Cin][NS] (time axis of size 1)
  const float *Wt, *bt, *Wc, *bc;        // lift
  const float *Wp, *bp;                  // projection (bp nullable)
  float* nu;                             // lift out / projection in / adjoint source
  float* u;                              // projection out
  const float* y;                        // target
  float* dnu;                            // adjoint field
  float* parts;                          // per-CTA float partials
  int plen;                              // partial row length
  double* dparts;                        // per-CTA fp64 partials (loss)
  const double* stats;                   // {||u - y||^2, ||y||^2} (global)
};
cudaError_t launch_net_lift_fwd(const NetParams& q, int num_sms, cudaStream_t st);
cudaError_t launch_net_proj_fwd(const NetParams& q, int num_sms, cudaStream_t st);
int net_loss_grid(const NetParams& q, int num_sms);
cudaError_t launch_net_loss_partial(const NetParams& q, int grid, cudaStream_t st);
cudaError_t launch_net_loss_finalize(const double* parts, int nrows, double* sums, float* out, cudaStream_t st);
int net_proj_bwd_grid(const NetParams& q, int num_sms);
cudaError_t launch_net_proj_bwd(const NetParams& q, int grid, cudaStream_t st);
int net_lift_bwd_grid(const NetParams& q, int num_sms);
cudaError_t launch_net_lift_bwd(const NetParams& q, int grid, cudaStream_t st);
cudaError_t launch_rowsum_strided(const float* rows, int nrows, long long stride, int len, float* out, int acc,
                                  cudaStream_t st);
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
                        float eps, int step, int num_sms, cudaStream_t st);

// exchange barrier over NVLink peer memory (peer.cu)
struct PeerBarrierParams {
  unsigned long long* peer_flags[FNO_MAXP];   // rank d's flag row (mapped over NVLink); this rank writes [rank]
  unsigned long long* my_flags;               // this rank's row: [d] = rank d's latest arrival epoch
  unsigned long long* epoch;                  // this rank's barrier count
  int P, rank;
};
cudaError_t launch_peer_barrier(const PeerBarrierParams& p, cudaStream_t st);

bool ac_pair_supported(int LZ, int LT);
bool b_size_supported(int L);

}  // namespace fno
