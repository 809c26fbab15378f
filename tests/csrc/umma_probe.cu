// GPU probe of the tcgen05 kind::tf32 operand layouts used by pass C
// (paper_2204_01205_b200/csrc/umma.cuh).  One CTA builds A (128 x 8) and
// B (N x 8) in shared memory in the interleaved core-matrix layouts, issues one
// MMA for several descriptor variants and compares D with a host GEMM.
// Built and run by tests/test_gpu_umma.py.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_2204_01205_b200/csrc/umma.cuh"

using namespace fno;

// variant bits: 1 = swap A lbo/sbo, 2 = swap B lbo/sbo, 4 = A stored K-major.
// Observed on B200: MN-major tf32 A with SWIZZLE_NONE yields D = 0 (variants
// 0-3), K-major A (variant 4, the layout pass C uses) is exact.
__global__ void probe(const float* Ag, const float* Bg, float* Dg, int N, int variant) {
  __shared__ __align__(1024) float As[128 * 8];
  __shared__ __align__(1024) float Bs[256 * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool a_kmajor = variant & 4;
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int m = e / 8, k = e % 8;
    int off;
    if (!a_kmajor) off = (m / 4) * 32 + (k % 8) * 4 + (m % 4);          // MN-major, C8 = 1
    else off = ((k / 4) * 16 + m / 8) * 32 + (m % 8) * 4 + (k % 4);      // K-major
    As[off] = Ag[m * 8 + k];
  }
  for (int e = tid; e < N * 8; e += blockDim.x) {
    const int n = e / 8, k = e % 8;
    const int off = ((k / 4) * (N / 8) + n / 8) * 32 + (n % 8) * 4 + (k % 4);
    Bs[off] = Bg[n * 8 + k];
  }
  if (warp == 0) tmem_alloc(&slot, 32 < N ? (N <= 64 ? 64 : 256) : 32);
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    uint32_t alb, asb, blb = (N / 8) * 128, bsb = 128;
    if (!a_kmajor) { alb = 128; asb = 128; } else { alb = 16 * 128; asb = 128; }
    if (variant & 1) { uint32_t t = alb; alb = asb; asb = t; }
    if (variant & 2) { uint32_t t = blb; blb = bsb; bsb = t; }
    const uint64_t ad = umma_sdesc(As, alb, asb);
    const uint64_t bd = umma_sdesc(Bs, blb, bsb);
    umma_tf32(tmem, ad, bd, umma_idesc_tf32(128, N, a_kmajor ? 0 : 1, 0), 0u);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 8) {
      float d[8];
      tmem_ld8(tmem + ((uint32_t)(32 * warp) << 16) + c0, d);
      for (int j = 0; j < 8; ++j) Dg[(32 * warp + lane) * N + c0 + j] = d[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 32 < N ? (N <= 64 ? 64 : 256) : 32); }
}

int main() {
  const int Ns[2] = {16, 32};
  int fails = 0;
  for (int ni = 0; ni < 2; ++ni) {
    const int N = Ns[ni];
    float *A, *B, *D;
    cudaMallocManaged(&A, 128 * 8 * 4);
    cudaMallocManaged(&B, N * 8 * 4);
    cudaMallocManaged(&D, 128 * N * 4);
    for (int i = 0; i < 128 * 8; ++i) A[i] = float((i * 7 + 3) % 13 - 6);
    for (int i = 0; i < N * 8; ++i) B[i] = float((i * 5 + 1) % 11 - 5);
    for (int variant = 0; variant < 5; ++variant) {
      for (int i = 0; i < 128 * N; ++i) D[i] = NAN;
      probe<<<1, 128>>>(A, B, D, N, variant);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("N=%d variant=%d CUDA error %s\n", N, variant, cudaGetErrorString(e)); return 2; }
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < 8; ++k) ref += double(A[m * 8 + k]) * B[n * 8 + k];
          double err = fabs(ref - D[m * N + n]);
          if (!(err <= maxerr)) maxerr = err;
        }
      printf("N=%d variant=%d (swapA=%d swapB=%d Akmajor=%d) maxerr=%g  D[0][0..3]=%g %g %g %g\n", N, variant,
             variant & 1, (variant >> 1) & 1, (variant >> 2) & 1, maxerr, D[0], D[1], D[2], D[3]);
      if (variant == 4 && maxerr > 0) fails++;
    }
    cudaFree(A); cudaFree(B); cudaFree(D);
  }
  printf(fails ? "FAIL\n" : "PASS\n");
  return fails ? 1 : 0;
}
