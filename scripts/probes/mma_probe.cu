// Throughput probe: legacy warp-level mma.sync (HMMA) on sm_100a, tf32 m16n8k8
// and bf16 m16n8k16, plus FFMA, to size the tensor-core vs FP32-pipe choice of
// the pass-C 1x1 / dW contractions.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int ILP>
__global__ void k_tf32(float* out, int iters) {
  unsigned a[4], b[2];
  float c[ILP][4];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  for (int j = 0; j < ILP; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ILP; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
  for (int j = 0; j < ILP; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
template <int ILP>
__global__ void k_bf16(float* out, int iters) {
  unsigned a[4], b[2];
  float c[ILP][4];
  for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x;
  for (int i = 0; i < 2; ++i) b[i] = 0x3f003f00u;
  for (int j = 0; j < ILP; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ILP; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
  for (int j = 0; j < ILP; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], 0.999f, 0.001f);
  }
  float s = 0.f;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  float* out; cudaMalloc(&out, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    int grid = sms, block = 32 * warps;
    float ms = timeit([&] { k_tf32<8><<<grid, block>>>(out, iters); });
    double fl = 2.0 * 16 * 8 * 8 * 8.0 * iters * grid * warps;
    printf("tf32 m16n8k8  warps/SM=%2d  %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    ms = timeit([&] { k_bf16<8><<<grid, block>>>(out, iters); });
    fl = 2.0 * 16 * 8 * 16 * 8.0 * iters * grid * warps;
    printf("bf16 m16n8k16 warps/SM=%2d  %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    ms = timeit([&] { k_ffma<<<grid, block>>>(out, iters / 4); });
    fl = 2.0 * 16 * 8 * (iters / 4) * double(grid) * block;
    printf("ffma          warps/SM=%2d  %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
