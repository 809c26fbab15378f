// Exchange barrier over NVLink peer memory.  With the peer
// exchange (fno_plan_connect_peers) the data of each repartition already
// travelled inside pass A / the y-inverse as direct stores into the owners'
// buffers; what remains is "every rank has finished storing".  One
// tiny kernel per exchange: thread d publishes this rank's arrival in rank d's
// flag row with a system-scope release store (through the CUDA-IPC mapping of
// d's workspace) and waits, with acquire loads, for rank d's arrival in its own
// row.  The epoch counter lives in device memory and advances inside the
// kernel, so the barrier replays correctly from a CUDA graph.  One such kernel
// per GPU, every GPU its own process: ranks never spin on one device.
#include "kernels.cuh"
#include "launch.h"

namespace fno {

__device__ __forceinline__ void st_release_sys(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}

__global__ void peer_barrier_kernel(PeerBarrierParams p) {
  __shared__ unsigned long long e;
  if (threadIdx.x == 0) {
    e = *p.epoch + 1;
    *p.epoch = e;
  }
  __syncthreads();
  const int d = threadIdx.x;
  if (d >= p.P) return;
  __threadfence_system();
  st_release_sys(p.peer_flags[d] + p.rank, e);   // "rank arrived" in rank d's row
  const unsigned long long* mine = p.my_flags + d;
  if (ld_acquire_sys(mine) >= e) return;
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(mine) < e) {
    __nanosleep(64);
    if (global_ns() - t0 > 4000000000ull) __trap();   // a rank that never arrives: fail, do not hang
  }
}

cudaError_t launch_peer_barrier(const PeerBarrierParams& p, cudaStream_t st) {
  peer_barrier_kernel<<<1, 64, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace fno
