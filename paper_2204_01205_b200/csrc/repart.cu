// Strided n-D box copy used by fno_repartition's pack / unpack (the
// repartition moves the intersection of a source box with a destination box).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

struct BoxCopy {
  const char* src;
  char* dst;
  long long src_ext[8], src_lo[8], dst_ext[8], dst_lo[8], cnt[8];
  long long total;
  int ndim;
  int elem_bytes;
};

template <typename W>
__global__ void box_copy_kernel(BoxCopy p) {
  const int words = p.elem_bytes / int(sizeof(W));
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < p.total; e += (long long)gridDim.x * blockDim.x) {
    long long r = e, so = 0, dof = 0, ss = 1, ds = 1;
    for (int d = p.ndim - 1; d >= 0; --d) {
      const long long i = r % p.cnt[d];
      r /= p.cnt[d];
      so += (p.src_lo[d] + i) * ss;
      dof += (p.dst_lo[d] + i) * ds;
      ss *= p.src_ext[d];
      ds *= p.dst_ext[d];
    }
    const W* s = reinterpret_cast<const W*>(p.src + so * p.elem_bytes);
    W* d = reinterpret_cast<W*>(p.dst + dof * p.elem_bytes);
    for (int w = 0; w < words; ++w) d[w] = s[w];
  }
}

}  // namespace

cudaError_t launch_box_copy(const void* src, const long long* src_ext, const long long* src_lo, void* dst,
                            const long long* dst_ext, const long long* dst_lo, const long long* cnt, int ndim,
                            size_t elem_bytes, cudaStream_t st) {
  BoxCopy p{};
  p.src = static_cast<const char*>(src);
  p.dst = static_cast<char*>(dst);
  p.ndim = ndim;
  p.elem_bytes = int(elem_bytes);
  p.total = 1;
  for (int d = 0; d < ndim; ++d) {
    p.src_ext[d] = src_ext[d];
    p.src_lo[d] = src_lo[d];
    p.dst_ext[d] = dst_ext[d];
    p.dst_lo[d] = dst_lo[d];
    p.cnt[d] = cnt[d];
    p.total *= cnt[d];
  }
  if (p.total == 0) return cudaSuccess;
  const long long blocks = (p.total + 255) / 256;
  const unsigned grid = unsigned(blocks < 148 * 16 ? blocks : 148 * 16);
  const uintptr_t a = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
  if (elem_bytes % 4 == 0 && (a & 3) == 0)
    box_copy_kernel<uint32_t><<<grid, 256, 0, st>>>(p);
  else
    box_copy_kernel<uint8_t><<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}
