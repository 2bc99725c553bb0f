// Ahead-of-time sm_100a helper kernels (the walk kernels themselves are
// specialised per program at compile time, see lower/ptx.cpp).
//
// max_abs_i64: per-variable max |x| over an int64 SoA coordinate array, the
// input to the host-side overflow proof for the exact int64 path (the
// reference's BigInt never overflows, bigint.hpp:18-81; we refuse instead).
// HBM-bound: 8 B read per coordinate, 16 B vector loads, grid sized to the SM
// count, one atomicMax per warp.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__device__ __forceinline__ unsigned long long uabs64(long long v) {
  // |INT64_MIN| = 2^63 as unsigned, larger than any provable bound.
  return v < 0 ? 0ull - static_cast<unsigned long long>(v)
               : static_cast<unsigned long long>(v);
}

__global__ void __launch_bounds__(256) max_abs_i64_kernel(const long long* __restrict__ x,
                                                          size_t n,
                                                          unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t n2 = n / 2;
  const auto* x2 = reinterpret_cast<const longlong2*>(x);
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  if (aligned) {
    for (size_t i = tid; i < n2; i += stride) {
      const longlong2 v = __ldg(x2 + i);
      m = max(m, max(uabs64(v.x), uabs64(v.y)));
    }
    if (tid == 0 && (n & 1)) m = max(m, uabs64(x[n - 1]));
  } else {
    for (size_t i = tid; i < n; i += stride) m = max(m, uabs64(__ldg(x + i)));
  }
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

}  // namespace

extern "C" cudaError_t pe_launch_max_abs_i64(const long long* x, size_t n,
                                             unsigned long long* out, int sms,
                                             cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const size_t want = (n / 2 + 255) / 256;
  const int grid = static_cast<int>(want < static_cast<size_t>(sms) * 8 ? (want ? want : 1)
                                                                        : static_cast<size_t>(sms) * 8);
  max_abs_i64_kernel<<<grid, 256, 0, stream>>>(x, n, out);
  return cudaGetLastError();
}
