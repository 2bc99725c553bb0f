// Walk VM kernels (ahead-of-time compiled for sm_100a): evaluate a program
// from its lowered op list (lower/vm.hpp) while its specialised kernel is
// still being compiled, so the first call on a new polynomial needs no
// ptxas run.
//
// One point per thread; the op list is staged through shared memory in
// chunks (every thread executes the same op: operand decoding is warp-
// uniform, no divergence); values live in a per-thread slot file (local
// memory, L1-resident). Arithmetic per domain is the specialised kernel's:
//   F64 / F64Strict  __fma_rn / __dmul_rn / __dadd_rn (never contracted)
//   I64F             the same on exact integers below 2^53 (host-proven)
//   I64              two's-complement int64 (wrap-free by the host proof)
//   Interval         reference interval.cpp:12-52: RN op, then one nextafter
//                    step outward per endpoint; products with the zero rule
//                    and the std::min/std::max({p1..p4}) scan order
// so results are bit-identical to the specialised kernels (which the tests
// check against the oracle and the unmodified reference).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

namespace {

constexpr std::uint32_t kCoef = 0x80000000u, kZero = 0x40000000u;
constexpr int kMaxVars = 16;
constexpr int kThreads = 128;
constexpr std::uint32_t kChunk = 256;  // ops staged per round

struct VmArgs {
  const std::uint32_t* code;
  const std::uint64_t* lo;
  const std::uint64_t* hi;
  const void* in[2 * kMaxVars];  // coordinates (intervals: lo_0, hi_0, lo_1, ...)
  void* out0;
  void* out1;
  unsigned long long n;
  unsigned* flag;
  unsigned long long bounds[kMaxVars];
  std::uint32_t nops, nvars, result;
};

__device__ __forceinline__ double as_f64(std::uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }

struct F64 {
  using T = double;
  static __device__ T zero() { return 0.0; }
  static __device__ T coef(const VmArgs& a, std::uint32_t k) { return as_f64(__ldg(a.lo + k)); }
  static __device__ T add(T x, T y) { return __dadd_rn(x, y); }
  static __device__ T mul(T x, T y) { return __dmul_rn(x, y); }
  static __device__ T fma(T x, T y, T z) { return __fma_rn(x, y, z); }
  static __device__ void load(const VmArgs& a, unsigned long long j, bool, T* r) {
    for (std::uint32_t v = 0; v < a.nvars; ++v) r[v] = __ldg(static_cast<const double*>(a.in[v]) + j);
  }
  static __device__ void store(const VmArgs& a, unsigned long long i, T v) {
    static_cast<double*>(a.out0)[i] = v;
  }
};

// exact integers on the FP64 pipe (|x| <= bound < 2^53, every intermediate
// below 2^53 by the host proof)
struct I64F : F64 {
  static __device__ void load(const VmArgs& a, unsigned long long j, bool valid, T* r) {
    for (std::uint32_t v = 0; v < a.nvars; ++v) {
      const long long x = __ldg(static_cast<const long long*>(a.in[v]) + j);
      const unsigned long long ax = x < 0 ? 0ull - static_cast<unsigned long long>(x) : x;
      if (valid && ax > a.bounds[v]) atomicOr(a.flag, 1u);
      r[v] = static_cast<double>(x);
    }
  }
  static __device__ void store(const VmArgs& a, unsigned long long i, T v) {
    static_cast<long long*>(a.out0)[i] = __double2ll_rn(v);
  }
};

struct I64 {
  using T = long long;
  static __device__ T zero() { return 0; }
  static __device__ T coef(const VmArgs& a, std::uint32_t k) { return static_cast<long long>(__ldg(a.lo + k)); }
  static __device__ T add(T x, T y) {
    return static_cast<long long>(static_cast<unsigned long long>(x) + static_cast<unsigned long long>(y));
  }
  static __device__ T mul(T x, T y) {
    return static_cast<long long>(static_cast<unsigned long long>(x) * static_cast<unsigned long long>(y));
  }
  static __device__ T fma(T x, T y, T z) { return add(mul(x, y), z); }
  static __device__ void load(const VmArgs& a, unsigned long long j, bool valid, T* r) {
    for (std::uint32_t v = 0; v < a.nvars; ++v) {
      const long long x = __ldg(static_cast<const long long*>(a.in[v]) + j);
      const unsigned long long ax = x < 0 ? 0ull - static_cast<unsigned long long>(x) : x;
      if (valid && ax > a.bounds[v]) atomicOr(a.flag, 1u);
      r[v] = x;
    }
  }
  static __device__ void store(const VmArgs& a, unsigned long long i, T v) {
    static_cast<long long*>(a.out0)[i] = v;
  }
};

struct IvVal {
  double lo, hi;
};

struct Interval {
  using T = IvVal;
  static __device__ T zero() { return {0.0, 0.0}; }
  static __device__ T coef(const VmArgs& a, std::uint32_t k) {
    return {as_f64(__ldg(a.lo + k)), as_f64(__ldg(a.hi + k))};
  }
  // std::nextafter(v, +inf) (up) / (v, -inf) (down) on the bit pattern:
  // +-0 -> +-denorm_min, NaN kept, +inf kept up / -inf kept down, otherwise
  // one step of the magnitude in the right direction
  static __device__ double step(double v, bool up) {
    const long long u = __double_as_longlong(v);
    const long long d = (u >> 63) | 1;
    const unsigned long long mag = static_cast<unsigned long long>(u) & 0x7FFFFFFFFFFFFFFFull;
    if (mag > 0x7FF0000000000000ull) return v;  // NaN
    if (mag == 0) return __longlong_as_double(up ? 1ll : static_cast<long long>(0x8000000000000001ull));
    if (up && u == 0x7FF0000000000000ll) return v;
    if (!up && static_cast<unsigned long long>(u) == 0xFFF0000000000000ull) return v;
    return __longlong_as_double(up ? u + d : u - d);
  }
  static __device__ double down(double v) { return step(v, false); }
  static __device__ double up(double v) { return step(v, true); }
  static __device__ T add(T x, T y) {  // interval_add (interval.cpp:36-41)
    return {down(__dadd_rn(x.lo, y.lo)), up(__dadd_rn(x.hi, y.hi))};
  }
  // endpoint product with the zero rule (interval.cpp:15-18)
  static __device__ double prod(double x, double y) {
    return (x == 0.0 || y == 0.0) ? 0.0 : __dmul_rn(x, y);
  }
  static __device__ T mul(T x, T y) {  // interval_mul (interval.cpp:43-52)
    const double p1 = prod(x.lo, y.lo), p2 = prod(x.lo, y.hi), p3 = prod(x.hi, y.lo),
                 p4 = prod(x.hi, y.hi);
    double mn = p1, mx = p1;  // std::min / std::max initializer-list scan order
    if (p2 < mn) mn = p2;
    if (mx < p2) mx = p2;
    if (p3 < mn) mn = p3;
    if (mx < p3) mx = p3;
    if (p4 < mn) mn = p4;
    if (mx < p4) mx = p4;
    return {down(mn), up(mx)};
  }
  static __device__ T fma(T x, T y, T z) { return add(mul(x, y), z); }  // (strict streams have none)
  static __device__ void load(const VmArgs& a, unsigned long long j, bool valid, T* r) {
    for (std::uint32_t v = 0; v < a.nvars; ++v) {
      const double lo = __ldg(static_cast<const double*>(a.in[2 * v]) + j);
      const double hi = __ldg(static_cast<const double*>(a.in[2 * v + 1]) + j);
      // reference Interval(lo, hi) rejects NaN endpoints and lo > hi
      // (interval.cpp:21-26): flag, the host reports EINVAL
      if (valid && !(lo <= hi)) atomicOr(a.flag, 2u);
      r[v] = {lo, hi};
    }
  }
  static __device__ void store(const VmArgs& a, unsigned long long i, T v) {
    static_cast<double*>(a.out0)[i] = v.lo;
    static_cast<double*>(a.out1)[i] = v.hi;
  }
};

template <class D, int MAXS>
__global__ void __launch_bounds__(kThreads) vm_kernel(const VmArgs a) {
  using T = typename D::T;
  __shared__ std::uint32_t sc[kChunk * 5];
  T r[MAXS];
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * kThreads + threadIdx.x;
  const bool valid = i < a.n;
  const unsigned long long j = valid ? i : a.n - 1;  // clamped: every thread reaches the barriers
  D::load(a, j, valid, r);
  auto fetch = [&](std::uint32_t o) -> T {
    if (o & kCoef) return D::coef(a, o & ~kCoef);
    if (o & kZero) return D::zero();
    return r[o];
  };
  for (std::uint32_t base = 0; base < a.nops; base += kChunk) {
    const std::uint32_t cnt = min(kChunk, a.nops - base);
    __syncthreads();
    for (std::uint32_t w = threadIdx.x; w < cnt * 5; w += kThreads) sc[w] = __ldg(a.code + base * 5 + w);
    __syncthreads();
    for (std::uint32_t k = 0; k < cnt; ++k) {
      const std::uint32_t* op = sc + 5 * k;
      const T x = fetch(op[2]), y = fetch(op[3]);
      T v;
      if (op[0] == 0) {
        v = D::add(x, y);
      } else if (op[0] == 1) {
        v = D::mul(x, y);
      } else {
        v = D::fma(x, y, fetch(op[4]));
      }
      r[op[1]] = v;
    }
  }
  if (valid) D::store(a, i, fetch(a.result));
}

template <class D>
cudaError_t launch_domain(const VmArgs& a, std::uint32_t nslots, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((a.n + kThreads - 1) / kThreads);
  if (nslots <= 16) {
    vm_kernel<D, 16><<<grid, kThreads, 0, s>>>(a);
  } else if (nslots <= 64) {
    vm_kernel<D, 64><<<grid, kThreads, 0, s>>>(a);
  } else if (nslots <= 256) {
    vm_kernel<D, 256><<<grid, kThreads, 0, s>>>(a);
  } else if (nslots <= 1024) {
    vm_kernel<D, 1024><<<grid, kThreads, 0, s>>>(a);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

extern "C" {

/// Largest slot file the VM kernels have.
unsigned pe_vm_max_slots(void) { return 1024; }

/// Launches the walk VM for `domain` (lower::Domain codes 0..4) over n points.
/// in: nvars coordinate pointers (intervals: 2 * nvars, lo/hi interleaved).
cudaError_t pe_launch_vm(int domain, const std::uint32_t* code, std::uint32_t nops,
                         std::uint32_t nslots, std::uint32_t result, const std::uint64_t* lo,
                         const std::uint64_t* hi, std::uint32_t nvars, const void* const* in,
                         void* out0, void* out1, unsigned long long n, unsigned* flag,
                         const unsigned long long* bounds, cudaStream_t stream) {
  if (nvars > kMaxVars || n == 0) return n == 0 ? cudaSuccess : cudaErrorInvalidValue;
  if (n > 0x7fffffffull * kThreads) return cudaErrorInvalidValue;
  VmArgs a{};
  a.code = code;
  a.lo = lo;
  a.hi = hi;
  const std::uint32_t nin = domain == 3 ? 2 * nvars : nvars;
  for (std::uint32_t v = 0; v < nin; ++v) a.in[v] = in[v];
  a.out0 = out0;
  a.out1 = out1;
  a.n = n;
  a.flag = flag;
  for (std::uint32_t v = 0; v < nvars && bounds; ++v) a.bounds[v] = bounds[v];
  a.nops = nops;
  a.nvars = nvars;
  a.result = result;
  switch (domain) {
    case 0:
    case 1: return launch_domain<F64>(a, nslots, stream);
    case 2: return launch_domain<I64>(a, nslots, stream);
    case 3: return launch_domain<Interval>(a, nslots, stream);
    case 4: return launch_domain<I64F>(a, nslots, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // extern "C"
