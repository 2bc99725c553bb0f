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

// ---------------------------------------------------------------------------
// narrow_limbs: K-limb two's-complement results -> int64, flagging (bit 8 of
// the status word) any value whose high limbs are not the sign extension of
// limb 0, i.e. that does not fit int64. Lets pe_eval_i64 stay exact when the
// int64 overflow proof fails but the results themselves fit (the reference
// BigInt has no overflow; its int64 conversion is what fails).
namespace {
struct LimbPtrs {
  const unsigned long long* p[8];
};

__global__ void __launch_bounds__(256) narrow_limbs_kernel(LimbPtrs l, int k, size_t n,
                                                           long long* __restrict__ out,
                                                           unsigned* __restrict__ flag) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  bool bad = false;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const unsigned long long v0 = l.p[0][i];
    const unsigned long long ext = static_cast<unsigned long long>(static_cast<long long>(v0) >> 63);
    for (int j = 1; j < k; ++j) bad |= l.p[j][i] != ext;
    out[i] = static_cast<long long>(v0);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 8u);
}
}  // namespace

extern "C" cudaError_t pe_launch_narrow_limbs(const unsigned long long* const* limbs, int k,
                                              size_t n, long long* out, unsigned* flag, int sms,
                                              cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (k < 1 || k > 8) return cudaErrorInvalidValue;
  LimbPtrs l{};
  for (int j = 0; j < k; ++j) l.p[j] = limbs[j];
  const size_t want = (n + 255) / 256;
  const int grid = static_cast<int>(want < static_cast<size_t>(sms) * 8 ? want
                                                                        : static_cast<size_t>(sms) * 8);
  narrow_limbs_kernel<<<grid, 256, 0, stream>>>(l, k, n, out, flag);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Pipe-peak microbenchmarks: the roofline denominators for the FP64-bound
// (C1/C2/C4/C5) and int64-MAD-bound (C3) walks. MEASURED_PEAKS.json carries
// only HBM and bf16 peaks, so bench.py measures these live on the same GPU.
// Each thread runs 8 independent dependency chains (enough ILP to saturate the
// pipe at full occupancy); the result is folded into a store so nothing is
// dead-code eliminated.
namespace {

// The multiplier is an immediate (1 - 2^-20 has a short encoding) and the
// addend a kernel parameter (uniform register): a DFMA with three 64-bit
// register operands measured ~3 % below the pipe rate the walk kernels reach
// (register-bank pressure), so the probe would not be an upper bound.
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
  (void)a;
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fma(r[k], 0.99999904632568359375, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  if (s == 1234.5) out[0] = s;  // never true in practice; keeps the chains live
}

__global__ void __launch_bounds__(256) imad64_peak_kernel(long long* out, int iters, long long a,
                                                          long long b) {
  long long r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = r[k] * a + b;
  }
  long long s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= r[k];
  if (s == 0x123456789LL) out[0] = s;
}

// FP64 tensor-core probe: mma.sync m8n8k4 f64
// (DMMA), 8 independent accumulator tiles per warp; one instruction is 8 x 8
// x 4 = 256 FMAs per warp (a DFMA: 32). Counted in FMAs, like the DFMA probe.
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters, double b) {
  double c[8][2];
  const double a = 0.99999904632568359375 + threadIdx.x * 1e-9;
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5) out[0] = s;
}

// one warp, one dependent DFMA chain: SM cycles per DFMA (latency)
__global__ void dfma_latency_kernel(double* out, long long* cycles, int iters, double a, double b) {
  double r = threadIdx.x * 1e-3;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) r = fma(r, a, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cycles = t1 - t0;
  if (r == 1234.5) out[0] = r;
}

}  // namespace

// Dependent-DFMA latency in SM cycles (single warp, 4096-deep chain).
extern "C" cudaError_t pe_measure_dfma_latency(double* cycles_per_op) {
  void* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, 64);
  if (e != cudaSuccess) return e;
  long long* cyc = reinterpret_cast<long long*>(static_cast<char*>(buf) + 32);
  long long h = 0;
  for (int rep = 0; rep < 2; ++rep) {
    dfma_latency_kernel<<<1, 32>>>(static_cast<double*>(buf), cyc, 4096, 0.999999, 1e-7);
  }
  e = cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  *cycles_per_op = static_cast<double>(h) / 4096.0;
  return e;
}

// ops/s for one (warm) launch; 1 op = one DFMA / one 64-bit multiply-add
extern "C" cudaError_t pe_measure_pipe_peak(int kind, int sms, double* ops_per_s) {
  const int blocks = sms * 8, threads = 256, iters = 4096;
  void* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, 64);
  if (e != cudaSuccess) return e;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  // 16 warm-up launches (~10 ms of FP64 work: the SM clock leaves any idle
  // state first — a short probe right after host-side setup read ~10 % low
  // and real kernels beat it), then the best of 16 timed launches
  float best_ms = 1e30f;
  constexpr int kWarm = 16, kReps = 32;
  for (int rep = 0; rep < kReps; ++rep) {
    cudaEventRecord(t0);
    if (kind == 0) {
      dfma_peak_kernel<<<blocks, threads>>>(static_cast<double*>(buf), iters, 0.999999, 1e-7);
    } else if (kind == 3) {
      dmma_peak_kernel<<<blocks, threads>>>(static_cast<double*>(buf), iters / 8, 1e-7);
    } else {
      imad64_peak_kernel<<<blocks, threads>>>(static_cast<long long*>(buf), iters,
                                              0x5851F42D4C957F2DLL, 0x14057B7EF767814FLL);
    }
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    if (rep >= kWarm && ms < best_ms) best_ms = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(buf);
  // FMAs per launch: DFMA / IMAD 8 chains x iters per thread; DMMA 8 tiles x
  // iters/8 instructions x 256 FMAs per warp = 8 x iters x 8 per thread
  *ops_per_s = kind == 3
                   ? static_cast<double>(blocks) * (threads / 32) * (iters / 8) * 8 * 256 / (best_ms * 1e-3)
                   : static_cast<double>(blocks) * threads * iters * 8 / (best_ms * 1e-3);
  return e;
}

// ---------------------------------------------------------------------------
// classify_intervals: the sign partition of the univariate interval fast path
// (lower/ptx.cpp, KernelImage::iv_partition). Interval i = [lo_i, hi_i] goes
//   lo > 0           -> idx[front++]      (x > 0 entry of the program)
//   hi < 0           -> idx[n-1-back++]   (x < 0 entry of the mirrored program)
//   otherwise        -> fixup list        (straddles / touches zero, NaN)
// and invalid intervals (NaN endpoint, lo > hi: reference interval.cpp:21-26)
// set bit 2 of the status word, a full fixup list bit 4 — the same status
// contract as the walk kernels. Each warp owns 512 consecutive intervals
// (16 rounds of 32, ballots kept in registers), so every list keeps point
// order inside a warp's range and the walk kernels' gathers stay coalesced;
// one atomicAdd per CTA and list. HBM-bound: 16 B read + <= 4 B written per
// interval.
namespace {
constexpr int kClsThreads = 256, kClsRounds = 16;
constexpr int kClsTile = kClsThreads * kClsRounds;

__global__ void __launch_bounds__(kClsThreads) classify_intervals_kernel(
    const double* __restrict__ lo, const double* __restrict__ hi, unsigned long long n,
    unsigned* __restrict__ idx, unsigned* __restrict__ counts, unsigned* __restrict__ fix_list,
    unsigned* __restrict__ fix_count, unsigned long long fix_cap, unsigned* __restrict__ flag) {
  __shared__ unsigned s_pos[kClsThreads / 32], s_neg[kClsThreads / 32];
  __shared__ unsigned s_base_pos, s_base_neg;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long w0 =
      static_cast<unsigned long long>(blockIdx.x) * kClsTile + static_cast<unsigned long long>(warp) * 32 * kClsRounds;
  const unsigned lt = (1u << lane) - 1u;
  unsigned mpos[kClsRounds], mneg[kClsRounds];
  unsigned npos = 0, nneg = 0;
  // all 16 rounds' loads in flight before the first ballot
  double vl[kClsRounds], vh[kClsRounds];
#pragma unroll
  for (int r = 0; r < kClsRounds; ++r) {
    const unsigned long long i = w0 + static_cast<unsigned long long>(r) * 32 + lane;
    vl[r] = i < n ? __ldg(lo + i) : 0.0;
    vh[r] = i < n ? __ldg(hi + i) : 0.0;
  }
#pragma unroll
  for (int r = 0; r < kClsRounds; ++r) {
    const unsigned long long i = w0 + static_cast<unsigned long long>(r) * 32 + lane;
    bool pos = false, neg = false, other = false;
    if (i < n) {
      const double l = vl[r], h = vh[r];
      const bool valid = l <= h;  // false for NaN endpoints
      if (!valid) atomicOr(flag, 2u);
      pos = valid && l > 0.0;
      neg = valid && h < 0.0;
      other = !pos && !neg;
    }
    mpos[r] = __ballot_sync(0xffffffffu, pos);
    mneg[r] = __ballot_sync(0xffffffffu, neg);
    const unsigned mo = __ballot_sync(0xffffffffu, other);
    if (mo) {  // rare: straddling / zero-touching / invalid intervals
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(fix_count, static_cast<unsigned>(__popc(mo)));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (other) {
        const unsigned long long slot = static_cast<unsigned long long>(base) + __popc(mo & lt);
        if (slot < fix_cap) {
          fix_list[slot] = static_cast<unsigned>(i);
        } else {
          atomicOr(flag, 4u);
        }
      }
    }
    npos += __popc(mpos[r]);
    nneg += __popc(mneg[r]);
  }
  if (lane == 0) {
    s_pos[warp] = npos;
    s_neg[warp] = nneg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned tp = 0, tn = 0;
    for (int w = 0; w < kClsThreads / 32; ++w) {
      const unsigned p = s_pos[w], q = s_neg[w];
      s_pos[w] = tp;
      s_neg[w] = tn;
      tp += p;
      tn += q;
    }
    s_base_pos = tp ? atomicAdd(&counts[0], tp) : 0;
    s_base_neg = tn ? atomicAdd(&counts[1], tn) : 0;
  }
  __syncthreads();
  unsigned op = s_base_pos + s_pos[warp], on = s_base_neg + s_neg[warp];
#pragma unroll
  for (int r = 0; r < kClsRounds; ++r) {
    const unsigned i = static_cast<unsigned>(w0 + static_cast<unsigned long long>(r) * 32 + lane);
    if ((mpos[r] >> lane) & 1u) idx[op + __popc(mpos[r] & lt)] = i;
    if ((mneg[r] >> lane) & 1u) idx[n - 1 - (on + __popc(mneg[r] & lt))] = i;
    op += __popc(mpos[r]);
    on += __popc(mneg[r]);
  }
}
}  // namespace

extern "C" cudaError_t pe_launch_classify_intervals(const double* lo, const double* hi,
                                                    unsigned long long n, unsigned* idx,
                                                    unsigned* counts, unsigned* fix_list,
                                                    unsigned* fix_count,
                                                    unsigned long long fix_cap, unsigned* flag,
                                                    cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const unsigned long long grid = (n + kClsTile - 1) / kClsTile;
  classify_intervals_kernel<<<static_cast<unsigned>(grid), kClsThreads, 0, stream>>>(
      lo, hi, n, idx, counts, fix_list, fix_count, fix_cap, flag);
  return cudaGetLastError();
}
