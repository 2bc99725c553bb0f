// Exact evaluation with arbitrary-width integers (the paper's Figure-1
// workload: dense polynomials with 64..2048-bit coefficients at 64..2048-bit
// points, reference BigIntDomain, bench.cpp:59-187), one point per CTA.
//
// The host (runtime/wide.cpp) lowers the program to the walk-VM op list
// (lower/vm.hpp, strict stream: the reference's adds and products) and
// bounds every value's magnitude, so each slot of the per-point arena has a
// fixed width in 64-bit limbs, two's complement, little-endian. A CTA walks
// the op list (warp-uniform) and executes each op cooperatively:
//   add  r = a + b     limb-parallel sum with a carry-lookahead scan
//                      (generate / propagate pairs, Kogge-Stone over the
//                      warp's lanes, then over the CTA's warps)
//   mul  r = a * b     magnitudes (negated in scratch if negative), column
//                      products: thread t owns result columns t, t + T, ...
//                      and sums a_i * b_(k-i) as 128-bit products into a
//                      192-bit accumulator; the three accumulator words are
//                      then added as three shifted numbers; negated if the
//                      operand signs differ
// Widths come from the host bound (|value| < 2^bits), so no op overflows its
// destination and the truncated two's-complement arithmetic is exact.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kMaxThreads = 256;  // CTA size is chosen per plan (32..256)
constexpr int kMaxWarps = kMaxThreads / 32;
constexpr std::uint32_t kCoef = 0x80000000u, kZero = 0x40000000u;
constexpr int kMaxVars = 16;

struct WideArgs {
  const std::uint32_t* code;     // 8 words per op (kind, dst, a, b, w_r, w_a, w_b, 0)
  const std::uint32_t* slot_off; // per slot: arena offset (limbs)
  const std::uint32_t* slot_w;   // per slot: width (limbs)
  const std::uint32_t* coef_off; // per coefficient: offset into coef_words
  const std::uint32_t* coef_w;   // per coefficient: width
  const std::uint64_t* coef_words;
  const std::uint64_t* in[kMaxVars];  // coords[v][i * point_limbs + k]
  std::uint64_t* out;                 // out[i * out_limbs + k]
  std::uint64_t* scratch;             // per CTA: arena + 5 * tmp_w limbs
  unsigned long long n;
  std::uint32_t nops, nvars, point_limbs, out_limbs, result, result_w, arena, tmp_w;
};

struct Num {
  const std::uint64_t* p;
  std::uint32_t w;  // limbs (0: zero)
};

__device__ __forceinline__ std::uint64_t limb(const Num& x, std::uint32_t k) {
  if (k < x.w) return x.p[k];
  return x.w && (x.p[x.w - 1] >> 63) ? ~0ull : 0ull;  // sign extension
}

// Carry-lookahead across the CTA. Each thread holds (g, p) for its chunk:
// g = carry out with carry in 0, p = carry out with carry in 1 (p >= g).
// Returns this thread's carry in (chunks are ordered by thread index).
__device__ bool block_carry_in(bool g, bool p, bool cin0, std::uint32_t* s_pair) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  // inclusive scan of (g, p) pairs: (g2,p2) o (g1,p1) = (g2 | (p2 & g1), p2 & p1)
  // represented as carry-out given carry-in 0 / 1
  bool c0 = g, c1 = p;
  for (int d = 1; d < 32; d <<= 1) {
    const bool l0 = __shfl_up_sync(0xffffffffu, c0, d), l1 = __shfl_up_sync(0xffffffffu, c1, d);
    if (lane >= d) {
      const bool n0 = l0 ? c1 : c0, n1 = l1 ? c1 : c0;
      c0 = n0;
      c1 = n1;
    }
  }
  // warp totals
  if (lane == 31) s_pair[warp] = (c0 ? 1u : 0u) | (c1 ? 2u : 0u);
  __syncthreads();
  if (threadIdx.x == 0) {
    bool c = cin0;
    for (int w = 0; w < nwarps; ++w) {
      const std::uint32_t t = s_pair[w];
      s_pair[nwarps + w] = c ? 1u : 0u;  // carry into warp w
      c = c ? (t & 2u) : (t & 1u);
    }
  }
  __syncthreads();
  const bool wcin = s_pair[nwarps + warp] != 0;
  // carry into this lane = exclusive scan applied to the warp's carry in
  const bool e0 = __shfl_up_sync(0xffffffffu, c0, 1), e1 = __shfl_up_sync(0xffffffffu, c1, 1);
  const bool cin = lane == 0 ? wcin : (wcin ? e1 : e0);
  __syncthreads();  // s_pair reused by the next call
  return cin;
}

// r[0, w) = x + y + cin0 (two's complement, truncated to w limbs); r may
// alias neither input (the host never allocates a destination slot that
// holds an operand).
__device__ void big_add(std::uint64_t* r, std::uint32_t w, const Num& x, const Num& y, bool cin0,
                        std::uint32_t* s_pair) {
  const std::uint32_t T = blockDim.x;
  const std::uint32_t chunk = (w + T - 1) / T;
  const std::uint32_t lo = threadIdx.x * chunk, hi = min(w, lo + chunk);
  bool g = false, p = true;  // carry out for carry in 0 / 1 over [lo, hi)
  for (std::uint32_t k = lo; k < hi; ++k) {
    const std::uint64_t s = limb(x, k) + limb(y, k);
    const bool c = s < limb(x, k);
    // carry in 0: out = c | (prev carry & s + ...): track both chains
    const bool g2 = c || (g && s == ~0ull);
    const bool p2 = c || (p && s == ~0ull);
    g = g2;
    p = p2;
  }
  if (lo >= hi) p = true, g = false;  // empty chunk: passes its carry through
  bool cin = block_carry_in(g, p, cin0, s_pair);
  for (std::uint32_t k = lo; k < hi; ++k) {
    const std::uint64_t a = limb(x, k), s = a + limb(y, k);
    const bool c1 = s < a;
    const std::uint64_t t = s + (cin ? 1ull : 0ull);
    const bool c2 = cin && t == 0;
    r[k] = t;
    cin = c1 || c2;
  }
  __syncthreads();
}

// r = -x over w limbs (~x + 1)
__device__ void big_neg(std::uint64_t* r, std::uint32_t w, const Num& x, std::uint32_t* s_pair,
                        std::uint64_t* tmp) {
  const std::uint32_t T = blockDim.x;
  for (std::uint32_t k = threadIdx.x; k < w; k += T) tmp[k] = ~limb(x, k);
  __syncthreads();
  big_add(r, w, Num{tmp, w}, Num{nullptr, 0}, true, s_pair);
}

__device__ __forceinline__ bool negative(const Num& x) { return x.w && (x.p[x.w - 1] >> 63); }

// Scratch of one CTA beside its arena: five buffers of tmp_w limbs.
struct Tmp {
  std::uint64_t *ta, *tb, *c0, *c1, *c2;
};

// r[0, w) = x * y, exact when |x * y| < 2^(64 w - 1); r aliases neither
// operand nor a scratch buffer.
__device__ void big_mul(std::uint64_t* r, std::uint32_t w, Num x, Num y, const Tmp& t,
                        std::uint32_t* s_pair) {
  const std::uint32_t T = blockDim.x;
  const bool nx = negative(x), ny = negative(y);
  if (nx) {  // magnitudes (the top limb may then use the sign bit: read as unsigned)
    big_neg(t.ta, x.w, x, s_pair, t.c0);
    x = Num{t.ta, x.w};
  }
  if (ny) {
    big_neg(t.tb, y.w, y, s_pair, t.c0);
    y = Num{t.tb, y.w};
  }
  // significant lengths (static widths are bounds; values are often shorter)
  __shared__ std::uint32_t s_w[2];
  if (threadIdx.x == 0) {
    std::uint32_t a = x.w, b = y.w;
    while (a && x.p[a - 1] == 0) --a;
    while (b && y.p[b - 1] == 0) --b;
    s_w[0] = a;
    s_w[1] = b;
  }
  __syncthreads();
  const std::uint32_t wa = s_w[0], wb = s_w[1];
  // column k: sum_i a_i * b_(k-i) as 192 bits (c0, c1, c2); thread t owns
  // columns t, t + T, ...
  for (std::uint32_t k = threadIdx.x; k < w; k += T) {
    std::uint64_t a0 = 0, a1 = 0, a2 = 0;
    const std::uint32_t i_lo = k + 1 > wb ? k + 1 - wb : 0, i_hi = min(k + 1, wa);
    for (std::uint32_t i = i_lo; i < i_hi; ++i) {
      const std::uint64_t u = x.p[i], v = y.p[k - i];
      const std::uint64_t plo = u * v, phi = __umul64hi(u, v);
      a0 += plo;
      const std::uint64_t c = a0 < plo;   // carry into a1
      std::uint64_t s = a1 + phi;
      std::uint64_t cc = s < a1;          // carry into a2
      s += c;
      cc += s < c;
      a1 = s;
      a2 += cc;
    }
    t.c0[k] = a0;
    t.c1[k] = a1;
    t.c2[k] = a2;
  }
  __syncthreads();
  // product = c0 + (c1 << 64) + (c2 << 128); every part is <= the product,
  // so each fits w limbs with the sign bit clear (the shifted-out limbs are 0)
  for (std::uint32_t k = threadIdx.x; k < w; k += T) {
    t.ta[k] = k >= 1 ? t.c1[k - 1] : 0;
    t.tb[k] = k >= 2 ? t.c2[k - 2] : 0;
  }
  __syncthreads();
  if (wa <= 1 || wb <= 1) {
    // one partial product per column: c2 is zero, product = c0 + (c1 << 64)
    if (nx == ny) {
      big_add(r, w, Num{t.c0, w}, Num{t.ta, w}, false, s_pair);
    } else {
      big_add(t.c1, w, Num{t.c0, w}, Num{t.ta, w}, false, s_pair);
      big_neg(r, w, Num{t.c1, w}, s_pair, t.tb);
    }
    return;
  }
  big_add(t.c1, w, Num{t.c0, w}, Num{t.ta, w}, false, s_pair);
  if (nx == ny) {
    big_add(r, w, Num{t.c1, w}, Num{t.tb, w}, false, s_pair);
  } else {
    big_add(t.c0, w, Num{t.c1, w}, Num{t.tb, w}, false, s_pair);
    big_neg(r, w, Num{t.c0, w}, s_pair, t.ta);
  }
}

// operand o of width w (the width its value was written with)
__device__ Num operand(const WideArgs& a, std::uint64_t* arena, std::uint32_t o, std::uint32_t w) {
  if (o & kZero) return Num{nullptr, 0};
  if (o & kCoef) {
    const std::uint32_t k = o & ~kCoef;
    return Num{a.coef_words + a.coef_off[k], a.coef_w[k]};
  }
  return Num{arena + a.slot_off[o], w};
}

__global__ void __launch_bounds__(kMaxThreads) wide_walk_kernel(const WideArgs a) {
  const std::uint32_t T = blockDim.x;
  __shared__ std::uint32_t s_pair[2 * kMaxWarps];
  std::uint64_t* arena = a.scratch + static_cast<size_t>(blockIdx.x) * (a.arena + 5ull * a.tmp_w);
  Tmp t;
  t.ta = arena + a.arena;
  t.tb = t.ta + a.tmp_w;
  t.c0 = t.tb + a.tmp_w;
  t.c1 = t.c0 + a.tmp_w;
  t.c2 = t.c1 + a.tmp_w;
  for (unsigned long long i = blockIdx.x; i < a.n; i += gridDim.x) {
    // coordinates into slots 0..nvars-1, sign-extended to the slot width
    for (std::uint32_t v = 0; v < a.nvars; ++v) {
      const Num x{a.in[v] + i * a.point_limbs, a.point_limbs};
      std::uint64_t* d = arena + a.slot_off[v];
      for (std::uint32_t k = threadIdx.x; k < a.slot_w[v]; k += T) d[k] = limb(x, k);
    }
    __syncthreads();
    for (std::uint32_t op = 0; op < a.nops; ++op) {
      const std::uint32_t* c = a.code + 8 * op;
      const std::uint32_t kind = c[0], dst = c[1];
      std::uint64_t* r = arena + a.slot_off[dst];
      const std::uint32_t w = c[4];
      const Num x = operand(a, arena, c[2], c[5]), y = operand(a, arena, c[3], c[6]);
      if (kind == 0) {
        big_add(r, w, x, y, false, s_pair);
      } else {
        big_mul(r, w, x, y, t, s_pair);
      }
    }
    const Num res = operand(a, arena, a.result, a.result_w);
    std::uint64_t* o = a.out + i * a.out_limbs;
    for (std::uint32_t k = threadIdx.x; k < a.out_limbs; k += T) o[k] = limb(res, k);
    __syncthreads();
  }
}

}  // namespace

extern "C" cudaError_t pe_launch_wide(const std::uint32_t* code, std::uint32_t nops,
                                      const std::uint32_t* slot_off, const std::uint32_t* slot_w,
                                      const std::uint32_t* coef_off, const std::uint32_t* coef_w,
                                      const std::uint64_t* coef_words, std::uint32_t nvars,
                                      const std::uint64_t* const* in, std::uint32_t point_limbs,
                                      std::uint64_t* out, std::uint32_t out_limbs,
                                      std::uint32_t result, std::uint32_t result_w,
                                      std::uint32_t arena,
                                      std::uint32_t tmp_w, std::uint64_t* scratch,
                                      unsigned grid, unsigned threads, unsigned long long n,
                                      cudaStream_t stream) {
  if (nvars > kMaxVars) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  WideArgs a{};
  a.code = code;
  a.slot_off = slot_off;
  a.slot_w = slot_w;
  a.coef_off = coef_off;
  a.coef_w = coef_w;
  a.coef_words = coef_words;
  for (std::uint32_t v = 0; v < nvars; ++v) a.in[v] = in[v];
  a.out = out;
  a.scratch = scratch;
  a.n = n;
  a.nops = nops;
  a.nvars = nvars;
  a.point_limbs = point_limbs;
  a.out_limbs = out_limbs;
  a.result = result;
  a.result_w = result_w;
  a.arena = arena;
  a.tmp_w = tmp_w;
  if (threads < 32 || threads > kMaxThreads || threads % 32) return cudaErrorInvalidValue;
  wide_walk_kernel<<<grid, threads, 0, stream>>>(a);
  return cudaGetLastError();
}

