// Exact evaluation with arbitrary-width integers (the paper's Figure-1
// workload: dense polynomials with 64..2048-bit coefficients at 64..2048-bit
// points, reference BigIntDomain, bench.cpp:59-187), one point per CTA.
//
// The host (runtime/wide.cpp) lowers the program to the walk-VM op list
// (lower/vm.hpp, fused stream: one multiply-add per record of the reference
// walk — exact integers give its value in any order) and bounds every
// value's magnitude, so each slot of the per-point arena has a
// fixed width in 64-bit limbs, two's complement, little-endian. A CTA walks
// the op list (warp-uniform) and executes each op cooperatively, one limb per
// lane:
//   add  r = a + b     rows of 32 limbs, the carries of a row resolved with
//                      two ballots and one integer addition (generate /
//                      propagate masks), the carry out of a row entering the
//                      next; several warps take ranges of rows and exchange
//                      (carry out, would-ripple) pairs
//   mul  r = a * b     magnitudes (negated if negative), column products in
//                      32 x 32-limb blocks held in registers: lane k of a
//                      warp owns column 32 C + k and gathers a_i by a
//                      broadcast shuffle and b_(k-i) by a window shuffle,
//                      128-bit products into a 192-bit accumulator; the three
//                      accumulator words are then added as three shifted
//                      numbers; negated if the operand signs differ
//   narrow ops (<= 32 limbs, most of a walk): warp 0 alone, operands loaded
//                      once, everything else in registers
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
  const std::uint32_t* code;     // 8 words per op (runtime/wide.hpp: resolved offsets), 16-byte aligned
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

// ---- one limb per lane: warp-wide helpers -----------------------------------

// Carries of a 32-lane addition: lane k generates (g) or propagates (p, with
// g and p exclusive). Bit k of the result is the carry INTO lane k, bit 32
// the carry out of lane 31. The chain c(k+1) = g(k) | (p(k) & c(k)) is the
// carry chain of the binary addition (G|P) + G + cin, and a sum's carries are
// sum ^ x ^ y.
__device__ __forceinline__ std::uint64_t lane_carries_out(bool g, bool p, bool cin) {
  const std::uint32_t G = __ballot_sync(0xffffffffu, g), P = __ballot_sync(0xffffffffu, p);
  const std::uint64_t X = G | P;
  return (X + G + (cin ? 1u : 0u)) ^ X ^ G;
}

// lane k: limb k of a + b + cin (mod 2^(64*32))
__device__ __forceinline__ std::uint64_t lanes_add(std::uint64_t a, std::uint64_t b, bool cin) {
  const std::uint64_t s = a + b;
  const std::uint64_t c = lane_carries_out(s < a, s == ~0ull, cin);
  return s + ((c >> (threadIdx.x & 31)) & 1u);
}

__device__ __forceinline__ std::uint64_t shfl64(std::uint64_t v, int src) {
  const std::uint32_t lo = __shfl_sync(0xffffffffu, static_cast<std::uint32_t>(v), src);
  const std::uint32_t hi = __shfl_sync(0xffffffffu, static_cast<std::uint32_t>(v >> 32), src);
  return (static_cast<std::uint64_t>(hi) << 32) | lo;
}

// (a2, a1, a0) += u * v: 128-bit product into a 192-bit accumulator on the
// carry flag (three instructions instead of compare-and-select carries)
__device__ __forceinline__ void mac192(std::uint64_t& a0, std::uint64_t& a1, std::uint64_t& a2,
                                       std::uint64_t u, std::uint64_t v) {
  asm("mad.lo.cc.u64 %0, %3, %4, %0;\n\tmadc.hi.cc.u64 %1, %3, %4, %1;\n\taddc.u64 %2, %2, 0;"
      : "+l"(a0), "+l"(a1), "+l"(a2)
      : "l"(u), "l"(v));
}

// Significant limbs of a magnitude (index of the top non-zero limb + 1),
// scanned a coalesced row of 32 limbs at a time from the top; every lane of
// the calling warp returns the length.
__device__ std::uint32_t significant_limbs(const Num& x) {
  const std::uint32_t lane = threadIdx.x & 31;
  for (std::uint32_t row = (x.w + 31) / 32; row-- > 0;) {
    const std::uint32_t k = 32 * row + lane;
    const std::uint32_t m = __ballot_sync(0xffffffffu, k < x.w && x.p[k] != 0);
    if (m) return 32 * row + 32 - __clz(m);
  }
  return 0;
}

// Rows [row_lo, row_hi) of 32 limbs of (inv ? ~x : x) + y + cin, one limb
// per lane, rows in turn (the carry out of a row enters the next). Stores
// limbs below w when `store`. Returns the carry out; *ones = every limb of
// the range came out all-ones (then a carry in of one more would ripple
// through the whole range).
__device__ bool add_rows(std::uint64_t* r, std::uint32_t w, const Num& x, bool inv, const Num& y,
                         bool cin, std::uint32_t row_lo, std::uint32_t row_hi, bool store,
                         bool* ones) {
  const std::uint32_t lane = threadIdx.x & 31;
  bool all = true;
  for (std::uint32_t row = row_lo; row < row_hi; ++row) {
    const std::uint32_t k = 32 * row + lane;
    const std::uint64_t a = inv ? ~limb(x, k) : limb(x, k), s = a + limb(y, k);
    const std::uint64_t c = lane_carries_out(s < a, s == ~0ull, cin);
    const std::uint64_t v = s + ((c >> lane) & 1u);
    if (store && k < w) r[k] = v;
    all = all && (k >= w || v == ~0ull);
    cin = (c >> 32) & 1u;
  }
  if (ones) *ones = __all_sync(0xffffffffu, all);
  return cin;
}

// r[0, w) = (inv ? ~x : x) + y + cin0 (two's complement, truncated to w
// limbs); r may alias neither input (the host never allocates a destination
// slot that holds an operand). Coalesced rows of 32 limbs; a CTA of several
// warps gives each a contiguous range of rows, resolves the carries between
// the ranges (carry out for carry in 0, and whether a carry in would ripple
// through) and runs the ranges again with their carry in.
__device__ void big_add(std::uint64_t* r, std::uint32_t w, const Num& x, const Num& y, bool cin0,
                        std::uint32_t* s_pair, bool inv = false) {
  const std::uint32_t nw = blockDim.x >> 5, wid = threadIdx.x >> 5;
  const std::uint32_t rows = (w + 31) / 32;
  if (nw == 1) {
    add_rows(r, w, x, inv, y, cin0, 0, rows, true, nullptr);
    __syncthreads();
    return;
  }
  const std::uint32_t per = (rows + nw - 1) / nw;
  const std::uint32_t lo = min(rows, wid * per), hi = min(rows, lo + per);
  bool ones = true;
  const bool g = add_rows(r, w, x, inv, y, false, lo, hi, false, &ones);
  if ((threadIdx.x & 31) == 0) s_pair[wid] = (g ? 1u : 0u) | (ones ? 2u : 0u);
  __syncthreads();
  if (threadIdx.x == 0) {
    bool c = cin0;
    for (std::uint32_t v = 0; v < nw; ++v) {
      const std::uint32_t t = s_pair[v];
      s_pair[nw + v] = c ? 1u : 0u;  // carry into warp v's range
      c = (t & 1u) || (c && (t & 2u));
    }
  }
  __syncthreads();
  add_rows(r, w, x, inv, y, s_pair[nw + wid] != 0, lo, hi, true, nullptr);
  __syncthreads();  // also: s_pair is reused by the next call
}

// r = -x over w limbs (~x + 1)
__device__ void big_neg(std::uint64_t* r, std::uint32_t w, const Num& x, std::uint32_t* s_pair) {
  big_add(r, w, x, Num{nullptr, 0}, true, s_pair, true);
}

__device__ __forceinline__ bool negative(const Num& x) { return x.w && (x.p[x.w - 1] >> 63); }

// Scratch of one CTA beside its arena: five buffers of tmp_w limbs.
struct Tmp {
  std::uint64_t *ta, *tb, *c0, *c1, *c2;
};

// r[0, w) = x * y, exact when |x * y| < 2^(64 w - 1); r aliases neither
// operand nor a scratch buffer.
// With `addend` (one-warp CTAs only): r = x * y + *addend, the sum taken
// in the pass that assembles the product.
__device__ void big_mul(std::uint64_t* r, std::uint32_t w, Num x, Num y, const Tmp& t,
                        std::uint32_t* s_pair, const Num* addend = nullptr) {
  const std::uint32_t T = blockDim.x;
  const bool nx = negative(x), ny = negative(y);
  if (nx) {  // magnitudes (the top limb may then use the sign bit: read as unsigned)
    big_neg(t.ta, x.w, x, s_pair);
    x = Num{t.ta, x.w};
  }
  if (ny) {
    big_neg(t.tb, y.w, y, s_pair);
    y = Num{t.tb, y.w};
  }
  // significant lengths (the static widths are bounds from the operands'
  // limb counts: values are often half as long), found by warp 0; the
  // shorter operand becomes x, the one whose limbs the inner loop steps over
  __shared__ std::uint32_t s_w[2];
  if (threadIdx.x < 32) {
    const std::uint32_t a = significant_limbs(x), b = significant_limbs(y);
    if (threadIdx.x == 0) {
      s_w[0] = a;
      s_w[1] = b;
    }
  }
  __syncthreads();
  if (s_w[0] > s_w[1]) {
    const Num z = x;
    x = y;
    y = z;
  }
  const std::uint32_t wa = min(s_w[0], s_w[1]), wb = max(s_w[0], s_w[1]);
  __syncthreads();  // s_w is rewritten by the next product
  // column k: sum_i a_i * b_(k-i) as 192 bits (c0, c1, c2). A warp owns
  // blocks of 32 columns (lane k: column 32 C + k) and works on 32 x 32-limb
  // operand blocks held one limb per lane: for block A_I of x the window of
  // y it meets is b[32 (C - I) + k - i], i = 0..31, i.e. block J = C - I for
  // k >= i and block J - 1 below. a_i is a broadcast shuffle, the window one
  // shuffle whose source lanes offer B_J or B_(J-1) by their position — two
  // coalesced loads per 1024 products instead of two loads per product.
  const int lane = threadIdx.x & 31;
  const std::uint32_t nbA = (wa + 31) / 32, nbB = (wb + 31) / 32, nbC = (w + 31) / 32;
  if (T == 32) {
    // One warp: the blocks of columns come in order, so the product is
    // assembled on the way — block C's limbs are a0 + (a1 one lane up) +
    // (a2 two lanes up), the top lanes of block C - 1 entering at the
    // bottom, as two chained additions whose carries run from block to
    // block; a negative product is negated in the same pass (~m + 1).
    std::uint64_t p1 = 0, p2a = 0, p2b = 0;  // a1 of lane 31, a2 of lanes 30 / 31, previous block
    const bool neg = nx != ny;
    bool c1 = false, c2 = false, cn = neg;
    for (std::uint32_t C = 0; C < nbC; ++C) {
      std::uint64_t a0 = 0, a1 = 0, a2 = 0;
      const std::uint32_t I_lo = C > nbB ? C - nbB : 0, I_hi = min(C + 1, nbA);
      for (std::uint32_t I = I_lo; I < I_hi; ++I) {
        const std::uint32_t J = C - I;
        const std::uint32_t ia = 32 * I + lane, ib = 32 * J + lane;
        const std::uint64_t A = ia < wa ? x.p[ia] : 0;
        const std::uint64_t BJ = ib < wb ? y.p[ib] : 0;
        const std::uint64_t BP = J >= 1 && ib - 32 < wb ? y.p[ib - 32] : 0;
        const int n_i = static_cast<int>(min(32u, wa - 32 * I));
        for (int i = 0; i < n_i; ++i) {
          const std::uint64_t u = shfl64(A, i);
          const std::uint64_t v = shfl64(lane <= 31 - i ? BJ : BP, (lane - i) & 31);
          mac192(a0, a1, a2, u, v);
        }
      }
      std::uint64_t t1 = shfl64(a1, (lane + 31) & 31), t2 = shfl64(a2, (lane + 30) & 31);
      if (lane == 0) t1 = p1, t2 = p2a;
      if (lane == 1) t2 = p2b;
      p1 = shfl64(a1, 31);
      p2a = shfl64(a2, 30);
      p2b = shfl64(a2, 31);
      std::uint64_t sum = a0 + t1;
      std::uint64_t cm = lane_carries_out(sum < a0, sum == ~0ull, c1);
      std::uint64_t s1 = sum + ((cm >> lane) & 1u);
      c1 = (cm >> 32) & 1u;
      sum = s1 + t2;
      cm = lane_carries_out(sum < s1, sum == ~0ull, c2);
      std::uint64_t m = sum + ((cm >> lane) & 1u);
      c2 = (cm >> 32) & 1u;
      const std::uint32_t k = 32 * C + lane;
      if (neg || addend) {  // (-m = ~m + 1) + addend, one more chained addition
        const std::uint64_t v = neg ? ~m : m;
        sum = v + (addend ? limb(*addend, k) : 0);
        cm = lane_carries_out(sum < v, sum == ~0ull, cn);
        m = sum + ((cm >> lane) & 1u);
        cn = (cm >> 32) & 1u;
      }
      if (k < w) r[k] = m;
    }
    __syncthreads();
    return;
  }
  {
    for (std::uint32_t C = threadIdx.x >> 5; C < nbC; C += T >> 5) {
      std::uint64_t a0 = 0, a1 = 0, a2 = 0;
      const std::uint32_t I_lo = C > nbB ? C - nbB : 0, I_hi = min(C + 1, nbA);
      for (std::uint32_t I = I_lo; I < I_hi; ++I) {
        const std::uint32_t J = C - I;
        const std::uint32_t ia = 32 * I + lane, ib = 32 * J + lane;
        const std::uint64_t A = ia < wa ? x.p[ia] : 0;
        const std::uint64_t BJ = ib < wb ? y.p[ib] : 0;
        const std::uint64_t BP = J >= 1 && ib - 32 < wb ? y.p[ib - 32] : 0;
        const int n_i = static_cast<int>(min(32u, wa - 32 * I));
        for (int i = 0; i < n_i; ++i) {
          const std::uint64_t u = shfl64(A, i);
          const std::uint64_t v = shfl64(lane <= 31 - i ? BJ : BP, (lane - i) & 31);
          mac192(a0, a1, a2, u, v);
        }
      }
      const std::uint32_t k = 32 * C + lane;
      if (k < w) {
        t.c0[k] = a0;
        t.c1[k] = a1;
        t.c2[k] = a2;
      }
    }
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
      big_neg(r, w, Num{t.c1, w}, s_pair);
    }
    return;
  }
  big_add(t.c1, w, Num{t.c0, w}, Num{t.ta, w}, false, s_pair);
  if (nx == ny) {
    big_add(r, w, Num{t.c1, w}, Num{t.tb, w}, false, s_pair);
  } else {
    big_add(t.c0, w, Num{t.c1, w}, Num{t.tb, w}, false, s_pair);
    big_neg(r, w, Num{t.c0, w}, s_pair);
  }
}

// ---- narrow values (<= 32 limbs) ---------------------------------------------
// Most ops of a walk are narrow (a dense polynomial's leaves and low tree
// levels). Warp 0 loads the operands once (lane k holds limb k), works in
// registers with shuffles and ballots, and stores the result: one memory
// round trip per op.

// r[0, w) = x + y for w <= 32 (called by the 32 lanes of warp 0)
__device__ void narrow_add(std::uint64_t* r, std::uint32_t w, const Num& x, const Num& y) {
  const std::uint32_t k = threadIdx.x & 31;
  const std::uint64_t s = lanes_add(limb(x, k), limb(y, k), false);
  if (k < w) r[k] = s;
}

// r[0, w) = x * y for w, x.w, y.w <= 32, exact when |x * y| < 2^(64 w - 1)
__device__ void narrow_mul(std::uint64_t* r, std::uint32_t w, const Num& x, const Num& y,
                           const Num* addend = nullptr) {
  const int k = threadIdx.x & 31;
  const bool nx = negative(x), ny = negative(y);
  // magnitudes, limb k in lane k (zero past the operand's width)
  std::uint64_t a = k < static_cast<int>(x.w) ? x.p[k] : 0, b = k < static_cast<int>(y.w) ? y.p[k] : 0;
  if (nx) a = lanes_add(k < static_cast<int>(x.w) ? ~a : 0, 0, true);
  if (ny) b = lanes_add(k < static_cast<int>(y.w) ? ~b : 0, 0, true);
  if (k >= static_cast<int>(x.w)) a = 0;  // the negation's carry stops at the width
  if (k >= static_cast<int>(y.w)) b = 0;
  // column k = sum_i a_i * b_(k-i) as 192 bits, stepping over the narrower operand
  std::uint32_t n_i = x.w;
  if (y.w < x.w) {
    const std::uint64_t z = a;
    a = b;
    b = z;
    n_i = y.w;
  }
  std::uint64_t a0 = 0, a1 = 0, a2 = 0;
  for (int i = 0; i < static_cast<int>(n_i); ++i) {
    const std::uint64_t u = shfl64(a, i);
    const std::uint64_t v = shfl64(b, (k - i) & 31);
    if (i <= k) mac192(a0, a1, a2, u, v);  // (lanes past y's width hold zero)
  }
  // product = A0 + (A1 << 64) + (A2 << 128)
  std::uint64_t s1 = shfl64(a1, (k + 31) & 31), s2 = shfl64(a2, (k + 30) & 31);
  if (k < 1) s1 = 0;
  if (k < 2) s2 = 0;
  std::uint64_t m = lanes_add(lanes_add(a0, s1, false), s2, false);
  if (nx != ny || addend) {  // (-m = ~m + 1) + addend
    m = lanes_add(nx != ny ? ~m : m, addend ? limb(*addend, k) : 0, nx != ny);
  }
  if (k < static_cast<int>(w)) r[k] = m;
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
    const uint4* code = reinterpret_cast<const uint4*>(a.code);
    uint4 c0 = __ldg(code), c1 = __ldg(code + 1);  // op 0 (one 32-byte record per op)
    for (std::uint32_t op = 0; op < a.nops;) {
      // kind, dst offset, a offset, b offset | width, width a, width b, flags
      const std::uint32_t kind = c0.x, w = c1.x, flags = c1.w;
      std::uint64_t* r = arena + c0.y;
      const Num x{(flags & 1u ? a.coef_words : arena) + c0.z, c1.y};
      const Num y{(flags & 2u ? a.coef_words : arena) + c0.w, c1.z};
      if (op + 1 < a.nops) {  // the next record arrives while this op runs
        c0 = __ldg(code + 2 * op + 2);
        c1 = __ldg(code + 2 * op + 3);
      }
      bool narrow = w <= 32 && x.w <= 32 && y.w <= 32;
      if (flags & 4u) {
        // a product read only by the sum in the next record (now in c0, c1):
        // e = x * y + c in one op, the product never written. Narrow pairs
        // always; wide ones where one warp assembles the product.
        const bool c_is_a = (flags & 8u) != 0;  // the product is the sum's b
        const Num c{(c1.w & (c_is_a ? 1u : 2u) ? a.coef_words : arena) + (c_is_a ? c0.z : c0.w),
                    c_is_a ? c1.y : c1.z};
        const std::uint32_t we = c1.x;
        narrow = narrow && we <= 32 && c.w <= 32;
        if (narrow || T == 32) {
          std::uint64_t* e = arena + c0.y;
          if (narrow) {
            if (threadIdx.x < 32) narrow_mul(e, we, x, y, &c);
            __syncthreads();
          } else {
            big_mul(e, we, x, y, t, s_pair, &c);
          }
          op += 2;
          if (op < a.nops) {
            c0 = __ldg(code + 2 * op);
            c1 = __ldg(code + 2 * op + 1);
          }
          continue;
        }
      }
      ++op;
      if (narrow) {
        if (threadIdx.x < 32) {
          if (kind == 0) {
            narrow_add(r, w, x, y);
          } else {
            narrow_mul(r, w, x, y);
          }
        }
        __syncthreads();  // the result is visible to the CTA's next op
      } else if (kind == 0) {
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

