// Lowering: FlatProgram -> register-scheduled instruction stream.
//
// The reference interprets its flat record list per point through a heap
// register file indexed at run time (eval.hpp:218-249, run_nested 208-213,
// power tables powers.hpp:50-72). On B200 every point is one thread and the
// record list is identical for all of them, so the walk is executed *once,
// symbolically, on the host*: register slots m[lazy]/m[parent] become SSA
// virtual registers, nested programs are inlined where the reference calls
// run_nested, and the per-point power table becomes a fixed DAG of
// multiplications. The result is a straight-line stream the PTX emitter turns
// into one specialised kernel per (program, domain).
//
// Two lowerings:
//  * lower_strict  — the reference op sequence verbatim, including adds into
//    a zero register (`m[parent] = add(m[parent], v)` with m[parent] == 0) and
//    the power-table multiplication order. Used where bit-identity with the
//    reference is the contract: IntervalDomain (interval.cpp:36-52) and the
//    optional bit-exact DoubleDomain mode.
//  * lower_fused   — same tree, same multiplications, but each record's
//    `(m + c) * x^d` + parent accumulation becomes one FMA: the record's
//    coefficient (scalar or nested result) is folded in as the addend the
//    moment its register goes live ("accumulator-init-with-coefficient",
//    SURVEY §8a rules). Used for fp64 (tolerance 1e-12 * sum|terms|) and
//    int64 (exact in any order once the host overflow proof holds).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "front/flat.hpp"

namespace polyeval::lower {

struct Operand {
  enum Kind : std::uint8_t { None = 0, Reg, Coef, Pow, Zero };
  Kind kind = None;
  std::uint32_t id = 0;  // Reg: virtual register; Coef: table slot; Pow: power id

  static Operand reg(std::uint32_t r) { return {Reg, r}; }
  static Operand coef(std::uint32_t k) { return {Coef, k}; }
  static Operand pow(std::uint32_t p) { return {Pow, p}; }
  static Operand zero() { return {Zero, 0}; }
  bool is(Kind k) const { return kind == k; }
};

enum class OpKind : std::uint8_t {
  Add,  // dst = a + b            (strict: a may be Zero)
  Mul,  // dst = a * b
  Fma,  // dst = a * b + c        (fused lowering only)
};

struct Op {
  OpKind kind;
  std::uint32_t dst;
  Operand a, b, c;
};

/// One entry of the per-variable power table: base^exponent.
struct Power {
  std::uint32_t var = 0;
  std::uint32_t exponent = 1;
  // exponent > 1: product of two earlier powers (memoized halving).
  std::uint32_t lo = 0, hi = 0;
};

template <typename C>
struct Stream {
  std::uint32_t nvars = 0;
  std::vector<Power> powers;       // topological: operands before products
  std::vector<Op> ops;             // the walk
  std::vector<C> coefs;            // coefficient table, first-use order
  // strict streams: outward nextafter steps applied when coefficient k is
  // injected (an interval zero-add of a constant, [next_down(0 + c.lo),
  // next_up(0 + c.hi)], folded on the host; fp64 0.0 + c == c needs none)
  std::vector<std::uint32_t> widen;
  // strict univariate streams: parity of the absolute exponent of the term
  // coefficient k belongs to (mirror_stream); `mirrorable` is false when the
  // program has nested sub-programs
  std::vector<std::uint8_t> odd;
  bool mirrorable = false;
  std::uint32_t nregs = 0;         // virtual registers used by `ops`
  Operand result;                  // Reg, Coef or Zero
  bool strict = false;

  // Counters for the roofline bookkeeping.
  std::uint64_t n_add = 0, n_mul = 0, n_fma = 0, n_zero_add = 0, n_folded = 0;
  std::uint64_t power_muls() const {
    std::uint64_t m = 0;
    for (const auto& p : powers) m += p.exponent > 1 ? 1 : 0;
    return m;
  }
};

template <typename C>
Stream<C> lower_strict(const front::FlatProgram<C>& program);

/// `fold_constants` = false keeps a constant + constant sum as an op (the
/// wide-integer plans carry placeholders for their coefficients: nothing may
/// be computed from them on the host).
template <typename C>
Stream<C> lower_fused(const front::FlatProgram<C>& program, bool fold_constants = true);

/// The strict stream of q(y) = p(-y): the same walk with the coefficients of
/// odd-exponent terms negated. Every primitive of the interval walk (RN
/// add/mul, nextafter, the product hull) commutes with negation, so q's walk
/// at -x mirrors p's at x register for register and ends in p(x) itself.
/// Returns false (no mirror) for nested programs or an unnegatable int64.
template <typename C>
bool mirror_stream(const Stream<C>& s, Stream<C>* out);

/// Interval value of coefficient k of a strict stream: the reference
/// injection (numeric.cpp:17-26: exact -> [c, c], else one ulp outward)
/// followed by the folded zero-add steps (one std::nextafter outward each).
struct IntervalWord {
  double lo, hi;
};
template <typename C>
IntervalWord interval_coefficient(const Stream<C>& s, std::size_t k);

/// Stable 64-bit FNV-1a over arbitrary bytes (cache keys, stream hashes).
inline std::uint64_t fnv1a(const void* data, std::size_t n,
                           std::uint64_t h = 1469598103934665603ull) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace polyeval::lower
