// Lowering of a FlatProgram into a straight-line register stream.
// See stream.hpp for the contract; reference walk: eval.hpp:208-249,
// power tables: powers.hpp:50-72.
#include "lower/stream.hpp"

#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <stdexcept>

namespace polyeval::lower {
namespace {

// Builds the per-variable power DAG by memoized halving, in the reference's
// recursion order (ensure(e) -> ensure(e/2), ensure(e - e/2), then multiply;
// powers.hpp:58-66), and returns [var][slot] -> power id.
template <typename C>
std::vector<std::vector<std::uint32_t>> build_powers(const front::FlatProgram<C>& prog,
                                                     Stream<C>& s) {
  std::vector<std::vector<std::uint32_t>> slot_to_power(prog.exponent_sets.size());
  for (std::size_t v = 0; v < prog.exponent_sets.size(); ++v) {
    const std::vector<std::uint32_t>& set = prog.exponent_sets[v];
    if (set.empty()) continue;
    std::map<std::uint32_t, std::uint32_t> memo;
    memo[1] = static_cast<std::uint32_t>(s.powers.size());
    s.powers.push_back(Power{static_cast<std::uint32_t>(v), 1, 0, 0});
    // explicit-stack version of the reference's recursive `ensure`
    auto ensure = [&](std::uint32_t root) {
      struct Frame {
        std::uint32_t e;
        int stage;
      };
      std::vector<Frame> st{{root, 0}};
      while (!st.empty()) {
        Frame& f = st.back();
        if (memo.count(f.e)) {
          st.pop_back();
          continue;
        }
        const std::uint32_t half = f.e / 2, rest = f.e - f.e / 2;
        if (f.stage == 0) {
          f.stage = 1;
          st.push_back({half, 0});
          continue;
        }
        if (f.stage == 1) {
          f.stage = 2;
          st.push_back({rest, 0});
          continue;
        }
        Power p{static_cast<std::uint32_t>(v), f.e, memo.at(half), memo.at(rest)};
        memo[f.e] = static_cast<std::uint32_t>(s.powers.size());
        s.powers.push_back(p);
        st.pop_back();
      }
    };
    for (std::uint32_t e : set) {
      ensure(e);
      slot_to_power[v].push_back(memo.at(e));
    }
  }
  return slot_to_power;
}

template <typename C>
struct Lowerer {
  Stream<C>& s;
  const std::vector<std::vector<std::uint32_t>>& pow_of;
  const front::FlatProgram<C>& fp;

  std::uint8_t cur_odd = 0;  // strict: parity of the record being lowered
  bool fold_constants = true;

  Operand new_reg() { return Operand::reg(s.nregs++); }
  Operand coef(const C& c, std::uint32_t widen = 0) {
    s.coefs.push_back(c);
    s.widen.push_back(widen);
    s.odd.push_back(cur_odd);
    return Operand::coef(static_cast<std::uint32_t>(s.coefs.size() - 1));
  }
  Operand power(std::uint32_t prog, std::int32_t slot) {
    return Operand::pow(pow_of.at(fp.progs[prog].var).at(static_cast<std::uint32_t>(slot)));
  }
  Operand emit(OpKind k, Operand a, Operand b, Operand c = {}) {
    if (s.strict && k == OpKind::Add && a.is(Operand::Zero) && b.is(Operand::Coef)) {
      // zero register + constant: a constant (one more outward step for
      // intervals), evaluated on the host instead of per point
      ++s.n_add;
      ++s.n_zero_add;
      ++s.n_folded;
      const std::uint8_t keep = cur_odd;
      cur_odd = s.odd[b.id];
      Operand r = coef(s.coefs[b.id], s.widen[b.id] + 1);
      cur_odd = keep;
      return r;
    }
    Operand d = new_reg();
    s.ops.push_back(Op{k, d.id, a, b, c});
    switch (k) {
      case OpKind::Add:
        ++s.n_add;
        if (a.is(Operand::Zero)) ++s.n_zero_add;
        break;
      case OpKind::Mul: ++s.n_mul; break;
      case OpKind::Fma: ++s.n_fma; break;
    }
    return d;
  }

  // ---- strict: the reference walk verbatim (eval.hpp:218-239) ----
  Operand strict(std::uint32_t prog) {
    const auto& P = fp.progs[prog];
    std::vector<Operand> m(P.regs, Operand::zero());
    const std::uint32_t last = P.count - 1;
    // parity of each record's absolute exponent: its own power plus its
    // consumer's (a record's value is added into the register its consumer
    // reads and multiplies by the consumer's power)
    std::vector<std::uint8_t> par(P.count, 0);
    if (s.mirrorable) {  // univariate only
      const auto up = front::consumers(fp, prog);
      for (std::uint32_t i = P.count; i-- > 0;) {
        const auto& rec = fp.rec(prog, i);
        const std::uint32_t d = rec.power >= 0 ? fp.exponent(prog, rec.power) : 0;
        const std::uint8_t above = up[i] == UINT32_MAX ? 0 : par[up[i]];
        par[i] = static_cast<std::uint8_t>((d + above) & 1u);
        if (rec.sub >= 0) s.mirrorable = false;
      }
    }
    for (std::uint32_t i = 0; i <= last; ++i) {
      const auto& rec = fp.rec(prog, i);
      cur_odd = par[i];
      Operand v = own(prog, i, true);                          // L224
      if (rec.reads) {                                         // L225-228
        v = emit(OpKind::Add, m[rec.lazy], v);
        m[rec.lazy] = Operand::zero();
      }
      if (rec.power >= 0) v = emit(OpKind::Mul, v, power(prog, rec.power));  // L229-232
      if (i == last) return v;                                 // L233-236
      Operand& slot = m[static_cast<std::uint32_t>(rec.parent)];  // L237-238
      slot = emit(OpKind::Add, slot, v);
    }
    return Operand::zero();
  }

  // ---- fused: one FMA per powered record, coefficient folded as addend ----
  // A record's "own" value is its scalar coefficient or its nested program's
  // result; it enters exactly once, either as the addend that makes the
  // record's register live or as a final add when the record is visited.
  Operand own(std::uint32_t prog, std::uint32_t i, bool strict_walk = false) {
    const auto& rec = fp.rec(prog, i);
    if (rec.sub < 0) return coef(rec.coef);
    const auto sub = static_cast<std::uint32_t>(rec.sub);
    return strict_walk ? strict(sub) : fused(sub);
  }

  Operand fused(std::uint32_t prog) {
    const auto& P = fp.progs[prog];
    const std::uint32_t n = P.count;
    const auto parent = front::consumers(fp, prog);
    std::vector<Operand> m(P.regs);  // None == not live
    std::vector<char> folded(n, 0);
    for (std::uint32_t i = 0; i < n; ++i) {
      const auto& rec = fp.rec(prog, i);
      Operand val;
      if (rec.reads) {
        Operand acc = m[rec.lazy];
        m[rec.lazy] = Operand{};
        if (acc.is(Operand::None)) throw std::logic_error("fused lowering: dead register read");
        val = folded[i] ? acc : emit(OpKind::Add, acc, own(prog, i));
      } else {
        val = own(prog, i);
      }
      if (i + 1 == n) {
        if (rec.power >= 0) return emit(OpKind::Mul, val, power(prog, rec.power));
        return val;
      }
      const std::uint32_t j = parent[i];
      if (j == UINT32_MAX) throw std::logic_error("fused lowering: record without parent");
      Operand& cur = m[static_cast<std::uint32_t>(rec.parent)];
      if (rec.power >= 0) {
        const Operand Pw = power(prog, rec.power);
        if (cur.is(Operand::None)) {
          if (!folded[j]) {
            folded[j] = 1;
            const Operand addend = own(prog, j);
            cur = emit(OpKind::Fma, val, Pw, addend);
          } else {
            cur = emit(OpKind::Mul, val, Pw);
          }
        } else {
          cur = emit(OpKind::Fma, val, Pw, cur);
        }
      } else {
        if (cur.is(Operand::None)) {
          if (!folded[j]) {
            folded[j] = 1;
            const Operand addend = own(prog, j);
            if (fold_constants && val.is(Operand::Coef) && addend.is(Operand::Coef)) {
              // constant + constant: fold on the host (same IEEE/int result
              // the device add would produce)
              cur = coef(fold_add(s.coefs[val.id], s.coefs[addend.id]));
            } else {
              cur = emit(OpKind::Add, val, addend);
            }
          } else {
            cur = val;
          }
        } else {
          cur = emit(OpKind::Add, cur, val);
        }
      }
    }
    return Operand::zero();
  }

  static C fold_add(C a, C b) {
    if constexpr (std::is_same_v<C, std::int64_t>) {
      return static_cast<C>(static_cast<std::uint64_t>(a) + static_cast<std::uint64_t>(b));
    } else {
      return a + b;
    }
  }
};

}  // namespace

template <typename C>
Stream<C> lower_strict(const front::FlatProgram<C>& program) {
  Stream<C> s;
  s.strict = true;
  s.nvars = program.nvars;
  s.mirrorable = s.nvars == 1;
  const auto pow_of = build_powers(program, s);
  Lowerer<C> L{s, pow_of, program};
  s.result = L.strict(0);
  return s;
}

template <typename C>
bool mirror_stream(const Stream<C>& s, Stream<C>* out) {
  if (!s.strict || !s.mirrorable || s.odd.size() != s.coefs.size()) return false;
  *out = s;
  for (std::size_t k = 0; k < s.coefs.size(); ++k) {
    if (!s.odd[k]) continue;
    if constexpr (std::is_same_v<C, std::int64_t>) {
      if (s.coefs[k] == INT64_MIN) return false;
    }
    out->coefs[k] = -s.coefs[k];
  }
  return true;
}

namespace {
IntervalWord inject(double c) { return {c, c}; }
IntervalWord inject(std::int64_t c) {
  const double d = static_cast<double>(c);  // round-to-nearest-even
  const bool exact = d < 9223372036854775808.0 && d >= -9223372036854775808.0 &&
                     static_cast<std::int64_t>(d) == c;
  if (exact) return {d, d};
  return {std::nextafter(d, -std::numeric_limits<double>::infinity()),
          std::nextafter(d, std::numeric_limits<double>::infinity())};
}
}  // namespace

template <typename C>
IntervalWord interval_coefficient(const Stream<C>& s, std::size_t k) {
  IntervalWord c = inject(s.coefs[k]);
  const std::uint32_t w = k < s.widen.size() ? s.widen[k] : 0;
  for (std::uint32_t i = 0; i < w; ++i) {
    c.lo = std::nextafter(c.lo, -std::numeric_limits<double>::infinity());
    c.hi = std::nextafter(c.hi, std::numeric_limits<double>::infinity());
  }
  return c;
}

template IntervalWord interval_coefficient(const Stream<double>&, std::size_t);
template IntervalWord interval_coefficient(const Stream<std::int64_t>&, std::size_t);

template bool mirror_stream(const Stream<double>&, Stream<double>*);
template bool mirror_stream(const Stream<std::int64_t>&, Stream<std::int64_t>*);

template <typename C>
Stream<C> lower_fused(const front::FlatProgram<C>& program, bool fold_constants) {
  Stream<C> s;
  s.strict = false;
  s.nvars = program.nvars;
  const auto pow_of = build_powers(program, s);
  Lowerer<C> L{s, pow_of, program};
  L.fold_constants = fold_constants;
  s.result = L.fused(0);
  return s;
}

template Stream<double> lower_strict(const front::FlatProgram<double>&);
template Stream<std::int64_t> lower_strict(const front::FlatProgram<std::int64_t>&);
template Stream<double> lower_fused(const front::FlatProgram<double>&, bool);
template Stream<std::int64_t> lower_fused(const front::FlatProgram<std::int64_t>&, bool);

}  // namespace polyeval::lower
