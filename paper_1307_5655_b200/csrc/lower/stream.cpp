// Lowering of a CompiledProgram into a straight-line register stream.
// See stream.hpp for the contract; reference walk: eval.hpp:208-249,
// power tables: powers.hpp:50-72.
#include "lower/stream.hpp"

#include <cstdint>
#include <map>
#include <stdexcept>

namespace polyeval::lower {
namespace {

// Builds the per-variable power DAG by memoized halving, in the reference's
// recursion order (ensure(e) -> ensure(e/2), ensure(e - e/2), then multiply;
// powers.hpp:58-66), and returns [var][slot] -> power id.
template <typename C>
std::vector<std::vector<std::uint32_t>> build_powers(const CompiledProgram<C>& prog,
                                                     Stream<C>& s) {
  std::vector<std::vector<std::uint32_t>> slot_to_power(prog.exponent_sets.size());
  for (std::size_t v = 0; v < prog.exponent_sets.size(); ++v) {
    const ExponentSet& set = prog.exponent_sets[v];
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
    for (std::uint32_t e : set.exponents) {
      ensure(e);
      slot_to_power[v].push_back(memo.at(e));
    }
  }
  return slot_to_power;
}

// For record i, the index of its parent record: the first later record that
// reads the register i accumulates into (register discipline of the lazy
// heights, reference tree.hpp:68-77).
template <typename C>
std::vector<std::uint32_t> parent_records(const CompiledProgram<C>& p) {
  const std::size_t n = p.records.size();
  std::vector<std::uint32_t> parent(n, UINT32_MAX);
  std::vector<std::uint32_t> next_reader(p.register_count, UINT32_MAX);
  for (std::size_t i = n; i-- > 0;) {
    const auto& r = p.records[i];
    if (r.parent_slot) parent[i] = next_reader[*r.parent_slot];
    if (r.reads_register) next_reader[r.lazy_slot] = static_cast<std::uint32_t>(i);
  }
  return parent;
}

template <typename C>
struct Lowerer {
  Stream<C>& s;
  const std::vector<std::vector<std::uint32_t>>& pow_of;

  std::uint8_t cur_odd = 0;  // strict: parity of the record being lowered

  Operand new_reg() { return Operand::reg(s.nregs++); }
  Operand coef(const C& c, std::uint32_t widen = 0) {
    s.coefs.push_back(c);
    s.widen.push_back(widen);
    s.odd.push_back(cur_odd);
    return Operand::coef(static_cast<std::uint32_t>(s.coefs.size() - 1));
  }
  Operand power(const CompiledProgram<C>& p, std::uint32_t slot) {
    return Operand::pow(pow_of.at(p.variable).at(slot));
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
  Operand strict(const CompiledProgram<C>& p) {
    std::vector<Operand> m(p.register_count, Operand::zero());
    const std::size_t last = p.records.size() - 1;
    // parity of each record's absolute exponent: its own power plus its
    // ancestors' (a record's value is added into the register its parent
    // reads and multiplies by the parent's power)
    std::vector<std::uint8_t> par(p.records.size(), 0);
    if (s.mirrorable && !p.records.empty()) {  // univariate only
      const auto parent = parent_records(p);
      for (std::size_t i = p.records.size(); i-- > 0;) {
        const auto& rec = p.records[i];
        std::uint32_t d = 0;
        if (rec.power_slot) d = p.exponent_sets.at(p.variable).exponents.at(*rec.power_slot);
        const std::uint8_t up = parent[i] == UINT32_MAX ? 0 : par[parent[i]];
        par[i] = static_cast<std::uint8_t>((d + up) & 1u);
        if (rec.sub) s.mirrorable = false;
      }
    }
    for (std::size_t i = 0; i <= last; ++i) {
      const auto& rec = p.records[i];
      cur_odd = par[i];
      Operand v = rec.sub ? strict(*rec.sub) : coef(rec.coeff);  // L224
      if (rec.reads_register) {                                   // L225-228
        v = emit(OpKind::Add, m[rec.lazy_slot], v);
        m[rec.lazy_slot] = Operand::zero();
      }
      if (rec.power_slot) v = emit(OpKind::Mul, v, power(p, *rec.power_slot));  // L229-232
      if (i == last) return v;                                    // L233-236
      Operand& slot = m[*rec.parent_slot];                        // L237-238
      slot = emit(OpKind::Add, slot, v);
    }
    return Operand::zero();
  }

  // ---- fused: one FMA per powered record, coefficient folded as addend ----
  // A record's "own" value is its scalar coefficient or its nested program's
  // result; it enters exactly once, either as the addend that makes the
  // record's register live or as a final add when the record is visited.
  Operand own(const CompiledProgram<C>& p, std::size_t i) {
    const auto& rec = p.records[i];
    return rec.sub ? fused(*rec.sub) : coef(rec.coeff);
  }

  Operand fused(const CompiledProgram<C>& p) {
    const std::size_t n = p.records.size();
    const auto parent = parent_records(p);
    std::vector<Operand> m(p.register_count);  // None == not live
    std::vector<char> folded(n, 0);
    for (std::size_t i = 0; i < n; ++i) {
      const auto& rec = p.records[i];
      Operand val;
      if (rec.reads_register) {
        Operand acc = m[rec.lazy_slot];
        m[rec.lazy_slot] = Operand{};
        if (acc.is(Operand::None)) throw std::logic_error("fused lowering: dead register read");
        val = folded[i] ? acc : emit(OpKind::Add, acc, own(p, i));
      } else {
        val = own(p, i);
      }
      if (i + 1 == n) {
        if (rec.power_slot) return emit(OpKind::Mul, val, power(p, *rec.power_slot));
        return val;
      }
      const std::uint32_t j = parent[i];
      if (j == UINT32_MAX) throw std::logic_error("fused lowering: record without parent");
      Operand& cur = m[*rec.parent_slot];
      if (rec.power_slot) {
        const Operand P = power(p, *rec.power_slot);
        if (cur.is(Operand::None)) {
          if (!folded[j]) {
            folded[j] = 1;
            const Operand addend = own(p, j);
            cur = emit(OpKind::Fma, val, P, addend);
          } else {
            cur = emit(OpKind::Mul, val, P);
          }
        } else {
          cur = emit(OpKind::Fma, val, P, cur);
        }
      } else {
        if (cur.is(Operand::None)) {
          if (!folded[j]) {
            folded[j] = 1;
            const Operand addend = own(p, j);
            if (val.is(Operand::Coef) && addend.is(Operand::Coef)) {
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
Stream<C> lower_strict(const CompiledProgram<C>& program) {
  Stream<C> s;
  s.strict = true;
  s.nvars = static_cast<std::uint32_t>(program.variable_count);
  s.mirrorable = s.nvars == 1;
  const auto pow_of = build_powers(program, s);
  Lowerer<C> L{s, pow_of};
  s.result = L.strict(program);
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

template bool mirror_stream(const Stream<double>&, Stream<double>*);
template bool mirror_stream(const Stream<std::int64_t>&, Stream<std::int64_t>*);

template <typename C>
Stream<C> lower_fused(const CompiledProgram<C>& program) {
  Stream<C> s;
  s.strict = false;
  s.nvars = static_cast<std::uint32_t>(program.variable_count);
  const auto pow_of = build_powers(program, s);
  Lowerer<C> L{s, pow_of};
  s.result = L.fused(program);
  return s;
}

template Stream<double> lower_strict(const CompiledProgram<double>&);
template Stream<std::int64_t> lower_strict(const CompiledProgram<std::int64_t>&);
template Stream<double> lower_fused(const CompiledProgram<double>&);
template Stream<std::int64_t> lower_fused(const CompiledProgram<std::int64_t>&);

}  // namespace polyeval::lower
