// Walk VM programs: see vm.hpp.
#include "lower/vm.hpp"

#include <cstring>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace polyeval::lower {
namespace {

std::uint64_t bits(double d) {
  std::uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

}  // namespace

template <typename C>
VmProgram build_vm(const Stream<C>& s, Domain d, bool distinct_dst) {
  if (d == Domain::I64K) throw std::invalid_argument("the walk VM has no K-limb domain");
  if ((d == Domain::F64Strict || d == Domain::Interval) && !s.strict) {
    throw std::logic_error("strict domain needs a strict stream");
  }
  VmProgram vm;
  vm.domain = d;
  vm.nvars = s.nvars;
  // values: coordinates [0, nvars), powers [nvars, nvars + P), registers
  // after; an exponent-1 power is its coordinate
  const std::uint32_t P = static_cast<std::uint32_t>(s.powers.size());
  const std::uint32_t base_reg = s.nvars + P;
  auto value_of = [&](const Operand& o) -> std::int64_t {
    switch (o.kind) {
      case Operand::Reg: return base_reg + o.id;
      case Operand::Pow:
        return s.powers[o.id].exponent == 1 ? s.powers[o.id].var : s.nvars + o.id;
      default: return -1;
    }
  };
  // the schedule: power products, then the walk
  struct VOp {
    std::uint32_t kind, dst;
    std::int64_t in[3];
    Operand src[3];
  };
  std::vector<VOp> ops;
  for (std::uint32_t p = 0; p < P; ++p) {
    const Power& pw = s.powers[p];
    if (pw.exponent == 1) continue;
    const Operand lo = Operand::pow(pw.lo), hi = Operand::pow(pw.hi);
    ops.push_back({1, s.nvars + p, {value_of(lo), value_of(hi), -1}, {lo, hi, {}}});
  }
  for (const Op& op : s.ops) {
    const std::uint32_t kind = op.kind == OpKind::Add ? 0 : op.kind == OpKind::Mul ? 1 : 2;
    ops.push_back({kind, base_reg + op.dst, {value_of(op.a), value_of(op.b), value_of(op.c)},
                   {op.a, op.b, op.c}});
  }
  // live ranges: last read of every value (the result is read after the end)
  const std::size_t nval = base_reg + s.nregs;
  std::vector<std::int64_t> last(nval, -1);
  for (std::size_t i = 0; i < ops.size(); ++i) {
    for (std::int64_t v : ops[i].in) {
      if (v >= 0) last[static_cast<std::size_t>(v)] = static_cast<std::int64_t>(i);
    }
  }
  const std::int64_t rv = value_of(s.result);
  if (rv >= 0) last[static_cast<std::size_t>(rv)] = static_cast<std::int64_t>(ops.size());
  // linear scan: coordinates sit in slots 0..nvars-1; a slot is released
  // after the op that reads its value for the last time (an op may write the
  // slot it frees: operands are read before the destination is written)
  std::vector<std::int64_t> slot_of(nval, -1);
  std::vector<std::uint32_t> free_slots;
  std::uint32_t top = s.nvars;
  for (std::uint32_t v = 0; v < s.nvars; ++v) slot_of[v] = v;
  auto operand = [&](const Operand& o, std::int64_t v) -> std::uint32_t {
    if (o.is(Operand::Coef)) return VmProgram::kCoef | o.id;
    if (o.is(Operand::Zero) || o.is(Operand::None)) return VmProgram::kZero;
    if (v < 0 || slot_of[static_cast<std::size_t>(v)] < 0) throw std::logic_error("VM: value read before written");
    return static_cast<std::uint32_t>(slot_of[static_cast<std::size_t>(v)]);
  };
  for (std::size_t i = 0; i < ops.size(); ++i) {
    const VOp& op = ops[i];
    std::uint32_t enc[3];
    for (int k = 0; k < 3; ++k) enc[k] = operand(op.src[k], op.in[k]);
    std::vector<std::uint32_t> released;
    for (int k = 0; k < 3; ++k) {  // release values read here for the last time
      const std::int64_t v = op.in[k];
      if (v >= 0 && last[static_cast<std::size_t>(v)] == static_cast<std::int64_t>(i) &&
          slot_of[static_cast<std::size_t>(v)] >= 0) {
        released.push_back(static_cast<std::uint32_t>(slot_of[static_cast<std::size_t>(v)]));
        slot_of[static_cast<std::size_t>(v)] = -1;
      }
    }
    if (!distinct_dst) free_slots.insert(free_slots.end(), released.begin(), released.end());
    std::uint32_t dst;
    if (last[op.dst] < 0) {
      dst = top;  // dead value (never read): any scratch slot
    } else if (!free_slots.empty()) {
      dst = free_slots.back();
      free_slots.pop_back();
    } else {
      dst = top++;
    }
    if (last[op.dst] >= 0) slot_of[op.dst] = dst;
    if (dst >= top) top = dst + 1;
    if (distinct_dst) free_slots.insert(free_slots.end(), released.begin(), released.end());
    vm.code.insert(vm.code.end(), {op.kind, dst, enc[0], enc[1], enc[2]});
  }
  vm.nops = static_cast<std::uint32_t>(ops.size());
  vm.result = s.result.is(Operand::Coef)   ? (VmProgram::kCoef | s.result.id)
              : s.result.is(Operand::Zero) ? VmProgram::kZero
                                           : static_cast<std::uint32_t>(slot_of[static_cast<std::size_t>(rv)]);
  vm.nslots = std::max<std::uint32_t>(top, 1);
  // coefficient words in the domain's format
  for (std::size_t k = 0; k < s.coefs.size(); ++k) {
    if (d == Domain::Interval) {
      const IntervalWord w = interval_coefficient(s, k);
      vm.lo.push_back(bits(w.lo));
      vm.hi.push_back(bits(w.hi));
    } else if (d == Domain::I64) {
      if constexpr (std::is_same_v<C, std::int64_t>) {
        vm.lo.push_back(static_cast<std::uint64_t>(s.coefs[k]));
      } else {
        throw std::invalid_argument("int64 domain needs integer coefficients");
      }
    } else {
      vm.lo.push_back(bits(static_cast<double>(s.coefs[k])));
    }
  }
  return vm;
}

template VmProgram build_vm(const Stream<double>&, Domain, bool);
template VmProgram build_vm(const Stream<std::int64_t>&, Domain, bool);

}  // namespace polyeval::lower
