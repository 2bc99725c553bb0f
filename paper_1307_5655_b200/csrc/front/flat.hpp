// FlatProgram: the compiled record walk of one polynomial, every program
// (root and nested coefficient programs) in one arena.
//
// Record semantics are the reference's CompiledProgram::Record
// (proj/core/include/polyeval/eval.hpp:32-54) — the walk contract of
// Evaluator::run_range (eval.hpp:218-249):
//   v = (reads ? m[lazy] : 0) + (sub >= 0 ? program sub at the point : coef)
//   m[lazy] = 0 if read;  v *= x_var^exponent_sets[var][power] if power >= 0
//   m[parent] += v, except the program's last record, which yields v.
// The layout is the C ABI's flattened form (pe_compiled_program / pe_record:
// programs by index, records contiguous per program), so a program imported
// from the reference (pe_program_from_compiled) and one built here
// (front/forest.hpp) are the same object.
#pragma once

#include <algorithm>
#include <cstdint>
#include <set>
#include <vector>

namespace polyeval::front {

template <typename C>
struct FlatProgram {
  struct Rec {
    C coef{};
    std::int32_t sub = -1;     // nested program index, or -1 (scalar coef)
    std::int32_t power = -1;   // index into exponent_sets[var of the program]
    std::uint32_t lazy = 0;    // register read (when `reads`)
    std::int32_t parent = -1;  // register accumulated into; -1 for the last record
    bool reads = false;
  };
  struct Prog {
    std::uint32_t var = 0;
    std::uint32_t regs = 1;               // register file size
    std::uint32_t first = 0, count = 0;   // records [first, first + count)
    std::vector<std::uint32_t> root_child_ends;  // ascending, program-local
  };

  std::uint32_t nvars = 0;
  std::vector<Prog> progs;  // [0] is the root program
  std::vector<Rec> recs;
  std::vector<std::vector<std::uint32_t>> exponent_sets;  // per variable, ascending, >= 1

  const Rec& rec(std::uint32_t prog, std::uint32_t i) const { return recs[progs[prog].first + i]; }
  std::uint32_t exponent(std::uint32_t prog, std::int32_t power) const {
    return exponent_sets[progs[prog].var][static_cast<std::uint32_t>(power)];
  }
};

/// Per-point walk statistics (reference op-count identities,
/// proj/tests/eval_test.cpp:182-216): adds = (records - 1) + #reads and
/// muls = #powered records, per program, summed; plus the memoized-halving
/// multiplications of the power tables.
struct WalkStats {
  std::uint64_t records = 0;
  std::uint64_t programs = 0;
  std::uint64_t walk_adds = 0;
  std::uint64_t walk_muls = 0;
  std::uint64_t power_muls = 0;
  std::uint32_t max_registers = 0;
};

/// Multiplications memoized halving spends on one exponent set
/// (x^e = x^(e/2) * x^(e - e/2), x^1 free; reference powers.hpp:50-72):
/// one per distinct exponent > 1 reachable from the set by halving.
inline std::uint64_t halving_muls(const std::vector<std::uint32_t>& set) {
  std::set<std::uint32_t> seen;
  std::vector<std::uint32_t> todo(set.begin(), set.end());
  while (!todo.empty()) {
    const std::uint32_t e = todo.back();
    todo.pop_back();
    if (e <= 1 || !seen.insert(e).second) continue;
    todo.push_back(e / 2);
    todo.push_back(e - e / 2);
  }
  return seen.size();
}

template <typename C>
WalkStats walk_stats(const FlatProgram<C>& fp) {
  WalkStats s;
  s.programs = fp.progs.size();
  for (const auto& p : fp.progs) {
    s.max_registers = std::max(s.max_registers, p.regs);
    s.records += p.count;
    s.walk_adds += p.count ? p.count - 1 : 0;
    for (std::uint32_t i = 0; i < p.count; ++i) {
      const auto& r = fp.recs[p.first + i];
      s.walk_adds += r.reads ? 1 : 0;
      s.walk_muls += r.power >= 0 ? 1 : 0;
    }
  }
  for (const auto& set : fp.exponent_sets) s.power_muls += halving_muls(set);
  return s;
}

/// For each record of program `prog`, the program-local index of the record
/// that consumes its value (the next record reading the register it
/// accumulates into), or UINT32_MAX for the last record.
template <typename C>
std::vector<std::uint32_t> consumers(const FlatProgram<C>& fp, std::uint32_t prog) {
  const auto& p = fp.progs[prog];
  std::vector<std::uint32_t> out(p.count, UINT32_MAX);
  std::vector<std::uint32_t> reader(p.regs, UINT32_MAX);
  for (std::uint32_t i = p.count; i-- > 0;) {
    const auto& r = fp.recs[p.first + i];
    if (r.parent >= 0) out[i] = reader[static_cast<std::uint32_t>(r.parent)];
    if (r.reads) reader[r.lazy] = i;
  }
  return out;
}

}  // namespace polyeval::front
