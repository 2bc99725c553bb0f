// Tree -> flat CompiledProgram (the reference's back-end compiler).
//
// Mirrors reference proj/core/include/polyeval/eval.hpp:32-57 (record layout)
// and proj/core/src/eval.cpp:8-69 (collect_exponents / compile_tree /
// compile), plus ExponentSet from powers.hpp:16-26 / powers.cpp:7-21.
// Records are in topological order with the root last; exponent sets are
// unioned per variable over nested programs and stored on the root program.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <optional>
#include <set>
#include <vector>

#include "front/tree.hpp"

namespace polyeval {

/// Sorted, deduplicated exponents >= 1 (reference powers.cpp:7-21).
struct ExponentSet {
  std::vector<std::uint32_t> exponents;

  static ExponentSet from_values(std::vector<std::uint32_t> values) {
    std::erase(values, 0u);
    std::sort(values.begin(), values.end());
    values.erase(std::unique(values.begin(), values.end()), values.end());
    return ExponentSet{std::move(values)};
  }
  bool empty() const noexcept { return exponents.empty(); }
  std::size_t size() const noexcept { return exponents.size(); }
  std::optional<std::size_t> index_of(std::uint32_t e) const noexcept {
    auto it = std::lower_bound(exponents.begin(), exponents.end(), e);
    if (it == exponents.end() || *it != e) return std::nullopt;
    return static_cast<std::size_t>(it - exponents.begin());
  }
};

template <typename C>
struct CompiledProgram {
  struct Record {
    C coeff{};
    std::unique_ptr<CompiledProgram> sub;  // nested coefficient program
    std::optional<std::uint32_t> power_slot;
    std::uint32_t lazy_slot = 0;
    std::optional<std::uint32_t> parent_slot;
    bool reads_register = false;
  };

  std::vector<Record> records;
  std::uint32_t register_count = 1;
  std::size_t variable = 0;
  std::vector<std::uint32_t> root_child_ends;

  // Root program only.
  std::size_t variable_count = 0;
  std::vector<ExponentSet> exponent_sets;  // indexed by variable
};

namespace detail {

template <typename C>
void collect_exponents(const EvaluationTree<C>& tree,
                       std::vector<std::set<std::uint32_t>>& per_variable) {
  auto& bucket = per_variable[tree.variable];
  for (const auto& node : tree.nodes) {
    if (node.partial_degree != 0) bucket.insert(node.partial_degree);
    if (node.has_sub()) collect_exponents(*node.sub_coeff, per_variable);
  }
}

template <typename C>
CompiledProgram<C> compile_tree(const EvaluationTree<C>& tree,
                                const std::vector<ExponentSet>& sets) {
  CompiledProgram<C> out;
  out.variable = tree.variable;
  out.records.reserve(tree.nodes.size());
  std::uint32_t max_lazy = 0;
  for (const auto& node : tree.nodes) {
    typename CompiledProgram<C>::Record rec;
    if (node.has_sub()) {
      rec.sub = std::make_unique<CompiledProgram<C>>(compile_tree(*node.sub_coeff, sets));
    } else {
      rec.coeff = node.coeff;
    }
    if (node.partial_degree != 0) {
      rec.power_slot = static_cast<std::uint32_t>(
          *sets[tree.variable].index_of(node.partial_degree));
    }
    rec.lazy_slot = node.lazy_height;
    if (node.parent) rec.parent_slot = tree.nodes[*node.parent].lazy_height;
    rec.reads_register = !node.children.empty();
    max_lazy = std::max(max_lazy, node.lazy_height);
    out.records.push_back(std::move(rec));
  }
  out.register_count = max_lazy + 1;
  out.root_child_ends = tree.root().children;
  std::sort(out.root_child_ends.begin(), out.root_child_ends.end());
  return out;
}

}  // namespace detail

/// Compiles an annotated tree (lazy heights computed) into a flat program
/// (reference eval.cpp:52-69).
template <typename C>
CompiledProgram<C> compile(const EvaluationTree<C>& tree) {
  const std::size_t nvars = std::max(tree.variables.size(), tree.variable + 1);
  std::vector<std::set<std::uint32_t>> gathered(nvars);
  detail::collect_exponents(tree, gathered);
  std::vector<ExponentSet> sets;
  sets.reserve(nvars);
  for (const auto& b : gathered) {
    sets.push_back(ExponentSet::from_values(std::vector<std::uint32_t>(b.begin(), b.end())));
  }
  CompiledProgram<C> out = detail::compile_tree(tree, sets);
  out.variable_count = tree.variables.size();
  out.exponent_sets = std::move(sets);
  return out;
}

/// Walk statistics pinned by the reference op-count identities
/// (eval_test.cpp:182-216): adds = (records-1) + #records_with_children,
/// muls = #records_with_power, summed over nested programs.
struct ProgramStats {
  std::uint64_t records = 0;
  std::uint64_t programs = 0;
  std::uint64_t walk_adds = 0;
  std::uint64_t walk_muls = 0;
  std::uint64_t power_muls = 0;  // memoized-halving table build, all variables
  std::uint32_t max_registers = 0;
};

template <typename C>
void accumulate_stats(const CompiledProgram<C>& p, ProgramStats& s) {
  s.programs += 1;
  s.max_registers = std::max(s.max_registers, p.register_count);
  for (std::size_t i = 0; i < p.records.size(); ++i) {
    const auto& r = p.records[i];
    s.records += 1;
    if (i + 1 != p.records.size()) s.walk_adds += 1;
    if (r.reads_register) s.walk_adds += 1;
    if (r.power_slot) s.walk_muls += 1;
    if (r.sub) accumulate_stats(*r.sub, s);
  }
}

/// Number of multiplications memoized halving performs for one exponent set
/// (reference powers.hpp:50-72: x^e = x^(e/2) * x^(e - e/2), x^1 free).
inline std::uint64_t power_table_muls(const ExponentSet& set) {
  std::set<std::uint32_t> memo{1};
  std::uint64_t muls = 0;
  std::vector<std::uint32_t> stack;
  for (std::uint32_t e : set.exponents) {
    // iterative post-order of ensure(e)
    stack.push_back(e);
    while (!stack.empty()) {
      const std::uint32_t top = stack.back();
      if (memo.count(top)) {
        stack.pop_back();
        continue;
      }
      const std::uint32_t h = top / 2, r = top - top / 2;
      const bool hv = memo.count(h) != 0, rv = memo.count(r) != 0;
      if (hv && rv) {
        memo.insert(top);
        ++muls;
        stack.pop_back();
      } else {
        if (!hv) stack.push_back(h);
        if (!rv && r != h) stack.push_back(r);
      }
    }
  }
  return muls;
}

template <typename C>
ProgramStats program_stats(const CompiledProgram<C>& p) {
  ProgramStats s;
  accumulate_stats(p, s);
  for (const auto& set : p.exponent_sets) s.power_muls += power_table_muls(set);
  return s;
}

}  // namespace polyeval
