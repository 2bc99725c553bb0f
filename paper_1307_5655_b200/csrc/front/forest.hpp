// Evaluation trees (paper Def. 1) over a canonical term table, built without
// recursion, plus lazy heights, the DOT rendering and compilation to a
// FlatProgram.
//
// Shape facts the builder relies on (they pin it to the reference's
// proj/core/src/tree.cpp:30-227 output, checked record for record against
// the unmodified reference in tests/test_front.py):
//  * Multivariate nesting (paper Remark 1) partitions the canonical table
//    into contiguous runs: inside a run that shares exponents 0..d-1, rows are
//    ordered by exponent d first, so the coefficient polynomial of x_d^a is a
//    contiguous sub-run, already canonical. A run that is one row with zero
//    exponents beyond d is a scalar; anything else is a nested tree in x_{d+1}.
//  * A tree's nodes are its distinct exponents E_0 > E_1 > ... in table order.
//    The scheme cuts a range [f, l) with base exponent s at s + f(E_f - s):
//    rows at or above the cut form the upper range (base s + f(.)), the rest
//    the lower range (same base); the root of a range is always its last
//    node, so every cut makes node (cut - 1) a child of node (l - 1). An
//    empty lower range only raises the base (the zero remainder, D5).
//  * Every node's full degree is its exponent, so partial degrees are
//    E_i - E_parent(i) (the root: E_root), and children appear in increasing
//    node index.
//  * Lazy heights (D2): a node with <= 1 child has height 0, otherwise
//    1 + the largest register usage among children 2..k; usage(i) =
//    max(height(i), usage(first child)).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "front/flat.hpp"
#include "front/split.hpp"
#include "front/terms.hpp"

namespace polyeval::front {

template <typename C>
struct Forest {
  struct Node {
    C coef{};
    std::int32_t sub = -1;      // nested tree index
    std::uint32_t exponent = 0; // absolute exponent in the tree's variable
    std::uint32_t pdeg = 0;     // partial degree
    std::int32_t parent = -1;   // tree-local node index
    std::uint32_t lazy = 0;
    std::uint32_t kids = 0, kid_first = 0;  // children in `kid_index`
  };
  struct Tree {
    std::uint32_t var = 0;
    std::uint32_t first = 0, count = 0;   // nodes [first, first + count)
    std::uint32_t row_lo = 0, row_hi = 0; // terms of the table it evaluates
  };

  const TermTable<C>* table = nullptr;
  std::vector<Tree> trees;  // [0] is the root tree
  std::vector<Node> nodes;
  std::vector<std::uint32_t> kid_index;  // tree-local child indices, grouped per node

  const Node& node(std::uint32_t t, std::uint32_t i) const { return nodes[trees[t].first + i]; }
  std::span<const std::uint32_t> children(std::uint32_t t, std::uint32_t i) const {
    const Node& n = node(t, i);
    return {kid_index.data() + n.kid_first, n.kids};
  }
};

namespace detail {

/// Parent links of one tree's nodes from its exponents (see the file header).
inline void link_tree(const std::vector<std::uint32_t>& E, const SplitRule& rule,
                      std::vector<std::int32_t>& parent) {
  struct Range {
    std::uint32_t f, l;
    std::uint64_t base;
  };
  const auto m = static_cast<std::uint32_t>(E.size());
  parent.assign(m, -1);
  std::vector<Range> work{{0, m, 0}};
  while (!work.empty()) {
    Range r = work.back();
    work.pop_back();
    const std::uint32_t root = r.l - 1;
    while (r.l - r.f > 1) {
      const std::uint64_t k = E[r.f] - r.base;
      const std::uint64_t s = rule(k);
      if (s < 1 || s > k) {
        throw std::invalid_argument("function scheme " + rule.name() + " gave " + std::to_string(s) +
                                    " for degree " + std::to_string(k) +
                                    " (a scheme split must lie in (0, k])");
      }
      const std::uint64_t cut = r.base + s;
      // first node of [f, l) whose exponent is below the cut (E descending)
      const auto it = std::partition_point(E.begin() + r.f, E.begin() + r.l,
                                           [cut](std::uint32_t e) { return e >= cut; });
      const auto mid = static_cast<std::uint32_t>(it - E.begin());
      if (mid == r.l) {  // nothing below the cut: only the base moves
        r.base = cut;
        continue;
      }
      parent[mid - 1] = static_cast<std::int32_t>(root);
      work.push_back({r.f, mid, cut});
      r.f = mid;
    }
  }
}

inline std::string coef_text(std::int64_t c) { return std::to_string(c); }
inline std::string coef_text(double c) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", c);
  return buf;
}

}  // namespace detail

/// Builds the forest of `table` with one rule per variable. The zero
/// polynomial is one node with coefficient 0.
template <typename C>
Forest<C> build_forest(const TermTable<C>& table, std::span<const SplitRule> rules) {
  if (rules.size() != table.nvars) throw std::invalid_argument("need exactly one scheme per variable");
  for (const auto& r : rules) r.check();
  Forest<C> F;
  F.table = &table;
  struct Job {
    std::uint32_t depth, lo, hi;
    std::int32_t owner;  // global node index that references the tree, or -1
  };
  std::vector<Job> jobs{{0, 0, static_cast<std::uint32_t>(table.size()), -1}};
  std::vector<std::uint32_t> E;
  std::vector<std::int32_t> parent;
  while (!jobs.empty()) {
    const Job job = jobs.back();
    jobs.pop_back();
    const auto t = static_cast<std::uint32_t>(F.trees.size());
    typename Forest<C>::Tree tree;
    tree.var = job.depth;
    tree.first = static_cast<std::uint32_t>(F.nodes.size());
    tree.row_lo = job.lo;
    tree.row_hi = job.hi;
    if (job.owner >= 0) F.nodes[static_cast<std::size_t>(job.owner)].sub = static_cast<std::int32_t>(t);
    // one node per run of equal exponent `depth`
    E.clear();
    std::vector<std::uint32_t> run_start;
    for (std::uint32_t r = job.lo; r < job.hi; ++r) {
      const std::uint32_t e = table.exp(r, job.depth);
      if (E.empty() || e != E.back()) {
        E.push_back(e);
        run_start.push_back(r);
      }
    }
    run_start.push_back(job.hi);
    if (E.empty()) {  // zero polynomial
      F.nodes.emplace_back();
      tree.count = 1;
      F.trees.push_back(tree);
      continue;
    }
    tree.count = static_cast<std::uint32_t>(E.size());
    detail::link_tree(E, rules[job.depth], parent);
    for (std::uint32_t k = 0; k < tree.count; ++k) {
      typename Forest<C>::Node nd;
      nd.exponent = E[k];
      nd.parent = parent[k];
      nd.pdeg = parent[k] < 0 ? E[k] : E[k] - E[static_cast<std::size_t>(parent[k])];
      const std::uint32_t lo = run_start[k], hi = run_start[k + 1];
      const std::uint32_t* row = table.row(lo);
      const bool scalar = hi - lo == 1 &&
                          std::all_of(row + job.depth + 1, row + table.nvars,
                                      [](std::uint32_t e) { return e == 0; });
      if (scalar) {
        nd.coef = table.coefs[lo];
      } else {
        if (job.depth + 1 >= table.nvars) throw std::logic_error("variables exhausted while nesting");
        jobs.push_back({job.depth + 1, lo, hi, static_cast<std::int32_t>(F.nodes.size())});
      }
      F.nodes.push_back(nd);
    }
    F.trees.push_back(tree);
  }
  // children lists (increasing index) and lazy heights, tree by tree
  F.kid_index.reserve(F.nodes.size());
  for (auto& tree : F.trees) {
    auto* nd = F.nodes.data() + tree.first;
    std::vector<std::uint32_t> cnt(tree.count + 1, 0);
    for (std::uint32_t i = 0; i < tree.count; ++i) {
      if (nd[i].parent >= 0) ++cnt[static_cast<std::uint32_t>(nd[i].parent)];
    }
    const auto base = static_cast<std::uint32_t>(F.kid_index.size());
    std::uint32_t at = base;
    for (std::uint32_t i = 0; i < tree.count; ++i) {
      nd[i].kid_first = at;
      nd[i].kids = 0;
      at += cnt[i];
    }
    F.kid_index.resize(at);
    for (std::uint32_t i = 0; i < tree.count; ++i) {
      if (nd[i].parent < 0) continue;
      auto& p = nd[static_cast<std::uint32_t>(nd[i].parent)];
      F.kid_index[p.kid_first + p.kids++] = i;
    }
    std::vector<std::uint32_t> usage(tree.count, 0);
    for (std::uint32_t i = 0; i < tree.count; ++i) {
      const std::uint32_t* kid = F.kid_index.data() + nd[i].kid_first;
      std::uint32_t h = 0;
      if (nd[i].kids > 1) {
        for (std::uint32_t c = 1; c < nd[i].kids; ++c) h = std::max(h, usage[kid[c]]);
        h += 1;
      }
      nd[i].lazy = h;
      usage[i] = nd[i].kids ? std::max(h, usage[kid[0]]) : h;
    }
  }
  return F;
}

/// Flattens the forest: tree t becomes program t, node k record k; power
/// slots index the per-variable union of the nonzero partial degrees.
template <typename C>
FlatProgram<C> compile_forest(const Forest<C>& F) {
  FlatProgram<C> fp;
  fp.nvars = F.table->nvars;
  fp.exponent_sets.assign(std::max<std::uint32_t>(fp.nvars, 1), {});
  for (const auto& tree : F.trees) {
    for (std::uint32_t i = 0; i < tree.count; ++i) {
      const auto& nd = F.nodes[tree.first + i];
      if (nd.pdeg) fp.exponent_sets[tree.var].push_back(nd.pdeg);
    }
  }
  for (auto& set : fp.exponent_sets) {
    std::sort(set.begin(), set.end());
    set.erase(std::unique(set.begin(), set.end()), set.end());
  }
  fp.recs.reserve(F.nodes.size());
  for (std::uint32_t t = 0; t < F.trees.size(); ++t) {
    const auto& tree = F.trees[t];
    typename FlatProgram<C>::Prog prog;
    prog.var = tree.var;
    prog.first = static_cast<std::uint32_t>(fp.recs.size());
    prog.count = tree.count;
    std::uint32_t top = 0;
    const auto& set = fp.exponent_sets[tree.var];
    for (std::uint32_t i = 0; i < tree.count; ++i) {
      const auto& nd = F.nodes[tree.first + i];
      typename FlatProgram<C>::Rec r;
      r.coef = nd.coef;
      r.sub = nd.sub;
      if (nd.pdeg) {
        r.power = static_cast<std::int32_t>(std::lower_bound(set.begin(), set.end(), nd.pdeg) - set.begin());
      }
      r.lazy = nd.lazy;
      r.reads = nd.kids > 0;
      if (nd.parent >= 0) r.parent = static_cast<std::int32_t>(F.nodes[tree.first + static_cast<std::uint32_t>(nd.parent)].lazy);
      top = std::max(top, nd.lazy);
      fp.recs.push_back(r);
    }
    prog.regs = top + 1;
    const auto root_kids = F.children(t, tree.count - 1);
    prog.root_child_ends.assign(root_kids.begin(), root_kids.end());
    fp.progs.push_back(std::move(prog));
  }
  return fp;
}

/// Text of the term rows [lo, hi) over the variables from `from_var` on, in
/// the reference's polynomial syntax (sign-separated monomials, coefficient
/// 1 elided before factors, x^e for e > 1; proj/core/src/parser.cpp:291-322).
/// A nested tree's rows still carry the outer exponents; they are skipped.
template <typename C>
std::string terms_text(const TermTable<C>& T, std::uint32_t lo, std::uint32_t hi,
                       std::uint32_t from_var, std::span<const std::string> names) {
  if (lo == hi) return "0";
  std::string s;
  for (std::uint32_t r = lo; r < hi; ++r) {
    const C c = T.coefs[r];
    const bool neg = c < C{};
    std::string mag = detail::coef_text(c);
    if (neg) {
      s += '-';
      mag.erase(0, 1);
    } else if (r != lo) {
      s += '+';
    }
    const std::uint32_t* e = T.row(r);
    const bool bare = std::all_of(e + from_var, e + T.nvars, [](std::uint32_t x) { return x == 0; });
    bool sep = false;
    if (bare || !(c == C{1} || c == C{-1})) {
      s += mag;
      sep = true;
    }
    for (std::uint32_t v = from_var; v < T.nvars; ++v) {
      if (!e[v]) continue;
      if (sep) s += '*';
      s += names[v];
      if (e[v] > 1) s += '^' + std::to_string(e[v]);
      sep = true;
    }
  }
  return s;
}

/// DOT digraph of the root tree: node labels "c=<coef or nested polynomial>
/// d=<partial degree> lh=<lazy height>", then the edges parent -> child
/// (reference to_dot, tree.cpp:290-309).
template <typename C>
std::string forest_dot(const Forest<C>& F, std::span<const std::string> names) {
  std::ostringstream os;
  os << "digraph evaluation_tree {\n";
  const auto& root = F.trees[0];
  for (std::uint32_t i = 0; i < root.count; ++i) {
    const auto& nd = F.node(0, i);
    os << "  n" << i << " [label=\"c=";
    if (nd.sub >= 0) {
      const auto& t = F.trees[static_cast<std::uint32_t>(nd.sub)];
      os << terms_text(*F.table, t.row_lo, t.row_hi, t.var, names);
    } else {
      os << detail::coef_text(nd.coef);
    }
    os << " d=" << nd.pdeg << " lh=" << nd.lazy << "\"];\n";
  }
  for (std::uint32_t i = 0; i < root.count; ++i) {
    for (std::uint32_t c : F.children(0, i)) os << "  n" << i << " -> n" << c << ";\n";
  }
  os << "}\n";
  return os.str();
}

}  // namespace polyeval::front
