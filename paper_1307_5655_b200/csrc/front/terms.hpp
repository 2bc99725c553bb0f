// Flat term tables: the polynomial as two parallel arrays (exponent rows and
// coefficients) in canonical order.
//
// Canonical order is the reference's (proj/core/src/polynomial.cpp:8-33):
// exponent rows strictly decreasing lexicographically, like terms merged in
// input order, zero coefficients dropped; the empty table is the zero
// polynomial. Here it is reached by sorting a permutation of row indices and
// folding runs of equal rows, with no per-term heap objects — the table is
// what the tree builder (front/forest.hpp) partitions by contiguous runs.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

namespace polyeval::front {

template <typename C>
struct TermTable {
  std::uint32_t nvars = 0;
  std::vector<std::uint32_t> exps;  // size() rows of nvars exponents
  std::vector<C> coefs;

  std::size_t size() const noexcept { return coefs.size(); }
  bool empty() const noexcept { return coefs.empty(); }
  const std::uint32_t* row(std::size_t t) const noexcept { return exps.data() + t * nvars; }
  std::uint32_t exp(std::size_t t, std::size_t v) const noexcept { return exps[t * nvars + v]; }
};

namespace detail {
inline bool is_zero(std::int64_t c) noexcept { return c == 0; }
inline bool is_zero(double c) noexcept { return c == 0.0; }
inline void accumulate(std::int64_t& acc, std::int64_t c) {
  if (__builtin_add_overflow(acc, c, &acc)) {
    throw std::overflow_error("int64 coefficient overflow while merging like terms");
  }
}
inline void accumulate(double& acc, double c) noexcept { acc += c; }
}  // namespace detail

/// Canonical table of `n` raw terms (`exps` row-major n x nvars).
///
/// Like terms are summed in their input order; a run whose sum is zero
/// vanishes. (The reference folds pairwise and drops a zero partial sum at
/// once — for int64 and for doubles the surviving values are the same, since
/// 0 + c == c exactly and a run that returns to zero restarts from c.)
template <typename C>
TermTable<C> canonical_terms(const std::uint32_t* exps, const C* coefs, std::size_t n,
                             std::uint32_t nvars) {
  std::vector<std::uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  auto row = [&](std::uint32_t t) { return exps + static_cast<std::size_t>(t) * nvars; };
  // descending rows; equal rows keep their input order (stable)
  std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
    const std::uint32_t* ra = row(a);
    const std::uint32_t* rb = row(b);
    for (std::uint32_t v = 0; v < nvars; ++v) {
      if (ra[v] != rb[v]) return ra[v] > rb[v];
    }
    return false;
  });
  TermTable<C> out;
  out.nvars = nvars;
  std::size_t i = 0;
  while (i < n) {
    std::size_t j = i + 1;
    while (j < n && std::equal(row(order[i]), row(order[i]) + nvars, row(order[j]))) ++j;
    C sum = coefs[order[i]];
    bool live = !detail::is_zero(sum);
    for (std::size_t k = i + 1; k < j; ++k) {
      const C c = coefs[order[k]];
      if (detail::is_zero(c)) continue;
      if (live) {
        detail::accumulate(sum, c);
      } else {
        sum = c;
      }
      live = !detail::is_zero(sum);
    }
    if (live) {
      out.coefs.push_back(sum);
      out.exps.insert(out.exps.end(), row(order[i]), row(order[i]) + nvars);
    }
    i = j;
  }
  return out;
}

}  // namespace polyeval::front
