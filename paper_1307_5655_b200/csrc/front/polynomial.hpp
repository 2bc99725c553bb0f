// Canonical sparse polynomial over a coefficient ring C (int64_t or double).
//
// Semantics follow the reference `Polynomial` (proj/core/include/polyeval/
// polynomial.hpp:15-76, proj/core/src/polynomial.cpp:8-110): terms strictly
// decreasing in lexicographic exponent order, like terms merged, zero
// coefficients dropped; the zero polynomial is the empty term list. The
// reference coefficients are BigInt only; this host front-end is
// templated over the coefficient type the batch kernels compute in.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace polyeval {

template <typename C>
struct Term {
  C coefficient{};
  std::vector<std::uint32_t> exponents;

  friend bool operator==(const Term& a, const Term& b) = default;
};

/// True if `a` precedes `b` in decreasing lexicographic exponent order
/// (reference polynomial.cpp:8-11).
inline bool term_order_before(const std::vector<std::uint32_t>& a,
                              const std::vector<std::uint32_t>& b) noexcept {
  return std::lexicographical_compare(b.begin(), b.end(), a.begin(), a.end());
}

namespace detail {
inline bool coeff_is_zero(std::int64_t c) { return c == 0; }
inline bool coeff_is_zero(double c) { return c == 0.0; }
inline std::int64_t coeff_add(std::int64_t a, std::int64_t b) {
  std::int64_t out;
  if (__builtin_add_overflow(a, b, &out)) {
    throw std::overflow_error("int64 coefficient overflow while merging terms");
  }
  return out;
}
inline double coeff_add(double a, double b) { return a + b; }
}  // namespace detail

template <typename C>
class Polynomial {
 public:
  Polynomial() = default;

  /// Sorts, merges like terms and drops zeros (reference polynomial.cpp:13-33).
  /// Throws std::invalid_argument on an exponent-width mismatch.
  static Polynomial canonicalize(std::vector<Term<C>> raw,
                                 std::vector<std::string> variables) {
    for (const auto& t : raw) {
      if (t.exponents.size() != variables.size()) {
        throw std::invalid_argument(
            "term exponent count does not match variable count");
      }
    }
    std::stable_sort(raw.begin(), raw.end(),
                     [](const Term<C>& a, const Term<C>& b) {
                       return term_order_before(a.exponents, b.exponents);
                     });
    Polynomial out;
    out.variables_ = std::move(variables);
    for (auto& t : raw) {
      if (!out.terms_.empty() && out.terms_.back().exponents == t.exponents) {
        out.terms_.back().coefficient =
            detail::coeff_add(out.terms_.back().coefficient, t.coefficient);
        if (detail::coeff_is_zero(out.terms_.back().coefficient)) {
          out.terms_.pop_back();
        }
      } else if (!detail::coeff_is_zero(t.coefficient)) {
        out.terms_.push_back(std::move(t));
      }
    }
    return out;
  }

  static Polynomial zero(std::vector<std::string> variables) {
    Polynomial out;
    out.variables_ = std::move(variables);
    return out;
  }

  const std::vector<std::string>& variables() const noexcept {
    return variables_;
  }
  const std::vector<Term<C>>& terms() const noexcept { return terms_; }
  bool is_zero() const noexcept { return terms_.empty(); }

  bool is_constant() const noexcept {
    if (terms_.empty()) return true;
    if (terms_.size() != 1) return false;
    return std::all_of(terms_[0].exponents.begin(), terms_[0].exponents.end(),
                       [](std::uint32_t e) { return e == 0; });
  }

  C constant_value() const {
    if (terms_.empty()) return C{};
    if (!is_constant()) {
      throw std::logic_error("constant_value() on a non-constant polynomial");
    }
    return terms_[0].coefficient;
  }

  /// Maximum exponent of a variable (reference polynomial.cpp:69-83).
  std::uint32_t degree(std::size_t variable_index) const {
    if (is_zero()) {
      throw std::domain_error("degree of the zero polynomial is undefined");
    }
    if (variable_index >= variables_.size()) {
      throw std::invalid_argument("variable index out of range");
    }
    std::uint32_t out = 0;
    for (const auto& t : terms_) out = std::max(out, t.exponents[variable_index]);
    return out;
  }

  friend bool operator==(const Polynomial& a, const Polynomial& b) = default;

 private:
  std::vector<std::string> variables_;
  std::vector<Term<C>> terms_;
};

}  // namespace polyeval
