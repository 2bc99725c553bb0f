// Function schemes (paper Def. 2): split f with 0 < f(k) <= k.
//
// Mirrors reference proj/core/include/polyeval/scheme.hpp:15-57 and
// proj/core/src/scheme.cpp:10-44, including discrepancy D1 (balanced is
// ceil(k/2), scheme.cpp:19). A scheme is a value; the C-ABI describes it by a
// small POD (`pe_scheme_desc`, builtin upper/lower + cutoff) so that every
// scheme reachable through the reference CLI grammar "upper:lower@N"
// (proj/tools/scheme_name.cpp:34-53) is expressible without callbacks.
#pragma once

#include <bit>
#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>

namespace polyeval {

class FunctionScheme {
 public:
  using SplitFn = std::function<std::uint64_t(std::uint64_t)>;

  FunctionScheme(std::string name, SplitFn split)
      : name_(std::move(name)), split_(std::move(split)) {}

  std::uint64_t split(std::uint64_t k) const { return split_(k); }
  const std::string& name() const noexcept { return name_; }

 private:
  std::string name_;
  SplitFn split_;
};

enum class BuiltinScheme : int { direct = 0, horner = 1, estrin = 2, balanced = 3 };

/// direct D(k)=k, horner H(k)=1, estrin E(k)=bit_floor(k), balanced
/// B(k)=(k+1)/2 (reference scheme.cpp:10-22).
inline FunctionScheme builtin_scheme(BuiltinScheme which) {
  switch (which) {
    case BuiltinScheme::direct:
      return {"direct", [](std::uint64_t k) { return k; }};
    case BuiltinScheme::horner:
      return {"horner", [](std::uint64_t) { return std::uint64_t{1}; }};
    case BuiltinScheme::estrin:
      return {"estrin", [](std::uint64_t k) { return std::bit_floor(k); }};
    case BuiltinScheme::balanced:
      return {"balanced", [](std::uint64_t k) { return (k + 1) / 2; }};
  }
  throw std::invalid_argument("unknown builtin scheme");
}

/// split(k) = upper(k) for k > cutoff, lower(k) otherwise
/// (reference scheme.cpp:24-34).
inline FunctionScheme threshold_combine(FunctionScheme upper,
                                        FunctionScheme lower,
                                        std::uint64_t cutoff) {
  if (cutoff < 1) throw std::invalid_argument("threshold cutoff must be >= 1");
  std::string name =
      upper.name() + ":" + lower.name() + "@" + std::to_string(cutoff);
  auto split = [upper = std::move(upper), lower = std::move(lower),
                cutoff](std::uint64_t k) {
    return k > cutoff ? upper.split(k) : lower.split(k);
  };
  return {std::move(name), std::move(split)};
}

struct SchemeViolation {
  std::uint64_t k = 0;
  std::uint64_t value = 0;
};

/// First k in [1, k_max] with split(k) outside (0, k] (reference
/// scheme.cpp:36-44).
inline std::optional<SchemeViolation> validate(const FunctionScheme& scheme,
                                               std::uint64_t k_max) {
  if (k_max < 1) throw std::invalid_argument("k_max must be >= 1");
  for (std::uint64_t k = 1; k <= k_max; ++k) {
    const std::uint64_t v = scheme.split(k);
    if (v == 0 || v > k) return SchemeViolation{k, v};
  }
  return std::nullopt;
}

/// Plain-data scheme description used across the C-ABI: `upper` alone when
/// cutoff == 0, else threshold_combine(upper, lower, cutoff).
struct SchemeDesc {
  int upper = static_cast<int>(BuiltinScheme::balanced);
  int lower = static_cast<int>(BuiltinScheme::horner);
  std::uint64_t cutoff = 0;
};

inline FunctionScheme scheme_from_desc(const SchemeDesc& d) {
  auto builtin = [](int id) {
    if (id < 0 || id > 3) throw std::invalid_argument("unknown builtin scheme id");
    return builtin_scheme(static_cast<BuiltinScheme>(id));
  };
  if (d.cutoff == 0) return builtin(d.upper);
  return threshold_combine(builtin(d.upper), builtin(d.lower), d.cutoff);
}

/// Parses "name" or "upper:lower@N" (reference tools/scheme_name.cpp:34-53).
inline std::optional<SchemeDesc> scheme_desc_from_name(std::string_view name) {
  auto id_of = [](std::string_view n) -> int {
    if (n == "direct") return 0;
    if (n == "horner") return 1;
    if (n == "estrin") return 2;
    if (n == "balanced") return 3;
    return -1;
  };
  const std::size_t colon = name.find(':');
  if (colon == std::string_view::npos) {
    const int id = id_of(name);
    if (id < 0) return std::nullopt;
    return SchemeDesc{id, id, 0};
  }
  const std::size_t at = name.find('@', colon + 1);
  if (at == std::string_view::npos) return std::nullopt;
  const int up = id_of(name.substr(0, colon));
  const int lo = id_of(name.substr(colon + 1, at - colon - 1));
  if (up < 0 || lo < 0) return std::nullopt;
  const std::string_view digits = name.substr(at + 1);
  if (digits.empty()) return std::nullopt;
  std::uint64_t cutoff = 0;
  for (char ch : digits) {
    if (ch < '0' || ch > '9') return std::nullopt;
    if (cutoff > (UINT64_MAX - 9) / 10) return std::nullopt;
    cutoff = cutoff * 10 + static_cast<std::uint64_t>(ch - '0');
  }
  if (cutoff < 1) return std::nullopt;
  return SchemeDesc{up, lo, cutoff};
}

}  // namespace polyeval
