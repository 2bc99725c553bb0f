// Function schemes (paper Def. 2) as plain data.
//
// A scheme maps a degree k >= 2 to the exponent s = f(k), 0 < s <= k, at
// which a term range is cut. The reference models a scheme as a named
// std::function (proj/core/include/polyeval/scheme.hpp:15-57,
// proj/core/src/scheme.cpp:10-44); everything its CLI can name is a builtin
// or one threshold combination "upper:lower@N" (tools/scheme_name.cpp:34-53),
// so here a scheme is the POD {upper, lower, cutoff} the C ABI already
// carries (pe_scheme_desc), evaluated by a switch.
//
//   direct   f(k) = k              horner  f(k) = 1
//   estrin   f(k) = 2^floor(lg k)  balanced f(k) = ceil(k / 2)   (D1)
#pragma once

#include <bit>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>

namespace polyeval::front {

enum class Builtin : int { direct = 0, horner = 1, estrin = 2, balanced = 3 };

inline std::uint64_t apply_builtin(int id, std::uint64_t k) {
  switch (static_cast<Builtin>(id)) {
    case Builtin::direct: return k;
    case Builtin::horner: return 1;
    case Builtin::estrin: return std::bit_floor(k);
    case Builtin::balanced: return k / 2 + (k & 1);
  }
  throw std::invalid_argument("unknown builtin scheme id " + std::to_string(id));
}

inline const char* builtin_label(int id) {
  static const char* const kNames[] = {"direct", "horner", "estrin", "balanced"};
  if (id < 0 || id > 3) throw std::invalid_argument("unknown builtin scheme id " + std::to_string(id));
  return kNames[id];
}

/// `upper` alone when cutoff == 0; otherwise `upper` for k > cutoff and
/// `lower` for k <= cutoff.
struct SplitRule {
  int upper = static_cast<int>(Builtin::balanced);
  int lower = static_cast<int>(Builtin::horner);
  std::uint64_t cutoff = 0;

  /// Throws std::invalid_argument for an unknown builtin id.
  void check() const {
    (void)builtin_label(upper);
    if (cutoff != 0) (void)builtin_label(lower);
  }
  std::uint64_t operator()(std::uint64_t k) const {
    return apply_builtin(cutoff != 0 && k <= cutoff ? lower : upper, k);
  }
  std::string name() const {
    std::string s = builtin_label(upper);
    if (cutoff == 0) return s;
    return s + ":" + builtin_label(lower) + "@" + std::to_string(cutoff);
  }
};

/// Smallest k in [1, k_max] where the rule leaves (0, k], if any.
inline std::optional<std::uint64_t> first_violation(const SplitRule& rule, std::uint64_t k_max) {
  for (std::uint64_t k = 1; k <= k_max; ++k) {
    const std::uint64_t s = rule(k);
    if (s < 1 || s > k) return k;
  }
  return std::nullopt;
}

/// "name" or "upper:lower@N" with N >= 1; nullopt for anything else.
inline std::optional<SplitRule> parse_rule(std::string_view text) {
  auto id = [](std::string_view w) -> int {
    for (int i = 0; i < 4; ++i) {
      if (w == builtin_label(i)) return i;
    }
    return -1;
  };
  const auto colon = text.find(':');
  if (colon == std::string_view::npos) {
    const int u = id(text);
    if (u < 0) return std::nullopt;
    return SplitRule{u, u, 0};
  }
  const auto at = text.find('@', colon);
  if (at == std::string_view::npos || at + 1 == text.size()) return std::nullopt;
  const int u = id(text.substr(0, colon)), l = id(text.substr(colon + 1, at - colon - 1));
  if (u < 0 || l < 0) return std::nullopt;
  std::uint64_t n = 0;
  for (char ch : text.substr(at + 1)) {
    if (ch < '0' || ch > '9' || n > UINT64_MAX / 10 - 1) return std::nullopt;
    n = n * 10 + static_cast<std::uint64_t>(ch - '0');
  }
  if (n == 0) return std::nullopt;
  return SplitRule{u, l, n};
}

}  // namespace polyeval::front
