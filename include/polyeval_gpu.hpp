// polyeval-b200 — header-only C++ wrapper over the C ABI (polyeval_b200.h).
//
// Mirrors the reference session API (proj/core/include/polyeval/eval.hpp:
// 69-90, Evaluator<D>(domain, program).evaluate(point)) for batches:
//
//   polyeval::gpu::Program prog = polyeval::gpu::Program::from_terms(
//       exponents, coeffs_i64, nterms, nvars, {"estrin"});
//   polyeval::gpu::BatchEvaluator<polyeval::gpu::BigIntDomain> ev(prog);
//   ev.evaluate({x.data(), y.data()}, n, out.data());
//
// Error mapping follows the reference (error.hpp:11-39, eval.hpp:98,186-188):
// PE_EINVAL -> std::invalid_argument, PE_ELOGIC -> std::logic_error,
// PE_EOVERFLOW -> std::overflow_error, PE_ECUDA -> std::runtime_error.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "polyeval_b200.h"

namespace polyeval::gpu {

inline void check(pe_status s) {
  if (s == PE_OK) return;
  const std::string msg = pe_last_error();
  switch (s) {
    case PE_EINVAL: throw std::invalid_argument(msg);
    case PE_EOVERFLOW: throw std::overflow_error(msg);
    case PE_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

/// "direct" | "horner" | "estrin" | "balanced" | "upper:lower@N"
/// (reference tools/scheme_name.cpp:34-53).
inline pe_scheme_desc scheme(const std::string& name) {
  auto id = [](const std::string& n) -> int {
    if (n == "direct") return PE_SCHEME_DIRECT;
    if (n == "horner") return PE_SCHEME_HORNER;
    if (n == "estrin") return PE_SCHEME_ESTRIN;
    if (n == "balanced") return PE_SCHEME_BALANCED;
    throw std::invalid_argument("unknown scheme '" + n + "'");
  };
  const auto colon = name.find(':');
  if (colon == std::string::npos) return pe_scheme_desc{id(name), id(name), 0};
  const auto at = name.find('@', colon + 1);
  if (at == std::string::npos) throw std::invalid_argument("bad scheme '" + name + "'");
  const unsigned long long cut = std::stoull(name.substr(at + 1));
  if (cut < 1) throw std::invalid_argument("threshold cutoff must be >= 1");
  return pe_scheme_desc{id(name.substr(0, colon)), id(name.substr(colon + 1, at - colon - 1)),
                        static_cast<std::uint64_t>(cut)};
}

/// Compiled program (the reference CompiledProgram; immutable, shareable).
class Program {
 public:
  template <typename Coeff>
  static Program from_terms(const std::uint32_t* exponents, const Coeff* coeffs,
                            std::size_t nterms, std::uint32_t nvars,
                            const std::vector<std::string>& schemes) {
    static_assert(std::is_same_v<Coeff, double> || std::is_same_v<Coeff, std::int64_t>,
                  "coefficients are double or int64_t");
    std::vector<pe_scheme_desc> s;
    for (std::uint32_t v = 0; v < nvars; ++v) {
      s.push_back(scheme(schemes.size() == 1 ? schemes[0] : schemes.at(v)));
    }
    pe_program* p = nullptr;
    check(pe_program_create(exponents, coeffs, nterms, nvars, s.data(),
                            std::is_same_v<Coeff, double> ? PE_COEFF_F64 : PE_COEFF_I64, &p));
    return Program(p, nvars);
  }

  /// An already compiled program (reference CompiledProgram, flattened; see
  /// pe_program_from_compiled and INTEGRATION.md).
  static Program from_compiled(const pe_compiled_program* programs, std::size_t nprograms,
                               std::uint32_t nvars, const std::uint32_t* const* exponent_sets,
                               const std::size_t* exponent_set_sizes, bool integer) {
    pe_program* p = nullptr;
    check(pe_program_from_compiled(programs, nprograms, nvars, exponent_sets, exponent_set_sizes,
                                   integer ? PE_COEFF_I64 : PE_COEFF_F64, &p));
    return Program(p, nvars);
  }

  /// Smallest 64-bit limb count (1..8) for |x_v| <= bounds[v]; 0 if > 8.
  std::uint32_t limbs_needed(const std::uint64_t* bounds) const {
    std::uint32_t k = 0;
    check(pe_program_limbs_needed(h_.get(), bounds, &k));
    return k;
  }

  const pe_program* get() const { return h_.get(); }
  std::uint32_t nvars() const { return nvars_; }

  pe_program_info_t info() const {
    pe_program_info_t i;
    check(pe_program_info(h_.get(), &i));
    return i;
  }

 private:
  Program(pe_program* p, std::uint32_t nv) : h_(p, &pe_program_destroy), nvars_(nv) {}
  std::shared_ptr<pe_program> h_;
  std::uint32_t nvars_;
};

struct DoubleDomain {
  using Value = double;
  bool strict = false;  // true: reference op order, bit-exact with DoubleDomain
};
struct BigIntDomain {
  using Value = std::int64_t;
};
struct IntervalDomain {
  using Value = double;  // SoA endpoints
};

/// Batch session (reference Evaluator<D>). Pointers may be device or host
/// memory; `stream` is a cudaStream_t for device pointers.
template <typename D>
class BatchEvaluator {
 public:
  BatchEvaluator(const Program& program, D domain = {}, int device = -1, void* stream = nullptr)
      : program_(program), domain_(domain) {
    exec_.device = device;
    exec_.stream = stream;
    exec_.synchronize = 1;
    if constexpr (std::is_same_v<D, DoubleDomain>) exec_.strict_f64 = domain.strict ? 1 : 0;
  }

  void evaluate(std::initializer_list<const typename D::Value*> coords, std::size_t n,
                typename D::Value* out) const {
    if (coords.size() != program_.nvars()) {
      throw std::invalid_argument("evaluation point arity mismatch");
    }
    std::vector<const typename D::Value*> c(coords);
    if constexpr (std::is_same_v<D, BigIntDomain>) {
      check(pe_eval_i64(program_.get(), c.data(), n, out, &exec_));
    } else {
      check(pe_eval_f64(program_.get(), c.data(), n, out, &exec_));
    }
  }

  /// BigIntDomain beyond int64: `limbs` 64-bit words per result (two's
  /// complement, little-endian), out_limbs[k][i] = word k of point i.
  void evaluate_limbs(std::initializer_list<const std::int64_t*> coords, std::size_t n,
                      std::uint32_t limbs, std::uint64_t* const* out_limbs) const {
    static_assert(std::is_same_v<D, BigIntDomain>, "exact integer domain only");
    if (coords.size() != program_.nvars()) {
      throw std::invalid_argument("evaluation point arity mismatch");
    }
    std::vector<const std::int64_t*> c(coords);
    check(pe_eval_limbs(program_.get(), c.data(), n, limbs, out_limbs, &exec_));
  }

  /// Reference evaluate_parallel (eval.hpp:97-140): identical results; the
  /// worker count is validated, the batch is spread over the GPU anyway.
  void evaluate_parallel(std::initializer_list<const typename D::Value*> coords, std::size_t n,
                         typename D::Value* out, unsigned workers) const {
    if (workers < 1) throw std::invalid_argument("workers must be >= 1");
    evaluate(coords, n, out);
  }

  /// Reference enable_register_check (eval.hpp:142-145), checked once per
  /// program (every point walks the same records).
  void enable_register_check(bool on) {
    if (on) check(pe_program_check_registers(program_.get()));
  }

  /// IntervalDomain: lo/hi coordinate arrays, lo/hi results.
  void evaluate(std::initializer_list<const double*> lo, std::initializer_list<const double*> hi,
                std::size_t n, double* out_lo, double* out_hi) const {
    static_assert(std::is_same_v<D, IntervalDomain>, "interval overload");
    if (lo.size() != program_.nvars() || hi.size() != program_.nvars()) {
      throw std::invalid_argument("evaluation point arity mismatch");
    }
    std::vector<const double*> l(lo), h(hi);
    check(pe_eval_interval(program_.get(), l.data(), h.data(), n, out_lo, out_hi, &exec_));
  }

 private:
  Program program_;
  D domain_;
  pe_exec exec_{};
};

}  // namespace polyeval::gpu
