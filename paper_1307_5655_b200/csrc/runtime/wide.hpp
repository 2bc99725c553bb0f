// Arbitrary-width exact evaluation (pe_eval_wide): the plan the wide-integer
// kernels (runtime/wide_kernels.cu) execute — the program's strict walk as a
// walk-VM op list (distinct destination slots), every value's limb width from
// a static magnitude bound, the per-point arena layout, and the coefficient
// words. See wide_kernels.cu for the arithmetic.
#pragma once

#include <cstdint>
#include <vector>

#include "front/flat.hpp"

namespace polyeval::rt {

struct WidePlan {
  // 8 words per op, operands resolved so the kernel decodes an op from one
  // 32-byte record: kind (0 add, 1 mul), arena offset of the destination,
  // offset of a, offset of b (arena limbs, or coef_words limbs for a
  // coefficient), result width, width of a, width of b (0: the operand is
  // zero), flags (bit 0: a is a coefficient, bit 1: b is; bit 2: a product
  // read only by the sum in the next record, bit 3: as that sum's b)
  std::vector<std::uint32_t> code;
  std::vector<std::uint32_t> slot_off, slot_w;
  std::vector<std::uint32_t> coef_off, coef_w;
  std::vector<std::uint64_t> coef_words;
  std::uint32_t nops = 0, nvars = 0, point_limbs = 0;
  std::uint32_t result = 0;        // VM operand
  std::uint32_t result_limbs = 0;  // width of the result value
  std::uint32_t arena = 0;         // limbs of slots per point
  std::uint32_t tmp_w = 1;         // widest op (multiplication scratch)
  double limb_products = 0;        // schoolbook 64x64 products per point (bound)
};

/// `coefs[t]` are the little-endian two's-complement words of term t; the
/// program's int64 coefficients are the placeholders t + 1 it was built
/// with (pe_program_create_wide).
WidePlan plan_wide(const front::FlatProgram<std::int64_t>& fp,
                   const std::vector<std::vector<std::uint64_t>>& coefs,
                   std::uint32_t point_limbs);

}  // namespace polyeval::rt
