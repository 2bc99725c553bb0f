// Wide-integer evaluation plans: see wide.hpp.
#include "runtime/wide.hpp"

#include <algorithm>
#include <stdexcept>

#include "lower/stream.hpp"
#include "lower/vm.hpp"

namespace polyeval::rt {
namespace {

// Magnitude bit length of a two's-complement word vector.
std::uint32_t magnitude_bits(const std::vector<std::uint64_t>& w) {
  if (w.empty()) return 0;
  const bool neg = w.back() >> 63;
  std::vector<std::uint64_t> m = w;
  if (neg) {  // -x = ~x + 1
    unsigned __int128 c = 1;
    for (auto& x : m) {
      const unsigned __int128 t = static_cast<unsigned __int128>(~x) + c;
      x = static_cast<std::uint64_t>(t);
      c = t >> 64;
    }
  }
  for (std::size_t k = m.size(); k-- > 0;) {
    if (m[k]) return static_cast<std::uint32_t>(64 * k + 64 - __builtin_clzll(m[k]));
  }
  return 0;
}

// Limbs of a two's-complement value with |v| <= 2^bits (bits + 1
// magnitude bits and a sign bit).
std::uint32_t limbs_for(std::uint64_t bits) {
  return static_cast<std::uint32_t>(std::max<std::uint64_t>(1, (bits + 2 + 63) / 64));
}

}  // namespace

WidePlan plan_wide(const front::FlatProgram<std::int64_t>& fp,
                   const std::vector<std::vector<std::uint64_t>>& coefs,
                   std::uint32_t point_limbs) {
  if (point_limbs == 0) throw std::invalid_argument("point_limbs must be >= 1");
  const lower::Stream<std::int64_t> s = lower::lower_strict(fp);
  const lower::VmProgram vm = lower::build_vm(s, lower::Domain::I64, true);
  WidePlan p;
  p.nvars = vm.nvars;
  p.point_limbs = point_limbs;
  p.nops = vm.nops;
  p.result = vm.result;
  // coefficient table (stream coefficient k carries the placeholder t + 1)
  std::vector<std::uint32_t> coef_bits(s.coefs.size());
  for (std::size_t k = 0; k < s.coefs.size(); ++k) {
    const std::int64_t ph = s.coefs[k];
    if (ph < 1 || static_cast<std::size_t>(ph) > coefs.size()) {
      throw std::logic_error("wide program: coefficient placeholder out of range");
    }
    const auto& w = coefs[static_cast<std::size_t>(ph - 1)];
    coef_bits[k] = magnitude_bits(w);
    const std::uint32_t width = limbs_for(coef_bits[k]);
    p.coef_off.push_back(static_cast<std::uint32_t>(p.coef_words.size()));
    p.coef_w.push_back(width);
    for (std::uint32_t j = 0; j < width; ++j) {
      p.coef_words.push_back(j < w.size() ? w[j] : (w.empty() || !(w.back() >> 63) ? 0 : ~0ull));
    }
  }
  // magnitude bounds |v| <= 2^bits, value by value in walk order (slots are
  // reused); a coordinate of L two's-complement limbs has |x| <= 2^(64L-1)
  const std::uint64_t coord_bits = 64ull * point_limbs - 1;
  std::vector<std::uint64_t> slot_bits(vm.nslots, 0);
  std::vector<std::uint32_t> slot_max(vm.nslots, 1);
  for (std::uint32_t v = 0; v < vm.nvars; ++v) {
    slot_bits[v] = coord_bits;
    slot_max[v] = std::max(point_limbs, limbs_for(coord_bits));
  }
  auto bits_of = [&](std::uint32_t o) -> std::uint64_t {
    if (o & lower::VmProgram::kZero) return 0;
    if (o & lower::VmProgram::kCoef) return coef_bits[o & ~lower::VmProgram::kCoef];
    return slot_bits[o];
  };
  auto width_of = [&](std::uint32_t o) -> std::uint32_t {
    if (o & lower::VmProgram::kZero) return 0;
    if (o & lower::VmProgram::kCoef) return p.coef_w[o & ~lower::VmProgram::kCoef];
    return limbs_for(slot_bits[o]);
  };
  for (std::uint32_t i = 0; i < vm.nops; ++i) {
    const std::uint32_t* c = vm.code.data() + 5 * i;
    const std::uint32_t kind = c[0], dst = c[1];
    if (kind == 2) throw std::logic_error("wide plans take strict streams (no fused ops)");
    const std::uint64_t ba = bits_of(c[2]), bb = bits_of(c[3]);
    const std::uint32_t wa = width_of(c[2]), wb = width_of(c[3]);
    const std::uint64_t br = kind == 0 ? std::max(ba, bb) + 1 : (ba && bb ? ba + bb : 0);
    if (br > (std::uint64_t{1} << 31)) throw std::overflow_error("wide evaluation: values beyond 2^31 bits");
    const std::uint32_t wr = limbs_for(br);
    slot_bits[dst] = br;
    slot_max[dst] = std::max(slot_max[dst], wr);
    p.tmp_w = std::max(p.tmp_w, wr);
    if (kind == 1) p.limb_products += static_cast<double>(wa) * wb;
    p.code.insert(p.code.end(), {kind, dst, c[2], c[3], wr, wa, wb, 0u});
  }
  p.result_limbs = width_of(vm.result);
  std::uint64_t off = 0;
  for (std::uint32_t sl = 0; sl < vm.nslots; ++sl) {
    p.slot_off.push_back(static_cast<std::uint32_t>(off));
    p.slot_w.push_back(slot_max[sl]);
    off += slot_max[sl];
  }
  if (off > UINT32_MAX / 2) throw std::overflow_error("wide evaluation: arena too large");
  p.arena = static_cast<std::uint32_t>(off);
  // resolve the operands of every op (slot -> arena offset, coefficient ->
  // offset into coef_words)
  for (std::uint32_t i = 0; i < p.nops; ++i) {
    std::uint32_t* c = p.code.data() + 8 * i;
    std::uint32_t flags = 0;
    for (int k = 0; k < 2; ++k) {
      std::uint32_t& o = c[2 + k];
      if (o & lower::VmProgram::kZero) {
        o = 0;
        c[5 + k] = 0;  // width 0: zero operand
      } else if (o & lower::VmProgram::kCoef) {
        o = p.coef_off[o & ~lower::VmProgram::kCoef];
        flags |= 1u << k;
      } else {
        o = p.slot_off[o];
      }
    }
    c[1] = p.slot_off[c[1]];
    c[7] = flags;
  }
  return p;
}

}  // namespace polyeval::rt
