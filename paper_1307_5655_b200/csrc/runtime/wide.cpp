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
  // The fused lowering (one multiply-add per record instead of product,
  // zero-add and sum): exact integers give the reference's value in any
  // order. No constant folding: the coefficients are placeholders.
  const lower::Stream<std::int64_t> s = lower::lower_fused(fp, false);
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
  // (one more slot: the product of a multiply-add where it is run as two ops)
  const std::uint32_t tmp_slot = vm.nslots;
  std::vector<std::uint64_t> slot_bits(vm.nslots + 1, 0);
  std::vector<std::uint32_t> slot_max(vm.nslots + 1, 1);
  std::vector<std::uint32_t> fuse;  // per record: flag bits 2, 3
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
  auto bound = [](std::uint64_t br) {
    if (br > (std::uint64_t{1} << 31)) throw std::overflow_error("wide evaluation: values beyond 2^31 bits");
    return limbs_for(br);
  };
  for (std::uint32_t i = 0; i < vm.nops; ++i) {
    const std::uint32_t* c = vm.code.data() + 5 * i;
    const std::uint32_t kind = c[0], dst = c[1];
    const std::uint64_t ba = bits_of(c[2]), bb = bits_of(c[3]);
    const std::uint32_t wa = width_of(c[2]), wb = width_of(c[3]);
    if (kind == 2) {
      // dst = a * b + c as a product into the extra slot and a sum, flagged
      // as a pair the kernel may run in one pass (the VM's destination is
      // distinct from all three operands)
      const std::uint64_t bc = bits_of(c[4]), bp = ba && bb ? ba + bb : 0;
      const std::uint32_t wc = width_of(c[4]), wp = bound(bp);
      const std::uint64_t br = std::max(bp, bc) + 1;
      const std::uint32_t wr = bound(br);
      slot_bits[tmp_slot] = bp;
      slot_max[tmp_slot] = std::max(slot_max[tmp_slot], wp);
      slot_bits[dst] = br;
      slot_max[dst] = std::max(slot_max[dst], wr);
      p.tmp_w = std::max(p.tmp_w, wr);
      p.limb_products += static_cast<double>(wa) * wb;
      p.code.insert(p.code.end(), {1u, tmp_slot, c[2], c[3], wp, wa, wb, 0u});
      p.code.insert(p.code.end(), {0u, dst, tmp_slot, c[4], wr, wp, wc, 0u});
      fuse.push_back(4u);  // the product is the sum's a
      fuse.push_back(0u);
      continue;
    }
    const std::uint64_t br = kind == 0 ? std::max(ba, bb) + 1 : (ba && bb ? ba + bb : 0);
    const std::uint32_t wr = bound(br);
    slot_bits[dst] = br;
    slot_max[dst] = std::max(slot_max[dst], wr);
    p.tmp_w = std::max(p.tmp_w, wr);
    if (kind == 1) p.limb_products += static_cast<double>(wa) * wb;
    p.code.insert(p.code.end(), {kind, dst, c[2], c[3], wr, wa, wb, 0u});
    fuse.push_back(0u);
  }
  p.nops = static_cast<std::uint32_t>(fuse.size());
  p.result_limbs = width_of(vm.result);
  std::uint64_t off = 0;
  for (std::uint32_t sl = 0; sl <= tmp_slot; ++sl) {
    p.slot_off.push_back(static_cast<std::uint32_t>(off));
    p.slot_w.push_back(slot_max[sl]);
    off += slot_max[sl];
  }
  if (off > UINT32_MAX / 2) throw std::overflow_error("wide evaluation: arena too large");
  p.arena = static_cast<std::uint32_t>(off);
  // A product whose only reader is the sum that follows it (r = a * b; e =
  // r + c: every node of a Horner chain or a balanced split) can be added
  // on the way: the product's record gets flag bit 2, bit 3 telling which
  // operand of the sum is the product. The kernel may then run the pair as
  // one op and never write r.
  for (std::uint32_t i = 0; i + 1 < p.nops; ++i) {
    const std::uint32_t* m = p.code.data() + 8 * i;
    const std::uint32_t* d = m + 8;
    if (fuse[i] || m[0] != 1 || d[0] != 0) continue;
    const std::uint32_t r = m[1];
    const bool in_a = d[2] == r, in_b = d[3] == r;
    if (in_a == in_b) continue;  // not read by the sum, or r + r
    bool dead = d[1] == r;       // the sum overwrites the slot ...
    for (std::uint32_t j = i + 2; !dead; ++j) {  // ... or nothing reads it before its next write
      if (j == p.nops) {
        dead = vm.result != r;
        break;
      }
      const std::uint32_t* q = p.code.data() + 8 * j;
      if (q[2] == r || q[3] == r) break;
      if (q[1] == r) dead = true;
    }
    // (the sum's destination may reuse a slot the product released: the
    // fused op would overwrite an operand it is still reading)
    if (dead && d[1] != r && d[1] != m[2] && d[1] != m[3]) fuse[i] = 4u | (in_b ? 8u : 0u);
  }
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
    c[7] = flags | fuse[i];
  }
  return p;
}

}  // namespace polyeval::rt
