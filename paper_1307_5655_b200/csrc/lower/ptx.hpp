// PTX emission for a lowered stream: one specialised sm_100a kernel per
// (program, domain). The kernel body is the straight-line walk; the frame
// around it (thread -> point mapping, SoA coordinate loads, power DAG,
// stores, domain checks) is fixed and hand-written below.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "lower/stream.hpp"

namespace polyeval::lower {

enum class Domain : int {
  F64 = 0,        // DoubleDomain, FMA-fused (tolerance contract)
  F64Strict = 1,  // DoubleDomain, reference op sequence, bit-exact
  I64 = 2,        // BigIntDomain restricted to a proven int64 range, exact
  Interval = 3,   // IntervalDomain, reference op sequence, bit-exact
  I64F = 4,       // BigIntDomain on a range proven below 2^53: the same exact
                  // integer results, computed on the FP64 FMA pipe (every
                  // intermediate is an integer of magnitude < 2^53, hence a
                  // double, hence every DFMA/DMUL is exact)
  I64K = 5,       // BigIntDomain on a range proven below 2^(64K-1): K-limb
                  // two's-complement integers (KernelShape::limbs), carry-chain
                  // multiply-adds mod 2^(64K) — exact by the proof
};

const char* domain_name(Domain d);

/// Where the coefficient words of a kernel live. Warp-uniform reads from the
/// constant bank fold into the FP64 instruction operand (c[0x3][imm]); the
/// 64 KB bank holds 8K words, kernel parameters another ~4K (c[0x0]); beyond
/// that coefficients stream from global memory through L1 (one LDG each).
struct CoefTiers {
  static constexpr std::uint32_t kConstCap = 8000;
  static constexpr std::uint32_t kParamCap = 3900;
  static constexpr std::uint32_t kSmemCap = 6140;  // 48 KB static shared less the mbarrier
};

struct KernelImage {
  std::string entry;               // kernel symbol
  std::string ptx;                 // full module text
  Domain domain = Domain::F64;
  std::uint32_t nvars = 0;
  std::uint32_t n_in = 0;          // pointer params for coordinates
  std::uint32_t n_out = 0;         // pointer params for results
  bool has_flag = false;           // u64 device pointer to a u32 status word
  bool has_bounds = false;         // nvars x u64 coordinate bounds (int64)
  std::vector<std::uint64_t> param_words;   // param-tier coefficient words
  std::vector<std::uint64_t> global_words;  // global-tier coefficient words
  std::uint32_t const_words = 0;
  std::uint32_t block = 128;
  std::uint32_t lanes = 1;         // points per thread (tile = block * lanes)
  bool interval_fast_path = false; // fast exact path + fixup entry (strict replay)
  std::uint32_t limbs = 1;         // I64K: 64-bit words per value (= result arrays)
  std::uint32_t chain_loops = 0;   // Hörner runs emitted as counted loops
  std::uint32_t sections = 1;      // sections of the walk (persistent grouped kernel when > 1)
  std::uint32_t group_tiles = 0;   // sectioned: tiles per CTA per section pass
  std::uint32_t scratch_values = 0;  // sectioned: values per point in the scratch slot
  std::string fix_entry;           // fixup kernel symbol (interval fast path)
  // sign-partitioned interval fast path (univariate): 1 = this module also
  // has `part_entry` (points with x > 0, taken from the front of a device
  // index list); 2 = module of the mirrored program q(y) = p(-y) whose only
  // entry `entry` takes points with x < 0 from the back of the list and
  // evaluates q at -x. Both entries take two extra parameters (list, counts).
  // 3 = `part_entry` is the one-pass split kernel (classify, pack by sign in
  // shared memory, evaluate p or q per packed slot); no mirror module.
  std::uint32_t iv_partition = 0;
  std::string part_entry;
  std::uint64_t iv_partition_min = 65536;  // smaller batches skip the partition
  std::uint32_t fix_block = 128;   // fixup kernel CTA size (.maxntid)
  std::uint32_t fix_ctas_per_sm = 4;  // fixup grid: CTAs per SM (.minnctapersm)
  bool fix_persistent = false;     // fixup entry strides over the list (grid: CTAs per SM x SMs)
  // instruction counts per point (roofline bookkeeping)
  std::uint64_t fp_ops = 0;        // FP64 add/mul/fma issued per point
  std::uint64_t int_ops = 0;       // int64 add/mul/mad per point
  std::uint64_t hash = 0;          // FNV-1a of `ptx`
};

/// Code-generation options of one program (the C ABI's pe_tuning). Every
/// field's 0 means "the measured default"; a program's kernels are generated
/// from the options it holds when the kernel is first needed.
struct Tuning {
  std::uint32_t lanes = 0;        // points per thread (1..8)
  std::uint32_t block = 0;        // threads per CTA (32..1024)
  std::uint32_t min_ctas = 0;     // .minnctapersm of the walk entry
  std::uint32_t sync_every = 0;   // walk ops between CTA barriers
  std::uint32_t section_ops = 0;  // ops per section of a long scalar walk; UINT32_MAX = one section
  std::uint32_t sched_window = 0; // list-scheduling window (1 = keep the walk order)
  std::uint32_t sched_distance = 0;
  std::uint32_t chain_min = 0;    // shortest Hörner run emitted as a loop; UINT32_MAX = never
  std::int32_t iv_fast = 0;       // interval fast path + fixup list (-1 = bit-level replay only)
  std::int32_t iv_mid = 0;        // fixup: finite-case replay first (-1 = bit-level only)
  std::int32_t iv_partition = 0;  // univariate sign partition (-1 off, 3 = one-pass split kernel)
  std::uint32_t group_tiles = 0;  // sections: tiles a CTA runs per section pass (default 4)
  std::int32_t word_layout = 0;   // sections: -1 = all uniform-bound words first (no per-section blocks)
  std::int32_t jit_mode = 0;      // 0 walk VM until the kernel is compiled, 1 always wait, 2 VM only
  std::uint64_t iv_partition_min = 0;  // smallest partitioned batch (default 65536)
};

/// Launch shape of a specialised kernel.
///  lanes       points per thread (P)
///  block       threads per CTA; `.maxntid block` caps ptxas at 65536/block
///              registers, so one CTA fills an SM's register file
///  sync_every  walk ops between CTA barriers (0 = none). Straight-line walks
///              are larger than the instruction caches; a barrier every few
///              KB of code keeps all warps of the CTA inside one code window,
///              so each instruction line is fetched once per SM, not per warp.
struct KernelShape {
  std::uint32_t lanes = 0;
  std::uint32_t block = 0;
  std::uint32_t sync_every = 0;
  // I64K: 64-bit limbs per value (1..8)
  std::uint32_t limbs = 0;
  // .minnctapersm of the walk entry (0 = none): caps ptxas at
  // 65536 / (block * min_ctas) registers
  std::uint32_t min_ctas = 0;
  // interval fast path partition role (KernelImage::iv_partition)
  std::uint32_t iv_partition = 0;
};

/// Measured defaults per domain and program size, then the tuning overrides.
KernelShape default_shape(Domain d, std::uint32_t powers, std::uint64_t distinct_coefs,
                          const Tuning& t);

/// `mirror` (interval domain, univariate, shape.iv_partition == 1): the
/// strict stream of q(y) = p(-y) (mirror_stream); when both programs'
/// coefficients fit the constant bank the module gains the one-pass sign
/// split entry (KernelImage::iv_partition 3).
template <typename C>
KernelImage emit_ptx(const Stream<C>& stream, Domain domain, KernelShape shape = {},
                     const Tuning& tuning = {}, const Stream<C>* mirror = nullptr);

}  // namespace polyeval::lower
