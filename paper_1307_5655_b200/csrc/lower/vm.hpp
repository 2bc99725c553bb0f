// Walk VM: a lowered stream as data for the ahead-of-time compiled
// interpreter kernels (runtime/vm_kernels.cu), so a new program's first
// evaluation does not wait for ptxas (0.5 s for a d1000 walk, seconds for
// C4-size programs; the reference builds and runs a program in
// milliseconds, bench.hpp:39-41 setup_ns).
//
// The straight-line SSA stream is register-allocated here, on the host:
// every value (coordinate, power, walk register) gets a slot of a per-thread
// slot file for exactly its live range (linear scan over the single
// straight-line schedule). Each op is five 32-bit words:
//   kind (0 add, 1 mul, 2 fma), dst slot, a, b, c
// with operands encoded as a slot index, kCoef | coefficient index, or kZero.
// Slots 0..nvars-1 hold the point's coordinates when the walk starts. The
// arithmetic is the stream's op sequence, unchanged — so the VM gives the
// specialised kernel's results bit for bit (tests/test_gpu_vm.py).
#pragma once

#include <cstdint>
#include <vector>

#include "lower/ptx.hpp"
#include "lower/stream.hpp"

namespace polyeval::lower {

struct VmProgram {
  static constexpr std::uint32_t kCoef = 0x80000000u;
  static constexpr std::uint32_t kZero = 0x40000000u;
  Domain domain = Domain::F64;
  std::uint32_t nvars = 0;
  std::uint32_t nslots = 0;   // slot file size (>= nvars)
  std::uint32_t nops = 0;
  std::uint32_t result = 0;   // operand
  std::vector<std::uint32_t> code;  // 5 words per op
  std::vector<std::uint64_t> lo;    // coefficient words in the domain's format
  std::vector<std::uint64_t> hi;    // interval upper endpoints (else empty)
};

/// `distinct_dst`: never give an op a destination slot that one of its
/// operands occupies (the wide-integer kernels write results limb by limb
/// while reading the operands).
template <typename C>
VmProgram build_vm(const Stream<C>& s, Domain d, bool distinct_dst = false);

}  // namespace polyeval::lower
