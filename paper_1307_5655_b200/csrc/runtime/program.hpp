// The program handle behind the C ABI: front-end result (tree + compiled
// program, reference semantics) plus lazily generated per-domain kernels.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <atomic>
#include <thread>

#include "front/flat.hpp"
#include "front/forest.hpp"
#include "front/split.hpp"
#include "front/terms.hpp"
#include "lower/ptx.hpp"
#include "lower/vm.hpp"
#include "runtime/wide.hpp"

extern "C" unsigned pe_vm_max_slots(void);

namespace polyeval::rt {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check_cuda(cudaError_t e, const char* what);

/// Device copies of a walk-VM program (op list + coefficient words).
struct VmDevice {
  void* code = nullptr;
  void* lo = nullptr;
  void* hi = nullptr;
};
struct VmImage {
  lower::VmProgram prog;
  std::map<int, VmDevice> dev;
};

/// One specialised kernel: generated PTX, its cubin, and the loaded handle
/// — or (vm set) the walk-VM form of the same stream for the AOT
/// interpreter kernels.
struct Artifact {
  std::unique_ptr<VmImage> vm;
  std::once_flag compiled;          // the cubin is built once (possibly in the background)
  std::atomic<bool> cubin_ready{false};
  lower::KernelImage image;
  std::vector<char> cubin;
  double compile_seconds = 0.0;
  cudaLibrary_t library = nullptr;
  cudaKernel_t kernel = nullptr;
  cudaKernel_t fix_kernel = nullptr;  // interval fast path: strict replay of listed points
  cudaKernel_t part_kernel = nullptr; // sign-partitioned fast path: x > 0 entry
  // sign-partitioned fast path: the mirrored program q(y) = p(-y), whose
  // kernel takes the x < 0 points (KernelImage::iv_partition == 2)
  std::unique_ptr<Artifact> mirror;
  std::map<int, void*> global_coefs;  // per device: global-tier coefficient words
  // per device ordinal: CUfunction of kernel / fix_kernel in that device's
  // primary context (driver-API launches skip the runtime's per-launch
  // library-kernel lookup); written once under the program mutex
  static constexpr int kMaxDevices = 64;
  std::array<void*, kMaxDevices> fn{};
  std::array<void*, kMaxDevices> fix_fn{};
  std::array<void*, kMaxDevices> part_fn{};
  /// The sign partition can run: this module has the x > 0 entry and the
  /// mirror module was generated with its x < 0 entry.
  bool partitioned() const {
    return image.iv_partition == 1 && mirror && mirror->image.iv_partition == 2;
  }
  Artifact() = default;
  Artifact(const Artifact&) = delete;
  Artifact& operator=(const Artifact&) = delete;
  /// Frees the per-device coefficient copies and unloads the library (the
  /// mirror module goes with its owner).
  ~Artifact();
};

/// Resolves a.fn / a.fix_fn for `device` (current device = `device`).
void bind_functions(Artifact& a, int device);

/// Host front-end state of one coefficient type: the canonical terms, the
/// evaluation trees (absent for pe_program_from_compiled) and the compiled
/// walk the kernels are generated from.
template <typename C>
struct Front {
  front::TermTable<C> terms;         // canonical (create) or one row per scalar record (import)
  std::unique_ptr<front::Forest<C>> forest;
  front::FlatProgram<C> flat;
};

/// Wide programs (pe_program_create_wide): the terms' coefficient words and
/// the plans per point width, with their device copies.
struct WideDevice {
  void *code = nullptr, *slot_off = nullptr, *slot_w = nullptr, *coef_off = nullptr,
       *coef_w = nullptr, *coef_words = nullptr;
};
struct WideFront {
  std::vector<std::vector<std::uint64_t>> coefs;  // by term, two's complement words
  std::map<std::uint32_t, WidePlan> plans;         // by point limbs
  std::map<std::pair<int, std::uint32_t>, WideDevice> dev;  // (device, point limbs)
  ~WideFront();
};

struct Program {
  std::uint32_t nvars = 0;
  bool integer = false;  // coefficient type int64 (else fp64)
  std::uint64_t nterms = 0;
  std::vector<std::string> variables;

  std::unique_ptr<Front<double>> f;         // fp64 coefficients
  std::unique_ptr<Front<std::int64_t>> i;   // int64 coefficients
  std::unique_ptr<WideFront> wide;          // multi-limb coefficients (i holds placeholders)

  front::WalkStats stats;
  lower::Tuning tuning;  // code-generation options (pe_program_set_tuning)
  // int64: largest B such that all |x_v| <= B is provably wrap-free;
  // variables absent from the polynomial get UINT64_MAX.
  std::vector<std::uint64_t> i64_uniform_bound;
  // same, for the exact-on-FP64 path: every intermediate below 2^53
  std::vector<std::uint64_t> i53_uniform_bound;

  mutable std::mutex mu;
  mutable std::array<std::unique_ptr<Artifact>, 5> artifacts;
  mutable std::array<std::unique_ptr<Artifact>, 5> vm_arts;  // walk-VM forms
  mutable std::vector<std::thread> jit_threads;              // background compiles
  mutable std::uint32_t jit_started = 0;                     // bit per domain
  mutable std::map<std::uint32_t, std::unique_ptr<Artifact>> limb_arts;  // I64K by limb count

  /// Generated (and compiled) artifact for a domain; thread-safe. With
  /// need_cubin it waits for a background compile of the same artifact.
  Artifact& artifact(lower::Domain d, bool need_cubin) const;
  /// The kernel a call launches on `device` (tuning.jit_mode): the
  /// specialised kernel once compiled; before that (default) the walk VM,
  /// while the specialised kernel compiles on a background thread.
  const Artifact& for_launch(lower::Domain d, int device) const;
  /// Walk-VM artifact for a domain, uploaded to `device`; null when the
  /// program's slot file exceeds the VM kernels'.
  Artifact* loaded_vm(lower::Domain d, int device) const;
  /// Loaded kernel handle + global-tier coefficients on `device`.
  Artifact& loaded(lower::Domain d, int device) const;
  /// K-limb exact integer kernel (Domain::I64K): generated (+ compiled), or
  /// loaded on `device`.
  Artifact& limb_artifact(std::uint32_t limbs, bool need_cubin) const;
  Artifact& loaded_limbs(std::uint32_t limbs, int device) const;
  /// Joins background compiles, unloads every kernel library and frees the
  /// device copies.
  void release() const;
  ~Program() { release(); }
};

/// Smallest K (1..8) with every intermediate provably below 2^(64K-1) for
/// |x_v| <= bounds[v] (log-domain bound: M <= T * max_t |c_t| prod X_v^a_tv,
/// with a safety margin); 0 if none.
std::uint32_t limbs_needed(const Program& p, const std::uint64_t* bounds);

/// Overflow proof for the exact int64 path: every intermediate of the walk
/// (fused or strict) is a partial sum of terms c_t * prod x_v^(a_tv - s_v),
/// bounded by M = sum_t |c_t| prod_v max(1, X_v)^a_tv; powers are bounded by
/// max(1, X_v)^max_e. Wrap-free iff M < 2^63 and every power < 2^63; with
/// limit_bits = 53 every intermediate is an exactly representable double.
bool i64_proof_holds(const Program& p, const std::uint64_t* bounds, int limit_bits = 63);

/// Largest B with the proof holding for |x_v| <= B on every variable present
/// in the polynomial (absent variables: unconstrained, or 2^53 for the FP64
/// tier, whose coordinates must be exact doubles).
std::vector<std::uint64_t> uniform_bounds(const Program& p, int limit_bits);

}  // namespace polyeval::rt
