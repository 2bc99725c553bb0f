// Program: the front-end result plus lazily generated per-domain kernels
// (lowering -> PTX -> cubin -> loaded library), the int64 overflow proof and
// the fp64 slicing of wide programs. See runtime/program.hpp.
#include "runtime/program.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <future>
#include <memory>
#include <thread>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "lower/ptx.hpp"
#include "lower/stream.hpp"
#include "runtime/jit.hpp"

namespace polyeval::rt {

namespace {
using u128 = unsigned __int128;
constexpr u128 kSat = (static_cast<u128>(1) << 100);

u128 sat_mul(u128 a, u128 b) {
  if (a == 0 || b == 0) return 0;
  if (a >= kSat || b >= kSat) return kSat;
  if (a > kSat / b) return kSat;
  return std::min<u128>(a * b, kSat);
}
u128 sat_pow(u128 base, std::uint32_t e) {
  u128 r = 1;
  while (e) {
    if (e & 1) r = sat_mul(r, base);
    e >>= 1;
    if (e) base = sat_mul(base, base);
  }
  return r;
}
}  // namespace

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                    cudaGetErrorString(e) + ")");
  }
}

bool i64_proof_holds(const Program& p, const std::uint64_t* bounds, int limit_bits) {
  const u128 limit = static_cast<u128>(1) << limit_bits;
  std::vector<u128> base(p.nvars);
  for (std::uint32_t v = 0; v < p.nvars; ++v) base[v] = std::max<u128>(1, bounds[v]);
  u128 m = 0;
  std::vector<std::uint32_t> max_e(p.nvars, 0);
  const auto& T = p.i->terms;
  for (std::size_t t = 0; t < T.size(); ++t) {
    const std::int64_t cf = T.coefs[t];
    const u128 c = cf < 0 ? static_cast<u128>(-(cf + 1)) + 1 : static_cast<u128>(cf);
    u128 term = c;
    for (std::uint32_t v = 0; v < p.nvars; ++v) {
      term = sat_mul(term, sat_pow(base[v], T.exp(t, v)));
      max_e[v] = std::max(max_e[v], T.exp(t, v));
    }
    m = std::min<u128>(m + term, kSat);
  }
  if (m >= limit) return false;
  for (std::uint32_t v = 0; v < p.nvars; ++v) {
    // coordinates themselves must be exact in the working type
    if (limit_bits < 63 && static_cast<u128>(bounds[v]) > limit) return false;
    if (sat_pow(base[v], max_e[v]) >= limit) return false;
  }
  return true;
}

std::vector<std::uint64_t> uniform_bounds(const Program& p, int limit_bits) {
  std::vector<std::uint64_t> out(p.nvars, UINT64_MAX);
  std::vector<bool> present(p.nvars, false);
  const auto& T = p.i->terms;
  for (std::size_t t = 0; t < T.size(); ++t) {
    for (std::uint32_t v = 0; v < p.nvars; ++v) present[v] = present[v] || T.exp(t, v) > 0;
  }
  // the exact-FP64 path converts coordinates to double: they must be < 2^53
  // even for variables absent from the polynomial
  const std::uint64_t absent = limit_bits == 53 ? (1ull << 53) : UINT64_MAX;
  for (std::uint32_t v = 0; v < p.nvars; ++v) out[v] = absent;
  std::uint64_t lo = 0, hi = limit_bits == 53 ? (1ull << 53) : (1ull << 62);
  std::vector<std::uint64_t> probe(p.nvars);
  auto ok = [&](std::uint64_t b) {
    for (std::uint32_t v = 0; v < p.nvars; ++v) probe[v] = present[v] ? b : 0;
    return i64_proof_holds(p, probe.data(), limit_bits);
  };
  if (!ok(0)) {
    lo = 0;
    for (std::uint32_t v = 0; v < p.nvars; ++v) out[v] = present[v] ? 0 : absent;
    // even X = 1 overflows: every evaluation is refused
    return out;
  }
  while (lo < hi) {  // largest b with ok(b)
    const std::uint64_t mid = lo + (hi - lo + 1) / 2;
    if (ok(mid)) lo = mid; else hi = mid - 1;
  }
  for (std::uint32_t v = 0; v < p.nvars; ++v) out[v] = present[v] ? lo : absent;
  return out;
}

namespace {
// Interval domain: the program's kernel (+ the mirror module when the sign
// partition applies, see lower/ptx.cpp and lower::mirror_stream).
template <typename C>
void emit_interval(const front::FlatProgram<C>& prog, std::uint32_t nvars, const lower::Tuning& t,
                   Artifact& a) {
  lower::KernelShape shape;
  if (nvars == 1 && t.iv_partition >= 0) shape.iv_partition = 1;
  const auto s = lower::lower_strict(prog);
  lower::Stream<C> q;
  const bool mirrored = shape.iv_partition == 1 && lower::mirror_stream(s, &q);
  // tuning iv_partition 3: the one-pass split kernel where it fits (reads and
  // writes each interval once; measured slower than the classifier path on
  // C5, 12.6 vs 10.5 ms per 1e8: profiles/r2_c5_split_vs_classify.jsonl)
  a.image = lower::emit_ptx(s, lower::Domain::Interval, shape, t,
                            mirrored && t.iv_partition == 3 ? &q : nullptr);
  // iv_partition 3: the split kernel carries both programs; 1: the
  // classifier path needs the mirrored program's module
  if (a.image.iv_partition != 1 || !mirrored) return;
  lower::KernelShape ms;
  ms.iv_partition = 2;
  auto m = std::make_unique<Artifact>();
  m->image = lower::emit_ptx(q, lower::Domain::Interval, ms, t);
  if (m->image.iv_partition == 2) a.mirror = std::move(m);
}
}  // namespace

Artifact& Program::artifact(lower::Domain d, bool need_cubin) const {
  std::unique_lock<std::mutex> lock(mu);
  auto& slot = artifacts[static_cast<int>(d)];
  if (!slot) {
    auto a = std::make_unique<Artifact>();
    const bool strict = d == lower::Domain::F64Strict || d == lower::Domain::Interval;
    if (d == lower::Domain::Interval) {
      // univariate programs get the sign-partitioned fast path: this module
      // gains an x > 0 entry, a mirror module evaluates q(y) = p(-y) at -x
      if (integer) {
        emit_interval(i->flat, nvars, tuning, *a);
      } else {
        emit_interval(f->flat, nvars, tuning, *a);
      }
    } else if (integer) {
      auto s = strict ? lower::lower_strict(i->flat) : lower::lower_fused(i->flat);
      a->image = lower::emit_ptx(s, d, {}, tuning);
    } else {
      if (d == lower::Domain::I64 || d == lower::Domain::I64F) {
        throw std::invalid_argument("pe_eval_i64 needs a program with int64 coefficients");
      }
      auto s = strict ? lower::lower_strict(f->flat) : lower::lower_fused(f->flat);
      a->image = lower::emit_ptx(s, d, {}, tuning);
    }
    slot = std::move(a);
  }
  Artifact& a = *slot;
  lock.unlock();  // ptxas runs outside the program lock
  if (need_cubin) {
    // once per artifact: a second caller (e.g. a blocking call while the
    // background compile runs) waits for the first
    std::call_once(a.compiled, [&a] {
      CompileResult r = compile_ptx_cached(a.image.ptx, a.image.entry);
      if (!r.ok) throw std::logic_error(r.log);
      std::vector<char> mirror_cubin;
      if (a.mirror) {
        CompileResult m = compile_ptx_cached(a.mirror->image.ptx, a.mirror->image.entry);
        if (!m.ok) throw std::logic_error(m.log);
        a.mirror->cubin = std::move(m.cubin);
        a.mirror->compile_seconds = m.seconds;
      }
      a.cubin = std::move(r.cubin);
      a.compile_seconds = r.seconds;
      a.cubin_ready.store(true, std::memory_order_release);
    });
  }
  return a;
}

const Artifact& Program::for_launch(lower::Domain d, int device) const {
  if (tuning.jit_mode == 1) return loaded(d, device);
  if (tuning.jit_mode == 2) {
    if (Artifact* v = loaded_vm(d, device)) return *v;
    throw std::invalid_argument("program too large for the walk VM (jit_mode 2)");
  }
  Artifact& a = artifact(d, false);
  if (a.cubin_ready.load(std::memory_order_acquire)) return loaded(d, device);
  {
    // first use: compile in the background, answer this call with the VM
    std::lock_guard<std::mutex> lock(mu);
    const int k = static_cast<int>(d);
    if (!(jit_started >> k & 1u)) {
      jit_started |= 1u << k;
      jit_threads.emplace_back([this, d] {
        try {
          artifact(d, true);
        } catch (...) {
          // a failing compile resurfaces (and throws) on the next blocking use
        }
      });
    }
  }
  if (Artifact* v = loaded_vm(d, device)) return *v;
  return loaded(d, device);  // beyond the VM's slot file: wait for the compile
}

Artifact* Program::loaded_vm(lower::Domain d, int device) const {
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = vm_arts[static_cast<int>(d)];
  if (!slot) {
    const bool strict = d == lower::Domain::F64Strict || d == lower::Domain::Interval;
    if (!integer && (d == lower::Domain::I64 || d == lower::Domain::I64F)) {
      throw std::invalid_argument("pe_eval_i64 needs a program with int64 coefficients");
    }
    auto a = std::make_unique<Artifact>();
    a->vm = std::make_unique<VmImage>();
    a->vm->prog = integer ? lower::build_vm(strict ? lower::lower_strict(i->flat)
                                                   : lower::lower_fused(i->flat), d)
                          : lower::build_vm(strict ? lower::lower_strict(f->flat)
                                                   : lower::lower_fused(f->flat), d);
    const bool iv = d == lower::Domain::Interval;
    const bool i64 = d == lower::Domain::I64 || d == lower::Domain::I64F;
    a->image.domain = d;
    a->image.nvars = nvars;
    a->image.n_in = iv ? 2 * nvars : nvars;
    a->image.n_out = iv ? 2 : 1;
    a->image.has_flag = iv || i64;
    a->image.has_bounds = i64;
    a->image.entry = std::string("pe_vm_") + lower::domain_name(d);
    slot = std::move(a);
  }
  Artifact& a = *slot;
  if (a.vm->prog.nslots > pe_vm_max_slots()) return nullptr;
  auto it = a.vm->dev.find(device);
  if (it == a.vm->dev.end()) {
    const lower::VmProgram& p = a.vm->prog;
    VmDevice dv;
    auto upload = [](void** dst, const void* src, size_t bytes, const char* what) {
      check_cuda(cudaMalloc(dst, std::max<size_t>(bytes, 8)), what);
      if (bytes) check_cuda(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), what);
    };
    upload(&dv.code, p.code.data(), p.code.size() * 4, "VM program upload");
    upload(&dv.lo, p.lo.data(), p.lo.size() * 8, "VM coefficient upload");
    if (!p.hi.empty()) upload(&dv.hi, p.hi.data(), p.hi.size() * 8, "VM coefficient upload");
    a.vm->dev[device] = dv;
  }
  return &a;
}

namespace {
// Loads an artifact's cubin (context-independent library) and uploads its
// global-tier coefficients to `device`. Caller holds the program mutex.
void ensure_loaded(Artifact& a, int device);
}  // namespace

Artifact& Program::loaded(lower::Domain d, int device) const {
  Artifact& a = artifact(d, true);
  std::lock_guard<std::mutex> lock(mu);
  ensure_loaded(a, device);
  return a;
}

Artifact& Program::limb_artifact(std::uint32_t limbs, bool need_cubin) const {
  if (!integer) throw std::invalid_argument("multi-limb evaluation needs int64 coefficients");
  if (limbs < 1 || limbs > 8) throw std::invalid_argument("limbs must be 1..8");
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = limb_arts[limbs];
  if (!slot) {
    slot = std::make_unique<Artifact>();
    lower::KernelShape shape;
    shape.limbs = limbs;
    slot->image = lower::emit_ptx(lower::lower_fused(i->flat), lower::Domain::I64K, shape, tuning);
  }
  if (need_cubin && slot->cubin.empty()) {
    CompileResult r = compile_ptx_cached(slot->image.ptx, slot->image.entry);
    if (!r.ok) throw std::logic_error(r.log);
    slot->cubin = std::move(r.cubin);
    slot->compile_seconds = r.seconds;
  }
  return *slot;
}

Artifact& Program::loaded_limbs(std::uint32_t limbs, int device) const {
  Artifact& a = limb_artifact(limbs, true);
  std::lock_guard<std::mutex> lock(mu);
  ensure_loaded(a, device);
  return a;
}

std::uint32_t limbs_needed(const Program& p, const std::uint64_t* bounds) {
  const auto& T = p.i->terms;
  if (T.empty()) return 1;
  std::vector<double> lx(p.nvars);
  for (std::uint32_t v = 0; v < p.nvars; ++v) {
    lx[v] = std::log2(std::max<double>(1.0, static_cast<double>(bounds[v])));
  }
  double worst = 0.0, max_pow = 0.0;
  for (std::size_t t = 0; t < T.size(); ++t) {
    const double c = std::fabs(static_cast<double>(T.coefs[t]));
    double bits = c > 0 ? std::log2(c) : 0.0;
    for (std::uint32_t v = 0; v < p.nvars; ++v) {
      bits += T.exp(t, v) * lx[v];
      max_pow = std::max(max_pow, T.exp(t, v) * lx[v]);
    }
    worst = std::max(worst, bits);
  }
  // M <= T * max term; 1e-6 relative + 1 bit of slack for log2 rounding
  const double need = std::max(worst + std::log2(static_cast<double>(T.size())), max_pow) *
                          (1 + 1e-6) + 1.0;
  for (std::uint32_t k = 1; k <= 8; ++k) {
    if (need < 64.0 * k - 1.0) return k;
  }
  return 0;
}

Artifact::~Artifact() {
  for (auto& [dev, ptr] : global_coefs) {
    if (cudaSetDevice(dev) == cudaSuccess) cudaFree(ptr);
  }
  if (vm) {
    for (auto& [dev, dv] : vm->dev) {
      if (cudaSetDevice(dev) != cudaSuccess) continue;
      cudaFree(dv.code);
      cudaFree(dv.lo);
      if (dv.hi) cudaFree(dv.hi);
    }
  }
  if (library) cudaLibraryUnload(library);
}

WideFront::~WideFront() {
  for (auto& [key, d] : dev) {
    if (cudaSetDevice(key.first) != cudaSuccess) continue;
    for (void* p : {d.code, d.slot_off, d.slot_w, d.coef_off, d.coef_w, d.coef_words}) cudaFree(p);
  }
}

void Program::release() const {
  std::vector<std::thread> jobs;
  {
    std::lock_guard<std::mutex> lock(mu);
    jobs.swap(jit_threads);
  }
  for (auto& t : jobs) t.join();
  std::lock_guard<std::mutex> lock(mu);
  for (auto& a : artifacts) a.reset();
  for (auto& a : vm_arts) a.reset();
  limb_arts.clear();
  jit_started = 0;
}

namespace {
void ensure_loaded(Artifact& a, int device) {
  if (a.library) bind_functions(a, device);
  if (!a.library) {
    check_cuda(cudaLibraryLoadData(&a.library, a.cubin.data(), nullptr, nullptr, 0, nullptr,
                                   nullptr, 0),
               "cudaLibraryLoadData");
    check_cuda(cudaLibraryGetKernel(&a.kernel, a.library, a.image.entry.c_str()),
               "cudaLibraryGetKernel");
    if (!a.image.fix_entry.empty()) {
      check_cuda(cudaLibraryGetKernel(&a.fix_kernel, a.library, a.image.fix_entry.c_str()),
                 "cudaLibraryGetKernel(fix)");
    }
    if (!a.image.part_entry.empty()) {
      check_cuda(cudaLibraryGetKernel(&a.part_kernel, a.library, a.image.part_entry.c_str()),
                 "cudaLibraryGetKernel(part)");
    }
    bind_functions(a, device);
  }
  if (a.mirror) ensure_loaded(*a.mirror, device);
  if (!a.image.global_words.empty() && !a.global_coefs.count(device)) {
    void* p = nullptr;
    const size_t bytes = a.image.global_words.size() * 8;
    check_cuda(cudaMalloc(&p, bytes), "cudaMalloc(global coefficients)");
    check_cuda(cudaMemcpy(p, a.image.global_words.data(), bytes, cudaMemcpyHostToDevice),
               "cudaMemcpy(global coefficients)");
    a.global_coefs[device] = p;
  }
}
}  // namespace

}  // namespace polyeval::rt
