// C ABI (include/polyeval_b200.h) over the host front-end, the lowering /
// PTX emitter, the in-process JIT and the launch runtime.
//
// Reference mapping: pe_program_create = build/build_multivariate +
// compute_lazy_heights + compile (tree.cpp:159-227, eval.cpp:52-69);
// pe_eval_* = Evaluator<D>::evaluate over a batch (eval.hpp:74-90), one GPU
// thread per point instead of one call per point.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "front/compile.hpp"
#include "lower/ptx.hpp"
#include "lower/stream.hpp"
#include "polyeval_b200.h"
#include "runtime/jit.hpp"
#include "runtime/program.hpp"

extern "C" cudaError_t pe_launch_max_abs_i64(const long long* x, size_t n,
                                             unsigned long long* out, int sms,
                                             cudaStream_t stream);
extern "C" cudaError_t pe_measure_pipe_peak(int kind, int sms, double* ops_per_s);

struct pe_program {
  polyeval::rt::Program impl;
};

namespace polyeval::rt {

namespace {
thread_local std::string g_last_error;
std::atomic<std::uint64_t> g_launches{0};

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
  for (const auto& t : p.terms_i) {
    const u128 c = t.coefficient < 0 ? static_cast<u128>(-(t.coefficient + 1)) + 1
                                     : static_cast<u128>(t.coefficient);
    u128 term = c;
    for (std::uint32_t v = 0; v < p.nvars; ++v) {
      term = sat_mul(term, sat_pow(base[v], t.exponents[v]));
      max_e[v] = std::max(max_e[v], t.exponents[v]);
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

namespace {

std::vector<std::uint64_t> uniform_bounds(const Program& p, int limit_bits) {
  std::vector<std::uint64_t> out(p.nvars, UINT64_MAX);
  std::vector<bool> present(p.nvars, false);
  for (const auto& t : p.terms_i) {
    for (std::uint32_t v = 0; v < p.nvars; ++v) present[v] = present[v] || t.exponents[v] > 0;
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

}  // namespace

Artifact& Program::artifact(lower::Domain d, bool need_cubin) const {
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = artifacts[static_cast<int>(d)];
  if (!slot) {
    auto a = std::make_unique<Artifact>();
    const bool strict = d == lower::Domain::F64Strict || d == lower::Domain::Interval;
    if (integer) {
      auto s = strict ? lower::lower_strict(*prog_i) : lower::lower_fused(*prog_i);
      a->image = lower::emit_ptx(s, d);
    } else {
      if (d == lower::Domain::I64 || d == lower::Domain::I64F) {
        throw std::invalid_argument("pe_eval_i64 needs a program with int64 coefficients");
      }
      auto s = strict ? lower::lower_strict(*prog_f) : lower::lower_fused(*prog_f);
      a->image = lower::emit_ptx(s, d);
    }
    slot = std::move(a);
  }
  if (need_cubin && slot->cubin.empty()) {
    CompileResult r = compile_ptx_cached(slot->image.ptx, slot->image.entry);
    if (!r.ok) throw std::logic_error(r.log);
    slot->cubin = std::move(r.cubin);
    slot->compile_seconds = r.seconds;
  }
  return *slot;
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

std::size_t Program::slice_count() const {
  if (integer || nvars < 2) return 1;
  std::size_t k = 0;
  if (const char* e = std::getenv("PE_SLICES")) k = static_cast<std::size_t>(std::atoi(e));
  if (k == 0) {
    // measured on C4 (profiles/r1_slices_c4.txt): straight-line kernels
    // beyond a few thousand records pay for instruction fetch and register
    // pressure (power tables); ~2k records per slice
    k = stats.records >= 8192 ? std::clamp<std::size_t>(stats.records / 2100, 2, 16) : 1;
  }
  return std::max<std::size_t>(1, k);
}

std::vector<const Artifact*> Program::f64_kernels(int device) const {
  const std::size_t k = slice_count();
  if (k <= 1) return {&loaded(lower::Domain::F64, device)};
  std::lock_guard<std::mutex> lock(mu);
  if (!slices_planned) {
    // terms are in decreasing lexicographic order: equal outer exponents are
    // contiguous; cut at outer-exponent boundaries near multiples of T/k
    const auto& terms = poly_f->terms();
    const std::size_t T = terms.size();
    std::vector<std::size_t> cuts{0};
    for (std::size_t i = 1; i < T && cuts.size() < k; ++i) {
      if (terms[i].exponents[0] != terms[i - 1].exponents[0] && i * k >= cuts.size() * T) {
        cuts.push_back(i);
      }
    }
    cuts.push_back(T);
    std::vector<FunctionScheme> fs;
    for (const auto& d : scheme_descs) fs.push_back(scheme_from_desc(d));
    for (std::size_t s = 0; s + 1 < cuts.size(); ++s) {
      std::vector<Term<double>> part(terms.begin() + static_cast<std::ptrdiff_t>(cuts[s]),
                                     terms.begin() + static_cast<std::ptrdiff_t>(cuts[s + 1]));
      Polynomial<double> sp = Polynomial<double>::canonicalize(std::move(part), variables);
      EvaluationTree<double> t = build_multivariate(sp, std::span<const FunctionScheme>(fs));
      compute_lazy_heights(t);
      slice_progs.push_back(std::make_unique<CompiledProgram<double>>(compile(t)));
      auto a = std::make_unique<Artifact>();
      lower::KernelShape shape;
      shape.accumulate = s > 0;
      a->image = lower::emit_ptx(lower::lower_fused(*slice_progs.back()), lower::Domain::F64, shape);
      CompileResult r = compile_ptx_cached(a->image.ptx, a->image.entry);
      if (!r.ok) throw std::logic_error(r.log);
      a->cubin = std::move(r.cubin);
      a->compile_seconds = r.seconds;
      slice_arts.push_back(std::move(a));
    }
    slices_planned = true;
  }
  std::vector<const Artifact*> out;
  for (auto& a : slice_arts) {
    ensure_loaded(*a, device);
    out.push_back(a.get());
  }
  return out;
}

namespace {
void ensure_loaded(Artifact& a, int device) {
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
  }
  if (!a.image.global_words.empty() && !a.global_coefs.count(device)) {
    void* p = nullptr;
    const size_t bytes = a.image.global_words.size() * 8;
    check_cuda(cudaMalloc(&p, bytes), "cudaMalloc(global coefficients)");
    check_cuda(cudaMemcpy(p, a.image.global_words.data(), bytes, cudaMemcpyHostToDevice),
               "cudaMemcpy(global coefficients)");
    a.global_coefs[device] = p;
  }
}

// ------------------------------------------------------------------ launch

struct LaunchArgs {
  std::vector<std::uint64_t> ins, outs;
  std::uint64_t n = 0;
  std::uint64_t flag = 0;
  std::vector<std::uint64_t> bounds;
  // interval fast path: fixup list (u32 point indices), counter, capacity
  std::uint64_t list = 0, count = 0, cap = 0;
};

int sm_count(int device) {
  static std::mutex m;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lock(m);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int n = 0;
  check_cuda(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device), "SM count");
  cache[device] = n;
  return n;
}

void launch(const Artifact& a, int device, const LaunchArgs& la, cudaStream_t stream) {
  const auto& img = a.image;
  std::uint64_t gcoef = 0;
  if (!img.global_words.empty()) gcoef = reinterpret_cast<std::uint64_t>(a.global_coefs.at(device));
  std::vector<std::uint64_t> vals;
  vals.reserve(img.n_in + img.n_out + 4 + img.nvars);
  for (auto v : la.ins) vals.push_back(v);
  for (auto v : la.outs) vals.push_back(v);
  vals.push_back(la.n);
  vals.push_back(gcoef);
  if (img.has_flag) vals.push_back(la.flag);
  if (img.has_bounds) {
    for (std::uint32_t v = 0; v < img.nvars; ++v) vals.push_back(la.bounds.at(v));
  }
  if (img.interval_fast_path) {
    if (!la.list || !la.count) throw std::logic_error("interval fast path needs a fixup list");
    vals.push_back(la.list);
    vals.push_back(la.count);
    vals.push_back(la.cap);
    check_cuda(cudaMemsetAsync(reinterpret_cast<void*>(la.count), 0, sizeof(unsigned), stream),
               "cudaMemsetAsync(fixup count)");
  }
  std::vector<void*> args;
  for (auto& v : vals) args.push_back(&v);
  if (!img.param_words.empty()) args.push_back(const_cast<std::uint64_t*>(img.param_words.data()));
  // Small batches: shrink the CTA (the kernel reads its tile size from
  // %ntid; .maxntid is only an upper bound) until every SM has work.
  std::uint64_t block = img.block;
  const std::uint64_t want_ctas = 2 * static_cast<std::uint64_t>(sm_count(device));
  while (block > 64 && block % 64 == 0 && (la.n + block * img.lanes - 1) / (block * img.lanes) < want_ctas) {
    block /= 2;
  }
  const std::uint64_t tile = block * img.lanes;
  const std::uint64_t grid = (la.n + tile - 1) / tile;
  if (grid > 0x7fffffffull) throw std::invalid_argument("batch too large for one launch");
  check_cuda(cudaLaunchKernel(reinterpret_cast<const void*>(a.kernel),
                              dim3(static_cast<unsigned>(grid)), dim3(static_cast<unsigned>(block)),
                              args.data(), 0, stream),
             "cudaLaunchKernel(walk)");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (img.interval_fast_path) {
    // strict replay of the points the fast path could not prove; it reads
    // the list length on the device, so no host round trip in between
    const unsigned fix_grid = static_cast<unsigned>(
        std::min<std::uint64_t>(2 * static_cast<std::uint64_t>(sm_count(device)),
                                (la.cap + 127) / 128));
    check_cuda(cudaLaunchKernel(reinterpret_cast<const void*>(a.fix_kernel), dim3(fix_grid ? fix_grid : 1),
                                dim3(128), args.data(), 0, stream),
               "cudaLaunchKernel(fixup)");
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
}

enum class MemKind { Host, Device };

MemKind classify(const void* p, int* device) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return MemKind::Host;
  }
  if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
    if (device) *device = attr.device;
    return MemKind::Device;
  }
  return MemKind::Host;
}

// Deferred-check state of one caller stream: an accumulating status word and
// a grow-only full-capacity interval fixup list, both stream-ordered.
struct StreamState {
  unsigned* status = nullptr;
  void* list = nullptr;
  unsigned* count = nullptr;
  std::uint64_t list_cap = 0;
};

struct DeviceCtx {
  static constexpr int kSlots = 3;
  cudaStream_t streams[kSlots] = {};
  std::vector<void*> buffers[kSlots];  // per slot: arrays of `cap` bytes
  size_t cap = 0;
  std::mutex mu;  // serialises host-staged calls on a device
  int sms = 0;
  std::mutex state_mu;
  std::map<cudaStream_t, StreamState> states;

  StreamState& state(cudaStream_t s, std::uint64_t need_list) {
    std::lock_guard<std::mutex> lock(state_mu);
    StreamState& st = states[s];
    if (!st.status) {
      check_cuda(cudaMalloc(reinterpret_cast<void**>(&st.status), 2 * sizeof(unsigned)),
                 "cudaMalloc(status)");
      check_cuda(cudaMemsetAsync(st.status, 0, 2 * sizeof(unsigned), s), "cudaMemsetAsync(status)");
      st.count = st.status + 1;
    }
    if (need_list > st.list_cap) {
      if (st.list) {
        check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        cudaFree(st.list);
      }
      check_cuda(cudaMalloc(&st.list, 4 * need_list), "cudaMalloc(fixup list)");
      st.list_cap = need_list;
    }
    return st;
  }
};

DeviceCtx& device_ctx(int device) {
  static std::mutex g;
  static std::map<int, std::unique_ptr<DeviceCtx>> ctxs;
  std::lock_guard<std::mutex> lock(g);
  auto& c = ctxs[device];
  if (!c) {
    c = std::make_unique<DeviceCtx>();
    for (auto& s : c->streams) check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    check_cuda(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device),
               "cudaDeviceGetAttribute");
  }
  return *c;
}

void ensure_buffers(DeviceCtx& c, size_t arrays, size_t bytes) {
  if (c.cap >= bytes && c.buffers[0].size() >= arrays) return;
  for (auto& slot : c.buffers) {
    for (void* p : slot) cudaFree(p);
    slot.clear();
  }
  c.cap = std::max(bytes, c.cap);
  for (auto& slot : c.buffers) {
    for (size_t i = 0; i < arrays; ++i) {
      void* p = nullptr;
      check_cuda(cudaMalloc(&p, c.cap), "cudaMalloc(staging)");
      slot.push_back(p);
    }
  }
}

int resolve_device(const pe_exec* ex, const void* probe, MemKind* kind) {
  int ptr_dev = -1;
  *kind = classify(probe, &ptr_dev);
  if (ex && ex->device >= 0) {
    if (*kind == MemKind::Device && ptr_dev >= 0 && ptr_dev != ex->device) {
      throw std::invalid_argument("device pointer does not belong to exec->device");
    }
    return ex->device;
  }
  if (*kind == MemKind::Device && ptr_dev >= 0) return ptr_dev;
  int cur = 0;
  check_cuda(cudaGetDevice(&cur), "cudaGetDevice");
  return cur;
}

// Flag word for domain checks: device u32, read back after the launch.
struct Flag {
  unsigned* dev = nullptr;
  cudaStream_t stream = nullptr;
  explicit Flag(cudaStream_t s) : stream(s) {
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&dev), sizeof(unsigned), s), "cudaMallocAsync(flag)");
    check_cuda(cudaMemsetAsync(dev, 0, sizeof(unsigned), s), "cudaMemsetAsync(flag)");
  }
  unsigned read() {
    unsigned h = 0;
    check_cuda(cudaMemcpyAsync(&h, dev, sizeof h, cudaMemcpyDeviceToHost, stream), "flag D2H");
    check_cuda(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    return h;
  }
  ~Flag() {
    if (dev) cudaFreeAsync(dev, stream);
  }
};

/// Runs `la` over [0, n): device pointers in place on `stream`; host pointers
/// through a 3-slot chunked H2D / kernel / D2H pipeline on the device's own
/// streams (copy engines overlap the walk of the neighbouring chunk).
/// `flag_dev` (may be null) is the device status word for domain checks.
// Device scratch for the interval fixup list: one (list, count) per pipeline
// slot. Capacity 1/16 of the chunk by default (special points are rare); the
// full chunk after an overflow.
struct FixupLists {
  std::vector<void*> lists, counts;
  std::uint64_t cap = 0;
  std::vector<cudaStream_t> streams;
  FixupLists(const Artifact& a, size_t chunk, bool full, const std::vector<cudaStream_t>& ss) {
    if (!a.image.interval_fast_path || chunk == 0) return;
    cap = full ? chunk : std::min<std::uint64_t>(chunk, chunk / 16 + 4096);
    streams = ss;
    for (auto s : ss) {
      void *l = nullptr, *c = nullptr;
      check_cuda(cudaMallocAsync(&l, 4 * cap, s), "cudaMallocAsync(fixup list)");
      check_cuda(cudaMallocAsync(&c, 4, s), "cudaMallocAsync(fixup count)");
      lists.push_back(l);
      counts.push_back(c);
    }
  }
  void bind(LaunchArgs& la, size_t slot) const {
    if (lists.empty()) return;
    la.list = reinterpret_cast<std::uint64_t>(lists[slot]);
    la.count = reinterpret_cast<std::uint64_t>(counts[slot]);
    la.cap = cap;
  }
  ~FixupLists() {
    for (size_t i = 0; i < lists.size(); ++i) {
      cudaFreeAsync(lists[i], streams[i]);
      cudaFreeAsync(counts[i], streams[i]);
    }
  }
};

// `arts` run in order on each chunk (wide fp64 programs: slice 0 stores,
// later slices accumulate); inputs are staged once per chunk for all of them.
void run_batch(const std::vector<const Artifact*>& arts, int device, MemKind kind, size_t n,
               const std::vector<const void*>& ins, const std::vector<void*>& outs,
               const LaunchArgs& proto, cudaStream_t user_stream, bool sync,
               bool full_fixup = false, const std::vector<size_t>& out_base = {}) {
  const size_t elem = 8;
  const Artifact& a = *arts.front();  // interval programs have exactly one
  // art i writes outs[out_base[i] .. out_base[i] + n_out) (default: from 0)
  auto launch_all = [&](const LaunchArgs& la, cudaStream_t st) {
    for (size_t i = 0; i < arts.size(); ++i) {
      LaunchArgs l = la;
      const size_t b = out_base.empty() ? 0 : out_base[i];
      l.outs.assign(la.outs.begin() + static_cast<std::ptrdiff_t>(b),
                    la.outs.begin() + static_cast<std::ptrdiff_t>(b + arts[i]->image.n_out));
      launch(*arts[i], device, l, st);
    }
  };
  if (kind == MemKind::Device) {
    const size_t max_chunk = size_t{1} << 30;
    // a caller-bound list (deferred checks) is reused; otherwise per call
    const bool own_list = proto.list == 0;
    FixupLists fix(a, own_list ? std::min(n, max_chunk) : 0, full_fixup, {user_stream});
    for (size_t off = 0; off < n; off += max_chunk) {
      LaunchArgs la = proto;
      if (own_list) fix.bind(la, 0);
      la.n = std::min(max_chunk, n - off);
      la.ins.clear();
      la.outs.clear();
      for (auto p : ins) la.ins.push_back(reinterpret_cast<std::uint64_t>(static_cast<const char*>(p) + off * elem));
      for (auto p : outs) la.outs.push_back(reinterpret_cast<std::uint64_t>(static_cast<char*>(p) + off * elem));
      launch_all(la, user_stream);
    }
    if (sync) check_cuda(cudaStreamSynchronize(user_stream), "cudaStreamSynchronize");
    return;
  }
  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  const size_t chunk = std::clamp<size_t>(n / 8, size_t{1} << 18, size_t{1} << 23);
  ensure_buffers(c, ins.size() + outs.size(), chunk * elem);
  cudaEvent_t flag_ready = nullptr;
  if (proto.flag) {
    // the flag was initialised on user_stream: order the slots after it
    check_cuda(cudaEventCreateWithFlags(&flag_ready, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(flag_ready, user_stream), "cudaEventRecord");
    for (auto s : c.streams) check_cuda(cudaStreamWaitEvent(s, flag_ready, 0), "cudaStreamWaitEvent");
  }
  FixupLists fix(a, chunk, full_fixup,
                 std::vector<cudaStream_t>(c.streams, c.streams + DeviceCtx::kSlots));
  size_t k = 0;
  for (size_t off = 0; off < n; off += chunk, ++k) {
    const int slot = static_cast<int>(k % DeviceCtx::kSlots);
    cudaStream_t s = c.streams[slot];
    const size_t m = std::min(chunk, n - off);
    LaunchArgs la = proto;
    fix.bind(la, static_cast<size_t>(slot));
    la.n = m;
    la.ins.clear();
    la.outs.clear();
    for (size_t i = 0; i < ins.size(); ++i) {
      void* d = c.buffers[slot][i];
      check_cuda(cudaMemcpyAsync(d, static_cast<const char*>(ins[i]) + off * elem, m * elem,
                                 cudaMemcpyHostToDevice, s),
                 "cudaMemcpyAsync(H2D)");
      la.ins.push_back(reinterpret_cast<std::uint64_t>(d));
    }
    for (size_t o = 0; o < outs.size(); ++o) {
      la.outs.push_back(reinterpret_cast<std::uint64_t>(c.buffers[slot][ins.size() + o]));
    }
    launch_all(la, s);
    for (size_t o = 0; o < outs.size(); ++o) {
      check_cuda(cudaMemcpyAsync(static_cast<char*>(outs[o]) + off * elem,
                                 c.buffers[slot][ins.size() + o], m * elem, cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(D2H)");
    }
  }
  for (auto s : c.streams) check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  if (flag_ready) cudaEventDestroy(flag_ready);
}

void run_batch(const Artifact& a, int device, MemKind kind, size_t n,
               const std::vector<const void*>& ins, const std::vector<void*>& outs,
               const LaunchArgs& proto, cudaStream_t user_stream, bool sync,
               bool full_fixup = false) {
  run_batch(std::vector<const Artifact*>{&a}, device, kind, n, ins, outs, proto, user_stream, sync,
            full_fixup);
}

// ------------------------------------------------------------------ errors

pe_status fail(pe_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

template <typename Fn>
pe_status guarded(Fn&& fn) {
  try {
    g_last_error.clear();
    return fn();
  } catch (const CudaError& e) {
    return fail(PE_ECUDA, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(PE_EINVAL, e.what());
  } catch (const std::overflow_error& e) {
    return fail(PE_EOVERFLOW, e.what());
  } catch (const std::domain_error& e) {
    return fail(PE_EINVAL, e.what());
  } catch (const std::logic_error& e) {
    return fail(PE_ELOGIC, e.what());
  } catch (const std::bad_alloc&) {
    return fail(PE_ELOGIC, "out of host memory");
  } catch (const std::exception& e) {
    return fail(PE_ELOGIC, e.what());
  }
}

template <typename C>
void build_program(Program& p, const std::uint32_t* exps, const C* coeffs, size_t nterms,
                   std::uint32_t nvars, const pe_scheme_desc* schemes,
                   std::unique_ptr<EvaluationTree<C>>& tree,
                   std::unique_ptr<CompiledProgram<C>>& prog) {
  std::vector<std::string> vars;
  for (std::uint32_t v = 0; v < nvars; ++v) vars.push_back(nvars <= 3 ? std::string(1, "xyz"[v]) : "x" + std::to_string(v));
  std::vector<Term<C>> raw(nterms);
  for (size_t t = 0; t < nterms; ++t) {
    raw[t].coefficient = coeffs[t];
    raw[t].exponents.assign(exps + t * nvars, exps + (t + 1) * nvars);
  }
  Polynomial<C> poly = Polynomial<C>::canonicalize(std::move(raw), vars);
  std::vector<FunctionScheme> fs;
  for (std::uint32_t v = 0; v < nvars; ++v) {
    fs.push_back(scheme_from_desc(SchemeDesc{schemes[v].upper, schemes[v].lower, schemes[v].cutoff}));
  }
  EvaluationTree<C> t = nvars == 1 ? build(poly, fs[0], 0)
                                   : build_multivariate(poly, std::span<const FunctionScheme>(fs));
  compute_lazy_heights(t);
  prog = std::make_unique<CompiledProgram<C>>(compile(t));
  tree = std::make_unique<EvaluationTree<C>>(std::move(t));
  p.nterms = poly.terms().size();
  p.variables = vars;
  p.stats = program_stats(*prog);
  if constexpr (std::is_same_v<C, std::int64_t>) {
    p.terms_i = poly.terms();
  } else {
    p.poly_f = std::make_unique<Polynomial<double>>(poly);
  }
  for (std::uint32_t v = 0; v < nvars; ++v) {
    p.scheme_descs.push_back(SchemeDesc{schemes[v].upper, schemes[v].lower, schemes[v].cutoff});
  }
}

}  // namespace
}  // namespace polyeval::rt

using namespace polyeval;
using namespace polyeval::rt;

extern "C" {

const char* pe_last_error(void) { return g_last_error.c_str(); }
const char* pe_version(void) { return "polyeval-b200 0.1 (sm_100a)"; }
uint64_t pe_launch_count(void) { return g_launches.load(); }

pe_status pe_program_create(const uint32_t* exponents, const void* coeffs, size_t nterms,
                            uint32_t nvars, const pe_scheme_desc* schemes,
                            pe_coeff_type coeff_type, pe_program** out) {
  return guarded([&]() -> pe_status {
    if (!out) return fail(PE_EINVAL, "out is null");
    *out = nullptr;
    if (nvars == 0) return fail(PE_EINVAL, "nvars must be >= 1");
    if (!schemes) return fail(PE_EINVAL, "schemes is null");
    if (nterms > 0 && (!exponents || !coeffs)) return fail(PE_EINVAL, "terms are null");
    if (coeff_type != PE_COEFF_F64 && coeff_type != PE_COEFF_I64) {
      return fail(PE_EINVAL, "unknown coefficient type");
    }
    auto h = std::make_unique<pe_program>();
    Program& p = h->impl;
    p.nvars = nvars;
    p.integer = coeff_type == PE_COEFF_I64;
    if (p.integer) {
      build_program(p, exponents, static_cast<const std::int64_t*>(coeffs), nterms, nvars, schemes,
                    p.tree_i, p.prog_i);
      p.i64_uniform_bound = uniform_bounds(p, 63);
      p.i53_uniform_bound = uniform_bounds(p, 53);
    } else {
      const double* c = static_cast<const double*>(coeffs);
      for (size_t t = 0; t < nterms; ++t) {
        if (!std::isfinite(c[t])) return fail(PE_EINVAL, "coefficient is not finite");
      }
      build_program(p, exponents, c, nterms, nvars, schemes, p.tree_f, p.prog_f);
    }
    *out = h.release();
    return PE_OK;
  });
}

void pe_program_destroy(pe_program* program) {
  if (!program) return;
  for (auto& a : program->impl.artifacts) {
    if (!a) continue;
    for (auto& [dev, ptr] : a->global_coefs) {
      if (cudaSetDevice(dev) == cudaSuccess) cudaFree(ptr);
    }
    if (a->library) cudaLibraryUnload(a->library);
  }
  delete program;
}

pe_status pe_program_info(const pe_program* program, pe_program_info_t* info) {
  return guarded([&]() -> pe_status {
    if (!program || !info) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    std::memset(info, 0, sizeof *info);
    info->nvars = p.nvars;
    info->max_registers = p.stats.max_registers;
    info->records = p.stats.records;
    info->programs = p.stats.programs;
    info->walk_adds = p.stats.walk_adds;
    info->walk_muls = p.stats.walk_muls;
    info->power_muls = p.stats.power_muls;
    info->terms = p.nterms;
    auto fill = [&](const auto& prog) {
      info->register_count = prog.register_count;
      info->root_children = static_cast<uint32_t>(prog.root_child_ends.size());
      for (size_t v = 0; v < prog.exponent_sets.size() && v < 8; ++v) {
        info->exponent_set_sizes[v] = static_cast<uint32_t>(prog.exponent_sets[v].size());
      }
    };
    if (p.integer) fill(*p.prog_i); else fill(*p.prog_f);
    return PE_OK;
  });
}

pe_status pe_program_exponents(const pe_program* program, uint32_t v, uint32_t* out, size_t cap,
                               size_t* count) {
  return guarded([&]() -> pe_status {
    if (!program || !count) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    const auto& sets = p.integer ? p.prog_i->exponent_sets : p.prog_f->exponent_sets;
    if (v >= sets.size()) return fail(PE_EINVAL, "variable index out of range");
    const auto& e = sets[v].exponents;
    *count = e.size();
    for (size_t i = 0; i < e.size() && i < cap && out; ++i) out[i] = e[i];
    return PE_OK;
  });
}

pe_status pe_program_records(const pe_program* program, int32_t* out, size_t cap, size_t* count) {
  return guarded([&]() -> pe_status {
    if (!program || !count) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    auto dump = [&](const auto& prog) {
      *count = prog.records.size();
      for (size_t i = 0; i < prog.records.size() && (i + 1) * 5 <= cap && out; ++i) {
        const auto& r = prog.records[i];
        out[5 * i + 0] = r.power_slot ? static_cast<int32_t>(*r.power_slot) : -1;
        out[5 * i + 1] = static_cast<int32_t>(r.lazy_slot);
        out[5 * i + 2] = r.parent_slot ? static_cast<int32_t>(*r.parent_slot) : -1;
        out[5 * i + 3] = r.reads_register ? 1 : 0;
        out[5 * i + 4] = r.sub ? 1 : 0;
      }
    };
    if (p.integer) dump(*p.prog_i); else dump(*p.prog_f);
    return PE_OK;
  });
}

pe_status pe_program_dot(const pe_program* program, char* out, size_t cap, size_t* len) {
  return guarded([&]() -> pe_status {
    if (!program || !len) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    const std::string dot = p.integer ? to_dot(*p.tree_i) : to_dot(*p.tree_f);
    *len = dot.size();
    if (out && cap) {
      const size_t k = std::min(cap - 1, dot.size());
      std::memcpy(out, dot.data(), k);
      out[k] = '\0';
    }
    return PE_OK;
  });
}

static lower::Domain to_domain(int32_t d) {
  if (d < 0 || d > 4) throw std::invalid_argument("unknown domain");
  return static_cast<lower::Domain>(d);
}

pe_status pe_program_kernel_stats(const pe_program* program, int32_t domain, uint64_t* fp_ops,
                                  uint64_t* int_ops, uint64_t* ptx_bytes) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "null argument");
    const Artifact& a = program->impl.artifact(to_domain(domain), false);
    if (fp_ops) *fp_ops = a.image.fp_ops;
    if (int_ops) *int_ops = a.image.int_ops;
    if (ptx_bytes) *ptx_bytes = a.image.ptx.size();
    return PE_OK;
  });
}

pe_status pe_program_ptx(const pe_program* program, int32_t domain, char* out, size_t cap,
                         size_t* len) {
  return guarded([&]() -> pe_status {
    if (!program || !len) return fail(PE_EINVAL, "null argument");
    const Artifact& a = program->impl.artifact(to_domain(domain), false);
    *len = a.image.ptx.size();
    if (out && cap) {
      const size_t k = std::min(cap - 1, a.image.ptx.size());
      std::memcpy(out, a.image.ptx.data(), k);
      out[k] = '\0';
    }
    return PE_OK;
  });
}

pe_status pe_program_i64_bounds(const pe_program* program, uint64_t* bound63, uint64_t* bound53) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    if (!p.integer) return fail(PE_EINVAL, "program has fp64 coefficients");
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (bound63) bound63[v] = p.i64_uniform_bound[v];
      if (bound53) bound53[v] = p.i53_uniform_bound[v];
    }
    return PE_OK;
  });
}

pe_status pe_program_f64_slices(const pe_program* program, uint32_t* slices) {
  return guarded([&]() -> pe_status {
    if (!program || !slices) return fail(PE_EINVAL, "null argument");
    *slices = static_cast<uint32_t>(program->impl.slice_count());
    return PE_OK;
  });
}

pe_status pe_program_compile_only(const pe_program* program, int32_t domain, uint64_t* cubin_bytes) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "null argument");
    const Artifact& a = program->impl.artifact(to_domain(domain), true);
    if (cubin_bytes) *cubin_bytes = a.cubin.size();
    return PE_OK;
  });
}

pe_status pe_measure_peak(int32_t device, int32_t kind, double* ops_per_s, int32_t* sms) {
  return guarded([&]() -> pe_status {
    if (!ops_per_s || (kind != 0 && kind != 1)) return fail(PE_EINVAL, "bad argument");
    if (device >= 0) check_cuda(cudaSetDevice(device), "cudaSetDevice");
    int dev = 0, n_sm = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    check_cuda(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev), "attr");
    check_cuda(pe_measure_pipe_peak(kind, n_sm, ops_per_s), "pipe peak microbenchmark");
    g_launches.fetch_add(5, std::memory_order_relaxed);
    if (sms) *sms = n_sm;
    return PE_OK;
  });
}

pe_status pe_synchronize(const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (exec && exec->device >= 0) check_cuda(cudaSetDevice(exec->device), "cudaSetDevice");
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    DeviceCtx& c = device_ctx(dev);
    unsigned* status = nullptr;
    {
      std::lock_guard<std::mutex> lock(c.state_mu);
      auto it = c.states.find(s);
      if (it != c.states.end()) status = it->second.status;
    }
    if (!status) return PE_OK;
    unsigned h = 0;
    check_cuda(cudaMemcpy(&h, status, sizeof h, cudaMemcpyDeviceToHost), "status D2H");
    if (h) check_cuda(cudaMemset(status, 0, sizeof h), "status reset");
    if (h & 2) return fail(PE_EINVAL, "invalid interval endpoints (NaN or lo > hi) in a deferred call");
    if (h & 1) {
      return fail(PE_EOVERFLOW,
                  "a coordinate exceeded the proven int64 bound in a deferred call "
                  "(re-run with synchronous checks to derive the batch bounds)");
    }
    if (h & 4) return fail(PE_ELOGIC, "interval fixup list overflow in a deferred call");
    return PE_OK;
  });
}

pe_status pe_eval_f64(const pe_program* program, const double* const* coords, size_t n,
                      double* out, const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    if (n == 0) return PE_OK;
    if (!coords || !out) return fail(PE_EINVAL, "null buffer");
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    const bool strict = exec && exec->strict_f64;
    MemKind kind;
    const int dev = resolve_device(exec, out, &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    const std::vector<const Artifact*> arts =
        strict ? std::vector<const Artifact*>{&p.loaded(lower::Domain::F64Strict, dev)}
               : p.f64_kernels(dev);
    std::vector<const void*> ins(coords, coords + p.nvars);
    std::vector<void*> outs{out};
    LaunchArgs la;
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    run_batch(arts, dev, kind, n, ins, outs, la, s, exec && exec->synchronize);
    return PE_OK;
  });
}

pe_status pe_eval_f64_multi(const pe_program* const* programs, size_t k,
                            const double* const* coords, size_t n, double* const* outs,
                            const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!programs || k == 0) return fail(PE_EINVAL, "no programs");
    if (n == 0) return PE_OK;
    if (!coords || !outs) return fail(PE_EINVAL, "null buffer");
    const std::uint32_t nv = programs[0] ? programs[0]->impl.nvars : 0;
    for (size_t j = 0; j < k; ++j) {
      if (!programs[j] || !outs[j]) return fail(PE_EINVAL, "null program or output");
      if (programs[j]->impl.nvars != nv) return fail(PE_EINVAL, "programs differ in variable count");
    }
    for (uint32_t v = 0; v < nv; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    MemKind kind;
    const int dev = resolve_device(exec, outs[0], &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    std::vector<const Artifact*> arts;
    std::vector<size_t> base;
    for (size_t j = 0; j < k; ++j) {
      for (const Artifact* a : programs[j]->impl.f64_kernels(dev)) {
        arts.push_back(a);
        base.push_back(j);
      }
    }
    std::vector<const void*> ins(coords, coords + nv);
    std::vector<void*> o(outs, outs + k);
    LaunchArgs la;
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    run_batch(arts, dev, kind, n, ins, o, la, s, exec && exec->synchronize, false, base);
    return PE_OK;
  });
}

pe_status pe_eval_interval(const pe_program* program, const double* const* lo,
                           const double* const* hi, size_t n, double* out_lo, double* out_hi,
                           const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    if (n == 0) return PE_OK;
    if (!lo || !hi || !out_lo || !out_hi) return fail(PE_EINVAL, "null buffer");
    std::vector<const void*> ins;
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!lo[v] || !hi[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
      ins.push_back(lo[v]);
      ins.push_back(hi[v]);
    }
    MemKind kind;
    const int dev = resolve_device(exec, out_lo, &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    const Artifact& a = p.loaded(lower::Domain::Interval, dev);
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    if (exec && exec->deferred_checks && kind == MemKind::Device) {
      // no host round trip: status accumulates on the stream, the fixup
      // list has full capacity (cannot overflow)
      StreamState& st = device_ctx(dev).state(s, std::min<size_t>(n, size_t{1} << 30));
      LaunchArgs la;
      la.flag = reinterpret_cast<std::uint64_t>(st.status);
      if (a.image.interval_fast_path) {
        la.list = reinterpret_cast<std::uint64_t>(st.list);
        la.count = reinterpret_cast<std::uint64_t>(st.count);
        la.cap = st.list_cap;
      }
      run_batch(a, dev, kind, n, ins, {out_lo, out_hi}, la, s, false);
      return PE_OK;
    }
    for (int attempt = 0; attempt < 2; ++attempt) {
      Flag flag(s);
      LaunchArgs la;
      la.flag = reinterpret_cast<std::uint64_t>(flag.dev);
      run_batch(a, dev, kind, n, ins, {out_lo, out_hi}, la, s, false, attempt == 1);
      const unsigned f = flag.read();
      if (f & 2) return fail(PE_EINVAL, "invalid interval endpoints (NaN or lo > hi)");
      if (!(f & 4)) return PE_OK;
      // more points needed the strict replay than the fixup list held:
      // re-run with a list as large as the batch (cannot overflow)
    }
    return fail(PE_ELOGIC, "interval fixup list overflowed at full capacity");
  });
}

pe_status pe_eval_i64(const pe_program* program, const int64_t* const* coords, size_t n,
                      int64_t* out, const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    if (!p.integer) return fail(PE_EINVAL, "pe_eval_i64 needs a program with int64 coefficients");
    if (n == 0) return PE_OK;
    if (!coords || !out) return fail(PE_EINVAL, "null buffer");
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    MemKind kind;
    const int dev = resolve_device(exec, out, &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    std::vector<const void*> ins(coords, coords + p.nvars);
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    const bool caller_bounds = exec && exec->i64_bounds;
    const bool force_int = exec && exec->i64_int_pipe;
    std::vector<std::uint64_t> bounds =
        caller_bounds ? std::vector<std::uint64_t>(exec->i64_bounds, exec->i64_bounds + p.nvars)
                      : p.i64_uniform_bound;
    if (caller_bounds && !i64_proof_holds(p, bounds.data())) {
      return fail(PE_EOVERFLOW, "int64 range proof fails for the asserted coordinate bounds");
    }
    if (exec && exec->deferred_checks && kind == MemKind::Device) {
      // no host round trip: the bound check writes the stream's status word
      const std::vector<std::uint64_t> b53 = caller_bounds ? bounds : p.i53_uniform_bound;
      const bool tier53 = !force_int && i64_proof_holds(p, b53.data(), 53);
      const Artifact& a =
          p.loaded(tier53 ? lower::Domain::I64F : lower::Domain::I64, dev);
      StreamState& st = device_ctx(dev).state(s, 0);
      LaunchArgs la;
      la.flag = reinterpret_cast<std::uint64_t>(st.status);
      la.bounds = tier53 ? b53 : bounds;
      run_batch(a, dev, kind, n, ins, {out}, la, s, false);
      return PE_OK;
    }
    // Tier 1: every intermediate provably below 2^53 -> exact integer
    // arithmetic on the FP64 FMA pipe (one DFMA per record instead of a
    // 3-IMAD 64-bit multiply-add). Same bits as the int64 kernel.
    const std::vector<std::uint64_t> b53 = caller_bounds ? bounds : p.i53_uniform_bound;
    if (!force_int && i64_proof_holds(p, b53.data(), 53)) {
      const Artifact& af = p.loaded(lower::Domain::I64F, dev);
      Flag flag(s);
      LaunchArgs la;
      la.flag = reinterpret_cast<std::uint64_t>(flag.dev);
      la.bounds = b53;
      run_batch(af, dev, kind, n, ins, {out}, la, s, false);
      if (flag.read() == 0) return PE_OK;
      if (caller_bounds) {
        return fail(PE_EOVERFLOW, "a coordinate exceeds the asserted int64 bound");
      }
    }
    // Tier 2: int64 multiply-adds, wrap-free by the 2^63 proof.
    const Artifact& a = p.loaded(lower::Domain::I64, dev);
    for (int attempt = 0; attempt < 2; ++attempt) {
      Flag flag(s);
      LaunchArgs la;
      la.flag = reinterpret_cast<std::uint64_t>(flag.dev);
      la.bounds = bounds;
      run_batch(a, dev, kind, n, ins, {out}, la, s, false);
      if (flag.read() == 0) return PE_OK;
      if (caller_bounds || attempt == 1) break;
      // Some coordinate exceeded the uniform bound: derive the batch's real
      // per-variable maxima and retry if the proof still holds.
      std::vector<std::uint64_t> actual(p.nvars, 0);
      if (kind == MemKind::Device) {
        unsigned long long* dmax = nullptr;
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&dmax), 8 * p.nvars, s), "cudaMallocAsync");
        check_cuda(cudaMemsetAsync(dmax, 0, 8 * p.nvars, s), "cudaMemsetAsync");
        const int sms = device_ctx(dev).sms;
        for (uint32_t v = 0; v < p.nvars; ++v) {
          check_cuda(pe_launch_max_abs_i64(reinterpret_cast<const long long*>(coords[v]), n, dmax + v,
                                           sms, s),
                     "max_abs_i64");
          g_launches.fetch_add(1, std::memory_order_relaxed);
        }
        check_cuda(cudaMemcpyAsync(actual.data(), dmax, 8 * p.nvars, cudaMemcpyDeviceToHost, s), "D2H");
        check_cuda(cudaFreeAsync(dmax, s), "cudaFreeAsync");
        check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      } else {
        for (uint32_t v = 0; v < p.nvars; ++v) {
          std::uint64_t m = 0;
          for (size_t i = 0; i < n; ++i) {
            const int64_t x = coords[v][i];
            const std::uint64_t ax = x < 0 ? 0ull - static_cast<std::uint64_t>(x) : static_cast<std::uint64_t>(x);
            m = std::max(m, ax);
          }
          actual[v] = m;
        }
      }
      if (!i64_proof_holds(p, actual.data())) break;
      bounds = actual;
    }
    return fail(PE_EOVERFLOW,
                "int64 evaluation could overflow for these coordinates (no CPU fallback)");
  });
}

}  // extern "C"
