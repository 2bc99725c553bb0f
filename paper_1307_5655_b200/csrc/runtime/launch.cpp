// Launch runtime: kernel launches, host-staged pipelines, per-device and
// per-stream state. See runtime/launch.hpp.
#include "runtime/launch.hpp"

#include <cuda.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <thread>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>

namespace polyeval::rt {

namespace {
// Driver entry points through the runtime (no libcuda link dependency).
using KernelGetFunctionFn = CUresult (*)(CUfunction*, CUkernel);
using OccupancyFn = CUresult (*)(int*, CUfunction, int, size_t);
using LaunchKernelFn = CUresult (*)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                                    unsigned, unsigned, CUstream, void**, void**);
struct Driver {
  KernelGetFunctionFn get_function = nullptr;
  LaunchKernelFn launch = nullptr;
  OccupancyFn occupancy = nullptr;
  Driver() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuKernelGetFunction", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      get_function = reinterpret_cast<KernelGetFunctionFn>(p);
    }
    if (cudaGetDriverEntryPoint("cuLaunchKernel", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      launch = reinterpret_cast<LaunchKernelFn>(p);
    }
    if (cudaGetDriverEntryPoint("cuOccupancyMaxActiveBlocksPerMultiprocessor", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      occupancy = reinterpret_cast<OccupancyFn>(p);
    }
    cudaGetLastError();
  }
};
const Driver& driver() {
  static const Driver d;
  return d;
}

// One launch: the cached CUfunction through cuLaunchKernel (measured 2.4 us
// of host time vs 3.8 us for cudaLaunchKernel on a library kernel,
// scripts/launch_overhead.cpp), else the runtime path.
void launch_one(cudaKernel_t k, void* fn, dim3 grid, dim3 block, void** args, cudaStream_t st,
                const char* what) {
  if (fn && driver().launch) {
    const CUresult r = driver().launch(static_cast<CUfunction>(fn), grid.x, grid.y, grid.z, block.x,
                                       block.y, block.z, 0, reinterpret_cast<CUstream>(st), args,
                                       nullptr);
    if (r != CUDA_SUCCESS) throw CudaError(std::string(what) + ": CUresult " + std::to_string(r));
    return;
  }
  check_cuda(cudaLaunchKernel(reinterpret_cast<const void*>(k), grid, block, args, 0, st), what);
}
}  // namespace

void bind_functions(Artifact& a, int device) {
  if (device < 0 || device >= Artifact::kMaxDevices || !driver().get_function) return;
  if (!a.fn[device] && a.kernel) {
    CUfunction f = nullptr;
    if (driver().get_function(&f, reinterpret_cast<CUkernel>(a.kernel)) == CUDA_SUCCESS) a.fn[device] = f;
  }
  if (!a.fix_fn[device] && a.fix_kernel) {
    CUfunction f = nullptr;
    if (driver().get_function(&f, reinterpret_cast<CUkernel>(a.fix_kernel)) == CUDA_SUCCESS) {
      a.fix_fn[device] = f;
    }
  }
  if (!a.part_fn[device] && a.part_kernel) {
    CUfunction f = nullptr;
    if (driver().get_function(&f, reinterpret_cast<CUkernel>(a.part_kernel)) == CUDA_SUCCESS) {
      a.part_fn[device] = f;
    }
  }
}

std::atomic<std::uint64_t>& launch_counter() {
  static std::atomic<std::uint64_t> n{0};
  return n;
}


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

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// pool; with its default release threshold (0) every synchronisation hands
// the memory back to the driver and the next call maps it again (C5: 400 MB
// per 1e8-interval call, ~4 ms). Keep it pooled instead.
void keep_pool_memory(int device) {
  static std::mutex m;
  static std::set<int> done;
  std::lock_guard<std::mutex> lock(m);
  if (!done.insert(device).second) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    std::uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}

extern "C" cudaError_t pe_launch_vm(int domain, const std::uint32_t* code, std::uint32_t nops,
                                    std::uint32_t nslots, std::uint32_t result,
                                    const std::uint64_t* lo, const std::uint64_t* hi,
                                    std::uint32_t nvars, const void* const* in, void* out0,
                                    void* out1, unsigned long long n, unsigned* flag,
                                    const unsigned long long* bounds, cudaStream_t stream);

extern "C" cudaError_t pe_launch_classify_intervals(const double* lo, const double* hi,
                                                    unsigned long long n, unsigned* idx,
                                                    unsigned* counts, unsigned* fix_list,
                                                    unsigned* fix_count,
                                                    unsigned long long fix_cap, unsigned* flag,
                                                    cudaStream_t stream);

namespace {
// Kernel argument values of one module, in entry_text's parameter order
// (the parameter-tier coefficient array is appended by the caller).
std::vector<std::uint64_t> arg_values(const Artifact& a, int device, const LaunchArgs& la,
                                      std::uint64_t pidx, std::uint64_t pcnt,
                                      std::uint64_t scratch = 0) {
  const auto& img = a.image;
  std::uint64_t gcoef = 0;
  if (!img.global_words.empty()) gcoef = reinterpret_cast<std::uint64_t>(a.global_coefs.at(device));
  std::vector<std::uint64_t> vals;
  vals.reserve(img.n_in + img.n_out + 8 + img.nvars);
  for (auto v : la.ins) vals.push_back(v);
  for (auto v : la.outs) vals.push_back(v);
  vals.push_back(la.n);
  vals.push_back(gcoef);
  if (img.has_flag) vals.push_back(la.flag);
  if (img.has_bounds) {
    for (std::uint32_t v = 0; v < img.nvars; ++v) vals.push_back(la.bounds.at(v));
  }
  if (img.interval_fast_path) {
    vals.push_back(la.list);
    vals.push_back(la.count);
    vals.push_back(la.cap);
  }
  if (img.iv_partition) {
    vals.push_back(pidx);
    vals.push_back(pcnt);
  }
  if (img.sections > 1) vals.push_back(scratch);
  return vals;
}

std::vector<void*> arg_ptrs(const Artifact& a, std::vector<std::uint64_t>& vals) {
  std::vector<void*> args;
  for (auto& v : vals) args.push_back(&v);
  if (!a.image.param_words.empty()) {
    args.push_back(const_cast<std::uint64_t*>(a.image.param_words.data()));
  }
  return args;
}

}  // namespace

namespace {
// Persistent sectioned kernel: one wave of CTAs (occupancy x SMs, at most
// one per group of tiles) and its stream-ordered scratch slots.
void launch_grouped(const Artifact& a, int device, const LaunchArgs& la, cudaStream_t stream) {
  const auto& img = a.image;
  const bool dev_ok = device >= 0 && device < Artifact::kMaxDevices;
  void* fn = dev_ok ? a.fn[device] : nullptr;
  int per_sm = 1;
  if (fn && driver().occupancy) {
    int k = 0;
    if (driver().occupancy(&k, static_cast<CUfunction>(fn), static_cast<int>(img.block), 0) ==
            CUDA_SUCCESS && k > 0) {
      per_sm = k;
    }
  }
  const std::uint64_t tile = static_cast<std::uint64_t>(img.block) * img.lanes;
  const std::uint64_t tiles = (la.n + tile - 1) / tile;
  const std::uint64_t groups = (tiles + img.group_tiles - 1) / img.group_tiles;
  const std::uint64_t grid =
      std::max<std::uint64_t>(1, std::min<std::uint64_t>(groups, static_cast<std::uint64_t>(per_sm) * sm_count(device)));
  const size_t bytes = static_cast<size_t>(grid * img.group_tiles * img.scratch_values * tile * 8);
  keep_pool_memory(device);
  void* scratch = nullptr;
  check_cuda(cudaMallocAsync(&scratch, bytes, stream), "cudaMallocAsync(section scratch)");
  std::vector<std::uint64_t> vals =
      arg_values(a, device, la, 0, 0, reinterpret_cast<std::uint64_t>(scratch));
  std::vector<void*> args = arg_ptrs(a, vals);
  launch_one(a.kernel, fn, dim3(static_cast<unsigned>(grid)), dim3(img.block), args.data(), stream,
             "launch(sectioned walk)");
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  check_cuda(cudaFreeAsync(scratch, stream), "cudaFreeAsync(section scratch)");
}
}  // namespace

void launch(const Artifact& a, int device, const LaunchArgs& la, cudaStream_t stream) {
  const auto& img = a.image;
  if (a.vm) {
    const lower::VmProgram& p = a.vm->prog;
    const VmDevice& dv = a.vm->dev.at(device);
    std::vector<const void*> in;
    for (auto v : la.ins) in.push_back(reinterpret_cast<const void*>(v));
    check_cuda(pe_launch_vm(static_cast<int>(p.domain), static_cast<const std::uint32_t*>(dv.code),
                            p.nops, p.nslots, p.result, static_cast<const std::uint64_t*>(dv.lo),
                            static_cast<const std::uint64_t*>(dv.hi), p.nvars, in.data(),
                            reinterpret_cast<void*>(la.outs.at(0)),
                            la.outs.size() > 1 ? reinterpret_cast<void*>(la.outs[1]) : nullptr, la.n,
                            reinterpret_cast<unsigned*>(la.flag),
                            la.bounds.empty() ? nullptr
                                              : reinterpret_cast<const unsigned long long*>(la.bounds.data()),
                            stream),
               "launch(walk VM)");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    return;
  }
  if (img.sections > 1) {
    launch_grouped(a, device, la, stream);
    return;
  }
  if (img.interval_fast_path) {
    if (!la.list || !la.count) throw std::logic_error("interval fast path needs a fixup list");
    check_cuda(cudaMemsetAsync(reinterpret_cast<void*>(la.count), 0, sizeof(unsigned), stream),
               "cudaMemsetAsync(fixup count)");
  }
  // below ~64K intervals the extra launches outweigh the cheaper walk
  const bool part = a.partitioned() && la.n <= 0xffffffffull && la.n >= img.iv_partition_min;
  // one-pass sign split (iv_partition 3): classify + pack + walk in one kernel
  const bool split = img.iv_partition == 3 && la.n <= 0xffffffffull && la.n >= img.iv_partition_min;
  void* scratch = nullptr;  // partition: n u32 point indices + 2 u32 list lengths
  if (part) {
    keep_pool_memory(device);
    check_cuda(cudaMallocAsync(&scratch, 4 * la.n + 8, stream), "cudaMallocAsync(partition)");
  }
  const std::uint64_t pidx = reinterpret_cast<std::uint64_t>(scratch);
  const std::uint64_t pcnt = part ? pidx + 4 * la.n : 0;
  std::vector<std::uint64_t> vals = arg_values(a, device, la, pidx, pcnt);
  std::vector<void*> args = arg_ptrs(a, vals);
  const bool dev_ok = device >= 0 && device < Artifact::kMaxDevices;
  if (part) {
    // sign partition: classify, then the x > 0 entry of this module and the
    // x < 0 entry of the mirror module, each over its list (device lengths);
    // intervals touching zero go straight to the fixup list
    check_cuda(cudaMemsetAsync(reinterpret_cast<void*>(pcnt), 0, 8, stream),
               "cudaMemsetAsync(partition counts)");
    check_cuda(pe_launch_classify_intervals(
                   reinterpret_cast<const double*>(la.ins.at(0)),
                   reinterpret_cast<const double*>(la.ins.at(1)), la.n,
                   reinterpret_cast<unsigned*>(pidx), reinterpret_cast<unsigned*>(pcnt),
                   reinterpret_cast<unsigned*>(la.list), reinterpret_cast<unsigned*>(la.count),
                   la.cap, reinterpret_cast<unsigned*>(la.flag), stream),
               "launch(classify)");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    const std::uint64_t tile = static_cast<std::uint64_t>(img.block) * img.lanes;
    const std::uint64_t grid = (la.n + tile - 1) / tile;
    if (grid > 0x7fffffffull) throw std::invalid_argument("batch too large for one launch");
    launch_one(a.part_kernel, dev_ok ? a.part_fn[device] : nullptr, dim3(static_cast<unsigned>(grid)),
               dim3(img.block), args.data(), stream, "launch(walk x>0)");
    const Artifact& m = *a.mirror;
    std::vector<std::uint64_t> mvals = arg_values(m, device, la, pidx, pcnt);
    std::vector<void*> margs = arg_ptrs(m, mvals);
    const std::uint64_t mtile = static_cast<std::uint64_t>(m.image.block) * m.image.lanes;
    launch_one(m.kernel, dev_ok ? m.fn[device] : nullptr,
               dim3(static_cast<unsigned>((la.n + mtile - 1) / mtile)), dim3(m.image.block),
               margs.data(), stream, "launch(walk x<0)");
    launch_counter().fetch_add(2, std::memory_order_relaxed);
  }
  // Small batches: shrink the CTA (the kernel reads its tile size from
  // %ntid; .maxntid is only an upper bound) until every SM has work. Looped
  // kernels (tiny code, no instruction-fetch sharing to lose) split finer,
  // which evens out the per-SM load of a batch of a few CTAs per SM.
  std::uint64_t block = img.block;
  const std::uint64_t want_ctas = (img.chain_loops ? 8 : 2) * static_cast<std::uint64_t>(sm_count(device));
  while (block > 64 && block % 64 == 0 && (la.n + block * img.lanes - 1) / (block * img.lanes) < want_ctas) {
    block /= 2;
  }
  const std::uint64_t tile = block * img.lanes;
  const std::uint64_t grid = (la.n + tile - 1) / tile;
  if (grid > 0x7fffffffull) throw std::invalid_argument("batch too large for one launch");
  if (split) {
    // persistent: 1024 threads per SM stride over the tiles
    const std::uint64_t stiles = (la.n + img.block - 1) / img.block;
    const std::uint64_t sgrid =
        std::min<std::uint64_t>(stiles, static_cast<std::uint64_t>(1024 / img.block) * sm_count(device));
    launch_one(a.part_kernel, dev_ok ? a.part_fn[device] : nullptr,
               dim3(static_cast<unsigned>(sgrid ? sgrid : 1)), dim3(img.block), args.data(), stream,
               "launch(walk split)");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
  } else if (!part) {
    launch_one(a.kernel, dev_ok ? a.fn[device] : nullptr, dim3(static_cast<unsigned>(grid)),
               dim3(static_cast<unsigned>(block)), args.data(), stream, "launch(walk)");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
  }
  if (img.interval_fast_path) {
    // strict replay of the points the fast path could not prove; it reads
    // the list length on the device, so no host round trip in between
    // one thread per list slot (the kernel has no grid-stride loop); threads
    // past the device-side count exit at once
    const std::uint64_t fb = img.fix_block;
    // (a caller-bound list can be larger than this call's batch)
    std::uint64_t fix_ctas = (std::min(la.cap, la.n) + fb - 1) / fb;
    if (img.fix_persistent) {
      fix_ctas = std::min<std::uint64_t>(fix_ctas, static_cast<std::uint64_t>(img.fix_ctas_per_sm) *
                                                       sm_count(device));
    }
    const unsigned fix_grid = static_cast<unsigned>(std::min<std::uint64_t>(0x7fffffffull, fix_ctas));
    launch_one(a.fix_kernel, dev_ok ? a.fix_fn[device] : nullptr,
               dim3(fix_grid ? fix_grid : 1), dim3(static_cast<unsigned>(fb)), args.data(), stream,
               "launch(fixup)");
    launch_counter().fetch_add(1, std::memory_order_relaxed);
  }
  if (scratch) check_cuda(cudaFreeAsync(scratch, stream), "cudaFreeAsync(partition)");
}


MemKind classify(const void* p, int* device, bool* pinned) {
  if (pinned) *pinned = false;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return MemKind::Host;
  }
  if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
    if (device) *device = attr.device;
    return MemKind::Device;
  }
  if (pinned) *pinned = attr.type == cudaMemoryTypeHost;
  return MemKind::Host;
}

DeviceCtx& device_ctx(int device) {
  static std::mutex g;
  static std::map<int, std::unique_ptr<DeviceCtx>> ctxs;
  std::lock_guard<std::mutex> lock(g);
  auto& c = ctxs[device];
  if (!c) {
    c = std::make_unique<DeviceCtx>();
    for (int i = 0; i < DeviceCtx::kMaxSlots; ++i) {
      check_cuda(cudaStreamCreateWithFlags(&c->streams[i], cudaStreamNonBlocking), "cudaStreamCreate");
      check_cuda(cudaEventCreateWithFlags(&c->done[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    check_cuda(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device),
               "cudaDeviceGetAttribute");
  }
  return *c;
}

Staging staging_of(const pe_exec* ex) {
  Staging s;
  if (ex) {
    s.chunk = static_cast<std::size_t>(ex->stage_chunk);
    s.slots = ex->stage_slots;
  }
  return s;
}

namespace {
void ensure_buffers(DeviceCtx& c, int slots, size_t arrays, size_t bytes, bool pinned) {
  const bool dev_ok = c.cap >= bytes && c.buffers[slots - 1].size() >= arrays;
  if (!dev_ok) {
    for (auto& slot : c.buffers) {
      for (void* p : slot) cudaFree(p);
      slot.clear();
    }
    c.cap = std::max(bytes, c.cap);
    for (int k = 0; k < DeviceCtx::kMaxSlots && k < slots; ++k) {
      for (size_t i = 0; i < arrays; ++i) {
        void* p = nullptr;
        check_cuda(cudaMalloc(&p, c.cap), "cudaMalloc(staging)");
        c.buffers[k].push_back(p);
      }
    }
  }
  if (!pinned) return;
  if (c.pinned_cap >= bytes && c.pinned[slots - 1].size() >= arrays) return;
  for (auto& slot : c.pinned) {
    for (void* p : slot) cudaFreeHost(p);
    slot.clear();
  }
  c.pinned_cap = std::max(bytes, c.pinned_cap);
  for (int k = 0; k < slots; ++k) {
    for (size_t i = 0; i < arrays; ++i) {
      void* p = nullptr;
      check_cuda(cudaHostAlloc(&p, c.pinned_cap, cudaHostAllocPortable), "cudaHostAlloc(staging)");
      c.pinned[k].push_back(p);
    }
  }
}

// Host memcpy of large pageable buffers into / out of page-locked staging:
// split over a few persistent worker threads (one thread's memcpy, ~10 GB/s,
// would be slower than PCIe).
class CopyPool {
 public:
  static CopyPool& get() {
    // never destroyed: its workers block on cv_ until the process ends
    static CopyPool* pool = new CopyPool;
    return *pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    const size_t parts = std::min<size_t>(workers_.size() + 1, std::max<size_t>(1, bytes >> 20));
    if (parts <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const size_t per = (bytes + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lock(mu_);
      for (size_t k = 1; k < parts; ++k) {
        const size_t lo = k * per, len = std::min(bytes, lo + per) - lo;
        jobs_.push_back({static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, len});
      }
      pending_ += parts - 1;
    }
    cv_.notify_all();
    std::memcpy(dst, src, std::min(per, bytes));
    std::unique_lock<std::mutex> lock(mu_);
    idle_.wait(lock, [&] { return pending_ == 0; });
  }

 private:
  struct Job {
    char* dst;
    const char* src;
    size_t len;
  };
  CopyPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    for (unsigned i = 0; i < std::min(7u, hw - 1); ++i) {
      workers_.emplace_back([this] { run(); });
      workers_.back().detach();
    }
  }
  void run() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return !jobs_.empty(); });
        j = jobs_.front();
        jobs_.pop_front();
      }
      std::memcpy(j.dst, j.src, j.len);
      std::lock_guard<std::mutex> lock(mu_);
      if (--pending_ == 0) idle_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, idle_;
  std::deque<Job> jobs_;
  size_t pending_ = 0;
  std::vector<std::thread> workers_;
};
}  // namespace

void copy_to_host(void* dst, const void* dev_src, size_t bytes, int device, cudaStream_t stream) {
  constexpr size_t kChunk = size_t{8} << 20;
  bool pinned = false;
  classify(dst, nullptr, &pinned);
  if (pinned || bytes < 2 * kChunk) {
    check_cuda(cudaMemcpyAsync(dst, dev_src, bytes, cudaMemcpyDeviceToHost, stream), "D2H");
    check_cuda(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    return;
  }
  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  for (int k = 0; k < 2; ++k) {
    if (!c.d2h_pinned[k]) {
      check_cuda(cudaHostAlloc(&c.d2h_pinned[k], kChunk, cudaHostAllocDefault), "cudaHostAlloc(D2H chunk)");
      check_cuda(cudaEventCreateWithFlags(&c.d2h_done[k], cudaEventDisableTiming), "cudaEventCreate");
    }
  }
  const size_t chunks = (bytes + kChunk - 1) / kChunk;
  auto len = [&](size_t i) { return std::min(kChunk, bytes - i * kChunk); };
  auto drain = [&](size_t i) {  // chunk i: wait for the copy engine, then the host copy
    check_cuda(cudaEventSynchronize(c.d2h_done[i & 1]), "cudaEventSynchronize");
    CopyPool::get().copy(static_cast<char*>(dst) + i * kChunk, c.d2h_pinned[i & 1], len(i));
  };
  for (size_t i = 0; i < chunks; ++i) {
    // (chunk i - 2, the previous user of this page-locked chunk, was drained in the last round)
    check_cuda(cudaMemcpyAsync(c.d2h_pinned[i & 1], static_cast<const char*>(dev_src) + i * kChunk, len(i),
                               cudaMemcpyDeviceToHost, stream),
               "D2H chunk");
    check_cuda(cudaEventRecord(c.d2h_done[i & 1], stream), "cudaEventRecord");
    if (i >= 1) drain(i - 1);
  }
  drain(chunks - 1);
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


/// Runs `la` over [0, n): device pointers in place on `stream`; host pointers
/// through a 3-slot chunked H2D / kernel / D2H pipeline on the device's own
/// streams (copy engines overlap the walk of the neighbouring chunk).
/// `flag_dev` (may be null) is the device status word for domain checks.
// Device scratch for the interval fixup list: one (list, count) per pipeline
// slot. Capacity 1/16 of the chunk by default (special points are rare); the
// full chunk after an overflow.
namespace {
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

}  // namespace

// `arts` run in order on each chunk; inputs are staged once per chunk for
// all of them (pe_eval_f64_multi).
void run_batch(const std::vector<const Artifact*>& arts, int device, MemKind kind, size_t n,
               const std::vector<const void*>& ins, const std::vector<void*>& outs,
               const LaunchArgs& proto, cudaStream_t user_stream, bool sync,
               bool full_fixup, const std::vector<size_t>& out_base, const Staging& staging) {
  const size_t elem = 8;
  const Artifact& a = *arts.front();  // interval programs have exactly one
  // every buffer must live where the output does (a host pointer handed to a
  // kernel, or a device pointer to a host memcpy, would be read blindly)
  bool all_pinned = true;
  {
    std::vector<const void*> all(ins.begin(), ins.end());
    all.insert(all.end(), outs.begin(), outs.end());
    for (const void* p : all) {
      int d = -1;
      bool pinned = false;
      const MemKind k = classify(p, &d, &pinned);
      if (k != kind) {
        throw std::invalid_argument(
            "coordinate and result buffers must all be device memory or all host memory");
      }
      if (k == MemKind::Device && d >= 0 && d != device) {
        throw std::invalid_argument("buffers live on different devices");
      }
      all_pinned = all_pinned && pinned;
    }
  }
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
  // Host buffers: chunk k runs on slot k % S — H2D, the walk kernels and D2H
  // on the slot's stream, so the copy engines overlap the neighbouring
  // chunks' walks. Pageable buffers additionally pass through page-locked
  // staging arrays: before chunk k is enqueued, the host waits for chunk
  // k - S (same slot), copies its results out and chunk k's inputs in, while
  // the GPU works on chunks k - S + 1 .. k - 1.
  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  const int S = staging.slots >= 2 && staging.slots <= DeviceCtx::kMaxSlots ? staging.slots : 3;
  // 16+ chunks keep the un-overlapped first H2D / last D2H short; >= 256K
  // points keep each walk launch large enough to fill the GPU
  size_t chunk = staging.chunk >= 4096 ? staging.chunk
                                       : std::clamp<size_t>(n / 16, size_t{1} << 18, size_t{1} << 22);
  chunk = std::min(chunk, std::max<size_t>(n, 1));
  const bool stage = !all_pinned;
  ensure_buffers(c, S, ins.size() + outs.size(), chunk * elem, stage);
  cudaEvent_t flag_ready = nullptr;
  if (proto.flag) {
    // the flag was initialised on user_stream: order the slots after it
    check_cuda(cudaEventCreateWithFlags(&flag_ready, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(flag_ready, user_stream), "cudaEventRecord");
    for (int i = 0; i < S; ++i) {
      check_cuda(cudaStreamWaitEvent(c.streams[i], flag_ready, 0), "cudaStreamWaitEvent");
    }
  }
  FixupLists fix(a, chunk, full_fixup, std::vector<cudaStream_t>(c.streams, c.streams + S));
  std::vector<size_t> slot_off(static_cast<size_t>(S), SIZE_MAX), slot_len(static_cast<size_t>(S), 0);
  auto drain = [&](int slot) {  // pageable: results of the slot's last chunk to the caller
    if (!stage || slot_off[static_cast<size_t>(slot)] == SIZE_MAX) return;
    check_cuda(cudaEventSynchronize(c.done[slot]), "cudaEventSynchronize");
    const size_t off = slot_off[static_cast<size_t>(slot)], m = slot_len[static_cast<size_t>(slot)];
    for (size_t o = 0; o < outs.size(); ++o) {
      CopyPool::get().copy(static_cast<char*>(outs[o]) + off * elem, c.pinned[slot][ins.size() + o],
                           m * elem);
    }
    slot_off[static_cast<size_t>(slot)] = SIZE_MAX;
  };
  size_t k = 0;
  for (size_t off = 0; off < n; off += chunk, ++k) {
    const int slot = static_cast<int>(k % static_cast<size_t>(S));
    cudaStream_t s = c.streams[slot];
    const size_t m = std::min(chunk, n - off);
    drain(slot);
    LaunchArgs la = proto;
    fix.bind(la, static_cast<size_t>(slot));
    la.n = m;
    la.ins.clear();
    la.outs.clear();
    for (size_t i = 0; i < ins.size(); ++i) {
      void* d = c.buffers[slot][i];
      const char* src = static_cast<const char*>(ins[i]) + off * elem;
      if (stage) {
        CopyPool::get().copy(c.pinned[slot][i], src, m * elem);
        src = static_cast<const char*>(c.pinned[slot][i]);
      }
      check_cuda(cudaMemcpyAsync(d, src, m * elem, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D)");
      la.ins.push_back(reinterpret_cast<std::uint64_t>(d));
    }
    for (size_t o = 0; o < outs.size(); ++o) {
      la.outs.push_back(reinterpret_cast<std::uint64_t>(c.buffers[slot][ins.size() + o]));
    }
    launch_all(la, s);
    for (size_t o = 0; o < outs.size(); ++o) {
      void* dst = stage ? c.pinned[slot][ins.size() + o] : static_cast<char*>(outs[o]) + off * elem;
      check_cuda(cudaMemcpyAsync(dst, c.buffers[slot][ins.size() + o], m * elem,
                                 cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(D2H)");
    }
    check_cuda(cudaEventRecord(c.done[slot], s), "cudaEventRecord");
    slot_off[static_cast<size_t>(slot)] = off;
    slot_len[static_cast<size_t>(slot)] = m;
  }
  for (size_t j = 0; j < static_cast<size_t>(S); ++j) {  // oldest chunk first
    drain(static_cast<int>((k + j) % static_cast<size_t>(S)));
  }
  for (int i = 0; i < S; ++i) check_cuda(cudaStreamSynchronize(c.streams[i]), "cudaStreamSynchronize");
  if (flag_ready) cudaEventDestroy(flag_ready);
}

void run_batch(const Artifact& a, int device, MemKind kind, size_t n,
               const std::vector<const void*>& ins, const std::vector<void*>& outs,
               const LaunchArgs& proto, cudaStream_t user_stream, bool sync,
               bool full_fixup, const Staging& staging) {
  run_batch(std::vector<const Artifact*>{&a}, device, kind, n, ins, outs, proto, user_stream, sync,
            full_fixup, {}, staging);
}

}  // namespace polyeval::rt
