// Launch runtime behind the C ABI: argument packing and launch of
// specialised kernels, pointer classification, the 3-slot host-staged
// H2D / walk / D2H pipeline, status words for domain checks, and the
// per-stream state of deferred checks.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

#include "polyeval_b200.h"
#include "runtime/program.hpp"

namespace polyeval::rt {

/// Kernels this library launched (pe_launch_count).
std::atomic<std::uint64_t>& launch_counter();

struct LaunchArgs {
  std::vector<std::uint64_t> ins, outs;
  std::uint64_t n = 0;
  std::uint64_t flag = 0;
  std::vector<std::uint64_t> bounds;
  // interval fast path: fixup list (u32 point indices), counter, capacity
  std::uint64_t list = 0, count = 0, cap = 0;
};

/// Host-buffer pipeline shape (pe_exec::stage_chunk / stage_slots; 0 = default).
struct Staging {
  std::size_t chunk = 0;  // points per chunk
  int slots = 0;          // chunks in flight (2..8)
};

int sm_count(int device);

/// Raises the release threshold of the device's default memory pool once, so
/// stream-ordered scratch stays mapped between calls.
void keep_pool_memory(int device);

/// Launches one artifact (and its interval fixup entry) on `stream`.
void launch(const Artifact& a, int device, const LaunchArgs& la, cudaStream_t stream);

enum class MemKind { Host, Device };

/// Device (or managed) memory vs host memory; `pinned` (optional) tells
/// page-locked host memory from pageable.
MemKind classify(const void* p, int* device, bool* pinned = nullptr);

// Deferred-check state of one caller stream: an accumulating status word and
// a grow-only full-capacity interval fixup list, both stream-ordered.
struct StreamState {
  unsigned* status = nullptr;
  void* list = nullptr;
  unsigned* count = nullptr;
  std::uint64_t list_cap = 0;
};

struct DeviceCtx {
  static constexpr int kMaxSlots = 8;
  cudaStream_t streams[kMaxSlots] = {};
  cudaEvent_t done[kMaxSlots] = {};
  std::vector<void*> buffers[kMaxSlots];  // per slot: device arrays of `cap` bytes
  std::vector<void*> pinned[kMaxSlots];   // per slot: page-locked host arrays (pageable callers)
  size_t cap = 0, pinned_cap = 0;
  void* d2h_pinned[2] = {};  // copy_to_host: two page-locked chunks
  cudaEvent_t d2h_done[2] = {};
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

DeviceCtx& device_ctx(int device);

/// Device -> host copy of a large result, ordered after the work queued on
/// `stream` and complete on return. A pageable destination is filled through
/// two page-locked chunks: the copy engine writes one while the host copy
/// pool moves the other into the caller's buffer (a plain cudaMemcpy to
/// pageable memory runs at a fraction of PCIe speed).
void copy_to_host(void* dst, const void* dev_src, size_t bytes, int device, cudaStream_t stream);

int resolve_device(const pe_exec* ex, const void* probe, MemKind* kind);

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

/// Runs the artifacts over [0, n): device pointers in place on
/// `user_stream`; host pointers through the chunked H2D / walk / D2H
/// pipeline on the device's own streams (pageable host memory additionally
/// through page-locked staging buffers). Every buffer must be of `kind`.
/// `arts` run in order per chunk; art i writes outs[out_base[i] ..] (default 0).
void run_batch(const std::vector<const Artifact*>& arts, int device, MemKind kind, size_t n,
               const std::vector<const void*>& ins, const std::vector<void*>& outs,
               const LaunchArgs& proto, cudaStream_t user_stream, bool sync,
               bool full_fixup = false, const std::vector<size_t>& out_base = {},
               const Staging& staging = {});
void run_batch(const Artifact& a, int device, MemKind kind, size_t n,
               const std::vector<const void*>& ins, const std::vector<void*>& outs,
               const LaunchArgs& proto, cudaStream_t user_stream, bool sync,
               bool full_fixup = false, const Staging& staging = {});

/// Staging options of a call (pe_exec fields).
Staging staging_of(const pe_exec* ex);

}  // namespace polyeval::rt
