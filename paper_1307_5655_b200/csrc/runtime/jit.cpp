#include "runtime/jit.hpp"

#include <nvPTXCompiler.h>

#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <functional>
#include <thread>

namespace polyeval::rt {

namespace {
const char* const kPtxasOptions[] = {"--gpu-name=sm_100a", "-O3", "--generate-line-info"};
constexpr int kPtxasOptionCount = 3;
}  // namespace

CompileResult compile_ptx(const std::string& ptx, const std::string& tag) {
  CompileResult out;
  const auto t0 = std::chrono::steady_clock::now();
  nvPTXCompilerHandle h = nullptr;
  if (nvPTXCompilerCreate(&h, ptx.size(), ptx.data()) != NVPTXCOMPILE_SUCCESS) {
    out.log = "nvPTXCompilerCreate failed for " + tag;
    return out;
  }
  const nvPTXCompileResult r = nvPTXCompilerCompile(h, kPtxasOptionCount, kPtxasOptions);
  size_t n = 0;
  if (r != NVPTXCOMPILE_SUCCESS) {
    nvPTXCompilerGetErrorLogSize(h, &n);
    std::string log(n, '\0');
    if (n) nvPTXCompilerGetErrorLog(h, log.data());
    out.log = "ptxas (sm_100a) failed for " + tag + ": " + log;
    nvPTXCompilerDestroy(&h);
    return out;
  }
  nvPTXCompilerGetInfoLogSize(h, &n);
  if (n) {
    std::string info(n, '\0');
    nvPTXCompilerGetInfoLog(h, info.data());
    out.log = info;
  }
  size_t sz = 0;
  nvPTXCompilerGetCompiledProgramSize(h, &sz);
  out.cubin.resize(sz);
  nvPTXCompilerGetCompiledProgram(h, out.cubin.data());
  nvPTXCompilerDestroy(&h);
  out.ok = true;
  out.seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

namespace {

std::string cache_dir() {
  if (const char* d = std::getenv("PE_CACHE_DIR")) {
    const std::string s(d);
    if (s == "off" || s == "0" || s.empty()) return {};
    return s;
  }
  if (const char* x = std::getenv("XDG_CACHE_HOME")) return std::string(x) + "/polyeval-b200";
  if (const char* h = std::getenv("HOME")) return std::string(h) + "/.cache/polyeval-b200";
  return {};
}

std::uint64_t fnv(const void* data, std::size_t n, std::uint64_t h) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}
std::uint64_t fnv(const std::string& s, std::uint64_t h) { return fnv(s.data(), s.size(), h); }

// The compiler identity and options enter the key: a cubin from another
// ptxas version or option set is never reused.
std::string compiler_tag() {
  unsigned major = 0, minor = 0;
  nvPTXCompilerGetVersion(&major, &minor);
  std::string t = "nvptxcompiler-" + std::to_string(major) + "." + std::to_string(minor);
  for (int i = 0; i < kPtxasOptionCount; ++i) t += std::string(" ") + kPtxasOptions[i];
  return t;
}

// Cache file: 8-byte magic, 8-byte payload length, 8-byte FNV-1a of the
// payload, payload. A short or corrupt file is treated as a miss.
constexpr std::uint64_t kMagic = 0x3130306d73626370ull;  // "pcbsm001"

}  // namespace

CompileResult compile_ptx_cached(const std::string& ptx, const std::string& tag, bool* cached) {
  if (cached) *cached = false;
  const std::string dir = cache_dir();
  if (dir.empty()) return compile_ptx(ptx, tag);
  static const std::string ctag = compiler_tag();
  char key[96];
  // two independent 64-bit hashes of (compiler identity, options, PTX text)
  // + PTX length: the PTX embeds target, coefficients and shape
  const std::uint64_t h1 = fnv(ptx, fnv(ctag, 1469598103934665603ull));
  const std::uint64_t h2 = fnv(ptx, fnv(ctag, 0x9E3779B97F4A7C15ull));
  std::snprintf(key, sizeof key, "%016llx%016llx_%zu", static_cast<unsigned long long>(h1),
                static_cast<unsigned long long>(h2), ptx.size());
  const std::string path = dir + "/" + key + ".sm100a.cubin";
  if (FILE* f = std::fopen(path.c_str(), "rb")) {
    std::uint64_t hdr[3] = {0, 0, 0};
    CompileResult out;
    if (std::fread(hdr, sizeof hdr, 1, f) == 1 && hdr[0] == kMagic && hdr[1] > 0 &&
        hdr[1] < (std::uint64_t{1} << 32)) {
      out.cubin.resize(static_cast<size_t>(hdr[1]));
      if (std::fread(out.cubin.data(), 1, out.cubin.size(), f) == out.cubin.size() &&
          fnv(out.cubin.data(), out.cubin.size(), 1469598103934665603ull) == hdr[2]) {
        std::fclose(f);
        out.ok = true;
        if (cached) *cached = true;
        return out;
      }
    }
    std::fclose(f);  // short / corrupt / other format: recompile and replace
  }
  CompileResult r = compile_ptx(ptx, tag);
  if (r.ok) {
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    // unique per writer (process, thread, call): concurrent compiles of the
    // same PTX never share a temporary; rename() publishes atomically
    static std::atomic<std::uint64_t> seq{0};
    const std::string tmp = path + ".tmp" + std::to_string(::getpid()) + "_" +
                            std::to_string(std::hash<std::thread::id>{}(std::this_thread::get_id())) +
                            "_" + std::to_string(seq.fetch_add(1));
    if (FILE* f = std::fopen(tmp.c_str(), "wb")) {
      const std::uint64_t hdr[3] = {kMagic, r.cubin.size(),
                                    fnv(r.cubin.data(), r.cubin.size(), 1469598103934665603ull)};
      const bool ok = std::fwrite(hdr, sizeof hdr, 1, f) == 1 &&
                      std::fwrite(r.cubin.data(), 1, r.cubin.size(), f) == r.cubin.size();
      const bool closed = std::fclose(f) == 0;
      if (ok && closed) {
        std::rename(tmp.c_str(), path.c_str());
      } else {
        std::remove(tmp.c_str());
      }
    }
  }
  return r;
}

}  // namespace polyeval::rt
