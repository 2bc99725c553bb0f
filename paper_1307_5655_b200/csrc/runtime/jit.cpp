#include "runtime/jit.hpp"

#include <nvPTXCompiler.h>

#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>

namespace polyeval::rt {

CompileResult compile_ptx(const std::string& ptx, const std::string& tag) {
  CompileResult out;
  const auto t0 = std::chrono::steady_clock::now();
  nvPTXCompilerHandle h = nullptr;
  if (nvPTXCompilerCreate(&h, ptx.size(), ptx.data()) != NVPTXCOMPILE_SUCCESS) {
    out.log = "nvPTXCompilerCreate failed for " + tag;
    return out;
  }
  const char* opts[] = {"--gpu-name=sm_100a", "-O3", "--generate-line-info"};
  const nvPTXCompileResult r = nvPTXCompilerCompile(h, 3, opts);
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

std::uint64_t fnv(const std::string& s, std::uint64_t h) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace

CompileResult compile_ptx_cached(const std::string& ptx, const std::string& tag, bool* cached) {
  if (cached) *cached = false;
  const std::string dir = cache_dir();
  if (dir.empty()) return compile_ptx(ptx, tag);
  char key[96];
  // two independent 64-bit hashes + length: the cubin depends only on the
  // PTX text (which embeds target, coefficients and shape) and ptxas options
  std::snprintf(key, sizeof key, "%016llx%016llx_%zu",
                static_cast<unsigned long long>(fnv(ptx, 1469598103934665603ull)),
                static_cast<unsigned long long>(fnv(ptx, 0x9E3779B97F4A7C15ull)), ptx.size());
  const std::string path = dir + "/" + key + ".sm100a.cubin";
  if (FILE* f = std::fopen(path.c_str(), "rb")) {
    CompileResult out;
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (n > 0) {
      out.cubin.resize(static_cast<size_t>(n));
      if (std::fread(out.cubin.data(), 1, out.cubin.size(), f) == out.cubin.size()) {
        std::fclose(f);
        out.ok = true;
        if (cached) *cached = true;
        return out;
      }
    }
    std::fclose(f);
  }
  CompileResult r = compile_ptx(ptx, tag);
  if (r.ok) {
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    const std::string tmp = path + ".tmp" + std::to_string(::getpid());
    if (FILE* f = std::fopen(tmp.c_str(), "wb")) {
      const bool ok = std::fwrite(r.cubin.data(), 1, r.cubin.size(), f) == r.cubin.size();
      std::fclose(f);
      if (ok) std::rename(tmp.c_str(), path.c_str());
      else std::remove(tmp.c_str());
    }
  }
  return r;
}

}  // namespace polyeval::rt
