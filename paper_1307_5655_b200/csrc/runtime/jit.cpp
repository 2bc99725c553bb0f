#include "runtime/jit.hpp"

#include <nvPTXCompiler.h>

#include <chrono>
#include <cstring>

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

}  // namespace polyeval::rt
