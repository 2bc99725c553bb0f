// PTX -> sm_100a cubin, in process (nvPTXCompiler, statically linked), and
// cubin -> loaded kernel handle (cudaLibrary, context-independent so the same
// handle launches on every device of the box).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace polyeval::rt {

struct CompileResult {
  bool ok = false;
  std::vector<char> cubin;
  std::string log;
  double seconds = 0.0;
};

/// ptxas for sm_100a with -O3 and line info; never touches a GPU.
CompileResult compile_ptx(const std::string& ptx, const std::string& tag);

/// compile_ptx behind an on-disk cubin cache keyed by the PTX text
/// (PE_CACHE_DIR, else $XDG_CACHE_HOME or ~/.cache /polyeval-b200;
/// PE_CACHE_DIR=off disables). `cached` reports a hit.
CompileResult compile_ptx_cached(const std::string& ptx, const std::string& tag,
                                 bool* cached = nullptr);

}  // namespace polyeval::rt
