// Driver for the INTEGRATION.md adapter (tests/test_integration_adapter.py
// extracts the adapter from INTEGRATION.md into integration_adapter.hpp and
// compiles this file against the unmodified reference headers and library).
//
//   integration_main          host checks only (no GPU needed)
//   integration_main gpu      also evaluates on the GPU vs Evaluator<D>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <polyeval/eval.hpp>
#include <polyeval/parser.hpp>
#include <polyeval/ring.hpp>
#include <polyeval/scheme.hpp>
#include <polyeval/tree.hpp>

#include "integration_adapter.hpp"

namespace {
int failures = 0;
void expect(bool ok, const char* what) {
  if (!ok) {
    std::printf("FAIL %s\n", what);
    ++failures;
  }
}

bool same_records(const pe_program* a, const pe_program* b) {
  std::size_t na = 0, nb = 0;
  pe_program_records(a, nullptr, 0, &na);
  pe_program_records(b, nullptr, 0, &nb);
  if (na != nb) return false;
  std::vector<std::int32_t> ra(5 * na), rb(5 * nb);
  pe_program_records(a, ra.data(), ra.size(), &na);
  pe_program_records(b, rb.data(), rb.size(), &nb);
  pe_program_info_t ia, ib;
  pe_program_info(a, &ia);
  pe_program_info(b, &ib);
  return ra == rb && std::memcmp(&ia, &ib, sizeof ia) == 0;
}
}  // namespace

int main(int argc, char** argv) {
  using namespace polyeval;
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  struct Case {
    const char* text;
    std::vector<std::string> schemes;
  } cases[] = {
      {"3*x^8 - x^7 + 2*x^6 + x^5 - 4*x^4 + 9*x^3 - 3*x^2 - 2*x + 1", {"balanced"}},
      {"x^2*y^2 + 2*x*y + 1", {"horner", "estrin"}},
      {"5*x^3*y*z^2 - 7*y^4 + 3*x*z^5 + 2*z - 11", {"balanced", "estrin:horner@2", "direct"}},
  };
  for (const auto& c : cases) {
    const Polynomial p = parse_polynomial(c.text);
    // the reference's own front end: trees per scheme, lazy heights, compile
    std::vector<FunctionScheme> fs;
    for (const auto& s : c.schemes) {
      const auto colon = s.find(':');
      auto builtin = [](const std::string& n) {
        return builtin_scheme(n == "direct" ? BuiltinScheme::direct
                              : n == "horner" ? BuiltinScheme::horner
                              : n == "estrin" ? BuiltinScheme::estrin
                                              : BuiltinScheme::balanced);
      };
      if (colon == std::string::npos) {
        fs.push_back(builtin(s));
      } else {
        const auto at = s.find('@');
        fs.push_back(threshold_combine(builtin(s.substr(0, colon)),
                                       builtin(s.substr(colon + 1, at - colon - 1)),
                                       std::stoull(s.substr(at + 1))));
      }
    }
    EvaluationTree tree = p.variables().size() == 1 ? build(p, fs[0], 0)
                                                    : build_multivariate(p, fs);
    compute_lazy_heights(tree);
    const CompiledProgram cp = compile(tree);
    // the adapter's two entry points
    const auto from_terms = gpu_adapter::compile_for_gpu(p, c.schemes, true);
    pe_program* lowered = gpu_adapter::lower_compiled(cp, true);
    expect(same_records(from_terms.get(), lowered), "adapter paths give the same program");
    expect(pe_program_info(lowered, nullptr) == PE_EINVAL, "null info argument rejected");
    pe_program_info_t info;
    pe_program_info(lowered, &info);
    expect(info.register_count == cp.register_count, "register_count");
    expect(info.records >= cp.records.size(), "records");
    if (gpu) {
      const std::size_t nv = p.variables().size();
      std::vector<std::vector<std::int64_t>> x(nv);
      const std::size_t n = 1000;
      for (std::size_t v = 0; v < nv; ++v) {
        for (std::size_t i = 0; i < n; ++i) x[v].push_back(static_cast<std::int64_t>((i * (v + 3)) % 7) - 3);
      }
      std::vector<std::int64_t> out(n);
      std::vector<const std::int64_t*> cols;
      for (auto& c2 : x) cols.push_back(c2.data());
      pe_exec ex{};
      ex.device = -1;
      expect(pe_eval_i64(lowered, cols.data(), n, out.data(), &ex) == PE_OK, "pe_eval_i64");
      Evaluator<BigIntDomain> ref(BigIntDomain{}, cp);
      bool equal = true;
      for (std::size_t i = 0; i < n; ++i) {
        std::vector<BigInt> pt;
        for (std::size_t v = 0; v < nv; ++v) pt.push_back(BigInt(x[v][i]));
        equal = equal && ref.evaluate(pt).to_decimal() == std::to_string(out[i]);
      }
      expect(equal, "GPU results equal the reference Evaluator<BigIntDomain>");
    }
    pe_program_destroy(lowered);
  }
  std::printf("%s %d failures\n", failures ? "FAILED" : "ok", failures);
  return failures ? 1 : 0;
}
