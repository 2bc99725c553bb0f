// C++ drop-in usage of the C ABI through include/polyeval_gpu.hpp: the
// reference worked example 3x^8-x^7+2x^6+x^5-4x^4+9x^3-3x^2-2x+1 at
// x = 2, 0, 1 (eval_test.cpp:80-93: 793, 1, 6) in every builtin scheme and
// every domain, plus the reference's exception mapping for an arity error.
#include <cstdio>
#include <stdexcept>

#include "polyeval_gpu.hpp"

int main() {
  using namespace polyeval::gpu;
  const std::uint32_t exps[] = {8, 7, 6, 5, 4, 3, 2, 1, 0};
  const std::int64_t ci[] = {3, -1, 2, 1, -4, 9, -3, -2, 1};
  const double cf[] = {3, -1, 2, 1, -4, 9, -3, -2, 1};
  const std::int64_t xi[] = {2, 0, 1};
  const double xf[] = {2, 0, 1};
  int bad = 0;
  for (const char* s : {"direct", "horner", "estrin", "balanced", "balanced:horner@2"}) {
    Program pi = Program::from_terms(exps, ci, 9, 1, {s});
    Program pf = Program::from_terms(exps, cf, 9, 1, {s});
    std::int64_t oi[3];
    double of[3], lo[3], hi[3];
    BatchEvaluator<BigIntDomain>(pi).evaluate({xi}, 3, oi);
    BatchEvaluator<DoubleDomain>(pf, DoubleDomain{true}).evaluate({xf}, 3, of);
    BatchEvaluator<IntervalDomain>(pf).evaluate({xf}, {xf}, 3, lo, hi);
    std::printf("%s %lld %lld %lld | %g %g %g | [%g,%g]\n", s, (long long)oi[0], (long long)oi[1],
                (long long)oi[2], of[0], of[1], of[2], lo[0], hi[0]);
    bad |= !(oi[0] == 793 && oi[1] == 1 && oi[2] == 6 && of[0] == 793 && of[1] == 1 && of[2] == 6 &&
             lo[0] <= 793 && hi[0] >= 793);
  }
  {  // BigInt beyond int64: 2 limbs, equal to the int64 path where both apply
    Program p = Program::from_terms(exps, ci, 9, 1, {"balanced"});
    const std::int64_t xs[] = {2, -3, 5};
    std::uint64_t l0[3], l1[3];
    std::uint64_t* limbs[] = {l0, l1};
    BatchEvaluator<BigIntDomain>(p).evaluate_limbs({xs}, 3, 2, limbs);
    std::int64_t ref[3];
    BatchEvaluator<BigIntDomain>(p).evaluate({xs}, 3, ref);
    for (int i = 0; i < 3; ++i) {
      const std::uint64_t ext = ref[i] < 0 ? ~0ull : 0ull;
      bad |= !(l0[i] == static_cast<std::uint64_t>(ref[i]) && l1[i] == ext);
    }
    std::printf("limbs %lld %lld %lld\n", (long long)ref[0], (long long)ref[1], (long long)ref[2]);
  }
  try {
    Program p = Program::from_terms(exps, ci, 9, 1, {"estrin"});
    BatchEvaluator<BigIntDomain>(p).evaluate({xi, xi}, 3, nullptr);
    bad = 1;
  } catch (const std::invalid_argument&) {
  }
  std::printf(bad ? "FAIL\n" : "OK\n");
  return bad;
}
