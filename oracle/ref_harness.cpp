// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C harness over the *unmodified* reference library (compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/). It
// drives the reference's own public API: Polynomial::canonicalize ->
// build / build_multivariate -> compute_lazy_heights -> compile ->
// Evaluator<D>::evaluate, one point per call (eval.hpp:74-90), one Evaluator
// session per host thread over a contiguous shard (the reference's documented
// concurrency contract, eval.hpp:59-68).
//
// fp64 coefficients: the reference Polynomial holds BigInt only,
// so each coefficient c is encoded as k = c * 2^S (S the smallest shift making
// every coefficient integral; BigInt::from_double_integral throws otherwise)
// and evaluated through ScaledDoubleDomain / ScaledIntervalDomain, whose
// from_integer(k) = ldexp(k.to_double(), -S) is exact. Everything else (walk,
// power tables, interval rounding) is the reference's code.
#include <polyeval/bigint.hpp>
#include <polyeval/eval.hpp>
#include <polyeval/interval.hpp>
#include <polyeval/polynomial.hpp>
#include <polyeval/ring.hpp>
#include <polyeval/scheme.hpp>
#include <polyeval/tree.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

using namespace polyeval;

namespace {

thread_local std::string g_err;

struct ScaledDoubleDomain {
  using Value = double;
  static constexpr bool exact = false;
  int shift = 0;
  Value zero() const { return 0.0; }
  Value add(const Value& a, const Value& b) const { return a + b; }
  Value mul(const Value& a, const Value& b) const { return a * b; }
  Value from_integer(const BigInt& c) const { return std::ldexp(c.to_double(), -shift); }
};

struct ScaledIntervalDomain {
  using Value = Interval;
  static constexpr bool exact = false;
  int shift = 0;
  Value zero() const { return Interval(); }
  Value add(const Value& a, const Value& b) const { return interval_add(a, b); }
  Value mul(const Value& a, const Value& b) const { return interval_mul(a, b); }
  Value from_integer(const BigInt& c) const {
    if (shift == 0) return IntervalDomain{}.from_integer(c);
    const double v = std::ldexp(c.to_double(), -shift);  // exact by construction
    return Interval(v, v);
  }
};

struct RefProgram {
  bool integer = false;
  int shift = 0;
  std::size_t nvars = 0;
  std::unique_ptr<EvaluationTree> tree;
  std::unique_ptr<CompiledProgram> program;
};

FunctionScheme scheme_of(int up, int lo, std::uint64_t cutoff) {
  auto b = [](int id) { return builtin_scheme(static_cast<BuiltinScheme>(id)); };
  if (cutoff == 0) return b(up);
  return threshold_combine(b(up), b(lo), cutoff);
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename D, typename In, typename Out, typename Conv>
void run_sharded(const RefProgram& rp, D domain, std::size_t n, int threads, In&& point_of,
                 Out* out, Conv&& conv) {
  threads = std::max(1, threads);
  const std::size_t per = (n + threads - 1) / threads;
  std::vector<std::exception_ptr> errors(threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      try {
        Evaluator<D> session(domain, *rp.program);
        std::vector<typename D::Value> point(rp.nvars);
        const std::size_t lo = t * per, hi = std::min(n, lo + per);
        for (std::size_t i = lo; i < hi; ++i) {
          point_of(i, point);
          out[i] = conv(session.evaluate(std::span<const typename D::Value>(point)));
        }
      } catch (...) {
        errors[t] = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errors) {
    if (e) std::rethrow_exception(e);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_create(const std::uint32_t* exps, const void* coeffs, std::size_t nterms,
               std::uint32_t nvars, const int* upper, const int* lower,
               const std::uint64_t* cutoff, int coeff_is_int, void** out) {
  return guarded([&] {
    auto rp = std::make_unique<RefProgram>();
    rp->integer = coeff_is_int != 0;
    rp->nvars = nvars;
    std::vector<std::string> vars;
    for (std::uint32_t v = 0; v < nvars; ++v) {
      vars.push_back(nvars <= 3 ? std::string(1, "xyz"[v]) : "x" + std::to_string(v));
    }
    int shift = 0;
    if (!rp->integer) {
      const double* c = static_cast<const double*>(coeffs);
      for (std::size_t t = 0; t < nterms; ++t) {
        if (c[t] == 0.0) continue;
        int e = 0;
        std::frexp(c[t], &e);
        shift = std::max(shift, 53 - e);
      }
    }
    rp->shift = shift;
    std::vector<Term> raw(nterms);
    for (std::size_t t = 0; t < nterms; ++t) {
      if (rp->integer) {
        raw[t].coefficient = BigInt(static_cast<const std::int64_t*>(coeffs)[t]);
      } else {
        raw[t].coefficient =
            BigInt::from_double_integral(std::ldexp(static_cast<const double*>(coeffs)[t], shift));
      }
      raw[t].exponents.assign(exps + t * nvars, exps + (t + 1) * nvars);
    }
    Polynomial p = Polynomial::canonicalize(std::move(raw), vars);
    std::vector<FunctionScheme> schemes;
    for (std::uint32_t v = 0; v < nvars; ++v) schemes.push_back(scheme_of(upper[v], lower[v], cutoff[v]));
    EvaluationTree tree = nvars == 1 ? build(p, schemes[0], 0) : build_multivariate(p, schemes);
    compute_lazy_heights(tree);
    rp->program = std::make_unique<CompiledProgram>(compile(tree));
    rp->tree = std::make_unique<EvaluationTree>(std::move(tree));
    *out = rp.release();
    return 0;
  });
}

void ref_destroy(void* h) { delete static_cast<RefProgram*>(h); }

int ref_dot(void* h, char* buf, std::size_t cap, std::size_t* len) {
  return guarded([&] {
    const std::string dot = to_dot(*static_cast<RefProgram*>(h)->tree);
    *len = dot.size();
    if (buf && cap) {
      const std::size_t k = std::min(cap - 1, dot.size());
      std::memcpy(buf, dot.data(), k);
      buf[k] = 0;
    }
    return 0;
  });
}

// records x 5: power_slot|-1, lazy_slot, parent_slot|-1, reads_register, has_sub
int ref_records(void* h, std::int32_t* out, std::size_t cap, std::size_t* count,
                std::uint32_t* register_count) {
  return guarded([&] {
    const CompiledProgram& p = *static_cast<RefProgram*>(h)->program;
    *count = p.records.size();
    *register_count = p.register_count;
    for (std::size_t i = 0; i < p.records.size() && (i + 1) * 5 <= cap; ++i) {
      const auto& r = p.records[i];
      out[5 * i] = r.power_slot ? static_cast<std::int32_t>(*r.power_slot) : -1;
      out[5 * i + 1] = static_cast<std::int32_t>(r.lazy_slot);
      out[5 * i + 2] = r.parent_slot ? static_cast<std::int32_t>(*r.parent_slot) : -1;
      out[5 * i + 3] = r.reads_register ? 1 : 0;
      out[5 * i + 4] = r.sub ? 1 : 0;
    }
    return 0;
  });
}

// Flattens the reference CompiledProgram (root + nested, pre-order) for
// pe_program_from_compiled: per record (coeff as fp64 — exact, k * 2^-S — and
// as int64 for integer programs; sub program index | -1, power_slot | -1,
// lazy_slot, parent_slot | -1, reads_register), per program (first record,
// record count, register_count, variable, first root_child_end, count).
// Call once with null buffers for the sizes.
int ref_export(void* h, double* rec_f64, std::int64_t* rec_i64, std::int32_t* rec_int,
               std::uint32_t* prog_info, std::uint32_t* ends, std::size_t* nrec,
               std::size_t* nprog, std::size_t* nends) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    std::size_t r = 0, pcount = 0, e = 0;
    auto visit = [&](auto&& self, const CompiledProgram& p) -> std::size_t {
      const std::size_t me = pcount++;
      const std::size_t first = r;
      r += p.records.size();
      const std::size_t first_end = e;
      e += p.root_child_ends.size();
      if (prog_info) {
        std::uint32_t* pi = prog_info + 6 * me;
        pi[0] = static_cast<std::uint32_t>(first);
        pi[1] = static_cast<std::uint32_t>(p.records.size());
        pi[2] = p.register_count;
        pi[3] = static_cast<std::uint32_t>(p.variable);
        pi[4] = static_cast<std::uint32_t>(first_end);
        pi[5] = static_cast<std::uint32_t>(p.root_child_ends.size());
        for (std::size_t k = 0; k < p.root_child_ends.size(); ++k) ends[first_end + k] = p.root_child_ends[k];
      }
      for (std::size_t i = 0; i < p.records.size(); ++i) {
        const auto& rec = p.records[i];
        std::int32_t sub = -1;
        if (rec.sub) sub = static_cast<std::int32_t>(self(self, *rec.sub));
        if (rec_int) {
          std::int32_t* ri = rec_int + 5 * (first + i);
          ri[0] = sub;
          ri[1] = rec.power_slot ? static_cast<std::int32_t>(*rec.power_slot) : -1;
          ri[2] = static_cast<std::int32_t>(rec.lazy_slot);
          ri[3] = rec.parent_slot ? static_cast<std::int32_t>(*rec.parent_slot) : -1;
          ri[4] = rec.reads_register ? 1 : 0;
          rec_f64[first + i] = rec.sub ? 0.0 : std::ldexp(rec.coeff.to_double(), -rp.shift);
          rec_i64[first + i] = rec.sub || !rp.integer ? 0 : std::stoll(rec.coeff.to_decimal());
        }
      }
      return me;
    };
    visit(visit, *rp.program);
    *nrec = r;
    *nprog = pcount;
    *nends = e;
    return 0;
  });
}

int ref_exponents(void* h, std::uint32_t v, std::uint32_t* out, std::size_t cap, std::size_t* count) {
  return guarded([&] {
    const CompiledProgram& p = *static_cast<RefProgram*>(h)->program;
    const auto& e = p.exponent_sets.at(v).exponents;
    *count = e.size();
    for (std::size_t i = 0; i < e.size() && i < cap; ++i) out[i] = e[i];
    return 0;
  });
}

int ref_eval_f64(void* h, const double* const* coords, std::size_t n, double* out, int threads) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    auto pt = [&](std::size_t i, std::vector<double>& p) {
      for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = coords[v][i];
    };
    auto id = [](double x) { return x; };
    if (rp.integer) {
      run_sharded(rp, DoubleDomain{}, n, threads, pt, out, id);
    } else {
      run_sharded(rp, ScaledDoubleDomain{rp.shift}, n, threads, pt, out, id);
    }
    return 0;
  });
}

int ref_eval_interval(void* h, const double* const* lo, const double* const* hi, std::size_t n,
                      double* out_lo, double* out_hi, int threads) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    auto pt = [&](std::size_t i, std::vector<Interval>& p) {
      for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = Interval(lo[v][i], hi[v][i]);
    };
    std::vector<Interval> res(n);
    auto id = [](const Interval& x) { return x; };
    run_sharded(rp, ScaledIntervalDomain{rp.integer ? 0 : rp.shift}, n, threads, pt, res.data(), id);
    for (std::size_t i = 0; i < n; ++i) {
      out_lo[i] = res[i].lo;
      out_hi[i] = res[i].hi;
    }
    return 0;
  });
}

// BigIntDomain; results must fit int64 (reported as an error otherwise).
int ref_eval_i64(void* h, const std::int64_t* const* coords, std::size_t n, std::int64_t* out,
                 int threads) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    if (!rp.integer) throw std::invalid_argument("integer evaluation needs integer coefficients");
    auto pt = [&](std::size_t i, std::vector<BigInt>& p) {
      for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = BigInt(coords[v][i]);
    };
    const BigInt lo = BigInt(INT64_MIN), hi = BigInt(INT64_MAX);
    auto conv = [&](const BigInt& b) -> std::int64_t {
      if (b < lo || b > hi) throw std::overflow_error("result does not fit int64");
      // decimal round trip keeps the harness independent of BigInt internals
      return std::stoll(b.to_decimal());
    };
    run_sharded(rp, BigIntDomain{}, n, threads, pt, out, conv);
    return 0;
  });
}

// BigInt results as K 64-bit limbs (little-endian two's complement):
// out[k * n + i] = word k of point i. Throws if a result needs more than
// 64K-1 bits. Decimal round trip, so the harness needs no BigInt internals.
int ref_eval_limbs(void* h, const std::int64_t* const* coords, std::size_t n, std::uint32_t K,
                   std::uint64_t* out, int threads) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    if (!rp.integer) throw std::invalid_argument("integer evaluation needs integer coefficients");
    auto pt = [&](std::size_t i, std::vector<BigInt>& p) {
      for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = BigInt(coords[v][i]);
    };
    std::vector<std::string> dec(n);
    run_sharded(rp, BigIntDomain{}, n, threads, pt, dec.data(),
                [](const BigInt& b) { return b.to_decimal(); });
    for (std::size_t i = 0; i < n; ++i) {
      const std::string& d = dec[i];
      const bool neg = !d.empty() && d[0] == '-';
      std::vector<std::uint64_t> mag(K + 1, 0);  // one spare limb detects overflow
      for (std::size_t c = neg ? 1 : 0; c < d.size(); ++c) {
        unsigned __int128 carry = static_cast<unsigned>(d[c] - '0');
        for (auto& w : mag) {
          const unsigned __int128 t = static_cast<unsigned __int128>(w) * 10 + carry;
          w = static_cast<std::uint64_t>(t);
          carry = t >> 64;
        }
      }
      // |value| must be < 2^(64K-1) (or == 2^(64K-1) when negative)
      const bool top_clear = mag[K] == 0 && (mag[K - 1] >> 63) == 0;
      if (!top_clear) throw std::overflow_error("result does not fit the limb count");
      if (neg) {  // two's complement
        unsigned __int128 c = 1;
        for (std::uint32_t k = 0; k < K; ++k) {
          const unsigned __int128 t = static_cast<unsigned __int128>(~mag[k]) + c;
          mag[k] = static_cast<std::uint64_t>(t);
          c = t >> 64;
        }
      }
      for (std::uint32_t k = 0; k < K; ++k) out[k * n + i] = mag[k];
    }
    return 0;
  });
}

}  // extern "C"

// ---- arbitrary-width integers (the paper's Figure-1 workload) ----

namespace {
BigInt big_of_words(const std::uint64_t* w, std::uint32_t L) {  // two's complement
  const bool neg = L && (w[L - 1] >> 63);
  std::vector<std::uint64_t> m(w, w + L);
  if (neg) {
    unsigned __int128 c = 1;
    for (auto& x : m) {
      const unsigned __int128 t = static_cast<unsigned __int128>(~x) + c;
      x = static_cast<std::uint64_t>(t);
      c = t >> 64;
    }
  }
  return BigInt::from_words(m, neg);
}

// one BigIntDomain session per thread over contiguous shards of the points
template <typename Fn>
void wide_sharded(const RefProgram& rp, std::size_t n, int threads, Fn&& per_point) {
  threads = std::max(1, threads);
  const std::size_t per = (n + threads - 1) / threads;
  std::vector<std::exception_ptr> errors(threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      try {
        Evaluator<BigIntDomain> session(BigIntDomain{}, *rp.program);
        const std::size_t lo = t * per, hi = std::min(n, lo + per);
        for (std::size_t i = lo; i < hi; ++i) per_point(session, i);
      } catch (...) {
        errors[t] = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errors) {
    if (e) std::rethrow_exception(e);
  }
}
}  // namespace

extern "C" {

// A program whose coefficient t is words[t*coeff_limbs .. +coeff_limbs)
// (two's complement), built by the reference's own canonicalize / build /
// lazy heights / compile.
int ref_create_wide(const std::uint32_t* exps, const std::uint64_t* words, std::uint32_t coeff_limbs,
                    std::size_t nterms, std::uint32_t nvars, const int* upper, const int* lower,
                    const std::uint64_t* cutoff, void** out) {
  return guarded([&] {
    auto rp = std::make_unique<RefProgram>();
    rp->integer = true;
    rp->nvars = nvars;
    std::vector<std::string> vars;
    for (std::uint32_t v = 0; v < nvars; ++v) {
      vars.push_back(nvars <= 3 ? std::string(1, "xyz"[v]) : "x" + std::to_string(v));
    }
    std::vector<Term> raw(nterms);
    for (std::size_t t = 0; t < nterms; ++t) {
      raw[t].coefficient = big_of_words(words + t * coeff_limbs, coeff_limbs);
      raw[t].exponents.assign(exps + t * nvars, exps + (t + 1) * nvars);
    }
    Polynomial p = Polynomial::canonicalize(std::move(raw), vars);
    std::vector<FunctionScheme> schemes;
    for (std::uint32_t v = 0; v < nvars; ++v) schemes.push_back(scheme_of(upper[v], lower[v], cutoff[v]));
    EvaluationTree tree = nvars == 1 ? build(p, schemes[0], 0) : build_multivariate(p, schemes);
    compute_lazy_heights(tree);
    rp->program = std::make_unique<CompiledProgram>(compile(tree));
    rp->tree = std::make_unique<EvaluationTree>(std::move(tree));
    *out = rp.release();
    return 0;
  });
}

// Compares results (out_limbs two's-complement words per point) with the
// reference BigInt results at the same points; *mismatches = differing points.
int ref_eval_wide_check(void* h, const std::uint64_t* const* coords, std::uint32_t point_limbs,
                        std::size_t n, const std::uint64_t* got, std::uint32_t out_limbs, int threads,
                        std::size_t* mismatches) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    std::vector<char> bad(n, 0);
    wide_sharded(rp, n, threads, [&](Evaluator<BigIntDomain>& s, std::size_t i) {
      std::vector<BigInt> pt(rp.nvars);
      for (std::size_t v = 0; v < rp.nvars; ++v) pt[v] = big_of_words(coords[v] + i * point_limbs, point_limbs);
      const BigInt want = s.evaluate(std::span<const BigInt>(pt));
      bad[i] = !(want == big_of_words(got + i * out_limbs, out_limbs));
    });
    *mismatches = static_cast<std::size_t>(std::count(bad.begin(), bad.end(), 1));
    return 0;
  });
}

// Wall time of evaluating the n points (BigIntDomain, `threads` sessions).
int ref_time_wide(void* h, const std::uint64_t* const* coords, std::uint32_t point_limbs, std::size_t n,
                  int threads, double* seconds) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    std::vector<std::vector<BigInt>> pts(n, std::vector<BigInt>(rp.nvars));
    for (std::size_t i = 0; i < n; ++i) {
      for (std::size_t v = 0; v < rp.nvars; ++v) pts[i][v] = big_of_words(coords[v] + i * point_limbs, point_limbs);
    }
    std::vector<std::size_t> sink(n);
    const auto t0 = std::chrono::steady_clock::now();
    wide_sharded(rp, n, threads, [&](Evaluator<BigIntDomain>& s, std::size_t i) {
      sink[i] = s.evaluate(std::span<const BigInt>(pts[i])).bit_length();
    });
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  });
}

// evaluate_parallel (intra-point threading, eval.hpp:97-140) for `n` points
int ref_eval_parallel_f64(void* h, const double* const* coords, std::size_t n, double* out,
                          unsigned workers) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    std::vector<double> p(rp.nvars);
    if (rp.integer) {
      Evaluator<DoubleDomain> s(DoubleDomain{}, *rp.program);
      for (std::size_t i = 0; i < n; ++i) {
        for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = coords[v][i];
        out[i] = s.evaluate_parallel(std::span<const double>(p), workers);
      }
    } else {
      Evaluator<ScaledDoubleDomain> s(ScaledDoubleDomain{rp.shift}, *rp.program);
      for (std::size_t i = 0; i < n; ++i) {
        for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = coords[v][i];
        out[i] = s.evaluate_parallel(std::span<const double>(p), workers);
      }
    }
    return 0;
  });
}

// evaluate_parallel in the interval and BigInt domains: seconds for `n`
// points (the results are checked elsewhere; this is the CPU-baseline leg)
int ref_time_parallel_interval(void* h, const double* const* lo, const double* const* hi,
                               std::size_t n, unsigned workers, double* seconds) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    Evaluator<ScaledIntervalDomain> s(ScaledIntervalDomain{rp.integer ? 0 : rp.shift}, *rp.program);
    std::vector<Interval> p(rp.nvars);
    double sink = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (std::size_t i = 0; i < n; ++i) {
      for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = Interval(lo[v][i], hi[v][i]);
      sink += s.evaluate_parallel(std::span<const Interval>(p), workers).lo;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (sink == 12345.678) *seconds += 0;  // keep the loop
    return 0;
  });
}

int ref_time_parallel_i64(void* h, const std::int64_t* const* coords, std::size_t n,
                          unsigned workers, double* seconds) {
  return guarded([&] {
    const RefProgram& rp = *static_cast<RefProgram*>(h);
    if (!rp.integer) throw std::invalid_argument("integer evaluation needs integer coefficients");
    Evaluator<BigIntDomain> s(BigIntDomain{}, *rp.program);
    std::vector<BigInt> p(rp.nvars);
    std::size_t sink = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (std::size_t i = 0; i < n; ++i) {
      for (std::size_t v = 0; v < rp.nvars; ++v) p[v] = BigInt(coords[v][i]);
      sink += s.evaluate_parallel(std::span<const BigInt>(p), workers).is_zero() ? 1 : 0;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (sink == static_cast<std::size_t>(-1)) *seconds += 0;
    return 0;
  });
}

}  // extern "C"
