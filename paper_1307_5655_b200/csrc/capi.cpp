// C ABI (include/polyeval_b200.h) over the host front-end, the lowering /
// PTX emitter, the in-process JIT and the launch runtime.
//
// Reference mapping: pe_program_create = canonicalize + build /
// build_multivariate + compute_lazy_heights + compile (polynomial.cpp:13-33,
// tree.cpp:159-227, eval.cpp:52-69), restated in front/*.hpp;
// pe_eval_* = Evaluator<D>::evaluate over a batch (eval.hpp:74-90), one GPU
// thread per point instead of one call per point.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "front/flat.hpp"
#include "front/forest.hpp"
#include "front/split.hpp"
#include "front/terms.hpp"
#include "lower/ptx.hpp"
#include "lower/stream.hpp"
#include "polyeval_b200.h"
#include "runtime/jit.hpp"
#include "runtime/launch.hpp"
#include "runtime/program.hpp"

extern "C" cudaError_t pe_launch_max_abs_i64(const long long* x, size_t n,
                                             unsigned long long* out, int sms,
                                             cudaStream_t stream);
extern "C" cudaError_t pe_measure_pipe_peak(int kind, int sms, double* ops_per_s);
extern "C" cudaError_t pe_launch_narrow_limbs(const unsigned long long* const* limbs, int k,
                                              size_t n, long long* out, unsigned* flag, int sms,
                                              cudaStream_t stream);
extern "C" cudaError_t pe_measure_dfma_latency(double* cycles_per_op);
extern "C" cudaError_t pe_launch_wide(const std::uint32_t* code, std::uint32_t nops,
                                      const std::uint32_t* slot_off, const std::uint32_t* slot_w,
                                      const std::uint32_t* coef_off, const std::uint32_t* coef_w,
                                      const std::uint64_t* coef_words, std::uint32_t nvars,
                                      const std::uint64_t* const* in, std::uint32_t point_limbs,
                                      std::uint64_t* out, std::uint32_t out_limbs,
                                      std::uint32_t result, std::uint32_t result_w,
                                      std::uint32_t arena, std::uint32_t tmp_w,
                                      std::uint64_t* scratch, unsigned grid, unsigned threads,
                                      unsigned long long n, cudaStream_t stream);

struct pe_program {
  polyeval::rt::Program impl;
};

namespace polyeval::rt {
namespace {
thread_local std::string g_last_error;

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

std::vector<std::string> variable_names(std::uint32_t nvars) {
  std::vector<std::string> out;
  for (std::uint32_t v = 0; v < nvars; ++v) {
    out.push_back(nvars <= 3 ? std::string(1, "xyz"[v]) : "x" + std::to_string(v));
  }
  return out;
}

template <typename C>
std::unique_ptr<Front<C>> build_front(Program& p, const std::uint32_t* exps, const C* coeffs,
                                      size_t nterms, std::uint32_t nvars,
                                      const pe_scheme_desc* schemes) {
  auto fr = std::make_unique<Front<C>>();
  fr->terms = front::canonical_terms(exps, coeffs, nterms, nvars);
  std::vector<front::SplitRule> rules;
  for (std::uint32_t v = 0; v < nvars; ++v) {
    rules.push_back(front::SplitRule{schemes[v].upper, schemes[v].lower, schemes[v].cutoff});
  }
  fr->forest = std::make_unique<front::Forest<C>>(
      front::build_forest(fr->terms, std::span<const front::SplitRule>(rules)));
  fr->flat = front::compile_forest(*fr->forest);
  p.nterms = fr->terms.size();
  p.variables = variable_names(nvars);
  p.stats = front::walk_stats(fr->flat);
  return fr;
}

// ---- pe_program_from_compiled: flat reference CompiledProgram -> FlatProgram ----

// Checks one program's register discipline (the reference's lazy-height
// contract, tree.hpp:68-77): every non-root record accumulates into a
// register a later record reads, every read register was accumulated into,
// and every slot is in range.
void check_program(const pe_compiled_program& src, std::uint32_t nvars,
                   const std::vector<std::vector<std::uint32_t>>& sets) {
  if (src.nrecords == 0 || !src.records) throw std::invalid_argument("program without records");
  if (src.register_count == 0) throw std::invalid_argument("register_count must be >= 1");
  if (src.variable >= nvars) throw std::invalid_argument("program variable out of range");
  const size_t n = src.nrecords;
  std::vector<char> pending_read(src.register_count, 0);  // scanning backwards
  for (size_t i = n; i-- > 0;) {
    const pe_record& r = src.records[i];
    if (r.lazy_slot >= src.register_count) throw std::invalid_argument("lazy_slot out of range");
    if (r.reads_register != 0 && r.reads_register != 1) {
      throw std::invalid_argument("reads_register must be 0 or 1");
    }
    if (r.power_slot < -1 ||
        (r.power_slot >= 0 && static_cast<size_t>(r.power_slot) >= sets[src.variable].size())) {
      throw std::invalid_argument("power_slot out of range");
    }
    if (i + 1 == n) {
      if (r.parent_slot != -1) throw std::invalid_argument("root record has a parent_slot");
    } else if (r.parent_slot < 0 || static_cast<std::uint32_t>(r.parent_slot) >= src.register_count) {
      throw std::invalid_argument("parent_slot out of range");
    } else if (!pending_read[static_cast<std::uint32_t>(r.parent_slot)]) {
      throw std::invalid_argument("record accumulates into a register no later record reads");
    }
    if (r.reads_register) pending_read[r.lazy_slot] = 1;
  }
  std::vector<char> written(src.register_count, 0);
  for (size_t i = 0; i < n; ++i) {
    const pe_record& r = src.records[i];
    if (r.reads_register) {
      if (!written[r.lazy_slot]) throw std::invalid_argument("record reads a register nothing wrote");
      written[r.lazy_slot] = 0;
    }
    if (i + 1 < n) written[static_cast<std::uint32_t>(r.parent_slot)] = 1;
  }
  if (src.nroot_child_ends > 0 && !src.root_child_ends) {
    throw std::invalid_argument("root_child_ends is null");
  }
  for (size_t k = 0; k < src.nroot_child_ends; ++k) {
    const std::uint32_t e = src.root_child_ends[k];
    if (e >= n || (k > 0 && e <= src.root_child_ends[k - 1])) {
      throw std::invalid_argument("root_child_ends must be ascending record indices");
    }
  }
}

// Imports the programs in the caller's numbering (programs[0] is the root;
// each nested program referenced exactly once, all reachable from the root).
template <typename C>
front::FlatProgram<C> import_programs(const pe_compiled_program* progs, size_t np,
                                      std::uint32_t nvars,
                                      std::vector<std::vector<std::uint32_t>> sets) {
  for (size_t k = 0; k < np; ++k) check_program(progs[k], nvars, sets);
  std::vector<int> refs(np, 0);
  for (size_t k = 0; k < np; ++k) {
    for (size_t i = 0; i < progs[k].nrecords; ++i) {
      const std::int32_t sub = progs[k].records[i].sub;
      if (sub == -1) continue;
      if (sub < -1 || static_cast<size_t>(sub) >= np) {
        throw std::invalid_argument("nested program index out of range");
      }
      if (sub == 0) throw std::invalid_argument("the root program cannot be nested");
      if (++refs[static_cast<size_t>(sub)] > 1) throw std::invalid_argument("program referenced more than once");
    }
  }
  // reachability from the root (each program has at most one referrer, so
  // an unreachable program would sit on a cycle or be unreferenced)
  std::vector<char> seen(np, 0);
  std::vector<size_t> todo{0};
  seen[0] = 1;
  while (!todo.empty()) {
    const size_t k = todo.back();
    todo.pop_back();
    for (size_t i = 0; i < progs[k].nrecords; ++i) {
      const std::int32_t sub = progs[k].records[i].sub;
      if (sub > 0 && !seen[static_cast<size_t>(sub)]) {
        seen[static_cast<size_t>(sub)] = 1;
        todo.push_back(static_cast<size_t>(sub));
      }
    }
  }
  for (size_t k = 0; k < np; ++k) {
    if (!seen[k]) throw std::invalid_argument("program not reachable from the root");
  }
  front::FlatProgram<C> fp;
  fp.nvars = nvars;
  fp.exponent_sets = std::move(sets);
  for (size_t k = 0; k < np; ++k) {
    const pe_compiled_program& src = progs[k];
    typename front::FlatProgram<C>::Prog pr;
    pr.var = src.variable;
    pr.regs = src.register_count;
    pr.first = static_cast<std::uint32_t>(fp.recs.size());
    pr.count = static_cast<std::uint32_t>(src.nrecords);
    pr.root_child_ends.assign(src.root_child_ends, src.root_child_ends + src.nroot_child_ends);
    for (size_t i = 0; i < src.nrecords; ++i) {
      const pe_record& r = src.records[i];
      typename front::FlatProgram<C>::Rec d;
      d.sub = r.sub;
      if (r.sub < 0) {
        if constexpr (std::is_same_v<C, double>) {
          if (!std::isfinite(r.coeff_f64)) throw std::invalid_argument("coefficient is not finite");
          d.coef = r.coeff_f64;
        } else {
          d.coef = r.coeff_i64;
        }
      }
      d.power = r.power_slot;
      d.lazy = r.lazy_slot;
      d.parent = r.parent_slot;
      d.reads = r.reads_register != 0;
      fp.recs.push_back(d);
    }
    fp.progs.push_back(std::move(pr));
  }
  return fp;
}

// The polynomial an imported program evaluates, one row per scalar record
// (like terms not merged): record i of a program over variable v contributes
// coef * v^(sum of the powers on its way to the program's last record), times
// the exponents of the enclosing programs. Every intermediate of the walk is
// a partial sum of these terms times a sub-product of their powers, so the
// int64 overflow proof over them is sound.
template <typename C>
front::TermTable<C> path_terms(const front::FlatProgram<C>& fp) {
  front::TermTable<C> T;
  T.nvars = fp.nvars;
  struct Frame {
    std::uint32_t prog;
    std::vector<std::uint32_t> prefix;
  };
  std::vector<Frame> todo{{0, std::vector<std::uint32_t>(fp.nvars, 0)}};
  while (!todo.empty()) {
    Frame fr = std::move(todo.back());
    todo.pop_back();
    const auto& P = fp.progs[fr.prog];
    const auto up = front::consumers(fp, fr.prog);
    std::vector<std::uint64_t> total(P.count, 0);
    for (std::uint32_t i = P.count; i-- > 0;) {
      const auto& r = fp.rec(fr.prog, i);
      const std::uint64_t own = r.power >= 0 ? fp.exponent(fr.prog, r.power) : 0;
      total[i] = own + (up[i] == UINT32_MAX ? 0 : total[up[i]]);
      if (total[i] + fr.prefix[P.var] > UINT32_MAX) {
        throw std::invalid_argument("exponent overflow in compiled program");
      }
    }
    for (std::uint32_t i = 0; i < P.count; ++i) {
      const auto& r = fp.rec(fr.prog, i);
      std::vector<std::uint32_t> row = fr.prefix;
      row[P.var] += static_cast<std::uint32_t>(total[i]);
      if (r.sub >= 0) {
        todo.push_back({static_cast<std::uint32_t>(r.sub), std::move(row)});
      } else if (r.coef != C{}) {
        T.coefs.push_back(r.coef);
        T.exps.insert(T.exps.end(), row.begin(), row.end());
      }
    }
  }
  return T;
}

template <typename C>
std::unique_ptr<Front<C>> import_front(Program& p, const pe_compiled_program* progs, size_t np,
                                       std::uint32_t nvars,
                                       std::vector<std::vector<std::uint32_t>> sets) {
  auto fr = std::make_unique<Front<C>>();
  fr->flat = import_programs<C>(progs, np, nvars, std::move(sets));
  fr->terms = path_terms(fr->flat);
  std::vector<std::vector<std::uint32_t>> keys;
  for (size_t t = 0; t < fr->terms.size(); ++t) {
    keys.emplace_back(fr->terms.row(t), fr->terms.row(t) + nvars);
  }
  std::sort(keys.begin(), keys.end());
  p.nterms = static_cast<std::uint64_t>(std::unique(keys.begin(), keys.end()) - keys.begin());
  p.variables = variable_names(nvars);
  p.stats = front::walk_stats(fr->flat);
  return fr;
}

// exec->devices: one host thread per device, each running the single-device
// call on its contiguous slice (host buffers only; each slice's results go
// straight to the caller's output, so the gather is the pipelines' D2H).
template <typename Fn>
pe_status across_devices(const pe_exec& ex, size_t n, const void* probe, Fn&& fn) {
  if (!ex.devices) return fail(PE_EINVAL, "devices is null");
  int ignored = -1;
  if (classify(probe, &ignored) == MemKind::Device) {
    return fail(PE_EINVAL, "multi-device calls take host buffers");
  }
  const size_t nd = static_cast<size_t>(ex.ndevices);
  const size_t per = (n + nd - 1) / nd;
  std::vector<pe_status> st(nd, PE_OK);
  std::vector<std::string> msg(nd);
  std::vector<std::thread> pool;
  for (size_t k = 0; k < nd; ++k) {
    const size_t lo = std::min(n, k * per), cnt = std::min(n, lo + per) - lo;
    if (cnt == 0) continue;
    pool.emplace_back([&, k, lo, cnt] {
      pe_exec e = ex;
      e.device = ex.devices[k];
      e.devices = nullptr;
      e.ndevices = 0;
      st[k] = fn(e, lo, cnt);
      if (st[k] != PE_OK) msg[k] = g_last_error;
    });
  }
  for (auto& t : pool) t.join();
  for (size_t k = 0; k < nd; ++k) {
    if (st[k] != PE_OK) return fail(st[k], "device " + std::to_string(ex.devices[k]) + ": " + msg[k]);
  }
  return PE_OK;
}

bool multi_device(const pe_exec* exec) { return exec && exec->ndevices > 0; }

}  // namespace
}  // namespace polyeval::rt

using namespace polyeval;
using namespace polyeval::rt;

extern "C" {

const char* pe_last_error(void) { return g_last_error.c_str(); }
const char* pe_version(void) { return "polyeval-b200 0.1 (sm_100a)"; }
uint64_t pe_launch_count(void) { return launch_counter().load(); }

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
      p.i = build_front(p, exponents, static_cast<const std::int64_t*>(coeffs), nterms, nvars,
                        schemes);
      p.i64_uniform_bound = uniform_bounds(p, 63);
      p.i53_uniform_bound = uniform_bounds(p, 53);
    } else {
      const double* c = static_cast<const double*>(coeffs);
      for (size_t t = 0; t < nterms; ++t) {
        if (!std::isfinite(c[t])) return fail(PE_EINVAL, "coefficient is not finite");
      }
      p.f = build_front(p, exponents, c, nterms, nvars, schemes);
    }
    *out = h.release();
    return PE_OK;
  });
}

pe_status pe_program_create_wide(const uint32_t* exponents, const uint64_t* coeff_words,
                                 uint32_t coeff_limbs, size_t nterms, uint32_t nvars,
                                 const pe_scheme_desc* schemes, pe_program** out) {
  return guarded([&]() -> pe_status {
    if (!out) return fail(PE_EINVAL, "out is null");
    *out = nullptr;
    if (nvars == 0) return fail(PE_EINVAL, "nvars must be >= 1");
    if (!schemes) return fail(PE_EINVAL, "schemes is null");
    if (coeff_limbs == 0) return fail(PE_EINVAL, "coeff_limbs must be >= 1");
    if (nterms > 0 && (!exponents || !coeff_words)) return fail(PE_EINVAL, "terms are null");
    if (nterms >= (std::size_t{1} << 62)) return fail(PE_EINVAL, "too many terms");
    // keep the nonzero terms; each gets the placeholder coefficient
    // (index + 1) the front end builds the tree with
    auto wf = std::make_unique<WideFront>();
    std::vector<std::uint32_t> exps;
    std::vector<std::int64_t> ph;
    for (size_t t = 0; t < nterms; ++t) {
      const uint64_t* w = coeff_words + t * coeff_limbs;
      if (std::all_of(w, w + coeff_limbs, [](uint64_t x) { return x == 0; })) continue;
      wf->coefs.emplace_back(w, w + coeff_limbs);
      exps.insert(exps.end(), exponents + t * nvars, exponents + (t + 1) * nvars);
      ph.push_back(static_cast<std::int64_t>(wf->coefs.size()));
    }
    std::vector<std::uint32_t> order(ph.size());
    for (std::uint32_t k = 0; k < order.size(); ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
      return std::lexicographical_compare(exps.begin() + a * nvars, exps.begin() + (a + 1) * nvars,
                                          exps.begin() + b * nvars, exps.begin() + (b + 1) * nvars);
    });
    for (size_t k = 1; k < order.size(); ++k) {
      if (std::equal(exps.begin() + order[k] * nvars, exps.begin() + (order[k] + 1) * nvars,
                     exps.begin() + order[k - 1] * nvars)) {
        return fail(PE_EINVAL, "wide programs need distinct exponent rows");
      }
    }
    auto h = std::make_unique<pe_program>();
    Program& p = h->impl;
    p.nvars = nvars;
    p.integer = true;
    p.i = build_front(p, exps.data(), ph.data(), ph.size(), nvars, schemes);
    p.wide = std::move(wf);
    *out = h.release();
    return PE_OK;
  });
}

pe_status pe_program_wide_limbs(const pe_program* program, uint32_t point_limbs,
                                uint32_t* out_limbs) {
  return guarded([&]() -> pe_status {
    if (!program || !out_limbs) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    if (!p.wide) return fail(PE_EINVAL, "not a wide program (pe_program_create_wide)");
    std::lock_guard<std::mutex> lock(p.mu);
    auto it = p.wide->plans.find(point_limbs);
    if (it == p.wide->plans.end()) {
      it = p.wide->plans.emplace(point_limbs, plan_wide(p.i->flat, p.wide->coefs, point_limbs)).first;
    }
    *out_limbs = it->second.result_limbs;
    return PE_OK;
  });
}

pe_status pe_eval_wide(const pe_program* program, const uint64_t* const* coords,
                       uint32_t point_limbs, size_t n, uint64_t* out, uint32_t out_limbs,
                       const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    if (!p.wide) return fail(PE_EINVAL, "not a wide program (pe_program_create_wide)");
    if (n == 0) return PE_OK;
    if (!coords || !out) return fail(PE_EINVAL, "null buffer");
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    if (p.nvars > 16) return fail(PE_EINVAL, "at most 16 variables");
    uint32_t need = 0;
    const pe_status st = pe_program_wide_limbs(program, point_limbs, &need);
    if (st != PE_OK) return st;
    if (out_limbs < need) {
      return fail(PE_EOVERFLOW, "results need " + std::to_string(need) + " limbs");
    }
    MemKind kind;
    const int dev = resolve_device(exec, out, &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    const WidePlan* plan;
    WideDevice dv;
    {
      std::lock_guard<std::mutex> lock(p.mu);
      plan = &p.wide->plans.at(point_limbs);
      auto& slot = p.wide->dev[{dev, point_limbs}];
      if (!slot.code) {
        auto up = [](void** d, const void* src, size_t bytes) {
          check_cuda(cudaMalloc(d, std::max<size_t>(bytes, 8)), "cudaMalloc(wide plan)");
          if (bytes) check_cuda(cudaMemcpy(*d, src, bytes, cudaMemcpyHostToDevice), "wide plan upload");
        };
        up(&slot.code, plan->code.data(), plan->code.size() * 4);
        up(&slot.slot_off, plan->slot_off.data(), plan->slot_off.size() * 4);
        up(&slot.slot_w, plan->slot_w.data(), plan->slot_w.size() * 4);
        up(&slot.coef_off, plan->coef_off.data(), plan->coef_off.size() * 4);
        up(&slot.coef_w, plan->coef_w.data(), plan->coef_w.size() * 4);
        up(&slot.coef_words, plan->coef_words.data(), plan->coef_words.size() * 8);
      }
      dv = slot;
    }
    // inputs / outputs on the device (host buffers are copied: the walk of
    // one point is long, so staging is a small part of a wide call)
    std::vector<const std::uint64_t*> din(p.nvars);
    std::vector<void*> owned;
    auto cleanup = [&] {
      for (void* q : owned) cudaFreeAsync(q, s);
    };
    try {
      for (uint32_t v = 0; v < p.nvars; ++v) {
        int d2 = -1;
        if (classify(coords[v], &d2) == MemKind::Device) {
          din[v] = coords[v];
        } else {
          void* q = nullptr;
          check_cuda(cudaMallocAsync(&q, n * point_limbs * 8, s), "cudaMallocAsync(wide input)");
          owned.push_back(q);
          check_cuda(cudaMemcpyAsync(q, coords[v], n * point_limbs * 8, cudaMemcpyHostToDevice, s),
                     "wide input H2D");
          din[v] = static_cast<const std::uint64_t*>(q);
        }
      }
      std::uint64_t* dout = out;
      if (kind != MemKind::Device) {
        void* q = nullptr;
        check_cuda(cudaMallocAsync(&q, n * out_limbs * 8, s), "cudaMallocAsync(wide output)");
        owned.push_back(q);
        dout = static_cast<std::uint64_t*>(q);
      }
      // CTA size by value width (a narrow walk would leave most of a wide
      // CTA idle at every barrier); as many CTAs as fit 1024 threads per SM,
      // at most 4 GB of arenas
      const int sms = device_ctx(dev).sms;
      unsigned threads = plan->tmp_w <= 64 ? 32 : plan->tmp_w <= 256 ? 64
                         : plan->tmp_w <= 1024 ? 128 : 256;
      // ... and by batch size: the walk is latency-bound per op (barriers,
      // dependent loads), so points in flight matter more than threads per
      // point. A CTA gets more than one warp only when the batch is too
      // small to fill 1024 threads per SM with one-warp CTAs
      // (profiles/r2_wide_cta_sweep.jsonl: 64-bit d1000 at 4096 points,
      // 65.6k -> 135.6k points/s with one-warp CTAs).
      unsigned by_batch = 32;
      while (by_batch < 256 && static_cast<std::uint64_t>(n) * by_batch * 2 <= 1024ull * sms) {
        by_batch *= 2;
      }
      threads = std::min(threads, by_batch);
      if (p.tuning.block >= 32 && p.tuning.block <= 256 && p.tuning.block % 32 == 0) {
        threads = p.tuning.block;  // pe_tuning.block: CTA size of the wide walk
      }
      const size_t per_cta = static_cast<size_t>(plan->arena) + 5ull * plan->tmp_w;
      const std::uint64_t by_mem = std::max<std::uint64_t>(1, (std::uint64_t{4} << 30) / (per_cta * 8));
      // pe_tuning.min_ctas: CTAs per SM of the wide walk (default: 1024 threads per SM)
      const std::uint64_t per_sm = p.tuning.min_ctas ? p.tuning.min_ctas : 1024 / threads;
      const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(
          {n, static_cast<std::uint64_t>(sms) * per_sm, by_mem}));
      void* scratch = nullptr;
      keep_pool_memory(dev);
      check_cuda(cudaMallocAsync(&scratch, grid * per_cta * 8, s), "cudaMallocAsync(wide arena)");
      owned.push_back(scratch);
      check_cuda(pe_launch_wide(static_cast<const std::uint32_t*>(dv.code), plan->nops,
                                static_cast<const std::uint32_t*>(dv.slot_off),
                                static_cast<const std::uint32_t*>(dv.slot_w),
                                static_cast<const std::uint32_t*>(dv.coef_off),
                                static_cast<const std::uint32_t*>(dv.coef_w),
                                static_cast<const std::uint64_t*>(dv.coef_words), p.nvars, din.data(),
                                point_limbs, dout, out_limbs, plan->result, plan->result_limbs,
                                plan->arena, plan->tmp_w, static_cast<std::uint64_t*>(scratch), grid,
                                threads, n, s),
                 "launch(wide walk)");
      launch_counter().fetch_add(1, std::memory_order_relaxed);
      if (kind != MemKind::Device) {
        copy_to_host(out, dout, n * out_limbs * 8, dev, s);  // complete on return
      }
      cleanup();
      if (kind == MemKind::Device && exec && exec->synchronize) {
        check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      }
    } catch (...) {
      cleanup();
      throw;
    }
    return PE_OK;
  });
}

pe_status pe_program_check_registers(const pe_program* program) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    // each program's walk leaves its register file clean iff every register
    // accumulated into is read again later (eval.hpp:225-238)
    auto clean = [](const auto& fp) -> bool {
      for (std::uint32_t k = 0; k < fp.progs.size(); ++k) {
        const auto& P = fp.progs[k];
        std::vector<char> live(P.regs, 0);
        for (std::uint32_t i = 0; i < P.count; ++i) {
          const auto& r = fp.rec(k, i);
          if (r.reads) live[r.lazy] = 0;
          if (i + 1 < P.count && r.parent >= 0) live[static_cast<std::uint32_t>(r.parent)] = 1;
        }
        if (std::find(live.begin(), live.end(), 1) != live.end()) return false;
      }
      return true;
    };
    const bool ok = p.integer ? clean(p.i->flat) : clean(p.f->flat);
    if (!ok) return fail(PE_ELOGIC, "register file not clean after walk");
    return PE_OK;
  });
}

pe_status pe_program_from_compiled(const pe_compiled_program* programs, size_t nprograms,
                                   uint32_t nvars, const uint32_t* const* exponent_sets,
                                   const size_t* exponent_set_sizes, pe_coeff_type coeff_type,
                                   pe_program** out) {
  return guarded([&]() -> pe_status {
    if (!out) return fail(PE_EINVAL, "out is null");
    *out = nullptr;
    if (!programs || nprograms == 0) return fail(PE_EINVAL, "no programs");
    if (nvars == 0) return fail(PE_EINVAL, "nvars must be >= 1");
    if (!exponent_sets || !exponent_set_sizes) return fail(PE_EINVAL, "exponent sets are null");
    if (coeff_type != PE_COEFF_F64 && coeff_type != PE_COEFF_I64) {
      return fail(PE_EINVAL, "unknown coefficient type");
    }
    std::vector<std::vector<std::uint32_t>> sets(nvars);
    for (uint32_t v = 0; v < nvars; ++v) {
      const size_t k = exponent_set_sizes[v];
      if (k > 0 && !exponent_sets[v]) return fail(PE_EINVAL, "exponent set is null");
      for (size_t i = 0; i < k; ++i) {
        const uint32_t e = exponent_sets[v][i];
        if (e == 0 || (i > 0 && e <= exponent_sets[v][i - 1])) {
          return fail(PE_EINVAL, "exponent sets must be ascending, distinct and >= 1");
        }
        sets[v].push_back(e);
      }
    }
    auto h = std::make_unique<pe_program>();
    Program& p = h->impl;
    p.nvars = nvars;
    p.integer = coeff_type == PE_COEFF_I64;
    if (p.integer) {
      p.i = import_front<std::int64_t>(p, programs, nprograms, nvars, std::move(sets));
      p.i64_uniform_bound = uniform_bounds(p, 63);
      p.i53_uniform_bound = uniform_bounds(p, 53);
    } else {
      p.f = import_front<double>(p, programs, nprograms, nvars, std::move(sets));
    }
    *out = h.release();
    return PE_OK;
  });
}

void pe_program_destroy(pe_program* program) { delete program; }

pe_status pe_program_set_tuning(pe_program* program, const pe_tuning* t) {
  return guarded([&]() -> pe_status {
    if (!program || !t) return fail(PE_EINVAL, "null argument");
    Program& p = program->impl;
    p.release();
    std::lock_guard<std::mutex> lock(p.mu);
    lower::Tuning& d = p.tuning;
    d.lanes = t->lanes;
    d.block = t->block;
    d.min_ctas = t->min_ctas;
    d.sync_every = t->sync_every;
    d.section_ops = t->section_ops;
    d.sched_window = t->sched_window;
    d.sched_distance = t->sched_distance;
    d.chain_min = t->chain_min;
    d.iv_fast = t->iv_fast;
    d.iv_mid = t->iv_mid;
    d.iv_partition = t->iv_partition;
    d.group_tiles = t->group_tiles;
    d.word_layout = t->word_layout;
    d.jit_mode = t->jit_mode;
    d.iv_partition_min = t->iv_partition_min;
    return PE_OK;
  });
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
    auto fill = [&](const auto& fp) {
      info->register_count = fp.progs[0].regs;
      info->root_children = static_cast<uint32_t>(fp.progs[0].root_child_ends.size());
      for (size_t v = 0; v < fp.exponent_sets.size() && v < 8; ++v) {
        info->exponent_set_sizes[v] = static_cast<uint32_t>(fp.exponent_sets[v].size());
      }
    };
    if (p.integer) fill(p.i->flat); else fill(p.f->flat);
    return PE_OK;
  });
}

pe_status pe_program_exponents(const pe_program* program, uint32_t v, uint32_t* out, size_t cap,
                               size_t* count) {
  return guarded([&]() -> pe_status {
    if (!program || !count) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    const auto& sets = p.integer ? p.i->flat.exponent_sets : p.f->flat.exponent_sets;
    if (v >= sets.size() || v >= p.nvars) return fail(PE_EINVAL, "variable index out of range");
    const auto& e = sets[v];
    *count = e.size();
    for (size_t i = 0; i < e.size() && i < cap && out; ++i) out[i] = e[i];
    return PE_OK;
  });
}

pe_status pe_program_records(const pe_program* program, int32_t* out, size_t cap, size_t* count) {
  return guarded([&]() -> pe_status {
    if (!program || !count) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    auto dump = [&](const auto& fp) {
      const std::uint32_t n = fp.progs[0].count;
      *count = n;
      for (size_t i = 0; i < n && (i + 1) * 5 <= cap && out; ++i) {
        const auto& r = fp.rec(0, static_cast<std::uint32_t>(i));
        out[5 * i + 0] = r.power;
        out[5 * i + 1] = static_cast<int32_t>(r.lazy);
        out[5 * i + 2] = r.parent;
        out[5 * i + 3] = r.reads ? 1 : 0;
        out[5 * i + 4] = r.sub >= 0 ? 1 : 0;
      }
    };
    if (p.integer) dump(p.i->flat); else dump(p.f->flat);
    return PE_OK;
  });
}

pe_status pe_program_dot(const pe_program* program, char* out, size_t cap, size_t* len) {
  return guarded([&]() -> pe_status {
    if (!program || !len) return fail(PE_EINVAL, "null argument");
    const Program& p = program->impl;
    if (p.integer ? !p.i->forest : !p.f->forest) {
      return fail(PE_EINVAL, "program was created from a compiled program and has no tree");
    }
    const std::span<const std::string> names(p.variables);
    const std::string dot = p.integer ? front::forest_dot(*p.i->forest, names)
                                      : front::forest_dot(*p.f->forest, names);
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

// domain codes 0..4, or PE_DOMAIN_LIMBS(K) = 0x100 | K for the K-limb kernel
static const Artifact& artifact_for(const Program& p, int32_t domain, bool need_cubin) {
  if (domain & 0x100) return p.limb_artifact(static_cast<std::uint32_t>(domain & 0xff), need_cubin);
  return p.artifact(to_domain(domain), need_cubin);
}

pe_status pe_program_kernel_stats(const pe_program* program, int32_t domain, uint64_t* fp_ops,
                                  uint64_t* int_ops, uint64_t* ptx_bytes) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "null argument");
    const Artifact& a = artifact_for(program->impl, domain, false);
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
    const Artifact& a = artifact_for(program->impl, domain, false);
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

pe_status pe_program_kernel_ready(const pe_program* program, int32_t domain, int32_t* ready) {
  return guarded([&]() -> pe_status {
    if (!program || !ready) return fail(PE_EINVAL, "null argument");
    const Artifact& a = program->impl.artifact(to_domain(domain), false);
    *ready = a.cubin_ready.load(std::memory_order_acquire) ? 1 : 0;
    return PE_OK;
  });
}

pe_status pe_program_f64_slices(const pe_program* program, uint32_t* slices) {
  return guarded([&]() -> pe_status {
    if (!program || !slices) return fail(PE_EINVAL, "null argument");
    *slices = program->impl.artifact(lower::Domain::F64, false).image.sections;
    return PE_OK;
  });
}

pe_status pe_program_compile_only(const pe_program* program, int32_t domain, uint64_t* cubin_bytes) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "null argument");
    const Artifact& a = artifact_for(program->impl, domain, true);
    if (cubin_bytes) *cubin_bytes = a.cubin.size();
    return PE_OK;
  });
}

pe_status pe_measure_peak(int32_t device, int32_t kind, double* ops_per_s, int32_t* sms) {
  return guarded([&]() -> pe_status {
    if (!ops_per_s || kind < 0 || kind > 3) return fail(PE_EINVAL, "bad argument");
    if (device >= 0) check_cuda(cudaSetDevice(device), "cudaSetDevice");
    int dev = 0, n_sm = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    check_cuda(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev), "attr");
    if (kind == 2) {
      check_cuda(pe_measure_dfma_latency(ops_per_s), "DFMA latency microbenchmark");
    } else {
      check_cuda(pe_measure_pipe_peak(kind, n_sm, ops_per_s), "pipe peak microbenchmark");
    }
    launch_counter().fetch_add(5, std::memory_order_relaxed);
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
    if (p.wide) return fail(PE_EINVAL, "a wide program evaluates through pe_eval_wide");
    if (n == 0) return PE_OK;
    if (!coords || !out) return fail(PE_EINVAL, "null buffer");
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    if (multi_device(exec)) {
      return across_devices(*exec, n, out, [&](const pe_exec& e, size_t lo, size_t cnt) {
        std::vector<const double*> c(p.nvars);
        for (uint32_t v = 0; v < p.nvars; ++v) c[v] = coords[v] + lo;
        return pe_eval_f64(program, c.data(), cnt, out + lo, &e);
      });
    }
    const bool strict = exec && exec->strict_f64;
    MemKind kind;
    const int dev = resolve_device(exec, out, &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    const std::vector<const Artifact*> arts{
        &p.for_launch(strict ? lower::Domain::F64Strict : lower::Domain::F64, dev)};
    std::vector<const void*> ins(coords, coords + p.nvars);
    std::vector<void*> outs{out};
    LaunchArgs la;
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    run_batch(arts, dev, kind, n, ins, outs, la, s, exec && exec->synchronize, false, {},
              staging_of(exec));
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
      if (programs[j]->impl.wide) return fail(PE_EINVAL, "a wide program evaluates through pe_eval_wide");
    }
    for (uint32_t v = 0; v < nv; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    if (multi_device(exec)) {
      return across_devices(*exec, n, outs[0], [&](const pe_exec& e, size_t lo, size_t cnt) {
        std::vector<const double*> c(nv);
        for (uint32_t v = 0; v < nv; ++v) c[v] = coords[v] + lo;
        std::vector<double*> o(k);
        for (size_t j = 0; j < k; ++j) o[j] = outs[j] + lo;
        return pe_eval_f64_multi(programs, k, c.data(), cnt, o.data(), &e);
      });
    }
    MemKind kind;
    const int dev = resolve_device(exec, outs[0], &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    std::vector<const Artifact*> arts;
    std::vector<size_t> base;
    for (size_t j = 0; j < k; ++j) {
      arts.push_back(&programs[j]->impl.for_launch(lower::Domain::F64, dev));
      base.push_back(j);
    }
    std::vector<const void*> ins(coords, coords + nv);
    std::vector<void*> o(outs, outs + k);
    LaunchArgs la;
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    run_batch(arts, dev, kind, n, ins, o, la, s, exec && exec->synchronize, false, base,
              staging_of(exec));
    return PE_OK;
  });
}

pe_status pe_eval_interval(const pe_program* program, const double* const* lo,
                           const double* const* hi, size_t n, double* out_lo, double* out_hi,
                           const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    if (p.wide) return fail(PE_EINVAL, "a wide program evaluates through pe_eval_wide");
    if (n == 0) return PE_OK;
    if (!lo || !hi || !out_lo || !out_hi) return fail(PE_EINVAL, "null buffer");
    std::vector<const void*> ins;
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!lo[v] || !hi[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
      ins.push_back(lo[v]);
      ins.push_back(hi[v]);
    }
    if (multi_device(exec)) {
      return across_devices(*exec, n, out_lo, [&](const pe_exec& e, size_t off, size_t cnt) {
        std::vector<const double*> l(p.nvars), h(p.nvars);
        for (uint32_t v = 0; v < p.nvars; ++v) {
          l[v] = lo[v] + off;
          h[v] = hi[v] + off;
        }
        return pe_eval_interval(program, l.data(), h.data(), cnt, out_lo + off, out_hi + off, &e);
      });
    }
    MemKind kind;
    const int dev = resolve_device(exec, out_lo, &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    const Artifact& a = p.for_launch(lower::Domain::Interval, dev);
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
      run_batch(a, dev, kind, n, ins, {out_lo, out_hi}, la, s, false, attempt == 1, staging_of(exec));
      const unsigned f = flag.read();
      if (f & 2) return fail(PE_EINVAL, "invalid interval endpoints (NaN or lo > hi)");
      if (!(f & 4)) return PE_OK;
      // more points needed the strict replay than the fixup list held:
      // re-run with a list as large as the batch (cannot overflow)
    }
    return fail(PE_ELOGIC, "interval fixup list overflowed at full capacity");
  });
}

// Per-variable max |x| of an int64 SoA batch (device reduction kernel or a
// host loop).
std::vector<std::uint64_t> batch_abs_max(const Program& p, const int64_t* const* coords, size_t n,
                                         MemKind kind, int dev, cudaStream_t s) {
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
      launch_counter().fetch_add(1, std::memory_order_relaxed);
    }
    check_cuda(cudaMemcpyAsync(actual.data(), dmax, 8 * p.nvars, cudaMemcpyDeviceToHost, s), "D2H");
    check_cuda(cudaFreeAsync(dmax, s), "cudaFreeAsync");
    check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  } else {
    for (uint32_t v = 0; v < p.nvars; ++v) {
      std::uint64_t m = 0;
      for (size_t i = 0; i < n; ++i) {
        const int64_t x = coords[v][i];
        m = std::max<std::uint64_t>(m, x < 0 ? 0ull - static_cast<std::uint64_t>(x) : static_cast<std::uint64_t>(x));
      }
      actual[v] = m;
    }
  }
  return actual;
}

pe_status pe_program_limbs_needed(const pe_program* program, const uint64_t* bounds,
                                  uint32_t* limbs) {
  return guarded([&]() -> pe_status {
    if (!program || !bounds || !limbs) return fail(PE_EINVAL, "null argument");
    if (!program->impl.integer) return fail(PE_EINVAL, "multi-limb evaluation needs int64 coefficients");
    *limbs = limbs_needed(program->impl, bounds);
    return PE_OK;
  });
}

pe_status pe_eval_limbs(const pe_program* program, const int64_t* const* coords, size_t n,
                        uint32_t limbs, uint64_t* const* out_limbs, const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    if (p.wide) return fail(PE_EINVAL, "a wide program evaluates through pe_eval_wide");
    if (!p.integer) return fail(PE_EINVAL, "pe_eval_limbs needs a program with int64 coefficients");
    if (limbs < 1 || limbs > 8) return fail(PE_EINVAL, "limbs must be 1..8");
    if (n == 0) return PE_OK;
    if (!coords || !out_limbs) return fail(PE_EINVAL, "null buffer");
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    for (uint32_t k = 0; k < limbs; ++k) {
      if (!out_limbs[k]) return fail(PE_EINVAL, "null output limb array");
    }
    if (multi_device(exec)) {
      return across_devices(*exec, n, out_limbs[0], [&](const pe_exec& e, size_t lo, size_t cnt) {
        std::vector<const int64_t*> c(p.nvars);
        for (uint32_t v = 0; v < p.nvars; ++v) c[v] = coords[v] + lo;
        std::vector<uint64_t*> o(limbs);
        for (uint32_t k = 0; k < limbs; ++k) o[k] = out_limbs[k] + lo;
        return pe_eval_limbs(program, c.data(), cnt, limbs, o.data(), &e);
      });
    }
    MemKind kind;
    const int dev = resolve_device(exec, out_limbs[0], &kind);
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    cudaStream_t s = exec ? static_cast<cudaStream_t>(exec->stream) : nullptr;
    // the batch's own maxima: the proof then covers exactly these points and
    // the kernel's per-point bound check cannot fire
    const std::vector<std::uint64_t> bounds =
        exec && exec->i64_bounds
            ? std::vector<std::uint64_t>(exec->i64_bounds, exec->i64_bounds + p.nvars)
            : batch_abs_max(p, coords, n, kind, dev, s);
    const std::uint32_t need = limbs_needed(p, bounds.data());
    if (need == 0 || need > limbs) {
      return fail(PE_EOVERFLOW, "values need " + (need ? std::to_string(need) : std::string("> 8")) +
                                    " limbs for these coordinates");
    }
    const Artifact& a = p.loaded_limbs(limbs, dev);
    std::vector<const void*> ins(coords, coords + p.nvars);
    std::vector<void*> outs(out_limbs, out_limbs + limbs);
    Flag flag(s);
    LaunchArgs la;
    la.flag = reinterpret_cast<std::uint64_t>(flag.dev);
    la.bounds = bounds;
    run_batch(a, dev, kind, n, ins, outs, la, s, false, false, staging_of(exec));
    if (flag.read() != 0) return fail(PE_EOVERFLOW, "a coordinate exceeds the asserted bound");
    return PE_OK;
  });
}

pe_status pe_eval_i64(const pe_program* program, const int64_t* const* coords, size_t n,
                      int64_t* out, const pe_exec* exec) {
  return guarded([&]() -> pe_status {
    if (!program) return fail(PE_EINVAL, "program is null");
    const Program& p = program->impl;
    if (p.wide) return fail(PE_EINVAL, "a wide program evaluates through pe_eval_wide");
    if (!p.integer) return fail(PE_EINVAL, "pe_eval_i64 needs a program with int64 coefficients");
    if (n == 0) return PE_OK;
    if (!coords || !out) return fail(PE_EINVAL, "null buffer");
    for (uint32_t v = 0; v < p.nvars; ++v) {
      if (!coords[v]) return fail(PE_EINVAL, "evaluation point arity mismatch");
    }
    if (multi_device(exec)) {
      return across_devices(*exec, n, out, [&](const pe_exec& e, size_t lo, size_t cnt) {
        std::vector<const int64_t*> c(p.nvars);
        for (uint32_t v = 0; v < p.nvars; ++v) c[v] = coords[v] + lo;
        return pe_eval_i64(program, c.data(), cnt, out + lo, &e);
      });
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
          p.for_launch(tier53 ? lower::Domain::I64F : lower::Domain::I64, dev);
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
      const Artifact& af = p.for_launch(lower::Domain::I64F, dev);
      Flag flag(s);
      LaunchArgs la;
      la.flag = reinterpret_cast<std::uint64_t>(flag.dev);
      la.bounds = b53;
      run_batch(af, dev, kind, n, ins, {out}, la, s, false, false, staging_of(exec));
      if (flag.read() == 0) return PE_OK;
      if (caller_bounds) {
        return fail(PE_EOVERFLOW, "a coordinate exceeds the asserted int64 bound");
      }
    }
    // Tier 2: int64 multiply-adds, wrap-free by the 2^63 proof.
    const Artifact& a = p.for_launch(lower::Domain::I64, dev);
    for (int attempt = 0; attempt < 2; ++attempt) {
      Flag flag(s);
      LaunchArgs la;
      la.flag = reinterpret_cast<std::uint64_t>(flag.dev);
      la.bounds = bounds;
      run_batch(a, dev, kind, n, ins, {out}, la, s, false, false, staging_of(exec));
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
          launch_counter().fetch_add(1, std::memory_order_relaxed);
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
    if (caller_bounds) {
      return fail(PE_EOVERFLOW, "a coordinate exceeds the asserted int64 bound");
    }
    // Tier 3: intermediates may leave int64, results may still fit: evaluate
    // in K 64-bit limbs (exact, the batch's own maxima) and narrow, flagging
    // results that do not fit (the reference's int64 conversion fails there).
    const std::vector<std::uint64_t> actual = batch_abs_max(p, coords, n, kind, dev, s);
    const std::uint32_t K = limbs_needed(p, actual.data());
    if (K == 0) {
      return fail(PE_EOVERFLOW, "intermediates exceed 511 bits for these coordinates");
    }
    const Artifact& ak = p.loaded_limbs(K, dev);
    std::vector<void*> limbs(K, nullptr);
    std::vector<std::vector<std::uint64_t>> host_limbs;
    if (kind == MemKind::Device) {
      for (auto& l : limbs) check_cuda(cudaMallocAsync(&l, 8 * n, s), "cudaMallocAsync(limbs)");
    } else {
      host_limbs.assign(K, std::vector<std::uint64_t>(n));
      for (std::uint32_t k = 0; k < K; ++k) limbs[k] = host_limbs[k].data();
    }
    Flag flag(s);
    LaunchArgs la;
    la.flag = reinterpret_cast<std::uint64_t>(flag.dev);
    la.bounds = actual;
    run_batch(ak, dev, kind, n, ins, limbs, la, s, false, false, staging_of(exec));
    bool fits = true;
    if (kind == MemKind::Device) {
      std::vector<const unsigned long long*> lp(K);
      for (std::uint32_t k = 0; k < K; ++k) lp[k] = static_cast<const unsigned long long*>(limbs[k]);
      check_cuda(pe_launch_narrow_limbs(lp.data(), static_cast<int>(K), n,
                                        reinterpret_cast<long long*>(out), flag.dev,
                                        device_ctx(dev).sms, s),
                 "narrow_limbs");
      launch_counter().fetch_add(1, std::memory_order_relaxed);
      for (auto l : limbs) check_cuda(cudaFreeAsync(l, s), "cudaFreeAsync(limbs)");
      const unsigned f = flag.read();
      if (f & 1) return fail(PE_ELOGIC, "limb evaluation saw a coordinate beyond its own maxima");
      fits = (f & 8) == 0;
    } else {
      if (flag.read() & 1) return fail(PE_ELOGIC, "limb evaluation saw a coordinate beyond its own maxima");
      for (size_t i = 0; i < n; ++i) {
        const std::uint64_t v0 = host_limbs[0][i];
        const std::uint64_t ext = static_cast<std::uint64_t>(static_cast<std::int64_t>(v0) >> 63);
        for (std::uint32_t k = 1; k < K; ++k) fits = fits && host_limbs[k][i] == ext;
        out[i] = static_cast<int64_t>(v0);
      }
    }
    if (!fits) return fail(PE_EOVERFLOW, "a result does not fit int64 (use pe_eval_limbs)");
    return PE_OK;
  });
}

}  // extern "C"
