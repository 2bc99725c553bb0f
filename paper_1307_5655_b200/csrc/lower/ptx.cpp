// PTX emitter: lowered stream -> sm_100a kernel text.
//
// Each thread evaluates P points ("lanes") of one CTA tile: point
// tile_base + lane * blockDim + tid, so every coordinate load and result
// store of a warp is one coalesced 256-byte access. The walk is emitted once
// per lane, interleaved op by op: a coefficient is loaded from the constant
// bank once and feeds P independent FMAs, which (a) divides the per-thread
// constant-load traffic — the MIO-queue limiter of a one-point-per-thread walk
// (profiles/) — by P and (b) gives the FP64 pipe P independent dependency
// chains. The power DAG and the walk are straight-line code over PTX virtual
// registers; ptxas does the physical allocation, which is the job the
// reference's lazy heights do for its heap register file (tree.hpp:68-77).
//
// Per-domain arithmetic:
//   F64 / F64Strict  add.rn / mul.rn / fma.rn (strict streams contain no FMA,
//                    and .rn instructions are never contracted by ptxas)
//   I64              add.s64 / mul.lo.s64 / mad.lo.s64 (wrap-free: the host
//                    proves the range, the kernel checks |x| <= bound)
//   Interval         reference interval.cpp:12-52 verbatim: RN op, then one
//                    nextafter step outward per endpoint; products use the
//                    zero rule and the std::min/std::max({p1..p4}) scan order.
#include "lower/ptx.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <type_traits>
#include <unordered_map>

namespace polyeval::lower {

const char* domain_name(Domain d) {
  switch (d) {
    case Domain::F64: return "f64";
    case Domain::F64Strict: return "f64strict";
    case Domain::I64: return "i64";
    case Domain::Interval: return "interval";
    case Domain::I64F: return "i64f";
    case Domain::I64K: return "i64k";
  }
  return "?";
}

KernelShape default_shape(Domain d, std::uint32_t powers, std::uint64_t distinct_coefs,
                          const Tuning& t) {
  // Measured on B200 (profiles/r1_shape_sweep.txt): the fp64 walk of a
  // one-point-per-thread kernel is bound by per-thread constant loads (MIO);
  // P points per thread share each coefficient load. One 512-thread CTA per
  // SM (ptxas capped at 128 registers) beats several 128-thread CTAs.
  // Coefficients: a DFMA reads at most one uniform register, so the walk's
  // coefficients split into uniform-bound words (paired 16-byte LDCU) and the
  // register-bound second coefficient of fma(c, x^d, c') leaves (paired
  // per-thread LDC) — profiles/r1_imm6_sweep.txt: C4 4.23 -> 3.71 ms per 4e6
  // points, C2 0.683 -> 0.646 ms per 1e7, C3 0.610 -> 0.579 ms per 1e7.
  KernelShape s;
  if (d == Domain::Interval) {
    s = {1, 512, 32};  // integer-pipe bound; no coefficient pressure
  } else if (d == Domain::I64K) {
    s = {1, 256, 0};   // K-limb registers: one point per thread
  } else if (powers > 32 || distinct_coefs < 64) {
    // very wide programs (large power tables): registers are the limit; few
    // distinct coefficients: independent sub-chains give enough ILP
    s = {1, 512, 0};
  } else {
    s = {4, 256, 0};
    s.min_ctas = 2;  // <= 128 registers: two CTAs (16 warps) per SM
  }
  // strict fp64 keeps every reference add: more live temporaries; a 512-wide
  // CTA caps ptxas at 128 registers so two CTAs fit an SM (C2 balanced d1000
  // strict: 174 registers at 256 wide, 2.54 -> 1.46 ms per 1e7 points)
  if (d == Domain::F64Strict && s.block < 512) s.block = 512;
  if (t.lanes >= 1 && t.lanes <= 8) s.lanes = t.lanes;
  if (t.block >= 32 && t.block <= 1024) s.block = t.block;
  if (t.sync_every) s.sync_every = t.sync_every;
  if (t.min_ctas) s.min_ctas = t.min_ctas;
  return s;
}

namespace {

std::uint64_t bits_of(double d) {
  std::uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

std::string hex64(std::uint64_t u) {
  char buf[24];
  std::snprintf(buf, sizeof buf, "0x%016llX", static_cast<unsigned long long>(u));
  return buf;
}

using IvCoef = IntervalWord;

// A Hörner-shaped run acc = fma(acc, B, c_j), j = 1..L, with one multiplier
// B and scalar coefficients is emitted as a counted loop over a constant
// array instead of L straight-line FMAs. The arithmetic is the same FMA
// sequence (bit-identical results); the kernel shrinks from ~16 B x L x P
// of code to one cached loop body, which removes the instruction-fetch
// bound of small batches (C1: 1e5 points, 26 us per straight-line launch,
// profiles/r1_launches_c1.csv).
struct ChainRun {
  std::size_t head = 0, last = 0;  // ops head+1..last form the loop
  Operand mult;
};

template <typename C>
std::vector<ChainRun> chain_runs(const Stream<C>& s, Domain d, std::uint32_t sync_every,
                                 std::uint64_t budget, std::uint32_t chain_min) {
  std::vector<ChainRun> runs;
  if (s.strict || sync_every != 0) return runs;
  if (d != Domain::F64 && d != Domain::I64F && d != Domain::I64) return runs;
  const std::size_t min_run = chain_min ? chain_min : 64;
  if (chain_min == UINT32_MAX) return runs;
  // uses of the value each op defines (registers may be redefined)
  const std::size_t n = s.ops.size();
  std::vector<std::uint32_t> uses(n, 0);
  std::unordered_map<std::uint32_t, std::size_t> last_def;
  auto read = [&](const Operand& o) {
    if (!o.is(Operand::Reg)) return;
    auto it = last_def.find(o.id);
    if (it != last_def.end()) ++uses[it->second];
  };
  for (std::size_t i = 0; i < n; ++i) {
    read(s.ops[i].a);
    read(s.ops[i].b);
    read(s.ops[i].c);
    last_def[s.ops[i].dst] = i;
  }
  read(s.result);
  // op j continues the chain of op j-1: acc operand is the previous value
  // (used once), same multiplier, scalar coefficient addend
  auto same = [](const Operand& x, const Operand& y) { return x.kind == y.kind && x.id == y.id; };
  auto link = [&](std::size_t j, Operand* mult) -> bool {
    const Op& p = s.ops[j - 1];
    const Op& o = s.ops[j];
    if (o.kind != OpKind::Fma || !o.c.is(Operand::Coef) || uses[j - 1] != 1) return false;
    Operand m;
    if (o.a.is(Operand::Reg) && o.a.id == p.dst) {
      m = o.b;
    } else if (o.b.is(Operand::Reg) && o.b.id == p.dst) {
      m = o.a;
    } else {
      return false;
    }
    if (!m.is(Operand::Pow) && !(m.is(Operand::Reg) && m.id != p.dst)) return false;
    if (mult->kind != Operand::None && !same(*mult, m)) return false;
    // the multiplier must not be redefined inside the run
    if (m.is(Operand::Reg) && o.dst == m.id) return false;
    *mult = m;
    return true;
  };
  for (std::size_t i = 1; i < n;) {
    Operand mult;
    std::size_t j = i;
    while (j < n && link(j, &mult)) ++j;
    const std::size_t len = j - i;  // ops i..j-1 continue the chain of op i-1
    const std::uint64_t words = len + 24;  // + prefetch padding (up to 3 trips)
    if (len >= min_run && words <= budget) {
      runs.push_back({i - 1, j - 1, mult});
      budget -= words;
    }
    i = len ? j : i + 1;
  }
  return runs;
}

template <typename C>
class Emitter {
 public:
  Emitter(const Stream<C>& s, Domain d, const KernelShape& shape, const Tuning& t,
          std::vector<std::size_t> cuts)
      : s_(s), d_(d), P_(shape.lanes), block_(shape.block), sync_every_(shape.sync_every),
        paired_(d != Domain::Interval && d != Domain::I64K), min_ctas_(shape.min_ctas),
        K_(d == Domain::I64K ? std::max<std::uint32_t>(1, shape.limbs) : 1),
        part_(shape.iv_partition), tuning_(t), cuts_(std::move(cuts)),
        group_tiles_(t.group_tiles ? t.group_tiles : 4) {
    if (K_ > 8) throw std::invalid_argument("at most 8 limbs");
  }

  /// The interval fast path of this program for one point as a function
  /// `name(lo, hi) -> (lo, hi, slow)`, preceded by its constant array under
  /// symbol `sym` (the split kernel's mirrored half lives in the program's
  /// module). Empty when the coefficients do not all fit the constant bank.
  std::string point_module(const std::string& name, std::uint32_t role, const std::string& sym) {
    sym_ = sym;
    assign_words();
    if (!(n_param_ == 0 && n_global_ == 0 && n_smem_ == 0) || !interval_fast_path_ok()) return {};
    const_words_ = n_const_;
    std::ostringstream m;
    m << ".const .align 16 .b64 " << sym_ << "[" << n_const_ << "] = {";
    for (std::uint32_t i = 0; i < n_const_; ++i) {
      if (i) m << (i % 8 == 0 ? ",\n  " : ", ");
      m << hex64(words_[i]);
    }
    m << "};\n\n" << point_function(name, role);
    return m.str();
  }
  std::uint32_t const_words() const { return const_words_; }
  void set_split_funcs(std::string text, std::uint32_t mirror_words) {
    split_funcs_ = std::move(text);
    mirror_words_ = mirror_words;
  }

  KernelImage run() {
    KernelImage img;
    img.domain = d_;
    img.nvars = s_.nvars;
    img.lanes = P_;
    img.block = block_;
    const bool iv = d_ == Domain::Interval;
    const bool i64 = d_ == Domain::I64 || d_ == Domain::I64F || d_ == Domain::I64K;
    img.n_in = iv ? 2 * s_.nvars : s_.nvars;
    img.n_out = iv ? 2 : K_;
    img.limbs = K_;
    img.has_flag = iv || i64;
    img.has_bounds = i64;
    if ((d_ == Domain::F64Strict || d_ == Domain::Interval) && !s_.strict) {
      throw std::logic_error("strict domain needs a strict stream");
    }

    assign_words();
    find_chain_runs();
    img.chain_loops = static_cast<std::uint32_t>(runs_.size());
    img.const_words = n_const_;
    img.param_words.assign(words_.begin() + n_const_, words_.begin() + n_const_ + n_param_);
    img.global_words.assign(words_.begin() + n_const_ + n_param_, words_.end());

    const bool fast = iv && interval_fast_path_ok();
    img.interval_fast_path = fast;
    img.entry = std::string("pe_walk_") + domain_name(d_);

    const bool part = fast && part_ != 0 && s_.nvars == 1;
    img.iv_partition = part ? part_ : 0;
    // one-pass sign split (the program's and the mirrored program's point
    // functions in this module): when both coefficient sets fit the bank
    const bool split = part && part_ == 1 && !split_funcs_.empty() && n_param_ == 0 &&
                       n_global_ == 0 && n_const_ + mirror_words_ <= CoefTiers::kConstCap;
    if (split) img.iv_partition = 3;
    if (part && part_ == 2) {
      // mirrored program: only the negative-coordinate entry
      img.entry += "_neg";
      reset_entry();
      gather_ = 2;
      emit_fast_body();
      gather_ = 0;
      std::ostringstream m;
      m << module_header(img, "interval-fast-path (x < 0, mirrored)");
      m << run_arrays_ << entry_text(img, img.entry, 0, min_ctas_);
      img.ptx = m.str();
      img.fp_ops = fp_ops_;
      img.int_ops = int_ops_;
      img.hash = fnv1a(img.ptx.data(), img.ptx.size());
      return img;
    }

    // main entry
    reset_entry();
    if (fast) {
      // exact fast path; points it cannot prove go to the fixup list
      emit_fast_body();
    } else if (cuts_.size() > 1) {
      emit_grouped(img);
    } else {
      emit_prologue();
      emit_powers();
      emit_walk();
      emit_epilogue();
    }
    img.sections = static_cast<std::uint32_t>(std::max<std::size_t>(1, cuts_.size()));
    const std::string main_entry = entry_text(img, img.entry, 0, min_ctas_);

    // fixup entry: exact replay of the listed points
    std::string fix_entry;
    if (fast) {
      img.fix_entry = img.entry + "_fix";
      const std::uint32_t lanes = P_, sync = sync_every_;
      P_ = 1;
      sync_every_ = 0;  // threads past the list length leave at once
      reset_entry();
      fix_ = true;
      // Persistent when the coefficients are all in the constant bank (a
      // function cannot read kernel parameters): a grid of a few CTAs per SM
      // strides over the list and calls the replay as a non-inlined
      // function per point — inside a loop ptxas would hoist the replay's
      // coefficient loads out and spill them. The list is sized for the
      // whole batch, so one thread per slot would launch n/128 CTAs that
      // mostly exit at once (C5: 0.59 ms of 12.2 per 1e8 intervals).
      const bool persistent = n_param_ == 0;
      img.fix_persistent = persistent;
      if (persistent) {
        emit_fix_function_prologue();
      } else {
        emit_fix_prologue();
      }
      if (tuning_.iv_mid >= 0) {
        // finite-case replay first; the bit-level replay only on %pmid
        decls_ << "  .reg .pred %pmid;\n  .reg .f64 %macc;\n";
        body_ << "  mov.f64 %macc, 0d0000000000000000;\n";
        for (std::uint32_t v = 0; v < s_.nvars; ++v) {
          for (bool hi : {false, true}) {
            body_ << "  fma.rn.f64 %macc, " << xr(v, 0, hi) << ", 0d0000000000000000, %macc;\n";
          }
        }
        medium_ = true;
        emit_powers();
        emit_walk();
        body_ << "  setp.nan.f64 %pmid, %macc, %macc;\n  @%pmid bra $Lexact;\n";
        emit_store();
        body_ << "  bra $Lnextpt;\n$Lexact:\n";
        medium_ = false;
      }
      emit_powers();
      emit_walk();
      emit_store();
      body_ << "$Lnextpt:\n";
      finish_entry();
      fix_ = false;
      // 128-thread CTAs, .minnctapersm 6 (<= 80 registers, no spills for
      // C5): the replay is latency-bound, so occupancy helps (C5 fixup per
      // 1e8: 612 -> 590 us at 6, 584 us at 8 but with spills;
      // profiles/r1_c5_fix_shape.txt).
      img.fix_block = 128;
      img.fix_ctas_per_sm = 6;
      if (persistent) {
        funcs_ += fix_function_text();
        reset_entry();
        emit_fix_loop();
        finish_entry();
      }
      fix_entry = entry_text(img, img.fix_entry, img.fix_block, img.fix_ctas_per_sm);
      P_ = lanes;
      sync_every_ = sync;
    }

    // positive-coordinate entry of the sign-partitioned fast path
    std::string part_entry;
    if (split) {
      const std::string ring2 = std::to_string(2 * split_ring(block_));
      funcs_ += ".shared .align 8 .b64 pe_sp_lo[" + ring2 + "];\n.shared .align 8 .b64 pe_sp_hi[" + ring2 +
                "];\n.shared .align 4 .b32 pe_sp_idx[" + ring2 + "];\n.shared .align 4 .b32 pe_sp_w[8];\n\n";
      funcs_ += split_funcs_ + point_function("pe_iv_pos", 1);
      img.part_entry = img.entry + "_split";
      reset_entry();
      emit_split_entry();
      finish_entry();
      // 1024 threads per SM (<= 64 registers) in CTAs of `block`
      part_entry = entry_text(img, img.part_entry, 0, 1024 / block_);
    } else if (part) {
      img.part_entry = img.entry + "_pos";
      reset_entry();
      gather_ = 1;
      emit_fast_body();
      gather_ = 0;
      part_entry = entry_text(img, img.part_entry, 0, min_ctas_);
    }

    std::ostringstream m;
    m << module_header(img, fast ? "interval-fast-path+fixup" : "");
    m << run_arrays_ << funcs_ << main_entry << fix_entry << part_entry;
    img.ptx = m.str();
    img.fp_ops = fp_ops_;
    img.int_ops = int_ops_;
    img.hash = fnv1a(img.ptx.data(), img.ptx.size());
    return img;
  }

 private:
  // ---------------- entries ----------------
  std::string module_header(const KernelImage& img, const char* note) const {
    std::ostringstream m;
    m << "//\n// polyeval-b200 generated kernel: domain=" << domain_name(d_)
      << " nvars=" << s_.nvars << " ops=" << s_.ops.size() << " powers=" << s_.powers.size()
      << " lanes=" << P_ << (*note ? " " : "") << note << "\n//\n";
    m << ".version 8.7\n.target sm_100a\n.address_size 64\n\n";
    if (n_smem_ > 0) {
      m << ".shared .align 16 .b64 pe_scoef[" << n_smem_ << "];\n"
        << ".shared .align 8 .b64 pe_mbar;\n\n";
    }
    if (n_const_ > 0) {
      m << ".const .align 16 .b64 " << sym_ << "[" << n_const_ << "] = {";
      for (std::uint32_t i = 0; i < n_const_; ++i) {
        if (i) m << (i % 8 == 0 ? ",\n  " : ", ");
        m << hex64(words_[i]);
      }
      m << "};\n\n";
    }
    (void)img;
    return m.str();
  }

  // Interval fast path entry body (main entry, or a partitioned entry when
  // gather_ != 0): prologue, power DAG, walk, exit to the fixup list / store.
  void emit_fast_body() {
    emit_prologue();
    decls_ << "  .reg .b64 %facc;\n  .reg .pred %pslow;\n  .reg .pred %pb<4>;\n";
    body_ << "  mov.b64 %facc, 0;\n";
    for (int i = 0; i < 4; ++i) body_ << "  setp.ne.b32 %pb" << i << ", %r3, %r3;\n";
    fast_ = true;
    emit_powers();
    emit_walk();
    emit_fast_exit();
    fast_ = false;
    finish_entry();
  }

  void reset_entry() {
    body_.str("");
    body_.clear();
    decls_.str("");
    decls_.clear();
    n_creg_ = n_tf_ = n_tu_ = n_tp_ = n_tr_ = 0;
    loop_decls_ = false;
    pending_.clear();
  }

  void finish_entry() {
    body_ << "$Ldone:\n  ret;\n";
    if (n_creg_ > 0) decls_ << "  .reg ." << ldty() << " %c<" << n_creg_ << ">;\n";
    if (n_tf_ > 0) decls_ << "  .reg .f64 %tf<" << n_tf_ << ">;\n";
    if (n_tu_ > 0) decls_ << "  .reg .b64 %tu<" << n_tu_ << ">;\n";
    if (n_tp_ > 0) decls_ << "  .reg .pred %tp<" << n_tp_ << ">;\n";
    if (n_tr_ > 0) decls_ << "  .reg .b32 %tr<" << n_tr_ << ">;\n";
  }

  // Both entries of a module take the same parameter list, so one argument
  // array launches either.
  std::string entry_text(const KernelImage& img, const std::string& name,
                         std::uint32_t maxntid = 0, std::uint32_t min_ctas = 0) const {
    if (maxntid == 0) maxntid = img.block;
    std::ostringstream m;
    m << ".visible .entry " << name << "(";
    bool first = true;
    auto param = [&](const std::string& decl) {
      m << (first ? "\n  " : ",\n  ") << decl;
      first = false;
    };
    for (std::uint32_t i = 0; i < img.n_in; ++i) param(".param .u64 pe_in" + std::to_string(i));
    for (std::uint32_t i = 0; i < img.n_out; ++i) param(".param .u64 pe_out" + std::to_string(i));
    param(".param .u64 pe_n");
    param(".param .u64 pe_gcoef");
    if (img.has_flag) param(".param .u64 pe_flag");
    if (img.has_bounds) {
      for (std::uint32_t v = 0; v < s_.nvars; ++v) param(".param .u64 pe_bound" + std::to_string(v));
    }
    if (img.interval_fast_path) {
      param(".param .u64 pe_list");
      param(".param .u64 pe_count");
      param(".param .u64 pe_cap");
    }
    if (img.iv_partition) {
      param(".param .u64 pe_pidx");
      param(".param .u64 pe_pcnt");
    }
    if (cuts_.size() > 1) param(".param .u64 pe_scratch");
    if (n_param_ > 0) param(".param .align 16 .b8 pe_pcoef[" + std::to_string(8 * n_param_) + "]");
    m << ")\n.maxntid " << maxntid << ", 1, 1\n";
    if (min_ctas) m << ".minnctapersm " << min_ctas << "\n";
    m << "{\n";
    m << "  .reg .pred %p<8>;\n  .reg .b32 %r<8>;\n  .reg .b64 %rd<24>;\n";
    m << decls_.str() << body_.str() << "}\n\n";
    return m.str();
  }

  // ---------------- coefficient words ----------------
  void assign_words() {
    coef_lo_.resize(s_.coefs.size());
    coef_hi_.resize(s_.coefs.size());
    std::unordered_map<std::uint64_t, std::uint32_t> dedup;
    auto word = [&](std::uint64_t w) {
      auto it = dedup.find(w);
      if (it != dedup.end()) return it->second;
      const auto idx = static_cast<std::uint32_t>(words_.size());
      words_.push_back(w);
      dedup.emplace(w, idx);
      return idx;
    };
    // Scalar domains: an FMA can take one uniform-register operand, so the
    // second coefficient of a two-coefficient op (fma(c, x^d, c'), the leaves
    // of every scheme) is register-bound. Uniform-bound words go to the
    // constant bank first, deduplicated, in first-use order (they arrive two
    // per 16-byte LDCU, load_word); the register-bound words follow as a
    // second region in first-use order (paired loads: ptxas turns those into
    // per-thread 16-byte LDCs, one issue slot per two coefficients).
    reg_bound_.assign(s_.coefs.size(), 0);
    const bool split = paired_;
    if (split) {
      for (const Op& op : s_.ops) {
        const int nc = op.a.is(Operand::Coef) + op.b.is(Operand::Coef) + op.c.is(Operand::Coef);
        if (nc < 2) continue;
        const Operand& r = op.c.is(Operand::Coef) ? op.c : op.b;  // keep one uniform operand
        reg_bound_[r.id] = 1;
      }
    }
    // Sectioned kernels place the words section by section (each section's
    // uniform-bound words, then its register-bound words): the constant
    // working set of a section is one contiguous block.
    std::vector<std::uint32_t> sec_of(s_.coefs.size(), 0);
    std::uint32_t nsec = 1;
    if (cuts_.size() > 1 && tuning_.word_layout >= 0) {
      nsec = static_cast<std::uint32_t>(cuts_.size());
      std::vector<char> seen(s_.coefs.size(), 0);
      std::uint32_t sec = 0;
      for (std::size_t i = 0; i < s_.ops.size(); ++i) {
        while (sec + 1 < cuts_.size() && i >= cuts_[sec]) ++sec;
        for (const Operand* o : {&s_.ops[i].a, &s_.ops[i].b, &s_.ops[i].c}) {
          if (o->is(Operand::Coef) && !seen[o->id]) {
            seen[o->id] = 1;
            sec_of[o->id] = sec;
          }
        }
      }
      if (s_.result.is(Operand::Coef) && !seen[s_.result.id]) sec_of[s_.result.id] = nsec - 1;
    }
    for (std::uint32_t sec = 0; sec < nsec; ++sec) {
    for (std::size_t k = 0; k < s_.coefs.size(); ++k) {
      if (sec_of[k] != sec) continue;
      if (split && reg_bound_[k]) continue;  // second region, below
      if (d_ == Domain::Interval) {
        const IvCoef c = ivcoef(k);
        coef_lo_[k] = word(bits_of(c.lo));
        coef_hi_[k] = word(bits_of(c.hi));
      } else if (d_ == Domain::I64 || d_ == Domain::I64F || d_ == Domain::I64K) {
        std::uint64_t w;
        if constexpr (std::is_same_v<C, std::int64_t>) {
          // I64F: |c| <= M < 2^53 by the host proof, so the double is exact
          w = d_ != Domain::I64F ? static_cast<std::uint64_t>(s_.coefs[k])
                                 : bits_of(static_cast<double>(s_.coefs[k]));
        } else {
          throw std::invalid_argument("int64 domain needs integer coefficients");
        }
        coef_lo_[k] = coef_hi_[k] = word(w);
      } else {
        const double c = static_cast<double>(s_.coefs[k]);
        coef_lo_[k] = coef_hi_[k] = word(bits_of(c));
      }
    }
    }
    if (words_.size() & 1) words_.push_back(0);  // region starts on a pair
    const auto region1 = static_cast<std::uint32_t>(words_.size());
    if (split) {
      for (std::uint32_t sec = 0; sec < nsec; ++sec) {
        for (std::size_t k = 0; k < s_.coefs.size(); ++k) {
          if (!reg_bound_[k] || sec_of[k] != sec) continue;
          coef_lo_[k] = coef_hi_[k] = static_cast<std::uint32_t>(words_.size());
          words_.push_back(scalar_word(k));
        }
        if (words_.size() & 1) words_.push_back(0);  // next section starts on a pair
      }
    }
    const auto n = static_cast<std::uint32_t>(words_.size());
    if (cuts_.size() > 1) {
      // Sectioned kernels: the section functions cannot read kernel
      // parameters. The uniform-bound words take the constant bank; the
      // register-bound ones (per-thread loads in any case) and any overflow
      // go to shared memory, filled once per CTA of the persistent kernel
      // (a global-memory tier here measured 30 % slower on C4: every word an
      // L1 round trip); beyond that, global memory.
      n_const_ = std::min(region1, CoefTiers::kConstCap);
      n_param_ = 0;
      n_smem_ = std::min(n - n_const_, CoefTiers::kSmemCap);
    } else {
      n_const_ = std::min(n, CoefTiers::kConstCap);
      n_param_ = std::min(n - n_const_, CoefTiers::kParamCap);
      n_smem_ = 0;
    }
    n_global_ = n - n_const_ - n_param_ - n_smem_;
  }

  // 64-bit word of scalar coefficient k as the kernel consumes it: the raw
  // integer for the int64 / K-limb kernels, otherwise the double (exact for
  // I64F by the host proof; RN for an integer polynomial evaluated in fp64)
  std::uint64_t scalar_word(std::size_t k) const {
    if constexpr (std::is_same_v<C, std::int64_t>) {
      if (d_ == Domain::I64 || d_ == Domain::I64K) return static_cast<std::uint64_t>(s_.coefs[k]);
    }
    return bits_of(static_cast<double>(s_.coefs[k]));
  }

  // Interval value of coefficient k: injection, then the folded zero-add
  // steps (std::nextafter outward, as interval_add would apply them).
  IvCoef ivcoef(std::size_t k) const { return interval_coefficient(s_, k); }

  // coefficient words / arithmetic registers
  // The fast interval path needs finite, nonzero, non-straddling coefficient
  // intervals (checked here once) and a walk that ends in a register.
  bool interval_fast_path_ok() const {
    if (tuning_.iv_fast < 0) return false;
    if (!s_.result.is(Operand::Reg)) return false;
    for (std::size_t k = 0; k < s_.coefs.size(); ++k) {
      const IvCoef c = ivcoef(k);
      if (!std::isfinite(c.lo) || !std::isfinite(c.hi) || c.lo == 0.0 || c.hi == 0.0) return false;
      if ((c.lo < 0) != (c.hi < 0)) return false;
    }
    return true;
  }

  bool intk() const { return d_ == Domain::I64 || d_ == Domain::I64K; }
  const char* ldty() const { return intk() ? "b64" : "f64"; }
  const char* rty() const { return intk() ? "s64" : "f64"; }
  // coordinates and results in memory
  bool int_io() const { return d_ == Domain::I64 || d_ == Domain::I64F || d_ == Domain::I64K; }
  const char* ioty() const { return int_io() ? "b64" : "f64"; }
  static std::string ln(std::uint32_t lane) { return "_" + std::to_string(lane); }

  // Loads coefficient word w into a fresh register (shared by all lanes).
  std::string load_word(std::uint32_t w) {
    if (paired_) {
      // paired uniform loads: words sit in first-use order, so an even word
      // and its odd neighbour arrive in one 16-byte LDCU (half the
      // coefficient-delivery issue slots of one LDCU per word)
      auto it = pending_.find(w);
      if (it != pending_.end()) {
        std::string r = it->second;
        pending_.erase(it);
        return r;
      }
      const bool pair_const = w < n_const_ && (w & 1) == 0 && w + 1 < n_const_;
      const bool pair_param = w >= n_const_ && w < n_const_ + n_param_ && ((w - n_const_) & 1) == 0 &&
                              w + 1 < n_const_ + n_param_;
      const bool pair_smem = w >= n_const_ && w < n_const_ + n_smem_ && ((w - n_const_) & 1) == 0 &&
                             w + 1 < n_const_ + n_smem_;
      if (pair_const || pair_param || pair_smem) {
        std::string r = "%c" + std::to_string(n_creg_++);
        std::string r2 = "%c" + std::to_string(n_creg_++);
        if (pair_const) {
          body_ << "  ld.const.v2." << ldty() << " {" << r << ", " << r2 << "}, [" << cbase() << "+"
                << 8 * w << "];\n";
        } else if (pair_smem) {
          body_ << "  ld.shared.v2." << ldty() << " {" << r << ", " << r2 << "}, [pe_scoef+"
                << 8 * (w - n_const_) << "];\n";
        } else {
          body_ << "  ld.param.v2." << ldty() << " {" << r << ", " << r2 << "}, [pe_pcoef+"
                << 8 * (w - n_const_) << "];\n";
        }
        pending_[w + 1] = r2;
        return r;
      }
    }
    std::string r = "%c" + std::to_string(n_creg_++);
    if (w < n_const_) {
      body_ << "  ld.const." << ldty() << " " << r << ", [" << cbase() << "+" << 8 * w << "];\n";
    } else if (w < n_const_ + n_param_) {
      body_ << "  ld.param." << ldty() << " " << r << ", [pe_pcoef+" << 8 * (w - n_const_) << "];\n";
    } else if (w < n_const_ + n_smem_) {
      body_ << "  ld.shared." << ldty() << " " << r << ", [pe_scoef+" << 8 * (w - n_const_) << "];\n";
    } else {
      body_ << "  ld.global.nc." << ldty() << " " << r << ", [%rd20+"
            << 8 * (w - n_const_ - n_param_) << "];\n";  // (smem words lead the global array)
    }
    return r;
  }

  // ---------------- operands ----------------
  std::string reg(std::uint32_t id, std::uint32_t lane, bool hi = false) const {
    if (d_ == Domain::Interval) {
      return std::string(fast_ ? "%f" : medium_ ? "%m" : "%") + (hi ? "vh" : "vl") + std::to_string(id) + ln(lane);
    }
    return "%v" + std::to_string(id) + ln(lane);
  }
  // section suffix of per-section power / coordinate copies (sections
  // after the first reload the coordinates and rebuild the powers they use)
  std::string sx() const { return sec_ ? "s" + std::to_string(sec_) : ""; }
  std::string pw(std::uint32_t id, std::uint32_t lane, bool hi = false) const {
    if (d_ == Domain::Interval) {
      return std::string(fast_ ? "%f" : medium_ ? "%m" : "%") + (hi ? "ph" : "pl") + std::to_string(id) + ln(lane);
    }
    return "%q" + std::to_string(id) + sx() + ln(lane);
  }
  std::string xr(std::uint32_t v, std::uint32_t lane, bool hi = false) const {
    if (d_ == Domain::Interval) return (hi ? "%xh" : "%xl") + std::to_string(v) + ln(lane);
    return "%x" + std::to_string(v) + sx() + ln(lane);
  }
  // integer coordinate as loaded (I64: the arithmetic register itself)
  std::string xi(std::uint32_t v, std::uint32_t lane) const {
    if (d_ == Domain::I64F || d_ == Domain::I64K) return "%xi" + std::to_string(v) + sx() + ln(lane);
    return xr(v, lane);
  }
  // I64K: limb j of a K-limb register name
  static std::string lb(const std::string& r, std::uint32_t j) { return r + "_l" + std::to_string(j); }

  // Coefficients are loaded once per op (before the lane loop) and shared.
  struct Loaded {
    std::string lo, hi;
  };
  Loaded load(const Operand& o) {
    if (!o.is(Operand::Coef)) return {};
    const std::string lo = load_word(coef_lo_[o.id]);
    const std::string hi = coef_hi_[o.id] == coef_lo_[o.id] ? lo : load_word(coef_hi_[o.id]);
    return {lo, hi};
  }
  std::string opnd(const Operand& o, const Loaded& l, std::uint32_t lane) const {
    switch (o.kind) {
      case Operand::Reg: return reg(o.id, lane);
      case Operand::Pow: return pw(o.id, lane);
      case Operand::Coef: return l.lo;
      case Operand::Zero: return d_ == Domain::I64 ? "0" : "0d0000000000000000";
      default: throw std::logic_error("bad operand");
    }
  }
  std::pair<std::string, std::string> ivop(const Operand& o, const Loaded& l,
                                           std::uint32_t lane) const {
    switch (o.kind) {
      case Operand::Reg: return {reg(o.id, lane, false), reg(o.id, lane, true)};
      case Operand::Pow: return {pw(o.id, lane, false), pw(o.id, lane, true)};
      case Operand::Coef: return {l.lo, l.hi};
      case Operand::Zero: return {"0d0000000000000000", "0d0000000000000000"};
      default: throw std::logic_error("bad operand");
    }
  }

  // ---------------- frame ----------------
  void emit_prologue() {
    const bool iv = d_ == Domain::Interval;
    // tile base = ctaid * (ntid * P) + tid; lane k at base + k * ntid
    body_ << "  mov.u32 %r1, %ctaid.x;\n  mov.u32 %r2, %ntid.x;\n  mov.u32 %r3, %tid.x;\n"
          << "  mul.wide.u32 %rd1, %r1, %r2;\n  mul.lo.u64 %rd1, %rd1, " << P_ << ";\n"
          << "  cvt.u64.u32 %rd2, %r3;\n  add.u64 %rd1, %rd1, %rd2;\n"
          << "  ld.param.u64 %rd3, [pe_n];\n";
    if (gather_) {
      // thread j of the grid takes list slot j; %rd3 becomes the list length
      // (device counter), %rd19 keeps n; a CTA past the end leaves as a whole
      body_ << "  mov.u64 %rd19, %rd3;\n  ld.param.u64 %rd22, [pe_pcnt];\n"
            << "  cvta.to.global.u64 %rd22, %rd22;\n  ld.global.u32 %r4, [%rd22+"
            << (gather_ == 2 ? 4 : 0) << "];\n  cvt.u64.u32 %rd3, %r4;\n"
            << "  mul.wide.u32 %rd22, %r1, %r2;\n  mul.lo.u64 %rd22, %rd22, " << P_ << ";\n"
            << "  setp.ge.u64 %p1, %rd22, %rd3;\n  @%p1 bra $Ldone;\n"
            << "  ld.param.u64 %rd21, [pe_pidx];\n  cvta.to.global.u64 %rd21, %rd21;\n";
    }
    emit_chain_warmup();
    if (sync_every_ == 0 && cuts_.size() <= 1) {
      // no CTA barriers: threads past the end leave immediately; with
      // barriers every thread stays (clamped loads, predicated stores)
      body_ << "  setp.ge.u64 %p1, %rd1, %rd3;\n  @%p1 bra $Ldone;\n";
    }
    body_ << "  sub.u64 %rd12, %rd3, 1;\n";  // last valid index (loads clamp to it)
    if (n_global_ > 0) {
      body_ << "  ld.param.u64 %rd20, [pe_gcoef];\n  cvta.to.global.u64 %rd20, %rd20;\n";
    }
    decls_ << "  .reg .b64 %ix<" << P_ << ">;\n  .reg .pred %pv<" << P_ << ">;\n";
    for (std::uint32_t k = 0; k < P_; ++k) {
      body_ << "  cvt.u64.u32 %rd13, %r2;\n  mul.lo.u64 %rd13, %rd13, " << k << ";\n"
            << "  add.u64 %rd13, %rd1, %rd13;\n  setp.lt.u64 %pv" << k << ", %rd13, %rd3;\n"
            << "  min.u64 %rd13, %rd13, %rd12;\n";
      if (gather_) {
        // list slot -> point index (front of the list, or back for x < 0)
        if (gather_ == 2) body_ << "  sub.u64 %rd13, %rd19, %rd13;\n  sub.u64 %rd13, %rd13, 1;\n";
        body_ << "  shl.b64 %rd22, %rd13, 2;\n  add.u64 %rd22, %rd21, %rd22;\n"
              << "  ld.global.u32 %r5, [%rd22];\n  cvt.u64.u32 %rd13, %r5;\n";
      }
      body_ << "  shl.b64 %ix" << k << ", %rd13, 3;\n";
    }
    for (std::uint32_t v = 0; v < s_.nvars; ++v) {
      for (std::uint32_t k = 0; k < P_; ++k) {
        if (iv) {
          decls_ << "  .reg .f64 " << xr(v, k, false) << ", " << xr(v, k, true) << ";\n";
        } else if (d_ == Domain::I64F) {
          decls_ << "  .reg .f64 " << xr(v, k) << ";\n  .reg .b64 " << xi(v, k) << ";\n";
        } else if (d_ == Domain::I64K) {
          decls_ << "  .reg .b64 " << xi(v, k) << ";\n";
          for (std::uint32_t j = 0; j < K_; ++j) decls_ << "  .reg .b64 " << lb(xr(v, k), j) << ";\n";
        } else {
          decls_ << "  .reg ." << ldty() << " " << xr(v, k) << ";\n";
        }
      }
    }
    const std::uint32_t nin = iv ? 2 * s_.nvars : s_.nvars;
    for (std::uint32_t i = 0; i < nin; ++i) {
      body_ << "  ld.param.u64 %rd5, [pe_in" << i << "];\n  cvta.to.global.u64 %rd5, %rd5;\n";
      for (std::uint32_t k = 0; k < P_; ++k) {
        const std::string dst = iv ? xr(i / 2, k, i % 2 == 1) : int_io() ? xi(i, k) : xr(i, k);
        body_ << "  add.u64 %rd6, %rd5, %ix" << k << ";\n  ld.global.nc." << ioty() << " " << dst
              << ", [%rd6];\n";
        if (d_ == Domain::I64F) {
          // exact: |x| <= bound < 2^53 is checked below before any result is used
          body_ << "  cvt.rn.f64.s64 " << xr(i, k) << ", " << xi(i, k) << ";\n";
        } else if (d_ == Domain::I64K) {  // sign-extend to K limbs
          body_ << "  mov.b64 " << lb(xr(i, k), 0) << ", " << xi(i, k) << ";\n";
          for (std::uint32_t j = 1; j < K_; ++j) {
            body_ << "  shr.s64 " << lb(xr(i, k), j) << ", " << xi(i, k) << ", 63;\n";
          }
        }
      }
    }
    if (iv && gather_ == 2) {
      // mirrored program: evaluate q at -x = [-hi, -lo]
      for (std::uint32_t v = 0; v < s_.nvars; ++v) {
        for (std::uint32_t k = 0; k < P_; ++k) {
          const std::string t = tmp_f();
          body_ << "  neg.f64 " << t << ", " << xr(v, k, true) << ";\n"
                << "  neg.f64 " << xr(v, k, true) << ", " << xr(v, k, false) << ";\n"
                << "  mov.f64 " << xr(v, k, false) << ", " << t << ";\n";
        }
      }
    }
    int label = 0;
    if (iv) {
      // Reference Interval(lo, hi) rejects NaN endpoints and lo > hi
      // (interval.cpp:21-26): flag and continue, the host reports EINVAL.
      for (std::uint32_t v = 0; v < s_.nvars; ++v) {
        for (std::uint32_t k = 0; k < P_; ++k, ++label) {
          body_ << "  setp.le.f64 %p2, " << xr(v, k, false) << ", " << xr(v, k, true) << ";\n"
                << "  @%p2 bra $Lok" << label << ";\n"
                << "  ld.param.u64 %rd7, [pe_flag];\n  cvta.to.global.u64 %rd7, %rd7;\n"
                << "  @%pv" << k << " st.global.u32 [%rd7], 2;\n$Lok" << label << ":\n";
        }
      }
    }
    if (int_io()) {
      // |x_v| <= bound_v, the range the host overflow proof assumed
      for (std::uint32_t v = 0; v < s_.nvars; ++v) {
        body_ << "  ld.param.u64 %rd8, [pe_bound" << v << "];\n";
        for (std::uint32_t k = 0; k < P_; ++k, ++label) {
          body_ << "  abs.s64 %rd9, " << xi(v, k) << ";\n"
                << "  setp.gt.u64 %p2, %rd9, %rd8;\n"
                << "  @!%p2 bra $Lbok" << label << ";\n"
                << "  ld.param.u64 %rd7, [pe_flag];\n  cvta.to.global.u64 %rd7, %rd7;\n"
                << "  @%pv" << k << " st.global.u32 [%rd7], 1;\n$Lbok" << label << ":\n";
        }
      }
    }
  }

  void emit_powers(const std::vector<char>* only = nullptr) {
    const std::size_t np = s_.powers.size();
    for (std::size_t i = 0; i < np; ++i) {
      const auto id = static_cast<std::uint32_t>(i);
      if (only && !(*only)[i]) continue;
      for (std::uint32_t k = 0; k < P_; ++k) {
        if (d_ == Domain::Interval) {
          decls_ << "  .reg .f64 " << pw(id, k, false) << ", " << pw(id, k, true) << ";\n";
        } else if (d_ == Domain::I64K) {
          for (std::uint32_t j = 0; j < K_; ++j) decls_ << "  .reg .b64 " << lb(pw(id, k), j) << ";\n";
        } else {
          decls_ << "  .reg ." << rty() << " " << pw(id, k) << ";\n";
        }
      }
    }
    psign_.assign(np, 0);
    for (std::size_t i = 0; i < np; ++i) {
      const Power& p = s_.powers[i];
      const auto id = static_cast<std::uint32_t>(i);
      if (only && !(*only)[i]) continue;
      for (std::uint32_t k = 0; k < P_; ++k) {
        if (p.exponent == 1) {
          if (d_ == Domain::Interval) {
            body_ << "  mov.f64 " << pw(id, k, false) << ", " << xr(p.var, k, false) << ";\n"
                  << "  mov.f64 " << pw(id, k, true) << ", " << xr(p.var, k, true) << ";\n";
            if (fast_) {
              // partitioned entries: the classifier guarantees 0 < lo
              if (!gather_) fcheck_straddle({pw(id, k, false), pw(id, k, true)});
              fcheck_finite(pw(id, k, false));
              fcheck_finite(pw(id, k, true));
            }
          } else if (d_ == Domain::I64K) {
            for (std::uint32_t j = 0; j < K_; ++j) {
              body_ << "  mov.b64 " << lb(pw(id, k), j) << ", " << lb(xr(p.var, k), j) << ";\n";
            }
          } else {
            body_ << "  mov." << ldty() << " " << pw(id, k) << ", " << xr(p.var, k) << ";\n";
          }
          continue;
        }
        if (d_ == Domain::Interval && fast_) {
          // A product of non-straddling intervals does not straddle — unless
          // it underflows: RN gives a zero endpoint and the outward step takes
          // it across. With both factor signs known the step is the integer
          // one, which turns a zero into a NaN (caught below); with an
          // unknown factor sign it is the directed add (fnext), which moves
          // a zero to -/+dmin like std::nextafter does, so the power must be
          // checked before anything trusts its sign (squares are "positive",
          // other powers take their sign from the upper endpoint): a power
          // that straddles sends the point to the exact replay.
          fast_mul(pw(id, k, false), pw(id, k, true), {pw(p.lo, k, false), pw(p.lo, k, true)},
                   {pw(p.hi, k, false), pw(p.hi, k, true)}, false, false, psign_[p.lo],
                   psign_[p.hi]);
          if (psign_[p.lo] * psign_[p.hi] == 0) fcheck_straddle({pw(id, k, false), pw(id, k, true)});
          fcheck_finite(pw(id, k, false));
          fcheck_finite(pw(id, k, true));
        } else if (d_ == Domain::Interval && medium_) {
          mid_mul(pw(id, k, false), pw(id, k, true), {pw(p.lo, k, false), pw(p.lo, k, true)},
                  {pw(p.hi, k, false), pw(p.hi, k, true)});
        } else if (d_ == Domain::Interval) {
          iv_mul(pw(id, k, false), pw(id, k, true), {pw(p.lo, k, false), pw(p.lo, k, true)},
                 {pw(p.hi, k, false), pw(p.hi, k, true)}, k == 0);
        } else if (d_ == Domain::I64K) {
          kmul(limbs_of(pw(id, k)), limbs_of(pw(p.lo, k)), limbs_of(pw(p.hi, k)));
          if (k == 0) ++int_ops_;
        } else if (d_ == Domain::I64) {
          body_ << "  mul.lo.s64 " << pw(id, k) << ", " << pw(p.lo, k) << ", " << pw(p.hi, k) << ";\n";
          if (k == 0) ++int_ops_;
        } else {
          body_ << "  mul.rn.f64 " << pw(id, k) << ", " << pw(p.lo, k) << ", " << pw(p.hi, k) << ";\n";
          if (k == 0) ++fp_ops_;
        }
      }
      // static sign: squares are positive, products of known signs known
      if (p.exponent > 1) {
        psign_[i] = p.lo == p.hi ? 1 : psign_[p.lo] * psign_[p.hi];
      }
      if (p.exponent == 1 && fast_ && gather_) psign_[i] = 1;  // 0 < x (classifier)
    }
  }

  void emit_walk() {
    declare_walk_regs();
    emit_ops(0, s_.ops.size());
  }

  // Sectioned walk (scalar domains, long streams). A straight-line walk of
  // 10k+ ops is larger than the SM's instruction and constant caches: if
  // every CTA ran the whole walk, each CTA would stream all of its code and
  // coefficients from the GPC caches again (C4: 78 % instruction-cache and
  // 85 % constant-cache hits, vs 99.5 % / 96 % for walks of ~3k ops). So the
  // op sequence is cut into sections where few walk values are live
  // (emit_ptx), and the kernel is persistent over groups of T tiles: a CTA
  // runs section 0 on T tiles, then section 1 on the same T tiles, ...;
  // each section's code and constants stay hot for T tiles. Each section is
  // a non-inlined .func called once per tile (inside a loop ptxas would hoist
  // the section's thousands of constant loads into registers), values live
  // across a cut go to a per-CTA scratch slot (L2-resident: grid x T x live x
  // tile words), coordinates are reloaded per tile (L2 hits after the first
  // section), each section rebuilds the powers it reads. The arithmetic is
  // the unsectioned op sequence, unchanged: results are bit-identical.
  void emit_grouped(KernelImage& img) {
    const std::uint32_t T = group_tiles_;
    const auto live = live_at_cuts();
    std::size_t L = 1;
    for (const auto& l : live) L = std::max(L, l.size());
    img.group_tiles = T;
    img.scratch_values = static_cast<std::uint32_t>(L);
    // the sections, one function each (kernel parameter names re-declared as
    // function parameters, so the frame helpers read them unchanged)
    std::vector<std::string> fparams;
    for (std::uint32_t i = 0; i < img.n_in; ++i) fparams.push_back("pe_in" + std::to_string(i));
    for (std::uint32_t i = 0; i < img.n_out; ++i) fparams.push_back("pe_out" + std::to_string(i));
    fparams.push_back("pe_n");
    fparams.push_back("pe_gcoef");
    if (img.has_flag) fparams.push_back("pe_flag");
    if (img.has_bounds) {
      for (std::uint32_t v = 0; v < s_.nvars; ++v) fparams.push_back("pe_bound" + std::to_string(v));
    }
    fparams.push_back("pe_tbase");  // first point index of the tile
    fparams.push_back("pe_slot");   // scratch slot of the tile
    std::size_t begin = 0;
    for (std::size_t k = 0; k < cuts_.size(); ++k) {
      const std::size_t end = cuts_[k];
      sec_ = static_cast<std::uint32_t>(k);
      reset_entry();
      decls_ << "  .reg .b64 %ix<" << P_ << ">;\n  .reg .pred %pv<" << P_ << ">;\n  .reg .b64 %gsl, %ga;\n";
      body_ << "  mov.u32 %r2, %ntid.x;\n  mov.u32 %r3, %tid.x;\n"
            << "  ld.param.u64 %rd3, [pe_n];\n  sub.u64 %rd12, %rd3, 1;\n"
            << "  ld.param.u64 %rd1, [pe_tbase];\n  cvt.u64.u32 %rd2, %r3;\n  add.u64 %rd1, %rd1, %rd2;\n"
            << "  ld.param.u64 %gsl, [pe_slot];\n  shl.b64 %rd14, %rd2, 3;\n  add.u64 %gsl, %gsl, %rd14;\n";
      if (n_smem_ + n_global_ > 0) {
        body_ << "  ld.param.u64 %rd20, [pe_gcoef];\n  cvta.to.global.u64 %rd20, %rd20;\n";
      }
      for (std::uint32_t q = 0; q < P_; ++q) {
        body_ << "  mul.wide.u32 %rd13, %r2, " << q << ";\n  add.u64 %rd13, %rd1, %rd13;\n"
              << "  setp.lt.u64 %pv" << q << ", %rd13, %rd3;\n  min.u64 %rd13, %rd13, %rd12;\n"
              << "  shl.b64 %ix" << q << ", %rd13, 3;\n";
      }
      emit_tile_coords(k == 0);
      // value j of lane q: %gsl + (j * ntid * P + q * ntid) * 8
      auto slot = [&](std::size_t j, std::uint32_t q) {
        body_ << "  mul.wide.u32 %ga, %r2, " << (j * P_ + q) * 8 << ";\n  add.u64 %ga, %ga, %gsl;\n";
      };
      declare_walk_regs();
      if (k > 0) {
        for (std::size_t j = 0; j < live[k - 1].size(); ++j) {
          for (std::uint32_t q = 0; q < P_; ++q) {
            slot(j, q);
            body_ << "  ld.global." << ldty() << " " << reg(live[k - 1][j], q) << ", [%ga];\n";
          }
        }
      }
      std::vector<char> need = powers_used(begin, end, k + 1 == cuts_.size());
      emit_powers(&need);
      emit_ops(begin, end);
      if (k + 1 < cuts_.size()) {
        for (std::size_t j = 0; j < live[k].size(); ++j) {
          for (std::uint32_t q = 0; q < P_; ++q) {
            slot(j, q);
            body_ << "  st.global." << ldty() << " [%ga], " << reg(live[k][j], q) << ";\n";
          }
        }
      } else {
        emit_store();
      }
      body_ << "  ret;\n";
      if (n_creg_ > 0) decls_ << "  .reg ." << ldty() << " %c<" << n_creg_ << ">;\n";
      if (n_tf_ > 0) decls_ << "  .reg .f64 %tf<" << n_tf_ << ">;\n";
      if (n_tu_ > 0) decls_ << "  .reg .b64 %tu<" << n_tu_ << ">;\n";
      if (n_tp_ > 0) decls_ << "  .reg .pred %tp<" << n_tp_ << ">;\n";
      if (n_tr_ > 0) decls_ << "  .reg .b32 %tr<" << n_tr_ << ">;\n";
      std::ostringstream f;
      f << ".func pe_section" << k << "(";
      for (std::size_t i = 0; i < fparams.size(); ++i) {
        f << (i ? ",\n  " : "\n  ") << ".param .u64 " << fparams[i];
      }
      f << ")\n{\n  .reg .pred %p<8>;\n  .reg .b32 %r<8>;\n  .reg .b64 %rd<24>;\n"
        << decls_.str() << body_.str() << "}\n\n";
      funcs_ += f.str();
      begin = end;
    }
    sec_ = 0;
    // the persistent kernel: groups of T tiles, each section over the group
    reset_entry();
    decls_ << "  .reg .b64 %gs, %gtl, %gn, %gb, %gstep, %gt, %gtile, %gsl, %gbase;\n"
           << "  .reg .pred %gp;\n  .reg .b64 %ka<" << fparams.size() << ">;\n";
    body_ << "  mov.u32 %r1, %ctaid.x;\n  mov.u32 %r2, %ntid.x;\n"
          << "  ld.param.u64 %rd3, [pe_n];\n"
          << "  ld.param.u64 %gs, [pe_scratch];\n  cvta.to.global.u64 %gs, %gs;\n"
          << "  mul.wide.u32 %gtl, %r2, " << P_ << ";\n"                       // tile = ntid * P
          << "  add.u64 %gn, %rd3, %gtl;\n  sub.u64 %gn, %gn, 1;\n  div.u64 %gn, %gn, %gtl;\n"
          << "  mul.wide.u32 %gb, %r1, " << T << ";\n"
          << "  mov.u32 %r4, %nctaid.x;\n  mul.wide.u32 %gstep, %r4, " << T << ";\n";
    for (std::size_t i = 0; i + 2 < fparams.size(); ++i) {
      body_ << "  ld.param.u64 %ka" << i << ", [" << fparams[i] << "];\n";
    }
    if (n_smem_ > 0) {
      // shared-tier words: one TMA bulk copy per CTA (cp.async.bulk, 1-D)
      // from the head of the global coefficient array, completing on an
      // mbarrier that every thread waits on before the first section
      body_ << "  ld.param.u64 %rd20, [pe_gcoef];\n  cvta.to.global.u64 %rd20, %rd20;\n"
            << "  mov.u64 %rd18, pe_scoef;\n  mov.u64 %rd19, pe_mbar;\n"
            << "  mov.u32 %r5, %tid.x;\n  setp.ne.u32 %p3, %r5, 0;\n  @%p3 bra $Lsarmed;\n"
            << "  mbarrier.init.shared::cta.b64 [%rd19], 1;\n  fence.proxy.async.shared::cta;\n"
            << "  mbarrier.arrive.expect_tx.shared::cta.b64 %rd17, [%rd19], " << 8 * n_smem_ << ";\n"
            << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%rd18], [%rd20], "
            << 8 * n_smem_ << ", [%rd19];\n"
            << "$Lsarmed:\n  bar.sync 0;\n$Lswait:\n"
            << "  mbarrier.try_wait.parity.shared::cta.b64 %p3, [%rd19], 0;\n  @!%p3 bra $Lswait;\n";
    }
    body_ << "$Lgroup:\n  setp.ge.u64 %gp, %gb, %gn;\n  @%gp bra.uni $Ldone;\n";
    for (std::size_t k = 0; k < cuts_.size(); ++k) {
      const std::string lt = "$Ltile" + std::to_string(k), le = "$Ltend" + std::to_string(k);
      body_ << "  mov.u64 %gt, 0;\n" << lt << ":\n"
            << "  add.u64 %gtile, %gb, %gt;\n  setp.ge.u64 %gp, %gtile, %gn;\n  @%gp bra.uni " << le << ";\n"
            << "  mul.lo.u64 %gbase, %gtile, %gtl;\n"
            // slot = scratch + ((ctaid * T + t) * L * tile) * 8
            << "  mul.wide.u32 %gsl, %r1, " << T << ";\n  add.u64 %gsl, %gsl, %gt;\n"
            << "  mul.lo.u64 %gsl, %gsl, %gtl;\n  mul.lo.u64 %gsl, %gsl, " << 8 * L << ";\n"
            << "  add.u64 %gsl, %gsl, %gs;\n  {\n";
      for (std::size_t i = 0; i < fparams.size(); ++i) {
        const std::string v = i + 2 == fparams.size() ? "%gbase" : i + 1 == fparams.size() ? "%gsl"
                                                                  : "%ka" + std::to_string(i);
        body_ << "  .param .u64 a" << i << ";\n  st.param.u64 [a" << i << "], " << v << ";\n";
      }
      body_ << "  call.uni pe_section" << k << ", (";
      for (std::size_t i = 0; i < fparams.size(); ++i) body_ << (i ? ", " : "") << "a" << i;
      body_ << ");\n  }\n"
            << "  add.u64 %gt, %gt, 1;\n  setp.lt.u64 %gp, %gt, " << T << ";\n  @%gp bra.uni " << lt << ";\n"
            << le << ":\n  bar.sync 0;\n";
    }
    body_ << "  add.u64 %gb, %gb, %gstep;\n  bra.uni $Lgroup;\n";
    finish_entry();
  }

  // SSA registers defined before each cut and read at or after it (or the
  // result), one list per cut except the last.
  std::vector<std::vector<std::uint32_t>> live_at_cuts() const {
    std::unordered_map<std::uint32_t, std::size_t> def, last;
    auto use = [&](const Operand& o, std::size_t at) {
      if (o.is(Operand::Reg)) last[o.id] = at;
    };
    for (std::size_t i = 0; i < s_.ops.size(); ++i) {
      use(s_.ops[i].a, i);
      use(s_.ops[i].b, i);
      use(s_.ops[i].c, i);
      def[s_.ops[i].dst] = i;
    }
    use(s_.result, s_.ops.size());
    std::vector<std::vector<std::uint32_t>> out(cuts_.size() > 0 ? cuts_.size() - 1 : 0);
    for (std::size_t c = 0; c + 1 < cuts_.size(); ++c) {
      for (const auto& [reg, d] : def) {
        auto it = last.find(reg);
        if (d < cuts_[c] && it != last.end() && it->second >= cuts_[c]) out[c].push_back(reg);
      }
      std::sort(out[c].begin(), out[c].end());
    }
    return out;
  }

  // Coordinates of the current tile (section-suffixed registers); the first
  // section also runs the int64 range checks.
  void emit_tile_coords(bool checks) {
    for (std::uint32_t v = 0; v < s_.nvars; ++v) {
      body_ << "  ld.param.u64 %rd5, [pe_in" << v << "];\n  cvta.to.global.u64 %rd5, %rd5;\n";
      for (std::uint32_t q = 0; q < P_; ++q) {
        if (d_ == Domain::I64F) {
          decls_ << "  .reg .f64 " << xr(v, q) << ";\n  .reg .b64 " << xi(v, q) << ";\n";
        } else {
          decls_ << "  .reg ." << ldty() << " " << xr(v, q) << ";\n";
        }
        body_ << "  add.u64 %rd6, %rd5, %ix" << q << ";\n  ld.global.nc." << ioty() << " "
              << (int_io() ? xi(v, q) : xr(v, q)) << ", [%rd6];\n";
        if (d_ == Domain::I64F) body_ << "  cvt.rn.f64.s64 " << xr(v, q) << ", " << xi(v, q) << ";\n";
      }
    }
    if (!checks || !int_io()) return;
    for (std::uint32_t v = 0; v < s_.nvars; ++v) {
      body_ << "  ld.param.u64 %rd8, [pe_bound" << v << "];\n";
      for (std::uint32_t q = 0; q < P_; ++q) {
        const std::string ok = "$Lgok" + std::to_string(v) + "_" + std::to_string(q);
        body_ << "  abs.s64 %rd9, " << xi(v, q) << ";\n  setp.gt.u64 %p2, %rd9, %rd8;\n"
              << "  @!%p2 bra " << ok << ";\n"
              << "  ld.param.u64 %rd7, [pe_flag];\n  cvta.to.global.u64 %rd7, %rd7;\n"
              << "  @%pv" << q << " st.global.u32 [%rd7], 1;\n" << ok << ":\n";
      }
    }
  }

  // Powers read by ops [begin, end) (and by the result, for the last
  // section), closed under the halving DAG.
  std::vector<char> powers_used(std::size_t begin, std::size_t end, bool last) const {
    std::vector<char> need(s_.powers.size(), 0);
    auto mark = [&](const Operand& o) {
      if (o.is(Operand::Pow)) need[o.id] = 1;
    };
    for (std::size_t i = begin; i < end; ++i) {
      mark(s_.ops[i].a);
      mark(s_.ops[i].b);
      mark(s_.ops[i].c);
    }
    if (last) mark(s_.result);
    for (std::size_t i = s_.powers.size(); i-- > 0;) {  // products follow their factors
      if (need[i] && s_.powers[i].exponent > 1) need[s_.powers[i].lo] = need[s_.powers[i].hi] = 1;
    }
    return need;
  }

  void declare_walk_regs() {
    for (std::uint32_t id = 0; id < s_.nregs; ++id) {
      std::ostringstream line;
      line << "  .reg .f64 ";
      if (intk()) line.str("  .reg .s64 ");
      line.seekp(0, std::ios_base::end);
      for (std::uint32_t k = 0; k < P_; ++k) {
        if (d_ == Domain::Interval) {
          line << (k ? ", " : "") << reg(id, k, false) << ", " << reg(id, k, true);
        } else if (d_ == Domain::I64K) {
          for (std::uint32_t j = 0; j < K_; ++j) line << (k || j ? ", " : "") << lb(reg(id, k), j);
        } else {
          line << (k ? ", " : "") << reg(id, k);
        }
      }
      line << ";\n";
      decls_ << line.str();
    }
  }

  void emit_ops(std::size_t begin, std::size_t end) {
    std::uint64_t since_sync = 0;
    std::size_t next_run = 0;
    for (std::size_t i = begin; i < end; ++i) {
      const Op& op = s_.ops[i];
      if (sync_every_ && ++since_sync == sync_every_) {
        body_ << "  bar.sync 0;\n";
        since_sync = 0;
      }
      if (d_ == Domain::Interval) {
        emit_iv_op(op);
      } else {
        emit_scalar_op(op);
        if (next_run < runs_.size() && runs_[next_run].head == i) {
          emit_chain_loop(runs_[next_run], next_run);
          i = runs_[next_run].last;
          ++next_run;
        }
      }
    }
  }

  // ---------------- chain loops ----------------
  // (see chain_runs above)

  // Constant-cache warm-up for the chain-loop arrays: thread t of every CTA
  // touches line t (64 B) of each array once, so the loop's one-trip-ahead
  // LDCU prefetch hits the SM's constant cache instead of paying one memory
  // round trip per trip on a cold cache (small batches after an L2 flush:
  // the loop is a single dependent chain of up to L/8 such misses). The
  // loaded word feeds a never-true comparison (coefficient words are finite,
  // touch is a prefetchu.L1 of the line.
  void emit_chain_warmup() {
    if (runs_.empty() || fix_) return;
    decls_ << "  .reg .b64 %wq<2>;\n  .reg .pred %wp<2>;\n  .reg .b32 %wl;\n";
    for (std::size_t idx = 0; idx < runs_.size(); ++idx) {
      const std::size_t words = runs_[idx].last - runs_[idx].head + loop_depth_ * kLoopU;
      const std::size_t lines = (words + 7) / 8;
      const std::string lbl = "$Lwarm" + std::to_string(idx);
      // for (line = tid; line < lines; line += ntid) touch(line)
      body_ << "  mov.u32 %wl, %r3;\n" << lbl << ":\n"
            << "  setp.ge.u32 %wp0, %wl, " << lines << ";\n  @%wp0 bra " << lbl << "e;\n"
            << "  cvta.const.u64 %wq0, pe_run" << idx
            << ";\n  mul.wide.u32 %wq1, %wl, 64;\n  add.u64 %wq0, %wq0, %wq1;\n"
            << "  prefetchu.L1 [%wq0];\n"
            << "  add.u32 %wl, %wl, %r2;\n  bra " << lbl << ";\n"
            << lbl << "e:\n";
    }
  }
  void find_chain_runs() {
    const std::uint64_t budget =
        n_const_ < CoefTiers::kConstCap ? CoefTiers::kConstCap - n_const_ : 0;
    runs_ = cuts_.size() > 1 ? std::vector<ChainRun>{}
                              : chain_runs(s_, d_, sync_every_, budget, tuning_.chain_min);
  }

  // Loop body: U steps; coefficients arrive as warp-uniform constant-bank
  // loads (LDCU) one iteration ahead of their use, so the load latency
  // overlaps the previous iteration's FMA chain. The array is padded with U
  // zero words so the last prefetch stays inside it. (Staging the words in
  // shared memory instead measured slower: 0.70 vs 0.59 ms per 1e7 C1 points,
  // per-thread LDS and +18 registers.)
  void emit_chain_loop(const ChainRun& run, std::size_t idx) {
    const std::uint32_t U = kLoopU, D = loop_depth_;
    const std::size_t L = run.last - run.head;
    const std::string arr = "pe_run" + std::to_string(idx);
    std::ostringstream a;
    a << ".const .align 16 .b64 " << arr << "[" << L + D * U << "] = {";
    for (std::size_t j = 0; j < L + D * U; ++j) {
      if (j) a << (j % 8 == 0 ? ",\n  " : ", ");
      a << (j < L ? hex64(words_[coef_lo_[s_.ops[run.head + 1 + j].c.id]]) : "0");
    }
    a << "};\n\n";
    run_arrays_ += a.str();
    // word sets: %lw0.. (this trip), %lw1.. (next trip), ... (depth D)
    auto set = [](std::uint32_t d) { return "%lw" + std::to_string(d) + "_"; };
    if (!loop_decls_) {
      decls_ << "  .reg .b64 %lp;\n  .reg .b32 %lc;\n  .reg .pred %lq;\n";
      for (std::uint32_t d = 0; d <= D; ++d) {
        decls_ << "  .reg ." << ldty() << " " << set(d) << "<" << U << ">;\n";
      }
      loop_decls_ = true;
    }
    const std::uint32_t acc = s_.ops[run.head].dst;
    const Loaded none;
    auto step = [&](std::uint32_t u, std::uint32_t si = 0) {
      for (std::uint32_t k = 0; k < P_; ++k) {
        const std::string r = reg(acc, k), m = opnd(run.mult, none, k);
        if (d_ == Domain::I64) {
          body_ << "  mad.lo.s64 " << r << ", " << r << ", " << m << ", " << set(si) << u << ";\n";
        } else {
          body_ << "  fma.rn.f64 " << r << ", " << r << ", " << m << ", " << set(si) << u << ";\n";
        }
      }
    };
    auto load8 = [&](const std::string& st, std::uint32_t off) {
      for (std::uint32_t u = 0; u < U; u += 2) {
        body_ << "  ld.const.v2." << ldty() << " {" << st << u << ", " << st << u + 1 << "}, [%lp+"
              << off + 8 * u << "];\n";
      }
    };
    const std::size_t iters = L / U, rem = L % U;
    const std::string lbl = "$Lrun" + std::to_string(idx);
    body_ << "  mov.u64 %lp, " << arr << ";\n";
    for (std::uint32_t d = 0; d < D; ++d) load8(set(d), 8 * U * d);
    {
      // rotating register sets, no moves: the loop body is R = D + 1 trips;
      // trip j uses set j and loads set (j + D) % R for the trip D ahead
      const std::uint32_t R = D + 1;
      const std::size_t outer = iters / R, tail = iters % R;
      if (outer > 0) {
        body_ << "  mov.u32 %lc, " << outer << ";\n" << lbl << ":\n";
        for (std::uint32_t j = 0; j < R; ++j) {
          load8(set((j + D) % R), 8 * U * (j + D));
          for (std::uint32_t u = 0; u < U; ++u) step(u, j);
        }
        body_ << "  add.u64 %lp, %lp, " << 8 * U * R << ";\n  sub.u32 %lc, %lc, 1;\n"
              << "  setp.ne.u32 %lq, %lc, 0;\n  @%lq bra.uni " << lbl << ";\n";
      }
      for (std::uint32_t j = 0; j < tail; ++j) {  // remaining full trips
        load8(set((j + D) % R), 8 * U * (j + D));
        for (std::uint32_t u = 0; u < U; ++u) step(u, j);
      }
      for (std::uint32_t u = 0; u < rem; ++u) step(u, static_cast<std::uint32_t>(tail));
    }
    const std::uint32_t dst = s_.ops[run.last].dst;
    if (dst != acc) {
      for (std::uint32_t k = 0; k < P_; ++k) {
        body_ << "  mov." << (d_ == Domain::I64 ? "b64" : "f64") << " " << reg(dst, k) << ", "
              << reg(acc, k) << ";\n";
      }
    }
    (d_ == Domain::I64 ? int_ops_ : fp_ops_) += L;
  }

  // ---------------- K-limb exact integers (Domain::I64K) ----------------
  // Values are K 64-bit limbs, two's complement, little-endian; arithmetic is
  // mod 2^(64K), which equals exact integer arithmetic because the host proof
  // bounds every intermediate below 2^(64K-1) in magnitude.
  std::vector<std::string> limbs_of(const std::string& r) const {
    std::vector<std::string> v;
    for (std::uint32_t j = 0; j < K_; ++j) v.push_back(lb(r, j));
    return v;
  }

  // Limbs of an operand; a coefficient is its int64 word, sign-extended by
  // immediates (0 / all ones).
  std::vector<std::string> opl(const Operand& o, const Loaded& l, std::uint32_t lane) const {
    switch (o.kind) {
      case Operand::Reg: return limbs_of(reg(o.id, lane));
      case Operand::Pow: return limbs_of(pw(o.id, lane));
      case Operand::Coef: {
        std::vector<std::string> v{l.lo};
        std::int64_t c = 0;
        if constexpr (std::is_same_v<C, std::int64_t>) c = s_.coefs[o.id];
        for (std::uint32_t j = 1; j < K_; ++j) v.push_back(c < 0 ? "-1" : "0");
        return v;
      }
      case Operand::Zero: return std::vector<std::string>(K_, "0");
      default: throw std::logic_error("bad operand");
    }
  }

  std::string reg_of(const std::string& x) {
    if (x.rfind('%', 0) == 0) return x;
    const std::string t = tmp_u();
    body_ << "  mov.b64 " << t << ", " << x << ";\n";
    return t;
  }

  // r = a + b (carry chain)
  void kadd(const std::vector<std::string>& r, const std::vector<std::string>& a,
            const std::vector<std::string>& b) {
    if (K_ == 1) {
      body_ << "  add.u64 " << r[0] << ", " << reg_of(a[0]) << ", " << b[0] << ";\n";
      return;
    }
    for (std::uint32_t j = 0; j < K_; ++j) {
      const char* op = j == 0 ? "add.cc" : (j + 1 < K_ ? "addc.cc" : "addc");
      body_ << "  " << op << ".u64 " << r[j] << ", " << reg_of(a[j]) << ", " << b[j] << ";\n";
    }
  }

  // One multiply-add carry chain: r[base + t] += half(a_i * b[t]) for t in [0, len).
  void mad_chain(const char* half, const std::vector<std::string>& r, std::uint32_t base,
                 const std::string& ai, const std::vector<std::string>& b, std::uint32_t len) {
    for (std::uint32_t t = 0; t < len; ++t) {
      std::string op = (t == 0 ? "mad." : "madc.") + std::string(half);
      if (t + 1 < len) op += ".cc";
      body_ << "  " << op << ".u64 " << r[base + t] << ", " << ai << ", " << reg_of(b[t]) << ", "
            << r[base + t] << ";\n";
    }
  }

  // r = a * b mod 2^(64K): truncated schoolbook, row i adds a_i * b shifted by
  // i limbs (low halves, then high halves, each one carry chain). A
  // coefficient operand goes in `a`, whose zero high limbs skip their rows.
  void kmul(const std::vector<std::string>& r, std::vector<std::string> a,
            std::vector<std::string> b) {
    if (a[0].rfind('%', 0) == 0 && a.size() > 1 && a[1].rfind('%', 0) == 0 &&
        !(b.size() > 1 && b[1].rfind('%', 0) == 0)) {
      std::swap(a, b);  // immediate-limbed operand (coefficient) first
    }
    const std::string a0 = reg_of(a[0]);
    for (std::uint32_t j = 0; j < K_; ++j) {
      body_ << "  mul.lo.u64 " << r[j] << ", " << a0 << ", " << reg_of(b[j]) << ";\n";
    }
    if (K_ > 1) mad_chain("hi", r, 1, a0, b, K_ - 1);
    for (std::uint32_t i = 1; i < K_; ++i) {
      if (a[i] == "0") continue;
      const std::string ai = reg_of(a[i]);
      mad_chain("lo", r, i, ai, b, K_ - i);
      if (K_ - i > 1) mad_chain("hi", r, i + 1, ai, b, K_ - i - 1);
    }
  }

  void emit_limb_op(const Op& op) {
    const Loaded la = load(op.a), lbd = load(op.b), lc = load(op.c);
    for (std::uint32_t k = 0; k < P_; ++k) {
      const auto d = limbs_of(reg(op.dst, k));
      const auto A = opl(op.a, la, k), B = opl(op.b, lbd, k);
      switch (op.kind) {
        case OpKind::Add:
          if (op.a.is(Operand::Zero)) {
            for (std::uint32_t j = 0; j < K_; ++j) body_ << "  mov.b64 " << d[j] << ", " << B[j] << ";\n";
          } else {
            kadd(d, A, B);
          }
          break;
        case OpKind::Mul:
          kmul(d, A, B);
          break;
        case OpKind::Fma:
          kmul(d, A, B);
          kadd(d, d, opl(op.c, lc, k));
          break;
      }
      if (k == 0) ++int_ops_;
    }
  }

  void emit_scalar_op(const Op& op) {
    if (d_ == Domain::I64K) {
      emit_limb_op(op);
      return;
    }
    const Loaded la = load(op.a), lb = load(op.b), lc = load(op.c);
    for (std::uint32_t k = 0; k < P_; ++k) {
      const std::string d = reg(op.dst, k);
      const std::string a = opnd(op.a, la, k), b = opnd(op.b, lb, k);
      if (d_ == Domain::I64) {
        switch (op.kind) {
          case OpKind::Add:
            if (op.a.is(Operand::Zero)) {
              body_ << "  mov.b64 " << d << ", " << b << ";\n";
            } else {
              body_ << "  add.s64 " << d << ", " << a << ", " << b << ";\n";
              if (k == 0) ++int_ops_;
            }
            break;
          case OpKind::Mul:
            body_ << "  mul.lo.s64 " << d << ", " << a << ", " << b << ";\n";
            if (k == 0) ++int_ops_;
            break;
          case OpKind::Fma:
            body_ << "  mad.lo.s64 " << d << ", " << a << ", " << b << ", " << opnd(op.c, lc, k)
                  << ";\n";
            if (k == 0) ++int_ops_;
            break;
        }
        continue;
      }
      switch (op.kind) {
        case OpKind::Add:
          body_ << "  add.rn.f64 " << d << ", " << a << ", " << b << ";\n";
          break;
        case OpKind::Mul:
          body_ << "  mul.rn.f64 " << d << ", " << a << ", " << b << ";\n";
          break;
        case OpKind::Fma:
          body_ << "  fma.rn.f64 " << d << ", " << a << ", " << b << ", " << opnd(op.c, lc, k) << ";\n";
          break;
      }
      if (k == 0) ++fp_ops_;
    }
  }

  // ---------------- interval primitives ----------------
  std::string tmp_f() { return "%tf" + std::to_string(n_tf_++); }
  std::string tmp_u() { return "%tu" + std::to_string(n_tu_++); }
  std::string tmp_p() { return "%tp" + std::to_string(n_tp_++); }
  std::string tmp_r() { return "%tr" + std::to_string(n_tr_++); }

  // dst = nextafter(src, +inf) (up) or nextafter(src, -inf) (down), exactly as
  // std::nextafter: +-0 -> +-denorm_min, NaN kept, +inf kept (up) / -inf kept
  // (down), otherwise one step of the magnitude in the right direction.
  void next(const std::string& dst, const std::string& src, bool up) {
    const std::string u = tmp_u(), s = tmp_u(), dlt = tmp_u(), r = tmp_u(), mag = tmp_u();
    const std::string pz = tmp_p(), pk = tmp_p();
    body_ << "  mov.b64 " << u << ", " << src << ";\n"
          << "  shr.s64 " << s << ", " << u << ", 63;\n"
          << "  or.b64 " << dlt << ", " << s << ", 1;\n"
          << (up ? "  add.s64 " : "  sub.s64 ") << r << ", " << u << ", " << dlt << ";\n"
          << "  and.b64 " << mag << ", " << u << ", 0x7FFFFFFFFFFFFFFF;\n"
          << "  setp.eq.u64 " << pz << ", " << mag << ", 0;\n"
          << "  selp.b64 " << r << ", " << (up ? "0x0000000000000001" : "0x8000000000000001")
          << ", " << r << ", " << pz << ";\n"
          << "  setp.gt.u64 " << pk << ", " << mag << ", 0x7FF0000000000000;\n"
          << "  setp.eq.or.u64 " << pk << ", " << u << ", "
          << (up ? "0x7FF0000000000000" : "0xFFF0000000000000") << ", " << pk << ";\n"
          << "  selp.b64 " << r << ", " << u << ", " << r << ", " << pk << ";\n"
          << "  mov.b64 " << dst << ", " << r << ";\n";
  }

  // interval_add (reference interval.cpp:36-41)
  void iv_add(const std::string& dlo, const std::string& dhi,
              const std::pair<std::string, std::string>& a,
              const std::pair<std::string, std::string>& b, bool a_is_zero, bool count) {
    if (a_is_zero) {
      // 0.0 + v == v up to the sign of zero, and nextafter maps +-0 alike
      next(dlo, b.first, false);
      next(dhi, b.second, true);
    } else {
      const std::string lo = tmp_f(), hi = tmp_f();
      body_ << "  add.rn.f64 " << lo << ", " << a.first << ", " << b.first << ";\n"
            << "  add.rn.f64 " << hi << ", " << a.second << ", " << b.second << ";\n";
      if (count) fp_ops_ += 2;
      next(dlo, lo, false);
      next(dhi, hi, true);
    }
  }

  // endpoint_product with the zero rule (reference interval.cpp:15-18)
  std::string eprod(const std::string& x, const std::string& y) {
    const std::string r = tmp_f();
    const std::string pz = tmp_p();
    body_ << "  mul.rn.f64 " << r << ", " << x << ", " << y << ";\n"
          << "  setp.eq.f64 " << pz << ", " << x << ", 0d0000000000000000;\n"
          << "  setp.eq.or.f64 " << pz << ", " << y << ", 0d0000000000000000, " << pz << ";\n"
          << "  selp.f64 " << r << ", 0d0000000000000000, " << r << ", " << pz << ";\n";
    return r;
  }

  // interval_mul (reference interval.cpp:43-52): hull of the four products in
  // std::min / std::max initializer-list scan order, then one step outward.
  void iv_mul(const std::string& dlo, const std::string& dhi,
              const std::pair<std::string, std::string>& a,
              const std::pair<std::string, std::string>& b, bool count) {
    const std::string p1 = eprod(a.first, b.first), p2 = eprod(a.first, b.second),
                      p3 = eprod(a.second, b.first), p4 = eprod(a.second, b.second);
    if (count) fp_ops_ += 4;
    const std::string mn = tmp_f(), mx = tmp_f();
    body_ << "  mov.f64 " << mn << ", " << p1 << ";\n  mov.f64 " << mx << ", " << p1 << ";\n";
    for (const std::string* p : {&p2, &p3, &p4}) {
      const std::string q = tmp_p();
      body_ << "  setp.lt.f64 " << q << ", " << *p << ", " << mn << ";\n"
            << "  selp.f64 " << mn << ", " << *p << ", " << mn << ", " << q << ";\n"
            << "  setp.lt.f64 " << q << ", " << mx << ", " << *p << ";\n"
            << "  selp.f64 " << mx << ", " << *p << ", " << mx << ", " << q << ";\n";
    }
    next(dlo, mn, false);
    next(dhi, mx, true);
  }

  // ---------------- interval replay, finite case ----------------
  // The fixup entry first replays a listed point with cheap primitives that
  // are exact as long as every value stays finite, and falls back to the
  // bit-level replay (next / iv_add / iv_mul above) only when a non-finite
  // value appeared (%pmid). With finite operands:
  //  * next_down(v) = RD(v - RN(|v| 2^-60 + dmin)): the subtracted amount is
  //    at least dmin and below the spacing of v, so the exact difference lies
  //    in [neighbour, v) — std::nextafter for every finite v including +-0
  //    (-> -dmin) and subnormals; next_up symmetric with RU.
  //  * interval_mul's zero rule only differs from RN(x*y) when the other
  //    operand is inf/NaN, or in the sign of a zero product; a zero's sign
  //    never survives the nextafter step that follows min/max (both +-0 step
  //    to -/+dmin), so plain products and min/max give the same endpoints.
  //  * the one zero this produces has the wrong sign: RD(dmin - dmin) is -0
  //    (std::nextafter(dmin, -inf) is +0), so the difference gets + (+0)
  //    in RN (-0 -> +0, everything else unchanged; next_down never returns
  //    -0); next_up(v) = -next_down(-v).
  void mnext(const std::string& dst, const std::string& src, bool up) {
    const std::string a = tmp_f(), t = tmp_f(), r = tmp_f();
    body_ << "  abs.f64 " << a << ", " << src << ";\n"
          << "  fma.rn.f64 " << t << ", " << a << ", 0d3C30000000000000, 0d0000000000000001;\n";
    if (up) {
      const std::string ns = tmp_f(), q = tmp_f();
      body_ << "  neg.f64 " << ns << ", " << src << ";\n"
            << "  sub.rm.f64 " << r << ", " << ns << ", " << t << ";\n"
            << "  add.rn.f64 " << q << ", " << r << ", 0d0000000000000000;\n"
            << "  neg.f64 " << dst << ", " << q << ";\n";
    } else {
      body_ << "  sub.rm.f64 " << r << ", " << src << ", " << t << ";\n"
            << "  add.rn.f64 " << dst << ", " << r << ", 0d0000000000000000;\n";
    }
    // inf or NaN result (DBL_MAX up, +inf down, overflow) poisons the
    // accumulator (0 * inf = NaN): the point then takes the exact replay
    body_ << "  fma.rn.f64 %macc, " << dst << ", 0d0000000000000000, %macc;\n";
  }

  void mid_add(const std::string& dlo, const std::string& dhi,
               const std::pair<std::string, std::string>& a,
               const std::pair<std::string, std::string>& b, bool a_is_zero) {
    if (a_is_zero) {
      mnext(dlo, b.first, false);
      mnext(dhi, b.second, true);
      return;
    }
    const std::string lo = tmp_f(), hi = tmp_f();
    body_ << "  add.rn.f64 " << lo << ", " << a.first << ", " << b.first << ";\n"
          << "  add.rn.f64 " << hi << ", " << a.second << ", " << b.second << ";\n";
    mnext(dlo, lo, false);
    mnext(dhi, hi, true);
  }

  void mid_mul(const std::string& dlo, const std::string& dhi,
               const std::pair<std::string, std::string>& a,
               const std::pair<std::string, std::string>& b) {
    const std::string p1 = tmp_f(), p2 = tmp_f(), p3 = tmp_f(), p4 = tmp_f();
    const std::string mn = tmp_f(), mx = tmp_f();
    body_ << "  mul.rn.f64 " << p1 << ", " << a.first << ", " << b.first << ";\n"
          << "  mul.rn.f64 " << p2 << ", " << a.first << ", " << b.second << ";\n"
          << "  mul.rn.f64 " << p3 << ", " << a.second << ", " << b.first << ";\n"
          << "  mul.rn.f64 " << p4 << ", " << a.second << ", " << b.second << ";\n"
          << "  mov.f64 " << mn << ", " << p1 << ";\n  mov.f64 " << mx << ", " << p1 << ";\n";
    // std::min / std::max scan order (no NaN can occur with finite operands)
    for (const std::string* p : {&p2, &p3, &p4}) {
      const std::string q = tmp_p(), r = tmp_p();
      body_ << "  setp.lt.f64 " << q << ", " << *p << ", " << mn << ";\n"
            << "  selp.f64 " << mn << ", " << *p << ", " << mn << ", " << q << ";\n"
            << "  setp.lt.f64 " << r << ", " << mx << ", " << *p << ";\n"
            << "  selp.f64 " << mx << ", " << *p << ", " << mx << ", " << r << ";\n";
    }
    mnext(dlo, mn, false);
    mnext(dhi, mx, true);
  }

  // ---------------- interval fast path ----------------
  // Same op sequence as the strict replay, cheaper primitives that are exact
  // under preconditions, plus a per-thread accumulator (%facc, sign bit) that
  // records every way a precondition can fail. A thread whose accumulator or
  // result says "special" re-runs the point through the strict replay, so
  // every result stays bit-identical to the reference.
  //
  //  * next_down/next_up of a finite nonzero double is -/+1 on its magnitude
  //    bits: u -/+ (s|1), s = u >> 63 (arith). This is std::nextafter except
  //    at +-0, +-inf and NaN; the failing cases flip the sign bit (+0 down,
  //    -0 up, canonical NaN up) or produce NaN (+inf up, -inf down), which
  //    the sign-flip accumulator and the final NaN/inf test catch.
  //  * a product of two intervals that do not straddle zero is, by
  //    monotonicity of RN, [RN(A1*B1), RN(A2*B2)] with the endpoint choice
  //    set by the two signs (interval_mul's min/max of four products,
  //    interval.cpp:43-52). Straddling register operands set the
  //    accumulator. Zero endpoints either give the same value as the zero
  //    rule or a zero that the next step flags; NaN/inf always reach one of
  //    the two products ({A1,A2} and {B1,B2} are both endpoint pairs).
  // nextafter of a value whose sign is unknown statically: RD(v - dmin) /
  // RU(v + dmin), dmin the smallest subnormal. For every finite v the exact
  // difference lies strictly between v and its neighbour on that side, or is
  // the neighbour itself (subnormal v), so directed rounding lands on
  // std::nextafter — zero included (-> -dmin / +dmin). Two cases differ:
  //  * +-inf: RD(+inf - dmin) stays +inf (std: DBL_MAX) — an infinite
  //    endpoint never turns finite on the fast path (a product with it is
  //    inf or NaN, a sum inf or NaN), so the final finiteness test sends
  //    the point to the exact replay;
  //  * v = +dmin down gives -0 (std: +0), v = -dmin up gives +0 (std: -0).
  //    A zero endpoint's sign is washed out by the next step (+-0 -/+ dmin
  //    is the same), by a product (the zero rule / a zero product is then
  //    stepped) and by a sum with a nonzero value; it is visible only as a
  //    result endpoint or, as the upper endpoint of a non-positive interval,
  //    through the straddle test (which flags it). Result endpoints equal
  //    to zero are flagged (emit_fast_exit).
  // One FP64 add per step, no "did not move" test (the former FMA-based
  // step needed an integer compare per step: 532 of C5's ~1350 ALU ops per
  // interval).
  void fnext(const std::string& dst, const std::string& src, bool up) {
    body_ << "  " << (up ? "add.rp" : "sub.rm") << ".f64 " << dst << ", " << src
          << ", 0d0000000000000001;\n";
  }

  // nextafter of a value whose sign is known statically (sign != 0): the
  // neighbour is the bit pattern +-1 (magnitude up for the outward step of
  // that sign, down for the inward one) — two 32-bit ALU adds, no check. It
  // is std::nextafter for every finite value of that sign including
  // subnormals; the cases where it is not (+0 down, -0 up, +-inf outward)
  // give NaN, and NaN/inf never turn finite again on the fast path, so the
  // final finiteness test sends such points to the strict replay. Unknown
  // sign: the FP64-pipe step with its "no move" test (fnext).
  void snext(const std::string& dst, const std::string& src, bool up, int sign) {
    if (sign == 0) {
      fnext(dst, src, up);
      return;
    }
    if (up == (sign > 0)) {
      // Outward step (magnitude grows) on the FP64 pipe, no check: RU(v +
      // v 2^-60) for v > 0 (RD for v < 0) lies strictly between v and its
      // outer neighbour for every finite nonzero v, subnormals included, so
      // directed rounding lands on std::nextafter (DBL_MAX -> inf, caught by
      // the final finiteness test). It does not move a zero — but the outer
      // endpoint of a same-sign interval is zero only if the inner one is
      // too, and the inner endpoint's integer step turns any zero into a NaN.
      body_ << "  fma." << (sign > 0 ? "rp" : "rm") << ".f64 " << dst << ", " << src
            << ", 0d3C30000000000000, " << src << ";\n";
      return;
    }
    // inward step: the bit pattern minus one (magnitude shrinks)
    const std::string u = tmp_u(), r = tmp_u();
    body_ << "  mov.b64 " << u << ", " << src << ";\n"
          << "  sub.s64 " << r << ", " << u << ", 1;\n"
          << "  mov.b64 " << dst << ", " << r << ";\n";
  }

  // sign: statically known sign of the sum (0 = unknown)
  void fast_add(const std::string& dlo, const std::string& dhi,
                const std::pair<std::string, std::string>& a,
                const std::pair<std::string, std::string>& b, bool a_is_zero, int sign = 0) {
    if (a_is_zero) {
      snext(dlo, b.first, false, sign);
      snext(dhi, b.second, true, sign);
      return;
    }
    const std::string lo = tmp_f(), hi = tmp_f();
    body_ << "  add.rn.f64 " << lo << ", " << a.first << ", " << b.first << ";\n"
          << "  add.rn.f64 " << hi << ", " << a.second << ", " << b.second << ";\n";
    snext(dlo, lo, false, sign);
    snext(dhi, hi, true, sign);
  }

  // accumulator |= (lo ^ hi): sign bit set iff the interval straddles zero
  // (or has a sign-mismatched zero endpoint) — only the high words matter
  void fcheck_straddle(const std::pair<std::string, std::string>& a) {
    const std::string ul = tmp_u(), uh = tmp_u(), x = tmp_u();
    body_ << "  mov.b64 " << ul << ", " << a.first << ";\n  mov.b64 " << uh << ", " << a.second
          << ";\n  xor.b64 " << x << ", " << ul << ", " << uh << ";\n  or.b64 %facc, %facc, " << x
          << ";\n";
  }

  // accumulator gets the sign bit if v is inf or NaN (exponent 0x7FF + 1
  // carries into the sign bit)
  void fcheck_finite(const std::string& v) {
    const std::string u = tmp_u(), e = tmp_u(), x = tmp_u();
    body_ << "  mov.b64 " << u << ", " << v << ";\n  add.s64 " << e << ", " << u
          << ", 0x0010000000000000;\n  xor.b64 " << x << ", " << e << ", " << u
          << ";\n  or.b64 %facc, %facc, " << x << ";\n";
  }

  // sa / sb: statically known sign of an operand (+1 / -1; 0 = decided at
  // run time from its upper endpoint). A known sign fixes which endpoints
  // pair up, so the corresponding selects (2 FSEL each) disappear.
  void fast_mul(const std::string& dlo, const std::string& dhi,
                const std::pair<std::string, std::string>& a,
                const std::pair<std::string, std::string>& b, bool check_a, bool check_b,
                int sa = 0, int sb = 0) {
    if (check_a && sa == 0) fcheck_straddle(a);
    if (check_b && sb == 0) fcheck_straddle(b);
    const std::string an = tmp_p(), bn = tmp_p(), ng = tmp_p();
    if (sa == 0) {
      const std::string ah = tmp_u();
      body_ << "  mov.b64 " << ah << ", " << a.second << ";\n  setp.lt.s64 " << an << ", " << ah
            << ", 0;\n";
    }
    if (sb == 0) {
      const std::string bh = tmp_u();
      body_ << "  mov.b64 " << bh << ", " << b.second << ";\n  setp.lt.s64 " << bn << ", " << bh
            << ", 0;\n";
    }
    if (sa == 0 && sb == 0) body_ << "  xor.pred " << ng << ", " << an << ", " << bn << ";\n";
    // pick(x_if_neg, x_if_pos, sign, pred)
    auto pick = [&](const std::string& if_neg, const std::string& if_pos, int sign,
                    const std::string& pred) {
      if (sign > 0) return if_pos;
      if (sign < 0) return if_neg;
      const std::string r = tmp_f();
      body_ << "  selp.f64 " << r << ", " << if_neg << ", " << if_pos << ", " << pred << ";\n";
      return r;
    };
    const std::string A1 = pick(a.second, a.first, sb, bn);
    const std::string A2 = pick(a.first, a.second, sb, bn);
    const std::string B1 = pick(b.second, b.first, sa, an);
    const std::string B2 = pick(b.first, b.second, sa, an);
    const std::string lo = tmp_f(), hi = tmp_f();
    body_ << "  mul.rn.f64 " << lo << ", " << A1 << ", " << B1 << ";\n"
          << "  mul.rn.f64 " << hi << ", " << A2 << ", " << B2 << ";\n";
    snext(dlo, lo, false, sa * sb);
    snext(dhi, hi, true, sa * sb);
  }

  // Static sign of an operand in the fast path: +1 / -1 when every
  // unflagged evaluation has that sign on both endpoints, 0 when unknown.
  // Coefficients are nonzero non-straddling (host-checked); squares are
  // positive; products and same-sign sums keep known signs (a known-sign
  // step turns a zero endpoint into a NaN, and powers stepped with the
  // unknown-sign step are straddle-checked where they are computed, so
  // "known" never hides a zero crossing).
  int sgn(const Operand& o) const {
    switch (o.kind) {
      case Operand::Coef: return ivcoef(o.id).lo > 0 ? 1 : -1;
      case Operand::Reg: return o.id < rsign_.size() ? rsign_[o.id] : 0;
      case Operand::Pow: return psign_[o.id];
      default: return 0;
    }
  }

  void emit_iv_op(const Op& op) {
    const Loaded la = load(op.a), lb = load(op.b);
    const int sa = fast_ ? sgn(op.a) : 0, sb = fast_ ? sgn(op.b) : 0;
    for (std::uint32_t k = 0; k < P_; ++k) {
      const std::string dlo = reg(op.dst, k, false), dhi = reg(op.dst, k, true);
      switch (op.kind) {
        case OpKind::Add:
          if (fast_) {
            const int sum_sign = op.a.is(Operand::Zero) ? sb : (sa == sb ? sa : 0);
            fast_add(dlo, dhi, ivop(op.a, la, k), ivop(op.b, lb, k), op.a.is(Operand::Zero),
                     sum_sign);
          } else if (medium_) {
            mid_add(dlo, dhi, ivop(op.a, la, k), ivop(op.b, lb, k), op.a.is(Operand::Zero));
          } else {
            iv_add(dlo, dhi, ivop(op.a, la, k), ivop(op.b, lb, k), op.a.is(Operand::Zero), k == 0);
          }
          break;
        case OpKind::Mul:
          if (fast_) {
            // coefficients are host-checked, powers checked where computed
            fast_mul(dlo, dhi, ivop(op.a, la, k), ivop(op.b, lb, k), op.a.is(Operand::Reg),
                     op.b.is(Operand::Reg), sa, sb);
          } else if (medium_) {
            mid_mul(dlo, dhi, ivop(op.a, la, k), ivop(op.b, lb, k));
          } else {
            iv_mul(dlo, dhi, ivop(op.a, la, k), ivop(op.b, lb, k), k == 0);
          }
          break;
        case OpKind::Fma:
          throw std::logic_error("interval streams are strict (no FMA)");
      }
    }
    if (fast_) {
      if (rsign_.size() <= op.dst) rsign_.resize(op.dst + 1, 0);
      int r = 0;
      if (op.kind == OpKind::Mul) {
        r = sa * sb;
      } else if (op.a.is(Operand::Zero)) {
        r = sb;
      } else if (sa == sb) {
        r = sa;
      }
      rsign_[op.dst] = r;
    }
  }

  // Interval fast path: if the accumulator or either result endpoint says
  // "special", the thread re-evaluates through the strict replay.
  void emit_fast_exit() {
    for (std::uint32_t k = 0; k < P_; ++k) {
      fcheck_finite(reg(s_.result.id, k, false));
      fcheck_finite(reg(s_.result.id, k, true));
      // a zero result endpoint may carry the wrong sign (fnext)
      for (bool hi : {false, true}) {
        body_ << "  setp.eq.or.f64 %pb" << (nb_ & 3) << ", " << reg(s_.result.id, k, hi)
              << ", 0d0000000000000000, %pb" << (nb_ & 3) << ";\n";
        ++nb_;
      }
    }
    // special: append the thread's valid point indices to the fixup list
    body_ << "  setp.lt.s64 %pslow, %facc, 0;\n"
          << "  or.pred %pslow, %pslow, %pb0;\n  or.pred %pslow, %pslow, %pb1;\n"
          << "  or.pred %pslow, %pslow, %pb2;\n  or.pred %pslow, %pslow, %pb3;\n"
          << "  @!%pslow bra $Lfaststore;\n"
          << "  ld.param.u64 %rd14, [pe_count];\n  cvta.to.global.u64 %rd14, %rd14;\n"
          << "  ld.param.u64 %rd15, [pe_list];\n  cvta.to.global.u64 %rd15, %rd15;\n"
          << "  ld.param.u64 %rd16, [pe_cap];\n"
          << "  ld.param.u64 %rd7, [pe_flag];\n  cvta.to.global.u64 %rd7, %rd7;\n";
    for (std::uint32_t k = 0; k < P_; ++k) {
      // list overflow (more special points than capacity): flag bit 4, the
      // host re-runs with a full-size list
      body_ << "  @%pv" << k << " atom.global.add.u32 %r4, [%rd14], 1;\n"
            << "  cvt.u64.u32 %rd17, %r4;\n  setp.lt.u64 %p3, %rd17, %rd16;\n"
            << "  not.pred %p4, %p3;\n  and.pred %p4, %p4, %pv" << k << ";\n"
            << "  @%p4 atom.global.or.b32 %r6, [%rd7], 4;\n"
            << "  and.pred %p3, %p3, %pv" << k << ";\n"
            << "  shr.u64 %rd18, %ix" << k << ", 3;\n  cvt.u32.u64 %r5, %rd18;\n"
            << "  shl.b64 %rd17, %rd17, 2;\n  add.u64 %rd17, %rd15, %rd17;\n"
            << "  @%p3 st.global.u32 [%rd17], %r5;\n";
    }
    body_ << "  bra $Ldone;\n$Lfaststore:\n";
    emit_store();
  }

  // Fixup entry: thread j takes list slot j of the first min(count, cap)
  // listed points and re-evaluates it (finite-case replay, then the
  // bit-level replay if needed); inputs were validated by the main entry or
  // the classifier.
  void emit_fix_prologue() {
    body_ << "  mov.u32 %r1, %ctaid.x;\n  mov.u32 %r2, %ntid.x;\n  mov.u32 %r3, %tid.x;\n"
          << "  mul.wide.u32 %rd1, %r1, %r2;\n  cvt.u64.u32 %rd2, %r3;\n  add.u64 %rd1, %rd1, %rd2;\n"
          << "  ld.param.u64 %rd14, [pe_count];\n  cvta.to.global.u64 %rd14, %rd14;\n"
          << "  ld.global.u32 %r5, [%rd14];\n  cvt.u64.u32 %rd3, %r5;\n"
          << "  ld.param.u64 %rd16, [pe_cap];\n  min.u64 %rd3, %rd3, %rd16;\n"
          << "  ld.param.u64 %rd15, [pe_list];\n  cvta.to.global.u64 %rd15, %rd15;\n";
    if (n_global_ > 0) {
      body_ << "  ld.param.u64 %rd20, [pe_gcoef];\n  cvta.to.global.u64 %rd20, %rd20;\n";
    }
    decls_ << "  .reg .b64 %ix<1>;\n  .reg .pred %pv<1>;\n";
    for (std::uint32_t v = 0; v < s_.nvars; ++v) {
      decls_ << "  .reg .f64 " << xr(v, 0, false) << ", " << xr(v, 0, true) << ";\n";
    }
    body_ << "$Lfix:\n  setp.ge.u64 %p1, %rd1, %rd3;\n  @%p1 bra $Ldone;\n"
          << "  shl.b64 %rd17, %rd1, 2;\n  add.u64 %rd17, %rd15, %rd17;\n"
          << "  ld.global.u32 %r6, [%rd17];\n  cvt.u64.u32 %rd13, %r6;\n"
          << "  shl.b64 %ix0, %rd13, 3;\n  setp.eq.u64 %pv0, %rd13, %rd13;\n";
    for (std::uint32_t i = 0; i < 2 * s_.nvars; ++i) {
      body_ << "  ld.param.u64 %rd5, [pe_in" << i << "];\n  cvta.to.global.u64 %rd5, %rd5;\n"
            << "  add.u64 %rd6, %rd5, %ix0;\n  ld.global.nc.f64 " << xr(i / 2, 0, i % 2 == 1)
            << ", [%rd6];\n";
    }
  }

  // Persistent fixup: the replay of one listed point as a function of the
  // point index (and the coordinate / result pointers, passed through from
  // the kernel's parameters of the same names).
  std::vector<std::string> fix_params() const {
    std::vector<std::string> ps;
    for (std::uint32_t i = 0; i < 2 * s_.nvars; ++i) ps.push_back("pe_in" + std::to_string(i));
    ps.push_back("pe_out0");
    ps.push_back("pe_out1");
    ps.push_back("pe_gcoef");
    ps.push_back("pe_pt");
    return ps;
  }
  void emit_fix_function_prologue() {
    if (n_global_ > 0) {
      body_ << "  ld.param.u64 %rd20, [pe_gcoef];\n  cvta.to.global.u64 %rd20, %rd20;\n";
    }
    decls_ << "  .reg .b64 %ix<1>;\n  .reg .pred %pv<1>;\n";
    for (std::uint32_t v = 0; v < s_.nvars; ++v) {
      decls_ << "  .reg .f64 " << xr(v, 0, false) << ", " << xr(v, 0, true) << ";\n";
    }
    body_ << "  ld.param.u64 %rd13, [pe_pt];\n  shl.b64 %ix0, %rd13, 3;\n"
          << "  setp.eq.u64 %pv0, %rd13, %rd13;\n";
    for (std::uint32_t i = 0; i < 2 * s_.nvars; ++i) {
      body_ << "  ld.param.u64 %rd5, [pe_in" << i << "];\n  cvta.to.global.u64 %rd5, %rd5;\n"
            << "  add.u64 %rd6, %rd5, %ix0;\n  ld.global.nc.f64 " << xr(i / 2, 0, i % 2 == 1)
            << ", [%rd6];\n";
    }
  }
  std::string fix_function_text() const {
    std::ostringstream f;
    const auto ps = fix_params();
    f << ".func pe_fix_point(";
    for (std::size_t i = 0; i < ps.size(); ++i) f << (i ? ",\n  " : "\n  ") << ".param .u64 " << ps[i];
    f << ")\n{\n  .reg .pred %p<8>;\n  .reg .b32 %r<8>;\n  .reg .b64 %rd<24>;\n" << decls_.str()
      << body_.str() << "}\n\n";
    return f.str();
  }
  // the kernel: slot = global thread index, strided by the grid, while
  // slot < min(count, cap)
  void emit_fix_loop() {
    const auto ps = fix_params();
    decls_ << "  .reg .b64 %fk<" << ps.size() << ">;\n";
    body_ << "  mov.u32 %r1, %ctaid.x;\n  mov.u32 %r2, %ntid.x;\n  mov.u32 %r3, %tid.x;\n"
          << "  mul.wide.u32 %rd1, %r1, %r2;\n  cvt.u64.u32 %rd2, %r3;\n  add.u64 %rd1, %rd1, %rd2;\n"
          << "  mov.u32 %r4, %nctaid.x;\n  mul.wide.u32 %rd4, %r4, %r2;\n"
          << "  ld.param.u64 %rd14, [pe_count];\n  cvta.to.global.u64 %rd14, %rd14;\n"
          << "  ld.global.u32 %r5, [%rd14];\n  cvt.u64.u32 %rd3, %r5;\n"
          << "  ld.param.u64 %rd16, [pe_cap];\n  min.u64 %rd3, %rd3, %rd16;\n"
          << "  ld.param.u64 %rd15, [pe_list];\n  cvta.to.global.u64 %rd15, %rd15;\n";
    for (std::size_t i = 0; i + 1 < ps.size(); ++i) {
      body_ << "  ld.param.u64 %fk" << i << ", [" << ps[i] << "];\n";
    }
    body_ << "$Lfix:\n  setp.ge.u64 %p1, %rd1, %rd3;\n  @%p1 bra $Ldone;\n"
          << "  shl.b64 %rd17, %rd1, 2;\n  add.u64 %rd17, %rd15, %rd17;\n"
          << "  ld.global.u32 %r6, [%rd17];\n  cvt.u64.u32 %fk" << ps.size() - 1 << ", %r6;\n  {\n";
    for (std::size_t i = 0; i < ps.size(); ++i) {
      body_ << "  .param .u64 a" << i << ";\n  st.param.u64 [a" << i << "], %fk" << i << ";\n";
    }
    body_ << "  call.uni pe_fix_point, (";
    for (std::size_t i = 0; i < ps.size(); ++i) body_ << (i ? ", " : "") << "a" << i;
    body_ << ");\n  }\n  add.u64 %rd1, %rd1, %rd4;\n  bra $Lfix;\n";
  }

  // ---------------- one-pass sign split (interval fast path) ----------------
  // role 1: the program at [lo, hi] with lo > 0; role 2: the mirrored
  // program q(y) = p(-y) at [-hi, -lo] (hi < 0). Statically positive
  // coordinate, no straddle checks (the split kernel classified it).
  std::string point_function(const std::string& name, std::uint32_t role) {
    const std::uint32_t lanes = P_, sync = sync_every_;
    P_ = 1;
    // no CTA barriers inside: only the threads holding a packed slot of this
    // sign call the function (a bar.sync here deadlocks the CTA)
    sync_every_ = 0;
    reset_entry();
    decls_ << "  .reg .f64 " << xr(0, 0, false) << ", " << xr(0, 0, true) << ";\n"
           << "  .reg .b64 %facc;\n  .reg .pred %pslow;\n  .reg .pred %pb<4>;\n";
    body_ << "  ld.param.f64 " << xr(0, 0, false) << ", [pe_a_lo];\n"
          << "  ld.param.f64 " << xr(0, 0, true) << ", [pe_a_hi];\n";
    if (role == 2) {
      const std::string t = tmp_f();
      body_ << "  neg.f64 " << t << ", " << xr(0, 0, true) << ";\n"
            << "  neg.f64 " << xr(0, 0, true) << ", " << xr(0, 0, false) << ";\n"
            << "  mov.f64 " << xr(0, 0, false) << ", " << t << ";\n";
    }
    body_ << "  mov.b64 %facc, 0;\n  mov.u32 %r3, 0;\n";
    for (int i = 0; i < 4; ++i) body_ << "  setp.ne.b32 %pb" << i << ", %r3, %r3;\n";
    fast_ = true;
    gather_ = role;
    emit_powers();
    emit_walk();
    const std::string rl = reg(s_.result.id, 0, false), rh = reg(s_.result.id, 0, true);
    fcheck_finite(rl);
    fcheck_finite(rh);
    for (const std::string* r : {&rl, &rh}) {  // a zero result may carry the wrong sign
      body_ << "  setp.eq.or.f64 %pb" << (nb_ & 3) << ", " << *r << ", 0d0000000000000000, %pb"
            << (nb_ & 3) << ";\n";
      ++nb_;
    }
    body_ << "  setp.lt.s64 %pslow, %facc, 0;\n"
          << "  or.pred %pslow, %pslow, %pb0;\n  or.pred %pslow, %pslow, %pb1;\n"
          << "  or.pred %pslow, %pslow, %pb2;\n  or.pred %pslow, %pslow, %pb3;\n"
          << "  selp.u32 pe_r_slow, 1, 0, %pslow;\n"
          << "  mov.f64 pe_r_lo, " << rl << ";\n  mov.f64 pe_r_hi, " << rh << ";\n";
    fast_ = false;
    gather_ = 0;
    body_ << "  ret;\n";
    if (n_creg_ > 0) decls_ << "  .reg ." << ldty() << " %c<" << n_creg_ << ">;\n";
    if (n_tf_ > 0) decls_ << "  .reg .f64 %tf<" << n_tf_ << ">;\n";
    if (n_tu_ > 0) decls_ << "  .reg .b64 %tu<" << n_tu_ << ">;\n";
    if (n_tp_ > 0) decls_ << "  .reg .pred %tp<" << n_tp_ << ">;\n";
    if (n_tr_ > 0) decls_ << "  .reg .b32 %tr<" << n_tr_ << ">;\n";
    std::ostringstream f;
    f << ".func (.reg .f64 pe_r_lo, .reg .f64 pe_r_hi, .reg .b32 pe_r_slow) " << name
      << "(.param .f64 pe_a_lo, .param .f64 pe_a_hi)\n{\n"
      << "  .reg .pred %p<8>;\n  .reg .b32 %r<8>;\n  .reg .b64 %rd<24>;\n" << decls_.str()
      << body_.str() << "}\n\n";
    P_ = lanes;
    sync_every_ = sync;
    return f.str();
  }

  // The split entry: a persistent kernel that reads and writes every
  // interval once. Each CTA strides over tiles of ntid consecutive intervals:
  // it classifies a tile (lo > 0 / hi < 0 / the rest -> fixup list, invalid ->
  // status bit 2) and appends the two signs to two ring queues in shared
  // memory (warp ballots + a CTA prefix give every interval its slot).
  // Whenever a queue holds a full CTA of intervals, every thread takes one and
  // all of them call that sign's point function (the program for x > 0, the
  // mirrored program for x < 0): warps never mix the two functions (a warp
  // that ran both in turn held its CTA twice as long — the first version of
  // this kernel, 12.6 ms per 1e8 on C5 against 10.5 for the classifier path)
  // and every lane is busy. What is left in the queues after the last tile is
  // flushed by partial CTAs. Queue capacity per sign: a power of two >= 2 * ntid.
  // Ring entries per sign (a power of two). A queue holds < 2 * ntid entries
  // after an append; with 4 * ntid slots the next tile's appends (reached
  // only through the tile barrier) cannot wrap onto slots a slower warp is
  // still to read for the current drain, so the drain needs no barrier of
  // its own. 512-thread CTAs would pass the 48 KB static limit: 2 * ntid
  // slots and a barrier after the drain's reads.
  static std::uint32_t split_ring(std::uint32_t block) {
    std::uint32_t r = 128;
    while (r < (block <= 256 ? 4 : 2) * block) r *= 2;
    return r;
  }
  void emit_split_entry() {
    const std::uint32_t ring = split_ring(block_);  // entries per sign, a power of two >= 2 * ntid
    decls_ << "  .reg .b64 %sa, %sb, %gt, %gnt, %gstep, %gix, %gnm1;\n"
           << "  .reg .pred %pv<1>, %sp, %sn, %so, %sx, %pfin, %pfull, %pgo, %pact;\n"
           << "  .reg .b32 %smp, %smn, %slt, %sw, %slane, %sslot, %sq, %sfl, %snw, %sm, %sgi;\n"
           << "  .reg .b32 %qhp, %qcp, %qhn, %qcn, %sk;\n"
           << "  .reg .f64 %sxl, %sxh, %srl, %srh;\n";
    body_ << "  mov.u32 %r1, %ctaid.x;\n  mov.u32 %r2, %ntid.x;\n  mov.u32 %r3, %tid.x;\n"
          << "  ld.param.u64 %rd3, [pe_n];\n  sub.u64 %gnm1, %rd3, 1;\n"
          << "  cvt.u64.u32 %rd2, %r3;\n  cvt.u64.u32 %rd4, %r2;\n"
          << "  add.u64 %gnt, %rd3, %rd4;\n  sub.u64 %gnt, %gnt, 1;\n  div.u64 %gnt, %gnt, %rd4;\n"
          << "  cvt.u64.u32 %gt, %r1;\n  mov.u32 %r4, %nctaid.x;\n  cvt.u64.u32 %gstep, %r4;\n"
          << "  ld.param.u64 %rd8, [pe_in0];\n  cvta.to.global.u64 %rd8, %rd8;\n"
          << "  ld.param.u64 %rd9, [pe_in1];\n  cvta.to.global.u64 %rd9, %rd9;\n"
          << "  ld.param.u64 %rd10, [pe_out0];\n  cvta.to.global.u64 %rd10, %rd10;\n"
          << "  ld.param.u64 %rd11, [pe_out1];\n  cvta.to.global.u64 %rd11, %rd11;\n"
          << "  ld.param.u64 %rd7, [pe_flag];\n  cvta.to.global.u64 %rd7, %rd7;\n"
          << "  ld.param.u64 %rd14, [pe_count];\n  cvta.to.global.u64 %rd14, %rd14;\n"
          << "  ld.param.u64 %rd15, [pe_list];\n  cvta.to.global.u64 %rd15, %rd15;\n"
          << "  ld.param.u64 %rd16, [pe_cap];\n"
          << "  and.b32 %slane, %r3, 31;\n  shr.u32 %sw, %r3, 5;\n  shr.u32 %snw, %r2, 5;\n"
          << "  mov.u32 %r4, 1;\n  shl.b32 %slt, %r4, %slane;\n  sub.u32 %slt, %slt, 1;\n"
          << "  mov.u32 %qhp, 0;\n  mov.u32 %qcp, 0;\n  mov.u32 %qhn, 0;\n  mov.u32 %qcn, 0;\n";
    // appends interval index `idx` (u32 register) to the fixup list under `pred`
    auto append = [&](const char* pred, const char* idx) {
      body_ << "  @" << pred << " atom.global.add.u32 %r4, [%rd14], 1;\n"
            << "  cvt.u64.u32 %rd17, %r4;\n  setp.lt.u64 %p3, %rd17, %rd16;\n"
            << "  not.pred %p4, %p3;\n  and.pred %p4, %p4, " << pred << ";\n"
            << "  @%p4 atom.global.or.b32 %r5, [%rd7], 4;\n"
            << "  and.pred %p3, %p3, " << pred << ";\n"
            << "  shl.b64 %rd17, %rd17, 2;\n  add.u64 %rd17, %rd15, %rd17;\n"
            << "  @%p3 st.global.u32 [%rd17], " << idx << ";\n";
    };
    // per-tile totals {x > 0, x < 0} rotate through three shared slots: the
    // slot of tile k+1 is cleared during tile k, whose readers of the slot
    // of tile k-2 are all past barrier k-1
    body_ << "  mov.u32 %sk, 0;\n  setp.ne.u32 %p5, %r3, 0;\n  @%p5 bra $Lsplit_init;\n"
          << "  mov.u32 %r4, 0;\n  st.shared.v2.u32 [pe_sp_w], {%r4, %r4};\n"
          << "  st.shared.v2.u32 [pe_sp_w+8], {%r4, %r4};\n  st.shared.v2.u32 [pe_sp_w+16], {%r4, %r4};\n"
          << "$Lsplit_init:\n  bar.sync 0;\n";
    body_ << "$Ltile:\n  setp.ge.u64 %pfin, %gt, %gnt;\n  @%pfin bra.uni $Lphase_pos;\n"
          << "  mul.lo.u64 %rd1, %gt, %rd4;\n  add.u64 %rd13, %rd1, %rd2;\n"
          << "  setp.lt.u64 %pv0, %rd13, %rd3;\n  min.u64 %rd13, %rd13, %gnm1;\n"
          << "  cvt.u32.u64 %sgi, %rd13;\n  shl.b64 %gix, %rd13, 3;\n"
          << "  add.u64 %rd6, %rd8, %gix;\n  ld.global.nc.f64 %sxl, [%rd6];\n"
          << "  add.u64 %rd6, %rd9, %gix;\n  ld.global.nc.f64 %sxh, [%rd6];\n"
          // the CTA's next tile is a grid stride away: bring its lines to L2
          << "  add.u64 %gt, %gt, %gstep;\n  mul.lo.u64 %rd1, %gt, %rd4;\n  add.u64 %rd13, %rd1, %rd2;\n"
          << "  min.u64 %rd13, %rd13, %gnm1;\n  shl.b64 %gix, %rd13, 3;\n"
          << "  add.u64 %rd6, %rd8, %gix;\n  prefetch.global.L2 [%rd6];\n"
          << "  add.u64 %rd6, %rd9, %gix;\n  prefetch.global.L2 [%rd6];\n"
          // classify (reference Interval(lo, hi) rejects NaN / lo > hi)
          << "  setp.le.f64 %sx, %sxl, %sxh;\n  and.pred %sx, %sx, %pv0;\n"
          << "  setp.gt.f64 %sp, %sxl, 0d0000000000000000;\n  and.pred %sp, %sp, %sx;\n"
          << "  setp.lt.f64 %sn, %sxh, 0d0000000000000000;\n  and.pred %sn, %sn, %sx;\n"
          << "  or.pred %so, %sp, %sn;\n  not.pred %so, %so;\n  and.pred %so, %so, %pv0;\n"
          << "  not.pred %p2, %sx;\n  and.pred %p2, %p2, %pv0;\n"
          << "  @%p2 atom.global.or.b32 %r5, [%rd7], 2;\n";
    append("%so", "%sgi");  // touching / straddling zero, invalid: the fixup replay (rare)
    // slots: warp ballots; lane 0 reserves the warp's run in each queue with
    // a shared-memory atomic on the tile's totals (queue order is free)
    body_ << "  vote.sync.ballot.b32 %smp, %sp, 0xffffffff;\n"
          << "  vote.sync.ballot.b32 %smn, %sn, 0xffffffff;\n"
          << "  setp.eq.u32 %p5, %slane, 0;\n  mov.u64 %sa, pe_sp_w;\n"
          << "  mul.wide.u32 %sb, %sk, 8;\n  add.u64 %sa, %sa, %sb;\n"
          << "  popc.b32 %r4, %smp;\n  popc.b32 %r5, %smn;\n  mov.u32 %r6, 0;\n  mov.u32 %r7, 0;\n"
          << "  @%p5 atom.shared.add.u32 %r6, [%sa], %r4;\n"
          << "  @%p5 atom.shared.add.u32 %r7, [%sa+4], %r5;\n"
          << "  shfl.sync.idx.b32 %r6, %r6, 0, 31, 0xffffffff;\n"
          << "  shfl.sync.idx.b32 %r7, %r7, 0, 31, 0xffffffff;\n"
          // thread 0 clears the next tile's totals
          << "  add.u32 %sq, %sk, 1;\n  setp.eq.u32 %p6, %sq, 3;\n  selp.u32 %sq, 0, %sq, %p6;\n"
          << "  setp.ne.u32 %p6, %r3, 0;\n  @%p6 bra $Lsplit_cleared;\n"
          << "  mov.u64 %sb, pe_sp_w;\n  mul.wide.u32 %rd17, %sq, 8;\n  add.u64 %sb, %sb, %rd17;\n"
          << "  mov.u32 %r4, 0;\n  st.shared.v2.u32 [%sb], {%r4, %r4};\n"
          << "$Lsplit_cleared:\n"
          // x > 0: ring slot (head + count + warp base + rank) mod ring
          << "  and.b32 %r4, %smp, %slt;\n  popc.b32 %r4, %r4;\n"
          << "  add.u32 %sslot, %r6, %r4;\n  add.u32 %sslot, %sslot, %qhp;\n"
          << "  add.u32 %sslot, %sslot, %qcp;\n  and.b32 %sslot, %sslot, " << ring - 1 << ";\n"
          // x < 0: the second half of the arrays
          << "  and.b32 %r4, %smn, %slt;\n  popc.b32 %r4, %r4;\n"
          << "  add.u32 %r5, %r7, %r4;\n  add.u32 %r5, %r5, %qhn;\n  add.u32 %r5, %r5, %qcn;\n"
          << "  and.b32 %r5, %r5, " << ring - 1 << ";\n  add.u32 %r5, %r5, " << ring << ";\n"
          << "  selp.u32 %sslot, %sslot, %r5, %sp;\n"
          << "  or.pred %p5, %sp, %sn;\n  @!%p5 bra $Lsplit_packed;\n"
          << "  mul.wide.u32 %sb, %sslot, 8;\n  mov.u64 %rd17, pe_sp_lo;\n  add.u64 %rd17, %rd17, %sb;\n"
          << "  st.shared.f64 [%rd17], %sxl;\n  mov.u64 %rd17, pe_sp_hi;\n  add.u64 %rd17, %rd17, %sb;\n"
          << "  st.shared.f64 [%rd17], %sxh;\n  mul.wide.u32 %sb, %sslot, 4;\n  mov.u64 %rd17, pe_sp_idx;\n"
          << "  add.u64 %rd17, %rd17, %sb;\n  st.shared.u32 [%rd17], %sgi;\n"
          << "$Lsplit_packed:\n  bar.sync 0;\n"
          << "  ld.shared.v2.u32 {%r6, %r7}, [%sa];\n"
          << "  add.u32 %qcp, %qcp, %r6;\n  add.u32 %qcn, %qcn, %r7;\n  mov.u32 %sk, %sq;\n";
    // one queue: while it holds a full CTA (or, after the last tile, anything)
    auto phase = [&](const char* tag, const char* head, const char* count, const char* fn,
                     std::uint32_t offset, const std::string& next) {
      const std::string t(tag);
      body_ << "$Lphase_" << t << ":\n"
            << "  setp.ge.u32 %pfull, " << count << ", %r2;\n"
            << "  setp.ne.u32 %pgo, " << count << ", 0;\n  and.pred %pgo, %pgo, %pfin;\n"
            << "  or.pred %pgo, %pgo, %pfull;\n  @!%pgo bra.uni " << next << ";\n"
            << "  min.u32 %sm, " << count << ", %r2;\n  setp.lt.u32 %pact, %r3, %sm;\n"
            << "  add.u32 %sslot, " << head << ", %r3;\n  and.b32 %sslot, %sslot, " << ring - 1 << ";\n";
      if (offset) body_ << "  add.u32 %sslot, %sslot, " << offset << ";\n";
      body_ << "  mul.wide.u32 %sb, %sslot, 8;\n  mov.u64 %sa, pe_sp_lo;\n  add.u64 %sa, %sa, %sb;\n"
            << "  ld.shared.f64 %sxl, [%sa];\n  mov.u64 %sa, pe_sp_hi;\n  add.u64 %sa, %sa, %sb;\n"
            << "  ld.shared.f64 %sxh, [%sa];\n  mul.wide.u32 %sb, %sslot, 4;\n  mov.u64 %sa, pe_sp_idx;\n"
            << "  add.u64 %sa, %sa, %sb;\n  ld.shared.u32 %sgi, [%sa];\n"
            // (slots of inactive threads: stale, unused)
            << (ring < 4 * block_ ? "  bar.sync 0;\n" : "") << "  @!%pact bra $Lskip_" << t << ";\n"
            // the call binds its own .param arguments (a st.param belongs to
            // the one call that follows it in its scope)
            << "  {\n  .param .f64 a0;\n  .param .f64 a1;\n"
            << "  st.param.f64 [a0], %sxl;\n  st.param.f64 [a1], %sxh;\n"
            << "  call (%srl, %srh, %sfl), " << fn << ", (a0, a1);\n  }\n"
            << "  setp.ne.u32 %p7, %sfl, 0;\n";
      append("%p7", "%sgi");  // not proven by the fast path: the fixup replay
      body_ << "  @%p7 bra $Lskip_" << t << ";\n"
            << "  cvt.u64.u32 %rd18, %sgi;\n  shl.b64 %rd18, %rd18, 3;\n"
            << "  add.u64 %rd6, %rd10, %rd18;\n  st.global.f64 [%rd6], %srl;\n"
            << "  add.u64 %rd6, %rd11, %rd18;\n  st.global.f64 [%rd6], %srh;\n"
            << "$Lskip_" << t << ":\n"
            << "  add.u32 " << head << ", " << head << ", %sm;\n"
            << "  sub.u32 " << count << ", " << count << ", %sm;\n"
            << "  bra.uni $Lphase_" << t << ";\n";
    };
    phase("pos", "%qhp", "%qcp", "pe_iv_pos", 0, "$Lphase_neg");
    phase("neg", "%qhn", "%qcn", "pe_iv_neg", ring, "$Lphases_done");
    body_ << "$Lphases_done:\n  @!%pfin bra.uni $Ltile;\n";
  }

  void emit_epilogue() {
    emit_store();
    finish_entry();
  }

  void emit_store() {
    const bool iv = d_ == Domain::Interval;
    const Loaded lr = load(s_.result);
    if (d_ == Domain::I64K) {
      for (std::uint32_t j = 0; j < K_; ++j) {
        body_ << "  ld.param.u64 %rd9, [pe_out" << j << "];\n  cvta.to.global.u64 %rd9, %rd9;\n";
        for (std::uint32_t k = 0; k < P_; ++k) {
          const std::string v = reg_of(opl(s_.result, lr, k)[j]);
          body_ << "  add.u64 %rd10, %rd9, %ix" << k << ";\n  @%pv" << k << " st.global.b64 [%rd10], "
                << v << ";\n";
        }
      }
      return;
    }
    for (std::uint32_t o = 0; o < (iv ? 2u : 1u); ++o) {
      body_ << "  ld.param.u64 %rd9, [pe_out" << o << "];\n  cvta.to.global.u64 %rd9, %rd9;\n";
      for (std::uint32_t k = 0; k < P_; ++k) {
        std::string val;
        if (iv) {
          auto r = ivop(s_.result, lr, k);
          val = o == 0 ? r.first : r.second;
        } else {
          val = opnd(s_.result, lr, k);
        }
        if (val.rfind('%', 0) != 0) {  // immediate zero: stage through a register
          const std::string t = tmp_u();
          body_ << "  mov.b64 " << t << ", 0;\n";
          val = t;
        } else if (d_ == Domain::I64F) {  // exact integer-valued double -> int64
          const std::string t = tmp_u();
          body_ << "  cvt.rni.s64.f64 " << t << ", " << val << ";\n";
          val = t;
        }
        body_ << "  add.u64 %rd10, %rd9, %ix" << k << ";\n";
        body_ << "  @%pv" << k << " st.global." << ioty() << " [%rd10], " << val << ";\n";
      }
    }
  }

  const Stream<C>& s_;
  Domain d_;
  std::uint32_t P_;
  std::uint32_t block_;
  std::uint32_t sync_every_;
  bool paired_;  // scalar domains: paired coefficient loads, register-bound second region
  std::uint32_t min_ctas_ = 0;
  std::uint32_t K_ = 1;  // I64K limbs
  std::uint32_t part_ = 0;    // KernelShape::iv_partition
  Tuning tuning_;
  std::vector<std::size_t> cuts_;  // section boundaries (op indices), ascending, ends with ops.size()
  std::uint32_t sec_ = 0;          // section being emitted
  std::uint32_t group_tiles_ = 4;  // sectioned kernels: tiles per CTA per section pass
  std::string funcs_;              // sectioned kernels: the section functions
  std::string sym_ = "pe_coef";    // name of the module's constant-bank coefficient array
  std::string cbase() const { return sym_; }
  std::string split_funcs_;        // the mirrored program's point function (+ its constants)
  bool fast_ = false;  // emitting the interval fast path
  bool medium_ = false;  // emitting the finite-case replay of the fixup entry
  std::uint32_t gather_ = 0;  // emitting a partitioned entry: 1 front (x > 0), 2 back (x < 0)
  bool fix_ = false;   // emitting the fixup entry
  std::uint32_t nb_ = 0;
  std::vector<int> rsign_, psign_;  // fast path: static signs of registers / powers
  static constexpr std::uint32_t kLoopU = 8;  // loop unroll (steps per trip)
  // Chain-loop coefficient prefetch: D trips ahead into rotating register
  // sets (loop body = D + 1 trips, no moves). The 1e5-point C1 kernel had 47 %
  // of its stall samples on the move of a one-trip-ahead set (waiting on its
  // LDCU); D = 2 rotating: C1 1e5 20.2 -> 18.6 us per call, 1e7 0.594 ->
  // 0.577 ms (profiles/r1_c1_small_batch.txt).
  static constexpr std::uint32_t loop_depth_ = 2;
  std::vector<ChainRun> runs_;
  std::string run_arrays_;
  bool loop_decls_ = false;
  std::vector<std::uint64_t> words_;
  std::unordered_map<std::uint32_t, std::string> pending_;  // second word of a loaded pair
  std::vector<char> reg_bound_;  // coefficient in the register-bound region
  std::vector<std::uint32_t> coef_lo_, coef_hi_;
  std::uint32_t n_const_ = 0, n_param_ = 0, n_smem_ = 0, n_global_ = 0;
  std::uint32_t const_words_ = 0, mirror_words_ = 0;
  std::uint32_t n_creg_ = 0, n_tf_ = 0, n_tu_ = 0, n_tp_ = 0, n_tr_ = 0;
  std::uint64_t fp_ops_ = 0, int_ops_ = 0;
  std::ostringstream body_, decls_;
};

}  // namespace

namespace {
// Latency-aware reordering of a fused stream (see emit_ptx):
// greedy list scheduling over a window of the next W unscheduled ops, taking
// the oldest op whose producers were emitted at least D ops earlier (else the
// oldest ready op), then renumbering coefficients by first use so paired
// constant loads stay adjacent. The ops are SSA (one definition per
// register), so any topological order computes the same values.
template <typename C>
Stream<C> schedule_stream(const Stream<C>& in, std::size_t W, std::size_t D,
                          const std::vector<std::size_t>& cuts) {
  const std::size_t n = in.ops.size();
  std::unordered_map<std::uint32_t, std::size_t> def;
  for (std::size_t i = 0; i < n; ++i) def[in.ops[i].dst] = i;
  std::vector<std::vector<std::size_t>> preds(n);
  for (std::size_t i = 0; i < n; ++i) {
    for (const Operand* o : {&in.ops[i].a, &in.ops[i].b, &in.ops[i].c}) {
      if (o->is(Operand::Reg)) {
        auto it = def.find(o->id);
        if (it != def.end() && it->second < i) preds[i].push_back(it->second);
      }
    }
  }
  std::vector<std::size_t> pos(n, SIZE_MAX), order;
  order.reserve(n);
  std::size_t first = 0;  // lowest unscheduled original index
  std::size_t sec = 0;    // ops never move across a section boundary
  while (order.size() < n) {
    while (first < n && pos[first] != SIZE_MAX) ++first;
    while (sec < cuts.size() && cuts[sec] <= first) ++sec;
    const std::size_t limit = sec < cuts.size() ? cuts[sec] : n;
    std::size_t pick = SIZE_MAX, fallback = SIZE_MAX;
    const std::size_t now = order.size();
    for (std::size_t i = first; i < limit && i < first + W; ++i) {
      if (pos[i] != SIZE_MAX) continue;
      bool ready = true, aged = true;
      for (std::size_t p : preds[i]) {
        if (pos[p] == SIZE_MAX) { ready = false; break; }
        if (pos[p] + D > now) aged = false;
      }
      if (!ready) continue;
      if (fallback == SIZE_MAX) fallback = i;
      if (aged) { pick = i; break; }
    }
    if (pick == SIZE_MAX) pick = fallback;
    pos[pick] = now;
    order.push_back(pick);
  }
  Stream<C> out = in;
  out.ops.clear();
  for (std::size_t i : order) out.ops.push_back(in.ops[i]);
  // coefficients by first use in the new order
  std::vector<std::uint32_t> remap(in.coefs.size(), UINT32_MAX);
  out.coefs.clear();
  out.widen.clear();
  out.odd.clear();
  auto use = [&](Operand& o) {
    if (!o.is(Operand::Coef)) return;
    if (remap[o.id] == UINT32_MAX) {
      remap[o.id] = static_cast<std::uint32_t>(out.coefs.size());
      out.coefs.push_back(in.coefs[o.id]);
      out.widen.push_back(o.id < in.widen.size() ? in.widen[o.id] : 0);
      out.odd.push_back(o.id < in.odd.size() ? in.odd[o.id] : 0);
    }
    o.id = remap[o.id];
  };
  for (auto& op : out.ops) {
    use(op.a);
    use(op.b);
    use(op.c);
  }
  use(out.result);
  for (std::size_t k = 0; k < in.coefs.size(); ++k) {  // unused (should not happen)
    if (remap[k] == UINT32_MAX) {
      remap[k] = static_cast<std::uint32_t>(out.coefs.size());
      out.coefs.push_back(in.coefs[k]);
      out.widen.push_back(k < in.widen.size() ? in.widen[k] : 0);
      out.odd.push_back(k < in.odd.size() ? in.odd[k] : 0);
    }
  }
  return out;
}

// Section boundaries of a long scalar walk: about `target` ops per section,
// each cut placed where the fewest walk values are live (they cross the
// boundary in registers), within a quarter section of its even position.
// Returns the ascending section ends (the last is ops.size()).
template <typename C>
std::vector<std::size_t> section_cuts(const Stream<C>& s, std::size_t target) {
  const std::size_t n = s.ops.size();
  if (target == 0 || n < target + target / 2) return {n};
  const std::size_t K = (n + target / 2) / target;
  // live[b]: values defined before op b and read at or after it
  std::unordered_map<std::uint32_t, std::size_t> def;
  std::vector<std::int64_t> diff(n + 2, 0);
  std::unordered_map<std::uint32_t, std::size_t> last_use;
  auto use = [&](const Operand& o, std::size_t at) {
    if (o.is(Operand::Reg)) last_use[o.id] = at;
  };
  for (std::size_t i = 0; i < n; ++i) {
    use(s.ops[i].a, i);
    use(s.ops[i].b, i);
    use(s.ops[i].c, i);
    def[s.ops[i].dst] = i;
  }
  use(s.result, n);
  for (const auto& [reg, d] : def) {
    auto it = last_use.find(reg);
    if (it == last_use.end() || it->second <= d) continue;
    diff[d + 1] += 1;
    diff[it->second + 1] -= 1;
  }
  std::vector<std::int64_t> live(n + 1, 0);
  std::int64_t run = 0;
  for (std::size_t b = 0; b <= n; ++b) {
    run += diff[b];
    live[b] = run;
  }
  std::vector<std::size_t> cuts;
  const std::size_t slack = std::max<std::size_t>(1, n / (4 * K));
  for (std::size_t k = 1; k < K; ++k) {
    const std::size_t t = k * n / K;
    std::size_t best = t;
    for (std::size_t b = t > slack ? t - slack : 1; b <= std::min(n - 1, t + slack); ++b) {
      const auto dist = [&](std::size_t x) { return x > t ? x - t : t - x; };
      if (live[b] < live[best] || (live[b] == live[best] && dist(b) < dist(best))) best = b;
    }
    if (cuts.empty() || best > cuts.back()) cuts.push_back(best);
  }
  cuts.push_back(n);
  return cuts;
}
}  // namespace

// the split entry's ring queues are sized from the CTA width (a power of two)
inline bool block_ok(std::uint32_t block) {
  return block >= 64 && block <= 512 && (block & (block - 1)) == 0;
}

template <typename C>
KernelImage emit_ptx(const Stream<C>& stream_in, Domain domain, KernelShape shape,
                     const Tuning& tuning, const Stream<C>* mirror) {
  const bool scalar = domain == Domain::F64 || domain == Domain::F64Strict ||
                      domain == Domain::I64 || domain == Domain::I64F;
  // Long scalar walks are emitted in sections (Emitter::emit_sectioned);
  // ~3k ops per section (profiles/r1_slices_c4.txt: C4 at 4-6 parts of
  // 2-3k records beat the 12.6k-record walk by 22 %).
  const std::size_t target = tuning.section_ops == UINT32_MAX ? 0
                             : tuning.section_ops        ? tuning.section_ops
                                                         : 3000;
  const std::vector<std::size_t> cuts =
      scalar ? section_cuts(stream_in, target) : std::vector<std::size_t>{stream_in.ops.size()};
  // Wide fused programs (power tables > 32 entries, one point per thread:
  // C4's trivariate walk) get the latency-aware reordering: their warps are
  // few (128 registers, most holding powers) and ptxas keeps the walk's
  // order, so 68 % of FP64 ops sat within 4 instructions of their producer
  // (profiles/r1_sched_sweep.txt: C4 3.71 -> 3.50 ms per 4e6 points; the
  // 4-lane C2/C3 kernels have ILP from their lanes and gain nothing).
  Stream<C> scheduled;
  const Stream<C>* sp = &stream_in;
  if (!stream_in.strict && (domain == Domain::F64 || domain == Domain::I64F)) {
    std::size_t W = 0, D = 0;
    if (tuning.sched_window) {
      W = tuning.sched_window;
      D = tuning.sched_distance;
    } else if (stream_in.powers.size() > 32 && (shape.lanes == 0 || shape.lanes == 1)) {
      W = 64;
      D = 8;
    }
    if (W > 1) {
      scheduled = schedule_stream(stream_in, W, D, cuts);
      sp = &scheduled;
    }
  }
  const Stream<C>& stream = *sp;
  std::unordered_map<std::uint64_t, int> distinct;
  for (const auto& c : stream.coefs) {
    std::uint64_t w;
    std::memcpy(&w, &c, 8);
    distinct.emplace(w, 0);
  }
  const KernelShape def = default_shape(domain, static_cast<std::uint32_t>(stream.powers.size()),
                                        distinct.size(), tuning);
  if (shape.lanes == 0) shape.lanes = def.lanes;
  if (shape.block == 0) shape.block = def.block;
  if (shape.sync_every == 0) shape.sync_every = def.sync_every;
  if (shape.min_ctas == 0) shape.min_ctas = def.min_ctas;
  if (shape.limbs == 0) shape.limbs = 1;
  Emitter<C> e(stream, domain, shape, tuning, cuts);
  if (mirror && domain == Domain::Interval && shape.iv_partition == 1 && block_ok(shape.block)) {
    // the one-pass sign split: the mirrored program's point function joins
    // this module under its own constant array
    KernelShape ms = shape;
    ms.iv_partition = 2;
    Emitter<C> eq(*mirror, domain, ms, tuning, {mirror->ops.size()});
    std::string text = eq.point_module("pe_iv_neg", 2, "pe_qcoef");
    if (!text.empty()) e.set_split_funcs(std::move(text), eq.const_words());
  }
  KernelImage img = e.run();
  img.iv_partition_min = tuning.iv_partition_min ? tuning.iv_partition_min : 65536;
  return img;
}

template KernelImage emit_ptx(const Stream<double>&, Domain, KernelShape, const Tuning&,
                              const Stream<double>*);
template KernelImage emit_ptx(const Stream<std::int64_t>&, Domain, KernelShape, const Tuning&,
                              const Stream<std::int64_t>*);

}  // namespace polyeval::lower
