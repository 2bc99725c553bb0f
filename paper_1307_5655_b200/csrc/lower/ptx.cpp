// PTX emitter: lowered stream -> sm_100a kernel text.
//
// Thread i evaluates point i (SoA coordinates, one coalesced 8-byte load per
// variable per thread). The power DAG and the walk are straight-line code over
// PTX virtual registers; ptxas performs the physical register allocation,
// which is exactly the job the reference's lazy heights do for its heap
// register file (tree.hpp:68-77). Per-domain arithmetic:
//   F64 / F64Strict  add.rn / mul.rn / fma.rn (strict streams contain no FMA,
//                    and .rn instructions are never contracted by ptxas)
//   I64              add.s64 / mul.lo.s64 / mad.lo.s64 (wrap-free: the host
//                    proves the range, the kernel checks |x| <= bound)
//   Interval         reference interval.cpp:12-52 verbatim: RN op, then one
//                    nextafter step outward per endpoint; products use the
//                    zero rule and the std::min/std::max({p1..p4}) scan order.
#include "lower/ptx.hpp"

#include <cmath>
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
  }
  return "?";
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

/// Interval injection of a coefficient (reference numeric.cpp:17-26 for
/// integers; fp64 coefficients are exact points).
struct IvCoef {
  double lo, hi;
};
IvCoef inject(double c) { return {c, c}; }
IvCoef inject(std::int64_t c) {
  const double d = static_cast<double>(c);  // round-to-nearest-even
  const bool exact = d < 9223372036854775808.0 && d >= -9223372036854775808.0 &&
                     static_cast<std::int64_t>(d) == c;
  if (exact) return {d, d};
  return {std::nextafter(d, -std::numeric_limits<double>::infinity()),
          std::nextafter(d, std::numeric_limits<double>::infinity())};
}

template <typename C>
class Emitter {
 public:
  Emitter(const Stream<C>& s, Domain d) : s_(s), d_(d) {}

  KernelImage run() {
    KernelImage img;
    img.domain = d_;
    img.nvars = s_.nvars;
    const bool iv = d_ == Domain::Interval;
    const bool i64 = d_ == Domain::I64;
    img.n_in = iv ? 2 * s_.nvars : s_.nvars;
    img.n_out = iv ? 2 : 1;
    img.has_flag = iv || i64;
    img.has_bounds = i64;
    if ((d_ == Domain::F64Strict || d_ == Domain::Interval) && !s_.strict) {
      throw std::logic_error("strict domain needs a strict stream");
    }

    assign_words();
    img.const_words = n_const_;
    img.param_words.assign(words_.begin() + n_const_, words_.begin() + n_const_ + n_param_);
    img.global_words.assign(words_.begin() + n_const_ + n_param_, words_.end());

    body_.str("");
    emit_prologue();
    emit_powers();
    emit_walk();
    emit_epilogue();

    std::ostringstream m;
    img.entry = std::string("pe_walk_") + domain_name(d_);
    m << "//\n// polyeval-b200 generated kernel: domain=" << domain_name(d_)
      << " nvars=" << s_.nvars << " ops=" << s_.ops.size()
      << " powers=" << s_.powers.size() << "\n//\n";
    m << ".version 8.7\n.target sm_100a\n.address_size 64\n\n";
    if (n_const_ > 0) {
      m << ".const .align 8 .b64 pe_coef[" << n_const_ << "] = {";
      for (std::uint32_t i = 0; i < n_const_; ++i) {
        if (i) m << (i % 8 == 0 ? ",\n  " : ", ");
        m << hex64(words_[i]);
      }
      m << "};\n\n";
    }
    m << ".visible .entry " << img.entry << "(";
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
    if (n_param_ > 0) param(".param .align 8 .b8 pe_pcoef[" + std::to_string(8 * n_param_) + "]");
    m << ")\n.maxntid " << img.block << ", 1, 1\n{\n";
    m << "  .reg .pred %p<8>;\n  .reg .b32 %r<8>;\n  .reg .b64 %rd<24>;\n";
    m << decls_.str();
    m << body_.str();
    m << "}\n";
    img.ptx = m.str();
    img.fp_ops = fp_ops_;
    img.int_ops = int_ops_;
    img.hash = fnv1a(img.ptx.data(), img.ptx.size());
    return img;
  }

 private:
  // ---------------- coefficient words ----------------
  void assign_words() {
    // word table: f64/i64 one word per coefficient slot; interval lo/hi,
    // shared when equal.
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
    for (std::size_t k = 0; k < s_.coefs.size(); ++k) {
      if (d_ == Domain::Interval) {
        const IvCoef c = inject(s_.coefs[k]);
        coef_lo_[k] = word(bits_of(c.lo));
        coef_hi_[k] = word(bits_of(c.hi));
      } else if (d_ == Domain::I64) {
        std::uint64_t w;
        if constexpr (std::is_same_v<C, std::int64_t>) {
          w = static_cast<std::uint64_t>(s_.coefs[k]);
        } else {
          throw std::invalid_argument("int64 domain needs integer coefficients");
        }
        coef_lo_[k] = coef_hi_[k] = word(w);
      } else {
        const double c = static_cast<double>(s_.coefs[k]);
        coef_lo_[k] = coef_hi_[k] = word(bits_of(c));
      }
    }
    const auto n = static_cast<std::uint32_t>(words_.size());
    n_const_ = std::min(n, CoefTiers::kConstCap);
    n_param_ = std::min(n - n_const_, CoefTiers::kParamCap);
    n_global_ = n - n_const_ - n_param_;
  }

  const char* ty() const { return d_ == Domain::I64 ? "s64" : "f64"; }
  const char* ldty() const { return d_ == Domain::I64 ? "b64" : "f64"; }

  // Loads coefficient word w into a fresh register, returns its name.
  std::string load_word(std::uint32_t w) {
    std::string r = "%c" + std::to_string(n_creg_++);
    if (w < n_const_) {
      body_ << "  ld.const." << ldty() << " " << r << ", [pe_coef+" << 8 * w << "];\n";
    } else if (w < n_const_ + n_param_) {
      body_ << "  ld.param." << ldty() << " " << r << ", [pe_pcoef+" << 8 * (w - n_const_) << "];\n";
    } else {
      body_ << "  ld.global.nc." << ldty() << " " << r << ", [%rd20+" << 8 * (w - n_const_ - n_param_)
            << "];\n";
    }
    return r;
  }

  // ---------------- operands ----------------
  std::string reg(std::uint32_t id, bool hi = false) const {
    if (d_ == Domain::Interval) return (hi ? "%vh" : "%vl") + std::to_string(id);
    return "%v" + std::to_string(id);
  }
  std::string pw(std::uint32_t id, bool hi = false) const {
    if (d_ == Domain::Interval) return (hi ? "%ph" : "%pl") + std::to_string(id);
    return "%q" + std::to_string(id);
  }
  // scalar operand text (f64 / i64)
  std::string opnd(const Operand& o) {
    switch (o.kind) {
      case Operand::Reg: return reg(o.id);
      case Operand::Pow: return pw(o.id);
      case Operand::Coef: return load_word(coef_lo_[o.id]);
      case Operand::Zero: return d_ == Domain::I64 ? "0" : "0d0000000000000000";
      default: throw std::logic_error("bad operand");
    }
  }
  // interval operand: pair of register texts
  std::pair<std::string, std::string> iv(const Operand& o) {
    switch (o.kind) {
      case Operand::Reg: return {reg(o.id, false), reg(o.id, true)};
      case Operand::Pow: return {pw(o.id, false), pw(o.id, true)};
      case Operand::Coef: {
        const std::string lo = load_word(coef_lo_[o.id]);
        const std::string hi =
            coef_hi_[o.id] == coef_lo_[o.id] ? lo : load_word(coef_hi_[o.id]);
        return {lo, hi};
      }
      case Operand::Zero: return {"0d0000000000000000", "0d0000000000000000"};
      default: throw std::logic_error("bad operand");
    }
  }

  // ---------------- frame ----------------
  void emit_prologue() {
    const bool iv = d_ == Domain::Interval;
    const std::uint32_t nin = iv ? 2 * s_.nvars : s_.nvars;
    // thread -> point
    body_ << "  mov.u32 %r1, %ctaid.x;\n  mov.u32 %r2, %ntid.x;\n  mov.u32 %r3, %tid.x;\n"
          << "  mul.wide.u32 %rd1, %r1, %r2;\n  cvt.u64.u32 %rd2, %r3;\n"
          << "  add.u64 %rd1, %rd1, %rd2;\n  ld.param.u64 %rd3, [pe_n];\n"
          << "  setp.ge.u64 %p1, %rd1, %rd3;\n  @%p1 bra $Ldone;\n"
          << "  shl.b64 %rd4, %rd1, 3;\n";
    if (n_global_ > 0) {
      body_ << "  ld.param.u64 %rd20, [pe_gcoef];\n  cvta.to.global.u64 %rd20, %rd20;\n";
    }
    // coordinates (SoA): one coalesced 8-byte load per variable (per endpoint)
    for (std::uint32_t i = 0; i < nin; ++i) {
      std::string dst;
      if (iv) {
        dst = (i % 2 == 0 ? "%xl" : "%xh") + std::to_string(i / 2);
      } else {
        dst = "%x" + std::to_string(i);
      }
      body_ << "  ld.param.u64 %rd5, [pe_in" << i << "];\n  cvta.to.global.u64 %rd5, %rd5;\n"
            << "  add.u64 %rd5, %rd5, %rd4;\n  ld.global.nc." << ldty() << " " << dst
            << ", [%rd5];\n";
    }
    if (iv) {
      decls_ << "  .reg .f64 %xl<" << s_.nvars << ">, %xh<" << s_.nvars << ">;\n";
      // Reference Interval(lo, hi) rejects NaN endpoints and lo > hi
      // (interval.cpp:21-26): flag and continue, the host reports EINVAL.
      for (std::uint32_t v = 0; v < s_.nvars; ++v) {
        body_ << "  setp.le.f64 %p2, %xl" << v << ", %xh" << v << ";\n"
              << "  @%p2 bra $Lok" << v << ";\n"
              << "  ld.param.u64 %rd6, [pe_flag];\n  cvta.to.global.u64 %rd6, %rd6;\n"
              << "  st.global.u32 [%rd6], 2;\n$Lok" << v << ":\n";
      }
    } else {
      decls_ << "  .reg ." << (d_ == Domain::I64 ? "b64" : "f64") << " %x<" << s_.nvars
             << ">;\n";
    }
    if (d_ == Domain::I64) {
      // |x_v| <= bound_v, the range the host overflow proof assumed
      for (std::uint32_t v = 0; v < s_.nvars; ++v) {
        body_ << "  ld.param.u64 %rd7, [pe_bound" << v << "];\n"
              << "  abs.s64 %rd8, %x" << v << ";\n"
              << "  setp.gt.u64 %p2, %rd8, %rd7;\n"
              << "  @!%p2 bra $Lbok" << v << ";\n"
              << "  ld.param.u64 %rd6, [pe_flag];\n  cvta.to.global.u64 %rd6, %rd6;\n"
              << "  st.global.u32 [%rd6], 1;\n$Lbok" << v << ":\n";
      }
    }
  }

  void emit_powers() {
    const std::size_t np = s_.powers.size();
    if (np == 0) return;
    if (d_ == Domain::Interval) {
      decls_ << "  .reg .f64 %pl<" << np << ">, %ph<" << np << ">;\n";
    } else {
      decls_ << "  .reg ." << (d_ == Domain::I64 ? "s64" : "f64") << " %q<" << np << ">;\n";
    }
    for (std::size_t i = 0; i < np; ++i) {
      const Power& p = s_.powers[i];
      if (p.exponent == 1) {
        if (d_ == Domain::Interval) {
          body_ << "  mov.f64 %pl" << i << ", %xl" << p.var << ";\n  mov.f64 %ph" << i << ", %xh"
                << p.var << ";\n";
        } else {
          body_ << "  mov." << (d_ == Domain::I64 ? "b64" : "f64") << " %q" << i << ", %x" << p.var
                << ";\n";
        }
        continue;
      }
      if (d_ == Domain::Interval) {
        iv_mul(pw(static_cast<std::uint32_t>(i), false), pw(static_cast<std::uint32_t>(i), true),
               {pw(p.lo, false), pw(p.lo, true)}, {pw(p.hi, false), pw(p.hi, true)});
      } else if (d_ == Domain::I64) {
        body_ << "  mul.lo.s64 %q" << i << ", %q" << p.lo << ", %q" << p.hi << ";\n";
        ++int_ops_;
      } else {
        body_ << "  mul.rn.f64 %q" << i << ", %q" << p.lo << ", %q" << p.hi << ";\n";
        ++fp_ops_;
      }
    }
  }

  void emit_walk() {
    if (s_.nregs > 0) {
      if (d_ == Domain::Interval) {
        decls_ << "  .reg .f64 %vl<" << s_.nregs << ">, %vh<" << s_.nregs << ">;\n";
      } else {
        decls_ << "  .reg ." << ty() << " %v<" << s_.nregs << ">;\n";
      }
    }
    for (const Op& op : s_.ops) {
      if (d_ == Domain::Interval) {
        emit_iv_op(op);
      } else {
        emit_scalar_op(op);
      }
    }
  }

  void emit_scalar_op(const Op& op) {
    const std::string d = reg(op.dst);
    if (d_ == Domain::I64) {
      switch (op.kind) {
        case OpKind::Add: {
          if (op.a.is(Operand::Zero)) {
            body_ << "  mov.b64 " << d << ", " << opnd(op.b) << ";\n";
          } else {
            const std::string a = opnd(op.a), b = opnd(op.b);
            body_ << "  add.s64 " << d << ", " << a << ", " << b << ";\n";
            ++int_ops_;
          }
          break;
        }
        case OpKind::Mul: {
          const std::string a = opnd(op.a), b = opnd(op.b);
          body_ << "  mul.lo.s64 " << d << ", " << a << ", " << b << ";\n";
          ++int_ops_;
          break;
        }
        case OpKind::Fma: {
          const std::string a = opnd(op.a), b = opnd(op.b), c = opnd(op.c);
          body_ << "  mad.lo.s64 " << d << ", " << a << ", " << b << ", " << c << ";\n";
          ++int_ops_;
          break;
        }
      }
      return;
    }
    switch (op.kind) {
      case OpKind::Add: {
        const std::string a = opnd(op.a), b = opnd(op.b);
        body_ << "  add.rn.f64 " << d << ", " << a << ", " << b << ";\n";
        break;
      }
      case OpKind::Mul: {
        const std::string a = opnd(op.a), b = opnd(op.b);
        body_ << "  mul.rn.f64 " << d << ", " << a << ", " << b << ";\n";
        break;
      }
      case OpKind::Fma: {
        const std::string a = opnd(op.a), b = opnd(op.b), c = opnd(op.c);
        body_ << "  fma.rn.f64 " << d << ", " << a << ", " << b << ", " << c << ";\n";
        break;
      }
    }
    ++fp_ops_;
  }

  // ---------------- interval primitives ----------------
  std::string tmp_f() {
    std::string r = "%tf" + std::to_string(n_tf_++);
    return r;
  }
  std::string tmp_u() { return "%tu" + std::to_string(n_tu_++); }
  std::string tmp_p() { return "%tp" + std::to_string(n_tp_++); }

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
              const std::pair<std::string, std::string>& b, bool a_is_zero) {
    if (a_is_zero) {
      // 0.0 + v == v up to the sign of zero, and nextafter maps +-0 alike
      next(dlo, b.first, false);
      next(dhi, b.second, true);
    } else {
      const std::string lo = tmp_f(), hi = tmp_f();
      body_ << "  add.rn.f64 " << lo << ", " << a.first << ", " << b.first << ";\n"
            << "  add.rn.f64 " << hi << ", " << a.second << ", " << b.second << ";\n";
      fp_ops_ += 2;
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
    fp_ops_ += 1;
    return r;
  }

  // interval_mul (reference interval.cpp:43-52): hull of the four products in
  // std::min / std::max initializer-list scan order, then one step outward.
  void iv_mul(const std::string& dlo, const std::string& dhi,
              const std::pair<std::string, std::string>& a,
              const std::pair<std::string, std::string>& b) {
    const std::string p1 = eprod(a.first, b.first), p2 = eprod(a.first, b.second),
                      p3 = eprod(a.second, b.first), p4 = eprod(a.second, b.second);
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

  void emit_iv_op(const Op& op) {
    const std::string dlo = reg(op.dst, false), dhi = reg(op.dst, true);
    switch (op.kind) {
      case OpKind::Add:
        iv_add(dlo, dhi, iv(op.a), iv(op.b), op.a.is(Operand::Zero));
        break;
      case OpKind::Mul:
        iv_mul(dlo, dhi, iv(op.a), iv(op.b));
        break;
      case OpKind::Fma:
        throw std::logic_error("interval streams are strict (no FMA)");
    }
  }

  void emit_epilogue() {
    const bool iv = d_ == Domain::Interval;
    if (iv) {
      std::pair<std::string, std::string> r = this->iv(s_.result);
      body_ << "  ld.param.u64 %rd9, [pe_out0];\n  cvta.to.global.u64 %rd9, %rd9;\n"
            << "  add.u64 %rd9, %rd9, %rd4;\n  st.global.f64 [%rd9], " << r.first << ";\n"
            << "  ld.param.u64 %rd10, [pe_out1];\n  cvta.to.global.u64 %rd10, %rd10;\n"
            << "  add.u64 %rd10, %rd10, %rd4;\n  st.global.f64 [%rd10], " << r.second << ";\n";
    } else {
      const std::string r = opnd(s_.result);
      body_ << "  ld.param.u64 %rd9, [pe_out0];\n  cvta.to.global.u64 %rd9, %rd9;\n"
            << "  add.u64 %rd9, %rd9, %rd4;\n  st.global." << ldty() << " [%rd9], " << r << ";\n";
    }
    body_ << "$Ldone:\n  ret;\n";
    if (n_creg_ > 0) decls_ << "  .reg ." << ldty() << " %c<" << n_creg_ << ">;\n";
    if (n_tf_ > 0) decls_ << "  .reg .f64 %tf<" << n_tf_ << ">;\n";
    if (n_tu_ > 0) decls_ << "  .reg .b64 %tu<" << n_tu_ << ">;\n";
    if (n_tp_ > 0) decls_ << "  .reg .pred %tp<" << n_tp_ << ">;\n";
  }

  const Stream<C>& s_;
  Domain d_;
  std::vector<std::uint64_t> words_;
  std::vector<std::uint32_t> coef_lo_, coef_hi_;
  std::uint32_t n_const_ = 0, n_param_ = 0, n_global_ = 0;
  std::uint32_t n_creg_ = 0, n_tf_ = 0, n_tu_ = 0, n_tp_ = 0;
  std::uint64_t fp_ops_ = 0, int_ops_ = 0;
  std::ostringstream body_, decls_;
};

}  // namespace

template <typename C>
KernelImage emit_ptx(const Stream<C>& stream, Domain domain) {
  Emitter<C> e(stream, domain);
  return e.run();
}

template KernelImage emit_ptx(const Stream<double>&, Domain);
template KernelImage emit_ptx(const Stream<std::int64_t>&, Domain);

}  // namespace polyeval::lower
