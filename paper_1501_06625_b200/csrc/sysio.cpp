// sysio.cpp -- hex limbs, system files and solution files (host only).
//
//   pt_hex_*                 hexio.hpp:16-24 / hexio.cpp:21-70 restated: 16 hex
//                            digits per binary64 limb, "#(h1 h2 ...)" arrays
//   pt_system_parse          parse_system      SPEC.md:147-152, grammar SPEC.md:197
//   pt_system_serialize      serialize_system
//   pt_solutions_write/read  solutions file
//
// System file grammar:
//   file    := "vars:" name{ name } NL  poly ";" { poly ";" }
//   poly    := [sign] term { sign term }
//   term    := coef [ "*" factor { "*" factor } ] | factor { "*" factor }
//   factor  := name [ "^" exponent ]
//   coef    := decimal | "(" [sign] decimal [ sign decimal "*" "i" ] ")"
//            | "#(" limbs ")" [ "+i#(" limbs ")" ]          (hex_complex, hexio.hpp:36-39)
// Whitespace (including newlines) separates tokens; ';' ends a polynomial.
// Hex coefficients with exactly L limbs are taken bit for bit (the point of
// the hex form); other limb counts go through RealTraits<R>::from_components
// (multiprec.hpp:393,406,421).  Decimal coefficients are strtod in D and
// digit-by-digit in the working precision for DD / QD.
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "inputs.hpp"

using namespace ptgen;

namespace {

constexpr char kHex[] = "0123456789abcdef";

int nib(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

std::string enc(double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  std::string out(16, '0');
  for (int i = 15; i >= 0; --i) {
    out[i] = kHex[b & 0xf];
    b >>= 4;
  }
  return out;
}

// hexio.cpp:34-46; throws std::invalid_argument-equivalent messages
bool dec(std::string_view t, double* v, std::string* err) {
  if (t.size() != 16) {
    *err = "hex limb must be 16 digits";
    return false;
  }
  uint64_t b = 0;
  for (char c : t) {
    const int x = nib(c);
    if (x < 0) {
      *err = "invalid hex digit in limb";
      return false;
    }
    b = (b << 4) | (uint64_t)x;
  }
  std::memcpy(v, &b, 8);
  return true;
}

std::string enc_limbs(const double* l, int n) {  // hexio.cpp:48-56
  std::string out = "#(";
  for (int i = 0; i < n; ++i) {
    if (i) out += ' ';
    out += enc(l[i]);
  }
  return out + ")";
}

// hexio.cpp:58-70
bool dec_limbs(std::string_view t, std::vector<double>* out, std::string* err) {
  if (t.size() < 4 || t.substr(0, 2) != "#(" || t.back() != ')') {
    *err = "hex limb array must look like #(...)";
    return false;
  }
  out->clear();
  size_t i = 2;
  const size_t end = t.size() - 1;
  while (i < end) {
    while (i < end && t[i] == ' ') ++i;
    if (i >= end) break;
    if (end - i < 16) {
      *err = "truncated hex limb";
      return false;
    }
    double v;
    if (!dec(t.substr(i, 16), &v, err)) return false;
    out->push_back(v);
    i += 16;
  }
  if (out->empty()) {
    *err = "empty hex limb array";
    return false;
  }
  return true;
}

// RealTraits<R>::from_components (multiprec.hpp:393,406,421) into L limbs
void from_components(const std::vector<double>& in, int L, double* out) {
  for (int l = 0; l < L; ++l) out[l] = 0.0;
  if ((int)in.size() == L) {  // bit-exact
    for (int l = 0; l < L; ++l) out[l] = in[l];
    return;
  }
  const int cnt = (int)in.size();
  if (L == 1) {
    out[0] = cnt > 0 ? in[0] : 0.0;
  } else if (L == 2) {
    ptk::dd r{0.0, 0.0};
    for (int i = 0; i < cnt && i < 2; ++i) r = ptk::r_add(r, ptk::dd{in[i], 0.0});
    out[0] = r.hi;
    out[1] = r.lo;
  } else {
    double m[4] = {0, 0, 0, 0};
    for (int i = 0; i < cnt && i < 4; ++i) m[i] = in[i];
    ptk::qd q;
    if (cnt <= 1) {
      double a[1] = {m[0]};
      q = ptk::qd_distill<1>(a);
    } else if (cnt == 2) {
      double a[2] = {m[0], m[1]};
      q = ptk::qd_distill<2>(a);
    } else if (cnt == 3) {
      double a[3] = {m[0], m[1], m[2]};
      q = ptk::qd_distill<3>(a);
    } else {
      q = ptk::qd_distill<4>(m);
    }
    for (int l = 0; l < 4; ++l) out[l] = q.c[l];
  }
}

// Decimal text -> L limbs.  D: strtod (correctly rounded).  DD / QD: the
// digits accumulated and scaled by 10^e in the working precision.
template <class R>
void decimal_in(const std::string& s, double* out) {
  using namespace ptk;
  constexpr int L = limbs_of<R>::L;
  bool neg = false;
  size_t i = 0;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  R v = rconst<R>(0.0);
  const R ten = rconst<R>(10.0);
  int e10 = 0;
  bool frac = false;
  for (; i < s.size(); ++i) {
    const char c = s[i];
    if (c == '.') {
      frac = true;
    } else if (c >= '0' && c <= '9') {
      v = r_add(r_mul(v, ten), rconst<R>((double)(c - '0')));
      if (frac) --e10;
    } else {
      break;
    }
  }
  if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) e10 += std::atoi(s.c_str() + i + 1);
  if (e10 > 0) v = r_mul(v, r_powi(ten, (unsigned)e10));
  if (e10 < 0) v = r_div(v, r_powi(ten, (unsigned)(-e10)));
  if (neg) v = r_neg(v);
  for (int l = 0; l < L; ++l) out[l] = r_limb(v, l);
}

void decimal_limbs(const std::string& s, int L, double* out) {
  for (int l = 0; l < L; ++l) out[l] = 0.0;
  if (L == 1) out[0] = std::strtod(s.c_str(), nullptr);
  else if (L == 2) decimal_in<ptk::dd>(s, out);
  else decimal_in<ptk::qd>(s, out);
}

template <class R>
void negate_limbs(double* c, int L) {
  ptk::cplx<R> v;
  for (int l = 0; l < L; ++l) {
    ptk::r_set_limb(v.re, l, c[l]);
    ptk::r_set_limb(v.im, l, c[L + l]);
  }
  v = ptk::c_neg(v);
  for (int l = 0; l < L; ++l) {
    c[l] = ptk::r_limb(v.re, l);
    c[L + l] = ptk::r_limb(v.im, l);
  }
}

// ---------------------------------------------------------------------------
// system-file parser
// ---------------------------------------------------------------------------
class Parser {
 public:
  Parser(std::string_view text, int L) : t_(text), L_(L) {}

  bool run(pt_sysbuf** out) {
    skip_ws();
    if (!lit("vars:")) return err("expected 'vars:' header line");
    // names up to the end of the first line
    while (true) {
      while (pos_ < t_.size() && (t_[pos_] == ' ' || t_[pos_] == '\t' || t_[pos_] == '\r')) adv();
      if (pos_ >= t_.size() || t_[pos_] == '\n') break;
      const size_t l0 = line_, c0 = col_;
      std::string nm = ident();
      if (nm.empty()) return err("bad variable name in 'vars:' line");
      if (nm == "i") return err_at(l0, c0, "'i' is the imaginary unit, not a variable name");
      if (names_.count(nm)) return err_at(l0, c0, "duplicate variable '" + nm + "'");
      const int idx = (int)names_.size();
      names_[nm] = idx;
    }
    if (names_.empty()) return err("no variables declared");
    std::vector<std::vector<Term>> eqs;
    while (true) {
      skip_ws();
      if (pos_ >= t_.size()) break;
      std::vector<Term> e;
      if (!poly(&e)) return false;
      eqs.push_back(std::move(e));
    }
    if (eqs.empty()) return err("empty polynomial list");
    canonicalize(eqs, L_);
    *out = emit((int)names_.size(), eqs, L_);
    return true;
  }

  std::string msg;

 private:
  std::string_view t_;
  int L_;
  size_t pos_ = 0, line_ = 1, col_ = 1;
  std::map<std::string, int> names_;

  void adv() {
    if (t_[pos_] == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    ++pos_;
  }
  void skip_ws() {
    while (pos_ < t_.size() && std::isspace((unsigned char)t_[pos_])) adv();
  }
  bool lit(std::string_view s) {
    if (t_.substr(pos_, s.size()) != s) return false;
    for (size_t k = 0; k < s.size(); ++k) adv();
    return true;
  }
  char peek() const { return pos_ < t_.size() ? t_[pos_] : '\0'; }
  bool err(const std::string& m) { return err_at(line_, col_, m); }
  bool err_at(size_t l, size_t c, const std::string& m) {
    msg = "line " + std::to_string(l) + ", column " + std::to_string(c) + ": " + m;
    return false;
  }
  std::string ident() {
    std::string s;
    if (pos_ < t_.size() && (std::isalpha((unsigned char)t_[pos_]) || t_[pos_] == '_')) {
      while (pos_ < t_.size() && (std::isalnum((unsigned char)t_[pos_]) || t_[pos_] == '_')) {
        s += t_[pos_];
        adv();
      }
    }
    return s;
  }
  std::string number() {  // decimal literal (no sign)
    std::string s;
    auto digits = [&]() {
      while (pos_ < t_.size() && std::isdigit((unsigned char)t_[pos_])) {
        s += t_[pos_];
        adv();
      }
    };
    digits();
    if (peek() == '.') {
      s += '.';
      adv();
      digits();
    }
    if (!s.empty() && (peek() == 'e' || peek() == 'E')) {
      const size_t save = pos_, sl = line_, sc = col_;
      std::string e = "e";
      adv();
      if (peek() == '+' || peek() == '-') {
        e += peek();
        adv();
      }
      if (std::isdigit((unsigned char)peek())) {
        s += e;
        digits();
      } else {
        pos_ = save;
        line_ = sl;
        col_ = sc;
      }
    }
    if (s == ".") s.clear();
    return s;
  }
  bool hex_real(double* out) {
    const size_t l0 = line_, c0 = col_;
    const size_t a = pos_;
    while (pos_ < t_.size() && t_[pos_] != ')') adv();
    if (pos_ >= t_.size()) return err_at(l0, c0, "unterminated hex limb array");
    adv();
    std::vector<double> limbs;
    std::string e;
    if (!dec_limbs(t_.substr(a, pos_ - a), &limbs, &e)) return err_at(l0, c0, e);
    from_components(limbs, L_, out);
    return true;
  }
  // coefficient -> c (2L limbs); true when one was read
  bool coef(double* c, bool* have) {
    *have = false;
    for (int q = 0; q < 2 * L_; ++q) c[q] = 0.0;
    if (peek() == '#') {
      if (!hex_real(c)) return false;
      if (lit("+i")) {
        if (peek() != '#') return err("expected '#(' after '+i'");
        if (!hex_real(c + L_)) return false;
      }
      *have = true;
      return true;
    }
    if (peek() == '(') {
      adv();
      skip_ws();
      bool neg = false;
      if (peek() == '+' || peek() == '-') {
        neg = peek() == '-';
        adv();
        skip_ws();
      }
      std::string re = number();
      if (re.empty()) return err("expected a number");
      decimal_limbs((neg ? "-" : "") + re, L_, c);
      skip_ws();
      if (peek() == '+' || peek() == '-') {
        const bool ineg = peek() == '-';
        adv();
        skip_ws();
        std::string im = number();
        if (im.empty()) return err("expected the imaginary part");
        skip_ws();
        if (!lit("*")) return err("expected '*i'");
        skip_ws();
        if (!lit("i")) return err("expected 'i'");
        decimal_limbs((ineg ? "-" : "") + im, L_, c + L_);
        skip_ws();
      }
      if (!lit(")")) return err("expected ')'");
      *have = true;
      return true;
    }
    if (std::isdigit((unsigned char)peek()) || peek() == '.') {
      std::string re = number();
      if (re.empty()) return err("bad number");
      decimal_limbs(re, L_, c);
      *have = true;
    }
    return true;
  }
  bool factor(std::map<int, int>* ex) {
    const size_t l0 = line_, c0 = col_;
    std::string nm = ident();
    if (nm.empty()) return err("expected a variable");
    auto it = names_.find(nm);
    if (it == names_.end()) {
      bool xdig = nm.size() > 1 && nm[0] == 'x';
      for (size_t k = 1; k < nm.size() && xdig; ++k) xdig = std::isdigit((unsigned char)nm[k]);
      return err_at(l0, c0, xdig ? "variable index out of range: " + nm : "unknown variable '" + nm + "'");
    }
    int e = 1;
    skip_ws();
    if (peek() == '^') {
      adv();
      skip_ws();
      std::string d;
      while (std::isdigit((unsigned char)peek())) {
        d += peek();
        adv();
      }
      if (d.empty()) return err("expected an exponent");
      e = std::atoi(d.c_str());
      if (e < 1) return err("exponent must be >= 1");
    }
    (*ex)[it->second] += e;
    return true;
  }
  bool term(bool neg, Term* out) {
    std::memset(out->c, 0, sizeof out->c);
    bool have = false;
    if (!coef(out->c, &have)) return false;
    std::map<int, int> ex;
    skip_ws();
    if (have) {
      while (peek() == '*') {
        adv();
        skip_ws();
        if (!factor(&ex)) return false;
        skip_ws();
      }
    } else {
      out->c[0] = 1.0;  // implicit unit coefficient
      if (!factor(&ex)) return false;
      skip_ws();
      while (peek() == '*') {
        adv();
        skip_ws();
        if (!factor(&ex)) return false;
        skip_ws();
      }
    }
    if (neg) {
      if (L_ == 1) negate_limbs<double>(out->c, 1);
      else if (L_ == 2) negate_limbs<ptk::dd>(out->c, 2);
      else negate_limbs<ptk::qd>(out->c, 4);
    }
    out->sup.assign(ex.begin(), ex.end());
    return true;
  }
  bool poly(std::vector<Term>* e) {
    bool first = true;
    while (true) {
      skip_ws();
      if (peek() == ';') {
        if (first) return err("empty polynomial");
        adv();
        return true;
      }
      if (pos_ >= t_.size()) return err("missing ';' at the end of the polynomial");
      bool neg = false;
      if (peek() == '+' || peek() == '-') {
        neg = peek() == '-';
        adv();
        skip_ws();
      } else if (!first) {
        return err("expected '+', '-' or ';'");
      }
      Term tm;
      if (!term(neg, &tm)) return false;
      e->push_back(std::move(tm));
      first = false;
    }
  }
};

char* dup_text(const std::string& s) {
  char* p = (char*)std::malloc(s.size() + 1);
  if (p) std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// tokenizer for solution files: whitespace separates tokens, except inside
// a "#(...)" array (a complex is "#(...)+i#(...)")
std::vector<std::pair<std::string, int>> tokens(std::string_view t) {
  std::vector<std::pair<std::string, int>> out;
  size_t i = 0;
  int line = 1;
  while (i < t.size()) {
    if (std::isspace((unsigned char)t[i])) {
      if (t[i] == '\n') ++line;
      ++i;
      continue;
    }
    std::string tok;
    const int l0 = line;
    int depth = 0;
    while (i < t.size() && (depth > 0 || !std::isspace((unsigned char)t[i]))) {
      if (t[i] == '(') ++depth;
      if (t[i] == ')') --depth;
      if (t[i] == '\n') ++line;
      tok += t[i++];
    }
    out.push_back({tok, l0});
  }
  return out;
}

const char* prec_name(pt_prec p) { return p == PT_D ? "d" : (p == PT_DD ? "dd" : "qd"); }

}  // namespace

extern "C" {

int pt_hex_encode_limb(double value, char* out) {
  if (!out) return fail(PT_E_INVAL, "null output");
  const std::string s = enc(value);
  std::memcpy(out, s.c_str(), 17);
  return PT_OK;
}

int pt_hex_decode_limb(const char* text, int32_t len, double* out) {
  if (!text || !out || len < 0) return fail(PT_E_INVAL, "null argument");
  std::string e;
  if (!dec(std::string_view(text, (size_t)len), out, &e)) return fail(PT_E_INVAL, e);
  return PT_OK;
}

int pt_hex_limbs(const double* limbs, int32_t count, char** out) {
  if (!limbs || !out || count < 0) return fail(PT_E_INVAL, "null argument");
  *out = dup_text(enc_limbs(limbs, count));
  return *out ? PT_OK : fail(PT_E_NOMEM, "out of memory");
}

int pt_parse_hex_limbs(const char* text, int32_t len, double* out, int32_t cap, int32_t* count) {
  if (!text || !count || len < 0) return fail(PT_E_INVAL, "null argument");
  std::vector<double> v;
  std::string e;
  if (!dec_limbs(std::string_view(text, (size_t)len), &v, &e)) return fail(PT_E_INVAL, e);
  *count = (int32_t)v.size();
  for (int i = 0; i < (int)v.size() && i < cap && out; ++i) out[i] = v[i];
  return PT_OK;
}

int pt_system_parse(const char* text, pt_prec prec, pt_sysbuf** out) {
  if (!text || !out) return fail(PT_E_INVAL, "null argument");
  if (prec != PT_D && prec != PT_DD && prec != PT_QD) return fail(PT_E_INVAL, "bad precision");
  Parser p(text, limbs(prec));
  if (!p.run(out)) return fail(PT_E_INVAL, p.msg);
  return PT_OK;
}

int pt_system_serialize(const pt_system_desc* s, pt_prec prec, char** out) {
  if (!s || !out) return fail(PT_E_INVAL, "null argument");
  const int L = limbs(prec);
  std::string o = "vars:";
  for (int v = 0; v < s->n_vars; ++v) o += " x" + std::to_string(v);
  o += "\n";
  const long T = s->n_terms;
  for (int i = 0; i < s->n_eqs; ++i) {
    bool first = true;
    for (int t = s->eq_ptr[i]; t < s->eq_ptr[i + 1]; ++t) {
      double re[4], im[4];
      for (int l = 0; l < L; ++l) {
        re[l] = s->coef[(size_t)l * T + t];
        im[l] = s->coef[(size_t)(L + l) * T + t];
      }
      if (!first) o += " + ";
      first = false;
      o += enc_limbs(re, L) + "+i" + enc_limbs(im, L);
      for (int q = s->term_ptr[t]; q < s->term_ptr[t + 1]; ++q) {
        if (s->var[q] < 0 || s->var[q] >= s->n_vars) return fail(PT_E_INVAL, "variable index out of range");
        o += "*x" + std::to_string(s->var[q]);
        if (s->exp[q] != 1) o += "^" + std::to_string(s->exp[q]);
      }
    }
    if (first) o += "0";  // the zero polynomial (all terms cancelled)
    o += ";\n";
  }
  *out = dup_text(o);
  return *out ? PT_OK : fail(PT_E_NOMEM, "out of memory");
}

// solutions <count> dim <n> precision <d|dd|qd>
// then per record:  solution <r> t #(..) residual #(..) update #(..)
//                   x<j> #(re limbs)+i#(im limbs)      (j = 0..n-1)
int pt_solutions_write(int32_t n, pt_prec prec, int32_t count, const double* t, const double* points,
                       const double* residual, const double* update, char** out) {
  if (!out || n < 0 || count < 0 || (count > 0 && (!t || !points || !residual || !update)))
    return fail(PT_E_INVAL, "bad solution arguments");
  const int L = limbs(prec);
  std::string o = "solutions " + std::to_string(count) + " dim " + std::to_string(n) + " precision " +
                  prec_name(prec) + "\n";
  for (int r = 0; r < count; ++r) {
    o += "solution " + std::to_string(r) + " t " + enc_limbs(t + r, 1) + " residual " + enc_limbs(residual + r, 1) +
         " update " + enc_limbs(update + r, 1) + "\n";
    const double* x = points + (size_t)r * 2 * L * n;
    for (int j = 0; j < n; ++j) {
      double re[4], im[4];
      for (int l = 0; l < L; ++l) {
        re[l] = x[(size_t)l * n + j];
        im[l] = x[(size_t)(L + l) * n + j];
      }
      o += "x" + std::to_string(j) + " " + enc_limbs(re, L) + "+i" + enc_limbs(im, L) + "\n";
    }
  }
  *out = dup_text(o);
  return *out ? PT_OK : fail(PT_E_NOMEM, "out of memory");
}

int pt_solutions_read(const char* text, pt_prec prec, int32_t cap, int32_t* count, int32_t* n, double* t,
                      double* points, double* residual, double* update) {
  if (!text || !count || !n) return fail(PT_E_INVAL, "null argument");
  const int L = limbs(prec);
  auto tk = tokens(text);
  size_t k = 0;
  auto bad = [&](const std::string& m) {
    const int line = k < tk.size() ? tk[k].second : (tk.empty() ? 1 : tk.back().second);
    return fail(PT_E_INVAL, "line " + std::to_string(line) + ": " + m);
  };
  auto expect = [&](const char* w) { return k < tk.size() && tk[k].first == w ? (++k, true) : false; };
  auto integer = [&](long* v) {
    if (k >= tk.size()) return false;
    char* end = nullptr;
    *v = std::strtol(tk[k].first.c_str(), &end, 10);
    if (!end || *end) return false;
    ++k;
    return true;
  };
  long cnt = 0, dim = 0;
  if (!expect("solutions") || !integer(&cnt)) return bad("expected 'solutions <count>'");
  if (!expect("dim") || !integer(&dim)) return bad("expected 'dim <n>'");
  if (!expect("precision") || k >= tk.size()) return bad("expected 'precision <d|dd|qd>'");
  ++k;
  if (cnt < 0 || dim < 0) return bad("negative count or dimension");
  *count = (int32_t)cnt;
  *n = (int32_t)dim;
  if (!points) return PT_OK;
  std::string e;
  std::vector<double> limbs;
  auto real1 = [&](double* out) {
    if (k >= tk.size() || !dec_limbs(tk[k].first, &limbs, &e)) return false;
    ++k;
    *out = limbs[0];
    return true;
  };
  for (long r = 0; r < cnt; ++r) {
    long idx = -1;
    if (!expect("solution") || !integer(&idx) || idx != r) return bad("expected 'solution " + std::to_string(r) + "'");
    double tv, rv, uv;
    if (!expect("t") || !real1(&tv)) return bad("expected 't #(...)'" + (e.empty() ? "" : ": " + e));
    if (!expect("residual") || !real1(&rv)) return bad("expected 'residual #(...)'");
    if (!expect("update") || !real1(&uv)) return bad("expected 'update #(...)'");
    const bool store = r < cap;
    if (store) {
      t[r] = tv;
      residual[r] = rv;
      update[r] = uv;
    }
    double* x = points + (size_t)r * 2 * L * dim;
    for (long j = 0; j < dim; ++j) {
      if (!expect(("x" + std::to_string(j)).c_str())) return bad("expected 'x" + std::to_string(j) + "'");
      if (k >= tk.size()) return bad("missing component");
      const std::string& z = tk[k].first;
      const size_t plus = z.find(")+i#(");
      if (plus == std::string::npos) return bad("component must be #(...)+i#(...)");
      double re[4], im[4];
      if (!dec_limbs(std::string_view(z).substr(0, plus + 1), &limbs, &e)) return bad(e);
      from_components(limbs, L, re);
      if (!dec_limbs(std::string_view(z).substr(plus + 3), &limbs, &e)) return bad(e);
      from_components(limbs, L, im);
      ++k;
      if (store)
        for (int l = 0; l < L; ++l) {
          x[(size_t)l * dim + j] = re[l];
          x[(size_t)(L + l) * dim + j] = im[l];
        }
    }
  }
  if (k != tk.size()) return bad("trailing text after the last solution");
  return PT_OK;
}

}  // extern "C"
