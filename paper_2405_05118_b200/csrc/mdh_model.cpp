#include "mdh_model.hpp"

#include <algorithm>
#include <cctype>
#include <deque>
#include <mutex>
#include <set>

#include "json.hpp"

namespace mdhb {

void fail(const std::string& code, const std::string& msg) { throw Error(code, msg); }

std::string ty_name(Ty t) { return t == Ty::I64 ? "i64" : "f64"; }

namespace {
const char kIdx[] = "ijklmnopqrstuvw";  // positional index names (views.cpp:11)
int idx_dim(char c) {
  for (int d = 0; kIdx[d]; ++d)
    if (kIdx[d] == c) return d + 1;
  return 0;
}
}  // namespace

// ---------------------------------------------------------------- affine
int64_t Affine::lo(const std::vector<int64_t>& n) const {
  int64_t v = c0;
  for (size_t d = 0; d < coeff.size(); ++d) v += coeff[d] < 0 ? coeff[d] * (n[d] - 1) : 0;
  return v;
}
int64_t Affine::hi(const std::vector<int64_t>& n) const {
  int64_t v = c0;
  for (size_t d = 0; d < coeff.size(); ++d) v += coeff[d] > 0 ? coeff[d] * (n[d] - 1) : 0;
  return v;
}

// Grammar of views.cpp:45-99: term := INT ['*' NAME] | NAME ['*' INT], joined by +/-.
Affine Affine::parse(const std::string& s, int D) {
  Affine a;
  a.coeff.assign(static_cast<size_t>(D), 0);
  size_t p = 0;
  auto sp = [&] { while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p; };
  auto bad = [&](const std::string& m) {
    fail("ParseError", m + " at column " + std::to_string(p + 1) + " in index expression '" + s + "'");
  };
  auto integer = [&] {
    int64_t k = 0;
    while (p < s.size() && std::isdigit(static_cast<unsigned char>(s[p]))) k = k * 10 + (s[p++] - '0');
    return k;
  };
  for (bool first = true;; first = false) {
    sp();
    if (p >= s.size()) {
      if (first) bad("empty index expression");
      break;
    }
    int64_t sign = 1;
    if (s[p] == '+' || s[p] == '-') {
      sign = s[p] == '-' ? -1 : 1;
      ++p;
      sp();
    } else if (!first) {
      bad("expected '+' or '-'");
    }
    int64_t k = 1;
    bool lead_int = false;
    if (p < s.size() && std::isdigit(static_cast<unsigned char>(s[p]))) {
      k = integer();
      lead_int = true;
      sp();
      if (p < s.size() && s[p] == '*') {
        ++p;
        sp();
      } else {
        a.c0 += sign * k;
        continue;
      }
    }
    if (p >= s.size() || !idx_dim(s[p])) bad("expected index name");
    int d = idx_dim(s[p]);
    if (d > D) bad("index name beyond dimension count");
    ++p;
    sp();
    if (!lead_int && p < s.size() && s[p] == '*') {
      ++p;
      sp();
      if (p >= s.size() || !std::isdigit(static_cast<unsigned char>(s[p]))) bad("expected integer factor");
      k = integer();
    }
    a.coeff[static_cast<size_t>(d - 1)] += sign * k;
  }
  return a;
}

// ---------------------------------------------------------------- scalar
namespace {

struct Lex {
  const std::string& s;
  size_t p = 0;
  int line = 1, col = 1;
  [[noreturn]] void die(const std::string& m) const {
    fail("ParseError", m + " at line " + std::to_string(line) + ", column " + std::to_string(col));
  }
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\t' || s[p] == '\n' || s[p] == '\r')) {
      if (s[p] == '\n') { ++line; col = 1; } else { ++col; }
      ++p;
    }
  }
  char peek() { ws(); return p < s.size() ? s[p] : '\0'; }
  void adv(size_t n) { p += n; col += static_cast<int>(n); }
  bool eat(char c) { if (peek() != c) return false; adv(1); return true; }
  void need(char c) { if (!eat(c)) die(std::string("expected '") + c + "'"); }
  std::string word() {
    ws();
    size_t b = p;
    while (p < s.size() && (std::isalpha(static_cast<unsigned char>(s[p])) || s[p] == '_')) adv(1);
    if (b == p) die("expected identifier");
    return s.substr(b, p - b);
  }
  Expr number() {
    ws();
    size_t b = p;
    bool real = false;
    while (p < s.size() && std::isdigit(static_cast<unsigned char>(s[p]))) adv(1);
    if (b == p) die("expected number");
    if (p < s.size() && s[p] == '.') {
      real = true;
      adv(1);
      while (p < s.size() && std::isdigit(static_cast<unsigned char>(s[p]))) adv(1);
    }
    if (p < s.size() && (s[p] == 'e' || s[p] == 'E')) {
      real = true;
      adv(1);
      if (p < s.size() && (s[p] == '+' || s[p] == '-')) adv(1);
      size_t dg = p;
      while (p < s.size() && std::isdigit(static_cast<unsigned char>(s[p]))) adv(1);
      if (dg == p) die("expected exponent digits");
    }
    std::string tok = s.substr(b, p - b);
    Expr e;
    e.k = EK::Lit;
    e.flit = real;
    if (real) {
      e.fv = std::strtod(tok.c_str(), nullptr);
      e.type = Ty::F64;
    } else {
      e.iv = std::strtoll(tok.c_str(), nullptr, 10);
      e.fv = static_cast<double>(e.iv);
    }
    return e;
  }
  int small() {
    Expr e = number();
    if (e.flit) die("expected integer");
    return static_cast<int>(e.iv);
  }
};

Expr node(EK k, std::vector<Expr> a) {
  Expr e;
  e.k = k;
  e.args = std::move(a);
  return e;
}

Expr p_sum(Lex& lx);

Expr p_atom(Lex& lx) {
  char c = lx.peek();
  if (c == '(') {
    lx.adv(1);
    Expr e = p_sum(lx);
    lx.need(')');
    return e;
  }
  if (c == '-') {  // unary minus folds into literals, else 0 - x
    lx.adv(1);
    Expr in = p_atom(lx);
    if (in.k == EK::Lit) {
      in.iv = -in.iv;
      in.fv = -in.fv;
      return in;
    }
    return node(EK::Sub, {Expr{}, std::move(in)});
  }
  if (std::isdigit(static_cast<unsigned char>(c))) return lx.number();
  std::string w = lx.word();
  if (w == "in") {
    Expr e;
    e.k = EK::In;
    lx.need('(');
    e.buf = lx.small();
    lx.need(',');
    e.acc = lx.small();
    lx.need(')');
    return e;
  }
  if (w == "idx") {
    Expr e;
    e.k = EK::Idx;
    lx.need('(');
    e.dim = lx.small();
    lx.need(')');
    return e;
  }
  struct Fn { const char* n; EK k; int arity; };
  static const Fn fns[] = {{"min", EK::Min, 2}, {"max", EK::Max, 2}, {"cmp", EK::Cmp, 2},
                           {"abs", EK::Abs, 1}, {"select", EK::Select, 3}};
  for (const Fn& f : fns) {
    if (w != f.n) continue;
    lx.need('(');
    std::vector<Expr> a;
    for (int k = 0; k < f.arity; ++k) {
      if (k) lx.need(',');
      a.push_back(p_sum(lx));
    }
    lx.need(')');
    return node(f.k, std::move(a));
  }
  lx.die("unknown function '" + w + "'");
}

Expr p_prod(Lex& lx) {
  Expr e = p_atom(lx);
  for (char c = lx.peek(); c == '*' || c == '/'; c = lx.peek()) {
    lx.adv(1);
    e = node(c == '*' ? EK::Mul : EK::Div, {std::move(e), p_atom(lx)});
  }
  return e;
}

Expr p_sum(Lex& lx) {
  Expr e = p_prod(lx);
  for (char c = lx.peek(); c == '+' || c == '-'; c = lx.peek()) {
    lx.adv(1);
    e = node(c == '+' ? EK::Add : EK::Sub, {std::move(e), p_prod(lx)});
  }
  return e;
}

// Literal-only subtrees may be retyped as f64 (scalar_expr.cpp:208-232).
bool widen(Expr& e) {
  switch (e.k) {
    case EK::Lit:
      if (!e.flit) {
        e.fv = static_cast<double>(e.iv);
        e.type = Ty::F64;
      }
      return true;
    case EK::In:
    case EK::Idx:
    case EK::Cmp:
      return e.type == Ty::F64;
    case EK::Select:
      if (!(widen(e.args[1]) && widen(e.args[2]))) return false;
      e.type = Ty::F64;
      return true;
    default:
      for (auto& a : e.args)
        if (!widen(a)) return false;
      e.type = Ty::F64;
      return true;
  }
}

Ty unify(Expr& a, Expr& b, const char* what) {
  if (a.type == b.type) return a.type;
  if (!widen(a.type == Ty::I64 ? a : b)) fail("MixedTypes", std::string(what) + " mixes i64 and f64 operands");
  return Ty::F64;
}

void type_of(Expr& e, const MdHom& h) {
  for (auto& a : e.args) type_of(a, h);
  switch (e.k) {
    case EK::Lit: e.type = e.flit ? Ty::F64 : Ty::I64; break;
    case EK::In:
      if (e.buf < 1 || e.buf > static_cast<int>(h.in.size()))
        fail("IndexOutOfBounds", "in(" + std::to_string(e.buf) + ",_) references a missing input buffer");
      if (e.acc < 1 || e.acc > static_cast<int>(h.in[static_cast<size_t>(e.buf - 1)].acc.size()))
        fail("IndexOutOfBounds", "in(" + std::to_string(e.buf) + "," + std::to_string(e.acc) +
                                     ") references a missing access");
      e.type = h.in[static_cast<size_t>(e.buf - 1)].type;
      break;
    case EK::Idx:
      if (e.dim < 1 || e.dim > h.D())
        fail("DimOutOfRange", "idx(" + std::to_string(e.dim) + ") with " + std::to_string(h.D()) + " dimensions");
      e.type = Ty::I64;
      break;
    case EK::Abs: e.type = e.args[0].type; break;
    case EK::Cmp:
      unify(e.args[0], e.args[1], "cmp");
      e.type = Ty::I64;
      break;
    case EK::Select:
      if (e.args[0].type != Ty::I64) fail("MixedTypes", "select condition must be i64");
      e.type = unify(e.args[1], e.args[2], "select");
      break;
    default: e.type = unify(e.args[0], e.args[1], "arithmetic"); break;
  }
}

Combine parse_combine(const std::string& s, int d) {
  Combine c;
  if (s == "cc") return c;
  auto bin = [&](const std::string& op) {
    if (op == "+") { c.op = Fold::Add; c.assoc_comm = true; }
    else if (op == "*" || op == "mul") { c.op = Fold::Mul; c.assoc_comm = true; }
    else if (op == "min") { c.op = Fold::Min; c.assoc_comm = true; }
    else if (op == "max") { c.op = Fold::Max; c.assoc_comm = true; }
    else if (op == "-") { c.op = Fold::Sub; }
    else if (op == "/") { c.op = Fold::Div; }
    else fail("UnknownOperator", "unknown binary operator '" + op + "'");
  };
  auto named = [&](const std::string& op) {
    const int k = combine_index(op);
    if (k >= 0) {  // registered custom operator
      const CustomCombine& cc = combine_at(k);
      c.op = Fold::Custom;
      c.custom = k;
      c.assoc_comm = cc.assoc && cc.comm;
      return;
    }
    bin(op);
  };
  if (s.rfind("pw:", 0) == 0) {
    c.kind = Combine::PW;
    named(s.substr(3));
    return c;
  }
  if (s.rfind("ps:", 0) == 0) {
    c.kind = Combine::PS;
    named(s.substr(3));
    return c;
  }
  fail("ParseError", "combine operator " + std::to_string(d) + ": '" + s + "' is not cc, pw:<op>, or ps:<op>");
}

template <class F>
auto guarded(const char* what, F&& f) {
  try {
    return f();
  } catch (const json::ParseFailure& pf) {
    fail("ParseError", std::string(what) + ": " + pf.msg);
  }
}

}  // namespace

std::vector<int64_t> MdHom::collapsed() const {
  std::vector<int64_t> c = sizes;
  for (size_t d = 0; d < c.size(); ++d)
    if (comb[d].kind == Combine::PW) c[d] = 1;
  return c;
}

int MdHom::fold() const {
  for (auto& c : comb)
    if (c.kind != Combine::CC) return c.op == Fold::Custom ? kCustomFoldBase + c.custom : static_cast<int>(c.op);
  return -1;
}

// ---- custom combine registry ------------------------------------------------
namespace {
// a deque keeps references stable while operators are appended; entries are
// never removed (a plan holds its operator's index)
std::mutex g_registry_mu;
std::deque<CustomCombine>& registry() {
  static std::deque<CustomCombine> r = [] {
    std::deque<CustomCombine> v;
    CustomCombine m;
    m.name = "max_prl";
    m.arity = 2;
    // (weight, record): larger weight wins, the lower record on ties
    m.body = "if (b0 > a0 || (b0 == a0 && b1 < a1)) { a0 = b0; a1 = b1; }";
    m.identity = {"INT64_MIN", "INT64_MAX"};
    m.assoc = m.comm = true;
    m.description = "PRL max: lexicographic max of (weight, -record) over the (out 1, out 2) pair";
    m.vm_op = 1;
    v.push_back(m);
    return v;
  }();
  return r;
}
}  // namespace

int register_combine(const CustomCombine& c) {
  std::lock_guard<std::mutex> lk(g_registry_mu);
  auto& r = registry();
  if (c.name.empty() || c.name.find_first_of(" :,\"") != std::string::npos)
    fail("ParseError", "combine operator name '" + c.name + "' is empty or contains a separator");
  static const std::set<std::string> builtin = {"+", "*", "mul", "min", "max", "-", "/"};
  if (builtin.count(c.name)) fail("InvalidConfig", "'" + c.name + "' is a built-in operator of the reference");
  if (c.arity < 1 || c.arity > 8) fail("OutOfRange", "combine operator arity must be in [1, 8]");
  if (c.body.empty()) fail("ParseError", "combine operator '" + c.name + "' has no body");
  for (size_t k = 0; k < r.size(); ++k)
    if (r[k].name == c.name) {
      if (r[k].vm_op) fail("InvalidConfig", "'" + c.name + "' is a built-in custom operator");
      r[k] = c;
      r[k].vm_op = 0;
      return static_cast<int>(k);
    }
  r.push_back(c);
  r.back().vm_op = 0;
  return static_cast<int>(r.size() - 1);
}

int combine_index(const std::string& name) {
  std::lock_guard<std::mutex> lk(g_registry_mu);
  auto& r = registry();
  for (size_t k = 0; k < r.size(); ++k)
    if (r[k].name == name) return static_cast<int>(k);
  return -1;
}

const CustomCombine& combine_at(int index) {
  std::lock_guard<std::mutex> lk(g_registry_mu);
  return registry().at(static_cast<size_t>(index));
}

std::vector<std::string> combine_names() {
  std::lock_guard<std::mutex> lk(g_registry_mu);
  std::vector<std::string> n;
  for (auto& c : registry()) n.push_back(c.name);
  return n;
}

int MdHom::n_in_access() const {
  int n = 0;
  for (auto& b : in) n += static_cast<int>(b.acc.size());
  return n;
}

int MdHom::in_comp(int buf, int acc) const {
  int n = 0;
  for (int b = 0; b < buf - 1; ++b) n += static_cast<int>(in[static_cast<size_t>(b)].acc.size());
  return n + acc - 1;
}

MdHom parse_md_hom(const std::string& text) {
  return guarded("computation", [&] {
    json::Value j = json::parse(text);
    MdHom h;
    h.name = j.at("name").as_str();
    for (auto& v : j.at("dims").a) h.dim_names.push_back(v.as_str());
    for (auto& v : j.at("sizes").a) h.sizes.push_back(v.as_int());
    if (h.dim_names.size() != h.sizes.size())
      fail("ParseError", "computation '" + h.name + "': dims and sizes disagree in length");
    const int D = h.D();
    auto bufs = [&](const json::Value& arr, std::vector<Buf>& out) {
      for (auto& jb : arr.a) {
        Buf b;
        b.name = jb.at("name").as_str();
        const std::string& t = jb.at("type").as_str();
        if (t == "i64") b.type = Ty::I64;
        else if (t == "f64") b.type = Ty::F64;
        else fail("ParseError", "buffer '" + b.name + "': unknown element type '" + t + "' (expected i64 or f64)");
        b.rank = static_cast<int>(jb.at("rank").as_int());
        for (auto& a : jb.at("accesses").a) {
          Access acc;
          const std::string& txt = a.as_str();
          size_t st = 0;
          for (;;) {
            size_t comma = txt.find(',', st);
            acc.idx.push_back(Affine::parse(txt.substr(st, comma == std::string::npos ? std::string::npos : comma - st), D));
            if (comma == std::string::npos) break;
            st = comma + 1;
          }
          b.acc.push_back(std::move(acc));
        }
        out.push_back(std::move(b));
      }
    };
    bufs(j.at("inputs"), h.in);
    bufs(j.at("outputs"), h.out);
    h.scalar_text = j.at("scalar").as_str();
    int d = 0;
    for (auto& v : j.at("combine").a) h.comb.push_back(parse_combine(v.as_str(), ++d));

    // structure (highlevel.cpp:15-59)
    if (D == 0) fail("DimOutOfRange", "computation '" + h.name + "' has no dimensions");
    for (int k = 0; k < D; ++k)
      if (h.sizes[static_cast<size_t>(k)] < 1)
        fail("OutOfRange", "dimension " + std::to_string(k + 1) + " of '" + h.name + "' has non-positive size");
    if (static_cast<int>(h.comb.size()) != D)
      fail("DimOutOfRange", "'" + h.name + "' declares " + std::to_string(h.comb.size()) +
                                " combine operators for " + std::to_string(D) + " dimensions");
    for (auto* side : {&h.in, &h.out}) {
      if (side->empty()) fail("IndexOutOfBounds", "'" + h.name + "' has an empty view");
      for (auto& b : *side) {
        if (b.rank < 1) fail("DimOutOfRange", "buffer '" + b.name + "' has rank " + std::to_string(b.rank));
        if (b.acc.empty()) fail("IndexOutOfBounds", "buffer '" + b.name + "' has no accesses");
        for (auto& a : b.acc)
          if (static_cast<int>(a.idx.size()) != b.rank)
            fail("DimOutOfRange", "buffer '" + b.name + "' access arity does not match rank");
      }
    }

    // scalar function: parse + typecheck (scalar_expr.cpp:318-381)
    Lex lx{h.scalar_text};
    while (lx.peek() != '\0') {
      if (lx.word() != "out") lx.die("expected 'out'");
      Assign a;
      lx.need('(');
      a.buf = lx.small();
      lx.need(',');
      a.acc = lx.small();
      lx.need(')');
      lx.need('=');
      a.e = p_sum(lx);
      h.assigns.push_back(std::move(a));
      if (!lx.eat(';')) break;
    }
    if (lx.peek() != '\0') lx.die("trailing input");
    if (h.assigns.empty()) lx.die("expected at least one out(...) assignment");
    std::vector<std::vector<bool>> seen;
    for (auto& b : h.out) seen.emplace_back(b.acc.size(), false);
    for (auto& a : h.assigns) {
      std::string tag = "out(" + std::to_string(a.buf) + "," + std::to_string(a.acc) + ")";
      if (a.buf < 1 || a.buf > static_cast<int>(h.out.size()))
        fail("IndexOutOfBounds", tag + " references a missing output buffer");
      if (a.acc < 1 || a.acc > static_cast<int>(h.out[static_cast<size_t>(a.buf - 1)].acc.size()))
        fail("IndexOutOfBounds", tag + " references a missing access");
      auto flag = seen[static_cast<size_t>(a.buf - 1)][static_cast<size_t>(a.acc - 1)];
      if (flag) fail("IndexOutOfBounds", tag + " assigned twice");
      seen[static_cast<size_t>(a.buf - 1)][static_cast<size_t>(a.acc - 1)] = true;
      type_of(a.e, h);
      Ty want = h.out[static_cast<size_t>(a.buf - 1)].type;
      if (a.e.type != want && !(want == Ty::F64 && widen(a.e)))
        fail("MixedTypes", tag + " expression type " + ty_name(a.e.type) + " does not match buffer type " +
                               ty_name(want));
    }
    for (size_t b = 0; b < seen.size(); ++b)
      for (size_t k = 0; k < seen[b].size(); ++k)
        if (!seen[b][k])
          fail("IndexOutOfBounds", "out(" + std::to_string(b + 1) + "," + std::to_string(k + 1) + ") never assigned");
    std::stable_sort(h.assigns.begin(), h.assigns.end(),
                     [](const Assign& x, const Assign& y) { return x.buf != y.buf ? x.buf < y.buf : x.acc < y.acc; });
    for (auto& c : h.comb)
      if (c.op == Fold::Custom && c.kind != Combine::CC) {
        const CustomCombine& op = combine_at(c.custom);
        if (static_cast<int>(h.assigns.size()) != op.arity)
          fail("MixedIncompatibleOperators", "combine operator '" + op.name + "' folds " + std::to_string(op.arity) +
                                                 " output components jointly; the scalar function assigns " +
                                                 std::to_string(h.assigns.size()));
      }
    return h;
  });
}

std::string md_hom_violation(const MdHom& e) {
  int first = -1;
  for (int d = 0; d < e.D(); ++d) {
    const Combine& c = e.comb[static_cast<size_t>(d)];
    if (c.kind == Combine::CC) continue;
    if (!c.assoc_comm)
      return "dimension " + std::to_string(d + 1) + " folds with an operator that is not associative and commutative";
    if (first < 0) {
      first = d;
      continue;
    }
    if (e.comb[static_cast<size_t>(first)].op != c.op || e.comb[static_cast<size_t>(first)].custom != c.custom)
      return "dimensions " + std::to_string(first + 1) + " and " + std::to_string(d + 1) +
             " fold with different operators";
  }
  return "";
}

std::vector<std::vector<int64_t>> infer_extents(const std::vector<Buf>& bufs, const std::vector<int64_t>& sizes) {
  std::vector<std::vector<int64_t>> out;
  for (auto& b : bufs) {
    std::vector<int64_t> ext(static_cast<size_t>(b.rank), 0);
    for (auto& a : b.acc)
      for (int r = 0; r < b.rank; ++r) {
        const Affine& f = a.idx[static_cast<size_t>(r)];
        int64_t lo = f.lo(sizes);
        if (lo < 0)
          fail("NegativeIndexReachable", "buffer '" + b.name + "' reaches coordinate " + std::to_string(lo));
        ext[static_cast<size_t>(r)] = std::max(ext[static_cast<size_t>(r)], f.hi(sizes) + 1);
      }
    out.push_back(std::move(ext));
  }
  return out;
}

Linear linearize(const Access& a, const std::vector<int64_t>& ext, int D) {
  Linear l;
  l.cj.assign(static_cast<size_t>(D), 0);
  int64_t stride = 1;
  for (int r = static_cast<int>(ext.size()) - 1; r >= 0; --r) {
    const Affine& f = a.idx[static_cast<size_t>(r)];
    l.c0 += stride * f.c0;
    for (int d = 0; d < D; ++d) l.cj[static_cast<size_t>(d)] += stride * f.coeff[static_cast<size_t>(d)];
    stride *= ext[static_cast<size_t>(r)];
  }
  return l;
}

// ---------------------------------------------------------------- ASM
const std::string& Asm::layer(int i) const {
  if (i < 1 || i > L()) fail("OutOfRange", "layer id " + std::to_string(i) + " not in 1.." + std::to_string(L()));
  return i <= M() ? mem[static_cast<size_t>(i - 1)] : core[static_cast<size_t>(i - 1 - M())];
}

int Asm::id(const std::string& n) const {
  for (int i = 1; i <= L(); ++i)
    if (layer(i) == n) return i;
  return -1;
}

Asm asm_preset(const std::string& n) {
  if (n == "OpenMP") return {n, {"MM", "L2", "L1"}, {"COR"}};
  if (n == "OpenMP+L3") return {n, {"MM", "L3", "L2", "L1"}, {"COR"}};
  if (n == "OpenMP+L3+SIMD") return {n, {"MM", "L3", "L2", "L1"}, {"COR", "SIMD"}};
  if (n == "CUDA") return {n, {"DM", "SM", "RM"}, {"SMX", "CC"}};
  if (n == "CUDA+WRP") return {n, {"DM", "SM", "RM"}, {"SMX", "WRP", "CC"}};
  if (n == "OpenCL") return {n, {"GM", "LM", "PM"}, {"CU", "PE"}};
  if (n == "MultiGPU") return {n, {"HM", "DM", "SM", "RM"}, {"GPU", "SMX", "CC"}};
  if (n == "MultiNodeMultiGPU") return {n, {"NM", "HM", "DM", "SM", "RM"}, {"NOD", "GPU", "SMX", "CC"}};
  if (n == "Artificial2+1") return {n, {"HM", "L1"}, {"COR"}};
  if (n == "B200") return {n, {"DM", "SM", "RM"}, {"SMX", "WRP", "CC"}};
  if (n == "MultiB200") return {n, {"HM", "DM", "SM", "RM"}, {"GPU", "SMX", "WRP", "CC"}};
  fail("UnknownPreset", "no abstract system model preset named '" + n + "'");
}

Asm resolve_asm(const std::string& arg) {
  if (arg.empty() || arg[0] != '{') return asm_preset(arg.empty() ? "B200" : arg);
  return guarded("ASM description", [&] {
    json::Value j = json::parse(arg);
    Asm m;
    m.name = j.has("name") ? j.at("name").as_str() : "inline";
    if (!j.has("mem") || j.at("mem").size() == 0) fail("ParseError", "ASM description needs a non-empty \"mem\" layer list");
    for (auto& v : j.at("mem").a) m.mem.push_back(v.as_str());
    if (j.has("core"))
      for (auto& v : j.at("core").a) m.core.push_back(v.as_str());
    std::set<std::string> names;
    for (int i = 1; i <= m.L(); ++i)
      if (!names.insert(m.layer(i)).second) fail("ParseError", "ASM layer name '" + m.layer(i) + "' appears twice");
    return m;
  });
}

// ---------------------------------------------------------------- config
namespace {
std::vector<int> iota_perm(int n) {
  std::vector<int> p(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) p[static_cast<size_t>(k)] = k + 1;
  return p;
}
std::vector<Level> lex_levels(int L, int D) {
  std::vector<Level> v;
  for (int l = 1; l <= L; ++l)
    for (int d = 1; d <= D; ++d) v.push_back({l, d});
  return v;
}
}  // namespace

Config baseline_config(const MdHom& e, const Asm& m) {
  const int L = m.L(), D = e.D(), LD = L * D;
  Config c;
  c.parts.assign(static_cast<size_t>(L), std::vector<int64_t>(static_cast<size_t>(D), 1));
  for (int d = 0; d < D; ++d) c.parts[0][static_cast<size_t>(d)] = e.sizes[static_cast<size_t>(d)];
  c.ord_de = c.ord_scalar = c.ord_re = lex_levels(L, D);
  c.ass_de = c.ass_scalar = c.ass_re = lex_levels(L, D);
  for (auto& b : e.in) {
    c.mem_de.push_back(std::vector<int>(static_cast<size_t>(LD), 1));
    c.layout_de.push_back(std::vector<std::vector<int>>(static_cast<size_t>(LD), iota_perm(b.rank)));
    c.mem_scalar_in.push_back(1);
    c.layout_scalar_in.push_back(iota_perm(b.rank));
  }
  for (auto& b : e.out) {
    c.mem_re.push_back(std::vector<int>(static_cast<size_t>(LD), 1));
    c.layout_re.push_back(std::vector<std::vector<int>>(static_cast<size_t>(LD), iota_perm(b.rank)));
    c.mem_scalar_out.push_back(1);
    c.layout_scalar_out.push_back(iota_perm(b.rank));
  }
  return c;
}

Config parse_config(const std::string& text, const MdHom& e, const Asm& m) {
  return guarded("config", [&] {
    json::Value j = json::parse(text);
    const int L = m.L(), D = e.D();
    const size_t LD = static_cast<size_t>(L * D);
    Config c = baseline_config(e, m);
    if (j.has("num_parts")) {
      const json::Value& np = j.at("num_parts");
      if (static_cast<int>(np.size()) != L)
        fail("ParseError", "num_parts must have one row per ASM layer (" + std::to_string(L) + ")");
      c.parts.clear();
      for (auto& row : np.a) {
        if (static_cast<int>(row.size()) != D)
          fail("ParseError", "num_parts rows must have one entry per dimension (" + std::to_string(D) + ")");
        std::vector<int64_t> r;
        for (auto& x : row.a) r.push_back(x.as_int());
        c.parts.push_back(std::move(r));
      }
    }
    auto ord = [&](const char* key, std::vector<Level>& dst) {
      if (!j.has(key)) return;
      dst.clear();
      for (auto& v : j.at(key).a) {
        if (v.size() != 2) fail("ParseError", std::string(key) + ": MDH level must be a [layer, dim] pair");
        dst.push_back({static_cast<int>(v[0].as_int()), static_cast<int>(v[1].as_int())});
      }
    };
    ord("ord_de", c.ord_de);
    ord("ord_scalar", c.ord_scalar);
    ord("ord_re", c.ord_re);
    auto ass = [&](const char* key, std::vector<Level>& dst) {
      if (!j.has(key)) return;
      const json::Value& a = j.at(key);
      if (a.size() != LD)
        fail("ParseError", std::string(key) + " must list one ASM level per MDH level (" + std::to_string(LD) + ")");
      dst.clear();
      for (auto& v : a.a) {
        if (v.size() != 2) fail("ParseError", std::string(key) + ": ASM level must be a [layer, dim] pair");
        Level l;
        if (v[0].is_str()) {
          l.layer = m.id(v[0].as_str());
          if (l.layer < 0) fail("ParseError", std::string(key) + ": unknown ASM layer '" + v[0].as_str() + "'");
        } else {
          l.layer = static_cast<int>(v[0].as_int());
          if (l.layer < 1 || l.layer > L) fail("ParseError", std::string(key) + ": ASM layer id out of range");
        }
        l.dim = static_cast<int>(v[1].as_int());
        dst.push_back(l);
      }
    };
    ass("ass_de", c.ass_de);
    ass("ass_scalar", c.ass_scalar);
    ass("ass_re", c.ass_re);
    auto region = [&](const json::Value& v, const std::string& ctx) {
      if (v.is_int()) {
        int r = static_cast<int>(v.i);
        if (r < 1 || r > m.M()) fail("ParseError", ctx + ": region id " + std::to_string(r) + " outside 1.." + std::to_string(m.M()));
        return r;
      }
      if (v.is_str()) {
        int r = m.id(v.s);
        if (r < 1 || r > m.M()) fail("ParseError", ctx + ": unknown region '" + v.s + "'");
        return r;
      }
      fail("ParseError", ctx + ": region must be a 1-based id or a region name");
    };
    auto buf_index = [&](const std::vector<Buf>& bs, const std::string& n) {
      for (size_t b = 0; b < bs.size(); ++b)
        if (bs[b].name == n) return static_cast<int>(b);
      return -1;
    };
    auto mem_phase = [&](const char* key, const std::vector<Buf>& bs, std::vector<std::vector<int>>& dst) {
      if (!j.has(key)) return;
      for (auto& kv : j.at(key).o) {
        int b = buf_index(bs, kv.first);
        if (b < 0) fail("ParseError", std::string(key) + ": unknown buffer '" + kv.first + "'");
        auto& row = dst[static_cast<size_t>(b)];
        std::string ctx = std::string(key) + "." + kv.first;
        if (kv.second.is_arr()) {
          if (kv.second.size() != LD) fail("ParseError", ctx + " must list one region per MDH level");
          for (size_t r = 0; r < LD; ++r) row[r] = region(kv.second[r], ctx);
        } else {
          int reg = region(kv.second, ctx);
          for (auto& x : row) x = reg;
        }
      }
    };
    mem_phase("mem_de", e.in, c.mem_de);
    mem_phase("mem_re", e.out, c.mem_re);
    auto perm = [&](const json::Value& v) {
      std::vector<int> p;
      for (auto& x : v.a) p.push_back(static_cast<int>(x.as_int()));
      return p;
    };
    auto layout_phase = [&](const char* key, const std::vector<Buf>& bs, std::vector<std::vector<std::vector<int>>>& dst) {
      if (!j.has(key)) return;
      for (auto& kv : j.at(key).o) {
        int b = buf_index(bs, kv.first);
        if (b < 0) fail("ParseError", std::string(key) + ": unknown buffer '" + kv.first + "'");
        auto& row = dst[static_cast<size_t>(b)];
        if (!kv.second.is_arr() || kv.second.size() == 0) fail("ParseError", std::string(key) + ": expected a layout");
        if (kv.second[0].is_arr()) {
          if (kv.second.size() != LD) fail("ParseError", std::string(key) + ": one layout per MDH level");
          for (size_t r = 0; r < LD; ++r) row[r] = perm(kv.second[r]);
        } else {
          std::vector<int> p = perm(kv.second);
          for (auto& x : row) x = p;
        }
      }
    };
    layout_phase("layout_de", e.in, c.layout_de);
    layout_phase("layout_re", e.out, c.layout_re);
    auto mem_scalar = [&](const char* key, const std::vector<Buf>& bs, std::vector<int>& dst) {
      if (!j.has(key)) return;
      for (auto& kv : j.at(key).o) {
        int b = buf_index(bs, kv.first);
        if (b < 0) fail("ParseError", std::string(key) + ": unknown buffer '" + kv.first + "'");
        dst[static_cast<size_t>(b)] = region(kv.second, key);
      }
    };
    mem_scalar("mem_scalar_in", e.in, c.mem_scalar_in);
    mem_scalar("mem_scalar_out", e.out, c.mem_scalar_out);
    auto layout_scalar = [&](const char* key, const std::vector<Buf>& bs, std::vector<std::vector<int>>& dst) {
      if (!j.has(key)) return;
      for (auto& kv : j.at(key).o) {
        int b = buf_index(bs, kv.first);
        if (b < 0) fail("ParseError", std::string(key) + ": unknown buffer '" + kv.first + "'");
        dst[static_cast<size_t>(b)] = perm(kv.second);
      }
    };
    layout_scalar("layout_scalar_in", e.in, c.layout_scalar_in);
    layout_scalar("layout_scalar_out", e.out, c.layout_scalar_out);
    if (j.has("c_dev")) c.c_dev = j.at("c_dev").as_int();
    return c;
  });
}

std::string config_json(const Config& c, const MdHom& e, const Asm& m) {
  using json::Value;
  Value j = Value::make_obj();
  Value np = Value::make_arr();
  for (auto& row : c.parts) {
    Value r = Value::make_arr();
    for (int64_t p : row) r.push(Value::make_int(p));
    np.push(std::move(r));
  }
  j.set("num_parts", std::move(np));
  auto lv = [](const std::vector<Level>& v) {
    Value a = Value::make_arr();
    for (auto& l : v) {
      Value p = Value::make_arr();
      p.push(Value::make_int(l.layer));
      p.push(Value::make_int(l.dim));
      a.push(std::move(p));
    }
    return a;
  };
  auto as = [&](const std::vector<Level>& v) {
    Value a = Value::make_arr();
    for (auto& l : v) {
      Value p = Value::make_arr();
      p.push(Value::make_str(m.layer(l.layer)));
      p.push(Value::make_int(l.dim));
      a.push(std::move(p));
    }
    return a;
  };
  j.set("ord_de", lv(c.ord_de));
  j.set("ord_scalar", lv(c.ord_scalar));
  j.set("ord_re", lv(c.ord_re));
  j.set("ass_de", as(c.ass_de));
  j.set("ass_scalar", as(c.ass_scalar));
  j.set("ass_re", as(c.ass_re));
  auto mem = [&](const std::vector<Buf>& bs, const std::vector<std::vector<int>>& mm) {
    Value g = Value::make_obj();
    for (size_t b = 0; b < bs.size() && b < mm.size(); ++b) {
      Value row = Value::make_arr();
      for (int r : mm[b]) row.push(Value::make_str(m.layer(r)));
      g.set(bs[b].name, std::move(row));
    }
    return g;
  };
  auto perm = [](const std::vector<int>& p) {
    Value a = Value::make_arr();
    for (int x : p) a.push(Value::make_int(x));
    return a;
  };
  auto lay = [&](const std::vector<Buf>& bs, const std::vector<std::vector<std::vector<int>>>& ll) {
    Value g = Value::make_obj();
    for (size_t b = 0; b < bs.size() && b < ll.size(); ++b) {
      Value row = Value::make_arr();
      for (auto& p : ll[b]) row.push(perm(p));
      g.set(bs[b].name, std::move(row));
    }
    return g;
  };
  j.set("mem_de", mem(e.in, c.mem_de));
  j.set("mem_re", mem(e.out, c.mem_re));
  j.set("layout_de", lay(e.in, c.layout_de));
  j.set("layout_re", lay(e.out, c.layout_re));
  auto ms = [&](const std::vector<Buf>& bs, const std::vector<int>& mm) {
    Value g = Value::make_obj();
    for (size_t b = 0; b < bs.size() && b < mm.size(); ++b) g.set(bs[b].name, Value::make_str(m.layer(mm[b])));
    return g;
  };
  auto ls = [&](const std::vector<Buf>& bs, const std::vector<std::vector<int>>& ll) {
    Value g = Value::make_obj();
    for (size_t b = 0; b < bs.size() && b < ll.size(); ++b) g.set(bs[b].name, perm(ll[b]));
    return g;
  };
  j.set("mem_scalar_in", ms(e.in, c.mem_scalar_in));
  j.set("mem_scalar_out", ms(e.out, c.mem_scalar_out));
  j.set("layout_scalar_in", ls(e.in, c.layout_scalar_in));
  j.set("layout_scalar_out", ls(e.out, c.layout_scalar_out));
  j.set("c_dev", Value::make_int(c.c_dev));
  return json::dump(j, 2) + "\n";
}

std::string config_violation(const Config& c, const MdHom& e, const Asm& m, bool model_rules) {
  const int L = m.L(), D = e.D(), LD = L * D, M = m.M();
  auto lvl = [](const Level& l) { return "(" + std::to_string(l.layer) + "," + std::to_string(l.dim) + ")"; };
  // shape
  bool ok = static_cast<int>(c.parts.size()) == L;
  for (auto& r : c.parts) ok = ok && static_cast<int>(r.size()) == D;
  for (auto* o : {&c.ord_de, &c.ord_scalar, &c.ord_re, &c.ass_de, &c.ass_scalar, &c.ass_re})
    ok = ok && static_cast<int>(o->size()) == LD;
  ok = ok && c.mem_de.size() == e.in.size() && c.layout_de.size() == e.in.size() &&
       c.mem_scalar_in.size() == e.in.size() && c.layout_scalar_in.size() == e.in.size() &&
       c.mem_re.size() == e.out.size() && c.layout_re.size() == e.out.size() &&
       c.mem_scalar_out.size() == e.out.size() && c.layout_scalar_out.size() == e.out.size();
  if (ok)
    for (auto* mm : {&c.mem_de, &c.mem_re})
      for (auto& row : *mm) ok = ok && static_cast<int>(row.size()) == LD;
  if (ok)
    for (auto* ll : {&c.layout_de, &c.layout_re})
      for (auto& row : *ll) ok = ok && static_cast<int>(row.size()) == LD;
  if (!ok) return "structure: configuration maps do not match the model/computation shape";
  // full partitioning (PAPER.md Parameter 0)
  for (int d = 0; d < D; ++d) {
    int64_t prod = 1;
    for (int l = 0; l < L; ++l) {
      int64_t p = c.parts[static_cast<size_t>(l)][static_cast<size_t>(d)];
      if (p < 1) return "full partitioning: part counts must be >= 1 in dimension " + std::to_string(d + 1);
      prod *= p;
    }
    if (prod != e.sizes[static_cast<size_t>(d)])
      return "full partitioning: part counts in dimension " + std::to_string(d + 1) + " multiply to " +
             std::to_string(prod) + ", size is " + std::to_string(e.sizes[static_cast<size_t>(d)]);
  }
  for (auto* o : {&c.ord_de, &c.ord_scalar, &c.ord_re}) {
    std::vector<bool> seen(static_cast<size_t>(LD), false);
    for (auto& l : *o) {
      if (l.layer < 1 || l.layer > L || l.dim < 1 || l.dim > D) return "order bijection: level " + lvl(l) + " outside the level set";
      size_t r = static_cast<size_t>((l.layer - 1) * D + l.dim - 1);
      if (seen[r]) return "order bijection: repeated level " + lvl(l);
      seen[r] = true;
    }
  }
  for (auto* a : {&c.ass_de, &c.ass_scalar, &c.ass_re}) {
    std::vector<bool> seen(static_cast<size_t>(LD), false);
    for (auto& l : *a) {
      if (l.layer < 1 || l.layer > L || l.dim < 1 || l.dim > D) return "assignment bijection: target " + lvl(l) + " outside the model";
      size_t r = static_cast<size_t>((l.layer - 1) * D + l.dim - 1);
      if (seen[r]) return "assignment bijection: two levels map onto one ASM level";
      seen[r] = true;
    }
  }
  auto region_ok = [&](int r) { return r >= 1 && r <= M; };
  for (auto* mm : {&c.mem_de, &c.mem_re})
    for (auto& row : *mm)
      for (int r : row)
        if (!region_ok(r)) return "region range: region " + std::to_string(r) + " outside 1.." + std::to_string(M);
  for (auto* ms : {&c.mem_scalar_in, &c.mem_scalar_out})
    for (int r : *ms)
      if (!region_ok(r)) return "region range: region " + std::to_string(r) + " outside 1.." + std::to_string(M);
  auto is_perm = [](const std::vector<int>& p, int n) {
    if (static_cast<int>(p.size()) != n) return false;
    std::vector<bool> s(static_cast<size_t>(n), false);
    for (int v : p) {
      if (v < 1 || v > n || s[static_cast<size_t>(v - 1)]) return false;
      s[static_cast<size_t>(v - 1)] = true;
    }
    return true;
  };
  for (size_t b = 0; b < e.in.size(); ++b) {
    for (auto& p : c.layout_de[b])
      if (!is_perm(p, e.in[b].rank)) return "layout permutation: layout_de['" + e.in[b].name + "']";
    if (!is_perm(c.layout_scalar_in[b], e.in[b].rank)) return "layout permutation: layout_scalar_in['" + e.in[b].name + "']";
  }
  for (size_t b = 0; b < e.out.size(); ++b) {
    for (auto& p : c.layout_re[b])
      if (!is_perm(p, e.out[b].rank)) return "layout permutation: layout_re['" + e.out[b].name + "']";
    if (!is_perm(c.layout_scalar_out[b], e.out[b].rank)) return "layout permutation: layout_scalar_out['" + e.out[b].name + "']";
  }
  if (!model_rules) return "";

  // model rules (tuning.cpp:172-225) + the B200 ones
  auto count_rule = [&](const std::string& core, int64_t bound, const std::string& rule) -> std::string {
    int layer = m.id(core);
    if (layer < 0) return "";
    for (auto* a : {&c.ass_de, &c.ass_scalar, &c.ass_re}) {
      int64_t prod = 1;
      for (int r = 0; r < LD; ++r)
        if ((*a)[static_cast<size_t>(r)].layer == layer) prod *= c.parts[static_cast<size_t>(r / D)][static_cast<size_t>(r % D)];
      if (prod > bound) return rule + ": " + std::to_string(prod) + " parts on " + core + ", limit is " + std::to_string(bound);
    }
    return "";
  };
  auto combine_rule = [&](const std::string& core, std::vector<std::string> allowed_names, const std::string& rule) -> std::string {
    int layer = m.id(core);
    if (layer < 0) return "";
    std::vector<int> allowed;
    for (auto& n : allowed_names)
      if (m.id(n) > 0 && m.id(n) <= M) allowed.push_back(m.id(n));
    for (int r = 0; r < LD; ++r) {
      if (c.ass_re[static_cast<size_t>(r)].layer != layer) continue;
      int l = r / D, d = r % D;
      if (c.parts[static_cast<size_t>(l)][static_cast<size_t>(d)] <= 1) continue;
      if (e.comb[static_cast<size_t>(d)].kind == Combine::CC) continue;
      for (size_t b = 0; b < e.out.size(); ++b) {
        int reg = c.mem_re[b][static_cast<size_t>(r)];
        if (std::find(allowed.begin(), allowed.end(), reg) == allowed.end())
          return rule + ": level (" + std::to_string(l + 1) + "," + std::to_string(d + 1) + ") combines on " + core +
                 " but stores '" + e.out[b].name + "' in " + m.layer(reg);
      }
    }
    return "";
  };
  std::string v;
  if (m.name == "CUDA") {
    if (!(v = count_rule("CC", 1024, "Number of CCs limited")).empty()) return v;
    if (!(v = combine_rule("SMX", {"DM"}, "SMXs combine in DM")).empty()) return v;
    if (!(v = combine_rule("CC", {"DM", "SM"}, "CCs combine in DM/SM")).empty()) return v;
  } else if (m.name == "CUDA+WRP" || m.name == "B200" || m.name == "MultiB200") {
    if (!(v = count_rule("CC", 1024, "Number of CCs limited")).empty()) return v;
    if (!(v = combine_rule("SMX", {"DM"}, "SMXs combine in DM")).empty()) return v;
    if (!(v = combine_rule("WRP", {"DM", "SM"}, "WRPs combine in DM/SM")).empty()) return v;
    if (m.name != "CUDA+WRP") {
      // B200 capacity: one CTA holds at most 1024 threads = WRP x CC parts.
      int w = m.id("WRP"), cc = m.id("CC");
      for (auto* a : {&c.ass_de, &c.ass_scalar, &c.ass_re}) {
        int64_t prod = 1;
        for (int r = 0; r < LD; ++r) {
          int lay = (*a)[static_cast<size_t>(r)].layer;
          if (lay == w || lay == cc) prod *= c.parts[static_cast<size_t>(r / D)][static_cast<size_t>(r % D)];
        }
        if (prod > 1024) return "Threads per CTA limited: " + std::to_string(prod) + " WRP x CC parts, limit is 1024";
      }
      if (m.name == "MultiB200")
        if (!(v = combine_rule("GPU", {"DM", "HM"}, "GPUs combine in DM (NCCL) or HM")).empty()) return v;
    }
  } else if (m.name == "OpenCL") {
    if (!(v = count_rule("PE", c.c_dev, "Number of PEs limited")).empty()) return v;
    if (!(v = combine_rule("CU", {"GM"}, "CUs combine in GM")).empty()) return v;
    if (!(v = combine_rule("PE", {"GM", "LM"}, "PEs combine in GM/LM")).empty()) return v;
  }
  return "";
}

std::vector<std::vector<int64_t>> parts_per_asm_layer(const Config& c, const MdHom& e, const Asm& m) {
  const int L = m.L(), D = e.D();
  std::vector<std::vector<int64_t>> P(static_cast<size_t>(L), std::vector<int64_t>(static_cast<size_t>(D), 1));
  for (int r = 0; r < L * D; ++r) {
    int l = r / D, d = r % D;
    int tgt = c.ass_re[static_cast<size_t>(r)].layer;
    P[static_cast<size_t>(tgt - 1)][static_cast<size_t>(d)] *= c.parts[static_cast<size_t>(l)][static_cast<size_t>(d)];
  }
  return P;
}

}  // namespace mdhb
