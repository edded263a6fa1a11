// The md_hom declaration and the Table-1 tuning space, as the B200 backend
// sees them.  This is the product-side front end behind the C ABI
// (include/mdh_b200.h): it reads the reference's own JSON dialect unchanged
// (proj/src/json_io.cpp:298-328 for computations, :128-237 for configs) and
// keeps the reference's error codes (proj/include/mdh/error.hpp:9-17) so a
// caller sees the same failures as with mdh::reference_execute.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mdhb {

// Same contract as mdh::Error: a stable code plus a human message.
struct Error : std::runtime_error {
  std::string code;
  Error(std::string c, const std::string& msg) : std::runtime_error(c + ": " + msg), code(std::move(c)) {}
};
[[noreturn]] void fail(const std::string& code, const std::string& msg);

enum class Ty { I64, F64 };  // the reference's value model (value.hpp:12)

// c0 + sum_d coeff[d] * i_d   (views.hpp:15-31)
struct Affine {
  int64_t c0 = 0;
  std::vector<int64_t> coeff;
  int64_t lo(const std::vector<int64_t>& n) const;  // min over [0, n_d)
  int64_t hi(const std::vector<int64_t>& n) const;  // max over [0, n_d)
  static Affine parse(const std::string& text, int D);
};

struct Access {
  std::vector<Affine> idx;  // one per buffer rank
};

struct Buf {
  std::string name;
  Ty type = Ty::I64;
  int rank = 0;
  std::vector<Access> acc;
};

// Scalar-function AST (scalar_expr.hpp:12-25).
enum class EK { Lit, In, Idx, Add, Sub, Mul, Div, Min, Max, Abs, Cmp, Select };
struct Expr {
  EK k = EK::Lit;
  bool flit = false;
  int64_t iv = 0;
  double fv = 0.0;
  int buf = 0, acc = 0, dim = 0;  // 1-based like the text form
  Ty type = Ty::I64;
  std::vector<Expr> args;
};
struct Assign {
  int buf = 1, acc = 1;
  Expr e;
};

enum class Fold { Add = 0, Sub = 1, Mul = 2, Div = 3, Min = 4, Max = 5, Custom = 6 };  // mda.hpp:52 (+ Custom)
struct Combine {
  enum Kind { CC, PW, PS } kind = CC;
  Fold op = Fold::Add;
  bool assoc_comm = false;  // mda.cpp:75-83: + * min max are declared assoc+comm
  int custom = -1;          // registry index when op == Fold::Custom
};

// ---- custom combine operators (API extension; the reference's BinOpKind is
// closed, mda.hpp:52, and its JSON accepts only the six named operators,
// json_io.cpp:58-64 / mda.cpp:75-83).  A registered operator folds the TUPLE
// of all output components of the scalar function jointly -- e.g. max_prl
// keeps the (weight, record) pair with the larger weight and, on ties, the
// lower record: PRL's custom combine.  It is used as
// pw:<name> or ps:<name> like a built-in operator.
struct CustomCombine {
  std::string name;
  int arity = 0;                      // output components folded jointly
  std::string body;                   // CUDA C statements over a0.. (accumulator, lvalues) and b0.. (next value)
  std::vector<std::string> identity;  // per component (C literal text), documentation + seeding
  bool assoc = false, comm = false;
  std::string description;
  int vm_op = 0;                      // > 0: also compiled into the generic device VM (built-ins)
};
constexpr int kCustomFoldBase = 100;  // MdHom::fold() of custom operator k = kCustomFoldBase + k
// registers (or replaces a same-named, not built-in) operator; returns its index
int register_combine(const CustomCombine& c);
int combine_index(const std::string& name);  // -1 when not registered
const CustomCombine& combine_at(int index);
std::vector<std::string> combine_names();

struct MdHom {
  std::string name;
  std::vector<std::string> dim_names;
  std::vector<int64_t> sizes;
  std::vector<Buf> in, out;
  std::string scalar_text;
  std::vector<Assign> assigns;  // typed, canonical (buf, acc) order
  std::vector<Combine> comb;

  int D() const { return static_cast<int>(sizes.size()); }
  std::vector<int64_t> collapsed() const;  // pw dims -> 1 (highlevel.cpp:65-75)
  int fold() const;                        // shared fold op of non-cc dims, -1 if none;
                                           // kCustomFoldBase + k for custom operator k
  int n_in_access() const;
  int in_comp(int buf, int acc) const;     // flat (buffer, access) position, 1-based args
};

MdHom parse_md_hom(const std::string& json_text);
// md_hom is partial (Lemma 2.9): all non-cc dims share one assoc+comm op.
// Empty string when valid, else the first violation (highlevel.cpp:72-102).
std::string md_hom_violation(const MdHom& e);
// 1 + max over accesses per rank; NegativeIndexReachable below 0 (views.cpp:164-184).
std::vector<std::vector<int64_t>> infer_extents(const std::vector<Buf>& bufs, const std::vector<int64_t>& sizes);

// Flat row-major offset of an access as an affine function of the md_hom
// index: off = c0 + sum_d cj[d] * i_d (the reference's AccessPlan,
// engine.cpp:266-286).
struct Linear {
  int64_t c0 = 0;
  std::vector<int64_t> cj;
};
Linear linearize(const Access& a, const std::vector<int64_t>& extents, int D);

// ---- abstract system model + Table-1 configuration --------------------
struct Asm {
  std::string name;
  std::vector<std::string> mem, core;
  int L() const { return static_cast<int>(mem.size() + core.size()); }
  int M() const { return static_cast<int>(mem.size()); }
  const std::string& layer(int id) const;  // 1-based, memory layers first
  int id(const std::string& n) const;      // -1 when absent
};
// Reference presets (asm_model.cpp:23-43) plus the B200 ones:
//   "B200"      {DM, SM, RM | SMX, WRP, CC}
//   "MultiB200" {HM, DM, SM, RM | GPU, SMX, WRP, CC}
Asm asm_preset(const std::string& name);
Asm resolve_asm(const std::string& arg);  // preset name or inline JSON

struct Level {
  int layer = 1, dim = 1;
};
struct Config {
  std::vector<std::vector<int64_t>> parts;  // [layer-1][dim-1]
  std::vector<Level> ord_de, ord_scalar, ord_re;
  std::vector<Level> ass_de, ass_scalar, ass_re;  // by level rank -> ASM level
  std::vector<std::vector<int>> mem_de, mem_re;   // [buffer][rank] -> region
  std::vector<std::vector<std::vector<int>>> layout_de, layout_re;
  std::vector<int> mem_scalar_in, mem_scalar_out;
  std::vector<std::vector<int>> layout_scalar_in, layout_scalar_out;
  int64_t c_dev = 1024;
};

Config baseline_config(const MdHom& e, const Asm& m);  // tuning.cpp:476-503
Config parse_config(const std::string& text, const MdHom& e, const Asm& m);
std::string config_json(const Config& c, const MdHom& e, const Asm& m);
// Structural rules + (optionally) the model rules of the ASM; returns
// "<rule>: <message>" of the first violation, or "" (tuning.cpp:41-228).
std::string config_violation(const Config& c, const MdHom& e, const Asm& m, bool model_rules);

// Product of parts placed on each ASM layer per MDH dimension, following
// ass_re (the placement the executor realises): P[asm_layer-1][dim-1].
std::vector<std::vector<int64_t>> parts_per_asm_layer(const Config& c, const MdHom& e, const Asm& m);

std::string ty_name(Ty t);

}  // namespace mdhb
