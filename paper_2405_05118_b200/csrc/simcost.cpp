// SimCost: the reference's input-free cost model of a Table-1 configuration
// (simulate_trace + cost, proj/src/interpreter.cpp:70-241; objective
// simcost_objective, proj/src/autotuner.cpp:58-62), restated over this
// repo's Config so the tuner can rank candidates without running them
// (SimCost-seeded tuning).
//
// Trace (per lowered step, lowering.cpp:56-118):
//   iv      every input footprint moves DM (region 1) -> the first de level's region
//   de k    a buffer moves when its (region, layout) differs from level k-1's
//   scalar  each access of each point reads its scalar-input region once; each
//           output access writes its scalar-output region once
//   re k    partials move from the next-inner staging (or the scalar output)
//           when (region, layout) differs
//   ov      the outermost re staging -> region 1
// Every move charges its element count to BOTH regions; fan-out counts a
// level's parts only when its ASM layer is a memory layer (step_fanout).
// cost = sum_r 2^(M - r + 1) * traffic_r (ascending r) + 1.0 * (de + scalar
// + re fan-out + 2).
#include <cmath>
#include <map>
#include <numeric>
#include <sstream>

#include "plan.hpp"

namespace mdhb {

namespace {

int64_t footprint(const std::vector<int64_t>& dims) {
  return std::accumulate(dims.begin(), dims.end(), int64_t{1}, std::multiplies<int64_t>());
}

}  // namespace

SimTrace simulate(const Config& c, const MdHom& e, const Asm& m) {
  std::string why = config_violation(c, e, m, false);
  if (!why.empty()) fail("InvalidConfig", "configuration violates \"" + why.substr(0, why.find(':')) + "\": " +
                                              (why.find(": ") == std::string::npos ? why : why.substr(why.find(": ") + 2)));
  const int D = static_cast<int>(e.sizes.size());
  const int M = m.M();
  auto parts = [&](const Level& l) { return c.parts[static_cast<size_t>(l.layer - 1)][static_cast<size_t>(l.dim - 1)]; };
  auto fanout = [&](const Level& asm_level, int64_t p) { return asm_level.layer <= M ? p : int64_t{1}; };
  auto rank = [&](const Level& l) { return (l.layer - 1) * D + (l.dim - 1); };

  std::vector<int64_t> in_fp, out_fp;
  for (const auto& dims : infer_extents(e.in, e.sizes)) in_fp.push_back(footprint(dims));
  for (const auto& dims : infer_extents(e.out, e.collapsed())) out_fp.push_back(footprint(dims));
  const int64_t n_total = footprint(e.sizes);

  SimTrace t;
  auto charge = [&](int from, int to, int64_t n) {
    t.reads += n;
    t.writes += n;
    t.traffic[from] += n;
    t.traffic[to] += n;
  };
  int64_t de_fan = 1, sc_fan = 1, re_fan = 1;

  // de-composition
  const size_t nde = c.ord_de.size();
  for (size_t b = 0; b < in_fp.size() && nde > 0; ++b)
    charge(1, c.mem_de[b][static_cast<size_t>(rank(c.ord_de[0]))], in_fp[b]);
  for (size_t k = 0; k < nde; ++k) {
    const Level& lv = c.ord_de[k];
    const int r = rank(lv);
    de_fan *= fanout(c.ass_de[static_cast<size_t>(r)], parts(lv));
    if (k >= 1) {
      const int rp = rank(c.ord_de[k - 1]);
      for (size_t b = 0; b < in_fp.size(); ++b) {
        const int r0 = c.mem_de[b][static_cast<size_t>(rp)], r1 = c.mem_de[b][static_cast<size_t>(r)];
        if (r0 != r1 || c.layout_de[b][static_cast<size_t>(rp)] != c.layout_de[b][static_cast<size_t>(r)]) charge(r0, r1, in_fp[b]);
      }
    }
  }
  // scalar phase
  for (size_t b = 0; b < e.in.size(); ++b) {
    const int64_t n = n_total * static_cast<int64_t>(e.in[b].acc.size());
    t.reads += n;
    t.traffic[c.mem_scalar_in[b]] += n;
  }
  for (size_t b = 0; b < e.out.size(); ++b) {
    const int64_t n = n_total * static_cast<int64_t>(e.out[b].acc.size());
    t.writes += n;
    t.traffic[c.mem_scalar_out[b]] += n;
  }
  for (size_t r = 0; r < c.ass_scalar.size(); ++r) {
    const Level lv{static_cast<int>(r) / D + 1, static_cast<int>(r) % D + 1};
    sc_fan *= fanout(c.ass_scalar[r], parts(lv));
  }
  // re-composition (levels inner -> outer as listed in ord_re), then ov
  const size_t nre = c.ord_re.size();
  for (size_t k = 0; k < nre; ++k) {
    const Level& lv = c.ord_re[k];
    const int r = rank(lv);
    re_fan *= fanout(c.ass_re[static_cast<size_t>(r)], parts(lv));
    for (size_t b = 0; b < out_fp.size(); ++b) {
      int ri;
      const std::vector<int>* li;
      if (k + 1 < nre) {
        const int rn = rank(c.ord_re[k + 1]);
        ri = c.mem_re[b][static_cast<size_t>(rn)];
        li = &c.layout_re[b][static_cast<size_t>(rn)];
      } else {
        ri = c.mem_scalar_out[b];
        li = &c.layout_scalar_out[b];
      }
      const int ro = c.mem_re[b][static_cast<size_t>(r)];
      if (ri != ro || *li != c.layout_re[b][static_cast<size_t>(r)]) charge(ri, ro, out_fp[b]);
    }
  }
  for (size_t b = 0; b < out_fp.size() && nre > 0; ++b)
    charge(c.mem_re[b][static_cast<size_t>(rank(c.ord_re[0]))], 1, out_fp[b]);
  t.depth = de_fan + sc_fan + re_fan + 2;
  return t;
}

double simcost(const SimTrace& t, const Asm& m) {
  double total = 0.0;
  for (const auto& kv : t.traffic) total += std::ldexp(1.0, m.M() - kv.first + 1) * static_cast<double>(kv.second);
  return total + 1.0 * static_cast<double>(t.depth);
}

// The lowered form's pretty text (LowLevelExpr::pretty, lowering.cpp:185-222;
// steps as lower() builds them, lowering.cpp:56-118): one de line per level in
// ord_de after the "iv" view stage, the scalar line, one re line per level in
// ord_re, then the "ov" view stage.
std::string lowered_text(const Config& c, const MdHom& e, const Asm& m) {
  std::string why = config_violation(c, e, m, false);
  if (!why.empty()) fail("InvalidConfig", "configuration violates \"" + why.substr(0, why.find(':')) + "\": " +
                                              (why.find(": ") == std::string::npos ? why : why.substr(why.find(": ") + 2)));
  const int D = e.D();
  auto letter = [](int d) { return d == 1 ? std::string("x") : d == 2 ? std::string("y") : d == 3 ? std::string("z") : "d" + std::to_string(d); };
  auto lvl = [&](const Level& l) { return "(" + std::to_string(l.layer) + "," + letter(l.dim) + ")"; };
  auto tag = [&](const Level& a) { return "(" + m.layer(a.layer) + "," + letter(a.dim) + ")"; };
  auto perm = [](const std::vector<int>& v) {
    std::string s = "(";
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    return s + ")";
  };
  auto rank = [&](const Level& l) { return (l.layer - 1) * D + (l.dim - 1); };
  auto opname = [](Fold f) {
    switch (f) {
      case Fold::Add: return "+";
      case Fold::Sub: return "-";
      case Fold::Mul: return "*";
      case Fold::Div: return "/";
      case Fold::Min: return "min";
      default: return "max";
    }
  };
  auto comb = [&](int dim) {
    const Combine& cb = e.comb[static_cast<size_t>(dim - 1)];
    if (cb.kind == Combine::CC) return std::string("cc");
    return std::string(cb.kind == Combine::PW ? "pw:" : "ps:") +
           (cb.op == Fold::Custom ? combine_at(cb.custom).name : std::string(opname(cb.op)));
  };
  std::ostringstream o;
  o << "lowered computation=" << e.name << " model=" << m.name << "\n";
  auto step = [&](const char* ph, const Level& l, const Level& a, const std::string& op, const std::vector<Buf>& bufs,
                  const std::vector<std::vector<int>>& mem, const std::vector<std::vector<std::vector<int>>>& lay) {
    const int r = rank(l);
    o << ph << " level=" << lvl(l) << " tag=" << tag(a) << " parts="
      << c.parts[static_cast<size_t>(l.layer - 1)][static_cast<size_t>(l.dim - 1)] << " op=" << op << " mem=[";
    for (size_t b = 0; b < bufs.size(); ++b)
      o << (b ? ", " : "") << bufs[b].name << ":" << m.layer(mem[b][static_cast<size_t>(r)]);
    o << "] layout=[";
    for (size_t b = 0; b < bufs.size(); ++b)
      o << (b ? ", " : "") << bufs[b].name << ":" << perm(lay[b][static_cast<size_t>(r)]);
    o << "]\n";
  };
  o << "de level=(-) tag=(-) op=iv\n";
  for (const Level& l : c.ord_de) step("de", l, c.ass_de[static_cast<size_t>(rank(l))], "cc_inv", e.in, c.mem_de, c.layout_de);
  o << "scalar level=(-) tag=(-) op=f ord=[";
  for (size_t i = 0; i < c.ord_scalar.size(); ++i) o << (i ? ", " : "") << lvl(c.ord_scalar[i]);
  o << "] ass=[";
  for (size_t i = 0; i < c.ass_scalar.size(); ++i) o << (i ? ", " : "") << tag(c.ass_scalar[i]);
  o << "] mem=[";
  for (size_t b = 0; b < e.in.size(); ++b) o << (b ? ", " : "") << "in " << e.in[b].name << ":" << m.layer(c.mem_scalar_in[b]);
  for (size_t b = 0; b < e.out.size(); ++b)
    o << (b || !e.in.empty() ? ", " : "") << "out " << e.out[b].name << ":" << m.layer(c.mem_scalar_out[b]);
  o << "] layout=[";
  for (size_t b = 0; b < e.in.size(); ++b) o << (b ? ", " : "") << "in " << e.in[b].name << ":" << perm(c.layout_scalar_in[b]);
  for (size_t b = 0; b < e.out.size(); ++b)
    o << (b || !e.in.empty() ? ", " : "") << "out " << e.out[b].name << ":" << perm(c.layout_scalar_out[b]);
  o << "]\n";
  for (const Level& l : c.ord_re) step("re", l, c.ass_re[static_cast<size_t>(rank(l))], comb(l.dim), e.out, c.mem_re, c.layout_re);
  o << "re level=(-) tag=(-) op=ov\n";
  return o.str();
}

std::string SimTrace::json(const Asm& m) const {
  std::ostringstream os;
  os << "{\"reads\": " << reads << ", \"writes\": " << writes << ", \"parallel_depth\": " << depth << ", \"regions\": {";
  bool first = true;
  for (const auto& kv : traffic) {
    os << (first ? "" : ", ") << "\"" << m.layer(kv.first) << "\": " << kv.second;
    first = false;
  }
  os << "}}";
  return os.str();
}

}  // namespace mdhb
