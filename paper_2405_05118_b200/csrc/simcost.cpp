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
