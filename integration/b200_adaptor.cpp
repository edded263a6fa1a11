// mdh::b200 -- see b200_adaptor.hpp.  Reference-side code: it uses only the
// reference's public headers and the B200 C ABI.
#include "b200_adaptor.hpp"

#include <cstring>
#include <limits>
#include <string>

#include "../include/mdh_b200.h"
#include "mdh/json_io.hpp"

namespace mdh::b200 {
namespace {

[[noreturn]] void rethrow_abi() {
  std::string m = mdh_b200_last_error();
  size_t k = m.find(": ");
  if (k == std::string::npos) throw Error("CudaError", m);
  throw Error(m.substr(0, k), m.substr(k + 2));
}

void check(int rc) {
  if (rc) rethrow_abi();
}

struct Plan {
  mdh_b200_plan* p = nullptr;
  Plan(const HighLevelExpr& e, const AsmModel* m, const TuningConfig* cfg, const Options& o) {
    mdh_b200_options opt;
    mdh_b200_default_options(&opt);
    opt.float_storage = o.f64_storage ? MDH_B200_F64 : MDH_B200_F32;
    opt.int_storage = MDH_B200_I64;
    opt.math = o.math;
    opt.device = o.device;
    const std::string comp = computation_to_json(e);
    std::string asm_json, cfg_json;
    if (m) {
      // inline ASM JSON (json_io.cpp:241-254 dialect): the B200 backend's
      // resolve_asm accepts the reference's presets and inline models alike
      asm_json = "{\"name\": \"" + m->name + "\", \"mem\": [";
      for (size_t i = 0; i < m->mem_layers.size(); ++i) asm_json += (i ? ", \"" : "\"") + m->mem_layers[i] + "\"";
      asm_json += "], \"core\": [";
      for (size_t i = 0; i < m->core_layers.size(); ++i) asm_json += (i ? ", \"" : "\"") + m->core_layers[i] + "\"";
      asm_json += "]}";
    }
    if (m && cfg) cfg_json = config_to_json(*cfg, e, *m);
    check(mdh_b200_plan_create(comp.c_str(), m ? asm_json.c_str() : nullptr, cfg ? cfg_json.c_str() : nullptr, &opt, &p));
  }
  ~Plan() {
    if (p) mdh_b200_plan_destroy(p);
  }
};

// Buffer (AoS Comp + defined mask, mda.hpp:25-37) <-> the plan's flat typed storage
std::vector<char> pack(const Buffer& b, int dtype, int64_t bytes) {
  for (uint8_t d : b.defined)
    if (!d) throw Error("Mismatch", "undefined input cell (engine.cpp:145-146 rejects it too)");
  std::vector<char> out(static_cast<size_t>(bytes));
  const size_t n = b.data.size();
  for (size_t t = 0; t < n; ++t) {
    const auto& c = b.data[t];
    switch (dtype) {
      case MDH_B200_F32: reinterpret_cast<float*>(out.data())[t] = static_cast<float>(c.f); break;
      case MDH_B200_F64: reinterpret_cast<double*>(out.data())[t] = c.f; break;
      case MDH_B200_I32: reinterpret_cast<int32_t*>(out.data())[t] = static_cast<int32_t>(c.i); break;
      default: reinterpret_cast<int64_t*>(out.data())[t] = c.i; break;
    }
  }
  return out;
}

// cells the output view writes (views.cpp:242-275): every access over the
// collapsed index box
void mark_defined(const HighLevelExpr& e, size_t b, Buffer& out) {
  const auto ranges = collapsed_ranges(e);
  std::vector<int64_t> strides(out.dims.size(), 1);
  for (int r = static_cast<int>(out.dims.size()) - 2; r >= 0; --r) strides[static_cast<size_t>(r)] = strides[static_cast<size_t>(r) + 1] * out.dims[static_cast<size_t>(r) + 1];
  for (const auto& acc : e.output_view.buffers[b].accesses)
    for_each_index(ranges, [&](const std::vector<int64_t>& i) {
      int64_t off = 0;
      for (size_t r = 0; r < acc.idx.size(); ++r) off += strides[r] * acc.idx[r].eval(i);
      out.defined[static_cast<size_t>(off)] = 1;
    });
}

std::vector<std::shared_ptr<Buffer>> run(const Plan& plan, const HighLevelExpr& e, const std::vector<std::shared_ptr<Buffer>>& inputs) {
  int nin = 0, nout = 0;
  check(mdh_b200_buffer_count(plan.p, 0, &nin));
  check(mdh_b200_buffer_count(plan.p, 1, &nout));
  if (static_cast<int>(inputs.size()) != nin)
    throw Error("BufferTooSmall", "expected " + std::to_string(nin) + " input buffers, got " + std::to_string(inputs.size()));
  std::vector<std::vector<char>> hin, hout;
  std::vector<int> odt;
  for (int b = 0; b < nin; ++b) {
    int64_t dims[16], bytes = 0;
    int rank = 0, dt = 0;
    check(mdh_b200_buffer_info(plan.p, 0, b, dims, &rank, &dt, &bytes));
    const Buffer& in = *inputs[static_cast<size_t>(b)];
    if (in.dims != std::vector<int64_t>(dims, dims + rank))
      throw Error("BufferTooSmall", "input buffer " + std::to_string(b) + " does not have the inferred extents");
    hin.push_back(pack(in, dt, bytes));
  }
  std::vector<std::shared_ptr<Buffer>> outs;
  for (int b = 0; b < nout; ++b) {
    int64_t dims[16], bytes = 0;
    int rank = 0, dt = 0;
    check(mdh_b200_buffer_info(plan.p, 1, b, dims, &rank, &dt, &bytes));
    hout.emplace_back(static_cast<size_t>(bytes));
    odt.push_back(dt);
    outs.push_back(std::make_shared<Buffer>(Buffer::make(std::vector<int64_t>(dims, dims + rank),
                                                         e.output_view.buffers[static_cast<size_t>(b)].type)));
  }
  std::vector<const void*> pin;
  std::vector<void*> pout;
  for (auto& v : hin) pin.push_back(v.data());
  for (auto& v : hout) pout.push_back(v.data());
  check(mdh_b200_run_host(plan.p, pin.data(), pout.data(), nullptr));
  for (int b = 0; b < nout; ++b) {
    Buffer& o = *outs[static_cast<size_t>(b)];
    mark_defined(e, static_cast<size_t>(b), o);
    const char* src = hout[static_cast<size_t>(b)].data();
    for (size_t t = 0; t < o.data.size(); ++t) {
      auto& c = o.data[t];
      if (!o.defined[t]) continue;
      switch (odt[static_cast<size_t>(b)]) {
        case MDH_B200_F32: c.f = reinterpret_cast<const float*>(src)[t]; break;
        case MDH_B200_F64: c.f = reinterpret_cast<const double*>(src)[t]; break;
        case MDH_B200_I32: c.i = reinterpret_cast<const int32_t*>(src)[t]; break;
        default: c.i = reinterpret_cast<const int64_t*>(src)[t]; break;
      }
    }
  }
  return outs;
}

// the reference's own well-formedness check first (highlevel.cpp:72-102)
void require_md_hom(const HighLevelExpr& e) {
  ValidationReport r = validate_md_hom(e);
  if (!r.ok) throw Error(r.violations.front().code, r.violations.front().message);
}

}  // namespace

std::vector<std::shared_ptr<Buffer>> execute(const HighLevelExpr& e, const std::vector<std::shared_ptr<Buffer>>& inputs,
                                             const Options& o) {
  require_md_hom(e);
  Plan plan(e, nullptr, nullptr, o);
  return run(plan, e, inputs);
}

std::vector<std::shared_ptr<Buffer>> execute(const HighLevelExpr& e, const AsmModel& m, const TuningConfig& cfg,
                                             const std::vector<std::shared_ptr<Buffer>>& inputs, const Options& o) {
  require_md_hom(e);
  Plan plan(e, &m, &cfg, o);
  return run(plan, e, inputs);
}

double time_objective(const HighLevelExpr& e, const AsmModel& m, const TuningConfig& cfg, const Options& o) {
  Plan plan(e, &m, &cfg, o);
  double med = 0.0, ker = 0.0;
  check(mdh_b200_time_synthetic(plan.p, 1, 5, 1, &med, &ker));  // 1 warm-up + 5 timed, as autotuner.cpp:112-119
  return med;
}

EvaluateFn time_evaluator(const HighLevelExpr& e, const AsmModel& m, const Options& o) {
  return [e, m, o](const TuningConfig& cfg) -> std::optional<double> {
    try {
      return time_objective(e, m, cfg, o);
    } catch (const Error&) {
      return std::numeric_limits<double>::infinity();
    }
  };
}

TuneResult tune(const HighLevelExpr& e, const AsmModel& m, const ModelConstraintSet& cs, int budget, uint64_t seed,
                const Options& o) {
  if (budget < 1) throw Error("InvalidConfig", "tuning budget must be at least 1, got " + std::to_string(budget));
  Rng rng(seed);
  ReducedSpace space = reduce_space(e, m);
  space.constraints = cs;
  TuneResult res;
  bool have = false;
  uint64_t best_hash = 0;
  // every evaluation goes through the device objective; failures are
  // recorded as +inf / invalid rows, the budget is exact
  EvaluateFn evaluate = [&](const TuningConfig& cfg) -> std::optional<double> {
    if (static_cast<int>(res.history.size()) >= budget) return std::nullopt;
    TuneEvent ev;
    ev.eval_index = static_cast<int>(res.history.size());
    ev.config_hash = config_hash(cfg, e, m);
    try {
      ev.objective = time_objective(e, m, cfg, o);
    } catch (const Error&) {
      ev.objective = std::numeric_limits<double>::infinity();
      ev.valid = false;
    }
    res.history.push_back(ev);
    const bool better = ev.valid && (!have || ev.objective < res.best_objective ||
                                     (ev.objective == res.best_objective && ev.config_hash < best_hash));
    if (better) {
      have = true;
      res.best = cfg;
      res.best_objective = ev.objective;
      best_hash = ev.config_hash;
    }
    return ev.objective;
  };
  const int n_random = std::min(budget, std::max(1, budget * 3 / 10));
  for (int k = 0; k < n_random; ++k) evaluate(space.sample(rng));
  const NeighborhoodFn nb = default_neighborhood(e, m, cs);
  bool settled = false;
  uint64_t settled_on = 0;
  while (static_cast<int>(res.history.size()) < budget) {
    if (have && !(settled && settled_on == best_hash)) {
      ClimbResult cr = hill_climb(res.best, res.best_objective, nb, evaluate,
                                  budget - static_cast<int>(res.history.size()), rng);
      if (!cr.converged) break;
      settled = true;
      settled_on = best_hash;
    } else {
      evaluate(space.sample(rng));
    }
  }
  if (!have) throw Error("NoValidConfigFound", "every evaluated configuration failed");
  return res;
}

}  // namespace mdh::b200
