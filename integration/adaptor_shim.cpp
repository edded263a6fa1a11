// TEST INFRASTRUCTURE: a C entry for ctypes tests of the reference-side
// binding (integration/b200_adaptor.*).  It runs the unmodified reference's
// reference_execute and mdh::b200::execute on the same inputs (the
// reference's generator, support.hpp:32-51: below(11) - 5, x0.25 for f64) and
// counts differing cells; and it drives the reference's own hill_climb /
// b200::tune with the device objective.
#include <cstring>
#include <limits>
#include <string>

#include "b200_adaptor.hpp"
#include "mdh/json_io.hpp"
#include "mdh/rng.hpp"

namespace {
thread_local std::string g_err;

int fail_with(const std::exception& ex) {
  g_err = ex.what();
  if (auto* e = dynamic_cast<const mdh::Error*>(&ex)) g_err = e->code + ": " + e->what();
  return 1;
}

std::vector<std::shared_ptr<mdh::Buffer>> make_inputs(const mdh::HighLevelExpr& e, uint64_t seed) {
  mdh::Rng rng(seed);
  auto sizes = mdh::infer_buffer_sizes(e.input_view, e.full_ranges());
  std::vector<std::shared_ptr<mdh::Buffer>> ins;
  for (size_t b = 0; b < sizes.size(); ++b) {
    const auto t = e.input_view.buffers[b].type;
    auto buf = std::make_shared<mdh::Buffer>(mdh::Buffer::make(sizes[b], t));
    for (size_t k = 0; k < buf->data.size(); ++k) {
      int64_t v = static_cast<int64_t>(rng.below(11)) - 5;
      buf->data[k].type = t;
      if (t == mdh::ScalarType::Int64) buf->data[k].i = v;
      else buf->data[k].f = 0.25 * static_cast<double>(v);
      buf->defined[k] = 1;
    }
    ins.push_back(buf);
  }
  return ins;
}

int64_t mismatches(const std::vector<std::shared_ptr<mdh::Buffer>>& a, const std::vector<std::shared_ptr<mdh::Buffer>>& b) {
  if (a.size() != b.size()) return -1;
  int64_t bad = 0;
  for (size_t k = 0; k < a.size(); ++k) {
    if (a[k]->dims != b[k]->dims) return -1;
    for (size_t t = 0; t < a[k]->data.size(); ++t) {
      if (a[k]->defined[t] != b[k]->defined[t]) {
        ++bad;
        continue;
      }
      if (!a[k]->defined[t]) continue;
      const auto &x = a[k]->data[t], &y = b[k]->data[t];
      if (x.type == mdh::ScalarType::Int64 ? x.i != y.i : x.f != y.f) ++bad;
    }
  }
  return bad;
}
}  // namespace

extern "C" {

const char* adaptor_last_error() { return g_err.c_str(); }

// reference_execute(e, in) vs b200::execute(e, in) [vs b200::execute(e, m, cfg, in)
// when asm/cfg are given]; *bad = number of differing cells (-1: shapes differ)
int adaptor_check_execute(const char* comp_json, const char* asm_name, const char* cfg_json, uint64_t seed,
                          int f64_storage, int math, int64_t* bad) {
  try {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    auto ins = make_inputs(e, seed);
    auto want = mdh::reference_execute(e, ins);
    mdh::b200::Options o;
    o.f64_storage = f64_storage != 0;
    o.math = math;
    if (asm_name && *asm_name) {
      mdh::AsmModel m = mdh::resolve_asm(asm_name);
      mdh::TuningConfig c = cfg_json && *cfg_json ? mdh::parse_config_json(cfg_json, e, m) : mdh::baseline_config(e, m);
      *bad = mismatches(mdh::b200::execute(e, m, c, ins, o), want);
    } else {
      *bad = mismatches(mdh::b200::execute(e, ins, o), want);
    }
    return 0;
  } catch (const std::exception& ex) {
    return fail_with(ex);
  }
}

// the reference's OWN hill_climb (autotuner.cpp:214-243) over its
// default_neighborhood, with the device objective as the EvaluateFn
int adaptor_hill_climb(const char* comp_json, const char* asm_name, int steps, uint64_t seed, double* start_obj,
                       double* best_obj, int* evaluations) {
  try {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_name);
    mdh::ModelConstraintSet cs = mdh::ModelConstraintSet::for_model(m);
    mdh::Rng rng(seed);
    mdh::ReducedSpace space = mdh::reduce_space(e, m);
    space.constraints = cs;
    mdh::TuningConfig start = space.sample(rng);
    auto ev = mdh::b200::time_evaluator(e, m);
    *start_obj = *ev(start);
    mdh::ClimbResult r = mdh::hill_climb(start, *start_obj, mdh::default_neighborhood(e, m, cs), ev, steps, rng);
    *best_obj = r.best_objective;
    *evaluations = r.evaluations;
    return 0;
  } catch (const std::exception& ex) {
    return fail_with(ex);
  }
}

int adaptor_tune(const char* comp_json, const char* asm_name, int budget, uint64_t seed, char* best_cfg, int64_t cap,
                 char* csv, int64_t csv_cap, double* best_obj) {
  try {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_name);
    mdh::TuneResult r = mdh::b200::tune(e, m, mdh::ModelConstraintSet::for_model(m), budget, seed);
    std::string c = mdh::config_to_json(r.best, e, m), h = mdh::history_csv(r);
    std::strncpy(best_cfg, c.c_str(), static_cast<size_t>(cap - 1));
    best_cfg[cap - 1] = '\0';
    std::strncpy(csv, h.c_str(), static_cast<size_t>(csv_cap - 1));
    csv[csv_cap - 1] = '\0';
    *best_obj = r.best_objective;
    return 0;
  } catch (const std::exception& ex) {
    return fail_with(ex);
  }
}

}  // extern "C"
