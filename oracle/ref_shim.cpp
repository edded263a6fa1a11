// TEST INFRASTRUCTURE: a C ABI over the UNMODIFIED reference library, built by
// oracle/Makefile into oracle/_ref/libmdh_ref.so.  Only tests/, smoke() and the
// bench's cpu_baseline / --impl reference legs load it, as the checker and the
// CPU baseline -- never as the product path.
//
// Every entry point forwards to one reference API call:
//   ref_execute        -> mdh::reference_execute          (include/mdh/highlevel.hpp:62-63)
//   ref_interpret      -> mdh::interpret(mdh::lower(...))  (include/mdh/interpreter.hpp:44-46)
//   ref_emit           -> mdh::emit                        (include/mdh/codegen.hpp:38)
//   ref_compiled_time  -> mdh::compiled_time_objective     (include/mdh/autotuner.hpp:73)
//   ref_lowered        -> mdh::lower(...).pretty()                 (lowering.cpp:185-222)
//   ref_simcost        -> mdh::simcost_objective           (include/mdh/autotuner.hpp:67)
//   ref_sample_config  -> mdh::sample / ReducedSpace::sample (include/mdh/tuning.hpp:64,80)
//   ref_validate       -> mdh::validate                    (include/mdh/tuning.hpp:57)
//   ref_tune           -> mdh::tune                        (include/mdh/autotuner.hpp:38)
// Buffers cross the boundary as flat row-major int64_t / double arrays at the
// extents infer_buffer_sizes gives (views.hpp:61); outputs come with a
// per-cell defined mask (mda.hpp:25-37).
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "mdh/autotuner.hpp"
#include "mdh/codegen.hpp"
#include "mdh/error.hpp"
#include "mdh/highlevel.hpp"
#include "mdh/interpreter.hpp"
#include "mdh/json_io.hpp"
#include "mdh/lowering.hpp"
#include "mdh/tuning.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const mdh::Error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = std::string("Exception: ") + e.what();
    return 2;
  }
}

int put_string(const std::string& s, char* buf, int64_t cap, int64_t* need) {
  if (need) *need = static_cast<int64_t>(s.size()) + 1;
  if (buf && cap > 0) {
    size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return 0;
}

std::vector<std::shared_ptr<mdh::Buffer>> wrap_inputs(const mdh::HighLevelExpr& e, const void* const* in) {
  auto dims = mdh::infer_buffer_sizes(e.input_view, e.full_ranges());
  std::vector<std::shared_ptr<mdh::Buffer>> bufs;
  for (size_t b = 0; b < dims.size(); ++b) {
    const auto& vb = e.input_view.buffers[b];
    auto buf = std::make_shared<mdh::Buffer>(mdh::Buffer::make(dims[b], vb.type));
    int64_t n = buf->flat_size();
    for (int64_t t = 0; t < n; ++t) {
      auto& c = buf->data[static_cast<size_t>(t)];
      c.type = vb.type;
      if (vb.type == mdh::ScalarType::Int64)
        c.i = static_cast<const int64_t*>(in[b])[t];
      else
        c.f = static_cast<const double*>(in[b])[t];
      buf->defined[static_cast<size_t>(t)] = 1;
    }
    bufs.push_back(buf);
  }
  return bufs;
}

void unwrap_outputs(const std::vector<std::shared_ptr<mdh::Buffer>>& outs, void* const* out, uint8_t* const* def) {
  for (size_t b = 0; b < outs.size(); ++b) {
    const mdh::Buffer& buf = *outs[b];
    int64_t n = buf.flat_size();
    for (int64_t t = 0; t < n; ++t) {
      const auto& c = buf.data[static_cast<size_t>(t)];
      if (buf.elem_type == mdh::ScalarType::Int64)
        static_cast<int64_t*>(out[b])[t] = c.i;
      else
        static_cast<double*>(out[b])[t] = c.f;
      if (def && def[b]) def[b][t] = buf.defined[static_cast<size_t>(t)];
    }
  }
}

mdh::TuningConfig config_of(const mdh::HighLevelExpr& e, const mdh::AsmModel& m, const char* cfg) {
  if (!cfg || !*cfg) return mdh::baseline_config(e, m);
  return mdh::parse_config_json(cfg, e, m);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// side 0 = inputs, 1 = outputs.  dims must hold >= 16 entries.
int ref_buffer_info(const char* comp_json, int side, int b, int64_t* dims, int* rank, int* is_float) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    const mdh::ViewSpec& v = side == 0 ? e.input_view : e.output_view;
    auto all = side == 0 ? mdh::infer_buffer_sizes(v, e.full_ranges())
                         : mdh::infer_buffer_sizes(v, mdh::collapsed_ranges(e));
    if (b < 0 || b >= static_cast<int>(all.size())) mdh::fail("OutOfRange", "buffer index");
    *rank = static_cast<int>(all[static_cast<size_t>(b)].size());
    for (int r = 0; r < *rank; ++r) dims[r] = all[static_cast<size_t>(b)][static_cast<size_t>(r)];
    *is_float = v.buffers[static_cast<size_t>(b)].type == mdh::ScalarType::Float64;
  });
}

int ref_execute(const char* comp_json, const void* const* in, void* const* out, uint8_t* const* def) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    unwrap_outputs(mdh::reference_execute(e, wrap_inputs(e, in)), out, def);
  });
}

int ref_interpret(const char* comp_json, const char* asm_arg, const char* cfg_json, const void* const* in,
                  void* const* out, uint8_t* const* def) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    mdh::TuningConfig c = config_of(e, m, cfg_json);
    unwrap_outputs(mdh::interpret(mdh::lower(e, m, c), e, wrap_inputs(e, in)).first, out, def);
  });
}

int ref_emit(const char* comp_json, const char* asm_arg, const char* cfg_json, char* buf, int64_t cap,
             int64_t* need) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    put_string(mdh::emit(mdh::lower(e, m, config_of(e, m, cfg_json)), e), buf, cap, need);
  });
}

int ref_lowered(const char* comp_json, const char* asm_arg, const char* cfg_json, char* buf, int64_t cap,
                int64_t* need) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    put_string(mdh::lower(e, m, config_of(e, m, cfg_json)).pretty(), buf, cap, need);
  });
}

int ref_compiled_time(const char* comp_json, const char* asm_arg, const char* cfg_json, double* secs) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    *secs = mdh::compiled_time_objective(e, m, config_of(e, m, cfg_json));
  });
}

int ref_simcost(const char* comp_json, const char* asm_arg, const char* cfg_json, double* cost) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    *cost = mdh::simcost_objective(e, m, config_of(e, m, cfg_json));
  });
}

int ref_sample_config(const char* comp_json, const char* asm_arg, uint64_t seed, int reduced, int model_rules,
                      char* buf, int64_t cap, int64_t* need) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    mdh::ModelConstraintSet cs = model_rules ? mdh::ModelConstraintSet::for_model(m) : mdh::ModelConstraintSet::none();
    mdh::TuningConfig c;
    if (reduced) {
      mdh::ReducedSpace rs = mdh::reduce_space(e, m);
      rs.constraints = cs;
      mdh::Rng rng(seed);
      c = rs.sample(rng);
    } else {
      c = mdh::sample(e, m, cs, seed);
    }
    put_string(mdh::config_to_json(c, e, m), buf, cap, need);
  });
}

// Returns 0 and writes "" when valid; writes "<rule>: <message>" of the first
// violation otherwise (still returning 0); nonzero only on parse errors.
int ref_validate(const char* comp_json, const char* asm_arg, const char* cfg_json, int model_rules, char* buf,
                 int64_t cap, int64_t* need) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    mdh::ModelConstraintSet cs = model_rules ? mdh::ModelConstraintSet::for_model(m) : mdh::ModelConstraintSet::none();
    mdh::ValidationReport r = mdh::validate(mdh::parse_config_json(cfg_json, e, m), e, m, cs);
    put_string(r.ok ? std::string() : r.violations[0].code + ": " + r.violations[0].message, buf, cap, need);
  });
}

int ref_fixture(const char* name, char* comp_buf, int64_t comp_cap, char* cfg_buf, int64_t cfg_cap, char* asm_buf,
                int64_t asm_cap) {
  return guard([&] {
    mdh::Fixture f = mdh::fixture(name);
    mdh::HighLevelExpr e = mdh::bundled_computation(f.spec_name);
    e.sizes = f.sizes;
    put_string(mdh::computation_to_json(e), comp_buf, comp_cap, nullptr);
    put_string(mdh::config_to_json(f.config, e, f.model), cfg_buf, cfg_cap, nullptr);
    put_string(f.model.name, asm_buf, asm_cap, nullptr);
  });
}

int ref_tune(const char* comp_json, const char* asm_arg, int budget, int compiled, uint64_t seed, char* best,
             int64_t best_cap, char* hist, int64_t hist_cap, double* best_obj) {
  return guard([&] {
    mdh::HighLevelExpr e = mdh::parse_computation_json(comp_json);
    mdh::AsmModel m = mdh::resolve_asm(asm_arg);
    mdh::TuneResult r = mdh::tune(e, m, mdh::ModelConstraintSet::for_model(m), budget,
                                  compiled ? mdh::Objective::CompiledTime : mdh::Objective::SimCost, seed);
    put_string(mdh::config_to_json(r.best, e, m), best, best_cap, nullptr);
    put_string(mdh::history_csv(r), hist, hist_cap, nullptr);
    *best_obj = r.best_objective;
  });
}

}  // extern "C"
