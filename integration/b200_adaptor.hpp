// Reference-side binding of the B200 backend: what a maintainer of the
// reference adds to its tree (e.g. proj/include/mdh/b200.hpp) to call the
// sm_100a executor through its C ABI (include/mdh_b200.h) with the
// reference's own types.  It compiles against the UNMODIFIED reference
// headers (/root/reference/proj/include) and links the reference library
// plus libmdh_b200.so; oracle/Makefile's `adaptor` target builds it here.
//
//   reference                                         drop-in here
//   ------------------------------------------------  -----------------------------------
//   reference_execute(e, inputs)  highlevel.hpp:62    b200::execute(e, inputs)
//   interpret(lower(e, m, cfg), e, inputs).outputs    b200::execute(e, m, cfg, inputs)
//     interpreter.hpp:44-46
//   compiled_time_objective(e, m, cfg)                b200::time_objective(e, m, cfg)
//     autotuner.hpp:73
//   EvaluateFn for hill_climb        autotuner.hpp:44  b200::time_evaluator(e, m)
//   tune(e, m, cs, budget, Objective::CompiledTime,   b200::tune(e, m, cs, budget, seed)
//        seed)  autotuner.hpp:40
#pragma once

#include <memory>
#include <optional>
#include <vector>

#include "mdh/asm_model.hpp"
#include "mdh/autotuner.hpp"
#include "mdh/highlevel.hpp"
#include "mdh/tuning.hpp"

namespace mdh::b200 {

struct Options {
  bool f64_storage = true;  // f64 buffers stored as double on the device (bit-identical to the oracle);
                            // false = FP32 storage (the BASELINE configs' arithmetic)
  int math = 0;             // 0 FFMA, 1 TF32, 2 BF16 (contraction family)
  int device = 0;
};

// reference_execute's contract: outputs at the inferred extents, defined
// exactly where the output view writes; mdh::Error with the reference's
// codes on failure (the C ABI's "<Code>: message" is rethrown).
std::vector<std::shared_ptr<Buffer>> execute(const HighLevelExpr& e, const std::vector<std::shared_ptr<Buffer>>& inputs,
                                             const Options& o = {});
// The configuration-ordered form (interpret(lower(...))): the plan is
// instantiated from (model, config).
std::vector<std::shared_ptr<Buffer>> execute(const HighLevelExpr& e, const AsmModel& m, const TuningConfig& cfg,
                                             const std::vector<std::shared_ptr<Buffer>>& inputs, const Options& o = {});

// compiled_time_objective's role: median seconds of the instantiated kernel
// on the plan's synthetic t % 7 + 1 inputs, CUDA events, L2 flushed (mdh_b200_time_synthetic).
double time_objective(const HighLevelExpr& e, const AsmModel& m, const TuningConfig& cfg, const Options& o = {});
// ... as the EvaluateFn hill_climb takes: nullopt never (failures -> +inf, as tune() records them)
EvaluateFn time_evaluator(const HighLevelExpr& e, const AsmModel& m, const Options& o = {});

// tune(..., Objective::CompiledTime, seed) with the device objective, from the
// reference's own search pieces: reduce_space().sample for 3/10 of the budget,
// then hill_climb over default_neighborhood, config_hash ties, exactly
// `budget` history rows.
TuneResult tune(const HighLevelExpr& e, const AsmModel& m, const ModelConstraintSet& cs, int budget, uint64_t seed,
                const Options& o = {});

}  // namespace mdh::b200
