/*
 * mdh_b200.h -- the drop-in C ABI of the B200 MDH executor.
 *
 * The reference executes an md_hom on the CPU in two ways, and this ABI
 * replaces both with sm_100a kernels behind one plan object:
 *
 *   reference                                             B200 replacement
 *   ----------------------------------------------------  ---------------------------
 *   mdh::reference_execute(expr, inputs)                  mdh_b200_plan_create (no config)
 *     proj/include/mdh/highlevel.hpp:62-63                + mdh_b200_run / mdh_b200_run_host
 *   mdh::interpret(mdh::lower(expr, model, cfg), ...)     mdh_b200_plan_create (with config)
 *     proj/include/mdh/interpreter.hpp:44-46,             + mdh_b200_run
 *     proj/include/mdh/lowering.hpp:71
 *   void mdh_kernel(const T* in..., T* out...)            mdh_b200_run (same argument order:
 *     emitted by mdh::emit, proj/include/mdh/codegen.hpp:38;  inputs then outputs, in view order,
 *     golden proj/data/golden/emitted_matvec_openmp.c:41   flat row-major at infer_buffer_sizes
 *                                                          extents, views.hpp:61)
 *   mdh::compile_and_run(program)                         mdh_b200_plan_create (kernel selection
 *     proj/include/mdh/codegen.hpp:47                     and instantiation; no host compiler)
 *   mdh::compiled_time_objective(expr, model, cfg)        mdh_b200_time (CUDA-event median,
 *     proj/include/mdh/autotuner.hpp:73                   L2 flushed between reps)
 *   mdh::tune(expr, model, cs, budget, objective, seed)   mdh_b200_tune (on-device objective)
 *     proj/include/mdh/autotuner.hpp:38
 *   mdh::validate(cfg, expr, model, constraints)          mdh_b200_validate_config
 *     proj/include/mdh/tuning.hpp:57
 *   mdh::lower(expr, model, cfg).pretty()                  mdh_b200_lowered (host only)
 *     proj/include/mdh/lowering.hpp:71
 *   mdh::simcost_objective(expr, model, cfg)              mdh_b200_simcost (host only)
 *     proj/include/mdh/autotuner.hpp:67;                  mdh_b200_tune_ex (objective choice,
 *     tune(..., Objective::SimCost, ...)                    SimCost seeding, start config)
 *
 * Inputs are the reference's own JSON texts, unchanged: the computation
 * (proj/src/json_io.cpp:298-328), an ASM preset name or inline ASM JSON
 * (json_io.cpp:477-488; the presets of asm_model.cpp:23-43 plus "B200" and
 * "MultiB200"), and a tuning configuration (json_io.cpp:128-237).
 *
 * Element storage: the reference's value model is i64/f64 (value.hpp:12).
 * On the device, f64-typed buffers are stored as float (MDH_B200_F32, the
 * default) or double; i64-typed buffers as int32 (MDH_B200_I32) or int64
 * (default).  mdh_b200_buffer_info reports what the plan expects.
 *
 * Errors: every call returns 0 on success and 1 on failure; the failure's
 * stable code and message (the reference's mdh::Error codes, error.hpp:9-17,
 * plus CudaError / Unsupported) are available from mdh_b200_last_error()
 * ("<Code>: <message>", thread-local).  There is no CPU fallback: a plan
 * whose kernels cannot run on the device fails loudly.
 */
#ifndef MDH_B200_H
#define MDH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mdh_b200_plan mdh_b200_plan;

enum mdh_b200_dtype { MDH_B200_F32 = 0, MDH_B200_F64 = 1, MDH_B200_I32 = 2, MDH_B200_I64 = 3 };

/* Arithmetic of the dense-contraction family (MatMul, MCC, CCSD(T), ...). */
enum mdh_b200_math {
  MDH_B200_MATH_FFMA = 0, /* FP32 FFMA on the CUDA cores */
  MDH_B200_MATH_TF32 = 1, /* tcgen05.mma kind::tf32, FP32 accumulate in TMEM */
  MDH_B200_MATH_BF16 = 2  /* tcgen05.mma kind::f16 on BF16-rounded operands, FP32 accumulate */
};

typedef struct {
  int float_storage; /* MDH_B200_F32 (default) or MDH_B200_F64 for f64-typed buffers */
  int int_storage;   /* MDH_B200_I64 (default) or MDH_B200_I32 for i64-typed buffers */
  int math;          /* enum mdh_b200_math, contraction family only */
  int device;        /* CUDA device ordinal the plan lives on */
  int family;        /* 0 = auto; 1 = force the generic md_hom kernel */
  int split_dim;     /* DEV layer (mplan / rank plans): 1-based dimension the GPU layer splits, 0 = automatic */
} mdh_b200_options;

/* Fills the defaults: F32 / I64 storage, FFMA math, device 0, auto family, automatic split. */
void mdh_b200_default_options(mdh_b200_options* opt);

/* Builds a plan: parses + validates the md_hom, checks the configuration
 * (NULL/"" = the planner's default for the selected kernel template),
 * selects and instantiates the sm_100a kernel template, allocates scratch. */
int mdh_b200_plan_create(const char* computation_json, const char* asm_model, const char* config_json,
                         const mdh_b200_options* opt, mdh_b200_plan** out);
int mdh_b200_plan_destroy(mdh_b200_plan* plan);

/* side 0 = inputs, 1 = outputs.  dims needs room for 16 entries. */
int mdh_b200_buffer_count(const mdh_b200_plan* plan, int side, int* count);
int mdh_b200_buffer_info(const mdh_b200_plan* plan, int side, int index, int64_t* dims, int* rank, int* dtype,
                         int64_t* bytes);

/* Device-resident execution, asynchronous on `stream` (a cudaStream_t, NULL =
 * the legacy default stream).  d_in / d_out hold device pointers in view
 * order -- the mdh_kernel argument order. */
int mdh_b200_run(mdh_b200_plan* plan, const void* const* d_in, void* const* d_out, void* stream);

/* End-to-end execution on HOST buffers (pinned or pageable): host->device
 * copies, the kernels, device->host copies, then a stream synchronize.
 * Copies are chunked and overlapped with compute where the kernel family
 * partitions along a concatenation dimension. */
int mdh_b200_run_host(mdh_b200_plan* plan, const void* const* h_in, void* const* h_out, void* stream);

/* The on-device objective (compiled_time_objective's role): `warmup` untimed
 * runs, then `reps` runs each bracketed by CUDA events, the L2 flushed
 * before every rep when flush_l2 != 0.  Writes the median seconds and, when
 * kernel_s is non-NULL, the median of the dominant kernel alone. */
int mdh_b200_time(mdh_b200_plan* plan, const void* const* d_in, void* const* d_out, int warmup, int reps,
                  int flush_l2, double* median_s, double* kernel_s);

/* compiled_time_objective exactly (proj/src/autotuner.cpp:64-129): synthetic
 * inputs owned by the plan, element t = t % 7 + 1 as that function's
 * generated main() fills them, then mdh_b200_time on them.  What the
 * reference-side EvaluateFn binding calls. */
int mdh_b200_time_synthetic(mdh_b200_plan* plan, int warmup, int reps, int flush_l2, double* median_s,
                            double* kernel_s);

/* JSON describing the plan: family, kernel template + its parameters, the
 * normalised Table-1 configuration, launches per run, algorithmic bytes and
 * flops per run. */
int mdh_b200_describe(const mdh_b200_plan* plan, char* buf, int64_t cap, int64_t* need);

/* Structural + model rules of the configuration; writes "" when valid or
 * "<rule>: <message>" of the first violation (tuning.hpp:57). */
int mdh_b200_validate_config(const char* computation_json, const char* asm_model, const char* config_json,
                             char* buf, int64_t cap, int64_t* need);

/* On-device auto-tuning over the template-instantiable part of the Table-1
 * space: 30% random samples, then first-improving hill climbing, objective
 * = mdh_b200_time (autotuner.cpp:245-305 with the objective replaced).
 * Writes the best configuration JSON and the history CSV
 * ("eval_index,config_hash,objective,valid"). */
int mdh_b200_tune(const char* computation_json, const char* asm_model, const mdh_b200_options* opt, int budget,
                  uint64_t seed, char* best_config, int64_t best_cap, char* history_csv, int64_t hist_cap,
                  double* best_seconds);

/* Tuning objectives of mdh_b200_tune_ex (autotuner.hpp:16, Objective). */
enum { MDH_B200_OBJ_TIME = 0, MDH_B200_OBJ_SIMCOST = 1 };

/* mdh_b200_tune with the reference's objective choice and two seeding
 * aids:
 *   objective       MDH_B200_OBJ_TIME: device time (as mdh_b200_tune);
 *                   MDH_B200_OBJ_SIMCOST: the input-free SimCost model
 *                   (simcost_objective, autotuner.cpp:58-62) -- no kernel runs
 *   simcost_seeded  non-zero: the random phase samples the cheapest quarter of
 *                   the candidates by SimCost instead of the whole space
 *   start_config    NULL or a configuration JSON (e.g. the published
 *                   tvm_gpu / ppcg_gpu fixtures) evaluated first, so hill
 *                   climbing can start from it
 * History rows, tie-breaking and the budget rule are mdh_b200_tune's;
 * *best_objective is seconds (TIME) or the SimCost value (SIMCOST). */
int mdh_b200_tune_ex(const char* computation_json, const char* asm_model, const mdh_b200_options* opt, int budget,
                     uint64_t seed, int objective, int simcost_seeded, const char* start_config, char* best_config,
                     int64_t best_cap, char* history_csv, int64_t hist_cap, double* best_objective);

/* The tuner's enumerated search space for a kernel family ("stencil",
 * "contraction", "prl", ...; host only): a JSON array of the canonical Table-1
 * configurations of every template instance the family offers for this
 * md_hom (the random phase samples it; hill climbing moves with the
 * reference's four neighbourhood moves and projects each neighbour onto the
 * instance it instantiates). */
int mdh_b200_tune_space(const char* computation_json, const char* asm_model, const mdh_b200_options* opt,
                        const char* family, char* buf, int64_t cap, int64_t* need);

/* SimCost of a configuration (NULL config = the baseline configuration,
 * tuning.cpp:476-503): mdh::simcost_objective(expr, model, cfg)
 * (autotuner.cpp:58-62 = cost(simulate_trace(lower(...)), default weights
 * 2^(M-r+1), alpha 1), interpreter.cpp:70-241).  Host only, no GPU.  The
 * trace totals are written as JSON {"reads", "writes", "parallel_depth",
 * "regions": {name: elements}}. */
int mdh_b200_simcost(const char* computation_json, const char* asm_model, const char* config_json, double* cost,
                     char* trace_json, int64_t cap, int64_t* need);

/* The lowered form of (computation, model, configuration) as the
 * reference's LowLevelExpr::pretty() prints it (lowering.cpp:185-222; `mdh
 * lower`): host only.  NULL config = the baseline configuration. */
int mdh_b200_lowered(const char* computation_json, const char* asm_model, const char* config_json, char* buf,
                     int64_t cap, int64_t* need);

/* CUDA C++ source of the kernel the plan compiled at plan time (the emitted
 * family, NVRTC); "" for the precompiled template families.  The B200
 * counterpart of mdh::emit (codegen.hpp:38-53, `mdh emit`). */
int mdh_b200_kernel_source(const mdh_b200_plan* plan, char* buf, int64_t cap, int64_t* need);

/* Custom combine operators (API extension, SURVEY §8(b) "Custom combine").
 * The reference's BinOpKind is closed (proj/include/mdh/mda.hpp:52) and its
 * JSON accepts only pw:/ps: over + * min max - / (proj/src/json_io.cpp:58-64,
 * proj/src/mda.cpp:75-83).  Here a registered operator is usable as
 * "pw:<name>" / "ps:<name>" in a computation's "combine" list.  It folds the
 * TUPLE of all output components of the scalar function jointly: `cuda_body`
 * is CUDA C statements over a0..a{arity-1} (the accumulator, lvalues) and
 * b0..b{arity-1} (the next value), compiled into the md_hom's kernel by NVRTC
 * (the emitted family).  md_hom validity (Lemma 2.9) requires assoc and comm.
 * Built in: "max_prl" (arity 2: larger weight, lower record on ties --
 * PRL's custom combine), also implemented by the PRL
 * template and the device VM.  Registering an existing user operator's name
 * replaces it; plans already created keep their compiled kernel. */
int mdh_b200_register_combine(const char* name, int arity, const char* cuda_body, const char* identity_csv,
                              int assoc, int comm, const char* description);
/* JSON array describing every registered custom operator. */
int mdh_b200_combine_info(char* buf, int64_t cap, int64_t* need);

/* ---- the multi-GPU DEV layer (the reference declares the
 * MultiGPU ASM, proj/src/asm_model.cpp:36-37, and GPU partials combining in
 * host memory, but never executes them).
 *
 * The md_hom is split over the GPU layer: along the dimension a MultiB200
 * configuration gives GPU-layer parts to, else the outermost ++ dimension that
 * splits uniformly (every output depending on it), else the outermost
 * point-wise one.  A ++ split needs no communication; a point-wise split
 * combines the shards' partial outputs with the dimension's operator in device
 * memory -- ncclAllReduce over NVLink (+ * min max, distinct devices) or the
 * peer-memory combine kernel (any operator incl. max_prl; several shards may
 * share one device).  Shard g reads the slab of each global input that starts
 * at `start` along `slab_rank` (-1: the whole buffer) and, for a ++ split,
 * writes the matching slab of each output; a point-wise split leaves the
 * combined result in shard 0's outputs. */
typedef struct mdh_b200_mplan mdh_b200_mplan;
int mdh_b200_mplan_create(const char* computation_json, const char* asm_model, const char* config_json,
                          const mdh_b200_options* opt, int n_gpus, const int* device_ids, mdh_b200_mplan** out);
int mdh_b200_mplan_destroy(mdh_b200_mplan* mplan);
/* JSON: split dimension/kind, combine path ("none" | "nccl" | "peer"), each shard's range and plan. */
int mdh_b200_mplan_describe(const mdh_b200_mplan* mplan, char* buf, int64_t cap, int64_t* need);
/* Shard g's local buffer (side 0 in, 1 out): its slab of the global buffer and its shape. */
int mdh_b200_mplan_shard_buffer(const mdh_b200_mplan* mplan, int g, int side, int b, int* slab_rank, int64_t* start,
                                int64_t* dims, int* rank, int* dtype, int64_t* bytes);
int mdh_b200_mplan_shard_plan(const mdh_b200_mplan* mplan, int g, mdh_b200_plan** plan);
/* d_in[g][b] / d_out[g][b]: shard-local device buffers; streams[g] (NULL = plan-owned). */
int mdh_b200_mplan_run(mdh_b200_mplan* mplan, const void* const* const* d_in, void* const* const* d_out,
                       void* const* streams);
/* End to end on GLOBAL host buffers: slabs scattered to the devices, run, outputs gathered. */
int mdh_b200_mplan_run_host(mdh_b200_mplan* mplan, const void* const* h_in, void* const* h_out);
/* `sweeps` iterations of a halo-1 stencil (one input = output + 1-cell halo,
 * split along dimension 1): after each sweep the output is written back into
 * the input's interior and each shard's two ghost planes are exchanged with
 * its neighbours (grouped ncclSend/Recv, or peer copies; MDHB_DEV_PEER=1
 * forces the latter). */
int mdh_b200_mplan_iterate(mdh_b200_mplan* mplan, void* const* const* d_v, void* const* const* d_w, int sweeps,
                           void* const* streams);
/* Median over `reps` of the MAX over shards of each shard's event-timed run. */
int mdh_b200_mplan_time(mdh_b200_mplan* mplan, const void* const* const* d_in, void* const* const* d_out, int warmup,
                        int reps, double* median_s);

/* One process per GPU (torch.distributed / torchrun): rank `rank` of `world`
 * builds the plan of its shard (same split rule as mdh_b200_mplan_create).
 * With `nccl_id` (128 bytes from mdh_b200_nccl_unique_id on one rank,
 * broadcast by the caller) a point-wise split all-reduces its outputs over
 * NCCL inside mdh_b200_run; with NULL the caller combines.  describe() gains
 * a "shard" member (range, per-buffer slab rank and start). */
int mdh_b200_nccl_unique_id(unsigned char* id128);
/* Host only: rank `rank`'s shard as the rank plan would build it -- JSON
 * {"computation": <shard md_hom>, "config": <shard config or null>,
 *  "shard": {split_dim, split_kind, range, in/out: [slab rank, start]}}. */
int mdh_b200_shard_spec(const char* computation_json, const char* asm_model, const char* config_json, int world,
                        int rank, int split_dim, char* buf, int64_t cap, int64_t* need);
int mdh_b200_rank_plan_create(const char* computation_json, const char* asm_model, const char* config_json,
                              const mdh_b200_options* opt, int world, int rank, const unsigned char* nccl_id,
                              mdh_b200_plan** out);

/* Number of kernel launches one mdh_b200_run issues. */
int mdh_b200_launches_per_run(const mdh_b200_plan* plan, int* launches);

const char* mdh_b200_last_error(void);
const char* mdh_b200_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MDH_B200_H */
