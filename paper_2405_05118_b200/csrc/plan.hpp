// Plan = an md_hom + a Table-1 configuration bound to one sm_100a kernel
// template instance.  The planner recognises the routine class of the md_hom
// (the "kernel family") and asks that family to instantiate itself from the
// configuration; every family also offers the canonical configuration of its
// default instance so callers may omit the config.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "mdh_model.hpp"

namespace mdhb {

enum class Store { F32 = 0, F64 = 1, I32 = 2, I64 = 3 };
inline size_t store_bytes(Store s) { return (s == Store::F32 || s == Store::I32) ? 4 : 8; }
inline const char* store_name(Store s) {
  switch (s) {
    case Store::F32: return "f32";
    case Store::F64: return "f64";
    case Store::I32: return "i32";
    default: return "i64";
  }
}

enum class Math { FFMA = 0, TF32 = 1, BF16 = 2 };

struct Options {
  Store fstore = Store::F32;
  Store istore = Store::I64;
  Math math = Math::FFMA;
  int device = 0;
  bool force_generic = false;
};

// Everything a family needs to know about the problem, precomputed once.
struct Problem {
  MdHom e;
  Asm m;
  Options opt;
  std::vector<std::vector<int64_t>> in_ext, out_ext;  // infer_buffer_sizes
  std::vector<Store> in_store, out_store;
  int64_t in_bytes = 0, out_bytes = 0;  // algorithmic bytes: every buffer once
  Store store_of(Ty t) const { return t == Ty::F64 ? opt.fstore : opt.istore; }
};

// One instantiated kernel template.
class Routine {
 public:
  virtual ~Routine() = default;
  virtual const char* family() const = 0;
  virtual std::string describe() const = 0;  // JSON object text (template parameters)
  virtual void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) = 0;
  virtual int launches() const = 0;
  virtual double flops() const { return 0.0; }  // algorithmic, per run
  virtual double bytes() const = 0;             // algorithmic, per run
  virtual const char* bound() const { return "hbm"; }
  // source of a kernel compiled at plan time (emitted family), else ""
  virtual std::string source() const { return ""; }
  // Chunked host<->device execution along a concatenation dimension, when
  // the family can overlap copies with compute (nullptr = whole-buffer copy).
  virtual bool supports_chunked_host() const { return false; }
  virtual void launch_host_chunked(const void* const* h_in, void* const* h_out, void* const* d_in, void* const* d_out,
                                   cudaStream_t s) {
    (void)h_in; (void)h_out; (void)d_in; (void)d_out; (void)s;
  }
  // Events recorded around the dominant kernel of launch() (mdh_b200_time's
  // kernel_s); null = not recording.  marked() says whether the last launch
  // recorded them (families whose run is one kernel leave it to the caller).
  void set_marks(cudaEvent_t a, cudaEvent_t b) {
    mark_a_ = a;
    mark_b_ = b;
    marked_ = false;
  }
  bool marked() const { return marked_; }

 protected:
  void mark_begin(cudaStream_t s) {
    if (mark_a_) cudaEventRecord(mark_a_, s);
  }
  void mark_end(cudaStream_t s) {
    if (mark_b_) {
      cudaEventRecord(mark_b_, s);
      marked_ = true;
    }
  }
  // records mark_begin now and mark_end when the scope exits (every return
  // path of a launch that follows the dominant kernel)
  struct MarkScope {
    Routine* r;
    cudaStream_t s;
    MarkScope(Routine* r_, cudaStream_t s_) : r(r_), s(s_) { r->mark_begin(s); }
    ~MarkScope() { r->mark_end(s); }
  };

 private:
  cudaEvent_t mark_a_ = nullptr, mark_b_ = nullptr;
  bool marked_ = false;
};

// Family factories.  Each returns nullptr when the md_hom is not of its
// routine class; throws Error("Unsupported", ...) when it is, but the given
// configuration is outside what its template can instantiate.  `cfg` may be
// null (use the family's default instance) -- on return, *cfg_out holds the
// canonical configuration of the chosen instance.
std::unique_ptr<Routine> make_prl(const Problem& p, const Config* cfg, Config* cfg_out);
std::unique_ptr<Routine> make_stencil(const Problem& p, const Config* cfg, Config* cfg_out);
std::unique_ptr<Routine> make_contraction(const Problem& p, const Config* cfg, Config* cfg_out);
std::unique_ptr<Routine> make_generic(const Problem& p, const Config* cfg, Config* cfg_out);
std::unique_ptr<Routine> make_scan(const Problem& p, const Config* cfg, Config* cfg_out);
std::unique_ptr<Routine> make_emitted(const Problem& p, const Config* cfg, Config* cfg_out);

// SimCost (simcost.cpp): the reference's input-free trace of a configuration
// (interpreter.cpp:70-210) and its cost (interpreter.cpp:232-241 with the
// default weights 2^(M-r+1) and alpha 1, autotuner.cpp:58-62).
struct SimTrace {
  std::map<int, int64_t> traffic;  // region id -> elements moved
  int64_t reads = 0, writes = 0, depth = 0;
  std::string json(const Asm& m) const;
};
SimTrace simulate(const Config& c, const MdHom& e, const Asm& m);
double simcost(const SimTrace& t, const Asm& m);
// LowLevelExpr::pretty() of lower(e, m, c) (lowering.cpp:56-118, 185-222)
std::string lowered_text(const Config& c, const MdHom& e, const Asm& m);

// The DEV layer for one process per GPU (dev_layer.cu): the rank's shard of
// the md_hom (computation JSON, shard config, a JSON "shard" member for
// describe()), and the routine wrapper that all-reduces a point-wise split's
// outputs over NCCL inside run().
std::string rank_shard(const std::string& comp_json, const Asm& m, const std::string& cfg_json, int world, int rank,
                       int split_dim, std::string* cfg_out, std::string* desc, int* fold, bool* pw);
std::unique_ptr<Routine> wrap_rank(std::unique_ptr<Routine> inner, const Problem& p, const std::string& desc, int fold,
                                   bool pw, const unsigned char* nccl_id, int world, int rank);

// The C ABI's thread-local last-error slot (abi.cu).
void set_last_error(const std::string& what);

// The candidate configurations a family can instantiate for this problem
// (the tuner's search space), canonical Table-1 form.
std::vector<Config> family_space(const Problem& p, const std::string& family);

// Table-1 configuration builder for the "B200" ASM {DM, SM, RM | SMX, WRP, CC}
// (and MultiB200 with HM/GPU).  Layer parts are given per ASM layer name;
// the MDH level order is SMX -> DM -> WRP -> CC -> SM -> RM (outer to inner),
// each MDH layer assigned to the ASM layer of the same role.
struct LayerParts {
  std::string layer;
  std::vector<int64_t> parts;  // per dimension
};
Config make_config(const Problem& p, const std::vector<LayerParts>& parts,
                   const std::vector<std::pair<std::string, std::string>>& staging_in,  // buffer -> region
                   const std::string& out_region);

// CUDA error check -> Error("CudaError", ...)
void cuda_check(cudaError_t err, const char* what);
#define MDHB_CUDA(x) ::mdhb::cuda_check((x), #x)

// Device properties cached per device.
int sm_count(int device);

}  // namespace mdhb
