// The multi-GPU DEV layer: one md_hom split over the GPU layer of the
// MultiB200 ASM {HM, DM, SM, RM | GPU, SMX, WRP, CC}.
//
// The reference declares this layer but never executes it: the MultiGPU ASM
// (proj/src/asm_model.cpp:36-37) has no constraint set and the paper says GPU
// partial results combine in host memory.  Here:
//
//   * a ++ (cc) dimension splits with NO communication -- shard g computes
//     the md_hom restricted to its index range (the homomorphic property,
//     PAPER.md:2532-2582; test_highlevel.cpp:203-221) on its own slab of the
//     inputs and writes its own slab of the outputs;
//   * a point-wise dimension splits too, but the shards' partial results then
//     combine with the dimension's operator in device memory: an NCCL
//     all-reduce over NVLink for + * min max on distinct devices, or this
//     file's peer-memory combine kernel (any operator, including the custom
//     tuple operator max_prl, and several shards on one device), folding the
//     shards in ascending order -- the order the unsplit fold visits them;
//   * an iterated stencil keeps the split and exchanges its ghost planes
//     between neighbouring shards after every sweep (grouped ncclSend/Recv,
//     or peer copies), SURVEY 8(e).
//
// Shards are ordinary plans (abi.cu) on the shard md_hom: sizes[dim] / G and
// every idx(dim) of the scalar function rebased to the global index
// (idx(dim) + offset), so index-dependent scalars (PRL's record id) stay
// global.  Views are not rewritten: a shard's inputs are the slabs of the
// global buffers starting at coefficient * offset along the rank the split
// dimension drives (replicated when no rank depends on it), so the same views
// address the slab from 0.
//
// One process may drive all G devices (mdh_b200_mplan_*), or each process of
// a torch.distributed job drives one device (mdh_b200_rank_plan_create) with
// an NCCL communicator built from a unique id the caller broadcasts.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/mdh_b200.h"
#include "json.hpp"
#include "plan.hpp"

namespace mdhb {
namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
// The product binds NCCL at run time (libnccl.so.2: the image's system copy, or
// the one torch already loaded), so the library links without it and a
// missing NCCL is a loud NcclError only for paths that need it.
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
  char internal[128];
};
enum NcclOp { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };
enum NcclType { kInt32 = 2, kInt64 = 4, kFloat32 = 7, kFloat64 = 8 };

struct Nccl {
  bool ok = false;
  std::string why;
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p && n.why.empty()) n.why = std::string("missing NCCL symbol ") + s;
      return p;
    };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
    n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    n.ok = n.why.empty();
  });
  return n;
}

void nccl_check(int rc, const char* what) {
  if (rc != 0)
    fail("NcclError", std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(rc) : "error " + std::to_string(rc)));
}

Nccl& need_nccl() {
  Nccl& n = nccl();
  if (!n.ok) fail("NcclError", n.why);
  return n;
}

// ---------------------------------------------------------------- the split
struct Slice {
  int rank = -1;       // buffer rank the split dimension drives (-1: replicated / whole buffer)
  int64_t coeff = 0;   // its coefficient (start of shard g = coeff * offset_g)
};

struct Split {
  int dim = -1;        // 0-based md_hom dimension split over the GPU layer
  int parts = 1;
  bool pw = false;     // point-wise dimension: shards' results combine
  int fold = -1;       // MdHom::fold() of the combine
  std::vector<Slice> in, out;  // per buffer (out: only for a cc split)
};

Slice slice_of(const Buf& b, int dim) {
  Slice s;
  for (auto& acc : b.acc)
    for (int r = 0; r < b.rank; ++r) {
      int64_t c = acc.idx[static_cast<size_t>(r)].coeff[static_cast<size_t>(dim)];
      if (c == 0) continue;
      if (c < 0) fail("Unsupported", "buffer '" + b.name + "': negative coefficient on the split dimension");
      if (s.rank >= 0 && (s.rank != r || s.coeff != c))
        fail("Unsupported", "buffer '" + b.name + "': the split dimension drives two ranks");
      s.rank = r;
      s.coeff = c;
    }
  return s;
}

// Which dimension the GPU layer splits: the config's GPU-layer parts when a
// MultiB200 configuration is given, else the outermost cc dimension that
// splits uniformly with every output depending on it, else the outermost
// point-wise dimension that splits uniformly.
Split choose_split(const MdHom& e, const Asm& m, const Config* cfg, int G, int split_dim) {
  Split s;
  s.parts = G;
  auto cc_ok = [&](int d) {
    if (e.sizes[static_cast<size_t>(d)] % G) return false;
    for (auto& b : e.out)
      if (slice_of(b, d).rank < 0) return false;  // every shard would write the same cells
    return true;
  };
  if (split_dim > 0) {  // caller's choice (mdh_b200_options::split_dim)
    if (split_dim > e.D()) fail("DimOutOfRange", "split_dim " + std::to_string(split_dim) + " of a " + std::to_string(e.D()) + "-D md_hom");
    s.dim = split_dim - 1;
  } else if (cfg && m.id("GPU") > 0) {
    auto P = parts_per_asm_layer(*cfg, e, m);
    const auto& gp = P[static_cast<size_t>(m.id("GPU") - 1)];
    int64_t prod = 1;
    for (int d = 0; d < e.D(); ++d) {
      prod *= gp[static_cast<size_t>(d)];
      if (gp[static_cast<size_t>(d)] > 1) {
        if (s.dim >= 0) fail("Unsupported", "the DEV layer splits one dimension over the GPU layer");
        s.dim = d;
      }
    }
    if (prod != G) fail("InvalidConfig", "GPU-layer parts (" + std::to_string(prod) + ") != number of devices (" + std::to_string(G) + ")");
    if (G == 1) s.dim = 0;
  } else {
    for (int d = 0; d < e.D() && s.dim < 0; ++d)
      if (e.comb[static_cast<size_t>(d)].kind == Combine::CC && cc_ok(d)) s.dim = d;
    for (int d = 0; d < e.D() && s.dim < 0; ++d)
      if (e.comb[static_cast<size_t>(d)].kind == Combine::PW && e.sizes[static_cast<size_t>(d)] % G == 0) s.dim = d;
    if (s.dim < 0) fail("NonDivisible", "no dimension splits uniformly into " + std::to_string(G) + " parts");
  }
  const Combine& c = e.comb[static_cast<size_t>(s.dim)];
  if (c.kind == Combine::PS) fail("Unsupported", "a prefix (ps) dimension does not split without a carry exchange");
  if (e.sizes[static_cast<size_t>(s.dim)] % G)
    fail("NonDivisible", "dimension " + std::to_string(s.dim + 1) + " does not split into " + std::to_string(G) + " uniform parts");
  s.pw = c.kind == Combine::PW;
  s.fold = e.fold();
  if (!s.pw && G > 1 && !cc_ok(s.dim)) fail("Unsupported", "an output does not depend on the split ++ dimension");
  for (auto& b : e.in) s.in.push_back(slice_of(b, s.dim));
  for (auto& b : e.out) s.out.push_back(s.pw ? Slice{} : slice_of(b, s.dim));
  return s;
}

// idx(dim+1) -> (idx(dim+1) + off) in the scalar text
std::string rebase_idx(const std::string& text, int dim, int64_t off) {
  if (off == 0) return text;
  std::string out;
  size_t p = 0;
  while (p < text.size()) {
    if (text.compare(p, 3, "idx") == 0 && (p == 0 || !std::isalnum(static_cast<unsigned char>(text[p - 1])))) {
      size_t q = p + 3;
      while (q < text.size() && std::isspace(static_cast<unsigned char>(text[q]))) ++q;
      if (q < text.size() && text[q] == '(') {
        size_t r = q + 1;
        while (r < text.size() && std::isspace(static_cast<unsigned char>(text[r]))) ++r;
        size_t ds = r;
        while (r < text.size() && std::isdigit(static_cast<unsigned char>(text[r]))) ++r;
        size_t de = r;
        while (r < text.size() && std::isspace(static_cast<unsigned char>(text[r]))) ++r;
        if (de > ds && r < text.size() && text[r] == ')' && std::stoi(text.substr(ds, de - ds)) == dim + 1) {
          out += "(idx(" + std::to_string(dim + 1) + ") + " + std::to_string(off) + ")";
          p = r + 1;
          continue;
        }
      }
    }
    out += text[p++];
  }
  return out;
}

std::string shard_computation(const std::string& comp_json, const MdHom& e, const Split& s, int g) {
  json::Value j = json::parse(comp_json);
  const int64_t step = e.sizes[static_cast<size_t>(s.dim)] / s.parts;
  json::Value sizes = json::Value::make_arr();
  for (int d = 0; d < e.D(); ++d) sizes.push(json::Value::make_int(d == s.dim ? step : e.sizes[static_cast<size_t>(d)]));
  j.set("sizes", sizes);
  j.set("scalar", json::Value::make_str(rebase_idx(e.scalar_text, s.dim, step * g)));
  return json::dump(j);
}

std::string shard_config(const std::string& cfg_json, const MdHom& e, const MdHom& es, const Asm& m, const Split& s) {
  Config c = parse_config(cfg_json, e, m);
  const int L = m.L(), D = e.D();
  const int gpu = m.id("GPU");
  for (int r = 0; r < L * D; ++r) {
    int l = r / D, d = r % D;
    if (d == s.dim && gpu > 0 && c.ass_re[static_cast<size_t>(r)].layer == gpu) c.parts[static_cast<size_t>(l)][static_cast<size_t>(d)] = 1;
  }
  return config_json(c, es, m);
}

// ---------------------------------------------------------------- combine kernels
constexpr int kMaxShards = 16;
struct Srcs {
  const void* p[kMaxShards];
  const void* q[kMaxShards];  // second component (tuple operators)
};

template <typename T>
__device__ __forceinline__ T fold_op(int op, T a, T b) {
  switch (op) {
    case 0: return a + b;
    case 2: return a * b;
    case 4: return b < a ? b : a;
    default: return b > a ? b : a;
  }
}

// dst = src[0] (+) src[1] (+) ... (+) src[n-1], ascending shard order (the
// unsplit fold's order over the split dimension).  dst may alias src[0].
template <typename T>
__global__ void combine_shards(T* dst, Srcs s, int n, int64_t count, int op) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(s.p[0])[i];
    for (int k = 1; k < n; ++k) acc = fold_op<T>(op, acc, static_cast<const T*>(s.p[k])[i]);
    dst[i] = acc;
  }
}

// max_prl over (key, payload) pairs held in two parallel buffers
template <typename K, typename V>
__global__ void combine_shards_max_prl(K* dk, V* dv, Srcs s, int n, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    K bk = static_cast<const K*>(s.p[0])[i];
    V bv = static_cast<const V*>(s.q[0])[i];
    for (int k = 1; k < n; ++k) {
      K ck = static_cast<const K*>(s.p[k])[i];
      V cv = static_cast<const V*>(s.q[k])[i];
      if (ck > bk || (ck == bk && cv < bv)) {
        bk = ck;
        bv = cv;
      }
    }
    dk[i] = bk;
    dv[i] = bv;
  }
}

template <typename K>
void launch_max_prl_v(Store vs, void* dk, void* dv, const Srcs& s, int n, int64_t count, cudaStream_t st, int grid) {
  if (vs == Store::I32) combine_shards_max_prl<K, int32_t><<<grid, 256, 0, st>>>(static_cast<K*>(dk), static_cast<int32_t*>(dv), s, n, count);
  else combine_shards_max_prl<K, long long><<<grid, 256, 0, st>>>(static_cast<K*>(dk), static_cast<long long*>(dv), s, n, count);
}

int nccl_type(Store st) {
  switch (st) {
    case Store::F32: return kFloat32;
    case Store::F64: return kFloat64;
    case Store::I32: return kInt32;
    default: return kInt64;
  }
}

int nccl_op(int fold) {
  switch (fold) {
    case 0: return kSum;
    case 2: return kProd;
    case 4: return kMin;
    case 5: return kMax;
    default: return -1;
  }
}

int64_t numel(const std::vector<int64_t>& ext) {
  int64_t n = 1;
  for (int64_t x : ext) n *= x;
  return n;
}

}  // namespace
}  // namespace mdhb

using mdhb::Store;

// ------------------------------------------------------------------ mplan
struct mdh_b200_mplan {
  std::string comp_json;
  mdhb::MdHom e;
  mdhb::Asm m;
  mdhb::Split split;
  int G = 1;
  std::vector<int> dev;
  std::vector<mdh_b200_plan*> shard;
  std::vector<cudaStream_t> stream;  // plan-owned, one per shard (run_host / time / iterate)
  std::vector<cudaEvent_t> done;      // per shard: its kernels finished (combine dependency)
  std::vector<mdhb::ncclComm_t> comm;  // one per shard when the devices are distinct and NCCL loads
  bool distinct = true;
  std::string combine_path;            // "none" | "nccl" | "peer"
  // per shard, per buffer: dims + bytes of the shard-local buffer, slab start along the driven rank
  std::vector<std::vector<std::vector<int64_t>>> in_dims, out_dims;
  std::vector<std::vector<int64_t>> in_start, out_start;
  std::vector<std::vector<int>> in_store, out_store;
  std::vector<std::vector<int64_t>> g_in_ext, g_out_ext;  // global extents
  // run_host device buffers
  std::vector<std::vector<void*>> h_in, h_out;
};

namespace {

std::vector<int64_t> buf_dims(mdh_b200_plan* p, int side, int b, int* dtype, int64_t* bytes) {
  int64_t dims[16];
  int rank = 0;
  if (mdh_b200_buffer_info(p, side, b, dims, &rank, dtype, bytes)) mdhb::fail("Internal", mdh_b200_last_error());
  return std::vector<int64_t>(dims, dims + rank);
}

template <class F>
int guard_mp(F&& f) {
  try {
    f();
    return 0;
  } catch (const mdhb::Error& e) {
    mdhb::set_last_error(e.what());
  } catch (const std::exception& e) {
    mdhb::set_last_error(std::string("Exception: ") + e.what());
  }
  return 1;
}

void put_text(const std::string& s, char* buf, int64_t cap, int64_t* need) {
  if (need) *need = static_cast<int64_t>(s.size()) + 1;
  if (buf && cap > 0) {
    size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
}

size_t store_size(int st) { return (st == MDH_B200_F32 || st == MDH_B200_I32) ? 4 : 8; }

// Copy a slab [start, start + dims[r]) along rank r between a global buffer
// (extents gext) and a shard-local one (extents dims), as a 2-D strided copy.
void copy_slab(void* dst, const void* src, bool to_local, const std::vector<int64_t>& gext, const std::vector<int64_t>& dims,
               int r, int64_t start, size_t es, cudaMemcpyKind kind, cudaStream_t s) {
  if (r < 0) {  // replicated: the whole buffer
    MDHB_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(mdhb::numel(gext)) * es, kind, s));
    return;
  }
  int64_t outer = 1, inner = 1;
  for (int k = 0; k < r; ++k) outer *= gext[static_cast<size_t>(k)];
  for (size_t k = static_cast<size_t>(r) + 1; k < gext.size(); ++k) inner *= gext[k];
  const size_t row = static_cast<size_t>(dims[static_cast<size_t>(r)] * inner) * es;
  const size_t gpitch = static_cast<size_t>(gext[static_cast<size_t>(r)] * inner) * es;
  const size_t goff = static_cast<size_t>(start * inner) * es;
  if (to_local)
    MDHB_CUDA(cudaMemcpy2DAsync(dst, row, static_cast<const char*>(src) + goff, gpitch, row, static_cast<size_t>(outer), kind, s));
  else
    MDHB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + goff, gpitch, src, row, row, static_cast<size_t>(outer), kind, s));
}

// Combine point-wise partials: shard g's outputs d_out[g][b]; the result lands
// in shard 0's buffers (NCCL all-reduce also leaves it in every shard's).
void combine(mdh_b200_mplan* mp, void* const* const* d_out, const std::vector<cudaStream_t>& st) {
  const int G = mp->G;
  if (!mp->split.pw || G == 1) return;
  const size_t nout = mp->e.out.size();
  if (mp->combine_path == "nccl") {
    auto& n = mdhb::need_nccl();
    const int op = mdhb::nccl_op(mp->split.fold);
    mdhb::nccl_check(n.GroupStart(), "ncclGroupStart");
    for (int g = 0; g < G; ++g) {
      MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
      for (size_t b = 0; b < nout; ++b) {
        void* p = d_out[g][b];
        const int64_t cnt = mdhb::numel(mp->out_dims[static_cast<size_t>(g)][b]);
        mdhb::nccl_check(n.AllReduce(p, p, static_cast<size_t>(cnt), mdhb::nccl_type(static_cast<Store>(mp->out_store[static_cast<size_t>(g)][b])),
                                     op, mp->comm[static_cast<size_t>(g)], st[static_cast<size_t>(g)]),
                         "ncclAllReduce");
      }
    }
    mdhb::nccl_check(n.GroupEnd(), "ncclGroupEnd");
    return;
  }
  // peer-memory combine on shard 0's device, after every shard finished
  const int d0 = mp->dev[0];
  MDHB_CUDA(cudaSetDevice(d0));
  for (int g = 1; g < G; ++g) {
    MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
    MDHB_CUDA(cudaEventRecord(mp->done[static_cast<size_t>(g)], st[static_cast<size_t>(g)]));
  }
  MDHB_CUDA(cudaSetDevice(d0));
  for (int g = 1; g < G; ++g) MDHB_CUDA(cudaStreamWaitEvent(st[0], mp->done[static_cast<size_t>(g)], 0));
  const int grid = 4 * mdhb::sm_count(d0);
  const int fold = mp->split.fold;
  if (fold >= mdhb::kCustomFoldBase) {  // tuple operator over two parallel output buffers
    mdhb::Srcs s{};
    for (int g = 0; g < G; ++g) {
      s.p[g] = d_out[g][0];
      s.q[g] = d_out[g][1];
    }
    const int64_t cnt = mdhb::numel(mp->out_dims[0][0]);
    const Store ks = static_cast<Store>(mp->out_store[0][0]), vs = static_cast<Store>(mp->out_store[0][1]);
    switch (ks) {
      case Store::F32: mdhb::launch_max_prl_v<float>(vs, d_out[0][0], d_out[0][1], s, G, cnt, st[0], grid); break;
      case Store::F64: mdhb::launch_max_prl_v<double>(vs, d_out[0][0], d_out[0][1], s, G, cnt, st[0], grid); break;
      case Store::I32: mdhb::launch_max_prl_v<int32_t>(vs, d_out[0][0], d_out[0][1], s, G, cnt, st[0], grid); break;
      default: mdhb::launch_max_prl_v<long long>(vs, d_out[0][0], d_out[0][1], s, G, cnt, st[0], grid); break;
    }
    MDHB_CUDA(cudaGetLastError());
    return;
  }
  for (size_t b = 0; b < nout; ++b) {
    mdhb::Srcs s{};
    for (int g = 0; g < G; ++g) s.p[g] = d_out[g][b];
    const int64_t cnt = mdhb::numel(mp->out_dims[0][b]);
    void* dst = d_out[0][b];
    switch (static_cast<Store>(mp->out_store[0][b])) {
      case Store::F32: mdhb::combine_shards<float><<<grid, 256, 0, st[0]>>>(static_cast<float*>(dst), s, G, cnt, fold); break;
      case Store::F64: mdhb::combine_shards<double><<<grid, 256, 0, st[0]>>>(static_cast<double*>(dst), s, G, cnt, fold); break;
      case Store::I32: mdhb::combine_shards<int32_t><<<grid, 256, 0, st[0]>>>(static_cast<int32_t*>(dst), s, G, cnt, fold); break;
      default: mdhb::combine_shards<long long><<<grid, 256, 0, st[0]>>>(static_cast<long long*>(dst), s, G, cnt, fold); break;
    }
    MDHB_CUDA(cudaGetLastError());
  }
}

std::vector<cudaStream_t> streams_of(mdh_b200_mplan* mp, void* const* streams) {
  std::vector<cudaStream_t> st(static_cast<size_t>(mp->G));
  for (int g = 0; g < mp->G; ++g) st[static_cast<size_t>(g)] = streams ? static_cast<cudaStream_t>(streams[g]) : mp->stream[static_cast<size_t>(g)];
  return st;
}

void run_shards(mdh_b200_mplan* mp, const void* const* const* d_in, void* const* const* d_out, const std::vector<cudaStream_t>& st) {
  for (int g = 0; g < mp->G; ++g) {
    if (mdh_b200_run(mp->shard[static_cast<size_t>(g)], d_in[g], d_out[g], st[static_cast<size_t>(g)]))
      mdhb::fail("CudaError", std::string("shard ") + std::to_string(g) + ": " + mdh_b200_last_error());
  }
  combine(mp, d_out, st);
}

}  // namespace

extern "C" {

int mdh_b200_mplan_create(const char* comp_json, const char* asm_model, const char* config_json,
                          const mdh_b200_options* opt, int n_gpus, const int* device_ids, mdh_b200_mplan** out) {
  return guard_mp([&] {
    if (!comp_json || !out || n_gpus < 1) mdhb::fail("InvalidConfig", "null argument or n_gpus < 1");
    if (n_gpus > mdhb::kMaxShards) mdhb::fail("OutOfRange", "at most 16 shards");
    auto mp = std::make_unique<mdh_b200_mplan>();
    mp->comp_json = comp_json;
    mp->e = mdhb::parse_md_hom(comp_json);
    std::string v = mdhb::md_hom_violation(mp->e);
    if (!v.empty()) mdhb::fail("MixedIncompatibleOperators", v);
    mp->m = mdhb::resolve_asm(asm_model ? asm_model : "MultiB200");
    mp->G = n_gpus;
    for (int g = 0; g < n_gpus; ++g) mp->dev.push_back(device_ids ? device_ids[g] : g);
    std::unique_ptr<mdhb::Config> cfg;
    if (config_json && *config_json) cfg = std::make_unique<mdhb::Config>(mdhb::parse_config(config_json, mp->e, mp->m));
    mp->split = mdhb::choose_split(mp->e, mp->m, cfg.get(), n_gpus, opt ? opt->split_dim : 0);
    // the point-wise combine: NCCL when it has the operator and every shard
    // has its own device, else the peer-memory kernel
    for (int a = 0; a < n_gpus; ++a)
      for (int b = a + 1; b < n_gpus; ++b)
        if (mp->dev[static_cast<size_t>(a)] == mp->dev[static_cast<size_t>(b)]) mp->distinct = false;
    mp->combine_path = "none";
    if (mp->split.pw && n_gpus > 1) {
      bool use_nccl = mp->distinct && mdhb::nccl_op(mp->split.fold) >= 0 && mdhb::nccl().ok && !std::getenv("MDHB_DEV_PEER");
      mp->combine_path = use_nccl ? "nccl" : "peer";
      if (mp->split.fold >= mdhb::kCustomFoldBase) {
        const auto& op = mdhb::combine_at(mp->split.fold - mdhb::kCustomFoldBase);
        if (op.name != "max_prl" || mp->e.out.size() != 2)
          mdhb::fail("Unsupported", "the DEV layer combines custom operator '" + op.name + "' only as max_prl over two output buffers");
      }
    }
    mdh_b200_options o;
    if (opt) o = *opt;
    else mdh_b200_default_options(&o);
    for (int g = 0; g < n_gpus; ++g) {
      std::string sj = mdhb::shard_computation(mp->comp_json, mp->e, mp->split, g);
      std::string sc;
      if (cfg) sc = mdhb::shard_config(config_json, mp->e, mdhb::parse_md_hom(sj), mp->m, mp->split);
      o.device = mp->dev[static_cast<size_t>(g)];
      mdh_b200_plan* p = nullptr;
      // shard plans: the configuration's own ASM when one is given (its GPU
      // parts set to 1), else the single-device B200 ASM for a MultiB200 split
      const std::string shard_asm = cfg ? (asm_model ? std::string(asm_model) : mp->m.name)
                                        : (mp->m.name == "MultiB200" ? std::string("B200")
                                                                     : (asm_model ? std::string(asm_model) : std::string("B200")));
      if (mdh_b200_plan_create(sj.c_str(), shard_asm.c_str(), cfg ? sc.c_str() : nullptr, &o, &p))
        mdhb::fail("Internal", std::string("shard ") + std::to_string(g) + ": " + mdh_b200_last_error());
      mp->shard.push_back(p);
      cudaStream_t s;
      MDHB_CUDA(cudaSetDevice(o.device));
      MDHB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      mp->stream.push_back(s);
      cudaEvent_t ev;
      MDHB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      mp->done.push_back(ev);
      std::vector<std::vector<int64_t>> id, od;
      std::vector<int> is, os;
      std::vector<int64_t> ist, ost;
      int nin = 0, nout = 0;
      mdh_b200_buffer_count(p, 0, &nin);
      mdh_b200_buffer_count(p, 1, &nout);
      const int64_t off = mp->e.sizes[static_cast<size_t>(mp->split.dim)] / n_gpus * g;
      for (int b = 0; b < nin; ++b) {
        int dt = 0;
        int64_t by = 0;
        id.push_back(buf_dims(p, 0, b, &dt, &by));
        is.push_back(dt);
        ist.push_back(mp->split.in[static_cast<size_t>(b)].coeff * off);
      }
      for (int b = 0; b < nout; ++b) {
        int dt = 0;
        int64_t by = 0;
        od.push_back(buf_dims(p, 1, b, &dt, &by));
        os.push_back(dt);
        ost.push_back(mp->split.out[static_cast<size_t>(b)].coeff * off);
      }
      mp->in_dims.push_back(id);
      mp->out_dims.push_back(od);
      mp->in_store.push_back(is);
      mp->out_store.push_back(os);
      mp->in_start.push_back(ist);
      mp->out_start.push_back(ost);
    }
    mp->g_in_ext = mdhb::infer_extents(mp->e.in, mp->e.sizes);
    mp->g_out_ext = mdhb::infer_extents(mp->e.out, mp->e.collapsed());
    // peer access for the combine kernel / halo copies (distinct devices)
    if (n_gpus > 1 && mp->distinct) {
      for (int a = 0; a < n_gpus; ++a)
        for (int b = 0; b < n_gpus; ++b) {
          if (a == b) continue;
          int can = 0;
          cudaDeviceCanAccessPeer(&can, mp->dev[static_cast<size_t>(a)], mp->dev[static_cast<size_t>(b)]);
          if (!can) continue;
          cudaSetDevice(mp->dev[static_cast<size_t>(a)]);
          cudaError_t err = cudaDeviceEnablePeerAccess(mp->dev[static_cast<size_t>(b)], 0);
          if (err != cudaSuccess && err != cudaErrorPeerAccessAlreadyEnabled) MDHB_CUDA(err);
          cudaGetLastError();
        }
      if (mdhb::nccl().ok && !std::getenv("MDHB_DEV_PEER")) {
        mp->comm.resize(static_cast<size_t>(n_gpus));
        mdhb::nccl_check(mdhb::nccl().CommInitAll(mp->comm.data(), n_gpus, mp->dev.data()), "ncclCommInitAll");
      }
    }
    *out = mp.release();
  });
}

int mdh_b200_mplan_destroy(mdh_b200_mplan* mp) {
  return guard_mp([&] {
    if (!mp) return;
    for (auto c : mp->comm)
      if (c) mdhb::nccl().CommDestroy(c);
    for (size_t g = 0; g < mp->shard.size(); ++g) {
      cudaSetDevice(mp->dev[g]);
      for (void* p : g < mp->h_in.size() ? mp->h_in[g] : std::vector<void*>{}) cudaFree(p);
      for (void* p : g < mp->h_out.size() ? mp->h_out[g] : std::vector<void*>{}) cudaFree(p);
      cudaStreamDestroy(mp->stream[g]);
      cudaEventDestroy(mp->done[g]);
      mdh_b200_plan_destroy(mp->shard[g]);
    }
    delete mp;
  });
}

int mdh_b200_mplan_describe(const mdh_b200_mplan* mp, char* buf, int64_t cap, int64_t* need) {
  return guard_mp([&] {
    std::ostringstream os;
    const auto& s = mp->split;
    os << "{\"n_gpus\": " << mp->G << ", \"devices\": [";
    for (int g = 0; g < mp->G; ++g) os << (g ? ", " : "") << mp->dev[static_cast<size_t>(g)];
    os << "], \"split_dim\": " << s.dim + 1 << ", \"split_kind\": \"" << (s.pw ? "pw" : "cc") << "\", \"combine\": \""
       << mp->combine_path << "\", \"shards\": [";
    for (int g = 0; g < mp->G; ++g) {
      int64_t need2 = 0;
      mdh_b200_describe(mp->shard[static_cast<size_t>(g)], nullptr, 0, &need2);
      std::string d(static_cast<size_t>(need2), '\0');
      mdh_b200_describe(mp->shard[static_cast<size_t>(g)], &d[0], need2, &need2);
      d.resize(std::strlen(d.c_str()));
      const int64_t step = mp->e.sizes[static_cast<size_t>(s.dim)] / mp->G;
      os << (g ? ", " : "") << "{\"range\": [" << step * g << ", " << step * (g + 1) << "], \"plan\": " << d << "}";
    }
    os << "]}";
    put_text(os.str(), buf, cap, need);
  });
}

int mdh_b200_mplan_shard_buffer(const mdh_b200_mplan* mp, int g, int side, int b, int* slab_rank, int64_t* start,
                                int64_t* dims, int* rank, int* dtype, int64_t* bytes) {
  return guard_mp([&] {
    if (g < 0 || g >= mp->G) mdhb::fail("OutOfRange", "shard index");
    const auto& D = side == 0 ? mp->in_dims[static_cast<size_t>(g)] : mp->out_dims[static_cast<size_t>(g)];
    if (b < 0 || b >= static_cast<int>(D.size())) mdhb::fail("OutOfRange", "buffer index");
    const auto& sl = side == 0 ? mp->split.in[static_cast<size_t>(b)] : mp->split.out[static_cast<size_t>(b)];
    *slab_rank = sl.rank;
    *start = side == 0 ? mp->in_start[static_cast<size_t>(g)][static_cast<size_t>(b)] : mp->out_start[static_cast<size_t>(g)][static_cast<size_t>(b)];
    *rank = static_cast<int>(D[static_cast<size_t>(b)].size());
    for (size_t r = 0; r < D[static_cast<size_t>(b)].size(); ++r) dims[r] = D[static_cast<size_t>(b)][r];
    *dtype = side == 0 ? mp->in_store[static_cast<size_t>(g)][static_cast<size_t>(b)] : mp->out_store[static_cast<size_t>(g)][static_cast<size_t>(b)];
    if (bytes) *bytes = mdhb::numel(D[static_cast<size_t>(b)]) * static_cast<int64_t>(store_size(*dtype));
  });
}

int mdh_b200_mplan_shard_plan(const mdh_b200_mplan* mp, int g, mdh_b200_plan** plan) {
  return guard_mp([&] {
    if (g < 0 || g >= mp->G) mdhb::fail("OutOfRange", "shard index");
    *plan = mp->shard[static_cast<size_t>(g)];
  });
}

int mdh_b200_mplan_run(mdh_b200_mplan* mp, const void* const* const* d_in, void* const* const* d_out, void* const* streams) {
  return guard_mp([&] { run_shards(mp, d_in, d_out, streams_of(mp, streams)); });
}

int mdh_b200_mplan_run_host(mdh_b200_mplan* mp, const void* const* h_in, void* const* h_out) {
  return guard_mp([&] {
    const int G = mp->G;
    const size_t nin = mp->e.in.size(), nout = mp->e.out.size();
    if (mp->h_in.empty()) {
      mp->h_in.resize(static_cast<size_t>(G));
      mp->h_out.resize(static_cast<size_t>(G));
      for (int g = 0; g < G; ++g) {
        MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
        for (size_t b = 0; b < nin; ++b) {
          void* d = nullptr;
          MDHB_CUDA(cudaMalloc(&d, std::max<size_t>(16, static_cast<size_t>(mdhb::numel(mp->in_dims[static_cast<size_t>(g)][b])) *
                                                               store_size(mp->in_store[static_cast<size_t>(g)][b]))));
          mp->h_in[static_cast<size_t>(g)].push_back(d);
        }
        for (size_t b = 0; b < nout; ++b) {
          void* d = nullptr;
          MDHB_CUDA(cudaMalloc(&d, std::max<size_t>(16, static_cast<size_t>(mdhb::numel(mp->out_dims[static_cast<size_t>(g)][b])) *
                                                               store_size(mp->out_store[static_cast<size_t>(g)][b]))));
          mp->h_out[static_cast<size_t>(g)].push_back(d);
        }
      }
    }
    auto st = streams_of(mp, nullptr);
    for (int g = 0; g < G; ++g) {
      MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
      for (size_t b = 0; b < nin; ++b)
        copy_slab(mp->h_in[static_cast<size_t>(g)][b], h_in[b], true, mp->g_in_ext[b], mp->in_dims[static_cast<size_t>(g)][b],
                  mp->split.in[b].rank, mp->in_start[static_cast<size_t>(g)][b], store_size(mp->in_store[static_cast<size_t>(g)][b]),
                  cudaMemcpyHostToDevice, st[static_cast<size_t>(g)]);
    }
    std::vector<const void* const*> din(static_cast<size_t>(G));
    std::vector<void* const*> dout(static_cast<size_t>(G));
    for (int g = 0; g < G; ++g) {
      din[static_cast<size_t>(g)] = mp->h_in[static_cast<size_t>(g)].data();
      dout[static_cast<size_t>(g)] = mp->h_out[static_cast<size_t>(g)].data();
    }
    run_shards(mp, din.data(), dout.data(), st);
    for (int g = 0; g < G; ++g) {
      if (mp->split.pw && g > 0) continue;  // the combined result is shard 0's
      MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
      for (size_t b = 0; b < nout; ++b)
        copy_slab(h_out[b], mp->h_out[static_cast<size_t>(g)][b], false, mp->g_out_ext[b], mp->out_dims[static_cast<size_t>(g)][b],
                  mp->split.out[b].rank, mp->out_start[static_cast<size_t>(g)][b], store_size(mp->out_store[static_cast<size_t>(g)][b]),
                  cudaMemcpyDeviceToHost, st[static_cast<size_t>(g)]);
    }
    for (int g = 0; g < G; ++g) MDHB_CUDA(cudaStreamSynchronize(st[static_cast<size_t>(g)]));
  });
}

// Iterated sweeps of a halo-1 stencil split along dimension 1: the shard's
// input slab v[g] holds its planes plus one ghost plane per side.  Per sweep:
// every shard runs v -> w; w is written back into v's interior; the ghost
// planes are refreshed from the neighbours' edge planes (grouped
// ncclSend/Recv when the shards own distinct devices and NCCL is up, else
// peer copies).  The outer boundary (global planes 0 and N+1, and every
// plane's boundary rows/columns) stays fixed.  On return v holds the state
// after `sweeps` sweeps and w the last sweep's output.
int mdh_b200_mplan_iterate(mdh_b200_mplan* mp, void* const* const* d_v, void* const* const* d_w, int sweeps,
                           void* const* streams) {
  return guard_mp([&] {
    const int G = mp->G;
    if (mp->e.in.size() != 1 || mp->e.out.size() != 1 || mp->split.pw || mp->split.dim != 0)
      mdhb::fail("Unsupported", "iterate: one input and one output, split along dimension 1");
    const auto& ge = mp->g_in_ext[0];
    const auto& go = mp->g_out_ext[0];
    if (ge.size() != go.size() || mp->in_store[0][0] != mp->out_store[0][0] || mp->split.in[0].rank != 0)
      mdhb::fail("Unsupported", "iterate: input and output must have the same rank and storage");
    for (size_t r = 0; r < ge.size(); ++r)
      if (ge[r] != go[r] + 2) mdhb::fail("Unsupported", "iterate: the input must be the output plus a 1-cell halo");
    const size_t es = store_size(mp->in_store[0][0]);
    int64_t plane = 1;  // elements of one input plane (ranks 1..)
    for (size_t r = 1; r < ge.size(); ++r) plane *= ge[r];
    auto st = streams_of(mp, streams);
    const bool use_nccl = !mp->comm.empty();
    for (int it = 0; it < sweeps; ++it) {
      run_shards(mp, reinterpret_cast<const void* const* const*>(d_v), d_w, st);
      for (int g = 0; g < G; ++g) {
        // w -> interior of v: a 3-D strided copy (depth = local planes)
        MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
        const auto& od = mp->out_dims[static_cast<size_t>(g)][0];
        const auto& id = mp->in_dims[static_cast<size_t>(g)][0];
        cudaMemcpy3DParms p{};
        const int64_t inner_out = od.back();
        // 3-D copies address (plane, row, element); for rank 3 rows are j, elements k
        if (od.size() != 3) mdhb::fail("Unsupported", "iterate: rank-3 stencils");
        char* vbase = static_cast<char*>(d_v[g][0]) + (static_cast<size_t>(plane) + static_cast<size_t>(id[2]) + 1) * es;
        p.srcPtr = make_cudaPitchedPtr(d_w[g][0], static_cast<size_t>(inner_out) * es, static_cast<size_t>(inner_out), static_cast<size_t>(od[1]));
        p.dstPtr = make_cudaPitchedPtr(vbase, static_cast<size_t>(id[2]) * es, static_cast<size_t>(id[2]), static_cast<size_t>(id[1]));
        p.extent = make_cudaExtent(static_cast<size_t>(inner_out) * es, static_cast<size_t>(od[1]), static_cast<size_t>(od[0]));
        p.kind = cudaMemcpyDeviceToDevice;
        MDHB_CUDA(cudaMemcpy3DAsync(&p, st[static_cast<size_t>(g)]));
      }
      if (G == 1) continue;
      // halo exchange: ghost plane 0 of shard g <- last interior plane of g-1;
      // ghost plane n+1 of g <- first interior plane of g+1
      for (int g = 0; g < G; ++g) {
        MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
        MDHB_CUDA(cudaEventRecord(mp->done[static_cast<size_t>(g)], st[static_cast<size_t>(g)]));
      }
      const size_t pbytes = static_cast<size_t>(plane) * es;
      if (use_nccl) {
        auto& n = mdhb::need_nccl();
        const int ty = mdhb::nccl_type(static_cast<Store>(mp->in_store[0][0]));
        mdhb::nccl_check(n.GroupStart(), "ncclGroupStart");
        for (int g = 0; g < G; ++g) {
          const int64_t nl = mp->in_dims[static_cast<size_t>(g)][0][0];  // local planes incl. ghosts
          char* v = static_cast<char*>(d_v[g][0]);
          cudaStream_t s = st[static_cast<size_t>(g)];
          mdhb::ncclComm_t c = mp->comm[static_cast<size_t>(g)];
          if (g > 0) {
            mdhb::nccl_check(n.Send(v + pbytes, static_cast<size_t>(plane), ty, g - 1, c, s), "ncclSend");
            mdhb::nccl_check(n.Recv(v, static_cast<size_t>(plane), ty, g - 1, c, s), "ncclRecv");
          }
          if (g + 1 < G) {
            mdhb::nccl_check(n.Send(v + static_cast<size_t>(nl - 2) * pbytes, static_cast<size_t>(plane), ty, g + 1, c, s), "ncclSend");
            mdhb::nccl_check(n.Recv(v + static_cast<size_t>(nl - 1) * pbytes, static_cast<size_t>(plane), ty, g + 1, c, s), "ncclRecv");
          }
        }
        mdhb::nccl_check(n.GroupEnd(), "ncclGroupEnd");
      } else {
        for (int g = 0; g < G; ++g) {
          MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
          cudaStream_t s = st[static_cast<size_t>(g)];
          const int64_t nl = mp->in_dims[static_cast<size_t>(g)][0][0];
          char* v = static_cast<char*>(d_v[g][0]);
          if (g > 0) {
            MDHB_CUDA(cudaStreamWaitEvent(s, mp->done[static_cast<size_t>(g - 1)], 0));
            const int64_t np = mp->in_dims[static_cast<size_t>(g - 1)][0][0];
            MDHB_CUDA(cudaMemcpyPeerAsync(v, mp->dev[static_cast<size_t>(g)],
                                          static_cast<char*>(d_v[g - 1][0]) + static_cast<size_t>(np - 2) * pbytes,
                                          mp->dev[static_cast<size_t>(g - 1)], pbytes, s));
          }
          if (g + 1 < G) {
            MDHB_CUDA(cudaStreamWaitEvent(s, mp->done[static_cast<size_t>(g + 1)], 0));
            MDHB_CUDA(cudaMemcpyPeerAsync(v + static_cast<size_t>(nl - 1) * pbytes, mp->dev[static_cast<size_t>(g)],
                                          static_cast<char*>(d_v[g + 1][0]) + pbytes, mp->dev[static_cast<size_t>(g + 1)], pbytes, s));
          }
        }
        // the next sweep must not overwrite an edge plane a neighbour is still reading
        for (int g = 0; g < G; ++g) {
          MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
          MDHB_CUDA(cudaEventRecord(mp->done[static_cast<size_t>(g)], st[static_cast<size_t>(g)]));
        }
        for (int g = 0; g < G; ++g) {
          MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
          if (g > 0) MDHB_CUDA(cudaStreamWaitEvent(st[static_cast<size_t>(g)], mp->done[static_cast<size_t>(g - 1)], 0));
          if (g + 1 < G) MDHB_CUDA(cudaStreamWaitEvent(st[static_cast<size_t>(g)], mp->done[static_cast<size_t>(g + 1)], 0));
        }
      }
    }
  });
}

// Device time of one mdh_b200_mplan_run: events on every shard's stream; the
// run's time is the MAX over shards (each bracketed on its own device), the
// L2 of every device left as the previous run left it (inputs above L2 size
// or rotated by the caller).
int mdh_b200_mplan_time(mdh_b200_mplan* mp, const void* const* const* d_in, void* const* const* d_out, int warmup,
                        int reps, double* median_s) {
  return guard_mp([&] {
    auto st = streams_of(mp, nullptr);
    for (int w = 0; w < warmup; ++w) run_shards(mp, d_in, d_out, st);
    const int G = mp->G;
    std::vector<cudaEvent_t> a(static_cast<size_t>(G)), b(static_cast<size_t>(G));
    for (int g = 0; g < G; ++g) {
      MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
      MDHB_CUDA(cudaEventCreate(&a[static_cast<size_t>(g)]));
      MDHB_CUDA(cudaEventCreate(&b[static_cast<size_t>(g)]));
    }
    std::vector<double> t;
    for (int k = 0; k < std::max(1, reps); ++k) {
      for (int g = 0; g < G; ++g) {
        MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
        MDHB_CUDA(cudaStreamSynchronize(st[static_cast<size_t>(g)]));
      }
      for (int g = 0; g < G; ++g) {
        MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
        MDHB_CUDA(cudaEventRecord(a[static_cast<size_t>(g)], st[static_cast<size_t>(g)]));
      }
      run_shards(mp, d_in, d_out, st);
      double mx = 0;
      for (int g = 0; g < G; ++g) {
        MDHB_CUDA(cudaSetDevice(mp->dev[static_cast<size_t>(g)]));
        MDHB_CUDA(cudaEventRecord(b[static_cast<size_t>(g)], st[static_cast<size_t>(g)]));
      }
      for (int g = 0; g < G; ++g) {
        MDHB_CUDA(cudaEventSynchronize(b[static_cast<size_t>(g)]));
        float ms = 0;
        MDHB_CUDA(cudaEventElapsedTime(&ms, a[static_cast<size_t>(g)], b[static_cast<size_t>(g)]));
        mx = std::max(mx, ms * 1e-3);
      }
      t.push_back(mx);
    }
    for (int g = 0; g < G; ++g) {
      cudaEventDestroy(a[static_cast<size_t>(g)]);
      cudaEventDestroy(b[static_cast<size_t>(g)]);
    }
    std::sort(t.begin(), t.end());
    *median_s = t[t.size() / 2];
  });
}

// ---------------------------------------------------------------- one process per GPU
int mdh_b200_nccl_unique_id(unsigned char* id128) {
  return guard_mp([&] {
    mdhb::ncclUniqueId id;
    mdhb::nccl_check(mdhb::need_nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id128, id.internal, 128);
  });
}

}  // extern "C"

// rank plans: the shard plan plus (optionally) an NCCL communicator; the
// combine of a point-wise split runs inside mdh_b200_run (plan.hpp RankCtx)
namespace mdhb {
struct RankCombine : Routine {
  std::unique_ptr<Routine> inner;
  ncclComm_t comm = nullptr;
  int op = -1;
  std::vector<int64_t> counts;
  std::vector<int> types;
  std::string shard_desc;
  const char* family() const override { return inner->family(); }
  std::string describe() const override {
    std::string d = inner->describe();
    if (!d.empty() && d.back() == '}') d.pop_back();
    return d + ", " + shard_desc + ", \"nccl_allreduce\": " + (comm ? "true" : "false") + "}";
  }
  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    inner->launch(d_in, d_out, s);
    if (comm) {
      auto& n = need_nccl();
      nccl_check(n.GroupStart(), "ncclGroupStart");
      for (size_t b = 0; b < counts.size(); ++b)
        nccl_check(n.AllReduce(d_out[b], d_out[b], static_cast<size_t>(counts[b]), types[b], op, comm, s), "ncclAllReduce");
      nccl_check(n.GroupEnd(), "ncclGroupEnd");
    }
  }
  int launches() const override { return inner->launches(); }
  double flops() const override { return inner->flops(); }
  double bytes() const override { return inner->bytes(); }
  const char* bound() const override { return inner->bound(); }
  std::string source() const override { return inner->source(); }
  ~RankCombine() override {
    if (comm) nccl().CommDestroy(comm);
  }
};

// used by abi.cu's mdh_b200_rank_plan_create
std::string rank_shard(const std::string& comp_json, const Asm& m, const std::string& cfg_json, int world, int rank,
                       int split_dim, std::string* cfg_out, std::string* desc, int* fold, bool* pw) {
  MdHom e = parse_md_hom(comp_json);
  std::unique_ptr<Config> cfg;
  if (!cfg_json.empty()) cfg = std::make_unique<Config>(parse_config(cfg_json, e, m));
  Split s = choose_split(e, m, cfg.get(), world, split_dim);
  std::string sj = shard_computation(comp_json, e, s, rank);
  if (cfg) *cfg_out = shard_config(cfg_json, e, parse_md_hom(sj), m, s);
  const int64_t step = e.sizes[static_cast<size_t>(s.dim)] / world;
  std::ostringstream os;
  os << "\"shard\": {\"world\": " << world << ", \"rank\": " << rank << ", \"split_dim\": " << s.dim + 1
     << ", \"split_kind\": \"" << (s.pw ? "pw" : "cc") << "\", \"range\": [" << step * rank << ", " << step * (rank + 1)
     << "], \"in\": [";
  for (size_t b = 0; b < s.in.size(); ++b)
    os << (b ? ", " : "") << "[" << s.in[b].rank << ", " << s.in[b].coeff * step * rank << "]";
  os << "], \"out\": [";
  for (size_t b = 0; b < s.out.size(); ++b)
    os << (b ? ", " : "") << "[" << s.out[b].rank << ", " << s.out[b].coeff * step * rank << "]";
  os << "]}";
  *desc = os.str();
  *fold = s.fold;
  *pw = s.pw;
  return sj;
}

std::unique_ptr<Routine> wrap_rank(std::unique_ptr<Routine> inner, const Problem& p, const std::string& desc, int fold,
                                   bool pw, const unsigned char* nccl_id, int world, int rank) {
  auto r = std::make_unique<RankCombine>();
  r->inner = std::move(inner);
  r->shard_desc = desc;
  if (pw && nccl_id) {  // (a 1-rank communicator all-reduces as the identity: the path runs on one GPU too)
    r->op = nccl_op(fold);
    if (r->op < 0) fail("Unsupported", "NCCL has no reduction for this combine operator");
    auto& n = need_nccl();
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_id, 128);
    nccl_check(n.CommInitRank(&r->comm, world, id, rank), "ncclCommInitRank");
    for (size_t b = 0; b < p.out_ext.size(); ++b) {
      r->counts.push_back(numel(p.out_ext[b]));
      r->types.push_back(nccl_type(p.out_store[b]));
    }
  }
  return r;
}
}  // namespace mdhb
