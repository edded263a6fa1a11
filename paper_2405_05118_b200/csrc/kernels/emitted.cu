// Emitted family: any md_hom without prefix-sum dims is
// compiled to its own CUDA kernel at plan time with NVRTC, for sm_100a.
// This is the B200 counterpart of the reference's code generator
// (proj/src/codegen.cpp:389-945: expr_c / fold_c at :198-251 emit the scalar
// function and the fold as C, the nest follows the lexicographic plan) and
// replaces the generic family's per-point bytecode interpretation
// (generic.cu, engine.cpp:134-176 semantics) by straight-line code:
//
//   * one thread per cell of the combined result (collapsed ranges); the
//     cell's cc coordinates are decoded with compile-time extents
//   * the point-wise dims become nested ascending loops -- the reference's
//     fold order (engine.cpp:177-189, first visit assigns), so f64 storage is
//     bit-identical to the oracle; the kernel is compiled with --fmad=false
//     (no contraction of a*b+c, as the reference's -ffp-contract=off build)
//   * every input / output access is its affine offset with the strides
//     folded in as literals; buffers are typed by their storage
//   * the scalar function is the reference's expression tree, typed as the
//     reference types it (i64 ops in long long, f64 ops in the float storage
//     type), with the VM's conventions for min/max argument order, cmp
//     (-1/0/1), select and integer division by zero
//
// NVRTC is loaded with dlopen (libnvrtc.so.12), the cubin with
// cudaLibraryLoadData; compiled kernels are cached per source text.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

#include "../plan.hpp"

namespace mdhb {
namespace {

// ---- NVRTC entry points (dlopen; no link-time dependency)
using nvrtcProgram = struct _nvrtcProgram*;
struct Nvrtc {
  int (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  int (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  int (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  int (*cubin)(nvrtcProgram, char*) = nullptr;
  int (*log_size)(nvrtcProgram, size_t*) = nullptr;
  int (*log)(nvrtcProgram, char*) = nullptr;
  int (*destroy)(nvrtcProgram*) = nullptr;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
    n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
    n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    n.log_size = reinterpret_cast<decltype(n.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.log_size && n.log && n.destroy;
  });
  return n;
}

constexpr int kMaxBuf = 16;
struct EmPtrs {
  const void* in[kMaxBuf];
  void* out[kMaxBuf];
};

// compiled kernels, shared by plans with the same source
struct Compiled {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
};
std::mutex g_mu;
std::map<std::string, Compiled>& cache() {
  static std::map<std::string, Compiled> c;
  return c;
}

Compiled compile_source(const std::string& src, int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  const std::string key = std::to_string(device) + "\n" + src;
  auto it = cache().find(key);
  if (it != cache().end()) return it->second;
  const Nvrtc& n = nvrtc();
  if (!n.ok) fail("Unsupported", "NVRTC (libnvrtc.so.12) not loadable");
  nvrtcProgram prog = nullptr;
  if (n.create(&prog, src.c_str(), "mdh_emitted.cu", 0, nullptr, nullptr) != 0) fail("CudaError", "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17", "--use_fast_math=false"};
  const int rc = n.compile(prog, 3, opts);
  if (rc != 0) {
    size_t ls = 0;
    n.log_size(prog, &ls);
    std::string log(ls, '\0');
    n.log(prog, &log[0]);
    n.destroy(&prog);
    fail("CompilerUnavailable", "NVRTC compile of the emitted kernel failed: " + log.substr(0, 2000));
  }
  size_t sz = 0;
  n.cubin_size(prog, &sz);
  std::string bin(sz, '\0');
  n.cubin(prog, &bin[0]);
  n.destroy(&prog);
  Compiled c;
  MDHB_CUDA(cudaLibraryLoadData(&c.lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  MDHB_CUDA(cudaLibraryGetKernel(&c.kern, c.lib, "mdh_emitted"));
  cache()[key] = c;
  return c;
}

const char* ctype(Store s) {
  switch (s) {
    case Store::F32: return "float";
    case Store::F64: return "double";
    case Store::I32: return "int";
    default: return "long long";
  }
}

class Emitter {
 public:
  Emitter(const Problem& p) : p_(p), e_(p.e) {}

  // shared prelude: typedefs and helpers of the emitted translation unit
  std::string prelude() {
    ft_ = p_.opt.fstore == Store::F64 ? "double" : "float";
    std::ostringstream s;
    s << "// emitted by mdh_b200 for md_hom '" << e_.name << "'\n"
      << "typedef long long i64;\ntypedef " << ft_ << " F;\n"
      << "struct Ptrs { const void* in[" << kMaxBuf << "]; void* out[" << kMaxBuf << "]; };\n"
      << "__device__ __forceinline__ i64 idiv(i64 a, i64 b) { return b == 0 ? 0 : a / b; }\n"
      << "template <class T> __device__ __forceinline__ i64 cmp3(T a, T b) { return a < b ? -1 : (a > b ? 1 : 0); }\n"
      << "template <class T> __device__ __forceinline__ T mn(T a, T b) { return b < a ? b : a; }\n"
      << "template <class T> __device__ __forceinline__ T mx(T a, T b) { return a < b ? b : a; }\n";
    return s.str();
  }
  std::string pointers() const {
    std::ostringstream s;
    for (size_t b = 0; b < e_.in.size(); ++b)
      s << "  const " << ctype(p_.in_store[b]) << "* __restrict__ in" << b << " = (const " << ctype(p_.in_store[b])
        << "*)p.in[" << b << "];\n";
    for (size_t b = 0; b < e_.out.size(); ++b)
      s << "  " << ctype(p_.out_store[b]) << "* __restrict__ out" << b << " = (" << ctype(p_.out_store[b]) << "*)p.out["
        << b << "];\n";
    return s.str();
  }
  // cc coordinates from `cell` (row-major over the collapsed ranges)
  std::string decode_cell() const {
    std::ostringstream s;
    s << "  i64 rem = cell;\n";
    for (int d = e_.D() - 1; d >= 0; --d) {
      if (e_.comb[static_cast<size_t>(d)].kind != Combine::CC) continue;
      s << "  const i64 i" << d << " = rem % " << e_.sizes[static_cast<size_t>(d)] << "LL; rem /= "
        << e_.sizes[static_cast<size_t>(d)] << "LL;\n";
    }
    return s.str();
  }
  std::string values(const std::string& ind) {
    std::ostringstream s;
    for (size_t c = 0; c < e_.assigns.size(); ++c) {
      const bool f = e_.assigns[c].e.type == Ty::F64;
      s << ind << "const " << (f ? "F" : "i64") << " v" << c << " = " << expr(e_.assigns[c].e) << ";\n";
    }
    return s.str();
  }
  std::string fold_in(const std::string& ind, const std::string& acc, const std::string& val, const std::string& first) {
    std::ostringstream s;
    const int fold = e_.fold();
    s << ind << "if (" << first << ") {\n";
    for (size_t c = 0; c < e_.assigns.size(); ++c) s << ind << "  " << acc << c << " = " << val << c << ";\n";
    s << ind << "} else {\n";
    if (fold >= kCustomFoldBase) {
      // registered custom operator: its body folds the whole component tuple
      // (a0.. = accumulator lvalues, b0.. = the next value)
      const CustomCombine& op = combine_at(fold - kCustomFoldBase);
      s << ind << "  {\n";
      for (size_t c = 0; c < e_.assigns.size(); ++c)
        s << ind << "    auto& a" << c << " = " << acc << c << ";\n" << ind << "    const auto b" << c << " = " << val << c << ";\n";
      s << ind << "    " << op.body << "\n" << ind << "  }\n";
    } else {
      for (size_t c = 0; c < e_.assigns.size(); ++c)
        s << ind << "  " << acc << c << " = " << fold_expr(fold, acc + std::to_string(c), val + std::to_string(c)) << ";\n";
    }
    s << ind << "}\n" << ind << first << " = false;\n";
    return s.str();
  }
  std::string stores(const std::string& acc) const {
    std::ostringstream s;
    int comp = 0;
    for (size_t b = 0; b < e_.out.size(); ++b)
      for (size_t a = 0; a < e_.out[b].acc.size(); ++a, ++comp) {
        Linear l = linearize(e_.out[b].acc[a], p_.out_ext[b], e_.D());
        const bool fsrc = e_.assigns[static_cast<size_t>(comp)].e.type == Ty::F64;
        const Store st = p_.out_store[b];
        std::string v = acc + std::to_string(comp);
        if (st == Store::I32) v = "(int)" + v;
        else if (st == Store::I64) v = fsrc ? "(i64)" + v : v;
        else v = std::string("(") + ctype(st) + ")" + v;
        s << "  out" << b << "[" << offset(l, true) << "] = " << v << ";\n";
      }
    return s.str();
  }

  // One thread per result cell, point-wise loops ascending (the reference's
  // lexicographic fold order).
  std::string source() {
    const int D = e_.D();
    std::ostringstream s;
    s << prelude() << "extern \"C\" __global__ void __launch_bounds__(128) mdh_emitted(Ptrs p) {\n"
      << "  const i64 cell = (i64)blockIdx.x * 128 + threadIdx.x;\n"
      << "  if (cell >= " << cells() << "LL) return;\n"
      << pointers() << decode_cell();
    const int fold = e_.fold();
    for (size_t c = 0; c < e_.assigns.size(); ++c)
      s << "  " << (e_.assigns[c].e.type == Ty::F64 ? "F" : "i64") << " acc" << c << " = 0;\n";
    if (fold >= 0) s << "  bool first = true;\n";
    std::string ind = "  ";
    for (int d = 0; d < D; ++d) {
      if (e_.comb[static_cast<size_t>(d)].kind == Combine::CC) continue;
      s << ind << "for (i64 i" << d << " = 0; i" << d << " < " << e_.sizes[static_cast<size_t>(d)] << "LL; ++i" << d << ") {\n";
      ind += "  ";
    }
    s << values(ind);
    if (fold >= 0) {
      s << fold_in(ind, "acc", "v", "first");
    } else {
      for (size_t c = 0; c < e_.assigns.size(); ++c) s << ind << "acc" << c << " = v" << c << ";\n";
    }
    for (int d = D - 1; d >= 0; --d)
      if (e_.comb[static_cast<size_t>(d)].kind != Combine::CC) {
        ind.resize(ind.size() - 2);
        s << ind << "}\n";
      }
    s << stores("acc") << "}\n";
    return s.str();
  }

  // Split-fiber reduction for few cells with long point-wise fibers (dot,
  // reduce, histo, ...): G CTAs per cell each fold a contiguous range of the
  // fiber (threads stride it, so the innermost unit-stride dim is read
  // coalesced), a fixed-order shuffle / shared-memory tree combines the
  // threads, and mdh_emitted_final folds the G partials of each cell in
  // order.  Deterministic; the fold is re-associated, so it is used only when
  // the reference's order cannot matter (integers, min/max) or the storage is
  // the FP32 tolerance mode.
  std::string source_split(int64_t G) {
    const int D = e_.D();
    const size_t NC = e_.assigns.size();
    int64_t L = 1;
    for (int d = 0; d < D; ++d)
      if (e_.comb[static_cast<size_t>(d)].kind != Combine::CC) L *= e_.sizes[static_cast<size_t>(d)];
    std::ostringstream s;
    s << prelude();
    // partial slot: 8 bytes per component + has flag, [cells * G]
    s << "struct Part {";
    for (size_t c = 0; c < NC; ++c) s << " " << (e_.assigns[c].e.type == Ty::F64 ? "F" : "i64") << " a" << c << ";";
    s << " int has; };\n";
    s << "extern \"C\" __global__ void __launch_bounds__(256) mdh_emitted(Ptrs p, Part* part) {\n"
      << "  const i64 cell = (i64)blockIdx.x / " << G << "LL, g = (i64)blockIdx.x % " << G << "LL;\n"
      << pointers() << decode_cell()
      << "  const i64 lo = g * " << L << "LL / " << G << "LL, hi = (g + 1) * " << L << "LL / " << G << "LL;\n";
    for (size_t c = 0; c < NC; ++c) s << "  " << (e_.assigns[c].e.type == Ty::F64 ? "F" : "i64") << " acc" << c << " = 0;\n";
    s << "  bool first = true;\n"
      << "  for (i64 t = lo + threadIdx.x; t < hi; t += 256) {\n"
      << "    i64 r = t;\n";
    for (int d = D - 1; d >= 0; --d) {
      if (e_.comb[static_cast<size_t>(d)].kind == Combine::CC) continue;
      s << "    const i64 i" << d << " = r % " << e_.sizes[static_cast<size_t>(d)] << "LL; r /= " << e_.sizes[static_cast<size_t>(d)]
        << "LL;\n";
    }
    s << values("    ") << fold_in("    ", "acc", "v", "first") << "  }\n";
    // warp tree (lane l takes lane l+o), then warps in order through shared memory
    s << "  int has = first ? 0 : 1;\n"
      << "  for (int o = 1; o < 32; o <<= 1) {\n"
      << "    const int oh = __shfl_down_sync(0xffffffffu, has, o);\n";
    for (size_t c = 0; c < NC; ++c) s << "    const auto o" << c << " = __shfl_down_sync(0xffffffffu, acc" << c << ", o);\n";
    s << "    if ((threadIdx.x & 31) + o < 32 && oh) {\n"
      << "      bool fst = !has;\n" << fold_in("      ", "acc", "o", "fst") << "      has = 1;\n    }\n  }\n"
      << "  __shared__ Part w[8];\n"
      << "  if ((threadIdx.x & 31) == 0) {";
    for (size_t c = 0; c < NC; ++c) s << " w[threadIdx.x >> 5].a" << c << " = acc" << c << ";";
    s << " w[threadIdx.x >> 5].has = has; }\n  __syncthreads();\n"
      << "  if (threadIdx.x == 0) {\n    bool fst = true;\n";
    for (size_t c = 0; c < NC; ++c) s << "    " << (e_.assigns[c].e.type == Ty::F64 ? "F" : "i64") << " b" << c << " = 0;\n";
    s << "    for (int k = 0; k < 8; ++k) {\n      if (!w[k].has) continue;\n";
    for (size_t c = 0; c < NC; ++c) s << "      const auto u" << c << " = w[k].a" << c << ";\n";
    s << fold_in("      ", "b", "u", "fst") << "    }\n"
      << "    Part q;";
    for (size_t c = 0; c < NC; ++c) s << " q.a" << c << " = b" << c << ";";
    s << " q.has = fst ? 0 : 1;\n    part[blockIdx.x] = q;\n  }\n}\n";
    // final: one thread per cell folds its G partials in order and stores
    s << "extern \"C\" __global__ void __launch_bounds__(128) mdh_emitted_final(Ptrs p, const Part* part) {\n"
      << "  const i64 cell = (i64)blockIdx.x * 128 + threadIdx.x;\n"
      << "  if (cell >= " << cells() << "LL) return;\n"
      << pointers() << decode_cell();
    for (size_t c = 0; c < NC; ++c) s << "  " << (e_.assigns[c].e.type == Ty::F64 ? "F" : "i64") << " acc" << c << " = 0;\n";
    s << "  bool first = true;\n"
      << "  for (i64 g = 0; g < " << G << "LL; ++g) {\n"
      << "    const Part q = part[cell * " << G << "LL + g];\n    if (!q.has) continue;\n";
    for (size_t c = 0; c < NC; ++c) s << "    const auto u" << c << " = q.a" << c << ";\n";
    s << fold_in("    ", "acc", "u", "first") << "  }\n" << stores("acc") << "}\n";
    return s.str();
  }

  // parts per cell for the split mode (0 = keep one thread per cell)
  int64_t split_parts(int sms) const {
    const int fold = e_.fold();
    if (fold < 0 || std::getenv("MDHB_EMIT_NO_SPLIT")) return 0;
    int64_t L = 1;
    for (int d = 0; d < e_.D(); ++d)
      if (e_.comb[static_cast<size_t>(d)].kind != Combine::CC) L *= e_.sizes[static_cast<size_t>(d)];
    const int64_t C = cells();
    if (L < 1024 || C >= 16384) return 0;
    // re-association is invisible for integers and min/max; FP32 storage is tolerance mode
    bool ok = true;  // (custom operators are declared associative + commutative by md_hom validity)
    for (auto& a : e_.assigns)
      if (a.e.type == Ty::F64 && (fold == 0 || fold == 2) && p_.opt.fstore == Store::F64) ok = false;
    if (!ok) return 0;
    int64_t G = std::max<int64_t>(1, (static_cast<int64_t>(sms) * 16 + C - 1) / C);
    G = std::min<int64_t>(G, std::max<int64_t>(1, L / 1024));
    return G;
  }

  int64_t cells() const {
    int64_t c = 1;
    for (int d = 0; d < e_.D(); ++d)
      if (e_.comb[static_cast<size_t>(d)].kind == Combine::CC) c *= e_.sizes[static_cast<size_t>(d)];
    return c;
  }

 private:
  std::string offset(const Linear& l, bool cc_only) const {
    std::ostringstream o;
    o << "(" << l.c0 << "LL";
    for (int d = 0; d < e_.D(); ++d) {
      const int64_t c = l.cj[static_cast<size_t>(d)];
      if (c == 0) continue;
      if (cc_only && e_.comb[static_cast<size_t>(d)].kind != Combine::CC) continue;
      o << " + " << c << "LL * i" << d;
    }
    o << ")";
    return o.str();
  }
  std::string fold_expr(int fold, const std::string& a, const std::string& v) const {
    switch (fold) {
      case 0: return a + " + " + v;
      case 2: return a + " * " + v;
      case 4: return "(" + v + " < " + a + " ? " + v + " : " + a + ")";
      case 5: return "(" + v + " > " + a + " ? " + v + " : " + a + ")";
      default: return v;
    }
  }
  std::string lit_f(double x) const {
    std::ostringstream o;
    o.precision(17);
    o << "(F)" << x;
    std::string s = o.str();
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
  }
  std::string expr(const Expr& x) {
    const bool f = x.type == Ty::F64;
    switch (x.k) {
      case EK::Lit: return f ? lit_f(x.fv) : "(" + std::to_string(x.iv) + "LL)";
      case EK::Idx: return "i" + std::to_string(x.dim - 1);
      case EK::In: {
        const int b = x.buf - 1;
        Linear l = linearize(e_.in[static_cast<size_t>(b)].acc[static_cast<size_t>(x.acc - 1)], p_.in_ext[static_cast<size_t>(b)], e_.D());
        return std::string("((") + (f ? "F" : "i64") + ")in" + std::to_string(b) + "[" + offset(l, false) + "])";
      }
      case EK::Abs: {
        const std::string a = expr(x.args[0]);
        return f ? "fabs" + std::string(ft_ == "float" ? "f" : "") + "(" + a + ")" : "((" + a + ") < 0 ? -(" + a + ") : (" + a + "))";
      }
      case EK::Cmp: {
        const bool af = x.args[0].type == Ty::F64;
        return "cmp3<" + std::string(af ? "F" : "i64") + ">(" + expr(x.args[0]) + ", " + expr(x.args[1]) + ")";
      }
      case EK::Select:
        return "((" + expr(x.args[0]) + ") != 0 ? (" + expr(x.args[1]) + ") : (" + expr(x.args[2]) + "))";
      case EK::Min: return std::string("mn<") + (f ? "F" : "i64") + ">(" + expr(x.args[0]) + ", " + expr(x.args[1]) + ")";
      case EK::Max: return std::string("mx<") + (f ? "F" : "i64") + ">(" + expr(x.args[0]) + ", " + expr(x.args[1]) + ")";
      case EK::Div:
        if (!f) return "idiv(" + expr(x.args[0]) + ", " + expr(x.args[1]) + ")";
        return "((F)(" + expr(x.args[0]) + " / " + expr(x.args[1]) + "))";
      default: {
        const char* op = x.k == EK::Add ? " + " : x.k == EK::Sub ? " - " : " * ";
        if (f) return "((F)(" + expr(x.args[0]) + op + expr(x.args[1]) + "))";
        return "(" + expr(x.args[0]) + op + expr(x.args[1]) + ")";
      }
    }
  }

  const Problem& p_;
  const MdHom& e_;
  std::string ft_;
};

class EmittedRoutine final : public Routine {
 public:
  explicit EmittedRoutine(const Problem& p) : p_(p) {}
  const char* family() const override { return "emitted"; }
  int launches() const override { return G_ ? 2 : 1; }
  std::string source() const override { return src_; }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  std::string describe() const override {
    std::ostringstream os;
    os << "{\"kernel\": \"mdh_emitted" << (G_ ? "_split" : "") << " (NVRTC sm_100a)\", \"cells\": " << cells_
       << ", \"fiber_parts\": " << G_ << ", \"source_bytes\": " << src_.size() << ", \"threads_per_cta\": " << (G_ ? 256 : 128) << "}";
    return os.str();
  }
  bool setup() {
    Emitter em(p_);
    cells_ = em.cells();
    MDHB_CUDA(cudaSetDevice(p_.opt.device));
    G_ = em.split_parts(sm_count(p_.opt.device));
    src_ = G_ ? em.source_split(G_) : em.source();
    k_ = compile_source(src_, p_.opt.device);
    if (G_) {
      std::lock_guard<std::mutex> lk(g_mu);
      MDHB_CUDA(cudaLibraryGetKernel(&kfinal_, k_.lib, "mdh_emitted_final"));
      // Part = one 8-byte slot per component + int flag, padded to 8
      part_bytes_ = static_cast<size_t>(cells_ * G_) * (8 * p_.e.assigns.size() + 8);
      MDHB_CUDA(cudaMalloc(&part_, part_bytes_));
    }
    const MdHom& e = p_.e;
    for (size_t b = 0; b < e.out.size(); ++b) {
      int64_t n = 1;
      for (int64_t x : p_.out_ext[b]) n *= x;
      out_cells_.push_back(n);
      zero_out_.push_back(cells_ * static_cast<int64_t>(e.out[b].acc.size()) < n);
    }
    return true;
  }
  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    const MdHom& e = p_.e;
    EmPtrs ptr{};
    for (size_t b = 0; b < e.in.size(); ++b) ptr.in[b] = d_in[b];
    for (size_t b = 0; b < e.out.size(); ++b) {
      ptr.out[b] = d_out[b];
      if (zero_out_[b])
        MDHB_CUDA(cudaMemsetAsync(d_out[b], 0, static_cast<size_t>(out_cells_[b]) * store_bytes(p_.out_store[b]), s));
    }
    if (cells_ == 0) return;
    MarkScope mark(this, s);
    if (G_) {
      void* args[] = {&ptr, &part_};
      MDHB_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(k_.kern), dim3(static_cast<unsigned>(cells_ * G_)), dim3(256),
                                 args, 0, s));
      MDHB_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(kfinal_), dim3(static_cast<unsigned>((cells_ + 127) / 128)),
                                 dim3(128), args, 0, s));
      return;
    }
    void* args[] = {&ptr};
    MDHB_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(k_.kern), dim3(static_cast<unsigned>((cells_ + 127) / 128)),
                               dim3(128), args, 0, s));
  }
  ~EmittedRoutine() override {
    if (part_) cudaFree(part_);
  }

 private:
  const Problem& p_;
  std::string src_;
  int64_t cells_ = 0, G_ = 0;
  Compiled k_;
  cudaKernel_t kfinal_ = nullptr;
  void* part_ = nullptr;
  size_t part_bytes_ = 0;
  std::vector<int64_t> out_cells_;
  std::vector<bool> zero_out_;
};

}  // namespace

std::unique_ptr<Routine> make_emitted(const Problem& p, const Config* cfg, Config* cfg_out) {
  const MdHom& e = p.e;
  if (std::getenv("MDHB_NO_EMIT")) return nullptr;
  for (auto& c : e.comb)
    if (c.kind == Combine::PS) return nullptr;  // prefix dims: generic VM (or the scan family)
  if (e.in.size() > static_cast<size_t>(kMaxBuf) || e.out.size() > static_cast<size_t>(kMaxBuf)) return nullptr;
  if (!nvrtc().ok) return nullptr;
  auto r = std::make_unique<EmittedRoutine>(p);
  r->setup();
  if (cfg_out) *cfg_out = cfg ? *cfg : baseline_config(e, p.m);
  return r;
}

}  // namespace mdhb
