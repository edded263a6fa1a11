// Generic md_hom family: any well-formed md_hom (cc / pw:op / ps:op dims, any
// affine views, any scalar function of the reference's language) executed
// on the device.  This is the catch-all that keeps the backend a drop-in for
// every computation the reference accepts; the routine classes of the
// BASELINE configs have specialised families (contraction, stencil, prl).
//
// Semantics follow engine::run (proj/src/engine.cpp:222-375) exactly:
//   * one thread owns one cell of the combined result (collapsed ranges,
//     engine.cpp:313-335) and folds the scalar function over its point-wise
//     fiber in ascending lexicographic order -- the lex_plan order
//     (engine.cpp:215-220), so f64 results are bit-identical to the oracle;
//   * the scalar function runs as the reference's stack bytecode
//     (engine.cpp:34-81, 134-176), interpreted per point;
//   * ps dims get an ascending in-place scan per dimension (engine.cpp:337-353);
//   * the result is scattered through the output view (views.cpp:242-275).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <sstream>

#include "../plan.hpp"

namespace mdhb {
namespace {

constexpr int kMaxD = 15;
constexpr int kMaxStack = 32;

enum Op : int32_t {
  LIT_I, LIT_F, IN_I, IN_F, IDX, ADD_I, ADD_F, SUB_I, SUB_F, MUL_I, MUL_F, DIV_I, DIV_F,
  MIN_I, MIN_F, MAX_I, MAX_F, ABS_I, ABS_F, CMP_I, CMP_F, SELECT
};

struct Instr {
  int32_t op, arg;
  int64_t ilit;
  double flit;
};

struct VmAccess {
  int64_t c0;
  int64_t cj[kMaxD];
  int32_t buf;    // buffer slot in the pointer array
  int32_t store;  // Store of that buffer
};

struct VmParams {
  int D;
  int64_t sizes[kMaxD];
  int32_t kind[kMaxD];   // 0 cc, 1 pw, 2 ps
  int64_t cstride[kMaxD];  // row-major stride of the collapsed result, 0 on pw dims
  int n_pw;
  int32_t pw_dims[kMaxD];
  int64_t cells;
  int fold;  // Fold enum, -1 none
  int custom_vm;  // built-in custom operator compiled into the VM (1 = max_prl), 0 none
  int n_in_acc;
  const VmAccess* in_acc;
  int n_comp;
  const int32_t* comp_start;
  const int32_t* comp_len;
  const int32_t* comp_float;
  const Instr* code;
  int n_out_acc;
  const VmAccess* out_acc;
  const int32_t* out_comp;
  // accumulator scratch (ps dims only): [comp][cells] as 8-byte slots
  int64_t* acc;
};

union Slot {
  int64_t i;
  double f;
};

template <typename FT>
__device__ __forceinline__ void load_in(Slot& s, const void* base, int store, int64_t off, bool want_float) {
  switch (store) {
    case 0: s.f = static_cast<double>(static_cast<const float*>(base)[off]); break;
    case 1: s.f = static_cast<const double*>(base)[off]; break;
    case 2: s.i = static_cast<const int32_t*>(base)[off]; break;
    default: s.i = static_cast<const int64_t*>(base)[off]; break;
  }
  (void)want_float;
}

// Float arithmetic happens in FT (float when buffers are stored as f32,
// double when stored as f64); slots carry doubles for uniformity.
template <typename FT>
__device__ __forceinline__ double fop(double a) { return static_cast<double>(static_cast<FT>(a)); }

template <typename FT>
__device__ void eval(const VmParams& P, const void* const* in, const int64_t* idx, const int64_t* off, Slot* out_vals) {
  Slot st[kMaxStack];
  for (int c = 0; c < P.n_comp; ++c) {
    const Instr* code = P.code + P.comp_start[c];
    int len = P.comp_len[c];
    int sp = 0;
    for (int k = 0; k < len; ++k) {
      Instr ins = code[k];
      switch (ins.op) {
        case LIT_I: st[sp++].i = ins.ilit; break;
        case LIT_F: st[sp++].f = fop<FT>(ins.flit); break;
        case IN_I:
        case IN_F: {
          const VmAccess& a = P.in_acc[ins.arg];
          load_in<FT>(st[sp], in[a.buf], a.store, off[ins.arg], ins.op == IN_F);
          ++sp;
          break;
        }
        case IDX: st[sp++].i = idx[ins.arg]; break;
        case ADD_I: --sp; st[sp - 1].i += st[sp].i; break;
        case SUB_I: --sp; st[sp - 1].i -= st[sp].i; break;
        case MUL_I: --sp; st[sp - 1].i *= st[sp].i; break;
        case DIV_I: --sp; st[sp - 1].i = st[sp].i == 0 ? 0 : st[sp - 1].i / st[sp].i; break;
        case ADD_F: --sp; st[sp - 1].f = fop<FT>(static_cast<FT>(st[sp - 1].f) + static_cast<FT>(st[sp].f)); break;
        case SUB_F: --sp; st[sp - 1].f = fop<FT>(static_cast<FT>(st[sp - 1].f) - static_cast<FT>(st[sp].f)); break;
        case MUL_F: --sp; st[sp - 1].f = fop<FT>(static_cast<FT>(st[sp - 1].f) * static_cast<FT>(st[sp].f)); break;
        case DIV_F: --sp; st[sp - 1].f = fop<FT>(static_cast<FT>(st[sp - 1].f) / static_cast<FT>(st[sp].f)); break;
        // std::min / std::max argument order (engine.cpp:166-169)
        case MIN_I: --sp; st[sp - 1].i = st[sp].i < st[sp - 1].i ? st[sp].i : st[sp - 1].i; break;
        case MIN_F: --sp; st[sp - 1].f = st[sp].f < st[sp - 1].f ? st[sp].f : st[sp - 1].f; break;
        case MAX_I: --sp; st[sp - 1].i = st[sp - 1].i < st[sp].i ? st[sp].i : st[sp - 1].i; break;
        case MAX_F: --sp; st[sp - 1].f = st[sp - 1].f < st[sp].f ? st[sp].f : st[sp - 1].f; break;
        case ABS_I: st[sp - 1].i = st[sp - 1].i < 0 ? -st[sp - 1].i : st[sp - 1].i; break;
        case ABS_F: st[sp - 1].f = fabs(st[sp - 1].f); break;
        case CMP_I: --sp; st[sp - 1].i = st[sp - 1].i < st[sp].i ? -1 : (st[sp - 1].i > st[sp].i ? 1 : 0); break;
        case CMP_F: --sp; st[sp - 1].i = st[sp - 1].f < st[sp].f ? -1 : (st[sp - 1].f > st[sp].f ? 1 : 0); break;
        case SELECT: sp -= 2; st[sp - 1] = st[sp - 1].i != 0 ? st[sp] : st[sp + 1]; break;
        default: break;
      }
    }
    out_vals[c] = st[0];
  }
}

template <typename FT>
__device__ __forceinline__ void fold_into(int fold, bool is_f, Slot& acc, Slot v) {
  if (is_f) {
    FT a = static_cast<FT>(acc.f), b = static_cast<FT>(v.f);
    switch (fold) {
      case 0: a = a + b; break;
      case 2: a = a * b; break;
      case 4: a = b < a ? b : a; break;
      case 5: a = b > a ? b : a; break;
      default: break;
    }
    acc.f = static_cast<double>(a);
  } else {
    switch (fold) {
      case 0: acc.i += v.i; break;
      case 2: acc.i *= v.i; break;
      case 4: acc.i = v.i < acc.i ? v.i : acc.i; break;
      case 5: acc.i = v.i > acc.i ? v.i : acc.i; break;
      default: break;
    }
  }
}

// built-in custom operators fold the whole component tuple; b better than a?
__device__ __forceinline__ bool tuple_better(int op, const int32_t* comp_float, const Slot* a, const Slot* b) {
  switch (op) {
    case 1: {  // max_prl: larger key (component 0), lower payload (component 1) on ties
      const bool gt = comp_float[0] ? b[0].f > a[0].f : b[0].i > a[0].i;
      const bool eq = comp_float[0] ? b[0].f == a[0].f : b[0].i == a[0].i;
      const bool lt1 = comp_float[1] ? b[1].f < a[1].f : b[1].i < a[1].i;
      return gt || (eq && lt1);
    }
    default: return false;
  }
}

__device__ __forceinline__ void store_out(void* base, int store, int64_t off, Slot v, bool is_f) {
  switch (store) {
    case 0: static_cast<float*>(base)[off] = static_cast<float>(is_f ? v.f : static_cast<double>(v.i)); break;
    case 1: static_cast<double*>(base)[off] = is_f ? v.f : static_cast<double>(v.i); break;
    case 2: static_cast<int32_t*>(base)[off] = static_cast<int32_t>(v.i); break;
    default: static_cast<int64_t*>(base)[off] = v.i; break;
  }
}

constexpr int kMaxComp = 8;
constexpr int kMaxBufs = 16;

// Buffer pointers travel by value in the kernel parameters.
struct Ptrs {
  const void* in[kMaxBufs];
  void* out[kMaxBufs];
};

// One thread per result cell: fold over the point-wise fiber, then either
// scatter (no ps dims) or park the folded value for the prefix pass.
template <typename FT>
__global__ void __launch_bounds__(128) vm_fold(VmParams P, Ptrs ptr, int direct) {
  const void* const* in = ptr.in;
  void* const* out = ptr.out;
  int64_t cell = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (cell >= P.cells) return;
  int64_t idx[kMaxD];
  int64_t rem = cell;
  for (int d = P.D - 1; d >= 0; --d) {
    if (P.kind[d] == 1) {
      idx[d] = 0;
      continue;
    }
    idx[d] = rem % P.sizes[d];
    rem /= P.sizes[d];
  }
  int64_t off[64];
  for (int a = 0; a < P.n_in_acc; ++a) {
    int64_t o = P.in_acc[a].c0;
    for (int d = 0; d < P.D; ++d) o += P.in_acc[a].cj[d] * idx[d];
    off[a] = o;
  }
  Slot acc[kMaxComp], v[kMaxComp];
  bool first = true;
  for (;;) {
    eval<FT>(P, in, idx, off, v);
    if (first) {
      for (int c = 0; c < P.n_comp; ++c) acc[c] = v[c];
      first = false;
    } else if (P.custom_vm) {
      if (tuple_better(P.custom_vm, P.comp_float, acc, v))
        for (int c = 0; c < P.n_comp; ++c) acc[c] = v[c];
    } else {
      for (int c = 0; c < P.n_comp; ++c) fold_into<FT>(P.fold, P.comp_float[c] != 0, acc[c], v[c]);
    }
    // advance the pw fiber odometer (innermost = highest dim)
    int k = P.n_pw - 1;
    for (; k >= 0; --k) {
      int d = P.pw_dims[k];
      if (idx[d] + 1 < P.sizes[d]) {
        ++idx[d];
        for (int a = 0; a < P.n_in_acc; ++a) off[a] += P.in_acc[a].cj[d];
        break;
      }
      for (int a = 0; a < P.n_in_acc; ++a) off[a] -= P.in_acc[a].cj[d] * idx[d];
      idx[d] = 0;
    }
    if (k < 0) break;
  }
  if (direct) {
    for (int a = 0; a < P.n_out_acc; ++a) {
      const VmAccess& oa = P.out_acc[a];
      int64_t o = oa.c0;
      for (int d = 0; d < P.D; ++d) o += oa.cj[d] * (P.kind[d] == 1 ? 0 : idx[d]);
      int c = P.out_comp[a];
      store_out(out[oa.buf], oa.store, o, acc[c], P.comp_float[c] != 0);
    }
  } else {
    for (int c = 0; c < P.n_comp; ++c) P.acc[static_cast<int64_t>(c) * P.cells + cell] = acc[c].i;
  }
}

// Ascending scan along ps dim `d` (engine.cpp:337-353): one thread per line.
template <typename FT>
__global__ void vm_prefix(VmParams P, int d, int64_t lines) {
  int64_t line = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (line >= lines) return;
  // enumerate cells with coordinate 0 along d: decompose `line` over the other dims
  int64_t base = 0, rem = line;
  for (int e = P.D - 1; e >= 0; --e) {
    if (e == d || P.kind[e] == 1) continue;
    base += (rem % P.sizes[e]) * P.cstride[e];
    rem /= P.sizes[e];
  }
  int64_t st = P.cstride[d];
  if (P.custom_vm) {  // tuple operator: the running best tuple carries forward
    Slot prev[kMaxComp], cur[kMaxComp];
    for (int c = 0; c < P.n_comp; ++c) prev[c].i = P.acc[static_cast<int64_t>(c) * P.cells + base];
    for (int64_t t = 1; t < P.sizes[d]; ++t) {
      for (int c = 0; c < P.n_comp; ++c) cur[c].i = P.acc[static_cast<int64_t>(c) * P.cells + base + t * st];
      if (tuple_better(P.custom_vm, P.comp_float, cur, prev))
        for (int c = 0; c < P.n_comp; ++c) cur[c] = prev[c];
      for (int c = 0; c < P.n_comp; ++c) P.acc[static_cast<int64_t>(c) * P.cells + base + t * st] = cur[c].i;
      for (int c = 0; c < P.n_comp; ++c) prev[c] = cur[c];
    }
    return;
  }
  for (int c = 0; c < P.n_comp; ++c) {
    int64_t* a = P.acc + static_cast<int64_t>(c) * P.cells;
    Slot prev;
    prev.i = a[base];
    for (int64_t t = 1; t < P.sizes[d]; ++t) {
      Slot cur;
      cur.i = a[base + t * st];
      fold_into<FT>(P.fold, P.comp_float[c] != 0, cur, prev);
      a[base + t * st] = cur.i;
      prev = cur;
    }
  }
}

__global__ void vm_scatter(VmParams P, Ptrs ptr) {
  void* const* out = ptr.out;
  int64_t cell = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (cell >= P.cells) return;
  int64_t idx[kMaxD];
  int64_t rem = cell;
  for (int d = P.D - 1; d >= 0; --d) {
    if (P.kind[d] == 1) {
      idx[d] = 0;
      continue;
    }
    idx[d] = rem % P.sizes[d];
    rem /= P.sizes[d];
  }
  for (int a = 0; a < P.n_out_acc; ++a) {
    const VmAccess& oa = P.out_acc[a];
    int64_t o = oa.c0;
    for (int d = 0; d < P.D; ++d) o += oa.cj[d] * idx[d];
    int c = P.out_comp[a];
    Slot v;
    v.i = P.acc[static_cast<int64_t>(c) * P.cells + cell];
    store_out(out[oa.buf], oa.store, o, v, P.comp_float[c] != 0);
  }
}

// ---------------------------------------------------------------- host side
int compile(const Expr& e, const MdHom& h, std::vector<Instr>& out) {
  const bool f = e.type == Ty::F64;
  auto emit = [&](Op op, int arg = 0, int64_t il = 0, double fl = 0.0) { out.push_back({op, arg, il, fl}); };
  switch (e.k) {
    case EK::Lit:
      if (f) emit(LIT_F, 0, 0, e.fv); else emit(LIT_I, 0, e.iv, 0.0);
      return 1;
    case EK::In: emit(f ? IN_F : IN_I, h.in_comp(e.buf, e.acc)); return 1;
    case EK::Idx: emit(IDX, e.dim - 1); return 1;
    case EK::Abs: {
      int d = compile(e.args[0], h, out);
      emit(f ? ABS_F : ABS_I);
      return d;
    }
    case EK::Cmp: {
      int d1 = compile(e.args[0], h, out), d2 = compile(e.args[1], h, out);
      emit(e.args[0].type == Ty::F64 ? CMP_F : CMP_I);
      return std::max(d1, 1 + d2);
    }
    case EK::Select: {
      int d1 = compile(e.args[0], h, out), d2 = compile(e.args[1], h, out), d3 = compile(e.args[2], h, out);
      emit(SELECT);
      return std::max({d1, 1 + d2, 2 + d3});
    }
    default: {
      int d1 = compile(e.args[0], h, out), d2 = compile(e.args[1], h, out);
      Op op;
      switch (e.k) {
        case EK::Add: op = f ? ADD_F : ADD_I; break;
        case EK::Sub: op = f ? SUB_F : SUB_I; break;
        case EK::Mul: op = f ? MUL_F : MUL_I; break;
        case EK::Div: op = f ? DIV_F : DIV_I; break;
        case EK::Min: op = f ? MIN_F : MIN_I; break;
        default: op = f ? MAX_F : MAX_I; break;
      }
      emit(op);
      return std::max(d1, 1 + d2);
    }
  }
}

class GenericRoutine final : public Routine {
 public:
  explicit GenericRoutine(const Problem& p) : p_(p) {
    const MdHom& e = p.e;
    const int D = e.D();
    if (D > kMaxD) fail("Unsupported", "generic family supports at most 15 dimensions");
    if (e.n_in_access() > 64) fail("Unsupported", "generic family supports at most 64 input accesses");
    if (static_cast<int>(e.assigns.size()) > kMaxComp) fail("Unsupported", "generic family supports at most 8 result components");
    if (e.in.size() > static_cast<size_t>(kMaxBufs) || e.out.size() > static_cast<size_t>(kMaxBufs))
      fail("Unsupported", "generic family supports at most 16 buffers per view");
    std::memset(&P_, 0, sizeof P_);
    P_.D = D;
    P_.fold = e.fold();
    if (P_.fold >= kCustomFoldBase) {
      const CustomCombine& op = combine_at(P_.fold - kCustomFoldBase);
      if (!op.vm_op)
        fail("Unsupported", "custom combine operator '" + op.name +
                                "' has no device-VM implementation (it runs through the emitted family, NVRTC, "
                                "which does not take ps dimensions)");
      P_.custom_vm = op.vm_op;
    }
    std::vector<int64_t> coll = e.collapsed();
    int64_t cells = 1;
    for (int d = D - 1; d >= 0; --d) {
      P_.sizes[d] = e.sizes[static_cast<size_t>(d)];
      P_.kind[d] = e.comb[static_cast<size_t>(d)].kind == Combine::CC ? 0 : (e.comb[static_cast<size_t>(d)].kind == Combine::PW ? 1 : 2);
      if (P_.kind[d] != 1) {
        P_.cstride[d] = cells;
        cells *= coll[static_cast<size_t>(d)];
      }
      if (P_.kind[d] == 2) has_ps_ = true;
    }
    P_.cells = cells;
    for (int d = 0; d < D; ++d)
      if (P_.kind[d] == 1) P_.pw_dims[P_.n_pw++] = d;
    // programs
    std::vector<Instr> code;
    std::vector<int32_t> start, len, isf;
    int depth = 1;
    for (auto& a : e.assigns) {
      start.push_back(static_cast<int32_t>(code.size()));
      depth = std::max(depth, compile(a.e, e, code));
      len.push_back(static_cast<int32_t>(code.size()) - start.back());
      isf.push_back(a.e.type == Ty::F64);
    }
    if (depth > kMaxStack) fail("Unsupported", "scalar function too deep for the device VM");
    // accesses
    std::vector<VmAccess> ia, oa;
    std::vector<int32_t> oc;
    for (size_t b = 0; b < e.in.size(); ++b)
      for (auto& acc : e.in[b].acc) {
        Linear l = linearize(acc, p.in_ext[b], D);
        VmAccess v{};
        v.c0 = l.c0;
        for (int d = 0; d < D; ++d) v.cj[d] = l.cj[static_cast<size_t>(d)];
        v.buf = static_cast<int32_t>(b);
        v.store = static_cast<int32_t>(p.in_store[b]);
        ia.push_back(v);
      }
    int comp = 0;
    for (size_t b = 0; b < e.out.size(); ++b)
      for (auto& acc : e.out[b].acc) {
        Linear l = linearize(acc, p.out_ext[b], D);
        VmAccess v{};
        v.c0 = l.c0;
        for (int d = 0; d < D; ++d) v.cj[d] = l.cj[static_cast<size_t>(d)];
        v.buf = static_cast<int32_t>(b);
        v.store = static_cast<int32_t>(p.out_store[b]);
        oa.push_back(v);
        oc.push_back(comp++);
      }
    // output cells nobody writes stay undefined in the reference; zero them
    // here so the buffers are deterministic (only when coverage is partial).
    for (size_t b = 0; b < e.out.size(); ++b) {
      int64_t n = 1;
      for (int64_t x : p.out_ext[b]) n *= x;
      int64_t reach = cells * static_cast<int64_t>(e.out[b].acc.size());
      zero_out_.push_back(reach < n);
    }
    P_.n_in_acc = static_cast<int>(ia.size());
    P_.n_out_acc = static_cast<int>(oa.size());
    P_.n_comp = static_cast<int>(start.size());
    size_t bytes = code.size() * sizeof(Instr) + (ia.size() + oa.size()) * sizeof(VmAccess) + 4 * sizeof(int32_t) * 64 + 4096;
    MDHB_CUDA(cudaSetDevice(p.opt.device));
    MDHB_CUDA(cudaMalloc(&blob_, bytes));
    char* cur = static_cast<char*>(blob_);
    auto put = [&](const void* src, size_t n) {
      void* dst = cur;
      if (n) MDHB_CUDA(cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice));
      cur += (n + 255) / 256 * 256;
      return dst;
    };
    P_.code = static_cast<const Instr*>(put(code.data(), code.size() * sizeof(Instr)));
    P_.in_acc = static_cast<const VmAccess*>(put(ia.data(), ia.size() * sizeof(VmAccess)));
    P_.out_acc = static_cast<const VmAccess*>(put(oa.data(), oa.size() * sizeof(VmAccess)));
    P_.out_comp = static_cast<const int32_t*>(put(oc.data(), oc.size() * sizeof(int32_t)));
    P_.comp_start = static_cast<const int32_t*>(put(start.data(), start.size() * sizeof(int32_t)));
    P_.comp_len = static_cast<const int32_t*>(put(len.data(), len.size() * sizeof(int32_t)));
    P_.comp_float = static_cast<const int32_t*>(put(isf.data(), isf.size() * sizeof(int32_t)));
    if (has_ps_) MDHB_CUDA(cudaMalloc(&P_.acc, static_cast<size_t>(P_.n_comp * cells) * sizeof(int64_t)));
    f64_ = p.opt.fstore == Store::F64;
  }
  ~GenericRoutine() override {
    if (blob_) cudaFree(blob_);
    if (P_.acc) cudaFree(P_.acc);
  }
  const char* family() const override { return "generic"; }
  std::string describe() const override {
    std::ostringstream os;
    os << "{\"kernel\": \"vm_fold<" << (f64_ ? "double" : "float") << ">\", \"cells\": " << P_.cells
       << ", \"pw_dims\": " << P_.n_pw << ", \"prefix\": " << (has_ps_ ? "true" : "false")
       << ", \"threads_per_cta\": 128}";
    return os.str();
  }
  int launches() const override {
    int n = 1;
    if (has_ps_) {
      for (int d = 0; d < P_.D; ++d) n += P_.kind[d] == 2;
      n += 1;
    }
    return n;
  }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    const MdHom& e = p_.e;
    Ptrs ptr{};
    for (size_t b = 0; b < e.in.size(); ++b) ptr.in[b] = d_in[b];
    for (size_t b = 0; b < e.out.size(); ++b) ptr.out[b] = d_out[b];
    for (size_t b = 0; b < e.out.size(); ++b)
      if (zero_out_[b]) {
        int64_t n = 1;
        for (int64_t x : p_.out_ext[b]) n *= x;
        MDHB_CUDA(cudaMemsetAsync(d_out[b], 0, static_cast<size_t>(n) * store_bytes(p_.out_store[b]), s));
      }
    unsigned grid = static_cast<unsigned>((P_.cells + 127) / 128);
    MarkScope mark(this, s);
    if (f64_)
      vm_fold<double><<<grid, 128, 0, s>>>(P_, ptr, has_ps_ ? 0 : 1);
    else
      vm_fold<float><<<grid, 128, 0, s>>>(P_, ptr, has_ps_ ? 0 : 1);
    MDHB_CUDA(cudaGetLastError());
    if (!has_ps_) return;
    for (int d = 0; d < P_.D; ++d) {
      if (P_.kind[d] != 2) continue;
      int64_t lines = P_.cells / P_.sizes[d];
      unsigned g = static_cast<unsigned>((lines + 127) / 128);
      if (f64_)
        vm_prefix<double><<<g, 128, 0, s>>>(P_, d, lines);
      else
        vm_prefix<float><<<g, 128, 0, s>>>(P_, d, lines);
      MDHB_CUDA(cudaGetLastError());
    }
    vm_scatter<<<grid, 128, 0, s>>>(P_, ptr);
    MDHB_CUDA(cudaGetLastError());
  }

 private:
  const Problem& p_;
  VmParams P_;
  void* blob_ = nullptr;
  bool has_ps_ = false;
  bool f64_ = false;
  std::vector<bool> zero_out_;
};

}  // namespace

std::unique_ptr<Routine> make_generic(const Problem& p, const Config* cfg, Config* cfg_out) {
  (void)cfg;
  if (cfg_out) *cfg_out = cfg ? *cfg : baseline_config(p.e, p.m);
  return std::make_unique<GenericRoutine>(p);
}

}  // namespace mdhb
