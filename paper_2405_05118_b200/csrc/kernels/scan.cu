// Scan family: md_homs with one prefix-sum dimension (`ps:op`, op in + * min
// max), every other dimension `++`, and the identity scalar function
// out(1,1) = in(1,1) -- the reference's scan.json and mbbs.json
// (proj/data/computations/; the prefix pass of engine.cpp:337-353 and the
// emitted scan of codegen.cpp:865-906).  SURVEY §8(f)2.
//
// Reference semantics: after the (trivial) fold, the result is scanned in
// place along the ps dim d in ascending order, acc[t] = acc[t] (+) acc[t-1],
// then scattered through the output view.  Every op the reference allows on
// ps dims is associative and commutative, so a parallel scan gives the same
// integers bit for bit; for float storage it gives a re-associated sum (the
// stated FP32 tolerance), and f64 storage stays on the generic family's
// sequential per-line scan (bit-exact fold order).
//
// Two kernels, chosen by where the scan dimension lies in memory:
//   * scan_tiles  -- the ps dim is unit-stride in input and output: a
//     single-pass decoupled look-back scan.  Tiles of 5120 elements (128
//     threads x 10 rounds x 4, 8 CTAs per SM so the look-back of one CTA hides
//     behind the loads of the others; rounds x threads x CTAs/SM swept over
//     17 shapes with tools/scan_variants.sh: 10 x 128 x 8 354 us, 8 x 128 x 8
//     367 us, 12 x 128 x 6 362 us, 16 x 128 x 4 405 us on 2^28 int32) are claimed in order from an atomic
//     counter; each publishes its aggregate, then its inclusive prefix, in a per-tile
//     status word (flag | value packed in 64 bits for 32-bit types, a flag
//     word fenced after the value otherwise).  Per element: one read, one
//     write -- the HBM roofline of a copy.
//   * scan_lines  -- the ps dim is strided (mbbs: scan over rows): one thread
//     per line walks it sequentially; neighbouring threads own neighbouring
//     lines, so every step is a coalesced row read and row write.
#include <algorithm>
#include <climits>
#include <cfloat>
#include <cstring>
#include <sstream>

#include "../plan.hpp"

namespace mdhb {
namespace {

#ifndef MDHB_SCAN_ROUNDS
#define MDHB_SCAN_ROUNDS 10
#endif
#ifndef MDHB_SCAN_THREADS
#define MDHB_SCAN_THREADS 128
#endif
#ifndef MDHB_SCAN_MINB
#define MDHB_SCAN_MINB 8
#endif
constexpr int SC_THREADS = MDHB_SCAN_THREADS, SC_ROUNDS = MDHB_SCAN_ROUNDS, SC_VEC = 4;
constexpr int SC_TILE = SC_THREADS * SC_ROUNDS * SC_VEC;  // elements per tile
constexpr int kScanMaxD = 15;

struct ScanArgs {
  const void* in;
  void* out;
  int64_t n;              // scan length (extent of dim d)
  int64_t lines;          // product of the other extents
  int64_t tiles_per_line;
  // line index -> base offsets: mixed radix over the other dims (outer -> inner)
  int nd;
  int64_t ext[kScanMaxD], cin[kScanMaxD], cout[kScanMaxD];
  int64_t in0, out0;      // constant offsets
  int64_t sin, sout;      // strides along d
  unsigned long long* status;   // [lines * tiles_per_line] (flag << 62 | value) or flags
  unsigned long long* values;   // 64-bit values (wide types)
  unsigned int* counter;
  int vec;                // 16-byte vector path allowed
};

template <typename T, int OP>
__device__ __forceinline__ T op_apply(T a, T b) {
  if (OP == 0) return a + b;
  if (OP == 2) return a * b;
  if (OP == 4) return b < a ? b : a;
  return b > a ? b : a;
}
template <typename T>
struct Lim;
template <>
struct Lim<float> {
  static __device__ float lo() { return -FLT_MAX; }
  static __device__ float hi() { return FLT_MAX; }
};
template <>
struct Lim<double> {
  static __device__ double lo() { return -DBL_MAX; }
  static __device__ double hi() { return DBL_MAX; }
};
template <>
struct Lim<int32_t> {
  static __device__ int32_t lo() { return INT_MIN; }
  static __device__ int32_t hi() { return INT_MAX; }
};
template <>
struct Lim<long long> {
  static __device__ long long lo() { return LLONG_MIN; }
  static __device__ long long hi() { return LLONG_MAX; }
};
template <typename T, int OP>
__device__ __forceinline__ T op_identity() {
  if (OP == 0) return T(0);
  if (OP == 2) return T(1);
  if (OP == 4) return Lim<T>::hi();
  return Lim<T>::lo();
}

__device__ __forceinline__ void line_base(const ScanArgs& a, int64_t line, int64_t& bi, int64_t& bo) {
  bi = a.in0;
  bo = a.out0;
  for (int q = a.nd - 1; q >= 0; --q) {
    const int64_t x = line % a.ext[q];
    line /= a.ext[q];
    bi += x * a.cin[q];
    bo += x * a.cout[q];
  }
}

template <typename T>
__device__ __forceinline__ unsigned long long to_bits(T v) {
  if (sizeof(T) == 4) {
    uint32_t u;
    memcpy(&u, &v, 4);
    return u;
  }
  unsigned long long u;
  memcpy(&u, &v, 8);
  return u;
}
template <typename T>
__device__ __forceinline__ T from_bits(unsigned long long u) {
  T v;
  if (sizeof(T) == 4) {
    uint32_t w = static_cast<uint32_t>(u);
    memcpy(&v, &w, 4);
  } else {
    memcpy(&v, &u, 8);
  }
  return v;
}

constexpr unsigned long long F_AGG = 1ull << 62, F_INC = 2ull << 62, F_MASK = 3ull << 62;

// status publication / observation.  32-bit types: one packed 64-bit word.
// 64-bit types: value in `values`, then a fence, then the flag in `status`.
template <typename T>
__device__ __forceinline__ void publish(const ScanArgs& a, int64_t slot, unsigned long long flag, T v) {
  if (sizeof(T) == 4) {
    atomicExch(a.status + slot, flag | to_bits(v));
  } else {
    // separate words for the aggregate and the inclusive prefix: a reader
    // that saw F_AGG must not pick up the later inclusive value
    atomicExch(a.values + 2 * slot + (flag == F_INC ? 1 : 0), to_bits(v));
    __threadfence();
    atomicExch(a.status + slot, flag);
  }
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
// Spins until tile `slot` has published; returns its flag and value.
template <typename T>
__device__ __forceinline__ unsigned long long observe(const ScanArgs& a, int64_t slot, T& v) {
  unsigned long long w;
  for (unsigned ns = 8;; ns = ns < 256 ? 2 * ns : ns) {
    w = sizeof(T) == 4 ? ld_relaxed(a.status + slot) : ld_acquire(a.status + slot);
    if (w & F_MASK) break;
    __nanosleep(ns);
  }
  if (sizeof(T) == 4) v = from_bits<T>(w & 0xffffffffull);
  else v = from_bits<T>(ld_relaxed(a.values + 2 * slot + ((w & F_MASK) == F_INC ? 1 : 0)));
  return w & F_MASK;
}

template <typename T, int OP>
__global__ void __launch_bounds__(SC_THREADS, MDHB_SCAN_MINB) scan_tiles(ScanArgs a) {
  __shared__ T wsum[SC_ROUNDS][SC_THREADS / 32];
  __shared__ T tile_prefix;
  __shared__ unsigned int s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(a.counter, 1u);
  __syncthreads();
  const int64_t id = s_tile;  // claimed in order: every predecessor is running or done
  const int64_t line = id / a.tiles_per_line, tile = id % a.tiles_per_line;
  int64_t bi, bo;
  line_base(a, line, bi, bo);
  const T* in = static_cast<const T*>(a.in) + bi;
  T* out = static_cast<T*>(a.out) + bo;
  const int64_t t0 = tile * SC_TILE;
  const T idn = op_identity<T, OP>();
  // ---- load: round r, thread t owns elements t0 + r*1024 + 4t .. +3 (coalesced rows)
  T v[SC_ROUNDS][SC_VEC];
#pragma unroll
  for (int r = 0; r < SC_ROUNDS; ++r) {
    const int64_t e = t0 + r * (SC_THREADS * SC_VEC) + tid * SC_VEC;
    if (a.vec && e + SC_VEC <= a.n) {
      if (sizeof(T) == 4) {
        const int4 q = __ldcs(reinterpret_cast<const int4*>(in + e));
        memcpy(&v[r][0], &q.x, 4), memcpy(&v[r][1], &q.y, 4), memcpy(&v[r][2], &q.z, 4), memcpy(&v[r][3], &q.w, 4);
      } else {
        const longlong2 q0 = __ldcs(reinterpret_cast<const longlong2*>(in + e));
        const longlong2 q1 = __ldcs(reinterpret_cast<const longlong2*>(in + e + 2));
        memcpy(&v[r][0], &q0.x, 8), memcpy(&v[r][1], &q0.y, 8), memcpy(&v[r][2], &q1.x, 8), memcpy(&v[r][3], &q1.y, 8);
      }
    } else {
#pragma unroll
      for (int k = 0; k < SC_VEC; ++k) v[r][k] = e + k < a.n ? in[(e + k) * a.sin] : idn;
    }
  }
  // ---- thread-local inclusive scans, then a block scan of the thread totals
  T tot[SC_ROUNDS];
#pragma unroll
  for (int r = 0; r < SC_ROUNDS; ++r) {
#pragma unroll
    for (int k = 1; k < SC_VEC; ++k) v[r][k] = op_apply<T, OP>(v[r][k - 1], v[r][k]);
    tot[r] = v[r][SC_VEC - 1];
  }
  T incl[SC_ROUNDS];
#pragma unroll
  for (int r = 0; r < SC_ROUNDS; ++r) {
    T x = tot[r];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = op_apply<T, OP>(y, x);
    }
    incl[r] = x;
    if (lane == 31) wsum[r][warp] = x;
  }
  __syncthreads();
  // warp prefixes within each round, and round totals
  T round_tot[SC_ROUNDS], warp_excl[SC_ROUNDS];
#pragma unroll
  for (int r = 0; r < SC_ROUNDS; ++r) {
    T acc = idn, mine = idn;
#pragma unroll
    for (int w = 0; w < SC_THREADS / 32; ++w) {
      if (w == warp) mine = acc;
      acc = op_apply<T, OP>(acc, wsum[r][w]);
    }
    warp_excl[r] = mine;
    round_tot[r] = acc;
  }
  T aggregate = idn;
#pragma unroll
  for (int r = 0; r < SC_ROUNDS; ++r) aggregate = op_apply<T, OP>(aggregate, round_tot[r]);
  // ---- decoupled look-back for the tile's exclusive prefix
  const int64_t slot = id;  // tile ids are line-major
  if (warp == 0) {
    if (tile == 0) {
      if (lane == 0) {
        publish<T>(a, slot, F_INC, aggregate);
        tile_prefix = idn;
      }
    } else {
      if (lane == 0) publish<T>(a, slot, F_AGG, aggregate);
      // warp-parallel look-back: lane l observes tile p - l; the window is
      // folded up to (and including) the newest inclusive prefix in it, else
      // entirely, and the walk moves 32 tiles further back.  The first tile
      // of the line is always inclusive, so the walk never leaves the line.
      const int64_t first = slot - tile;
      T prefix = idn;
      for (int64_t p = slot - 1;; p -= 32) {
        const int64_t q = p - lane;
        T v = idn;
        unsigned long long f = F_INC;
        if (q >= first) f = observe<T>(a, q, v);
        const unsigned inc = __ballot_sync(0xffffffffu, f == F_INC);
        const int stop = inc ? __ffs(inc) - 1 : 31;  // lanes 0..stop contribute
        if (lane > stop) v = idn;
        // fold the window, older tiles (higher lanes) on the left
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const T y = __shfl_down_sync(0xffffffffu, v, o);
          if (lane + o < 32) v = op_apply<T, OP>(y, v);
        }
        prefix = op_apply<T, OP>(__shfl_sync(0xffffffffu, v, 0), prefix);
        if (inc) break;
      }
      if (lane == 0) {
        publish<T>(a, slot, F_INC, op_apply<T, OP>(prefix, aggregate));
        tile_prefix = prefix;
      }
    }
  }
  __syncthreads();
  const T tp = tile_prefix;
  // ---- outputs: tile prefix (+) earlier rounds (+) earlier warps (+) earlier lanes (+) local
  T run = tp;
#pragma unroll
  for (int r = 0; r < SC_ROUNDS; ++r) {
    T ex = __shfl_up_sync(0xffffffffu, incl[r], 1);
    if (lane == 0) ex = idn;
    const T base = op_apply<T, OP>(op_apply<T, OP>(run, warp_excl[r]), ex);
    T o[SC_VEC];
#pragma unroll
    for (int k = 0; k < SC_VEC; ++k) o[k] = op_apply<T, OP>(base, v[r][k]);
    run = op_apply<T, OP>(run, round_tot[r]);
    const int64_t e = t0 + r * (SC_THREADS * SC_VEC) + tid * SC_VEC;
    if (a.vec && e + SC_VEC <= a.n) {
      if (sizeof(T) == 4) {
        int4 q;
        memcpy(&q.x, &o[0], 4), memcpy(&q.y, &o[1], 4), memcpy(&q.z, &o[2], 4), memcpy(&q.w, &o[3], 4);
        __stcs(reinterpret_cast<int4*>(out + e), q);
      } else {
        longlong2 q0, q1;
        memcpy(&q0.x, &o[0], 8), memcpy(&q0.y, &o[1], 8), memcpy(&q1.x, &o[2], 8), memcpy(&q1.y, &o[3], 8);
        __stcs(reinterpret_cast<longlong2*>(out + e), q0);
        __stcs(reinterpret_cast<longlong2*>(out + e + 2), q1);
      }
    } else {
#pragma unroll
      for (int k = 0; k < SC_VEC; ++k)
        if (e + k < a.n) out[(e + k) * a.sout] = o[k];
    }
  }
}

// strided scan dimension: one thread per line, sequential along d
template <typename T, int OP>
__global__ void __launch_bounds__(256) scan_lines(ScanArgs a) {
  const int64_t line = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  if (line >= a.lines) return;
  int64_t bi, bo;
  line_base(a, line, bi, bo);
  const T* in = static_cast<const T*>(a.in) + bi;
  T* out = static_cast<T*>(a.out) + bo;
  T run = in[0];
  out[0] = run;
  for (int64_t t = 1; t < a.n; ++t) {
    run = op_apply<T, OP>(run, in[t * a.sin]);  // acc[t] = acc[t] (+) acc[t-1]: commutative ops
    out[t * a.sout] = run;
  }
}

bool identity_scalar(const MdHom& e) {
  if (e.assigns.size() != 1 || e.in.size() != 1 || e.out.size() != 1) return false;
  if (e.in[0].acc.size() != 1 || e.out[0].acc.size() != 1) return false;
  const Expr& f = e.assigns[0].e;
  return f.k == EK::In && f.buf == 1 && f.acc == 1 && e.in[0].type == e.out[0].type;
}

class ScanRoutine final : public Routine {
 public:
  ScanRoutine(const Problem& p, int d) : p_(p), d_(d) {}
  ~ScanRoutine() override {
    if (scratch_) cudaFree(scratch_);
  }
  const char* family() const override { return "scan"; }
  int launches() const override { return tiles_ ? 1 : 1; }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  std::string describe() const override {
    std::ostringstream os;
    os << "{\"kernel\": \"" << (tiles_ ? "scan_tiles<" : "scan_lines<") << store_name(st_) << "," << op_name() << ">\""
       << ", \"n\": " << a_.n << ", \"lines\": " << a_.lines;
    if (tiles_) os << ", \"tile\": " << SC_TILE << ", \"tiles\": " << a_.lines * a_.tiles_per_line << ", \"vector\": " << (a_.vec ? "true" : "false");
    os << ", \"threads\": 256}";
    return os.str();
  }
  const char* op_name() const {
    switch (op_) {
      case 0: return "add";
      case 2: return "mul";
      case 4: return "min";
      default: return "max";
    }
  }

  bool setup() {
    const MdHom& e = p_.e;
    const int D = e.D();
    op_ = static_cast<int>(e.comb[static_cast<size_t>(d_)].op);
    if (op_ != 0 && op_ != 2 && op_ != 4 && op_ != 5) return false;
    st_ = p_.in_store[0];
    if (p_.out_store[0] != st_) return false;
    Linear li = linearize(e.in[0].acc[0], p_.in_ext[0], D);
    Linear lo = linearize(e.out[0].acc[0], p_.out_ext[0], D);
    a_.n = e.sizes[static_cast<size_t>(d_)];
    a_.sin = li.cj[static_cast<size_t>(d_)];
    a_.sout = lo.cj[static_cast<size_t>(d_)];
    a_.in0 = li.c0;
    a_.out0 = lo.c0;
    a_.lines = 1;
    a_.nd = 0;
    for (int x = 0; x < D; ++x) {
      if (x == d_) continue;
      if (a_.nd >= kScanMaxD) return false;
      a_.ext[a_.nd] = e.sizes[static_cast<size_t>(x)];
      a_.cin[a_.nd] = li.cj[static_cast<size_t>(x)];
      a_.cout[a_.nd] = lo.cj[static_cast<size_t>(x)];
      a_.lines *= e.sizes[static_cast<size_t>(x)];
      ++a_.nd;
    }
    // output view must be injective over the scanned box (single writer per cell)
    tiles_ = a_.sin == 1 && a_.sout == 1 && a_.n >= 2 * SC_TILE;
    if (!tiles_ && (a_.lines < 1024 && a_.n > 4096)) tiles_ = a_.sin == 1 && a_.sout == 1;
    if (tiles_) {
      a_.tiles_per_line = (a_.n + SC_TILE - 1) / SC_TILE;
      const int64_t esz = static_cast<int64_t>(store_bytes(st_));
      bool vec = true;
      for (int q = 0; q < a_.nd; ++q) vec = vec && (a_.cin[q] * esz) % 16 == 0 && (a_.cout[q] * esz) % 16 == 0;
      vec = vec && (a_.in0 * esz) % 16 == 0 && (a_.out0 * esz) % 16 == 0;
      a_.vec = vec ? 1 : 0;
      const int64_t nt = a_.lines * a_.tiles_per_line;
      status_bytes_ = static_cast<size_t>(nt) * 8 * (esz == 8 ? 3 : 1) + 256;
      MDHB_CUDA(cudaSetDevice(p_.opt.device));
      MDHB_CUDA(cudaMalloc(&scratch_, status_bytes_));
      a_.counter = static_cast<unsigned int*>(scratch_);
      a_.status = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch_) + 256);
      a_.values = esz == 8 ? a_.status + nt : nullptr;
    } else {
      a_.tiles_per_line = 1;
    }
    return true;
  }

  template <typename T>
  void go(cudaStream_t s) {
    if (tiles_) {
      const int64_t nt = a_.lines * a_.tiles_per_line;
      // counter + flags reset (the value words need no reset: read only after a flag)
      MDHB_CUDA(cudaMemsetAsync(scratch_, 0, 256 + static_cast<size_t>(nt) * 8, s));
      switch (op_) {
        case 0: scan_tiles<T, 0><<<static_cast<unsigned>(nt), SC_THREADS, 0, s>>>(a_); break;
        case 2: scan_tiles<T, 2><<<static_cast<unsigned>(nt), SC_THREADS, 0, s>>>(a_); break;
        case 4: scan_tiles<T, 4><<<static_cast<unsigned>(nt), SC_THREADS, 0, s>>>(a_); break;
        default: scan_tiles<T, 5><<<static_cast<unsigned>(nt), SC_THREADS, 0, s>>>(a_); break;
      }
    } else {
      const unsigned g = static_cast<unsigned>((a_.lines + 255) / 256);
      switch (op_) {
        case 0: scan_lines<T, 0><<<g, 256, 0, s>>>(a_); break;
        case 2: scan_lines<T, 2><<<g, 256, 0, s>>>(a_); break;
        case 4: scan_lines<T, 4><<<g, 256, 0, s>>>(a_); break;
        default: scan_lines<T, 5><<<g, 256, 0, s>>>(a_); break;
      }
    }
    MDHB_CUDA(cudaGetLastError());
  }

  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    a_.in = d_in[0];
    a_.out = d_out[0];
    // cells of the output buffer the view does not reach stay zero (generic family rule)
    if (zero_out_) MDHB_CUDA(cudaMemsetAsync(d_out[0], 0, static_cast<size_t>(out_cells_) * store_bytes(st_), s));
    MarkScope mark(this, s);
    switch (st_) {
      case Store::F32: go<float>(s); break;
      case Store::F64: go<double>(s); break;
      case Store::I32: go<int32_t>(s); break;
      default: go<long long>(s); break;
    }
  }

  bool zero_out_ = false;
  int64_t out_cells_ = 0;

 private:
  const Problem& p_;
  int d_;
  int op_ = 0;
  Store st_ = Store::I64;
  bool tiles_ = false;
  ScanArgs a_{};
  void* scratch_ = nullptr;
  size_t status_bytes_ = 0;
};

}  // namespace

std::unique_ptr<Routine> make_scan(const Problem& p, const Config* cfg, Config* cfg_out) {
  const MdHom& e = p.e;
  int d = -1;
  for (int x = 0; x < e.D(); ++x) {
    const auto k = e.comb[static_cast<size_t>(x)].kind;
    if (k == Combine::PW) return nullptr;
    if (k == Combine::PS) {
      if (d >= 0) return nullptr;  // one scan dim
      d = x;
    }
  }
  if (d < 0 || !identity_scalar(e)) return nullptr;
  // f64 storage keeps the reference's sequential fold order (generic family)
  if (e.in[0].type == Ty::F64 && p.opt.fstore == Store::F64) return nullptr;
  if (cfg) fail("Unsupported", "scan template is not instantiated from a configuration");
  auto r = std::make_unique<ScanRoutine>(p, d);
  if (!r->setup()) return nullptr;
  int64_t n = 1;
  for (int64_t x : p.out_ext[0]) n *= x;
  int64_t reach = 1;
  for (int64_t x : e.sizes) reach *= x;
  r->out_cells_ = n;
  r->zero_out_ = reach < n;
  if (cfg_out) *cfg_out = baseline_config(e, p.m);
  return r;
}

}  // namespace mdhb
