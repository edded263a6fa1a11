// PRL family: probabilistic record linkage with the max_PRL custom combine,
// expressed in the reference's own spec language as a packed key folded
// with pw:max (specs/prl_max.json; SURVEY §8 "PRL reconstructed"):
//
//   best[q] = max_r  ( sum_f select(cmp(Q[q][f], D[r][f]), 0, W[f]) ) * S + (C - r)
//
// The key orders candidates by match weight, then by the lowest record id,
// so max over r is order-independent and the result is bit-exact however
// the records are split -- which is what lets the record dimension (a
// point-wise dim) be split across CTAs (SMX) and combined in DM with a
// 64-bit atomicMax, and across GPUs with an NCCL max reduction.
//
// The hot loop is integer-ALU bound (2^35 pairs, ~17.6 MB of data).  A
// de-composition pre-pass (the D4 "layout" parameter) re-encodes the int
// fields as 7-bit codes packed four to a 32-bit word whenever every field
// value lies in a 128-wide window, and the weights as signed bytes; then one
// pair costs LOP3 + IADD + LOP3 (per-byte equality) + DP4A (weighted count)
// + IMAD (key) + IMNMX (fold) -- six instructions for four field compares.
// When the data does not fit that encoding the same kernel takes an exact
// 64-bit path (a device-side flag decides; no host round trip).
//
// The same template also runs the UNPACKED form with the registered custom
// combine operator max_prl (mdh_model.cpp registry; specs/prl_max_prl.json):
//
//   (weight[q], record[q]) = max_prl over r of ( sum_f select(...), r )
//
// i.e. two output buffers folded jointly -- larger weight, lower record on
// ties.  Internally the fast paths pack (w, r) exactly like the spec form
// with S = 2^ceil(log2(max(records, 128))); every thread's best is unpacked
// to a (w, r) pair and committed with a 128-bit compare-and-swap (lexicographic
// max, order-independent); the exact path folds pairs without packing, so
// no weight range is excluded.  prl_unpack writes the two outputs.
#include <climits>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "../plan.hpp"

namespace mdhb {
namespace {

constexpr int kMaxF = 4;  // fields of the packed fast path
constexpr int NT = 256;

struct PrlArgs {
  const void* Q;  // [nq][eq] int32/int64
  const void* D;  // [nr][ed]
  const void* W;  // [ew]
  int64_t* best;  // [nq] (through the output access: best[q * ob_stride])
  int q_is64, d_is64, w_is64, out_is64;
  int64_t nq, nr;
  int64_t qs, ds;  // row strides (elements) of Q and D
  int F;
  int qf[kMaxF], df[kMaxF], wf[kMaxF];  // column of Q / D, element of W per term
  int64_t S, C;
  int64_t out_stride;
  // pre-pass scratch
  uint32_t* qp;   // [nq]
  uint32_t* dp;   // [nr]
  int* info;      // [0] fast-path flag, [1] packed weights, [2] S / 128,
                  // [3] weights * 16 as unsigned bytes, [4] five-instruction path flag
  int qt;         // queries per thread
  int allow5;     // five-instruction path permitted (MDHB_PRL_5=1)
  uint32_t one;   // 1 (keeps the byte-compare add an IMAD, see add7f_fma)
  int rsplit;     // record splits (grid.y)
  // max_prl (unpacked pair) mode
  int pair;                  // 1: fold (w, r) pairs with max_prl
  int lgS;                   // S = 2^lgS, C = S - 1 internally
  unsigned long long* pairs;  // [nq][2] (w, r), 16-byte aligned scratch
  void* out_r;                // record output (weight output is `best`)
  int64_t roff;               // global index of local record 0 (a DEV-layer shard's offset)
  int r_is64;
  int64_t r_stride;
};

__device__ __forceinline__ int64_t ld(const void* p, int is64, int64_t i) {
  return is64 ? static_cast<const int64_t*>(p)[i] : static_cast<int64_t>(static_cast<const int32_t*>(p)[i]);
}

// Grid pass 1: per-CTA min / max of every compared field value.
__global__ void __launch_bounds__(512) prl_range(PrlArgs a, long long* part) {
  __shared__ long long smin[16], smax[16];
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < a.nq * a.F; i += stride) {
    long long v = ld(a.Q, a.q_is64, (i / a.F) * a.qs + a.qf[i % a.F]);
    mn = min(mn, v);
    mx = max(mx, v);
  }
  for (int64_t i = i0; i < a.nr * a.F; i += stride) {
    long long v = ld(a.D, a.d_is64, (i / a.F) * a.ds + a.df[i % a.F]);
    mn = min(mn, v);
    mx = max(mx, v);
  }
  for (int s = 16; s > 0; s >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, s));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, s));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = mn;
    smax[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      mn = min(mn, smin[w]);
      mx = max(mx, smax[w]);
    }
    part[2 * blockIdx.x] = mn;
    part[2 * blockIdx.x + 1] = mx;
  }
}

// Grid pass 2: every CTA folds the partials itself (no extra launch), decides
// the fast path (value window <= 128, weights fit a signed byte, the 32-bit
// key cannot overflow), then re-encodes fields as 7-bit codes packed into
// bytes; unused byte slots hold 0 in both Q and D with weight 0.  Also seeds
// best[] with the identity of max.
__global__ void __launch_bounds__(512) prl_pack(PrlArgs a, const long long* part, int nparts) {
  __shared__ int s_fast;
  __shared__ long long s_base;
  if (threadIdx.x == 0) {
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    for (int b = 0; b < nparts; ++b) {
      mn = min(mn, part[2 * b]);
      mx = max(mx, part[2 * b + 1]);
    }
    bool ok = a.F <= kMaxF && mx >= mn && (mx - mn) <= 127 && a.S % 128 == 0 && a.S > 0 && a.S / 128 <= INT_MAX;
    long long wpos = 0, wneg = 0;
    uint32_t wp = 0;
    for (int t = 0; t < a.F; ++t) {
      long long w = ld(a.W, a.w_is64, a.wf[t]);
      ok = ok && w >= -128 && w <= 127;
      if (w > 0) wpos += w; else wneg += w;
      wp |= (static_cast<uint32_t>(static_cast<int8_t>(w)) & 0xFFu) << (8 * t);
    }
    if (ok) {  // the packed 32-bit key must hold wsum * S + (C - r) for every pair
      long long lo = wneg * a.S + (a.C - (a.nr - 1)), hi = wpos * a.S + a.C;
      ok = lo >= INT_MIN && hi <= INT_MAX;
    }
    // five-instruction variant: weights in [0, 15] scaled by 16 into unsigned
    // bytes, so DP4A yields 2^11 * wsum and its accumulator adds the
    // tile-local reversed record index: key_local = wsum * 2^11 + (2047 - k)
    bool ok5 = ok && a.S >= 2048 && a.allow5;
    uint32_t wp16 = 0;
    for (int t = 0; t < a.F; ++t) {
      long long w = ld(a.W, a.w_is64, a.wf[t]);
      ok5 = ok5 && w >= 0 && w <= 15;
      wp16 |= (static_cast<uint32_t>(w * 16) & 0xFFu) << (8 * t);
    }
    s_fast = ok ? 1 : 0;
    s_base = mn;
    if (blockIdx.x == 0) {
      a.info[0] = s_fast;
      a.info[1] = static_cast<int>(wp);
      a.info[2] = ok ? static_cast<int>(a.S / 128) : 0;
      a.info[3] = static_cast<int>(wp16);
      a.info[4] = ok5 ? 1 : 0;
    }
  }
  __syncthreads();
  const int fast = s_fast;
  const long long base = s_base;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q = i; q < a.nq; q += stride) {
    if (fast) {
      uint32_t w = 0;
      for (int t = 0; t < a.F; ++t)
        w |= static_cast<uint32_t>(ld(a.Q, a.q_is64, q * a.qs + a.qf[t]) - base) << (8 * t);
      a.qp[q] = w;
    }
    if (a.pair) {
      a.pairs[2 * q] = static_cast<unsigned long long>(LLONG_MIN);  // max_prl identity (-inf, +inf)
      a.pairs[2 * q + 1] = static_cast<unsigned long long>(LLONG_MAX);
    } else if (a.out_is64) {
      a.best[q * a.out_stride] = LLONG_MIN;
    } else {
      reinterpret_cast<int32_t*>(a.best)[q * a.out_stride] = INT_MIN;
    }
  }
  if (!fast) return;
  for (int64_t r = i; r < a.nr; r += stride) {
    uint32_t w = 0;
    for (int t = 0; t < a.F; ++t)
      w |= static_cast<uint32_t>(ld(a.D, a.d_is64, r * a.ds + a.df[t]) - base) << (8 * t);
    a.dp[r] = w;
  }
}

// (x & 0x7F7F7F7F) + 0x7F7F7F7F as an integer multiply-add: the add runs on
// the FMA pipe (IMAD) instead of the integer ALU pipe, which the byte
// compares (LOP3) and the fold (VIMNMX) already saturate.  `one` is a kernel
// argument equal to 1 so ptxas cannot fold the multiply back into an IADD3.
__device__ __forceinline__ uint32_t add7f_fma(uint32_t xm, uint32_t one) {
  uint32_t t;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(xm), "r"(one), "r"(0x7F7F7F7Fu));
  return t;
}

// max_prl commit: lexicographic max of (w, -r) by 128-bit compare-and-swap
__device__ __forceinline__ void commit_pair(unsigned long long* slot, long long w, long long r) {
  unsigned __int128* p = reinterpret_cast<unsigned __int128*>(slot);
  unsigned __int128 cur = *reinterpret_cast<volatile unsigned __int128*>(p);
  for (;;) {
    const long long cw = static_cast<long long>(static_cast<unsigned long long>(cur));
    const long long cr = static_cast<long long>(static_cast<unsigned long long>(cur >> 64));
    if (!(w > cw || (w == cw && r < cr))) return;
    const unsigned __int128 nv = (static_cast<unsigned __int128>(static_cast<unsigned long long>(r)) << 64) |
                                 static_cast<unsigned long long>(w);
    const unsigned __int128 prev = atomicCAS(p, cur, nv);
    if (prev == cur) return;
    cur = prev;
  }
}

// max_prl: unpack each thread's packed best key (fast paths) and commit
template <int QT>
__device__ __forceinline__ void commit_pairs_packed(const PrlArgs& a, int64_t q0, const long long (&best)[QT]) {
  const long long S = 1LL << a.lgS;
#pragma unroll
  for (int j = 0; j < QT; ++j) {
    int64_t q = q0 + static_cast<int64_t>(j) * NT;
    if (q >= a.nq) continue;
    const long long w = best[j] >> a.lgS;  // floor: the low part is in [0, S)
    const long long r = (S - 1) - (best[j] & (S - 1));
    commit_pair(a.pairs + 2 * q, w, r);
  }
}

template <int QT>
__device__ __forceinline__ void commit_best(const PrlArgs& a, int64_t q0, const long long (&best)[QT]) {
#pragma unroll
  for (int j = 0; j < QT; ++j) {
    int64_t q = q0 + static_cast<int64_t>(j) * NT;
    if (q >= a.nq) continue;
    if (a.out_is64) {
      atomicMax(reinterpret_cast<long long*>(a.best) + q * a.out_stride, best[j]);
    } else {
      atomicMax(reinterpret_cast<int*>(a.best) + q * a.out_stride, static_cast<int>(best[j]));
    }
  }
}

// grid.x: query tiles of NT*QT queries (thread t owns q0 + j*NT), grid.y:
// record splits.  Records stream through shared memory in tiles.
template <int QT>
__global__ void __launch_bounds__(NT) prl_main(PrlArgs a) {
  constexpr int RT = 2048;  // records per shared-memory tile
  __shared__ uint2 tile[RT];
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * NT * QT + threadIdx.x;
  const int64_t per = (a.nr + a.rsplit - 1) / a.rsplit;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.y) * per;
  const int64_t r_end = min(a.nr, r_begin + per);
  if (r_end <= r_begin) return;  // empty record split: nothing to fold
  long long best64[QT];
  if (a.info[4]) {
    // ---- five instructions per pair: LOP3 (xor & mask) + IADD + LOP3 (byte
    // equality) + DP4A (2^11 * weighted count + reversed tile index) + IMNMX.
    // The tile's best local key converts to the global key once per tile.
    const uint32_t wp16 = static_cast<uint32_t>(a.info[3]);
    uint32_t qp[QT];
    int best[QT];
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      int64_t q = q0 + static_cast<int64_t>(j) * NT;
      qp[j] = q < a.nq ? a.qp[q] : 0u;
      best[j] = INT_MIN;
    }
    uint32_t* tile1 = reinterpret_cast<uint32_t*>(tile);
    for (int64_t rt = r_begin; rt < r_end; rt += RT) {
      const int n = static_cast<int>(r_end - rt < RT ? r_end - rt : RT);
      __syncthreads();
      for (int k = threadIdx.x; k < n; k += NT) tile1[k] = a.dp[rt + k];
      __syncthreads();
      int loc[QT];
#pragma unroll
      for (int j = 0; j < QT; ++j) loc[j] = -1;
#pragma unroll 4
      for (int k = 0; k < n; ++k) {
        const uint32_t rec = tile1[k];
        const uint32_t krev = static_cast<uint32_t>(RT - 1 - k);
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          const uint32_t x = qp[j] ^ rec;
          const uint32_t t = add7f_fma(x & 0x7F7F7F7Fu, a.one);
          const uint32_t eq = ~t & 0x80808080u;
          int key;
          asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(key) : "r"(eq), "r"(wp16), "r"(krev));
          loc[j] = max(loc[j], key);
        }
      }
#pragma unroll
      for (int j = 0; j < QT; ++j) {
        const int wsum = loc[j] >> 11;
        const int64_t r = rt + (RT - 1 - (loc[j] & (RT - 1)));
        const int g = static_cast<int>(static_cast<int64_t>(wsum) * a.S + (a.C - r));  // fits: host/pack checked
        best[j] = max(best[j], g);
      }
    }
#pragma unroll
    for (int j = 0; j < QT; ++j) best64[j] = best[j];
  } else if (a.info[0]) {
    // ---- packed fast path (32-bit keys, exact while info[0] holds)
    const uint32_t wp = static_cast<uint32_t>(a.info[1]);
    const int sdiv = a.info[2];
    uint32_t qp[QT];
    int best[QT];
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      int64_t q = q0 + static_cast<int64_t>(j) * NT;
      qp[j] = q < a.nq ? a.qp[q] : 0u;
      best[j] = INT_MIN;
    }
    for (int64_t rt = r_begin; rt < r_end; rt += RT) {
      const int n = static_cast<int>(r_end - rt < RT ? r_end - rt : RT);
      __syncthreads();
      for (int k = threadIdx.x; k < n; k += NT)
        tile[k] = make_uint2(a.dp[rt + k], static_cast<uint32_t>(static_cast<int>(a.C - (rt + k))));
      __syncthreads();
#pragma unroll 4
      for (int k = 0; k < n; ++k) {
        const uint2 rec = tile[k];
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          const uint32_t x = qp[j] ^ rec.x;
          const uint32_t t = add7f_fma(x & 0x7F7F7F7Fu, a.one);  // bit 7 set per non-zero byte
          const uint32_t eq = ~t & 0x80808080u;                // codes < 128: x's bit 7 is 0
          int dot;
          asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(dot) : "r"(eq), "r"(wp), "r"(0));
          const int key = dot * sdiv + static_cast<int>(rec.y);  // = wsum * S + (C - r)
          best[j] = max(best[j], key);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < QT; ++j) best64[j] = best[j];
  } else if (a.pair) {
    // ---- exact max_prl path: (w, r) pairs folded without packing
    long long bw[QT], br[QT];
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      bw[j] = LLONG_MIN;
      br[j] = LLONG_MAX;
    }
    for (int64_t r = r_begin; r < r_end; ++r) {
#pragma unroll
      for (int j = 0; j < QT; ++j) {
        int64_t q = q0 + static_cast<int64_t>(j) * NT;
        if (q >= a.nq) continue;
        long long w = 0;
        for (int t = 0; t < a.F; ++t) {
          long long x = ld(a.Q, a.q_is64, q * a.qs + a.qf[t]);
          long long y = ld(a.D, a.d_is64, r * a.ds + a.df[t]);
          w += x == y ? ld(a.W, a.w_is64, a.wf[t]) : 0;
        }
        if (w > bw[j] || r == r_begin) {  // ascending r: ties keep the lower record
          bw[j] = w;
          br[j] = r;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      int64_t q = q0 + static_cast<int64_t>(j) * NT;
      if (q < a.nq) commit_pair(a.pairs + 2 * q, bw[j], br[j]);
    }
    return;
  } else {
    // ---- exact 64-bit path: the scalar function as written, per pair
#pragma unroll
    for (int j = 0; j < QT; ++j) best64[j] = LLONG_MIN;
    for (int64_t r = r_begin; r < r_end; ++r) {
#pragma unroll
      for (int j = 0; j < QT; ++j) {
        int64_t q = q0 + static_cast<int64_t>(j) * NT;
        if (q >= a.nq) continue;
        long long w = 0;
        for (int t = 0; t < a.F; ++t) {
          long long x = ld(a.Q, a.q_is64, q * a.qs + a.qf[t]);
          long long y = ld(a.D, a.d_is64, r * a.ds + a.df[t]);
          w += x == y ? ld(a.W, a.w_is64, a.wf[t]) : 0;
        }
        long long key = static_cast<long long>(static_cast<unsigned long long>(w) * static_cast<unsigned long long>(a.S) +
                                               static_cast<unsigned long long>(a.C - r));
        best64[j] = max(best64[j], key);
      }
    }
  }
  if (a.pair) commit_pairs_packed<QT>(a, q0, best64);
  else commit_best<QT>(a, q0, best64);
}

// max_prl: the folded pairs -> the two output buffers (storage i64 or i32)
__global__ void prl_unpack(PrlArgs a) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= a.nq) return;
  const long long w = static_cast<long long>(a.pairs[2 * q]), r = static_cast<long long>(a.pairs[2 * q + 1]) + a.roff;
  if (a.out_is64) a.best[q * a.out_stride] = w;
  else reinterpret_cast<int32_t*>(a.best)[q * a.out_stride] = static_cast<int32_t>(w);
  if (a.r_is64) static_cast<int64_t*>(a.out_r)[q * a.r_stride] = r;
  else static_cast<int32_t*>(a.out_r)[q * a.r_stride] = static_cast<int32_t>(r);
}

// ---------------------------------------------------------------- host
struct Term {
  int qb, qa, db, da, wb, wa;  // (buffer, access), 1-based
};

bool collect_terms(const Expr& e, std::vector<Term>& out) {
  if (e.k == EK::Add) return collect_terms(e.args[0], out) && collect_terms(e.args[1], out);
  if (e.k != EK::Select) return false;
  const Expr& c = e.args[0];
  if (c.k != EK::Cmp || c.args[0].k != EK::In || c.args[1].k != EK::In) return false;
  const Expr& z = e.args[1];
  if (z.k != EK::Lit || z.flit || z.iv != 0) return false;
  const Expr& w = e.args[2];
  if (w.k != EK::In) return false;
  out.push_back({c.args[0].buf, c.args[0].acc, c.args[1].buf, c.args[1].acc, w.buf, w.acc});
  return true;
}

class PrlRoutine final : public Routine {
 public:
  PrlRoutine(const Problem& p, PrlArgs a, int ib[3]) : p_(p), a_(a) {
    std::memcpy(ib_, ib, sizeof ib_);
    MDHB_CUDA(cudaSetDevice(p.opt.device));
    nparts_ = 2 * sm_count(p.opt.device);
    size_t head = 256 + static_cast<size_t>(nparts_) * 16;
    MDHB_CUDA(cudaMalloc(&scratch_, static_cast<size_t>(a.nq + a.nr) * 4 + head));
    a_.info = static_cast<int*>(scratch_);
    // the five-instruction path measured slower on B200 (8.24 vs 7.93 ms at
    // 2^15 x 2^20: IDP.4A.U8.U8 + VIMNMX per pair vs the six-instruction mix);
    // kept selectable (MDHB_PRL_5=1), bit-exact either way
    a_.allow5 = std::getenv("MDHB_PRL_5") ? 1 : 0;
    a_.one = 1;
    part_ = reinterpret_cast<long long*>(static_cast<char*>(scratch_) + 256);
    a_.qp = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch_) + head);
    a_.dp = a_.qp + a.nq;
    if (a_.pair) MDHB_CUDA(cudaMalloc(&pairs_, static_cast<size_t>(a.nq) * 16 + 16));
    a_.pairs = static_cast<unsigned long long*>(pairs_);
  }
  ~PrlRoutine() override {
    if (scratch_) cudaFree(scratch_);
    if (pairs_) cudaFree(pairs_);
  }
  const char* family() const override { return "prl"; }
  const char* bound() const override { return "int"; }
  int launches() const override { return a_.pair ? 4 : 3; }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  // integer work: F compares + F selects + F adds + key + fold per pair
  double flops() const override { return static_cast<double>(a_.nq) * static_cast<double>(a_.nr) * (3.0 * a_.F + 3.0); }
  double pairs() const { return static_cast<double>(a_.nq) * static_cast<double>(a_.nr); }
  std::string describe() const override {
    std::ostringstream os;
    os << "{\"kernel\": \"prl_main<" << a_.qt << ">\", \"queries\": " << a_.nq << ", \"records\": " << a_.nr
       << ", \"fields\": " << a_.F << ", \"queries_per_thread\": " << a_.qt << ", \"threads\": " << NT
       << ", \"record_splits\": " << a_.rsplit << ", \"record_tile\": 2048, \"pairs\": " << pairs()
       << ", \"combine\": \"" << (a_.pair ? "pw:max_prl (weight, record) pairs, 128-bit CAS" : "pw:max packed key, 64-bit atomicMax")
       << "\"}";
    return os.str();
  }
  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    PrlArgs a = a_;
    a.Q = d_in[ib_[0]];
    a.D = d_in[ib_[1]];
    a.W = d_in[ib_[2]];
    a.best = static_cast<int64_t*>(d_out[0]);
    if (a.pair) a.out_r = d_out[1];
    prl_range<<<nparts_, 512, 0, s>>>(a, part_);
    MDHB_CUDA(cudaGetLastError());
    prl_pack<<<nparts_, 512, 0, s>>>(a, part_, nparts_);
    MDHB_CUDA(cudaGetLastError());
    dim3 grid(static_cast<unsigned>((a.nq + NT * a.qt - 1) / (NT * a.qt)), static_cast<unsigned>(a.rsplit));
    mark_begin(s);
    switch (a.qt) {
      case 4: prl_main<4><<<grid, NT, 0, s>>>(a); break;
      case 16: prl_main<16><<<grid, NT, 0, s>>>(a); break;
      default: prl_main<8><<<grid, NT, 0, s>>>(a); break;
    }
    mark_end(s);
    MDHB_CUDA(cudaGetLastError());
    if (a.pair) {
      prl_unpack<<<static_cast<unsigned>((a.nq + 255) / 256), 256, 0, s>>>(a);
      MDHB_CUDA(cudaGetLastError());
    }
  }

 private:
  const Problem& p_;
  PrlArgs a_;
  void* pairs_ = nullptr;
  int ib_[3];
  int nparts_ = 0;
  long long* part_ = nullptr;
  void* scratch_ = nullptr;
};

// matches  <const> - idx(r)  and  <lit> * <sum>  / <sum> * <lit>
// idx(r) or idx(r) + lit / lit + idx(r) (a DEV-layer shard rebases idx(r) to
// the global record index): the dim and the constant offset
bool idx_plus(const Expr& e, int* dim, int64_t* off) {
  if (e.k == EK::Idx) {
    *dim = e.dim - 1;
    *off = 0;
    return true;
  }
  if (e.k != EK::Add) return false;
  for (int s = 0; s < 2; ++s) {
    const Expr& a = e.args[static_cast<size_t>(s)];
    const Expr& b = e.args[static_cast<size_t>(1 - s)];
    if (a.k == EK::Idx && b.k == EK::Lit && !b.flit) {
      *dim = a.dim - 1;
      *off = b.iv;
      return true;
    }
  }
  return false;
}

bool split_key(const Expr& e, const Expr** sum, int64_t* S, int64_t* C, int* rdim) {
  if (e.k != EK::Add) return false;
  for (int s = 0; s < 2; ++s) {
    const Expr& m = e.args[static_cast<size_t>(s)];
    const Expr& c = e.args[static_cast<size_t>(1 - s)];
    if (m.k != EK::Mul || c.k != EK::Sub) continue;
    int dim = -1;
    int64_t off = 0;
    if (c.args[0].k != EK::Lit || c.args[0].flit || !idx_plus(c.args[1], &dim, &off)) continue;
    for (int t = 0; t < 2; ++t) {
      const Expr& lit = m.args[static_cast<size_t>(t)];
      if (lit.k == EK::Lit && !lit.flit) {
        *sum = &m.args[static_cast<size_t>(1 - t)];
        *S = lit.iv;
        *C = c.args[0].iv - off;  // C - (r + off) = (C - off) - r
        *rdim = dim;
        return true;
      }
    }
  }
  return false;
}

}  // namespace

std::unique_ptr<Routine> make_prl(const Problem& p, const Config* cfg, Config* cfg_out) {
  const MdHom& e = p.e;
  if (e.D() != 2 || e.in.size() != 3) return nullptr;
  int rdim = -1;
  const Expr* sum = nullptr;
  int64_t S = 0, C = 0, roff = 0;
  bool pair = false;
  if (e.out.size() == 1 && e.out[0].acc.size() == 1 && e.assigns.size() == 1) {
    // packed form: best = weight * S + (C - idx(r)) folded with pw:max
    if (!split_key(e.assigns[0].e, &sum, &S, &C, &rdim)) return nullptr;
    if (e.comb[static_cast<size_t>(rdim)].kind != Combine::PW || e.comb[static_cast<size_t>(rdim)].op != Fold::Max)
      return nullptr;
  } else if (e.out.size() == 2 && e.out[0].acc.size() == 1 && e.out[1].acc.size() == 1 && e.assigns.size() == 2) {
    // unpacked form: (weight, idx(r)) folded with the custom pw:max_prl
    rdim = e.comb[0].kind == Combine::PW ? 0 : 1;
    const Combine& c = e.comb[static_cast<size_t>(rdim)];
    if (c.kind != Combine::PW || c.op != Fold::Custom || combine_at(c.custom).name != "max_prl") return nullptr;
    int idim = -1;
    if (!idx_plus(e.assigns[1].e, &idim, &roff) || idim != rdim || e.out[1].type != Ty::I64) return nullptr;
    sum = &e.assigns[0].e;
    int lg = 7;
    while ((int64_t(1) << lg) < e.sizes[static_cast<size_t>(rdim)]) ++lg;
    if (lg > 40) return nullptr;
    S = int64_t(1) << lg;
    C = S - 1;
    pair = true;
  } else {
    return nullptr;
  }
  const int qdim = 1 - rdim;
  if (e.comb[static_cast<size_t>(qdim)].kind != Combine::CC) return nullptr;
  std::vector<Term> terms;
  if (!collect_terms(*sum, terms) || terms.empty() || terms.size() > static_cast<size_t>(kMaxF)) return nullptr;
  for (auto& b : e.in)
    if (b.type != Ty::I64) return nullptr;
  if (e.out[0].type != Ty::I64) return nullptr;
  // roles: Q buffer reads (q, const), D reads (r, const), W reads (const)
  auto role = [&](int buf, int acc, int dim) -> int {  // column index, -1 if not of the form
    const Buf& b = e.in[static_cast<size_t>(buf - 1)];
    const Access& a = b.acc[static_cast<size_t>(acc - 1)];
    if (dim < 0) {
      if (b.rank != 1 || a.idx[0].coeff[0] != 0 || a.idx[0].coeff[1] != 0) return -1;
      return static_cast<int>(a.idx[0].c0);
    }
    if (b.rank != 2) return -1;
    const Affine &r0 = a.idx[0], &r1 = a.idx[1];
    if (r0.c0 != 0 || r0.coeff[static_cast<size_t>(dim)] != 1 || r0.coeff[static_cast<size_t>(1 - dim)] != 0) return -1;
    if (r1.coeff[0] != 0 || r1.coeff[1] != 0) return -1;
    return static_cast<int>(r1.c0);
  };
  PrlArgs a{};
  int ib[3] = {-1, -1, -1};
  a.F = static_cast<int>(terms.size());
  for (size_t t = 0; t < terms.size(); ++t) {
    Term tm = terms[t];
    // cmp is symmetric for the equality test: orient Q (reads q) first
    if (role(tm.qb, tm.qa, qdim) < 0) {
      std::swap(tm.qb, tm.db);
      std::swap(tm.qa, tm.da);
    }
    int qc = role(tm.qb, tm.qa, qdim), dc = role(tm.db, tm.da, rdim), wc = role(tm.wb, tm.wa, -1);
    if (qc < 0 || dc < 0 || wc < 0) return nullptr;
    int bufs[3] = {tm.qb - 1, tm.db - 1, tm.wb - 1};
    for (int k = 0; k < 3; ++k) {
      if (ib[k] >= 0 && ib[k] != bufs[k]) return nullptr;
      ib[k] = bufs[k];
    }
    a.qf[t] = qc;
    a.df[t] = dc;
    a.wf[t] = wc;
  }
  if (ib[0] == ib[1] || ib[0] == ib[2] || ib[1] == ib[2]) return nullptr;
  // output(s): best[q] (pair mode: weight[q], record[q])
  for (size_t b = 0; b < e.out.size(); ++b) {
    const Affine& o = e.out[b].acc[0].idx[0];
    if (e.out[b].rank != 1 || o.c0 != 0 || o.coeff[static_cast<size_t>(qdim)] != 1) return nullptr;
  }
  a.pair = pair ? 1 : 0;
  if (pair) {
    a.lgS = 0;
    while ((int64_t(1) << a.lgS) < S) ++a.lgS;
    a.r_is64 = p.out_store[1] == Store::I64;
    a.r_stride = 1;
    a.roff = roff;
  }
  a.nq = e.sizes[static_cast<size_t>(qdim)];
  a.nr = e.sizes[static_cast<size_t>(rdim)];
  a.qs = p.in_ext[static_cast<size_t>(ib[0])][1];
  a.ds = p.in_ext[static_cast<size_t>(ib[1])][1];
  a.q_is64 = p.in_store[static_cast<size_t>(ib[0])] == Store::I64;
  a.d_is64 = p.in_store[static_cast<size_t>(ib[1])] == Store::I64;
  a.w_is64 = p.in_store[static_cast<size_t>(ib[2])] == Store::I64;
  a.out_is64 = p.out_store[0] == Store::I64;
  a.S = S;
  a.C = C;
  a.out_stride = 1;
  a.qt = 8;
  a.rsplit = 64;
  if (a.nq * a.nr < (int64_t(1) << 22)) a.rsplit = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, a.nr / 256)));
  if (cfg) {
    auto P = parts_per_asm_layer(*cfg, e, p.m);
    int smx = p.m.id("SMX"), rm = p.m.id("RM");
    if (smx < 0 || rm < 0) fail("Unsupported", "prl template needs SMX and RM layers");
    int64_t qt = P[static_cast<size_t>(rm - 1)][static_cast<size_t>(qdim)];
    int64_t rs = P[static_cast<size_t>(smx - 1)][static_cast<size_t>(rdim)];
    if (qt != 4 && qt != 8 && qt != 16) fail("Unsupported", "prl template: RM parts of the query dim in {4, 8, 16}");
    a.qt = static_cast<int>(qt);
    a.rsplit = static_cast<int>(rs);
  }
  if (cfg_out) {
    int64_t qtile = NT * a.qt;
    if (a.nq % qtile == 0 && a.nr % a.rsplit == 0 && (a.nr / a.rsplit) % 2048 == 0 && p.m.id("WRP") > 0) {
      std::vector<int64_t> smx(2), dm(2), wrp(2, 1), cc(2, 1), sm(2, 1), rmv(2, 1);
      smx[static_cast<size_t>(qdim)] = a.nq / qtile;
      smx[static_cast<size_t>(rdim)] = a.rsplit;
      dm[static_cast<size_t>(qdim)] = 1;
      dm[static_cast<size_t>(rdim)] = a.nr / a.rsplit / 2048;
      wrp[static_cast<size_t>(qdim)] = NT / 32;
      cc[static_cast<size_t>(qdim)] = 32;
      sm[static_cast<size_t>(rdim)] = 2048;
      rmv[static_cast<size_t>(qdim)] = a.qt;
      *cfg_out = make_config(p, {{"SMX", smx}, {"DM", dm}, {"WRP", wrp}, {"CC", cc}, {"SM", sm}, {"RM", rmv}},
                             {{e.in[static_cast<size_t>(ib[1])].name, "SM"}, {e.in[static_cast<size_t>(ib[0])].name, "RM"}},
                             "RM");
    } else {
      *cfg_out = cfg ? *cfg : baseline_config(e, p.m);
    }
  }
  return std::make_unique<PrlRoutine>(p, a, ib);
}

}  // namespace mdhb

namespace mdhb {
// Tuning space of the PRL template: queries per thread (RM parts of q) x
// record splits (SMX parts of r, combined in DM by atomicMax).
std::vector<Config> prl_space(const Problem& p) {
  std::vector<Config> out;
  const MdHom& e = p.e;
  if (p.m.id("SMX") < 0 || p.m.id("WRP") < 0 || e.D() != 2) return out;
  int rdim = e.comb[0].kind == Combine::PW ? 0 : 1, qdim = 1 - rdim;
  int64_t nq = e.sizes[static_cast<size_t>(qdim)], nr = e.sizes[static_cast<size_t>(rdim)];
  for (int64_t qt : {4, 8, 16})
    for (int64_t rs : {16, 32, 64, 128, 256}) {
      int64_t qtile = 256 * qt;
      if (nq % qtile || nr % rs || (nr / rs) % 2048) continue;
      std::vector<int64_t> smx(2), dm(2, 1), wrp(2, 1), cc(2, 1), sm(2, 1), rm(2, 1);
      smx[static_cast<size_t>(qdim)] = nq / qtile;
      smx[static_cast<size_t>(rdim)] = rs;
      dm[static_cast<size_t>(rdim)] = nr / rs / 2048;
      wrp[static_cast<size_t>(qdim)] = 8;
      cc[static_cast<size_t>(qdim)] = 32;
      sm[static_cast<size_t>(rdim)] = 2048;
      rm[static_cast<size_t>(qdim)] = qt;
      out.push_back(make_config(p, {{"SMX", smx}, {"DM", dm}, {"WRP", wrp}, {"CC", cc}, {"SM", sm}, {"RM", rm}}, {}, "RM"));
    }
  return out;
}
}  // namespace mdhb
