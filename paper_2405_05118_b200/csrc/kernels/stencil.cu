// Stencil family: concatenation-only md_homs whose scalar function is a
// weighted sum of shifted reads of one rank-3 buffer (Jacobi3D,
// proj/data/computations/jacobi3d.json; BASELINE config 2).
//
//   w[i][j][k] = sum_t  wt_t * v[i + o_t0][j + o_t1][k + o_t2],   o_t in {0,1,2}^3
//
// Every dimension is `++`, so the re-composition is a disjoint, coalesced,
// vectorised store of each thread's cells (no reduction).  De-composition:
//   SMX  : the grid tiles (k: TK=128, j: TJ, i: TI planes per CTA)
//   DM   : each CTA streams its TI output planes sequentially (2.5D blocking)
//   SM   : a 4-slot ring of input planes (tile + 1-cell halo) in shared memory
//   WRP/CC: 8 warps x 32 lanes; lane -> 4 consecutive k, warp -> TJ/8 rows j
//   RM   : 4 (k) x 2 (j) outputs per thread; the centre rows of the last two
//          planes stay in registers as the CTA marches along i, so each
//          plane row is read from shared memory once per use class.
// Algorithmic traffic per run: every input cell read once + every output cell
// written once = 4 * (514^3 + 512^3) B for the BASELINE size.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "../plan.hpp"

namespace mdhb {
namespace {

constexpr int TK = 128;           // outputs along k per CTA
constexpr int NTHREADS = 256;
constexpr int PITCH = TK + 8;     // smem row pitch (floats): 16B-aligned rows, room for the halo

struct StencilArgs {
  const float* v;   // input base (already offset by nothing; halo offsets are in o_*)
  float* w;
  int64_t n0, n1, n2;     // output extents (i, j, k)
  int64_t e0, e1, e2;     // input extents (row-major strides from e1, e2)
  int ti;                 // output planes per CTA
  // weights of the 7-point star, in slot order: centre, i-1, i+1, j-1, j+1, k-1, k+1
  float wc, wim, wip, wjm, wjp, wkm, wkp;
  int pf;                 // star7_s32: L2 prefetch distance in planes (0 = off)
};

// Star-7 stencil with the centre at offset (1,1,1): reads v[i+1+di][j+1+dj][k+1+dk].
template <int TJ>
__global__ void __launch_bounds__(NTHREADS, 3) star7_kernel(StencilArgs a) {
  constexpr int ROWS = TJ + 2;
  constexpr int JPT = TJ / 8;  // j rows per thread (8 warps along j)
  static_assert(JPT == 2, "thread tile is 4 (k) x 2 (j)");
  __shared__ __align__(16) float ring[4][ROWS][PITCH];

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * TK;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * TJ;
  const int64_t i0 = static_cast<int64_t>(blockIdx.z) * a.ti;
  const int64_t plane = a.e1 * a.e2;
  const int kl = lane * 4;          // local k of this thread's first output
  const int jl = warp * JPT;        // local j of this thread's first output

  // cooperative plane loader: ROWS x (TK+2) cells, cell (r, c) = v[ip][j0+r][k0+c]
  constexpr int CELLS = ROWS * (TK + 2);
  constexpr int PER = (CELLS + NTHREADS - 1) / NTHREADS;
  float pre[PER];
  const int64_t kmax = a.e2 - k0;  // cells available in this row (tile edge)
  auto fetch = [&](int64_t ip) {
    const float* src = a.v + ip * plane + j0 * a.e2 + k0;
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      int cidx = tid + t * NTHREADS;
      int r = cidx / (TK + 2), c = cidx - r * (TK + 2);
      float x = 0.f;
      if (cidx < CELLS && c < kmax && j0 + r < a.e1 && ip < a.e0) x = __ldg(src + static_cast<int64_t>(r) * a.e2 + c);
      pre[t] = x;
    }
  };
  auto commit = [&](int slot) {
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      int cidx = tid + t * NTHREADS;
      if (cidx < CELLS) {
        int r = cidx / (TK + 2), c = cidx - r * (TK + 2);
        ring[slot][r][c] = pre[t];
      }
    }
  };
  // 6 consecutive floats of row r of a slot, starting at local column kl
  auto row6 = [&](int slot, int r, float (&x)[6]) {
    float4 q = *reinterpret_cast<const float4*>(&ring[slot][r][kl]);
    float2 h = *reinterpret_cast<const float2*>(&ring[slot][r][kl + 4]);
    x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w; x[4] = h.x; x[5] = h.y;
  };

  // prologue: input planes i0 .. i0+2 in slots 0..2, plane i0+3 in flight
  // (output plane i needs input planes i, i+1, i+2)
  fetch(i0);
  commit(0);
  fetch(i0 + 1);
  commit(1);
  fetch(i0 + 2);
  commit(2);
  fetch(i0 + 3);
  __syncthreads();
  // registers: centre rows (jl+1 .. jl+JPT) of the previous / current input plane
  float cprev[JPT][4], ccur[JPT][6];
#pragma unroll
  for (int jj = 0; jj < JPT; ++jj) {
    float x[6];
    row6(0, jl + 1 + jj, x);
#pragma unroll
    for (int c = 0; c < 4; ++c) cprev[jj][c] = x[c + 1];
    row6(1, jl + 1 + jj, ccur[jj]);
  }
  const int iend = static_cast<int>(a.n0 - i0 < a.ti ? a.n0 - i0 : a.ti);
  for (int t = 0; t < iend; ++t) {
    if (t > 0) __syncthreads();  // plane i0+t+2 (committed last iteration) is visible
    const int s_cur = (t + 1) & 3, s_nxt = (t + 2) & 3;
    float nxt[JPT][6], jm[6], jp[6];
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) row6(s_nxt, jl + 1 + jj, nxt[jj]);
    row6(s_cur, jl, jm);            // row j-1 of the first output row
    row6(s_cur, jl + JPT + 1, jp);  // row j+1 of the last output row
    const int64_t i = i0 + t;
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
      const float* up = jj == 0 ? jm : ccur[jj - 1];
      const float* dn = jj == JPT - 1 ? jp : ccur[jj + 1];
      float o[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float acc = a.wc * ccur[jj][kk + 1];
        acc = fmaf(a.wim, cprev[jj][kk], acc);
        acc = fmaf(a.wip, nxt[jj][kk + 1], acc);
        acc = fmaf(a.wjm, up[kk + 1], acc);
        acc = fmaf(a.wjp, dn[kk + 1], acc);
        acc = fmaf(a.wkm, ccur[jj][kk], acc);
        acc = fmaf(a.wkp, ccur[jj][kk + 2], acc);
        o[kk] = acc;
      }
      const int64_t j = j0 + jl + jj, k = k0 + kl;
      if (j < a.n1 && k < a.n2) {
        float* dst = a.w + (i * a.n1 + j) * a.n2 + k;
        if (k + 4 <= a.n2 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          __stcs(reinterpret_cast<float4*>(dst), make_float4(o[0], o[1], o[2], o[3]));
        } else {
          for (int kk = 0; kk < 4 && k + kk < a.n2; ++kk) dst[kk] = o[kk];
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
#pragma unroll
      for (int c = 0; c < 4; ++c) cprev[jj][c] = ccur[jj][c + 1];
#pragma unroll
      for (int c = 0; c < 6; ++c) ccur[jj][c] = nxt[jj][c];
    }
    // slot (t+3)&3 is not read in this iteration: park plane i0+t+3 there and
    // put plane i0+t+4 in flight; both are consumed a full iteration later
    commit((t + 3) & 3);
    fetch(i0 + t + 4);
  }
}


// ---------------------------------------------------------------------------
// v2: the same 2.5D scheme with the plane rows moved by the TMA engine
// (cp.async.bulk, one 16-byte-aligned bulk copy per row, completion tracked
// by an mbarrier per ring slot).  No load/store instructions are spent on
// staging, and NSLOT-2 planes stay in flight per CTA, which is what keeps
// enough bytes outstanding to run at copy bandwidth.  Rows whose global
// offset is not 16-byte aligned are copied from the aligned address below
// them; the per-row float shift (0 or 2 for the BASELINE extents) is
// re-applied when the row is read from shared memory.
#ifndef MDHB_STENCIL_NSLOT
#define MDHB_STENCIL_NSLOT 6
#endif
#ifndef MDHB_STENCIL_WS_MINB
#define MDHB_STENCIL_WS_MINB 3
#endif
constexpr int NSLOT = MDHB_STENCIL_NSLOT;  // ring slots
constexpr int PD = NSLOT - 1;            // planes in flight ahead of compute
constexpr int BPITCH = TK + 8;           // floats per smem row: 128 + halo 2 + shift <= 3, 16B rounded

__device__ __forceinline__ uint32_t s_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int TJ>
__global__ void __launch_bounds__(NTHREADS, 3) star7_bulk(StencilArgs a) {
  constexpr int ROWS = TJ + 2;
  constexpr int JPT = TJ / 8;
  extern __shared__ __align__(128) float sring[];  // [NSLOT][ROWS][BPITCH]
  __shared__ __align__(8) uint64_t full[NSLOT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * TK;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * TJ;
  const int64_t i0 = static_cast<int64_t>(blockIdx.z) * a.ti;
  const int kl = lane * 4, jl = warp * JPT;
  const int iend = static_cast<int>(a.n0 - i0 < a.ti ? a.n0 - i0 : a.ti);
  const int nplanes = iend + 2;  // input planes i0 .. i0+iend+1

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // row r of input plane p -> slot p % NSLOT (warp 0 issues, lane r copies row r)
  auto issue = [&](int p) {
    if (warp != 0 || p >= nplanes) return;
    const int s = p % NSLOT;
    const int64_t ip = i0 + p;
    if (lane == 0) {
      uint32_t bytes = 0;
      for (int r = 0; r < ROWS; ++r) {
        int64_t off = (ip * a.e1 + j0 + r) * a.e2 + k0;
        uint32_t sh = static_cast<uint32_t>(off & 3);
        bytes += (sh * 4 + (TK + 2) * 4 + 15) & ~15u;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[s])), "r"(bytes) : "memory");
    }
    __syncwarp();
    for (int r = lane; r < ROWS; r += 32) {
      int64_t off = (ip * a.e1 + j0 + r) * a.e2 + k0;
      uint32_t sh = static_cast<uint32_t>(off & 3);
      uint32_t bytes = (sh * 4 + (TK + 2) * 4 + 15) & ~15u;
      const float* src = a.v + (off - sh);
      float* dst = sring + (static_cast<size_t>(s) * ROWS + r) * BPITCH;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(&full[s])) : "memory");
    }
  };
  auto wait_plane = [&](int p) {
    const int s = p % NSLOT;
    const uint32_t parity = static_cast<uint32_t>((p / NSLOT) & 1);
    uint32_t done = 0;
    for (uint32_t spin = 0; !done; ++spin) {
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                   : "=r"(done) : "r"(s_u32(&full[s])), "r"(parity) : "memory");
      if (spin > (1u << 26)) __trap();
    }
  };
  // 6 floats of row r of plane p starting at local column c
  auto row6 = [&](int p, int r, int c, float (&x)[6]) {
    const int64_t off = ((i0 + p) * a.e1 + j0 + r) * a.e2 + k0;
    const int sh = static_cast<int>(off & 3);
    const float* row = sring + (static_cast<size_t>(p % NSLOT) * ROWS + r) * BPITCH + sh + c;
    if ((sh & 1) == 0) {
      float2 u = *reinterpret_cast<const float2*>(row), v = *reinterpret_cast<const float2*>(row + 2),
             w = *reinterpret_cast<const float2*>(row + 4);
      x[0] = u.x; x[1] = u.y; x[2] = v.x; x[3] = v.y; x[4] = w.x; x[5] = w.y;
    } else {
#pragma unroll
      for (int q = 0; q < 6; ++q) x[q] = row[q];
    }
  };

  for (int p = 0; p < PD && p < nplanes; ++p) issue(p);
  wait_plane(0);
  wait_plane(1);
  float cprev[JPT][4], ccur[JPT][6];
#pragma unroll
  for (int jj = 0; jj < JPT; ++jj) {
    float x[6];
    row6(0, jl + 1 + jj, kl, x);
#pragma unroll
    for (int c = 0; c < 4; ++c) cprev[jj][c] = x[c + 1];
    row6(1, jl + 1 + jj, kl, ccur[jj]);
  }
  for (int t = 0; t < iend; ++t) {
    wait_plane(t + 2);
    float nxt[JPT][6], jm[6], jp[6];
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) row6(t + 2, jl + 1 + jj, kl, nxt[jj]);
    row6(t + 1, jl, kl, jm);
    row6(t + 1, jl + JPT + 1, kl, jp);
    const int64_t i = i0 + t;
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
      const float* up = jj == 0 ? jm : ccur[jj - 1];
      const float* dn = jj == JPT - 1 ? jp : ccur[jj + 1];
      float o[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float acc = a.wc * ccur[jj][kk + 1];
        acc = fmaf(a.wim, cprev[jj][kk], acc);
        acc = fmaf(a.wip, nxt[jj][kk + 1], acc);
        acc = fmaf(a.wjm, up[kk + 1], acc);
        acc = fmaf(a.wjp, dn[kk + 1], acc);
        acc = fmaf(a.wkm, ccur[jj][kk], acc);
        acc = fmaf(a.wkp, ccur[jj][kk + 2], acc);
        o[kk] = acc;
      }
      const int64_t j = j0 + jl + jj, k = k0 + kl;
      if (j < a.n1 && k < a.n2) {
        float* dst = a.w + (i * a.n1 + j) * a.n2 + k;
        if (k + 4 <= a.n2 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          __stcs(reinterpret_cast<float4*>(dst), make_float4(o[0], o[1], o[2], o[3]));
        } else {
          for (int kk = 0; kk < 4 && k + kk < a.n2; ++kk) dst[kk] = o[kk];
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
#pragma unroll
      for (int c = 0; c < 4; ++c) cprev[jj][c] = ccur[jj][c + 1];
#pragma unroll
      for (int c = 0; c < 6; ++c) ccur[jj][c] = nxt[jj][c];
    }
    // every thread is done with plane t+1 (its last reader): the slot of plane
    // t + PD (== slot of plane t + PD - NSLOT <= t - 2) may be refilled
    __syncthreads();
    issue(t + PD);
  }
}


// ---------------------------------------------------------------------------
// v3 (default): warp-specialised.  Warp 8 is the producer: it streams input
// planes into the NSLOT ring with cp.async.bulk (one copy per row, tx-counted
// on full[slot]) as soon as the 8 compute warps release a slot (empty[slot],
// one arrival per warp).  Compute warps never meet a CTA-wide barrier; they
// rotate three register row-sets (previous / current / next plane) with a
// 3-way unrolled loop so no register copies are needed.
constexpr int WS_THREADS = 288;  // 8 compute warps + 1 producer warp

struct Rows {
  float r[2][6];  // the thread's centre rows (j = jl+1, jl+2), cols kl .. kl+5
};

__device__ __forceinline__ void ld6(const float* row, int sh, float (&x)[6]) {
  if ((sh & 1) == 0) {
    float2 u = *reinterpret_cast<const float2*>(row), v = *reinterpret_cast<const float2*>(row + 2),
           w = *reinterpret_cast<const float2*>(row + 4);
    x[0] = u.x; x[1] = u.y; x[2] = v.x; x[3] = v.y; x[4] = w.x; x[5] = w.y;
  } else {
#pragma unroll
    for (int q = 0; q < 6; ++q) x[q] = row[q];
  }
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0; !done; ++spin) {
    asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(done) : "r"(s_u32(bar)), "r"(parity) : "memory");
    if (spin > (1u << 26)) __trap();
  }
}

__global__ void __launch_bounds__(WS_THREADS, MDHB_STENCIL_WS_MINB) star7_ws(StencilArgs a) {
  constexpr int TJ = 16, ROWS = TJ + 2;
  extern __shared__ __align__(128) float sring[];  // [NSLOT][ROWS][BPITCH]
  __shared__ __align__(8) uint64_t full[NSLOT], empty[NSLOT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * TK;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * TJ;
  const int64_t i0 = static_cast<int64_t>(blockIdx.z) * a.ti;
  const int iend = static_cast<int>(a.n0 - i0 < a.ti ? a.n0 - i0 : a.ti);
  const int nplanes = iend + 2;
  // low two bits of flat offsets decide each row's 16-byte shift
  const uint32_t pstride = static_cast<uint32_t>(a.e1 * a.e2);
  const uint32_t base0 = static_cast<uint32_t>((i0 * a.e1 + j0) * a.e2 + k0);
  const uint32_t rstride = static_cast<uint32_t>(a.e2);

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(s_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 8) {
    // ---------------- producer
    const float* vbase = a.v + ((i0 * a.e1 + j0) * a.e2 + k0);
    for (int p = 0; p < nplanes; ++p) {
      const int s = p % NSLOT;
      if (p >= NSLOT) mbar_wait_parity(&empty[s], static_cast<uint32_t>((p / NSLOT - 1) & 1));
      uint32_t bytes = 0, sh = 0;
      if (lane < ROWS) {
        sh = (base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(lane) * rstride) & 3u;
        bytes = (sh * 4 + (TK + 2) * 4 + 15) & ~15u;
      }
      uint32_t total = bytes;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[s])), "r"(total) : "memory");
      __syncwarp();
      if (lane < ROWS && i0 + p < a.e0) {
        const float* src = vbase + static_cast<int64_t>(p) * (a.e1 * a.e2) + static_cast<int64_t>(lane) * a.e2 - sh;
        float* dst = sring + (static_cast<size_t>(s) * ROWS + lane) * BPITCH;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(&full[s])) : "memory");
      }
    }
    return;
  }

  // ---------------- 8 compute warps: 4 (k) x 2 (j) outputs per thread
  const int kl = lane * 4, jl = warp * 2;
  auto rowptr = [&](int p, int r, int& sh) {
    sh = static_cast<int>((base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(r) * rstride) & 3u);
    return sring + (static_cast<size_t>(p % NSLOT) * ROWS + r) * BPITCH + sh + kl;
  };
  auto load_centre = [&](int p, Rows& R) {
    int sh;
    const float* q0 = rowptr(p, jl + 1, sh);
    ld6(q0, sh, R.r[0]);
    const float* q1 = rowptr(p, jl + 2, sh);
    ld6(q1, sh, R.r[1]);
  };
  auto release = [&](int p) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(&empty[p % NSLOT])) : "memory");
  };
  float* wout = a.w + (i0 * a.n1 + j0 + jl) * a.n2 + k0 + kl;
  const int64_t wplane = a.n1 * a.n2;
  const bool kin = k0 + kl + 4 <= a.n2;

  auto step = [&](int t, const Rows& P, const Rows& C, Rows& N) {
    mbar_wait_parity(&full[(t + 2) % NSLOT], static_cast<uint32_t>(((t + 2) / NSLOT) & 1));
    load_centre(t + 2, N);
    float jm[6], jp[6];
    int sh;
    const float* qm = rowptr(t + 1, jl, sh);
    ld6(qm, sh, jm);
    const float* qp = rowptr(t + 1, jl + 3, sh);
    ld6(qp, sh, jp);
    release(t + 1);  // plane t+1 has no readers after this step
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const float* up = jj == 0 ? jm : C.r[0];
      const float* dn = jj == 1 ? jp : C.r[1];
      float o[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float acc = a.wc * C.r[jj][kk + 1];
        acc = fmaf(a.wim, P.r[jj][kk + 1], acc);
        acc = fmaf(a.wip, N.r[jj][kk + 1], acc);
        acc = fmaf(a.wjm, up[kk + 1], acc);
        acc = fmaf(a.wjp, dn[kk + 1], acc);
        acc = fmaf(a.wkm, C.r[jj][kk], acc);
        acc = fmaf(a.wkp, C.r[jj][kk + 2], acc);
        o[kk] = acc;
      }
      const int64_t j = j0 + jl + jj;
      if (j < a.n1 && kin) {
        __stcs(reinterpret_cast<float4*>(wout + t * wplane + jj * a.n2), make_float4(o[0], o[1], o[2], o[3]));
      } else if (j < a.n1) {
        for (int kk = 0; kk < 4 && k0 + kl + kk < a.n2; ++kk) wout[t * wplane + jj * a.n2 + kk] = o[kk];
      }
    }
  };

  Rows R0, R1, R2;
  mbar_wait_parity(&full[0], 0);
  mbar_wait_parity(&full[1], 0);
  load_centre(0, R0);
  load_centre(1, R1);
  release(0);
  int t = 0;
  for (; t + 3 <= iend; t += 3) {
    step(t, R0, R1, R2);
    step(t + 1, R1, R2, R0);
    step(t + 2, R2, R0, R1);
  }
  if (t < iend) step(t, R0, R1, R2), ++t;
  if (t < iend) step(t, R1, R2, R0), ++t;
}


// ---------------------------------------------------------------------------
// v3b (lean registers): star7_ws with only the 4 centre columns of each
// plane's two rows kept in registers across steps; the centre plane's k-1 /
// k+4 halo values are re-read from shared memory in the step that uses them
// (the plane is still resident until that step releases it).  24 instead of
// 36 carried floats -> <= 56 registers -> 4 CTAs per SM, i.e. one more
// producer warp and ring per SM keeping HBM reads in flight.
struct Rows4 {
  float r[2][4];
};
__device__ __forceinline__ void ld4c(const float* row, int sh, float (&x)[4]) {
  // columns 1..4 of the 6-wide window at `row` (sh even: float2-aligned at row)
  if ((sh & 1) == 0) {
    float2 u = *reinterpret_cast<const float2*>(row), v = *reinterpret_cast<const float2*>(row + 2),
           w = *reinterpret_cast<const float2*>(row + 4);
    x[0] = u.y; x[1] = v.x; x[2] = v.y; x[3] = w.x;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = row[q + 1];
  }
}

// TS variant: every warp stages its two output rows of the plane in shared
// memory and its lane 0 writes them with two 512-byte bulk copies
// (cp.async.bulk.global.shared::cta), double-buffered per warp -- the store
// traffic leaves the LSU / L1 path for the TMA engine.  Full tiles only.
template <int NS, int MINB, bool TS>
__global__ void __launch_bounds__(WS_THREADS, MINB) star7_lean(StencilArgs a) {
  constexpr int TJ = 16, ROWS = TJ + 2;
  extern __shared__ __align__(128) float sring[];  // [NS][ROWS][BPITCH] (+ TS: [8 warps][2 bufs][2 rows][TK])
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * TK;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * TJ;
  const int64_t i0 = static_cast<int64_t>(blockIdx.z) * a.ti;
  const int iend = static_cast<int>(a.n0 - i0 < a.ti ? a.n0 - i0 : a.ti);
  const int nplanes = iend + 2;
  const uint32_t pstride = static_cast<uint32_t>(a.e1 * a.e2);
  const uint32_t base0 = static_cast<uint32_t>((i0 * a.e1 + j0) * a.e2 + k0);
  const uint32_t rstride = static_cast<uint32_t>(a.e2);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(s_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 8) {
    const float* vbase = a.v + ((i0 * a.e1 + j0) * a.e2 + k0);
    for (int p = 0; p < nplanes; ++p) {
      const int s = p % NS;
      if (p >= NS) mbar_wait_parity(&empty[s], static_cast<uint32_t>((p / NS - 1) & 1));
      uint32_t bytes = 0, sh = 0;
      if (lane < ROWS) {
        sh = (base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(lane) * rstride) & 3u;
        bytes = (sh * 4 + (TK + 2) * 4 + 15) & ~15u;
      }
      uint32_t total = bytes;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[s])), "r"(total) : "memory");
      __syncwarp();
      if (lane < ROWS && i0 + p < a.e0) {
        const float* src = vbase + static_cast<int64_t>(p) * (a.e1 * a.e2) + static_cast<int64_t>(lane) * a.e2 - sh;
        float* dst = sring + (static_cast<size_t>(s) * ROWS + lane) * BPITCH;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(&full[s])) : "memory");
      }
    }
    return;
  }

  const int kl = lane * 4, jl = warp * 2;
  auto rowptr = [&](int p, int r, int& sh) {
    sh = static_cast<int>((base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(r) * rstride) & 3u);
    return sring + (static_cast<size_t>(p % NS) * ROWS + r) * BPITCH + sh + kl;
  };
  auto load_centre = [&](int p, Rows4& R) {
    int sh;
    const float* q0 = rowptr(p, jl + 1, sh);
    ld4c(q0, sh, R.r[0]);
    const float* q1 = rowptr(p, jl + 2, sh);
    ld4c(q1, sh, R.r[1]);
  };
  auto release = [&](int p) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(&empty[p % NS])) : "memory");
  };
  float* wout = a.w + (i0 * a.n1 + j0 + jl) * a.n2 + k0 + kl;
  const int64_t wplane = a.n1 * a.n2;
  const bool kin = k0 + kl + 4 <= a.n2;

  // TS: this warp's output staging, 2 buffers x 2 rows x TK floats
  float* sout = sring + static_cast<size_t>(NS) * ROWS * BPITCH + static_cast<size_t>(warp) * 4 * TK;
  auto step = [&](int t, const Rows4& P, const Rows4& C, Rows4& N) {
    if (TS) {
      // the bulk store issued two steps ago from this buffer must have read it
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
    }
    mbar_wait_parity(&full[(t + 2) % NS], static_cast<uint32_t>(((t + 2) / NS) & 1));
    load_centre(t + 2, N);
    float jm[4], jp[4], hl[2], hr[2];
    int sh;
    ld4c(rowptr(t + 1, jl, sh), sh, jm);
    ld4c(rowptr(t + 1, jl + 3, sh), sh, jp);
    {
      const float* c0 = rowptr(t + 1, jl + 1, sh);
      hl[0] = c0[0];
      hr[0] = c0[5];
      const float* c1 = rowptr(t + 1, jl + 2, sh);
      hl[1] = c1[0];
      hr[1] = c1[5];
    }
    release(t + 1);
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const float* up = jj == 0 ? jm : C.r[0];
      const float* dn = jj == 1 ? jp : C.r[1];
      float o[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float km = kk == 0 ? hl[jj] : C.r[jj][kk - 1];
        const float kp = kk == 3 ? hr[jj] : C.r[jj][kk + 1];
        float acc = a.wc * C.r[jj][kk];
        acc = fmaf(a.wim, P.r[jj][kk], acc);
        acc = fmaf(a.wip, N.r[jj][kk], acc);
        acc = fmaf(a.wjm, up[kk], acc);
        acc = fmaf(a.wjp, dn[kk], acc);
        acc = fmaf(a.wkm, km, acc);
        acc = fmaf(a.wkp, kp, acc);
        o[kk] = acc;
      }
      const int64_t j = j0 + jl + jj;
      if (TS) {
        *reinterpret_cast<float4*>(sout + ((t & 1) * 2 + jj) * TK + kl) = make_float4(o[0], o[1], o[2], o[3]);
      } else if (j < a.n1 && kin) {
        __stcs(reinterpret_cast<float4*>(wout + t * wplane + jj * a.n2), make_float4(o[0], o[1], o[2], o[3]));
      } else if (j < a.n1) {
        for (int kk = 0; kk < 4 && k0 + kl + kk < a.n2; ++kk) wout[t * wplane + jj * a.n2 + kk] = o[kk];
      }
    }
    if (TS) {
      // generic-proxy writes -> async proxy, then lane 0 ships both rows
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       ::"l"(wout - kl + t * wplane + jj * a.n2), "r"(s_u32(sout + ((t & 1) * 2 + jj) * TK)),
                       "r"(static_cast<uint32_t>(TK * 4)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  };

  Rows4 R0, R1, R2;
  mbar_wait_parity(&full[0], 0);
  mbar_wait_parity(&full[1], 0);
  load_centre(0, R0);
  load_centre(1, R1);
  release(0);
  int t = 0;
  for (; t + 3 <= iend; t += 3) {
    step(t, R0, R1, R2);
    step(t + 1, R1, R2, R0);
    step(t + 2, R2, R0, R1);
  }
  if (t < iend) step(t, R0, R1, R2), ++t;
  if (t < iend) step(t, R1, R2, R0), ++t;
  if (TS && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// v5 (strided lanes, conflict-free): the lean kernel is bound by shared
// memory wavefronts (ncu: l1tex 90%, mio_throttle) because each lane owns 4
// consecutive k -- its windows are 8-byte reads at a 16-byte lane stride,
// 4-way bank conflicts.  Here lane l owns columns l, l+32, l+64, l+96 of the
// tile: every read of a row is one 4-byte word per lane at consecutive
// addresses (one wavefront per 32 values, whatever the row's alignment
// shift), the k-halos are plain reads one word left / right, and each store
// instruction writes 128 contiguous bytes.  Same ring, producer and
// register rotation along i as star7_lean.
struct Rows8 {
  float r[2][4];
};

// TKC = k columns per CTA tile (128, 256 or 512): wider tiles read longer
// contiguous row segments (528 / 1040 / 2064 bytes) at the price of more
// j-halo rows per output (TJ = 2048 / TKC rows: 16 / 8 / 4).  Each warp owns
// RW rows x CW columns, lane l the columns l + 32 m of them (M = CW / 32).
template <int TKC>
__host__ __device__ constexpr int CWDIV() { return (TKC * (2048 / TKC)) / 8; }

template <int TKC>
struct S32Shape {
  static constexpr int TJ = 2048 / TKC;                 // rows per CTA
  static constexpr int RW = TJ >= 8 ? TJ / 8 : 1;       // rows per warp
  static constexpr int CW = TJ >= 8 ? TKC : TKC * TJ / 8;  // columns per warp
  static constexpr int M = CW / 32;                     // columns per lane
  static constexpr int PITCH = TKC + 8;                 // smem row pitch (floats)
  static_assert(RW * M == 8, "8 output values per thread per plane");
};

template <int NS, int MINB, int TKC = 128>
__global__ void __launch_bounds__(WS_THREADS, MINB) star7_s32(StencilArgs a) {
  using SH = S32Shape<TKC>;
  constexpr int TJ = SH::TJ, ROWS = TJ + 2, RW = SH::RW, M = SH::M, PITCH = SH::PITCH;
  extern __shared__ __align__(128) float sring[];  // [NS][ROWS][PITCH]
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * TKC;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * TJ;
  const int64_t i0 = static_cast<int64_t>(blockIdx.z) * a.ti;
  const int iend = static_cast<int>(a.n0 - i0 < a.ti ? a.n0 - i0 : a.ti);
  const int nplanes = iend + 2;
  const uint32_t pstride = static_cast<uint32_t>(a.e1 * a.e2);
  const uint32_t base0 = static_cast<uint32_t>((i0 * a.e1 + j0) * a.e2 + k0);
  const uint32_t rstride = static_cast<uint32_t>(a.e2);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(s_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 8) {
    const float* vbase = a.v + ((i0 * a.e1 + j0) * a.e2 + k0);
    for (int p = 0; p < nplanes; ++p) {
      const int s = p % NS;
      if (p >= NS) mbar_wait_parity(&empty[s], static_cast<uint32_t>((p / NS - 1) & 1));
      uint32_t bytes = 0, sh = 0;
      if (lane < ROWS) {
        sh = (base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(lane) * rstride) & 3u;
        bytes = (sh * 4 + (TKC + 2) * 4 + 15) & ~15u;
      }
      uint32_t total = bytes;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[s])), "r"(total) : "memory");
      __syncwarp();
      if (lane < ROWS && i0 + p < a.e0) {
        const float* src = vbase + static_cast<int64_t>(p) * (a.e1 * a.e2) + static_cast<int64_t>(lane) * a.e2 - sh;
        float* dst = sring + (static_cast<size_t>(s) * ROWS + lane) * PITCH;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(&full[s])) : "memory");
      }
    }
    return;
  }

  // this warp's rows and columns
  const int jl = TJ >= 8 ? warp * RW : (warp * CWDIV<TKC>()) / TKC;
  const int cl = TJ >= 8 ? 0 : (warp * CWDIV<TKC>()) % TKC;
  const uint32_t ring0 = s_u32(sring) + static_cast<uint32_t>(cl + lane) * 4u;
  auto rowaddr = [&](int p, int r) {
    const uint32_t sh = (base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(r) * rstride) & 3u;
    return ring0 + (static_cast<uint32_t>(((p % NS) * ROWS + r) * PITCH) + sh) * 4u;
  };
  auto ld1 = [](uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
  };
  auto load_row = [&](uint32_t ra, float (&x)[M]) {  // centres of columns lane + 32 m
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = ld1(ra + static_cast<uint32_t>(32 * m + 1) * 4u);
  };
  struct RowsW {
    float r[RW][M];
  };
  auto load_centre = [&](int p, RowsW& R) {
#pragma unroll
    for (int q = 0; q < RW; ++q) load_row(rowaddr(p, jl + 1 + q), R.r[q]);
  };
  auto release = [&](int p) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(&empty[p % NS])) : "memory");
  };
  float* wout = a.w + (i0 * a.n1 + j0 + jl) * a.n2 + k0 + cl + lane;
  const int64_t wplane = a.n1 * a.n2;

  auto step = [&](int t, const RowsW& P, const RowsW& C, RowsW& N) {
    mbar_wait_parity(&full[(t + 2) % NS], static_cast<uint32_t>(((t + 2) / NS) & 1));
    load_centre(t + 2, N);
    // plane t + 1 stays resident until every read below is done: the j /
    // k neighbours are read just in time (few live registers)
#pragma unroll
    for (int jj = 0; jj < RW; ++jj) {
      float up[M], dn[M];
      if (jj == 0) load_row(rowaddr(t + 1, jl), up);
      else
#pragma unroll
        for (int m = 0; m < M; ++m) up[m] = C.r[jj - 1][m];
      if (jj == RW - 1) load_row(rowaddr(t + 1, jl + RW + 1), dn);
      else
#pragma unroll
        for (int m = 0; m < M; ++m) dn[m] = C.r[jj + 1][m];
      const uint32_t ra = rowaddr(t + 1, jl + 1 + jj);
      const int64_t j = j0 + jl + jj;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        float acc = a.wc * C.r[jj][m];
        acc = fmaf(a.wim, P.r[jj][m], acc);
        acc = fmaf(a.wip, N.r[jj][m], acc);
        acc = fmaf(a.wjm, up[m], acc);
        acc = fmaf(a.wjp, dn[m], acc);
        acc = fmaf(a.wkm, ld1(ra + static_cast<uint32_t>(32 * m) * 4u), acc);
        acc = fmaf(a.wkp, ld1(ra + static_cast<uint32_t>(32 * m + 2) * 4u), acc);
        if (j < a.n1 && k0 + cl + lane + 32 * m < a.n2) __stcs(wout + t * wplane + jj * a.n2 + 32 * m, acc);
      }
    }
    release(t + 1);
  };

  RowsW R0, R1, R2;
  mbar_wait_parity(&full[0], 0);
  mbar_wait_parity(&full[1], 0);
  load_centre(0, R0);
  load_centre(1, R1);
  release(0);
  int t = 0;
  for (; t + 3 <= iend; t += 3) {
    step(t, R0, R1, R2);
    step(t + 1, R1, R2, R0);
    step(t + 2, R2, R0, R1);
  }
  if (t < iend) step(t, R0, R1, R2), ++t;
  if (t < iend) step(t, R1, R2, R0), ++t;
}

// ---------------------------------------------------------------------------
// v4 (default): persistent + warp-specialised.  The (tile, i-plane) step
// space (n2/TK * n1/TJ tiles x n0 planes) is cut into `gridDim.x` contiguous
// equal ranges, one per resident CTA, so every SM streams the same number of
// planes (no wave tail) and consecutive segments of a CTA reuse the ring: a
// global plane sequence number q drives slot = q % NSLOT and mbarrier parity.
// Work units: mode 0 = one contiguous range of (tile, plane) steps per CTA;
// mode 1 = grid-stride over (tile, TI-plane chunk) items in launch-grid order,
// so concurrently running CTAs hold neighbouring tiles (halo rows hit L2)
// while each CTA's ring pipeline stays warm from one item to the next.
struct Work {
  int64_t tile, ilo, ihi;
};
__device__ __forceinline__ bool next_work(int mode, const StencilArgs& a, int64_t tiles, int64_t total, int64_t& cursor,
                                          Work& w) {
  if (mode == 0) {
    const int64_t g_end = total * (blockIdx.x + 1) / gridDim.x;
    if (cursor >= g_end) return false;
    w.tile = cursor / a.n0;
    w.ilo = cursor % a.n0;
    w.ihi = min(a.n0, w.ilo + (g_end - cursor));
    cursor = w.ihi == a.n0 ? (w.tile + 1) * a.n0 : g_end;
    return true;
  }
  const int64_t chunks = (a.n0 + a.ti - 1) / a.ti;
  if (cursor >= tiles * chunks) return false;
  w.tile = cursor % tiles;
  w.ilo = (cursor / tiles) * a.ti;
  w.ihi = min(a.n0, w.ilo + a.ti);
  cursor += gridDim.x;
  return true;
}

template <int MINB>
__global__ void __launch_bounds__(WS_THREADS, MINB) star7_pers(StencilArgs a, int64_t tiles_k, int64_t total, int mode) {
  constexpr int TJ = 16, ROWS = TJ + 2;
  extern __shared__ __align__(128) float sring[];
  __shared__ __align__(8) uint64_t full[NSLOT], empty[NSLOT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tiles = total / a.n0;
  const int64_t cursor0 = mode == 0 ? total * blockIdx.x / gridDim.x : blockIdx.x;
  const uint32_t pstride = static_cast<uint32_t>(a.e1 * a.e2), rstride = static_cast<uint32_t>(a.e2);

  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(s_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 8) {
    // ---------------- producer: walk the same segments, one plane per q
    uint32_t q = 0;
    int64_t cursor = cursor0;
    Work wk;
    while (next_work(mode, a, tiles, total, cursor, wk)) {
      const int64_t tile = wk.tile, ilo = wk.ilo, ihi = wk.ihi;
      const int64_t k0 = (tile % tiles_k) * TK, j0 = (tile / tiles_k) * TJ;
      const uint32_t base0 = static_cast<uint32_t>((ilo * a.e1 + j0) * a.e2 + k0);
      const float* vbase = a.v + ((ilo * a.e1 + j0) * a.e2 + k0);
      const int np = static_cast<int>(ihi - ilo) + 2;
      for (int p = 0; p < np; ++p, ++q) {
        const int s = static_cast<int>(q % NSLOT);
        if (q >= NSLOT) mbar_wait_parity(&empty[s], (q / NSLOT - 1) & 1);
        uint32_t bytes = 0, sh = 0;
        if (lane < ROWS) {
          sh = (base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(lane) * rstride) & 3u;
          bytes = (sh * 4 + (TK + 2) * 4 + 15) & ~15u;
        }
        uint32_t tot = bytes;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[s])), "r"(tot) : "memory");
        __syncwarp();
        if (lane < ROWS) {
          const float* src = vbase + static_cast<int64_t>(p) * (a.e1 * a.e2) + static_cast<int64_t>(lane) * a.e2 - sh;
          float* dst = sring + (static_cast<size_t>(s) * ROWS + lane) * BPITCH;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(&full[s])) : "memory");
        }
      }
    }
    return;
  }

  // ---------------- compute warps
  const int kl = lane * 4, jl = warp * 2;
  uint32_t q = 0;
  int64_t cursor = cursor0;
  Work wk;
  while (next_work(mode, a, tiles, total, cursor, wk)) {
    const int64_t tile = wk.tile, ilo = wk.ilo, ihi = wk.ihi;
    const int64_t k0 = (tile % tiles_k) * TK, j0 = (tile / tiles_k) * TJ;
    const uint32_t base0 = static_cast<uint32_t>((ilo * a.e1 + j0) * a.e2 + k0);
    const int n = static_cast<int>(ihi - ilo);
    const uint32_t q0 = q;
    auto rowptr = [&](int p, int r, int& sh) {
      sh = static_cast<int>((base0 + static_cast<uint32_t>(p) * pstride + static_cast<uint32_t>(r) * rstride) & 3u);
      return sring + (static_cast<size_t>((q0 + p) % NSLOT) * ROWS + r) * BPITCH + sh + kl;
    };
    auto wait = [&](int p) { mbar_wait_parity(&full[(q0 + p) % NSLOT], ((q0 + p) / NSLOT) & 1); };
    auto release = [&](int p) {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(&empty[(q0 + p) % NSLOT])) : "memory");
    };
    auto load_centre = [&](int p, Rows& R) {
      int sh;
      const float* p0 = rowptr(p, jl + 1, sh);
      ld6(p0, sh, R.r[0]);
      const float* p1 = rowptr(p, jl + 2, sh);
      ld6(p1, sh, R.r[1]);
    };
    float* wout = a.w + (ilo * a.n1 + j0 + jl) * a.n2 + k0 + kl;
    const int64_t wplane = a.n1 * a.n2;
    const bool kin = k0 + kl + 4 <= a.n2;
    auto step = [&](int t, const Rows& P, const Rows& C, Rows& N) {
      wait(t + 2);
      load_centre(t + 2, N);
      float jm[6], jp[6];
      int sh;
      const float* pm = rowptr(t + 1, jl, sh);
      ld6(pm, sh, jm);
      const float* pp = rowptr(t + 1, jl + 3, sh);
      ld6(pp, sh, jp);
      release(t + 1);
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const float* up = jj == 0 ? jm : C.r[0];
        const float* dn = jj == 1 ? jp : C.r[1];
        float o[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          float acc = a.wc * C.r[jj][kk + 1];
          acc = fmaf(a.wim, P.r[jj][kk + 1], acc);
          acc = fmaf(a.wip, N.r[jj][kk + 1], acc);
          acc = fmaf(a.wjm, up[kk + 1], acc);
          acc = fmaf(a.wjp, dn[kk + 1], acc);
          acc = fmaf(a.wkm, C.r[jj][kk], acc);
          acc = fmaf(a.wkp, C.r[jj][kk + 2], acc);
          o[kk] = acc;
        }
        if (j0 + jl + jj < a.n1) {
          float* dst = wout + t * wplane + jj * a.n2;
          if (kin) {
            __stcs(reinterpret_cast<float4*>(dst), make_float4(o[0], o[1], o[2], o[3]));
          } else {
            for (int kk = 0; kk < 4 && k0 + kl + kk < a.n2; ++kk) dst[kk] = o[kk];
          }
        }
      }
    };
    Rows R0, R1, R2;
    wait(0);
    wait(1);
    load_centre(0, R0);
    load_centre(1, R1);
    release(0);
    int t = 0;
    for (; t + 3 <= n; t += 3) {
      step(t, R0, R1, R2);
      step(t + 1, R1, R2, R0);
      step(t + 2, R2, R0, R1);
    }
    if (t < n) step(t, R0, R1, R2), ++t;
    if (t < n) step(t, R1, R2, R0), ++t;
    release(n + 1);  // the last plane was only read as "next"
    q += static_cast<uint32_t>(n + 2);
  }
}

// ---------------------------------------------------------------- host
// Recognises  sum_t lit_t * in(1, a_t)  (any association of + over terms,
// literal on either side of *, a bare in(1,a) = weight 1).
bool linear_terms(const Expr& e, std::vector<std::pair<double, int>>& terms) {
  if (e.k == EK::Add) return linear_terms(e.args[0], terms) && linear_terms(e.args[1], terms);
  if (e.k == EK::In && e.buf == 1) {
    terms.push_back({1.0, e.acc});
    return true;
  }
  if (e.k == EK::Mul) {
    const Expr *lit = nullptr, *in = nullptr;
    for (int s = 0; s < 2; ++s) {
      if (e.args[static_cast<size_t>(s)].k == EK::Lit) lit = &e.args[static_cast<size_t>(s)];
      if (e.args[static_cast<size_t>(s)].k == EK::In) in = &e.args[static_cast<size_t>(s)];
    }
    if (lit && in && in->buf == 1) {
      terms.push_back({lit->type == Ty::F64 ? lit->fv : static_cast<double>(lit->iv), in->acc});
      return true;
    }
  }
  return false;
}

// Schedules of the star-7 template (which kernel streams the planes):
//   LEAN     TMA-bulk producer warp + smem plane ring, centre columns in registers
//            (star7_s32: lanes strided by 32 columns; star7_lean: 4 adjacent columns per lane)
//   LEAN_TS  LEAN with the output staged in smem and written by TMA stores
//   WS       producer warp + ring, every neighbour read from smem (star7_ws)
//   PERS     WS on persistent CTAs striding over (tile, i-chunk) items (star7_pers)
//   PLAIN    no producer: the compute warps load their rows themselves (star7_kernel)
enum StencilSched { S_LEAN = 0, S_LEAN_TS = 1, S_WS = 2, S_PERS = 3, S_PLAIN = 4 };

class StencilRoutine final : public Routine {
 public:
  StencilRoutine(const Problem& p, StencilArgs a, int tj, bool bulk, int sched, int tkc = 128)
      : p_(p), a_(a), tj_(tj), bulk_(bulk && sched != S_PLAIN), ws_(bulk_ && sched != S_PLAIN),
        pers_(ws_ && sched == S_PERS), ts_(sched == S_LEAN_TS) {
    if (sched == S_WS || sched == S_PERS || !ws_) lean_ = 0;
    tkc_ = tkc;
  }
  const char* family() const override { return "stencil"; }
  std::string describe() const override {
    std::ostringstream os;
    const std::string kname = s32_ && lean_ && !ts_ok() ? "star7_s32<" + std::to_string(tkc_ != 128 ? 5 : s32_ / 10) + "," +
                                                                std::to_string(tkc_ != 128 ? 3 : s32_ % 10) +
                                                                (tkc_ != 128 ? "," + std::to_string(tkc_) : std::string()) + ">"
                              : lean_ && ts_ok() ? std::string("star7_lean<4,4,tma_store>")
                              : lean_ ? "star7_lean<" + std::to_string(lean_ / 10) + "," + std::to_string(lean_ % 10) + ">"
                                    : std::string(pers_ ? "star7_pers<" : ws_ ? "star7_ws<" : bulk_ ? "star7_bulk<" : "star7_kernel<") +
                                          std::to_string(tj_) + ">";
    const bool s32 = s32_ && lean_ && !ts_ok();
    const int tk = s32 ? tkc_ : TK, tj = s32 ? 2048 / tkc_ : tj_;
    os << "{\"kernel\": \"" << kname << "\", \"TK\": " << tk << ", \"TJ\": " << tj << ", \"TI\": " << a_.ti
       << ", \"threads\": " << (ws_ ? WS_THREADS : NTHREADS) << ", \"smem_ring_slots\": " << (lean_ ? lean_ / 10 : bulk_ ? NSLOT : 4)
       << ", \"ctas_per_sm\": " << (lean_ ? lean_ % 10 : 3) << ", \"grid\": [" << (a_.n2 + tk - 1) / tk << ", "
       << (a_.n1 + tj - 1) / tj << ", " << grid().z << "]}";
    return os.str();
  }
  dim3 grid() const {
    return dim3(static_cast<unsigned>((a_.n2 + TK - 1) / TK), static_cast<unsigned>((a_.n1 + tj_ - 1) / tj_),
                static_cast<unsigned>((a_.n0 + a_.ti - 1) / a_.ti));
  }
  int launches() const override { return 1; }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  double flops() const override { return 13.0 * static_cast<double>(a_.n0 * a_.n1 * a_.n2); }

  // End-to-end on host buffers, pipelined along the ++ dimension i: chunk c's
  // input planes go up on one copy engine while chunk c-1 computes and chunk
  // c-2's output planes come down on the other (the homomorphic split again:
  // every chunk is the same md_hom over a sub-range of i).
  bool supports_chunked_host() const override { return true; }
  void launch_host_chunked(const void* const* h_in, void* const* h_out, void* const* d_in, void* const* d_out,
                           cudaStream_t s) override {
    constexpr int kChunks = 16;
    if (!h2d_) {
      MDHB_CUDA(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
      MDHB_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
      for (int c = 0; c < kChunks + 2; ++c) {
        MDHB_CUDA(cudaEventCreateWithFlags(&ev_in_[c], cudaEventDisableTiming));
        MDHB_CUDA(cudaEventCreateWithFlags(&ev_cmp_[c], cudaEventDisableTiming));
      }
    }
    const int64_t pin = a_.e1 * a_.e2, pout = a_.n1 * a_.n2;
    const int64_t ci = (a_.n0 + kChunks - 1) / kChunks;
    const char* hi_in = static_cast<const char*>(h_in[0]);
    char* hi_out = static_cast<char*>(h_out[0]);
    char* dv = static_cast<char*>(d_in[0]);
    char* dw = static_cast<char*>(d_out[0]);
    MDHB_CUDA(cudaEventRecord(ev_in_[kChunks], s));  // respect work already queued on s
    MDHB_CUDA(cudaStreamWaitEvent(h2d_, ev_in_[kChunks], 0));
    int64_t copied = 0;
    int c = 0;
    for (int64_t lo = 0; lo < a_.n0; lo += ci, ++c) {
      const int64_t hi = std::min(a_.n0, lo + ci);
      const int64_t need = std::min(a_.e0, hi + 2);
      MDHB_CUDA(cudaMemcpyAsync(dv + copied * pin * 4, hi_in + copied * pin * 4,
                                static_cast<size_t>((need - copied) * pin * 4), cudaMemcpyHostToDevice, h2d_));
      copied = need;
      MDHB_CUDA(cudaEventRecord(ev_in_[c], h2d_));
      MDHB_CUDA(cudaStreamWaitEvent(s, ev_in_[c], 0));
      StencilArgs a = a_;
      a.n0 = hi - lo;
      a.e0 = a_.e0 - lo;
      const void* din[1] = {dv + lo * pin * 4};
      void* dout[1] = {dw + lo * pout * 4};
      StencilArgs keep = a_;
      a_ = a;
      launch(din, dout, s);
      a_ = keep;
      MDHB_CUDA(cudaEventRecord(ev_cmp_[c], s));
      MDHB_CUDA(cudaStreamWaitEvent(d2h_, ev_cmp_[c], 0));
      MDHB_CUDA(cudaMemcpyAsync(hi_out + lo * pout * 4, dw + lo * pout * 4, static_cast<size_t>((hi - lo) * pout * 4),
                                cudaMemcpyDeviceToHost, d2h_));
    }
    MDHB_CUDA(cudaEventRecord(ev_cmp_[kChunks], d2h_));
    MDHB_CUDA(cudaStreamWaitEvent(s, ev_cmp_[kChunks], 0));
  }
  ~StencilRoutine() override {
    if (h2d_) {
      cudaStreamDestroy(h2d_);
      cudaStreamDestroy(d2h_);
      for (int c = 0; c < 18; ++c) {
        cudaEventDestroy(ev_in_[c]);
        cudaEventDestroy(ev_cmp_[c]);
      }
    }
  }
  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    StencilArgs a = a_;
    a.v = static_cast<const float*>(d_in[0]);
    a.w = static_cast<float*>(d_out[0]);
    const size_t smem = static_cast<size_t>(NSLOT) * 18 * BPITCH * sizeof(float);
    MarkScope mark(this, s);
    if (pers_) {
      auto kern = minb_ == 2 ? star7_pers<2> : star7_pers<3>;
      MDHB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      if (!ctas_) {
        int occ = 0;
        MDHB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WS_THREADS, smem));
        ctas_ = std::max(1, occ) * sm_count(p_.opt.device);
      }
      const int64_t tiles_k = (a.n2 + TK - 1) / TK, tiles = tiles_k * ((a.n1 + 15) / 16);
      const int64_t total = tiles * a.n0;
      const int mode = std::getenv("MDHB_STENCIL_RANGES") ? 0 : 1;
      const int64_t items = tiles * ((a.n0 + a.ti - 1) / a.ti);
      const int grid_p = static_cast<int>(std::min<int64_t>(ctas_, mode ? items : std::max<int64_t>(1, total / 4)));
      kern<<<grid_p, WS_THREADS, smem, s>>>(a, tiles_k, total, mode);
    } else if (s32_ && lean_ && !ts_ok()) {
      a.pf = pf_;
      void (*k)(StencilArgs) = tkc_ == 256 ? star7_s32<5, 3, 256>
                               : tkc_ == 512 ? star7_s32<5, 3, 512>
                               : s32_ == 53  ? star7_s32<5, 3>
                               : s32_ == 63  ? star7_s32<6, 3>
                               : s32_ == 73  ? star7_s32<7, 3>
                               : s32_ == 44  ? star7_s32<4, 4>
                                             : star7_s32<5, 4>;
      const int ns = tkc_ != 128 ? 5 : s32_ / 10;
      const size_t lsmem = static_cast<size_t>(ns) * (2048 / tkc_ + 2) * (tkc_ + 8) * sizeof(float);
      MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lsmem)));
      const dim3 g(static_cast<unsigned>((a.n2 + tkc_ - 1) / tkc_), static_cast<unsigned>((a.n1 + 2048 / tkc_ - 1) / (2048 / tkc_)),
                   static_cast<unsigned>((a.n0 + a.ti - 1) / a.ti));
      k<<<g, WS_THREADS, lsmem, s>>>(a);
    } else if (lean_) {
      void (*k)(StencilArgs) = nullptr;
      const bool ts = ts_ok();
      if (ts) k = star7_lean<4, 4, true>;
      else if (lean_ == 53) k = star7_lean<5, 3, false>;
      else if (lean_ == 54) k = star7_lean<5, 4, false>;
      else if (lean_ == 44) k = star7_lean<4, 4, false>;
      else if (lean_ == 45) k = star7_lean<4, 5, false>;
      else k = star7_lean<6, 3, false>;
      const size_t lsmem = static_cast<size_t>(ts ? 4 : lean_ / 10) * 18 * BPITCH * sizeof(float) +
                           (ts ? static_cast<size_t>(8) * 4 * TK * sizeof(float) : 0);
      MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lsmem)));
      k<<<grid(), WS_THREADS, lsmem, s>>>(a);
    } else if (ws_) {
      MDHB_CUDA(cudaFuncSetAttribute(star7_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      star7_ws<<<grid(), WS_THREADS, smem, s>>>(a);
    } else if (bulk_) {
      MDHB_CUDA(cudaFuncSetAttribute(star7_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      star7_bulk<16><<<grid(), NTHREADS, smem, s>>>(a);
    } else {
      star7_kernel<16><<<grid(), NTHREADS, 0, s>>>(a);
    }
    MDHB_CUDA(cudaGetLastError());
  }

 private:
  const Problem& p_;
  StencilArgs a_;
  int tj_;
  bool bulk_;
  bool ws_;
  bool pers_;
  int ctas_ = 0;
  // strided-lane variant (star7_s32): NS*10+MINB, 0 = off
  // (default for the LEAN schedule: 206 vs 210 us at 512^3 on one box, bit-identical;
  // MDHB_STENCIL_LEAN selects the packed-lane star7_lean rings instead)
  int s32_ = std::getenv("MDHB_STENCIL_S32") ? std::atoi(std::getenv("MDHB_STENCIL_S32"))
                                            : (std::getenv("MDHB_STENCIL_LEAN") ? 0 : 53);
  int pf_ = std::getenv("MDHB_STENCIL_PF") ? std::atoi(std::getenv("MDHB_STENCIL_PF")) : 0;
  // star7_s32 k columns per CTA tile (128 / 256 / 512; rows 16 / 8 / 4)
  int tkc_ = 128;
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
  cudaEvent_t ev_in_[18] = {}, ev_cmp_[18] = {};
  int minb_ = std::getenv("MDHB_STENCIL_MINB") ? std::atoi(std::getenv("MDHB_STENCIL_MINB")) : 2;
  // lean-register variant (default): 5 ring slots, 4 CTAs per SM (NS*10+MINB; 0 = star7_ws)
  int lean_ = std::getenv("MDHB_STENCIL_LEAN") ? std::atoi(std::getenv("MDHB_STENCIL_LEAN")) : 54;
  bool ts_ = false;
  // TMA-store variant: full tiles, 16-byte aligned output rows
  bool ts_ok() const { return ts_ && a_.n2 % TK == 0 && a_.n1 % 16 == 0 && (a_.n2 * 4) % 16 == 0; }
};

}  // namespace

// ---- Table-1 instantiation (B200 ASM {DM, SM, RM | SMX, WRP, CC}; MDH
// layer order SMX -> DM -> WRP -> CC -> SM -> RM):
//   SMX(i, j, k) = grid (i-chunks, j/16, k/128); DM(i) = ti planes streamed
//   per CTA; DM(j) > 1 = CTAs walk several tiles (persistent); WRP(j) 8 x
//   RM(j) 2 = 16 rows, CC(k) 32 x RM(k) 4 = 128 columns per CTA.
//   Regions of v: at the SM layer SM = staged by the TMA producer, DM = read
//   by the compute warps (PLAIN); at the RM layer RM = centre columns held in
//   registers (LEAN), SM = re-read from the ring (WS).  Region of w at the SM
//   layer: SM = staged for TMA stores (LEAN_TS), else stored from registers.
struct StencilKnobs {
  int ti = 32;
  int sched = S_LEAN;
  int tkc = 128;  // k columns per CTA tile (LEAN: 128 / 256 / 512 with 16 / 8 / 4 rows; other schedules 128)
};

int region_at(const Config& c, const std::vector<std::vector<int>>& mem, size_t buf, int asm_layer, bool re, int D) {
  const auto& ass = re ? c.ass_re : c.ass_de;
  for (size_t r = 0; r < ass.size(); ++r)
    if (ass[r].layer == asm_layer && static_cast<int>(r) % D == 0) return mem[buf][r];
  return 0;
}

StencilKnobs stencil_knobs(const Problem& p, const Config& c) {
  const MdHom& e = p.e;
  const int smx = p.m.id("SMX"), dm = p.m.id("DM"), sm = p.m.id("SM"), rm = p.m.id("RM");
  if (smx < 0 || dm < 0 || sm < 0 || rm < 0) fail("Unsupported", "stencil template needs SMX, DM, SM and RM layers");
  auto P = parts_per_asm_layer(c, e, p.m);
  for (const char* other : {"GPU", "HM"})
    if (p.m.id(other) > 0)
      for (int64_t x : P[static_cast<size_t>(p.m.id(other) - 1)])
        if (x != 1) fail("Unsupported", std::string("stencil template: ") + other + " parts belong to the DEV layer");
  auto at = [&](int layer, int d) { return P[static_cast<size_t>(layer - 1)][static_cast<size_t>(d)]; };
  StencilKnobs k;
  const int64_t tj = e.sizes[1] % (at(smx, 1) * at(dm, 1)) ? 0 : e.sizes[1] / (at(smx, 1) * at(dm, 1));
  const int64_t tk = e.sizes[2] % (at(smx, 2) * at(dm, 2)) ? 0 : e.sizes[2] / (at(smx, 2) * at(dm, 2));
  if (!((tj == 16 && tk == 128) || (tj == 8 && tk == 256) || (tj == 4 && tk == 512)))
    fail("Unsupported", "stencil template tiles (j, k) by (16, 128), (8, 256) or (4, 512) per CTA");
  k.tkc = static_cast<int>(tk);
  if (e.sizes[0] % at(smx, 0)) fail("Unsupported", "stencil template needs uniform i-chunks");
  k.ti = static_cast<int>(e.sizes[0] / at(smx, 0));
  const bool persistent = at(dm, 1) > 1 || at(dm, 2) > 1;
  const int D = e.D();
  const int v_sm = region_at(c, c.mem_de, 0, sm, false, D), v_rm = region_at(c, c.mem_de, 0, rm, false, D);
  const int w_sm = region_at(c, c.mem_re, 0, sm, true, D);
  if (persistent) k.sched = S_PERS;
  else if (v_sm == dm) k.sched = S_PLAIN;
  else if (v_rm == rm) k.sched = w_sm == sm ? S_LEAN_TS : S_LEAN;
  else k.sched = S_WS;
  if (k.tkc != 128 && k.sched != S_LEAN) fail("Unsupported", "only the LEAN schedule takes 256- / 512-column tiles");
  return k;
}

Config stencil_canonical(const Problem& p, const StencilKnobs& k) {
  const MdHom& e = p.e;
  const int64_t tj = 2048 / k.tkc;
  const int64_t gj = e.sizes[1] / tj, gk = e.sizes[2] / k.tkc;
  const bool pers = k.sched == S_PERS && gj % 2 == 0;
  // threads: 8 warps over j (x 2 column halves at 512), 32 lanes over k, per
  // thread 8 values: 2 rows x 4 columns (128), 1 x 8 (256, 512)
  const std::vector<int64_t> wrp = k.tkc == 512 ? std::vector<int64_t>{1, 4, 2} : std::vector<int64_t>{1, 8, 1};
  const std::vector<int64_t> rmv = k.tkc == 128 ? std::vector<int64_t>{1, 2, 4} : std::vector<int64_t>{1, 1, 8};
  std::vector<LayerParts> lp = {{"SMX", {e.sizes[0] / k.ti, pers ? gj / 2 : gj, gk}}, {"DM", {k.ti, pers ? 2 : 1, 1}},
                                {"WRP", wrp}, {"CC", {1, 1, 32}}, {"SM", {1, 1, 1}}, {"RM", rmv}};
  Config c = make_config(p, lp, {{e.in[0].name, k.sched == S_PLAIN ? "DM" : "SM"}}, "RM");
  const int D = e.D(), sm = p.m.id("SM"), rm = p.m.id("RM"), dm = p.m.id("DM");
  for (size_t r = 0; r < c.ass_de.size(); ++r) {
    if (c.ass_de[r].layer == rm) c.mem_de[0][r] = (k.sched == S_LEAN || k.sched == S_LEAN_TS) ? rm : (k.sched == S_PLAIN ? dm : sm);
    if (c.ass_re[r].layer == sm && k.sched == S_LEAN_TS) c.mem_re[0][r] = sm;
  }
  (void)D;
  return c;
}

std::unique_ptr<Routine> make_stencil(const Problem& p, const Config* cfg, Config* cfg_out) {
  const MdHom& e = p.e;
  if (e.D() != 3 || e.in.size() != 1 || e.out.size() != 1 || e.assigns.size() != 1) return nullptr;
  for (auto& c : e.comb)
    if (c.kind != Combine::CC) return nullptr;
  const Buf& in = e.in[0];
  const Buf& out = e.out[0];
  if (in.rank != 3 || out.rank != 3 || out.acc.size() != 1 || in.type != Ty::F64) return nullptr;
  // output access: identity (w[i][j][k])
  for (int r = 0; r < 3; ++r) {
    const Affine& f = out.acc[0].idx[static_cast<size_t>(r)];
    if (f.c0 != 0) return nullptr;
    for (int d = 0; d < 3; ++d)
      if (f.coeff[static_cast<size_t>(d)] != (d == r ? 1 : 0)) return nullptr;
  }
  // input accesses: identity + offsets; must form the 7-point star around (1,1,1)
  std::vector<std::array<int64_t, 3>> off;
  for (auto& acc : in.acc) {
    std::array<int64_t, 3> o{};
    for (int r = 0; r < 3; ++r) {
      const Affine& f = acc.idx[static_cast<size_t>(r)];
      for (int d = 0; d < 3; ++d)
        if (f.coeff[static_cast<size_t>(d)] != (d == r ? 1 : 0)) return nullptr;
      o[static_cast<size_t>(r)] = f.c0;
    }
    off.push_back(o);
  }
  std::vector<std::pair<double, int>> terms;
  if (!linear_terms(e.assigns[0].e, terms)) return nullptr;
  // star slots: centre, i-1, i+1, j-1, j+1, k-1, k+1 (offsets relative to 1)
  const int64_t slot_off[7][3] = {{1, 1, 1}, {0, 1, 1}, {2, 1, 1}, {1, 0, 1}, {1, 2, 1}, {1, 1, 0}, {1, 1, 2}};
  double w[7] = {0, 0, 0, 0, 0, 0, 0};
  for (auto& t : terms) {
    auto& o = off[static_cast<size_t>(t.second - 1)];
    int slot = -1;
    for (int s = 0; s < 7; ++s)
      if (o[0] == slot_off[s][0] && o[1] == slot_off[s][1] && o[2] == slot_off[s][2]) slot = s;
    if (slot < 0) return nullptr;  // not a star-7 read
    w[slot] += t.first;
  }
  if (p.opt.fstore != Store::F32) return nullptr;  // f64 storage -> generic (bit-exact) path

  StencilArgs a{};
  a.n0 = e.sizes[0];
  a.n1 = e.sizes[1];
  a.n2 = e.sizes[2];
  a.e0 = p.in_ext[0][0];
  a.e1 = p.in_ext[0][1];
  a.e2 = p.in_ext[0][2];
  a.wc = static_cast<float>(w[0]);
  a.wim = static_cast<float>(w[1]);
  a.wip = static_cast<float>(w[2]);
  a.wjm = static_cast<float>(w[3]);
  a.wjp = static_cast<float>(w[4]);
  a.wkm = static_cast<float>(w[5]);
  a.wkp = static_cast<float>(w[6]);
  // the input must hold the 1-cell halo the star reads
  if (p.in_ext[0][0] < a.n0 + 2 || a.e1 < a.n1 + 2 || a.e2 < a.n2 + 2) return nullptr;

  const int TJ = 16;
  int ti = 32;
  int sched = S_LEAN;
  if (std::getenv("MDHB_STENCIL_V1") || std::getenv("MDHB_STENCIL_V2")) sched = S_PLAIN;  // dev aids
  if (std::getenv("MDHB_STENCIL_PERS")) sched = S_PERS;
  if (std::getenv("MDHB_STENCIL_TS")) sched = S_LEAN_TS;
  // LEAN: the widest k tile whose full tiles cover the output (longer
  // contiguous row reads: 172 vs 207 us at 512^3 for 512 vs 128 columns)
  int tkc = 128;
  for (int c : {512, 256})
    if (a.n2 % c == 0 && a.n1 % (2048 / c) == 0) {
      tkc = c;
      break;
    }
  if (const char* f = std::getenv("MDHB_STENCIL_TKC")) tkc = std::atoi(f);
  if (cfg) {
    StencilKnobs k = stencil_knobs(p, *cfg);
    ti = k.ti;
    sched = k.sched;
    tkc = k.tkc;
  }
  if (sched != S_LEAN) tkc = 128;
  if (const char* f = std::getenv("MDHB_STENCIL_TI")) ti = std::max(1, std::atoi(f));
  a.ti = ti;
  // TMA bulk row copies need every copied span inside the allocation: the
  // buffer size must be 16-byte rounded (rows overrun at most to the next
  // 16-byte boundary) and the k tiles must not reach past the row end.
  const int64_t vbytes = p.in_ext[0][0] * a.e1 * a.e2 * 4;
  // the producer copies whole (tile + halo) rows: full j and k tiles keep every
  // copy inside the buffer (ragged shapes take the PLAIN schedule)
  const bool bulk = vbytes % 16 == 0 && a.n2 % tkc == 0 && a.n1 % (2048 / tkc) == 0;
  if (cfg && sched != S_PLAIN && !bulk) fail("Unsupported", "stencil producer schedules need 16-byte rows and full j / k tiles");
  if (cfg && sched == S_LEAN_TS && (a.n1 % 16 || (a.n2 * 4) % 16)) fail("Unsupported", "TMA-store epilogue needs full tiles");
  if (cfg_out) {
    if (a.n1 % (2048 / tkc) || a.n2 % tkc || a.n0 % ti || p.m.id("WRP") < 0 || p.m.id("SMX") < 0)
      *cfg_out = baseline_config(e, p.m);
    else
      *cfg_out = stencil_canonical(p, {ti, sched, bulk ? tkc : 128});
  }
  return std::make_unique<StencilRoutine>(p, a, TJ, bulk, sched, tkc);
}

}  // namespace mdhb

namespace mdhb {
bool stencil_project(const Problem& p, const Config& c, Config* canon) {
  *canon = stencil_canonical(p, stencil_knobs(p, c));
  return true;
}

// Tuning space of the stencil template: i-planes per CTA (every divisor of
// the i extent) x the five schedules, as canonical configurations.
std::vector<Config> stencil_space(const Problem& p) {
  std::vector<Config> out;
  const MdHom& e = p.e;
  if (p.m.id("SMX") < 0 || p.m.id("WRP") < 0 || e.D() != 3) return out;
  if (e.sizes[1] % 16 || e.sizes[2] % 128) return out;
  for (int sched = S_LEAN; sched <= S_PLAIN; ++sched)
    for (int tkc : {128, 256, 512}) {
      if (tkc != 128 && (sched != S_LEAN || e.sizes[2] % tkc || e.sizes[1] % (2048 / tkc))) continue;
      for (int64_t ti = 1; ti <= e.sizes[0]; ti *= 2) {
        if (e.sizes[0] % ti) continue;
        if (sched == S_PERS && (e.sizes[1] / 16) % 2) continue;
        out.push_back(stencil_canonical(p, {static_cast<int>(ti), sched, tkc}));
      }
    }
  return out;
}
}  // namespace mdhb
