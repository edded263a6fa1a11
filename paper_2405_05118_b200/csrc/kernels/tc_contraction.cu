// Tensor-core instance of the contraction template (MATH_TF32):
// TMA -> 128B-swizzled shared memory -> tcgen05.mma.kind::tf32 -> TMEM ->
// tcgen05.ld epilogue -> C through the additive offset tables.
//
// Each operand is described as a TMA box over its own buffer (no im2col,
// no transposes): every buffer rank's index function is an affine sum of
// md_hom dims, so a tile origin maps to per-rank coordinates
//   coord[r] = c0_r + sum_{d in row dims} c_rd * origin_d + sum_{d in K} c_rd * k_d
// which the planner tabulates per row tile and per k-tile.  A K-major
// operand needs a K dim with unit coefficient in its innermost rank (32
// elements = one 128-byte swizzle row per k-tile); an MN-major operand needs
// a row dim there (32-element slabs) and the K dim in another rank.  MCC
// over NHWC is therefore a plain 4-D box {32 c, 8 q, 8 p, 2 n} of the input
// (the implicit GEMM needs no gather), and MatMul's B[k][n] is MN-major.
//
// CTA = 6 warps: warp 0 issues TMA, warp 1 owns TMEM and issues the MMAs
// (one elected thread), warps 2-5 drain TMEM (lane quarter = warp % 4).
// Pipelines: STAGES smem slots (full/empty mbarriers), one accumulator
// (BM = 128 lanes x BN fp32 columns of TMEM).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sstream>

#include "contraction_common.hpp"
#include "tc_gemm.cuh"

namespace mdhb {
namespace ctr {
namespace {

constexpr int BM = 128;
constexpr int BKE = 32;  // k elements per tile = one 128-byte swizzle row of fp32
constexpr int MAXR = 5;  // TMA rank limit

constexpr int MAXKD = 6;  // K dims handled by the producer's odometer

struct TcArgs {
  float* C;
  const int32_t *tCm, *tCn, *cm, *cn;
  const int32_t *a_mc, *b_nc;  // [tiles][MAXR] TMA coordinates of the row-tile origins (innermost first)
  int a_rank, b_rank;
  int nk, tilesM, tilesN;
  int cvec;
  // k-tile -> TMA coordinate offsets, as a mixed-radix odometer over the K
  // dims (innermost = the dim stepped by 32): kext digits, kstep elements per
  // digit, per-rank coefficients for A and B.  Computed in registers by the
  // producer thread -- no table loads on the TMA issue path.
  int nkd;
  int kext[MAXKD], kstep[MAXKD];
  int kca[MAXKD][MAXR], kcb[MAXKD][MAXR];
  // Table-1 instantiation (plan-time knobs): M tiles per raster group (the
  // SMX parts of the M dim, 0 = 8), and the K-split's starting coordinates
  // (SMX parts of the K dim: split s starts at ka0 / kb0)
  int group_m;
  int ka0[MAXR], kb0[MAXR];
  // packed operands whose K is not a multiple of the 128-byte k-tile: the
  // last k-step lands 32- or 64-byte rows (SWIZZLE_32B / 64B) through the
  // tail tensor maps instead of a zero-padded 128-byte step (0 = none)
  int tail_bytes;
};

template <int BN, int STAGES, bool B_MN>
__global__ void __launch_bounds__(192, 1)
    tc_gemm_tf32(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, TcArgs g) {
  constexpr uint32_t A_BYTES = BM * BKE * 4;
  constexpr uint32_t B_BYTES = BN * BKE * 4;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = tc::warp_uniform(), lane = threadIdx.x & 31;
  // grouped raster over (tilesM x tilesN) for L2 reuse
  const int GROUP_M = g.group_m > 0 ? g.group_m : 8;
  const int x = blockIdx.x;
  const int per_group = GROUP_M * g.tilesN;
  const int first_m = (x / per_group) * GROUP_M;
  const int gsz = min(g.tilesM - first_m, GROUP_M);
  const int tm = first_m + (x % per_group) % gsz;
  const int tn = (x % per_group) / gsz;

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tma_a);
    tc::tma_prefetch(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tmem_full, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    int am0[MAXR], bn0[MAXR], ka[MAXR], kb[MAXR], dig[MAXKD];
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      am0[r] = g.a_mc[tm * MAXR + r];
      bn0[r] = g.b_nc[tn * MAXR + r];
      ka[r] = g.ka0[r];
      kb[r] = g.kb0[r];
    }
#pragma unroll
    for (int q = 0; q < MAXKD; ++q) dig[q] = 0;
    for (int kt = 0; kt < g.nk; ++kt) {
      const int s = kt % STAGES, it = kt / STAGES;
      if (kt >= STAGES) tc::mbar_wait(&empty[s], (it - 1) & 1);
      tc::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      uint8_t* sa = smem + s * STAGE_BYTES;
      uint8_t* sb = sa + A_BYTES;
      int c[MAXR];
#pragma unroll
      for (int r = 0; r < MAXR; ++r) c[r] = am0[r] + ka[r];
      tc::tma_load(sa, &tma_a, &full[s], g.a_rank, c);
#pragma unroll
      for (int r = 0; r < MAXR; ++r) c[r] = bn0[r] + kb[r];
      if (B_MN) {
        for (int j = 0; j < BN / 32; ++j) {
          int cj[MAXR];
#pragma unroll
          for (int r = 0; r < MAXR; ++r) cj[r] = c[r];
          cj[0] += 32 * j;
          tc::tma_load(sb + j * (BKE * 128), &tma_b, &full[s], g.b_rank, cj);
        }
      } else {
        tc::tma_load(sb, &tma_b, &full[s], g.b_rank, c);
      }
      // advance the K odometer (innermost digit last)
      for (int q = g.nkd - 1; q >= 0; --q) {
        if (++dig[q] < g.kext[q]) {
#pragma unroll
          for (int r = 0; r < MAXR; ++r) {
            ka[r] += g.kca[q][r] * g.kstep[q];
            kb[r] += g.kcb[q][r] * g.kstep[q];
          }
          break;
        }
#pragma unroll
        for (int r = 0; r < MAXR; ++r) {
          ka[r] -= g.kca[q][r] * g.kstep[q] * (g.kext[q] - 1);
          kb[r] -= g.kcb[q][r] * g.kstep[q] * (g.kext[q] - 1);
        }
        dig[q] = 0;
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = tc::instr_desc(2, 0, B_MN ? 1 : 0, BM, BN);
    for (int kt = 0; kt < g.nk; ++kt) {
      const int s = kt % STAGES, it = kt / STAGES;
      tc::mbar_wait(&full[s], it & 1);
      tc::tc_fence_after();
      const uint32_t sa = tc::smem_u32(smem + s * STAGE_BYTES);
      const uint32_t sb = sa + A_BYTES;
#pragma unroll
      for (int k = 0; k < BKE / 8; ++k) {
        const uint64_t da = tc::sw128_desc(sa + k * 32, 16, 1024);
        // MN-major fp32 operands live in the 32-byte-atom 128B swizzle (layout 1):
        // LBO = stride of 32-element MN slabs, SBO = stride of 4-row K atoms
        const uint64_t db = B_MN ? tc::umma_desc(sb + k * 1024, BKE * 128, 512, 1) : tc::sw128_desc(sb + k * 32, 16, 1024);
        tc::mma<true>(tmem, da, db, idesc, (kt | k) != 0 ? 1u : 0u);
      }
      tc::mma_commit(&empty[s]);  // frees the slot once these MMAs have read it
    }
    tc::mma_commit(tmem_full);
  } else if (warp >= 2) {
    // ---------------- epilogue: TMEM -> registers -> C
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    tc::mbar_wait(tmem_full, 0);
    tc::tc_fence_after();
    float* crow = g.C + g.tCm[tm] + g.cm[row] + g.tCn[tn];
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      tc::tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), r);
      if (g.cvec) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(crow + g.cn[c0 + j]) =
              make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) crow[g.cn[c0 + j]] = __uint_as_float(r[j]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// De-composition layout pass (Table-1 D4, layout_de = [2,1]): an MN-major
// operand B[k][n] is rewritten K-major as Bt[n][k] so the MMA reads both
// operands K-major -- MN-major fp32 operands run the tensor pipe at half
// rate on sm_100 (measured: 237 vs 464 TFLOP/s at 8192^3).
__global__ void __launch_bounds__(256) transpose_kn(const float* __restrict__ src, int64_t sk, int64_t sn,
                                                   float* __restrict__ dst, int K, int N) {
  __shared__ float t[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows per pass
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    int k = k0 + r, n = n0 + tx;
    t[r][tx] = (k < K && n < N) ? __ldcs(src + k * sk + n * sn) : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    int n = n0 + r, k = k0 + tx;
    if (n < N && k < K) dst[static_cast<int64_t>(n) * K + k] = t[tx][r];
  }
}


// Operand packing pass (Table-1 D4 layout_de for views no TMA box can
// describe, e.g. CCSD(T)'s A[g][d][a][b] with the contraction index outermost
// and 24-wide M dims): the operand is gathered through the contraction
// template's additive offset tables into a K-major [tile][row][Kp] scratch
// (K zero-padded to a multiple of 32), i.e. exactly the order in which the
// MMA tiles consume it.  Consecutive threads walk k, so the writes coalesce.
__global__ void __launch_bounds__(256) pack_kmajor(const float* __restrict__ src, float* __restrict__ dst,
                                                   const int32_t* __restrict__ tile_off, const int32_t* __restrict__ row_off,
                                                   const int32_t* __restrict__ k_off, int rows, int K, int Kp, int64_t total) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < total; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int k = static_cast<int>(i % Kp);
    const int64_t rr = i / Kp;
    const int r = static_cast<int>(rr % rows);
    const int64_t t = rr / rows;
    dst[i] = k < K ? __ldg(src + tile_off[t] + row_off[r] + k_off[k]) : 0.f;
  }
}

// Epilogue store of one 32 x 32 block drained from TMEM (lane = row, r[j] =
// column c0 + j) through this warp's staging square (stg) to C rows at
// tbase + rtab[row] + cn[column]:
//  * cvec (columns in aligned runs of 4): rows land in 144-byte-pitch smem
//    rows by STS.128; lane l then reads row 4 s + l / 8, columns 4 (l % 8) ..
//    +3 (LDS.128, conflict-free at that pitch) and stores them with one
//    STG.128 -- each store instruction writes 4 rows x 128 contiguous bytes;
//  * else the 33-word-pitch transpose: lane = column, one STG.32 per row.
__device__ __forceinline__ void epi_block(const uint32_t (&r)[32], uint32_t stg, uint32_t rtab, float* C, int64_t tbase,
                                          const int32_t* cn, int c0, int lane, bool cvec) {
  if (cvec) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + lane * 144 + j * 16), "r"(r[4 * j]),
                   "r"(r[4 * j + 1]), "r"(r[4 * j + 2]), "r"(r[4 * j + 3])
                   : "memory");
    __syncwarp();
    const int sub = lane & 7, rq = lane >> 3;
    float* cc = C + tbase + cn[c0 + 4 * sub];
#pragma unroll
    for (int s0 = 0; s0 < 8; s0 += 4) {
      int ro[4];
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = 4 * (s0 + u) + rq;
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(ro[u]) : "r"(rtab + row * 4));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                     : "r"(stg + row * 144 + sub * 16));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) __stcs(reinterpret_cast<float4*>(cc + ro[u]), v[u]);
    }
    __syncwarp();
    return;
  }
#pragma unroll
  for (int j = 0; j < 32; ++j)
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(stg + (lane * 33 + j) * 4), "r"(r[j]) : "memory");
  __syncwarp();
  float* cc = C + tbase + cn[c0 + lane];
  // 8 rows per batch: 16 shared loads in flight before the 8 stores (a
  // load -> store -> load chain per row left each warp waiting one
  // shared-load latency per 128-byte store)
#pragma unroll
  for (int r0 = 0; r0 < 32; r0 += 8) {
    int ro[8];
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      asm volatile("ld.shared.s32 %0, [%1];" : "=r"(ro[u]) : "r"(rtab + (r0 + u) * 4));
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[u]) : "r"(stg + ((r0 + u) * 33 + lane) * 4));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) __stcs(cc + ro[u], v[u]);
  }
  __syncwarp();
}

// shared-memory layout of tc_gemm_pers: A ring | B ring (or resident B) |
// barriers (256 B) | epilogue staging (4 warps x 32 x 33 floats)
#define EPI_OFF(ST, BNV, BSLOTS) \
  (static_cast<size_t>(ST) * BM * BKE * 4 + static_cast<size_t>(BSLOTS) * (BNV) * BKE * 4 + 256)
// epilogue warps: 2 per TMEM lane quarter (splitting the tile's columns), or
// 1 per quarter when a resident B
// (resident B) or a 256-wide tile's 4-stage ring leaves no room for 8 squares
__host__ __device__ constexpr int epi_warps(bool rb, int bn) { return (rb && bn <= 128) || bn >= 256 ? 4 : 8; }
__host__ __device__ constexpr size_t epi_bytes(bool rb, int bn) { return epi_warps(rb, bn) * (32 * 36 * 4 + 32 * 8); }

// bf16 packing (MATH_BF16): the same gather, converting to bf16 (round to
// nearest even).  k-fast: consecutive threads walk k (coalesced when k is the
// operand's unit-stride direction).  row-fast: a 32 x 32 (row, k) block goes
// through shared memory so that reads walk the rows (MatMul's B[k][n]) and
// writes walk k.
__global__ void __launch_bounds__(256) pack_kmajor_bf16(const float* __restrict__ src, uint16_t* __restrict__ dst,
                                                        const int32_t* __restrict__ tile_off, const int32_t* __restrict__ row_off,
                                                        const int32_t* __restrict__ k_off, int rows, int K, int Kp, int64_t total) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < total; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int k = static_cast<int>(i % Kp);
    const int64_t rr = i / Kp;
    const int r = static_cast<int>(rr % rows);
    const int64_t t = rr / rows;
    const float v = k < K ? __ldg(src + tile_off[t] + row_off[r] + k_off[k]) : 0.f;
    dst[i] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
  }
}
template <typename OutT>
__global__ void __launch_bounds__(256) pack_rows(const float* __restrict__ src, OutT* __restrict__ dst,
                                                 const int32_t* __restrict__ tile_off, const int32_t* __restrict__ row_off,
                                                 const int32_t* __restrict__ k_off, int rows, int K, int Kp, int64_t n_rows) {
  __shared__ float t[32][33];
  const int k0 = blockIdx.x * 32;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int kk = ty; kk < 32; kk += 8) {  // read: lanes along rows
    const int64_t gr = r0 + tx;
    const int k = k0 + kk;
    float v = 0.f;
    if (gr < n_rows && k < K) v = __ldg(src + tile_off[gr / rows] + row_off[gr % rows] + k_off[k]);
    t[kk][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int rr = ty; rr < 32; rr += 8) {  // write: lanes along k
    const int64_t gr = r0 + rr;
    if (gr < n_rows && k0 + tx < Kp) {
      if constexpr (sizeof(OutT) == 2) dst[gr * Kp + k0 + tx] = __bfloat16_as_ushort(__float2bfloat16_rn(t[tx][rr]));
      else dst[gr * Kp + k0 + tx] = t[tx][rr];
    }
  }
}

// Vectorised layout passes for plain 2-D operands (the MatMul case):
//   transpose64<OutT>: dst[n][k] (pitch Kp, zero-padded past K) from src with
//     n unit-stride and k stride sk -- 64 x 64 tiles, 16-byte reads along n,
//     16-byte writes along k (4 fp32 or 8 bf16)
//   convert_kvec_bf16: dst[r][k] (pitch Kp) from src rows of K contiguous
//     floats (row stride sr) -- 8 k per thread, two 16-byte reads, one write
template <typename OutT>
__global__ void __launch_bounds__(256) transpose64(const float* __restrict__ src, int64_t sk, OutT* __restrict__ dst, int K,
                                                   int N, int Kp) {
  __shared__ float t[64][65];
  const int k0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // 64 k-rows x 16 float4 along n
    const int c = tid + 256 * i, kk = c >> 4, n4 = (c & 15) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k0 + kk < K && n0 + n4 + 3 < N) v = __ldcs(reinterpret_cast<const float4*>(src + (k0 + kk) * sk + n0 + n4));
    t[kk][n4] = v.x;
    t[kk][n4 + 1] = v.y;
    t[kk][n4 + 2] = v.z;
    t[kk][n4 + 3] = v.w;
  }
  __syncthreads();
  constexpr int V = sizeof(OutT) == 4 ? 4 : 8;  // k per 16-byte store
#pragma unroll
  for (int i = 0; i < (64 * 64 / V) / 256; ++i) {
    const int c = tid + 256 * i, nn = c / (64 / V), kq = (c % (64 / V)) * V;
    if (n0 + nn >= N || k0 + kq >= Kp) continue;
    OutT* d = dst + static_cast<int64_t>(n0 + nn) * Kp + k0 + kq;
    if (sizeof(OutT) == 4) {
      *reinterpret_cast<float4*>(d) = make_float4(t[kq][nn], t[kq + 1][nn], t[kq + 2][nn], t[kq + 3][nn]);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const __nv_bfloat162 b2 = __floats2bfloat162_rn(t[kq + 2 * h][nn], t[kq + 2 * h + 1][nn]);
        w[h] = *reinterpret_cast<const uint32_t*>(&b2);
      }
      *reinterpret_cast<uint4*>(d) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}
__global__ void __launch_bounds__(256) convert_kvec_bf16(const float* __restrict__ src, int64_t sr, uint16_t* __restrict__ dst,
                                                         int K, int Kp, int64_t n_rows) {
  const int per = Kp / 8;
  const int64_t total = n_rows * per;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < total; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int64_t r = i / per;
    const int k = static_cast<int>(i - r * per) * 8;
    float v[8];
    if (k + 8 <= K) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(src + r * sr + k));
      const float4 b = __ldcs(reinterpret_cast<const float4*>(src + r * sr + k + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = k + j < K ? src[r * sr + k + j] : 0.f;
    }
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
      w[h] = *reinterpret_cast<const uint32_t*>(&b2);
    }
    *reinterpret_cast<uint4*>(dst + r * Kp + k) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Persistent variant: one CTA per SM walks the tile list; two TMEM
// accumulators (2 x BN columns) let the epilogue warps drain tile i while
// the MMA warp already accumulates tile i+1.  With RB (resident B) the whole
// K extent of B for the single N tile is loaded once per CTA and stays in
// shared memory -- MCC's 147 KB filter -- so only A streams from HBM.
template <int BN, int STAGES, bool B_MN, bool RB, bool BF16 = false>
__global__ void __launch_bounds__(64 + 32 * epi_warps(RB, BN), 1)
    tc_gemm_pers(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, TcArgs g,
                 const __grid_constant__ CUtensorMap tma_at, const __grid_constant__ CUtensorMap tma_bt) {
  constexpr uint32_t A_BYTES = BM * BKE * 4;
  constexpr uint32_t B_BYTES = BN * BKE * 4;
  constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  const uint32_t b_slots = RB ? static_cast<uint32_t>(g.nk) : STAGES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + b_slots * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* bfull = empty + STAGES;
  uint64_t* tfull = bfull + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // per epilogue warp: a 32 x 33 staging square (row-major in, column-major out)
  float* stage_base = reinterpret_cast<float*>(smem + EPI_OFF(STAGES, BN, b_slots));
  const int warp = tc::warp_uniform(), lane = threadIdx.x & 31;
  const int ntiles = g.tilesM * g.tilesN;
  const int GROUP_M = g.group_m > 0 ? g.group_m : 8;
  auto tile_mn = [&](int x, int& tm, int& tn) {
    const int per_group = GROUP_M * g.tilesN;
    const int first_m = (x / per_group) * GROUP_M;
    const int gsz = min(g.tilesM - first_m, GROUP_M);
    tm = first_m + (x % per_group) % gsz;
    tn = (x % per_group) / gsz;
  };
  // RB: CTA b keeps N tile b % tilesN resident and walks the M tiles
  // b / tilesN, + lanes, ... (lanes = gridDim / tilesN CTAs per N tile), so
  // only A streams; else tiles x = b, b + gridDim, ... in raster order
  const int lanes = RB ? static_cast<int>(gridDim.x) / g.tilesN : 1;
  const int tn_res = RB ? static_cast<int>(blockIdx.x) % g.tilesN : 0;
  const int sub = RB ? static_cast<int>(blockIdx.x) / g.tilesN : 0;
  const int my_tiles = RB ? (g.tilesM - sub + lanes - 1) / lanes
                          : (ntiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
  auto tile_of = [&](int j, int& tm, int& tn) {
    if (RB) {
      tm = sub + j * lanes;
      tn = tn_res;
    } else {
      tile_mn(static_cast<int>(blockIdx.x) + j * static_cast<int>(gridDim.x), tm, tn);
    }
  };
  const int tb = g.tail_bytes;  // bytes per row of the last k-step (0: full 128-byte step)
  const int nk = g.nk;
  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tma_a);
    tc::tma_prefetch(&tma_b);
    if (tb) {
      tc::tma_prefetch(&tma_at);
      tc::tma_prefetch(&tma_bt);
    }
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(bfull, 1);
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], epi_warps(RB, BN));  // one arrival per epilogue warp
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto kstep = [&](int (&dig)[MAXKD], int (&ka)[MAXR], int (&kb)[MAXR]) {
    for (int q = g.nkd - 1; q >= 0; --q) {
      if (++dig[q] < g.kext[q]) {
#pragma unroll
        for (int r = 0; r < MAXR; ++r) {
          ka[r] += g.kca[q][r] * g.kstep[q];
          kb[r] += g.kcb[q][r] * g.kstep[q];
        }
        return;
      }
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        ka[r] -= g.kca[q][r] * g.kstep[q] * (g.kext[q] - 1);
        kb[r] -= g.kcb[q][r] * g.kstep[q] * (g.kext[q] - 1);
      }
      dig[q] = 0;
    }
  };

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    if (RB) {  // all of B for the (single) N tile, once
      int dig[MAXKD] = {0, 0, 0, 0, 0, 0}, ka[MAXR], kb[MAXR];
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        ka[r] = g.ka0[r];
        kb[r] = g.kb0[r];
      }
      tc::mbar_arrive_expect_tx(bfull, tb ? static_cast<uint32_t>(nk - 1) * B_BYTES + static_cast<uint32_t>(BN * tb)
                                          : static_cast<uint32_t>(nk) * B_BYTES);
      for (int kt = 0; kt < nk; ++kt) {
        int c[MAXR];
#pragma unroll
        for (int r = 0; r < MAXR; ++r) c[r] = g.b_nc[tn_res * MAXR + r] + kb[r];
        tc::tma_load(sB + kt * B_BYTES, tb && kt == nk - 1 ? &tma_bt : &tma_b, bfull, g.b_rank, c);
        kstep(dig, ka, kb);
      }
    }
    uint32_t it = 0;
    for (int j = 0; j < my_tiles; ++j) {
      int tm, tn;
      tile_of(j, tm, tn);
      int am0[MAXR], bn0[MAXR], ka[MAXR], kb[MAXR], dig[MAXKD];
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        am0[r] = g.a_mc[tm * MAXR + r];
        bn0[r] = g.b_nc[tn * MAXR + r];
        ka[r] = g.ka0[r];
        kb[r] = g.kb0[r];
      }
#pragma unroll
      for (int q = 0; q < MAXKD; ++q) dig[q] = 0;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const uint32_t s = it % STAGES;
        const bool tail = tb && kt == nk - 1;
        if (it >= STAGES) tc::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        tc::mbar_arrive_expect_tx(&full[s], tail ? static_cast<uint32_t>((BM + (RB ? 0 : BN)) * tb) : A_BYTES + (RB ? 0u : B_BYTES));
        int c[MAXR];
#pragma unroll
        for (int r = 0; r < MAXR; ++r) c[r] = am0[r] + ka[r];
        tc::tma_load(sA + s * A_BYTES, tail ? &tma_at : &tma_a, &full[s], g.a_rank, c);
        if (!RB) {
#pragma unroll
          for (int r = 0; r < MAXR; ++r) c[r] = bn0[r] + kb[r];
          if (tail) {
            tc::tma_load(sB + s * B_BYTES, &tma_bt, &full[s], g.b_rank, c);
          } else if (B_MN) {
            for (int j = 0; j < BN / 32; ++j) {
              int cj[MAXR];
#pragma unroll
              for (int r = 0; r < MAXR; ++r) cj[r] = c[r];
              cj[0] += 32 * j;
              tc::tma_load(sB + s * B_BYTES + j * (BKE * 128), &tma_b, &full[s], g.b_rank, cj);
            }
          } else {
            tc::tma_load(sB + s * B_BYTES, &tma_b, &full[s], g.b_rank, c);
          }
        }
        kstep(dig, ka, kb);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: whole warp, uniform operands, one elected lane issues
    constexpr uint32_t idesc = tc::instr_desc(BF16 ? 1 : 2, 0, B_MN ? 1 : 0, BM, BN);  // kind::f16 bf16 | kind::tf32
    if (RB) tc::mbar_wait_warp(bfull, 0);
    uint32_t it = 0, tl = 0;
    for (int j = 0; j < my_tiles; ++j, ++tl) {
      const uint32_t acc = tl & 1;
      if (tl >= 2) tc::mbar_wait_warp(&tempty[acc], ((tl / 2) - 1) & 1);
      tc::tc_fence_after();
      const uint32_t dtm = tmem + acc * BN;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const uint32_t s = it % STAGES;
        tc::mbar_wait_warp(&full[s], (it / STAGES) & 1);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(sA + s * A_BYTES);
        const uint32_t sb = tc::smem_u32(sB + (RB ? static_cast<uint32_t>(kt) : s) * B_BYTES);
        if (tb && kt == nk - 1) {
          // tail k-step: 32- / 64-byte swizzled rows (8-row atoms of 8 x tb bytes)
          const uint32_t lt = tb == 32 ? 6u : 4u;
          for (int k = 0; k < tb / 32; ++k) {
            const uint64_t da = tc::umma_desc(sa + k * 32, 16, 8 * tb, lt);
            const uint64_t db = tc::umma_desc(sb + k * 32, 16, 8 * tb, lt);
            tc::mma_warp<!BF16>(dtm, da, db, idesc, (kt | k) != 0 ? 1u : 0u);
          }
        } else {
#pragma unroll
        for (int k = 0; k < BKE / 8; ++k) {
          const uint64_t da = tc::sw128_desc(sa + k * 32, 16, 1024);
          const uint64_t db = B_MN ? tc::umma_desc(sb + k * 1024, BKE * 128, 512, 1) : tc::sw128_desc(sb + k * 32, 16, 1024);
          tc::mma_warp<!BF16>(dtm, da, db, idesc, (kt | k) != 0 ? 1u : 0u);
        }
        }
        tc::mma_commit_warp(&empty[s]);
      }
      tc::mma_commit_warp(&tfull[acc]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue warps: TMEM -> registers -> 32x32 smem
    // transpose -> C.  After the transpose lane j holds column c0 + j of 32
    // consecutive rows, so each store instruction writes one row's 32
    // columns: 128 contiguous bytes whenever the tile's columns are
    // contiguous in C (MatMul, MCC, CCSD(T) with a full (e, f) block) --
    // instead of 32 scattered 16-byte pieces, one per TMEM lane / C row.
    constexpr int NH = epi_warps(RB, BN) / 4;  // column parts per lane quarter
    const int q = warp & 3, half = (warp - 2) >> 2;  // lane quarter, column part
    const int ew = warp - 2;
    // shared (.shared window) addresses of this warp's staging square and row table
    const uint32_t stg = tc::smem_u32(stage_base) + static_cast<uint32_t>(ew) * (32 * 36 * 4 + 32 * 8);
    const uint32_t rtab = stg + 32 * 36 * 4;
    constexpr int CH = (BN / 32 + NH - 1) / NH;  // 32-column chunks per column part
    uint32_t tl = 0;
    for (int j = 0; j < my_tiles; ++j, ++tl) {
      int tm, tn;
      tile_of(j, tm, tn);
      const uint32_t acc = tl & 1;
      // row table: C offset of TMEM lane q*32 + r (tile origin folded in)
      // C offset of TMEM lane q*32 + r = tile origin + cm[q*32 + r] (row table in smem)
      const int64_t tbase = static_cast<int64_t>(g.tCm[tm]) + g.tCn[tn];
      asm volatile("st.shared.s32 [%0], %1;" ::"r"(rtab + lane * 4), "r"(g.cm[q * 32 + lane]) : "memory");
      tc::mbar_wait(&tfull[acc], (tl / 2) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < CH; ++ch) {
        const int c0 = (half * CH + ch) * 32;
        if (c0 >= BN) break;
        uint32_t r[32];
        tc::tmem_ld32(tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), r);
        epi_block(r, stg, rtab, g.C, tbase, g.cn, c0, lane, g.cvec != 0);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs on one TPC
// computes a 256 x BN tile with M = 256 MMAs issued by the leader.  Each CTA
// lands its own 128 rows of A and HALF of the BN rows of B (the MMA reads
// the peer's half at the same shared-memory offsets), so per SM the ring
// moves A + B/2 per k-tile instead of A + B -- the single-CTA kernel is
// shared-memory-bandwidth bound (TMA writes + MMA reads of 96 KB per k-tile
// at BN = 256).  Both CTAs' TMA loads complete on the leader's full[s]
// barrier; the leader's MMA commits multicast to both CTAs' empty[s] /
// tfull[a]; both CTAs' epilogue warps release the accumulator on the
// leader's tempty[a].  Each CTA drains its own 128 TMEM lanes x BN columns.
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2sm(void* dst, const void* tmap, uint32_t mbar_cluster, int rank, const int* c) {
  const uint32_t d = tc::smem_u32(dst);
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(d), "l"(tmap), "r"(mbar_cluster), "r"(c[0]), "r"(c[1]) : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(d), "l"(tmap), "r"(mbar_cluster), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                   ::"r"(d), "l"(tmap), "r"(mbar_cluster), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
      break;
    default:
      asm volatile("cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                   ::"r"(d), "l"(tmap), "r"(mbar_cluster), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
      break;
  }
}

// 2-D TMA load into this CTA AND the CTAs of `mask` (same smem offsets);
// with cta_group::2 each destination's complete_tx lands on its pair
// leader's barrier (the even CTA of the pair)
__device__ __forceinline__ void tma_load_2sm_mc(void* dst, const void* tmap, uint32_t mbar_cluster, uint16_t mask,
                                                const int* c) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.cta_group::2"
      " [%0], [%1, {%3, %4}], [%2], %5;"
      ::"r"(tc::smem_u32(dst)), "l"(tmap), "r"(mbar_cluster), "r"(c[0]), "r"(c[1]), "h"(mask) : "memory");
}

// MC: a cluster of FOUR CTAs = two CTA pairs on the tiles (tm, 2n) and
// (tm, 2n + 1), which share their A rows: CTA r lands half of its A tile
// (64 rows, multicast) in itself and in CTA r ^ 2, so each A row crosses
// from L2 once per cluster instead of once per pair.  A stage is reused only
// after BOTH pairs' MMAs released it (empty[s] counts two commits, each
// multicast to all four CTAs).
//
// WIDE: the pair's tile is 256 rows x TWO adjacent N tiles (2 * BN = 512
// columns): each k-step lands A once for both halves (48 KB per CTA per
// 32-deep k-step for 2^21 MACs instead of 32 KB for 2^20), so the operand
// bytes crossing from L2 per MAC drop by a quarter.  The 512-column
// accumulator fills TMEM, so it is single-buffered: the epilogue drains half
// 0 then half 1, releasing each on its own tempty barrier, and the next
// tile's first MMAs into a half wait only for that half.
template <int BN, int STAGES, bool BF16 = false, bool B_MN = false, bool MC = false, bool WIDE = false>
__global__ void __launch_bounds__(64 + 32 * 4, 1)
    tc_gemm_2sm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, TcArgs g, int b_row_rank) {
  constexpr int EPW = 4;
  constexpr int NH = WIDE ? 2 : 1;  // N tiles per pair tile
  static_assert(!WIDE || (BN == 256 && !MC), "WIDE: BN 256, no multicast");
  constexpr uint32_t A_BYTES = BM * BKE * 4;
  constexpr uint32_t B_BYTES = (BN / 2) * BKE * 4;  // this CTA's half of one N tile of B
  constexpr uint32_t TMEM_COLS = WIDE ? 512 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * NH * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stage_base = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);
  const int warp = tc::warp_uniform(), lane = threadIdx.x & 31;
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const uint32_t rank = crank & 1u;           // rank within the CTA pair
  const uint32_t lead_rank = crank & ~1u;     // the pair leader's cluster rank
  const int pp = static_cast<int>(crank >> 1);  // MC: pair index within the cluster
  const bool leader = rank == 0;
  const int pair = MC ? static_cast<int>(blockIdx.x) >> 2 : static_cast<int>(blockIdx.x) >> 1;
  const int npairs = MC ? static_cast<int>(gridDim.x) >> 2 : static_cast<int>(gridDim.x) >> 1;
  const int tilesM2 = g.tilesM / 2;  // 256-row tiles
  const int tilesNs = MC || WIDE ? g.tilesN / 2 : g.tilesN;  // MC: pairs of N tiles per cluster work item
  const int ntiles = tilesM2 * tilesNs;
  const int GROUP_M = g.group_m > 0 ? g.group_m : 8;
  auto tile_mn = [&](int x, int& tm, int& tn) {
    const int per_group = GROUP_M * tilesNs;
    const int first_m = (x / per_group) * GROUP_M;
    const int gsz = min(tilesM2 - first_m, GROUP_M);
    tm = first_m + (x % per_group) % gsz;
    tn = (x % per_group) / gsz;
    if (MC) tn = 2 * tn + pp;
    if (WIDE) tn = 2 * tn;  // first of the tile's two N tiles
  };
  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tma_a);
    tc::tma_prefetch(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], MC ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 2 * EPW);  // leader's copy: the epilogue warps of both CTAs
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::tc_fence_before();
  // both CTAs' barriers exist before anyone touches the peer's
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs): own A rows, own half of B
    const uint32_t full_leader0 = peer_addr(tc::smem_u32(&full[0]), lead_rank);
    uint32_t it = 0;
    for (int x = pair; x < ntiles; x += npairs) {
      int tm, tn;
      tile_mn(x, tm, tn);
      const int ta = 2 * tm + static_cast<int>(rank);
      int am0[MAXR], bn0[MAXR], bn1[MAXR], ka[MAXR], kb[MAXR], dig[MAXKD];
#pragma unroll
      for (int r = 0; r < MAXR; ++r) {
        am0[r] = g.a_mc[ta * MAXR + r];
        bn0[r] = g.b_nc[tn * MAXR + r] + (r == b_row_rank ? static_cast<int>(rank) * (BN / 2) : 0);
        if (WIDE) bn1[r] = g.b_nc[(tn + 1) * MAXR + r] + (r == b_row_rank ? static_cast<int>(rank) * (BN / 2) : 0);
        ka[r] = g.ka0[r];
        kb[r] = g.kb0[r];
      }
#pragma unroll
      for (int q = 0; q < MAXKD; ++q) dig[q] = 0;
      for (int kt = 0; kt < g.nk; ++kt, ++it) {
        const uint32_t s = it % STAGES;
        if (it >= STAGES) tc::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        if (leader) tc::mbar_arrive_expect_tx(&full[s], 2 * (A_BYTES + NH * B_BYTES));
        const uint32_t fb = full_leader0 + s * 8;
        int c[MAXR];
#pragma unroll
        for (int r = 0; r < MAXR; ++r) c[r] = am0[r] + ka[r];
        if (MC) {  // half pp of this CTA's A rows, into this CTA and its twin in the other pair
          c[1] += pp * (BM / 2);
          tma_load_2sm_mc(sA + s * A_BYTES + pp * (A_BYTES / 2), &tma_a, fb,
                          static_cast<uint16_t>((1u << crank) | (1u << (crank ^ 2u))), c);
        } else {
          tma_load_2sm(sA + s * A_BYTES, &tma_a, fb, g.a_rank, c);
        }
#pragma unroll
        for (int r = 0; r < MAXR; ++r) c[r] = bn0[r] + kb[r];
        if (B_MN) {  // MN-major B: this CTA's BN/2 columns as 32-column slabs (no layout pass)
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            if (h) {
#pragma unroll
              for (int r = 0; r < MAXR; ++r) c[r] = bn1[r] + kb[r];
            }
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) {
              int cj[MAXR];
#pragma unroll
              for (int r = 0; r < MAXR; ++r) cj[r] = c[r];
              cj[0] += 32 * j;
              tma_load_2sm(sB + (s * NH + h) * B_BYTES + j * (BKE * 128), &tma_b, fb, g.b_rank, cj);
            }
          }
        } else {
          tma_load_2sm(sB + s * NH * B_BYTES, &tma_b, fb, g.b_rank, c);
          if (WIDE) {
#pragma unroll
            for (int r = 0; r < MAXR; ++r) c[r] = bn1[r] + kb[r];
            tma_load_2sm(sB + s * NH * B_BYTES + B_BYTES, &tma_b, fb, g.b_rank, c);
          }
        }
        for (int q = g.nkd - 1; q >= 0; --q) {
          if (++dig[q] < g.kext[q]) {
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
              ka[r] += g.kca[q][r] * g.kstep[q];
              kb[r] += g.kcb[q][r] * g.kstep[q];
            }
            break;
          }
#pragma unroll
          for (int r = 0; r < MAXR; ++r) {
            ka[r] -= g.kca[q][r] * g.kstep[q] * (g.kext[q] - 1);
            kb[r] -= g.kcb[q][r] * g.kstep[q] * (g.kext[q] - 1);
          }
          dig[q] = 0;
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader only): M = 256 across the pair
    constexpr uint32_t idesc = tc::instr_desc(BF16 ? 1 : 2, 0, B_MN ? 1 : 0, 2 * BM, BN);
    uint32_t it = 0, tl = 0;
    for (int x = pair; x < ntiles; x += npairs, ++tl) {
      const uint32_t acc = WIDE ? 0u : tl & 1;
      if (!WIDE && tl >= 2) tc::mbar_wait_warp(&tempty[acc], ((tl / 2) - 1) & 1);
      tc::tc_fence_after();
      for (int kt = 0; kt < g.nk; ++kt, ++it) {
        const uint32_t s = it % STAGES;
        tc::mbar_wait_warp(&full[s], (it / STAGES) & 1);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(sA + s * A_BYTES);
#pragma unroll
        for (int k = 0; k < BKE / 8; ++k)
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          if (WIDE && kt == 0 && k == 0 && tl >= 1) {  // this half drained by the previous tile's epilogue
            tc::mbar_wait_warp(&tempty[h], (tl - 1) & 1);
            tc::tc_fence_after();
          }
          const uint32_t dtm = tmem + acc * BN + h * BN;
          const uint32_t sb = tc::smem_u32(sB + (s * NH + h) * B_BYTES);
          const uint64_t da = tc::sw128_desc(sa + k * 32, 16, 1024);
          const uint64_t db = B_MN ? tc::umma_desc(sb + k * 1024, BKE * 128, 512, 1) : tc::sw128_desc(sb + k * 32, 16, 1024);
          const uint32_t accum = (kt | k) != 0 ? 1u : 0u;
          if (BF16)
            asm volatile(
                "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtm), "l"(da), "l"(db), "r"(idesc),
                "r"(accum));
          else
            asm volatile(
                "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtm), "l"(da), "l"(db), "r"(idesc),
                "r"(accum));
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                     ::"r"(tc::smem_u32(&empty[s])), "h"(static_cast<uint16_t>(MC ? 0xF : 3)) : "memory");
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                   ::"r"(tc::smem_u32(&tfull[acc])), "h"(static_cast<uint16_t>(3u << lead_rank)) : "memory");
    }
  } else if (warp >= 2) {
    // ---------------- epilogue warps (both CTAs): own 128 TMEM lanes
    const int q = warp & 3;
    const uint32_t stg = tc::smem_u32(stage_base) + static_cast<uint32_t>(warp - 2) * (32 * 36 * 4 + 32 * 8);
    const uint32_t rtab = stg + 32 * 36 * 4;
    const uint32_t tempty_leader0 = peer_addr(tc::smem_u32(&tempty[0]), lead_rank);
    uint32_t tl = 0;
    for (int x = pair; x < ntiles; x += npairs, ++tl) {
      int tm, tn;
      tile_mn(x, tm, tn);
      const int ta = 2 * tm + static_cast<int>(rank);
      const uint32_t acc = WIDE ? 0u : tl & 1;
      tc::mbar_wait(&tfull[acc], (WIDE ? tl : tl / 2) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < NH; ++h) {
      const int64_t tbase = static_cast<int64_t>(g.tCm[ta]) + g.tCn[tn + h];
      if (h == 0) asm volatile("st.shared.s32 [%0], %1;" ::"r"(rtab + lane * 4), "r"(g.cm[q * 32 + lane]) : "memory");
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t rv[32];
        tc::tmem_ld32(tmem + (acc + h) * BN + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), rv);
        epi_block(rv, stg, rtab, g.C, tbase, g.cn, c0, lane, g.cvec != 0);
      }
      if (WIDE || h == NH - 1) {
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader0 + (acc + h) * 8) : "memory");
      }
      }
    }
  }
  tc::tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ---------------------------------------------------------------- host
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  if (!fn) fail("CudaError", "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// TMA description of one operand.
struct View {
  int buf = 0;
  int rank = 0;                       // TMA rank (= buffer rank)
  cuuint64_t dims[MAXR], strides[MAXR];  // innermost first; strides in bytes (strides[0] unused)
  cuuint32_t box[MAXR];
  std::vector<int> row_dims;          // smem row order (outer -> inner)
  std::vector<int64_t> row_box;
  bool mn = false;                    // MN-major (slabs of 32 along the inner row dim)
  bool bf16 = false;                  // packed bf16 operand (64 elements per 128-byte row)
  int swz_bytes = 128;                // row bytes of the swizzle (tail views: 32 / 64)
  int kin = -1;                       // the K dim stepped by 32 per k-tile
  std::vector<std::vector<int64_t>> coef;  // [TMA rank][dim]
  std::vector<int64_t> c0;            // [TMA rank]
};

// Describes operand `b` (buffer) as a TMA view. `rows` = its row dims
// (M for A, N for B), `K` = the contraction dims, `row_target` = BM or BN.
bool describe_view(const Problem& p, int b, const std::vector<int>& rows, const std::vector<int>& K,
                   int64_t row_target, bool allow_mn, View& v, std::string* why) {
  const MdHom& e = p.e;
  const Buf& buf = e.in[static_cast<size_t>(b)];
  const int R = buf.rank, D = e.D();
  if (R > MAXR) return *why = "rank > 5", false;
  v.buf = b;
  v.rank = R;
  v.coef.assign(static_cast<size_t>(R), std::vector<int64_t>(static_cast<size_t>(D), 0));
  v.c0.assign(static_cast<size_t>(R), 0);
  int64_t stride = 4;
  for (int t = 0; t < R; ++t) {  // t = TMA dim (innermost first), rank index R-1-t
    const Affine& f = buf.acc[0].idx[static_cast<size_t>(R - 1 - t)];
    v.dims[t] = static_cast<cuuint64_t>(p.in_ext[static_cast<size_t>(b)][static_cast<size_t>(R - 1 - t)]);
    v.strides[t] = static_cast<cuuint64_t>(stride);
    if (t > 0 && stride % 16) return *why = "TMA stride not a multiple of 16 bytes", false;
    stride *= static_cast<int64_t>(v.dims[t]);
    v.c0[static_cast<size_t>(t)] = f.c0;
    for (int d = 0; d < D; ++d) v.coef[static_cast<size_t>(t)][static_cast<size_t>(d)] = f.coeff[static_cast<size_t>(d)];
  }
  auto is_row = [&](int d) { return std::find(rows.begin(), rows.end(), d) != rows.end(); };
  auto is_k = [&](int d) { return std::find(K.begin(), K.end(), d) != K.end(); };
  // the inner TMA dim decides the majorness
  std::vector<int> inner;
  for (int d = 0; d < D; ++d)
    if (v.coef[0][static_cast<size_t>(d)] != 0) inner.push_back(d);
  if (inner.size() != 1 || v.coef[0][static_cast<size_t>(inner[0])] != 1) return *why = "inner rank is not a single unit-stride dim", false;
  int di = inner[0];
  // row dims per rank (at most one, coefficient 1)
  std::vector<int> rank_row(static_cast<size_t>(R), -1);
  for (int t = 0; t < R; ++t)
    for (int d = 0; d < D; ++d) {
      int64_t c = v.coef[static_cast<size_t>(t)][static_cast<size_t>(d)];
      if (c == 0) continue;
      if (is_row(d)) {
        if (c != 1 || rank_row[static_cast<size_t>(t)] >= 0) return *why = "row dim with non-unit coefficient or shared rank", false;
        rank_row[static_cast<size_t>(t)] = d;
      } else if (!is_k(d)) {
        return *why = "operand depends on a dim outside its row / K groups", false;
      }
    }
  for (int d : rows) {
    int cnt = 0;
    for (int t = 0; t < R; ++t) cnt += rank_row[static_cast<size_t>(t)] == d;
    if (cnt != 1) return *why = "row dim not in exactly one rank", false;
  }
  for (int t = 0; t < R; ++t) v.box[t] = 1;
  if (is_k(di)) {
    // K-major: box 32 along the inner K dim, row boxes (outer -> inner by rank)
    if (e.sizes[static_cast<size_t>(di)] % BKE) return *why = "inner K extent not a multiple of 32", false;
    v.mn = false;
    v.kin = di;
    v.box[0] = BKE;
    // factor the row target over the row ranks, innermost rank first
    int64_t rem = row_target;
    for (int t = 1; t < R; ++t) {
      int d = rank_row[static_cast<size_t>(t)];
      if (d < 0) continue;
      int64_t gcd = std::gcd(e.sizes[static_cast<size_t>(d)], rem);
      if (gcd > 256) gcd = 256;
      v.box[t] = static_cast<cuuint32_t>(gcd);
      rem /= gcd;
    }
    if (rem != 1) return *why = "row tile cannot be formed as a TMA box", false;
    for (int t = R - 1; t >= 1; --t)
      if (rank_row[static_cast<size_t>(t)] >= 0) {
        v.row_dims.push_back(rank_row[static_cast<size_t>(t)]);
        v.row_box.push_back(v.box[t]);
      }
  } else {
    // MN-major: inner rank = a row dim, 32-element slabs; K dim in another rank
    if (!allow_mn) return *why = "MN-major operand not supported here", false;
    if (rows.size() != 1 || rank_row[0] != di) return *why = "MN-major operand needs a single row dim", false;
    if (e.sizes[static_cast<size_t>(di)] % row_target || row_target % 32) return *why = "row tile does not split into slabs", false;
    int tk = -1;
    for (int t = 1; t < R; ++t)
      for (int d : K)
        if (v.coef[static_cast<size_t>(t)][static_cast<size_t>(d)] == 1 && e.sizes[static_cast<size_t>(d)] % BKE == 0) tk = t;
    if (tk < 0) return *why = "no K rank with unit coefficient", false;
    int kd = -1;
    for (int d : K)
      if (v.coef[static_cast<size_t>(tk)][static_cast<size_t>(d)] == 1) kd = d;
    v.mn = true;
    v.kin = kd;
    v.box[0] = 32;
    v.box[tk] = BKE;
    v.row_dims = {di};
    v.row_box = {row_target};
  }
  return true;
}

// coordinates (TMA order) of an origin given per-dim values
std::vector<int32_t> coords(const View& v, const std::vector<int64_t>& origin, bool with_c0) {
  std::vector<int32_t> c(MAXR, 0);
  for (int t = 0; t < v.rank; ++t) {
    int64_t x = with_c0 ? v.c0[static_cast<size_t>(t)] : 0;
    for (size_t d = 0; d < origin.size(); ++d) x += v.coef[static_cast<size_t>(t)][d] * origin[d];
    c[static_cast<size_t>(t)] = static_cast<int32_t>(x);
  }
  return c;
}

// Template parameters a Table-1 configuration sets (tc_knobs below):
// N tile, kernel form, M-tiles per raster group, K split, B layout pass.
struct TcKnobs {
  bool set = false;   // read from a configuration (else the planner's menu)
  int bn = 0;         // N tile = RM parts of the N dim
  int form = -1;      // 0 one CTA per tile, 1 persistent CTAs (DM parts of M > 1), 2 CTA pair (256-row tiles)
  int group = 0;      // M tiles per raster group = SMX parts of M (persistent forms), 0 = 8
  int split = 1;      // K split = SMX parts of K (SMXs combine in DM: ordered reduction)
  int transpose = -1; // B rewritten K-major (layout_de of B = [2, 1]) 1, read as stored 0
  bool rbn = false;   // DM parts of N = every N tile: one-CTA tiles with B resident per CTA
};

// split-K combine: C += ws[0] + ws[1] + ... in split order (the k order of
// the unsplit fold)
__global__ void splitk_reduce(float* __restrict__ C, const float* __restrict__ ws, int parts, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = C[i];
    for (int s = 0; s < parts; ++s) acc += ws[static_cast<int64_t>(s) * n + i];
    C[i] = acc;
  }
}

class TcRoutine final : public Routine {
 public:
  TcRoutine(const Problem& p, const Groups& g, const TcKnobs& k = {}) : p_(p), g_(g), kn_(k) {}
  ~TcRoutine() override {
    if (ws_) cudaFree(ws_);
    if (blob_) cudaFree(blob_);
    if (bt_) cudaFree(bt_);
    if (pa_) cudaFree(pa_);
    if (pb_) cudaFree(pb_);
  }
  const char* family() const override { return "contraction"; }
  const char* bound() const override { return "tensor"; }
  int launches() const override {
    return (packed_ ? 3 : (transposeB_ ? 2 : 1)) + (kn_.split > 1 ? kn_.split : 0);
  }
  double flops() const override { return 2.0 * static_cast<double>(M_) * static_cast<double>(N_) * static_cast<double>(K_); }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  std::string describe() const override {
    std::ostringstream os;
 os << "{\"kernel\": \"" << (two_sm_ ? "tc_gemm_2sm<" : pers_ ? "tc_gemm_pers<" : "tc_gemm_tf32<") << (wide_ ? 2 * BN_ : BN_) << ","
       << (two_sm_ ? st2_ : pers_ ? pstages_ : stages_) << ","
       << (va_.mn ? "A_MN" : "A_K") << "," << (vb_.mn ? "B_MN" : "B_K") << (rb_ && pers_ ? ",B_RESIDENT" : "")
       << ">\", \"math\": \"" << (bf16_ ? "bf16" : "tf32") << "\", \"M\": " << M_ << ", \"N\": " << N_ << ", \"K\": " << K_
       << ", \"BM\": " << BM << ", \"BN\": " << (wide_ ? 2 * BN_ : BN_) << ", \"BK\": " << BKE << ", \"stages\": " << stages_
       << ", \"umma\": \"tcgen05.mma.cta_group::1.kind::" << (bf16_ ? "f16 (bf16) M128xN" : "tf32 M128xN") << BN_
       << (bf16_ ? "xK16" : "xK8") << "\", \"tiles\": "
       << static_cast<int64_t>(tilesM_) * tilesN_ << ", \"tmem_cols\": " << (wide_ ? 2 * BN_ : BN_)
       << ", \"b_layout\": \"" << (packed_ ? "packed K-major (pack_kmajor pre-pass, both operands)" : transposeB_ ? "K-major copy (layout_de [2,1] pre-pass)" : (vb_.mn ? "MN-major" : "K-major"))
       << "\"";
    if (packed_) os << ", \"K_padded\": " << Kp_;
    if (two_sm_) os << ", \"cta_pair\": \"tc_gemm_2sm<" << BN_ << "," << st2_ << ">: tcgen05.mma.cta_group::2 M256xN" << BN_ << (bf16_ ? "xK16 (bf16)" : "xK8") << "\"";
    if (wide_) os << ", \"wide\": \"256 x " << 2 * BN_ << " pair tiles: two N" << BN_ << " MMAs per k-step share one A landing, TMEM 512 columns single-buffered\"";
    if (mc_) os << ", \"a_multicast\": \"clusters of 4 (two pairs on adjacent N tiles), A halves multicast\", \"clusters\": " << mc_clusters_;
    os << ", \"raster_group_m\": " << (args_.group_m > 0 ? args_.group_m : 8) << ", \"k_split\": " << kn_.split
       << ", \"from_config\": " << (kn_.set ? "true" : "false");
    os << "}";
    return os.str();
  }

  bool setup(int BN, std::string* why) {
    const MdHom& e = p_.e;
    M_ = prod_sizes(e, g_.Md);
    N_ = prod_sizes(e, g_.Nd);
    K_ = prod_sizes(e, g_.Kd);
    std::string w;
    bf16_ = p_.opt.math == Math::BF16;
    if (bf16_) return setup_packed(BN, why);  // operands converted + packed (layout_de) for kind::f16
    if (!describe_view(p_, g_.a_buf, g_.Md, g_.Kd, BM, false, va_, &w) ||
        !describe_view(p_, g_.b_buf, g_.Nd, g_.Kd, BN, true, vb_, &w) || va_.kin != vb_.kin) {
      if (setup_packed(BN, why)) return true;
      *why = w + "; packed: " + *why;
      return false;
    }
    if (vb_.mn && g_.Nd.size() == 1 && g_.Kd.size() == 1 && !std::getenv("MDHB_TC_NO_TRANSPOSE") && kn_.transpose != 0) {
      // rewrite B K-major into scratch: Bt[n][k]
      const int dn = g_.Nd[0], dk = g_.Kd[0];
      const int64_t Nn = e.sizes[static_cast<size_t>(dn)], Kk = e.sizes[static_cast<size_t>(dk)];
      if (Kk % BKE == 0 && Nn % BN == 0) {
        View t;
        t.buf = vb_.buf;
        t.rank = 2;
        t.dims[0] = static_cast<cuuint64_t>(Kk);
        t.dims[1] = static_cast<cuuint64_t>(Nn);
        t.strides[0] = 4;
        t.strides[1] = static_cast<cuuint64_t>(Kk * 4);
        t.box[0] = BKE;
        t.box[1] = static_cast<cuuint32_t>(BN);
        t.coef.assign(2, std::vector<int64_t>(static_cast<size_t>(e.D()), 0));
        t.coef[0][static_cast<size_t>(dk)] = 1;
        t.coef[1][static_cast<size_t>(dn)] = 1;
        t.c0 = {0, 0};
        t.mn = false;
        t.kin = dk;
        t.row_dims = {dn};
        t.row_box = {BN};
        if (BN > 256 || t.strides[1] % 16) return *why = "transposed view not TMA-able", false;
        vb_ = t;
        transposeB_ = true;
        tK_ = Kk;
        tN_ = Nn;
        MDHB_CUDA(cudaMalloc(&bt_, static_cast<size_t>(Kk * Nn) * 4));
      }
    }
    if (va_.kin != vb_.kin) return *why = "operands step different K dims", false;
    BN_ = BN;
    stages_ = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
    // row tiles: boxes over the row dims in the views' smem order
    auto tiles = [&](const View& v, std::vector<std::vector<int64_t>>& origins) {
      std::vector<int64_t> gext;
      for (size_t q = 0; q < v.row_dims.size(); ++q) {
        int64_t n = e.sizes[static_cast<size_t>(v.row_dims[q])];
        if (n % v.row_box[q]) return false;
        gext.push_back(n / v.row_box[q]);
      }
      int64_t cnt = 1;
      for (auto x : gext) cnt *= x;
      std::vector<int64_t> l(gext.size(), 0);
      for (int64_t t = 0; t < cnt; ++t) {
        std::vector<int64_t> o(static_cast<size_t>(e.D()), 0);
        for (size_t q = 0; q < l.size(); ++q) o[static_cast<size_t>(v.row_dims[q])] = l[q] * v.row_box[q];
        origins.push_back(o);
        for (int q = static_cast<int>(l.size()) - 1; q >= 0; --q) {
          if (++l[static_cast<size_t>(q)] < gext[static_cast<size_t>(q)]) break;
          l[static_cast<size_t>(q)] = 0;
        }
      }
      return true;
    };
    std::vector<std::vector<int64_t>> om, on;
    if (!tiles(va_, om) || !tiles(vb_, on)) return *why = "row tiles do not divide", false;
    tilesM_ = static_cast<int>(om.size());
    tilesN_ = static_cast<int>(on.size());
    // k-tiles: the K dims (kin stepped by 32, the rest by 1), kin innermost
    std::vector<int> kd;
    std::vector<int64_t> kext, kstep;
    for (int d : g_.Kd)
      if (d != va_.kin) {
        kd.push_back(d);
        kext.push_back(e.sizes[static_cast<size_t>(d)]);
        kstep.push_back(1);
      }
    kd.push_back(va_.kin);
    kext.push_back(e.sizes[static_cast<size_t>(va_.kin)] / BKE);
    kstep.push_back(BKE);
    nk_ = static_cast<int>(K_ / BKE);
    if (kd.size() > static_cast<size_t>(MAXKD)) return *why = "more than 6 contraction dims", false;
    args_.nkd = static_cast<int>(kd.size());
    for (size_t q = 0; q < kd.size(); ++q) {
      args_.kext[q] = static_cast<int>(kext[q]);
      args_.kstep[q] = static_cast<int>(kstep[q]);
      for (int t = 0; t < MAXR; ++t) {
        args_.kca[q][t] = t < va_.rank ? static_cast<int>(va_.coef[static_cast<size_t>(t)][static_cast<size_t>(kd[q])]) : 0;
        args_.kcb[q][t] = t < vb_.rank ? static_cast<int>(vb_.coef[static_cast<size_t>(t)][static_cast<size_t>(kd[q])]) : 0;
      }
    }
    // epilogue tables in the smem row orders of A (TMEM lanes) and B (columns)
    std::vector<int64_t> tCm, tCn, cm, cn;
    for (auto& o : om) {
      int64_t x = g_.lc.c0;
      for (int d = 0; d < e.D(); ++d) x += g_.lc.cj[static_cast<size_t>(d)] * o[static_cast<size_t>(d)];
      tCm.push_back(x);
    }
    for (auto& o : on) {
      int64_t x = 0;
      for (int d = 0; d < e.D(); ++d) x += g_.lc.cj[static_cast<size_t>(d)] * o[static_cast<size_t>(d)];
      tCn.push_back(x);
    }
    std::vector<int64_t> ones_m(va_.row_dims.size(), 1), ones_n(vb_.row_dims.size(), 1);
    cm = box_offsets(va_.row_dims, va_.row_box, g_.lc.cj, ones_m);
    cn = box_offsets(vb_.row_dims, vb_.row_box, g_.lc.cj, ones_n);
    auto mod4 = [](const std::vector<int64_t>& v) {
      for (auto x : v)
        if (x % 4) return false;
      return true;
    };
    bool grp = cn.size() % 4 == 0;
    for (size_t t = 0; grp && t < cn.size(); t += 4)
      for (size_t j = 1; j < 4; ++j) grp = grp && cn[t + j] == cn[t] + static_cast<int64_t>(j);
    cvec_ = grp && mod4(cn) && mod4(cm) && mod4(tCm) && mod4(tCn);
    c_run_ = run_of(cn);
    // coordinate tables
    std::vector<int64_t> amc, bnc;
    for (auto& o : om) for (auto c : coords(va_, o, true)) amc.push_back(c);
    for (auto& o : on) for (auto c : coords(vb_, o, true)) bnc.push_back(c);
    const std::vector<int64_t>* ts[6] = {&tCm, &tCn, &cm, &cn, &amc, &bnc};
    size_t total = 0;
    for (auto* t : ts) total += (t->size() + 64) / 64 * 64;
    std::vector<int32_t> host(total, 0);
    size_t cur = 0, offs[6];
    for (int q = 0; q < 6; ++q) {
      offs[q] = cur;
      for (int64_t x : *ts[q]) {
        if (x > INT32_MAX || x < INT32_MIN) return *why = "offsets exceed int32", false;
        host[cur++] = static_cast<int32_t>(x);
      }
      cur = (cur + 64) / 64 * 64;
    }
    MDHB_CUDA(cudaSetDevice(p_.opt.device));
    MDHB_CUDA(cudaMalloc(&blob_, std::max<size_t>(cur, 64) * 4));
    MDHB_CUDA(cudaMemcpy(blob_, host.data(), cur * 4, cudaMemcpyHostToDevice));
    const int32_t* base = static_cast<const int32_t*>(blob_);
    args_.tCm = base + offs[0];
    args_.tCn = base + offs[1];
    args_.cm = base + offs[2];
    args_.cn = base + offs[3];
    args_.a_mc = base + offs[4];
    args_.b_nc = base + offs[5];
    args_.a_rank = va_.rank;
    args_.b_rank = vb_.rank;
    args_.nk = nk_;
    args_.tilesM = tilesM_;
    args_.tilesN = tilesN_;
    args_.cvec = cvec_ && !std::getenv("MDHB_TC_EPI32");  // dev aid: the one-row-per-store epilogue
    smem_ = static_cast<size_t>(stages_) * (BM + BN) * BKE * 4 + 1024 + 256;
    // persistent instance: resident B when the single N tile's K extent fits
    auto rb_need = [&](int st) { return static_cast<size_t>(nk_) * BN * BKE * 4 + st * BM * BKE * 4 + 1024 + 256 + epi_bytes(true, BN); };
    const int rb_st = rb_need(4) <= 227 * 1024 ? 4 : 3;
    const size_t rb_bytes = rb_need(rb_st);
    rb_ = tilesN_ == 1 && !vb_.mn && (BN == 64 || BN == 128) && rb_bytes <= 227 * 1024;
    pstages_ = rb_ ? rb_st : pers_stages(BN);
    psmem_ = rb_ ? rb_bytes : static_cast<size_t>(pstages_) * (BM + BN) * BKE * 4 + 1024 + 256 + epi_bytes(false, BN);
    decide_rb_multi(BN);
    pers_ = !std::getenv("MDHB_TC_NONPERSISTENT");
    return finish_knobs(why);
  }

  // The configuration's knobs on top of the instance: kernel form, raster
  // group, K split (workspace for the partials)
  bool finish_knobs(std::string* why) {
    if (kn_.set) {
      pers_ = kn_.form >= 1;
      if (kn_.transpose == 1 && vb_.mn && !transposeB_) return *why = "K-major B copy unavailable", false;
    }
    decide_2sm();
    if (kn_.set && (kn_.form == 2) != two_sm_) return *why = "CTA-pair instance unavailable for this tile", false;
    if (kn_.set && (kn_.bn == 512) != wide_) return *why = "256 x 512 CTA-pair tile unavailable (K-major B, N % 512)", false;
    if (kn_.set && kn_.rbn != (rb_ && tilesN_ > 1)) return *why = "resident-B instance unavailable (BN 192, K-major B, smem)", false;
    if (!pers_ && BN_ == 192) return *why = "no one-CTA-per-tile instance with BN 192", false;
    if (!pers_ && bf16_) return *why = "no one-CTA-per-tile kind::f16 instance", false;
    args_.group_m = kn_.group;
    // 256 x 512 pair tiles: raster groups of 16 row tiles (1% over 8 at 8192^3)
    if (!kn_.set && wide_ && (tilesM_ / 2) % 16 == 0) args_.group_m = 16;
    if (const char* f = std::getenv("MDHB_TC_GROUP")) args_.group_m = std::atoi(f);  // dev aid
    if (kn_.split > 1) {
      if (args_.kext[0] % kn_.split) return *why = "K split does not divide the outer K digit", false;
      int64_t n = 1;
      for (int64_t x : p_.out_ext[0]) n *= x;
      ws_n_ = n;
      MDHB_CUDA(cudaMalloc(&ws_, static_cast<size_t>(n) * static_cast<size_t>(kn_.split - 1) * sizeof(float)));
    }
    return true;
  }

  // Packed-operand instance: both operands gathered K-major into scratch in
  // tile order (pack_kmajor), so any view the contraction family accepts
  // reaches the tensor cores; C is written through the FFMA template's tables.
  bool setup_packed(int BN, std::string* why) {
    const MdHom& e = p_.e;
    std::vector<int64_t> Tm = factor_box(e, g_.Md, BM), Tn = factor_box(e, g_.Nd, BN);
    if (Tm.empty() || Tn.empty()) return *why = "row tiles cannot be formed", false;
    const int ek = bf16_ ? 2 * BKE : BKE;  // elements per 128-byte k-tile row
    const int esz = bf16_ ? 2 : 4;
    Kp_ = (K_ + ek - 1) / ek * ek;
    // K tail: the last k-step as 32- / 64-byte rows instead of a padded
    // 128-byte one (persistent one-CTA instances, BN 64 / 192)
    int tail_bytes = 0;
    // (TF32: 163-164 vs 166 us on CCSD(T); BF16 within noise, so opt-in there
    // with MDHB_TC_KTAIL=1)
    if (K_ % ek && K_ > ek && (BN == 192 || BN == 64) && !std::getenv("MDHB_TC_NO_KTAIL") && !std::getenv("MDHB_TC_NONPERSISTENT") &&
        !(kn_.set && kn_.form == 0) && (!bf16_ || std::getenv("MDHB_TC_KTAIL"))) {
      const int64_t rem = (K_ % ek) * esz;
      tail_bytes = rem <= 32 ? 32 : rem <= 64 ? 64 : 0;
      if (tail_bytes) Kp_ = K_ / ek * ek + tail_bytes / esz;
    }
    if ((M_ + N_) * Kp_ * esz > (int64_t(1) << 30)) return *why = "packed operands exceed 1 GiB", false;
    auto ones = [](size_t n) { return std::vector<int64_t>(n, 1); };
    auto grid_of = [&](const std::vector<int>& dims, const std::vector<int64_t>& T, std::vector<int64_t>& gext) {
      for (size_t q = 0; q < dims.size(); ++q) gext.push_back(e.sizes[static_cast<size_t>(dims[q])] / T[q]);
    };
    std::vector<int64_t> gm, gn, fullK;
    grid_of(g_.Md, Tm, gm);
    grid_of(g_.Nd, Tn, gn);
    for (int d : g_.Kd) fullK.push_back(e.sizes[static_cast<size_t>(d)]);
    std::vector<int64_t> tAm = box_offsets(g_.Md, gm, g_.la.cj, Tm), tBn = box_offsets(g_.Nd, gn, g_.lb.cj, Tn);
    std::vector<int64_t> tCm = box_offsets(g_.Md, gm, g_.lc.cj, Tm), tCn = box_offsets(g_.Nd, gn, g_.lc.cj, Tn);
    std::vector<int64_t> am = box_offsets(g_.Md, Tm, g_.la.cj, ones(Tm.size())), bn = box_offsets(g_.Nd, Tn, g_.lb.cj, ones(Tn.size()));
    std::vector<int64_t> cm = box_offsets(g_.Md, Tm, g_.lc.cj, ones(Tm.size())), cn = box_offsets(g_.Nd, Tn, g_.lc.cj, ones(Tn.size()));
    std::vector<int64_t> ak = box_offsets(g_.Kd, fullK, g_.la.cj, ones(fullK.size())), bk = box_offsets(g_.Kd, fullK, g_.lb.cj, ones(fullK.size()));
    for (auto& v : tAm) v += g_.la.c0;
    for (auto& v : tBn) v += g_.lb.c0;
    for (auto& v : tCm) v += g_.lc.c0;
    tilesM_ = static_cast<int>(tAm.size());
    tilesN_ = static_cast<int>(tBn.size());
    BN_ = BN;
    stages_ = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
    nk_ = static_cast<int>((Kp_ + ek - 1) / ek);
    auto view2 = [&](int buf, int64_t rows_total, int box_rows) {
      View v;
      v.buf = buf;
      v.rank = 2;
      v.dims[0] = static_cast<cuuint64_t>(Kp_);
      v.dims[1] = static_cast<cuuint64_t>(rows_total);
      v.strides[0] = 4;
      v.strides[1] = static_cast<cuuint64_t>(Kp_ * esz);
      v.box[0] = static_cast<cuuint32_t>(ek);
      v.bf16 = bf16_;
      v.box[1] = static_cast<cuuint32_t>(box_rows);
      v.mn = false;
      return v;
    };
    va_ = view2(g_.a_buf, M_, BM);
    vb_ = view2(g_.b_buf, N_, BN);
    tail_ = tail_bytes > 0;
    args_.tail_bytes = tail_bytes;
    if (tail_) {
      vat_ = va_;
      vbt_ = vb_;
      vat_.box[0] = vbt_.box[0] = static_cast<cuuint32_t>(tail_bytes / esz);
      vat_.swz_bytes = vbt_.swz_bytes = tail_bytes;
    }
    args_.nkd = 1;
    args_.kext[0] = nk_;
    args_.kstep[0] = ek;
    for (int t = 0; t < MAXR; ++t) args_.kca[0][t] = args_.kcb[0][t] = t == 0 ? 1 : 0;
    std::vector<int64_t> amc, bnc;
    for (int t = 0; t < tilesM_; ++t) for (int r = 0; r < MAXR; ++r) amc.push_back(r == 1 ? int64_t(t) * BM : 0);
    for (int t = 0; t < tilesN_; ++t) for (int r = 0; r < MAXR; ++r) bnc.push_back(r == 1 ? int64_t(t) * BN : 0);
    bool grp = cn.size() % 4 == 0;
    for (size_t t = 0; grp && t < cn.size(); t += 4)
      for (size_t j = 1; j < 4; ++j) grp = grp && cn[t + j] == cn[t] + static_cast<int64_t>(j);
    auto mod4 = [](const std::vector<int64_t>& v) {
      for (auto x : v)
        if (x % 4) return false;
      return true;
    };
    cvec_ = grp && mod4(cn) && mod4(cm) && mod4(tCm) && mod4(tCn);
    c_run_ = run_of(cn);
    const std::vector<int64_t>* ts[12] = {&tCm, &tCn, &cm, &cn, &amc, &bnc, &tAm, &am, &ak, &tBn, &bn, &bk};
    size_t cur = 0, offs[12];
    std::vector<int32_t> host;
    for (int q = 0; q < 12; ++q) {
      offs[q] = cur;
      for (int64_t x : *ts[q]) {
        if (x > INT32_MAX || x < INT32_MIN) return *why = "offsets exceed int32", false;
        host.push_back(static_cast<int32_t>(x));
        ++cur;
      }
      while (cur % 64) host.push_back(0), ++cur;
    }
    MDHB_CUDA(cudaSetDevice(p_.opt.device));
    MDHB_CUDA(cudaMalloc(&blob_, std::max<size_t>(cur, 64) * 4));
    MDHB_CUDA(cudaMemcpy(blob_, host.data(), cur * 4, cudaMemcpyHostToDevice));
    const int32_t* base = static_cast<const int32_t*>(blob_);
    args_.tCm = base + offs[0];
    args_.tCn = base + offs[1];
    args_.cm = base + offs[2];
    args_.cn = base + offs[3];
    args_.a_mc = base + offs[4];
    args_.b_nc = base + offs[5];
    pk_ = {base + offs[6], base + offs[7], base + offs[8], base + offs[9], base + offs[10], base + offs[11]};
    args_.a_rank = 2;
    args_.b_rank = 2;
    args_.nk = nk_;
    args_.tilesM = tilesM_;
    args_.tilesN = tilesN_;
    args_.cvec = cvec_ && !std::getenv("MDHB_TC_EPI32");  // dev aid: the one-row-per-store epilogue
    MDHB_CUDA(cudaMalloc(&pa_, static_cast<size_t>(M_ * Kp_) * esz));
    MDHB_CUDA(cudaMalloc(&pb_, static_cast<size_t>(N_ * Kp_) * esz));
    // bf16 packing reads along the operand's unit-stride direction
    a_rowfast_ = am.size() > 1 && am[1] - am[0] == 1 && !(ak.size() > 1 && ak[1] - ak[0] == 1);
    b_rowfast_ = bn.size() > 1 && bn[1] - bn[0] == 1 && !(bk.size() > 1 && bk[1] - bk[0] == 1);
    // plain 2-D operands (global row r = t*rows + local at base + r*sr, k at k*sk):
    // vectorised convert (sk == 1) or 64x64 transposing convert (sr == 1)
    auto plain = [](const std::vector<int64_t>& toff, const std::vector<int64_t>& roff, const std::vector<int64_t>& koff,
                    int64_t& base, int64_t& sr, int64_t& sk) {
      if (roff.size() < 2 || koff.size() < 2) return false;
      base = toff[0] + roff[0];
      sr = roff[1] - roff[0];
      sk = koff[1] - koff[0];
      const int64_t rows = static_cast<int64_t>(roff.size());
      for (size_t r = 0; r < roff.size(); ++r)
        if (roff[r] != roff[0] + static_cast<int64_t>(r) * sr) return false;
      for (size_t t = 0; t < toff.size(); ++t)
        if (toff[t] + roff[0] != base + static_cast<int64_t>(t) * rows * sr) return false;
      for (size_t k = 0; k < koff.size(); ++k)
        if (koff[k] != static_cast<int64_t>(k) * sk) return false;
      return true;
    };
    auto mode = [&](const std::vector<int64_t>& toff, const std::vector<int64_t>& roff, const std::vector<int64_t>& koff,
                    PlainPack& pp) {
      int64_t base, sr, sk;
      pp.kind = 0;
      if (!bf16_ || !plain(toff, roff, koff, base, sr, sk)) return;
      if (sk == 1 && K_ % 8 == 0 && base % 4 == 0 && sr % 4 == 0) pp = {1, base, sr};
      else if (sr == 1 && base % 4 == 0 && sk % 4 == 0) pp = {2, base, sk};
    };
    mode(tAm, am, ak, ppa_);
    mode(tBn, bn, bk, ppb_);
    packed_ = true;
    smem_ = static_cast<size_t>(stages_) * (BM + BN) * BKE * 4 + 1024 + 256;
    rb_ = false;
    pstages_ = pers_stages(BN);
    psmem_ = static_cast<size_t>(pstages_) * (BM + BN) * BKE * 4 + 1024 + 256 + epi_bytes(false, BN);
    decide_rb_multi(BN);
    pers_ = !std::getenv("MDHB_TC_NONPERSISTENT");
    return finish_knobs(why);
  }

  // Many N tiles: each CTA keeps one N tile of B resident and walks M tiles,
  // so only A crosses from L2 per tile -- when the N tiles spread over the
  // SMs with little idle (CCSD(T): 72 tiles x 2 CTAs of 148 SMs)
  void decide_rb_multi(int BN) {
    if (rb_ || tilesN_ <= 1 || BN != 192 || vb_.mn) return;
    int lanes;
    if (kn_.set) {
      if (!kn_.rbn || kn_.group <= 0 || tilesM_ % kn_.group) return;
      lanes = tilesM_ / kn_.group;
    } else {
      if (std::getenv("MDHB_TC_NO_RBN")) return;
      const int sms = sm_count(p_.opt.device);
      lanes = sms / tilesN_;
      while (lanes > 1 && tilesM_ % lanes) --lanes;
      if (lanes < 1 || tilesM_ < 4 * lanes || (sms - lanes * tilesN_) * 16 > sms) return;
    }
    auto need = [&](int st) { return static_cast<size_t>(nk_) * BN * BKE * 4 + st * BM * BKE * 4 + 1024 + 256 + epi_bytes(true, BN); };
    int st = 4;  // 5: same time, 7: slower (CCSD(T))
    while (st > 3 && need(st) > 227 * 1024) --st;
    if (need(st) > 227 * 1024) return;
    rb_ = true;
    rbn_lanes_ = lanes;
    pstages_ = st;
    psmem_ = need(st);
  }

  // CTA-pair instance: K-major B whose tile rows live in one TMA rank (the
  // half-box split), an even number of 128-row tiles, BN 128 / 256
  void decide_2sm() {
    two_sm_ = false;
    if (std::getenv("MDHB_TC_1SM") || !pers_ || rb_ || (BN_ != 256 && BN_ != 128) || tilesM_ % 2) return;
    if (kn_.set && kn_.form != 2) return;
    if (vb_.mn) {
      // MN-major B (TF32, no layout pass): 32-column slabs, this CTA's half
      // of the N tile from column rank * BN / 2 of the innermost TMA dim
      if (bf16_ || vb_.box[0] != 32 || BN_ != 256 || std::getenv("MDHB_TC_2SM_NO_MN")) return;
      b_row_rank_ = 0;
      vb2_ = vb_;
      st2_ = 6;
      smem2_ = static_cast<size_t>(st2_) * (BM + BN_ / 2) * BKE * 4 + 1024 + 256 + 4 * (32 * 36 * 4 + 32 * 8);
      two_sm_ = smem2_ <= 227 * 1024;
      // 256 x 512 pair tiles reading B MN-major (dev aid)
      wide_ = two_sm_ && tilesN_ % 2 == 0 && (kn_.set ? kn_.bn == 512 : std::getenv("MDHB_TC_WIDE_MN") != nullptr);
      if (wide_) {
        st2_ = 4;
        smem2_ = static_cast<size_t>(st2_) * (BM + BN_) * BKE * 4 + 1024 + 256 + 4 * (32 * 36 * 4 + 32 * 8);
      }
      return;
    }
    int row_rank = -1;
    for (int t = 1; t < vb_.rank; ++t) {
      if (vb_.box[t] == static_cast<cuuint32_t>(BN_)) {
        if (row_rank >= 0) return;
        row_rank = t;
      } else if (vb_.box[t] != 1) {
        return;
      }
    }
    if (row_rank < 0) return;
    b_row_rank_ = row_rank;
    vb2_ = vb_;
    vb2_.box[row_rank] = static_cast<cuuint32_t>(BN_ / 2);
    st2_ = BN_ == 256 ? 6 : 8;
    smem2_ = static_cast<size_t>(st2_) * (BM + BN_ / 2) * BKE * 4 + 1024 + 256 + 4 * (32 * 36 * 4 + 32 * 8);
    two_sm_ = smem2_ <= 227 * 1024;
    // clusters of two pairs sharing A by multicast (plain 2-D A views)
    mc_ = two_sm_ && BN_ == 256 && tilesN_ % 2 == 0 && va_.rank == 2 && va_.row_dims.size() <= 1 && va_.box[1] == BM &&
          std::getenv("MDHB_TC_MC") != nullptr;
    if (mc_) {
      vaH_ = va_;
      vaH_.box[1] = BM / 2;
    }
    // 256 x 512 pair tiles (two adjacent N tiles, one A landing per k-step):
    // the default wherever they divide N; a configuration picks it by RM
    // parts of N = 512
    wide_ = two_sm_ && !mc_ && BN_ == 256 && tilesN_ % 2 == 0 &&
            (kn_.set ? kn_.bn == 512 : std::getenv("MDHB_TC_NARROW") == nullptr);
    if (wide_) {
      st2_ = 4;
      smem2_ = static_cast<size_t>(st2_) * (BM + BN_) * BKE * 4 + 1024 + 256 + 4 * (32 * 36 * 4 + 32 * 8);
      if (smem2_ > 227 * 1024) wide_ = false;
    }
    if (!wide_ && two_sm_) smem2_ = static_cast<size_t>(st2_) * (BM + BN_ / 2) * BKE * 4 + 1024 + 256 + 4 * (32 * 36 * 4 + 32 * 8);
  }
  bool packed() const { return packed_; }
  // the knobs of the planner's default instance (for its canonical config)
  bool knobs_default(TcKnobs* k) const {
    k->set = true;
    k->form = two_sm_ ? 2 : pers_ ? 1 : 0;
    k->bn = wide_ ? 2 * BN_ : BN_;
    k->group = k->form == 0 ? (two_sm_ ? tilesM_ / 2 : tilesM_) : (wide_ && (tilesM_ / 2) % 16 == 0 ? 16 : 8);
    k->rbn = rb_ && tilesN_ > 1 && pers_;
    if (k->rbn) k->group = tilesM_ / rbn_lanes_;
    else if (k->form != 0 && (two_sm_ ? tilesM_ / 2 : tilesM_) % 8) return false;
    k->split = 1;
    k->transpose = bf16_ ? -1 : (transposeB_ ? 1 : 0);
    return true;
  }
  int64_t c_run() const { return c_run_; }
  static int64_t run_of(const std::vector<int64_t>& cn) {
    int64_t n = 1;
    while (n < static_cast<int64_t>(cn.size()) && cn[static_cast<size_t>(n)] == cn[0] + n) ++n;
    return n;
  }
  // ring depth of the persistent kernel (fits 227 KB with the epilogue staging)
  static int pers_stages(int BN) { return BN >= 192 ? 4 : (BN >= 128 ? 5 : 6); }

  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    const void* A = d_in[va_.buf];
    const void* B = d_in[vb_.buf];
    if (packed_ && bf16_) {
      const int sms = sm_count(p_.opt.device);
      auto pack = [&](const void* src, void* dst, const int32_t* t, const int32_t* r, const int32_t* k, int rows, int64_t n_rows,
                      bool rowfast) {
        if (rowfast) {
          dim3 g(static_cast<unsigned>((Kp_ + 31) / 32), static_cast<unsigned>((n_rows + 31) / 32));
          pack_rows<uint16_t><<<g, 256, 0, s>>>(static_cast<const float*>(src), static_cast<uint16_t*>(dst), t, r, k, rows,
                                                 static_cast<int>(K_), static_cast<int>(Kp_), n_rows);
        } else {
          const int64_t tot = n_rows * Kp_;
          pack_kmajor_bf16<<<static_cast<unsigned>(std::min<int64_t>(8 * sms, (tot + 255) / 256)), 256, 0, s>>>(
              static_cast<const float*>(src), static_cast<uint16_t*>(dst), t, r, k, rows, static_cast<int>(K_),
              static_cast<int>(Kp_), tot);
        }
        MDHB_CUDA(cudaGetLastError());
      };
      auto plain_pack = [&](const void* src, void* dst, const PlainPack& pp, int64_t n_rows) {
        const float* base = static_cast<const float*>(src) + pp.base;
        if (pp.kind == 1) {
          const int64_t tot = n_rows * (Kp_ / 8);
          convert_kvec_bf16<<<static_cast<unsigned>(std::min<int64_t>(8 * sms, (tot + 255) / 256)), 256, 0, s>>>(
              base, pp.stride, static_cast<uint16_t*>(dst), static_cast<int>(K_), static_cast<int>(Kp_), n_rows);
        } else {
          dim3 g(static_cast<unsigned>((n_rows + 63) / 64), static_cast<unsigned>((Kp_ + 63) / 64));
          transpose64<__nv_bfloat16><<<g, 256, 0, s>>>(base, pp.stride, static_cast<__nv_bfloat16*>(dst), static_cast<int>(K_),
                                                       static_cast<int>(n_rows), static_cast<int>(Kp_));
        }
        MDHB_CUDA(cudaGetLastError());
      };
      if (ppa_.kind) plain_pack(A, pa_, ppa_, M_);
      else pack(A, pa_, pk_[0], pk_[1], pk_[2], BM, M_, a_rowfast_);
      if (ppb_.kind) plain_pack(B, pb_, ppb_, N_);
      else pack(B, pb_, pk_[3], pk_[4], pk_[5], BN_, N_, b_rowfast_);
      A = pa_;
      B = pb_;
    } else if (packed_) {
      const int sms = sm_count(p_.opt.device);
      // rows unit-stride (CCSD(T)'s A[g][d][a][b] along b): 32 x 32 blocks
      // through shared memory, reads along rows and writes along k; else
      // k-fast gathers
      auto pack = [&](const void* src, void* dst, const int32_t* t, const int32_t* r, const int32_t* k, int rows, int64_t n_rows,
                      bool rowfast) {
        if (rowfast && !std::getenv("MDHB_TC_NO_ROWPACK")) {
          dim3 g(static_cast<unsigned>((Kp_ + 31) / 32), static_cast<unsigned>((n_rows + 31) / 32));
          pack_rows<float><<<g, 256, 0, s>>>(static_cast<const float*>(src), static_cast<float*>(dst), t, r, k, rows,
                                              static_cast<int>(K_), static_cast<int>(Kp_), n_rows);
        } else {
          const int64_t tot = n_rows * Kp_;
          pack_kmajor<<<static_cast<unsigned>(std::min<int64_t>(8 * sms, (tot + 255) / 256)), 256, 0, s>>>(
              static_cast<const float*>(src), static_cast<float*>(dst), t, r, k, rows, static_cast<int>(K_),
              static_cast<int>(Kp_), tot);
        }
        MDHB_CUDA(cudaGetLastError());
      };
      pack(A, pa_, pk_[0], pk_[1], pk_[2], BM, M_, a_rowfast_);
      pack(B, pb_, pk_[3], pk_[4], pk_[5], BN_, N_, b_rowfast_);
      A = pa_;
      B = pb_;
    }
    if (transposeB_) {
      const float* src = static_cast<const float*>(B) + g_.lb.c0;
      const int64_t sk = g_.lb.cj[static_cast<size_t>(g_.Kd[0])], sn = g_.lb.cj[static_cast<size_t>(g_.Nd[0])];
      if (sn == 1 && sk % 4 == 0 && g_.lb.c0 % 4 == 0 && tN_ % 4 == 0) {
        dim3 tg(static_cast<unsigned>((tN_ + 63) / 64), static_cast<unsigned>((tK_ + 63) / 64));
        transpose64<float><<<tg, 256, 0, s>>>(src, sk, static_cast<float*>(bt_), static_cast<int>(tK_), static_cast<int>(tN_),
                                              static_cast<int>(tK_));
      } else {
        dim3 tg(static_cast<unsigned>((tN_ + 31) / 32), static_cast<unsigned>((tK_ + 31) / 32));
        transpose_kn<<<tg, 256, 0, s>>>(src, sk, sn, static_cast<float*>(bt_), static_cast<int>(tK_), static_cast<int>(tN_));
      }
      MDHB_CUDA(cudaGetLastError());
      B = bt_;
    }
    if (A != last_a_) {
      encode(mc_ ? vaH_ : va_, A, &ma_);
      if (tail_) encode(vat_, A, &mat_);
      last_a_ = A;
    }
    if (B != last_b_) {
      encode(vb_, B, &mb_);
      if (tail_) encode(vbt_, B, &mbt_);
      if (two_sm_) encode(vb2_, B, &mb2_);
      last_b_ = B;
    }
    MarkScope mark(this, s);  // the GEMM kernel(s) below are the dominant ones
    float* C = static_cast<float*>(d_out[0]);
    const int S = kn_.split;
    for (int sp = 0; sp < S; ++sp) {
      TcArgs a = args_;
      a.C = sp == 0 ? C : static_cast<float*>(ws_) + static_cast<int64_t>(sp - 1) * ws_n_;
      if (S > 1) {  // split sp: the outer K digit's range [sp, sp + 1) * kext / S
        const int part = args_.kext[0] / S;
        a.kext[0] = part;
        a.nk = args_.nk / S;
        for (int r = 0; r < MAXR; ++r) {
          a.ka0[r] = args_.kca[0][r] * args_.kstep[0] * part * sp;
          a.kb0[r] = args_.kcb[0][r] * args_.kstep[0] * part * sp;
        }
      }
      launch_gemm(a, s);
    }
    if (S > 1) {
      splitk_reduce<<<4 * sm_count(p_.opt.device), 256, 0, s>>>(C, static_cast<const float*>(ws_), S - 1, ws_n_);
      MDHB_CUDA(cudaGetLastError());
    }
  }

  void launch_gemm(TcArgs& a, cudaStream_t s) {
    if (two_sm_ && mc_) {
      cudaLaunchConfig_t lc = {};
      lc.blockDim = dim3(64 + 32 * 4);
      lc.dynamicSmemBytes = smem2_;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 4;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      void (*k)(const CUtensorMap, const CUtensorMap, TcArgs, int) =
          bf16_ ? tc_gemm_2sm<256, 6, true, false, true> : tc_gemm_2sm<256, 6, false, false, true>;
      MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2_)));
      if (!mc_clusters_) {  // co-resident clusters of 4 (GPC-limited, fewer than SMs / 4)
        lc.gridDim = dim3(4 * 64);
        MDHB_CUDA(cudaOccupancyMaxActiveClusters(&mc_clusters_, reinterpret_cast<const void*>(k), &lc));
        mc_clusters_ = std::max(1, mc_clusters_);
      }
      const int clusters = std::min(mc_clusters_, (tilesM_ / 2) * (tilesN_ / 2));
      lc.gridDim = dim3(static_cast<unsigned>(4 * clusters));
      MDHB_CUDA(cudaLaunchKernelEx(&lc, k, ma_, mb2_, a, b_row_rank_));
      return;
    }
    if (two_sm_) {
      const int sms = sm_count(p_.opt.device);
      const int pairs = std::min(sms / 2, (tilesM_ / 2) * (wide_ ? tilesN_ / 2 : tilesN_));
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(static_cast<unsigned>(2 * pairs));
      lc.blockDim = dim3(64 + 32 * 4);
      lc.dynamicSmemBytes = smem2_;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      void (*k)(const CUtensorMap, const CUtensorMap, TcArgs, int) =
          wide_ ? (bf16_ ? tc_gemm_2sm<256, 4, true, false, false, true>
                         : vb_.mn ? tc_gemm_2sm<256, 4, false, true, false, true> : tc_gemm_2sm<256, 4, false, false, false, true>)
          : vb_.mn ? tc_gemm_2sm<256, 6, false, true>
          : bf16_ ? (BN_ == 256 ? tc_gemm_2sm<256, 6, true> : tc_gemm_2sm<128, 8, true>)
                  : (BN_ == 256 ? tc_gemm_2sm<256, 6> : tc_gemm_2sm<128, 8>);
      MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2_)));
      MDHB_CUDA(cudaLaunchKernelEx(&lc, k, ma_, mb2_, a, b_row_rank_));
      return;
    }
    if (pers_) {
      const int sms = sm_count(p_.opt.device);
      dim3 pgrid(static_cast<unsigned>(rb_ && tilesN_ > 1 ? rbn_lanes_ * tilesN_ : std::min(sms, tilesM_ * tilesN_)));
#define MDHB_TCP(BNV, ST, MN, RBV)                                                                           \
  if (BN_ == BNV && vb_.mn == MN && rb_ == RBV && pstages_ == ST) {                                         \
    auto k = bf16_ ? tc_gemm_pers<BNV, ST, MN, RBV, true> : tc_gemm_pers<BNV, ST, MN, RBV, false>;          \
    MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(psmem_))); \
    k<<<pgrid, 64 + 32 * epi_warps(RBV, BNV), psmem_, s>>>(ma_, mb_, a, tail_ ? mat_ : ma_, tail_ ? mbt_ : mb_);                                              \
    MDHB_CUDA(cudaGetLastError());                                                                          \
    return;                                                                                                 \
  }
      if (psmem_ > 227 * 1024) fail("Unsupported", "tensor-core instance exceeds 227 KB of shared memory");
      MDHB_TCP(256, 4, false, false) MDHB_TCP(256, 4, true, false) MDHB_TCP(192, 4, false, false)
      MDHB_TCP(128, 5, false, false) MDHB_TCP(128, 5, true, false) MDHB_TCP(64, 6, false, false)
      MDHB_TCP(64, 4, false, true) MDHB_TCP(64, 3, false, true) MDHB_TCP(128, 4, false, true)
      MDHB_TCP(128, 3, false, true) MDHB_TCP(192, 4, false, true) MDHB_TCP(192, 3, false, true)
#undef MDHB_TCP
    }
    dim3 grid(static_cast<unsigned>(tilesM_ * tilesN_));
#define MDHB_TC(BNV, ST, MN)                                                                              \
  if (BN_ == BNV && vb_.mn == MN) {                                                                      \
    auto k = tc_gemm_tf32<BNV, ST, MN>;                                                                  \
    MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_))); \
    k<<<grid, 192, smem_, s>>>(ma_, mb_, a);                                                             \
    MDHB_CUDA(cudaGetLastError());                                                                       \
    return;                                                                                              \
  }
    MDHB_TC(256, 4, true) MDHB_TC(256, 4, false) MDHB_TC(128, 6, true) MDHB_TC(128, 6, false)
    MDHB_TC(64, 8, true) MDHB_TC(64, 8, false)
#undef MDHB_TC
    fail("Unsupported", "no tensor-core instance for this tile");
  }

 private:
  void encode(const View& v, const void* ptr, CUtensorMap* m) {
    cuuint32_t estr[MAXR] = {1, 1, 1, 1, 1};
    CUresult r = encoder()(m, v.bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           static_cast<cuuint32_t>(v.rank), const_cast<void*>(ptr),
                           v.dims, v.strides + 1, v.box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           v.mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                           : v.swz_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                           : v.swz_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  }

  const Problem& p_;
  Groups g_;
  TcKnobs kn_;
  void* ws_ = nullptr;
  int64_t ws_n_ = 0;
  View va_, vb_;
  int64_t M_ = 0, N_ = 0, K_ = 0;
  int BN_ = 0, stages_ = 0, nk_ = 0, tilesM_ = 0, tilesN_ = 0;
  bool cvec_ = false;
  size_t smem_ = 0;
  void* blob_ = nullptr;
  TcArgs args_{};
  CUtensorMap ma_{}, mb_{};
  CUtensorMap mat_{}, mbt_{};  // tail k-step views of packed operands
  View vat_, vbt_;
  bool tail_ = false;
  const void* last_a_ = nullptr;
  const void* last_b_ = nullptr;
  bool transposeB_ = false;
  int64_t tK_ = 0, tN_ = 0;
  void* bt_ = nullptr;
  bool pers_ = false, rb_ = false;
  int rbn_lanes_ = 0;  // resident B over many N tiles: CTAs per N tile
  int pstages_ = 0;
  size_t psmem_ = 0;
  bool packed_ = false;
  int64_t Kp_ = 0, c_run_ = 1;
  bool two_sm_ = false;
  bool mc_ = false;  // CTA-pair clusters of 4 sharing A by TMA multicast
  bool wide_ = false;  // CTA-pair tiles of 256 x 2 BN (two N tiles per A landing)
  int mc_clusters_ = 0;
  View vaH_;
  bool bf16_ = false, a_rowfast_ = false, b_rowfast_ = false;
  struct PlainPack {
    int kind = 0;  // 0 table gather, 1 vectorised convert (k unit-stride), 2 64x64 transpose (rows unit-stride)
    int64_t base = 0, stride = 0;
  };
  PlainPack ppa_, ppb_;
  int b_row_rank_ = 1, st2_ = 0;
  size_t smem2_ = 0;
  View vb2_;
  CUtensorMap mb2_{};
  void *pa_ = nullptr, *pb_ = nullptr;
  std::array<const int32_t*, 6> pk_{};  // packing tables: tAm, am, ak, tBn, bn, bk
};

}  // namespace

// ---- Table-1 instantiation of the tensor-core GEMM (MatMul-shaped md_homs:
// one M, one N, one K dim).  ASM layers, MDH layer order DM -> SMX -> WRP ->
// CC -> SM -> RM (the persistent schedule: a CTA's sequential tile loop is
// the DM layer around the concurrent SMX layer):
//   SMX(m) x DM(m) = M tiles; SMX(m) = M tiles per raster group; DM(m) > 1
//     = persistent CTAs walking groups, DM(m) = 1 = one CTA per tile
//   WRP(m) x CC(m) = rows per tile: 128 (4 epilogue warps x 32 TMEM lanes), 256 = CTA pair
//   SMX(n) = N tiles, RM(n) = BN (TMEM columns each epilogue thread drains)
//   SM(k) = the 128-byte k-tile (32 TF32 / 64 BF16), DM(k) = k-tiles per split,
//   SMX(k) = K split, partials combined in DM ("SMXs combine in DM")
//   layout_de of B = [2, 1]: B rewritten K-major by a layout pass
bool gemm_shaped(const Groups& g) { return g.Md.size() == 1 && g.Nd.size() == 1 && g.Kd.size() == 1; }
int k_tile(const Problem& p) { return p.opt.math == Math::BF16 ? 2 * BKE : BKE; }
bool b_mn_major(const Groups& g) { return std::llabs(g.lb.cj[static_cast<size_t>(g.Nd[0])]) == 1; }

TcKnobs tc_knobs(const Problem& p, const Groups& g, const Config& c) {
  const MdHom& e = p.e;
  const Asm& m = p.m;
  const int smx = m.id("SMX"), dm = m.id("DM"), wrp = m.id("WRP"), cc = m.id("CC"), sm = m.id("SM"), rm = m.id("RM");
  if (smx < 0 || dm < 0 || wrp < 0 || cc < 0 || sm < 0 || rm < 0) fail("Unsupported", "tensor-core template needs the B200 (CUDA+WRP) layers");
  auto P = parts_per_asm_layer(c, e, m);
  for (const char* other : {"GPU", "HM"})
    if (m.id(other) > 0)
      for (int64_t x : P[static_cast<size_t>(m.id(other) - 1)])
        if (x != 1) fail("Unsupported", std::string("tensor-core template: ") + other + " parts belong to the DEV layer");
  const int dm_ = g.Md[0], dn = g.Nd[0], dk = g.Kd[0];
  auto at = [&](int layer, int d) { return P[static_cast<size_t>(layer - 1)][static_cast<size_t>(d)]; };
  auto below = [&](int d) { return at(wrp, d) * at(cc, d) * at(sm, d) * at(rm, d); };
  TcKnobs k;
  k.set = true;
  const int64_t tm = below(dm_);
  if (tm != BM && tm != 2 * BM) fail("Unsupported", "tensor-core tile rows (WRP x CC x SM x RM of M) must be 128 or 256");
  k.bn = static_cast<int>(below(dn));
  if (k.bn != 64 && k.bn != 128 && k.bn != 192 && k.bn != 256 && !(k.bn == 512 && tm == 2 * BM))
    fail("Unsupported", "tensor-core N tile must be 64, 128, 192 or 256 (512 for CTA-pair tiles)");
  if (below(dk) != k_tile(p)) fail("Unsupported", "tensor-core k-tile (SM x ... of K) must be one 128-byte row");
  const int64_t cols = e.sizes[static_cast<size_t>(dn)] / k.bn;
  if (at(dm, dn) != 1) {
    // DM parts of N = one per N tile: each CTA keeps its N tile of B resident
    // and walks SMX parts of M tiles (the CTAs of one N tile = DM parts of M)
    if (tm != BM || at(dm, dn) != cols || at(smx, dn) != 1 || at(smx, dk) != 1)
      fail("Unsupported", "tensor-core template: DM parts of N must be 1, or one per 128-row-tile N tile (resident B, no K split)");
    k.rbn = true;
  }
  k.split = static_cast<int>(at(smx, dk));
  const int64_t rows = e.sizes[static_cast<size_t>(dm_)] / tm;
  if (k.rbn) {
    k.form = 1;
    k.group = static_cast<int>(at(smx, dm_));
  } else if (tm == 2 * BM) {
    k.form = 2;
    k.group = static_cast<int>(at(smx, dm_));
  } else if (at(dm, dm_) > 1) {
    k.form = 1;
    k.group = static_cast<int>(at(smx, dm_));
  } else {
    k.form = 0;
    k.group = static_cast<int>(rows);
  }
  k.transpose = 0;
  const auto& lay = c.layout_de[static_cast<size_t>(g.b_buf)];
  for (auto& l : lay)
    if (l.size() == 2 && l[0] == 2 && l[1] == 1) k.transpose = 1;
  if (p.opt.math == Math::BF16) k.transpose = -1;  // bf16 operands are always packed K-major
  else if (!b_mn_major(g) && k.transpose == 1) fail("Unsupported", "B is stored K-major already");
  return k;
}

Config tc_canonical(const Problem& p, const Groups& g, const TcKnobs& k) {
  const MdHom& e = p.e;
  const int D = e.D(), dm_ = g.Md[0], dn = g.Nd[0], dk = g.Kd[0];
  const int64_t tm = k.form == 2 ? 2 * BM : BM, ek = k_tile(p);
  const int64_t rows = e.sizes[static_cast<size_t>(dm_)] / tm, cols = e.sizes[static_cast<size_t>(dn)] / k.bn;
  const int64_t grp = k.form == 0 ? rows : k.group;
  std::vector<int64_t> DMv(static_cast<size_t>(D), 1), SMXv(DMv), WRPv(DMv), CCv(DMv), SMv(DMv), RMv(DMv);
  DMv[static_cast<size_t>(dm_)] = rows / grp;
  SMXv[static_cast<size_t>(dm_)] = grp;
  (k.rbn ? DMv : SMXv)[static_cast<size_t>(dn)] = cols;
  SMXv[static_cast<size_t>(dk)] = k.split;
  DMv[static_cast<size_t>(dk)] = e.sizes[static_cast<size_t>(dk)] / ek / k.split;
  WRPv[static_cast<size_t>(dm_)] = tm / 32;
  CCv[static_cast<size_t>(dm_)] = 32;
  SMv[static_cast<size_t>(dk)] = ek;
  RMv[static_cast<size_t>(dn)] = k.bn;
  Config c = make_config(p, {{"DM", DMv}, {"SMX", SMXv}, {"WRP", WRPv}, {"CC", CCv}, {"SM", SMv}, {"RM", RMv}},
                         {{e.in[static_cast<size_t>(g.a_buf)].name, "SM"}, {e.in[static_cast<size_t>(g.b_buf)].name, "SM"}}, "RM");
  if (k.transpose == 1)
    for (auto& l : c.layout_de[static_cast<size_t>(g.b_buf)]) l = {2, 1};
  return c;
}

// Every instance the tensor-core GEMM template offers for this problem, as
// canonical configurations (the tuner's search space).
std::vector<Config> tc_space(const Problem& p, const Groups& g) {
  std::vector<Config> out;
  if (!gemm_shaped(g) || p.m.id("WRP") < 0 || p.m.id("SMX") < 0) return out;
  const MdHom& e = p.e;
  const int64_t M = e.sizes[static_cast<size_t>(g.Md[0])], N = e.sizes[static_cast<size_t>(g.Nd[0])],
                K = e.sizes[static_cast<size_t>(g.Kd[0])], ek = k_tile(p);
  if (K % ek) return out;
  const bool bf16 = p.opt.math == Math::BF16, mn = b_mn_major(g);
  for (int form = 0; form < 3; ++form)
    for (int bn : {512, 256, 192, 128, 64}) {
      if (N % bn) continue;
      if ((form == 0 && (bn == 192 || bf16)) || (form == 2 && bn != 512 && bn != 256 && bn != 128)) continue;
      if (bn == 512 && form != 2) continue;
      const int64_t tm = form == 2 ? 2 * BM : BM;
      if (M % tm) continue;
      const int64_t rows = M / tm;
      for (int tr : {0, 1}) {
        if (bf16 && tr) continue;
        if (!bf16 && !mn && tr) continue;
        if (form == 1 && bn == 192 && !(mn && !tr && !bf16))  // resident-B instances: CTAs per N tile 1, 2, 4
          for (int64_t lanes : {1, 2, 4}) {
            if (rows % lanes || rows / lanes < 4 || N / bn < 2) continue;
            if ((K / ek) * bn * 128 + 3 * BM * 128 + 1280 + epi_bytes(true, bn) > 227 * 1024) continue;  // B resident in smem
            TcKnobs k;
            k.set = true;
            k.form = 1;
            k.bn = bn;
            k.group = static_cast<int>(rows / lanes);
            k.transpose = bf16 ? -1 : (mn ? tr : 0);
            k.rbn = true;
            Config c = tc_canonical(p, g, k);
            if (config_violation(c, e, p.m, true).empty()) out.push_back(c);
          }
        if (!bf16 && mn && !tr && ((form == 2 && bn != 256 && bn != 512) || bn == 192 || (bn == 64 && form == 1))) continue;  // no MN-major instance
        for (int split : {1, 2, 4}) {
          if ((K / ek) % split) continue;
          std::vector<int64_t> groups;
          if (form == 0) groups = {rows};
          else
            for (int64_t gp = 1; gp < rows && gp <= 64; gp *= 2)
              if (rows % gp == 0) groups.push_back(gp);
          for (int64_t gp : groups) {
            TcKnobs k;
            k.set = true;
            k.form = form;
            k.bn = bn;
            k.group = static_cast<int>(gp);
            k.split = split;
            k.transpose = bf16 ? -1 : (mn ? tr : 0);
            Config c = tc_canonical(p, g, k);
            if (config_violation(c, e, p.m, true).empty()) out.push_back(c);
          }
        }
      }
    }
  return out;
}

bool tc_project(const Problem& p, const Groups& g, const Config& c, Config* canon) {
  if (!gemm_shaped(g) || p.opt.math == Math::FFMA) return false;
  *canon = tc_canonical(p, g, tc_knobs(p, g, c));
  return true;
}

std::unique_ptr<Routine> make_tc_contraction(const Problem& p, const Groups& g, const Config* cfg, Config* cfg_out,
                                             std::string* why) {
  // N-tile menu; among the instances that set up, prefer a direct TMA view
  // over packed operands, then the longest contiguous run of C per tile row
  // (the epilogue's store width), then the wider tile.
  {
    std::string w;
    if (auto conv = make_tc_conv(p, g, &w)) {
      if (cfg_out) *cfg_out = cfg ? *cfg : baseline_config(p.e, p.m);
      return conv;
    }
  }
  TcKnobs kn;
  if (cfg && gemm_shaped(g)) kn = tc_knobs(p, g, *cfg);  // Unsupported when outside the template
  std::vector<int> menu = {256, 192, 128, 64};
  if (const char* f = std::getenv("MDHB_TC_BN")) menu = {std::atoi(f)};
  if (kn.set) menu = {kn.bn == 512 ? 256 : kn.bn};  // 512: two 256-column N tiles per CTA-pair tile
  std::unique_ptr<TcRoutine> best;
  int64_t best_score = -1;
  for (int bn : menu) {
    auto r = std::make_unique<TcRoutine>(p, g, kn);
    std::string w;
    if (!r->setup(bn, &w)) {
      *why = w;
      continue;
    }
    const int64_t score = (r->packed() ? 0 : 1000000) + r->c_run() * 1000 + bn;
    if (score > best_score) best_score = score, best = std::move(r);
  }
  if (kn.set && !best) fail("Unsupported", "tensor-core template cannot instantiate this configuration: " + *why);
  if (best && cfg_out) {
    if (gemm_shaped(g) && p.m.id("WRP") > 0 && p.m.id("SMX") > 0 && (kn.set || best->knobs_default(&kn)))
      *cfg_out = tc_canonical(p, g, kn);
    else
      *cfg_out = cfg ? *cfg : baseline_config(p.e, p.m);
  }
  return best;
}

}  // namespace ctr
}  // namespace mdhb
