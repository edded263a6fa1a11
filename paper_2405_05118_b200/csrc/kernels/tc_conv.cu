// Tensor-core (tcgen05 kind::tf32) instance for the multi-channel convolution
// md_hom over NHWC (MCC, BASELINE config 4; the reference's mcc.json with
// NHWC/KRSC/NPQK views):
//
//   O[n][p][q][k] = sum_{r,s,c}  I[n][p+r][q+s][c] * F[k][r][s][c]
//
// The generic tensor-core contraction re-reads the input once per filter tap
// (r,s) -- 9 TMA boxes per output tile.  Here the input patch a tile needs is
// loaded ONCE per 32-channel chunk and all R*S taps are issued from it by
// shifting the UMMA shared-memory descriptor:
//
//   * tile = 16 output rows (p) x 8 output columns (q) of one image = 128 MMA
//     rows (M), all K output channels as N (64);  P is padded to 16 (rows past
//     P are computed on TMA zero-fill and never stored)
//   * patch = (16+R-1) x (8+S-1) input pixels x 32 channels, landed by one 5-D
//     TMA box {4 c, 8+S-1 q, 16+R-1 p, 8 c-groups, 1 n} without swizzle, i.e.
//     [c-group][p'][q'][4 c]: every 16-byte core-matrix row is one pixel's 4
//     channels, 8 consecutive q' are 128 contiguous bytes
//   * tap (r,s), k-step j: A descriptor start = patch + 2j*plane + (r*Wq+s)*16,
//     M-direction core stride 16*Wq bytes (next p), K-direction core stride
//     plane bytes (next 4 channels) -- the K-major no-swizzle canonical layout
//   * the filter (K x R*S*C, K-major) stays resident in shared memory, 128B
//     swizzled, loaded once per CTA
//
// Warp roles as tc_gemm_pers: warp 0 TMA, warp 1 TMEM + MMA issue (one
// thread), warps 2-5 drain the double-buffered TMEM accumulator through a
// 32x32 smem transpose into coalesced 256-byte C rows.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <sstream>

#include "contraction_common.hpp"
#include "tc_gemm.cuh"

namespace mdhb {
namespace ctr {
namespace {

constexpr int CV_BM = 128, CV_TP = 16, CV_TQ = 8, CV_BKE = 32;

struct ConvArgs {
  float* O;
  int N, P, Q, K;          // output extents (K = output channels = BN)
  int R, S, C;             // taps and input channels
  int HP, WQ;              // patch extents (CV_TP + R - 1, CV_TQ + S - 1)
  int pblocks, qblocks;    // tiles per image
  int64_t on, op, oq;      // output strides (elements)
  uint32_t plane;          // bytes of one 4-channel plane of the patch (HP * WQ * 16)
  uint32_t lbo, sbo;       // descriptor core-matrix strides (K direction, M direction)
  int ek;                  // channels per k-tile row of 128 bytes (32 fp32 / 64 bf16)
  int sw;                  // 1: pixel-major 128B-swizzled patch (4-D box {32 c, WQ, HP, 1})
  int bo_mode;             // descriptor base-offset rule for shifted swizzled rows (dev)
  int tma_store;           // 1: output tiles leave through TMA tensor stores (NPQK view, clipped at P)
};

__device__ __forceinline__ uint64_t nosw_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return tc::umma_desc(saddr, lbo, sbo, 0);
}

template <int BN, bool BF16 = false, int PSTAGES = 2>
__global__ void __launch_bounds__(192, 1)
    tc_conv_tf32(const __grid_constant__ CUtensorMap tma_i, const __grid_constant__ CUtensorMap tma_f,
                 const __grid_constant__ CUtensorMap tma_o, ConvArgs g) {
  constexpr uint32_t B_BYTES = BN * CV_BKE * 4;      // one 128-byte-row k-tile of the filter (32 fp32 / 64 bf16)
  constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int ktiles = g.R * g.S * (g.C / g.ek);
  const int chunks = g.C / g.ek;
  const uint32_t patch_bytes = 8 * g.plane;           // 8 planes of 4 channels = 32 channels
  const uint32_t patch_slot = (patch_bytes + 1023) & ~1023u;
  uint8_t* sB = smem;                                 // resident filter [ktiles][BN][32] (128B swizzle)
  uint8_t* sP = smem + static_cast<size_t>(ktiles) * B_BYTES;  // patch ring
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + PSTAGES * patch_slot);
  uint64_t* empty = full + PSTAGES;
  uint64_t* bfull = empty + PSTAGES;
  uint64_t* tfull = bfull + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stage_base = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);
  // TMA-store staging: 1024-aligned, 8 KB per epilogue warp (two 128B-swizzled 32-channel halves)
  const uint32_t ostage = (tc::smem_u32(full) + 256 + 1023) & ~1023u;
  const int warp = tc::warp_uniform(), lane = threadIdx.x & 31;
  const int per_img = g.pblocks * g.qblocks;
  const int ntiles = g.N * per_img;

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tma_i);
    tc::tma_prefetch(&tma_f);
    for (int s = 0; s < PSTAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(bfull, 1);
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: the filter once, then one patch per (tile, chunk)
    tc::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(ktiles) * B_BYTES);
    for (int kt = 0; kt < ktiles; ++kt) {
      int c[5] = {kt * g.ek, 0, 0, 0, 0};
      tc::tma_load(sB + static_cast<size_t>(kt) * B_BYTES, &tma_f, bfull, 2, c);
    }
    uint32_t it = 0;
    for (int x = blockIdx.x; x < ntiles; x += gridDim.x) {
      const int n = x / per_img, rem = x % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
      for (int cc = 0; cc < chunks; ++cc, ++it) {
        const uint32_t s = it % PSTAGES;
        if (it >= PSTAGES) tc::mbar_wait(&empty[s], ((it / PSTAGES) - 1) & 1);
        tc::mbar_arrive_expect_tx(&full[s], patch_bytes);
        if (g.sw) {
          int c[5] = {cc * g.ek, qb * CV_TQ, pb * CV_TP, n, 0};
          tc::tma_load(sP + s * patch_slot, &tma_i, &full[s], 4, c);
        } else {
          int c[5] = {0, qb * CV_TQ, pb * CV_TP, cc * 8, n};
          tc::tma_load(sP + s * patch_slot, &tma_i, &full[s], 5, c);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp walks the loop with uniform
    // operands, one elected lane issues.  Descriptors are built once and
    // advanced by adding 16-byte units to the start-address field (shared
    // addresses < 256 KB never carry out of its 14 bits).
    constexpr uint32_t idesc = tc::instr_desc(BF16 ? 1 : 2, 0, 0, CV_BM, BN);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint64_t da0 = g.sw ? tc::umma_desc(tc::smem_u32(sP), 16, static_cast<uint32_t>(g.WQ) * 128, 2)
                              : nosw_desc(tc::smem_u32(sP), g.lbo, g.sbo);
    const uint64_t db0 = tc::sw128_desc(tc::smem_u32(sB), 16, 1024);
    const uint32_t tap_u = g.sw ? 8 : 1;                         // one pixel, 16-byte units
    const uint32_t j_u = g.sw ? 2 : (2 * g.plane) >> 4;          // next 8 (tf32) / 16 (bf16) channels
    const uint32_t slot_u = patch_slot >> 4, btap_u = (static_cast<uint32_t>(chunks) * B_BYTES) >> 4;
    tc::mbar_wait_warp(bfull, 0);
    uint32_t it = 0, tl = 0;
    for (int x = blockIdx.x; x < ntiles; x += gridDim.x, ++tl) {
      const uint32_t acc = tl & 1;
      if (tl >= 2) tc::mbar_wait_warp(&tempty[acc], ((tl / 2) - 1) & 1);
      tc::tc_fence_after();
      const uint32_t dtm = tm + acc * BN;
      for (int cc = 0; cc < chunks; ++cc, ++it) {
        const uint32_t s = it % PSTAGES;
        tc::mbar_wait_warp(&full[s], (it / PSTAGES) & 1);
        tc::tc_fence_after();
        const uint64_t dA = da0 + s * slot_u;
        uint64_t dB = db0 + ((static_cast<uint32_t>(cc) * B_BYTES) >> 4);
        uint32_t first = cc == 0 ? 1u : 0u;
        for (int r = 0; r < g.R; ++r)
          for (int ss = 0; ss < g.S; ++ss, dB += btap_u) {
            const uint32_t t = static_cast<uint32_t>(r * g.WQ + ss);
            const uint64_t a = dA + t * tap_u + (g.bo_mode ? static_cast<uint64_t>(t & 7) << 49 : 0);
#pragma unroll
            for (int j = 0; j < CV_BKE / 8; ++j) {
              tc::mma_warp<!BF16>(dtm, a + j * j_u, dB + 2 * j, idesc, first ? 0u : 1u);
              first = 0;
            }
          }
        tc::mma_commit_warp(&empty[s]);
      }
      tc::mma_commit_warp(&tfull[acc]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: TMEM -> 32x32 smem transpose -> C rows
    const int q = warp & 3;
    if (g.tma_store) {
      // TMEM lane = output pixel, columns = channels: each lane owns a 256-byte
      // output row; lanes write their rows 128B-swizzled (conflict-free) and one
      // lane stores the warp's 4 p x 8 q x 64 k box (rows past P are clipped)
      const uint32_t stg = ostage + static_cast<uint32_t>(warp - 2) * 8192;
      uint32_t tl = 0;
      for (int x = blockIdx.x; x < ntiles; x += gridDim.x, ++tl) {
        const int n = x / per_img, rem = x % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
        const uint32_t acc = tl & 1;
        tc::mbar_wait(&tfull[acc], (tl / 2) & 1);
        tc::tc_fence_after();
        if (lane == 0) tc::bulk_wait_read0();
        __syncwarp();
#pragma unroll
        for (int h = 0; h < BN / 32; ++h) {
          uint32_t rv[32];
          tc::tmem_ld32(tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(h * 32), rv);
          const uint32_t row = stg + static_cast<uint32_t>(h) * 4096 + static_cast<uint32_t>(lane) * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((c ^ (lane & 7)) << 4)), "r"(rv[4 * c]),
                         "r"(rv[4 * c + 1]), "r"(rv[4 * c + 2]), "r"(rv[4 * c + 3])
                         : "memory");
        }
        tc::tc_fence_before();
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&tempty[acc]);
#pragma unroll
          for (int h = 0; h < BN / 32; ++h)
            tc::tma_store4(&tma_o, stg + static_cast<uint32_t>(h) * 4096, h * 32, qb * CV_TQ, pb * CV_TP + q * 4, n);
          tc::bulk_commit();
        }
      }
      if (lane == 0) tc::bulk_wait0();
    } else {
    const uint32_t stg = tc::smem_u32(stage_base) + static_cast<uint32_t>(warp - 2) * (32 * 33 * 4 + 32 * 8);
    const uint32_t rtab = stg + 32 * 33 * 4;
    uint32_t tl = 0;
    for (int x = blockIdx.x; x < ntiles; x += gridDim.x, ++tl) {
      const int n = x / per_img, rem = x % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
      const uint32_t acc = tl & 1;
      // TMEM lane m = pp * 8 + qq  ->  output pixel (n, pb*16 + pp, qb*8 + qq); -1 = padding row
      const int m = q * 32 + lane, p = pb * CV_TP + m / CV_TQ, qq = qb * CV_TQ + m % CV_TQ;
      const int64_t rowoff = p < g.P ? n * g.on + p * g.op + qq * g.oq : -1;
      asm volatile("st.shared.s64 [%0], %1;" ::"r"(rtab + lane * 8), "l"(rowoff) : "memory");
      tc::mbar_wait(&tfull[acc], (tl / 2) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t rv[32];
        tc::tmem_ld32(tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), rv);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(stg + (lane * 33 + j) * 4), "r"(rv[j]) : "memory");
        __syncwarp();
        float* cc = g.O + c0 + lane;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          int64_t ro;
          float v;
          asm volatile("ld.shared.s64 %0, [%1];" : "=l"(ro) : "r"(rtab + rr * 8) : "memory");
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(stg + (rr * 33 + lane) * 4) : "memory");
          if (ro >= 0) __stcs(cc + ro, v);
        }
        __syncwarp();
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// BF16 instance with the fp32 -> bf16 conversion fused (MDHB_CONV_BF16F):
// the producer lands each 32-channel fp32 half-chunk of the patch with a 4-D
// TMA box {32 c, WQ, HP, 1} into a 2-slot staging ring; four converter warps
// turn two halves into one 64-channel bf16 patch slot -- pixel rows of 128
// bytes written with the 128-byte swizzle TMA would apply (16-byte chunk
// index XOR address bits 7..9) -- fence them into the async proxy and arrive
// on the slot's full barrier.  The MMA warp and the TMA-store epilogue are
// tc_conv_tf32<BF16>'s.  The input is read once as fp32; no bf16 copy of it
// exists in HBM.
template <int BN, int PST, int FS, int EH>
__global__ void __launch_bounds__(320, 1)
    tc_conv_bf16f(const __grid_constant__ CUtensorMap tma_i, const __grid_constant__ CUtensorMap tma_f,
                  const __grid_constant__ CUtensorMap tma_o, ConvArgs g) {
  constexpr uint32_t B_BYTES = BN * 128;  // one 64-channel bf16 k-tile of the filter
  constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int chunks = g.C / 64;
  const int ktiles = g.R * g.S * chunks;
  const int npx = g.HP * g.WQ;
  const uint32_t patch_bytes = static_cast<uint32_t>(npx) * 128;
  // slots need only 128-byte alignment: the bf16 slots' swizzle is a function
  // of absolute address bits on both sides (converter stores, UMMA reads)
  const uint32_t patch_slot = patch_bytes;
  uint8_t* sB = smem;
  uint8_t* sP = sB + static_cast<size_t>(ktiles) * B_BYTES;  // bf16 patch ring
  uint8_t* sF = sP + static_cast<size_t>(PST) * patch_slot;  // fp32 staging ring
  uint64_t* full = reinterpret_cast<uint64_t*>(sF + FS * patch_slot);
  uint64_t* empty = full + PST;
  uint64_t* sfull = empty + PST;
  uint64_t* sempty = sfull + FS;
  uint64_t* bfull = sempty + FS;
  uint64_t* tfull = bfull + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t ostage = (tc::smem_u32(full) + 256 + 1023) & ~1023u;
  const int warp = tc::warp_uniform(), lane = threadIdx.x & 31;
  const int per_img = g.pblocks * g.qblocks;
  const int ntiles = g.N * per_img;

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tma_i);
    tc::tma_prefetch(&tma_f);
    for (int s = 0; s < PST; ++s) {
      tc::mbar_init(&full[s], 4);   // one arrival per converter warp
      tc::mbar_init(&empty[s], 1);  // MMA commit
    }
    for (int s = 0; s < FS; ++s) {
      tc::mbar_init(&sfull[s], 1);
      tc::mbar_init(&sempty[s], 4);
    }
    tc::mbar_init(bfull, 1);
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: the bf16 filter once, then fp32 half-chunks
    tc::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(ktiles) * B_BYTES);
    for (int kt = 0; kt < ktiles; ++kt) {
      int c[5] = {kt * 64, 0, 0, 0, 0};
      tc::tma_load(sB + static_cast<size_t>(kt) * B_BYTES, &tma_f, bfull, 2, c);
    }
    uint32_t it = 0;
    for (int x = blockIdx.x; x < ntiles; x += gridDim.x) {
      const int n = x / per_img, rem = x % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
      for (int h = 0; h < 2 * chunks; ++h, ++it) {
        const uint32_t s = it % FS;
        if (it >= FS) tc::mbar_wait(&sempty[s], ((it / FS) - 1) & 1);
        tc::mbar_arrive_expect_tx(&sfull[s], patch_bytes);
        int c[5] = {h * 32, qb * CV_TQ, pb * CV_TP, n, 0};
        tc::tma_load(sF + s * patch_slot, &tma_i, &sfull[s], 4, c);
      }
    }
  } else if (warp >= 6) {
    // ---------------- converters: two fp32 halves -> one swizzled bf16 slot
    const int ct = threadIdx.x - 192;  // 0..127
    uint32_t it = 0, ps = 0;
    for (int x = blockIdx.x; x < ntiles; x += gridDim.x) {
      for (int cc = 0; cc < chunks; ++cc, ++ps) {
        const uint32_t s = ps % PST;
        if (ps >= PST) tc::mbar_wait(&empty[s], ((ps / PST) - 1) & 1);
        const uint32_t dst = tc::smem_u32(sP + s * patch_slot);
        for (int h = 0; h < 2; ++h, ++it) {
          const uint32_t fs = it % FS;
          tc::mbar_wait(&sfull[fs], (it / FS) & 1);
          const uint32_t src = tc::smem_u32(sF + fs * patch_slot);
          for (int i = ct; i < npx * 8; i += 128) {
            const int px = i >> 3, c4 = i & 7;
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(src + static_cast<uint32_t>(px) * 128 + c4 * 16));
            __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
            const uint32_t row = dst + static_cast<uint32_t>(px) * 128;
            const uint32_t chunk = static_cast<uint32_t>(h * 4 + (c4 >> 1)) ^ ((row >> 7) & 7u);
            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(row + chunk * 16 + (c4 & 1) * 8),
                         "r"(*reinterpret_cast<uint32_t*>(&lo)), "r"(*reinterpret_cast<uint32_t*>(&hi))
                         : "memory");
          }
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&sempty[fs]);
        }
        tc::fence_proxy_async();  // generic-proxy writes -> visible to tcgen05 (async proxy)
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp, uniform descriptors)
    constexpr uint32_t idesc = tc::instr_desc(1, 0, 0, CV_BM, BN);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint64_t da0 = tc::umma_desc(tc::smem_u32(sP), 16, static_cast<uint32_t>(g.WQ) * 128, 2);
    const uint64_t db0 = tc::sw128_desc(tc::smem_u32(sB), 16, 1024);
    const uint32_t slot_u = patch_slot >> 4, btap_u = (static_cast<uint32_t>(chunks) * B_BYTES) >> 4;
    tc::mbar_wait_warp(bfull, 0);
    uint32_t it = 0, tl = 0;
    for (int x = blockIdx.x; x < ntiles; x += gridDim.x, ++tl) {
      const uint32_t acc = tl & 1;
      if (tl >= 2) tc::mbar_wait_warp(&tempty[acc], ((tl / 2) - 1) & 1);
      tc::tc_fence_after();
      const uint32_t dtm = tm + acc * BN;
      for (int cc = 0; cc < chunks; ++cc, ++it) {
        const uint32_t s = it % PST;
        tc::mbar_wait_warp(&full[s], (it / PST) & 1);
        tc::tc_fence_after();
        const uint64_t dA = da0 + s * slot_u;
        uint64_t dB = db0 + ((static_cast<uint32_t>(cc) * B_BYTES) >> 4);
        uint32_t first = cc == 0 ? 1u : 0u;
        for (int r = 0; r < g.R; ++r)
          for (int ss = 0; ss < g.S; ++ss, dB += btap_u) {
            const uint64_t a = dA + static_cast<uint32_t>(r * g.WQ + ss) * 8;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              tc::mma_warp<false>(dtm, a + j * 2, dB + 2 * j, idesc, first ? 0u : 1u);
              first = 0;
            }
          }
        tc::mma_commit_warp(&empty[s]);
      }
      tc::mma_commit_warp(&tfull[acc]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (TMA tensor stores), as tc_conv_tf32; EH = 32-channel
    // halves buffered per warp (1: the second half waits for the first's smem read)
    const int q = warp & 3;
    const uint32_t stg = ostage + static_cast<uint32_t>(warp - 2) * 4096 * EH;
    uint32_t tl = 0;
    for (int x = blockIdx.x; x < ntiles; x += gridDim.x, ++tl) {
      const int n = x / per_img, rem = x % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
      const uint32_t acc = tl & 1;
      tc::mbar_wait(&tfull[acc], (tl / 2) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int h = 0; h < BN / 32; ++h) {
        if (EH == 1 || h == 0) {
          if (lane == 0) tc::bulk_wait_read0();
          __syncwarp();
        }
        uint32_t rv[32];
        tc::tmem_ld32(tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(h * 32), rv);
        const uint32_t hb = stg + static_cast<uint32_t>(EH == 1 ? 0 : h) * 4096;
        const uint32_t row = hb + static_cast<uint32_t>(lane) * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((c ^ (lane & 7)) << 4)), "r"(rv[4 * c]),
                       "r"(rv[4 * c + 1]), "r"(rv[4 * c + 2]), "r"(rv[4 * c + 3])
                       : "memory");
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store4(&tma_o, hb, h * 32, qb * CV_TQ, pb * CV_TP + q * 4, n);
          tc::bulk_commit();
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) tc::bulk_wait0();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// CTA-pair instance (cta_group::2): the two CTAs of a cluster take two
// output tiles, each lands its own input patches, and each holds HALF of the
// resident filter (32 of the 64 output channels); the leader issues
// M = 256 x N = 64 MMAs that read the peer's patch and filter half at the same
// shared-memory offsets.  Per SM the MMA reads A + B/2 (and the filter's
// smem footprint halves, leaving room for a deeper patch ring).
__device__ __forceinline__ uint32_t cv_peer(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

template <int BN, int PSTAGES, bool BF16 = false>
__global__ void __launch_bounds__(192, 1)
    tc_conv_2sm(const __grid_constant__ CUtensorMap tma_i, const __grid_constant__ CUtensorMap tma_f,
                const __grid_constant__ CUtensorMap tma_o, ConvArgs g) {
  constexpr uint32_t B_BYTES = (BN / 2) * CV_BKE * 4;  // this CTA's half of one filter k-tile (128-byte rows)
  constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int chunks = g.C / g.ek;
  const int ktiles = g.R * g.S * chunks;
  const uint32_t patch_bytes = g.sw ? static_cast<uint32_t>(g.HP * g.WQ) * 128 : 8 * g.plane;
  const uint32_t patch_slot = (patch_bytes + 1023) & ~1023u;
  uint8_t* sB = smem;
  uint8_t* sP = smem + ((static_cast<size_t>(ktiles) * B_BYTES + 1023) & ~size_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + PSTAGES * patch_slot);
  uint64_t* empty = full + PSTAGES;
  uint64_t* bfull = empty + PSTAGES;
  uint64_t* tfull = bfull + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stage_base = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);
  const uint32_t ostage = (tc::smem_u32(full) + 256 + 1023) & ~1023u;
  const int warp = tc::warp_uniform(), lane = threadIdx.x & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const bool leader = rank == 0;
  const int per_img = g.pblocks * g.qblocks;
  const int ntiles = g.N * per_img;
  const int npairs_tiles = (ntiles + 1) / 2;  // pair items: tiles 2x (leader) and 2x+1 (peer)
  const int pair = static_cast<int>(blockIdx.x) >> 1, npairs = static_cast<int>(gridDim.x) >> 1;

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tma_i);
    tc::tma_prefetch(&tma_f);
    for (int s = 0; s < PSTAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(bfull, 1);
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 8);  // leader's copy: 4 epilogue warps x 2 CTAs
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs); everything completes on the leader's barriers
    const uint32_t bfull_leader = cv_peer(tc::smem_u32(bfull), 0);
    const uint32_t full_leader0 = cv_peer(tc::smem_u32(&full[0]), 0);
    // this CTA's filter half: output channels rank*BN/2 .. +BN/2, every k-tile
    if (leader) tc::mbar_arrive_expect_tx(bfull, 2u * static_cast<uint32_t>(ktiles) * B_BYTES);
    for (int kt = 0; kt < ktiles; ++kt) {
      int c[2] = {kt * g.ek, static_cast<int>(rank) * (BN / 2)};
      uint32_t d = tc::smem_u32(sB + static_cast<size_t>(kt) * B_BYTES);
      asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(d), "l"(&tma_f), "r"(bfull_leader), "r"(c[0]), "r"(c[1]) : "memory");
    }
    uint32_t it = 0;
    for (int x = pair; x < npairs_tiles; x += npairs) {
      // a ragged last pair: the peer re-loads the leader's tile (its rows are not stored)
      const int t = min(2 * x + static_cast<int>(rank), ntiles - 1);
      const int n = t / per_img, rem = t % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
      for (int cc = 0; cc < chunks; ++cc, ++it) {
        const uint32_t s = it % PSTAGES;
        if (it >= PSTAGES) tc::mbar_wait(&empty[s], ((it / PSTAGES) - 1) & 1);
        if (leader) tc::mbar_arrive_expect_tx(&full[s], 2 * patch_bytes);
        const uint32_t d = tc::smem_u32(sP + s * patch_slot);
        if (g.sw)
          asm volatile("cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                       ::"r"(d), "l"(&tma_i), "r"(full_leader0 + s * 8), "r"(cc * g.ek), "r"(qb * CV_TQ), "r"(pb * CV_TP), "r"(n)
                       : "memory");
        else
          asm volatile("cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                       ::"r"(d), "l"(&tma_i), "r"(full_leader0 + s * 8), "r"(0), "r"(qb * CV_TQ), "r"(pb * CV_TP), "r"(cc * 8), "r"(n)
                       : "memory");
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader warp, one elected lane): M = 256 (two tiles) x N = BN;
    // descriptors advanced by 16-byte units as in tc_conv_tf32
    constexpr uint32_t idesc = tc::instr_desc(BF16 ? 1 : 2, 0, 0, 2 * CV_BM, BN);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint64_t da0 = g.sw ? tc::umma_desc(tc::smem_u32(sP), 16, static_cast<uint32_t>(g.WQ) * 128, 2)
                              : nosw_desc(tc::smem_u32(sP), g.lbo, g.sbo);
    const uint64_t db0 = tc::sw128_desc(tc::smem_u32(sB), 16, 1024);
    const uint32_t tap_u = g.sw ? 8 : 1;
    const uint32_t j_u = g.sw ? 2 : (2 * g.plane) >> 4;
    const uint32_t slot_u = patch_slot >> 4, btap_u = (static_cast<uint32_t>(chunks) * B_BYTES) >> 4;
    tc::mbar_wait_warp(bfull, 0);
    uint32_t it = 0, tl = 0;
    for (int x = pair; x < npairs_tiles; x += npairs, ++tl) {
      const uint32_t acc = tl & 1;
      if (tl >= 2) tc::mbar_wait_warp(&tempty[acc], ((tl / 2) - 1) & 1);
      tc::tc_fence_after();
      const uint32_t dtm = tm + acc * BN;
      for (int cc = 0; cc < chunks; ++cc, ++it) {
        const uint32_t s = it % PSTAGES;
        tc::mbar_wait_warp(&full[s], (it / PSTAGES) & 1);
        tc::tc_fence_after();
        const uint64_t dA = da0 + s * slot_u;
        uint64_t dB = db0 + ((static_cast<uint32_t>(cc) * B_BYTES) >> 4);
        uint32_t first = cc == 0 ? 1u : 0u;
        for (int r = 0; r < g.R; ++r)
          for (int ss = 0; ss < g.S; ++ss, dB += btap_u) {
            const uint64_t a = dA + static_cast<uint32_t>(r * g.WQ + ss) * tap_u;
#pragma unroll
            for (int j = 0; j < CV_BKE / 8; ++j) {
              if (BF16)
                asm volatile(
                    "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtm), "l"(a + j * j_u),
                    "l"(dB + 2 * j), "r"(idesc), "r"(first ? 0u : 1u));
              else
                asm volatile(
                    "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtm), "l"(a + j * j_u),
                    "l"(dB + 2 * j), "r"(idesc), "r"(first ? 0u : 1u));
              first = 0;
            }
          }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
            ::"r"(tc::smem_u32(&empty[s])), "h"(static_cast<uint16_t>(3)) : "memory");
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
          ::"r"(tc::smem_u32(&tfull[acc])), "h"(static_cast<uint16_t>(3)) : "memory");
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (both CTAs): own tile, own 128 TMEM lanes
    const int q = warp & 3;
    const uint32_t tempty_leader0 = cv_peer(tc::smem_u32(&tempty[0]), 0);
    uint32_t tl = 0;
    if (g.tma_store) {
      const uint32_t stg = ostage + static_cast<uint32_t>(warp - 2) * 8192;
      for (int x = pair; x < npairs_tiles; x += npairs, ++tl) {
        const int t = 2 * x + static_cast<int>(rank);
        const int n = t / per_img, rem = t % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
        const uint32_t acc = tl & 1;
        tc::mbar_wait(&tfull[acc], (tl / 2) & 1);
        tc::tc_fence_after();
        if (lane == 0) tc::bulk_wait_read0();
        __syncwarp();
#pragma unroll
        for (int h = 0; h < BN / 32; ++h) {
          uint32_t rv[32];
          tc::tmem_ld32(tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(h * 32), rv);
          const uint32_t row = stg + static_cast<uint32_t>(h) * 4096 + static_cast<uint32_t>(lane) * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((c ^ (lane & 7)) << 4)), "r"(rv[4 * c]),
                         "r"(rv[4 * c + 1]), "r"(rv[4 * c + 2]), "r"(rv[4 * c + 3])
                         : "memory");
        }
        tc::tc_fence_before();
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader0 + acc * 8) : "memory");
          if (t < ntiles) {
#pragma unroll
            for (int h = 0; h < BN / 32; ++h)
              tc::tma_store4(&tma_o, stg + static_cast<uint32_t>(h) * 4096, h * 32, qb * CV_TQ, pb * CV_TP + q * 4, n);
          }
          tc::bulk_commit();
        }
      }
      if (lane == 0) tc::bulk_wait0();
    } else {
      const uint32_t stg = tc::smem_u32(stage_base) + static_cast<uint32_t>(warp - 2) * (32 * 33 * 4 + 32 * 8);
      const uint32_t rtab = stg + 32 * 33 * 4;
      for (int x = pair; x < npairs_tiles; x += npairs, ++tl) {
        const int tr = 2 * x + static_cast<int>(rank);
        const bool mine = tr < ntiles;
        const int t = mine ? tr : ntiles - 1;
        const int n = t / per_img, rem = t % per_img, pb = rem / g.qblocks, qb = rem % g.qblocks;
        const uint32_t acc = tl & 1;
        const int m = q * 32 + lane, p = pb * CV_TP + m / CV_TQ, qq = qb * CV_TQ + m % CV_TQ;
        const int64_t rowoff = (mine && p < g.P) ? n * g.on + p * g.op + qq * g.oq : -1;
        asm volatile("st.shared.s64 [%0], %1;" ::"r"(rtab + lane * 8), "l"(rowoff) : "memory");
        tc::mbar_wait(&tfull[acc], (tl / 2) & 1);
        tc::tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t rv[32];
          tc::tmem_ld32(tmem + acc * BN + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), rv);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(stg + (lane * 33 + j) * 4), "r"(rv[j]) : "memory");
          __syncwarp();
          float* cc = g.O + c0 + lane;
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) {
            int64_t ro;
            float v;
            asm volatile("ld.shared.s64 %0, [%1];" : "=l"(ro) : "r"(rtab + rr * 8) : "memory");
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(stg + (rr * 33 + lane) * 4) : "memory");
            if (ro >= 0) __stcs(cc + ro, v);
          }
          __syncwarp();
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader0 + acc * 8) : "memory");
      }
    }
  }
  tc::tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

__global__ void __launch_bounds__(256) to_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n8) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < n8; i += static_cast<int64_t>(gridDim.x) * 256) {
    const float4 a = __ldcs(reinterpret_cast<const float4*>(src) + 2 * i);
    const float4 b = __ldcs(reinterpret_cast<const float4*>(src) + 2 * i + 1);
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w),
                         h2 = __floats2bfloat162_rn(b.x, b.y), h3 = __floats2bfloat162_rn(b.z, b.w);
    uint4 w;
    w.x = *reinterpret_cast<const uint32_t*>(&h0);
    w.y = *reinterpret_cast<const uint32_t*>(&h1);
    w.z = *reinterpret_cast<const uint32_t*>(&h2);
    w.w = *reinterpret_cast<const uint32_t*>(&h3);
    reinterpret_cast<uint4*>(dst)[i] = w;
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn conv_encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) fail("CudaError", "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// single-dim affine index function: coefficient 1 on `d` only, no offset
bool is_dim(const Affine& f, int d) {
  if (f.c0 != 0) return false;
  for (size_t x = 0; x < f.coeff.size(); ++x)
    if (f.coeff[x] != (static_cast<int>(x) == d ? 1 : 0)) return false;
  return true;
}
// two-dim sum i_a + i_b
bool is_sum(const Affine& f, int a, int b) {
  if (f.c0 != 0) return false;
  for (size_t x = 0; x < f.coeff.size(); ++x)
    if (f.coeff[x] != ((static_cast<int>(x) == a || static_cast<int>(x) == b) ? 1 : 0)) return false;
  return true;
}
int only_dim(const Affine& f) {
  int d = -1;
  for (size_t x = 0; x < f.coeff.size(); ++x)
    if (f.coeff[x] != 0) {
      if (d >= 0 || f.coeff[x] != 1) return -1;
      d = static_cast<int>(x);
    }
  return f.c0 == 0 ? d : -1;
}

class ConvRoutine final : public Routine {
 public:
  ConvRoutine(const Problem& p, int ib, int fb) : p_(p), ib_(ib), fb_(fb) {}
  const char* family() const override { return "contraction"; }
  const char* bound() const override { return "tensor"; }
  int launches() const override { return fused_ ? 2 : bf16_ ? 3 : 1; }
  double flops() const override {
    return 2.0 * a_.N * a_.P * a_.Q * static_cast<double>(a_.K) * a_.R * a_.S * a_.C;
  }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  std::string describe() const override {
    std::ostringstream os;
    os << "{\"kernel\": \"" << (two_sm_ ? "tc_conv_2sm<" : fused_ ? "tc_conv_bf16f<" : bf16_ ? "tc_conv_bf16<" : "tc_conv_tf32<") << a_.K
       << ">\", \"math\": \"" << (bf16_ ? "bf16" : "tf32") << "\", \"M\": "
       << static_cast<int64_t>(a_.N) * a_.P * a_.Q << ", \"N\": " << a_.K << ", \"K\": " << a_.R * a_.S * a_.C
       << ", \"tile\": \"16 p x 8 q x " << a_.K << " k\", \"patch\": [" << a_.HP << ", " << a_.WQ << ", 32]"
       << ", \"taps_per_patch\": " << a_.R * a_.S << ", \"tiles\": " << static_cast<int64_t>(a_.N) * a_.pblocks * a_.qblocks
       << ", \"patch_stages\": " << (two_sm_ ? pst2_ : pst_) << ", \"patch_layout\": \"" << (a_.sw ? "pixel-major 128B swizzle" : "[c-group][p][q][4c] no swizzle")
       << "\", \"umma\": \"tcgen05.mma.cta_group::" << (two_sm_ ? "2" : "1") << ".kind::" << (bf16_ ? "f16 (bf16) M" : "tf32 M")
       << (two_sm_ ? 256 : 128) << "xN" << a_.K
       << (bf16_ ? "xK16" : "xK8") << ", A no-swizzle shifted descriptors, B resident 128B-swizzled\", \"smem\": " << smem_
       << (fused_ ? ", \"conversion\": \"input fp32 -> bf16 in-kernel (4 converter warps, bf16 + fp32 slot rings); to_bf16 of the filter per run\""
                  : bf16_ ? ", \"conversion\": \"to_bf16 of input and filter per run\"" : "")
       << ", \"epilogue\": \"" << (a_.tma_store ? "TMA tensor store (128B-swizzled 4p x 8q x 32k boxes)" : "smem transpose + st.global")
       << "\"}";
    return os.str();
  }

  bool setup(std::string* why) {
    const MdHom& e = p_.e;
    const Buf& I = e.in[static_cast<size_t>(ib_)];
    const Buf& F = e.in[static_cast<size_t>(fb_)];
    const Buf& O = e.out[0];
    // dims: n p q k (cc), r s c (pw), read off the views
    const int dn = only_dim(O.acc[0].idx[0]), dp = only_dim(O.acc[0].idx[1]), dq = only_dim(O.acc[0].idx[2]),
              dk = only_dim(O.acc[0].idx[3]);
    const int dr = only_dim(F.acc[0].idx[1]), ds = only_dim(F.acc[0].idx[2]), dc = only_dim(F.acc[0].idx[3]);
    if (dn < 0 || dp < 0 || dq < 0 || dk < 0 || dr < 0 || ds < 0 || dc < 0) return *why = "not an NHWC convolution", false;
    if (!is_dim(F.acc[0].idx[0], dk) || !is_dim(I.acc[0].idx[0], dn) || !is_sum(I.acc[0].idx[1], dp, dr) ||
        !is_sum(I.acc[0].idx[2], dq, ds) || !is_dim(I.acc[0].idx[3], dc))
      return *why = "not an NHWC convolution", false;
    auto sz = [&](int d) { return static_cast<int>(e.sizes[static_cast<size_t>(d)]); };
    a_.N = sz(dn), a_.P = sz(dp), a_.Q = sz(dq), a_.K = sz(dk), a_.R = sz(dr), a_.S = sz(ds), a_.C = sz(dc);
    const auto& ie = p_.in_ext[static_cast<size_t>(ib_)];  // [N][H][W][C]
    const auto& oe = p_.out_ext[0];                      // [N][P][Q][K]
    if (a_.K != 64) return *why = "conv instance: 64 output channels", false;
    bf16_ = p_.opt.math == Math::BF16;
    a_.ek = bf16_ ? 2 * CV_BKE : CV_BKE;
    if (a_.C % a_.ek || a_.Q % CV_TQ) return *why = "conv instance: C % (32 fp32 | 64 bf16), Q % 8", false;
    if (ie[3] != a_.C) return *why = "conv instance: input channel extent", false;
    a_.HP = CV_TP + a_.R - 1;
    a_.WQ = CV_TQ + a_.S - 1;
    a_.pblocks = (a_.P + CV_TP - 1) / CV_TP;
    a_.qblocks = a_.Q / CV_TQ;
    a_.on = oe[1] * oe[2] * oe[3];
    a_.op = oe[2] * oe[3];
    a_.oq = oe[3];
    a_.plane = static_cast<uint32_t>(a_.HP * a_.WQ * 16);
    const char* swap = std::getenv("MDHB_CONV_SWAP_LBO");
    a_.lbo = swap ? static_cast<uint32_t>(16 * a_.WQ) : a_.plane;
    a_.sbo = swap ? a_.plane : static_cast<uint32_t>(16 * a_.WQ);
    // pixel-major 128B-swizzled patch (shifted taps need no base offset: the
    // swizzle follows absolute smem address bits) -- bit-exact, measured
    // slower than the [c-group][p][q][4c] layout; selectable (MDHB_CONV_SW128=1)
    // pixel-major 128B-swizzled patch (rows = 128-byte pixel slices) is the
    // default; the [c-group][p][q][4c] no-swizzle layout stays selectable
    a_.sw = std::getenv("MDHB_CONV_NOSW") ? 0 : 1;
    a_.bo_mode = std::getenv("MDHB_CONV_BO") ? std::atoi(std::getenv("MDHB_CONV_BO")) : 0;
    if (a_.sw && (a_.WQ * 128) / 16 >= (1 << 14)) a_.sw = 0;
    const int ktiles = a_.R * a_.S * (a_.C / a_.ek);
    const size_t patch_slot = (8 * static_cast<size_t>(a_.plane) + 1023) / 1024 * 1024;
    pst_ = bf16_ ? 4 : 2;  // the bf16 filter is half the bytes: room for a deeper patch ring
    // epilogue: TMA tensor stores of 128B-swizzled 4 p x 8 q x 32 k boxes from
    // 8 KB per warp (needs 16-byte output strides), else the smem-transpose path
    a_.tma_store = (oe[3] * 4) % 16 == 0 && !std::getenv("MDHB_CONV_NO_TMA_STORE") ? 1 : 0;
    auto smem_of = [&](int pst) {
      const size_t epi = a_.tma_store ? 1024 + 4 * 8192 : 4 * (32 * 33 * 4 + 32 * 8);
      return static_cast<size_t>(ktiles) * a_.K * CV_BKE * 4 + pst * patch_slot + 256 + epi + 1024;
    };
    smem_ = smem_of(pst_);
    if (bf16_ && smem_ > 227 * 1024) smem_ = smem_of(pst_ = 2);
    if (smem_ > 227 * 1024 && a_.tma_store) {
      a_.tma_store = 0;
      smem_ = smem_of(pst_);
    }
    if (smem_ > 227 * 1024) return *why = "conv instance: filter + patches exceed shared memory", false;
    // CTA-pair instance: half the filter per CTA, the freed shared memory
    // deepens the patch ring (up to 6 stages)
    auto smem2_of = [&](int pst) {
      const size_t epi = a_.tma_store ? 1024 + 4 * 8192 : 4 * (32 * 33 * 4 + 32 * 8);
      return ((static_cast<size_t>(ktiles) * (a_.K / 2) * CV_BKE * 4 + 1023) / 1024 * 1024) + pst * patch_slot + 256 + epi + 1024;
    };
    pst2_ = 6;
    while (pst2_ > 3 && smem2_of(pst2_) > 227 * 1024) --pst2_;
    smem2_ = smem2_of(pst2_);
    // default for TF32 (0.121 vs 0.142 ms at conv2_x); the bf16 pair measured
    // slower than the single-CTA bf16 instance (selectable: MDHB_CONV_2SM=1)
    two_sm_ = smem2_ <= 227 * 1024 && !std::getenv("MDHB_CONV_1SM") && !std::getenv("MDHB_TC_1SM") &&
              (!bf16_ || std::getenv("MDHB_CONV_2SM"));
    if (a_.plane / 16 >= (1u << 14)) return *why = "conv instance: patch plane too large for a descriptor", false;
    // bf16 with the conversion fused into the conv kernel (default; measured
    // 0.102 vs 0.128 ms with the separate to_bf16 pass; MDHB_CONV_NO_BF16F=1 off)
    if (bf16_ && a_.sw && a_.tma_store && !std::getenv("MDHB_CONV_NO_BF16F") && !std::getenv("MDHB_CONV_2SM")) {
      const size_t slot = (static_cast<size_t>(a_.HP) * a_.WQ * 128 + 1023) / 1024 * 1024;
      // rings: bf16 slots + fp32 staging slots (128-byte aligned) and the
      // epilogue's per-warp buffer of 1 or 2 32-channel halves
      const size_t slot128 = static_cast<size_t>(a_.HP) * a_.WQ * 128;
      auto fsm = [&](int nslots, int eh) {
        return static_cast<size_t>(ktiles) * a_.K * 128 + nslots * slot128 + 256 + 1024 + 4 * 4096 * eh + 1024;
      };
      (void)slot;
      if (const char* v = std::getenv("MDHB_CONV_BF16F_CFG")) {  // "PST,FS,EH" (dev)
        std::sscanf(v, "%d,%d,%d", &pstf_, &fsf_, &ehf_);
      } else if (fsm(6, 1) <= 227 * 1024) {
        pstf_ = 3, fsf_ = 3, ehf_ = 1;  // measured: 3 + 3 0.091 ms, 2 + 4 0.101, 2 + 3 (2 halves) 0.104
      } else {
        pstf_ = 2, fsf_ = 3, ehf_ = 2;
      }
      smemf_ = fsm(pstf_ + fsf_, ehf_);
      fused_ = smemf_ <= 227 * 1024;
    }
    // input and filter extents for the tensor maps
    H_ = ie[1];
    W_ = ie[2];
    FK_ = static_cast<int64_t>(a_.R) * a_.S * a_.C;
    if (p_.in_ext[static_cast<size_t>(fb_)][1] != a_.R || p_.in_ext[static_cast<size_t>(fb_)][2] != a_.S ||
        p_.in_ext[static_cast<size_t>(fb_)][3] != a_.C)
      return *why = "conv instance: filter extents", false;
    return true;
  }

  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    const void* I = d_in[ib_];
    const void* F = d_in[fb_];
    const int sms0 = sm_count(p_.opt.device);
    if (fused_) {
      // the filter alone is converted (147 KB); the input is read as fp32 by the kernel
      const int64_t nf = FK_ * a_.K;
      if (!fbf_) MDHB_CUDA(cudaMalloc(&fbf_, static_cast<size_t>(nf) * 2 + 16));
      to_bf16<<<static_cast<unsigned>(std::min<int64_t>(8 * sms0, (nf / 8 + 255) / 256)), 256, 0, s>>>(
          static_cast<const float*>(F), static_cast<__nv_bfloat16*>(fbf_), nf / 8);
      MDHB_CUDA(cudaGetLastError());
      if (!bf_maps_) {
        cuuint64_t fd[2] = {static_cast<cuuint64_t>(FK_), static_cast<cuuint64_t>(a_.K)};
        cuuint64_t fs[1] = {static_cast<cuuint64_t>(FK_) * 2};
        cuuint32_t fbx[2] = {64, static_cast<cuuint32_t>(a_.K)};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = conv_encoder()(&mf_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, fbf_, fd, fs, fbx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (bf16 conv filter) failed");
        bf_maps_ = true;
      }
      if (I != last_i_) {
        // fp32 input, pixel-major {C, W, H, N}, box {32 c, WQ, HP, 1}, no swizzle: [HP][WQ][32] staging
        cuuint64_t d4[4] = {static_cast<cuuint64_t>(a_.C), static_cast<cuuint64_t>(W_), static_cast<cuuint64_t>(H_),
                            static_cast<cuuint64_t>(a_.N)};
        cuuint64_t s4[3] = {static_cast<cuuint64_t>(a_.C) * 4, static_cast<cuuint64_t>(W_ * a_.C) * 4,
                            static_cast<cuuint64_t>(H_ * W_ * a_.C) * 4};
        cuuint32_t b4[4] = {32, static_cast<cuuint32_t>(a_.WQ), static_cast<cuuint32_t>(a_.HP), 1};
        cuuint32_t e4[4] = {1, 1, 1, 1};
        CUresult r = conv_encoder()(&mi_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(I), d4, s4, b4, e4,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (fused bf16 conv input) failed");
        last_i_ = I;
      }
      last_f_ = F;
    } else if (bf16_) {
      // operand conversion (layout_de): fp32 views -> bf16 copies of the same layout
      const int64_t ni = static_cast<int64_t>(a_.N) * H_ * W_ * a_.C, nf = FK_ * a_.K;
      if (!ibf_) {
        MDHB_CUDA(cudaMalloc(&ibf_, static_cast<size_t>(ni) * 2));
        MDHB_CUDA(cudaMalloc(&fbf_, static_cast<size_t>(nf) * 2 + 16));
      }
      to_bf16<<<static_cast<unsigned>(std::min<int64_t>(8 * sms0, (ni / 8 + 255) / 256)), 256, 0, s>>>(
          static_cast<const float*>(I), static_cast<__nv_bfloat16*>(ibf_), ni / 8);
      to_bf16<<<static_cast<unsigned>(std::min<int64_t>(8 * sms0, (nf / 8 + 255) / 256)), 256, 0, s>>>(
          static_cast<const float*>(F), static_cast<__nv_bfloat16*>(fbf_), nf / 8);
      MDHB_CUDA(cudaGetLastError());
      if (!bf_maps_) {
        const int64_t C = a_.C;
        cuuint64_t dims[5] = {8, static_cast<cuuint64_t>(W_), static_cast<cuuint64_t>(H_), static_cast<cuuint64_t>(C / 8),
                              static_cast<cuuint64_t>(a_.N)};
        cuuint64_t strides[4] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(W_ * C) * 2, 16,
                                 static_cast<cuuint64_t>(H_ * W_ * C) * 2};
        cuuint32_t box[5] = {8, static_cast<cuuint32_t>(a_.WQ), static_cast<cuuint32_t>(a_.HP), 8, 1};
        cuuint32_t es[5] = {1, 1, 1, 1, 1};
        CUresult r;
        if (a_.sw) {
          // pixel-major: {C, W, H, N}, box {64 c, WQ, HP, 1}, 128-byte swizzle
          cuuint64_t d4[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W_), static_cast<cuuint64_t>(H_),
                              static_cast<cuuint64_t>(a_.N)};
          cuuint64_t s4[3] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(W_ * C) * 2,
                              static_cast<cuuint64_t>(H_ * W_ * C) * 2};
          cuuint32_t b4[4] = {64, static_cast<cuuint32_t>(a_.WQ), static_cast<cuuint32_t>(a_.HP), 1};
          r = conv_encoder()(&mi_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, ibf_, d4, s4, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
          r = conv_encoder()(&mi_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, ibf_, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (bf16 conv input) failed");
        cuuint64_t fd[2] = {static_cast<cuuint64_t>(FK_), static_cast<cuuint64_t>(a_.K)};
        cuuint64_t fs[1] = {static_cast<cuuint64_t>(FK_) * 2};
        cuuint32_t fbx[2] = {64, static_cast<cuuint32_t>(a_.K)};
        r = conv_encoder()(&mf_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, fbf_, fd, fs, fbx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (bf16 conv filter) failed");
        fbx[1] = static_cast<cuuint32_t>(a_.K / 2);  // the CTA pair's filter halves
        r = conv_encoder()(&mf2_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, fbf_, fd, fs, fbx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (bf16 conv filter half) failed");
        bf_maps_ = true;
      }
      last_i_ = I;
      last_f_ = F;
    }
    if (I != last_i_) {
      // 5-D view of I: {4 c, W, H, C/4 c-groups, N}; the c-group stride (16 B)
      // is smaller than the pixel stride -- TMA strides need not be ordered
      cuuint64_t dims[5] = {4, static_cast<cuuint64_t>(W_), static_cast<cuuint64_t>(H_),
                            static_cast<cuuint64_t>(a_.C / 4), static_cast<cuuint64_t>(a_.N)};
      cuuint64_t strides[4] = {static_cast<cuuint64_t>(a_.C) * 4, static_cast<cuuint64_t>(W_ * a_.C) * 4, 16,
                               static_cast<cuuint64_t>(H_ * W_ * a_.C) * 4};
      if (a_.sw) {
        // pixel-major: {C, W, H, N}, box {32 c, WQ, HP, 1}, 128-byte swizzle
        cuuint64_t d4[4] = {static_cast<cuuint64_t>(a_.C), static_cast<cuuint64_t>(W_), static_cast<cuuint64_t>(H_),
                            static_cast<cuuint64_t>(a_.N)};
        cuuint64_t s4[3] = {static_cast<cuuint64_t>(a_.C) * 4, static_cast<cuuint64_t>(W_ * a_.C) * 4,
                            static_cast<cuuint64_t>(H_ * W_ * a_.C) * 4};
        cuuint32_t b4[4] = {CV_BKE, static_cast<cuuint32_t>(a_.WQ), static_cast<cuuint32_t>(a_.HP), 1};
        cuuint32_t e4[4] = {1, 1, 1, 1};
        CUresult r4 = conv_encoder()(&mi_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(I), d4, s4, b4, e4,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r4 != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (conv input, swizzled) failed");
      }
      cuuint32_t box[5] = {4, static_cast<cuuint32_t>(a_.WQ), static_cast<cuuint32_t>(a_.HP), 8, 1};
      cuuint32_t es[5] = {1, 1, 1, 1, 1};
      CUresult r = a_.sw ? CUDA_SUCCESS
                         : conv_encoder()(&mi_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void*>(I), dims, strides, box,
                                          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (conv input) failed (" + std::to_string(static_cast<int>(r)) + ")");
      last_i_ = I;
    }
    if (F != last_f_) {
      cuuint64_t dims[2] = {static_cast<cuuint64_t>(FK_), static_cast<cuuint64_t>(a_.K)};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(FK_) * 4};
      cuuint32_t box[2] = {CV_BKE, static_cast<cuuint32_t>(a_.K)};
      cuuint32_t es[2] = {1, 1};
      CUresult r = conv_encoder()(&mf_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(F), dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (conv filter) failed (" + std::to_string(static_cast<int>(r)) + ")");
      box[1] = static_cast<cuuint32_t>(a_.K / 2);  // the CTA pair's filter halves
      r = conv_encoder()(&mf2_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(F), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (conv filter half) failed (" + std::to_string(static_cast<int>(r)) + ")");
      last_f_ = F;
    }
    if (a_.tma_store && d_out[0] != last_o_) {
      // O[N][P][Q][K] as {K, Q, P, N}, box {32 k, 8 q, 4 p, 1 n}, 128-byte swizzle
      const auto& oe = p_.out_ext[0];
      cuuint64_t dims[4] = {static_cast<cuuint64_t>(oe[3]), static_cast<cuuint64_t>(oe[2]), static_cast<cuuint64_t>(oe[1]),
                            static_cast<cuuint64_t>(oe[0])};
      cuuint64_t strides[3] = {static_cast<cuuint64_t>(oe[3]) * 4, static_cast<cuuint64_t>(oe[2] * oe[3]) * 4,
                               static_cast<cuuint64_t>(oe[1] * oe[2] * oe[3]) * 4};
      cuuint32_t box[4] = {32, CV_TQ, 4, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = conv_encoder()(&mo_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d_out[0], dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (conv output) failed (" + std::to_string(static_cast<int>(r)) + ")");
      last_o_ = d_out[0];
    }
    MarkScope mark(this, s);  // the convolution kernel below is the dominant one
    ConvArgs a = a_;
    a.O = static_cast<float*>(d_out[0]);
    const int sms = sm_count(p_.opt.device);
    if (two_sm_) {
      const int64_t tiles = static_cast<int64_t>(a_.N) * a_.pblocks * a_.qblocks;
      const int pairs = static_cast<int>(std::min<int64_t>(sms / 2, (tiles + 1) / 2));
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(static_cast<unsigned>(2 * pairs));
      lc.blockDim = dim3(192);
      lc.dynamicSmemBytes = smem2_;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      auto k = bf16_ ? (pst2_ >= 6 ? tc_conv_2sm<64, 6, true> : pst2_ == 5 ? tc_conv_2sm<64, 5, true>
                        : pst2_ == 4 ? tc_conv_2sm<64, 4, true> : tc_conv_2sm<64, 3, true>)
                     : (pst2_ >= 6 ? tc_conv_2sm<64, 6> : pst2_ == 5 ? tc_conv_2sm<64, 5>
                        : pst2_ == 4 ? tc_conv_2sm<64, 4> : tc_conv_2sm<64, 3>);
      MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2_)));
      MDHB_CUDA(cudaLaunchKernelEx(&lc, k, mi_, mf2_, mo_, a));
      return;
    }
    const int64_t tiles = static_cast<int64_t>(a_.N) * a_.pblocks * a_.qblocks;
    if (fused_) {
      auto kf = tc_conv_bf16f<64, 3, 3, 1>;
      if (pstf_ == 2 && fsf_ == 3 && ehf_ == 2) kf = tc_conv_bf16f<64, 2, 3, 2>;
      else if (pstf_ == 2 && fsf_ == 4 && ehf_ == 1) kf = tc_conv_bf16f<64, 2, 4, 1>;
      else if (pstf_ == 4 && fsf_ == 2 && ehf_ == 1) kf = tc_conv_bf16f<64, 4, 2, 1>;
      else if (pstf_ == 3 && fsf_ == 2 && ehf_ == 2) kf = tc_conv_bf16f<64, 3, 2, 2>;
      else if (!(pstf_ == 3 && fsf_ == 3 && ehf_ == 1)) fail("Unsupported", "fused bf16 conv: slot configuration");
      MDHB_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smemf_)));
      kf<<<static_cast<unsigned>(std::min<int64_t>(sms, tiles)), 320, smemf_, s>>>(mi_, mf_, mo_, a);
      MDHB_CUDA(cudaGetLastError());
      return;
    }
    auto k = bf16_ ? (pst_ == 4 ? tc_conv_tf32<64, true, 4> : tc_conv_tf32<64, true, 2>) : tc_conv_tf32<64>;
    MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
    k<<<static_cast<unsigned>(std::min<int64_t>(sms, tiles)), 192, smem_, s>>>(mi_, mf_, mo_, a);
    MDHB_CUDA(cudaGetLastError());
  }

 private:
  const Problem& p_;
  int ib_, fb_;
  ConvArgs a_{};
  int64_t H_ = 0, W_ = 0, FK_ = 0;
  size_t smem_ = 0, smem2_ = 0;
  bool two_sm_ = false;
  bool bf16_ = false, bf_maps_ = false;
  int pst_ = 2, pst2_ = 3, pstf_ = 2, fsf_ = 4, ehf_ = 1;
  bool fused_ = false;
  size_t smemf_ = 0;
  void *ibf_ = nullptr, *fbf_ = nullptr;

 public:
  ~ConvRoutine() override {
    if (ibf_) cudaFree(ibf_);
    if (fbf_) cudaFree(fbf_);
  }

 private:
  CUtensorMap mi_{}, mf_{}, mf2_{}, mo_{};
  const void* last_o_ = nullptr;
  const void* last_i_ = nullptr;
  const void* last_f_ = nullptr;
};

}  // namespace

bool nhwc_conv_shape(const Problem& p, int ib, int fb, ConvShape* cs, std::string* why) {
  const MdHom& e = p.e;
  if (e.D() != 7 || e.in.size() != 2 || e.out.size() != 1) return *why = "not a 7-dim two-input md_hom", false;
  const Buf& I = e.in[static_cast<size_t>(ib)];
  const Buf& F = e.in[static_cast<size_t>(fb)];
  const Buf& O = e.out[0];
  if (I.rank != 4 || F.rank != 4 || O.rank != 4) return *why = "not an NHWC convolution", false;
  const int dn = only_dim(O.acc[0].idx[0]), dp = only_dim(O.acc[0].idx[1]), dq = only_dim(O.acc[0].idx[2]),
            dk = only_dim(O.acc[0].idx[3]);
  const int dr = only_dim(F.acc[0].idx[1]), ds = only_dim(F.acc[0].idx[2]), dc = only_dim(F.acc[0].idx[3]);
  if (dn < 0 || dp < 0 || dq < 0 || dk < 0 || dr < 0 || ds < 0 || dc < 0) return *why = "not an NHWC convolution", false;
  if (!is_dim(F.acc[0].idx[0], dk) || !is_dim(I.acc[0].idx[0], dn) || !is_sum(I.acc[0].idx[1], dp, dr) ||
      !is_sum(I.acc[0].idx[2], dq, ds) || !is_dim(I.acc[0].idx[3], dc))
    return *why = "not an NHWC convolution", false;
  auto sz = [&](int d) { return static_cast<int>(e.sizes[static_cast<size_t>(d)]); };
  cs->ib = ib;
  cs->fb = fb;
  cs->N = sz(dn), cs->P = sz(dp), cs->Q = sz(dq), cs->K = sz(dk), cs->R = sz(dr), cs->S = sz(ds), cs->C = sz(dc);
  const auto& ie = p.in_ext[static_cast<size_t>(ib)];
  const auto& fe = p.in_ext[static_cast<size_t>(fb)];
  cs->H = ie[1];
  cs->W = ie[2];
  cs->oe = p.out_ext[0];
  if (ie[3] != cs->C || fe[0] != cs->K || fe[1] != cs->R || fe[2] != cs->S || fe[3] != cs->C || cs->oe[3] != cs->K)
    return *why = "conv extents", false;
  return true;
}

std::unique_ptr<Routine> make_tc_conv(const Problem& p, const Groups& g, std::string* why) {
  if (std::getenv("MDHB_TC_NO_CONV")) return nullptr;
  const MdHom& e = p.e;
  if (e.D() != 7 || e.in.size() != 2 || e.out.size() != 1) return nullptr;
  // the input is the operand with a 2-dim index function; the filter the other
  for (int ib : {g.a_buf, g.b_buf}) {
    const int fb = ib == g.a_buf ? g.b_buf : g.a_buf;
    if (e.in[static_cast<size_t>(ib)].rank != 4 || e.in[static_cast<size_t>(fb)].rank != 4 || e.out[0].rank != 4) continue;
    auto r = std::make_unique<ConvRoutine>(p, ib, fb);
    std::string w;
    if (r->setup(&w)) return r;
    *why = w;
  }
  return nullptr;
}

}  // namespace ctr
}  // namespace mdhb
