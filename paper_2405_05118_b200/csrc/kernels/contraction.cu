// Contraction family: md_homs of the form
//
//     out(m, n) = sum_k  A[a0 + a(m,k)] * B[b0 + b(k,n)]        (pw:+ over k)
//
// where the scalar function is in(1,1) * in(2,1), the point-wise dims (K)
// fold with +, the concatenation dims split into M (read by A only) and N
// (read by B only), and the output access is a permutation of the cc dims.
// This covers MatVec, MatMul, the ResNet-50 FC layer, MCC (implicit GEMM
// over NHWC: M = (n,p,q), N = k, K = (r,s,c)) and the CCSD(T) triples
// contraction (M = (a,b,d), N = (c,e,f), K = g) -- BASELINE configs 1, 3-5.
//
// Every affine view linearises to  off = c0 + sum_d c_d * i_d  (the
// reference's AccessPlan, engine.cpp:266-286), so the A/B/C addresses split
// additively into per-tile, per-local-row/column and per-k parts.  The
// planner precomputes those parts as small int32 tables; the kernels never
// see the md_hom, only tables -- which is what lets one template serve every
// view permutation (TCCG-style contractions without transposes).
//
// Tiling follows the Table-1 levels of the B200 ASM:
//   SMX : a box tile of the M dims (BM cells) x a box of the N dims (BN)
//   DM  : the CTA's sequential k-tile loop (K / BK steps)
//   CC  : (BM/8) x (BN/8) threads
//   SM  : A and B k-tiles (BK = 8) double-buffered in shared memory
//   RM  : an 8 x 8 register tile per thread (two 4-row x two 4-col quads)
// Re-composition of K happens entirely in registers (each output cell has a
// single writer), so the store is a plain coalesced write of C.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <set>
#include <sstream>

#include "../plan.hpp"
#include "contraction_common.hpp"
#include "tc_gemm.cuh"

namespace mdhb {
namespace {
using namespace ctr;

constexpr int BK = 8;
enum { LD_SCALAR = 0, LD_K4 = 1, LD_MN4 = 2 };  // vector direction of 16-byte loads

struct GemmArgs {
  const float* A;
  const float* B;
  float* C;
  const int32_t *tAm, *tCm, *tBn, *tCn;  // per tile (A/C row part, B/C column part)
  const int32_t *am, *cm, *bn, *cn;      // per local row / column of a tile
  const int32_t *ak, *bk;                // per k
  int K, tilesM, tilesN;
  int sak, sbk;  // per-k strides inside one k-tile (sgemm_pipe: ak[k0 + j] = ak[k0] + j * sak)
  int klin;      // sgemm_pipe: ak[k] = k * sak and bk[k] = k * sbk for EVERY k -- no per-k-tile table read
  int group_m;   // row tiles per raster group (Table-1: SMX parts of the innermost M dim; 0 = 8)
};

struct GemvArgs {
  const float* A;
  const float* x;
  float* y;
  const int32_t *am, *cm;
  int64_t M;
  int K;
};

template <int BM, int BN, int AMODE, int BMODE, bool CVEC>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 256 / ((BM / 8) * (BN / 8)) * 2) sgemm_tiled(GemmArgs g) {
  constexpr int NT = (BM / 8) * (BN / 8);
  constexpr int TXN = BN / 8;
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % TXN, ty = tid / TXN;

  // grouped raster: GROUP_M row-tiles sweep the N tiles together (L2 reuse)
  const int GROUP_M = g.group_m > 0 ? g.group_m : 8;
  const int x = blockIdx.x;
  const int per_group = GROUP_M * g.tilesN;
  const int first_m = (x / per_group) * GROUP_M;
  const int gsz = min(g.tilesM - first_m, GROUP_M);
  const int tm = first_m + (x % per_group) % gsz;
  const int tn = (x % per_group) / gsz;

  const float* __restrict__ A = g.A + g.tAm[tm];
  const float* __restrict__ B = g.B + g.tBn[tn];

  // ---- per-thread load slots (fixed across k-tiles)
  constexpr int AG = AMODE == LD_SCALAR ? BM * BK : BM * BK / 4;  // load groups per tile
  constexpr int BG = BMODE == LD_SCALAR ? BN * BK : BN * BK / 4;
  constexpr int AP = (AG + NT - 1) / NT, BP = (BG + NT - 1) / NT;
  constexpr int AW = AMODE == LD_SCALAR ? 1 : 4, BW = BMODE == LD_SCALAR ? 1 : 4;
  int a_row[AP], a_k[AP], b_col[BP], b_k[BP];
  int32_t a_off[AP], b_off[BP];
#pragma unroll
  for (int p = 0; p < AP; ++p) {
    int gi = tid + p * NT;
    if (AMODE == LD_K4) { a_row[p] = gi >> 1; a_k[p] = (gi & 1) * 4; }
    else if (AMODE == LD_MN4) { a_k[p] = gi / (BM / 4); a_row[p] = (gi % (BM / 4)) * 4; }
    else { a_k[p] = gi / BM; a_row[p] = gi % BM; }
    a_off[p] = gi < AG ? g.am[a_row[p]] : 0;
  }
#pragma unroll
  for (int p = 0; p < BP; ++p) {
    int gi = tid + p * NT;
    if (BMODE == LD_K4) { b_col[p] = gi >> 1; b_k[p] = (gi & 1) * 4; }
    else if (BMODE == LD_MN4) { b_k[p] = gi / (BN / 4); b_col[p] = (gi % (BN / 4)) * 4; }
    else { b_k[p] = gi / BN; b_col[p] = gi % BN; }
    b_off[p] = gi < BG ? g.bn[b_col[p]] : 0;
  }
  float ra[AP][AW], rb[BP][BW];

  auto load = [&](int k0) {
#pragma unroll
    for (int p = 0; p < AP; ++p) {
      if (tid + p * NT >= AG) continue;
      const float* src = A + a_off[p] + g.ak[k0 + a_k[p]];
      if (AW == 4) {
        float4 v = __ldg(reinterpret_cast<const float4*>(src));
        ra[p][0] = v.x; ra[p][AW > 1 ? 1 : 0] = v.y; ra[p][AW > 2 ? 2 : 0] = v.z; ra[p][AW > 3 ? 3 : 0] = v.w;
      } else {
        ra[p][0] = __ldg(src);
      }
    }
#pragma unroll
    for (int p = 0; p < BP; ++p) {
      if (tid + p * NT >= BG) continue;
      const float* src = B + b_off[p] + g.bk[k0 + b_k[p]];
      if (BW == 4) {
        float4 v = __ldg(reinterpret_cast<const float4*>(src));
        rb[p][0] = v.x; rb[p][BW > 1 ? 1 : 0] = v.y; rb[p][BW > 2 ? 2 : 0] = v.z; rb[p][BW > 3 ? 3 : 0] = v.w;
      } else {
        rb[p][0] = __ldg(src);
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int p = 0; p < AP; ++p) {
      if (tid + p * NT >= AG) continue;
      if (AMODE == LD_K4) {
#pragma unroll
        for (int j = 0; j < AW; ++j) As[buf][a_k[p] + j][a_row[p]] = ra[p][j];
      } else if (AMODE == LD_MN4) {
        *reinterpret_cast<float4*>(&As[buf][a_k[p]][a_row[p]]) = make_float4(ra[p][0], ra[p][AW > 1 ? 1 : 0], ra[p][AW > 2 ? 2 : 0], ra[p][AW > 3 ? 3 : 0]);
      } else {
        As[buf][a_k[p]][a_row[p]] = ra[p][0];
      }
    }
#pragma unroll
    for (int p = 0; p < BP; ++p) {
      if (tid + p * NT >= BG) continue;
      if (BMODE == LD_K4) {
#pragma unroll
        for (int j = 0; j < BW; ++j) Bs[buf][b_k[p] + j][b_col[p]] = rb[p][j];
      } else if (BMODE == LD_MN4) {
        *reinterpret_cast<float4*>(&Bs[buf][b_k[p]][b_col[p]]) = make_float4(rb[p][0], rb[p][BW > 1 ? 1 : 0], rb[p][BW > 2 ? 2 : 0], rb[p][BW > 3 ? 3 : 0]);
      } else {
        Bs[buf][b_k[p]][b_col[p]] = rb[p][0];
      }
    }
  };

  float2 acc[8][4];  // column pairs, FFMA2 (see sgemm_pipe)
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);

  const int nk = g.K / BK;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][BM / 2 + ty * 4]);
      float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][BN / 2 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), make_float2(b[2 * j], b[2 * j + 1]), acc[i][j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }

  // ---- epilogue: each C cell has exactly one writer
  float* __restrict__ C = g.C + g.tCm[tm] + g.tCn[tn];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = i < 4 ? ty * 4 + i : BM / 2 + ty * 4 + (i - 4);
    float* crow = C + g.cm[r];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h * (BN / 2) + tx * 4;
      if (CVEC) {
        *reinterpret_cast<float4*>(crow + g.cn[c]) =
            make_float4(acc[i][h * 2].x, acc[i][h * 2].y, acc[i][h * 2 + 1].x, acc[i][h * 2 + 1].y);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) crow[g.cn[c + j]] = j & 1 ? acc[i][h * 2 + j / 2].y : acc[i][h * 2 + j / 2].x;
      }
    }
  }
}

// y[cm[m]] = sum_k A[am[m] + k] * x[k]  -- MatVec (N = 1), rows contiguous in k.
// One warp owns ROWS rows and streams them with 16-byte loads, sharing each
// x chunk across its rows; the K reduction is a warp shuffle (CC -> RM).
template <int ROWS>
__global__ void __launch_bounds__(128) gemv_rows(GemvArgs g) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t m0 = warp * ROWS;
  if (m0 >= g.M) return;
  const float4* x4 = reinterpret_cast<const float4*>(g.x);
  const float4* rows[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
    rows[r] = reinterpret_cast<const float4*>(g.A + g.am[(m0 + r < g.M) ? (m0 + r) : (g.M - 1)]);
  float acc[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) acc[r] = 0.f;
  const int n4 = g.K / 4;
  constexpr int U = 4;
  int k = lane;
  for (; k + 32 * (U - 1) < n4; k += 32 * U) {
    float4 xv[U], av[ROWS][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xv[u] = __ldg(x4 + k + 32 * u);
#pragma unroll
      for (int r = 0; r < ROWS; ++r) av[r][u] = __ldcs(rows[r] + k + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        acc[r] = fmaf(av[r][u].x, xv[u].x, acc[r]);
        acc[r] = fmaf(av[r][u].y, xv[u].y, acc[r]);
        acc[r] = fmaf(av[r][u].z, xv[u].z, acc[r]);
        acc[r] = fmaf(av[r][u].w, xv[u].w, acc[r]);
      }
  }
  for (; k < n4; k += 32) {
    float4 xv = __ldg(x4 + k);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      float4 av = __ldcs(rows[r] + k);
      acc[r] = fmaf(av.x, xv.x, acc[r]);
      acc[r] = fmaf(av.y, xv.y, acc[r]);
      acc[r] = fmaf(av.z, xv.z, acc[r]);
      acc[r] = fmaf(av.w, xv.w, acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], s);
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
      if (m0 + r < g.M) g.y[g.cm[m0 + r]] = acc[r];
  }
}


// Skinny contraction (small M, e.g. the ResNet-50 FC layer 16 x 1000 x 2048):
// a 128-row tile would idle 7/8 of its rows, so K is split across CTAs
// instead.  Thread t of CTA (nt, ks) owns column n = nt*256 + t for all M
// rows (M accumulators in registers) over the k-slice ks; B rows stream
// coalesced along n, the A slice is staged once in shared memory and read
// as broadcasts.  Partial sums land in a [splits][M][N] scratch and a second
// pass folds them in fixed split order (deterministic).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn tensor_map_encoder() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    fail("CudaError", "cuTensorMapEncodeTiled unavailable");
  return reinterpret_cast<EncodeFn>(p);
}

struct SkinnyArgs {
  const float* A;
  const float* B;
  float* part;
  float* C;
  const int32_t *am, *ak, *bk, *bn, *cm, *cn;
  int M, N, K, ks;  // ks = k per split
  int splits;
  int64_t sak, sbk;  // affine k strides of A and B (skinny_cluster)
  int* counter;      // per N strip arrival counters (skinny_cluster<..., LAST>)
  // aff = 1: am[m] = m sam, bn[n] = n sbn, cm[m] = m scm, cn[n] = n scn -- the
  // offsets are computed, so no table read (an L2 round trip) sits before the
  // first copy or the last store (skinny_cluster)
  int64_t sam, sbn, scm, scn;
  int aff;
  // txfold = 1 (opt-in MDHB_SKINNY_TXFOLD=1; 5.68 vs 5.64 us, DESIGN): the
  // slices' pushes are st.async remote stores that complete bytes on the
  // owner's mbarrier; each owner waits for its own inbox only (no second
  // cluster-wide barrier)
  int txfold;
};

template <int MT>
__global__ void __launch_bounds__(256) skinny_partial(SkinnyArgs g) {
  extern __shared__ float sA[];  // [M][ks]
  const int n = blockIdx.x * 256 + threadIdx.x;
  const int k0 = blockIdx.y * g.ks;
  for (int i = threadIdx.x; i < g.M * g.ks; i += 256) {
    int m = i / g.ks, k = i - m * g.ks;
    sA[i] = __ldg(g.A + g.am[m] + g.ak[k0 + k]);
  }
  __syncthreads();
  if (n >= g.N) return;
  float acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m] = 0.f;
  const float* Bn = g.B + g.bn[n];
#pragma unroll 4
  for (int k = 0; k < g.ks; ++k) {
    const float b = __ldcs(Bn + g.bk[k0 + k]);
#pragma unroll
    for (int m = 0; m < MT; ++m)
      if (m < g.M) acc[m] = fmaf(sA[m * g.ks + k], b, acc[m]);
  }
  float* out = g.part + static_cast<int64_t>(blockIdx.y) * g.M * g.N;
#pragma unroll
  for (int m = 0; m < MT; ++m)
    if (m < g.M) out[m * g.N + n] = acc[m];
}

__global__ void __launch_bounds__(256) skinny_fold(SkinnyArgs g) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= g.M * g.N) return;
  const int m = i / g.N, n = i - m * g.N;
  float s = g.part[i];
  for (int sp = 1; sp < g.splits; ++sp) s += g.part[static_cast<int64_t>(sp) * g.M * g.N + i];
  g.C[g.cm[m] + g.cn[n]] = s;
}


// Skinny contraction v2 (vector operands): K is split across the CS CTAs of a
// thread-block cluster and re-composed in distributed shared memory, so no
// partial sums ever reach global memory and there is one launch per run.
//   SMX : blockIdx.x = a strip of NW = 32 columns of N; blockIdx.y = one of
//         CS k-slices (the cluster), KS = K / CS rows of B per CTA
//   SM  : the CTA's whole B slice [KS][32] and A slice [MT][KS] land in shared
//         memory through 16-byte cp.async in 4 commit groups (stages), so
//         compute on stage s overlaps the flight of stages s+1..3
//   CC  : 256 threads = 4 k-quarters x 8 m-groups x 8 column quads
//   RM  : MT/8 rows x 4 columns per thread, 4 k per step (float4 A reads)
// Re-composition of K: k-quarters meet in shared memory (WRP -> SM), the CS
// slices meet over DSMEM (SM -> cluster), each CTA folding 1/CS of the
// outputs in fixed slice order -- deterministic, single writer per C cell.
//
// LAST = true (no cluster): the k-slices meet in global memory instead -- each
// CTA writes its folded [MT][NW] partial to the plan's workspace, fences, and
// bumps the strip's arrival counter; the CTA that arrives last folds the
// strip's partials in slice order (deterministic, single writer) and resets
// the counter for the next run.  CTAs that finish early leave at once (no
// cluster barrier waits on the slowest slice).
#ifndef MDHB_FC_BISECT
#define MDHB_FC_BISECT 0  // development bisection builds only (tools/fc_bisect.sh): 1 no FMAs, 2 no cluster fold, 4 no loads
#endif
// TMAB: the B slice lands by one 2-D TMA tensor copy per stage ({32 columns,
// KS/4 rows} boxes, zero fill past N) on an mbarrier instead of 8 16-byte
// cp.async per thread; A keeps cp.async.
template <int MT, int KS, bool LAST = false, int NW = 32, int MG = 8, bool TMAB = false>
__global__ void __launch_bounds__(256) skinny_cluster(SkinnyArgs g, const __grid_constant__ CUtensorMap tmb) {
  // NW columns per CTA strip: 256 threads = KQN k-parts x MG m-groups x NW/4
  // column quads; thread rows mg + MG i (i < R) -- one warp's MG row groups
  // read distinct bank quads of the KS + 4 pitch.  MG = 4 (R = 4 rows per
  // thread) halves the shared-memory wavefronts per FMA against MG = 8.
  constexpr int CQN = NW / 4, KQN = 256 / (MG * CQN);
  constexpr int NSTG = 4, R = MT / MG, SL = KS / NSTG, KQ = SL / KQN, AKQ = SL / 4, AP = KS + 4;
  static_assert(KQN >= 1 && KQ % 4 == 0, "k per thread per stage must be a multiple of 4");
  extern __shared__ __align__(1024) float sm[];
  float* Bs = sm;                 // [KS][NW]
  float* As = Bs + KS * NW;       // [MT][KS + 4]
  float* red = As + MT * AP;      // [KQN][MT][NW]   k-part partials
  float* inbox = red + KQN * MT * NW;  // [CS][MT*NW/CS]  slices pushed by the cluster's CTAs
  const int tid = threadIdx.x;
  const int kq = tid / (MG * CQN), mg = (tid / CQN) % MG, cq = tid % CQN;
  const int n0 = blockIdx.x * NW;
  const int kbase = blockIdx.y * KS;
  constexpr bool TB = TMAB && !(MDHB_FC_BISECT & 4);
  // stage barriers after the inbox (dynamic smem: Bs, the TMA destination,
  // stays at the 1024-byte aligned base -- no static smem shifts it)
  uint64_t* bbar = reinterpret_cast<uint64_t*>(inbox + MT * NW);
  if (TB) {
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < NSTG; ++s) tc::mbar_init(&bbar[s], 1);
      tc::fence_barrier_init();
    }
    __syncthreads();
  }
  // every CTA of the cluster must be running before anyone writes into its
  // shared memory: arrive now, wait just before the DSMEM pushes
  uint64_t* fbar = bbar + NSTG;  // txfold: this CTA's inbox barrier
  if (!LAST && !(MDHB_FC_BISECT & 2)) {
    if (g.txfold) {
      if (tid == 0) {
        uint32_t ncta;
        asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
        tc::mbar_init(fbar, 1);
        tc::fence_barrier_init();
        tc::mbar_arrive_expect_tx(fbar, (MT * NW / ncta) * 4 * ncta);  // every slice pushes per floats
      }
      // release: the barrier init is visible to the cluster before any push
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    } else {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    }
  }
  // ---- issue every stage's copies up front (NSTG commit groups).  k offsets
  // are affine (g.sak == 1, g.sbk per k), so one table read per row / column
  // precedes the copies and nothing serialises the issue on load latency.
  const int bq = tid % (NW / 4), bk0 = tid / (NW / 4);
  const bool bok = n0 + bq * 4 < g.N;
  const float* bsrc = g.B + (bok ? (g.aff ? (n0 + bq * 4) * g.sbn : g.bn[n0 + bq * 4]) + static_cast<int64_t>(kbase) * g.sbk : 0);
  constexpr int ACH = (MT * AKQ + 255) / 256;
  const float* asrc[ACH];
  int adst[ACH];
  bool aok[ACH];
#pragma unroll
  for (int i = 0; i < ACH; ++i) {
    const int c = tid + 256 * i, m = c / AKQ;
    aok[i] = c < MT * AKQ && m < g.M;
    adst[i] = m * AP + (c % AKQ) * 4;
    asrc[i] = g.A + (aok[i] ? (g.aff ? m * g.sam : g.am[m]) + kbase + (c % AKQ) * 4 : 0);
  }
  // programmatic dependent launch: everything above touches only plan-owned
  // tables; the operands may be produced by the previous kernel in the
  // stream, so wait for it here (no-op without the PDL launch attribute) and
  // let the next kernel's prologue start.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
#pragma unroll
  for (int s = 0; s < NSTG; ++s) {
#pragma unroll
    for (int i = 0; i < ACH; ++i)
      if (!(MDHB_FC_BISECT & 4) && tid + 256 * i < MT * AKQ)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(As + adst[i] + s * SL))),
                     "l"(asrc[i] + s * SL), "r"(aok[i] ? 16 : 0));
    if (TB && tid == 0) {
      const int c[2] = {n0, kbase + s * SL};
      tc::mbar_arrive_expect_tx(&bbar[s], SL * NW * 4);
      tc::tma_load(Bs + s * SL * NW, &tmb, &bbar[s], 2, c);
    }
#pragma unroll
    for (int k = s * SL + bk0; k < (s + 1) * SL && !(MDHB_FC_BISECT & 4) && !TB; k += 256 / (NW / 4))
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(Bs + k * NW + bq * 4))),
                   "l"(bsrc + static_cast<int64_t>(k) * g.sbk), "r"(bok ? 16 : 0));
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // column pairs updated by FFMA2 (two fma.rn per instruction, bit-identical
  // to scalar FFMA): half the FMA instructions
  float2 acc[R][2];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  auto stage = [&](int s) {
    if (MDHB_FC_BISECT & 1) return;
    const int k0 = s * SL + kq * KQ;
#pragma unroll
    for (int k = k0; k < k0 + KQ; k += 4) {
      float a[R][4];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(As + (mg + MG * i) * AP + k);
        a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float4 b = *reinterpret_cast<const float4*>(Bs + (k + kk) * NW + cq * 4);
#pragma unroll
        for (int i = 0; i < R; ++i) {
          acc[i][0] = __ffma2_rn(make_float2(a[i][kk], a[i][kk]), make_float2(b.x, b.y), acc[i][0]);
          acc[i][1] = __ffma2_rn(make_float2(a[i][kk], a[i][kk]), make_float2(b.z, b.w), acc[i][1]);
        }
      }
    }
  };
  asm volatile("cp.async.wait_group 3;" ::: "memory");
  if (TB) tc::mbar_wait(&bbar[0], 0);
  __syncthreads();
  stage(0);
  asm volatile("cp.async.wait_group 2;" ::: "memory");
  if (TB) tc::mbar_wait(&bbar[1], 0);
  __syncthreads();
  stage(1);
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  if (TB) tc::mbar_wait(&bbar[2], 0);
  __syncthreads();
  stage(2);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (TB) tc::mbar_wait(&bbar[3], 0);
  __syncthreads();
  stage(3);
  // ---- k-quarters meet in shared memory (fixed order)
#pragma unroll
  for (int i = 0; i < R; ++i)
    *reinterpret_cast<float4*>(red + (kq * MT + mg + MG * i) * NW + cq * 4) = make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
  __syncthreads();
  if (LAST) {
    // ---- k-slices meet in global memory, the last arrival folds
    __shared__ int last;
    float* mine = g.part + (static_cast<int64_t>(blockIdx.x) * gridDim.y + blockIdx.y) * (MT * NW);
    for (int o = tid; o < MT * NW; o += 256) {
      float v = red[o];
#pragma unroll
      for (int q = 1; q < KQN; ++q) v += red[q * MT * NW + o];
      mine[o] = v;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(g.counter + blockIdx.x, 1) == static_cast<int>(gridDim.y) - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const float* strip = g.part + static_cast<int64_t>(blockIdx.x) * gridDim.y * (MT * NW);
    for (int o = tid; o < MT * NW; o += 256) {
      float v = 0.f;
      for (int c = 0; c < static_cast<int>(gridDim.y); ++c) v += __ldcg(strip + c * (MT * NW) + o);
      const int m = o / NW, n = n0 + o % NW;
      if (m < g.M && n < g.N) g.C[g.aff ? m * g.scm + n * g.scn : g.cm[m] + g.cn[n]] = v;
    }
    if (tid == 0) g.counter[blockIdx.x] = 0;  // ready for the next run (stream order)
    return;
  }
  // ---- k-slices meet over DSMEM: output o belongs to CTA o / per of the
  // cluster; every CTA pushes its partial of o into slot [my rank] of the
  // owner's inbox (remote stores, no round trips), one cluster barrier, then
  // each owner folds its inbox in rank order -- deterministic.
  if (MDHB_FC_BISECT & 2) {  // no cluster fold (wrong results): slice 0 writes its own partial
    if (blockIdx.y == 0)
      for (int o = tid; o < MT * NW; o += 256) {
        const int m = o / NW, n = n0 + o % NW;
        if (m < g.M && n < g.N) g.C[g.aff ? m * g.scm + n * g.scn : g.cm[m] + g.cn[n]] = red[o];
      }
    return;
  }
  uint32_t rank, cs;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  const int per = MT * NW / static_cast<int>(cs);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  for (int o = tid; o < MT * NW; o += 256) {
    float v = red[o];
#pragma unroll
    for (int q = 1; q < KQN; ++q) v += red[q * MT * NW + o];
    const uint32_t owner = static_cast<uint32_t>(o / per);
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(inbox + rank * per + o % per));
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(owner));
    if (g.txfold) {
      uint32_t rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(tc::smem_u32(fbar)), "r"(owner));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(remote), "f"(v), "r"(rbar)
                   : "memory");
    } else {
      asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
    }
  }
  if (g.txfold) {
    if (tid >= per) return;  // the owner's threads wait for its inbox bytes
    tc::mbar_wait(fbar, 0);
  } else {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  for (int t = tid; t < per; t += 256) {
    float s = 0.f;
    for (uint32_t c = 0; c < cs; ++c) s += inbox[c * per + t];
    const int o = static_cast<int>(rank) * per + t;
    const int m = o / NW, n = n0 + o % NW;
    if (m < g.M && n < g.N) g.C[g.aff ? m * g.scm + n * g.scn : g.cm[m] + g.cn[n]] = s;
  }
}


// MatVec v2: a CTA of 8 warps owns 2 rows; warp w reduces K-slice w, every
// lane issues all of its 2 x V 16-byte loads of M (and V of x) before the
// first FMA, so a full 64 MiB matrix is in flight after one pass of CTAs.
// Partial dot products meet in shared memory (WRP combine in SM, the
// CUDA+WRP model rule) and one lane per row writes the result.
template <int V>
__global__ void __launch_bounds__(256) gemv_split(GemvArgs g) {
  constexpr int ROWS = 2;
  __shared__ float part[8][ROWS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * ROWS;
  const int kq = g.K / 8;  // floats per warp slice
  const float4* x4 = reinterpret_cast<const float4*>(g.x + warp * kq);
  float4 av[ROWS][V], xv[V];
  int32_t amr[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) amr[r] = g.am[m0 + r < g.M ? m0 + r : g.M - 1];  // plan-owned table
  asm volatile("griddepcontrol.wait;" ::: "memory");  // operands may come from the previous kernel (PDL)
  asm volatile("griddepcontrol.launch_dependents;");
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const float4* row = reinterpret_cast<const float4*>(g.A + amr[r] + warp * kq);
#pragma unroll
    for (int u = 0; u < V; ++u) av[r][u] = __ldcs(row + lane + 32 * u);
  }
#pragma unroll
  for (int u = 0; u < V; ++u) xv[u] = __ldg(x4 + lane + 32 * u);
  float acc[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    acc[r] = 0.f;
#pragma unroll
    for (int u = 0; u < V; ++u) {
      acc[r] = fmaf(av[r][u].x, xv[u].x, acc[r]);
      acc[r] = fmaf(av[r][u].y, xv[u].y, acc[r]);
      acc[r] = fmaf(av[r][u].z, xv[u].z, acc[r]);
      acc[r] = fmaf(av[r][u].w, xv[u].w, acc[r]);
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], s);
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < ROWS; ++r) part[warp][r] = acc[r];
  }
  __syncthreads();
  if (threadIdx.x < ROWS && m0 + threadIdx.x < g.M) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += part[w][threadIdx.x];
    g.y[g.cm[m0 + threadIdx.x]] = s;
  }
}


// FFMA template v2 (vector operand modes): global -> shared with cp.async
// (16-byte LDGSTS, no register staging, no spills), a 4-stage ring, one
// barrier per k-tile.  A in K4 mode is kept [m][k] in shared memory and
// read as one 16-byte vector per row per 4 k; MN4 operands are [k][rows].
// The register tile and epilogue are those of sgemm_tiled.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <bool AK4, bool CVEC, int TN>
__global__ void __launch_bounds__(256, TN == 8 ? 2 : 1) sgemm_async(GemmArgs g) {
  constexpr int BM = 128, BN = 16 * TN, ST = 4, NQ = TN / 4;  // NQ column quads per thread
  __shared__ __align__(16) float As[ST][BM * BK];
  __shared__ __align__(16) float Bs[ST][BK * BN];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int GROUP_M = g.group_m > 0 ? g.group_m : 8;
  const int x = blockIdx.x;
  const int per_group = GROUP_M * g.tilesN;
  const int first_m = (x / per_group) * GROUP_M;
  const int gsz = min(g.tilesM - first_m, GROUP_M);
  const int tm = first_m + (x % per_group) % gsz;
  const int tn = (x % per_group) / gsz;
  const float* __restrict__ A = g.A + g.tAm[tm];
  const float* __restrict__ B = g.B + g.tBn[tn];
  int a_r, a_k, a_dst;
  if (AK4) { a_r = tid >> 1; a_k = (tid & 1) * 4; a_dst = a_r * BK + a_k; }
  else { a_k = tid >> 5; a_r = (tid & 31) * 4; a_dst = a_k * BM + a_r; }
  constexpr int BCH = BK * BN / 4 / 256;  // 16-byte B chunks per thread
  int b_k[BCH], b_dst[BCH];
  const float* b_src[BCH];
#pragma unroll
  for (int c = 0; c < BCH; ++c) {
    const int ch = tid + c * 256;
    b_k[c] = ch / (BN / 4);
    const int col = (ch % (BN / 4)) * 4;
    b_dst[c] = b_k[c] * BN + col;
    b_src[c] = B + g.bn[col];
  }
  const float* a_src = A + g.am[a_r];
  const int nk = g.K / BK;
  auto issue = [&](int kt) {
    const int s = kt % ST, k0 = kt * BK;
    cp_async16(&As[s][a_dst], a_src + g.ak[k0 + a_k]);
#pragma unroll
    for (int c = 0; c < BCH; ++c) cp_async16(&Bs[s][b_dst[c]], b_src[c] + g.bk[k0 + b_k[c]]);
  };
#pragma unroll
  for (int p = 0; p < ST - 1; ++p) {
    if (p < nk) issue(p);
    cp_async_commit();
  }
  float2 acc[8][TN / 2];  // column pairs, FFMA2 (see sgemm_pipe)
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TN / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    if (kt + ST - 1 < nk) issue(kt + ST - 1);
    cp_async_commit();
    const float* as = As[kt % ST];
    const float* bs = Bs[kt % ST];
#pragma unroll
    for (int kq = 0; kq < BK; kq += 4) {
      float a4[8][4];
      if (AK4) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i < 4 ? ty * 4 + i : BM / 2 + ty * 4 + (i - 4);
          float4 v = *reinterpret_cast<const float4*>(as + r * BK + kq);
          a4[i][0] = v.x; a4[i][1] = v.y; a4[i][2] = v.z; a4[i][3] = v.w;
        }
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float a[8];
        if (AK4) {
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = a4[i][kk];
        } else {
          float4 a0 = *reinterpret_cast<const float4*>(as + (kq + kk) * BM + ty * 4);
          float4 a1 = *reinterpret_cast<const float4*>(as + (kq + kk) * BM + BM / 2 + ty * 4);
          a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
        }
        float b[TN];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          float4 v = *reinterpret_cast<const float4*>(bs + (kq + kk) * BN + q * (BN / NQ) + tx * 4);
          b[4 * q] = v.x; b[4 * q + 1] = v.y; b[4 * q + 2] = v.z; b[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < TN / 2; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), make_float2(b[2 * j], b[2 * j + 1]), acc[i][j]);
      }
    }
  }
  cp_async_wait<0>();
  float* __restrict__ C = g.C + g.tCm[tm] + g.tCn[tn];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = i < 4 ? ty * 4 + i : BM / 2 + ty * 4 + (i - 4);
    float* crow = C + g.cm[r];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = q * (BN / NQ) + tx * 4;
      if (CVEC) {
        *reinterpret_cast<float4*>(crow + g.cn[c]) =
            make_float4(acc[i][q * 2].x, acc[i][q * 2].y, acc[i][q * 2 + 1].x, acc[i][q * 2 + 1].y);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) crow[g.cn[c + j]] = j & 1 ? acc[i][q * 2 + j / 2].y : acc[i][q * 2 + j / 2].x;
      }
    }
  }
}

// FFMA template v3: 128 x 128 CTA tile, 8 x 8 register tile per thread
// (two 4-row x two 4-column quads, conflict-free 16-byte shared reads),
// <= 128 registers so two CTAs (16 warps) share an SM, and a 4-stage
// cp.async ring of BKT-deep k-tiles in MN-major shared layout [k][m] /
// [k][n].  Operands whose MN dim is 16-byte contiguous land with 16-byte
// copies (V16); any other view -- K-contiguous A (MatMul), permuted tensors
// (CCSD(T)), the filter of MCC -- lands element-wise with 4-byte copies that
// are coalesced along k and transpose on the fly (no pre-pass, no registers).
// Fragments of step k+1 are read from shared memory while step k's 64 FFMAs
// issue (register double buffering).
//   SMX : one 128 x 128 tile of (M, N) per CTA (grouped raster)
//   DM  : the K / BKT k-tiles;  SM : the 4-slot ring;  CC : 16 x 16 threads
//   RM  : 8 x 8 accumulators per thread
template <int BM, int BN, int BKT>
struct PipeSmem {
  static constexpr int PA = BM + 4, PB = BN + 4;  // row pitch (floats): breaks k-stride bank aliasing of the 4-byte fills
  static constexpr int STAGES = BKT >= 32 ? 3 : 4;
  static constexpr int FLOATS = STAGES * BKT * (PA + PB);
};

template <int BM, int BN, bool AV, bool BV, bool CVEC, int BKT>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 512 / ((BM / 8) * (BN / 8))) sgemm_pipe(GemmArgs g) {
  constexpr int NT = (BM / 8) * (BN / 8);  // threads: one 8 x 8 register tile each
  using SM = PipeSmem<BM, BN, BKT>;
  constexpr int PA = SM::PA, PB = SM::PB, ST = SM::STAGES, TX = BN / 8;
  static_assert(NT == 256 || NT == 128, "8 x 8 register tiles over 128 or 256 threads");
  extern __shared__ __align__(16) float psm[];
  float* As = psm;                   // [ST][BKT][PA]
  float* Bs = psm + ST * BKT * PA;   // [ST][BKT][PB]
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int GROUP_M = g.group_m > 0 ? g.group_m : 8;
  const int x = blockIdx.x;
  const int per_group = GROUP_M * g.tilesN;
  const int first_m = (x / per_group) * GROUP_M;
  const int gsz = min(g.tilesM - first_m, GROUP_M);
  const int tm = first_m + (x % per_group) % gsz;
  const int tn = (x % per_group) / gsz;
  const float* __restrict__ A = g.A + g.tAm[tm];
  const float* __restrict__ B = g.B + g.tBn[tn];

  // ---- fill slots, fixed across k-tiles.  Inside a k-tile the k offsets
  // are affine (host-checked), so a slot's source is  base(k-tile) + off[p]
  // with one uniform table read per k-tile and one IMAD.WIDE per copy.
  // V16: 16-byte chunk c = tid + NT p -> k = c / (X/4), mn = (c % (X/4)) * 4
  // S4 : element e = tid + NT p      -> k = e % BKT,    mn = e / BKT
  constexpr int TA = AV ? BM * BKT / 4 : BM * BKT, TB = BV ? BN * BKT / 4 : BN * BKT;  // fills per k-tile
  constexpr int NA = (TA + NT - 1) / NT, NB = (TB + NT - 1) / NT;
  int a_off[NA], b_off[NB];
#pragma unroll
  for (int p = 0; p < NA; ++p) {
    const int c = tid + NT * p;
    const int k = AV ? c / (BM / 4) : c % BKT, m = AV ? (c % (BM / 4)) * 4 : c / BKT;
    a_off[p] = c < TA ? g.am[m] + k * g.sak : 0;
  }
#pragma unroll
  for (int p = 0; p < NB; ++p) {
    const int c = tid + NT * p;
    const int k = BV ? c / (BN / 4) : c % BKT, n = BV ? (c % (BN / 4)) * 4 : c / BKT;
    b_off[p] = c < TB ? g.bn[n] + k * g.sbk : 0;
  }
  // shared destinations: slot p sits at a fixed offset from slot 0
  const int a_dst0 = AV ? (tid / (BM / 4)) * PA + (tid % (BM / 4)) * 4 : (tid % BKT) * PA + tid / BKT;
  const int b_dst0 = BV ? (tid / (BN / 4)) * PB + (tid % (BN / 4)) * 4 : (tid % BKT) * PB + tid / BKT;
  constexpr int A_STEP = AV ? (NT / (BM / 4)) * PA : NT / BKT;  // floats between slots p and p+1
  constexpr int B_STEP = BV ? (NT / (BN / 4)) * PB : NT / BKT;
  // K = nfull * BKT + ktail: a last, partial k-tile of ktail (a multiple of
  // 8) rows is filled and folded without padding (CCSD(T): 72 = 4 x 16 + 8)
  const int nfull = g.K / BKT, ktail = g.K - nfull * BKT;
  const int nk = nfull + (ktail ? 1 : 0);
  auto issue = [&](int kt) {
    const int s = kt % ST, k0 = kt * BKT;
    const int kcount = kt < nfull ? BKT : ktail;
    // the k-tile's base: linear in k0 when the offsets are globally affine,
    // else one table read (its latency sits right before the copies)
    const float* abase = A + (g.klin ? static_cast<int64_t>(k0) * g.sak : __ldg(g.ak + k0));
    const float* bbase = B + (g.klin ? static_cast<int64_t>(k0) * g.sbk : __ldg(g.bk + k0));
    const uint32_t as = static_cast<uint32_t>(__cvta_generic_to_shared(As + s * BKT * PA + a_dst0));
    const uint32_t bs = static_cast<uint32_t>(__cvta_generic_to_shared(Bs + s * BKT * PB + b_dst0));
#pragma unroll
    for (int p = 0; p < NA; ++p) {
      if (TA % NT && tid + NT * p >= TA) continue;
      if ((AV ? (tid + NT * p) / (BM / 4) : (tid + NT * p) % BKT) >= kcount) continue;
      if (AV) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(as + p * A_STEP * 4), "l"(abase + a_off[p]));
      else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(as + p * A_STEP * 4), "l"(abase + a_off[p]));
    }
#pragma unroll
    for (int p = 0; p < NB; ++p) {
      if (TB % NT && tid + NT * p >= TB) continue;
      if ((BV ? (tid + NT * p) / (BN / 4) : (tid + NT * p) % BKT) >= kcount) continue;
      if (BV) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(bs + p * B_STEP * 4), "l"(bbase + b_off[p]));
      else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(bs + p * B_STEP * 4), "l"(bbase + b_off[p]));
    }
  };
#pragma unroll
  for (int p = 0; p < ST - 1; ++p) {
    if (p < nk) issue(p);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // accumulators as column pairs: acc[i][jj] = (C[i][2 jj], C[i][2 jj + 1]),
  // updated by FFMA2 (two fma.rn per instruction, the row value broadcast
  // from a scalar register): half the FMA instructions of scalar FFMA,
  // bit-identical results
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 2) : "memory");
    __syncthreads();
    if (kt + ST - 1 < nk) issue(kt + ST - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* as = As + (kt % ST) * BKT * PA + ty * 4;
    const float* bs = Bs + (kt % ST) * BKT * PB + tx * 4;
    float4 fa[2][2], fb[2][2];
    fa[0][0] = *reinterpret_cast<const float4*>(as);
    fa[0][1] = *reinterpret_cast<const float4*>(as + BM / 2);
    fb[0][0] = *reinterpret_cast<const float4*>(bs);
    fb[0][1] = *reinterpret_cast<const float4*>(bs + BN / 2);
    const int kcount = kt < nfull ? BKT : ktail;
#pragma unroll
    for (int k = 0; k < BKT; ++k) {
      if (BKT > 8 && k == 8 && kcount == 8) break;  // the partial last k-tile
      const int cur = k & 1, nxt = cur ^ 1;
      if (k + 1 < BKT && (BKT == 8 || k + 1 != 8 || kcount != 8)) {
        fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * PA);
        fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * PA + BM / 2);
        fb[nxt][0] = *reinterpret_cast<const float4*>(bs + (k + 1) * PB);
        fb[nxt][1] = *reinterpret_cast<const float4*>(bs + (k + 1) * PB + BN / 2);
      }
      const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                          fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
      const float2 b[4] = {make_float2(fb[cur][0].x, fb[cur][0].y), make_float2(fb[cur][0].z, fb[cur][0].w),
                           make_float2(fb[cur][1].x, fb[cur][1].y), make_float2(fb[cur][1].z, fb[cur][1].w)};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), b[j], acc[i][j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  float* __restrict__ C = g.C + g.tCm[tm] + g.tCn[tn];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = i < 4 ? ty * 4 + i : BM / 2 + ty * 4 + (i - 4);
    float* crow = C + g.cm[r];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h * (BN / 2) + tx * 4;
      if (CVEC) {
        *reinterpret_cast<float4*>(crow + g.cn[c]) =
            make_float4(acc[i][h * 2].x, acc[i][h * 2].y, acc[i][h * 2 + 1].x, acc[i][h * 2 + 1].y);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) crow[g.cn[c + j]] = j & 1 ? acc[i][h * 2 + j / 2].y : acc[i][h * 2 + j / 2].x;
      }
    }
  }
}

// sgemm_pipe with a K-contiguous A tile (MCC's implicit im2col: a k-tile is
// 16 channels of one filter tap, 64 contiguous bytes of the NHWC input per
// output pixel).  The tile lands row-major [BM][16] through 16-byte copies
// along k -- 4 per thread per k-tile instead of the 16 transposing 4-byte
// copies of the S4 form, a quarter of the L1 fill wavefronts -- and the
// fragments are read as float4 along k (8 rows x 4 k per LDS.128 group, the
// same LDS count per FFMA as the M-major form).  Rows are 64 bytes with the
// 16-byte quads XOR-swizzled by (row & 3), and thread rows are interleaved
// (ty + TY i), so one warp's four row groups read distinct bank quads (no
// padding: 4 stages keep 4 CTAs per SM).  The k-group loop stays rolled: fully
// unrolled, ptxas renames the accumulators across groups and pays ~170 MOVs
// per k-tile.  Accumulation order per output (k ascending, FFMA2 column
// pairs) is that of sgemm_pipe: bit-identical results.
template <int BM, int BN, int BKT>
struct PipeAkSmem {
  static constexpr int PA = BKT, PB = BN + 4;
  static constexpr int STAGES = 4;
  static constexpr int FLOATS = STAGES * (BM * PA + BKT * PB);
};

template <int BM, int BN, bool BV, bool CVEC, int BKT>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 512 / ((BM / 8) * (BN / 8))) sgemm_pipe_ak(GemmArgs g) {
  constexpr int NT = (BM / 8) * (BN / 8);
  using SM = PipeAkSmem<BM, BN, BKT>;
  constexpr int PA = SM::PA, PB = SM::PB, ST = SM::STAGES, TX = BN / 8, TY = BM / 8;
  static_assert(BKT == 16, "16-deep k-tiles: 4 swizzled quads per row (partial last tile of 8)");
  extern __shared__ __align__(16) float psm[];
  float* As = psm;                   // [ST][BM][PA]
  float* Bs = psm + ST * BM * PA;    // [ST][BKT][PB]
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int GROUP_M = g.group_m > 0 ? g.group_m : 8;
  const int x = blockIdx.x;
  const int per_group = GROUP_M * g.tilesN;
  const int first_m = (x / per_group) * GROUP_M;
  const int gsz = min(g.tilesM - first_m, GROUP_M);
  const int tm = first_m + (x % per_group) % gsz;
  const int tn = (x % per_group) / gsz;
  const float* __restrict__ A = g.A + g.tAm[tm];
  const float* __restrict__ B = g.B + g.tBn[tn];
  // A: 16-byte chunk c = tid + NT p -> row c / (BKT/4), k quad c % (BKT/4)
  constexpr int KQ = BKT / 4, TA = BM * KQ, NA = TA / NT;
  static_assert(TA % NT == 0, "A chunks per thread");
  constexpr int TB = BV ? BN * BKT / 4 : BN * BKT, NB = (TB + NT - 1) / NT;
  int a_off[NA];
#pragma unroll
  for (int p = 0; p < NA; ++p) a_off[p] = g.am[(tid + NT * p) / KQ] + ((tid + NT * p) % KQ) * 4;
  int b_off[NB];
#pragma unroll
  for (int p = 0; p < NB; ++p) {
    const int c = tid + NT * p;
    const int k = BV ? c / (BN / 4) : c % BKT, n = BV ? (c % (BN / 4)) * 4 : c / BKT;
    b_off[p] = c < TB ? g.bn[n] + k * g.sbk : 0;
  }
  const int b_dst0 = BV ? (tid / (BN / 4)) * PB + (tid % (BN / 4)) * 4 : (tid % BKT) * PB + tid / BKT;
  constexpr int B_STEP = BV ? (NT / (BN / 4)) * PB : NT / BKT;
  const int nfull = g.K / BKT, ktail = g.K - nfull * BKT;
  const int nk = nfull + (ktail ? 1 : 0);
  auto issue = [&](int kt) {
    const int s = kt % ST, k0 = kt * BKT;
    const int kcount = kt < nfull ? BKT : ktail;
    const float* abase = A + (g.klin ? static_cast<int64_t>(k0) : __ldg(g.ak + k0));
    const float* bbase = B + (g.klin ? static_cast<int64_t>(k0) * g.sbk : __ldg(g.bk + k0));
    const uint32_t as = static_cast<uint32_t>(__cvta_generic_to_shared(As + s * BM * PA));
    const uint32_t bs = static_cast<uint32_t>(__cvta_generic_to_shared(Bs + s * BKT * PB + b_dst0));
#pragma unroll
    for (int p = 0; p < NA; ++p) {
      const int c = tid + NT * p;
      if ((c % KQ) * 4 >= kcount) continue;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(as + ((c / KQ) * PA + (((c % KQ) ^ ((c / KQ) & 3)) * 4)) * 4),
                   "l"(abase + a_off[p]));
    }
#pragma unroll
    for (int p = 0; p < NB; ++p) {
      if (TB % NT && tid + NT * p >= TB) continue;
      if ((BV ? (tid + NT * p) / (BN / 4) : (tid + NT * p) % BKT) >= kcount) continue;
      if (BV) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(bs + p * B_STEP * 4), "l"(bbase + b_off[p]));
      else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(bs + p * B_STEP * 4), "l"(bbase + b_off[p]));
    }
  };
#pragma unroll
  for (int p = 0; p < ST - 1; ++p) {
    if (p < nk) issue(p);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 2) : "memory");
    __syncthreads();
    if (kt + ST - 1 < nk) issue(kt + ST - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* as = As + (kt % ST) * BM * PA + ty * PA;
    const float* bs = Bs + (kt % ST) * BKT * PB + tx * 4;
    const int kgroups = (kt < nfull ? BKT : ktail) / 4;
#pragma unroll 1
    for (int kg = 0; kg < kgroups; ++kg) {
      float4 fa[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) fa[i] = *reinterpret_cast<const float4*>(as + i * TY * PA + ((kg ^ (ty & 3)) * 4));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = kg * 4 + kk;
        const float4 f0 = *reinterpret_cast<const float4*>(bs + k * PB);
        const float4 f1 = *reinterpret_cast<const float4*>(bs + k * PB + BN / 2);
        const float2 b[4] = {make_float2(f0.x, f0.y), make_float2(f0.z, f0.w), make_float2(f1.x, f1.y), make_float2(f1.z, f1.w)};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float a = kk == 0 ? fa[i].x : kk == 1 ? fa[i].y : kk == 2 ? fa[i].z : fa[i].w;
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __ffma2_rn(make_float2(a, a), b[j], acc[i][j]);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  float* __restrict__ C = g.C + g.tCm[tm] + g.tCn[tn];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float* crow = C + g.cm[ty + TY * i];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = h * (BN / 2) + tx * 4;
      if (CVEC) {
        *reinterpret_cast<float4*>(crow + g.cn[c]) =
            make_float4(acc[i][h * 2].x, acc[i][h * 2].y, acc[i][h * 2 + 1].x, acc[i][h * 2 + 1].y);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) crow[g.cn[c + j]] = j & 1 ? acc[i][h * 2 + j / 2].y : acc[i][h * 2 + j / 2].x;
      }
    }
  }
}

// B layout pass: Bp[k][t * BN + c] = B[tBn[t] + bn[c] + bk[k]] (n in N-tile
// order; consecutive threads walk n).
__global__ void __launch_bounds__(256) bpack(const float* __restrict__ B, float* __restrict__ Bp, const int32_t* __restrict__ tBn,
                                             const int32_t* __restrict__ bn, const int32_t* __restrict__ bk, int bnl, int64_t ntot,
                                             int64_t total) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < total; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int64_t k = i / ntot, n = i - k * ntot;
    const int t = static_cast<int>(n / bnl), c = static_cast<int>(n - static_cast<int64_t>(t) * bnl);
    Bp[i] = __ldg(B + tBn[t] + bn[c] + bk[k]);
  }
}

// A layout pass: Ap[k][m] = A[tAm[m / bml] + am[m % bml] + ak[k]] (m in
// M-tile order) -- the K-contiguous A of a large MatMul transposed once per
// run through 32 x 32 shared-memory tiles (reads along k, writes along m), so
// the template fills A with 16-byte M-major copies instead of 4-byte
// transposing ones.
__global__ void __launch_bounds__(256) apack_t(const float* __restrict__ A, float* __restrict__ Ap,
                                               const int32_t* __restrict__ tAm, const int32_t* __restrict__ am,
                                               const int32_t* __restrict__ ak, int bml, int64_t mtot, int K) {
  // 64 (m) x 64 (k) tile: 16-byte reads along k (the rows of A are
  // K-contiguous with 16-byte aligned starts, host-checked), 16-byte writes
  // along m
  __shared__ float tile[64][65];
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int k0 = blockIdx.y * 64;
  const int t = threadIdx.x, q = (t & 15) * 4, r = t >> 4;  // 16 quads x 16 rows
  const int64_t kb = ak[k0];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = r + 16 * i;
    const int64_t m = m0 + row;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (m < mtot && k0 + q < K) v = __ldg(reinterpret_cast<const float4*>(A + tAm[m / bml] + am[m % bml] + kb + q));
    tile[q + 0][row] = v.x;
    tile[q + 1][row] = v.y;
    tile[q + 2][row] = v.z;
    tile[q + 3][row] = v.w;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kr = r + 16 * i;
    const int64_t m = m0 + q;
    if (k0 + kr < K && m < mtot)
      *reinterpret_cast<float4*>(Ap + static_cast<int64_t>(k0 + kr) * mtot + m) =
          make_float4(tile[kr][q], tile[kr][q + 1], tile[kr][q + 2], tile[kr][q + 3]);
  }
}

// ---------------------------------------------------------------- host
// Programmatic dependent launch for the latency-bound kernels (MDHB_NO_PDL=1 off)
bool pdl_enabled() {
  static const bool on = std::getenv("MDHB_NO_PDL") == nullptr;
  return on;
}

// every offset 16-byte aligned (in floats)
bool all_mod4(const std::vector<int64_t>& v) {
  for (int64_t x : v)
    if (x % 4) return false;
  return true;
}
// offsets come in aligned runs of 4 consecutive floats (one 16-byte vector)
bool groups4(const std::vector<int64_t>& v) {
  if (v.size() % 4) return false;
  for (size_t t = 0; t < v.size(); t += 4) {
    if (v[t] % 4) return false;
    for (size_t j = 1; j < 4; ++j)
      if (v[t + j] != v[t] + static_cast<int64_t>(j)) return false;
  }
  return true;
}

class GemmRoutine final : public Routine {
 public:
  GemmRoutine(const Problem& p, Groups g) : p_(p), g_(std::move(g)) {}
  ~GemmRoutine() override {
    if (blob_) cudaFree(blob_);
    if (part_) cudaFree(part_);
    if (lpart_) cudaFree(lpart_);
    if (lcnt_) cudaFree(lcnt_);
    if (bp_tab_) cudaFree(bp_tab_);
    if (bp_) cudaFree(bp_);
    if (ap_tab_) cudaFree(ap_tab_);
    if (ap_) cudaFree(ap_);
  }
  const char* family() const override { return "contraction"; }
  double flops() const override { return 2.0 * static_cast<double>(M_) * static_cast<double>(N_) * static_cast<double>(K_); }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  const char* bound() const override { return (gemv_ || skinny_) ? "hbm" : "fp32"; }
  int launches() const override { return (skinny_ && !cluster_ ? 2 : 1) + (bpack_n_ ? 1 : 0) + (apack_m_ ? 1 : 0); }

  // Builds tables; returns false when this template cannot realise the problem.
  bool setup(int BM, int BN, const std::vector<int64_t>& Tm_in, const std::vector<int64_t>& Tn_in) {
    const MdHom& e = p_.e;
    M_ = prod_sizes(e, g_.Md);
    N_ = prod_sizes(e, g_.Nd);
    K_ = prod_sizes(e, g_.Kd);
    std::vector<int64_t> ones;
    auto scale1 = [](size_t n) { return std::vector<int64_t>(n, 1); };
    std::vector<int64_t> fullK;
    for (int d : g_.Kd) fullK.push_back(e.sizes[static_cast<size_t>(d)]);
    std::vector<int64_t> ak = box_offsets(g_.Kd, fullK, g_.la.cj, scale1(g_.Kd.size()));
    std::vector<int64_t> bk = box_offsets(g_.Kd, fullK, g_.lb.cj, scale1(g_.Kd.size()));
    const int64_t a0 = g_.la.c0, b0 = g_.lb.c0, c0 = g_.lc.c0;
    std::vector<int64_t> tAm, tCm, tBn, tCn, am, cm, bn, cn;
    gemv_ = g_.Nd.empty();
    if (!gemv_ && M_ <= 32 && ((N_ >= 64 && K_ >= 256) || K_ >= 128) && Tm_in.empty()) {
      // skinny: split K so that ~2 waves of CTAs stream B
      std::vector<int64_t> fullM, fullN;
      for (int d : g_.Md) fullM.push_back(e.sizes[static_cast<size_t>(d)]);
      for (int d : g_.Nd) fullN.push_back(e.sizes[static_cast<size_t>(d)]);
      am = box_offsets(g_.Md, fullM, g_.la.cj, scale1(g_.Md.size()));
      cm = box_offsets(g_.Md, fullM, g_.lc.cj, scale1(g_.Md.size()));
      bn = box_offsets(g_.Nd, fullN, g_.lb.cj, scale1(g_.Nd.size()));
      cn = box_offsets(g_.Nd, fullN, g_.lc.cj, scale1(g_.Nd.size()));
      for (auto& v : am) v += a0;
      for (auto& v : bn) v += b0;
      for (auto& v : cm) v += c0;
      // v2 (cluster, DSMEM re-composition): 16-byte operand groups along k
      // for A and along n for B, N % 4 == 0, K split 8 (else 4, 2) ways into
      // slices that are multiples of 64 and fit shared memory
      auto affine = [](const std::vector<int64_t>& v) {
        for (size_t k = 1; k < v.size(); ++k)
          if (v[k] - v[k - 1] != v[1] - v[0]) return false;
        return v.size() > 1;
      };
      if (groups4(bn) && all_mod4(bk) && groups4(ak) && all_mod4(am) && N_ % 4 == 0 && affine(ak) && affine(bk) &&
          ak[0] == 0 && bk[0] == 0 && ak[1] == 1 && !std::getenv("MDHB_SKINNY_V1")) {
        sak_ = ak[1];
        sbk_ = bk[1];
        std::vector<int> css = {8, 4, 2};
        if (const char* f = std::getenv("MDHB_SKINNY_CS")) css.insert(css.begin(), std::atoi(f));
        for (int cs : css) {
          const int64_t ks = K_ / cs;
          const int64_t mt = M_ <= 16 ? 16 : 32;
          if (K_ % (cs * 64) || ks > 1024 || (ks & (ks - 1))) continue;
          if ((ks * 32 + mt * (ks + 4) + 5 * mt * 32) * 4 > 200 * 1024) continue;
          skinny_ = cluster_ = true;
          ks_ = static_cast<int>(ks);
          splits_ = cs;
          last_ = std::getenv("MDHB_SKINNY_LAST") != nullptr;
          if (const char* f = std::getenv("MDHB_SKINNY_NW")) nw_ = std::atoi(f);
          if (nw_ != 32 && (mt != 16 || last_ || (ks != 128 && ks != 256) || N_ % 4)) nw_ = 32;
          // 4 m-groups x 4 rows per thread where the k-parts keep whole 4-k steps
          mg_ = (mt == 16 && nw_ == 32 && ks >= 128 && !std::getenv("MDHB_SKINNY_MG8")) ? 4 : 8;
          if (last_) {  // workspace [strips][splits][mt * 32] + per-strip counters (zeroed once)
            const int64_t strips = (N_ + 31) / 32;
            MDHB_CUDA(cudaMalloc(&lpart_, static_cast<size_t>(strips * cs * mt * 32) * sizeof(float)));
            MDHB_CUDA(cudaMalloc(&lcnt_, static_cast<size_t>(strips) * sizeof(int)));
            MDHB_CUDA(cudaMemset(lcnt_, 0, static_cast<size_t>(strips) * sizeof(int)));
          }
          {  // affine row / column offsets (the dense FC): computed in the kernel
            auto lin = [](const std::vector<int64_t>& v, int64_t& st) {
              st = v.size() > 1 ? v[1] - v[0] : 0;
              for (size_t i = 0; i < v.size(); ++i)
                if (v[i] != static_cast<int64_t>(i) * st) return false;
              return true;
            };
            saff_[4] = lin(am, saff_[0]) && lin(bn, saff_[1]) && lin(cm, saff_[2]) && lin(cn, saff_[3]) &&
                       !std::getenv("MDHB_SKINNY_TABLES");
          }
          tables(am, ak, bk, bn, cm, cn, {}, {}, {}, {});
          return true;
        }
      }
      int64_t ntiles = (N_ + 255) / 256;
      int64_t want = std::max<int64_t>(1, 2 * sm_count(p_.opt.device) / ntiles);
      int64_t ks = 64;
      while (ks * 2 <= K_ / want && ks < 1024) ks *= 2;
      while (K_ % ks) ks /= 2;
      if (ks < 8) return false;
      skinny_ = true;
      ks_ = static_cast<int>(ks);
      splits_ = static_cast<int>(K_ / ks);
      MDHB_CUDA(cudaMalloc(&part_, static_cast<size_t>(splits_) * M_ * N_ * sizeof(float)));
      tables(am, ak, bk, bn, cm, cn, {}, {}, {}, {});
      return true;
    }
    if (gemv_) {
      // rows must be contiguous in k, x contiguous too
      for (int64_t k = 0; k < K_; ++k)
        if (ak[static_cast<size_t>(k)] != k || bk[static_cast<size_t>(k)] != k) return false;
      std::vector<int64_t> fullM;
      for (int d : g_.Md) fullM.push_back(e.sizes[static_cast<size_t>(d)]);
      am = box_offsets(g_.Md, fullM, g_.la.cj, scale1(g_.Md.size()));
      cm = box_offsets(g_.Md, fullM, g_.lc.cj, scale1(g_.Md.size()));
      if (K_ % 4 || a0 % 4 || b0 % 4) return false;
      for (auto& v : am) {
        if ((v + a0) % 4) return false;
        v += a0;
      }
      for (auto& v : cm) v += c0;
      tables(am, cm, {}, {}, {}, {}, {}, {}, {}, {});
      return true;
    }
    if (K_ % BK) return false;
    std::vector<int64_t> Tm = Tm_in.empty() ? factor_box(e, g_.Md, BM) : Tm_in;
    std::vector<int64_t> Tn = Tn_in.empty() ? factor_box(e, g_.Nd, BN) : Tn_in;
    if (Tm.empty() || Tn.empty()) return false;
    int64_t pm = 1, pn = 1;
    for (size_t q = 0; q < Tm.size(); ++q) {
      if (e.sizes[static_cast<size_t>(g_.Md[q])] % Tm[q]) return false;
      pm *= Tm[q];
    }
    for (size_t q = 0; q < Tn.size(); ++q) {
      if (e.sizes[static_cast<size_t>(g_.Nd[q])] % Tn[q]) return false;
      pn *= Tn[q];
    }
    if (pm != BM || pn != BN) return false;
    Tm_ = Tm;
    Tn_ = Tn;
    BM_ = BM;
    BN_ = BN;
    auto grid_of = [&](const std::vector<int>& dims, const std::vector<int64_t>& T) {
      std::vector<int64_t> gext, sc;
      for (size_t q = 0; q < dims.size(); ++q) {
        gext.push_back(e.sizes[static_cast<size_t>(dims[q])] / T[q]);
        sc.push_back(T[q]);
      }
      return std::make_pair(gext, sc);
    };
    auto [gm, sm] = grid_of(g_.Md, Tm);
    auto [gn, sn] = grid_of(g_.Nd, Tn);
    tAm = box_offsets(g_.Md, gm, g_.la.cj, sm);
    tCm = box_offsets(g_.Md, gm, g_.lc.cj, sm);
    tBn = box_offsets(g_.Nd, gn, g_.lb.cj, sn);
    tCn = box_offsets(g_.Nd, gn, g_.lc.cj, sn);
    am = box_offsets(g_.Md, Tm, g_.la.cj, scale1(Tm.size()));
    cm = box_offsets(g_.Md, Tm, g_.lc.cj, scale1(Tm.size()));
    bn = box_offsets(g_.Nd, Tn, g_.lb.cj, scale1(Tn.size()));
    cn = box_offsets(g_.Nd, Tn, g_.lc.cj, scale1(Tn.size()));
    for (auto& v : tAm) v += a0;
    for (auto& v : tBn) v += b0;
    for (auto& v : tCm) v += c0;
    tilesM_ = static_cast<int>(tAm.size());
    tilesN_ = static_cast<int>(tBn.size());
    {
      // raster group = SMX parts of the innermost M dim's tile grid: a given
      // group must divide that grid; the default is its largest divisor <= 8
      const int64_t gl = gm.empty() ? 1 : gm.back();
      inner_rows_ = gl;
      if (group_ > 0 && gl % group_) return false;
      if (group_ <= 0) {
        group_ = 1;
        for (int q = 8; q >= 1; --q)
          if (gl % q == 0) {
            group_ = q;
            break;
          }
      }
    }
    // vector load / store directions
    if (groups4(ak) && all_mod4(am) && all_mod4(tAm)) amode_ = LD_K4;
    else if (groups4(am) && all_mod4(ak) && all_mod4(tAm)) amode_ = LD_MN4;
    else amode_ = LD_SCALAR;
    if (groups4(bn) && all_mod4(bk) && all_mod4(tBn)) bmode_ = LD_MN4;
    else if (groups4(bk) && all_mod4(bn) && all_mod4(tBn)) bmode_ = LD_K4;
    else bmode_ = LD_SCALAR;
    cvec_ = groups4(cn) && all_mod4(cm) && all_mod4(tCm) && all_mod4(tCn);
    // layout_de pass for a small B that no 16-byte fill can read (CCSD(T)'s
    // B[e][f][g][c] against an (c, e, f) N tile): gather it once per run into
    // Bp[k][n] with n in N-tile order, so the template reads B with 16-byte
    // MN-major copies
    if (bmode_ != LD_MN4 && N_ % 4 == 0 && BN % 4 == 0 && K_ * N_ * 4 <= (int64_t(64) << 20) &&
        !std::getenv("MDHB_NO_BPACK")) {
      bp_tBn_ = tBn;
      bp_bn_ = bn;
      bp_bk_ = bk;
      const int64_t ntot = static_cast<int64_t>(tilesN_) * BN;
      for (size_t t = 0; t < tBn.size(); ++t) tBn[t] = static_cast<int64_t>(t) * BN;
      for (size_t c = 0; c < bn.size(); ++c) bn[c] = static_cast<int64_t>(c);
      for (size_t k = 0; k < bk.size(); ++k) bk[k] = static_cast<int64_t>(k) * ntot;
      bpack_n_ = ntot;
      bmode_ = LD_MN4;
    }
    // layout_de pass for a large K-contiguous A (MatMul's A[i][k]) re-read by
    // many N tiles: transposed once per run into M-major tile order (16-byte
    // fills; measured 20.27 vs 21.12 ms at 8192^3 for the GEMM itself)
    if (amode_ == LD_K4 && tilesN_ >= 16 && BM % 32 == 0 && !std::getenv("MDHB_NO_APACK")) {
      const int64_t mtot = static_cast<int64_t>(tilesM_) * BM;
      bool kcontig = K_ % 4 == 0 && all_mod4(tAm) && all_mod4(am) && ak[0] % 4 == 0;
      for (size_t k = 0; k < ak.size() && kcontig; ++k) kcontig = ak[k] == ak[0] + static_cast<int64_t>(k);
      if (kcontig && mtot % 64 == 0 && K_ * mtot * 4 <= (int64_t(1) << 30) && K_ * mtot < INT32_MAX) {
        ap_tAm_ = tAm;
        ap_am_ = am;
        ap_ak_ = ak;
        for (size_t t = 0; t < tAm.size(); ++t) tAm[t] = static_cast<int64_t>(t) * BM;
        for (size_t r = 0; r < am.size(); ++r) am[r] = static_cast<int64_t>(r);
        for (size_t k = 0; k < ak.size(); ++k) ak[k] = static_cast<int64_t>(k) * mtot;
        apack_m_ = mtot;
        amode_ = LD_MN4;
      }
    }
    {
      // k offsets affine inside every k-tile of the pipe template: the
      // deepest k-tile (32 for 128 x 128 tiles, else 16, else 8) that keeps
      // both operands affine and divides K
      // a partial last k-tile of 8 (K % bkt == 8) unless a configuration
      // names the k-tile (its Table-1 form has no partial tiles)
      const bool ktail_ok = bk_want_ == 0 && !std::getenv("MDHB_SGEMM_NO_KTAIL");
      auto tile_aff = [&](const std::vector<int64_t>& v, int64_t bkt, int& stride) {
        if (v.size() < 2 || (K_ % bkt && !(ktail_ok && bkt > 8 && K_ % bkt == 8 && K_ > bkt))) return false;
        const int64_t sd = v[1] - v[0];
        for (size_t k = 0; k < v.size(); ++k)
          if (v[k] != v[k / bkt * bkt] + static_cast<int64_t>(k % bkt) * sd) return false;
        stride = static_cast<int>(sd);
        return true;
      };
      pbk_ = 0;
      for (int bkt : {32, 16, 8}) {
        if (bkt == 32 && !(BM == 128 && BN == 128)) continue;
        if (bk_want_ && bkt != bk_want_) continue;  // the configuration's k-tile (SM parts of K)
        if (tile_aff(ak, bkt, psak_) && tile_aff(bk, bkt, psbk_)) {
          pbk_ = bkt;
          break;
        }
      }
      tile_affine_ = pbk_ > 0;
      auto lin = [&](const std::vector<int64_t>& v, int stride) {
        for (size_t k = 0; k < v.size(); ++k)
          if (v[k] != static_cast<int64_t>(k) * stride) return false;
        return true;
      };
      klin_ = tile_affine_ && lin(ak, psak_) && lin(bk, psbk_) && !std::getenv("MDHB_SGEMM_NO_KLIN");
    }
    tables(tAm, tCm, tBn, tCn, am, cm, bn, cn, ak, bk);
    if (apack_m_) {
      std::vector<int32_t> h;
      for (auto* v : {&ap_tAm_, &ap_am_, &ap_ak_})
        for (int64_t x : *v) {
          if (x > INT32_MAX || x < INT32_MIN) fail("Unsupported", "A offsets exceed int32");
          h.push_back(static_cast<int32_t>(x));
        }
      MDHB_CUDA(cudaMalloc(&ap_tab_, h.size() * sizeof(int32_t)));
      MDHB_CUDA(cudaMemcpy(ap_tab_, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      MDHB_CUDA(cudaMalloc(&ap_, static_cast<size_t>(K_ * apack_m_) * sizeof(float)));
    }
    if (bpack_n_) {
      // gather tables (original B offsets) + the packed copy
      std::vector<int32_t> h;
      for (auto* v : {&bp_tBn_, &bp_bn_, &bp_bk_})
        for (int64_t x : *v) {
          if (x > INT32_MAX || x < INT32_MIN) fail("Unsupported", "B offsets exceed int32");
          h.push_back(static_cast<int32_t>(x));
        }
      MDHB_CUDA(cudaMalloc(&bp_tab_, h.size() * sizeof(int32_t)));
      MDHB_CUDA(cudaMemcpy(bp_tab_, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      MDHB_CUDA(cudaMalloc(&bp_, static_cast<size_t>(K_ * bpack_n_) * sizeof(float)));
    }
    return true;
  }

  std::string describe() const override {
    std::ostringstream os;
    const char* mn[] = {"scalar", "k4", "mn4"};
    if (cluster_) {
      os << "{\"kernel\": \"skinny_cluster<" << (M_ <= 16 ? 16 : 32) << (last_ ? ",last_block>" : ">") << "\", \"M\": " << M_ << ", \"N\": " << N_
         << ", \"K\": " << K_ << ", \"k_per_cta\": " << ks_ << ", \"cluster\": " << splits_
         << ", \"ctas\": " << (N_ + 31) / 32 * splits_ << ", \"rows_per_thread\": " << (M_ <= 16 ? 16 : 32) / mg_ << ", \"threads\": 256}";
      return os.str();
    }
    if (skinny_) {
      os << "{\"kernel\": \"skinny_partial<" << (M_ <= 16 ? 16 : 32) << ">+skinny_fold\", \"M\": " << M_
         << ", \"N\": " << N_ << ", \"K\": " << K_ << ", \"k_per_split\": " << ks_ << ", \"splits\": " << splits_
         << ", \"threads\": 256}";
      return os.str();
    }
    if (gemv_) {
      const bool split = K_ % 1024 == 0 && K_ / 1024 <= 8 && !std::getenv("MDHB_GEMV_V1");
      os << "{\"kernel\": \"" << (split ? "gemv_split<" + std::to_string(K_ / 1024) + ">" : std::string("gemv_rows<2>"))
         << "\", \"M\": " << M_ << ", \"K\": " << K_ << ", \"threads\": " << (split ? 256 : 128) << "}";
      return os.str();
    }
    const std::string kname = pipe_ok() ? "sgemm_pipe<" + std::to_string(BM_) + "x" + std::to_string(BN_) + "," +
                                              std::string(pipe_av() ? "V16" : pipe_ak() ? "K16" : "S4") + "," +
                                              (pipe_bv() ? "V16" : "S4") + ",BK" + std::to_string(pipe_bk()) + ">"
                              : (async_ok() ? "sgemm_async<" : "sgemm_tiled<") + std::to_string(BM_) + "," +
                                    std::to_string(BN_) + ">";
    os << "{\"kernel\": \"" << kname << "\", \"M\": " << M_ << ", \"N\": " << N_
       << ", \"K\": " << K_ << ", \"BK\": " << (pipe_ok() ? pipe_bk() : BK) << ", \"threads\": " << (async_ok() || pipe_ok() ? 256 : (BM_ / 8) * (BN_ / 8)) << ", \"a_load\": \""
       << mn[amode_] << "\", \"b_load\": \"" << mn[bmode_] << "\", \"c_store\": \"" << (cvec_ ? "v4" : "scalar")
       << "\", \"tiles\": " << static_cast<int64_t>(tilesM_) * tilesN_ << ", \"raster_group_m\": " << group_;
    if (!note_.empty()) os << ", \"tc_declined\": \"" << note_ << "\"";
    os << "}";
    return os.str();
  }

  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    const float* A = static_cast<const float*>(d_in[g_.a_buf]);
    const float* B = static_cast<const float*>(d_in[g_.b_buf]);
    float* C = static_cast<float*>(d_out[0]);
    if (cluster_) {
      SkinnyArgs a{A, B, lpart_, C, tab_[0], tab_[1], tab_[2], tab_[3], tab_[4], tab_[5], static_cast<int>(M_),
                   static_cast<int>(N_), static_cast<int>(K_), ks_, splits_, sak_, sbk_, lcnt_, saff_[0], saff_[1],
                   saff_[2], saff_[3], static_cast<int>(saff_[4]), !last_ && std::getenv("MDHB_SKINNY_TXFOLD") != nullptr};  // opt-in: measured no faster
      const int mt = M_ <= 16 ? 16 : 32;
      const int nw = nw_, kqn = 256 / (mg_ * (nw / 4));
      const size_t smem = (static_cast<size_t>(ks_) * nw + static_cast<size_t>(mt) * (ks_ + 4) + (kqn + 1) * mt * nw) * sizeof(float) +
                          8 * sizeof(uint64_t);  // + the TMA stage barriers and the inbox barrier
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(static_cast<unsigned>((N_ + nw - 1) / nw), static_cast<unsigned>(splits_));
      lc.blockDim = dim3(256);
      lc.dynamicSmemBytes = smem;
      lc.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 1;
      at[0].val.clusterDim.y = static_cast<unsigned>(splits_);
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = last_ ? 0 : 1;  // PDL measured slower for the cluster kernel (6.6 -> 7.7 us)
      void (*kern)(SkinnyArgs, CUtensorMap) = nullptr;
      // B by TMA tensor copies (opt-in MDHB_SKINNY_TMA=1: bit-identical, but
      // 5.71 vs 5.52 us for the FC -- DESIGN, dead ends): dense FC (affine,
      // unit column stride, 16-byte row pitch and base), 4 x 4 thread tiles
      const bool tmab = mg_ == 4 && !last_ && saff_[4] && saff_[1] == 1 && (sbk_ * 4) % 16 == 0 && K_ % ks_ == 0 &&
                        reinterpret_cast<uintptr_t>(B) % 16 == 0 && std::getenv("MDHB_SKINNY_TMA");
      if (tmab && B != last_b_) {
        static EncodeFn enc = tensor_map_encoder();
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(N_), static_cast<cuuint64_t>(K_)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(sbk_) * 4};
        cuuint32_t box[2] = {32, static_cast<cuuint32_t>(ks_ / 4)};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tmb_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(B), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (FC B slice) failed");
        last_b_ = B;
      }
#define MDHB_SK(KS)                                                                                          \
  if (ks_ == KS)                                                                                             \
    kern = last_ ? (mt == 16 ? skinny_cluster<16, KS, true> : skinny_cluster<32, KS, true>)                  \
                 : (mt == 16 ? skinny_cluster<16, KS> : skinny_cluster<32, KS>);
#define MDHB_SK4(KS)                                                                                    \
  if (ks_ == KS) kern = last_ ? skinny_cluster<16, KS, true, 32, 4>                                      \
                       : tmab ? skinny_cluster<16, KS, false, 32, 4, true> : skinny_cluster<16, KS, false, 32, 4>;
      if (nw == 32 && mg_ == 8) {
        MDHB_SK(64) MDHB_SK(128) MDHB_SK(256) MDHB_SK(512) MDHB_SK(1024)
      }
      if (nw == 32 && mg_ == 4) {
        MDHB_SK4(128) MDHB_SK4(256) MDHB_SK4(512) MDHB_SK4(1024)
      }
#undef MDHB_SK
#undef MDHB_SK4
      // wider column strips (longer contiguous B row segments): MT 16 only
      if (nw == 64 && mt == 16) kern = ks_ == 128 ? skinny_cluster<16, 128, false, 64> : ks_ == 256 ? skinny_cluster<16, 256, false, 64> : nullptr;
      if (nw == 128 && mt == 16) kern = ks_ == 128 ? skinny_cluster<16, 128, false, 128> : ks_ == 256 ? skinny_cluster<16, 256, false, 128> : nullptr;
      if (!kern) fail("Unsupported", "no skinny_cluster instance for this strip / slice");
      if (smem > 48 * 1024) MDHB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      if (splits_ > 8 && !last_) MDHB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      MDHB_CUDA(cudaLaunchKernelEx(&lc, kern, a, tmb_));
      return;
    }
    if (skinny_) {
      SkinnyArgs a{A, B, part_, C, tab_[0], tab_[1], tab_[2], tab_[3], tab_[4], tab_[5], static_cast<int>(M_),
                   static_cast<int>(N_), static_cast<int>(K_), ks_, splits_, 0, 0};
      dim3 grid(static_cast<unsigned>((N_ + 255) / 256), static_cast<unsigned>(splits_));
      size_t smem = static_cast<size_t>(M_) * ks_ * sizeof(float);
      // the attribute goes on the instance actually launched
      void (*kp)(SkinnyArgs) = M_ <= 16 ? skinny_partial<16> : skinny_partial<32>;
      if (smem > 48 * 1024) MDHB_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      mark_begin(s);
      kp<<<grid, 256, smem, s>>>(a);
      mark_end(s);
      MDHB_CUDA(cudaGetLastError());
      skinny_fold<<<static_cast<unsigned>((M_ * N_ + 255) / 256), 256, 0, s>>>(a);
      MDHB_CUDA(cudaGetLastError());
      return;
    }
    if (gemv_) {
      GemvArgs a{A, B + g_.lb.c0, C, tab_[0], tab_[1], M_, static_cast<int>(K_)};
      const int V = static_cast<int>(K_ / 1024);
      if (K_ % 1024 == 0 && (V == 1 || V == 2 || V == 4 || V == 8) && !std::getenv("MDHB_GEMV_V1")) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(static_cast<unsigned>((M_ + 1) / 2));
        lc.blockDim = dim3(256);
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        lc.attrs = at;
        lc.numAttrs = 1;
        void (*k)(GemvArgs) = V == 1 ? gemv_split<1> : V == 2 ? gemv_split<2> : V == 4 ? gemv_split<4> : gemv_split<8>;
        MDHB_CUDA(cudaLaunchKernelEx(&lc, k, a));
        MDHB_CUDA(cudaGetLastError());
        return;
      }
      constexpr int ROWS = 2;
      int64_t warps = (M_ + ROWS - 1) / ROWS;
      unsigned grid = static_cast<unsigned>((warps * 32 + 127) / 128);
      gemv_rows<ROWS><<<grid, 128, 0, s>>>(a);
      MDHB_CUDA(cudaGetLastError());
      return;
    }
    if (apack_m_) {
      const int32_t* ta = static_cast<const int32_t*>(ap_tab_);
      const int nt = static_cast<int>(ap_tAm_.size()), bml = static_cast<int>(ap_am_.size());
      dim3 grid(static_cast<unsigned>(apack_m_ / 64), static_cast<unsigned>((K_ + 63) / 64));
      apack_t<<<grid, 256, 0, s>>>(A, static_cast<float*>(ap_), ta, ta + nt, ta + nt + bml, bml, apack_m_, static_cast<int>(K_));
      MDHB_CUDA(cudaGetLastError());
      A = static_cast<const float*>(ap_);
    }
    if (bpack_n_) {
      const int32_t* tb = static_cast<const int32_t*>(bp_tab_);
      const int nt = static_cast<int>(bp_tBn_.size()), bnl = static_cast<int>(bp_bn_.size());
      const int64_t total = K_ * bpack_n_;
      bpack<<<static_cast<unsigned>(std::min<int64_t>(8 * sm_count(p_.opt.device), (total + 255) / 256)), 256, 0, s>>>(
          B, static_cast<float*>(bp_), tb, tb + nt, tb + nt + bnl, bnl, bpack_n_, total);
      MDHB_CUDA(cudaGetLastError());
      B = static_cast<const float*>(bp_);
    }
    GemmArgs a{A, B, C, tab_[0], tab_[1], tab_[2], tab_[3], tab_[4], tab_[5], tab_[6], tab_[7], tab_[8], tab_[9],
               static_cast<int>(K_), tilesM_, tilesN_, psak_, psbk_, klin_ ? 1 : 0, group_};
    mark_begin(s);
    dispatch(a, s);
    mark_end(s);
    MDHB_CUDA(cudaGetLastError());
  }

  Config canonical(const Config* given) const;
  bool is_gemv() const { return gemv_; }
  bool is_skinny() const { return skinny_ || cluster_; }
  bool uses_async() const { return async_ok(); }
  bool uses_pipe() const { return pipe_ok(); }
  // Table-1 knobs, set before setup(): k-tile (0 = deepest affine) and raster group (0 = default)
  void set_knobs(int bk, int group) {
    bk_want_ = bk;
    group_ = group;
  }
  int k_tile() const { return pipe_ok() ? pbk_ : BK; }
  int64_t inner_row_tiles() const { return inner_rows_; }

 private:
  void tables(const std::vector<int64_t>& t0, const std::vector<int64_t>& t1, const std::vector<int64_t>& t2,
              const std::vector<int64_t>& t3, const std::vector<int64_t>& t4, const std::vector<int64_t>& t5,
              const std::vector<int64_t>& t6, const std::vector<int64_t>& t7, const std::vector<int64_t>& t8,
              const std::vector<int64_t>& t9) {
    const std::vector<int64_t>* ts[10] = {&t0, &t1, &t2, &t3, &t4, &t5, &t6, &t7, &t8, &t9};
    size_t total = 0;
    for (auto* t : ts) total += (t->size() + 64) * sizeof(int32_t);
    std::vector<int32_t> host(total / sizeof(int32_t), 0);
    size_t cur = 0;
    size_t offs[10];
    for (int q = 0; q < 10; ++q) {
      offs[q] = cur;
      for (int64_t v : *ts[q]) {
        if (v > INT32_MAX || v < INT32_MIN) fail("Unsupported", "contraction offsets exceed int32");
        host[cur++] = static_cast<int32_t>(v);
      }
      cur = (cur + 64) / 64 * 64;
    }
    MDHB_CUDA(cudaSetDevice(p_.opt.device));
    MDHB_CUDA(cudaMalloc(&blob_, std::max<size_t>(cur, 64) * sizeof(int32_t)));
    MDHB_CUDA(cudaMemcpy(blob_, host.data(), cur * sizeof(int32_t), cudaMemcpyHostToDevice));
    for (int q = 0; q < 10; ++q) tab_[q] = static_cast<const int32_t*>(blob_) + offs[q];
  }

  template <int BM, int BN>
  void dispatch2(const GemmArgs& a, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(tilesM_ * tilesN_));
    dim3 block((BM / 8) * (BN / 8));
#define MDHB_G(AMo, BMo, CV) \
  if (amode_ == AMo && bmode_ == BMo && cvec_ == CV) { sgemm_tiled<BM, BN, AMo, BMo, CV><<<grid, block, 0, s>>>(a); return; }
#define MDHB_G2(AMo, BMo) MDHB_G(AMo, BMo, true) MDHB_G(AMo, BMo, false)
    MDHB_G2(LD_K4, LD_MN4) MDHB_G2(LD_K4, LD_K4) MDHB_G2(LD_K4, LD_SCALAR)
    MDHB_G2(LD_MN4, LD_MN4) MDHB_G2(LD_MN4, LD_K4) MDHB_G2(LD_MN4, LD_SCALAR)
    MDHB_G2(LD_SCALAR, LD_MN4) MDHB_G2(LD_SCALAR, LD_K4) MDHB_G2(LD_SCALAR, LD_SCALAR)
#undef MDHB_G2
#undef MDHB_G
  }
  bool async_ok() const {
    return BM_ == 128 && (BN_ == 128 || BN_ == 256) && bmode_ == LD_MN4 && amode_ != LD_SCALAR &&
           !std::getenv("MDHB_SGEMM_V1");
  }
  template <int TN>
  void dispatch_async(const GemmArgs& a, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(tilesM_ * tilesN_));
    if (amode_ == LD_K4) {
      if (cvec_) sgemm_async<true, true, TN><<<grid, 256, 0, s>>>(a); else sgemm_async<true, false, TN><<<grid, 256, 0, s>>>(a);
    } else {
      if (cvec_) sgemm_async<false, true, TN><<<grid, 256, 0, s>>>(a); else sgemm_async<false, false, TN><<<grid, 256, 0, s>>>(a);
    }
  }
  // v3 (sgemm_pipe): 128 x 128 tiles, any operand view (V16 where the MN dim
  // is 16-byte contiguous, else 4-byte fills), K a multiple of the k-tile
  bool pipe_ok() const {
    return ((BM_ == 128 && BN_ == 128) || (BM_ == 256 && BN_ == 64) || (BM_ == 128 && BN_ == 64)) && K_ % 8 == 0 &&
           tile_affine_ && !std::getenv("MDHB_SGEMM_V2");
  }
  int pipe_bk() const { return pbk_; }
  bool pipe_av() const { return amode_ == LD_MN4; }
  bool pipe_bv() const { return bmode_ == LD_MN4; }
  // K-contiguous A tile (16-byte fills along k): A is K4 with unit k stride
  // inside 16-deep k-tiles (MCC's implicit im2col).  Opt-in (MDHB_PIPE_AK=1):
  // bit-identical but 1186 vs 1164 us on MCC FFMA N=256 (DESIGN, dead ends)
  bool pipe_ak() const { return amode_ == LD_K4 && psak_ == 1 && pbk_ == 16 && std::getenv("MDHB_PIPE_AK"); }
  template <int PBM, int PBN, int BKT>
  void dispatch_pipe(const GemmArgs& a, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(tilesM_ * tilesN_));
    const size_t smem = PipeSmem<PBM, PBN, BKT>::FLOATS * sizeof(float);
    void (*k)(GemmArgs) = nullptr;
    if constexpr (BKT == 16) {
      if (pipe_ak()) {
        const size_t smem_ak = PipeAkSmem<PBM, PBN, 16>::FLOATS * sizeof(float);
        if (pipe_bv()) k = cvec_ ? sgemm_pipe_ak<PBM, PBN, true, true, 16> : sgemm_pipe_ak<PBM, PBN, true, false, 16>;
        else k = cvec_ ? sgemm_pipe_ak<PBM, PBN, false, true, 16> : sgemm_pipe_ak<PBM, PBN, false, false, 16>;
        MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_ak)));
        k<<<grid, (PBM / 8) * (PBN / 8), smem_ak, s>>>(a);
        return;
      }
    }
#define MDHB_P(AV, BV, CV) \
  if (pipe_av() == AV && pipe_bv() == BV && cvec_ == CV) k = sgemm_pipe<PBM, PBN, AV, BV, CV, BKT>;
    MDHB_P(true, true, true) MDHB_P(true, true, false) MDHB_P(true, false, true) MDHB_P(true, false, false)
    MDHB_P(false, true, true) MDHB_P(false, true, false) MDHB_P(false, false, true) MDHB_P(false, false, false)
#undef MDHB_P
    MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k<<<grid, (PBM / 8) * (PBN / 8), smem, s>>>(a);
  }
  void dispatch(const GemmArgs& a, cudaStream_t s) {
    if (pipe_ok()) {
      if (BM_ == 256) return pipe_bk() == 16 ? dispatch_pipe<256, 64, 16>(a, s) : dispatch_pipe<256, 64, 8>(a, s);
      if (BN_ == 64) return pipe_bk() == 16 ? dispatch_pipe<128, 64, 16>(a, s) : dispatch_pipe<128, 64, 8>(a, s);
      if (pipe_bk() == 32) return dispatch_pipe<128, 128, 32>(a, s);
      return pipe_bk() == 16 ? dispatch_pipe<128, 128, 16>(a, s) : dispatch_pipe<128, 128, 8>(a, s);
    }
    if (async_ok()) return BN_ == 256 ? dispatch_async<16>(a, s) : dispatch_async<8>(a, s);
    if (BM_ == 128 && BN_ == 128) return dispatch2<128, 128>(a, s);
    if (BM_ == 128 && BN_ == 64) return dispatch2<128, 64>(a, s);
    if (BM_ == 64 && BN_ == 128) return dispatch2<64, 128>(a, s);
    return dispatch2<64, 64>(a, s);
  }

  const Problem& p_;
  Groups g_;
  int64_t M_ = 0, N_ = 0, K_ = 0;
  int BM_ = 0, BN_ = 0, tilesM_ = 0, tilesN_ = 0;
  std::vector<int64_t> Tm_, Tn_;
  int amode_ = 0, bmode_ = 0;
  bool cvec_ = false, gemv_ = false, skinny_ = false, cluster_ = false, last_ = false;
  float* lpart_ = nullptr;
  int* lcnt_ = nullptr;
  int nw_ = 32;  // skinny_cluster column strip width
  int mg_ = 8;   // skinny_cluster m-groups (rows per thread = MT / mg_)
  CUtensorMap tmb_{};           // skinny_cluster: B slice tensor map (TMA), re-encoded when B moves
  const float* last_b_ = nullptr;
  int64_t saff_[5] = {0, 0, 0, 0, 0};  // skinny_cluster: sam, sbn, scm, scn, affine flag
  int ks_ = 0, splits_ = 0;
  int64_t sak_ = 0, sbk_ = 0;
  bool tile_affine_ = false;
  // B layout pass (bpack): original gather tables, packed copy, its row length
  std::vector<int64_t> bp_tBn_, bp_bn_, bp_bk_;
  void* bp_tab_ = nullptr;
  void* bp_ = nullptr;
  int64_t bpack_n_ = 0;
  // A layout pass (apack_t): original tables, transposed copy, its row length
  std::vector<int64_t> ap_tAm_, ap_am_, ap_ak_;
  void* ap_tab_ = nullptr;
  void* ap_ = nullptr;
  int64_t apack_m_ = 0;
  int psak_ = 0, psbk_ = 0, pbk_ = 0;
  // Table-1 knobs: k-tile (SM parts of K; 0 = the deepest affine one) and
  // raster group (SMX parts of the innermost M dim; resolved in setup)
  int bk_want_ = 0, group_ = 0;
  int64_t inner_rows_ = 1;  // row tiles of the innermost M dim
  bool klin_ = false;
  float* part_ = nullptr;
  void* blob_ = nullptr;

 public:
  std::string note_;  // why a requested tensor-core instance was declined

 private:
  const int32_t* tab_[10] = {};
};

// Places `factors` (inner first) onto the box extents T (inner -> outer):
// returns per-dim [layer] parts.
void place(const std::vector<int64_t>& T, const std::vector<std::pair<int, int64_t>>& factors,
           std::vector<std::vector<int64_t>>& parts_by_layer, const std::vector<int>& dims, bool& exact) {
  std::vector<int64_t> rem = T;
  int q = static_cast<int>(T.size()) - 1;
  for (auto [layer, f] : factors) {
    while (f > 1 && q >= 0) {
      int64_t g = std::gcd(f, rem[static_cast<size_t>(q)]);
      if (g == 1) {
        if (rem[static_cast<size_t>(q)] == 1) { --q; continue; }
        exact = false;
        break;
      }
      parts_by_layer[static_cast<size_t>(layer)][static_cast<size_t>(dims[static_cast<size_t>(q)])] *= g;
      rem[static_cast<size_t>(q)] /= g;
      f /= g;
      if (rem[static_cast<size_t>(q)] == 1) --q;
    }
    if (f > 1) exact = false;
  }
  // leftovers stay sequential in registers of the tile (RM)
  for (size_t t = 0; t < T.size(); ++t)
    parts_by_layer[5][static_cast<size_t>(dims[t])] *= rem[t];
}

Config GemmRoutine::canonical(const Config* given) const {
  if (given) return *given;
  const MdHom& e = p_.e;
  // the skinny split-K instance tiles N by 256 threads with a masked tail:
  // not a uniform partition, reported as the baseline configuration
  if (skinny_) return baseline_config(e, p_.m);
  if (p_.m.id("SMX") < 0 || p_.m.id("CC") < 0) return baseline_config(e, p_.m);
  const int D = e.D();
  // layers: 0 SMX, 1 DM, 2 WRP, 3 CC, 4 SM, 5 RM
  std::vector<std::vector<int64_t>> L(6, std::vector<int64_t>(static_cast<size_t>(D), 1));
  bool exact = true;
  if (gemv_) {
    // rows: SMX = M/8 (4 warps x 2 rows per CTA), WRP 4, RM 2; k: CC 32, RM 4, DM rest
    for (int d : g_.Md) L[0][static_cast<size_t>(d)] = e.sizes[static_cast<size_t>(d)];
    std::vector<int64_t> T(g_.Md.size(), 1);
    if (!g_.Md.empty()) {
      int64_t inner = e.sizes[static_cast<size_t>(g_.Md.back())];
      if (inner % 8 == 0) {
        L[0][static_cast<size_t>(g_.Md.back())] = inner / 8;
        L[2][static_cast<size_t>(g_.Md.back())] = 4;
        L[5][static_cast<size_t>(g_.Md.back())] = 2;
      }
    }
    for (int d : g_.Kd) L[1][static_cast<size_t>(d)] = e.sizes[static_cast<size_t>(d)];
    if (!g_.Kd.empty()) {
      int dk = g_.Kd.back();
      int64_t n = e.sizes[static_cast<size_t>(dk)];
      if (n % 128 == 0) {
        L[1][static_cast<size_t>(dk)] = n / 128;
        L[3][static_cast<size_t>(dk)] = 32;
        L[5][static_cast<size_t>(dk)] = 4;
      }
    }
  } else {
    for (size_t q = 0; q < g_.Md.size(); ++q)
      L[0][static_cast<size_t>(g_.Md[q])] = e.sizes[static_cast<size_t>(g_.Md[q])] / Tm_[q];
    for (size_t q = 0; q < g_.Nd.size(); ++q)
      L[0][static_cast<size_t>(g_.Nd[q])] = e.sizes[static_cast<size_t>(g_.Nd[q])] / Tn_[q];
    if (!g_.Md.empty()) {  // raster groups: SMX = rows per group, DM = groups (innermost M dim)
      const size_t dl = static_cast<size_t>(g_.Md.back());
      const int64_t gl = L[0][dl];
      if (group_ > 0 && gl % group_ == 0) {
        L[0][dl] = group_;
        L[1][dl] = gl / group_;
      }
    }
    place(Tm_, {{5, 4}, {3, BM_ / 8}, {5, 2}}, L, g_.Md, exact);
    place(Tn_, {{5, 4}, {3, BN_ / 8}, {5, 2}}, L, g_.Nd, exact);
    int64_t bk = pipe_ok() ? pbk_ : BK;  // the k-tile the instance runs
    for (int q = static_cast<int>(g_.Kd.size()) - 1; q >= 0; --q) {
      int d = g_.Kd[static_cast<size_t>(q)];
      int64_t g = std::gcd(bk, e.sizes[static_cast<size_t>(d)]);
      L[4][static_cast<size_t>(d)] = g;
      L[1][static_cast<size_t>(d)] = e.sizes[static_cast<size_t>(d)] / g;
      bk /= g;
    }
  }
  // sanity: per-dim products must equal the sizes, else report the baseline
  for (int d = 0; d < D; ++d) {
    int64_t p = 1;
    for (int l = 0; l < 6; ++l) p *= L[static_cast<size_t>(l)][static_cast<size_t>(d)];
    if (p != e.sizes[static_cast<size_t>(d)]) exact = false;
  }
  if (!exact) return baseline_config(e, p_.m);
  std::vector<LayerParts> lp = {{"SMX", L[0]}, {"DM", L[1]}, {"WRP", L[2]}, {"CC", L[3]}, {"SM", L[4]}, {"RM", L[5]}};
  return make_config(p_, lp, {{e.in[static_cast<size_t>(g_.a_buf)].name, "SM"}, {e.in[static_cast<size_t>(g_.b_buf)].name, "SM"}}, "RM");
}

}  // namespace

// Recognises the contraction routine class and splits the dims into groups.
bool analyze_contraction(const Problem& p, Groups& g) {
  const MdHom& e = p.e;
  const int D = e.D();
  if (e.assigns.size() != 1 || e.out.size() != 1 || e.out[0].acc.size() != 1 || e.in.size() != 2) return false;
  const Expr& f = e.assigns[0].e;
  if (f.k != EK::Mul || f.args[0].k != EK::In || f.args[1].k != EK::In) return false;
  if (f.args[0].buf == f.args[1].buf) return false;
  if (e.in[0].acc.size() != 1 || e.in[1].acc.size() != 1) return false;
  if (e.in[0].type != Ty::F64 || e.in[1].type != Ty::F64 || e.out[0].type != Ty::F64) return false;
  if (p.opt.fstore != Store::F32) return false;  // f64 storage: the generic path is the bit-exact one
  int npw = 0;
  for (auto& c : e.comb) {
    if (c.kind == Combine::PS) return false;
    if (c.kind == Combine::PW) {
      if (c.op != Fold::Add) return false;
      ++npw;
    }
  }
  if (npw == 0) return false;
  // output access: every rank is exactly one cc dim, coefficient 1, no offset
  std::vector<int> seen(static_cast<size_t>(D), 0);
  for (auto& af : e.out[0].acc[0].idx) {
    int nz = -1, cnt = 0;
    for (int d = 0; d < D; ++d)
      if (af.coeff[static_cast<size_t>(d)] != 0) {
        nz = d;
        ++cnt;
      }
    if (cnt != 1 || af.coeff[static_cast<size_t>(nz)] != 1 || af.c0 != 0) return false;
    if (e.comb[static_cast<size_t>(nz)].kind != Combine::CC) return false;
    seen[static_cast<size_t>(nz)]++;
  }
  for (int d = 0; d < D; ++d)
    if (e.comb[static_cast<size_t>(d)].kind == Combine::CC && seen[static_cast<size_t>(d)] != 1) return false;

  g.a_buf = f.args[0].buf - 1;
  g.b_buf = f.args[1].buf - 1;
  g.la = linearize(e.in[static_cast<size_t>(g.a_buf)].acc[0], p.in_ext[static_cast<size_t>(g.a_buf)], D);
  g.lb = linearize(e.in[static_cast<size_t>(g.b_buf)].acc[0], p.in_ext[static_cast<size_t>(g.b_buf)], D);
  g.lc = linearize(e.out[0].acc[0], p.out_ext[0], D);
  for (int d = 0; d < D; ++d) {
    bool da = g.la.cj[static_cast<size_t>(d)] != 0, db = g.lb.cj[static_cast<size_t>(d)] != 0;
    if (e.comb[static_cast<size_t>(d)].kind == Combine::PW) {
      g.Kd.push_back(d);
    } else if (da && db) {
      return false;  // batch dims: generic family
    } else if (da) {
      g.Md.push_back(d);
    } else {
      g.Nd.push_back(d);  // B-only, or read by neither (broadcast)
    }
  }
  if (g.Md.empty()) {  // make the streamed operand "A"
    std::swap(g.a_buf, g.b_buf);
    std::swap(g.la, g.lb);
    std::swap(g.Md, g.Nd);
  }
  if (g.Md.empty()) return false;
  // dim order inside each group: largest output stride outermost; K by A stride
  auto by = [&](const std::vector<int64_t>& cj) {
    return [&cj](int x, int y) { return std::llabs(cj[static_cast<size_t>(x)]) > std::llabs(cj[static_cast<size_t>(y)]); };
  };
  // M dims: A-contiguous dim innermost (16-byte loads of A along m when A is
  // M-major, e.g. CCSD(T)'s A[g][d][a][b]); N dims: C-contiguous innermost
  // (vector stores of the big output); K dims: unit-stride operand innermost.
  std::stable_sort(g.Md.begin(), g.Md.end(), by(g.la.cj));
  std::stable_sort(g.Nd.begin(), g.Nd.end(), by(g.lc.cj));
  {
    // K innermost = the dim where A (else B) has unit stride
    bool a_unit = false;
    for (int d : g.Kd) a_unit = a_unit || std::llabs(g.la.cj[static_cast<size_t>(d)]) == 1;
    std::stable_sort(g.Kd.begin(), g.Kd.end(), by(a_unit ? g.la.cj : g.lb.cj));
  }

  return true;
}

std::unique_ptr<Routine> make_contraction(const Problem& p, const Config* cfg, Config* cfg_out) {
  Groups g;
  if (!analyze_contraction(p, g)) return nullptr;
  const MdHom& e = p.e;
  std::string tc_why;
  if (p.opt.math != Math::FFMA) {
    auto tc = make_tc_contraction(p, g, cfg, cfg_out, &tc_why);
    if (tc) return tc;
  } else if (!cfg && std::getenv("MDHB_FFMA_CONV")) {
    // NHWC convolutions: the patch-reuse FFMA instance first (dev aid)
    std::string w;
    if (auto conv = make_ffma_conv(p, g, &w)) return conv;
  }
  auto r = std::make_unique<GemmRoutine>(p, g);
  r->note_ = tc_why;
  bool ok = false;
  if (cfg) {
    // instantiate from the configuration's per-dim tile boxes
    auto P = parts_per_asm_layer(*cfg, e, p.m);
    int smx = p.m.id("SMX"), gpu = p.m.id("GPU"), dm = p.m.id("DM"), sml = p.m.id("SM");
    if (smx < 0) fail("Unsupported", "contraction template needs an SMX layer");
    auto at = [&](int layer, int d) { return layer > 0 ? P[static_cast<size_t>(layer - 1)][static_cast<size_t>(d)] : int64_t(1); };
    std::vector<int64_t> Tm, Tn;
    int64_t bm = 1, bn = 1;
    // tile grid of an M / N dim = its SMX x DM (x GPU) parts; on the
    // innermost M dim SMX = row tiles per raster group, DM = groups
    for (size_t q = 0; q < g.Md.size(); ++q) {
      const int d = g.Md[q];
      if (q + 1 < g.Md.size() && at(dm, d) != 1) fail("Unsupported", "contraction template: DM parts of an outer M dim must be 1");
      int64_t grid = at(smx, d) * at(dm, d) * at(gpu, d);
      Tm.push_back(e.sizes[static_cast<size_t>(d)] / grid);
      bm *= Tm.back();
    }
    const int want_group = g.Md.empty() ? 0 : static_cast<int>(at(smx, g.Md.back()));
    for (int d : g.Nd) {
      if (at(dm, d) != 1) fail("Unsupported", "contraction template: DM parts of an N dim must be 1");
      int64_t grid = at(smx, d) * at(gpu, d);
      Tn.push_back(e.sizes[static_cast<size_t>(d)] / grid);
      bn *= Tn.back();
    }
    int64_t kt = 1;
    for (int d : g.Kd) {
      if (at(smx, d) != 1) fail("Unsupported", "contraction template does not split K across CTAs");
      kt *= at(sml, d);
    }
    // the k-tile = SM parts of K (8, 16 or 32: the pipelined template's ring depth)
    const int want_bk = kt == 8 || kt == 16 || kt == 32 ? static_cast<int>(kt) : 0;
    if (!want_bk && kt != 1) fail("Unsupported", "contraction template: k-tile (SM parts of K) must be 8, 16 or 32");
    bool menu = (bm == 128 || bm == 64) && (bn == 128 || bn == 64);
    r->set_knobs(want_bk, want_group);
    if (g.Nd.empty()) {
      ok = r->setup(0, 0, {}, {});
    } else if (!menu || !(ok = r->setup(static_cast<int>(bm), static_cast<int>(bn), Tm, Tn))) {
      fail("Unsupported", "contraction template instantiates BM, BN in {64, 128} with K % 8 == 0, a raster group dividing the row tiles");
    }
    if (ok && want_bk && r->k_tile() != want_bk)
      fail("Unsupported", "contraction template: k-tile 16 / 32 needs the pipelined 128-wide instance with affine k offsets");
  } else {
    const bool wide = std::getenv("MDHB_SGEMM_WIDE") != nullptr;
    const bool m64 = std::getenv("MDHB_PIPE_128x64") != nullptr;
    // long K: the pipelined 128 x 64 instance first (4 CTAs of 128 threads
    // per SM: 18.06 vs 18.65 ms for 128 x 128 at MatMul 8192^3 with FFMA2 --
    // tools/space_sweep.py); short K (a few k-tiles per output tile): the
    // 128 x 128 menu, whose 32-deep k-tiles amortise the per-tile work
    // (CCSD(T), K = 72: 525 vs 549 us)
    int64_t Kall = 1;
    for (int d : g.Kd) Kall *= e.sizes[static_cast<size_t>(d)];
    if (!std::getenv("MDHB_PIPE_128x128") && Kall >= 512) {
      auto r64 = std::make_unique<GemmRoutine>(p, g);
      r64->note_ = tc_why;
      if (r64->setup(128, 64, {}, {}) && r64->uses_pipe()) {
        if (cfg_out) *cfg_out = r64->canonical(cfg);
        return r64;
      }
    }
    // NHWC convolutions the pipelined implicit GEMM cannot tile (P x Q not
    // 128-row tiles): the patch-reuse FFMA instance (ffma_conv.cu).  Where
    // both apply the implicit GEMM is faster since FFMA2 (MCC conv2_x:
    // 1.133 vs 1.178 ms)
    if (p.opt.math == Math::FFMA) {
      std::string w;
      if (auto conv = make_ffma_conv(p, g, &w)) return conv;
    }
    const int menu[6][2] = {{128, wide ? 256 : 128}, {128, 128}, {m64 ? 128 : 256, 64}, {128, 64}, {64, 128}, {64, 64}};
    for (auto& t : menu) {
      ok = r->setup(t[0], t[1], {}, {});
      if (ok) {
        if ((t[1] == 256 && !r->uses_async()) || (t[0] == 256 && !r->uses_pipe())) {
          r = std::make_unique<GemmRoutine>(p, g);
          ok = false;
          continue;
        }
        break;
      }
    }
  }
  if (!ok) return nullptr;
  if (cfg_out) *cfg_out = r->canonical(cfg);
  return r;
}

}  // namespace mdhb

namespace mdhb {
// Tuning space of the FFMA contraction template: the (BM, BN) tile menu,
// each instance reported through its canonical Table-1 configuration.
bool contraction_project(const Problem& p, const Config& c, Config* canon) {
  Groups g;
  if (!analyze_contraction(p, g)) return false;
  return tc_project(p, g, c, canon);
}

std::vector<Config> contraction_space(const Problem& p) {
  std::vector<Config> out;
  Groups g;
  if (!analyze_contraction(p, g)) return out;
  if (p.opt.math != Math::FFMA) {
    out = tc_space(p, g);
    if (!out.empty()) return out;
  }
  // FFMA instances: tile (BM, BN) x k-tile (SM parts of K: 8 / 16 / 32,
  // the pipelined template's) x raster group (SMX parts of the innermost M
  // dim, dividing its row tiles)
  const int menu[4][2] = {{128, 128}, {128, 64}, {64, 128}, {64, 64}};
  std::set<std::string> seen;
  for (auto& t : menu) {
    std::vector<int> groups;
    {
      GemmRoutine r(p, g);
      if (!r.setup(t[0], t[1], {}, {})) continue;
      if (r.is_gemv() || r.is_skinny()) {
        Config c = r.canonical(nullptr);
        if (config_violation(c, p.e, p.m, true).empty()) out.push_back(c);
        break;
      }
      for (int64_t q = 1; q <= 64 && q <= r.inner_row_tiles(); ++q)  // divisors of the row tiles
        if (r.inner_row_tiles() % q == 0) groups.push_back(static_cast<int>(q));
    }
    for (int bk : {8, 16, 32})
      for (int grp : groups) {
        GemmRoutine r(p, g);
        r.set_knobs(bk, grp);
        if (!r.setup(t[0], t[1], {}, {}) || r.k_tile() != bk) continue;
        Config c = r.canonical(nullptr);
        if (!config_violation(c, p.e, p.m, true).empty()) continue;
        if (seen.insert(config_json(c, p.e, p.m)).second) out.push_back(c);
      }
  }
  return out;
}
}  // namespace mdhb
