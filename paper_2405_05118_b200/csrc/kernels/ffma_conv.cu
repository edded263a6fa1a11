// FP32 FFMA instance for the multi-channel convolution md_hom over NHWC
// (MCC, BASELINE config 4; the reference's mcc.json views, evaluated by the
// reference executor as the 7-dim fold of md_hom.hpp / interpreter.cpp):
//
//   O[n][p][q][k] = sum_{r,s,c}  I[n][p+r][q+s][c] * F[k][r][s][c]
//
// The generic FFMA contraction (sgemm_pipe) reads the implicit-GEMM A operand
// through offset tables, one 4-byte copy per element and tap.  Here a CTA
// owns PB output rows x all Q columns x all 64 output channels of one image:
//
//   * per 8-channel chunk, the input patch (PB + R - 1 rows x Q + S - 1
//     pixels x 8 channels, pixel-major as in HBM) and the filter chunk
//     (pre-transposed once per run to [c/8][r][s][c%8][k'], k' interleaving
//     the 8 channel groups' half-rows) land in shared
//     memory with 16-byte cp.async copies, three chunks in flight
//   * thread = 8 output pixels along q x 8 output channels; per (r, channel
//     pair) it loads the 8 + S - 1 input pixels it needs ONCE (LDS.64: two
//     channels) and reuses them for all S taps -- the S shifts are register
//     renames -- against 2 x LDS.128 of filter per tap: 384 FFMA per 22 LDS
//   * warps = 8 channel groups x 4 output rows; a warp's A loads hit 4
//     distinct rows (row stride = 8 or 24 words mod 32: conflict-free), its
//     B loads 8 distinct 32-byte filter segments (broadcast)
//   * stores: 8 channel-group lanes write one pixel's 256 contiguous bytes
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <sstream>

#include "contraction_common.hpp"
#include "tc_gemm.cuh"

namespace mdhb {
namespace ctr {
namespace {

constexpr int FC_CC = 8;  // channels per chunk
constexpr int FC_ST = 3;  // chunks in flight
constexpr int FC_K = 64;  // output channels (8 groups of 8)

struct FConvArgs {
  const float* I;
  const float* FT;  // [C/8][R][S][8][64]
  float* O;
  int P, Q, C;
  int64_t H;
  int PB, QG, pblocks;  // rows per CTA, column groups (QT columns each), row blocks per image
  int rsw, prow;        // patch row stride (words), patch rows
  int64_t in_n, in_h;   // input strides: image, row (pixel stride = C)
  int64_t on, op;       // output strides: image, row (pixel stride = 64)
};

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int R, int S, int QT, int MAXT>
__global__ void __launch_bounds__(MAXT, 2) ffma_conv(FConvArgs g) {
  extern __shared__ __align__(16) float sm[];
  constexpr int AW = QT + S - 1;  // input pixels one thread reads per row
  const int patch_words = g.prow * g.rsw;
  constexpr int filt_words = R * S * FC_CC * FC_K;
  const int stage_words = patch_words + filt_words;
  const int tid = threadIdx.x, T = blockDim.x;
  const int kg = tid & 7, pp = (tid >> 3) & 3, rest = tid >> 5;
  const int qg = rest % g.QG, pl = (rest / g.QG) * 4 + pp;  // 8-column group, local output row
  const int n = blockIdx.x / g.pblocks, p0 = (blockIdx.x % g.pblocks) * g.PB;
  const int chunks = g.C / FC_CC;
  const float* In = g.I + n * g.in_n;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const int wq = g.Q + S - 1;

  auto fill = [&](int ch, int st) {
    const uint32_t sp = sbase + static_cast<uint32_t>(st * stage_words) * 4;
    // patch: row by row, 2 x 16 B per pixel (no divisions in the index math)
    for (int row = 0; row < g.prow; ++row) {
      const int64_t hr = p0 + row;
      const float* srow = In + min(hr, g.H - 1) * g.in_h + ch * FC_CC;
      const uint32_t drow = sp + static_cast<uint32_t>(row * g.rsw) * 4;
      for (int x = tid; x < 2 * wq; x += T)
        cp16(drow + static_cast<uint32_t>(x) * 16, srow + static_cast<int64_t>(x >> 1) * g.C + (x & 1) * 4, hr < g.H ? 16u : 0u);
    }
    const uint32_t sf = sp + static_cast<uint32_t>(patch_words) * 4;
    const float* fsrc = g.FT + static_cast<int64_t>(ch) * filt_words;
    for (int i = tid; i < filt_words / 4; i += T) cp16(sf + static_cast<uint32_t>(i) * 16, fsrc + 4 * i, 16u);
  };

  float acc[QT][8];
#pragma unroll
  for (int j = 0; j < QT; ++j)
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) acc[j][kk] = 0.f;

#pragma unroll
  for (int st = 0; st < FC_ST - 1; ++st) {
    if (st < chunks) fill(st, st);
    cp_commit();
  }
  for (int ch = 0; ch < chunks; ++ch) {
    cp_wait<FC_ST - 2>();
    __syncthreads();
    {
      const int nx = ch + FC_ST - 1;
      if (nx < chunks) fill(nx, nx % FC_ST);
      cp_commit();
    }
    const float* sp = sm + (ch % FC_ST) * stage_words;
    const float* sf = sp + patch_words;
#pragma unroll 1
    for (int c = 0; c < FC_CC; c += 2) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float2 a[AW];
        const float* ar = sp + (pl + r) * g.rsw + qg * QT * FC_CC + c;
#pragma unroll
        for (int j = 0; j < AW; ++j) a[j] = *reinterpret_cast<const float2*>(ar + j * FC_CC);
        // filter rows for (s, cc) double-buffered in registers: the next
        // sub-block's LDS.128s are in flight during this one's 64 FFMAs
        // a 64-k filter row is stored [half][kg][4]: the 8 groups' first
        // halves fill one 128-byte line (conflict-free LDS.128), then the second
        const float* bb = sf + (r * S * FC_CC + c) * FC_K + kg * 4;
        float4 n0 = *reinterpret_cast<const float4*>(bb), n1 = *reinterpret_cast<const float4*>(bb + 32);
#pragma unroll
        for (int sub = 0; sub < 2 * S; ++sub) {
          const int s = sub >> 1, cc = sub & 1;
          const float b[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
          if (sub + 1 < 2 * S) {
            const float* bn = bb + ((((sub + 1) >> 1) * FC_CC) + ((sub + 1) & 1)) * FC_K;
            n0 = *reinterpret_cast<const float4*>(bn);
            n1 = *reinterpret_cast<const float4*>(bn + 32);
          }
#pragma unroll
          for (int j = 0; j < QT; ++j) {
            const float av = cc ? a[j + s].y : a[j + s].x;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) acc[j][kk] = fmaf(av, b[kk], acc[j][kk]);
          }
        }
      }
    }
  }
  const int p = p0 + pl;
  if (p < g.P) {
    float* o = g.O + n * g.on + static_cast<int64_t>(p) * g.op + (qg * QT) * FC_K + kg * 8;
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      __stcs(reinterpret_cast<float4*>(o + j * FC_K), make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]));
      __stcs(reinterpret_cast<float4*>(o + j * FC_K + 4), make_float4(acc[j][4], acc[j][5], acc[j][6], acc[j][7]));
    }
  }
}

// mbarrier form of ffma_conv: each chunk lands with a 4-D TMA box of the
// input ({8 c, boxpx px, prow rows, 1 n}, rows past H zero-filled; boxpx =
// Q + S - 1 rounded so the row stride is 8 or 24 words mod 32) plus one bulk
// copy of the filter chunk, completing on the slot's full mbarrier; each warp
// releases a slot on its empty mbarrier (count 8).  Lane 0 of warp 0 issues
// chunk ch + 1 at the top of iteration ch into the slot chunk ch - 2 used --
// no CTA-wide barrier per chunk, so warps drift freely within the ring.
template <int R, int S, int QT>
__global__ void __launch_bounds__(256, 2) ffma_conv_tma(const __grid_constant__ CUtensorMap tmi, FConvArgs g) {
  // used directly (not re-aligned through a generic pointer) so the loads
  // below stay LDS; the dynamic window starts 128-byte aligned (checked)
  extern __shared__ __align__(128) float sm[];
  constexpr int AW = QT + S - 1;
  constexpr int filt_words = R * S * FC_CC * FC_K;
  const int patch_words = (g.prow * g.rsw + 31) & ~31;  // 128-byte aligned filter
  if (tc::smem_u32(sm) & 127) __trap();
  const int stage_words = patch_words + filt_words;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + FC_ST * stage_words);
  uint64_t* empty = full + FC_ST;
  const int tid = threadIdx.x, lane = tid & 31;
  const int n = blockIdx.x / g.pblocks, p0 = (blockIdx.x % g.pblocks) * g.PB;
  const int chunks = g.C / FC_CC;
  const uint32_t pbytes = static_cast<uint32_t>(g.prow * g.rsw) * 4;
  auto issue = [&](int ch) {
    const int st = ch % FC_ST;
    if (ch >= FC_ST) tc::mbar_wait(&empty[st], ((ch / FC_ST) - 1) & 1);
    tc::mbar_arrive_expect_tx(&full[st], pbytes + filt_words * 4);
    float* dst = sm + st * stage_words;
    int c[4] = {ch * FC_CC, 0, p0, n};
    tc::tma_load(dst, &tmi, &full[st], 4, c);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tc::smem_u32(dst + patch_words)),
                 "l"(g.FT + static_cast<int64_t>(ch) * filt_words), "r"(filt_words * 4), "r"(tc::smem_u32(&full[st]))
                 : "memory");
  };
  if (tid == 0) {
    for (int st = 0; st < FC_ST; ++st) {
      tc::mbar_init(&full[st], 1);
      tc::mbar_init(&empty[st], 8);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmi);
    for (int ch = 0; ch < FC_ST - 1 && ch < chunks; ++ch) issue(ch);
  }
  __syncthreads();
  const int kg = tid & 7, pp = (tid >> 3) & 3, rest = tid >> 5;
  const int qg = rest % g.QG, pl = (rest / g.QG) * 4 + pp;
  float acc[QT][8];
#pragma unroll
  for (int j = 0; j < QT; ++j)
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) acc[j][kk] = 0.f;
  for (int ch = 0; ch < chunks; ++ch) {
    const int st = ch % FC_ST;
    if (tid == 0 && ch + FC_ST - 1 < chunks) issue(ch + FC_ST - 1);
    __syncwarp();
    tc::mbar_wait(&full[st], (ch / FC_ST) & 1);
    const float* sp = sm + st * stage_words;
    const float* sf = sp + patch_words;
#pragma unroll 1
    for (int c = 0; c < FC_CC; c += 2) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float2 a[AW];
        const float* ar = sp + (pl + r) * g.rsw + qg * QT * FC_CC + c;
#pragma unroll
        for (int j = 0; j < AW; ++j) a[j] = *reinterpret_cast<const float2*>(ar + j * FC_CC);
        const float* bb = sf + (r * S * FC_CC + c) * FC_K + kg * 4;
        float4 n0 = *reinterpret_cast<const float4*>(bb), n1 = *reinterpret_cast<const float4*>(bb + 32);
#pragma unroll
        for (int sub = 0; sub < 2 * S; ++sub) {
          const int s = sub >> 1, cc = sub & 1;
          const float b[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
          if (sub + 1 < 2 * S) {
            const float* bn = bb + ((((sub + 1) >> 1) * FC_CC) + ((sub + 1) & 1)) * FC_K;
            n0 = *reinterpret_cast<const float4*>(bn);
            n1 = *reinterpret_cast<const float4*>(bn + 32);
          }
#pragma unroll
          for (int j = 0; j < QT; ++j) {
            const float av = cc ? a[j + s].y : a[j + s].x;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) acc[j][kk] = fmaf(av, b[kk], acc[j][kk]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[st]);
  }
  const int p = p0 + pl;
  if (p < g.P) {
    float* o = g.O + n * g.on + static_cast<int64_t>(p) * g.op + (qg * QT) * FC_K + kg * 8;
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      __stcs(reinterpret_cast<float4*>(o + j * FC_K), make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]));
      __stcs(reinterpret_cast<float4*>(o + j * FC_K + 4), make_float4(acc[j][4], acc[j][5], acc[j][6], acc[j][7]));
    }
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn fconv_encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) fail("CudaError", "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// F[k][r][s][c] -> FT[c/8][r][s][c%8][half][kg][4], k = kg * 8 + half * 4 + e
__global__ void __launch_bounds__(256) filter_ct(const float* __restrict__ F, float* __restrict__ FT, int R, int S, int C) {
  const int total = FC_K * R * S * C;
  for (int i = blockIdx.x * 256 + threadIdx.x; i < total; i += gridDim.x * 256) {
    const int slot = i % FC_K, k = ((slot >> 2) & 7) * 8 + (slot >> 5) * 4 + (slot & 3);
    int t = i / FC_K;
    const int cc = t % FC_CC;
    t /= FC_CC;
    const int s = t % S;
    t /= S;
    const int r = t % R;
    const int ch = t / R;
    const int c = ch * FC_CC + cc;
    FT[i] = __ldg(F + ((static_cast<int64_t>(k) * R + r) * S + s) * C + c);
  }
}

class FfmaConvRoutine final : public Routine {
 public:
  explicit FfmaConvRoutine(const Problem& p) : p_(p) {}
  ~FfmaConvRoutine() override {
    if (ft_) cudaFree(ft_);
  }
  const char* family() const override { return "contraction"; }
  const char* bound() const override { return "fp32"; }
  int launches() const override { return 2; }
  double flops() const override {
    return 2.0 * cs_.N * cs_.P * cs_.Q * static_cast<double>(cs_.K) * cs_.R * cs_.S * cs_.C;
  }
  double bytes() const override { return static_cast<double>(p_.in_bytes + p_.out_bytes); }
  std::string describe() const override {
    std::ostringstream os;
    os << "{\"kernel\": \"" << (tma_ ? "ffma_conv_tma<" : "ffma_conv<") << cs_.R << "x" << cs_.S << ">\", \"math\": \"ffma\", \"M\": "
       << static_cast<int64_t>(cs_.N) * cs_.P * cs_.Q << ", \"N\": " << cs_.K << ", \"K\": " << cs_.R * cs_.S * cs_.C
       << ", \"tile\": \"" << a_.PB << " p x " << cs_.Q << " q x 64 k\", \"threads\": " << threads_
       << ", \"thread_tile\": \"" << qt_ << " q x 8 k\", \"chunk_channels\": " << FC_CC << ", \"stages\": " << FC_ST
       << ", \"smem\": " << smem_ << ", \"ctas\": " << static_cast<int64_t>(cs_.N) * a_.pblocks
       << ", \"layout_pass\": \"filter_ct: F[k][r][s][c] -> [c/8][r][s][c%8][k] per run\"}";
    return os.str();
  }

  bool setup(const ConvShape& cs, std::string* why) {
    cs_ = cs;
    if (cs.K != FC_K) return *why = "ffma conv: 64 output channels", false;
    if (cs.R != 3 || cs.S != 3) return *why = "ffma conv: 3x3 taps", false;
    if (cs.C % FC_CC) return *why = "ffma conv: C % 8", false;
    // thread = QT columns: 8, or 7 when that gives 8 full warps (Q = 56)
    qt_ = cs.Q % 56 == 0 && cs.Q / 7 == 8 ? 7 : 8;
    if (cs.Q % qt_ || cs.Q / qt_ > 8) return *why = "ffma conv: Q % 8 == 0, Q <= 64", false;
    if (cs.W != cs.Q + cs.S - 1 || cs.H < cs.P + cs.R - 1) return *why = "ffma conv: valid-convolution extents", false;
    a_.QG = cs.Q / qt_;
    const int pm = std::max(1, 256 / (32 * a_.QG));
    a_.PB = 4 * pm;
    threads_ = 32 * a_.QG * pm;
    a_.pblocks = (cs.P + a_.PB - 1) / a_.PB;
    a_.prow = a_.PB + cs.R - 1;
    int rsw = (cs.Q + cs.S - 1) * FC_CC;
    while (rsw % 32 != 8 && rsw % 32 != 24) rsw += 4;
    a_.rsw = rsw;
    a_.P = cs.P;
    a_.Q = cs.Q;
    a_.C = cs.C;
    a_.H = cs.H;
    a_.in_h = cs.W * cs.C;
    a_.in_n = cs.H * a_.in_h;
    a_.op = cs.oe[2] * cs.oe[3];
    a_.on = cs.oe[1] * a_.op;
    if (cs.oe[2] != cs.Q) return *why = "ffma conv: output row extent", false;
    smem_ = static_cast<size_t>(FC_ST) * (a_.prow * a_.rsw + cs.R * cs.S * FC_CC * FC_K) * 4;
    if (smem_ > 113 * 1024) return *why = "ffma conv: stages exceed half the shared memory", false;
    // warp-specialised TMA instance (default): the TMA box lands rows densely,
    // so the box is one pixel wider when that makes the stride 8 / 24 mod 32
    tma_ = !std::getenv("MDHB_FCONV_CPASYNC");
    if (tma_) {
      boxpx_ = cs.Q + cs.S - 1;
      while ((boxpx_ * FC_CC) % 32 != 8 && (boxpx_ * FC_CC) % 32 != 24) ++boxpx_;
      if (boxpx_ > 256 || a_.prow > 256 || threads_ != 256) tma_ = false;
    }
    if (tma_) {
      a_.rsw = boxpx_ * FC_CC;
      const size_t pw = (static_cast<size_t>(a_.prow) * a_.rsw + 31) & ~size_t(31);
      smem_ = FC_ST * (pw + cs.R * cs.S * FC_CC * FC_K) * 4 + 2 * FC_ST * 8;
      if (smem_ > 113 * 1024) tma_ = false;
    }
    if (!tma_) {
      a_.rsw = rsw;
      smem_ = static_cast<size_t>(FC_ST) * (a_.prow * a_.rsw + cs.R * cs.S * FC_CC * FC_K) * 4;
    }
    return true;
  }

  void launch(const void* const* d_in, void* const* d_out, cudaStream_t s) override {
    const int nf = FC_K * cs_.R * cs_.S * cs_.C;
    if (!ft_) MDHB_CUDA(cudaMalloc(&ft_, static_cast<size_t>(nf) * 4));
    filter_ct<<<std::min(4 * sm_count(p_.opt.device), (nf + 255) / 256), 256, 0, s>>>(
        static_cast<const float*>(d_in[cs_.fb]), static_cast<float*>(ft_), cs_.R, cs_.S, cs_.C);
    MDHB_CUDA(cudaGetLastError());
    MarkScope mark(this, s);  // the convolution kernel below is the dominant one
    FConvArgs a = a_;
    a.I = static_cast<const float*>(d_in[cs_.ib]);
    a.FT = static_cast<const float*>(ft_);
    a.O = static_cast<float*>(d_out[0]);
    if (tma_) {
      if (a.I != last_i_) {
        cuuint64_t dims[4] = {static_cast<cuuint64_t>(cs_.C), static_cast<cuuint64_t>(cs_.W), static_cast<cuuint64_t>(cs_.H),
                              static_cast<cuuint64_t>(cs_.N)};
        cuuint64_t strides[3] = {static_cast<cuuint64_t>(cs_.C) * 4, static_cast<cuuint64_t>(cs_.W * cs_.C) * 4,
                                 static_cast<cuuint64_t>(cs_.H * cs_.W * cs_.C) * 4};
        cuuint32_t box[4] = {FC_CC, static_cast<cuuint32_t>(boxpx_), static_cast<cuuint32_t>(a_.prow), 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = fconv_encoder()(&tmi_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(a.I), dims, strides, box, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail("CudaError", "cuTensorMapEncodeTiled (ffma conv input) failed (" + std::to_string(static_cast<int>(r)) + ")");
        last_i_ = a.I;
      }
      auto k = qt_ == 7 ? ffma_conv_tma<3, 3, 7> : ffma_conv_tma<3, 3, 8>;
      MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
      k<<<static_cast<unsigned>(static_cast<int64_t>(cs_.N) * a_.pblocks), 256, smem_, s>>>(tmi_, a);
      MDHB_CUDA(cudaGetLastError());
      return;
    }
    auto k = qt_ == 7 ? ffma_conv<3, 3, 7, 256> : threads_ <= 224 ? ffma_conv<3, 3, 8, 224> : ffma_conv<3, 3, 8, 256>;
    MDHB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
    k<<<static_cast<unsigned>(static_cast<int64_t>(cs_.N) * a_.pblocks), threads_, smem_, s>>>(a);
    MDHB_CUDA(cudaGetLastError());
  }

 private:
  const Problem& p_;
  ConvShape cs_;
  FConvArgs a_{};
  int threads_ = 0, qt_ = 8, boxpx_ = 0;
  bool tma_ = false;
  CUtensorMap tmi_{};
  const void* last_i_ = nullptr;
  size_t smem_ = 0;
  void* ft_ = nullptr;
};

}  // namespace

std::unique_ptr<Routine> make_ffma_conv(const Problem& p, const Groups& g, std::string* why) {
  if (std::getenv("MDHB_NO_FFMA_CONV")) return nullptr;
  if (p.e.D() != 7 || p.e.in.size() != 2 || p.e.out.size() != 1) return nullptr;
  for (int ib : {g.a_buf, g.b_buf}) {
    const int fb = ib == g.a_buf ? g.b_buf : g.a_buf;
    ConvShape cs;
    std::string w;
    if (!nhwc_conv_shape(p, ib, fb, &cs, &w)) {
      *why = w;
      continue;
    }
    auto r = std::make_unique<FfmaConvRoutine>(p);
    if (r->setup(cs, &w)) return r;
    *why = w;
  }
  return nullptr;
}

}  // namespace ctr
}  // namespace mdhb
