// Development probe for the tcgen05 TF32 path: one 128 x BN tile, K = 32.
// Prints TMA-landed shared memory and the TMEM accumulator against a host
// reference, for B K-major and B MN-major.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2405_05118_b200/csrc/kernels \
//        tools/tc_debug.cu -o /tmp/tc_debug -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "tc_gemm.cuh"

using namespace mdhb::tc;

constexpr int BM = 128, BN = 64, BK = 32;

template <bool B_MN>
__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* out,
                      float* smem_dump, uint32_t lbo, uint32_t sbo, uint32_t kstep, uint32_t layout) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + BM * BK * 4;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + BN * BK * 4);
  uint64_t* done = bar + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, (BM + BN) * BK * 4);
    int c[5] = {0, 0, 0, 0, 0};
    tma_load(sa, &ta, bar, 2, c);
    if (B_MN) {
      for (int j = 0; j < BN / 32; ++j) {
        int cj[5] = {32 * j, 0, 0, 0, 0};
        tma_load(sb + j * 4096, &tb, bar, 2, cj);
      }
    } else {
      tma_load(sb, &tb, bar, 2, c);
    }
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < (BM + BN) * BK; i += blockDim.x) smem_dump[i] = reinterpret_cast<float*>(smem)[i];
  __syncthreads();
  if (threadIdx.x == 32) {
    tc_fence_after();
    constexpr uint32_t idesc = instr_desc(2, 0, B_MN ? 1 : 0, BM, BN);
    uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    for (int k = 0; k < BK / 8; ++k) {
      uint64_t da = sw128_desc(a0 + k * 32, 16, 1024);
      uint64_t db = B_MN ? umma_desc(b0 + k * kstep, lbo, sbo, layout) : sw128_desc(b0 + k * 32, 16, 1024);
      mma<true>(tmem, da, db, idesc, k > 0);
    }
    mma_commit(done);
  }
  if (warp >= 4) {  // warps 4..7 -> lane quarters 0..3
    mbar_wait(done, 0);
    tc_fence_after();
    int q = warp & 3;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c0, r);
      for (int j = 0; j < 32; ++j) out[(q * 32 + lane) * BN + c0 + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 64);
}

int main() {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  Enc enc = reinterpret_cast<Enc>(fp);
  std::vector<float> A(BM * BK), Bk(BN * BK), Bn(BK * BN);
  for (int m = 0; m < BM; ++m)
    for (int k = 0; k < BK; ++k) A[m * BK + k] = ((m * 7 + k * 3) % 11 - 5) * 0.25f;
  for (int n = 0; n < BN; ++n)
    for (int k = 0; k < BK; ++k) {
      float v = ((n * 5 + k * 2) % 9 - 4) * 0.25f;
      Bk[n * BK + k] = v;  // [N][K]
      Bn[k * BN + n] = v;  // [K][N]
    }
  float *dA, *dB, *dO, *dS;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, Bk.size() * 4);
  cudaMalloc(&dO, BM * BN * 4);
  cudaMalloc(&dS, (BM + BN) * BK * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  cuuint64_t adims[2] = {BK, BM}, astr[1] = {BK * 4};
  cuuint32_t abox[2] = {BK, BM}, es[2] = {1, 1};
  printf("encA %d\n", enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, adims, astr, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  uint32_t variants[6][5] = {{4096, 512, 1024, 1, 1}, {512, 4096, 1024, 1, 1}, {4096, 1024, 1024, 1, 1}, {4096, 512, 1024, 1, 0}, {4096, 1024, 1024, 2, 0}, {4096, 512, 512, 1, 1}};
  for (int vi = 0; vi < 7; ++vi) {
    int mn = vi > 0;
    uint32_t* V = variants[vi > 0 ? vi - 1 : 0];
    printf("variant lbo=%u sbo=%u kstep=%u layout=%u tma32b=%u\n", V[0], V[1], V[2], V[3], V[4]);
    if (mn == 0) {
      cudaMemcpy(dB, Bk.data(), Bk.size() * 4, cudaMemcpyHostToDevice);
      cuuint64_t bd[2] = {BK, BN}, bs[1] = {BK * 4};
      cuuint32_t bb[2] = {BK, BN};
      printf("encB %d\n", enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, bd, bs, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    } else {
      cudaMemcpy(dB, Bn.data(), Bn.size() * 4, cudaMemcpyHostToDevice);
      cuuint64_t bd[2] = {BN, BK}, bs[1] = {BN * 4};
      cuuint32_t bb[2] = {32, BK};
      printf("encB %d\n", enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, bd, bs, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              V[4] ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    }
    cudaMemset(dO, 0, BM * BN * 4);
    size_t smem = (BM + BN) * BK * 4 + 2048;
    if (mn) {
      cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      probe<true><<<1, 256, smem>>>(ta, tb, dO, dS, V[0], V[1], V[2], V[3]);
    } else {
      cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      probe<false><<<1, 256, smem>>>(ta, tb, dO, dS, 16, 1024, 32, 2);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("B %s-major: kernel %s\n", mn ? "MN" : "K", cudaGetErrorString(e));
    std::vector<float> O(BM * BN), S((BM + BN) * BK);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
    printf("  smem A[0..7]: ");
    for (int i = 0; i < 8; ++i) printf("%g ", S[i]);
    printf("\n  host A[0..7]: ");
    for (int i = 0; i < 8; ++i) printf("%g ", A[i]);
    printf("\n  smem B[0..7]: ");
    for (int i = 0; i < 8; ++i) printf("%g ", S[BM * BK + i]);
    int bad = 0;
    double maxerr = 0;
    for (int m = 0; m < BM; ++m)
      for (int n = 0; n < BN; ++n) {
        double ref = 0;
        for (int k = 0; k < BK; ++k) ref += A[m * BK + k] * Bk[n * BK + k];
        double err = std::fabs(ref - O[m * BN + n]);
        maxerr = std::max(maxerr, err);
        bad += err > 1e-6;
      }
    printf("\n  C[0][0..3] = %g %g %g %g ; bad %d / %d, maxerr %g\n", O[0], O[1], O[2], O[3], bad, BM * BN, maxerr);
  }
  return 0;
}
