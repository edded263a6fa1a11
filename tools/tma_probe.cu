// Dev probe: one 2-D TMA tile load (box {32, 1}, no swizzle) into shared
// memory from a chosen thread, then a copy-out; prints whether it worked.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap tv, float* out, int issuer, int c0, int c1) {
  __shared__ __align__(128) float buf[64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == issuer) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(128u) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su(buf)), "l"(&tv), "r"(c0), "r"(c1), "r"(su(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(done) : "r"(su(&bar)) : "memory");
  if (threadIdx.x < 32) out[threadIdx.x] = buf[threadIdx.x];
}

int main() {
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(fp);
  const int W = 520, H = 27;
  float* d; float* o;
  cudaMalloc(&d, W * H * 4); cudaMalloc(&o, 32 * 4);
  float h[W * H]; for (int i = 0; i < W * H; ++i) h[i] = i;
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 4; ++variant) {
    CUtensorMap m;
    cuuint64_t dims[2] = {W, H}, str[1] = {W * 4};
    cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int threads = variant < 2 ? 32 : 288, issuer = variant < 2 ? 0 : 256, c0 = variant % 2 ? 5 : 0;
    probe<<<1, threads>>>(m, o, issuer, c0, 3);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[32];
    cudaMemcpy(ho, o, sizeof ho, cudaMemcpyDeviceToHost);
    printf("variant %d encode %d kernel %s out[0]=%g out[31]=%g (want %d)\n", variant, (int)r, cudaGetErrorString(e), ho[0], ho[31], 3 * W + c0);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
