// Standalone check of the TMA + mbarrier helpers used by k_forward_tma:
// load a 96 x 16 box of 8-byte elements from a padded 2-D array and compare.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

struct Maps { CUtensorMap a, b; };

__global__ void probe(const __grid_constant__ Maps maps, float2* out, int c0, int r0, int variant) {
  extern __shared__ __align__(128) unsigned char smem[];
  float2* buf = reinterpret_cast<float2*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 96 * 16 * 8);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    if (variant & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(96 * 16 * 8) : "memory");
    const CUtensorMap* m = (variant & 2) ? &maps.b : &maps.a;
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(buf)),
        "l"(m), "r"(c0), "r"(r0), "r"(smem_u32(bar)) : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 96 * 16; i += blockDim.x) out[i] = buf[i];
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) { printf("no entry point\n"); return 1; }
  auto enc = reinterpret_cast<EncodeTiledFn>(p);
  const int pitch = 1122, rows = 64;
  std::vector<float2> h(pitch * rows);
  for (int r = 0; r < rows; ++r) for (int c = 0; c < pitch; ++c) h[r * pitch + c] = make_float2(r, c);
  float2 *d, *o;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 96 * 16 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  Maps maps;
  const cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch * 8};
  const cuuint32_t box[2] = {96, 16}, es[2] = {1, 1};
  CUresult r1 = enc(&maps.a, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  maps.b = maps.a;
  printf("encode rc=%d sizeof(Maps)=%zu align=%zu\n", (int)r1, sizeof(Maps), alignof(Maps));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 16 * 8 + 64);
  for (int variant = 0; variant < 4; ++variant) {
    cudaMemset(o, 0, 96 * 16 * 8);
    probe<<<1, 128, 96 * 16 * 8 + 64>>>(maps, o, 100, 5, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess) return 2;
    std::vector<float2> ho(96 * 16);
    cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 16; ++r) for (int c = 0; c < 96; ++c) {
      float2 v = ho[r * 96 + c];
      if (v.x != 5 + r || v.y != 100 + c) ++bad;
    }
    printf("  mismatches %d (first %f %f)\n", bad, ho[0].x, ho[0].y);
  }
  // out-of-bounds box (negative column) -> zero fill
  probe<<<1, 128, 96 * 16 * 8 + 64>>>(maps, o, -40, 60, 1);
  printf("oob: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
