// Vary one factor at a time from the working probe: threads, smem bytes, barrier offset.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
struct Maps { CUtensorMap a, b; };
__global__ void probe(const __grid_constant__ Maps maps, float2* out, int bar_off, int cx, int cy) {
  extern __shared__ __align__(128) unsigned char smem[];
  float2* buf = reinterpret_cast<float2*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + bar_off);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(96 * 16 * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(buf)), "l"(&maps.a), "r"(cx), "r"(cy), "r"(smem_u32(bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 1536; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
  const int threads = atoi(argv[1]), smem = atoi(argv[2]), bar_off = atoi(argv[3]), pitch = atoi(argv[4]), rows = atoi(argv[5]);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<EncodeTiledFn>(p);
  std::vector<float2> h(pitch * rows);
  for (int r = 0; r < rows; ++r) for (int c = 0; c < pitch; ++c) h[r * pitch + c] = make_float2(r, c);
  float2 *d, *o; cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 1536 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  Maps maps;
  const cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows}; const cuuint64_t strides[1] = {(cuuint64_t)pitch * 8};
  const cuuint32_t box[2] = {96, 16}, es[2] = {1, 1};
  CUresult r = enc(&maps.a, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  maps.b = maps.a;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, threads, smem>>>(maps, o, bar_off, atoi(argv[6]), atoi(argv[7]));
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float2> ho(1536); cudaMemcpy(ho.data(), o, 1536 * 8, cudaMemcpyDeviceToHost);
  printf("threads=%d smem=%d bar=%d pitch=%d rows=%d enc=%d -> %s  first=(%g,%g)\n", threads, smem, bar_off, pitch, rows, (int)r, cudaGetErrorString(e), ho[0].x, ho[0].y);
  return 0;
}
