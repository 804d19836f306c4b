// Reproduce k_forward_tma's TMA usage: 256 threads, 51.5 KB smem, two 96x16 boxes
// per barrier at offsets 0/12288 (stage 0) and 24576/36864 (stage 1), mbarriers at 49152.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
struct Maps { CUtensorMap row, row_m, col, col_m; };

__global__ void __launch_bounds__(256) probe(const __grid_constant__ Maps maps, float2* out, int rows,
                                             int variant, int nloads, int rowmode) {
  extern __shared__ __align__(128) unsigned char smem[];
  float2* stage = reinterpret_cast<float2*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 49152);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool trans = (blockIdx.x & 1) && (variant & 1);
  const CUtensorMap* mm = trans ? &maps.col : &maps.row;
  const CUtensorMap* mmm = trans ? &maps.col_m : &maps.row_m;
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < 2; ++i) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[i])),
                     "r"(nloads * 12288) : "memory");
        const int col = (((int)(blockIdx.x % 40) - 20 + 49) & ~1);
        const int row = rowmode == 0 ? (i * 16 + blockIdx.x) % rows : (rowmode == 1 ? 0 : (i * 16) % rows);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(stage + (i * 2) * 1536)),
                     "l"(mm), "r"(col), "r"(row), "r"(smem_u32(&full[i])) : "memory");
        if (nloads == 2) asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(stage + (i * 2 + 1) * 1536)),
                     "l"(mmm), "r"(col), "r"(row), "r"(smem_u32(&full[i])) : "memory");
      }
    }
    __syncwarp();
  }
  for (int i = 0; i < 2; ++i)
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                 ::"r"(smem_u32(&full[i])), "r"(0) : "memory");
  if (blockIdx.x == 0) for (int k = threadIdx.x; k < 1536; k += 256) out[k] = stage[k];
}

int main(int argc, char** argv) {
  const int nloads = atoi(argv[1]), rowmode = atoi(argv[2]), ctas = atoi(argv[3]), nsel = atoi(argv[4]);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<EncodeTiledFn>(p);
  for (int n : {nsel}) {
    const int pitch = (n + 98) & ~1, rows = n;
    std::vector<float2> h(pitch * rows);
    for (int r = 0; r < rows; ++r) for (int c = 0; c < pitch; ++c) h[r * pitch + c] = make_float2(r, c);
    float2 *d[4], *o;
    for (auto& x : d) { cudaMalloc(&x, h.size() * 8); cudaMemcpy(x, h.data(), h.size() * 8, cudaMemcpyHostToDevice); }
    cudaMalloc(&o, 1536 * 8);
    Maps maps;
    CUtensorMap* ms[4] = {&maps.row, &maps.row_m, &maps.col, &maps.col_m};
    for (int k = 0; k < 4; ++k) {
      const cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
      const cuuint64_t strides[1] = {(cuuint64_t)pitch * 8};
      const cuuint32_t box[2] = {96, 16}, es[2] = {1, 1};
      CUresult r = enc(ms[k], CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d[k], dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) printf("encode %d failed %d\n", k, (int)r);
    }
    const size_t smem = 51504;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int variant = 0; variant < 2; ++variant) {
      probe<<<ctas, 256, smem>>>(maps, o, rows, variant, nloads, rowmode);
      printf("n=%d variant %d: %s\n", n, variant, cudaGetErrorString(cudaDeviceSynchronize()));
    }
  }
  return 0;
}
