// Solver metrics on the device (run()'s record rows, solvers.py:382-390): the
// squared distance ||x - ref||^2 accumulated in float64 with a fixed-order
// two-kernel reduction (deterministic), so recording a row costs two small
// launches and an 8-byte async read-back instead of a host synchronisation.
#include <cuda_runtime.h>

#include "imask_b200.h"

namespace {

constexpr int kBlocks = IMASK_SQDIST_SCRATCH - 1;
constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

__global__ void __launch_bounds__(kThreads)
k_sq_dist_partial(const float* __restrict__ x, const float* __restrict__ ref, int64_t n,
                  double* __restrict__ out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (int64_t)kBlocks * kThreads) {
    const double d = (double)x[i] - (ref ? (double)ref[i] : 0.0);
    s = fma(d, d, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) out[1 + blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) k_sq_dist_final(double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < kBlocks; i += kThreads) s += out[1 + i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[0] = s;
}

}  // namespace

extern "C" IMASK_API int imask_sq_dist(const float* x, const float* ref, int64_t n, double* out,
                                       void* stream) {
  if (!x || !out || n < 0) return IMASK_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  k_sq_dist_partial<<<kBlocks, kThreads, 0, s>>>(x, ref, n, out);
  k_sq_dist_final<<<1, kThreads, 0, s>>>(out);
  return cudaGetLastError() == cudaSuccess ? IMASK_OK : IMASK_ECUDA;
}
