// Solver metrics on the device (run()'s record rows, solvers.py:382-390): the
// squared distance ||x - ref||^2 accumulated in float64 with a fixed-order
// reduction (block partials summed in block order by the last block), so
// recording a row costs one small launch and an 8-byte async read-back
// instead of a host synchronisation.
#include <cuda_runtime.h>

#include "imask_b200.h"

namespace {

constexpr int kBlocks = IMASK_SQDIST_SCRATCH - 2;
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

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// rows == nullptr: *result = ||x - ref||^2. Otherwise a metric row: at slot
// k = rows[0] (a 64-bit counter) rows[2 + 2k] = ||x - ref||^2 and
// rows[3 + 2k] = the device's global timer (ns) when the value was final,
// then the counter advances -- no host involvement per row.
__global__ void __launch_bounds__(kThreads)
k_sq_dist(const float* __restrict__ x, const float* __restrict__ ref, int64_t n,
          double* __restrict__ out, double* __restrict__ result, double* __restrict__ rows) {
  // out[1 .. kBlocks]: block partials; out[kBlocks + 1] (as an unsigned counter):
  // blocks done. The last block to finish sums the partials in block order, so
  // the result does not depend on scheduling.
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (int64_t)kBlocks * kThreads) {
    const double d = (double)x[i] - (ref ? (double)ref[i] : 0.0);
    s = fma(d, d, s);
  }
  s = block_sum(s);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    out[1 + blockIdx.x] = s;
    __threadfence();
    unsigned int* done = reinterpret_cast<unsigned int*>(out + 1 + kBlocks);
    last = atomicAdd(done, 1u) == kBlocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int i = threadIdx.x; i < kBlocks; i += kThreads) t += ((volatile double*)out)[1 + i];
  t = block_sum(t);
  if (threadIdx.x == 0) {
    if (rows) {
      unsigned long long* slot = reinterpret_cast<unsigned long long*>(rows);
      const unsigned long long k = *slot;
      rows[2 + 2 * k] = t;
      rows[3 + 2 * k] = (double)globaltimer_ns();
      *slot = k + 1;
    } else {
      *result = t;
    }
    *reinterpret_cast<unsigned int*>(out + 1 + kBlocks) = 0u;  // re-arm for the next call
  }
}

}  // namespace

extern "C" IMASK_API int imask_sq_dist(const float* x, const float* ref, int64_t n, double* out,
                                       double* result, void* stream) {
  if (!x || !out || n < 0) return IMASK_EINVAL;
  k_sq_dist<<<kBlocks, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, ref, n, out, result ? result : out, nullptr);
  return cudaGetLastError() == cudaSuccess ? IMASK_OK : IMASK_ECUDA;
}

extern "C" IMASK_API int imask_metric_row(const float* x, const float* ref, int64_t n,
                                          double* scratch, double* rows, void* stream) {
  if (!x || !scratch || !rows || n < 0) return IMASK_EINVAL;
  k_sq_dist<<<kBlocks, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, ref, n, scratch, nullptr, rows);
  return cudaGetLastError() == cudaSuccess ? IMASK_OK : IMASK_ECUDA;
}
