// Device helpers of the solver metric rows (run()'s record rows,
// solvers.py:382-390): float64 block sums in a fixed order and the device timer,
// shared by the stand-alone reduction (metrics.cu) and the image-side SAGA
// kernels that fold the row in (sketch.cu).
#pragma once
#include <cuda_runtime.h>

namespace imask {

// Sum of v over a block of kT threads (a multiple of 32, <= 1024): xor tree in
// each warp, then the warp sums by one warp -- the same order every launch.
// Every thread of the block must call it; the result is valid in thread 0.
template <int kT>
__device__ __forceinline__ double metric_block_sum(double v) {
  __shared__ double red[kT / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // red may still be read by a previous call
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < kT / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

__device__ __forceinline__ unsigned long long metric_timer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Block-level tail of a fused metric row: `s` is this thread's partial of
// ||x - ref||^2. part[1 + block] receives the block sums; the last block to
// finish (counter at part[1 + n_blocks], zero before the launch and re-armed
// here) adds them in block order and writes rows[2 + 2k] = sum,
// rows[3 + 2k] = timer at slot k = rows[0] (a 64-bit counter), k -> k + 1.
template <int kT>
__device__ __forceinline__ void metric_row_tail(double s, double* __restrict__ part,
                                                double* __restrict__ rows, unsigned block,
                                                unsigned n_blocks) {
  s = metric_block_sum<kT>(s);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[1 + block] = s;
    __threadfence();
    unsigned int* done = reinterpret_cast<unsigned int*>(part + 1 + n_blocks);
    last = atomicAdd(done, 1u) == n_blocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned i = threadIdx.x; i < n_blocks; i += kT) t += ((volatile double*)part)[1 + i];
  t = metric_block_sum<kT>(t);
  if (threadIdx.x == 0) {
    unsigned long long* slot = reinterpret_cast<unsigned long long*>(rows);
    const unsigned long long k = *slot;
    rows[2 + 2 * k] = t;
    rows[3 + 2 * k] = (double)metric_timer_ns();
    *slot = k + 1;
    *reinterpret_cast<unsigned int*>(part + 1 + n_blocks) = 0u;
  }
}

}  // namespace imask
