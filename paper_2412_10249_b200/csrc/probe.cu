// Measurement helper for bench.py's roofline: the projectors are
// FP32-issue bound, and the FP32 peak is not in MEASURED_PEAKS.json, so it is
// measured here with an FFMA-chain microbenchmark on the live clocks.
#include <cuda_runtime.h>

#include "imask_b200.h"

namespace {

constexpr int kChains = 8;

// kChains independent FFMA chains per thread; the result is stored only when
// an impossible condition holds, which keeps the chains alive without traffic.
__global__ void __launch_bounds__(256) k_ffma_chain(float* sink, int iters, float a, float b) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      v[c] = fmaf(v[c], a, b);
      v[c] = fmaf(v[c], a, b);
      v[c] = fmaf(v[c], a, b);
      v[c] = fmaf(v[c], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == -1.2345f) sink[threadIdx.x] = s;
}

}  // namespace

extern "C" IMASK_API int imask_probe_ffma_peak(int device, double* ffma_per_s) {
  if (!ffma_per_s) return IMASK_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return IMASK_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(float)) != cudaSuccess) return IMASK_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, iters = 4096;
  const float a = 0.999f, b = 1e-4f;
  for (int w = 0; w < 3; ++w) k_ffma_chain<<<blocks, 256>>>(sink, iters, a, b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_ffma_chain<<<blocks, 256>>>(sink, iters, a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return IMASK_ECUDA;
  *ffma_per_s = (double)blocks * 256.0 * iters * kChains * 4 / (best * 1e-3);
  return IMASK_OK;
}
