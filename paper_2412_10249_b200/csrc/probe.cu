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

// Shared-memory read stream: every warp reads conflict-free 128-bit words
// (lane-contiguous), the pattern that moves 128 B per wavefront.
__global__ void __launch_bounds__(256) k_lds_stream(float* sink, int iters) {
  __shared__ float4 buf[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    buf[i] = make_float4(i * 1e-3f, 1.f, 2.f, 3.f);
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 v = buf[(idx + u * 256) & 2047];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    idx = (idx + 32) & 2047;
  }
  if (acc.x + acc.y + acc.z + acc.w == -1.2345f) sink[threadIdx.x] = acc.x;
}

}  // namespace

extern "C" IMASK_API int imask_probe_smem_peak(int device, double* bytes_per_s) {
  if (!bytes_per_s) return IMASK_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return IMASK_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(float)) != cudaSuccess) return IMASK_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, iters = 2048;
  for (int w = 0; w < 3; ++w) k_lds_stream<<<blocks, 256>>>(sink, iters);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_lds_stream<<<blocks, 256>>>(sink, iters);
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
  *bytes_per_s = (double)blocks * 256.0 * iters * 8 * 16 / (best * 1e-3);
  return IMASK_OK;
}

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
