// What a small HBM-streaming kernel can reach on B200 when timed like bench.py's
// hbm_kernels (one cold launch between CUDA events) and when timed back to back
// over rotating buffer sets larger than L2. Mimics the image-side SAGA update
// (read x, sum [, tab, bp]; write x, sum [, tab]) on d = 1024^2 floats.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

struct Bufs { float *x, *sum, *tab, *bp; };

__global__ void k_empty() {}

__global__ void k_flush(const float4* __restrict__ p, size_t n, float* sink) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(p + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345f) *sink = acc;
}

// one float4 per array per thread; kFull: 4 reads 3 writes, else 2 reads 2 writes
template <bool kFull>
__global__ void __launch_bounds__(256) k_one(Bufs b, float s) {
  const size_t g = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  float4 sum = *reinterpret_cast<const float4*>(b.sum + g);
  float4 xv = *reinterpret_cast<const float4*>(b.x + g);
  float4 tab = make_float4(0, 0, 0, 0), pn = make_float4(1, 2, 3, 4);
  if (kFull) {
    tab = *reinterpret_cast<const float4*>(b.tab + g);
    pn = __ldg(reinterpret_cast<const float4*>(b.bp + g));
  }
  float4 d = make_float4(pn.x - tab.x, pn.y - tab.y, pn.z - tab.z, pn.w - tab.w);
  xv.x = fmaf(-s, d.x + sum.x, xv.x); xv.y = fmaf(-s, d.y + sum.y, xv.y);
  xv.z = fmaf(-s, d.z + sum.z, xv.z); xv.w = fmaf(-s, d.w + sum.w, xv.w);
  sum.x = fmaf(0.25f, d.x, sum.x); sum.y = fmaf(0.25f, d.y, sum.y);
  sum.z = fmaf(0.25f, d.z, sum.z); sum.w = fmaf(0.25f, d.w, sum.w);
  *reinterpret_cast<float4*>(b.sum + g) = sum;
  *reinterpret_cast<float4*>(b.x + g) = xv;
  if (kFull) *reinterpret_cast<float4*>(b.tab + g) = pn;
}

// U float4 per array per thread, all loads issued before any use
template <bool kFull, int U>
__global__ void __launch_bounds__(256) k_multi(Bufs b, float s, size_t n4) {
  const size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  float4 sum[U], xv[U], tab[U], pn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const size_t g = (base + (size_t)u * blockDim.x) * 4;
    sum[u] = *reinterpret_cast<const float4*>(b.sum + g);
    xv[u] = *reinterpret_cast<const float4*>(b.x + g);
    if (kFull) {
      tab[u] = *reinterpret_cast<const float4*>(b.tab + g);
      pn[u] = __ldg(reinterpret_cast<const float4*>(b.bp + g));
    } else {
      tab[u] = make_float4(0, 0, 0, 0);
      pn[u] = make_float4(1, 2, 3, 4);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const size_t g = (base + (size_t)u * blockDim.x) * 4;
    float4 d = make_float4(pn[u].x - tab[u].x, pn[u].y - tab[u].y, pn[u].z - tab[u].z, pn[u].w - tab[u].w);
    float4 x = xv[u], sm = sum[u];
    x.x = fmaf(-s, d.x + sm.x, x.x); x.y = fmaf(-s, d.y + sm.y, x.y);
    x.z = fmaf(-s, d.z + sm.z, x.z); x.w = fmaf(-s, d.w + sm.w, x.w);
    sm.x = fmaf(0.25f, d.x, sm.x); sm.y = fmaf(0.25f, d.y, sm.y);
    sm.z = fmaf(0.25f, d.z, sm.z); sm.w = fmaf(0.25f, d.w, sm.w);
    *reinterpret_cast<float4*>(b.sum + g) = sm;
    *reinterpret_cast<float4*>(b.x + g) = x;
    if (kFull) *reinterpret_cast<float4*>(b.tab + g) = pn[u];
  }
}

int main() {
  const size_t d = 1024 * 1024;
  const int K = 20;  // rotating sets: K * 29 MB > L2
  std::vector<Bufs> sets(K);
  for (auto& b : sets) {
    CK(cudaMalloc(&b.x, d * 4)); CK(cudaMalloc(&b.sum, d * 4));
    CK(cudaMalloc(&b.tab, d * 4)); CK(cudaMalloc(&b.bp, d * 4));
    CK(cudaMemset(b.x, 0, d * 4)); CK(cudaMemset(b.sum, 0, d * 4));
    CK(cudaMemset(b.tab, 0, d * 4)); CK(cudaMemset(b.bp, 0, d * 4));
  }
  float4* fl; float* sink;
  const size_t fn = (size_t)512 * 1024 * 1024 / 16;
  CK(cudaMalloc(&fl, fn * 16)); CK(cudaMemset(fl, 0, fn * 16)); CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto flush = [&] { k_flush<<<148 * 8, 256>>>(fl, fn, sink); };

  auto run = [&](const char* name, double bytes, auto launch) {
    // cold single launches
    std::vector<float> t;
    for (int r = 0; r < 25; ++r) {
      flush();
      cudaEventRecord(e0);
      launch(sets[r % K]);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 5) t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    const float cold = t[t.size() / 2];
    // back to back over rotating sets
    t.clear();
    for (int r = 0; r < 8; ++r) {
      flush();
      cudaEventRecord(e0);
      for (int k = 0; k < K; ++k) launch(sets[k]);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) t.push_back(ms / K);
    }
    std::sort(t.begin(), t.end());
    const float b2b = t[t.size() / 2];
    printf("%-34s cold %6.2f us %6.0f GB/s | back-to-back %6.2f us %6.0f GB/s\n", name, cold * 1e3,
           bytes / (cold * 1e-3) / 1e9, b2b * 1e3, bytes / (b2b * 1e-3) / 1e9);
    CK(cudaGetLastError());
  };
  const size_t n4 = d / 4;
  run("empty kernel", 0.0, [&](Bufs) { k_empty<<<1, 32>>>(); });
  run("coarse-like 1024x256 U1", 16.0 * d, [&](Bufs b) { k_one<false><<<n4 / 256, 256>>>(b, 0.1f); });
  run("coarse-like 2048x128 U1", 16.0 * d, [&](Bufs b) { k_one<false><<<n4 / 128, 128>>>(b, 0.1f); });
  run("coarse-like 512x256 U2", 16.0 * d, [&](Bufs b) { k_multi<false, 2><<<n4 / 512, 256>>>(b, 0.1f, n4); });
  run("coarse-like 256x256 U4", 16.0 * d, [&](Bufs b) { k_multi<false, 4><<<n4 / 1024, 256>>>(b, 0.1f, n4); });
  run("coarse-like 1024x128 U2", 16.0 * d, [&](Bufs b) { k_multi<false, 2><<<n4 / 256, 128>>>(b, 0.1f, n4); });
  run("full-like 1024x256 U1", 28.0 * d, [&](Bufs b) { k_one<true><<<n4 / 256, 256>>>(b, 0.1f); });
  run("full-like 2048x128 U1", 28.0 * d, [&](Bufs b) { k_one<true><<<n4 / 128, 128>>>(b, 0.1f); });
  run("full-like 512x256 U2", 28.0 * d, [&](Bufs b) { k_multi<true, 2><<<n4 / 512, 256>>>(b, 0.1f, n4); });
  run("full-like 1024x128 U2", 28.0 * d, [&](Bufs b) { k_multi<true, 2><<<n4 / 256, 128>>>(b, 0.1f, n4); });
  run("full-like 256x256 U4", 28.0 * d, [&](Bufs b) { k_multi<true, 4><<<n4 / 1024, 256>>>(b, 0.1f, n4); });
  return 0;
}
