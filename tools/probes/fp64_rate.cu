// FP64 vs FP32 FMA throughput probe (independent chains, all SMs).
#include <cstdio>
template <typename T>
__global__ void k(T* out, T a, T b, int iters) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <typename T>
void run(const char* name) {
  T* o; cudaMalloc(&o, sizeof(T) * 148 * 8 * 256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  k<T><<<148 * 8, 256>>>(o, (T)0.999, (T)0.001, 10);
  cudaEventRecord(e0);
  k<T><<<148 * 8, 256>>>(o, (T)0.999, (T)0.001, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fmas = 148.0 * 8 * 256 * iters * 64;
  printf("%s: %.3f ms  %.2f TFMA/s  (%.1f per clk per SM at 1.965 GHz)\n", name, ms, fmas / ms / 1e9, fmas / (ms * 1e-3) / 148 / 1.965e9);
}
int main() { run<float>("fp32"); run<double>("fp64"); return 0; }
