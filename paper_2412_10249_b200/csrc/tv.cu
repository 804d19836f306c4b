// TV + nonnegativity prox on the device: the fast
// gradient projection on the gradient-field dual variable of
// prox_tv_nonneg (reference proxlib.py:102-148), restated:
//   primal = max(xp - G^T m, 0)
//   q'     = P_w(m + G primal / 8)          (per-pixel projection onto the radius-w ball)
//   m'     = q' + ((t-1)/t') (q' - q),     t' = (1 + sqrt(1 + 4 t^2)) / 2
// until ||q' - q|| / max(1, ||q'||) < tol or inner_iters, then
//   out = max(xp - G^T q, 0).
// G is the forward-difference gradient with a zero last row / column
// (proxlib.py:66-93); G^T is minus its divergence.
//
// One launch per iteration: a 32 x 32 tile stages the momentum field with a
// one-pixel halo and xp, evaluates the primal on the tile plus its bottom and
// right neighbours, and updates q (in place, each pixel reads only its own
// old q) and the next momentum (ping-pong: neighbours read the old one). The
// progress norms are reduced in float64 in a fixed order by the last block
// to finish, which raises a device flag that turns the remaining launches
// into no-ops, so the whole prox is stream-ordered with no host round trip.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "imask_b200.h"

namespace imask {
namespace {

constexpr int kTvT = 32;
constexpr int kTvThreads = 256;

struct TvScratch {
  float *q, *mom0, *mom1;  // 2 planes each (row differences, column differences)
  double* part;            // 2 per block
  unsigned* counter;
  int* done;
};

__device__ __forceinline__ double tv_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  v = threadIdx.x < kTvThreads / 32 ? red[threadIdx.x] : 0.0;
  if (threadIdx.x < 32) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

// G^T m at (r, c) from a staged field (row-difference plane mr, column plane mc)
__device__ __forceinline__ float gt_at(const float (*mr)[kTvT + 2], const float (*mc)[kTvT + 2],
                                       int i, int j, int r, int c, int n) {
  // i, j: staged indices of (r, c); the tile stages rows r0-1.. and cols c0-1..
  float v = 0.f;
  if (r < n - 1) v -= mr[i][j];
  if (r >= 1) v += mr[i - 1][j];
  if (c < n - 1) v -= mc[i][j];
  if (c >= 1) v += mc[i][j - 1];
  return v;
}

__global__ void __launch_bounds__(kTvThreads)
k_tv_iter(const float* __restrict__ xp, int n, float w, float step, float coef, double tol,
          TvScratch sc, const float* __restrict__ mom_in, float* __restrict__ mom_out) {
  if (*(volatile int*)sc.done) return;
  __shared__ float mr[kTvT + 2][kTvT + 2], mc[kTvT + 2][kTvT + 2];  // rows r0-1 .. r0+32
  __shared__ float pr[kTvT + 1][kTvT + 1];                        // primal, rows r0 .. r0+32
  __shared__ double red[kTvThreads / 32];
  __shared__ bool last;
  const size_t d = (size_t)n * n;
  const int r0 = blockIdx.y * kTvT, c0 = blockIdx.x * kTvT;
  for (int e = threadIdx.x; e < (kTvT + 2) * (kTvT + 2); e += kTvThreads) {
    const int i = e / (kTvT + 2), j = e % (kTvT + 2);
    const int r = r0 - 1 + i, c = c0 - 1 + j;
    const bool in = r >= 0 && r < n && c >= 0 && c < n;
    mr[i][j] = in ? mom_in[(size_t)r * n + c] : 0.f;
    mc[i][j] = in ? mom_in[d + (size_t)r * n + c] : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < (kTvT + 1) * (kTvT + 1); e += kTvThreads) {
    const int i = e / (kTvT + 1), j = e % (kTvT + 1);
    const int r = r0 + i, c = c0 + j;
    float p = 0.f;
    if (r < n && c < n) p = fmaxf(__ldg(xp + (size_t)r * n + c) - gt_at(mr, mc, i + 1, j + 1, r, c, n), 0.f);
    pr[i][j] = p;
  }
  __syncthreads();
  double dq2 = 0.0, q2 = 0.0;
  for (int e = threadIdx.x; e < kTvT * kTvT; e += kTvThreads) {
    const int i = e / kTvT, j = e % kTvT;
    const int r = r0 + i, c = c0 + j;
    if (r >= n || c >= n) continue;
    const size_t p = (size_t)r * n + c;
    const float gr = r < n - 1 ? pr[i + 1][j] - pr[i][j] : 0.f;
    const float gc = c < n - 1 ? pr[i][j + 1] - pr[i][j] : 0.f;
    float qr = fmaf(step, gr, mr[i + 1][j + 1]);
    float qc = fmaf(step, gc, mc[i + 1][j + 1]);
    const float nrm = hypotf(qr, qc);
    const float shrink = w / fmaxf(nrm, w);
    qr *= shrink;
    qc *= shrink;
    const float qor = sc.q[p], qoc = sc.q[d + p];
    mom_out[p] = fmaf(coef, qr - qor, qr);
    mom_out[d + p] = fmaf(coef, qc - qoc, qc);
    sc.q[p] = qr;
    sc.q[d + p] = qc;
    const double er = (double)qr - qor, ec = (double)qc - qoc;
    dq2 += er * er + ec * ec;
    q2 += (double)qr * qr + (double)qc * qc;
  }
  dq2 = tv_block_sum(dq2, red);
  q2 = tv_block_sum(q2, red);
  const int nblocks = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    sc.part[2 * bid] = dq2;
    sc.part[2 * bid + 1] = q2;
    __threadfence();
    last = atomicAdd(sc.counter, 1u) == (unsigned)nblocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += kTvThreads) {
    a += ((volatile double*)sc.part)[2 * i];
    b += ((volatile double*)sc.part)[2 * i + 1];
  }
  a = tv_block_sum(a, red);
  b = tv_block_sum(b, red);
  if (threadIdx.x == 0) {
    *sc.counter = 0u;
    const double progress = sqrt(a) / fmax(1.0, sqrt(b));
    if (progress < tol) *sc.done = 1;
  }
}

__global__ void __launch_bounds__(kTvThreads)
k_tv_final(const float* xp, int n, const float* __restrict__ q, float* out) {
  const size_t d = (size_t)n * n;
  const size_t p = (size_t)blockIdx.x * kTvThreads + threadIdx.x;
  if (p >= d) return;
  const int r = (int)(p / n), c = (int)(p % n);
  float g = 0.f;
  if (r < n - 1) g -= q[p];
  if (r >= 1) g += q[p - n];
  if (c < n - 1) g -= q[d + p];
  if (c >= 1) g += q[d + p - 1];
  out[p] = fmaxf(xp[p] - g, 0.f);
}

size_t tv_blocks(int n) { return (size_t)((n + kTvT - 1) / kTvT) * ((n + kTvT - 1) / kTvT); }

}  // namespace
}  // namespace imask

using namespace imask;

extern "C" IMASK_API int64_t imask_prox_tv_scratch_bytes(int side) {
  if (side < 1) return 0;
  const size_t d = (size_t)side * side;
  return (int64_t)(6 * d * sizeof(float) + 2 * tv_blocks(side) * sizeof(double) + 16);
}

extern "C" IMASK_API int imask_prox_tv_nonneg(int side, const float* xp, float* out, double sigma,
                                              double mu_g, int inner_iters, double inner_tol,
                                              void* scratch, void* stream) {
  if (side < 1 || !xp || !out || !scratch) return IMASK_EINVAL;
  if (!(sigma > 0.0) || !(mu_g > 0.0) || inner_iters < 0) return IMASK_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t d = (size_t)side * side;
  const size_t nb = tv_blocks(side);
  TvScratch sc;
  float* f = reinterpret_cast<float*>(scratch);
  sc.q = f;
  sc.mom0 = f + 2 * d;
  sc.mom1 = f + 4 * d;
  sc.part = reinterpret_cast<double*>(f + 6 * d);
  sc.counter = reinterpret_cast<unsigned*>(sc.part + 2 * nb);
  sc.done = reinterpret_cast<int*>(sc.counter + 1);
  // q = m = 0, counters re-armed, not done
  if (cudaMemsetAsync(scratch, 0, imask_prox_tv_scratch_bytes(side), s) != cudaSuccess)
    return IMASK_ECUDA;
  const float w = (float)(sigma * mu_g), step = 1.0f / 8.0f;  // GRAD_NORM_SQ (proxlib.py:12)
  dim3 grid((side + kTvT - 1) / kTvT, (side + kTvT - 1) / kTvT);
  double t = 1.0;
  for (int k = 0; k < inner_iters; ++k) {
    const double t_new = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    const float coef = (float)((t - 1.0) / t_new);
    const float* min = (k & 1) ? sc.mom1 : sc.mom0;
    float* mout = (k & 1) ? sc.mom0 : sc.mom1;
    k_tv_iter<<<grid, kTvThreads, 0, s>>>(xp, side, w, step, coef, inner_tol, sc, min, mout);
    t = t_new;
  }
  k_tv_final<<<(unsigned)((d + kTvThreads - 1) / kTvThreads), kTvThreads, 0, s>>>(xp, side, sc.q,
                                                                                  out);
  return cudaGetLastError() == cudaSuccess ? IMASK_OK : IMASK_ECUDA;
}
