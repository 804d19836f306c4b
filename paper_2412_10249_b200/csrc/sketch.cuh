// Tile-local compensation helpers shared by the compensate and SAGA kernels.
#pragma once
#include "imask_common.cuh"

namespace imask {

constexpr int kMaxLevels = 12;

struct CompParams {
  int r;
  float p[kMaxLevels];  // p[i-1] = probability of level i
  float pr;             // p_r
};

struct ResumParams {
  int r;
  float p[kMaxLevels];
  int factor[kMaxLevels];
  long long offset[kMaxLevels];  // phi table row offsets
};

// Levels 1..r-1 of the 2x2-mean pyramid of the ts x ts tile, packed one
// after another in `pyr` (level j has side ts >> j). Block-wide; ends synced.
__device__ __forceinline__ void build_pyramid(const float* tile, float* pyr, int ts, int r) {
  const float* src = tile;
  float* dst = pyr;
  int sn = ts;
  for (int lev = 1; lev < r; ++lev) {
    const int dn = sn >> 1;
    for (int e = threadIdx.x; e < dn * dn; e += blockDim.x) {
      const int rr = e / dn, cc = e % dn;
      const float* s0 = src + (2 * rr) * sn + 2 * cc;
      dst[e] = ((s0[0] + s0[1]) + (s0[sn] + s0[sn + 1])) * 0.25f;
    }
    __syncthreads();
    src = dst;
    dst += dn * dn;
    sn = dn;
  }
}

// (v - acc)/p_r with acc = sum over levels i = 1..r-1 (coarsest first) of
// p_i * (level r-i pyramid value of pixel (py, px))  (mrsketch.py:141-153).
__device__ __forceinline__ float compensated(float v, const float* pyr, int ts,
                                             const CompParams& cp, int py, int px) {
  if (cp.r == 1) return v;  // S_1 = I (mrsketch.py:137-138)
  // offsets of pyramid levels: level j starts after levels 1..j-1
  float acc = 0.f;
  for (int i = 1; i < cp.r; ++i) {
    const int j = cp.r - i;
    int off = 0;
    for (int l = 1; l < j; ++l) off += (ts >> l) * (ts >> l);
    const int sj = ts >> j;
    const float term = cp.p[i - 1] * pyr[off + (py >> j) * sj + (px >> j)];
    acc = (i == 1) ? term : acc + term;
  }
  return (v - acc) / cp.pr;
}

}  // namespace imask
