// Kernels (3) and (4): the multiresolution sketch family and the fused SAGA
// updates.
//   restrict   : T_f block mean                 (mrsketch.py:23-32)
//   prolong    : alpha * U_f replication        (mrsketch.py:35-41, 54-55)
//   compensate : S_r = (I - sum_{i<r} p_i S_i)/p_r by a tile-local pyramid
//                (mrsketch.py:133-153); block means are aligned to the
//                2^(r-1) grid, so every 2^(r-1)-tile is independent.
//   prepare    : coarse image -> the forward projector's pair layouts
//                P[row][c+1] = (u[row][c], u[row][c+1]-u[row][c]), c = -1..n-1,
//                and the same on the transpose, zero outside the image.
//   saga_image : image side of sketch_step (solvers.py:204-214): new adjoint
//                product (prolonged /f^2 or compensated), table row, phi_sum,
//                primal ridge prox (proxlib.py:51-55), one pass over HBM.
//   resum      : _resum (solvers.py:184-191).
#include "imask_common.cuh"
#include "sketch.cuh"

namespace imask {

// ---- restriction / prolongation -------------------------------------------

// thread per coarse pixel (small factors)
__global__ void k_restrict_small(const float* __restrict__ x, float* __restrict__ u, int side,
                                 int f) {
  const int n = side / f;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  const int R = idx / n, C = idx % n;
  const float* base = x + (size_t)R * f * side + (size_t)C * f;
  float s = 0.f;
  for (int i = 0; i < f; ++i) {
    float rs = 0.f;
    for (int j = 0; j < f; ++j) rs += __ldg(base + (size_t)i * side + j);
    s += rs;
  }
  u[idx] = s * (1.0f / (float)(f * f));
}

// warp per coarse pixel (factors >= 16)
__global__ void k_restrict_warp(const float* __restrict__ x, float* __restrict__ u, int side,
                                int f) {
  const int n = side / f;
  const int w = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= n * n) return;
  const int R = w / n, C = w % n;
  const float* base = x + (size_t)R * f * side + (size_t)C * f;
  float s = 0.f;
  for (int e = lane; e < f * f; e += 32) s += __ldg(base + (size_t)(e / f) * side + (e % f));
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) u[w] = s * (1.0f / (float)(f * f));
}

__global__ void k_prolong(const float* __restrict__ u, float* __restrict__ x, int side, int f,
                          float alpha) {
  const int n = side / f;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)side * side) return;
  const int row = (int)(idx / side), col = (int)(idx % side);
  x[idx] = alpha * __ldg(u + (size_t)(row / f) * n + col / f);
}

// ---- compensation -----------------------------------------------------------

template <int TT>
__global__ void __launch_bounds__(256)
k_compensate(const float* __restrict__ x, float* __restrict__ out, int side, CompParams cp) {
  __shared__ float tile[TT * TT];
  __shared__ float pyr[TT * TT / 3 + 8];
  const int ts = side / (int)gridDim.x;  // the launcher's tile (cover_tile): divides side, <= TT
  const int x0 = blockIdx.x * ts, y0 = blockIdx.y * ts;
  IMASK_CHECK_RANGE(50, (long long)(gridDim.x * ts) - side, 1);  // the tiles cover the image exactly
  IMASK_CHECK_RANGE(51, ts, TT + 1);
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x) {
    IMASK_CHECK_RANGE(52, (size_t)(y0 + e / ts) * side + x0 + e % ts, (long long)side * side);
    tile[e] = __ldg(x + (size_t)(y0 + e / ts) * side + x0 + e % ts);
  }
  __syncthreads();
  build_pyramid(tile, pyr, ts, cp.r);
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x) {
    const int py = e / ts, px = e % ts;
    out[(size_t)(y0 + py) * side + x0 + px] = compensated(tile[e], pyr, ts, cp, py, px);
  }
}

// Fast path (side % 32 == 0, r <= 6): a 32 x 32 tile held as one float4 per
// thread (256 threads; thread t holds row py = t >> 3, pixels px = 4 (t & 7) ..
// px + 3). The block-mean pyramid is built in registers: level 1 (2 x 2 means)
// and level 2 (4 x 4) by warp shuffles (a warp holds four pixel rows), levels
// 3..5 by warp 0 from the 8 x 8 level-2 values, with the additions of
// build_pyramid in the same order, ((s00 + s01) + (s10 + s11)) * 0.25. The
// compensation's accumulation keeps the reference's order too (coarsest level
// first, mrsketch.py:141-153): warp 0 folds levels r-1..3 per level-3 node,
// then every thread adds the level-2 and level-1 terms of its pixels.
struct Pyr32Smem {
  float l2[64];  // level-2 values (8 x 8)
  float a3[16];  // per level-3 node: the accumulated terms of levels r-1..3
};

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void pyr32_low(const float4 v, float& l1a, float& l1b, float& l2) {
  const float h0 = v.x + v.y, h1 = v.z + v.w;  // horizontal pair sums of this row
  const float o0 = __shfl_xor_sync(kFull, h0, 8), o1 = __shfl_xor_sync(kFull, h1, 8);  // row py ^ 1
  const bool odd = (threadIdx.x >> 3) & 1;
  l1a = (odd ? (o0 + h0) : (h0 + o0)) * 0.25f;  // level-1 node (py >> 1, 2 (t & 7))
  l1b = (odd ? (o1 + h1) : (h1 + o1)) * 0.25f;  // level-1 node (py >> 1, 2 (t & 7) + 1)
  const float t = l1a + l1b;
  const float ot = __shfl_xor_sync(kFull, t, 16);  // level-1 row (py >> 1) ^ 1
  const bool bot = (threadIdx.x >> 4) & 1;
  l2 = (bot ? (ot + t) : (t + ot)) * 0.25f;  // level-2 node (py >> 2, t & 7)
}

// Warp 0 (after the level-2 values are in sm.l2): levels 3, 4 and 5. Lane l < 16
// holds the level-3 node (l >> 2, l & 3); L4a / L5 are that node's ancestors;
// lanes 0..3 also hold the level-4 node (l >> 1, l & 1) in L4.
__device__ __forceinline__ void pyr32_high(const Pyr32Smem& sm, float& L3, float& L4, float& L4a,
                                           float& L5) {
  const int l = threadIdx.x & 31;
  const int R = (l >> 2) & 3, C = l & 3;
  const float* q = sm.l2 + (2 * R) * 8 + 2 * C;
  L3 = ((q[0] + q[1]) + (q[8] + q[9])) * 0.25f;
  const int b4 = ((l >> 1) & 1) * 8 + (l & 1) * 2;
  const float a = __shfl_sync(kFull, L3, b4), b = __shfl_sync(kFull, L3, b4 + 1),
              c = __shfl_sync(kFull, L3, b4 + 4), d = __shfl_sync(kFull, L3, b4 + 5);
  L4 = ((a + b) + (c + d)) * 0.25f;
  const float e0 = __shfl_sync(kFull, L4, 0), e1 = __shfl_sync(kFull, L4, 1),
              e2 = __shfl_sync(kFull, L4, 2), e3 = __shfl_sync(kFull, L4, 3);
  L5 = ((e0 + e1) + (e2 + e3)) * 0.25f;
  L4a = __shfl_sync(kFull, L4, (R >> 1) * 2 + (C >> 1));
}

// S_r of the thread's four pixels (block-wide: every thread of the CTA calls it).
__device__ __forceinline__ float4 comp32(const float4 v, const CompParams& cp, Pyr32Smem& sm) {
  const int r = cp.r;
  if (r == 1) return v;  // S_1 = I (mrsketch.py:137-138)
  float l1a, l1b, l2;
  pyr32_low(v, l1a, l1b, l2);
  float acc = 0.f;
  if (r >= 4) {
    const int py = threadIdx.x >> 3;
    if ((py & 3) == 0) sm.l2[(py >> 2) * 8 + (threadIdx.x & 7)] = l2;
    __syncthreads();
    if (threadIdx.x < 32) {
      float L3, L4, L4a, L5;
      pyr32_high(sm, L3, L4, L4a, L5);
      float A = 0.f;
      if (r >= 6) A = A + cp.p[r - 6] * L5;
      if (r >= 5) A = A + cp.p[r - 5] * L4a;
      A = A + cp.p[r - 4] * L3;
      if (threadIdx.x < 16) sm.a3[threadIdx.x] = A;
    }
    __syncthreads();
    acc = sm.a3[(py >> 3) * 4 + ((threadIdx.x & 7) >> 1)];
  }
  if (r >= 3) acc = acc + cp.p[r - 3] * l2;
  const float pl = cp.p[r - 2];  // level-1 term (factor 2), last in the telescoping order
  const float a0 = acc + pl * l1a, a1 = acc + pl * l1b;
  return make_float4((v.x - a0) / cp.pr, (v.y - a0) / cp.pr, (v.z - a1) / cp.pr,
                     (v.w - a1) / cp.pr);
}

__global__ void __launch_bounds__(256)
k_compensate32(const float* __restrict__ x, float* __restrict__ out, int side, CompParams cp) {
  __shared__ __align__(16) Pyr32Smem sm;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, px = (threadIdx.x & 7) * 4;
  const size_t g = (size_t)(y0 + py) * side + x0 + px;
  const float4 v = __ldg(reinterpret_cast<const float4*>(x + g));
  *reinterpret_cast<float4*>(out + g) = comp32(v, cp, sm);
}

// Restriction by a power-of-two factor f = 2^lg <= 32 (side % 32 == 0): each
// CTA loads a 32 x 32 tile of x with 128-bit loads, builds the block-mean
// pyramid up to level lg and writes the tile's (32/f)^2 coarse pixels.
__global__ void __launch_bounds__(256)
k_restrict32(const float* __restrict__ x, float* __restrict__ u, int side, int lg) {
  __shared__ __align__(16) Pyr32Smem sm;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, c8 = threadIdx.x & 7;
  const float4 v =
      __ldg(reinterpret_cast<const float4*>(x + (size_t)(y0 + py) * side + x0 + c8 * 4));
  float l1a, l1b, l2;
  pyr32_low(v, l1a, l1b, l2);
  const int n = side >> lg;
  if (lg == 1) {
    if ((py & 1) == 0)
      *reinterpret_cast<float2*>(u + (size_t)((y0 >> 1) + (py >> 1)) * n + (x0 >> 1) + 2 * c8) =
          make_float2(l1a, l1b);
    return;
  }
  if (lg == 2) {
    if ((py & 3) == 0) u[(size_t)((y0 >> 2) + (py >> 2)) * n + (x0 >> 2) + c8] = l2;
    return;
  }
  if ((py & 3) == 0) sm.l2[(py >> 2) * 8 + c8] = l2;
  __syncthreads();
  if (threadIdx.x < 32) {
    float L3, L4, L4a, L5;
    pyr32_high(sm, L3, L4, L4a, L5);
    const int l = threadIdx.x;
    if (lg == 3 && l < 16)
      u[(size_t)((y0 >> 3) + (l >> 2)) * n + (x0 >> 3) + (l & 3)] = L3;
    else if (lg == 4 && l < 4)
      u[(size_t)((y0 >> 4) + (l >> 1)) * n + (x0 >> 4) + (l & 1)] = L4;
    else if (lg == 5 && l == 0)
      u[(size_t)(y0 >> 5) * n + (x0 >> 5)] = L5;
  }
}

// The adjoint's split planes summed for four consecutive pixels, planes in
// order (k_adjoint_reduce's order; used where the planes are many pixels).
__device__ __forceinline__ float4 planes_sum4(const ImageSaga& sg, size_t g) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* p = sg.planes + g;
  for (int s = 0; s < sg.n_planes; ++s, p += sg.plane_len) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(p));
    v.x += w.x;
    v.y += w.y;
    v.z += w.z;
    v.w += w.w;
  }
  return v;
}

__device__ __forceinline__ float saga_px(float pn, float& tab, float& sum, float& xv,
                                         const ImageSaga& sg) {
  const float d = pn - tab;
  const float xi = d + sum;
  sum = fmaf(sg.p_i, d, sum);
  tab = pn;
  xv = fmaf(-sg.s, xi, xv) * sg.inv_den;
  return d;
}

// Full level, fast path: phi_new = S_r(bp) by the 32x32 tile pyramid, then the
// SAGA image update, all with 128-bit accesses.
__global__ void __launch_bounds__(256, 6)  // 40 registers: 888 of the 1024 CTAs of a 1024^2 image resident
k_saga_image_full32(const float* __restrict__ bp, int side, CompParams cp, ImageSaga sg) {
  __shared__ __align__(16) Pyr32Smem sm;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, px = (threadIdx.x & 7) * 4;
  const size_t g = (size_t)(y0 + py) * side + x0 + px;
  // the table row, the sum and x were last written by the previous step, which
  // completed before this step's adjoint (a plain launch) started: they are
  // loaded before the programmatic wait, overlapping the adjoint's tail
  IMASK_CHECK_RANGE(64, (long long)(((uintptr_t)(sg.phi_tab + g) | (uintptr_t)(sg.phi_sum + g) |
                                      (uintptr_t)(sg.x + g)) & 15), 1);  // 128-bit accesses aligned
  float4 tab = *reinterpret_cast<const float4*>(sg.phi_tab + g);
  float4 sum = *reinterpret_cast<const float4*>(sg.phi_sum + g);
  float4 xv = *reinterpret_cast<const float4*>(sg.x + g);
  griddep_wait();  // bp (or the split planes) come from the stream predecessor (the adjoint)
  // planes summed in order (step_image fuses the reduction here only when the
  // reduce kernels would use that order too)
  const float4 v = sg.n_planes > 0 ? planes_sum4(sg, g)
                                   : __ldg(reinterpret_cast<const float4*>(bp + g));
  const float4 xo = xv;
  const float4 pn = comp32(v, cp, sm);
  saga_px(pn.x, tab.x, sum.x, xv.x, sg);
  saga_px(pn.y, tab.y, sum.y, xv.y, sg);
  saga_px(pn.z, tab.z, sum.z, xv.z, sg);
  saga_px(pn.w, tab.w, sum.w, xv.w, sg);
  *reinterpret_cast<float4*>(sg.phi_tab + g) = tab;
  *reinterpret_cast<float4*>(sg.phi_sum + g) = sum;
  *reinterpret_cast<float4*>(sg.x + g) = xv;
  extrapolate4(sg, g, xo, xv);
}

// Coarse level, fast path (side % 32 == 0, f <= 32): 32 x 32 full-resolution
// tile, four contiguous pixels per thread, 128-bit accesses to x / phi_sum.
__global__ void __launch_bounds__(256)
k_saga_image_coarse32(const float* __restrict__ bp, int side, int lg, float inv_f2, ImageSaga sg) {
  __shared__ float cv[256];  // the tile's (32/f)^2 coarse backprojection values (planes mode)
  const int n = side >> lg;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int lt = 5 - lg, tc = 1 << lt;  // coarse pixels per tile side
  const int py = threadIdx.x >> 3, px = (threadIdx.x & 7) * 4;
  const int row = y0 + py, col = x0 + px;
  const size_t g = (size_t)row * side + col;
  const int qrow = (row >> lg) * n;
  // state written by the previous step (complete before this step's adjoint, a
  // plain launch, started): loaded before the programmatic wait
  float4 sum = *reinterpret_cast<const float4*>(sg.phi_sum + g);
  float4 xv = *reinterpret_cast<const float4*>(sg.x + g);
  float po[4];
  IMASK_CHECK_RANGE(65, (long long)(((uintptr_t)(sg.phi_sum + g) | (uintptr_t)(sg.x + g)) & 15), 1);
  IMASK_CHECK_RANGE(66, qrow + ((col + 3) >> lg), (long long)n * n);
#pragma unroll
  for (int k = 0; k < 4; ++k) po[k] = sg.phi_tab[qrow + ((col + k) >> lg)];
  griddep_wait();  // bp (or the split planes) come from the stream predecessor (the adjoint)
  if (sg.n_planes > 0) {
    // sum the adjoint's split planes for this tile's coarse pixels in the order of
    // k_adjoint_reduce_warp (many planes, few pixels) or k_adjoint_reduce
    const int P = sg.n_planes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (P >= 32 && n * n <= 65536) {
      for (int c = warp; c < tc * tc; c += 8) {
        const int q = ((y0 >> lg) + (c >> lt)) * n + (x0 >> lg) + (c & (tc - 1));
        float v = 0.f;
        for (int s = lane; s < P; s += 32) v += __ldg(sg.planes + (size_t)s * sg.plane_len + q);
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) cv[c] = v;
      }
    } else {
      for (int c = threadIdx.x; c < tc * tc; c += blockDim.x) {
        const int q = ((y0 >> lg) + (c >> lt)) * n + (x0 >> lg) + (c & (tc - 1));
        float v = 0.f;
        for (int s = 0; s < P; ++s) v += __ldg(sg.planes + (size_t)s * sg.plane_len + q);
        cv[c] = v;
      }
    }
    __syncthreads();
  }
  const float4 xo = xv;
  float pn[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = qrow + ((col + k) >> lg);
    const float b = sg.n_planes > 0
                        ? cv[(((row >> lg) - (y0 >> lg)) << lt) + ((col + k) >> lg) - (x0 >> lg)]
                        : __ldg(bp + q);
    pn[k] = b * inv_f2;
  }
  float d;
  d = pn[0] - po[0]; { const float xi = d + sum.x; sum.x = fmaf(sg.p_i, d, sum.x); xv.x = fmaf(-sg.s, xi, xv.x) * sg.inv_den; }
  d = pn[1] - po[1]; { const float xi = d + sum.y; sum.y = fmaf(sg.p_i, d, sum.y); xv.y = fmaf(-sg.s, xi, xv.y) * sg.inv_den; }
  d = pn[2] - po[2]; { const float xi = d + sum.z; sum.z = fmaf(sg.p_i, d, sum.z); xv.z = fmaf(-sg.s, xi, xv.z) * sg.inv_den; }
  d = pn[3] - po[3]; { const float xi = d + sum.w; sum.w = fmaf(sg.p_i, d, sum.w); xv.w = fmaf(-sg.s, xi, xv.w) * sg.inv_den; }
  *reinterpret_cast<float4*>(sg.phi_sum + g) = sum;
  *reinterpret_cast<float4*>(sg.x + g) = xv;
  extrapolate4(sg, g, xo, xv);
  __syncthreads();  // every old table value of this tile's blocks has been read
  if ((int)threadIdx.x < tc * tc) {
    const int q = ((y0 >> lg) + (threadIdx.x >> lt)) * n + (x0 >> lg) + (threadIdx.x & (tc - 1));
    sg.phi_tab[q] = (sg.n_planes > 0 ? cv[threadIdx.x] : __ldg(bp + q)) * inv_f2;
  }
}

// ---- projector staging ------------------------------------------------------

// Pair layouts of the n x n image u for the forward projector, rows padded by
// kPadC zero columns on each side (imask_common.cuh):
//   P  [R][c + 1 + kPadC] = (u[R][c], u[R][c+1] - u[R][c])          c in [-1-kPadC, n-1+kPadC]
//   PT [C][r + 1 + kPadC] = (u[r][C], u[r+1][C] - u[r][C])          r in [-1-kPadC, n-1+kPadC]
// For the mirror-symmetric forward (PM != nullptr) the pairs of u and of the
// left-right mirrored image um[R][c] = u[R][n-1-c] (whose transposed layout is
// PT with its bands reversed) are regrouped as value and difference planes,
// so one 8-byte read feeds a ray and its mirror with packed FP32 adds:
//   P  [R][i] = (P_u[R][i].x,  P_um[R][i].x)    PM [R][i] = (P_u[R][i].y,  P_um[R][i].y)
//   PT [C][i] = (PT[C][i].x, PT[n-1-C][i].x)    PTM[C][i] = (PT[C][i].y, PT[n-1-C][i].y)
// with u = 0 outside the image. The grid tiles the padded index range in both
// dimensions; each 32x32 tile (plus a one-element halo on each side) is staged
// in shared memory so the row-major and the transposed writes are coalesced.
__global__ void __launch_bounds__(256)
k_prepare(const float* __restrict__ u, int n, float2* __restrict__ P, float2* __restrict__ PT,
          float2* __restrict__ PM, float2* __restrict__ PTM, bool diff) {
  // t[rr][cc] = u[r0 + rr][c0 - 1 + cc]; for the symmetric layout also the tile
  // of the mirrored image um[R][C] = u[R][n-1-C] at the same coordinates, so
  // every output is one coalesced float2 (a value of u, the same of um)
  __shared__ float t[33][35];
  __shared__ float tm[33][35];
  griddep_wait();  // u comes from the stream predecessor (restriction / compensation)
  const bool sym = PM != nullptr;
  const int pitch = pair_pitch(n);
  const int r0 = blockIdx.y * 32 - 1 - kPadC, c0 = blockIdx.x * 32 - 1 - kPadC;
  for (int e = threadIdx.x; e < 33 * 34; e += blockDim.x) {
    const int rr = e / 34, cc = e % 34;
    const int R = r0 + rr, C = c0 - 1 + cc;
    const bool in = R >= 0 && R < n && C >= 0 && C < n;
    t[rr][cc] = in ? __ldg(u + (size_t)R * n + C) : 0.f;
    if (sym) tm[rr][cc] = in ? __ldg(u + (size_t)R * n + (n - 1 - C)) : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int rr = e / 32, cc = e % 32;
    // row-major pairs: real rows, padded column index
    {
      const int R = r0 + rr, C = c0 + cc, idx = C + 1 + kPadC;
      if (R >= 0 && R < n && idx < pitch) {
        const float v = t[rr][cc + 1], dv = t[rr][cc + 2] - v;
        const size_t o = (size_t)R * pitch + idx;
        if (!sym) {
          P[o] = make_float2(v, dv);
        } else {
          // value planes (u, um) in P, difference planes (d, dm) in PM (only
          // when the forward reads them; the value-plane kernels subtract)
          const float vm = tm[rr][cc + 1];
          P[o] = make_float2(v, vm);
          if (diff) PM[o] = make_float2(dv, tm[rr][cc + 2] - vm);
        }
      }
    }
    // transposed pairs: real columns, padded row index (consecutive threads walk rows of u)
    {
      const int C = c0 + rr, idx = r0 + cc + 1 + kPadC;
      if (C >= 0 && C < n && idx < pitch) {
        const float v = t[cc][rr + 1], dv = t[cc + 1][rr + 1] - v;
        const size_t o = (size_t)C * pitch + idx;
        if (!sym) {
          PT[o] = make_float2(v, dv);
        } else {
          // band C of the transposed image and of the transposed mirror image
          // (= band n-1-C of the transposed image)
          const float vm = tm[cc][rr + 1];
          PT[o] = make_float2(v, vm);
          if (diff) PTM[o] = make_float2(dv, tm[cc + 1][rr + 1] - vm);
        }
      }
    }
  }
}

// Fused staging for the value-plane forwards (the mirror-symmetric plans of
// the whole angle set): x goes to the value planes P, PT of level f = 2^lg
// in one kernel. Each CTA loads a 32 x 32 tile of x (128-bit loads), forms its
// (32/f)^2 values of u = T_f x (the restriction pyramid of k_restrict32) or,
// at the full level, u = S_r x (comp32 of k_compensate32) -- the same float
// operations, so P and PT are bit-identical to restriction / compensation +
// k_prepare -- and writes each value twice per plane: P[R][c].x = u[R][c] and
// P[R][n-1-c].y = u[R][c] (the mirror pairing), likewise along the transpose.
// Tiles on the image edge write the rows' zero padding; every entry of the
// n x pitch planes is written, so the planes need no clearing between levels.
__global__ void __launch_bounds__(256)
k_stage32(const float* __restrict__ x, int side, int lg, CompParams cp, float2* __restrict__ P,
          float2* __restrict__ PT) {
  __shared__ __align__(16) Pyr32Smem sm;
  __shared__ float ut[32][33];  // the tile's u values, w x w (w = 32 >> lg)
  const int n = side >> lg, w = 32 >> lg;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, c8 = threadIdx.x & 7;
  const float4 v =
      __ldg(reinterpret_cast<const float4*>(x + (size_t)(y0 + py) * side + x0 + c8 * 4));
  if (lg == 0) {
    const float4 o = comp32(v, cp, sm);
    ut[py][4 * c8] = o.x;
    ut[py][4 * c8 + 1] = o.y;
    ut[py][4 * c8 + 2] = o.z;
    ut[py][4 * c8 + 3] = o.w;
  } else {
    float l1a, l1b, l2;
    pyr32_low(v, l1a, l1b, l2);
    if (lg == 1) {
      if ((py & 1) == 0) {
        ut[py >> 1][2 * c8] = l1a;
        ut[py >> 1][2 * c8 + 1] = l1b;
      }
    } else if (lg == 2) {
      if ((py & 3) == 0) ut[py >> 2][c8] = l2;
    } else {
      if ((py & 3) == 0) sm.l2[(py >> 2) * 8 + c8] = l2;
      __syncthreads();
      if (threadIdx.x < 32) {
        float L3, L4, L4a, L5;
        pyr32_high(sm, L3, L4, L4a, L5);
        const int l = threadIdx.x;
        if (lg == 3 && l < 16) ut[l >> 2][l & 3] = L3;
        if (lg == 4 && l < 4) ut[l >> 1][l & 1] = L4;
        if (lg == 5 && l == 0) ut[0][0] = L5;
      }
    }
  }
  __syncthreads();
  // the planes may still be read by the previous level's forward (the stream
  // predecessor): write them only once it is done
  griddep_wait();
  const int R0 = y0 >> lg, C0 = x0 >> lg;
  const size_t pitch = (size_t)pair_pitch(n);
  float* Pf = reinterpret_cast<float*>(P);
  float* PTf = reinterpret_cast<float*>(PT);
  const int nw = w * w;
  for (int e = threadIdx.x; e < nw; e += blockDim.x) {
    const int rr = e / w, cc = e % w;  // consecutive threads along a row of u
    const int R = R0 + rr, C = C0 + cc;
    const float val = ut[rr][cc];
    IMASK_CHECK_RANGE(60, R * pitch + C + 1 + kPadC, (long long)n * pitch);
    IMASK_CHECK_RANGE(61, R * pitch + (n - 1 - C) + 1 + kPadC, (long long)n * pitch);
    Pf[2 * (R * pitch + C + 1 + kPadC)] = val;
    Pf[2 * (R * pitch + (n - 1 - C) + 1 + kPadC) + 1] = val;
  }
  for (int e = threadIdx.x; e < nw; e += blockDim.x) {
    const int cc = e / w, rr = e % w;  // consecutive threads along a column of u
    const int R = R0 + rr, C = C0 + cc;
    const float val = ut[rr][cc];
    IMASK_CHECK_RANGE(62, C * pitch + R + 1 + kPadC, (long long)n * pitch);
    IMASK_CHECK_RANGE(63, (n - 1 - C) * pitch + R + 1 + kPadC, (long long)n * pitch);
    PTf[2 * (C * pitch + R + 1 + kPadC)] = val;
    PTf[2 * ((n - 1 - C) * pitch + R + 1 + kPadC) + 1] = val;
  }
  // zero padding: P rows of the left / right edge tiles, PT rows of the top / bottom
  constexpr int kPadL = kPadC + 1;  // indices 0 .. kPadC (c = -1 - kPadC .. -1)
  const int padR = (int)pitch - (n + 1 + kPadC);  // indices n + 1 + kPadC .. pitch - 1
  const float2 z = make_float2(0.f, 0.f);
  if (C0 == 0)
    for (int e = threadIdx.x; e < w * kPadL; e += blockDim.x)
      P[(R0 + e / kPadL) * pitch + e % kPadL] = z;
  if (C0 + w == n)
    for (int e = threadIdx.x; e < w * padR; e += blockDim.x)
      P[(R0 + e / padR) * pitch + n + 1 + kPadC + e % padR] = z;
  if (R0 == 0)
    for (int e = threadIdx.x; e < w * kPadL; e += blockDim.x)
      PT[(C0 + e / kPadL) * pitch + e % kPadL] = z;
  if (R0 + w == n)
    for (int e = threadIdx.x; e < w * padR; e += blockDim.x)
      PT[(C0 + e / padR) * pitch + n + 1 + kPadC + e % padR] = z;
}

// ---- SAGA image side --------------------------------------------------------

// Coarse level (factor f > 1): phi_new = U_f(bp)/f^2 is constant on f x f
// blocks, so the table row is stored compactly (one value per coarse pixel).
// A CTA owns whole blocks (tile side ts is a multiple of f), reads every old
// row value it needs, synchronises, then replaces the row entries it owns.
__global__ void __launch_bounds__(256)
k_saga_image_coarse(const float* __restrict__ bp, int side, int f, int ts, float inv_f2,
                    ImageSaga sg) {
  const int n = side / f;
  const int x0 = blockIdx.x * ts, y0 = blockIdx.y * ts;
  IMASK_CHECK_RANGE(56, (long long)(gridDim.x * ts) - side, 1);  // the tiles cover the image exactly
  IMASK_CHECK_RANGE(57, ts % f, 1);                              // and hold whole f x f blocks
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x) {
    const int row = y0 + e / ts, col = x0 + e % ts;
    const int q = (row / f) * n + col / f;
    const size_t p = (size_t)row * side + col;
    IMASK_CHECK_RANGE(58, q, (long long)n * n);
    IMASK_CHECK_RANGE(59, p, (long long)side * side);
    const float pn = __ldg(bp + q) * inv_f2;
    const float d = pn - sg.phi_tab[q];
    const float ps = sg.phi_sum[p];
    const float xi = d + ps;
    sg.phi_sum[p] = fmaf(sg.p_i, d, ps);
    const float xo = sg.x[p], xn = fmaf(-sg.s, xi, xo) * sg.inv_den;
    sg.x[p] = xn;
    extrapolate(sg, p, xo, xn);
  }
  __syncthreads();
  const int tc = ts / f;
  for (int e = threadIdx.x; e < tc * tc; e += blockDim.x) {
    const int q = (y0 / f + e / tc) * n + x0 / f + e % tc;
    sg.phi_tab[q] = __ldg(bp + q) * inv_f2;
  }
}

// Full level: phi_new = S_r(bp) computed tile-locally, then the update.
template <int TT>
__global__ void __launch_bounds__(256)
k_saga_image_full(const float* __restrict__ bp, int side, CompParams cp, ImageSaga sg) {
  __shared__ float tile[TT * TT];
  __shared__ float pyr[TT * TT / 3 + 8];
  const int ts = side / (int)gridDim.x;  // the launcher's tile (cover_tile): divides side, <= TT
  const int x0 = blockIdx.x * ts, y0 = blockIdx.y * ts;
  IMASK_CHECK_RANGE(53, (long long)(gridDim.x * ts) - side, 1);
  IMASK_CHECK_RANGE(54, ts, TT + 1);
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x) {
    IMASK_CHECK_RANGE(55, (size_t)(y0 + e / ts) * side + x0 + e % ts, (long long)side * side);
    tile[e] = __ldg(bp + (size_t)(y0 + e / ts) * side + x0 + e % ts);
  }
  __syncthreads();
  build_pyramid(tile, pyr, ts, cp.r);
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x) {
    const int py = e / ts, px = e % ts;
    const size_t p = (size_t)(y0 + py) * side + x0 + px;
    const float pn = compensated(tile[e], pyr, ts, cp, py, px);
    const float d = pn - sg.phi_tab[p];
    const float ps = sg.phi_sum[p];
    const float xi = d + ps;
    sg.phi_sum[p] = fmaf(sg.p_i, d, ps);
    sg.phi_tab[p] = pn;
    const float xo = sg.x[p], xn = fmaf(-sg.s, xi, xo) * sg.inv_den;
    sg.x[p] = xn;
    extrapolate(sg, p, xo, xn);
  }
}

// ---- sinogram-side SAGA update as its own pass --------------------------------
// psi_new = K_i x from the projector, then solvers.py:205-215 per bin (psi row,
// psi_sum, dual prox) with 128-bit accesses; used where the forward kernel is
// better off without the epilogue's prefetched state (large levels).
template <bool kVec>
__global__ void __launch_bounds__(256)
k_saga_sino(const float* __restrict__ psi_new, size_t m, SinoSaga sg) {
  const size_t q4 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (kVec && q4 + 4 <= m) {
    // every operand 16-byte aligned: one 128-bit access per array and thread.
    // y, b, the table row and the sum were last written by the previous step,
    // complete before this step's staging (a plain launch) started: loaded
    // before the programmatic wait
    const float4 yv = *reinterpret_cast<const float4*>(sg.y_in + q4);
    const float4 bv = __ldg(reinterpret_cast<const float4*>(sg.b + q4));
    float4 po = make_float4(0.f, 0.f, 0.f, 0.f), ps = po;
    if (sg.psi_tab) {
      po = *reinterpret_cast<const float4*>(sg.psi_tab + q4);
      ps = *reinterpret_cast<const float4*>(sg.psi_sum + q4);
    }
    griddep_wait();  // psi_new comes from the stream predecessor (the forward)
    const float4 v = __ldg(reinterpret_cast<const float4*>(psi_new + q4));
    const float vals[4] = {v.x, v.y, v.z, v.w}, pos[4] = {po.x, po.y, po.z, po.w},
                pss[4] = {ps.x, ps.y, ps.z, ps.w}, ys[4] = {yv.x, yv.y, yv.z, yv.w},
                bs[4] = {bv.x, bv.y, bv.z, bv.w};
    float nsum[4], ny[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // sino_update's arithmetic (solvers.py:205-215)
      const float d = vals[k] - pos[k];
      const float zeta = d + pss[k];
      nsum[k] = fmaf(sg.p_i, d, pss[k]);
      const float yn = fmaf(sg.sigma, zeta, ys[k]);
      ny[k] = (yn - sg.sigma * bs[k]) * sg.inv_1ps;
    }
    if (sg.psi_tab) {
      *reinterpret_cast<float4*>(sg.psi_sum + q4) = make_float4(nsum[0], nsum[1], nsum[2], nsum[3]);
      *reinterpret_cast<float4*>(sg.psi_tab + q4) = v;
    }
    *reinterpret_cast<float4*>(sg.y + q4) = make_float4(ny[0], ny[1], ny[2], ny[3]);
  } else {
    griddep_wait();
    for (size_t q = q4; q < m && q < q4 + 4; ++q) sino_update(sg, q, sino_load(sg, q), psi_new[q]);
  }
}

cudaError_t launch_saga_sino(const float* psi_new, size_t m, const SinoSaga& sg, cudaStream_t s) {
  const size_t threads = (m + 3) / 4;
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool vec = al(psi_new) && al(sg.y_in) && al(sg.y) && al(sg.b) &&
                   (!sg.psi_tab || (al(sg.psi_tab) && al(sg.psi_sum)));
  if (vec)
    return launch_pdl(k_saga_sino<true>, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s,
                      psi_new, m, sg);
  return launch_pdl(k_saga_sino<false>, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s,
                    psi_new, m, sg);
}

// ---- PDHG primal step (solvers.py:335-337) -----------------------------------
// x' = (x - tau K^T y) / (1 + tau mu_g) (ridge prox), xbar = x' + theta (x' - x).
__global__ void __launch_bounds__(256)
k_pdhg_image(const float* __restrict__ bp, float* __restrict__ x, float* __restrict__ xbar,
             size_t d, float tau, float inv_den, float theta) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  const float xo = x[i];
  const float xn = fmaf(-tau, __ldg(bp + i), xo) * inv_den;
  x[i] = xn;
  xbar[i] = fmaf(theta, xn - xo, xn);
}

cudaError_t launch_pdhg_image(const float* bp, float* x, float* xbar, size_t d, float tau,
                              float inv_den, float theta, cudaStream_t s) {
  k_pdhg_image<<<(unsigned)((d + 255) / 256), 256, 0, s>>>(bp, x, xbar, d, tau, inv_den, theta);
  return cudaGetLastError();
}

// ---- resum (solvers.py:184-191) --------------------------------------------

__global__ void k_resum_image(const float* __restrict__ phi_tab, float* __restrict__ phi_sum,
                              int side, ResumParams rp) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (size_t)side * side) return;
  const int row = (int)(p / side), col = (int)(p % side);
  float acc = 0.f;
  for (int i = 0; i < rp.r; ++i) {
    const int f = rp.factor[i], n = side / f;
    const float v = rp.p[i] * __ldg(phi_tab + rp.offset[i] + (size_t)(row / f) * n + col / f);
    acc = (i == 0) ? v : acc + v;
  }
  phi_sum[p] = acc;
}

__global__ void k_resum_sino(const float* __restrict__ psi_tab, float* __restrict__ psi_sum,
                             size_t m, ResumParams rp) {
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  float acc = 0.f;
  for (int i = 0; i < rp.r; ++i) {
    const float v = rp.p[i] * __ldg(psi_tab + (size_t)i * m + q);
    acc = (i == 0) ? v : acc + v;
  }
  psi_sum[q] = acc;
}

// ---- launchers --------------------------------------------------------------

static inline unsigned blocks_for(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_restrict(const float* x, float* u, int side, int f, cudaStream_t s) {
  const int n = side / f;
  if (side % 32 == 0 && f >= 2 && f <= 32) {
    int lg = 0;
    while ((1 << lg) < f) ++lg;
    if ((1 << lg) == f) {
      k_restrict32<<<dim3(side / 32, side / 32), 256, 0, s>>>(x, u, side, lg);
      return cudaGetLastError();
    }
  }
  if (f >= 16) {
    k_restrict_warp<<<blocks_for((size_t)n * n * 32, 256), 256, 0, s>>>(x, u, side, f);
  } else {
    k_restrict_small<<<blocks_for((size_t)n * n, 256), 256, 0, s>>>(x, u, side, f);
  }
  return cudaGetLastError();
}

cudaError_t launch_prolong(const float* u, float* x, int side, int f, float alpha,
                           cudaStream_t s) {
  k_prolong<<<blocks_for((size_t)side * side, 256), 256, 0, s>>>(u, x, side, f, alpha);
  return cudaGetLastError();
}

static inline int comp_tile(int r) { return (r <= 6) ? 32 : 64; }

// Tile side of the generic (any-size) kernels: the largest multiple of `align`
// (the block side the tile must hold whole: 2^(r-1) for the compensation
// pyramid, f for the coarse image update) that is <= cap and divides `side`,
// so the grid side / ts covers the image exactly. (side / 32 tiles of 32 left
// the last side % 32 rows and columns of a 48^2 image untouched.)
static inline int cover_tile(int side, int align, int cap) {
  int best = align;
  for (int ts = align; ts <= cap && ts <= side; ts += align)
    if (side % ts == 0) best = ts;
  return best;
}

cudaError_t launch_compensate(const float* x, float* out, int side, const CompParams& cp,
                              cudaStream_t s) {
  if (side % 32 == 0 && cp.r <= 6) {
    k_compensate32<<<dim3(side / 32, side / 32), 256, 0, s>>>(x, out, side, cp);
    return cudaGetLastError();
  }
  const int TT = comp_tile(cp.r);
  const int ts = cover_tile(side, 1 << (cp.r - 1), TT);
  dim3 grid(side / ts, side / ts);
  if (TT == 32)
    k_compensate<32><<<grid, 256, 0, s>>>(x, out, side, cp);
  else
    k_compensate<64><<<grid, 256, 0, s>>>(x, out, side, cp);
  return cudaGetLastError();
}

bool debug_bounds_read_sketch(unsigned long long* out4, bool reset) {
  return bounds_read(out4, reset);
}

bool stage32_ok(int side, int f, int r) { return side % 32 == 0 && f <= 32 && r <= 6; }

cudaError_t launch_stage32(const float* x, int side, int f, const CompParams& cp, float2* P,
                           float2* PT, cudaStream_t s) {
  int lg = 0;
  while ((1 << lg) < f) ++lg;
  launch_pdl(k_stage32, dim3(side / 32, side / 32), dim3(256), 0, s, x, side, lg, cp, P, PT);
  return cudaGetLastError();
}

cudaError_t launch_prepare(const float* u, int n, float2* P, float2* PT, float2* PM,
                           float2* PTM, bool diff, cudaStream_t s) {
  const int tiles = (pair_pitch(n) + 31) / 32;
  dim3 grid(tiles, tiles);
  launch_pdl(k_prepare, grid, dim3(256), 0, s, u, n, P, PT, PM, PTM, diff);
  return cudaGetLastError();
}

cudaError_t launch_saga_image_coarse(const float* bp, int side, int f, const ImageSaga& sg,
                                     cudaStream_t s) {
  if (side % 32 == 0 && f <= 32 && 32 % f == 0) {
    int lg = 0;
    while ((1 << lg) < f) ++lg;
    launch_pdl(k_saga_image_coarse32, dim3(side / 32, side / 32), dim3(256), 0, s, bp, side, lg,
               1.0f / (float)(f * f), sg);
    return cudaGetLastError();
  }
  const int ts = cover_tile(side, f, f > 32 ? f : 32);
  dim3 grid(side / ts, side / ts);
  k_saga_image_coarse<<<grid, 256, 0, s>>>(bp, side, f, ts, 1.0f / (float)(f * f), sg);
  return cudaGetLastError();
}

cudaError_t launch_saga_image_full(const float* bp, int side, const CompParams& cp,
                                   const ImageSaga& sg, cudaStream_t s) {
  if (side % 32 == 0 && cp.r <= 6) {
    launch_pdl(k_saga_image_full32, dim3(side / 32, side / 32), dim3(256), 0, s, bp, side, cp, sg);
    return cudaGetLastError();
  }
  const int TT = comp_tile(cp.r);
  const int ts = cover_tile(side, 1 << (cp.r - 1), TT);
  dim3 grid(side / ts, side / ts);
  if (TT == 32)
    k_saga_image_full<32><<<grid, 256, 0, s>>>(bp, side, cp, sg);
  else
    k_saga_image_full<64><<<grid, 256, 0, s>>>(bp, side, cp, sg);
  return cudaGetLastError();
}

cudaError_t launch_resum(const float* phi_tab, float* phi_sum, int side, const float* psi_tab,
                         float* psi_sum, size_t m, const ResumParams& rp, cudaStream_t s) {
  k_resum_image<<<blocks_for((size_t)side * side, 256), 256, 0, s>>>(phi_tab, phi_sum, side, rp);
  k_resum_sino<<<blocks_for(m, 256), 256, 0, s>>>(psi_tab, psi_sum, m, rp);
  return cudaGetLastError();
}

}  // namespace imask
