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
  const int ts = min(TT, side);
  const int x0 = blockIdx.x * ts, y0 = blockIdx.y * ts;
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x)
    tile[e] = __ldg(x + (size_t)(y0 + e / ts) * side + x0 + e % ts);
  __syncthreads();
  build_pyramid(tile, pyr, ts, cp.r);
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x) {
    const int py = e / ts, px = e % ts;
    out[(size_t)(y0 + py) * side + x0 + px] = compensated(tile[e], pyr, ts, cp, py, px);
  }
}

// Fast path (side % 32 == 0, r <= 6): 32 x 32 tile, four contiguous pixels per
// thread with 128-bit loads/stores; the pyramid terms of levels >= 2 are shared
// by the four pixels, so acc = (sum over levels r-1..2, coarsest first) + the
// level-1 term, which keeps the reference's accumulation order.
struct CompTile32 {
  float tile[32 * 32];
  float pyr[16 * 16 + 8 * 8 + 4 * 4 + 2 * 2 + 1];
};

__device__ __forceinline__ void comp32_build(CompTile32& sm, int r) {
  // level j has side 32 >> j at offset off(j) = sum_{l<j} (32 >> l)^2 (level 1 at 0)
  const float* src = sm.tile;
  float* dst = sm.pyr;
  int sn = 32;
  for (int lev = 1; lev < r; ++lev) {
    const int dn = sn >> 1;
    if ((int)threadIdx.x < dn * dn) {
      const int rr = threadIdx.x / dn, cc = threadIdx.x % dn;
      const float* s0 = src + (2 * rr) * sn + 2 * cc;
      dst[threadIdx.x] = ((s0[0] + s0[1]) + (s0[sn] + s0[sn + 1])) * 0.25f;
    }
    __syncthreads();
    src = dst;
    dst += dn * dn;
    sn = dn;
  }
}

// S_r of the four pixels (py, px..px+3) of the staged tile.
__device__ __forceinline__ float4 comp32_quad(const CompTile32& sm, const CompParams& cp, int py,
                                             int px) {
  const float4 v = *reinterpret_cast<const float4*>(&sm.tile[py * 32 + px]);
  if (cp.r == 1) return v;  // S_1 = I (mrsketch.py:137-138)
  float shared_acc = 0.f;
  bool first = true;
  for (int i = 1; i < cp.r - 1; ++i) {  // levels j = r-1 .. 2
    const int j = cp.r - i;
    const int sj = 32 >> j;
    const int off = (1024 - (1 << (12 - 2 * j))) / 3;  // sum of (32 >> l)^2, l < j
    const float term = cp.p[i - 1] * sm.pyr[off + (py >> j) * sj + (px >> j)];
    shared_acc = first ? term : shared_acc + term;
    first = false;
  }
  const float pl = cp.p[cp.r - 2];  // level-1 term (factor 2), last in the telescoping order
  const float t0 = pl * sm.pyr[(py >> 1) * 16 + (px >> 1)];
  const float t1 = pl * sm.pyr[(py >> 1) * 16 + (px >> 1) + 1];
  const float a0 = first ? t0 : shared_acc + t0;
  const float a1 = first ? t1 : shared_acc + t1;
  return make_float4((v.x - a0) / cp.pr, (v.y - a0) / cp.pr, (v.z - a1) / cp.pr,
                     (v.w - a1) / cp.pr);
}

__global__ void __launch_bounds__(256)
k_compensate32(const float* __restrict__ x, float* __restrict__ out, int side, CompParams cp) {
  __shared__ __align__(16) CompTile32 sm;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, px = (threadIdx.x & 7) * 4;
  const size_t g = (size_t)(y0 + py) * side + x0 + px;
  *reinterpret_cast<float4*>(&sm.tile[py * 32 + px]) = __ldg(reinterpret_cast<const float4*>(x + g));
  __syncthreads();
  comp32_build(sm, cp.r);
  *reinterpret_cast<float4*>(out + g) = comp32_quad(sm, cp, py, px);
}

// Restriction by a power-of-two factor f = 2^lg <= 32 (side % 32 == 0): each
// CTA stages a 32 x 32 tile of x with 128-bit loads, builds the block-mean
// pyramid in shared memory and writes the tile's (32/f)^2 coarse pixels.
__global__ void __launch_bounds__(256)
k_restrict32(const float* __restrict__ x, float* __restrict__ u, int side, int lg) {
  __shared__ __align__(16) CompTile32 sm;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, px = (threadIdx.x & 7) * 4;
  *reinterpret_cast<float4*>(&sm.tile[py * 32 + px]) =
      __ldg(reinterpret_cast<const float4*>(x + (size_t)(y0 + py) * side + x0 + px));
  __syncthreads();
  comp32_build(sm, lg + 1);
  const int sj = 32 >> lg, n = side >> lg;
  const int off = (1024 - (1 << (12 - 2 * lg))) / 3;  // pyramid offset of level lg
  if ((int)threadIdx.x < sj * sj) {
    const int rr = threadIdx.x / sj, cc = threadIdx.x % sj;
    u[(size_t)((y0 >> lg) + rr) * n + (x0 >> lg) + cc] = sm.pyr[off + rr * sj + cc];
  }
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
__global__ void __launch_bounds__(256)
k_saga_image_full32(const float* __restrict__ bp, int side, CompParams cp, ImageSaga sg) {
  __shared__ __align__(16) CompTile32 sm;
  griddep_wait();  // bp comes from the stream predecessor (the adjoint reduction)
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, px = (threadIdx.x & 7) * 4;
  const size_t g = (size_t)(y0 + py) * side + x0 + px;
  *reinterpret_cast<float4*>(&sm.tile[py * 32 + px]) = __ldg(reinterpret_cast<const float4*>(bp + g));
  float4 tab = *reinterpret_cast<const float4*>(sg.phi_tab + g);
  float4 sum = *reinterpret_cast<const float4*>(sg.phi_sum + g);
  float4 xv = *reinterpret_cast<const float4*>(sg.x + g);
  const float4 xo = xv;
  __syncthreads();
  comp32_build(sm, cp.r);
  const float4 pn = comp32_quad(sm, cp, py, px);
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
k_saga_image_coarse32(const float* __restrict__ bp, int side, int f, float inv_f2, ImageSaga sg) {
  griddep_wait();  // bp comes from the stream predecessor (the adjoint reduction)
  const int n = side / f;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int py = threadIdx.x >> 3, px = (threadIdx.x & 7) * 4;
  const int row = y0 + py, col = x0 + px;
  const size_t g = (size_t)row * side + col;
  const int qrow = (row / f) * n;
  float4 sum = *reinterpret_cast<const float4*>(sg.phi_sum + g);
  float4 xv = *reinterpret_cast<const float4*>(sg.x + g);
  const float4 xo = xv;
  float pn[4], po[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = qrow + (col + k) / f;
    pn[k] = __ldg(bp + q) * inv_f2;
    po[k] = sg.phi_tab[q];
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
  const int tc = 32 / f;
  if ((int)threadIdx.x < tc * tc) {
    const int q = (y0 / f + threadIdx.x / tc) * n + x0 / f + threadIdx.x % tc;
    sg.phi_tab[q] = __ldg(bp + q) * inv_f2;
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
          float2* __restrict__ PM, float2* __restrict__ PTM) {
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
          // value planes (u, um) in P, difference planes (d, dm) in PM
          const float vm = tm[rr][cc + 1];
          P[o] = make_float2(v, vm);
          PM[o] = make_float2(dv, tm[rr][cc + 2] - vm);
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
          PTM[o] = make_float2(dv, tm[cc + 1][rr + 1] - vm);
        }
      }
    }
  }
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
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x) {
    const int row = y0 + e / ts, col = x0 + e % ts;
    const int q = (row / f) * n + col / f;
    const size_t p = (size_t)row * side + col;
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
  const int ts = min(TT, side);
  const int x0 = blockIdx.x * ts, y0 = blockIdx.y * ts;
  for (int e = threadIdx.x; e < ts * ts; e += blockDim.x)
    tile[e] = __ldg(bp + (size_t)(y0 + e / ts) * side + x0 + e % ts);
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
__global__ void __launch_bounds__(256)
k_saga_sino(const float* __restrict__ psi_new, size_t m, SinoSaga sg) {
  griddep_wait();  // psi_new comes from the stream predecessor (the forward)
  const size_t q4 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (q4 + 4 <= m) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(psi_new + q4));
    const float vals[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) sino_update(sg, q4 + k, sino_load(sg, q4 + k), vals[k]);
  } else {
    for (size_t q = q4; q < m; ++q) sino_update(sg, q, sino_load(sg, q), psi_new[q]);
  }
}

cudaError_t launch_saga_sino(const float* psi_new, size_t m, const SinoSaga& sg, cudaStream_t s) {
  const size_t threads = (m + 3) / 4;
  return launch_pdl(k_saga_sino, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s,
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

cudaError_t launch_compensate(const float* x, float* out, int side, const CompParams& cp,
                              cudaStream_t s) {
  if (side % 32 == 0 && cp.r <= 6) {
    k_compensate32<<<dim3(side / 32, side / 32), 256, 0, s>>>(x, out, side, cp);
    return cudaGetLastError();
  }
  const int TT = comp_tile(cp.r);
  const int ts = side < TT ? side : TT;
  dim3 grid(side / ts, side / ts);
  if (TT == 32)
    k_compensate<32><<<grid, 256, 0, s>>>(x, out, side, cp);
  else
    k_compensate<64><<<grid, 256, 0, s>>>(x, out, side, cp);
  return cudaGetLastError();
}

cudaError_t launch_prepare(const float* u, int n, float2* P, float2* PT, float2* PM,
                           float2* PTM, cudaStream_t s) {
  const int tiles = (pair_pitch(n) + 31) / 32;
  dim3 grid(tiles, tiles);
  launch_pdl(k_prepare, grid, dim3(256), 0, s, u, n, P, PT, PM, PTM);
  return cudaGetLastError();
}

cudaError_t launch_saga_image_coarse(const float* bp, int side, int f, const ImageSaga& sg,
                                     cudaStream_t s) {
  if (side % 32 == 0 && f <= 32 && 32 % f == 0) {
    launch_pdl(k_saga_image_coarse32, dim3(side / 32, side / 32), dim3(256), 0, s, bp, side, f,
               1.0f / (float)(f * f), sg);
    return cudaGetLastError();
  }
  int ts = f > 32 ? f : 32;
  if (ts > side) ts = side;
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
  const int ts = side < TT ? side : TT;
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
