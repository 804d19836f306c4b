// Kernels (1) and (2): exact-chord forward projector and its matched
// pixel-driven adjoint, at any sketch level (pixel width h = factor).
//
// Forward (ray-driven gather): one thread per ray (angle a, detector j); a
// warp is 32 consecutive detectors of one angle, so sinogram writes are
// coalesced and the 32 rays of a warp sweep adjacent pixels of each band.
// The image is pre-staged (prepare kernel, sketch.cu) as "pair" rows
// P[band][c+1] = (u[c], u[c+1]-u[c]) so one 8-byte load per band yields both
// chord partners: sum_band u[c0] + g*(u[c0+1]-u[c0]) == (1-g)u[c0] + g u[c0+1].
// Row-family angles read the row-major pair image, column-family angles the
// transposed one, so both families read along contiguous memory.
//
// Adjoint (pixel-driven gather, no atomics): one thread per 4 pixels of a
// 32x32 tile, looping over all angles; per angle the pixel's footprint covers
// nb detector bins whose weights come from the same trapezoid the forward's
// chords integrate (reference operator: ctmodel.py:73-154).
#include "imask_common.cuh"

namespace imask {

// rows b in [lo, hi) where the ray's left chord partner floor(xi) is in [-1, n-1]
__device__ __forceinline__ bool band_ok(long long X0, long long step, int b, int n) {
  long long X = X0 + (long long)b * step;
  return X >= -(1LL << 32) && X < ((long long)n << 32);
}

__device__ void band_range(long long X0, long long step, int n, int* lo_out, int* hi_out) {
  int lo, hi;
  if (step == 0) {
    bool ok = band_ok(X0, 0, 0, n);
    lo = 0;
    hi = ok ? n : 0;
  } else {
    double x0 = (double)X0, st = (double)step;
    double e1 = (-kFix - x0) / st;
    double e2 = ((double)n * kFix - x0) / st;
    double elo = fmin(e1, e2), ehi = fmax(e1, e2);
    elo = fmax(elo, 0.0);
    ehi = fmin(ehi + 1.0, (double)n);
    lo = (int)ceil(elo) - 1;
    if (lo < 0) lo = 0;
    if (lo > n) lo = n;
    hi = (int)ehi;
    if (hi > n) hi = n;
    if (hi < lo) hi = lo;
    // exact fix-up (the valid set is an interval)
    while (lo > 0 && band_ok(X0, step, lo - 1, n)) --lo;
    while (lo < n && !band_ok(X0, step, lo, n)) ++lo;
    if (hi < lo) hi = lo;
    while (hi < n && band_ok(X0, step, hi, n)) ++hi;
    while (hi > lo && !band_ok(X0, step, hi - 1, n)) --hi;
  }
  *lo_out = lo;
  *hi_out = hi;
}

template <bool kSaga>
__global__ void __launch_bounds__(256)
k_forward(const float2* __restrict__ P, const float2* __restrict__ PT, int n, int pitch,
          const FwdAngle* __restrict__ ang, int n_loc, int n_det, float* __restrict__ sino,
          SinoSaga saga) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int a = blockIdx.y * 8 + warp;
  if (a >= n_loc) return;
  const int j = blockIdx.x * 32 + lane;
  const FwdAngle A = ang[a];
  const float2* __restrict__ img = A.transposed ? PT : P;
  float acc = 0.f;
  if (j < n_det) {
    const long long X0 = __double2ll_rn(fma((double)j, A.xi_dj, A.xi_base) * kFix);
    int lo, hi;
    band_range(X0, A.step, n, &lo, &hi);
    long long X = X0 + (long long)lo * A.step;
    const float2* prow = img + (size_t)lo * pitch + 1;
    const float S = A.S, B = A.B;
    const long long step = A.step;
#pragma unroll 4
    for (int b = lo; b < hi; ++b) {
      const int c0 = (int)(X >> 32);
      const float g = __saturatef(fmaf(onep_from_frac((uint32_t)X), S, B));
      const float2 v = __ldg(prow + c0);
      acc += v.x;
      acc = fmaf(g, v.y, acc);
      X += step;
      prow += pitch;
    }
    acc *= A.wsc;
    const size_t q = (size_t)a * n_det + j;
    if (kSaga) {
      // sinogram side of sketch_step (solvers.py:205-215): psi row, psi_sum, dual prox
      const float po = saga.psi_tab[q];
      const float d = acc - po;
      const float ps = saga.psi_sum[q];
      const float zeta = d + ps;
      saga.psi_sum[q] = fmaf(saga.p_i, d, ps);
      saga.psi_tab[q] = acc;
      const float yv = fmaf(saga.sigma, zeta, saga.y[q]);
      saga.y[q] = (yv - saga.sigma * saga.b[q]) * saga.inv_1ps;
    } else {
      sino[q] = acc;
    }
  }
}

constexpr int kAdjChunk = 64;   // angles staged per smem round
constexpr int kTile = 32;       // pixels per tile side
constexpr int kRowsPerThread = 4;

struct AdjStage {
  long long E;  // Q32.32 of (eta - R) at the tile origin, plus 2^32-1 (ceil bias)
  long long Dc, Ds;
  float kneg, Rk, R, wsc;
  int nb, axis;
};

// NB > 0: compile-time bin count (all non-axis angles at factor 1 have 2 bins)
template <int NB>
__global__ void __launch_bounds__(256)
k_adjoint(const float* __restrict__ sino, float* __restrict__ out, int n, int n_loc, int n_det,
          const AdjAngle* __restrict__ ang) {
  __shared__ AdjStage st[kAdjChunk];
  const int x0 = blockIdx.x * kTile, y0 = blockIdx.y * kTile;
  const int dx = threadIdx.x & 31, dy = threadIdx.x >> 5;  // rows dy + 8k
  float acc[kRowsPerThread];
#pragma unroll
  for (int k = 0; k < kRowsPerThread; ++k) acc[k] = 0.f;

  for (int a0 = 0; a0 < n_loc; a0 += kAdjChunk) {
    const int na = min(kAdjChunk, n_loc - a0);
    __syncthreads();
    for (int t = threadIdx.x; t < na; t += blockDim.x) {
      const AdjAngle A = ang[a0 + t];
      AdjStage s;
      const double eta = A.eta0 + (double)x0 * A.ch + (double)y0 * A.sh;
      s.E = __double2ll_rn(eta * kFix) + 0xFFFFFFFFLL;
      s.Dc = A.Dc;
      s.Ds = A.Ds;
      s.kneg = A.kneg;
      s.Rk = A.Rk;
      s.R = A.R;
      s.wsc = A.wsc;
      s.nb = A.nb;
      s.axis = A.axis;
      st[t] = s;
    }
    __syncthreads();
    for (int t = 0; t < na; ++t) {
      const AdjStage s = st[t];
      const float* __restrict__ yrow = sino + (size_t)(a0 + t) * n_det;
      long long E = s.E + (long long)dx * s.Dc + (long long)dy * s.Ds;
      const long long E8 = 8LL * s.Ds;
#pragma unroll
      for (int k = 0; k < kRowsPerThread; ++k) {
        const int lo = (int)(E >> 32);
        const float onep = onep_from_frac(~(uint32_t)E);  // 1 + (ceil(v) - v)
        float part = 0.f;
        if (s.axis) {
          // half-open box [eta - h/2, eta + h/2): bins lo .. lo+nb-1, weight h
          for (int bb = 0; bb < s.nb; ++bb) {
            const int jj = lo + bb;
            if (jj >= 0 && jj < n_det) part += __ldg(yrow + jj);
          }
        } else if (NB > 0) {
#pragma unroll
          for (int bb = 0; bb < NB; ++bb) {
            const int jj = lo + bb;
            const float u = onep + (float)(bb - 1) - s.R;
            const float w = __saturatef(fmaf(fabsf(u), s.kneg, s.Rk));
            if (jj >= 0 && jj < n_det) part = fmaf(w, __ldg(yrow + jj), part);
          }
        } else {
          for (int bb = 0; bb < s.nb; ++bb) {
            const int jj = lo + bb;
            const float u = onep + (float)(bb - 1) - s.R;
            const float w = __saturatef(fmaf(fabsf(u), s.kneg, s.Rk));
            if (jj >= 0 && jj < n_det) part = fmaf(w, __ldg(yrow + jj), part);
          }
        }
        acc[k] = fmaf(s.wsc, part, acc[k]);
        E += E8;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kRowsPerThread; ++k) {
    const int row = y0 + dy + 8 * k, col = x0 + dx;
    if (row < n && col < n) out[(size_t)row * n + col] = acc[k];
  }
}

// ---- launchers ----------------------------------------------------------

cudaError_t launch_forward(const float2* P, const float2* PT, int n, const FwdAngle* ang,
                           int n_loc, int n_det, float* sino, const SinoSaga* saga,
                           cudaStream_t stream) {
  dim3 grid((n_det + 31) / 32, (n_loc + 7) / 8);
  if (saga) {
    k_forward<true><<<grid, 256, 0, stream>>>(P, PT, n, n + 1, ang, n_loc, n_det, nullptr, *saga);
  } else {
    SinoSaga none{};
    k_forward<false><<<grid, 256, 0, stream>>>(P, PT, n, n + 1, ang, n_loc, n_det, sino, none);
  }
  return cudaGetLastError();
}

cudaError_t launch_adjoint(const float* sino, float* out, int n, int factor, int n_loc,
                           int n_det, const AdjAngle* ang, cudaStream_t stream) {
  dim3 grid((n + kTile - 1) / kTile, (n + kTile - 1) / kTile);
  if (factor == 1) {
    k_adjoint<2><<<grid, 256, 0, stream>>>(sino, out, n, n_loc, n_det, ang);
  } else {
    k_adjoint<0><<<grid, 256, 0, stream>>>(sino, out, n, n_loc, n_det, ang);
  }
  return cudaGetLastError();
}

}  // namespace imask
