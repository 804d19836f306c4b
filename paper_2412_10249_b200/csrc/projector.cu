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
// Adjoint (pixel-driven gather, no atomics): see the adjoint section below;
// per angle a pixel's footprint covers nb detector bins whose weights are the
// trapezoid the forward's chords integrate (reference operator:
// ctmodel.py:73-154).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>

#include <cooperative_groups.h>

#include "imask_common.cuh"

namespace cg = cooperative_groups;

namespace imask {

// bands b in [lo, hi) where the ray's left chord partner floor(xi) is in [-1, n-1]
__device__ __forceinline__ bool band_ok(long long X0, long long step, int b, int n) {
  const long long X = X0 + (long long)b * step;
  return X >= -(1LL << 32) && X < ((long long)n << 32);
}

__device__ __forceinline__ void band_range(long long X0, long long step, double inv_step, int n,
                                           int* lo_out, int* hi_out) {
  int lo, hi;
  if (step == 0) {
    lo = 0;
    hi = band_ok(X0, 0, 0, n) ? n : 0;
  } else {
    // float64 estimate (no division: inv_step = 2^32/step), then exact integer fix-up
    const double x0 = (double)X0 * (1.0 / kFix);
    const double e1 = (-1.0 - x0) * inv_step;
    const double e2 = ((double)n - x0) * inv_step;
    const double elo = fmax(fmin(e1, e2), -1.0), ehi = fmin(fmax(e1, e2), (double)n + 1.0);
    lo = min(max((int)ceil(elo), 0), n);
    hi = min(max((int)ceil(ehi), lo), n);
    // the bands of a ray are one interval and the estimate is within a band of
    // it, so the first band is searched no further than the estimated end + 1
    // (a ray that has left the image before band 0 used to walk all n bands
    // here: half the instructions of a prologue-only launch at n = 1024)
    const int guard = hi + 1;
    while (lo > 0 && band_ok(X0, step, lo - 1, n)) --lo;
    while (lo < n && lo <= guard && !band_ok(X0, step, lo, n)) ++lo;
    if (lo >= n || lo > guard) {
      lo = hi = 0;  // no band
    } else {
      if (hi < lo) hi = lo;
      while (hi < n && band_ok(X0, step, hi, n)) ++hi;
      while (hi > lo && !band_ok(X0, step, hi - 1, n)) --hi;
    }
  }
  *lo_out = lo;
  *hi_out = hi;
}

// The band offset is folded into the integer word of the Q32.32 position:
// Y = X + b * pitch * 2^32, so hi(Y) is directly the pair-image index of the
// left chord partner and one 64-bit add advances both position and band.
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
  // lanes past n_det trace the last detector's ray (result discarded)
  const int jr = min(j, n_det - 1);
  SinoIn sin;
  if (kSaga && j < n_det) sin = sino_load(saga, (size_t)a * n_det + j);
  const long long X0 = __double2ll_rn(fma((double)jr, A.xi_dj, A.xi_base) * kFix);
  int lo, hi;
  band_range(X0, A.step, A.inv_step, n, &lo, &hi);
  // the warp walks the union of its lanes' band ranges in lockstep, so every
  // load instruction reads one image row (coalesced); a lane outside its own
  // range reads the zero padding of the row (kPadC), so no predicate is needed
  int wlo = lo < hi ? lo : n, whi = lo < hi ? hi : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    wlo = min(wlo, __shfl_xor_sync(0xffffffffu, wlo, o));
    whi = max(whi, __shfl_xor_sync(0xffffffffu, whi, o));
  }
  // Y = X + (band * pitch + 1 + kPadC) * 2^32: hi(Y) is the pair-image index
  const long long dYl = A.step + ((long long)pitch << 32);
  Fix32 Y = fix_from(X0 + (long long)wlo * dYl + ((long long)(1 + kPadC) << 32));
  const Fix32 dY = fix_from(dYl);
  const float S = A.S, B = A.B;
  int b = wlo;
#pragma unroll 1
  for (; b + 4 <= whi; b += 4) {
    float2 v[4];
    float g[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      IMASK_CHECK_RANGE(10, Y.hi, (long long)n * pitch);
      v[k] = __ldg(img + Y.hi);
      g[k] = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
      fix_add(Y, dY);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc += v[k].x;
      acc = fmaf(g[k], v[k].y, acc);
    }
  }
  for (; b < whi; ++b) {
    const float2 v = __ldg(img + Y.hi);
    const float g = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
    acc += v.x;
    acc = fmaf(g, v.y, acc);
    fix_add(Y, dY);
  }
  if (j < n_det) {
    acc *= A.wsc;
    const size_t q = (size_t)a * n_det + j;
    if (kSaga) {
      // sinogram side of sketch_step (solvers.py:205-215): psi row, psi_sum, dual prox
      sino_update(saga, q, sin, acc);
    } else {
      sino[q] = acc;
    }
  }
}

// Mirror-symmetric forward (full, even-sized angle set): ray (a, j) and ray
// (n-a, j) are mirror images (theta -> pi-theta, x -> -x), so one warp walks
// both with the same fixed-point position: band b of the mirrored ray reads
// the mirrored pair image (PM: rows reversed left-right; PTM: PT with its
// bands reversed) at the same index. entries[e] = (a, mirror angle or -1);
// angle 0 is traced alone (its tie rule is not mirror-invariant) and so is
// the self-mirrored angle n/2.
template <bool kSaga>
__global__ void __launch_bounds__(256, 6)  // (256, 8) caps it at 32 registers and spills
k_forward_sym(const float2* __restrict__ P, const float2* __restrict__ PT,
              const float2* __restrict__ PM, const float2* __restrict__ PTM, int n, int pitch,
              const FwdAngle* __restrict__ ang, const int2* __restrict__ entries, int n_entries,
              int n_det, float* __restrict__ sino, SinoSaga saga) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.y * 8 + warp;
  if (e >= n_entries) return;
  const int2 ent = entries[e];
  const int a = ent.x, am = ent.y;
  const int j = blockIdx.x * 32 + lane;
  const FwdAngle A = ang[a];
  const float2* __restrict__ img = A.transposed ? PT : P;
  const float2* __restrict__ imgm = A.transposed ? PTM : PM;
  const int jr = min(j, n_det - 1);
  SinoIn sin[2];
  if (kSaga && j < n_det) {
    sin[0] = sino_load(saga, (size_t)a * n_det + j);
    if (am >= 0) sin[1] = sino_load(saga, (size_t)am * n_det + j);
  }
  const long long X0 = __double2ll_rn(fma((double)jr, A.xi_dj, A.xi_base) * kFix);
  int lo, hi;
  band_range(X0, A.step, A.inv_step, n, &lo, &hi);
  int wlo = lo < hi ? lo : n, whi = lo < hi ? hi : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    wlo = min(wlo, __shfl_xor_sync(0xffffffffu, wlo, o));
    whi = max(whi, __shfl_xor_sync(0xffffffffu, whi, o));
  }
  const long long dYl = A.step + ((long long)pitch << 32);
  Fix32 Y = fix_from(X0 + (long long)wlo * dYl + ((long long)(1 + kPadC) << 32));
  const Fix32 dY = fix_from(dYl);
  const float S = A.S, B = A.B;
  griddep_wait();  // the pair images come from the stream predecessor (k_prepare)
  // img holds value pairs (u, um), imgm difference pairs (d, dm) (k_prepare):
  // (acc, accm) += (u, um) + g * (d, dm) with packed FP32 ops
  float2 acc2 = make_float2(0.f, 0.f);
  int b = wlo;
#pragma unroll 1
  for (; b + 4 <= whi; b += 4) {
    float2 v[4], vd[4];
    float g[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      IMASK_CHECK_RANGE(11, Y.hi, (long long)n * pitch);
      v[k] = __ldg(img + Y.hi);
      vd[k] = __ldg(imgm + Y.hi);
      g[k] = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
      fix_add(Y, dY);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc2 = fadd2(acc2, v[k]);
      acc2 = ffma2(g[k], vd[k], acc2);
    }
  }
  for (; b < whi; ++b) {
    const float2 v = __ldg(img + Y.hi), vd = __ldg(imgm + Y.hi);
    const float g = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
    acc2 = fadd2(acc2, v);
    acc2 = ffma2(g, vd, acc2);
    fix_add(Y, dY);
  }
  const float acc = acc2.x, accm = acc2.y;
  if (j < n_det) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = r == 0 ? a : am;
      if (row < 0) break;
      const float val = (r == 0 ? acc : accm) * A.wsc;
      const size_t q = (size_t)row * n_det + j;
      if (kSaga) {
        sino_update(saga, q, sin[r], val);
      } else {
        sino[q] = val;
      }
    }
  }
}

// Quad form of k_forward_sym (the plan's rows closed under a -> n/2 - a too):
// entry (a, n-a, n/2-a, n/2+a) of the TMA forward's list, one position walk for
// four rays -- the transpose partners read PT / PTM at the same index as P /
// PM (the ray through u at pi/2 - theta is the ray through u^T at theta).
// Singles and the pair (n/4, 3n/4) come as entries with -1 slots; padding
// entries (all -1) idle. L1-cached loads: the coarse levels, where the images
// fit on chip and the walks are short.
#ifndef IMASK_FWDQ_UNROLL
#define IMASK_FWDQ_UNROLL 4
#endif
#ifndef IMASK_FWDQ_MINB
#define IMASK_FWDQ_MINB 4
#endif
template <bool kSaga, bool kVal>
__global__ void __launch_bounds__(256, IMASK_FWDQ_MINB)
k_forward_quad(const float2* __restrict__ P, const float2* __restrict__ PT,
               const float2* __restrict__ PM, const float2* __restrict__ PTM, int n, int pitch,
               const FwdAngle* __restrict__ ang, const int4* __restrict__ entries, int n_entries,
               int n_det, float* __restrict__ sino, SinoSaga saga) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.y * 8 + warp;
  if (e >= n_entries) return;
  const int4 ent = entries[e];
  const int rows[4] = {ent.x, ent.y, ent.z, ent.w};
  const int tab = ent.x >= 0 ? ent.x : ent.z;  // the entry's parameter row
  if (tab < 0) return;
  const int j = blockIdx.x * 32 + lane;
  const FwdAngle A = ang[tab];
  const int jr = min(j, n_det - 1);
  SinoIn sin[4];
  if (kSaga && j < n_det) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (rows[r] >= 0) sin[r] = sino_load(saga, (size_t)rows[r] * n_det + j);
  }
  const long long X0 = __double2ll_rn(fma((double)jr, A.xi_dj, A.xi_base) * kFix);
  int lo, hi;
  band_range(X0, A.step, A.inv_step, n, &lo, &hi);
  int wlo = lo < hi ? lo : n, whi = lo < hi ? hi : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    wlo = min(wlo, __shfl_xor_sync(0xffffffffu, wlo, o));
    whi = max(whi, __shfl_xor_sync(0xffffffffu, whi, o));
  }
  const long long dYl = A.step + ((long long)pitch << 32);
  Fix32 Y = fix_from(X0 + (long long)wlo * dYl + ((long long)(1 + kPadC) << 32));
  const Fix32 dY = fix_from(dYl);
  const float S = A.S, B = A.B;
  griddep_wait();  // the pair images come from the stream predecessor (k_prepare)
  float2 acc2 = make_float2(0.f, 0.f), accT = make_float2(0.f, 0.f);
  int b = wlo;
  // kU bands per iteration: 4 kU independent 8-byte loads in flight per thread
  // (the walk is bound by the latency of its L1 loads)
  constexpr int kU = IMASK_FWDQ_UNROLL;
#pragma unroll 1
  for (; b + kU <= whi; b += kU) {
    float2 v[kU], vd[kU], vt[kU], vdt[kU];
    float g[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      IMASK_CHECK_RANGE(12, (long long)Y.hi + (kVal ? 1 : 0), (long long)n * pitch);
      v[k] = __ldg(P + Y.hi);
      vt[k] = __ldg(PT + Y.hi);
      if (kVal) {  // difference pairs as P[c+1] - P[c] (k_prepare's subtraction)
        vd[k] = __ldg(P + Y.hi + 1);
        vdt[k] = __ldg(PT + Y.hi + 1);
      } else {
        vd[k] = __ldg(PM + Y.hi);
        vdt[k] = __ldg(PTM + Y.hi);
      }
      g[k] = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
      fix_add(Y, dY);
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      if (kVal) {
        vd[k] = fsub2(vd[k], v[k]);
        vdt[k] = fsub2(vdt[k], vt[k]);
      }
      acc2 = fadd2(acc2, v[k]);
      acc2 = ffma2(g[k], vd[k], acc2);
      accT = fadd2(accT, vt[k]);
      accT = ffma2(g[k], vdt[k], accT);
    }
  }
  for (; b < whi; ++b) {
    IMASK_CHECK_RANGE(13, (long long)Y.hi + (kVal ? 1 : 0), (long long)n * pitch);
    const float g = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
    const float2 v = __ldg(P + Y.hi), vt = __ldg(PT + Y.hi);
    const float2 vd = kVal ? fsub2(__ldg(P + Y.hi + 1), v) : __ldg(PM + Y.hi);
    const float2 vdt = kVal ? fsub2(__ldg(PT + Y.hi + 1), vt) : __ldg(PTM + Y.hi);
    acc2 = fadd2(acc2, v);
    acc2 = ffma2(g, vd, acc2);
    accT = fadd2(accT, vt);
    accT = ffma2(g, vdt, accT);
    fix_add(Y, dY);
  }
  if (j < n_det) {
    const float vals[4] = {acc2.x, acc2.y, accT.x, accT.y};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (rows[r] < 0) continue;
      const float val = vals[r] * A.wsc;
      const size_t q = (size_t)rows[r] * n_det + j;
      if (kSaga) {
        sino_update(saga, q, sin[r], val);
      } else {
        sino[q] = val;
      }
    }
  }
}

// ---- TMA-staged mirror-symmetric forward ---------------------------------------
//
// Same rays and arithmetic as k_forward_sym, but the image data come from
// shared memory: a CTA (8 angle entries of one family, each with its mirror,
// x 32 detectors; a warp takes 4 entries x 8 detectors) walks its bands in
// chunks of kFB; for every chunk the
// exact window of kFWc pair columns its rays touch is fetched for the image
// and its mirror by two cp.async.bulk.tensor.2d loads (double-buffered,
// mbarrier full/empty pipeline; TMA zero-fills outside the tensor). The warps
// then read the window with LDS.64 instead of L1-cached LDG, so the eight
// neighbouring angles share one on-chip copy. A CTA whose window would exceed
// kFWc (very wide angle spread) falls back to global loads. Window origins are
// rounded down to an even pair index: a tensor copy must start 16-byte aligned.
constexpr int kFB = 16;           // bands per chunk (pair mode)
constexpr int kFBQuad = 8;        // bands per chunk (quad mode: twice the images)
#ifndef IMASK_FWD_FBQ
#define IMASK_FWD_FBQ 16
#endif
// quad mode on value planes stages two images per chunk, like pair mode on both
// planes: chunks of 16 bands halve the per-chunk work of every warp (barrier
// wait, window origin, position rebuild, release: ~80 of the ~210 instructions
// a warp spent per 8-band chunk)
constexpr int kFBQuadVal = IMASK_FWD_FBQ;
#ifndef IMASK_FWD_ENTRIES
#define IMASK_FWD_ENTRIES 8
#endif
#ifndef IMASK_FWD_WINDOW
#define IMASK_FWD_WINDOW 96
#endif
constexpr int kFE = IMASK_FWD_ENTRIES;  // entries per CTA (4 per warp row, kFE / 4 warp rows)
constexpr int kFThreads = kFE * 32;     // 8 detectors x 4 entries per warp, 32 detectors per CTA
constexpr int kFWc = IMASK_FWD_WINDOW;  // window width in pair columns: the TMA box; the
                                        // window write costs kFWc / (32 kFE) of the reads
constexpr int kFMaxChunks = 1024;  // side up to 8192 (the tables hold the launch's own chunk count)

struct TmaMaps {
  CUtensorMap row, row_m, col, col_m;  // P, PM, PT, PTM of one level
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

struct FwdWarpInfo {
  long long x0_first, x0_last, step;
  int lo, hi;  // union of the lockstep band ranges (lo >= hi: idle)
};

// kQuad: each entry is up to four rays at the same fixed-point positions --
// angle a (row family), its mirror n-a, its transpose partner n/2-a (column
// family: the ray through u at pi/2 - theta is the ray through u^T at theta)
// and that one's mirror n/2+a -- so a CTA stages four windows per chunk (the
// value and difference planes of P and of PT) and every position, weight and
// address is computed once for four rays. Pair mode (kQuad = false): entries
// (a, n-a), one ray family per CTA.
#ifndef IMASK_FWD2_MINB
#define IMASK_FWD2_MINB 4
#endif
#ifndef IMASK_FWD1_MINB
#define IMASK_FWD1_MINB 4  // 64 registers, 4 CTAs per SM: f=1 step -1% (A/B)
#endif
// kK = 2 (value planes, pixel width >= 2): each thread traces two adjacent
// detectors of its entries. Their positions are < 1 column apart (xi_dj =
// 1/(max(|c|,|s|) h) <= 1/sqrt2 for h >= 2), so the second ray's pair column is
// the first's or the next: the three value pairs c, c+1, c+2 serve both rays
// (3 window reads per plane and band instead of 4), and the second ray's
// (value, difference) is selected by the carry -- the same float operations
// as kK = 1, so the sinograms are bit-identical. A CTA covers 64 detectors.
template <bool kSaga, bool kQuad, bool kVal, int kK = 1>
__global__ void __launch_bounds__(kFThreads, kK == 2 ? IMASK_FWD2_MINB : IMASK_FWD1_MINB)
k_forward_tma(const __grid_constant__ TmaMaps maps, const float2* __restrict__ P,
              const float2* __restrict__ PT, const float2* __restrict__ PM,
              const float2* __restrict__ PTM, int n, int pitch, const FwdAngle* __restrict__ ang,
              const int4* __restrict__ entries, int n_entries, int row_ctas, int n_det,
              float* __restrict__ sino, SinoSaga saga, int nch_cap, const int* __restrict__ tab_in,
              int* __restrict__ tab_out) {
  constexpr int FB = kQuad ? (kVal ? kFBQuadVal : kFBQuad) : kFB;  // bands per chunk
  // staged images per chunk: kVal stages only the value planes (P, and PT in
  // quad mode) and forms the difference pair of column c as P[c+1] - P[c], the
  // subtraction k_prepare does for the difference planes (bit-identical sums,
  // half the window bytes and shared memory, two more packed adds per band);
  // otherwise the value and difference planes are staged
  constexpr int NI = (kQuad ? 2 : 1) * (kVal ? 1 : 2);
  constexpr int NR = kQuad ? 4 : 2;          // rays (sinogram rows) per entry
  constexpr int kBox = FB * kFWc;            // float2 per image per stage
  extern __shared__ __align__(128) unsigned char smem[];
  float2* stage = reinterpret_cast<float2*>(smem);  // [2 stages][NI images][FB][kFWc]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * NI * kBox * sizeof(float2));
  uint64_t* empty = full + 2;
  FwdWarpInfo* info = reinterpret_cast<FwdWarpInfo*>(empty + 2);
  int* cmin_tab = reinterpret_cast<int*>(info + kFE);
  int* ctl = cmin_tab + nch_cap;  // [0] overflow, [1] first band, [2] chunks, then cmax_tab

  // A warp holds 4 entries x 8 consecutive detectors (lane = 8 q + d): each
  // half-warp's 8-byte window reads then span ~10 pair columns of one band,
  // never two slots 16 apart (the bank period), so a read is 2 wavefronts
  // where 32 detectors of one angle (up to 45 columns) cost up to 4.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q4 = lane >> 3;
  const int e = blockIdx.y * kFE + (warp >> 2) * 4 + q4;
  const int4 ent = e < n_entries ? entries[e] : make_int4(-1, -1, -1, -1);
  const int rows[4] = {ent.x, ent.y, ent.z, ent.w};
  const int tab = ent.x >= 0 ? ent.x : ent.z;  // the entry's parameter row
  const bool valid = tab >= 0;
  static_assert(kK == 1 || kVal, "two detectors per thread read value planes");
  const int j = blockIdx.x * 32 * kK + (warp & 3) * 8 * kK + (lane & 7) * kK;
  const int jr = min(j, n_det - 1);
  const int j1 = j + 1, jr1 = min(j1, n_det - 1);  // kK = 2: the second detector
  FwdAngle A{};
  if (valid) A = ang[tab];
  SinoIn sin[NR];
  if (kSaga && valid && j < n_det) {  // (kK = 2: the second ray's inputs load at the end)
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (rows[r] >= 0) sin[r] = sino_load(saga, (size_t)rows[r] * n_det + j);
  }
  long long X0 = 0, X1 = 0;
  int lo = n, hi = 0;
  if (valid) {
    X0 = __double2ll_rn(fma((double)jr, A.xi_dj, A.xi_base) * kFix);
    band_range(X0, A.step, A.inv_step, n, &lo, &hi);
    if (lo >= hi) {
      lo = n;
      hi = 0;
    }
    if constexpr (kK == 2) {
      X1 = __double2ll_rn(fma((double)jr1, A.xi_dj, A.xi_base) * kFix);
      int lo1, hi1;
      band_range(X1, A.step, A.inv_step, n, &lo1, &hi1);
      if (lo1 < hi1) {
        lo = min(lo, lo1);
        hi = max(hi, hi1);
      }
    }
  }
  int wlo = lo, whi = hi;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    wlo = min(wlo, __shfl_xor_sync(0xffffffffu, wlo, o));
    whi = max(whi, __shfl_xor_sync(0xffffffffu, whi, o));
  }
  // per entry slot (8 per CTA): positions of its first and last detector and the
  // union of the lockstep band ranges of the four warps holding it (every lane
  // walks its warp's whole range)
  int* cmax_tab = ctl + 4;  // [nch_cap]
  // The chunk tables of a CTA (overflow flag, first band, chunk count, window
  // origin per chunk) depend on the geometry only: they are built once per
  // plan and level by a launch of this kernel with tab_out set (which stops
  // after writing them) and read back here -- the atomics and five of the
  // seven barriers of the prologue go (ncu: the prologue was 10% of the
  // instructions but 27% of the stall samples of the f=8 forward).
  const int tab_stride = nch_cap + 3;
  const size_t cta = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
  if (tab_in) {
    const int* row = tab_in + cta * tab_stride;
    if (threadIdx.x < 3) ctl[threadIdx.x] = row[threadIdx.x];
    const int nrow = min(row[2], nch_cap);
    for (int t = threadIdx.x; t < nrow; t += blockDim.x) cmin_tab[t] = row[3 + t];
  } else {
  if (threadIdx.x < kFE) {
    info[threadIdx.x] = FwdWarpInfo{0, 0, 0, n, 0};
    ctl[0] = 0;
  }
  __syncthreads();
  const int slot = (warp >> 2) * 4 + q4;
  if ((lane & 7) == 0 && valid) {
    FwdWarpInfo& I = info[slot];
    if ((warp & 3) == 0) I.x0_first = X0;
    if ((warp & 3) == 0) I.step = A.step;
    atomicMin(&I.lo, wlo);
    atomicMax(&I.hi, whi);
  }
  {
    const long long x_last = __shfl_sync(0xffffffffu, kK == 2 ? X1 : X0, lane | 7);
    if ((lane & 7) == 0 && valid && (warp & 3) == 3) info[slot].x0_last = x_last;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int blo = n, bhi = 0;
    for (int w = 0; w < kFE; ++w) {
      blo = min(blo, info[w].lo);
      bhi = max(bhi, info[w].hi);
    }
    ctl[1] = blo;
    ctl[2] = bhi > blo ? (bhi - blo + FB - 1) / FB : 0;
    if (ctl[2] > nch_cap) ctl[0] = 1;
  }
  __syncthreads();
  {
  const int blo = ctl[1], nch = ctl[2];
  // window (first pair column) of every chunk: extremes of the affine positions,
  // one (chunk, entry slot) item per thread
  if (!ctl[0]) {
    for (int t = threadIdx.x; t < nch; t += blockDim.x) {
      cmin_tab[t] = INT_MAX;
      cmax_tab[t] = INT_MIN;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < nch * kFE; it += blockDim.x) {
      const int t = it / kFE;
      const FwdWarpInfo& I = info[it % kFE];
      const int b0 = blo + t * FB;
      const int bs = max(b0, I.lo), be = min(b0 + FB, I.hi) - 1;
      if (bs > be) continue;
      const int c0 = (int)((I.x0_first + bs * I.step) >> 32), c1 = (int)((I.x0_first + be * I.step) >> 32),
                c2 = (int)((I.x0_last + bs * I.step) >> 32), c3 = (int)((I.x0_last + be * I.step) >> 32);
      atomicMin(&cmin_tab[t], min(min(c0, c1), min(c2, c3)));
      atomicMax(&cmax_tab[t], max(max(c0, c1), max(c2, c3)));
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nch; t += blockDim.x) {
      int cmn = cmin_tab[t], cmx = cmax_tab[t];
      if (cmn > cmx) cmn = cmx = 0;  // no warp walks this chunk
      // TMA needs a 16-byte aligned start in the inner dimension: even pair index
      const int corig = ((cmn + 1 + kPadC) & ~1) - 1 - kPadC;
      // kVal reads c .. c + 1; kK = 2 reads c .. c + 2 from the first ray's c
      if (cmx + (kVal ? 1 : 0) + (kK == 2 ? 1 : 0) - corig + 1 > kFWc) atomicExch(&ctl[0], 1);
      cmin_tab[t] = corig;
    }
  }
  }
  }  // !tab_in
  __syncthreads();
  const int blo = ctl[1], nch = ctl[2];
  if (tab_out) {
    int* row = tab_out + cta * tab_stride;
    if (threadIdx.x < 3) row[threadIdx.x] = ctl[threadIdx.x];
    const int nrow = min(ctl[2], nch_cap);
    for (int t = threadIdx.x; t < nrow; t += blockDim.x) row[3 + t] = cmin_tab[t];
    return;
  }
  // everything above reads only tables and the solver state; the pair images
  // come from the stream predecessor (k_prepare)
  griddep_wait();
  // pair mode: one ray family per CTA, the row-family CTAs first, so the family
  // (and the tensor-map pointers below) is uniform, derived from blockIdx
  const bool trans = !kQuad && (int)blockIdx.y >= row_ctas;
  // value pairs (u, um) and difference pairs (d, dm) (k_prepare's symmetric
  // layout): (acc, accm) += (u, um) + g * (d, dm) with packed FP32 ops; accT
  // the same for the transpose partners (kQuad)
  float2 acc2 = make_float2(0.f, 0.f), accT = make_float2(0.f, 0.f);
  float2 acc2b = make_float2(0.f, 0.f), accTb = make_float2(0.f, 0.f);  // kK = 2: 2nd ray
  const float S = A.S, B = A.B;
  const Fix32 dX1 = fix_from(X1 - X0);  // kK = 2: second ray's offset (< 1 column)

  if (ctl[0]) {
    // fallback: global (L1) loads over the lane's own band range (a warp holds
    // four entries, whose angles may be far apart in a sparse angle subset:
    // outside its own range a lane's position can leave the zero padding)
    if (valid) {
      const float2* __restrict__ img = trans ? PT : P;
      const float2* __restrict__ imgd = trans ? PTM : PM;
      const long long dYl = A.step + ((long long)pitch << 32);
      Fix32 Y = fix_from(X0 + (long long)lo * dYl + ((long long)(1 + kPadC) << 32));
      const Fix32 dY = fix_from(dYl);
      for (int b = lo; b < hi; ++b) {
        const float g = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
        const float2 v = __ldg(img + Y.hi);
        acc2 = fadd2(acc2, v);
        acc2 = ffma2(g, kVal ? fsub2(__ldg(img + Y.hi + 1), v) : __ldg(imgd + Y.hi), acc2);
        if (kQuad) {
          const float2 vt = __ldg(PT + Y.hi);
          accT = fadd2(accT, vt);
          accT = ffma2(g, kVal ? fsub2(__ldg(PT + Y.hi + 1), vt) : __ldg(PTM + Y.hi), accT);
        }
        fix_add(Y, dY);
      }
      if constexpr (kK == 2) {
        int lo1, hi1;
        band_range(X1, A.step, A.inv_step, n, &lo1, &hi1);
        Fix32 Y1 = fix_from(X1 + (long long)lo1 * dYl + ((long long)(1 + kPadC) << 32));
        for (int b = lo1; b < hi1; ++b) {
          const float g = __saturatef(fmaf(onep_from_frac(Y1.lo), S, B));
          const float2 v = __ldg(img + Y1.hi);
          acc2b = fadd2(acc2b, v);
          acc2b = ffma2(g, fsub2(__ldg(img + Y1.hi + 1), v), acc2b);
          if (kQuad) {
            const float2 vt = __ldg(PT + Y1.hi);
            accTb = fadd2(accTb, vt);
            accTb = ffma2(g, fsub2(__ldg(PT + Y1.hi + 1), vt), accTb);
          }
          fix_add(Y1, dY);
        }
      }
    }
  } else if (nch > 0) {
    const CUtensorMap* mp[4] = {trans ? &maps.col : &maps.row,
                                kVal ? &maps.col : (trans ? &maps.col_m : &maps.row_m), &maps.col,
                                &maps.col_m};
    constexpr uint32_t kTx = NI * kBox * sizeof(float2);
    if (threadIdx.x == 0) {
      mbar_init(&full[0], 1);
      mbar_init(&full[1], 1);
      mbar_init(&empty[0], kFThreads / 32);
      mbar_init(&empty[1], kFThreads / 32);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // producer: warp 0 enters warp-uniformly, one lane issues the bulk tensor copies
    if (warp == 0) {
      if (lane == 0) {
        for (int i = 0; i < 2 && i < nch; ++i) {
          mbar_expect_tx(&full[i], kTx);
          const int col = cmin_tab[i] + 1 + kPadC, row = blo + i * FB;
#pragma unroll
          for (int k = 0; k < NI; ++k)
            tma_load_2d(stage + (i * NI + k) * kBox, mp[k], col, row, &full[i]);
        }
      }
      __syncwarp();
    }
    const Fix32 dYw = fix_from(A.step + ((long long)kFWc << 32));
    for (int i = 0; i < nch; ++i) {
      const int s = i & 1;
      const int b0 = blo + i * FB;
      mbar_wait(&full[s], (i >> 1) & 1);
      const int bs = max(b0, wlo), be = min(b0 + FB, whi);
      if (valid && bs < be) {
        // image k of this stage sits k * kBox elements on; the stage offset
        // rides in the position's integer word
        const float2* win = stage;
        const long long X = X0 + (long long)bs * A.step;
        Fix32 Y = fix_from(X + ((long long)((bs - b0) * kFWc - cmin_tab[i] + s * NI * kBox) << 32));
        int b = bs;
#if IMASK_BOUNDS_CHECK
        // element index relative to the first image of this stage: band row
        // (b - b0), column within [0, kFWc - partners)
        auto chk = [&](const Fix32& y, int band) {
          const long long rel = (long long)y.hi - (long long)s * NI * kBox;
          IMASK_CHECK_RANGE(20, rel - (long long)(band - b0) * kFWc,
                            kFWc - (kVal ? 1 : 0) - (kK == 2 ? 1 : 0));
        };
#else
        auto chk = [](const Fix32&, int) {};
#endif
        if constexpr (kK == 2) {
          // three value pairs per plane feed both rays; the second ray's pair
          // (value, difference) is the first's or the next one's (carry)
          for (; b < be; ++b) {
            chk(Y, b);
            float2 v3[3], t3[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              v3[c] = win[Y.hi + c];
              if (kQuad) t3[c] = win[Y.hi + kBox + c];
            }
            Fix32 Y1 = Y;
            fix_add(Y1, dX1);
            const bool c1 = Y1.hi != Y.hi;
            const float g0 = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
            const float g1 = __saturatef(fmaf(onep_from_frac(Y1.lo), S, B));
            const float2 d0 = fsub2(v3[1], v3[0]), d1 = fsub2(v3[2], v3[1]);
            acc2 = fadd2(acc2, v3[0]);
            acc2 = ffma2(g0, d0, acc2);
            acc2b = fadd2(acc2b, c1 ? v3[1] : v3[0]);
            acc2b = ffma2(g1, c1 ? d1 : d0, acc2b);
            if (kQuad) {
              const float2 e0 = fsub2(t3[1], t3[0]), e1 = fsub2(t3[2], t3[1]);
              accT = fadd2(accT, t3[0]);
              accT = ffma2(g0, e0, accT);
              accTb = fadd2(accTb, c1 ? t3[1] : t3[0]);
              accTb = ffma2(g1, c1 ? e1 : e0, accTb);
            }
            fix_add(Y, dYw);
          }
        }
        for (; kK == 1 && b + 4 <= be; b += 4) {
          float2 v[4], vd[4], vt[4], vdt[4];
          float g[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            chk(Y, b + k);
            v[k] = win[Y.hi];
            if (kVal) {
              vd[k] = win[Y.hi + 1];  // value pair of column c + 1 (difference below)
              if (kQuad) {
                vt[k] = win[Y.hi + kBox];
                vdt[k] = win[Y.hi + kBox + 1];
              }
            } else {
              vd[k] = win[Y.hi + kBox];
              if (kQuad) {
                vt[k] = win[Y.hi + 2 * kBox];
                vdt[k] = win[Y.hi + 3 * kBox];
              }
            }
            g[k] = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
            fix_add(Y, dYw);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (kVal) {
              vd[k] = fsub2(vd[k], v[k]);
              if (kQuad) vdt[k] = fsub2(vdt[k], vt[k]);
            }
            acc2 = fadd2(acc2, v[k]);
            acc2 = ffma2(g[k], vd[k], acc2);
            if (kQuad) {
              accT = fadd2(accT, vt[k]);
              accT = ffma2(g[k], vdt[k], accT);
            }
          }
        }
        for (; kK == 1 && b < be; ++b) {
          chk(Y, b);
          const float g = __saturatef(fmaf(onep_from_frac(Y.lo), S, B));
          const float2 v = win[Y.hi];
          const float2 vd = kVal ? fsub2(win[Y.hi + 1], v) : win[Y.hi + kBox];
          acc2 = fadd2(acc2, v);
          acc2 = ffma2(g, vd, acc2);
          if (kQuad) {
            const float2 vt = win[Y.hi + (kVal ? 1 : 2) * kBox];
            const float2 vdt = kVal ? fsub2(win[Y.hi + kBox + 1], vt) : win[Y.hi + 3 * kBox];
            accT = fadd2(accT, vt);
            accT = ffma2(g, vdt, accT);
          }
          fix_add(Y, dYw);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (warp == 0 && i + 2 < nch) {
        // refill this stage with chunk i+2 once all eight warps have released it
        mbar_wait(&empty[s], (i >> 1) & 1);
        if (lane == 0) {
          mbar_expect_tx(&full[s], kTx);
          const int col = cmin_tab[i + 2] + 1 + kPadC, row = blo + (i + 2) * FB;
#pragma unroll
          for (int k = 0; k < NI; ++k)
            tma_load_2d(stage + (s * NI + k) * kBox, mp[k], col, row, &full[s]);
        }
        __syncwarp();
      }
    }
  }
  if (valid && j < n_det) {
    const float vals[4] = {acc2.x, acc2.y, accT.x, accT.y};
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (rows[r] < 0) continue;
      const float val = vals[r] * A.wsc;
      const size_t q = (size_t)rows[r] * n_det + j;
      if (kSaga) {
        sino_update(saga, q, sin[r], val);
      } else {
        sino[q] = val;
      }
    }
  }
  if (kK == 2 && valid && j1 < n_det) {
    const float vals[4] = {acc2b.x, acc2b.y, accTb.x, accTb.y};
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (rows[r] < 0) continue;
      const float val = vals[r] * A.wsc;
      const size_t q = (size_t)rows[r] * n_det + j1;
      if (kSaga) {
        sino_update(saga, q, sino_load(saga, q), val);
      } else {
        sino[q] = val;
      }
    }
  }
}

int forward_tma_bands(bool quad, bool val) { return quad ? (val ? kFBQuadVal : kFBQuad) : kFB; }

// chunk-table entries a launch on an n-band image needs
static int forward_tma_chunk_cap(int n, bool quad, bool val) {
  const int fb = forward_tma_bands(quad, val);
  const int cap = (n + fb - 1) / fb + 2;
  return cap < kFMaxChunks ? cap : kFMaxChunks;
}

// ints of the per-CTA chunk tables of a level's TMA forward (build: a launch
// of the kernel with tab_out)
bool forward_tma_val(int ctas);
size_t forward_tma_table_len(int n, int n_det, int n_entries, bool quad, bool two_det) {
  const int kk = two_det ? 2 : 1;
  const size_t ctas = (size_t)((n_det + 32 * kk - 1) / (32 * kk)) * ((n_entries + kFE - 1) / kFE);
  const bool val = two_det || forward_tma_val(0);
  return ctas * (size_t)(forward_tma_chunk_cap(n, quad, val) + 3);
}

size_t forward_tma_smem(bool val, bool quad, int nch_cap) {
  // two stages of (1 or 2) x (quad: 2) images of FB bands x kFWc pairs
  const size_t ni = (quad ? 2 : 1) * (val ? 1 : 2);
  return 2 * ni * forward_tma_bands(quad, val) * kFWc * sizeof(float2) + 4 * sizeof(uint64_t) +
         kFE * sizeof(FwdWarpInfo) + (2 * (size_t)nch_cap + 4) * sizeof(int);
}

namespace {
int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}
}  // namespace

// Value-plane staging (kVal): its CTAs take half the shared memory, so they
// co-reside with the concurrent adjoint's (f=1 step 932 -> 907 us on one GPU)
// while the projection alone runs as fast. On a small grid (an angle shard: a
// fraction of a wave, latency-bound along each CTA's band walk) the extra
// packed subtractions make the projection alone slower (1/4 shard's f=1
// forward 169 -> 188 us), but with the fused staging x -> value planes
// (k_stage32) the shard steps are faster too (f=1 step: 1/8 shard 167.5 ->
// 161.3 us on rank 0, 148.8 -> 138.7 us on rank 7; 1/4 shard 270 -> 262 us),
// so every grid stages value planes (IMASK_FWD_VAL=0: both planes).
bool forward_tma_val(int ctas) {
  (void)ctas;
  const int forced = knob(Knob::kFwdVal, -1);
  if (forced == 0 || forced == 1) return forced == 1;
  return true;
}

bool forward_tma_val_grid(int n_det, int n_entries) {
  return forward_tma_val(((n_det + 31) / 32) * ((n_entries + kFE - 1) / kFE));
}

cudaError_t launch_forward_tma(const TmaMaps& maps, const float2* P, const float2* PT,
                               const float2* PM, const float2* PTM, int n, const FwdAngle* ang,
                               const int4* entries, int n_entries, int row_ctas, bool quad,
                               int n_det, float* sino, const SinoSaga* saga, cudaStream_t stream,
                               bool two_det, const int* tab_in, int* tab_out) {
  const int kk = two_det ? 2 : 1;
  dim3 grid((n_det + 32 * kk - 1) / (32 * kk), (n_entries + kFE - 1) / kFE);
  const bool val = two_det || forward_tma_val((int)(grid.x * grid.y));
  const int cap = forward_tma_chunk_cap(n, quad, val);
  const size_t smem = forward_tma_smem(val, quad, cap);
  SinoSaga none{};
  const SinoSaga sg = saga ? *saga : none;
  float* out = saga ? nullptr : sino;
#define FWD_TMA(S_, Q_, V_, K_)                                                                  \
  launch_pdl(k_forward_tma<S_, Q_, V_, K_>, grid, dim3(kFThreads), smem, stream, maps, P, PT, PM, \
             PTM, n, pair_pitch(n), ang, entries, n_entries, row_ctas, n_det, out, sg, cap, tab_in, \
             tab_out)
#define FWD_TMA_V(S_, Q_)                                 \
  if (two_det) FWD_TMA(S_, Q_, true, 2);                  \
  else if (val) FWD_TMA(S_, Q_, true, 1);                 \
  else FWD_TMA(S_, Q_, false, 1)
  if (saga) {
    if (quad) { FWD_TMA_V(true, true); } else { FWD_TMA_V(true, false); }
  } else {
    if (quad) { FWD_TMA_V(false, true); } else { FWD_TMA_V(false, false); }
  }
#undef FWD_TMA_V
#undef FWD_TMA
  return cudaGetLastError();
}

// ---- adjoint -----------------------------------------------------------------
//
// Pixel-driven gather, no atomics. A CTA owns a T x T pixel tile and a range of
// angles (grid.z splits the angles when the level has few tiles; the per-split
// partial images are then summed in a fixed order by k_adjoint_reduce, so the
// result is deterministic). For each chunk of angles the CTA stages, per angle,
// the W-bin window of the sinogram the tile's footprint can touch, pre-scaled
// by that angle's chord scale. Pixel positions are Q32.32 fixed point whose
// integer word is the window slot: exact integer increments per column/row,
// so ties on gridlines (axis-parallel rays, integer detector offsets) are
// decided exactly, and 1 + frac is one LEA.HI away from the fraction word.
//
// With v = eta - R - window base for a pixel, the candidate bins are
// floor(v)+1 .. floor(v)+nb and bin b has offset u_b = (2 - R + b) - onep,
// onep = 1 + frac(v); oblique weights are sat(|u| * kneg + Rk) (the trapezoid),
// axis-parallel angles use v - 2^-32 (ceil rule of the half-open box) and
// constant weights (kneg = 0, Rk = 1 for the h bins of the box).

constexpr int kAdjThreads = 128;
// pixels per thread (one column of a tile): 8 where the per-angle setup must be
// amortised (factors 1-4), 2 at coarse factors where the bin loop dominates
// and small angle chunks keep the large windows within shared memory

struct AdjStage {
  long long E0;     // Q32.32 of v at the tile origin (minus one ulp for axis angles), integer
                    // word offset by this angle's window slot base t*W
  long long Dc, Ds;
  long long estep;  // Ds * (rows between a thread's pixels)
  float c0;         // 2 - R
  float kneg, Rk;   // trapezoid weight: sat(|u| * kneg + Rk)
  float k1a, k1b;   // factor-1 path: w1 = sat(onep * k1a + k1b)
  int nb;           // candidate bins per pixel
  int axis;
  int jb;           // window slot 0 holds detector bin jb
  float wsc;
};

__device__ __forceinline__ float onep32(uint32_t frac) {
  return __uint_as_float(0x3F800000u + (frac >> 9));
}

template <bool kPair, bool kSym>
struct AdjWin;  // staged window element: bins (k, k+1) for the pair path, rows (a, n-a) for kSym
template <> struct AdjWin<false, false> { using T = float; };
template <> struct AdjWin<false, true> { using T = float2; };
template <> struct AdjWin<true, false> { using T = float2; };
template <> struct AdjWin<true, true> { using T = float4; };

// kPair: factor-1 path (two bins per pixel, T = 32).
// T: tile side; lanes = T*T/8 threads share one angle, G = 128/lanes angle groups.
// kSym (mirror symmetry, full angle set of even size): the grid covers the
// left half of the image; pixel p = (col,row) at angle a has the same detector
// bins and weights as its mirror m(p) = (n-1-col,row) at angle n-a (theta ->
// pi-theta, x -> -x), so each weight evaluation accumulates into both pixels,
// reading rows a and n-a from one staged window element. Angle 0 is excluded
// from the loop (the half-open tie rule flips under the mirror); its box is
// added per pixel in the epilogue (add_a0). Angles [a_begin, a_end) are split
// over grid.z, a thread-block cluster of cz splits reduces on chip, and plane
// z / cz of `out` receives the cluster's partial image.
// Pixel k of thread slot p (0 <= p < lanes) within a T x T tile. The lanes of
// a warp cover a compact 8 x 4 pixel block at every k, so one window read
// touches few distinct bins (ideally ~8|cos| + 4|sin| + 1 slots, many lanes
// broadcast) instead of a 32-pixel row's ~32:
//   T = 32 (lanes 128): fixed column 8*warp + 4*half + p%4, rows (p/4)%4 + 4k
//   T = 16 (lanes 32) : columns 4*half + p%4 + 8*(k&1), rows (p/4)%4 + 4*(k>>1)
//   T = 8  (lanes 32) : column 4*half + p%4, rows (p/4)%4 + 4k
template <int T>
__device__ __forceinline__ void adj_pixel(int p, int k, int& dx, int& dy) {
  // (each half-warp is a 4 x 4 sub-block, whose window reads stay within one
  // bank period at factors 2 and 4)
  if constexpr (T == 32) {
    dx = ((p >> 5) << 3) + (((p >> 4) & 1) << 2) + (p & 3);
    dy = ((p >> 2) & 3) + 4 * k;
  } else if constexpr (T == 16) {
    dx = (((p >> 4) & 1) << 2) + (p & 3) + 8 * (k & 1);
    dy = ((p >> 2) & 3) + 4 * (k >> 1);
  } else {
    dx = (((p >> 4) & 1) << 2) + (p & 3);
    dy = ((p >> 2) & 3) + 4 * k;
  }
}

// Angle 0 (cos = 1, sin = 0) at pixel (row, col): the half-open box covers the
// bins ceil(v) .. ceil(v) + nb - 1, v = eta - R (exact in double: half-integers),
// each with weight 1 -- the kernel's axis rule, summed in bin order.
__device__ __forceinline__ float angle0_value(const float* __restrict__ sino, const AdjAngle& A,
                                              int row, int col, int n_det) {
  const int j0 = (int)ceil(A.eta0 + (double)col * A.ch + (double)row * A.sh);
  float v = 0.f;
  for (int b = 0; b < A.nb; ++b) {
    const int j = j0 + b;
    if (j >= 0 && j < n_det) v += __ldg(sino + j) * A.wsc;
  }
  return v;
}

#ifndef IMASK_ADJ_STAGE_NB
#define IMASK_ADJ_STAGE_NB 2
#endif
#ifndef IMASK_ADJ_PAIR_MINB
#define IMASK_ADJ_PAIR_MINB 7  // factor 1: 72 registers with two angles staged per round
#endif
#ifndef IMASK_ADJ_SYM_MINB
#define IMASK_ADJ_SYM_MINB 8  // 64 registers: f=1 adjoint 514.7 -> 512.4 us, f=8 80.3 -> 78.4 us, every step -0.2..-1% (A/B, two rounds)
#endif
// kRP (row pairs; factor 1, mirror symmetry, T = 32): a thread's eight pixels
// are four pairs of vertically adjacent pixels. At f = 1 the lower pixel's
// footprint sits sin(theta) in [0, 1] bins further on (angles in [0, pi)),
// so its two bins are the upper pixel's two or the next two: one window of
// single bins (y_a[k], y_{n-a}[k]) read at k, k+1, k+2 feeds both pixels
// and their mirrors (3 LDS.64 per pixel pair and angle instead of 2 LDS.128)
// with packed FMAs, the same float operations in the same order as the
// pair path, so the backprojection is bit-identical.
template <int T, bool kRP>
__device__ __forceinline__ void adj_pix(int p, int k, int& dx, int& dy) {
  if constexpr (kRP) {
    dx = ((p >> 5) << 3) + (((p >> 4) & 1) << 2) + (p & 3);
    dy = 2 * (((p >> 2) & 3) + 4 * (k >> 1)) + (k & 1);
  } else {
    adj_pixel<T>(p, k, dx, dy);
  }
}

template <bool kPair, int T, bool kSym, int kPPT, bool kRP = false>
__global__ void __launch_bounds__(kAdjThreads, kSym ? (kPair ? IMASK_ADJ_PAIR_MINB : IMASK_ADJ_SYM_MINB) : 8)
k_adjoint(const float* __restrict__ sino, float* __restrict__ out, int n, int W, int CA,
          int a_begin, int a_per_split, int a_end, int n_mirror, int n_det,
          const AdjAngle* __restrict__ ang, int add_a0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  static_assert(!kRP || (kPair && kSym && T == 32 && kPPT == 8), "row pairs: f = 1 symmetric");
  using WinT = typename AdjWin<kPair && !kRP, kSym>::T;
  constexpr int lanes = T * T / kPPT;
  constexpr int G = kAdjThreads / lanes;
  static_assert(lanes == (T == 32 ? 128 : 32), "adj_pixel layout");
  constexpr int NACC = kSym ? 2 : 1;
  AdjStage* st = reinterpret_cast<AdjStage*>(smem_raw);
  float* red = reinterpret_cast<float*>(st + CA);
  WinT* win = reinterpret_cast<WinT*>(red + kAdjThreads * kPPT * NACC);

  const int tid = threadIdx.x;
  const int grp = tid / lanes;
  const int pix0 = tid % lanes;
  const int x0 = blockIdx.x * T, y0 = blockIdx.y * T;
  const int a_lo = a_begin + blockIdx.z * a_per_split;
  const int a_hi = min(a_end, a_lo + a_per_split);
  int dx, dy;
  adj_pix<T, kRP>(pix0, 0, dx, dy);
  const int warp = tid >> 5, lane = tid & 31;
  float acc[NACC][kPPT];
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int k = 0; k < kPPT; ++k) acc[q][k] = 0.f;

  for (int a0 = a_lo; a0 < a_hi; a0 += CA) {
    const int na = min(CA, a_hi - a0);
    __syncthreads();
    for (int t = tid; t < na; t += kAdjThreads) {
      const AdjAngle A = ang[a0 + t];
      const double eta = A.eta0 + (double)x0 * A.ch + (double)y0 * A.sh;  // eta - R at origin
      const double emin = eta + fmin(0.0, (T - 1) * A.ch) + fmin(0.0, (T - 1) * A.sh);
      const int jb = (int)floor(emin) - 1;
      AdjStage s;
      s.E0 = __double2ll_rn((eta - (double)jb) * kFix) - (A.axis ? 1 : 0) +
             ((long long)(t * W) << 32);
      s.Dc = A.Dc;
      s.Ds = A.Ds;
      s.estep = 4 * A.Ds;  // next pixel of a thread: 4 rows down (T = 16: see estep2)
      s.c0 = 2.0f - A.R;
      s.axis = A.axis;
      if (A.axis) {
        s.kneg = 0.f;
        s.Rk = 1.f;
        s.k1a = 0.f;
        s.k1b = 0.f;  // factor 1: the box holds one bin
      } else {
        s.kneg = A.kneg;
        s.Rk = A.Rk;
        // factor 1: u1 = (3 - R) - onep > 0, so w1 = sat(onep * (-kneg) + Rk + kneg * (3 - R))
        s.k1a = -A.kneg;
        s.k1b = A.Rk + A.kneg * (3.0f - A.R);
      }
      s.nb = A.nb;
      s.jb = jb + 1;
      s.wsc = A.wsc;
      st[t] = s;
    }
    __syncthreads();
    // stage windows (one warp per angle): W bins scaled by wsc, zero outside the detector
    constexpr int kNL = (kPair && !kRP ? 2 : 1) * (kSym ? 2 : 1);  // global loads per window element
    auto interior = [&](int t) { return st[t].jb >= 0 && st[t].jb + W + 1 <= n_det; };
    // one element of an interior window: its loads (l), then the scaled element
    auto load_elem = [&](const float* yp, const float* mp, unsigned k, float (&l)[kNL]) {
      l[0] = __ldg(yp + k);
      if constexpr (kRP) {
        l[1] = __ldg(mp + k);
      } else if constexpr (kPair && kSym) {
        l[1] = __ldg(yp + k + 1);
        l[2] = __ldg(mp + k);
        l[3] = __ldg(mp + k + 1);
      } else if constexpr (kPair) {
        l[1] = __ldg(yp + k + 1);
      } else if constexpr (kSym) {
        l[1] = __ldg(mp + k);
      }
    };
    auto store_elem = [&](WinT* wt, unsigned k, const float (&l)[kNL], float wsc) {
      if constexpr (kNL == 4) {
        wt[k] = make_float4(l[0] * wsc, l[1] * wsc, l[2] * wsc, l[3] * wsc);
      } else if constexpr (kNL == 2) {
        wt[k] = make_float2(l[0] * wsc, l[1] * wsc);
      } else {
        wt[k] = l[0] * wsc;
      }
    };
    for (int t = warp; t < na; t += kAdjThreads / 32) {
      const int jb = st[t].jb;
      const float wsc = st[t].wsc;
      const float* yrow = sino + (size_t)(a0 + t) * n_det;
      const float* mrow = sino + (size_t)(kSym ? n_mirror - (a0 + t) : 0) * n_det;
      if constexpr (!kPair) {
        if (interior(t)) {
          // window inside the detector (almost every tile and angle): no edge
          // tests, 32-bit offsets from two per-angle pointers (the tested loop
          // below spends ~35 instructions per 32 bins, mostly on predicates and
          // 64-bit addresses)
          const float* yp = yrow + jb;
          const float* mp = mrow + jb;
          WinT* wt = win + t * W;
#pragma unroll 4
          for (unsigned k = lane; k < (unsigned)W; k += 32) {
            const float v0 = __ldg(yp + k) * wsc;
            if constexpr (kSym) {
              wt[k] = make_float2(v0, __ldg(mp + k) * wsc);
            } else {
              wt[k] = v0;
            }
          }
          continue;
        }
      } else if (interior(t)) {
        // window inside the detector (almost every tile and angle): no edge
        // tests, 32-bit offsets from two per-angle pointers. Two angles of this
        // warp go together, two lane-chunks of each per round: up to 4 kNL
        // independent loads are in flight before the first is used (ncu's
        // source page of the f=1 kernel: the multiplies waiting on these loads
        // held 11% of all stall samples, staging 30% with 12% of the
        // instructions).
        // (factor-1 kernel only, at 72 registers: f=1 adjoint 513 -> 505 us; the
        // coarse kernels got slower with it -- f=4 115 -> 118 us, f=16 54 -> 62 us --
        // and keep one angle and one lane-chunk per round)
        // kNB consecutive angles of this warp (t, t + 4, ...) go together while
        // they are interior
        constexpr int kNB = IMASK_ADJ_STAGE_NB;
        constexpr int kStep = kAdjThreads / 32;
        int nbat = 1;
        while (nbat < kNB && t + nbat * kStep < na && interior(t + nbat * kStep)) ++nbat;
        const float* ypb[kNB];
        const float* mpb[kNB];
        float wscb[kNB];
#pragma unroll
        for (int q = 0; q < kNB; ++q) {
          const int tq = t + (q < nbat ? q : 0) * kStep;
          const int jq = st[tq].jb;
          ypb[q] = sino + (size_t)(a0 + tq) * n_det + jq;
          mpb[q] = sino + (size_t)(kSym ? n_mirror - (a0 + tq) : 0) * n_det + jq;
          wscb[q] = st[tq].wsc;
        }
        for (unsigned k = lane; k < (unsigned)W; k += 64) {
          float la[kNB][kNL], lb[kNB][kNL];
          const bool more = k + 32 < (unsigned)W;
#pragma unroll
          for (int q = 0; q < kNB; ++q)
            if (q < nbat) {
              load_elem(ypb[q], mpb[q], k, la[q]);
              if (more) load_elem(ypb[q], mpb[q], k + 32, lb[q]);
            }
#pragma unroll
          for (int q = 0; q < kNB; ++q)
            if (q < nbat) {
              WinT* wq = win + (t + q * kStep) * W;
              store_elem(wq, k, la[q], wscb[q]);
              if (more) store_elem(wq, k + 32, lb[q], wscb[q]);
            }
        }
        t += (nbat - 1) * kStep;  // those angles are done
        continue;
      }
      for (int k = lane; k < W; k += 32) {
        const int j = jb + k;
        const bool in0 = j >= 0 && j < n_det, in1 = j + 1 >= 0 && j + 1 < n_det;
        const float v0 = in0 ? __ldg(yrow + j) * wsc : 0.f;
        if constexpr (kRP) {
          win[t * W + k] = make_float2(v0, in0 ? __ldg(mrow + j) * wsc : 0.f);
        } else if constexpr (kPair && kSym) {
          win[t * W + k] = make_float4(v0, in1 ? __ldg(yrow + j + 1) * wsc : 0.f,
                                       in0 ? __ldg(mrow + j) * wsc : 0.f,
                                       in1 ? __ldg(mrow + j + 1) * wsc : 0.f);
        } else if constexpr (kPair) {
          win[t * W + k] = make_float2(v0, in1 ? __ldg(yrow + j + 1) * wsc : 0.f);
        } else if constexpr (kSym) {
          win[t * W + k] = make_float2(v0, in0 ? __ldg(mrow + j) * wsc : 0.f);
        } else {
          win[t * W + k] = v0;
        }
      }
    }
    __syncthreads();
    if constexpr (kRP) {
      const float2* win2 = reinterpret_cast<const float2*>(win);
#pragma unroll 2
      for (int t = 0; t < na; ++t) {
        const AdjStage s = st[t];
        Fix32 e = fix_from(s.E0 + (long long)dx * s.Dc + (long long)dy * s.Ds);
        const Fix32 estep = fix_from(8 * s.Ds);  // next pair: 8 rows down
        const Fix32 eds = fix_from(s.Ds);        // the lower pixel: one row down
#pragma unroll
        for (int k2 = 0; k2 < kPPT / 2; ++k2) {
          IMASK_CHECK_RANGE(32, (long long)e.hi - (long long)t * W, W - 2);
          const float2 v0 = win2[e.hi], v1 = win2[e.hi + 1], v2 = win2[e.hi + 2];
          Fix32 eb = e;
          fix_add(eb, eds);
          const bool cy = eb.hi != e.hi;
          const float oa = onep32(e.lo), ob = onep32(eb.lo);
          const float w0a = __saturatef(fmaf(fabsf(s.c0 - oa), s.kneg, s.Rk));
          const float w1a = __saturatef(fmaf(oa, s.k1a, s.k1b));
          const float w0b = __saturatef(fmaf(fabsf(s.c0 - ob), s.kneg, s.Rk));
          const float w1b = __saturatef(fmaf(ob, s.k1a, s.k1b));
          float2 pa = make_float2(acc[0][2 * k2], acc[1][2 * k2]);
          float2 pb = make_float2(acc[0][2 * k2 + 1], acc[1][2 * k2 + 1]);
          pa = ffma2(w0a, v0, pa);
          pa = ffma2(w1a, v1, pa);
          pb = ffma2(w0b, cy ? v1 : v0, pb);
          pb = ffma2(w1b, cy ? v2 : v1, pb);
          acc[0][2 * k2] = pa.x;
          acc[1][2 * k2] = pa.y;
          acc[0][2 * k2 + 1] = pb.x;
          acc[1][2 * k2 + 1] = pb.y;
          fix_add(e, estep);
        }
      }
    } else if constexpr (kPair) {
#pragma unroll 2
      for (int t = 0; t < na; ++t) {
        const AdjStage s = st[t];
        Fix32 e = fix_from(s.E0 + (long long)dx * s.Dc + (long long)dy * s.Ds);
        const Fix32 estep = fix_from(s.estep);
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
          IMASK_CHECK_RANGE(30, (long long)e.hi - (long long)t * W, W);
          const WinT pr = win[e.hi];
          const float onep = onep32(e.lo);
          const float w0 = __saturatef(fmaf(fabsf(s.c0 - onep), s.kneg, s.Rk));
          const float w1 = __saturatef(fmaf(onep, s.k1a, s.k1b));
          acc[0][k] = fmaf(w0, pr.x, acc[0][k]);
          acc[0][k] = fmaf(w1, pr.y, acc[0][k]);
          if constexpr (kSym) {
            acc[NACC - 1][k] = fmaf(w0, pr.z, acc[NACC - 1][k]);
            acc[NACC - 1][k] = fmaf(w1, pr.w, acc[NACC - 1][k]);
          }
          fix_add(e, estep);
        }
      }
    } else {
      for (int t = grp; t < na; t += G) {
        const AdjStage s = st[t];
        Fix32 e = fix_from(s.E0 + (long long)dx * s.Dc + (long long)dy * s.Ds);
        // T = 16 alternates +8 columns / (-8 columns, +4 rows) between pixels
        const Fix32 estep = fix_from(T == 16 ? 8 * s.Dc : s.estep);
        const Fix32 estep2 = fix_from(s.estep - 8 * s.Dc);
        // bins outer, pixels inner: independent accumulation chains
        int base[kPPT];
        float u[kPPT];
#pragma unroll
        for (int k = 0; k < kPPT; ++k) {
          base[k] = (int)e.hi;
          IMASK_CHECK_RANGE(31, (long long)e.hi - (long long)t * W, W - s.nb + 1);
          u[k] = s.c0 - onep32(e.lo);
          fix_add(e, (T == 16 && (k & 1)) ? estep2 : estep);
        }
        auto bin = [&](int b) {
#pragma unroll
          for (int k = 0; k < kPPT; ++k) {
            const float w = __saturatef(fmaf(fabsf(u[k]), s.kneg, s.Rk));
            const WinT v = win[base[k] + b];
            if constexpr (kSym) {
              acc[0][k] = fmaf(w, v.x, acc[0][k]);
              acc[NACC - 1][k] = fmaf(w, v.y, acc[NACC - 1][k]);
            } else {
              acc[0][k] = fmaf(w, v, acc[0][k]);
            }
            u[k] += 1.0f;
          }
        };
        if (s.nb == 3) {
          // factor 2 (every oblique angle has 3 candidate bins): fully unrolled,
          // the bin offsets become immediate offsets of the window reads
#pragma unroll
          for (int b = 0; b < 3; ++b) bin(b);
        } else {
          for (int b = 0; b < s.nb; ++b) bin(b);
        }
      }
    }
  }
  // Epilogue. Value i = (q * kPPT + k) * lanes + p of this CTA's tile (q: the
  // pixel or its mirror, k: the thread's k-th pixel, p: the lane slot). With a
  // thread-block cluster along grid.z (the angle splits of one tile), the
  // cluster's CTAs put their tiles in shared memory and each sums a slice of
  // the pixels over the cluster ranks in rank order (DSMEM reads), so one
  // plane per cluster is written instead of one per split (deterministic).
  // Angle 0 (unpaired under the mirror, add_a0) is added on plane 0.
  cg::cluster_group cluster = cg::this_cluster();
  const int cz = (int)cluster.num_blocks();
  float* dst = out + (size_t)(blockIdx.z / cz) * n * n;
  const bool a0 = add_a0 && blockIdx.z < (unsigned)cz;
  auto store = [&](int i, float v) {
    const int q = i / (lanes * kPPT), r = i % (lanes * kPPT);
    int px, py;
    adj_pix<T, kRP>(r % lanes, r / lanes, px, py);
    const int row = y0 + py;
    const int col = q == 0 ? x0 + px : n - 1 - (x0 + px);
    if (row < n && col >= 0 && col < n) {
      if (a0) v += angle0_value(sino, ang[0], row, col, n_det);
      dst[(size_t)row * n + col] = v;
    }
  };
  constexpr int kVals = NACC * lanes * kPPT;
  float* tb = reinterpret_cast<float*>(win);  // the windows are dead after the angle loop
  __syncthreads();
  if (G > 1) {
    // fixed-order sum over the angle groups
#pragma unroll
    for (int q = 0; q < NACC; ++q)
#pragma unroll
      for (int k = 0; k < kPPT; ++k)
        red[((q * G + grp) * kPPT + k) * lanes + pix0] = acc[q][k];
    __syncthreads();
    for (int i = tid; i < kVals; i += kAdjThreads) {
      const int q = i / (lanes * kPPT), r = i % (lanes * kPPT);
      const int k = r / lanes, p = r % lanes;
      float v = 0.f;
      for (int g = 0; g < G; ++g) v += red[((q * G + g) * kPPT + k) * lanes + p];
      if (cz > 1) tb[i] = v; else store(i, v);
    }
  } else {
#pragma unroll
    for (int q = 0; q < NACC; ++q)
#pragma unroll
      for (int k = 0; k < kPPT; ++k) {
        const int i = (q * kPPT + k) * lanes + pix0;
        if (cz > 1) tb[i] = acc[q][k]; else store(i, acc[q][k]);
      }
  }
  if (cz > 1) {
    cluster.sync();
    const int chunk = (kVals + cz - 1) / cz;
    const int lo = (int)cluster.block_rank() * chunk;
    const int hi = min(kVals, lo + chunk);
    for (int i = lo + tid; i < hi; i += kAdjThreads) {
      float v = 0.f;
      for (int rk = 0; rk < cz; ++rk) v += cluster.map_shared_rank(tb, rk)[i];
      store(i, v);
    }
    cluster.sync();  // keep this CTA's tile alive until every rank has read it
  }
}

// Many planes, few pixels (coarse levels): a warp per pixel, lane l sums
// planes l, l+32, ... and a fixed xor tree combines the lanes (deterministic).
__global__ void k_adjoint_reduce_warp(const float* __restrict__ part, float* __restrict__ out,
                                      int npix, int S) {
  griddep_wait();
  const int p = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= npix) return;
  float v = 0.f;
  for (int s = lane; s < S; s += 32) v += __ldg(part + (size_t)s * npix + p);
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) out[p] = v;
}

// Sum of the per-split partial images in split order (deterministic).
__global__ void k_adjoint_reduce(const float* __restrict__ part, float* __restrict__ out,
                                 int npix, int S) {
  griddep_wait();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  float v = 0.f;
  for (int s = 0; s < S; ++s) v += __ldg(part + (size_t)s * npix + p);
  out[p] = v;
}

// ---- launchers ----------------------------------------------------------

// The L1 quad forward forms the difference pairs from the value planes: half
// the L1 footprint (f=16 step 93.5 -> 91.5 us on one GPU).
bool forward_l1_val() {
  return knob(Knob::kFwdValL1, 1) == 1;
}

cudaError_t launch_forward(const float2* P, const float2* PT, const float2* PM, const float2* PTM,
                           int n, const FwdAngle* ang, int n_loc, int n_det,
                           const int2* sym_entries, int n_entries, const int4* quad_entries,
                           int n_quad_entries, float* sino, const SinoSaga* saga,
                           cudaStream_t stream) {
  SinoSaga none{};
  if (quad_entries) {
    dim3 grid((n_det + 31) / 32, (n_quad_entries + 7) / 8);
    const bool val = forward_l1_val();
#define FWD_QUAD(S_, V_, OUT_, SG_)                                                        \
  launch_pdl(k_forward_quad<S_, V_>, grid, dim3(256), 0, stream, P, PT, PM, PTM, n, pair_pitch(n), \
             ang, quad_entries, n_quad_entries, n_det, OUT_, SG_)
    if (saga) {
      if (val) FWD_QUAD(true, true, (float*)nullptr, *saga); else FWD_QUAD(true, false, (float*)nullptr, *saga);
    } else {
      if (val) FWD_QUAD(false, true, sino, none); else FWD_QUAD(false, false, sino, none);
    }
#undef FWD_QUAD
    return cudaGetLastError();
  }
  if (sym_entries) {
    dim3 grid((n_det + 31) / 32, (n_entries + 7) / 8);
    if (saga)
      launch_pdl(k_forward_sym<true>, grid, dim3(256), 0, stream, P, PT, PM, PTM, n,
                 pair_pitch(n), ang, sym_entries, n_entries, n_det, (float*)nullptr, *saga);
    else
      launch_pdl(k_forward_sym<false>, grid, dim3(256), 0, stream, P, PT, PM, PTM, n,
                 pair_pitch(n), ang, sym_entries, n_entries, n_det, sino, none);
    return cudaGetLastError();
  }
  dim3 grid((n_det + 31) / 32, (n_loc + 7) / 8);
  if (saga) {
    k_forward<true><<<grid, 256, 0, stream>>>(P, PT, n, pair_pitch(n), ang, n_loc, n_det, nullptr,
                                              *saga);
  } else {
    k_forward<false><<<grid, 256, 0, stream>>>(P, PT, n, pair_pitch(n), ang, n_loc, n_det, sino,
                                               none);
  }
  return cudaGetLastError();
}

// Opt-in shared memory beyond 48 KB (called once per device at plan creation,
// outside any stream capture).
void init_kernel_attributes() {
#define FWD_ATTR(S_, Q_, V_)                                                                  \
  cudaFuncSetAttribute(k_forward_tma<S_, Q_, V_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       (int)forward_tma_smem(V_, Q_, kFMaxChunks))
  FWD_ATTR(true, false, false);
  FWD_ATTR(false, false, false);
  FWD_ATTR(true, true, false);
  FWD_ATTR(false, true, false);
  FWD_ATTR(true, false, true);
  FWD_ATTR(false, false, true);
  FWD_ATTR(true, true, true);
  FWD_ATTR(false, true, true);
#undef FWD_ATTR
#define FWD_ATTR2(S_, Q_)                                                                    \
  cudaFuncSetAttribute(k_forward_tma<S_, Q_, true, 2>,                                       \
                       cudaFuncAttributeMaxDynamicSharedMemorySize,                            \
                       (int)forward_tma_smem(true, Q_, kFMaxChunks))
  FWD_ATTR2(true, true);
  FWD_ATTR2(false, true);
  FWD_ATTR2(true, false);
  FWD_ATTR2(false, false);
#undef FWD_ATTR2
#define ADJ_ATTR(P_, T_, S_, K_)                                                          \
  cudaFuncSetAttribute(k_adjoint<P_, T_, S_, K_>,                                        \
                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
  cudaFuncSetAttribute(k_adjoint<true, 32, true, 8, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  ADJ_ATTR(true, 32, false, 8);
  ADJ_ATTR(true, 32, true, 8);
  ADJ_ATTR(false, 32, false, 8);
  ADJ_ATTR(false, 32, true, 8);
  ADJ_ATTR(false, 16, false, 8);
  ADJ_ATTR(false, 16, true, 8);
  ADJ_ATTR(false, 8, false, 2);
  ADJ_ATTR(false, 8, true, 2);
#undef ADJ_ATTR
}

// Tile / split choice of the adjoint at one level (shared with the plan's
// scratch sizing): T = 32 at factors 1-2, 16 at factors 4-8 and, for plans of
// >= 512 angles, 16; else 8;
// T shrinks to the next power of two >= n (>= 8) for small images. The angle
// splits S give the grid ~16-28 CTAs per SM; with mirror symmetry (sym) the
// grid covers half the tiles. Splits are grouped into thread-block clusters of
// cz (<= 8, S a multiple of cz) that reduce their partial tiles on chip, so
// the level writes S / cz planes.
void adjoint_layout(int n, int factor, int n_loc, bool sym, int* T_out, int* S_out,
                    int* cz_out = nullptr) {
  // (measured beside the value-plane forward: 16 at f = 8 -> step -4% on the
  // whole set and on shards; 16 at f = 16 -> -1..2% on the whole set, slower
  // on 1/4 and 1/8 shards, which keep 8; at f = 32 16 is faster with the L2
  // warm (60.5 -> 54.8 us) but slower after an L2 flush (67 -> 70 us), so 8)
  int T = factor <= 2 ? 32 : (factor <= 8 || (factor <= 16 && n_loc >= 512) ? 16 : 8);
  {
    const int tt = knob_for_factor(Knob::kAdjTile, factor, T);
    if (tt == 8 || tt == 16 || tt == 32) T = tt;
  }
  int np2 = 8;
  while (np2 < n) np2 <<= 1;
  if (T > np2) T = np2;
  int tiles = ((n + T - 1) / T) * ((n + T - 1) / T);
  if (sym) tiles /= 2;
  // angle splits: ~16-20 CTAs per SM. (At f >= 16 a lighter grid, ~4 per SM,
  // makes an L2-warm step faster by leaving room for the concurrent forward
  // chain, but a cold-L2 step slower: the windows' HBM latency needs the CTAs.)
  // (factor 1 with many angles: 28 per SM, measured -1% on the whole-set step
  // with the value-plane forward beside it; a 1/4 or 1/8 shard is slower so)
  // (factor 2 on plans of >= 512 angles: 24 per SM, f=2 step 377 -> 373 us)
  int per_sm = factor == 1 ? (n_loc >= 512 ? 28 : 20) : (factor == 2 && n_loc >= 512 ? 24 : 16);
  {
    const int cc = knob_for_factor(Knob::kAdjCtas, factor, per_sm);
    if (cc > 0) per_sm = cc;
  }
  const int target = per_sm * sm_count();
  int S = (target + tiles - 1) / tiles;
  const int max_s = n_loc / 8 > 1 ? n_loc / 8 : 1;
  if (S > max_s) S = max_s;
  if (S < 1) S = 1;
  // Clusters measured slower at every level of config D (f=1 adjoint 515 ->
  // 549 us with clusters of 8, f=4 118 -> 144 us; 2 and 4 in between): the
  // co-scheduling of a cluster's CTAs costs more SM time than the plane
  // round trip through L2 saves, so the default is no cluster (A/B knob).
  const int cz_knob = knob(Knob::kAdjCluster, 1);
  const int cz_max = cz_knob < 1 ? 1 : (cz_knob > 8 ? 8 : cz_knob);
  const int cz = S < cz_max ? S : cz_max;
  S = (S / cz) * cz;
  *T_out = T;
  *S_out = S;
  if (cz_out) *cz_out = cz;
}

// Mirror symmetry applies when the slab is the whole, even-sized angle set and
// the left half of the image is a whole number of tiles (T is a power of two,
// so n % (2T) == 0).
bool adjoint_sym_ok(int n, int factor, int n_loc, bool mirror_layout) {
  int T, S;
  adjoint_layout(n, factor, n_loc, false, &T, &S);
  return mirror_layout && n_loc >= 2 && n % (2 * T) == 0;
}

int adjoint_planes(int n, int factor, int n_loc, bool sym, int sym_s) {
  int T, S, cz;
  adjoint_layout(n, factor, n_loc, sym, &T, &S, &cz);
  (void)sym_s;  // angle 0 is added in the symmetric kernel's epilogue
  const int planes = S / cz;
  return planes > 1 ? planes : 0;
}

template <bool kPair, int T, bool kSym, bool kRP = false>
static void adj_launch_(dim3 grid, size_t smem, cudaStream_t stream, int cz, const float* sino,
                        float* dst, int n, int W, int CA, int a_begin, int per_split, int a_end,
                        int n_mirror, int n_det, const AdjAngle* ang, int add_a0) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kAdjThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = (unsigned)cz;
  cfg.attrs = attr;
  cfg.numAttrs = cz > 1 ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_adjoint<kPair, T, kSym, (T >= 16 ? 8 : 2), kRP>, sino, dst, n, W,
                     CA, a_begin, per_split, a_end, n_mirror, n_det, ang, add_a0);
}

static void adj_dispatch(bool pair, int T, bool sym, dim3 grid, size_t smem, cudaStream_t stream,
                         int cz, const float* sino, float* dst, int n, int W, int CA, int a_begin,
                         int per_split, int a_end, int n_mirror, int n_det, const AdjAngle* ang,
                         int add_a0, bool rp = false) {
  if (rp) {
    adj_launch_<true, 32, true, true>(grid, smem, stream, cz, sino, dst, n, W, CA, a_begin,
                                      per_split, a_end, n_mirror, n_det, ang, add_a0);
    return;
  }
#define ADJ_CALL(P_, T_, S_)                                                                   \
  adj_launch_<P_, T_, S_>(grid, smem, stream, cz, sino, dst, n, W, CA, a_begin, per_split, a_end, \
                          n_mirror, n_det, ang, add_a0)
  if (pair) {
    if (sym) ADJ_CALL(true, 32, true); else ADJ_CALL(true, 32, false);
  } else if (T == 32) {
    if (sym) ADJ_CALL(false, 32, true); else ADJ_CALL(false, 32, false);
  } else if (T == 16) {
    if (sym) ADJ_CALL(false, 16, true); else ADJ_CALL(false, 16, false);
  } else {
    if (sym) ADJ_CALL(false, 8, true); else ADJ_CALL(false, 8, false);
  }
#undef ADJ_CALL
}

static size_t adj_smem(bool pair, bool sym, int T, int W, int* CA_io) {
  const int ppt = T >= 16 ? 8 : 2;
  const int lanes = T * T / ppt;
  const int G = kAdjThreads / lanes;
  const size_t elem = sizeof(float) * (pair ? 2 : 1) * (sym ? 2 : 1);
  // up to 32 angles per chunk, fewer for wide windows (keep ~7 CTAs per SM)
  const size_t cap = (size_t)knob(Knob::kAdjWinKb, 20) * 1024;
  int CA = 32;
  while (CA > G && (size_t)CA * W * elem > cap) CA >>= 1;
  if (CA < G) CA = G;
  *CA_io = CA;
  // the window region also holds the CTA's tile for the cluster reduction
  const size_t tile = sizeof(float) * T * T * (sym ? 2 : 1);
  const size_t win = (size_t)CA * W * elem;
  return (size_t)CA * sizeof(AdjStage) + kAdjThreads * ppt * (sym ? 2 : 1) * sizeof(float) +
         (win > tile ? win : tile);
}

// Reduction mode of the split planes, shared by the reduce kernels and the
// image-side kernels that fold the reduction in (k_saga_image_coarse32 repeats
// the predicate): warp per pixel (lane-strided
// planes, xor tree) for many planes and few pixels, else planes in order.
static bool adjoint_reduce_warp(int npix, int planes) { return planes >= 32 && npix <= 65536; }

static void adj_reduce(const float* partial, float* out, int npix, int S, cudaStream_t stream) {
  if (adjoint_reduce_warp(npix, S))
    launch_pdl(k_adjoint_reduce_warp, dim3((npix * 32 + 255) / 256), dim3(256), 0, stream,
               partial, out, npix, S);
  else
    launch_pdl(k_adjoint_reduce, dim3((npix + 255) / 256), dim3(256), 0, stream, partial, out,
               npix, S);
}

// defer_planes != nullptr: the split planes are left unreduced (the consumer
// sums them) and their count is returned there (0: the result is in out).
cudaError_t launch_adjoint_reduce(const float* partial, float* out, int npix, int S,
                                  cudaStream_t stream) {
  adj_reduce(partial, out, npix, S, stream);
  return cudaGetLastError();
}

cudaError_t launch_adjoint(const float* sino, float* out, float* partial, int n, int factor,
                           int n_loc, int n_det, const AdjAngle* ang, int sym_s,
                           cudaStream_t stream, const SideStream& side, int* launches,
                           int* defer_planes) {
  (void)side;
  if (defer_planes) *defer_planes = 0;
  const bool sym = adjoint_sym_ok(n, factor, n_loc, sym_s >= 0);
  int T, S, cz;
  adjoint_layout(n, factor, n_loc, sym, &T, &S, &cz);
  const bool pair = (factor == 1 && T == 32);
  const int W = (int)floor(1.41422 * T * factor) + 6;
  const int planes = S / cz;
  float* dst = planes > 1 ? partial : out;
  int CA;
  // factor 1 with mirror symmetry: the row-pair kernel (single-bin windows) is
  // bit-identical but measured slower (whole-set f=1 adjoint 515 -> 524 us,
  // 1/8 shard 81 -> 85 us: the carry selects cost more issue than the 25%
  // fewer shared wavefronts save), so it is an A/B switch, off by default
  const bool rp = pair && sym && knob(Knob::kAdjRowPair, 0) != 0;
  const size_t smem = adj_smem(pair && !rp, sym, T, W, &CA);
  if (sym) {
    // rows [sym_s, n_loc) with their mirrors over the left-half tiles; the
    // unpaired angle 0 (rows [0, sym_s)) in the epilogue
    const int per_split = (n_loc - sym_s + S - 1) / S;
    dim3 grid(n / (2 * T), (n + T - 1) / T, S);
    adj_dispatch(pair, T, true, grid, smem, stream, cz, sino, dst, n, W, CA, sym_s, per_split,
                 n_loc, sym_s + n_loc - 1, n_det, ang, sym_s > 0 ? 1 : 0, rp);
  } else {
    const int per_split = (n_loc + S - 1) / S;
    dim3 grid((n + T - 1) / T, (n + T - 1) / T, S);
    adj_dispatch(pair, T, false, grid, smem, stream, cz, sino, dst, n, W, CA, 0, per_split, n_loc,
                 n_loc, n_det, ang, 0);
  }
  *launches = 1;
  if (planes > 1) {
    if (defer_planes) {
      *defer_planes = planes;
    } else {
      adj_reduce(partial, out, n * n, planes, stream);
      *launches = 2;
    }
  }
  return cudaGetLastError();
}

}  // namespace imask

namespace imask {
// this file's index-check counters (imask_common.cuh: IMASK_BOUNDS_CHECK)
bool debug_bounds_read_projector(unsigned long long* out4, bool reset) {
  return bounds_read(out4, reset);
}
int forward_tma_entries_per_cta() { return kFE; }
int forward_tma_window() { return kFWc; }
}  // namespace imask
