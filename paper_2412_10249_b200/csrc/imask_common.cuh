// Shared definitions of the sm_100a ImaSk kernels.
//
// Ray/pixel geometry (reference ctmodel.py:73-154, restated in
// oracle/ct_oracle.py): pixel (row, col) of the n x n grid of width h has
// centre X = -half + (col+.5)h, Y = -half + (row+.5)h, half = n*h/2 (= side/2
// at every level); ray (a, j) is the line X cos + Y sin = t_j,
// t_j = j - (n_det-1)/2.
//
// Positions along a ray and across a pixel's footprint are carried in signed
// Q32.32 fixed point (int64): the integer word is a pixel / detector index,
// the fraction word feeds the weights through a float built from its top 23
// bits. Stepping is an exact integer add, so no drift builds up along a ray
// and ties on gridlines (axis-parallel rays with integer offsets) are decided
// exactly, as the reference's half-open rule requires (ctmodel.py:99-114).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace imask {

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// (and run its independent prologue) while its stream predecessor drains; it
// must call griddep_wait() before reading anything the predecessor writes.
// In a kernel launched normally griddep_wait() returns at once.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

constexpr double kFix = 4294967296.0;  // 2^32

// Debug build (-DIMASK_BOUNDS_CHECK=1): the kernels check their computed
// indices against the range they must stay in -- every shared-memory window
// read of the projectors and pair-image read of the L1 forwards, every plane
// write of the staging kernels, every table / tile access of the any-size
// sketch and image-side kernels -- and count violations in a per-file device
// word the host reads with imask_debug_bounds. compute-sanitizer is closed on
// the B200 pool, so this build, run through the GPU test suite
// (tools/gpu_bounds_check.sh), stands in for memcheck on computed indices.
#ifndef IMASK_BOUNDS_CHECK
#define IMASK_BOUNDS_CHECK 0
#endif
#if IMASK_BOUNDS_CHECK
static __device__ unsigned long long g_bounds[4];  // violations, first: site code, index, limit
static __device__ __noinline__ void bounds_fail(int code, long long idx, long long limit) {
  if (atomicAdd(&g_bounds[0], 1ull) == 0ull) {
    g_bounds[1] = (unsigned long long)code;
    g_bounds[2] = (unsigned long long)idx;
    g_bounds[3] = (unsigned long long)limit;
  }
}
#define IMASK_CHECK_RANGE(code, idx, limit)                                       \
  do {                                                                            \
    const long long i_ = (long long)(idx), l_ = (long long)(limit);               \
    if (i_ < 0 || i_ >= l_) bounds_fail(code, i_, l_);                            \
  } while (0)
// out4 = this translation unit's {violations, first site code, index, limit}
// (all ones when the device word cannot be read)
static inline bool bounds_read(unsigned long long* out4, bool reset) {
  out4[0] = out4[1] = out4[2] = out4[3] = ~0ull;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    out4[1] = (unsigned long long)e;
    out4[2] = 1;
    return true;
  }
  unsigned long long v[4];
  e = cudaMemcpyFromSymbol(v, g_bounds, sizeof(v));
  if (e != cudaSuccess) {
    out4[1] = (unsigned long long)e;
    out4[2] = 2;
    return true;
  }
  for (int i = 0; i < 4; ++i) out4[i] = v[i];
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_bounds, z, sizeof(z));
  }
  return true;
}
#else
#define IMASK_CHECK_RANGE(code, idx, limit) ((void)0)
static inline bool bounds_read(unsigned long long* out4, bool reset) {
  (void)reset;
  out4[0] = out4[1] = out4[2] = out4[3] = 0;
  return false;
}
#endif

// Path and tuning switches, read once from the environment (host code only).
// Unset, the product defaults apply. They exist to select the alternative
// code paths the bit-identity tests compare (IMASK_NO_QUAD, IMASK_NO_TMA,
// IMASK_FWD_VAL, IMASK_FWD_VAL_L1) and for A/B measurement runs (the others,
// tools/gpu_ab_env.sh); DESIGN.md lists what each one measured.
enum class Knob {
  kNoTma,            // IMASK_NO_TMA: forward through L1 loads only
  kNoQuad,           // IMASK_NO_QUAD: pair (mirror-only) entries, no four-ray quads
  kNoQuadL1,         // IMASK_NO_QUAD_L1: coarse levels through the pair L1 kernel
  kFwdVal,           // IMASK_FWD_VAL (0/1): TMA forward value-plane staging forced off/on
  kFwdValL1,         // IMASK_FWD_VAL_L1 (0/1): L1 quad forward value planes
  kTmaMinN,          // IMASK_TMA_MIN_N: smallest coarse side on the TMA forward (128)
  kAdjAfterStageMinN,  // IMASK_ADJ_AFTER_STAGE_MIN_N: step order threshold
  kSagaSplitMinN,    // IMASK_SAGA_SPLIT_MIN_N: separate sinogram SAGA pass threshold
  kAdjWinKb,         // IMASK_ADJ_WIN_KB: adjoint window budget per CTA (20)
  kAdjCluster,       // IMASK_ADJ_CLUSTER: adjoint cluster size (1 = none)
  kAdjTile,          // IMASK_ADJ_TILE: "f:T,..." adjoint tile per factor
  kAdjCtas,          // IMASK_ADJ_CTAS: "f:ctas_per_sm,..." adjoint split target
  kFwdTwoDet,        // IMASK_FWD_TWO_DET (0/1): two detectors per thread in the TMA forward (f >= 2)
  kFusedStage,       // IMASK_FUSED_STAGE (0/1): x -> value planes in one kernel
  kFwdTwoDetMinWaves,  // IMASK_FWD_TWO_DET_MIN_WAVES: two-detector grids need >= this x SMs CTAs
  kAdjRowPair,       // IMASK_ADJ_ROW_PAIR (0/1): the f=1 symmetric adjoint on row pairs (off)
  kFwdTwoDetMinN,    // IMASK_FWD_TWO_DET_MIN_N: smallest coarse side with two detectors per thread (512)
  kFwdTables,        // IMASK_FWD_TABLES (0/1): TMA forward reads its CTAs' prebuilt chunk tables (1)
  kCount
};
// Integer value of a switch, or `dflt` when unset (a set-but-valueless flag
// reads as 1).
int knob(Knob k, int dflt);
// Per-factor value of a "f:v,f:v" list switch, or `dflt`.
int knob_for_factor(Knob k, int factor, int dflt);

// Zero columns on each side of every pair-image row (see k_forward): a lane
// walking its warp's band range outside its own valid range is at most
// 31*sqrt(2) < 48 columns from a lane inside it, so it reads zeros instead of
// needing a predicate. Column c in [-1-kPadC, n-1+kPadC] is stored at index
// c + 1 + kPadC of a row of pitch >= n + 2*kPadC + 1, rounded up to an even
// number of float2 so rows are 16-byte aligned (TMA tensor-map strides).
constexpr int kPadC = 48;
__host__ __device__ inline int pair_pitch(int n) { return (n + 2 * kPadC + 2) & ~1; }

// Forward projector, one entry per (level factor, local angle).
// A ray crosses `n` bands (pixel rows, or columns when |sin| > |cos|); at
// band b its band coordinate is xi = xi_base + j*xi_dj + b*(step/2^32), in
// pixel-index units measured from the centre of pixel 0. The band's chord
// (length wsc/scale) splits between pixel floor(xi) and floor(xi)+1 with
// fractions (1-g, g), g = sat(onep*S + B), onep = 1 + frac(xi).
struct FwdAngle {
  double xi_base;
  double xi_dj;
  double inv_step;  // 2^32 / step (0 when step == 0): band-range estimate without division
  long long step;
  float S, B;
  float wsc;       // h / max(|cos|,|sin|) * scale
  int transposed;  // 0: bands are rows (row-major image), 1: columns (transposed image)
};

// Adjoint projector, one entry per (level factor, local angle).
// For pixel (col,row) the footprint covers detector coordinates
// eta = X cos + Y sin + (n_det-1)/2 within +-R, a trapezoid of height
// wsc/scale, plateau half-width |a-b|, support half-width R = a+b
// (a = |cos|h/2, b = |sin|h/2). eta0 is eta at pixel (0,0) minus R.
// Inside a CTA tile, positions are Q32.32 fixed point relative to the tile's
// staged sinogram window (Dc, Ds = per-column / per-row increments).
struct AdjAngle {
  double eta0;
  double ch, sh;       // cos*h, sin*h
  long long Dc, Ds;    // Q32.32 of ch, sh
  float R;             // support half-width in detector units
  float kneg, Rk;      // w = sat(|u|*kneg + Rk), kneg = -1/(2 min(a,b)), Rk = R/(2 min(a,b))
  float wsc;           // h / max(|cos|,|sin|) * scale
  int nb;              // candidate bins per pixel
  int axis;            // 1: axis-parallel half-open box rule
};

// Q32.32 position held as two 32-bit words; one add-with-carry pair advances it
// and the integer word is used directly as an index (no 64-bit shifts).
struct Fix32 {
  uint32_t lo, hi;
};
__device__ __forceinline__ Fix32 fix_from(long long v) {
  return Fix32{(uint32_t)(unsigned long long)v, (uint32_t)((unsigned long long)v >> 32)};
}
__device__ __forceinline__ void fix_add(Fix32& a, const Fix32& d) {
  asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;"
      : "+r"(a.lo), "+r"(a.hi)
      : "r"(d.lo), "r"(d.hi));
}

// 1 + (top 23 bits of a Q0.32 fraction) as a float in [1, 2)
__device__ __forceinline__ float onep_from_frac(uint32_t frac) {
  return __uint_as_float((frac >> 9) | 0x3F800000u);
}

// Packed FP32 (FADD2 / FFMA2, sm_100): both lanes of a float2 in one
// instruction, each rounded exactly like the scalar fadd / fmaf.
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return r;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 r;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return r;
}
// c + g * b with the scalar g broadcast
__device__ __forceinline__ float2 ffma2(float g, float2 b, float2 c) {
  float2 r;
  const float2 gg = make_float2(g, g);
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&r))
      : "l"(*reinterpret_cast<const unsigned long long*>(&gg)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return r;
}

struct SinoSaga {  // sinogram side of the SAGA step, fused into the forward epilogue
  float* psi_tab;        // level row of the psi table
  float* psi_sum;
  const float* y_in;  // y^k
  float* y;           // y^{k+1} (== y_in for the in-place update)
  const float* b;
  float p_i;
  float sigma;
  float inv_1ps;  // 1 / (1 + sigma)
};

// Optional second stream for work that can overlap a kernel on the main
// stream: fork = record on main + wait on side; join = record on side + wait on
// main. stream == nullptr: everything stays on the main stream.
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

// Inputs of the sinogram-side update of one ray, loaded before the band walk
// so their latency hides behind it; sino_update then applies solvers.py:205-215
// (psi row, psi_sum, dual prox) with the new projection value.
struct SinoIn {
  float po = 0.f, ps = 0.f, yv = 0.f, bv = 0.f;
};
// psi_tab == nullptr is the PDHG dual step (solvers.py:333-334): no tables, so
// zeta = val and y' = (y + sigma K xbar - sigma b) / (1 + sigma).
__device__ __forceinline__ SinoIn sino_load(const SinoSaga& sg, size_t q) {
  SinoIn in;
  if (sg.psi_tab) {
    in.po = sg.psi_tab[q];
    in.ps = sg.psi_sum[q];
  }
  in.yv = sg.y_in[q];
  in.bv = __ldg(sg.b + q);
  return in;
}
__device__ __forceinline__ void sino_update(const SinoSaga& sg, size_t q, const SinoIn& in,
                                            float val) {
  const float d = val - in.po;
  const float zeta = d + in.ps;
  if (sg.psi_tab) {
    sg.psi_sum[q] = fmaf(sg.p_i, d, in.ps);
    sg.psi_tab[q] = val;
  }
  const float yv = fmaf(sg.sigma, zeta, in.yv);
  sg.y[q] = (yv - sg.sigma * in.bv) * sg.inv_1ps;
}

struct ImageSaga {
  float* phi_tab;  // level row of the phi table (coarse, or full at the full level)
  float* phi_sum;
  float* x;
  float p_i;
  float s;        // sigma / mu
  float inv_den;  // 1 / (1 + s*mu_g)
  float* xbar = nullptr;  // sketch_seq_step: xbar = x' + theta (x' - x) (nullptr: none)
  float theta = 0.f;
  // n_planes > 0: the backprojection is the sum of n_planes partial planes of
  // the adjoint's angle splits (plane stride plane_len), reduced here in the
  // order of k_adjoint_reduce / k_adjoint_reduce_warp instead of read from bp
  const float* planes = nullptr;
  int n_planes = 0;
  long long plane_len = 0;
};

// Primal extrapolation of sketch_seq_step (solvers.py:296-300) for one pixel /
// four pixels, given the old and the new primal value.
__device__ __forceinline__ void extrapolate(const ImageSaga& sg, size_t p, float xo, float xn) {
  if (sg.xbar) sg.xbar[p] = fmaf(sg.theta, xn - xo, xn);
}
__device__ __forceinline__ void extrapolate4(const ImageSaga& sg, size_t p, float4 xo, float4 xn) {
  if (sg.xbar)
    *reinterpret_cast<float4*>(sg.xbar + p) =
        make_float4(fmaf(sg.theta, xn.x - xo.x, xn.x), fmaf(sg.theta, xn.y - xo.y, xn.y),
                    fmaf(sg.theta, xn.z - xo.z, xn.z), fmaf(sg.theta, xn.w - xo.w, xn.w));
}

}  // namespace imask
