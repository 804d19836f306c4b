// C-ABI of the ImaSk B200 hot path (declared in include/imask_b200.h).
//
// The plan replaces the reference's per-geometry projector cache
// (_projector_pair, ctmodel.py:157-167): instead of a CSR matrix it holds the
// float64-derived per-angle parameter tables of every level factor (a few KB)
// and the staging buffers of the forward projector. Everything else is
// caller-owned device memory.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>

#include "imask_b200.h"
#include "imask_common.cuh"
#include "sketch.cuh"

namespace imask {
cudaError_t launch_forward(const float2* P, const float2* PT, const float2* PM, const float2* PTM,
                           int n, const FwdAngle* ang, int n_loc, int n_det,
                           const int2* sym_entries, int n_entries, const int4* quad_entries,
                           int n_quad_entries, float* sino, const SinoSaga* saga,
                           cudaStream_t stream);
cudaError_t launch_adjoint(const float* sino, float* out, float* partial, int n, int factor,
                           int n_loc, int n_det, const AdjAngle* ang, int sym_s,
                           cudaStream_t stream, const SideStream& side, int* launches,
                           int* defer_planes = nullptr);
int adjoint_planes(int n, int factor, int n_loc, bool sym, int sym_s);
cudaError_t launch_adjoint_reduce(const float* partial, float* out, int npix, int S,
                                  cudaStream_t stream);
bool adjoint_sym_ok(int n, int factor, int n_loc, bool full_even_set);
cudaError_t launch_restrict(const float* x, float* u, int side, int f, cudaStream_t s);
cudaError_t launch_prolong(const float* u, float* x, int side, int f, float alpha,
                           cudaStream_t s);
cudaError_t launch_compensate(const float* x, float* out, int side, const CompParams& cp,
                              cudaStream_t s);
cudaError_t launch_prepare(const float* u, int n, float2* P, float2* PT, float2* PM,
                           float2* PTM, bool diff, cudaStream_t s);
bool stage32_ok(int side, int f, int r);
cudaError_t launch_stage32(const float* x, int side, int f, const CompParams& cp, float2* P,
                           float2* PT, cudaStream_t s);
bool forward_tma_val_grid(int n_det, int n_entries);
bool forward_l1_val();
cudaError_t launch_saga_image_coarse(const float* bp, int side, int f, const ImageSaga& sg,
                                     cudaStream_t s);
cudaError_t launch_saga_image_full(const float* bp, int side, const CompParams& cp,
                                   const ImageSaga& sg, cudaStream_t s);
cudaError_t launch_saga_sino(const float* psi_new, size_t m, const SinoSaga& sg, cudaStream_t s);
cudaError_t launch_pdhg_image(const float* bp, float* x, float* xbar, size_t d, float tau,
                              float inv_den, float theta, cudaStream_t s);
cudaError_t launch_resum(const float* phi_tab, float* phi_sum, int side, const float* psi_tab,
                         float* psi_sum, size_t m, const ResumParams& rp, cudaStream_t s);
void init_kernel_attributes();
int forward_tma_entries_per_cta();
int forward_tma_window();
bool debug_bounds_read_projector(unsigned long long* out4, bool reset);
bool debug_bounds_read_sketch(unsigned long long* out4, bool reset);
int forward_tma_bands(bool quad, bool val);
struct TmaMaps {
  CUtensorMap row, row_m, col, col_m;
};
cudaError_t launch_forward_tma(const TmaMaps& maps, const float2* P, const float2* PT,
                               const float2* PM, const float2* PTM, int n, const FwdAngle* ang,
                               const int4* entries, int n_entries, int row_ctas, bool quad,
                               int n_det, float* sino, const SinoSaga* saga, cudaStream_t stream,
                               bool two_det, const int* tab_in, int* tab_out);
size_t forward_tma_table_len(int n, int n_det, int n_entries, bool quad, bool two_det);
}  // namespace imask

struct imask_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int device = 0;
};

namespace imask {

namespace {
const char* const kKnobNames[(int)Knob::kCount] = {
    "IMASK_NO_TMA", "IMASK_NO_QUAD", "IMASK_NO_QUAD_L1", "IMASK_FWD_VAL", "IMASK_FWD_VAL_L1",
    "IMASK_TMA_MIN_N", "IMASK_ADJ_AFTER_STAGE_MIN_N", "IMASK_SAGA_SPLIT_MIN_N",
    "IMASK_ADJ_WIN_KB", "IMASK_ADJ_CLUSTER", "IMASK_ADJ_TILE", "IMASK_ADJ_CTAS",
    "IMASK_FWD_TWO_DET", "IMASK_FUSED_STAGE", "IMASK_FWD_TWO_DET_MIN_WAVES",
    "IMASK_ADJ_ROW_PAIR", "IMASK_FWD_TWO_DET_MIN_N", "IMASK_FWD_TABLES"};

std::string g_knob_vals[(int)Knob::kCount];
bool g_knob_set[(int)Knob::kCount];
std::mutex g_knob_mu;
bool g_knobs_read = false;

void read_knobs() {
  for (int i = 0; i < (int)Knob::kCount; ++i) {
    const char* e = std::getenv(kKnobNames[i]);
    g_knob_set[i] = e != nullptr;
    g_knob_vals[i] = e ? e : "";
  }
  g_knobs_read = true;
}

const char* knob_raw(Knob k) {
  std::lock_guard<std::mutex> lk(g_knob_mu);
  if (!g_knobs_read) read_knobs();
  return g_knob_set[(int)k] ? g_knob_vals[(int)k].c_str() : nullptr;
}
}  // namespace

int knob(Knob k, int dflt) {
  const char* e = knob_raw(k);
  if (!e) return dflt;
  return *e ? std::atoi(e) : 1;
}

int knob_for_factor(Knob k, int factor, int dflt) {
  const char* e = knob_raw(k);
  int v = dflt;
  for (const char* q = e; q && *q;) {
    int ff = 0, vv = 0;
    if (std::sscanf(q, "%d:%d", &ff, &vv) == 2 && ff == factor) v = vv;
    while (*q && *q != ',') ++q;
    if (*q) ++q;
  }
  return v;
}

}  // namespace imask

using namespace imask;

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct LevelTables {
  FwdAngle* fwd = nullptr;  // device
  AdjAngle* adj = nullptr;  // device
  bool tma = false;         // tensor maps of the pair images at this level are valid
  bool two_det = false;     // every TMA entry's detectors are < 1 column apart (and ascend):
                            // the two-detectors-per-thread forward applies
  TmaMaps maps{};           // boxes of 96 x 16 (pair mode) or 96 x 8 bands (quad mode)
  int* fwd_tab = nullptr;   // device: per-CTA chunk tables of the TMA forward (geometry only)
  bool fwd_tab_val = false;  // the staging mode (value planes) they were built for
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D map over a pair image of one level: {pitch, n} 8-byte elements, box of
// kFWc columns x box_h bands (projector.cu: 96 x 16 in pair mode, 96 x 8 in quad mode).
bool encode_pair_map(CUtensorMap* map, void* base, int n, unsigned box_h) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || !base) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)pair_pitch(n), (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)pair_pitch(n) * sizeof(float2)};
  const cuuint32_t box[2] = {(cuuint32_t)forward_tma_window(), box_h};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

struct imask_plan {
  int side, n_angles, n_det, n_loc, r, device;
  std::vector<int> angle_idx;  // global angle index of every local sinogram row
  int sym_s = 0;               // symmetric layout: rows [0, sym_s) unpaired (angle 0),
                               // rows [sym_s, n_loc) mirror-paired as i <-> sym_s + n_loc - 1 - i
  double scale;
  std::vector<double> probs, cosv, sinv;
  std::vector<int> factors;        // factor of level i (0-based)
  std::vector<long long> phi_off;  // phi table offsets
  std::map<int, LevelTables> tables;
  std::mutex mu;
  float2* P = nullptr;
  float2* PT = nullptr;
  float2* PM = nullptr;   // mirrored pair images (mirror-symmetric forward)
  float2* PTM = nullptr;
  bool sym = false;       // whole, even-sized angle set: mirror-symmetric kernels
  int2* fwd_entries = nullptr;  // (angle, mirror angle or -1) per forward warp
  int n_entries = 0;
  int4* tma_entries = nullptr;  // TMA forward entries, 8 per CTA (-1 = none):
                                // quad mode (a, n-a, n/2-a, n/2+a); pair mode (a, n-a, -1, -1)
                                // grouped by ray family
  int n_tma_entries = 0;
  std::vector<int4> tma_entries_host;  // host copy of tma_entries
  int tma_row_ctas = 0;         // pair mode: CTAs [0, tma_row_ctas) hold row-family entries
  bool tma_quad = false;        // the local rows are closed under a -> n/2 - a as well
  float* u = nullptr;
  float* sino_tmp = nullptr;
  float* adj_partial = nullptr;  // per-split partial backprojections (coarse levels)
  SideStream aux;                // angle-0 plane of the symmetric adjoint
  SideStream aux2;               // forward chain of imask_sketch_step, concurrent with the adjoint
  cudaEvent_t ev_staged = nullptr;  // aux2: x has been read (restriction / compensation done)
  size_t adj_partial_len = 0;
  std::vector<float*> retired;   // replaced scratch buffers, freed with the plan
  int64_t scratch = 0;
  CompParams cp{};
  ResumParams rp{};
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(IMASK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return IMASK_OK;
}

#define LAUNCH(expr, what)                                   \
  do {                                                       \
    ++g_launches;                                            \
    int _rc = cuda_check((expr), what);                      \
    if (_rc != IMASK_OK) return _rc;                         \
  } while (0)

// Float64 per-angle parameters of one level factor (see imask_common.cuh).
void build_tables(const imask_plan& pl, int f, std::vector<FwdAngle>& fw,
                  std::vector<AdjAngle>& ad) {
  const double h = (double)f;
  const double half = pl.side / 2.0;  // n*h/2 at every level
  const double t0 = -(pl.n_det - 1) / 2.0;
  fw.resize(pl.n_loc);
  ad.resize(pl.n_loc);
  for (int a = 0; a < pl.n_loc; ++a) {
    const double c = pl.cosv[a], s = pl.sinv[a];
    const double ac = std::fabs(c), as = std::fabs(s);
    const bool axis = (c == 0.0 || s == 0.0);
    FwdAngle F{};
    double step, tau, wmax;
    if (ac >= as) {  // bands are pixel rows: x where the ray meets the row centre line
      F.transposed = 0;
      F.xi_dj = 1.0 / (c * h);
      F.xi_base = t0 / (c * h) + (half - h / 2) * s / (c * h) + half / h - 0.5;
      step = -s / c;
      tau = as / ac;
      wmax = h / ac;
    } else {  // bands are pixel columns (transposed image)
      F.transposed = 1;
      F.xi_dj = 1.0 / (s * h);
      F.xi_base = t0 / (s * h) + (half - h / 2) * c / (s * h) + half / h - 0.5;
      step = -c / s;
      tau = ac / as;
      wmax = h / as;
    }
    F.step = std::llrint(step * kFix);
    F.inv_step = F.step != 0 ? kFix / (double)F.step : 0.0;
    if (axis) {
      // g = [frac >= 1/2]: the ray on a gridline goes to the upper/right pixel
      F.S = 16777216.0f;   // 2^24
      F.B = -25165822.0f;  // 2 - 1.5*2^24
    } else {
      F.S = (float)(1.0 / tau);
      F.B = (float)(-(3.0 - tau) / (2.0 * tau));
    }
    F.wsc = (float)(wmax * pl.scale);
    fw[a] = F;

    AdjAngle A{};
    A.ch = c * h;
    A.sh = s * h;
    const double R = (ac + as) * h / 2.0;
    A.eta0 = (-half + h / 2.0) * (c + s) + (pl.n_det - 1) / 2.0 - R;
    A.Dc = std::llrint(A.ch * kFix);
    A.Ds = std::llrint(A.sh * kFix);
    A.R = (float)R;
    A.wsc = (float)(wmax * pl.scale);
    if (axis) {
      A.axis = 1;
      A.nb = f;
      A.kneg = 0.f;
      A.Rk = 0.f;
    } else {
      const double kk = 1.0 / (std::fmin(ac, as) * h);  // 1/(R - plateau half-width)
      A.axis = 0;
      A.nb = (int)std::floor(2.0 * R) + 1;
      A.kneg = (float)(-kk);
      A.Rk = (float)(R * kk);
    }
    ad[a] = A;
  }
}

int get_tables(imask_plan* pl, int f, LevelTables** out) {
  std::lock_guard<std::mutex> lk(pl->mu);
  auto it = pl->tables.find(f);
  if (it == pl->tables.end()) {
    std::vector<FwdAngle> fw;
    std::vector<AdjAngle> ad;
    build_tables(*pl, f, fw, ad);
    LevelTables t;
    if (pl->n_loc > 0) {
      int rc = cuda_check(cudaMalloc(&t.fwd, sizeof(FwdAngle) * pl->n_loc), "cudaMalloc");
      if (rc) return rc;
      rc = cuda_check(cudaMalloc(&t.adj, sizeof(AdjAngle) * pl->n_loc), "cudaMalloc");
      if (rc) return rc;
      rc = cuda_check(cudaMemcpy(t.fwd, fw.data(), sizeof(FwdAngle) * pl->n_loc,
                                 cudaMemcpyHostToDevice),
                      "cudaMemcpy");
      if (rc) return rc;
      rc = cuda_check(cudaMemcpy(t.adj, ad.data(), sizeof(AdjAngle) * pl->n_loc,
                                 cudaMemcpyHostToDevice),
                      "cudaMemcpy");
      if (rc) return rc;
    }
    if (pl->sym && pl->tma_entries) {
      // the two-detector forward needs 0 < xi_dj < 1 for every entry's parameter row
      bool ok = f >= 2 && knob(Knob::kFwdTwoDet, 1) != 0;
      for (const int4& e4 : pl->tma_entries_host) {
        const int row = e4.x >= 0 ? e4.x : e4.z;
        if (row >= 0 && !(fw[row].xi_dj > 0.0 && fw[row].xi_dj < 0.999)) ok = false;
      }
      // a small grid (an angle shard) runs latency-bound along each CTA's band
      // walk: halving its CTAs costs more than the shared reads save (1/8 shard
      // f=2 forward 71 -> 97 us), so two detectors only where the two-detector
      // grid still fills >= IMASK_FWD_TWO_DET_MIN_WAVES x SM count CTAs
      const long long ctas2 = (long long)((pl->n_det + 63) / 64) *
                              (long long)((pl->n_tma_entries + forward_tma_entries_per_cta() - 1) /
                                          forward_tma_entries_per_cta());
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl->device);
      if (ctas2 < (long long)knob(Knob::kFwdTwoDetMinWaves, 6) * sms) ok = false;
      // with 16-band chunks (half the per-chunk work per ray) one detector per
      // thread is faster on coarse sides below 512 (config D, in the step:
      // f=4 223 -> 217 us, f=8 137 -> 132 us); at n = 512 the two-detector
      // kernel's smaller footprint beside the adjoint still wins (354 vs 359 us)
      if (pl->side / f < knob(Knob::kFwdTwoDetMinN, 512)) ok = false;
      t.two_det = ok;
    }
    if (pl->sym && !knob(Knob::kNoTma, 0)) {
      const int n = pl->side / f;
      // box height = bands per chunk of the TMA kernel this level launches
      const bool val = t.two_det || forward_tma_val_grid(pl->n_det, pl->n_tma_entries);
      const unsigned bh = (unsigned)forward_tma_bands(pl->tma_quad, val);
      t.tma = encode_pair_map(&t.maps.row, pl->P, n, bh) &&
              encode_pair_map(&t.maps.row_m, pl->PM, n, bh) &&
              encode_pair_map(&t.maps.col, pl->PT, n, bh) &&
              encode_pair_map(&t.maps.col_m, pl->PTM, n, bh);
      if (t.tma && pl->tma_entries && pl->n_loc > 0 && n >= knob(Knob::kTmaMinN, 128)) {
        // the CTAs' chunk tables, built once by the kernel itself (tab_out)
        const size_t len = forward_tma_table_len(n, pl->n_det, pl->n_tma_entries, pl->tma_quad,
                                                 t.two_det);
        int rc = cuda_check(cudaMalloc(&t.fwd_tab, sizeof(int) * len), "cudaMalloc fwd_tab");
        if (rc) return rc;
        rc = cuda_check(launch_forward_tma(t.maps, pl->P, pl->PT, pl->PM, pl->PTM, n, t.fwd,
                                           pl->tma_entries, pl->n_tma_entries, pl->tma_row_ctas,
                                           pl->tma_quad, pl->n_det, pl->sino_tmp, nullptr, nullptr,
                                           t.two_det, nullptr, t.fwd_tab),
                        "forward tables");
        if (!rc) rc = cuda_check(cudaDeviceSynchronize(), "forward tables");
        if (rc) return rc;
        t.fwd_tab_val = val;
      }
    }
    it = pl->tables.emplace(f, t).first;
  }
  *out = &it->second;
  return IMASK_OK;
}

int ensure_partial(imask_plan* pl, int f) {
  const int n = pl->side / f;
  const bool sym = adjoint_sym_ok(n, f, pl->n_loc, pl->sym);
  const size_t need = (size_t)adjoint_planes(n, f, pl->n_loc, sym, pl->sym_s) * n * n;
  if (need > pl->adj_partial_len) {
    // the plan is created with room for every factor of its family; a larger
    // factor served later (backproject at another f) gets a new buffer, and the
    // old one is retired, not freed: captured step graphs may still point at it
    if (pl->adj_partial) pl->retired.push_back(pl->adj_partial);
    pl->adj_partial = nullptr;
    pl->adj_partial_len = 0;
    int rc = cuda_check(cudaMalloc(&pl->adj_partial, need * sizeof(float)), "cudaMalloc partial");
    if (rc) return rc;
    pl->adj_partial_len = need;
    pl->scratch += (int64_t)(need * sizeof(float));
  }
  return IMASK_OK;
}

int run_adjoint(imask_plan* pl, int f, const float* sino, float* out, const AdjAngle* ang,
                cudaStream_t s, int* defer_planes = nullptr) {
  int launches = 0;
  cudaError_t e = launch_adjoint(sino, out, pl->adj_partial, pl->side / f, f, pl->n_loc, pl->n_det,
                                 ang, pl->sym ? pl->sym_s : -1, s, pl->aux, &launches,
                                 defer_planes);
  g_launches += launches;
  return cuda_check(e, "adjoint");
}

// Step order at large levels: the adjoint is enqueued behind the forward's
// input staging, so the forward kernel is dispatched first. Launched
// together, the adjoint's many short CTAs (~30 KB shared memory each) fill
// every SM, and the forward's 58 KB CTAs only get slots as the adjoint drains,
// which serialises the two; dispatched first, the forward's CTAs are resident
// and the adjoint's fill the space around them. Measured (config D, L2 flushed
// between steps): f = 1/2/4 steps -3/-4/-3% on one GPU and -21/-15/-14% on an
// eighth-angle shard; at coarse levels (n < 256) the staging delay costs more
// than the overlap gains, so the two chains start together there.
// With value-plane staging the whole-set forward's CTAs are small enough to
// share the SMs at n = 256 as well (f=4 step on one GPU 238 -> 229 us without
// the wait), so there the order applies from n = 512; an angle shard keeps it
// from n = 256 (1/8 shard, f=4: 53 us with the wait, 63 us without).
bool adjoint_after_staging(const imask_plan* pl, int level0) {
  const int forced = knob(Knob::kAdjAfterStageMinN, 0);
  const int min_n = forced > 0 ? forced : (2 * pl->n_loc > pl->n_angles ? 512 : 256);
  return pl->side / pl->factors[level0] >= min_n;
}

// TMA staging pays off where the band walks are long; coarse grids use L1 loads
bool forward_uses_tma(const imask_plan* pl, const LevelTables* t, int n) {
  return t->tma && pl->tma_entries && n >= knob(Knob::kTmaMinN, 128);
}

bool forward_quad_l1(const imask_plan* pl) {
  return pl->tma_quad && !knob(Knob::kNoQuadL1, 0);
}

// Whether the forward run_forward picks at this level reads the difference
// planes PM / PTM: the value-plane kernels form the differences from P / PT,
// so k_prepare skips those two planes for them (half its writes).
bool forward_reads_diff(const imask_plan* pl, const LevelTables* t, int n) {
  if (!pl->sym) return false;  // plain layout: P holds (u, d) pairs itself
  if (forward_uses_tma(pl, t, n))
    return !t->two_det && !forward_tma_val_grid(pl->n_det, pl->n_tma_entries);
  if (forward_quad_l1(pl)) return !forward_l1_val();
  return true;  // k_forward_sym
}

// The prebuilt chunk tables, when they match the kernel this launch picks (the
// path switches can be re-read after the plan was built: chunk sizes differ
// between the value-plane and the two-plane kernels).
const int* forward_tables(const imask_plan* pl, const LevelTables* t) {
  if (!t->fwd_tab || !knob(Knob::kFwdTables, 1)) return nullptr;
  const bool val = t->two_det || forward_tma_val_grid(pl->n_det, pl->n_tma_entries);
  return val == t->fwd_tab_val ? t->fwd_tab : nullptr;
}

int prepare_for_forward(imask_plan* pl, const LevelTables* t, const float* u, int n,
                        cudaStream_t s) {
  LAUNCH(launch_prepare(u, n, pl->P, pl->PT, pl->PM, pl->PTM, forward_reads_diff(pl, t, n), s),
         "prepare");
  return IMASK_OK;
}

int run_forward(imask_plan* pl, int f, const LevelTables* t, float* sino, const SinoSaga* saga,
                cudaStream_t s) {
  const int n = pl->side / f;
  ++g_launches;
  cudaError_t e;
  if (forward_uses_tma(pl, t, n))
    e = launch_forward_tma(t->maps, pl->P, pl->PT, pl->PM, pl->PTM, n, t->fwd, pl->tma_entries,
                           pl->n_tma_entries, pl->tma_row_ctas, pl->tma_quad, pl->n_det, sino,
                           saga, s, t->two_det, forward_tables(pl, t), nullptr);
  else {
    const bool quad = forward_quad_l1(pl);
    e = launch_forward(pl->P, pl->PT, pl->PM, pl->PTM, n, t->fwd, pl->n_loc, pl->n_det,
                       pl->fwd_entries, pl->n_entries, quad ? pl->tma_entries : nullptr,
                       pl->n_tma_entries, sino, saga, s);
  }
  return cuda_check(e, "forward");
}

int check_factor(const imask_plan* pl, int f) {
  if (f < 1 || pl->side % f != 0)
    return fail(IMASK_EINVAL, "side " + std::to_string(pl->side) + " not divisible by factor " +
                                  std::to_string(f));
  return IMASK_OK;
}

int check_params(const imask_step_params* prm) {
  if (!prm) return fail(IMASK_EINVAL, "null step parameters");
  if (!(prm->sigma > 0.0) || !(prm->g_kind == 1 || prm->mu_g > 0.0))
    return fail(IMASK_EINVAL, "sigma and mu_g must be positive");
  if (!(prm->mu > 0.0)) return fail(IMASK_EINVAL, "mu must be positive");
  if (prm->g_kind == 1 && (!(prm->tv_mu > 0.0) || prm->tv_iters < 0 || !prm->tv_scratch))
    return fail(IMASK_EINVAL, "TV step needs tv_mu > 0, tv_iters >= 0 and tv_scratch");
  if (prm->g_kind != 0 && prm->g_kind != 1) return fail(IMASK_EINVAL, "unknown g_kind");
  return IMASK_OK;
}

int check_level0(const imask_plan* pl, int level0) {
  if (level0 < 0 || level0 >= pl->r)
    return fail(IMASK_ELEVEL, "level " + std::to_string(level0 + 1) + " out of range 1.." +
                                  std::to_string(pl->r));
  return IMASK_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

}  // namespace

namespace {

int step_image(imask_plan* pl, const imask_state* st, int level0, const imask_step_params* prm,
               float* xbar, double theta, void* stream, int planes = 0);

// Restriction (or compensation at the full level) of x into pl->u, then the
// pair images of the forward projector.
int stage_forward_input(imask_plan* pl, const float* x, int level0, cudaStream_t s) {
  const int f = pl->factors[level0];
  const int n = pl->side / f;
  if (pl->n_loc > 0 && pl->sym && knob(Knob::kFusedStage, 1) != 0 &&
      stage32_ok(pl->side, f, pl->r)) {
    LevelTables* t;
    int rc;
    if ((rc = get_tables(pl, f, &t))) return rc;
    if (!forward_reads_diff(pl, t, n)) {
      // value-plane forwards: x -> P, PT in one kernel (restriction or
      // compensation fused into the pair-plane staging)
      LAUNCH(launch_stage32(x, pl->side, f, pl->cp, pl->P, pl->PT, s), "stage");
      return IMASK_OK;
    }
  }
  if (level0 < pl->r - 1)
    LAUNCH(launch_restrict(x, pl->u, pl->side, f, s), "restrict");
  else
    LAUNCH(launch_compensate(x, pl->u, pl->side, pl->cp, s), "compensate");
  if (pl->n_loc == 0) return IMASK_OK;
  LevelTables* t;
  int rc;
  if ((rc = get_tables(pl, f, &t))) return rc;
  return prepare_for_forward(pl, t, pl->u, n, s);
}

// psi_new = K_i u on this slab fused with the sinogram-side SAGA update.
int forward_saga(imask_plan* pl, const imask_state* st, int level0, const imask_step_params* prm,
                 const LevelTables* t, cudaStream_t stream, bool in_place = false) {
  if (pl->n_loc == 0) return IMASK_OK;
  const int f = pl->factors[level0];
  int rc;
  const size_t m = (size_t)pl->n_loc * pl->n_det;
  SinoSaga sg;
  sg.psi_tab = st->psi_tab + (size_t)level0 * m;
  sg.psi_sum = st->psi_sum;
  sg.y_in = st->y;
  sg.y = st->y_next && !in_place ? st->y_next : st->y;
  sg.b = st->b;
  sg.p_i = (float)pl->probs[level0];
  sg.sigma = (float)prm->sigma;
  sg.inv_1ps = (float)(1.0 / (1.0 + prm->sigma));
  const int split_forced = knob(Knob::kSagaSplitMinN, 0);
  // measured: a win from n = 1024 with the two-plane forward; with value-plane
  // staging (the whole angle set) from n = 512 too (f=2 step 401 -> 378 us)
  const int split_min_n =
      split_forced > 0 ? split_forced : (2 * pl->n_loc > pl->n_angles ? 512 : 1024);
  if (pl->side / f >= split_min_n) {
    // large levels: projection into scratch, then the update as its own pass
    if ((rc = run_forward(pl, f, t, pl->sino_tmp, nullptr, S(stream)))) return rc;
    LAUNCH(launch_saga_sino(pl->sino_tmp, m, sg, S(stream)), "saga_sino");
    return IMASK_OK;
  }
  if ((rc = run_forward(pl, f, t, nullptr, &sg, S(stream)))) return rc;
  return IMASK_OK;
}

}  // namespace

extern "C" {

const char* imask_version(void) { return "imask_b200 0.1 (sm_100a)"; }
const char* imask_last_error(void) { return g_err.c_str(); }
int imask_last_launch_count(void) { return g_launches; }

int imask_plan_create(int side, int n_angles, int n_det, int angle_begin, int angle_end,
                      const double* cos_tab, const double* sin_tab, int r, const double* probs,
                      double scale, int device, imask_plan** out) {
  g_err.clear();
  if (angle_begin < 0 || angle_end > n_angles || angle_begin > angle_end) {
    if (out) *out = nullptr;
    return fail(IMASK_EINVAL, "angle slab [" + std::to_string(angle_begin) + ", " +
                                  std::to_string(angle_end) + ") outside 0.." +
                                  std::to_string(n_angles));
  }
  std::vector<int> idx;
  for (int a = angle_begin; a < angle_end; ++a) idx.push_back(a);
  return imask_plan_create_list(side, n_angles, n_det, (int)idx.size(), idx.data(), cos_tab,
                                sin_tab, r, probs, scale, device, out);
}

int imask_plan_create_list(int side, int n_angles, int n_det, int n_loc, const int* angle_idx,
                           const double* cos_tab, const double* sin_tab, int r,
                           const double* probs, double scale, int device, imask_plan** out) {
  g_err.clear();
  g_launches = 0;
  if (!out) return fail(IMASK_EINVAL, "out must not be null");
  *out = nullptr;
  if (side < 1) return fail(IMASK_EINVAL, "side must be positive");
  if (n_angles < 1 || n_det < 1) return fail(IMASK_EINVAL, "n_angles and n_det must be positive");
  if (n_loc < 0 || n_loc > n_angles || (n_loc > 0 && !angle_idx))
    return fail(IMASK_EINVAL, "bad angle list");
  {
    std::vector<char> seen(n_angles, 0);
    for (int i = 0; i < n_loc; ++i) {
      const int a = angle_idx[i];
      if (a < 0 || a >= n_angles || seen[a])
        return fail(IMASK_EINVAL, "angle list entry " + std::to_string(a) +
                                      " out of range or repeated");
      seen[a] = 1;
    }
  }
  if (r < 1 || r > 7) return fail(IMASK_EINVAL, "levels r must be in 1..7");
  const int coarsest = 1 << (r - 1);
  if (side % coarsest != 0)
    return fail(IMASK_EINVAL, "side " + std::to_string(side) + " not divisible by 2^(r-1) = " +
                                  std::to_string(coarsest));
  double psum = 0.0;
  for (int i = 0; i < r; ++i) {
    if (!(probs[i] > 0.0)) return fail(IMASK_EINVAL, "all probabilities must be positive");
    psum += probs[i];
  }
  if (std::fabs(psum - 1.0) > 1e-12)
    return fail(IMASK_EINVAL, "probabilities sum to " + std::to_string(psum) + ", expected 1");
  if ((n_loc > 0) && (!cos_tab || !sin_tab)) return fail(IMASK_EINVAL, "angle tables missing");
  for (int a = 0; a < n_loc; ++a)
    if (cos_tab[a] == 0.0 && sin_tab[a] == 0.0)
      return fail(IMASK_EINVAL, "angle with cos = sin = 0");

  DeviceGuard g(device);
  init_kernel_attributes();
  imask_plan* pl = new imask_plan();
  pl->side = side;
  pl->n_angles = n_angles;
  pl->n_det = n_det;
  pl->angle_idx.assign(angle_idx, angle_idx + n_loc);
  pl->n_loc = n_loc;
  pl->r = r;
  pl->device = device;
  pl->scale = scale;
  pl->probs.assign(probs, probs + r);
  pl->cosv.assign(cos_tab, cos_tab + n_loc);
  pl->sinv.assign(sin_tab, sin_tab + n_loc);
  long long off = 0;
  pl->cp.r = r;
  pl->rp.r = r;
  for (int i = 0; i < r; ++i) {
    const int f = 1 << (r - 1 - i);
    pl->factors.push_back(f);
    pl->phi_off.push_back(off);
    const long long n = side / f;
    pl->cp.p[i] = (float)probs[i];
    pl->rp.p[i] = (float)probs[i];
    pl->rp.factor[i] = f;
    pl->rp.offset[i] = off;
    // rows start 16-byte aligned (the 128-bit image-side kernels read them as
    // float4: 3^2 + 6^2 + ... of a 96^2 / r = 6 family is not a multiple of 4)
    off = (off + n * n + 3) & ~3LL;
  }
  pl->cp.pr = (float)probs[r - 1];

  const size_t pair_bytes = sizeof(float2) * (size_t)side * pair_pitch(side);
  const size_t img_bytes = sizeof(float) * (size_t)side * side;
  const size_t sino_bytes = sizeof(float) * (size_t)n_loc * n_det;
  int rc = IMASK_OK;
  // Mirror symmetry (theta -> pi - theta is angle a -> n_angles - a): usable when
  // the local rows are [angle 0 (optional)] + a list whose row i holds the
  // mirror of row sym_s + n_loc - 1 - i (the full set 0..n-1 and the
  // mirror-closed shards of shard_angles both have this layout).
  pl->sym = false;
  for (int s0 = 0; s0 <= 1 && !pl->sym; ++s0) {
    if (n_loc - s0 < 2 || (s0 == 1 && angle_idx[0] != 0)) continue;
    bool ok = true;
    for (int i = s0; i < n_loc && ok; ++i) {
      const int a = angle_idx[i], am = angle_idx[s0 + n_loc - 1 - i];
      ok = a != 0 && am == n_angles - a;
    }
    if (ok) {
      pl->sym = true;
      pl->sym_s = s0;
    }
  }
  if (pl->sym) {
    std::vector<int2> ent;  // local rows (row, mirror row or -1)
    for (int i = 0; i < pl->sym_s; ++i) ent.push_back(make_int2(i, -1));  // angle 0 alone:
                                                                         // tie rule not mirror-invariant
    for (int i = pl->sym_s; i < n_loc; ++i) {
      const int im = pl->sym_s + n_loc - 1 - i;
      if (i < im) ent.push_back(make_int2(i, im));
      else if (i == im) ent.push_back(make_int2(i, -1));  // self-mirrored (pi/2)
    }
    pl->n_entries = (int)ent.size();
    // TMA forward: 8 entries of one ray family per CTA (rows vs columns of the image)
    std::vector<int2> rowf, colf;
    for (const int2& e2 : ent)
      (std::fabs(cos_tab[e2.x]) >= std::fabs(sin_tab[e2.x]) ? rowf : colf).push_back(e2);
    std::vector<int2> tent;
    for (auto* lst : {&rowf, &colf}) {
      for (const int2& e2 : *lst) tent.push_back(e2);
      const size_t fe = (size_t)forward_tma_entries_per_cta();
      while (tent.size() % fe) tent.push_back(make_int2(-1, -1));
      if (lst == &rowf) pl->tma_row_ctas = (int)(tent.size() / fe);
    }
    // quad mode when every row's transpose partner n/2 - a (pi/2 - theta) is local
    // too: the singles 0 and n/2 (a transposed-family entry), entries
    // (a, n-a, n/2-a, n/2+a) for 0 < a < n/4, then the pair (n/4, 3n/4)
    std::vector<int4> qent;
    if (n_angles % 4 == 0 && !knob(Knob::kNoQuad, 0)) {
      std::vector<int> loc(n_angles, -1);
      for (int i = 0; i < n_loc; ++i) loc[angle_idx[i]] = i;
      const int h = n_angles / 2, qn = n_angles / 4;
      int covered = 0;
      bool ok = true;
      // the axis singles first, beside the near-axis quads (a CTA's lanes walk
      // one lockstep band range, so its entries must be geometrically close)
      if (loc[0] >= 0) {
        qent.push_back(make_int4(loc[0], -1, -1, -1));
        ++covered;
      }
      if (loc[h] >= 0) {
        qent.push_back(make_int4(-1, -1, loc[h], -1));
        ++covered;
      }
      for (int a = 1; a < qn && ok; ++a) {
        const int r0 = loc[a], r1 = loc[n_angles - a], r2 = loc[h - a], r3 = loc[h + a];
        const int have = (r0 >= 0) + (r1 >= 0) + (r2 >= 0) + (r3 >= 0);
        if (have == 0) continue;
        if (have != 4) ok = false;
        qent.push_back(make_int4(r0, r1, r2, r3));
        covered += 4;
      }
      if (ok && loc[qn] >= 0 && loc[3 * qn] >= 0) {
        qent.push_back(make_int4(loc[qn], loc[3 * qn], -1, -1));
        covered += 2;
      } else if (loc[qn] >= 0 || loc[3 * qn] >= 0) {
        ok = false;
      }
      if (!ok || covered != n_loc) qent.clear();
    }
    std::vector<int4> tent4;
    if (!qent.empty()) {
      pl->tma_quad = true;
      tent4 = qent;
      const size_t fe = (size_t)forward_tma_entries_per_cta();
      while (tent4.size() % fe) tent4.push_back(make_int4(-1, -1, -1, -1));
      pl->tma_row_ctas = (int)(tent4.size() / fe);
    } else {
      for (const int2& e2 : tent) tent4.push_back(make_int4(e2.x, e2.y, -1, -1));
    }
    pl->n_tma_entries = (int)tent4.size();
    pl->tma_entries_host = tent4;
    if ((rc = cuda_check(cudaMalloc(&pl->tma_entries, sizeof(int4) * tent4.size()), "cudaMalloc")) ||
        (rc = cuda_check(cudaMemcpy(pl->tma_entries, tent4.data(), sizeof(int4) * tent4.size(),
                                    cudaMemcpyHostToDevice),
                         "cudaMemcpy"))) {
      imask_plan_destroy(pl);
      return rc;
    }
    if ((rc = cuda_check(cudaMalloc(&pl->fwd_entries, sizeof(int2) * ent.size()), "cudaMalloc")) ||
        (rc = cuda_check(cudaMemcpy(pl->fwd_entries, ent.data(), sizeof(int2) * ent.size(),
                                    cudaMemcpyHostToDevice),
                         "cudaMemcpy"))) {
      imask_plan_destroy(pl);
      return rc;
    }
  }
  if ((rc = cuda_check(cudaMalloc(&pl->P, pair_bytes), "cudaMalloc P")) ||
      (rc = cuda_check(cudaMalloc(&pl->PT, pair_bytes), "cudaMalloc PT")) ||
      (pl->sym && (rc = cuda_check(cudaMalloc(&pl->PM, pair_bytes), "cudaMalloc PM"))) ||
      (pl->sym && (rc = cuda_check(cudaMalloc(&pl->PTM, pair_bytes), "cudaMalloc PTM"))) ||
      (rc = cuda_check(cudaMalloc(&pl->u, img_bytes), "cudaMalloc u")) ||
      (rc = cuda_check(cudaMalloc(&pl->sino_tmp, sino_bytes > 0 ? sino_bytes : 4),
                       "cudaMalloc sino"))) {
    imask_plan_destroy(pl);
    return rc;
  }
  if ((rc = cuda_check(cudaStreamCreateWithFlags(&pl->aux.stream, cudaStreamNonBlocking),
                       "side stream")) ||
      (rc = cuda_check(cudaEventCreateWithFlags(&pl->aux.fork, cudaEventDisableTiming), "event")) ||
      (rc = cuda_check(cudaEventCreateWithFlags(&pl->aux.join, cudaEventDisableTiming), "event")) ||
      (rc = cuda_check(cudaStreamCreateWithFlags(&pl->aux2.stream, cudaStreamNonBlocking),
                       "side stream")) ||
      (rc = cuda_check(cudaEventCreateWithFlags(&pl->aux2.fork, cudaEventDisableTiming), "event")) ||
      (rc = cuda_check(cudaEventCreateWithFlags(&pl->aux2.join, cudaEventDisableTiming), "event")) ||
      (rc = cuda_check(cudaEventCreateWithFlags(&pl->ev_staged, cudaEventDisableTiming), "event"))) {
    imask_plan_destroy(pl);
    return rc;
  }
  pl->scratch = (int64_t)((pl->sym ? 4 : 2) * pair_bytes + img_bytes + sino_bytes);
  for (int f : pl->factors) {
    LevelTables* t;
    if ((rc = get_tables(pl, f, &t)) || (rc = ensure_partial(pl, f))) {
      imask_plan_destroy(pl);
      return rc;
    }
  }
  *out = pl;
  return IMASK_OK;
}

int imask_debug_bounds(unsigned long long* out4, int reset) {
  if (!out4) return fail(IMASK_EINVAL, "out4 is null");
  // projector.cu's counters, then sketch.cu's (the first failing site wins)
  unsigned long long b[4] = {0, 0, 0, 0};
  const bool on = debug_bounds_read_projector(out4, reset != 0);
  debug_bounds_read_sketch(b, reset != 0);
  if (out4[0] == ~0ull || b[0] == ~0ull) {
    const unsigned long long* bad = out4[0] == ~0ull ? out4 : b;
    return fail(IMASK_ECUDA, std::string("bounds counters unreadable (") +
                                 (out4[0] == ~0ull ? "projector" : "sketch") + ", " +
                                 (bad[2] == 1 ? "synchronize" : "memcpy") + ": " +
                                 cudaGetErrorString((cudaError_t)bad[1]) + ")");
  }
  if (out4[0] == 0) {
    out4[1] = b[1];
    out4[2] = b[2];
    out4[3] = b[3];
  }
  out4[0] += b[0];
  return on ? 1 : 0;
}

int imask_reload_switches(void) {
  std::lock_guard<std::mutex> lk(g_knob_mu);
  read_knobs();
  return IMASK_OK;
}

int imask_plan_destroy(imask_plan* pl) {
  if (!pl) return IMASK_OK;
  DeviceGuard g(pl->device);
  for (auto& kv : pl->tables) {
    cudaFree(kv.second.fwd);
    cudaFree(kv.second.adj);
    cudaFree(kv.second.fwd_tab);
  }
  cudaFree(pl->P);
  cudaFree(pl->PT);
  cudaFree(pl->PM);
  cudaFree(pl->PTM);
  cudaFree(pl->fwd_entries);
  cudaFree(pl->tma_entries);
  cudaFree(pl->u);
  cudaFree(pl->sino_tmp);
  cudaFree(pl->adj_partial);
  for (float* p : pl->retired) cudaFree(p);
  if (pl->aux.stream) cudaStreamDestroy(pl->aux.stream);
  if (pl->aux.fork) cudaEventDestroy(pl->aux.fork);
  if (pl->aux.join) cudaEventDestroy(pl->aux.join);
  if (pl->aux2.stream) cudaStreamDestroy(pl->aux2.stream);
  if (pl->aux2.fork) cudaEventDestroy(pl->aux2.fork);
  if (pl->aux2.join) cudaEventDestroy(pl->aux2.join);
  if (pl->ev_staged) cudaEventDestroy(pl->ev_staged);
  delete pl;
  return IMASK_OK;
}

int64_t imask_plan_scratch_bytes(const imask_plan* pl) { return pl ? pl->scratch : 0; }
int imask_plan_symmetric(const imask_plan* pl) {
  return !pl || !pl->sym ? 0 : (pl->tma_quad ? 2 : 1);
}

int imask_project(imask_plan* pl, int factor, const float* u, int64_t u_len, float* sino,
                  int64_t sino_len, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_factor(pl, factor);
  if (rc) return rc;
  const int n = pl->side / factor;
  if (u_len != (int64_t)n * n)
    return fail(IMASK_EDIM, "operator expects domain dim " + std::to_string((int64_t)n * n) +
                                ", got vector of length " + std::to_string(u_len));
  if (sino_len != (int64_t)pl->n_loc * pl->n_det)
    return fail(IMASK_EDIM, "operator expects range dim " +
                                std::to_string((int64_t)pl->n_loc * pl->n_det) +
                                ", got vector of length " + std::to_string(sino_len));
  DeviceGuard g(pl->device);
  LevelTables* t;
  if ((rc = get_tables(pl, factor, &t))) return rc;
  if (pl->n_loc == 0) return IMASK_OK;
  if ((rc = prepare_for_forward(pl, t, u, n, S(stream)))) return rc;
  if ((rc = run_forward(pl, factor, t, sino, nullptr, S(stream)))) return rc;
  return IMASK_OK;
}

int imask_backproject(imask_plan* pl, int factor, const float* sino, int64_t sino_len, float* u,
                      int64_t u_len, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_factor(pl, factor);
  if (rc) return rc;
  const int n = pl->side / factor;
  if (sino_len != (int64_t)pl->n_loc * pl->n_det)
    return fail(IMASK_EDIM, "operator adjoint expects range dim " +
                                std::to_string((int64_t)pl->n_loc * pl->n_det) +
                                ", got vector of length " + std::to_string(sino_len));
  if (u_len != (int64_t)n * n)
    return fail(IMASK_EDIM, "operator adjoint output has domain dim " +
                                std::to_string((int64_t)n * n) + ", got buffer of length " +
                                std::to_string(u_len));
  DeviceGuard g(pl->device);
  LevelTables* t;
  if ((rc = get_tables(pl, factor, &t))) return rc;
  if (pl->n_loc == 0) {
    LAUNCH(cudaMemsetAsync(u, 0, sizeof(float) * n * n, S(stream)), "memset");
    return IMASK_OK;
  }
  if ((rc = ensure_partial(pl, factor))) return rc;
  return run_adjoint(pl, factor, sino, u, t->adj, S(stream));
}

int imask_restrict(int side, int factor, const float* x, float* u, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (side < 1 || factor < 1 || side % factor != 0)
    return fail(IMASK_EINVAL, "side " + std::to_string(side) + " not divisible by factor " +
                                  std::to_string(factor));
  LAUNCH(launch_restrict(x, u, side, factor, S(stream)), "restrict");
  return IMASK_OK;
}

int imask_prolong(int side, int factor, const float* u, float* x, float alpha, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (side < 1 || factor < 1 || side % factor != 0)
    return fail(IMASK_EINVAL, "side " + std::to_string(side) + " not divisible by factor " +
                                  std::to_string(factor));
  LAUNCH(launch_prolong(u, x, side, factor, alpha, S(stream)), "prolong");
  return IMASK_OK;
}

int imask_compensate(int side, int r, const double* probs, const float* x, float* out,
                     void* stream) {
  g_err.clear();
  g_launches = 0;
  if (r < 1 || r > 7) return fail(IMASK_EINVAL, "levels r must be in 1..7");
  if (side < 1 || side % (1 << (r - 1)) != 0)
    return fail(IMASK_EINVAL, "side " + std::to_string(side) + " not divisible by 2^(r-1) = " +
                                  std::to_string(1 << (r - 1)));
  CompParams cp{};
  cp.r = r;
  for (int i = 0; i < r; ++i) cp.p[i] = (float)probs[i];
  cp.pr = (float)probs[r - 1];
  LAUNCH(launch_compensate(x, out, side, cp, S(stream)), "compensate");
  return IMASK_OK;
}

int imask_sketch_forward(imask_plan* pl, int level, const float* x, float* sino, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level - 1);
  if (rc) return rc;
  DeviceGuard g(pl->device);
  const int f = pl->factors[level - 1];
  const int n = pl->side / f;
  LevelTables* t;
  if ((rc = get_tables(pl, f, &t))) return rc;
  if (level < pl->r)
    LAUNCH(launch_restrict(x, pl->u, pl->side, f, S(stream)), "restrict");
  else
    LAUNCH(launch_compensate(x, pl->u, pl->side, pl->cp, S(stream)), "compensate");
  if (pl->n_loc == 0) return IMASK_OK;
  if ((rc = prepare_for_forward(pl, t, pl->u, n, S(stream)))) return rc;
  if ((rc = run_forward(pl, f, t, sino, nullptr, S(stream)))) return rc;
  return IMASK_OK;
}

int imask_sketch_adjoint(imask_plan* pl, int level, const float* sino, float* out,
                         void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level - 1);
  if (rc) return rc;
  DeviceGuard g(pl->device);
  const int f = pl->factors[level - 1];
  const int n = pl->side / f;
  LevelTables* t;
  if ((rc = get_tables(pl, f, &t))) return rc;
  if (pl->n_loc == 0)
    LAUNCH(cudaMemsetAsync(pl->u, 0, sizeof(float) * n * n, S(stream)), "memset");
  else
    if ((rc = run_adjoint(pl, f, sino, pl->u, t->adj, S(stream)))) return rc;
  if (level < pl->r)
    LAUNCH(launch_prolong(pl->u, out, pl->side, f, 1.0f / (float)(f * f), S(stream)), "prolong");
  else
    LAUNCH(launch_compensate(pl->u, out, pl->side, pl->cp, S(stream)), "compensate");
  return IMASK_OK;
}

int imask_draw_levels(uint64_t seed, int64_t k0, int64_t count, const double* cum_probs, int r,
                      int32_t* out) {
  g_err.clear();
  if (r < 1 || !cum_probs || (count > 0 && !out)) return fail(IMASK_EINVAL, "bad arguments");
  for (int64_t n = 0; n < count; ++n) {
    const double u = imask_uniform_at(seed, k0 + n);
    int idx = 0;
    while (idx < r && cum_probs[idx] <= u) ++idx;  // searchsorted(..., side="right")
    out[n] = idx < r - 1 ? idx : r - 1;
  }
  return IMASK_OK;
}

double imask_uniform_at(uint64_t seed, int64_t k) {
  uint64_t z = mix64(seed + kGolden * (uint64_t)(k + 1));
  z = mix64(z + kGolden);
  return (double)(z >> 11) * 0x1.0p-53;
}

int imask_step_adjoint(imask_plan* pl, const imask_state* st, int level0, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  DeviceGuard g(pl->device);
  const int f = pl->factors[level0];
  const int n = pl->side / f;
  LevelTables* t;
  if ((rc = get_tables(pl, f, &t))) return rc;
  if (pl->n_loc == 0)
    LAUNCH(cudaMemsetAsync(st->bp, 0, sizeof(float) * n * n, S(stream)), "memset");
  else
    if ((rc = run_adjoint(pl, f, st->y, st->bp, t->adj, S(stream)))) return rc;
  return IMASK_OK;
}

int imask_step_forward(imask_plan* pl, const imask_state* st, int level0,
                       const imask_step_params* prm, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  if (!(prm->sigma > 0.0)) return fail(IMASK_EINVAL, "sigma must be positive");
  DeviceGuard g(pl->device);
  const int f = pl->factors[level0];
  LevelTables* t;
  if ((rc = get_tables(pl, f, &t))) return rc;
  if ((rc = stage_forward_input(pl, st->x, level0, S(stream)))) return rc;
  cudaEventRecord(pl->ev_staged, S(stream));  // for imask_step_wait_staging
  return forward_saga(pl, st, level0, prm, t, S(stream));
}

int imask_step_wait_staging(imask_plan* pl, int level0, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  if (!adjoint_after_staging(pl, level0)) return IMASK_OK;
  return cuda_check(cudaStreamWaitEvent(S(stream), pl->ev_staged, 0), "wait staging");
}

int imask_step_image(imask_plan* pl, const imask_state* st, int level0,
                     const imask_step_params* prm, void* stream) {
  return step_image(pl, st, level0, prm, nullptr, 0.0, stream);
}

int imask_seq_step(imask_plan* pl, const imask_state* st, int level0,
                   const imask_step_params* prm, double theta, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  if ((rc = check_params(prm))) return rc;
  if (!(theta >= 0.0 && theta <= 1.0)) return fail(IMASK_EINVAL, "theta_extrap must lie in [0, 1]");
  if (!st->xbar) return fail(IMASK_EINVAL, "sketch_seq_step needs st->xbar");
  DeviceGuard g(pl->device);
  const int f = pl->factors[level0];
  const int n = pl->side / f;
  LevelTables* t;
  if ((rc = get_tables(pl, f, &t))) return rc;
  const cudaStream_t s = S(stream);
  // forward memory from the extrapolated point, dual first (in place) ...
  if ((rc = stage_forward_input(pl, st->xbar, level0, s))) return rc;
  if ((rc = forward_saga(pl, st, level0, prm, t, s, true))) return rc;
  // ... then the adjoint memory from the new dual, the primal step and xbar
  if (pl->n_loc == 0)
    LAUNCH(cudaMemsetAsync(st->bp, 0, sizeof(float) * n * n, s), "memset");
  else if ((rc = run_adjoint(pl, f, st->y, st->bp, t->adj, s)))
    return rc;
  const int launches = g_launches;
  if ((rc = step_image(pl, st, level0, prm, st->xbar, theta, stream))) return rc;
  g_launches += launches;
  return IMASK_OK;
}

}  // extern "C"

namespace {

int step_image(imask_plan* pl, const imask_state* st, int level0, const imask_step_params* prm,
               float* xbar, double theta, void* stream, int planes) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  if ((rc = check_params(prm))) return rc;
  DeviceGuard g(pl->device);
  const int f = pl->factors[level0];
  ImageSaga sg;
  sg.xbar = xbar;
  sg.theta = (float)theta;
  sg.phi_tab = st->phi_tab + pl->phi_off[level0];
  sg.phi_sum = st->phi_sum;
  sg.x = st->x;
  if (planes > 0) {
    const int n = pl->side / f;
    // the full-level kernel sums planes in order only; many planes over few
    // pixels (the reduce kernels' warp-tree order) keep the explicit reduction
    const bool warp_order = planes >= 32 && (long long)n * n <= 65536;
    const bool fused = pl->side % 32 == 0 &&
                       (level0 < pl->r - 1 ? (f <= 32 && 32 % f == 0) : (pl->r <= 6 && !warp_order));
    if (fused) {  // the adjoint's split planes, reduced inside the image kernel
      sg.planes = pl->adj_partial;
      sg.n_planes = planes;
      sg.plane_len = (long long)n * n;
    } else {
      LAUNCH(launch_adjoint_reduce(pl->adj_partial, st->bp, n * n, planes, S(stream)), "reduce");
    }
  }
  sg.p_i = (float)pl->probs[level0];
  const double s = prm->sigma / prm->mu;
  const bool tv = prm->g_kind == 1;
  sg.s = (float)s;
  sg.inv_den = tv ? 1.0f : (float)(1.0 / (1.0 + s * prm->mu_g));  // TV: x - s xi, prox below
  if (tv && xbar) return fail(IMASK_EINVAL, "the sequential variant takes the ridge g only");
  if (level0 < pl->r - 1)
    LAUNCH(launch_saga_image_coarse(st->bp, pl->side, f, sg, S(stream)), "saga_image");
  else
    LAUNCH(launch_saga_image_full(st->bp, pl->side, pl->cp, sg, S(stream)), "saga_image_full");
  if (tv) {
    // x' = prox_{s g}(x - s xi) in place: memset + tv_iters iterations + recovery
    const int trc = imask_prox_tv_nonneg(pl->side, st->x, st->x, s, prm->tv_mu, prm->tv_iters,
                                         prm->tv_tol, prm->tv_scratch, stream);
    if (trc) return fail(trc, std::string("prox_tv_nonneg: ") + cudaGetErrorString(cudaGetLastError()));
    g_launches += prm->tv_iters + 1;  // iteration kernels + the recovery (plus one memset)
  }
  return IMASK_OK;
}

}  // namespace

extern "C" {

int imask_sketch_step(imask_plan* pl, const imask_state* st, int level0,
                      const imask_step_params* prm, void* stream) {
  g_err.clear();
  g_launches = 0;
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  if ((rc = check_params(prm))) return rc;
  DeviceGuard g(pl->device);
  const int f = pl->factors[level0];
  const int n = pl->side / f;
  LevelTables* t;
  if ((rc = get_tables(pl, f, &t))) return rc;
  const cudaStream_t s = S(stream);
  int planes = 0;  // > 0: the adjoint's split planes are left for the image kernel to sum
  if (pl->n_loc == 0) {
    LAUNCH(cudaMemsetAsync(st->bp, 0, sizeof(float) * n * n, s), "memset");
  } else if (st->y_next) {
    // double-buffered dual: the whole forward chain (staging + projection +
    // sinogram-side update into y_next) overlaps the adjoint of y^k; the image
    // update waits for the adjoint and for the staging's read of x
    cudaEventRecord(pl->aux2.fork, s);
    cudaStreamWaitEvent(pl->aux2.stream, pl->aux2.fork, 0);
    if ((rc = stage_forward_input(pl, st->x, level0, pl->aux2.stream))) return rc;
    cudaEventRecord(pl->ev_staged, pl->aux2.stream);
    if ((rc = forward_saga(pl, st, level0, prm, t, pl->aux2.stream))) return rc;
    cudaEventRecord(pl->aux2.join, pl->aux2.stream);
    const bool after = adjoint_after_staging(pl, level0);
    if (after) cudaStreamWaitEvent(s, pl->ev_staged, 0);
    if ((rc = run_adjoint(pl, f, st->y, st->bp, t->adj, s, &planes))) return rc;
    if (!after) cudaStreamWaitEvent(s, pl->ev_staged, 0);
    const int launches = g_launches;
    if ((rc = step_image(pl, st, level0, prm, nullptr, 0.0, stream, planes))) return rc;
    g_launches += launches;
    cudaStreamWaitEvent(s, pl->aux2.join, 0);
    return cuda_check(cudaGetLastError(), "fork/join");
  } else {
    // the forward's input staging (restriction / compensation + pair images)
    // reads only x, so it runs on the side stream while the adjoint reads y
    cudaEventRecord(pl->aux.fork, s);
    cudaStreamWaitEvent(pl->aux.stream, pl->aux.fork, 0);
    if ((rc = stage_forward_input(pl, st->x, level0, pl->aux.stream))) return rc;
    if ((rc = run_adjoint(pl, f, st->y, st->bp, t->adj, s, &planes))) return rc;
    cudaEventRecord(pl->aux.join, pl->aux.stream);
    cudaStreamWaitEvent(s, pl->aux.join, 0);
    if ((rc = cuda_check(cudaGetLastError(), "fork/join"))) return rc;
    if ((rc = forward_saga(pl, st, level0, prm, t, s))) return rc;
  }
  const int launches = g_launches;
  if ((rc = step_image(pl, st, level0, prm, nullptr, 0.0, stream, planes))) return rc;
  g_launches += launches;
  return IMASK_OK;
}

namespace {

// Capture one imask_sketch_step into a new graph (not instantiated).
int capture_step(imask_plan* pl, const imask_state* st, int level0, const imask_step_params* prm,
                 cudaGraph_t* graph, int* launches) {
  cudaStream_t s;
  int rc;
  if ((rc = cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create")))
    return rc;
  *graph = nullptr;
  rc = cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
  int step_rc = IMASK_OK;
  if (!rc) step_rc = imask_sketch_step(pl, st, level0, prm, s);
  const int n_launch = g_launches;
  const std::string step_err = g_err;
  cudaError_t end = rc ? cudaSuccess : cudaStreamEndCapture(s, graph);
  if (!rc && step_rc) rc = fail(step_rc, step_err);
  if (!rc) rc = cuda_check(end, "end capture");
  cudaStreamDestroy(s);
  if (rc && *graph) {
    cudaGraphDestroy(*graph);
    *graph = nullptr;
  }
  if (launches) *launches = n_launch;
  return rc;
}

}  // namespace

int imask_step_graph_create(imask_plan* pl, const imask_state* st, int level0,
                            const imask_step_params* prm, imask_graph** out, int* launches) {
  g_err.clear();
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  if (!out) return fail(IMASK_EINVAL, "out must not be null");
  DeviceGuard g(pl->device);
  imask_graph* gr = new imask_graph();
  gr->device = pl->device;
  int n_launch = 0;
  rc = capture_step(pl, st, level0, prm, &gr->graph, &n_launch);
  if (!rc) rc = cuda_check(cudaGraphInstantiate(&gr->exec, gr->graph, 0), "graph instantiate");
  // upload the executable graph now, so its first launch does not pay for it
  if (!rc) rc = cuda_check(cudaGraphUpload(gr->exec, pl->aux2.stream), "graph upload");
  if (rc) {
    imask_graph_destroy(gr);
    return rc;
  }
  *out = gr;
  if (launches) *launches = n_launch;
  g_launches = 0;
  return IMASK_OK;
}

int imask_step_graph_update(imask_graph* gr, imask_plan* pl, const imask_state* st, int level0,
                            const imask_step_params* prm) {
  g_err.clear();
  if (!gr) return fail(IMASK_EINVAL, "null graph");
  int rc = check_level0(pl, level0);
  if (rc) return rc;
  DeviceGuard g(pl->device);
  cudaGraph_t fresh = nullptr;
  if ((rc = capture_step(pl, st, level0, prm, &fresh, nullptr))) return rc;
  // same topology, new kernel arguments: patch the executable graph in place
  cudaGraphExecUpdateResultInfo info;
  if (cudaGraphExecUpdate(gr->exec, fresh, &info) != cudaSuccess) {
    cudaGetLastError();  // clear the update failure; instantiate afresh
    cudaGraphExec_t exec = nullptr;
    rc = cuda_check(cudaGraphInstantiate(&exec, fresh, 0), "graph instantiate");
    if (rc) {
      cudaGraphDestroy(fresh);
      return rc;
    }
    cudaGraphExecDestroy(gr->exec);
    gr->exec = exec;
    if ((rc = cuda_check(cudaGraphUpload(gr->exec, pl->aux2.stream), "graph upload"))) {
      cudaGraphDestroy(fresh);
      return rc;
    }
  }
  if (gr->graph) cudaGraphDestroy(gr->graph);
  gr->graph = fresh;
  g_launches = 0;
  return IMASK_OK;
}

int imask_graph_launch(imask_graph* gr, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (!gr) return fail(IMASK_EINVAL, "null graph");
  return cuda_check(cudaGraphLaunch(gr->exec, S(stream)), "graph launch");
}

int imask_graph_destroy(imask_graph* gr) {
  if (!gr) return IMASK_OK;
  DeviceGuard g(gr->device);
  if (gr->exec) cudaGraphExecDestroy(gr->exec);
  if (gr->graph) cudaGraphDestroy(gr->graph);
  delete gr;
  return IMASK_OK;
}

int imask_pdhg_step(imask_plan* pl, const imask_pdhg_state* st, const imask_pdhg_params* prm,
                    void* stream) {
  g_err.clear();
  g_launches = 0;
  if (!pl || !st || !prm) return fail(IMASK_EINVAL, "null argument");
  if (!(prm->sigma > 0.0) || !(prm->tau > 0.0) || !(prm->mu_g > 0.0))
    return fail(IMASK_EINVAL, "sigma, tau and mu_g must be positive");
  DeviceGuard g(pl->device);
  const int n = pl->side;
  LevelTables* t;
  int rc;
  if ((rc = get_tables(pl, 1, &t))) return rc;
  const cudaStream_t s = S(stream);
  if (pl->n_loc > 0) {
    // dual step: K xbar fused with the conjugate prox in the forward epilogue
    if ((rc = prepare_for_forward(pl, t, st->xbar, n, s))) return rc;
    SinoSaga sg{};
    sg.psi_tab = nullptr;  // no SAGA tables: zeta = K xbar
    sg.psi_sum = nullptr;
    sg.y_in = st->y;
    sg.y = st->y;
    sg.b = st->b;
    sg.sigma = (float)prm->sigma;
    sg.inv_1ps = (float)(1.0 / (1.0 + prm->sigma));
    if ((rc = run_forward(pl, 1, t, nullptr, &sg, s))) return rc;
    // primal step from the new dual
    if ((rc = run_adjoint(pl, 1, st->y, st->bp, t->adj, s))) return rc;
  } else {
    LAUNCH(cudaMemsetAsync(st->bp, 0, sizeof(float) * n * n, s), "memset");
  }
  LAUNCH(launch_pdhg_image(st->bp, st->x, st->xbar, (size_t)n * n, (float)prm->tau,
                           (float)(1.0 / (1.0 + prm->tau * prm->mu_g)), (float)prm->theta, s),
         "pdhg image");
  return IMASK_OK;
}

int imask_resum(imask_plan* pl, const imask_state* st, void* stream) {
  g_err.clear();
  g_launches = 0;
  DeviceGuard g(pl->device);
  const size_t m = (size_t)pl->n_loc * pl->n_det;
  ++g_launches;
  LAUNCH(launch_resum(st->phi_tab, st->phi_sum, pl->side, st->psi_tab, st->psi_sum, m, pl->rp,
                      S(stream)),
         "resum");
  return IMASK_OK;
}

}  // extern "C"
