/*
 * imask_b200.h -- C-ABI of the B200-native ImaSk hot path (arXiv 2412.10249).
 *
 * Drop-in boundary for the reference package `mrtomo` (pure Python/scipy,
 * /root/reference/pkg/src/mrtomo). Each entry point names the reference
 * interface it replaces (file:line relative to pkg/src/mrtomo). All device
 * buffers are caller-owned CUDA allocations passed as plain pointers; all
 * calls are stream-ordered and asynchronous (no host sync) unless noted;
 * `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *
 * Layouts (float32 everywhere):
 *   image   side x side, row-major, y increasing with row   (ctmodel.py:76-79)
 *   coarse  (side/f) x (side/f), same convention, pixel width f (ctmodel.py:194-204)
 *   sino    n_loc x n_det, angle-major, detector fastest     (ctmodel.py:176)
 *           n_loc = angle_end - angle_begin (this rank's angle slab)
 *
 * Return codes: IMASK_OK, or one of the IMASK_E* codes below with a message
 * retrievable through imask_last_error() (thread-local). The Python host maps
 * IMASK_EDIM to linops.DimensionMismatch and IMASK_EINVAL / IMASK_ELEVEL to
 * ValueError with the reference's messages (linops.py:19-55, mrsketch.py:120-122).
 */
#ifndef IMASK_B200_H
#define IMASK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IMASK_API __attribute__((visibility("default")))

#define IMASK_OK 0
#define IMASK_EINVAL 1 /* invalid argument / configuration      -> ValueError        */
#define IMASK_EDIM 2   /* vector length does not match geometry  -> DimensionMismatch */
#define IMASK_ELEVEL 3 /* sketch level out of range 1..r         -> ValueError        */
#define IMASK_ECUDA 4  /* CUDA runtime error                     -> RuntimeError      */
#define IMASK_MAX_LEVELS 12

/* Opaque plan; owns the per-angle tables and device scratch (staged pair
 * images, sinogram staging, adjoint split planes). The scratch is shared by
 * every call on the plan, so calls on one plan must be stream-ordered with
 * respect to each other (one stream, or caller-ordered streams); use one plan
 * per concurrent stream. */
typedef struct imask_plan imask_plan;

/* Solver state of one rank: every pointer is a device buffer.
 * Mirrors SaddleState (solvers.py:119-140) with compact coarse phi rows:
 *   x, phi_sum           : side*side
 *   phi_tab              : level i (1-based) holds (side/f_i)^2 values at
 *                          offset o_i, o_1 = 0, o_{i+1} = o_i + (side/f_i)^2
 *                          rounded up to a multiple of 4 (rows start 16-byte
 *                          aligned); total o_{r+1}. Rows hold U_f^T-scaled
 *                          coarse values; the reference stores the same
 *                          values replicated to full resolution
 *   y, b, psi_sum        : n_loc*n_det (this rank's slab)
 *   psi_tab              : r * n_loc*n_det, level i at offset (i-1)*n_loc*n_det
 *   bp                   : side*side scratch for the (partial) backprojection
 *   y_next               : n_loc*n_det or NULL (see below) */
typedef struct imask_state {
  float* x;
  float* y;
  const float* b;
  float* phi_sum;
  float* psi_sum;
  float* phi_tab;
  float* psi_tab;
  float* bp;
  /* Optional second dual buffer (n_loc*n_det). When set, the forward writes
   * y^{k+1} here instead of updating y in place, so imask_sketch_step runs
   * the forward concurrently with the adjoint (which reads y^k); the caller
   * swaps y and y_next after each step. NULL: in-place update. */
  float* y_next;
  /* Extrapolated primal point of the sequential variant (imask_seq_step):
   * side*side, or NULL. */
  float* xbar;
} imask_state;

/* Per-iteration scalars of sketch_step (solvers.py:194-221) with the ridge
 * prox (proxlib.py:51-63) and the quadratic-data conjugate prox
 * (proxlib.py:30-48). */
typedef struct imask_step_params {
  double sigma; /* dual step sigma; primal step is sigma/mu */
  double mu;    /* solver strong-convexity parameter mu      */
  double mu_g;  /* ridge weight of g(x) = mu_g/2 ||x||^2      */
  /* g_kind 1: g = TV + nonnegativity (tv_nonneg_fn, proxlib.py:151-166) with
   * weight tv_mu instead of the ridge: the primal step is then
   * x' = prox_tv_nonneg(x - s xi, s) (imask_prox_tv_nonneg, tv_iters inner
   * iterations, tolerance tv_tol, device scratch tv_scratch of
   * imask_prox_tv_scratch_bytes(side) bytes); mu_g is ignored. 0: ridge. */
  int g_kind;
  int tv_iters;
  double tv_tol;
  double tv_mu;
  void* tv_scratch;
} imask_step_params;

/* Library version string. */
IMASK_API const char* imask_version(void);
/* Message of the last failing call on this thread ("" if none). */
IMASK_API const char* imask_last_error(void);

/* ---- plan ------------------------------------------------------------- */

/* Geometry + sketch family of one rank. Replaces Geometry (ctmodel.py:38-70),
 * the per-geometry projector cache _projector_pair (ctmodel.py:157-167) and
 * the SketchFamily probabilities/factors (mrsketch.py:76-118).
 *   side, n_angles, n_det : Geometry(side, n_angles, n_detectors)
 *   angle_begin/end       : this rank's contiguous angle slab [begin, end)
 *   cos_tab, sin_tab      : float64 cos/sin of the slab's angles a*pi/n_angles,
 *                           ALREADY snapped to 0 below 1e-14 (ctmodel.py:88-93);
 *                           a ray family is axis-parallel iff one is exactly 0
 *   r, probs              : levels and selection probabilities (level i has
 *                           factor 2^(r-i), mrsketch.py:107-109)
 *   scale                 : operator scale (1/||K|| when normalised,
 *                           expcli.py:173-180; 1.0 otherwise)
 *   device                : CUDA device ordinal the plan lives on            */
IMASK_API int imask_plan_create(int side, int n_angles, int n_det, int angle_begin,
                                int angle_end, const double* cos_tab, const double* sin_tab,
                                int r, const double* probs, double scale, int device,
                                imask_plan** out);
/* Same, for an arbitrary set of angles: local sinogram row i holds global
 * angle angle_idx[i] (distinct, in [0, n_angles)); cos_tab / sin_tab are in
 * local row order. Mirror-symmetric kernels are used when the rows are
 * [angle 0 (optional)] followed by a list whose row i is the mirror
 * (n_angles - a) of row (first + last - i), as the full set and the
 * mirror-closed multi-GPU shards are (paper_2412_10249_b200.ctmodel.shard_angles). */
IMASK_API int imask_plan_create_list(int side, int n_angles, int n_det, int n_loc,
                                     const int* angle_idx, const double* cos_tab,
                                     const double* sin_tab, int r, const double* probs,
                                     double scale, int device, imask_plan** out);
IMASK_API int imask_plan_destroy(imask_plan* plan);
/* 0: no mirror layout; 1: the plan's angle rows have the mirror layout above
 * (symmetric kernels in use); 2: in addition they are closed under the
 * transpose a -> n_angles/2 - a (four-ray TMA forward). */
IMASK_API int imask_plan_symmetric(const imask_plan* plan);
/* Scratch bytes the plan owns on the device (for memory accounting). */
IMASK_API int64_t imask_plan_scratch_bytes(const imask_plan* plan);

/* ---- projector (kernels 1 and 2) ------------------------------------ */

/* sino = R_f u : exact-chord forward projection of a coarse image.
 * Replaces coarse_projector(geom, f).apply (ctmodel.py:194-204) and, for
 * f = 1, projector_op(geom).apply / project (ctmodel.py:170-191). */
IMASK_API int imask_project(imask_plan* plan, int factor, const float* u, int64_t u_len,
                            float* sino, int64_t sino_len, void* stream);
/* u = R_f^T sino : matched pixel-driven backprojection, no atomics.
 * Replaces coarse_projector(geom, f).adjoint_apply and backproject
 * (ctmodel.py:179-185,194-204). */
IMASK_API int imask_backproject(imask_plan* plan, int factor, const float* sino,
                                int64_t sino_len, float* u, int64_t u_len, void* stream);

/* ---- sketch family (kernel 3) ----------------------------------------- */

/* u = T_f x (block mean).  Replaces decimate (mrsketch.py:23-32) and
 * decimate_op(side, f).apply (mrsketch.py:44-57). */
IMASK_API int imask_restrict(int side, int factor, const float* x, float* u, void* stream);
/* x = alpha * U_f u (replication).  alpha = 1: upsample (mrsketch.py:35-41);
 * alpha = 1/f^2: decimate_op adjoint (mrsketch.py:54-55). */
IMASK_API int imask_prolong(int side, int factor, const float* u, float* x, float alpha,
                            void* stream);
/* out = S_r x, the full-resolution compensation (mrsketch.py:133-153) of the
 * family (r, probs). S_r is symmetric, so this is also its adjoint
 * (mrsketch.py:155-160). Requires side % 2^(r-1) == 0, r <= 7. */
IMASK_API int imask_compensate(int side, int r, const double* probs, const float* x, float* out,
                               void* stream);
/* sino = K_i x and out = K_i^T sino for the sketched operator of level i
 * (1-based): coarse mode K_i = R_f T_f for i < r, K_r = K S_r
 * (sketch_forward, mrsketch.py:181-204). x / out are full resolution. */
IMASK_API int imask_sketch_forward(imask_plan* plan, int level, const float* x, float* sino,
                                   void* stream);
IMASK_API int imask_sketch_adjoint(imask_plan* plan, int level, const float* sino, float* out,
                                   void* stream);

/* ---- sketched SAGA iteration (kernel 4) -------------------------------- */

/* Host-side level schedule, bit-exact with draw_level (solvers.py:30-48):
 * out[n] = draw_level(seed, k0 + n, cum_probs) for n in [0, count).
 * cum_probs = numpy.cumsum(probs) (solvers.py:81). Pure host function. */
IMASK_API int imask_draw_levels(uint64_t seed, int64_t k0, int64_t count,
                                const double* cum_probs, int r, int32_t* out);
/* uniform_at(seed, k) (solvers.py:37-41). Pure host function. */
IMASK_API double imask_uniform_at(uint64_t seed, int64_t k);

/* One parallel ImaSk iteration at 0-based level index `level0` (the value
 * draw_level returns) on one GPU: replaces sketch_step (solvers.py:194-221)
 * minus the host bookkeeping (k, cost, resum cadence stay on the host).
 * Equivalent to step_adjoint + step_forward + step_image below; with
 * st->y_next set, the forward chain runs on a plan-owned side stream
 * concurrently with the adjoint (fork/join with events, so the call stays
 * stream-ordered and graph-capturable). */
IMASK_API int imask_sketch_step(imask_plan* plan, const imask_state* st, int level0,
                                const imask_step_params* prm, void* stream);
/* The three phases of one iteration, for angle-sharded multi-GPU runs:
 *  step_adjoint : st->bp = partial (this slab) coarse backprojection R_f^T y
 *                 (or K^T y at the full level), reads y^k.
 *  step_forward : psi_new = K_i x^k on this slab, fused with the sinogram-
 *                 side SAGA update (psi table row, psi_sum, y prox) writing
 *                 y^{k+1} to st->y_next (or in place when it is NULL, in
 *                 which case it must be enqueued after step_adjoint).
 *  step_image   : after st->bp has been all-reduced over ranks: phi_new,
 *                 phi table row, phi_sum and the x prox (x^k -> x^{k+1}).
 *                 Must be enqueued after step_forward's image read. */
IMASK_API int imask_step_adjoint(imask_plan* plan, const imask_state* st, int level0,
                                 void* stream);
IMASK_API int imask_step_forward(imask_plan* plan, const imask_state* st, int level0,
                                 const imask_step_params* prm, void* stream);
/* Step order (no reference counterpart: scheduling only): at large levels
 * (coarse side >= 256) makes `stream` wait until the input staging of the last
 * imask_step_forward on this plan is done, so an adjoint enqueued next on
 * `stream` starts after the forward kernel has its SM slots (see DESIGN.md,
 * step DAG); a no-op at coarse levels. */
IMASK_API int imask_step_wait_staging(imask_plan* plan, int level0, void* stream);
IMASK_API int imask_step_image(imask_plan* plan, const imask_state* st, int level0,
                               const imask_step_params* prm, void* stream);
/* One iteration of the deterministic primal-dual reference solver on the
 * unsketched operator K (the plan's f = 1 projector, with its scale),
 * replacing the loop body of pdhg_solve / run(..., "pdhg") (solvers.py:
 * 331-337, 433-446) for the ridge g and the quadratic-data conjugate f*:
 *   y    <- (y + sigma K xbar - sigma b) / (1 + sigma)
 *   x'   <- (x - tau K^T y) / (1 + tau mu_g)
 *   xbar <- x' + theta (x' - x);  x <- x'
 * Buffers: x, xbar, bp (scratch): side*side; y, b: n_loc*n_det. Single GPU
 * (the adjoint is not reduced over ranks). */
typedef struct imask_pdhg_state {
  float* x;
  float* xbar;
  float* y;
  const float* b;
  float* bp;
} imask_pdhg_state;
typedef struct imask_pdhg_params {
  double sigma, tau, theta; /* pdhg_parameters (solvers.py:308-318) */
  double mu_g;              /* ridge weight of g */
} imask_pdhg_params;
IMASK_API int imask_pdhg_step(imask_plan* plan, const imask_pdhg_state* st,
                              const imask_pdhg_params* prm, void* stream);
/* One sequential-update iteration with primal extrapolation, ImaSk-Seq
 * (sketch_seq_step, solvers.py:265-305): psi_new = K_i xbar with the
 * sinogram-side update and the dual prox (y in place), then phi_new =
 * K_i^T y_new with the image-side update and the primal prox, then
 * xbar = x' + theta (x' - x). theta in [0, 1]; st->xbar required. */
IMASK_API int imask_seq_step(imask_plan* plan, const imask_state* st, int level0,
                             const imask_step_params* prm, double theta, void* stream);
/* Recompute phi_sum / psi_sum from the tables in index order (_resum,
 * solvers.py:184-191). */
IMASK_API int imask_resum(imask_plan* plan, const imask_state* st, void* stream);

/* CUDA graph of one single-GPU iteration at level0 (imask_sketch_step with the
 * state pointers and scalars baked in), so a run loop issues one launch per
 * iteration. The graph stays valid while the plan and the state buffers live.
 * *launches receives the number of kernels one replay executes. */
typedef struct imask_graph imask_graph;
IMASK_API int imask_step_graph_create(imask_plan* plan, const imask_state* st, int level0,
                                      const imask_step_params* prm, imask_graph** out,
                                      int* launches);
/* Re-target an existing step graph to another state / step parameters of the
 * same plan and level (new kernel arguments, same topology): the graph is
 * re-captured and the executable graph patched in place (cudaGraphExecUpdate),
 * which costs a fraction of a fresh instantiation. */
IMASK_API int imask_step_graph_update(imask_graph* graph, imask_plan* plan,
                                      const imask_state* st, int level0,
                                      const imask_step_params* prm);
IMASK_API int imask_graph_launch(imask_graph* graph, void* stream);
IMASK_API int imask_graph_destroy(imask_graph* graph);

/* Number of kernel launches the last imask_* device call on this thread
 * enqueued (instrumentation for the benchmark's gpu_launches count). */
IMASK_API int imask_last_launch_count(void);

/* ||x - ref||^2 (ref may be NULL: ||x||^2) accumulated in float64 with a
 * fixed-order reduction, written to *result (a device double; NULL: out[0]);
 * `out` is device scratch of IMASK_SQDIST_SCRATCH doubles, ZERO-INITIALISED
 * before the first call (it holds a completion counter each call re-arms).
 * Backs the rel_dist / psnr columns of run()'s record rows (_metrics,
 * solvers.py:382-390) without a host sync. */
#define IMASK_SQDIST_SCRATCH 298
IMASK_API int imask_sq_dist(const float* x, const float* ref, int64_t n, double* out,
                            double* result, void* stream);
/* One metric row of run() (solvers.py:403-405) recorded on the device: with
 * k = rows[0] read as a uint64 counter, rows[2 + 2k] = ||x - ref||^2 (float64,
 * fixed order; n = 0 gives 0) and rows[3 + 2k] = the device global timer in ns
 * when it was final; the counter then advances. `rows` is device memory of
 * 2 + 2 * capacity doubles with rows[0] = 0 initially; `scratch` as for
 * imask_sq_dist. A run's rows are read back once at the end. */
IMASK_API int imask_metric_row(const float* x, const float* ref, int64_t n, double* scratch,
                               double* rows, void* stream);

/* TV + nonnegativity prox (prox_tv_nonneg, proxlib.py:102-148):
 * out = argmin_u 0.5||u - xp||^2 + sigma mu_g ||grad u||_{1,2} + [u >= 0]
 * by the fast gradient projection on the dual gradient field (step 1/8,
 * at most inner_iters iterations, stopping when the relative dual progress
 * drops below inner_tol), for a side x side image; out may alias xp.
 * `scratch` is device memory of imask_prox_tv_scratch_bytes(side) bytes. One
 * launch per inner iteration, no host synchronisation. */
IMASK_API int64_t imask_prox_tv_scratch_bytes(int side);
IMASK_API int imask_prox_tv_nonneg(int side, const float* xp, float* out, double sigma,
                                   double mu_g, int inner_iters, double inner_tol, void* scratch,
                                   void* stream);

/* Test / measurement helper (no reference counterpart): re-read the IMASK_*
 * path switches from the environment (imask_common.cuh lists them; they are
 * otherwise read once). Plans created afterwards use the new values. */
IMASK_API int imask_reload_switches(void);

/* Debug helper (no reference counterpart): the index checks of a library built
 * with -DIMASK_BOUNDS_CHECK=1 (every shared-memory window read of the
 * projectors and every pair-image read of the L1 forwards against the range
 * it must stay in). out4 = {violations, first site code, first index, first
 * limit}; reset != 0 clears the counter. Returns 1 when the checks are
 * compiled in, 0 when not (out4 zeroed), < 0 on error. */
IMASK_API int imask_debug_bounds(unsigned long long* out4, int reset);

/* Measurement helper (no reference counterpart): thread-level FP32 FFMA
 * throughput of `device` from an FFMA-chain microbenchmark, the FP32-issue
 * denominator of bench.py's roofline. */
IMASK_API int imask_probe_ffma_peak(int device, double* ffma_per_s);
/* Measurement helper: aggregate shared-memory read bandwidth of `device`
 * (conflict-free 128-bit loads on every SM), the denominator of the
 * projectors' shared-memory roofline in bench.py. */
IMASK_API int imask_probe_smem_peak(int device, double* bytes_per_s);

#ifdef __cplusplus
}
#endif
#endif /* IMASK_B200_H */
