/* ===========================================================================
 * sss.h — C ABI of the B200-native hot path of Student Splatting and Scooping
 * (SSS, arXiv 2503.10148).  Citations "PAPER.md:l" are lines of the paper's
 * text; "Rnn" are the readings listed in
 * DESIGN.md §1 where the paper is silent or ambiguous.
 *
 * Conventions common to every entry point
 * ---------------------------------------
 *  - All array pointers are DEVICE pointers (CUDA global memory) unless the
 *    argument is marked "host".  Every call is asynchronous on `stream`
 *    (a cudaStream_t passed as void*; NULL = the legacy default stream).
 *  - Ownership: the caller allocates and frees every buffer.  The library
 *    allocates nothing and keeps no global mutable state, so calls on
 *    different streams may run concurrently.  Workspaces are sized by the
 *    matching *_workspace() query.
 *  - Component parameters are SoA planes of stride n (sss_params): plane p of
 *    component i is at base[p * n + i].  With K = (D+1)^2 SH coefficients per
 *    channel: mean[3], log_scale[3], rot[4] (w,x,y,z, not necessarily unit),
 *    raw_nu[1], raw_opacity[1], sh[3K] (plane 3k + channel).  When the six
 *    pointers are consecutive slices of one allocation the whole set is a
 *    single flat buffer of (12 + 3K) * n floats (used for the NCCL all-reduce).
 *  - Errors: argument validation returns synchronously (SSS_ERR_ARG /
 *    SSS_ERR_SHAPE) and launches nothing; a failed launch returns
 *    SSS_ERR_CUDA; sss_last_error() gives a thread-local message.
 *    Instance overflow in sss_bin_sort is reported on the device (see there).
 * ======================================================================== */
#ifndef SSS_H_
#define SSS_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SSS_API __attribute__((visibility("default")))
#else
#define SSS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SSS_OK = 0,
  SSS_ERR_ARG = 1,      /* null pointer, n < 0, sh_degree outside [0,3], bad camera */
  SSS_ERR_SHAPE = 2,    /* zero-size image, views of different sizes, too many bins */
  SSS_ERR_CAPACITY = 3, /* bin capacity exceeded (sss_check_overflow) */
  SSS_ERR_CUDA = 4      /* CUDA launch / runtime error */
} sss_status;

#define SSS_TILE 16          /* tile edge in pixels */
#define SSS_MAX_BINS 5632    /* bins per view (tiles >> bin_shift); bounded by the scatter CTA's shared memory */
#define SSS_REC_FLOATS 8     /* floats per projected geometry record (32 B) */
#define SSS_COL_FLOATS 4     /* floats per projected colour record (16 B) */
#define SSS_G2D_FLOATS 10    /* floats per screen-space gradient record (40 B) */
#define SSS_TILE_LISTS 2     /* composited-entry lists per tile (one per 16x8 strip) */

/* Pinhole camera (host struct).  p_cam = rot * x + trans (rot row-major,
 * world->camera; OpenCV axes x right, y down, z forward).  Pixel (i, j) has its
 * centre at (i + 1/2, j + 1/2).  Eq. 4's W, t and the perspective Jacobian J
 * (R4, R5); z_near culls components (R24). */
typedef struct {
  float rot[9];
  float trans[3];
  float fx, fy, cx, cy;
  int32_t width, height;
  float z_near;
} sss_camera;

/* Component parameters ("mean mu, covariance Sigma (S and R),
 * colour c, opacity o, degree parameter nu"), device SoA planes, see above.
 * nu = min(1 + softplus(raw_nu), 1e4) (R1); o = tanh(raw_opacity)
 * (R2); S = diag(exp(log_scale)) (R3); R = R(q / |q|).
 * The same struct describes gradients and Adam moments (same layout).
 * variant: 0 for SSS, or the paper's ablation variants (PAPER.md:1109-1111,
 * R32) as SSS_VARIANT_* flags; every entry point taking the parameter set
 * honours them (the projected records carry the kernel). */
#define SSS_VARIANT_POSITIVE 1 /* o = sigmoid(raw_opacity): "positive t-dis" (settings 1-2) */
#define SSS_VARIANT_GAUSSIAN 2 /* 3DGS Gaussian kernel exp(-h/2) (nu unused; inv_nu = 0 in the record) */
#define SSS_VARIANT_LOWPASS 4  /* +0.3 on the diagonal of Sigma2D (setting 1) */
/* block > 0 (gradients only: sss_render_bwd's grad, sss_project_bwd_range's
 * grad, sss_sghmc_step's grad): component-blocked layout for the overlapped
 * multi-GPU exchange.  The set is then one flat buffer at `mean` of
 * ceil(n / block) blocks of [block_planes][block] floats (block_planes >=
 * 12 + 3K, the rest padding): plane p of component i is at
 * mean[(i / block) * block_planes * block + p * block + i % block]; the other
 * five pointers are ignored.  A block is contiguous, so its exchange can
 * start as soon as the components of that block are done.  Everywhere else
 * block must be 0. */
typedef struct {
  int64_t n;
  int32_t sh_degree;
  int32_t variant;
  float* mean;
  float* log_scale;
  float* rot;
  float* raw_nu;
  float* raw_opacity;
  float* sh;
  int64_t block;
  int32_t block_planes;
  int32_t reserved;
} sss_params;

/* Per-(view, component) projection (output of sss_project).
 *  rec   [V][n][8] floats: {mx, my, A, B2}, {C, hmax, o, inv_nu} with
 *        (A, B2/2, C) the conic (Sigma2D)^-1 and hmax the L9 cutoff --
 *        32-byte records, so the geometry of a component is one sector
 *  col   [V][n][4] floats: {e, r, g, b}, e = -(nu+2)/2 and (r,g,b) the
 *        clamped SH colour (the compositors' third record)
 *  depth [V][n] camera-space z of the mean, fp32 (the sort key source, R8).
 *  rect  [V][n][4] int16 inclusive tile rect x0,y0,x1,y1; x0 > x1 = culled.
 * Memory: 60 B per (view, component). */
typedef struct {
  int64_t n;
  int32_t n_views;
  int32_t reserved;
  float* rec;
  float* depth;
  int16_t* rect;
  float* col;
} sss_projected;

/* Depth-ordered bin lists (output of sss_bin_sort).  A bin is a square of
 * 2^bin_shift x 2^bin_shift tiles; bin_shift = 0 gives the classic per-tile
 * lists.  For view v the entries of bin b are ids[v*capacity + ranges[2(v*nb+b)]
 * ... + ranges[2(v*nb+b)+1]) in (depth, index) order (R8).
 *  ids      [V][capacity] component indices
 *  keys     nullable [V][capacity]: bin << 32 | float bits of depth
 *  ranges   [V][n_bins][2] start, end (absolute offsets within the view)
 *  totals   [V] instance count of the view (written even on overflow)
 *  max_per_bin  0: every list is complete.  > 0: truncated lists -- bin b
 *           holds only the first min(len_b, max_per_bin) entries of its list
 *           (a pixel stops after W < 1e-4, R11, so the raster reads only a
 *           front part of each list: ~2 % of the entries at config 5).  The
 *           raster then continues a truncated list, for a tile that still has
 *           a live pixel at its end, with sorted[v][resume[v][b] ...
 *           n_vis[v]) filtered by the tile rect, which is exactly the rest of
 *           the tile's list; images and gradients are unchanged.
 *  sorted   [V][n] (nullable if max_per_bin == 0): the view's visible
 *           components in (depth, index) order (first n_vis[v] entries)
 *  n_vis    [V] (nullable if max_per_bin == 0): visible components per view
 *  resume   [V][n_bins] (nullable if max_per_bin == 0): position in sorted
 *           one past the bin's last materialised entry; n_vis[v] if the
 *           list is complete
 *  used     [V][n_bins] nullable: adaptive truncation.  sss_render_fwd with
 *           these bins writes each bin's consumption (the list length its
 *           tiles needed: up to the last composited entry if every pixel of
 *           the tile stopped, 2^30 if some pixel is still live at the end);
 *           the next sss_bin_sort caps bin b at min(max_per_bin, 1.25 used + 256)
 *           (no cap for used < 0 or >= 2^30: initialise to -1) and resets
 *           used to 0 for the forward that follows.  Truncation (either
 *           kind) never changes the raster's results; a tile that needs
 *           more than its bin kept reads the tail (slower).
 *  tmask    [V][capacity] nullable (bin_shift <= 2; needs pr->rec): per
 *           materialised entry, bit ly * 2^bin_shift + lx is set for the
 *           tiles of its bin whose 16x16 block of pixel centres the
 *           component's h <= hmax ellipse (R9) may reach -- conservative:
 *           a cleared bit guarantees no pixel of that tile passes the
 *           raster's fp32 inclusion test; a set bit may be a tile it misses
 *           (also outside the tile rect).  The raster filters a bin's listed
 *           entries by this bit instead of by the tile rect (a truncated
 *           list's tail stays rect-filtered), which drops the rect's false
 *           positives (~43 % of the entries a config-5 forward tile visits)
 *           before they are staged; results are unchanged.  Computed by
 *           sss_bin_sort after the scatter (one extra kernel).
 *  overflow [1] set to 1 if any totals[v] > capacity (then nothing is
 *           scattered for that view and its ranges are empty; grow and
 *           retry).  Sticky: sss_bin_sort only ever sets it; the caller
 *           zeroes it (so one check after many calls sees every overflow;
 *           sss_sghmc_step can be told to skip its update when it is set). */
typedef struct {
  int32_t bin_shift;
  int32_t n_views;
  int64_t capacity;
  int32_t* ids;
  uint64_t* keys;
  int32_t* ranges;
  int64_t* totals;
  int32_t* overflow;
  int32_t max_per_bin;
  int32_t reserved;
  int32_t* sorted;
  int32_t* n_vis;
  int32_t* resume;
  int32_t* used;
  uint16_t* tmask;
} sss_bins;

/* Rendered frames (output of sss_render_fwd; all views share one size).
 *  rgb       [V][3][H][W]  C(u) of Eq. 7 + bg * W (unclamped, R21)
 *  final_T   [V][H][W]     final transmittance W
 *  n_contrib [V][H][W]     number of composited (included) components (R23);
 *                          optional diagnostic: NULL = not counted (the backward
 *                          does not read it)
 *  last      [V][H][W]     private: bin-list offset one past the last
 *                          composited entry (start of the backward replay)
 *  tile_list [V][tiles][SSS_TILE_LISTS][tile_cap],
 *  tile_count [V][tiles][SSS_TILE_LISTS]: private, nullable (both or
 *            neither): per 16x8 strip of a tile (rows 0-7, rows 8-15), the
 *            bin-list offsets of the entries some pixel of the strip
 *            composited, in order; the backward replays only those (a strip
 *            with tile_count > tile_cap falls back to the full range) */
typedef struct {
  float* rgb;
  float* final_T;
  int32_t* n_contrib;
  int32_t* last;
  int32_t* tile_list;
  int32_t* tile_count;
  int32_t tile_cap;
  int32_t reserved;
} sss_frame;

/* Hyper-parameters of one sampler step (host struct; PAPER.md:151-163,
 * 1492-1523, R14-R19).  lr is eps of Eq. 10 (the mu step), noise the std eta
 * of the pre-gate mu noise (R15), gate = sigmoid(-gate_k (|o| - gate_t)) (R16),
 * grad_scale multiplies every gradient (1/V for the multi-view mean, R26). */
typedef struct {
  float lr, friction, noise, gate_k, gate_t;
  int32_t burn_in; /* 1: F dropped, noise premultiplied by Sigma (R18) */
  int32_t g_adam;  /* 1: use Adam's m^/(sqrt(v^)+eps) as g in the mu update (R17) */
  float lr_scale, lr_rot, lr_nu, lr_opacity, lr_sh;
  float beta1, beta2, adam_eps, grad_scale;
  int64_t step;    /* 1-based step (Adam bias correction, noise counter) */
  uint64_t seed;   /* Philox4x32-10 key */
  /* Eq. 8 regularizers (R27), folded into the step:
   * eps_o sum_i |o_i| adds eps_o sign(o)(1 - o^2) to d raw_opacity and
   * eps_sigma sum_ij sqrt(lambda_ij) adds eps_sigma exp(s_j) to d log_scale_j
   * (after grad_scale).  0, 0 = the BASELINE L1 objective. */
  float eps_o, eps_sigma;
  /* NEXT-3 mean update: 0 gated SGHMC (Eq. 10), 1 SGLD (F disabled,
   * PAPER.md:161), 2 Adam on the means with lr (setting 1's optimiser). */
  int32_t mu_mode;
  /* Plane range [plane_begin, plane_end) this call updates (0, 0 = all):
   * the ZeRO-1 sharded step of the multi-GPU path updates only the planes
   * its rank owns after a reduce-scatter of the gradient, then the ranks
   * all-gather the parameters (SURVEY.md §8(e) option 2).  Every plane's
   * update reads the pre-update parameters, so a split into ranges equals
   * the full update bit for bit. */
  int32_t plane_begin, plane_end;
  int32_t reserved;
  /* Device int32 flag (nullable): if *skip_if != 0 when the kernel runs, the
   * step writes nothing (pass sss_bins.overflow so an iteration whose
   * binning overflowed -- its views rendered as background -- never moves
   * the parameters, moments or momentum; the caller grows and replays). */
  const int32_t* skip_if;
  /* Device sss_step_state (nullable): if set, the 1-based step is read from
   * step_state->step on the device (hp->step is ignored) and incremented by
   * the call, so a CUDA graph that captured the call replays successive
   * steps (host values are frozen in a captured launch). */
  struct sss_step_state* step_state;
} sss_sghmc_hparams;

/* Device-resident step counter of a graph-captured sampler (see above).
 * Initialise step to the first step (>= 1); the rest is scratch. */
typedef struct sss_step_state {
  int64_t step;
  float inv_b1t, inv_b2t;  /* 1 / (1 - beta^t) of the step being applied */
  uint32_t ctr2, ctr3;     /* Philox counter words (the step) */
  int64_t reserved;
} sss_step_state;

/* flags for sss_render_bwd */
#define SSS_BWD_NU_GRAD_PAPER 1 /* use the printed dT/dnu of PAPER.md:1301-1314 (R13) */
#define SSS_BWD_RASTER_ONLY 2   /* run only the a4 raster half (fills the workspace) */
#define SSS_BWD_PROJECTION_ONLY 4 /* run only the a5 projection half (consumes it) */
#define SSS_BWD_TARGET_U8 16    /* target is uint8 [V][3][H][W] (8-bit images, as the
                                   paper's datasets): value u / 255 (fp32, correctly
                                   rounded division) -- a quarter of the bytes */
#define SSS_BWD_GRAD_ASSIGN 8   /* grad = result instead of grad += result: every
                                   component's gradient is written (zeros where no
                                   view touched it) and the old contents are not
                                   read -- saves zeroing grad before a one-batch step */

/* a1 — projection of every component into V views (Eq. 4,
 * 1116-1215 SM forward, 1077-1079 nu range / truncation / no low-pass).
 * p: device params; cams: host array of n_views cameras (all the same size);
 * out: device buffers sized as documented at sss_projected.
 * Returns SSS_ERR_ARG / SSS_ERR_SHAPE on invalid input. */
SSS_API sss_status sss_project(const sss_params* p, const sss_camera* cams, int32_t n_views,
                       sss_projected* out, void* stream);

/* Bytes of device scratch sss_bin_sort needs for n components, n_views views
 * of cams[0]'s size and the given bin_shift.  0 on invalid input. */
SSS_API size_t sss_bin_sort_workspace(int64_t n, int32_t n_views, const sss_camera* cams,
                              int32_t bin_shift);

/* a2 — bin every visible component into the bins its tile rect overlaps and
 * order each bin's list by (fp32 depth, component index) (R8).  Implements a
 * stable LSD radix sort of the depth keys followed by a stable counting
 * scatter by bin.  ws: device scratch of at least sss_bin_sort_workspace()
 * bytes.  out->bin_shift, capacity, ids, ranges, totals, overflow must be set
 * (keys optional; sorted, n_vis, resume required when max_per_bin > 0).
 * totals and the capacity count materialised entries.  Overflow is
 * device-side (see sss_bins).  SSS_ERR_SHAPE if
 * the view has more than SSS_MAX_BINS bins or more than 1024 bins along an
 * axis (raise bin_shift).  The capacity also sizes the scatter's shared-
 * memory stage (capacity / chunks of 1024 components); chunks above it take
 * a slower direct path, so size it near the instance count. */
SSS_API sss_status sss_bin_sort(const sss_projected* pr, const sss_camera* cams, int32_t n_views,
                        void* ws, size_t ws_bytes, sss_bins* out, void* stream);

/* Synchronising helper: waits for `stream`, returns SSS_ERR_CAPACITY if the
 * overflow flag of `bins` is set, SSS_OK otherwise. */
SSS_API sss_status sss_check_overflow(const sss_bins* bins, void* stream);

/* a3 — signed front-to-back compositing, Eq. 7:
 * per pixel, components of its tile in bin order that pass the fp32 gate
 * h <= hmax (R9) are composited with a = clamp(o T2D, -0.99, 0.99) (R10);
 * a pixel stops after the component that makes W < 1e-4 (R11); bg (host[3])
 * is added times the final W (R12). */
SSS_API sss_status sss_render_fwd(const sss_projected* pr, const sss_bins* bins, const sss_camera* cams,
                          int32_t n_views, const float* bg, sss_frame* out, void* stream);

/* Bytes of device scratch sss_render_bwd needs (screen-space gradient records
 * [V][n][SSS_G2D_FLOATS] floats, private layout: the geometry moments
 * sum dh (dx, dy, dx^2, dx dy, dy^2) (5), d colour (3), d o, d nu).  The scratch must be ZERO before the first call; every
 * call leaves it zero again (the projection-backward consumes and clears it). */
SSS_API size_t sss_render_bwd_workspace(int64_t n, int32_t n_views);

/* a4 + a5 (+ a6) — closed-form backward of
 * sss_render_fwd with gating frozen (R22), accumulated (+=) into grad over all
 * views.  Image gradient: d_rgb [V][3][H][W] if non-NULL, else the fused L1
 * loss against target [V][3][H][W] (fp32, or uint8 with SSS_BWD_TARGET_U8):
 * dL/dC = sign(C - target) / (3 H W) per
 * view (Eq. 8's L1 term, R20); in that case loss_out (device float[1],
 * nullable) is incremented by sum_v mean|C - target|.  fwd must be the
 * output of sss_render_fwd for the same inputs.  flags: SSS_BWD_*. */
SSS_API sss_status sss_render_bwd(const sss_params* p, const sss_projected* pr, const sss_bins* bins,
                          const sss_camera* cams, int32_t n_views, const float* bg,
                          const sss_frame* fwd, const float* d_rgb, const void* target,
                          float* loss_out, sss_params* grad, void* ws, size_t ws_bytes,
                          int32_t flags, void* stream);

/* a5 alone, for the components [i0, i1): the projection backward (see
 * sss_render_bwd) consuming and clearing their screen-space gradient records
 * in ws (filled by sss_render_bwd with SSS_BWD_RASTER_ONLY) and adding their
 * parameter gradients to grad (plain or component-blocked layout).  Calls for
 * disjoint ranges may be issued one after the other so that each block's
 * gradient exchange overlaps the next block's computation. */
SSS_API sss_status sss_project_bwd_range(const sss_params* p, const sss_camera* cams, int32_t n_views,
                                         void* ws, size_t ws_bytes, sss_params* grad, int64_t i0, int64_t i1,
                                         void* stream);

/* Bytes of device scratch sss_image_loss needs for n_views views of
 * height x width (the three SSIM partial-derivative maps over the valid
 * window positions).  0 on invalid input. */
SSS_API size_t sss_image_loss_workspace(int32_t n_views, int32_t height, int32_t width);

/* NEXT-1 — image part of Eq. 8 for a batch of views:
 *   L_v = (1 - eps_dssim) mean|C - T| + eps_dssim (1 - SSIM(C, T)),
 * SSIM the mean over channels and valid 11x11 window positions of the local
 * SSIM with a Gaussian window (sigma 1.5, K1 0.01, K2 0.03, range 1; R28).
 * rgb, target: [V][3][H][W] device; d_rgb (out, overwritten): dL_v/dC in the
 * same layout, ready for sss_render_bwd's d_rgb; loss (device float[1],
 * nullable) is incremented by sum_v L_v.  eps_dssim in [0, 1]; with
 * eps_dssim > 0 both sides must be >= 11 pixels (else SSS_ERR_SHAPE).
 * ws: at least sss_image_loss_workspace() bytes. */
SSS_API sss_status sss_image_loss(const float* rgb, const float* target, int32_t n_views, int32_t height,
                                  int32_t width, float eps_dssim, float* d_rgb, float* loss, void* ws,
                                  size_t ws_bytes, void* stream);

/* Settings of one recycling pass (host struct; R29-R31). */
typedef struct {
  float threshold; /* dead iff |o| < threshold (0.005, the gate threshold) */
  float cap_frac;  /* at most floor(cap_frac * n) dead relocated per pass (0.05) */
  int32_t n_max;   /* at most n_max members per group incl. the target, in [2, 64] (R29) */
  int32_t reserved;
  uint64_t seed;   /* Philox4x32-10 key of the multinomial draws */
  int64_t step;    /* draw counter (the pass's iteration number) */
} sss_relocate_params;

/* Bytes of device scratch sss_relocate needs for n components. */
SSS_API size_t sss_relocate_workspace(int64_t n);

/* NEXT-2 — one component-recycling pass in place (PAPER.md:168-183 Eqs.
 * 11-12, 1317-1460; 1081 multinomial over opacity).  Dead components
 * (|o| < threshold) are moved onto live targets drawn with probability
 * proportional to |o|; each group of N members (target + dead) takes the
 * target's mean, rotation, nu and SH, o_new with (1 - o_new)^N = 1 - o_old
 * and Sigma_new = o_old^2 (beta(1/2,(nu+2)/2)/K)^2 Sigma_old (Eq. 12,
 * nu_new = nu_old); momentum and Adam moments of the members are reset.
 * p, adam_m, adam_v must each be one flat [P][n] device buffer (planes
 * consecutive, as sss_params documents); momentum [3][n].  target_of
 * (device int32[n], nullable): the target of every relocated component, -1
 * elsewhere.  n_moved (device int64[1]): number relocated.  n < 2^31. */
SSS_API sss_status sss_relocate(sss_params* p, sss_params* adam_m, sss_params* adam_v, float* momentum,
                                const sss_relocate_params* rp, int32_t* target_of, int64_t* n_moved,
                                void* ws, size_t ws_bytes, void* stream);

/* a7 — one sampler step in place (Eq. 10, 1492-1523; Adam on
 * every non-mean group).  p, adam_m, adam_v: device
 * planes (same n / sh_degree); grad read-only; momentum [3][n] device; hp host.
 * Noise: Philox4x32-10 keyed by hp->seed, counter (i, hp->step) (R14). */
SSS_API sss_status sss_sghmc_step(sss_params* p, const sss_params* grad, sss_params* adam_m,
                          sss_params* adam_v, float* momentum, const sss_sghmc_hparams* hp,
                          void* stream);

/* Measurement infrastructure (not on the hot path): microbenchmarks of the
 * current device's FP32 pipe and MUFU throughput (the
 * roofline denominators are measured, not assumed).  out (host double[7]):
 * scalar FFMA lane-ops/s, FFMA2 lane-ops/s (2 per lane), MUFU ex2, lg2 and
 * rcp ops/s, SM count, SM clock in kHz.  Synchronous; ~0.1 s.  0 = ok. */
SSS_API int sss_alu_peaks(double* out);

SSS_API const char* sss_status_string(sss_status s);
SSS_API const char* sss_last_error(void);
/* Number of kernel launches issued by this thread since the last reset. */
SSS_API int64_t sss_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* SSS_H_ */
