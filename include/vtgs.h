/* vtgs.h — C ABI of the B200-native view-tied Gaussian splatting hot path.
 *
 * The one data-parallel hot path of VTGaussian-SLAM (arxiv 2506.02741): differentiable
 * splatting of view-tied isotropic 3D Gaussians — the render-and-backprop step that every
 * tracking (§3.3, Eq. 1) and mapping (§3.4, Eq. 2)
 * iteration repeats.  Five parts (BASELINE.json north_star):
 *   (1) vtgs_instantiate  — view-tied Gaussians from keyframe depth / RGB / pose
 *   (2) vtgs_render_fwd   — projection to an isotropic footprint + 16×16 tile binning,
 *   (3)                     device sort on (tile | depth),
 *   (4)                     per-tile front-to-back compositing of colour, depth, silhouette
 *   (5) vtgs_render_bwd   — reverse-order backward: colour / opacity / radius (mapping) and
 *                           6-DoF camera pose (tracking) gradients
 * Every stage is a hand-written sm_100a CUDA kernel in libvtgs.so.  There is no CPU fallback:
 * without a CUDA device every call returns VTGS_ERR_NO_DEVICE / VTGS_ERR_CUDA.
 *
 * Conventions (DESIGN.md §3 lists every reading of the paper taken here):
 *   - fp32 throughout.  Arrays are C-contiguous.  "float4[N]" means N×4 floats, 16-byte aligned.
 *   - Images are row-major H×W (colour H×W×3, interleaved), pixel (x, y) centred at integer
 *     coordinates, OpenCV camera axes (x right, y down, z forward).
 *   - A pose is camera-to-world: unit quaternion (w, x, y, z) + translation in metres
 *     (SPEC.md:29-34); q is normalised inside every call.
 *   - Gaussian slot gid = k·H·W + y·W + x for pixel (x, y) of keyframe k.  State is two
 *     float4 arrays: pos_rad = (X_w, Y_w, Z_w, r) and col_opa = (c_r, c_g, c_b, o) — the
 *     5 learnable scalars of PAPER.md:116-117 (§3.2) plus the derived centre.  r = 0 marks an
 *     invalid slot (depth 0) that is never rendered.
 *   - Pointers are DEVICE pointers owned by the caller unless marked (host).  All calls
 *     except those marked "synchronous" are asynchronous on `stream` (a cudaStream_t; NULL =
 *     legacy default stream) and may be captured in a CUDA graph.
 *   - Errors are returned, never thrown.  Argument errors are detected before any launch.
 *     Device-side capacity overflow (more tile pairs than the context holds) is recorded on
 *     the device and reported by the next synchronous call (vtgs_get_stats / vtgs_check).
 *     CUDA launch errors return VTGS_ERR_CUDA with detail in vtgs_last_error().
 */
#ifndef VTGS_H
#define VTGS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VTGS_ABI_VERSION 4

#if defined(__GNUC__)
#define VTGS_API __attribute__((visibility("default")))
#else
#define VTGS_API
#endif

typedef int32_t vtgs_status;
enum {
    VTGS_OK = 0,
    VTGS_ERR_INVALID_ARG = -1, /* NULL required pointer, fx/fy ≤ 0, cx ∉ (0, W), cy ∉ (0, H) */
    VTGS_ERR_SHAPE = -2,       /* size exceeds the context's limits, or inconsistent sizes */
    VTGS_ERR_CAPACITY = -3,    /* tile pairs exceeded max_pairs during a forward */
    VTGS_ERR_CUDA = -4,        /* a CUDA call failed; see vtgs_last_error */
    VTGS_ERR_STATE = -5,       /* render_bwd without a preceding render_fwd on this context */
    VTGS_ERR_NO_DEVICE = -6    /* no CUDA device: there is no CPU fallback */
};

/* SPEC.md:22-27 (CameraIntrinsics).  fx, fy > 0; 0 < cx < width; 0 < cy < height. */
typedef struct vtgs_intrinsics {
    float fx, fy, cx, cy;
    int32_t width, height;
} vtgs_intrinsics;

/* SPEC.md:29-34 (Pose): camera-to-world, q = (w, x, y, z) (normalised inside), t in metres. */
typedef struct vtgs_pose {
    float q[4];
    float t[3];
} vtgs_pose;

typedef struct vtgs_ctx vtgs_ctx;

/* ABI version of the loaded library (== VTGS_ABI_VERSION of the header it was built from). */
VTGS_API int32_t vtgs_abi_version(void);

/* Create a context on CUDA device `device`.  The context OWNS all scratch of the path, sized
 * for at most `max_gaussians` slots, images up to max_width × max_height (≤ 65535 each), and
 * `max_pairs` (Gaussian, tile) pairs per forward (0 ⇒ 2·max_gaussians + 262144; the five configs
 * need ≤ 1.75 per slot).  Scratch ≈ 32 B per slot + 85 B per pair (the 8 per-tile sub-lists and
 * their masks dominate).  One context serves one in-flight forward/backward: use one per stream.
 * Synchronous. */
VTGS_API vtgs_status vtgs_create(vtgs_ctx **out, int32_t device, int64_t max_gaussians, int32_t max_width,
                        int32_t max_height, int64_t max_pairs);
/* Release the context and its scratch (synchronises the device first).  NULL is a no-op. */
VTGS_API vtgs_status vtgs_destroy(vtgs_ctx *ctx);
/* Static description of a status code. */
VTGS_API const char *vtgs_status_string(vtgs_status s);
/* Detail of the last error on `ctx` ("" if none).  Valid until the next call on ctx. */
VTGS_API const char *vtgs_last_error(const vtgs_ctx *ctx);

/* (1) Instantiation — PAPER.md:110 (§3.1 "initialize Gaussians by centering them at all
 * pixels with valid depth values"), PAPER.md:119 (§3.2), PAPER.md:696-699 (Supp. A,
 * r = D_GT / f).
 *   depth   [K×H×W] metres, ≤ 0 or non-finite = invalid; rgb [K×H×W×3] in [0,1];
 *   kf_poses[K] device array of vtgs_pose (camera-to-world of each keyframe);
 *   opacity_init [K×H×W] or NULL (then every valid slot gets opacity_default);
 *   out pos_rad float4[K·H·W] = (R_k·X_c + t_k, d / f_mean), X_c = ((x−cx)d/fx, (y−cy)d/fy, d);
 *   out col_opa float4[K·H·W] = (rgb, opacity).  Invalid slots are written as all zeros.
 *   n_valid: device int64 or NULL, OVERWRITTEN with the number of valid slots (SPEC.md:440
 *   "count = valid pixels").
 *   H, W = intr.height, intr.width.  N = K·H·W > max_gaussians → VTGS_ERR_CAPACITY. */
VTGS_API vtgs_status vtgs_instantiate(vtgs_ctx *ctx, const float *depth, const float *rgb,
                             const vtgs_pose *kf_poses, int32_t K, vtgs_intrinsics intr,
                             const float *opacity_init, float opacity_default, float *pos_rad,
                             float *col_opa, int64_t *n_valid, void *stream);

/* Densification on a regular frame — PAPER.md:192 ("complement Gaussians at pixels uncovered by
 * the current Gaussians' renderings"), PAPER.md:261 ("0.5 as a mask threshold to determine if
 * current Gaussians ... cover a pixel").  A new Gaussian at every pixel with
 * valid depth (> 0, finite) and silhouette < threshold (strict), initialised exactly as
 * vtgs_instantiate does, appended in row-major pixel order (deterministic).
 *   depth [H×W], rgb [H×W×3], pose (device vtgs_pose of the frame), silhouette [H×W] (the
 *   section rendered from that pose by vtgs_render_fwd), opacity [H×W] or NULL (→ default).
 *   pos_rad_out / col_opa_out float4 (device, capacity H×W, e.g. the section's arrays + N):
 *   the first *n_new rows are written; n_new: device int64, OVERWRITTEN.
 * Asynchronous on `stream` (read n_new after synchronising). */
VTGS_API vtgs_status vtgs_densify(vtgs_ctx *ctx, const float *depth, const float *rgb, const vtgs_pose *pose,
                         vtgs_intrinsics intr, const float *silhouette, float threshold, const float *opacity,
                         float opacity_default, float *pos_rad_out, float *col_opa_out, int64_t *n_new,
                         void *stream);

/* Visibility mask of a frame to a section — PAPER.md:186 (§3.3 "Visibility Check": a point is
 * visible to a view "if its projected depth is within 1% of the interpolated depth at its
 * projection on the depth map"; the section's mask is the union over its head, middle and last
 * frames).  Every valid pixel of `depth` (the frame, at device `pose`) is
 * back-projected, transformed into each reference view r (ref_poses[r], device) and tested:
 * z > 0.01, projection inside [0, W−1] × [0, H−1], bilinear reference depth valid (four
 * neighbours > 0), |z − d_r| ≤ tol·d_r (tol = 0.01 in the paper).
 *   depth [H×W], ref_depth [R×H×W] (device), 1 ≤ R ≤ 8; mask [H×W] uint8 (device, OVERWRITTEN:
 *   1 = visible to some reference) — pass it as vtgs_l1_loss.vis_mask for Eq. 1's W_i;
 *   n_visible: device int64 or NULL (OVERWRITTEN with the count).  Asynchronous on `stream`. */
VTGS_API vtgs_status vtgs_visibility_mask(vtgs_ctx *ctx, const float *depth, const vtgs_pose *pose,
                                 const float *ref_depth, const vtgs_pose *ref_poses, int32_t R,
                                 vtgs_intrinsics intr, float tol, uint8_t *mask, int64_t *n_visible,
                                 void *stream);

/* Per-candidate visible-point counts for selecting the overlapping section of a head frame —
 * PAPER.md:180 (§3.3 "Selecting Overlapping Section S^o": "we project the depth D_i from the
 * initialized pose to each one frame in the overlap candidate view list. We count the number of
 * visible points to each candidate view, and select the candidate views that have more visible
 * points than a threshold γ"), SPEC.md:382-386 steps (1)-(3).  Same per-point test as
 * vtgs_visibility_mask, but each candidate r is counted alone (no union):
 *   depth [H×W] (the head frame, at device `pose` = its initialised pose), ref_depth [R×H×W] and
 *   ref_poses[R] (device) the candidate views, 1 ≤ R ≤ 65535;
 *   counts: device int64[R], OVERWRITTEN with the visible valid pixels per candidate;
 *   n_valid: device int64 or NULL, OVERWRITTEN with the frame's valid pixels (the fraction's
 *   denominator, PAPER.md:700 γ = 0.26 / 0.24 is a fraction).  Asynchronous on `stream`.
 * Errors: NULL argument → VTGS_ERR_INVALID_ARG; R out of range → VTGS_ERR_SHAPE. */
VTGS_API vtgs_status vtgs_visibility_counts(vtgs_ctx *ctx, const float *depth, const vtgs_pose *pose,
                                   const float *ref_depth, const vtgs_pose *ref_poses, int32_t R,
                                   vtgs_intrinsics intr, float tol, int64_t *counts, int64_t *n_valid,
                                   void *stream);

/* (2)–(4) Forward render of N Gaussians from `view` — PAPER.md:146 (Eq. 1 `splat`),
 * PAPER.md:192 (Eq. 2 multi-set render: concatenate the sets, pass the union).
 *   projection: X_c = Rᵀ(X_w − t), culled if r ≤ 0 or z ≤ 0.01 m; σ = max(f_mean·r/z, 0.3) px;
 *   footprint = integer pixel rect within ±3σ; binned to every 16×16 tile the rect overlaps;
 *   per tile sorted by (depth, gid); each pixel composites, front to back, the Gaussians of its
 *   tile whose rect contains it and with d² ≤ 9σ²: α = min(o·exp(−d²/2σ²), 0.999), skipped if
 *   α < 1/255, stopped before the first Gaussian that would take T below 1e-4.
 *   view: DEVICE pointer to one vtgs_pose (so a graph-captured loop can update it in place);
 *   the forward copies it on the device, so it may be reused as soon as the call is enqueued.
 *   out color [H×W×3], depth [H×W] (Σ αT z, unnormalised), silhouette [H×W] (Σ αT).
 * N > max_gaussians → VTGS_ERR_CAPACITY; N < 0 → VTGS_ERR_SHAPE.
 * The context remembers pos_rad, col_opa and the three output pointers: they must stay valid
 * and unmodified until the matching vtgs_render_bwd. */
VTGS_API vtgs_status vtgs_render_fwd(vtgs_ctx *ctx, const float *pos_rad, const float *col_opa, int64_t N,
                            const vtgs_pose *view, vtgs_intrinsics intr, float *color, float *depth,
                            float *silhouette, void *stream);

/* Fused masked-L1 loss of Eq. 1 / the L1 terms of Eq. 2:
 *   loss = w_color·Σ m_c ‖C − C̃‖₁ · s_c + w_depth·Σ m_d |D − D̃| · s_d
 *   U = [D̃ > 0];  W = U ∧ [S > 0.99] ∧ vis
 *   color_mask_mode 0: m_c = 1 (Eq. 2), 1: m_c = W (Eq. 1)
 *   depth_mask_mode 0: m_d = U (Eq. 2), 1: m_d = W (Eq. 1)
 *   normalize 0: s = 1 (sum form), 1: s = 1 / Σ m (mean over masked pixels; 0 if
 *   the mask is empty).  Upstream gradients use sgn(0) = 0.
 *   extra_dcolor [H×W×3] (device, may be NULL) is added to the colour upstream gradient — the
 *   SSIM term of Eq. 2 from vtgs_ssim_loss, so the full mapping objective
 *   ρ‖V − V'‖₁ + τ L_S + σ U‖D − D'‖₁ runs through one backward. */
typedef struct vtgs_l1_loss {
    const float *target_rgb;   /* [H×W×3] */
    const float *target_depth; /* [H×W], 0 = invalid */
    const uint8_t *vis_mask;   /* [H×W] or NULL (= all visible) */
    float w_color, w_depth;
    int32_t color_mask_mode, depth_mask_mode, normalize;
    const float *extra_dcolor;  /* [H×W×3] or NULL */
} vtgs_l1_loss;

/* SSIM term of the mapping objective Eq. 2 — PAPER.md:195-201 ("τ L_S(V_i, V_i') ... L_S is the
 * SSIM loss"), τ = 0.2 in the paper's experiments.  DESIGN.md reading R24: 11×11
 * Gaussian window σ = 1.5, C1 = 0.01², C2 = 0.03², per colour channel, zero padding outside the
 * image, L_S = 1 − mean of the SSIM map over all pixels and channels.
 *   color (the render V') and target_rgb (V) [height×width×3], device.
 *   d_color [height×width×3] (device, may be NULL): dL/dV' of τ·L_S is ACCUMULATED (+=) — pass
 *   it as vtgs_l1_loss.extra_dcolor (or add it to dL_dcolor) for vtgs_render_bwd.
 *   loss_out (device float, may be NULL) is OVERWRITTEN with τ·L_S.
 * Errors: image smaller than the 11×11 window → VTGS_ERR_SHAPE; larger than the context's
 * max_width × max_height → VTGS_ERR_CAPACITY.  Asynchronous on `stream`; the loss is summed
 * in a fixed order (deterministic). */
VTGS_API vtgs_status vtgs_ssim_loss(vtgs_ctx *ctx, const float *color, const float *target_rgb, int32_t width,
                           int32_t height, float tau, float *d_color, float *loss_out, void *stream);

enum { VTGS_GRAD_COLOR = 1, VTGS_GRAD_OPACITY = 2, VTGS_GRAD_RADIUS = 4, VTGS_GRAD_POSE = 8,
       VTGS_GRAD_POSITION = 16, VTGS_GRAD_DETERMINISTIC = 32 };

/* (5) Backward of the LAST vtgs_render_fwd on this context — SPEC.md:197-205 (chain through
 * the α/T recurrence, the footprint σ = f·r/z, the projection), SPEC.md:223 (pose gradient on
 * the ambient quaternion 4 + translation 3), PAPER.md:201 ("Only {g}^k are learnable").
 *   Upstream: either dL_dcolor [H×W×3] / dL_ddepth / dL_dsil [H×W] (NULL entries = 0) when
 *   `loss` is NULL, or the fused L1 loss above when `loss` is non-NULL (the dL_* must be NULL).
 *   want: OR of VTGS_GRAD_*.  learn_begin ≤ gid < learn_end receive attribute gradients.
 *   d_col_opa float4[N] (dc_r, dc_g, dc_b, do) and d_radius [N] are ACCUMULATED (+=, the
 *   caller zeroes them), so multi-view mapping is a loop of fwd/bwd pairs.  Either may be NULL
 *   when the corresponding want bits are clear.
 *   d_position float4[N]: with VTGS_GRAD_POSITION, dL/dX_w (x, y, z; w untouched) of every
 *   Gaussian centre is ACCUMULATED (+=) — the input of the head-frame bundle adjustment
 *   (vtgs_keyframe_pose_grad); NULL when not wanted.  Not restricted to
 *   [learn_begin, learn_end).
 *   d_pose [7] (dq_w, dq_x, dq_y, dq_z, dt_x, dt_y, dt_z) is OVERWRITTEN (NULL if not wanted).
 *   loss_out: device float, OVERWRITTEN with the loss value (NULL = not needed; requires loss).
 * Attribute gradients are summed with float atomics across tiles: run-to-run results can
 * differ in the last bits — unless want has VTGS_GRAD_DETERMINISTIC: then the
 * per-(Gaussian, sub-tile) partials are summed as int64 fixed point (2⁻⁴⁰ resolution, |sum| <
 * 8.4e6), independent of arrival order, and added to d_col_opa / d_radius by one more pass
 * ("privatized buffers merged deterministically"; the context allocates 40 B per
 * Gaussian on first use).  The pose gradient is always reduced in a fixed order. */
VTGS_API vtgs_status vtgs_render_bwd(vtgs_ctx *ctx, const float *dL_dcolor, const float *dL_ddepth,
                            const float *dL_dsil, const vtgs_l1_loss *loss, uint32_t want,
                            int64_t learn_begin, int64_t learn_end, float *d_col_opa,
                            float *d_radius, float *d_position, float *d_pose, float *loss_out,
                            void *stream);

/* Head-frame bundle adjustment — PAPER.md:248-250 (§3.5: "back-propagate gradients to update
 * the camera pose of the head frame").  A view-tied centre is its keyframe's back-projected
 * depth pixel, X_w = R_k X_k + t_k, so
 *   dL/dt_k = Σ_{g ∈ k} dL/dX_w,g,   dL/dR_k = Σ_{g ∈ k} dL/dX_w,g X_kᵀ,  X_k = R_kᵀ(X_w − t_k),
 * then through R(q̂), q̂ = q/|q|.  Keyframe k owns slots [k·slots_per_kf,
 * (k+1)·slots_per_kf) (vtgs_instantiate's layout); invalid slots (r = 0) are skipped.
 *   pos_rad float4[K·slots_per_kf] (device), d_position float4[...] (device, from
 *   vtgs_render_bwd with VTGS_GRAD_POSITION), kf_poses vtgs_pose[K] (device);
 *   d_kf_pose float[K×7] (device) is OVERWRITTEN (dq 4, dt 3 per keyframe).
 * The total gradient of a head frame that is also the rendered view is d_pose + d_kf_pose[k].
 * Sums are fp64 in a fixed order (deterministic).  Asynchronous on `stream`. */
VTGS_API vtgs_status vtgs_keyframe_pose_grad(vtgs_ctx *ctx, const float *pos_rad, const float *d_position,
                                    const vtgs_pose *kf_poses, int32_t K, int64_t slots_per_kf,
                                    float *d_kf_pose, void *stream);

/* One Adam step on a device pose (β1 = 0.9, β2 = 0.999, ε = 1e-8; learning
 * rates lr_rot for q and lr_trans for t), then q ← q/|q|.
 *   adam_state: device float[16] = m[7], v[7], step, unused; zero it to restart. */
VTGS_API vtgs_status vtgs_pose_adam_step(vtgs_ctx *ctx, vtgs_pose *pose, const float *d_pose,
                                float *adam_state, float lr_rot, float lr_trans, void *stream);

/* Work counters of the last forward.  Synchronous (synchronises `stream`). */
typedef struct vtgs_stats {
    int64_t n_gaussians; /* N of the last forward */
    int64_t n_pairs;     /* P: (Gaussian, tile) pairs */
    int64_t e_eval;      /* (pixel, Gaussian) evaluations inside the footprint, before the cut-off */
    int64_t e_comp;      /* composited (pixel, Gaussian) pairs */
    int64_t max_tile;    /* longest tile list */
    int64_t overflow;    /* 1 if P exceeded max_pairs (outputs then zero) */
    int64_t launches;    /* kernels this context has launched since it was created */
} vtgs_stats;
VTGS_API vtgs_status vtgs_get_stats(vtgs_ctx *ctx, vtgs_stats *out /* host */, void *stream);
/* The forward's e_eval / e_comp counters cost a few instructions per evaluation; they are on by
 * default and can be switched off (then both read 0; n_pairs / max_tile are always kept). */
VTGS_API vtgs_status vtgs_set_work_counters(vtgs_ctx *ctx, int32_t enable);

/* Per-kernel device timing (CUDA events recorded on the launching stream around every kernel
 * while enabled; not for use inside CUDA-graph capture).  Stages, in order:
 *   0 project_count, 1 scan_tiles, 2 emit_pairs, 3 tile_sort, 4 composite_fwd, 5 l1_count,
 *   6 composite_bwd, 7 pose_finalize, 8 instantiate, 9 pose_adam, 10 keyframe_pose_grad, 11 ssim,
 *   12 densify, 13 visibility. */
#define VTGS_NUM_STAGES 14
VTGS_API vtgs_status vtgs_set_profiling(vtgs_ctx *ctx, int32_t enable);
/* Synchronous: sum of event-timed milliseconds (ms[VTGS_NUM_STAGES], host) and the number of
 * event-timed launch scopes (counts[VTGS_NUM_STAGES], host, may be NULL; launches made while
 * profiling was off are not counted) per stage since the previous call; resets. */
VTGS_API vtgs_status vtgs_get_profile(vtgs_ctx *ctx, double *ms, int64_t *counts, void *stream);

/* Measurement hook (not on the path): the FP32 FMA peak (TFLOP/s, an FMA = 2 flops) and the
 * MUFU ex2.approx throughput (ops/s) of `device`, measured by two microbenchmark kernels (every
 * SM, 64 warps, 8 independent chains per thread; best of 4) — the roofline denominators of the
 * ALU-bound compositing kernels.  Synchronous. */
VTGS_API vtgs_status vtgs_measure_peaks(int32_t device, double *fp32_tflops, double *ex2_per_s);

/* Synchronise `stream` and report a deferred device-side error (VTGS_ERR_CAPACITY) or a CUDA
 * error.  Synchronous. */
VTGS_API vtgs_status vtgs_check(vtgs_ctx *ctx, void *stream);

/* Test hook: copy the last forward's tile lists to HOST memory.  tile_start (host) gets
 * ntiles+1 offsets (ntiles = ⌈W/16⌉·⌈H/16⌉, row-major tiles); sorted_gid (host) gets P gids
 * when P ≤ cap (else only *P_out is written).  Synchronous. */
VTGS_API vtgs_status vtgs_export_tiles(vtgs_ctx *ctx, int64_t *tile_start, int32_t *sorted_gid, int64_t cap,
                              int64_t *P_out, void *stream);

/* End-to-end mapping/tracking step with HOST buffers (the bench's e2e leg): copies the target
 * frame (host rgb [H×W×3], host depth [H×W]) and the view pose (host) to device scratch owned
 * by the context, runs render_fwd + fused-L1 render_bwd exactly as above, and copies the loss
 * (and, if d_pose_host is non-NULL, the 7 pose gradients) back to the host.  pos_rad /
 * col_opa / d_col_opa / d_radius / color / depth / silhouette are DEVICE buffers (the model
 * state and the outputs stay resident).  The targets upload on a context-owned second stream
 * while projection, sort and forward run (the backward waits for them); host buffers should be
 * pinned for the copy to be asynchronous.  Synchronous (returns after the loss is on the host).
 * The 5N attribute gradients (and the images) stay on the device: only the loss (4 B) and, with
 * VTGS_GRAD_POSE, the 7 pose gradients come back.  A forward whose tile pairs exceeded the
 * context's capacity returns VTGS_ERR_CAPACITY here (render and gradients empty). */
VTGS_API vtgs_status vtgs_step_host(vtgs_ctx *ctx, const float *pos_rad, const float *col_opa, int64_t N,
                           const vtgs_pose *view_host, vtgs_intrinsics intr,
                           const float *target_rgb_host, const float *target_depth_host,
                           float w_color, float w_depth, int32_t color_mask_mode,
                           int32_t depth_mask_mode, int32_t normalize, uint32_t want,
                           int64_t learn_begin, int64_t learn_end, float *color, float *depth,
                           float *silhouette, float *d_col_opa, float *d_radius,
                           float *loss_host, float *d_pose_host, void *stream);

/* vtgs_step_host with the target frame in the formats an RGB-D sensor (and the paper's datasets:
 * 8-bit RGB, 16-bit depth images) deliver it: rgb8_host [H×W×3] uint8, depth16_host [H×W]
 * uint16 (0 = no depth), depth_scale = metres per depth unit (e.g. 1/5000).  The 5 B/pixel are
 * uploaded (instead of 16 B/pixel of fp32) on the context's copy stream and widened on the device
 * right before the backward: c = v / 255 (IEEE fp32 division), z = d · depth_scale (one fp32
 * multiply) — exactly the fp32 targets a host-side conversion with the same two operations gives,
 * so the step equals vtgs_step_host on those targets.  Everything else as vtgs_step_host. */
VTGS_API vtgs_status vtgs_step_host_sensor(vtgs_ctx *ctx, const float *pos_rad, const float *col_opa, int64_t N,
                                  const vtgs_pose *view_host, vtgs_intrinsics intr,
                                  const uint8_t *rgb8_host, const uint16_t *depth16_host, float depth_scale,
                                  float w_color, float w_depth, int32_t color_mask_mode,
                                  int32_t depth_mask_mode, int32_t normalize, uint32_t want,
                                  int64_t learn_begin, int64_t learn_end, float *color, float *depth,
                                  float *silhouette, float *d_col_opa, float *d_radius,
                                  float *loss_host, float *d_pose_host, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* VTGS_H */
