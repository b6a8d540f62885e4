/* oracle/vtgs_oracle.c — the CPU ORACLE for the view-tied splatting hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product path
 * (paper_2506_02741_b200/) never touches it and shares no code, header, helper or constant
 * table with it.
 *
 * What it computes — a plain, slow, obviously-correct definition of each step, written from
 * PAPER.md / SPEC.md (citations at each function; P:n = PAPER.md line n, S:n = SPEC.md line n):
 *   or_instantiate_*  (a1)  back-projected view-tied Gaussians
 *   or_project_*      (a2)  isotropic screen footprint
 *   or_tile_lists_*   (a3)  16×16 tile lists in (z, gid) order
 *   or_render_*       (a4)  per-pixel front-to-back compositing
 *   or_render_bwd_*   (a5)  derivative of the compositing closed form
 *   or_keyframe_pose_grad_*  head-frame bundle adjustment: keyframe poses
 *   or_l1_upstream          masked L1 terms of Eq. 1 / Eq. 2
 *   or_ssim_loss            SSIM term τ·L_S of Eq. 2 and its gradient
 *   or_densify_f32          regular-frame densification (S < 0.5)
 *   or_visibility_*         visibility mask to a section (1% depth band)
 * Two builds of the same source (oracle_impl.inc): *_f32 takes every decision in fp32 (the
 * kernel's precision) with fp64 values; *_f64 is fp64 throughout.
 *
 * Pinning (tests/test_oracle_pins.py): SPEC worked examples, closed
 * forms for one and two Gaussians, the termination / truncation / floor / clamp special cases,
 * invariants, brute-force tile lists, central finite differences in fp64
 * for colour, opacity, radius and the 7 pose parameters.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC (no FMA
 * contraction, so every fp32 decision quantity is rounded exactly as DESIGN.md §3 states).
 * OpenMP: the forward render runs its pixel rows in parallel (results independent of the thread
 * count); the backward splits the pixels into row bands with private accumulators merged in
 * band order.  OMP_NUM_THREADS=1 gives the single-core oracle.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* memory budget of the backward's per-thread accumulator copies (bytes; env OR_BWD_MEM overrides) */
#ifndef OR_BWD_MEM
#define OR_BWD_MEM 16.0e9
#endif
#include <stdlib.h>
#include <string.h>

#define DEC float
#define FN(name) name##_f32
#include "oracle_impl.inc"
#undef DEC
#undef FN
#undef OR_EPS_DEC
#undef OR_EPS_VAL
#undef OR_ALPHA_MIN
#undef OR_ALPHA_MAX
#undef OR_T_MIN

#define DEC double
#define FN(name) name##_f64
#include "oracle_impl.inc"
#undef DEC
#undef FN

/* ---------------------------------------------------------------------------------------
 * Masked L1 terms of the tracking objective Eq. 1:
 *     α·W_i‖V_i − V_i'‖₁ + β·W_i‖D_i − D_i'‖₁
 * and of the mapping objective Eq. 2 without its SSIM term:
 *     ρ‖V_i − V_i'‖₁ + σ·U_i‖D_i − D_i'‖₁
 * Masks: U_i = [D̃ > 0] ("removes pixels without valid depth values");
 *        W_i = [D̃ > 0] ∧ [S > 0.99] ∧ vis ("removes pixels either without depth values or
 *        uncovered by the rendering ... or invisible"; 0.99 from S:336).
 * color_mask_mode 0: colour term over all pixels (Eq. 2); 1: over W_i (Eq. 1).
 * depth_mask_mode 0: U_i (Eq. 2); 1: W_i (Eq. 1).
 * normalize 0: sum over pixels (‖·‖₁ sums the 3 channels); 1: divided by the mask's pixel
 * count ("mean absolute difference over masked pixels"; empty mask → 0).
 * Upstream gradients are the subgradient with sgn(0) = 0.
 * Returns the loss value; writes gC (H×W×3), gD, gS (gS ≡ 0).
 * Near-tie flags (the kernel renders in fp32, so its residual can take the other side of
 * sgn): a (pixel, component) is flagged when its residual is nonzero but within `band` of 0
 * (DESIGN.md §3 derives `band` from the measured GPU-vs-oracle render difference), and a whole
 * pixel when S lies within 1e-5 of 0.99 under a W-mask.  `flag` (H×W, may be NULL) marks
 * flagged pixels; `flip` (H×W×4, may be NULL) gets, per flagged component (3 colour channels,
 * depth), the largest change of its upstream gradient the other branch could cause, 2·w·s
 * (0 elsewhere) — the tests turn it into a per-Gaussian allowance by running or_render_bwd
 * on it.  (A residual that is exactly 0 — e.g. a clipped black target rendered from black
 * Gaussians — is exactly 0 in fp32 too.)
 * ------------------------------------------------------------------------------------- */
double or_l1_upstream(const double *C, const double *D, const double *S, const double *tC,
                      const double *tD, const unsigned char *vis, int64_t npx, double w_color,
                      double w_depth, int color_mask_mode, int depth_mask_mode, int normalize,
                      double *gC, double *gD, double *gS, int32_t *flag, double band, double *flip)
{
    int64_t nc = 0, nd = 0;
    for (int64_t p = 0; p < npx; ++p) {
        const int U = tD[p] > 0.0;
        const int Wm = U && S[p] > 0.99 && (vis ? vis[p] != 0 : 1);
        nc += color_mask_mode ? Wm : 1;
        nd += depth_mask_mode ? Wm : U;
    }
    const double sc = normalize ? (nc ? 1.0 / (double)nc : 0.0) : 1.0;
    const double sd = normalize ? (nd ? 1.0 / (double)nd : 0.0) : 1.0;
    double loss = 0.0;
    for (int64_t p = 0; p < npx; ++p) {
        const int U = tD[p] > 0.0;
        const int Wm = U && S[p] > 0.99 && (vis ? vis[p] != 0 : 1);
        const int mc = color_mask_mode ? Wm : 1;
        const int md = depth_mask_mode ? Wm : U;
        const int mflip = (color_mask_mode || depth_mask_mode) && U && fabs(S[p] - 0.99) < 1e-5;
        int fl = mflip;
        double fw[4] = {0.0, 0.0, 0.0, 0.0};
        for (int c = 0; c < 3; ++c) {
            const double r = C[3 * p + c] - tC[3 * p + c];
            const int near = mc && r != 0.0 && fabs(r) < band;
            if (near || (mflip && color_mask_mode)) { fl = 1; fw[c] = 2.0 * fabs(w_color * sc); }
            gC[3 * p + c] = mc ? w_color * sc * (double)((r > 0) - (r < 0)) : 0.0;
            loss += mc ? w_color * sc * fabs(r) : 0.0;
        }
        const double r = D[p] - tD[p];
        const int near = md && r != 0.0 && fabs(r) < band;
        if (near || (mflip && depth_mask_mode)) { fl = 1; fw[3] = 2.0 * fabs(w_depth * sd); }
        gD[p] = md ? w_depth * sd * (double)((r > 0) - (r < 0)) : 0.0;
        loss += md ? w_depth * sd * fabs(r) : 0.0;
        gS[p] = 0.0;
        if (flag) flag[p] = fl;
        if (flip)
            for (int c = 0; c < 4; ++c) flip[4 * p + c] = fw[c];
    }
    return loss;
}

/* ---------------------------------------------------------------------------------------
 * SSIM term of the mapping objective Eq. 2 ("τ L_S(V_i, V_i') ... L_S is the SSIM
 * loss"; τ = 0.2).  The paper fixes no variant; reading R24 takes the standard
 * one: 11×11 Gaussian window with σ = 1.5 normalised to sum 1, C1 = 0.01²,
 * C2 = 0.03², applied to each colour channel with zero padding outside the image ("same"
 * output size), L_S = 1 − mean of the SSIM map over all pixels and the 3 channels.
 * Plain definition: for every pixel p and channel c the five window moments are summed
 * directly over the 121 window taps,
 *     μx = Σ w x, μy = Σ w y, σx² = Σ w x² − μx², σy² = Σ w y² − μy², σxy = Σ w x y − μx μy,
 *     SSIM_p = (2 μx μy + C1)(2 σxy + C2) / ((μx² + μy² + C1)(σx² + σy² + C2)),
 * and the gradient of τ·L_S w.r.t. x (the render) is the chain rule through those moments
 * written out per (window centre p, tap q):
 *     ∂SSIM_p/∂x_q = w_{q−p} [∂S/∂μx + 2 x_q ∂S/∂Exx + y_q ∂S/∂Exy]
 * with ∂S/∂μx = S(2μy/A1 − 2μy/A2 − 2μx/B1 + 2μx/B2), ∂S/∂Exx = −S/B2, ∂S/∂Exy = 2S/A2
 * (A1 = 2μxμy + C1, A2 = 2σxy + C2, B1 = μx² + μy² + C1, B2 = σx² + σy² + C2).
 * fp64 throughout.  x, y: H×W×3 (x = render, y = target).  Returns τ·L_S; writes grad (H×W×3,
 * overwritten, may be NULL) and the SSIM map (H×W×3, may be NULL).
 * ------------------------------------------------------------------------------------- */
double or_ssim_loss(const double *x, const double *y, int W, int H, double tau, double *grad, double *smap)
{
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double w[11][11], g1[11], gs = 0.0;
    for (int i = 0; i < 11; ++i) {
        g1[i] = exp(-((double)(i - 5) * (i - 5)) / (2.0 * 1.5 * 1.5));
        gs += g1[i];
    }
    for (int i = 0; i < 11; ++i)
        for (int j = 0; j < 11; ++j) w[i][j] = (g1[i] / gs) * (g1[j] / gs);
    const int64_t npx = (int64_t)W * H;
    double *dS = (double *)malloc(sizeof(double) * 3 * (size_t)npx * 3);   /* ∂S/∂μx, ∂S/∂Exx, ∂S/∂Exy */
    if (!dS) return NAN;
    double sum = 0.0;
    for (int py = 0; py < H; ++py)
        for (int px = 0; px < W; ++px)
            for (int c = 0; c < 3; ++c) {
                double mx = 0, my = 0, exx = 0, eyy = 0, exy = 0;
                for (int i = 0; i < 11; ++i)
                    for (int j = 0; j < 11; ++j) {
                        const int qy = py + i - 5, qx = px + j - 5;
                        if (qx < 0 || qy < 0 || qx >= W || qy >= H) continue;   /* zero padding */
                        const double a = x[3 * ((int64_t)qy * W + qx) + c], b = y[3 * ((int64_t)qy * W + qx) + c];
                        mx += w[i][j] * a;
                        my += w[i][j] * b;
                        exx += w[i][j] * a * a;
                        eyy += w[i][j] * b * b;
                        exy += w[i][j] * a * b;
                    }
                const double A1 = 2 * mx * my + C1, A2 = 2 * (exy - mx * my) + C2;
                const double B1 = mx * mx + my * my + C1, B2 = (exx - mx * mx) + (eyy - my * my) + C2;
                const double S = A1 * A2 / (B1 * B2);
                const int64_t k = 3 * ((int64_t)py * W + px) + c;
                if (smap) smap[k] = S;
                sum += S;
                dS[3 * k + 0] = S * (2 * my / A1 - 2 * my / A2 - 2 * mx / B1 + 2 * mx / B2);
                dS[3 * k + 1] = -S / B2;
                dS[3 * k + 2] = 2 * S / A2;
            }
    const double n = 3.0 * (double)npx;
    if (grad) {
        const double dLdS = -tau / n;   /* L = τ (1 − Σ S / n) */
        for (int64_t i = 0; i < 3 * npx; ++i) grad[i] = 0.0;
        for (int py = 0; py < H; ++py)
            for (int px = 0; px < W; ++px)
                for (int c = 0; c < 3; ++c) {
                    const int64_t k = 3 * ((int64_t)py * W + px) + c;
                    for (int i = 0; i < 11; ++i)
                        for (int j = 0; j < 11; ++j) {
                            const int qy = py + i - 5, qx = px + j - 5;
                            if (qx < 0 || qy < 0 || qx >= W || qy >= H) continue;
                            const int64_t q = 3 * ((int64_t)qy * W + qx) + c;
                            grad[q] += dLdS * w[i][j] * (dS[3 * k] + 2 * x[q] * dS[3 * k + 1] + y[q] * dS[3 * k + 2]);
                        }
                }
    }
    free(dS);
    return tau * (1.0 - sum / n);
}

/* ---------------------------------------------------------------------------------------
 * Densification on a regular frame ("complement Gaussians at pixels uncovered by the
 * current Gaussians' renderings"; "we will choose 0.5 as a mask threshold to determine if
 * current Gaussians in S_k cover a pixel, if they do not, we will initialize a Gaussian as a
 * complement").  A pixel gets a new Gaussian iff its depth is valid (> 0, finite)
 * and the section's silhouette there is below the threshold (strict <).  The new Gaussians are
 * initialised exactly as or_instantiate does and appended in row-major pixel
 * order.  depth [H,W], rgb [H,W,3], pose [7], sil [H,W], opacity [H,W] or NULL; out pos_rad /
 * col_opa [H·W,4] (the first `count` rows written).  Returns count.
 * ------------------------------------------------------------------------------------- */
int64_t or_densify_f32(const double *depth, const double *rgb, const double *pose, const double *intr, int W,
                       int H, const double *sil, double threshold, const double *opacity,
                       double opacity_default, double *pos_rad, double *col_opa)
{
    const int64_t npx = (int64_t)W * H;
    double *pr = (double *)malloc(sizeof(double) * 4 * (size_t)npx);
    double *co = (double *)malloc(sizeof(double) * 4 * (size_t)npx);
    if (!pr || !co) return -1;
    or_instantiate_f32(depth, rgb, pose, 1, intr, W, H, opacity, opacity_default, pr, co);
    int64_t n = 0;
    for (int64_t p = 0; p < npx; ++p) {
        const double d = (double)(float)depth[p];
        if (!(d > 0.0) || !isfinite(d)) continue;
        if (!((float)sil[p] < (float)threshold)) continue;
        for (int i = 0; i < 4; ++i) {
            pos_rad[4 * n + i] = pr[4 * p + i];
            col_opa[4 * n + i] = co[4 * p + i];
        }
        ++n;
    }
    free(pr);
    free(co);
    return n;
}

/* ---------------------------------------------------------------------------------------
 * One Adam step on a camera pose (S:207-215 adam_step: "standard first/second-moment update,
 * β1=0.9, β2=0.999, ε=1e-8 ... quaternion renormalized after step"; learning rates per group —
 * rotation lr_rot for q, translation lr_trans for t, "lr_rot, lr_trans").  fp64:
 *   t ← t + 1;  m ← β1 m + (1−β1) g;  v ← β2 v + (1−β2) g²;
 *   p ← p − lr · (m / (1 − β1^t)) / (√(v / (1 − β2^t)) + ε);  q ← q / |q|.
 * pose[7] = (q w,x,y,z, t x,y,z) and state[15] = m[7], v[7], step are updated in place.
 * ------------------------------------------------------------------------------------- */
void or_pose_adam(double *pose, const double *g, double *state, double lr_rot, double lr_trans)
{
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double t = state[14] + 1.0;
    state[14] = t;
    const double c1 = 1.0 - pow(b1, t), c2 = 1.0 - pow(b2, t);
    for (int i = 0; i < 7; ++i) {
        state[i] = b1 * state[i] + (1.0 - b1) * g[i];
        state[7 + i] = b2 * state[7 + i] + (1.0 - b2) * g[i] * g[i];
        const double lr = i < 4 ? lr_rot : lr_trans;
        pose[i] -= lr * (state[i] / c1) / (sqrt(state[7 + i] / c2) + eps);
    }
    const double n = sqrt(pose[0] * pose[0] + pose[1] * pose[1] + pose[2] * pose[2] + pose[3] * pose[3]);
    for (int i = 0; i < 4; ++i) pose[i] /= n;
}
