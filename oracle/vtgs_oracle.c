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
 * Two builds of the same source (oracle_impl.inc): *_f32 takes every decision in fp32 (the
 * kernel's precision) with fp64 values; *_f64 is fp64 throughout.
 *
 * Pinning (tests/test_oracle_pins.py): SPEC worked examples, closed
 * forms for one and two Gaussians, the termination / truncation / floor / clamp special cases,
 * invariants, brute-force tile lists, central finite differences in fp64
 * for colour, opacity, radius and the 7 pose parameters.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC (no FMA contraction,
 * so every fp32 decision quantity is rounded exactly as DESIGN.md §3 states).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEC float
#define FN(name) name##_f32
#include "oracle_impl.inc"
#undef DEC
#undef FN
#undef OR_EPS_A
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
 * Returns the loss value; writes gC (H×W×3), gD, gS (gS ≡ 0).  `flag` (H×W, may be NULL) is
 * set where a residual is nonzero but within 5e-5 of 0, or S within 1e-5 of 0.99, i.e. where
 * the kernel's fp32 render could take the other branch of sgn or of the mask.  (A residual
 * that is exactly 0 — e.g. a clipped black target rendered from black Gaussians — is exactly 0
 * in fp32 too.)
 * ------------------------------------------------------------------------------------- */
double or_l1_upstream(const double *C, const double *D, const double *S, const double *tC,
                      const double *tD, const unsigned char *vis, int64_t npx, double w_color,
                      double w_depth, int color_mask_mode, int depth_mask_mode, int normalize,
                      double *gC, double *gD, double *gS, int32_t *flag)
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
        int fl = (color_mask_mode || depth_mask_mode) && U && fabs(S[p] - 0.99) < 1e-5;
        for (int c = 0; c < 3; ++c) {
            const double r = C[3 * p + c] - tC[3 * p + c];
            if (mc && r != 0.0 && fabs(r) < 5e-5) fl = 1;
            gC[3 * p + c] = mc ? w_color * sc * (double)((r > 0) - (r < 0)) : 0.0;
            loss += mc ? w_color * sc * fabs(r) : 0.0;
        }
        const double r = D[p] - tD[p];
        if (md && r != 0.0 && fabs(r) < 5e-5) fl = 1;
        gD[p] = md ? w_depth * sd * (double)((r > 0) - (r < 0)) : 0.0;
        loss += md ? w_depth * sd * fabs(r) : 0.0;
        gS[p] = 0.0;
        if (flag) flag[p] = fl;
    }
    return loss;
}
