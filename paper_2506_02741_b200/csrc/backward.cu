// (5) Reverse-order backward of the compositing — SPEC.md:197-205, :223-224, :232;
// north_star part (5); fused masked-L1 prologue of Eq. 1 / Eq. 2
// (PAPER.md:195-201).  DESIGN.md §3 steps 8-11.
//
// One CTA per 16×16 tile, one thread per pixel, same sub-tile / compaction scheme as the
// forward.  Each pixel walks its composited Gaussians back to front, recovering
// T_i = T_{i+1} / (1 − α_i) from the saved final transmittance, with the running "behind"
// accumulators ā ← α·x + (1 − α)·ā.
//   * attribute gradients (mapping): warp-shuffle reduction per Gaussian → shared-memory
//     accumulator per staged entry → one float4 + one float global atomic per (Gaussian, tile);
//   * pose gradient (tracking): each lane chains its pairs straight into 12 register
//     accumulators (Σ g, Σ X_c gᵀ), reduced per CTA in fp64 into a per-tile partial; a
//     one-CTA kernel sums the partials in a fixed order and applies the rotation chain.
#include <stddef.h>
#include <stdlib.h>

#include "composite_common.cuh"

namespace vtgs {

constexpr unsigned kFull = kFullMask;

struct BwdArgs {
    const float4 *proj;
    const float *thr;             // per Gaussian packed (D_c, D_clamp), k_project_count
    const float4 *col_opa;
    const float4 *pos_rad;
    const uint32_t *tile_count;
    const uint32_t *tile_start;
    const uint32_t *sub_lists;
    const uint32_t *sub_count;
    const uint32_t *sub_masks;   // the forward's per-entry candidate pixel masks (lane_mask within D_c)
    int W, H, ntx;
    const float *color, *depth, *sil, *T_final;
    const uint32_t *last;
    const float *dC, *dD, *dS;
    const float *tC, *tD;
    const uint8_t *vis;
    const float *extra_dc;
    float wc, wd;
    int cmode, dmode, normalize;
    const DevScalars *dev;
    const vtgs_pose *view;
    vtgs_intrinsics in;
    int64_t learn_begin, learn_end;
    uint32_t want;
    float4 *d_col_opa;
    float *d_radius;
    float4 *d_position;
    double *partials;
    unsigned long long *det;   // VTGS_GRAD_DETERMINISTIC: int64 fixed-point accumulators [N][5], else NULL
    uint64_t sub_cap;          // entries of sub_lists / sub_masks (checked build)
    int64_t N;                 // Gaussians (checked build)
};

// Deterministic attribute-gradient merge ("merged deterministically"): the
// per-(Gaussian, sub-tile) partials are rounded to int64 multiples of 2⁻⁴⁰ and summed with
// integer atomics — integer addition is associative, so the sum is the same whatever order the
// warps arrive in — then k_det_finalize adds them (as fp32) to the caller's buffers.
constexpr double kDetScale = 1099511627776.0;   // 2^40: resolution 9.1e-13, range ±8.4e6
__device__ __forceinline__ void det_add(unsigned long long *q, float v) {
    if (v != 0.f) atomicAdd(q, (unsigned long long)__double2ll_rn((double)v * kDetScale));
}

// index of the highest set bit (bfind: one FLO; 0xffffffff for 0) — `31 − __clz` costs the
// compiler an extra subtract and an XOR per use
__device__ __forceinline__ int msb_index(unsigned x) {
    unsigned r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return (int)r;
}

__device__ __forceinline__ float sgnf(float r) { return (float)((r > 0.0f) - (r < 0.0f)); }

// Per-pixel upstream gradient (explicit, or the fused masked-L1 prologue of Eq. 1 / Eq. 2),
// the saved forward state, and the pixel's reference colour / depth (its normalised render):
// the behind-accumulators are kept relative to it, so c − c̄ and z − z̄ — differences of nearly
// equal values when view-tied layers sit on one surface — keep fp32 relative precision.
struct PixelUp {
    float g0, g1, g2, gD, gS, T, r0, r1, r2, rz;
    uint32_t L;
    double lossv;
};

template <bool LOSS>
__device__ __forceinline__ PixelUp pixel_upstream(const BwdArgs &p, int px, int py, bool inside) {
    PixelUp u{0.f, 0.f, 0.f, 0.f, 0.f, 1.0f, 0.f, 0.f, 0.f, 0.f, 0u, 0.0};
    if (!inside) return u;
    const int pix = py * p.W + px;
    if (LOSS) {
        const float tDv = p.tD[pix];
        const float Sv = p.sil[pix];
        const bool U = tDv > 0.0f;
        const bool Wm = U && Sv > 0.99f && (p.vis ? p.vis[pix] != 0 : true);
        const bool mc = p.cmode ? Wm : true;
        const bool md = p.dmode ? Wm : U;
        float sc = 1.0f, sd = 1.0f;
        if (p.normalize) {
            sc = p.dev->count_c ? 1.0f / (float)p.dev->count_c : 0.0f;
            sd = p.dev->count_d ? 1.0f / (float)p.dev->count_d : 0.0f;
        }
        if (mc) {
            const float e0 = p.color[3 * pix] - p.tC[3 * pix];
            const float e1 = p.color[3 * pix + 1] - p.tC[3 * pix + 1];
            const float e2 = p.color[3 * pix + 2] - p.tC[3 * pix + 2];
            const float k = p.wc * sc;
            u.g0 = k * sgnf(e0); u.g1 = k * sgnf(e1); u.g2 = k * sgnf(e2);
            u.lossv += (double)k * ((double)fabsf(e0) + (double)fabsf(e1) + (double)fabsf(e2));
        }
        if (p.extra_dc) {   // e.g. the SSIM term of Eq. 2 (vtgs_ssim_loss)
            u.g0 += p.extra_dc[3 * pix]; u.g1 += p.extra_dc[3 * pix + 1]; u.g2 += p.extra_dc[3 * pix + 2];
        }
        if (md) {
            const float e = p.depth[pix] - tDv;
            const float k = p.wd * sd;
            u.gD = k * sgnf(e);
            u.lossv += (double)k * (double)fabsf(e);
        }
    } else {
        if (p.dC) { u.g0 = p.dC[3 * pix]; u.g1 = p.dC[3 * pix + 1]; u.g2 = p.dC[3 * pix + 2]; }
        if (p.dD) u.gD = p.dD[pix];
        if (p.dS) u.gS = p.dS[pix];
    }
    u.T = p.T_final[pix];
    u.L = p.last[pix];
    const float Sv = p.sil[pix];
    if (Sv > 0.0f) {
        const float inv = 1.0f / Sv;
        u.r0 = p.color[3 * pix] * inv; u.r1 = p.color[3 * pix + 1] * inv; u.r2 = p.color[3 * pix + 2] * inv;
        u.rz = p.depth[pix] * inv;
    }
    return u;
}

// Per batch of 32 sub-list entries the backward runs in two phases (composite_common.cuh):
//   phase 1 — lane i = pixel walks ITS candidate entries back to front, recovering T_i and the
//             behind-accumulator, and writes (ω = α_i T_i, dL/dα_i·w_i·[α unclamped]) into the
//             warp's 32×32 matrix M[entry][pixel] (0 for pairs that were not composited);
//   phase 2 — lane j = entry walks the pixels its footprint covers and sums that entry's
//             colour / opacity / σ / (u, v, z) gradient from M and the per-pixel upstream — a
//             per-Gaussian reduction with no shuffles; attribute gradients leave with one
//             float4 + one float global atomic per (Gaussian, sub-tile), the pose chain is
//             applied per (Gaussian, sub-tile) into the lane's 12 accumulators.
// One warp per sub-tile (4×8, composite_common.cuh), kBwdWarps warps per CTA, no block barriers.
constexpr int kBwdWarps = 2;
struct __align__(16) BwdStage {
    float4 A[32];   // u, v, D_c, escale
    float4 B[32];   // c, o
    float2 L[32];   // z, D_clamp
};

template <bool ATTR, bool POSE, bool LOSS, int MINB = 1>
__global__ void __launch_bounds__(kBwdWarps * 32, MINB) k_composite_bwd(BwdArgs p) {
    // per warp, one block: A (u, v, D_c, escale) | B (c, o) | L (z, D_clamp) — one base register
    // and immediate offsets address all three of a candidate's loads
    __shared__ BwdStage sS[kBwdWarps];
    __shared__ float4 sX[kBwdWarps][POSE ? 32 : 1];  // X_c and ±σ (−: σ clamped)
    __shared__ float4 sG[kBwdWarps][32];             // per pixel (g_C, g_D)
    // [kBwdWarps][32 entries][32 pixels]: phase 1 writes column = own lane (conflict-free per
    // half-warp phase of the 64-bit stores), phase 2 reads row = own lane, walking its pixel bits
    // from a lane-rotated start so the half-warp's reads spread over the banks
    extern __shared__ float2 sMdyn[];

    const int gsub = blockIdx.x * kBwdWarps + (int)(threadIdx.x >> 5);
    const int tile = gsub >> 3;
    const int wl_ = threadIdx.x >> 5;
    const int sub = gsub & 7;  // sub-tile 0..7 of the tile
    float2 (*M)[32] = reinterpret_cast<float2 (*)[32]>(sMdyn + (size_t)wl_ * 32 * 32);
    const char *sbase = reinterpret_cast<const char *>(&sS[wl_]);
    const int ty = tile / p.ntx, tx = tile - ty * p.ntx;
    const unsigned lane = lane_id();
    const int sx = sub_x0(tx, sub), sy = sub_y0(ty, sub);
    const int px = sx + pix_dx((int)lane), py = sy + pix_dy((int)lane);
    const bool inside = px < p.W && py < p.H;
    const float pxf = (float)px, pyf = (float)py;
    const int n = (int)p.tile_count[tile];
    const uint32_t *list = p.sub_lists + (size_t)8 * p.tile_start[tile] + (size_t)sub * n;
    const uint32_t *mlist = p.sub_masks + (size_t)8 * p.tile_start[tile] + (size_t)sub * n;
    VTGS_CHECK((uint64_t)8 * p.tile_start[tile] + (uint64_t)(sub + 1) * n <= p.sub_cap);
    PoseR P;
    if (POSE) pose_rotation(*p.view, P);

    const PixelUp up = pixel_upstream<LOSS>(p, px, py, inside);
    float g0 = up.g0, g1 = up.g1, g2 = up.g2, gD = up.gD, gS = up.gS, T = up.T;
    const float r0 = up.r0, r1 = up.r1, r2 = up.r2, rz = up.rz;
    uint32_t L = up.L;
    const double lossv = up.lossv;
    const bool on = inside && L > 0 && (g0 != 0.f || g1 != 0.f || g2 != 0.f || gD != 0.f || gS != 0.f);
    if (!on) L = 0;
    sG[wl_][lane] = make_float4(g0, g1, g2, gD);
    const unsigned onmask = __ballot_sync(kFullMask, on);
    const int wmax = (int)__reduce_max_sync(kFullMask, L);  // sub-list positions < wmax matter
    VTGS_CHECK(wmax <= (int)p.sub_count[tile * 8 + sub]);

    // Behind-accumulator, relative to the pixel's references and already dotted with the
    // (constant) upstream gradient: Fb = Σ_{j behind} w_j f_j with f_j = g_C·(c_j − c_ref) +
    // g_D (z_j − z_ref), w_j = α_j T_j / T_{i+1}; Tb = 1 − Σ w_j = Π (1 − α_j).  Then
    //   g·(x_i − x̄) + g_S (1 − S̄) = f_i − Fb + Kr·Tb,   Kr = g_C·c_ref + g_D z_ref + g_S,
    // one scalar recursion instead of one per channel, and no difference of nearly equal
    // colours / depths is ever formed in fp32 (R23).
    float Fb = 0.f, Tb = 1.0f;
    const float Kr = g0 * r0 + g1 * r1 + g2 * r2 + gD * rz + gS;
    float h0 = 0.f, h1 = 0.f, h2 = 0.f;
    float K00 = 0.f, K01 = 0.f, K02 = 0.f, K10 = 0.f, K11 = 0.f, K12 = 0.f, K20 = 0.f, K21 = 0.f, K22 = 0.f;
    const float fmean = 0.5f * (p.in.fx + p.in.fy);

    const int bb_top = wmax > 0 ? ((wmax - 1) >> 5) << 5 : -32;
    EntryRegs nxt;
    fetch_entry(nxt, list, bb_top + (int)lane, wmax, p.proj, p.col_opa, p.thr);
    uint32_t mnx = load_mask(mlist, bb_top + (int)lane, wmax);
    for (int bb = bb_top; bb >= 0; bb -= 32) {
        const EntryRegs cur = nxt;
        const uint32_t mcur = mnx;
        fetch_entry(nxt, list, bb - 32 + (int)lane, wmax, p.proj, p.col_opa, p.thr);
        mnx = load_mask(mlist, bb - 32 + (int)lane, wmax);  // next (lower) batch
        const int jj = bb + (int)lane;
        unsigned mj = 0u;
        float s2j = 1.0f;
        if (jj < wmax) {   // wmax ≤ the sub-list length
            VTGS_CHECK((int64_t)cur.g < p.N && cur.pr.z > 0.0f);
            const float s = fabsf(cur.pr.w);
            s2j = __fmul_rn(s, s);
            const float2 th = thr_unpack(cur.th, s2j);
            sS[wl_].A[lane] = make_float4(cur.pr.x, cur.pr.y, th.x, exp_scale(s2j));
            sS[wl_].B[lane] = cur.co;
            sS[wl_].L[lane] = make_float2(cur.pr.z, th.y);
            if (POSE)   // camera-space centre from the projection (x = (u − cx)·z / fx, …)
                sX[wl_][lane] = make_float4((cur.pr.x - p.in.cx) * cur.pr.z * rcp_approx(p.in.fx),
                                            (cur.pr.y - p.in.cy) * cur.pr.z * rcp_approx(p.in.fy), cur.pr.z, cur.pr.w);
            mj = mcur & onmask;   // the forward's candidate pixels with a nonzero upstream
        }
        __syncwarp();
        // candidates at positions ≥ the pixel's `last` were not composited: drop them from the
        // lane's column (phase 1) and, through the transposed threshold masks, from each entry's
        // pixel set (phase 2); the rest are re-decided exactly as the forward decided (d² ≤ D_c)
        const int rem = (int)L - bb;
        const unsigned alive = rem >= 32 ? 0xffffffffu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
        unsigned bits = transpose32(mj, lane) & alive;
        mj &= transpose32(alive, lane);
        // ---- phase 1: lane = pixel, back to front, two pairs per iteration: both pairs' loads,
        // α (the forward's exact bits), 1/(1−α) and f carry no loop state and are computed
        // together; the recursion (T, Fb, Tb) then runs over the two in order ----
        auto stage_a = [&](int k, bool v, float &a, float &rc, float &wgt, float &fi, bool &comp, bool &aclamp) {
            float4 A, B;
            float2 lo;
            if (v) {   // predicated loads: lanes without a candidate add no shared-memory traffic
                const char *pk = sbase + 16 * k;
                A = *reinterpret_cast<const float4 *>(pk);
                B = *reinterpret_cast<const float4 *>(pk + offsetof(BwdStage, B));
                lo = *reinterpret_cast<const float2 *>(sbase + offsetof(BwdStage, L) + 8 * k);
            }
            const float d2 = pair_d2(pxf, pyf, A.x, A.y);
            comp = v && d2 <= A.z;         // the forward's exact decision (3σ and the α floor)
            a = pair_alpha(d2, A.w, B.w, lo.y, wgt);   // the forward's α (same entry data, thresholds)
            aclamp = d2 <= lo.y;
            rc = rcp_approx(1.0f - a);
            fi = g0 * (B.x - r0) + g1 * (B.y - r1) + g2 * (B.z - r2) + gD * (lo.x - rz);
        };
        // branch-free: every value is computed and a pair that was not composited selects the
        // old state (a branch here cost a reconvergence per pair)
        auto stage_b = [&](int k, bool comp, bool aclamp, float a, float rc, float wgt, float fi, bool store) {
            const float oma = 1.0f - a;
            const float Ti = T * rc;
            const float om = comp ? a * Ti : 0.f;
            // M.y = dL/dα · w (0 when α is clamped): phase 2 needs only that product
            const float dAe = (comp && !aclamp) ? Ti * (fi - Fb + Kr * Tb) * wgt : 0.f;
            Fb = comp ? a * fi + oma * Fb : Fb;
            Tb = comp ? oma * Tb : Tb;
            T = comp ? Ti : T;
            if (store) M[k][lane] = make_float2(om, dAe);   // predicated: no second candidate, no store
        };
        while (bits) {
            const int k0 = msb_index(bits);
            bits ^= 1u << k0;
            const bool v1 = bits != 0u;
            const int k1 = msb_index(bits) & 31;
            if (v1) bits ^= 1u << k1;
            float a0, rc0, w0, f0, a1, rc1, w1, f1;
            bool c0, cl0, c1, cl1;
            stage_a(k0, true, a0, rc0, w0, f0, c0, cl0);
            stage_a(k1, v1, a1, rc1, w1, f1, c1, cl1);
            stage_b(k0, c0, cl0, a0, rc0, w0, f0, true);
            stage_b(k1, c1, cl1, a1, rc1, w1, f1, v1);   // c1 is false without a second candidate
        }
        __syncwarp();
        // ---- phase 2: lane = entry, over the pixels that composited it, two pixels per
        // iteration (both pixels' M and upstream loads issued before either is accumulated) ----
        if (mj) {
            const float4 B = cur.co;
            const float z = cur.pr.z;
            float dc0 = 0.f, dc1 = 0.f, dc2 = 0.f, dop = 0.f, sw2 = 0.f, swx = 0.f, swy = 0.f, dzd = 0.f;
            unsigned mm = __funnelshift_r(mj, mj, lane);  // rotate right by lane
            const float ux = cur.pr.x, uy = cur.pr.y;
            // branch-free: a pair that was not composited holds (0, 0) in M and adds exact zeros
            auto accum = [&](int i, float2 md, float4 gp) {
                dc0 = fmaf(gp.x, md.x, dc0);
                dc1 = fmaf(gp.y, md.x, dc1);
                dc2 = fmaf(gp.z, md.x, dc2);
                dzd = fmaf(gp.w, md.x, dzd);
                const float dx = (float)(sx + pix_dx(i)) - ux, dy = (float)(sy + pix_dy(i)) - uy;
                const float d2 = dx * dx + dy * dy;
                const float dw = md.y;  // dL/dα · w  (= ∂L/∂o contribution; 0 when α clamped)
                dop += dw;
                sw2 = fmaf(dw, d2, sw2);
                swx = fmaf(dw, dx, swx);
                swy = fmaf(dw, dy, swy);
            };
            while (mm) {
                const int i0 = ((__ffs(mm) - 1) + (int)lane) & 31;
                mm &= mm - 1u;
                const bool v1 = mm != 0u;
                const int i1 = ((__ffs(mm) - 1) + (int)lane) & 31;
                mm &= mm - 1u;
                const float2 md0 = M[lane][i0];
                const float4 gp0 = sG[wl_][i0];
                float2 md1 = make_float2(0.f, 0.f);
                float4 gp1 = make_float4(0.f, 0.f, 0.f, 0.f);
                if (v1) {
                    md1 = M[lane][i1];
                    gp1 = sG[wl_][i1];
                }
                accum(i0, md0, gp0);
                accum(i1, md1, gp1);   // zeros when there is no second pixel
            }
            // dL/dw·w = dL/dα·o·w;  ∂w/∂σ = w d²/σ³, ∂w/∂u = w (x−u)/σ², ∂w/∂v = w (y−v)/σ²
            const float s = fabsf(cur.pr.w);
            const float inv_s2 = rcp_approx(s * s);
            const float dsg = B.w * sw2 * inv_s2 * rcp_approx(s);
            if (ATTR && (int64_t)cur.g >= p.learn_begin && (int64_t)cur.g < p.learn_end) {
                const bool wc = p.want & VTGS_GRAD_COLOR, wo = p.want & VTGS_GRAD_OPACITY;
                const float dr = ((p.want & VTGS_GRAD_RADIUS) && cur.pr.w > 0.f) ? dsg * fmean * rcp_approx(z) : 0.f;
                if (p.det) {   // deterministic merge: fixed-point integer atomics
                    unsigned long long *q = p.det + (size_t)5 * cur.g;
                    if (wc) { det_add(q, dc0); det_add(q + 1, dc1); det_add(q + 2, dc2); }
                    if (wo) det_add(q + 3, dop);
                    det_add(q + 4, dr);
                } else {
                    if ((wc && (dc0 != 0.f || dc1 != 0.f || dc2 != 0.f)) || (wo && dop != 0.f))
                        atomicAdd(&p.d_col_opa[cur.g],
                                  make_float4(wc ? dc0 : 0.f, wc ? dc1 : 0.f, wc ? dc2 : 0.f, wo ? dop : 0.f));
                    if (dr != 0.f) atomicAdd(&p.d_radius[cur.g], dr);  // ∂σ/∂r = f/z
                }
            }
            if (POSE) {
                const float4 X = sX[wl_][lane];
                const float du = B.w * swx * inv_s2, dv = B.w * swy * inv_s2;
                const float iz = rcp_approx(z);
                float dzt = dzd - (du * (cur.pr.x - p.in.cx) + dv * (cur.pr.y - p.in.cy)) * iz;
                if (X.w > 0.f) dzt -= dsg * s * iz;  // ∂σ/∂z = −σ/z (unclamped)
                const float gx = du * p.in.fx * iz, gy = dv * p.in.fy * iz, gz = dzt;
                if ((p.want & VTGS_GRAD_POSITION) && (gx != 0.f || gy != 0.f || gz != 0.f))   // dL/dX_w = R g
                    atomicAdd(&p.d_position[cur.g],
                              make_float4(P.R[0] * gx + P.R[1] * gy + P.R[2] * gz, P.R[3] * gx + P.R[4] * gy + P.R[5] * gz,
                                          P.R[6] * gx + P.R[7] * gy + P.R[8] * gz, 0.f));
                h0 += gx; h1 += gy; h2 += gz;
                K00 = fmaf(X.x, gx, K00); K01 = fmaf(X.x, gy, K01); K02 = fmaf(X.x, gz, K02);
                K10 = fmaf(X.y, gx, K10); K11 = fmaf(X.y, gy, K11); K12 = fmaf(X.y, gz, K12);
                K20 = fmaf(X.z, gx, K20); K21 = fmaf(X.z, gy, K21); K22 = fmaf(X.z, gz, K22);
            }
        }
        __syncwarp();
    }

    if (!POSE && LOSS) {   // loss only (mapping): lanes → warp → CTA, one contiguous double per CTA
        double v = lossv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
        if (lane == 0) reinterpret_cast<double *>(&sS[wl_].A[0])[0] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < kBwdWarps; ++i) s += reinterpret_cast<const double *>(&sS[i].A[0])[0];
            p.partials[blockIdx.x] = s;   // k_loss_finalize: row order, coalesced
        }
    }
    if (POSE) {   // fixed-order reduction: lanes → warp → CTA (one partial per CTA)
        // each warp's 13 doubles go into its own (now dead) row of sA: no extra shared memory
        // (K7's occupancy is shared-memory bound: 11 two-warp CTAs per SM need ≤ 19.9 KB each)
        double v[13] = {h0, h1, h2, K00, K01, K02, K10, K11, K12, K20, K21, K22, lossv};
#pragma unroll
        for (int q = 0; q < 13; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(kFullMask, v[q], o);
        }
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 13; ++q) reinterpret_cast<double *>(&sS[wl_].A[0])[q] = v[q];
        __syncthreads();
        if (threadIdx.x < 13) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < kBwdWarps; ++i) s += reinterpret_cast<const double *>(&sS[i].A[0])[threadIdx.x];
            p.partials[(size_t)blockIdx.x * 16 + threadIdx.x] = s;
        }
    }
}

// ------------------------------------------------------------------------------------------
// Pose-only backward (tracking, Eq. 1: "keep all Gaussians in the scene fixed, and merely
// optimize the pose"), ring walk.  The pose gradient is linear in the per-pair
// terms, so each composited pair's dL/dX_c goes straight into the lane's 12 accumulators
// (Σ g, Σ X_c gᵀ): no per-Gaussian reduction, so the lanes walk back to front ACROSS batch
// boundaries at their own pace over a ring of R resident batches, like the forward's ring
// (k_composite_fwd_ring): a lane only waits when it needs a batch not yet built and the ring is
// R batches ahead of the slowest lane.  The lane's candidates are the forward's
// candidates, re-decided with the forward's exact thresholds (d² ≤ D_c, candidates before `last`).
// Per entry the slot keeps A = (u, v, D_c, escale), B = (c, o), Xq = (X_c.x, X_c.y, z, o/σ²) and
// (±1/z (−: σ clamped, ∂σ/∂z = 0), D_clamp); per pair
//   q = (o/σ²)·dL/dα·w,  g = (q·dx·fx/z, q·dy·fy/z, g_D·ω − q·dx·(u−cx)/z − q·dy·(v−cy)/z − q·d²·[1/z])
// ------------------------------------------------------------------------------------------
template <int R>
struct PoseRing {
    float4 A[R * 32];        // u, v, D_c, escale
    float4 B[R * 32];        // c, o
    float4 Xq[R * 32];       // X_c.x, X_c.y, z, o/σ²
    float2 iz[R * 32];       // ±1/z (−: σ clamped), D_clamp
    uint32_t bits[R * 32];   // per lane: its composited entries of the batch (bit k = entry k)
};

constexpr int kPoseRingWarps = 2;
constexpr int kPoseInner = 8;   // lane-independent steps between warp checks (4 → 8: tracking backward 14.5 → 14.0 ms per frame)

template <int R, bool LOSS>
__global__ void __launch_bounds__(kPoseRingWarps * 32) k_composite_bwd_pose_ring(BwdArgs p) {
    extern __shared__ float4 pose_ring_smem[];
    static_assert((R & (R - 1)) == 0, "ring depth must be a power of two");
    const int wl_ = threadIdx.x >> 5;
    PoseRing<R> &ring = reinterpret_cast<PoseRing<R> *>(pose_ring_smem)[wl_];
    const int gsub = blockIdx.x * kPoseRingWarps + wl_;
    const int tile = gsub >> 3;
    const int sub = gsub & 7;
    const int ty = tile / p.ntx, tx = tile - ty * p.ntx;
    const unsigned lane = lane_id();
    const int sx = sub_x0(tx, sub), sy = sub_y0(ty, sub);
    const int px = sx + pix_dx((int)lane), py = sy + pix_dy((int)lane);
    const bool inside = px < p.W && py < p.H;
    const float pxf = (float)px, pyf = (float)py;
    const int n = (int)p.tile_count[tile];
    const uint32_t *list = p.sub_lists + (size_t)8 * p.tile_start[tile] + (size_t)sub * n;
    const uint32_t *mlist = p.sub_masks + (size_t)8 * p.tile_start[tile] + (size_t)sub * n;
    const int cnt = (int)p.sub_count[tile * 8 + sub];
    VTGS_CHECK(cnt <= n && (uint64_t)8 * p.tile_start[tile] + (uint64_t)(sub + 1) * n <= p.sub_cap);
    const PixelUp up = pixel_upstream<LOSS>(p, px, py, inside);
    const float g0 = up.g0, g1 = up.g1, g2 = up.g2, gD = up.gD, gS = up.gS;
    const float r0 = up.r0, r1 = up.r1, r2 = up.r2, rz = up.rz;
    float T = up.T;
    const bool on = inside && up.L > 0 && (g0 != 0.f || g1 != 0.f || g2 != 0.f || gD != 0.f || gS != 0.f);
    const int L = on ? (int)up.L : 0;
    const unsigned onmask = __ballot_sync(kFullMask, on);
    const int wmax = (int)__reduce_max_sync(kFullMask, (unsigned)L);
    const int bb_top = wmax > 0 ? ((wmax - 1) >> 5) << 5 : -32;
    const int nb = (bb_top >> 5) + 1;   // batch t covers sub-list positions [bb_top − 32t, +32)
    float Fb = 0.f, Tb = 1.0f;
    const float Kr = g0 * r0 + g1 * r1 + g2 * r2 + gD * rz + gS;
    float h0 = 0.f, h1 = 0.f, h2 = 0.f;
    float K00 = 0.f, K01 = 0.f, K02 = 0.f, K10 = 0.f, K11 = 0.f, K12 = 0.f, K20 = 0.f, K21 = 0.f, K22 = 0.f;
    const float fx = p.in.fx, fy = p.in.fy, cxp = p.in.cx, cyp = p.in.cy;

    EntryStream st;
    stream_start(st, list, bb_top + (int)lane, bb_top - 32 + (int)lane, cnt, p.proj, p.col_opa, p.thr);
    uint32_t mnx = load_mask(mlist, bb_top + (int)lane, wmax);
    const float ifx = 1.0f / fx, ify = 1.0f / fy;
    int built = 0;
    auto build = [&]() {
        const int bb = bb_top - 32 * built;
        const int slot = (built & (R - 1)) * 32;
        unsigned mj = 0u;
        if (bb + (int)lane < wmax) {   // wmax ≤ cnt
            const EntryRegs &e = st.e;
            VTGS_CHECK((int64_t)e.g < p.N && e.pr.z > 0.0f && wmax <= cnt);
            const float s = fabsf(e.pr.w);
            const float s2 = __fmul_rn(s, s);
            const float2 th = thr_unpack(e.th, s2);
            ring.A[slot + lane] = make_float4(e.pr.x, e.pr.y, th.x, exp_scale(s2));
            ring.B[slot + lane] = e.co;
            // X_c from the projection itself (x = (u − cx)·z / fx, …): no gather of the world centre
            const float iz = rcp_approx(e.pr.z);
            ring.Xq[slot + lane] = make_float4((e.pr.x - cxp) * e.pr.z * ifx, (e.pr.y - cyp) * e.pr.z * ify, e.pr.z,
                                               e.co.w * rcp_approx(s2));
            ring.iz[slot + lane] = make_float2(e.pr.w > 0.f ? iz : -iz, th.y);
            mj = mnx & onmask;   // the forward's candidate pixels with a nonzero upstream
        }
        // positions ≥ the pixel's `last` were not composited
        const int rem = L - bb;
        const unsigned alive = rem >= 32 ? 0xffffffffu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
        ring.bits[slot + lane] = transpose32(mj, lane) & alive;
        ++built;
        const int nidx = bb - 32 + (int)lane;
        stream_next(st, list, bb - 64 + (int)lane, cnt, p.proj, p.col_opa, p.thr);
        mnx = load_mask(mlist, nidx, wmax);
    };
    while (built < nb && built < R) build();
    __syncwarp();

    int b = -1;
    unsigned cur = 0u;
    int soff = 0;
    auto advance = [&]() {
        ++b;
        soff = (b & (R - 1)) * 32;
        cur = ring.bits[soff + lane];
    };
    for (;;) {
#pragma unroll
        for (int it = 0; it < kPoseInner; ++it) {
            if (cur == 0u && b + 1 < built) advance();
            const bool has = cur != 0u;
            const int k = 31 - __clz(cur);   // highest remaining entry (back to front)
            cur &= ~(1u << (k & 31));
            float4 A, B;
            if (has) {   // predicated loads: idle lanes add no shared-memory traffic
                A = ring.A[soff + k];
                B = ring.B[soff + k];
            }
            const float dx = __fsub_rn(pxf, A.x), dy = __fsub_rn(pyf, A.y);
            const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
            if (has && d2 <= A.z) {   // composited: the forward's exact decision
                const float4 Xq = ring.Xq[soff + k];
                const float2 izl = ring.iz[soff + k];
                const float izs = izl.x;
                float wgt;
                const float a = pair_alpha(d2, A.w, B.w, izl.y, wgt);   // the forward's α
                const bool aclamp = d2 <= izl.y;
                const float oma = 1.0f - a;
                const float Ti = T * rcp_approx(oma);
                const float om = a * Ti;
                const float fi = g0 * (B.x - r0) + g1 * (B.y - r1) + g2 * (B.z - r2) + gD * (Xq.z - rz);
                const float dAe = aclamp ? 0.f : Ti * (fi - Fb + Kr * Tb) * wgt;
                Fb = a * fi + oma * Fb;
                Tb = oma * Tb;
                T = Ti;
                const float iz = fabsf(izs), kz = izs > 0.f ? izs : 0.f;
                const float q = Xq.w * dAe;
                const float du = q * dx, dv = q * dy;
                const float gx = du * fx * iz, gy = dv * fy * iz;
                const float gz = gD * om - (du * (A.x - cxp) + dv * (A.y - cyp)) * iz - q * d2 * kz;
                const float X0 = Xq.x, X1 = Xq.y, X2 = Xq.z;
                h0 += gx; h1 += gy; h2 += gz;
                K00 = fmaf(X0, gx, K00); K01 = fmaf(X0, gy, K01); K02 = fmaf(X0, gz, K02);
                K10 = fmaf(X1, gx, K10); K11 = fmaf(X1, gy, K11); K12 = fmaf(X1, gz, K12);
                K20 = fmaf(X2, gx, K20); K21 = fmaf(X2, gy, K21); K22 = fmaf(X2, gz, K22);
            }
        }
        while (cur == 0u && b + 1 < built) advance();
        const bool live = cur != 0u || b + 1 < nb;
        if (!__any_sync(kFullMask, live)) break;
        const bool blocked = cur == 0u && b + 1 < nb && b + 1 >= built;
        if (__any_sync(kFullMask, blocked)) {
            const int need = !live ? 0x7fffffff : (cur ? b : b + 1);   // earliest batch still needed
            const int lo = (int)__reduce_min_sync(kFullMask, (unsigned)need);
            if (built < nb && built < lo + R) {
                while (built < nb && built < lo + R) build();
                __syncwarp();
            }
        }
    }

    __shared__ double sRed[kPoseRingWarps][13];   // fixed-order reduction: lanes → warp → CTA
    double v[13] = {h0, h1, h2, K00, K01, K02, K10, K11, K12, K20, K21, K22, up.lossv};
#pragma unroll
    for (int q = 0; q < 13; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(kFullMask, v[q], o);
    }
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 13; ++q) sRed[wl_][q] = v[q];
    __syncthreads();
    if (threadIdx.x < 13) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < kPoseRingWarps; ++i) s += sRed[i][threadIdx.x];
        p.partials[(size_t)blockIdx.x * 16 + threadIdx.x] = s;
    }
}

// ------------------------------------------------------------------------------------------
// Mapping backward as a ring walk (VTGS_BWD_RING): phase 1 (lane = pixel) walks its candidates
// back to front ACROSS batch boundaries at its own pace over R resident batches, like the
// forward's ring, and writes each pair's (ω, dL/dα·w) into a per-warp shared-memory pair ring
// at a popc-ranked slot: entry k's pairs sit at base_k + rank of the pixel in k's pixel mask.
// Phase 2 (lane = entry) runs per batch once every lane has passed it, reads the entry's pairs
// in pixel order and leaves with the same per-(Gaussian, sub-tile) atomics as k_composite_bwd.
// The arithmetic per pair and per entry is that of k_composite_bwd (same decisions, same α,
// same recursion, same per-entry summation order), only the schedule differs.
// ------------------------------------------------------------------------------------------
template <int R>
struct BwdRing {
    float4 A[R * 32];         // u, v, D_c, escale
    float4 B[R * 32];         // c, o
    float4 Z[R * 32];         // z, D_clamp, σ (signed: − when clamped), gid (bits)
    uint2 EM[R * 32];         // entry: pixel mask (candidate ∧ upstream ≠ 0 ∧ before the pixel's last), pair base
    uint32_t bits[R * 32];    // pixel lane: its entries of the batch (bit k = entry k)
};
constexpr int kRingPairs = 1024;   // ≥ 32 × 32: any one batch fits, so the walk cannot deadlock
constexpr int kRingInner = 6;      // lane-independent steps between warp checks
template <int R>
__host__ __device__ constexpr size_t bwd_ring_warp_bytes() {
    return sizeof(BwdRing<R>) + sizeof(float2) * kRingPairs + sizeof(float4) * 32;
}

template <int R, bool LOSS>
__global__ void __launch_bounds__(kBwdWarps * 32) k_composite_bwd_ring(BwdArgs p) {
    extern __shared__ float4 bwd_ring_smem[];
    static_assert((R & (R - 1)) == 0, "ring depth must be a power of two");
    constexpr unsigned CP = kRingPairs;
    const int wl_ = threadIdx.x >> 5;
    char *wbase = reinterpret_cast<char *>(bwd_ring_smem) + (size_t)wl_ * bwd_ring_warp_bytes<R>();
    BwdRing<R> &ring = *reinterpret_cast<BwdRing<R> *>(wbase);
    float2 *pairs = reinterpret_cast<float2 *>(wbase + sizeof(BwdRing<R>));
    float4 *sG = reinterpret_cast<float4 *>(wbase + sizeof(BwdRing<R>) + sizeof(float2) * CP);
    const int gsub = blockIdx.x * kBwdWarps + wl_;
    const int tile = gsub >> 3;
    const int sub = gsub & 7;
    const int ty = tile / p.ntx, tx = tile - ty * p.ntx;
    const unsigned lane = lane_id();
    const unsigned lmlt = lanemask_lt();
    const int sx = sub_x0(tx, sub), sy = sub_y0(ty, sub);
    const int px = sx + pix_dx((int)lane), py = sy + pix_dy((int)lane);
    const bool inside = px < p.W && py < p.H;
    const float pxf = (float)px, pyf = (float)py;
    const int n = (int)p.tile_count[tile];
    const uint32_t *list = p.sub_lists + (size_t)8 * p.tile_start[tile] + (size_t)sub * n;
    const uint32_t *mlist = p.sub_masks + (size_t)8 * p.tile_start[tile] + (size_t)sub * n;
    const int cnt = (int)p.sub_count[tile * 8 + sub];
    VTGS_CHECK(cnt <= n && (uint64_t)8 * p.tile_start[tile] + (uint64_t)(sub + 1) * n <= p.sub_cap);
    const PixelUp up = pixel_upstream<LOSS>(p, px, py, inside);
    const float g0 = up.g0, g1 = up.g1, g2 = up.g2, gD = up.gD, gS = up.gS;
    const float r0 = up.r0, r1 = up.r1, r2 = up.r2, rz = up.rz;
    float T = up.T;
    const bool on = inside && up.L > 0 && (g0 != 0.f || g1 != 0.f || g2 != 0.f || gD != 0.f || gS != 0.f);
    const int L = on ? (int)up.L : 0;
    sG[lane] = make_float4(g0, g1, g2, gD);
    const unsigned onmask = __ballot_sync(kFullMask, on);
    const int wmax = (int)__reduce_max_sync(kFullMask, (unsigned)L);
    VTGS_CHECK(wmax <= cnt);
    const int bb_top = wmax > 0 ? ((wmax - 1) >> 5) << 5 : -32;
    const int nb = (bb_top >> 5) + 1;   // batch t covers sub-list positions [bb_top − 32t, +32)
    float Fb = 0.f, Tb = 1.0f;          // behind-accumulators (k_composite_bwd)
    const float Kr = g0 * r0 + g1 * r1 + g2 * r2 + gD * rz + gS;
    const float fmean = 0.5f * (p.in.fx + p.in.fy);

    EntryStream st;
    stream_start(st, list, bb_top + (int)lane, bb_top - 32 + (int)lane, cnt, p.proj, p.col_opa, p.thr);
    uint32_t mnx = load_mask(mlist, bb_top + (int)lane, wmax);
    int built = 0;          // batches committed (visible to phase 1)
    int flushed = 0;        // batches reduced by phase 2
    unsigned head = 0u, tail = 0u;   // pair ring in use: [tail, head)
    bool pend = false;      // batch `built` staged (slot written) but its pairs not yet allocated
    unsigned pem = 0u, pbits = 0u;   // the staged batch: entry lane's pixel mask, pixel lane's entries
    auto stage = [&]() {
        const int bb = bb_top - 32 * built;
        const int slot = (built & (R - 1)) * 32;
        unsigned mj = 0u;
        if (bb + (int)lane < wmax) {
            const EntryRegs &e = st.e;
            VTGS_CHECK((int64_t)e.g < p.N && e.pr.z > 0.0f);
            const float s = fabsf(e.pr.w);
            const float s2 = __fmul_rn(s, s);
            const float2 th = thr_unpack(e.th, s2);
            ring.A[slot + lane] = make_float4(e.pr.x, e.pr.y, th.x, exp_scale(s2));
            ring.B[slot + lane] = e.co;
            ring.Z[slot + lane] = make_float4(e.pr.z, th.y, e.pr.w, __uint_as_float(e.g));
            mj = mnx & onmask;   // the forward's candidate pixels with a nonzero upstream
        }
        const int rem = L - bb;  // positions ≥ the pixel's `last` were not composited
        const unsigned alive = rem >= 32 ? 0xffffffffu : (rem <= 0 ? 0u : ((1u << rem) - 1u));
        pbits = transpose32(mj, lane) & alive;
        pem = mj & transpose32(alive, lane);
        pend = true;
        stream_next(st, list, bb - 64 + (int)lane, cnt, p.proj, p.col_opa, p.thr);
        mnx = load_mask(mlist, bb - 32 + (int)lane, wmax);
    };
    auto try_commit = [&]() {
        const unsigned c = __popc(pem);
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(kFullMask, incl, o);
            if ((int)lane >= o) incl += t;
        }
        const unsigned tot = __shfl_sync(kFullMask, incl, 31);
        if (head - tail + tot > CP) return;
        const int slot = (built & (R - 1)) * 32;
        ring.EM[slot + lane] = make_uint2(pem, head + incl - c);
        ring.bits[slot + lane] = pbits;
        head += tot;
        ++built;
        pend = false;
    };
    // phase 2 of batch f (lane = entry): the entry's pairs in ascending pixel order
    auto reduce = [&](int f) {
        const int slot = (f & (R - 1)) * 32;
        const uint2 em = ring.EM[slot + lane];
        const unsigned mj = em.x;
        if (mj) {
            const float4 A = ring.A[slot + lane];
            const float4 Zs = ring.Z[slot + lane];
            const float o = ring.B[slot + lane].w;
            const float ux = A.x, uy = A.y, z = Zs.x, sg = Zs.z;
            const uint32_t g = __float_as_uint(Zs.w);
            float dc0 = 0.f, dc1 = 0.f, dc2 = 0.f, dop = 0.f, sw2 = 0.f;
            auto accum = [&](int i, float2 md, float4 gp) {
                if (md.x != 0.f) {   // composited (ω > 0 for every composited pair)
                    dc0 = fmaf(gp.x, md.x, dc0);
                    dc1 = fmaf(gp.y, md.x, dc1);
                    dc2 = fmaf(gp.z, md.x, dc2);
                    const float dx = (float)(sx + pix_dx(i)) - ux, dy = (float)(sy + pix_dy(i)) - uy;
                    const float d2 = dx * dx + dy * dy;
                    dop += md.y;
                    sw2 = fmaf(md.y, d2, sw2);
                }
            };
            unsigned mm = mj;
            unsigned q = em.y;
            while (mm) {
                const int i0 = __ffs(mm) - 1;
                mm &= mm - 1u;
                const bool v1 = mm != 0u;
                const int i1 = (__ffs(mm) - 1) & 31;
                mm &= mm - 1u;
                const float2 md0 = pairs[q & (CP - 1)];
                const float4 gp0 = sG[i0];
                float2 md1 = make_float2(0.f, 0.f);
                float4 gp1;
                if (v1) {
                    md1 = pairs[(q + 1) & (CP - 1)];
                    gp1 = sG[i1];
                }
                q += 2;
                accum(i0, md0, gp0);
                accum(i1, md1, gp1);
            }
            const float s = fabsf(sg);
            const float inv_s2 = rcp_approx(s * s);
            const float dsg = o * sw2 * inv_s2 * rcp_approx(s);
            if ((int64_t)g >= p.learn_begin && (int64_t)g < p.learn_end) {
                const bool wc = p.want & VTGS_GRAD_COLOR, wo = p.want & VTGS_GRAD_OPACITY;
                const float dr = ((p.want & VTGS_GRAD_RADIUS) && sg > 0.f) ? dsg * fmean * rcp_approx(z) : 0.f;
                if (p.det) {
                    unsigned long long *qd = p.det + (size_t)5 * g;
                    if (wc) { det_add(qd, dc0); det_add(qd + 1, dc1); det_add(qd + 2, dc2); }
                    if (wo) det_add(qd + 3, dop);
                    det_add(qd + 4, dr);
                } else {
                    if ((wc && (dc0 != 0.f || dc1 != 0.f || dc2 != 0.f)) || (wo && dop != 0.f))
                        atomicAdd(&p.d_col_opa[g],
                                  make_float4(wc ? dc0 : 0.f, wc ? dc1 : 0.f, wc ? dc2 : 0.f, wo ? dop : 0.f));
                    if (dr != 0.f) atomicAdd(&p.d_radius[g], dr);
                }
            }
        }
        tail = __shfl_sync(kFullMask, em.y + __popc(mj), 31);   // the batch's pairs are free again
    };

    while (built < nb && built < R) {   // first fill: R batches (or what the pair ring holds)
        stage();
        try_commit();
        if (pend) break;
    }
    __syncwarp();

    int b = -1;
    unsigned cur = 0u;
    int soff = 0;
    auto advance = [&]() {
        ++b;
        soff = (b & (R - 1)) * 32;
        cur = ring.bits[soff + lane];
    };
    for (;;) {
#pragma unroll
        for (int it = 0; it < kRingInner; ++it) {
            if (cur == 0u && b + 1 < built) advance();
            const bool has = cur != 0u;
            const int k = 31 - __clz(cur);   // highest remaining entry (back to front)
            cur &= ~(1u << (k & 31));
            float4 A, B;
            float2 Zl;
            uint2 em;
            if (has) {   // predicated loads: idle lanes add no shared-memory traffic
                A = ring.A[soff + k];
                B = ring.B[soff + k];
                Zl = *reinterpret_cast<const float2 *>(&ring.Z[soff + k]);
                em = ring.EM[soff + k];
            }
            const float d2 = pair_d2(pxf, pyf, A.x, A.y);
            float om = 0.f, dAe = 0.f;
            if (has && d2 <= A.z) {   // composited: the forward's exact decision
                float wgt;
                const float a = pair_alpha(d2, A.w, B.w, Zl.y, wgt);   // the forward's α
                const bool aclamp = d2 <= Zl.y;
                const float oma = 1.0f - a;
                const float Ti = T * rcp_approx(oma);
                om = a * Ti;
                const float fi = g0 * (B.x - r0) + g1 * (B.y - r1) + g2 * (B.z - r2) + gD * (Zl.x - rz);
                dAe = aclamp ? 0.f : Ti * (fi - Fb + Kr * Tb) * wgt;
                Fb = a * fi + oma * Fb;
                Tb = oma * Tb;
                T = Ti;
            }
            if (has) pairs[(em.y + __popc(em.x & lmlt)) & (CP - 1)] = make_float2(om, dAe);
        }
        while (cur == 0u && b + 1 < built) advance();
        const bool live = cur != 0u || b + 1 < nb;
        if (!__any_sync(kFullMask, live)) break;
        const unsigned need = !live ? 0x7fffffffu : (unsigned)(cur ? b : b + 1);   // earliest batch still needed
        const int lo = (int)__reduce_min_sync(kFullMask, need);
        if (flushed < lo && flushed < built) {
            __syncwarp();   // phase 1's pair stores before phase 2's loads
            do reduce(flushed++);
            while (flushed < lo && flushed < built);
        }
        const bool blocked = cur == 0u && b + 1 < nb && b + 1 >= built;
        if (__any_sync(kFullMask, blocked)) {   // lazy build: up to the furthest batch a live lane needs
            const int hi = (int)__reduce_max_sync(kFullMask, live ? need : 0u);
            const int target = min(min(nb, flushed + R), hi + 1);
            if (pend) try_commit();
            while (!pend && built < target) {
                stage();
                try_commit();
            }
            __syncwarp();
        }
    }
    __syncwarp();
    while (flushed < built) reduce(flushed++);

    if (LOSS) {   // fixed-order loss reduction: lanes → warp → CTA (the contiguous rows k_loss_finalize sums)
        double v = up.lossv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
        __shared__ double sRedL[kBwdWarps];
        if (lane == 0) sRedL[wl_] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < kBwdWarps; ++i) s += sRedL[i];
            p.partials[blockIdx.x] = s;   // k_loss_finalize: row order, coalesced
        }
    }
}

// mask counts for the mean-normalised loss (normalize = 1)
__global__ void __launch_bounds__(256) k_l1_count(const float *__restrict__ sil, const float *__restrict__ tD,
                                                  const uint8_t *__restrict__ vis, int npx, int cmode,
                                                  int dmode, DevScalars *dev) {
    unsigned cc = 0, cd = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npx; i += gridDim.x * blockDim.x) {
        const bool U = tD[i] > 0.0f;
        const bool Wm = U && sil[i] > 0.99f && (vis ? vis[i] != 0 : true);
        cc += cmode ? Wm : 1u;
        cd += dmode ? Wm : U;
    }
    cc = __reduce_add_sync(kFull, cc);   // warp → block (shared) → one atomic pair per block
    cd = __reduce_add_sync(kFull, cd);
    __shared__ unsigned sc[8], sd[8];
    const int w = threadIdx.x >> 5;
    if (lane_id() == 0) { sc[w] = cc; sd[w] = cd; }
    __syncthreads();
    if (threadIdx.x < 32) {
        const unsigned a = __reduce_add_sync(kFull, threadIdx.x < 8 ? sc[threadIdx.x] : 0u);
        const unsigned b = __reduce_add_sync(kFull, threadIdx.x < 8 ? sd[threadIdx.x] : 0u);
        if (threadIdx.x == 0) {
            atomicAdd(&dev->count_c, a);
            atomicAdd(&dev->count_d, b);
        }
    }
}

// Fixed-order sum of the per-tile partials, then the rotation chain (DESIGN.md §3 step 11):
//   dL/dt = −R Σg,  dL/dR = R Σ X_c gᵀ,  dL/dq̂ = Σ_ab (dL/dR)_ab ∂R_ab/∂q̂,
//   dL/dq = (dL/dq̂ − q̂ (q̂·dL/dq̂)) / |q|.
constexpr int kFinThreads = 256;
constexpr int kFinBlocks = 64;

// Two-level fixed-order reduction: block b sums rows [b·R, (b+1)·R) of the per-CTA partials
// into partials2[b]; the last block to finish (ticket) sums partials2[0 .. kFinBlocks) in index
// order — deterministic, and the row loads of the 64 blocks run in parallel.
// Fixed-order block sum of 13 values: butterfly within each warp, then warp 0 over the warps'
// sums; the result lands in red[0][0..12].
__device__ __forceinline__ void block_sum13(double acc[13], double (*red)[13]) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int q = 0; q < 13; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(kFull, acc[q], o);
    }
    __syncthreads();   // red may still be read by the caller's previous use
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 13; ++q) red[w][q] = acc[q];
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int q = 0; q < 13; ++q) {
            double v = lane < kFinThreads / 32 ? red[lane][q] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            acc[q] = v;
        }
        __syncwarp();
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 13; ++q) red[0][q] = acc[q];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kFinThreads) k_pose_finalize(const double *__restrict__ partials, int T,
                                                               const vtgs_pose *__restrict__ view,
                                                               float *__restrict__ d_pose,
                                                               float *__restrict__ loss_out,
                                                               double *__restrict__ partials2,
                                                               unsigned int *__restrict__ ticket) {
    __shared__ double red[kFinThreads / 32][13];
    __shared__ bool last;
    const int tid = threadIdx.x;
    const int R = (T + kFinBlocks - 1) / kFinBlocks;
    const int r0 = blockIdx.x * R, r1 = min(T, r0 + R);
    double acc[13];
#pragma unroll
    for (int q = 0; q < 13; ++q) acc[q] = 0.0;
    for (int t = r0 + tid; t < r1; t += kFinThreads) {
        const double2 *r = reinterpret_cast<const double2 *>(partials + (size_t)t * 16);
        double x[14];
#pragma unroll
        for (int h = 0; h < 7; ++h) {
            const double2 d = __ldg(r + h);
            x[2 * h] = d.x;
            x[2 * h + 1] = d.y;
        }
#pragma unroll
        for (int q = 0; q < 13; ++q) acc[q] += x[q];
    }
    block_sum13(acc, red);
    if (tid < 13) partials2[blockIdx.x * 16 + tid] = red[0][tid];
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(ticket, 1u) == kFinBlocks - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
#pragma unroll
    for (int q = 0; q < 13; ++q) acc[q] = 0.0;
    if (tid < kFinBlocks)
#pragma unroll
        for (int q = 0; q < 13; ++q) acc[q] = __ldcg(partials2 + tid * 16 + q);
    block_sum13(acc, red);
    if (tid == 0) *ticket = 0u;
    if (tid == 0) {
        if (loss_out) *loss_out = (float)red[0][12];
        if (d_pose) {
            PoseR P;
            pose_rotation(*view, P);
            const double h[3] = {red[0][0], red[0][1], red[0][2]};
            double K[9];
            for (int i = 0; i < 9; ++i) K[i] = red[0][3 + i];
            double R[9];
            for (int i = 0; i < 9; ++i) R[i] = (double)P.R[i];
            double G[9];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    G[3 * a + b] = R[3 * a] * K[b] + R[3 * a + 1] * K[3 + b] + R[3 * a + 2] * K[6 + b];
            for (int a = 0; a < 3; ++a) d_pose[4 + a] = (float)-(R[3 * a] * h[0] + R[3 * a + 1] * h[1] + R[3 * a + 2] * h[2]);
            const double w = P.qhat[0], x = P.qhat[1], y = P.qhat[2], z = P.qhat[3];
            // ∂R/∂w, ∂R/∂x, ∂R/∂y, ∂R/∂z of the unit-quaternion matrix (row-major)
            const double Dw[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
            const double Dx[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
            const double Dy[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
            const double Dz[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
            double gq[4] = {0, 0, 0, 0};
            for (int i = 0; i < 9; ++i) {
                gq[0] += G[i] * Dw[i];
                gq[1] += G[i] * Dx[i];
                gq[2] += G[i] * Dy[i];
                gq[3] += G[i] * Dz[i];
            }
            const double dot = gq[0] * w + gq[1] * x + gq[2] * y + gq[3] * z;
            const double qh[4] = {w, x, y, z};
            for (int i = 0; i < 4; ++i) d_pose[i] = (float)((gq[i] - qh[i] * dot) / P.qnorm);
        }
    }
}

// Loss only (mapping): the fixed-order sum of the per-CTA loss partials (one contiguous double per
// backward CTA, so the loads coalesce), one CTA.
constexpr int kLossThreads = 1024;
__global__ void __launch_bounds__(kLossThreads) k_loss_finalize(const double *__restrict__ partials, int T,
                                                                float *__restrict__ loss_out) {
    __shared__ double red[kLossThreads / 32];
    const int tid = threadIdx.x;
    // all of a thread's loads in flight together, summed in row order
    constexpr int kU = 16;
    double x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const int t = tid + u * kLossThreads;
        x[u] = t < T ? __ldg(partials + t) : 0.0;
    }
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += x[u];
    for (int t = tid + kU * kLossThreads; t < T; t += kLossThreads) acc += __ldg(partials + t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid < 32) {
        double v = red[tid];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (tid == 0) *loss_out = (float)v;
    }
}

// Deterministic merge, second half: fixed point → fp32, added (+=) to the caller's buffers in
// Gaussian order; the accumulators are zeroed for the next call.
__global__ void __launch_bounds__(256) k_det_finalize(unsigned long long *__restrict__ det, int64_t g0, int64_t g1,
                                                      uint32_t want, float4 *__restrict__ d_col_opa,
                                                      float *__restrict__ d_radius) {
    for (int64_t g = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < g1; g += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long *q = det + (size_t)5 * g;   // 40-byte rows: 8-byte loads
        const ulonglong2 a = make_ulonglong2(q[0], q[1]);
        const ulonglong2 b = make_ulonglong2(q[2], q[3]);
        const unsigned long long c = q[4];
        if ((a.x | a.y | b.x | b.y | c) == 0ull) continue;
        const double k = 1.0 / kDetScale;
        if (want & (VTGS_GRAD_COLOR | VTGS_GRAD_OPACITY)) {
            float4 d = d_col_opa[g];
            d.x += (float)((double)(long long)a.x * k);
            d.y += (float)((double)(long long)a.y * k);
            d.z += (float)((double)(long long)b.x * k);
            d.w += (float)((double)(long long)b.y * k);
            d_col_opa[g] = d;
        }
        if (want & VTGS_GRAD_RADIUS) d_radius[g] += (float)((double)(long long)c * k);
        q[0] = q[1] = q[2] = q[3] = q[4] = 0ull;
    }
}

constexpr size_t kBwdDynSmem = sizeof(float2) * kBwdWarps * 32 * 32;

static int pose_direct() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("VTGS_BWD_POSE");
        v = e ? atoi(e) : 1;   // 1: pose-only ring kernel, 0: the general two-phase kernel
    }
    return v;
}

static int bwd_minb() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("VTGS_BWD_MINB");
        v = e ? atoi(e) : 11;  // 11 (default): the mapping backward held to 11 two-warp CTAs per SM (≤ 93
                               // registers) — shared memory allows 10–11 anyway; 12 (80 registers)
                               // makes ptxas rematerialise phase 1's f; 0: the compiler's choice (~107)
    }
    return v;
}

template <bool A, bool P, bool L>
static void launch_bwd_t(const BwdArgs &a, int T, cudaStream_t s) {
    if constexpr (A && !P) {
        if (bwd_minb() == 12) {
            k_composite_bwd<A, P, L, 12><<<T * (8 / kBwdWarps), kBwdWarps * 32, kBwdDynSmem, s>>>(a);
            return;
        }
        if (bwd_minb() == 11) {
            k_composite_bwd<A, P, L, 11><<<T * (8 / kBwdWarps), kBwdWarps * 32, kBwdDynSmem, s>>>(a);
            return;
        }
    }
    k_composite_bwd<A, P, L><<<T * (8 / kBwdWarps), kBwdWarps * 32, kBwdDynSmem, s>>>(a);
}

// Shared memory is the occupancy limit of the two-phase backward (19.7 KB per two-warp CTA: 11
// CTAs need the largest carve-out; the entry gathers hit L1 < 10 % of the time anyway).
static int bwd_carveout() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("VTGS_BWD_CARVEOUT");
        v = e ? atoi(e) : 100;   // percent of the unified L1 / shared storage given to shared memory
    }
    return v;
}

static int bwd_ring() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("VTGS_BWD_RING");
        v = e ? atoi(e) : 0;   // 1: the mapping backward (attributes only) as a ring walk
    }
    return v;
}
constexpr int kBwdRingR = 4;
constexpr size_t kBwdRingSmem = kBwdWarps * bwd_ring_warp_bytes<kBwdRingR>();

template <bool L>
static cudaError_t set_bwd_ring_attr() {
    cudaError_t e = cudaFuncSetAttribute(k_composite_bwd_ring<kBwdRingR, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kBwdRingSmem);
    if (!e) e = cudaFuncSetAttribute(k_composite_bwd_ring<kBwdRingR, L>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return e;
}

template <bool A, bool P, bool L>
static cudaError_t set_bwd_attr() {
    cudaError_t e = cudaFuncSetAttribute(k_composite_bwd<A, P, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kBwdDynSmem);
    if (!e && bwd_carveout() >= 0)
        e = cudaFuncSetAttribute(k_composite_bwd<A, P, L>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 bwd_carveout());
    if constexpr (A && !P) {
        if (!e) e = cudaFuncSetAttribute(k_composite_bwd<A, P, L, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kBwdDynSmem);
        if (!e && bwd_carveout() >= 0)
            e = cudaFuncSetAttribute(k_composite_bwd<A, P, L, 12>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     bwd_carveout());
        if (!e) e = cudaFuncSetAttribute(k_composite_bwd<A, P, L, 11>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kBwdDynSmem);
        if (!e && bwd_carveout() >= 0)
            e = cudaFuncSetAttribute(k_composite_bwd<A, P, L, 11>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     bwd_carveout());
    }
    return e;
}

cudaError_t backward_set_attributes() {
    cudaError_t e = set_bwd_attr<false, false, false>();
    if (!e) e = set_bwd_attr<false, false, true>();
    if (!e) e = set_bwd_attr<false, true, false>();
    if (!e) e = set_bwd_attr<false, true, true>();
    if (!e) e = set_bwd_attr<true, false, false>();
    if (!e) e = set_bwd_attr<true, false, true>();
    if (!e) e = set_bwd_attr<true, true, false>();
    if (!e) e = set_bwd_attr<true, true, true>();
    if (!e) e = set_bwd_ring_attr<false>();
    if (!e) e = set_bwd_ring_attr<true>();
    return e;
}

cudaError_t launch_backward(Ctx &c, const float *dC, const float *dD, const float *dS,
                            const vtgs_l1_loss *loss, uint32_t want, int64_t learn_begin,
                            int64_t learn_end, float4 *d_col_opa, float *d_radius, float4 *d_position,
                            float *d_pose, float *loss_out, cudaStream_t s) {
    const int W = c.intr.width, H = c.intr.height;
    const int ntx = (W + kTile - 1) / kTile, nty = (H + kTile - 1) / kTile, T = ntx * nty;
    cudaError_t err;
    BwdArgs a{};
    a.proj = c.proj; a.thr = c.thr; a.col_opa = c.col_opa; a.pos_rad = c.pos_rad;
    a.tile_count = c.tile_count; a.tile_start = c.tile_start; a.sub_lists = c.sub_lists; a.sub_count = c.sub_count;
    a.sub_masks = c.sub_masks;
    a.W = W; a.H = H; a.ntx = ntx;
    a.color = c.color; a.depth = c.depth; a.sil = c.sil; a.T_final = c.T_final; a.last = c.last;
    a.dC = dC; a.dD = dD; a.dS = dS;
    a.dev = c.dev; a.view = c.view_copy; a.in = c.intr;
    a.learn_begin = learn_begin; a.learn_end = learn_end; a.want = want;
    a.d_col_opa = d_col_opa; a.d_radius = d_radius; a.d_position = d_position; a.partials = c.partials;
    a.sub_cap = (uint64_t)8 * c.max_pairs; a.N = c.N;
    const bool L = loss != nullptr;
    if (L) {
        a.tC = loss->target_rgb; a.tD = loss->target_depth; a.vis = loss->vis_mask; a.extra_dc = loss->extra_dcolor;
        a.wc = loss->w_color; a.wd = loss->w_depth;
        a.cmode = loss->color_mask_mode; a.dmode = loss->depth_mask_mode; a.normalize = loss->normalize;
        if (a.normalize) {
            if ((err = cudaMemsetAsync(&c.dev->count_c, 0, 2 * sizeof(unsigned int), s))) return err;
            int g = (W * H + 255) / 256;
            if (g > c.num_sms * 2) g = c.num_sms * 2;
            LaunchScope ls(&c, kL1Count, s);
            k_l1_count<<<g, 256, 0, s>>>(c.sil, a.tD, a.vis, W * H, a.cmode, a.dmode, c.dev);
            if ((err = cudaGetLastError())) return err;
        }
    }
    const bool A = (want & (VTGS_GRAD_COLOR | VTGS_GRAD_OPACITY | VTGS_GRAD_RADIUS)) != 0;
    const bool DET = A && (want & VTGS_GRAD_DETERMINISTIC) != 0;
    if (DET) {   // the fixed-point accumulators (N×5 int64), allocated zeroed on first use
        if (c.det_cap < c.N) {
            if (c.det) cudaFree(c.det);
            c.det = nullptr;
            c.det_cap = 0;
            if ((err = cudaMalloc((void **)&c.det, sizeof(unsigned long long) * 5 * (size_t)(c.N > 0 ? c.N : 1))))
                return err;
            if ((err = cudaMemsetAsync(c.det, 0, sizeof(unsigned long long) * 5 * (size_t)(c.N > 0 ? c.N : 1), s)))
                return err;
            c.det_cap = c.N;
        }
        a.det = c.det;
    }
    const bool P = (want & VTGS_GRAD_POSE) != 0 && d_pose != nullptr;
    const bool X = (want & VTGS_GRAD_POSITION) != 0 && d_position != nullptr;   // same chain as the pose
    if (!X) a.want &= ~(uint32_t)VTGS_GRAD_POSITION;
    const int sel = (A ? 4 : 0) | ((P || X) ? 2 : 0) | (L ? 1 : 0);
    if (P && !A && !X && pose_direct()) {   // tracking: pose-only backward without the per-Gaussian reduction
        LaunchScope ls(&c, kCompBwd, s);
        constexpr int R = 4;
        const size_t sm = sizeof(PoseRing<R>) * kPoseRingWarps;
        static_assert(kPoseRingWarps == kBwdWarps, "k_pose_finalize rows: one partial per CTA of kBwdWarps warps");
        if (L) k_composite_bwd_pose_ring<R, true><<<T * (8 / kPoseRingWarps), kPoseRingWarps * 32, sm, s>>>(a);
        else k_composite_bwd_pose_ring<R, false><<<T * (8 / kPoseRingWarps), kPoseRingWarps * 32, sm, s>>>(a);
    } else if (A && !P && !X && bwd_ring()) {   // mapping: attribute gradients, ring walk
        LaunchScope ls(&c, kCompBwd, s);
        if (L) k_composite_bwd_ring<kBwdRingR, true><<<T * (8 / kBwdWarps), kBwdWarps * 32, kBwdRingSmem, s>>>(a);
        else k_composite_bwd_ring<kBwdRingR, false><<<T * (8 / kBwdWarps), kBwdWarps * 32, kBwdRingSmem, s>>>(a);
    } else {
    {
    LaunchScope ls(&c, kCompBwd, s);
    switch (sel) {
        case 0: launch_bwd_t<false, false, false>(a, T, s); break;
        case 1: launch_bwd_t<false, false, true>(a, T, s); break;
        case 2: launch_bwd_t<false, true, false>(a, T, s); break;
        case 3: launch_bwd_t<false, true, true>(a, T, s); break;
        case 4: launch_bwd_t<true, false, false>(a, T, s); break;
        case 5: launch_bwd_t<true, false, true>(a, T, s); break;
        case 6: launch_bwd_t<true, true, false>(a, T, s); break;
        default: launch_bwd_t<true, true, true>(a, T, s); break;
    }
    }
    }
    if ((err = cudaGetLastError())) return err;
    if (DET) {
        const int64_t g0 = learn_begin < 0 ? 0 : learn_begin, g1 = learn_end > c.N ? c.N : learn_end;
        if (g1 > g0) {
            LaunchScope ls(&c, kCompBwd, s);
            int grid = (int)((g1 - g0 + 255) / 256);
            if (grid > c.num_sms * 16) grid = c.num_sms * 16;
            k_det_finalize<<<grid, 256, 0, s>>>(c.det, g0, g1, want, d_col_opa, d_radius);
            if ((err = cudaGetLastError())) return err;
        }
    }
    if (P || (L && loss_out)) {
        LaunchScope ls(&c, kFinalize, s);
        const int rows = T * (8 / kBwdWarps);
        if (!P) k_loss_finalize<<<1, kLossThreads, 0, s>>>(c.partials, rows, loss_out);
        else k_pose_finalize<<<kFinBlocks, kFinThreads, 0, s>>>(c.partials, rows, c.view_copy, P ? d_pose : nullptr,
                                                           L ? loss_out : nullptr, c.partials + (size_t)c.max_tiles * 8 * 16,
                                                           &c.dev->fin_ticket);
        if ((err = cudaGetLastError())) return err;
    }
    return cudaSuccess;
}


// Head-frame bundle adjustment: per keyframe k, the 12 sums Σ dL/dX_w and
// Σ dL/dX_w X_kᵀ over its slots (X_k = R_kᵀ(X_w − t_k), fp64), then the rotation chain.  One
// CTA per keyframe, fixed-order block reduction (deterministic).
__global__ void __launch_bounds__(256) k_keyframe_pose_grad(const float4 *__restrict__ pos_rad,
                                                            const float4 *__restrict__ d_position,
                                                            const vtgs_pose *__restrict__ kf_poses,
                                                            int64_t spk, float *__restrict__ d_kf) {
    __shared__ double red[256][12];
    __shared__ PoseR P;
    const int k = blockIdx.x, tid = threadIdx.x;
    if (tid == 0) pose_rotation(kf_poses[k], P);
    __syncthreads();
    const double w = P.qhat[0], x = P.qhat[1], y = P.qhat[2], z = P.qhat[3];
    // fp64 rotation from the normalised quaternion (X_k recovered without fp32 rounding of R)
    const double Rd[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                          2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                          2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    const double t0 = kf_poses[k].t[0], t1 = kf_poses[k].t[1], t2 = kf_poses[k].t[2];
    double acc[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i] = 0.0;
    const int64_t b = (int64_t)k * spk;
    for (int64_t i = tid; i < spk; i += 256) {
        const float4 pr = __ldg(pos_rad + b + i);
        if (!(pr.w > 0.f)) continue;
        const float4 g = __ldg(d_position + b + i);
        const double d0 = (double)pr.x - t0, d1 = (double)pr.y - t1, d2 = (double)pr.z - t2;
        const double X[3] = {Rd[0] * d0 + Rd[3] * d1 + Rd[6] * d2, Rd[1] * d0 + Rd[4] * d1 + Rd[7] * d2,
                             Rd[2] * d0 + Rd[5] * d1 + Rd[8] * d2};
        const double G[3] = {g.x, g.y, g.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            acc[a] += G[a];
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[3 + 3 * a + c] += G[a] * X[c];
        }
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) red[tid][i] = acc[i];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (tid < s)
#pragma unroll
            for (int i = 0; i < 12; ++i) red[tid][i] += red[tid + s][i];
        __syncthreads();
    }
    if (tid == 0) {
        const double *M = &red[0][3];   // dL/dR_k (row-major), dL/dt_k = red[0][0..2]
        const double Dw[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
        const double Dx[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
        const double Dy[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
        const double Dz[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
        double gq[4] = {0, 0, 0, 0};
        for (int i = 0; i < 9; ++i) {
            gq[0] += M[i] * Dw[i];
            gq[1] += M[i] * Dx[i];
            gq[2] += M[i] * Dy[i];
            gq[3] += M[i] * Dz[i];
        }
        const double dot = gq[0] * w + gq[1] * x + gq[2] * y + gq[3] * z;
        const double qh[4] = {w, x, y, z};
        for (int i = 0; i < 4; ++i) d_kf[7 * k + i] = (float)((gq[i] - qh[i] * dot) / P.qnorm);
        for (int a = 0; a < 3; ++a) d_kf[7 * k + 4 + a] = (float)red[0][a];
    }
}

cudaError_t launch_keyframe_pose_grad(Ctx &c, const float4 *pos_rad, const float4 *d_position,
                                      const vtgs_pose *kf_poses, int K, int64_t spk, float *d_kf, cudaStream_t s) {
    LaunchScope ls(&c, kKfPose, s);
    k_keyframe_pose_grad<<<K, 256, 0, s>>>(pos_rad, d_position, kf_poses, spk, d_kf);
    return cudaGetLastError();
}

// One Adam step on the device pose, then q ← q / |q|.
__global__ void k_pose_adam(vtgs_pose *pose, const float *__restrict__ g, float *state, float lr_rot,
                            float lr_trans) {
    if (threadIdx.x != 0) return;
    const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
    const float step = state[14] + 1.0f;
    state[14] = step;
    const float c1 = 1.0f - powf(b1, step), c2 = 1.0f - powf(b2, step);
    float prm[7] = {pose->q[0], pose->q[1], pose->q[2], pose->q[3], pose->t[0], pose->t[1], pose->t[2]};
    for (int i = 0; i < 7; ++i) {
        const float m = b1 * state[i] + (1.0f - b1) * g[i];
        const float v = b2 * state[7 + i] + (1.0f - b2) * g[i] * g[i];
        state[i] = m;
        state[7 + i] = v;
        const float lr = i < 4 ? lr_rot : lr_trans;
        prm[i] -= lr * (m / c1) / (sqrtf(v / c2) + eps);
    }
    const float n = sqrtf(prm[0] * prm[0] + prm[1] * prm[1] + prm[2] * prm[2] + prm[3] * prm[3]);
    for (int i = 0; i < 4; ++i) pose->q[i] = prm[i] / n;
    for (int i = 0; i < 3; ++i) pose->t[i] = prm[4 + i];
}

cudaError_t launch_pose_adam(Ctx &c, vtgs_pose *pose, const float *d_pose, float *state, float lr_rot,
                             float lr_trans, cudaStream_t s) {
    LaunchScope ls(&c, kPoseAdam, s);
    k_pose_adam<<<1, 32, 0, s>>>(pose, d_pose, state, lr_rot, lr_trans);
    return cudaGetLastError();
}

}  // namespace vtgs
