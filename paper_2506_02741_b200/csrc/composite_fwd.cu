// (4) Per-tile front-to-back compositing of colour, depth and silhouette — PAPER.md:146
// (Eq. 1 `splat`), α floor 1/255 from north_star (4).
// Decision arithmetic exactly as DESIGN.md §3 step 7.  Work decomposition: composite_common.cuh
// (one warp per 4×8 sub-tile, lane = pixel, per-lane candidate lists by bit transpose).
#include <stdlib.h>

#include "composite_common.cuh"

namespace vtgs {

struct FwdArgs {
    const float4 *proj;
    const float *thr;      // per Gaussian packed (D_c, D_clamp), k_project_count
    const float4 *col_opa;
    const uint32_t *tile_count;
    const uint32_t *tile_start;
    const uint32_t *sub_lists;
    const uint32_t *sub_count;
    uint32_t *sub_masks;   // per sub-list entry: its candidate pixels (lane_mask within D_c), read by the backward
    int W, H, ntx;
    float *color, *depth, *sil, *T_final;
    uint32_t *last;
    DevScalars *dev;
    uint64_t sub_cap;   // entries of sub_lists / sub_masks (checked build)
    int64_t N;          // Gaussians (checked build)
};

constexpr int kFwdWarps = 2;  // warps (sub-tiles) per CTA: small CTAs retire independently

// Ring walk.  The warp builds 32-entry batches of its sub-list into a ring of R slots (entry
// data A = (u, v, 9σ², o), B = (c_r, c_g, c_b, z), and per lane the bit column of the entries
// whose footprint can touch its pixel).  Each lane then walks ITS candidates front to back at
// its own pace: a lane only waits when it reaches the batch not yet built and the ring is full
// (R batches ahead of the slowest live lane).  Compared with walking batch by batch in lock
// step (the warp runs max-over-lanes candidates per batch), the warp runs ≈ max-over-lanes of
// the whole-list candidate count — tools/sim_batches.py: lane efficiency 0.27 → 0.87 at R = 16.
#ifndef VTGS_FWD_INNER
#define VTGS_FWD_INNER 6
#endif
constexpr int kInner = VTGS_FWD_INNER;         // lane-independent steps between warp checks

template <int R, bool STATS>
struct FwdRing {
    float4 A[R * 32];        // u, v, D_c, escale = −½log2(e)/σ²
    float4 B[R * 32];        // c_r, c_g, c_b, o
    float Z[R * 32];         // z
    uint32_t bits[R * 32];   // per lane: its candidate entries of the batch (bit 31 − j = entry j)
    float S9[STATS ? R * 32 : 1];   // 9σ² (the work counter's 3σ test)
};

// AHEAD: how far past the furthest batch a lane needs the warp builds when it has to build (the
// ring's R bounds it too); batches built past the point where every pixel terminates are wasted
template <int R, bool STATS, int MINB, int AHEAD = R>
__global__ void __launch_bounds__(kFwdWarps * 32, MINB) k_composite_fwd_ring(FwdArgs p) {
    extern __shared__ float4 fwd_smem[];
    static_assert((R & (R - 1)) == 0, "ring depth must be a power of two");
    const int wl = threadIdx.x >> 5;
    FwdRing<R, STATS> &ring = reinterpret_cast<FwdRing<R, STATS> *>(fwd_smem)[wl];
    const int gsub = blockIdx.x * kFwdWarps + wl;
    const int tile = gsub >> 3;
    const int ty = tile / p.ntx, tx = tile - ty * p.ntx;
    const int w = gsub & 7;
    const unsigned lane = lane_id();
    const int sx = sub_x0(tx, w), sy = sub_y0(ty, w);
    const int px = sx + pix_dx((int)lane), py = sy + pix_dy((int)lane);
    const bool inside = px < p.W && py < p.H;
    const float pxf = (float)px, pyf = (float)py;
    const int n = (int)p.tile_count[tile];
    const uint32_t *list = p.sub_lists + (size_t)8 * p.tile_start[tile] + (size_t)w * n;
    uint32_t *mout = p.sub_masks + (size_t)8 * p.tile_start[tile] + (size_t)w * n;
    const int cnt = (int)p.sub_count[tile * 8 + w];
    const int nb = (cnt + 31) >> 5;
    VTGS_CHECK(cnt <= n && (uint64_t)8 * p.tile_start[tile] + (uint64_t)(w + 1) * n <= p.sub_cap);
    const unsigned inmask = __ballot_sync(kFullMask, inside);

    EntryStream st;
    stream_start(st, list, (int)lane, 32 + (int)lane, cnt, p.proj, p.col_opa, p.thr);
    const EntryRegs &nxt = st.e;
    int built = 0;
    // build batch `built` from the prefetched registers, prefetch the one after it
    auto build = [&]() {
        const int slot = (built & (R - 1)) * 32;
        const int idx = built * 32 + (int)lane;
        unsigned mj = 0u;
        if (idx < cnt) {
            VTGS_CHECK((int64_t)nxt.g < p.N && nxt.pr.z > 0.0f);
            const float s = fabsf(nxt.pr.w);
            const float s2 = __fmul_rn(s, s);
            const float s9 = __fmul_rn(9.0f, s2);
            const float dc = thr_unpack(nxt.th, s2).x;
            ring.A[slot + lane] = make_float4(nxt.pr.x, nxt.pr.y, dc, exp_scale(s2));
            ring.B[slot + lane] = nxt.co;
            ring.Z[slot + lane] = nxt.pr.z;
            if (STATS) ring.S9[slot + lane] = s9;
            // candidates: the pixels within D_c (the work counters also want the whole 3σ disc)
            const unsigned m0 = lane_mask(make_float4(nxt.pr.x, nxt.pr.y, STATS ? s9 : dc, 0.f),
                                          rect_from_proj(nxt.pr, p.W, p.H), sx, sy);
            mout[idx] = m0;   // the backward walks the same candidates and re-takes the same exact decisions
            mj = m0 & inmask;
        }
        ring.bits[slot + lane] = __brev(transpose32(mj, lane));  // bit 31 − j = entry j
        ++built;
        stream_next(st, list, (built + 1) * 32 + (int)lane, cnt, p.proj, p.col_opa, p.thr);
    };
    while (built < nb && built < R && built <= AHEAD) build();
    __syncwarp();

    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, D = 0.f, Sl = 0.f;
    uint32_t lastc = 0, ne = 0, nc = 0;
    // lane state: batch b, its remaining candidate bits cur (bit 31 − j = entry j, so the lowest
    // remaining entry is the highest set bit, one FLO), the address of the batch's entry 31,
    // and 1 + the sub-list position of its entry 31.
    // Finished (terminated, walked the whole list, or outside the image) ⇔ cur == 0 && b + 1 ≥ nb
    // (terminated and outside lanes park at b = kDoneB).
    constexpr int kDoneB = 0x3fffffff;   // b of a finished lane: b + 1 ≥ nb and ≥ built
    int b = inside ? -1 : kDoneB;
    unsigned cur = 0u;
    int soff = 0;
    int lbase = 0;
    auto advance = [&]() {
        ++b;
        soff = (b & (R - 1)) * 32;
        cur = ring.bits[soff + lane];
        lbase = b * 32 + 32;
    };
    for (;;) {
        // a few lane-independent steps between warp-level checks (a blocked lane idles ≤ kInner);
        // branch-free body: every lane runs the same predicated instructions
#pragma unroll
        for (int it = 0; it < kInner; ++it) {
            if (cur == 0u && b + 1 < built) advance();
            const bool has = cur != 0u;
            const int hb = 31 - __clz(cur);                // highest set bit = lowest remaining entry
            cur &= ~(1u << (hb & 31));
            const int k = soff + 31 - hb;                  // ring index of entry 31 − hb
            float4 A, Bc;                                  // unused unless `has` (comp includes it)
            float zk;
            if (has) {   // predicated loads: idle lanes add no shared-memory traffic
                A = ring.A[k];
                Bc = ring.B[k];
                zk = ring.Z[k];
            }
            const float d2 = pair_d2(pxf, pyf, A.x, A.y);
            const bool comp = has && d2 <= A.z;            // 3σ truncation and α floor, exact
            float w;
            const float a = pair_alpha_value(d2, A.w, Bc.w, w);   // value only (clamp decision: backward)
            const float Tn = __fmul_rn(T, __fsub_rn(1.0f, a));
            const bool term = comp && Tn < kTMin;
            const bool acc = comp && !term;
            const float om = a * T;
            if (acc) {   // predicated: Bc is garbage for lanes without a candidate
                C0 = fmaf(Bc.x, om, C0);
                C1 = fmaf(Bc.y, om, C1);
                C2 = fmaf(Bc.z, om, C2);
                D = fmaf(zk, om, D);
                Sl += om;
                T = Tn;
                lastc = (uint32_t)(lbase - hb);
            }
            if (STATS) {
                float s9 = 0.f;
                if (has) s9 = ring.S9[k];
                ne += (has && d2 <= s9) ? 1u : 0u;
                nc += acc ? 1u : 0u;
            }
            if (term) {   // finished: past every batch (a constant, so nb need not stay live)
                cur = 0u;
                b = kDoneB;
            }
        }
        // lanes whose next word was empty: catch up before the warp-level check
        while (cur == 0u && b + 1 < built) advance();
        const bool live = cur != 0u || b + 1 < nb;
        if (!__any_sync(kFullMask, live)) break;
        const bool blocked = cur == 0u && b + 1 < nb && b + 1 >= built;
        if (__any_sync(kFullMask, blocked)) {
            const int need = !live ? 0x7fffffff : (cur ? b : b + 1);  // earliest batch still needed
            const int lo = __reduce_min_sync(kFullMask, need);
            int target = lo + R < nb ? lo + R : nb;
            if (AHEAD < R) {
                const int hi = (int)__reduce_max_sync(kFullMask, live ? (unsigned)need : 0u);
                target = min(target, hi + 1 + AHEAD);
            }
            if (built < target) {
                while (built < target) build();
                __syncwarp();
            }
        }
    }
    if (inside) {
        const int pix = py * p.W + px;
        VTGS_CHECK(lastc <= (uint32_t)cnt && T >= kTMin);
        p.color[3 * pix + 0] = C0;
        p.color[3 * pix + 1] = C1;
        p.color[3 * pix + 2] = C2;
        p.depth[pix] = D;
        p.sil[pix] = Sl;
        p.T_final[pix] = T;
        p.last[pix] = lastc;
    }
    if (STATS) {
        unsigned long long a = ne, bsum = nc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(kFullMask, a, o);
            bsum += __shfl_xor_sync(kFullMask, bsum, o);
        }
        if (lane == 0 && (a | bsum)) {
            atomicAdd(&p.dev->e_eval, a);
            atomicAdd(&p.dev->e_comp, bsum);
        }
    }
}

static int fwd_variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("VTGS_FWD");
        v = e ? atoi(e) : 0;   // 0 (default): R = 4, 14 two-warp CTAs per SM (≤ 72 registers), lazy
                               // build; 14: the same with an eager ring fill; 4: R = 4 at the
                               // compiler's register count; 8: R = 8; 812: R = 8, 12 CTAs/SM
    }
    return v;
}

template <int R, bool STATS, int MINB, int AHEAD>
static cudaError_t launch_ring_s(const FwdArgs &a, int T, cudaStream_t s) {
    const size_t sm = sizeof(FwdRing<R, STATS>) * kFwdWarps;
    cudaError_t e = cudaFuncSetAttribute(k_composite_fwd_ring<R, STATS, MINB, AHEAD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e) return e;
    k_composite_fwd_ring<R, STATS, MINB, AHEAD><<<T * 8 / kFwdWarps, kFwdWarps * 32, sm, s>>>(a);
    return cudaGetLastError();
}

template <int R, int MINB, int AHEAD = R>
static cudaError_t launch_ring(const FwdArgs &a, int T, bool stats, cudaStream_t s) {
    return stats ? launch_ring_s<R, true, MINB, AHEAD>(a, T, s) : launch_ring_s<R, false, MINB, AHEAD>(a, T, s);
}

cudaError_t launch_composite_fwd(Ctx &c, cudaStream_t s) {
    const int W = c.intr.width, H = c.intr.height;
    const int ntx = (W + kTile - 1) / kTile, nty = (H + kTile - 1) / kTile;
    FwdArgs a{c.proj, c.thr, c.col_opa, c.tile_count, c.tile_start, c.sub_lists, c.sub_count, c.sub_masks, W, H, ntx,
              c.color, c.depth, c.sil, c.T_final, c.last, c.dev, (uint64_t)8 * c.max_pairs, c.N};
    switch (fwd_variant()) {
        case 8: return launch_ring<8, 1>(a, ntx * nty, c.count_work, s);
        case 812: return launch_ring<8, 12>(a, ntx * nty, c.count_work, s);
        case 14: return launch_ring<4, 14>(a, ntx * nty, c.count_work, s);   // eager ring fill
        case 4: return launch_ring<4, 1>(a, ntx * nty, c.count_work, s);
        default: return launch_ring<4, 14, 0>(a, ntx * nty, c.count_work, s);   // lazy build
    }
}

}  // namespace vtgs
