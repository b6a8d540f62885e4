// (4) Per-tile front-to-back compositing of colour, depth and silhouette — PAPER.md:146
// (Eq. 1 `splat`), α floor 1/255 from north_star (4).
// Decision arithmetic exactly as DESIGN.md §3 step 7.  Work decomposition: composite_common.cuh
// (one warp per 8×4 sub-tile, lane = pixel, per-lane candidate lists by bit transpose).
#include "composite_common.cuh"

namespace vtgs {

struct FwdArgs {
    const float4 *proj;
    const uint2 *rect;
    const float4 *col_opa;
    const uint32_t *tile_count;
    const uint32_t *tile_start;
    const uint32_t *sub_lists;
    const uint32_t *sub_count;
    int W, H, ntx;
    float *color, *depth, *sil, *T_final;
    uint32_t *last;
    DevScalars *dev;
};

constexpr int kFwdWarps = 2;  // warps (8×4 sub-tiles) per CTA: small CTAs retire independently

__global__ void __launch_bounds__(kFwdWarps * 32, 16) k_composite_fwd(FwdArgs p) {
    __shared__ float4 sA[kFwdWarps][32];  // u, v, 9σ², −log2(e)/(2σ²) of the warp's current batch
    __shared__ float4 sB[kFwdWarps][32];  // colour, opacity
    __shared__ float sZ[kFwdWarps][32];

    const int wl = threadIdx.x >> 5;
    const int gsub = blockIdx.x * kFwdWarps + wl;
    const int tile = gsub >> 3;
    const int ty = tile / p.ntx, tx = tile - ty * p.ntx;
    const int w = gsub & 7;
    const unsigned lane = lane_id();
    const int sx = tx * kTile + (w & 1) * 8, sy = ty * kTile + (w >> 1) * 4;
    const int px = sx + (lane & 7), py = sy + (lane >> 3);
    const bool inside = px < p.W && py < p.H;
    const float pxf = (float)px, pyf = (float)py;
    const int n = (int)p.tile_count[tile];
    const uint32_t *list = p.sub_lists + (size_t)8 * p.tile_start[tile] + (size_t)w * n;
    const int cnt = (int)p.sub_count[tile * 8 + w];

    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, D = 0.f, Sl = 0.f;
    uint32_t lastc = 0, ne = 0, nc = 0;
    bool done = !inside;
    unsigned active = __ballot_sync(kFullMask, !done);

    EntryRegs nxt;
    fetch_entry(nxt, list, (int)lane, cnt, p.proj, p.col_opa, p.rect);
    for (int bb = 0; bb < cnt && active; bb += 32) {
        const EntryRegs cur = nxt;
        fetch_entry(nxt, list, bb + 32 + (int)lane, cnt, p.proj, p.col_opa, p.rect);  // next batch
        unsigned mj = 0u;
        if (bb + (int)lane < cnt) {
            const float4 A = entry_geom(cur.pr);
            sA[wl][lane] = A;
            sB[wl][lane] = cur.co;
            sZ[wl][lane] = cur.pr.z;
            mj = lane_mask(A, cur.r, sx, sy) & active;
        }
        __syncwarp();
        unsigned bits = transpose32(mj, lane);
        while (bits) {
            const int k = __ffs(bits) - 1;
            bits &= bits - 1u;
            const float4 A = sA[wl][k];
            const float dx = __fsub_rn(pxf, A.x), dy = __fsub_rn(pyf, A.y);
            const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
            if (d2 <= A.z) {
                ++ne;
                const float4 B = sB[wl][k];
                const float a = fminf(__fmul_rn(B.w, fast_exp2(d2 * A.w)), kAlphaMax);
                if (a >= 1.0f / 255.0f) {
                    const float Tn = __fmul_rn(T, __fsub_rn(1.0f, a));
                    if (Tn < kTMin) {
                        done = true;
                        bits = 0u;
                    } else {
                        const float om = a * T;
                        C0 = fmaf(B.x, om, C0);
                        C1 = fmaf(B.y, om, C1);
                        C2 = fmaf(B.z, om, C2);
                        D = fmaf(sZ[wl][k], om, D);
                        Sl += om;
                        T = Tn;
                        lastc = (uint32_t)(bb + k + 1);
                        ++nc;
                    }
                }
            }
        }
        active = __ballot_sync(kFullMask, !done);
        __syncwarp();
    }
    if (inside) {
        const int pix = py * p.W + px;
        p.color[3 * pix + 0] = C0;
        p.color[3 * pix + 1] = C1;
        p.color[3 * pix + 2] = C2;
        p.depth[pix] = D;
        p.sil[pix] = Sl;
        p.T_final[pix] = T;
        p.last[pix] = lastc;
    }
    unsigned long long a = ne, b = nc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(kFullMask, a, o);
        b += __shfl_xor_sync(kFullMask, b, o);
    }
    if (lane == 0 && (a | b)) {
        atomicAdd(&p.dev->e_eval, a);
        atomicAdd(&p.dev->e_comp, b);
    }
}

cudaError_t launch_composite_fwd(Ctx &c, cudaStream_t s) {
    const int W = c.intr.width, H = c.intr.height;
    const int ntx = (W + kTile - 1) / kTile, nty = (H + kTile - 1) / kTile;
    FwdArgs a{c.proj, c.rect, c.col_opa, c.tile_count, c.tile_start, c.sub_lists, c.sub_count, W, H, ntx,
              c.color, c.depth, c.sil, c.T_final, c.last, c.dev};
    k_composite_fwd<<<ntx * nty * 8 / kFwdWarps, kFwdWarps * 32, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace vtgs
