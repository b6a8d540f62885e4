// composite_common.cuh — machinery shared by the forward and backward compositing kernels.
//
// Work decomposition (DESIGN.md §4 K6/K7).  Every 16×16 tile is split into eight 4×8 sub-tiles
// and the tile sort also emits, per sub-tile, the (depth-ordered) sub-list of the tile entries
// whose footprint rect touches that sub-tile.  One WARP owns one sub-tile (lane = pixel) and
// walks its sub-list independently of every other warp — no block barriers, so a warp whose
// pixels are all saturated stops at once.  The sub-list is consumed 32 entries at a time:
//   1. lane j gathers entry j (prefetched one batch ahead through registers) and builds the
//      32-bit mask of the warp's pixels inside the entry's rect and, conservatively, inside its
//      3σ disc;
//   2. the 32×32 bit matrix is transposed across the warp (5 shuffle stages), so lane i holds
//      the bits of exactly the entries that can touch ITS pixel;
//   3. each lane walks only its own candidates (the forward front to back; the backward back
//      to front, then a second phase where lane j sums entry j's gradient over its pixels).
#pragma once

#include "vtgs_internal.cuh"

namespace vtgs {

constexpr unsigned kFullMask = 0xffffffffu;

// Sub-tile geometry: each 16×16 tile is split into 8 sub-tiles of kSubW × kSubH pixels, one warp
// each, lane = pixel (y − sy)·kSubW + (x − sx).  Default 4 × 8 (4 columns × 2 rows of sub-tiles,
// s = column + 4·row): depth-sorted batches spread over a tall sub-tile's pixels a little more
// evenly than over a wide one (the lane models of tests/models/sim_bwd_ring.py: lock-step
// phase-1 steps −10 %, ring steps −6 %).  -DVTGS_SUB_8x4 builds the round-1 shape (8 × 4).
#ifdef VTGS_SUB_8x4
constexpr int kSubW = 8, kSubH = 4;
#else
constexpr int kSubW = 4, kSubH = 8;
#endif
constexpr int kSubCols = kTile / kSubW;
static_assert(kSubW * kSubH == 32 && kTile % kSubW == 0 && kTile % kSubH == 0, "a warp per sub-tile");
__device__ __forceinline__ int sub_x0(int tx, int s) { return tx * kTile + (s % kSubCols) * kSubW; }
__device__ __forceinline__ int sub_y0(int ty, int s) { return ty * kTile + (s / kSubCols) * kSubH; }
__device__ __forceinline__ int pix_dx(int i) { return i % kSubW; }   // pixel / lane index → offsets
__device__ __forceinline__ int pix_dy(int i) { return i / kSubW; }

// One sub-list entry held in registers (gathered one batch ahead).
struct EntryRegs {
    uint32_t g;
    float4 pr;
    float4 co;
    float th;    // the packed (D_c, D_clamp) of k_project_count (thr_pack / thr_unpack)
};

__device__ __forceinline__ void fetch_entry(EntryRegs &er, const uint32_t *__restrict__ list, int idx, int n,
                                            const float4 *__restrict__ proj, const float4 *__restrict__ col,
                                            const float *__restrict__ thr) {
    if (idx >= 0 && idx < n) {
        er.g = __ldg(list + idx);
        er.pr = __ldg(proj + er.g);
        er.co = __ldg(col + er.g);
        er.th = __ldg(thr + er.g);
    }
}

// Two-level prefetch along a sub-list: the gid of the batch after next is loaded one batch
// earlier than its attributes (a gather through that gid), so a build never waits on the
// dependent list → gid → attribute chain, only on loads issued a whole batch before.
struct EntryStream {
    EntryRegs e;   // entry (this lane's) of the next batch to build
    uint32_t gn;   // gid of the batch after it
    bool gv;
};

__device__ __forceinline__ void stream_start(EntryStream &s, const uint32_t *__restrict__ list, int idx0, int idx1,
                                             int n, const float4 *__restrict__ proj, const float4 *__restrict__ col,
                                             const float *__restrict__ thr) {
    fetch_entry(s.e, list, idx0, n, proj, col, thr);
    s.gv = idx1 >= 0 && idx1 < n;
    if (s.gv) s.gn = __ldg(list + idx1);
}

// e ← the attributes of gid gn; gn ← the gid at idx2
__device__ __forceinline__ void stream_next(EntryStream &s, const uint32_t *__restrict__ list, int idx2, int n,
                                            const float4 *__restrict__ proj, const float4 *__restrict__ col,
                                            const float *__restrict__ thr) {
    if (s.gv) {
        s.e.g = s.gn;
        s.e.pr = __ldg(proj + s.gn);
        s.e.co = __ldg(col + s.gn);
        s.e.th = __ldg(thr + s.gn);
    }
    s.gv = idx2 >= 0 && idx2 < n;
    if (s.gv) s.gn = __ldg(list + idx2);
}

// The forward stores each sub-list entry's pixel mask (lane_mask, below) next to the sub-list;
// the backward reads it instead of recomputing it (same entry, same sub-tile, same mask).
__device__ __forceinline__ uint32_t load_mask(const uint32_t *__restrict__ mlist, int idx, int n) {
    return (idx >= 0 && idx < n) ? __ldg(mlist + idx) : 0u;
}

// ---- α of a (pixel, Gaussian) pair: ONE definition for every compositing kernel -----------
// DESIGN.md §3 step 7: w = exp((−0.5·d²)/σ²), α = min(o·w, 0.999), skipped iff α < 1/255.  The
// decisions are taken on the oracle's bits — w the correctly rounded fp32 exp of the fp32
// argument fl(fl(−0.5·d²)/s2), s2 = fl(σ·σ) — and every one of them is MONOTONE in d² (each
// rounding step is monotone): "α ≥ 1/255" ⇔ d² ≤ D_floor and "o·w > 0.999" (clamped) ⇔
// d² ≤ D_clamp, for per-Gaussian fp32 thresholds that k_project_count finds once per view with
// the exact arithmetic (alpha_thresholds).  The compositing kernels then decide with compares
// only; the VALUE of an unclamped α uses the fast w = ex2.approx(d²·escale),
// escale = −½log2(e)·rcp(s2) (relative error ≤ ~1e-6, a value difference, never a decision).
// The forward and the backward read the same thresholds, so they composite the same pairs.
constexpr float kAlphaMin = 1.0f / 255.0f;
constexpr float kNegHalfLog2e = -0.5f * kLog2e;

// −½log2(e)/s2 for the α VALUE (never a decision): one approximate reciprocal, the same
// instructions in every kernel, so the forward and the backward use the same bits
__device__ __forceinline__ float exp_scale(float s2) { return kNegHalfLog2e * rcp_approx(s2); }

__device__ __forceinline__ float f32_next(float x) { return __uint_as_float(__float_as_uint(x) + 1u); }   // x ≥ 0
__device__ __forceinline__ float f32_prev(float x) { return __uint_as_float(__float_as_uint(x) - 1u); }   // x > 0

// Largest fp32 d² in [0, cap] whose exact raw α passes (raw ≥ thr, or raw > thr when strict), −1
// if d² = 0 already fails.  Each step of raw(d²) = fl(o · RN₃₂(exp(x))), x = fl(fl(−0.5 d²)/s2),
// is monotone, so the boundary is found stage by stage without evaluating exp:
//   1. w_min = the smallest fp32 w with fl(o·w) passing (fp32 arithmetic, a step or two);
//   2. RN₃₂(e^x) ≥ w_min ⇔ e^x > m, m = the midpoint between w_min and its predecessor (e^x is
//      never exactly m for fp32 x ≠ 0), ⇔ x > L = ln m: x_min = the smallest fp32 above L
//      (one fp64 log; its 1e-16 error matters only if L lies within 1e-16 of an fp32 number);
//   3. the largest d² with fl(fl(−0.5 d²)/s2) ≥ x_min, walking from −2·s2·x_min with the
//      oracle's own fp32 operations.
static __device__ __noinline__ float alpha_threshold_d2(float s2, float o, float thr, bool strict, float cap) {
    auto ok_w = [&](float w) {
        const float r = __fmul_rn(o, w);
        return strict ? r > thr : r >= thr;
    };
    if (!ok_w(1.0f)) return -1.0f;                 // d² = 0: w = exp(0) = 1 exactly
    float w = __fdiv_rn(thr, o);
    if (!(w > 0.0f)) return cap;
    if (ok_w(w)) {
        for (int i = 0; i < 4 && w > 0.0f && ok_w(f32_prev(w)); ++i) w = f32_prev(w);
    } else {
        for (int i = 0; i < 4 && !ok_w(w); ++i) w = f32_next(w);
    }
    if (w > 1.0f) return -1.0f;
    auto xd = [&](float d) { return __fdiv_rn(__fmul_rn(-0.5f, d), s2); };
    const double m = 0.5 * ((double)f32_prev(w) + (double)w);
    const double L = log(m);                       // x must exceed L (L < 0 since m < 1)
    float xm = (float)L;                           // round to nearest, then the smallest fp32 > L
    if ((double)xm <= L) xm = __uint_as_float(__float_as_uint(xm) - 1u);   // negative: −1 ulp moves up
    if (xd(cap) >= xm) return cap;
    float d = (float)fmin(fmax(-2.0 * (double)s2 * (double)xm, 0.0), (double)cap);
    if (xd(d) >= xm) {
        for (int i = 0; i < 64 && d < cap && xd(f32_next(d)) >= xm; ++i) d = f32_next(d);
    } else {
        for (int i = 0; i < 64 && d > 0.0f && xd(d) < xm; ++i) d = f32_prev(d);
    }
    return d;
}

// The common case without the search: o ≤ 0.999 (never clamped) and either o < 1/255 (nothing
// passes: at d² = 0 the raw α is o itself) or o ≥ kOpaFast: at the disc's rim d² = fl(9·s2) the
// argument fl(fl(−0.5 d²)/s2) is −4.5 within 2 ulp, so w ≥ e^−4.5·(1 − 7e-7) there and
// fl(o·w) ≥ 1/255 whenever o ≥ (1/255)·e^4.5·(1 + 1e-5) = 0.353012… — the whole disc passes.
// Returns false when the exact search (alpha_thresholds) is needed (o in [1/255, 0.3530), or
// o > 0.999).
constexpr float kOpaFast = 0.35302f;   // ≥ (1/255)·e^4.5·(1 + 1e-5) = 0.3530119…
__device__ __forceinline__ bool alpha_thresholds_fast(float s2, float o, float2 &th) {
    if (o > kAlphaMax || (o >= kAlphaMin && o < kOpaFast)) return false;
    th = make_float2(o >= kAlphaMin ? __fmul_rn(9.0f, s2) : -1.0f, -1.0f);
    return true;
}

// One float per Gaussian carries both thresholds: D_c ≥ 0 (not clampable, D_clamp = −1); −1 (no
// pixel passes); ≤ −2 for a clampable Gaussian (o > 0.999), which always passes its whole disc
// (o·w at the rim ≥ 0.999·e^−4.5 > 1/255, so D_c = fl(9·s2)) — the value is −D_clamp − 2.
__device__ __forceinline__ float thr_pack(float2 t, float s2) {
    return t.y >= 0.0f ? -t.y - 2.0f : t.x;
}
__device__ __forceinline__ float2 thr_unpack(float th, float s2) {
    return th <= -2.0f ? make_float2(__fmul_rn(9.0f, s2), -th - 2.0f) : make_float2(th, -1.0f);
}

// (D_c, D_clamp) of a Gaussian with σ² = s2 and opacity o: composited-eligible ⇔ d² ≤ D_c =
// min(D_floor, fl(9·s2)) (the 3σ truncation and the α floor in one compare), clamped ⇔
// d² ≤ D_clamp (−1: never; w ≤ 1 so only o > 0.999 can clamp).
__device__ __forceinline__ float2 alpha_thresholds(float s2, float o) {
    const float cap = __fmul_rn(9.0f, s2);
    const float dc = alpha_threshold_d2(s2, o, kAlphaMin, false, cap);
    const float dcl = o > kAlphaMax ? alpha_threshold_d2(s2, o, kAlphaMax, true, cap) : -1.0f;
    return make_float2(dc, dcl);
}

// α VALUE of a pair (the decision d² ≤ D_c is the caller's): 0.999 when clamped (d² ≤ D_clamp),
// else min(o·w, 0.999) with the fast w = 2^(d²·escale) (relative error ≤ ~1.1e-6 against the
// oracle's o·w).  The forward passes dcl = −1: its α value needs no clamp decision (an exact-vs-
// fast difference at the clamp is a value difference of ~1e-6); the backward passes D_clamp, for
// ∂α/∂o = 0 on clamped pairs.  w is returned for the backward's chain.
__device__ __forceinline__ float pair_alpha(float d2, float escale, float o, float dcl, float &w) {
    w = fast_exp2(d2 * escale);
    return d2 <= dcl ? kAlphaMax : fminf(o * w, kAlphaMax);
}

// pair_alpha with dcl = −1 (the forward): d² ≥ 0 never passes d² ≤ −1, so the same value
// without the compare and select the compiler cannot drop
__device__ __forceinline__ float pair_alpha_value(float d2, float escale, float o, float &w) {
    w = fast_exp2(d2 * escale);
    return fminf(o * w, kAlphaMax);
}

// d² of pixel (xf, yf) to centre (u, v), DESIGN.md §3 step 7 (no FMA contraction)
__device__ __forceinline__ float pair_d2(float xf, float yf, float u, float v) {
    const float dx = __fsub_rn(xf, u), dy = __fsub_rn(yf, v);
    return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

#ifdef VTGS_SUB_8x4
// Mask of the warp's 32 pixels (bit = (y−sy)·8 + (x−sx)) inside the entry's rect and,
// conservatively, inside its disc d² ≤ 9σ².  The exact fp32 test is re-done per pixel in the
// compositing loops; this mask only has to be a superset of the pixels that pass it: row y
// is kept iff fl(dy·dy) ≤ 9σ² (the same fp32 dy² the exact test adds to a non-negative dx²),
// and its columns are widened by 0.01 px around u ± √(9σ² − dy²).
__device__ __forceinline__ unsigned lane_mask(const float4 A, const uint2 r, int sx, int sy) {
    const int x0 = max((int)(r.x & 0xffffu), sx), x1 = min((int)(r.x >> 16), sx + 7);
    const int y0 = max((int)(r.y & 0xffffu), sy), y1 = min((int)(r.y >> 16), sy + 3);
    const float fsy = (float)sy;
    unsigned m = 0;
    // the sub-tile's 4 rows, branch-free (lanes are entries with different row ranges: a loop
    // over each entry's rows diverged); a row outside the rect or the disc selects 0
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float dy = __fsub_rn(fsy + (float)j, A.y);
        const float dy2 = __fmul_rn(dy, dy);
        // the exact test accepts |dx| up to √(r2 + ½ulp(9σ²)) (dx² + dy² rounds down onto 9σ²):
        // widen by A.z·2⁻²³ ≥ ½ulp before the root, then by 0.01 px for the approximate rsqrt
        const float r2 = A.z - dy2 + A.z * 1.1920929e-7f;           // ≥ 0 on a kept row
        const float hw = r2 * rsqrt_approx(fmaxf(r2, 1e-30f)) + 0.01f; // √r2 (+ ≤ 2⁻²² rel.) + margin
        const int xa = max(x0, (int)ceilf(A.x - hw)), xb = min(x1, (int)floorf(A.x + hw));
        const bool ok = sy + j >= y0 && sy + j <= y1 && dy2 <= A.z && xa <= xb;
        const unsigned lo = (unsigned)min(max(xa - sx, 0), 7), hi = (unsigned)min(max(xb - sx, 0), 7);
        const unsigned row = (0xffu >> (7u - hi)) & (0xffu << lo);
        m |= ok ? row << (8 * j) : 0u;
    }
    return m;
}
#else
// Mask of the warp's 32 pixels (bit = (y−sy)·4 + (x−sx)) inside the entry's rect and,
// conservatively, inside its disc d² ≤ D_c.  The exact fp32 test is re-done per pixel in the
// compositing loops; this mask only has to be a superset of the pixels that pass it: column x is
// kept iff fl(dx·dx) ≤ D_c (the same fp32 dx² the exact test adds to a non-negative dy²), and its
// rows are widened by 0.01 px around v ± √(D_c − dx²) — the 8 × 4 shape's row test with x and y
// exchanged (the exact test is symmetric in them).  Branch-free over the sub-tile's 4 columns.
__device__ __forceinline__ unsigned lane_mask(const float4 A, const uint2 r, int sx, int sy) {
    const int x0 = max((int)(r.x & 0xffffu), sx), x1 = min((int)(r.x >> 16), sx + 3);
    const int y0 = max((int)(r.y & 0xffffu), sy), y1 = min((int)(r.y >> 16), sy + 7);
    const float fsx = (float)sx;
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float dx = __fsub_rn(fsx + (float)j, A.x);
        const float dx2 = __fmul_rn(dx, dx);
        // the exact test accepts |dy| up to √(r2 + ½ulp(D_c)) (dx² + dy² rounds down onto D_c):
        // widen by A.z·2⁻²³ ≥ ½ulp before the root, then by 0.01 px for the approximate rsqrt
        const float r2 = A.z - dx2 + A.z * 1.1920929e-7f;
        const float hh = r2 * rsqrt_approx(fmaxf(r2, 1e-30f)) + 0.01f;
        const int ya = max(y0, (int)ceilf(A.y - hh)), yb = min(y1, (int)floorf(A.y + hh));
        const bool ok = sx + j >= x0 && sx + j <= x1 && dx2 <= A.z && ya <= yb;
        const unsigned lo = (unsigned)min(max(ya - sy, 0), 7), hi = (unsigned)min(max(yb - sy, 0), 7);
        const unsigned col = 0x11111111u & (0xffffffffu << (4 * lo)) & (0xffffffffu >> (28 - 4 * hi));
        m |= ok ? col << j : 0u;
    }
    return m;
}
#endif

// The entry's ±3σ pixel rect recomputed from its projection with exactly k_project_count's fp32
// operations (|proj.w| is the clamped σ it used), so the compositing kernels need not gather it.
__device__ __forceinline__ uint2 rect_from_proj(const float4 pr, int W, int H) {
    const float e = __fmul_rn(3.0f, fabsf(pr.w));
    const float Wm1 = (float)(W - 1), Hm1 = (float)(H - 1);
    const float cx0 = ceilf(__fsub_rn(pr.x, e)), cx1 = floorf(__fadd_rn(pr.x, e));
    const float cy0 = ceilf(__fsub_rn(pr.y, e)), cy1 = floorf(__fadd_rn(pr.y, e));
    const int x0 = cx0 < 0.0f ? 0 : (int)cx0, x1 = cx1 > Wm1 ? (int)Wm1 : (int)cx1;
    const int y0 = cy0 < 0.0f ? 0 : (int)cy0, y1 = cy1 > Hm1 ? (int)Hm1 : (int)cy1;
    return make_uint2((uint32_t)x0 | ((uint32_t)x1 << 16), (uint32_t)y0 | ((uint32_t)y1 << 16));
}

// 32×32 bit-matrix transpose across the warp: lane j holds row j on entry, lane i holds
// column i on exit (bit j of the result = bit i of lane j's input).
__device__ __forceinline__ unsigned transpose32(unsigned x, unsigned lane) {
    const unsigned M[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int s = 16 >> i;
        const unsigned y = __shfl_xor_sync(kFullMask, x, s);
        x = (lane & s) ? ((x & ~M[i]) | ((y & ~M[i]) >> s)) : ((x & M[i]) | ((y & M[i]) << s));
    }
    return x;
}

#ifdef VTGS_SUB_8x4
// Bit s (s = 2k + c) set iff the rect touches sub-tile (c, k) = pixels
// [tx0 + 8c, tx0 + 8c + 7] × [ty0 + 4k, ty0 + 4k + 3] of the tile at (tx0, ty0).
__device__ __forceinline__ unsigned subtile_bits(uint2 r, int tx0, int ty0) {
    const int x0 = (int)(r.x & 0xffffu), x1 = (int)(r.x >> 16);
    const int y0 = (int)(r.y & 0xffffu), y1 = (int)(r.y >> 16);
    const unsigned cols = (x0 <= tx0 + 7 ? 1u : 0u) | (x1 >= tx0 + 8 ? 2u : 0u);
    // sub-tile rows k0 .. k1 the rect touches (the rect overlaps the tile: k0 ≤ 3, k1 ≥ 0)
    const int k0 = max(y0 - ty0, 0) >> 2, k1 = min(y1 - ty0, 15) >> 2;
    const unsigned rows = (0xffu >> (6 - 2 * k1)) & (0xffu << (2 * k0)) & 0x55u;   // bit 2k per row k
    return ((cols & 1u) ? rows : 0u) | ((cols & 2u) ? rows << 1 : 0u);
}
#else
// Bit s (s = c + 4k) set iff the rect touches sub-tile (c, k) = pixels
// [tx0 + 4c, tx0 + 4c + 3] × [ty0 + 8k, ty0 + 8k + 7] of the tile at (tx0, ty0).
__device__ __forceinline__ unsigned subtile_bits(uint2 r, int tx0, int ty0) {
    const int x0 = (int)(r.x & 0xffffu), x1 = (int)(r.x >> 16);
    const int y0 = (int)(r.y & 0xffffu), y1 = (int)(r.y >> 16);
    // sub-tile columns c0 .. c1 and rows k0 .. k1 the rect touches (it overlaps the tile)
    const int c0 = max(x0 - tx0, 0) >> 2, c1 = min(x1 - tx0, 15) >> 2;
    const int k0 = max(y0 - ty0, 0) >> 3, k1 = min(y1 - ty0, 15) >> 3;
    const unsigned cols = (0xfu >> (3 - c1)) & (0xfu << c0);
    return (k0 == 0 ? cols : 0u) | (k1 == 1 ? cols << 4 : 0u);
}
#endif

}  // namespace vtgs
