// (2)–(4) Forward render: projection + 16×16 tile binning, per-tile depth sort, per-tile
// front-to-back compositing.  PAPER.md:146 (Eq. 1 `splat`), SPEC.md:124-150, :169-175,
// BASELINE.json north_star parts (2)-(4).
//
// Launch sequence (all on the caller's stream, no host synchronisation, graph-capturable):
//   memset(tile_count) → k_project_count → k_scan_tiles → k_emit_pairs → k_tile_sort
//   → k_composite_fwd
// Pairs are bucketed by tile with warp-aggregated atomics (one global atomic per distinct tile
// per warp), then each tile's bucket is sorted in shared memory by (z bits, gid) — one
// bucket-scatter pass plus an on-chip sort instead of a multi-pass global 64-bit radix sort
// (K4/K5).
#include <stdlib.h>

#include "composite_common.cuh"

namespace vtgs {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------------------------------
// K2: projection, culling, footprint rect, tile counts.  DESIGN.md §3 steps 3-5.
// ------------------------------------------------------------------------------------------
struct Footprint {
    bool vis;
    float u, v, z, s;
    bool clamped;
    int x0, y0, x1, y1;
};

__device__ __forceinline__ Footprint project_one(float4 pr, const PoseR &P, const vtgs_intrinsics &in,
                                                 float fmean, float Wm1, float Hm1) {
    Footprint f;
    f.vis = false;
    float xc[3];
    view_transform(P.R, P.t, pr, xc);
    const float z = xc[2];
    if (!(pr.w > 0.0f) || !(z > kNearClip)) return f;
    const float u = __fadd_rn(__fdiv_rn(__fmul_rn(in.fx, xc[0]), z), in.cx);
    const float v = __fadd_rn(__fdiv_rn(__fmul_rn(in.fy, xc[1]), z), in.cy);
    if (!isfinite(u) || !isfinite(v)) return f;
    const float s0 = __fdiv_rn(__fmul_rn(fmean, pr.w), z);
    const bool clamped = s0 < kSigmaMin;
    const float s = clamped ? kSigmaMin : s0;
    const float e = __fmul_rn(3.0f, s);
    if (__fadd_rn(u, e) < 0.0f || __fsub_rn(u, e) > Wm1 || __fadd_rn(v, e) < 0.0f || __fsub_rn(v, e) > Hm1)
        return f;
    const float cx0 = ceilf(__fsub_rn(u, e)), cx1 = floorf(__fadd_rn(u, e));
    const float cy0 = ceilf(__fsub_rn(v, e)), cy1 = floorf(__fadd_rn(v, e));
    f.x0 = cx0 < 0.0f ? 0 : (int)cx0;
    f.x1 = cx1 > Wm1 ? (int)Wm1 : (int)cx1;
    f.y0 = cy0 < 0.0f ? 0 : (int)cy0;
    f.y1 = cy1 > Hm1 ? (int)Hm1 : (int)cy1;
    if (f.x0 > f.x1 || f.y0 > f.y1) return f;
    f.vis = true;
    f.u = u; f.v = v; f.z = z; f.s = s; f.clamped = clamped;
    return f;
}

__global__ void __launch_bounds__(256) k_project_count(const float4 *__restrict__ pos_rad,
                                                       const float4 *__restrict__ col_opa, int64_t N,
                                                       const vtgs_pose *__restrict__ view,
                                                       vtgs_intrinsics in, int ntx,
                                                       float4 *__restrict__ proj,
                                                       uint2 *__restrict__ rect,
                                                       float *__restrict__ thr,
                                                       uint32_t *__restrict__ tile_count) {
    __shared__ PoseR P;
    if (threadIdx.x == 0) pose_rotation(*view, P);
    __syncthreads();
    const float fmean = __fmul_rn(0.5f, __fadd_rn(in.fx, in.fy));
    const float Wm1 = (float)(in.width - 1), Hm1 = (float)(in.height - 1);
    const int64_t Nr = (N + 31) & ~(int64_t)31;  // whole warps iterate together
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    __shared__ uint32_t qg[8][64];   // per warp: Gaussians waiting for the exact threshold search
    __shared__ float qs[8][64];      // and their σ
    const int wq = threadIdx.x >> 5;
    int qn = 0;
    // the next iteration's state is loaded one iteration ahead (the loop is latency-bound)
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float4 pr_next = g0 < N ? __ldg(pos_rad + g0) : make_float4(0.f, 0.f, 0.f, 0.f);
    float o_next = g0 < N ? __ldg(&col_opa[g0].w) : 0.f;
    for (int64_t g = g0; g < Nr; g += stride) {
        Footprint f;
        f.vis = false;
        bool slow = false;
        const float4 pr_g = pr_next;
        const float o_g = o_next;
        if (g + stride < N) {
            pr_next = __ldg(pos_rad + g + stride);
            o_next = __ldg(&col_opa[g + stride].w);
        }
        if (g < N) {
            f = project_one(pr_g, P, in, fmean, Wm1, Hm1);
            proj[g] = f.vis ? make_float4(f.u, f.v, f.z, f.clamped ? -f.s : f.s) : make_float4(0.f, 0.f, 0.f, 0.f);
            rect[g] = f.vis ? make_uint2((uint32_t)f.x0 | ((uint32_t)f.x1 << 16), (uint32_t)f.y0 | ((uint32_t)f.y1 << 16))
                            : make_uint2(0xffffffffu, 0xffffffffu);
            // exact α decision thresholds in d² (composite_common.cuh), once per Gaussian per view:
            // the common case here, the search for the rest on a dense work list (no divergence)
            float2 th = make_float2(-1.f, -1.f);
            slow = f.vis && !alpha_thresholds_fast(__fmul_rn(f.s, f.s), o_g, th);
            thr[g] = th.x;
        }
        // the Gaussians the fast test could not settle join the warp's queue; every 32 of them the
        // whole warp runs the exact search, one per lane (no divergence, no global atomics)
        const unsigned sm = __ballot_sync(kFull, slow);
        if (sm) {
            if (slow) {
                const int at = qn + __popc(sm & lanemask_lt());
                qg[wq][at] = (uint32_t)g;
                qs[wq][at] = f.s;
            }
            qn += __popc(sm);
            __syncwarp();
            if (qn >= 32) {
                const uint32_t gq = qg[wq][lane_id()];
                const float sq = qs[wq][lane_id()];
                thr[gq] = thr_pack(alpha_thresholds(__fmul_rn(sq, sq), __ldg(&col_opa[gq].w)), 0.f);
                __syncwarp();
                qn -= 32;
                if ((int)lane_id() < qn) {
                    qg[wq][lane_id()] = qg[wq][32 + lane_id()];
                    qs[wq][lane_id()] = qs[wq][32 + lane_id()];
                }
                __syncwarp();
            }
        }
        const int tx0 = f.vis ? f.x0 >> 4 : 0, ty0 = f.vis ? f.y0 >> 4 : 0;
        const int ntg = f.vis ? (f.x1 >> 4) - tx0 + 1 : 0;
        const int cnt = f.vis ? ntg * ((f.y1 >> 4) - ty0 + 1) : 0;
        // tiles in row-major order, (kx, ky) stepped incrementally (no integer division)
        int kx = 0, trow = ty0 * ntx + tx0;
        for (int k = 0; __any_sync(kFull, k < cnt); ++k) {
            const int tile = k < cnt ? trow + kx : -1;
            if (++kx == ntg) { kx = 0; trow += ntx; }
            const unsigned peers = __match_any_sync(kFull, tile);
            if (tile >= 0 && (int)lane_id() == __ffs(peers) - 1) atomicAdd(&tile_count[tile], (uint32_t)__popc(peers));
        }
    }
    if ((int)lane_id() < qn) {   // the queue's remainder
        const uint32_t gq = qg[wq][lane_id()];
        const float sq = qs[wq][lane_id()];
        thr[gq] = thr_pack(alpha_thresholds(__fmul_rn(sq, sq), __ldg(&col_opa[gq].w)), 0.f);
    }
}

// ------------------------------------------------------------------------------------------
// K3: exclusive scan of the tile counts (one CTA; ≤ a few thousand tiles).  On capacity
// overflow every count is zeroed (the render is empty) and the overflow flag is raised.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_scan_tiles(uint32_t *__restrict__ tile_count,
                                                     uint32_t *__restrict__ tile_start,
                                                     uint32_t *__restrict__ cursor, int T,
                                                     unsigned long long cap,
                                                     DevScalars *__restrict__ dev,
                                                     const vtgs_pose *__restrict__ view,
                                                     vtgs_pose *__restrict__ view_copy,
                                                     uint32_t *__restrict__ radix_list) {
    if (threadIdx.x == 0) *view_copy = *view;  // the backward reads the copy (caller may reuse view)
    __shared__ unsigned long long warp_sum[32];
    __shared__ unsigned int warp_max[32];
    __shared__ unsigned long long total_s;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int per = (T + 1023) / 1024;
    const int b = tid * per, e = min(b + per, T);
    unsigned long long s = 0;
    unsigned int mx = 0;
    for (int i = b; i < e; ++i) {
        s += tile_count[i];
        mx = max(mx, tile_count[i]);
    }
    unsigned long long incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane == 31) warp_sum[w] = incl;
    if (lane == 0) warp_max[w] = mx;
    __syncthreads();
    if (w == 0) {
        unsigned long long v = warp_sum[lane];
        unsigned int m = warp_max[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFull, v, o);
            if (lane >= o) v += y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
        warp_sum[lane] = v;
        if (lane == 31) {
            total_s = v;
            dev->n_pairs = v;
            dev->max_tile = m;
            dev->overflow = v > cap ? 1u : 0u;
        }
    }
    __syncthreads();
    const bool overflow = total_s > cap;
    unsigned long long run = incl - s + (w > 0 ? warp_sum[w - 1] : 0ull);
    for (int i = b; i < e; ++i) {
        const uint32_t c = tile_count[i];
        tile_start[i] = overflow ? 0u : (uint32_t)run;
        cursor[i] = overflow ? 0u : (uint32_t)run;
        if (overflow) tile_count[i] = 0;
        run += c;
    }
    if (tid == 0) tile_start[T] = overflow ? 0u : (uint32_t)total_s;
}

// ------------------------------------------------------------------------------------------
// K4: scatter (z bits, gid) into each tile's bucket (order inside a bucket is arbitrary; the
// per-tile sort below makes it (z, gid)).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_emit_pairs(const float4 *__restrict__ proj,
                                                    const uint2 *__restrict__ rect, int64_t N, int ntx,
                                                    const uint32_t *__restrict__ tile_start,
                                                    uint32_t *__restrict__ cursor,
                                                    uint32_t *__restrict__ keys,
                                                    uint32_t *__restrict__ vals,
                                                    uint8_t *__restrict__ pbits,
                                                    const DevScalars *__restrict__ dev) {
    if (dev->overflow) return;
    const int64_t Nr = (N + 31) & ~(int64_t)31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const unsigned lane = lane_id();
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < Nr; g += stride) {
        int cnt = 0, ntg = 1, tx0 = 0, ty0 = 0;
        uint32_t zb = 0;
        uint2 r = make_uint2(0u, 0u);
        if (g < N) {
            r = rect[g];
            if (r.x != 0xffffffffu) {
                const int x0 = r.x & 0xffff, x1 = r.x >> 16, y0 = r.y & 0xffff, y1 = r.y >> 16;
                tx0 = x0 >> 4;
                ty0 = y0 >> 4;
                ntg = (x1 >> 4) - tx0 + 1;
                cnt = ntg * ((y1 >> 4) - ty0 + 1);
                zb = __float_as_uint(proj[g].z);
            }
        }
        int kx = 0, ky = 0;   // (tile column, row) offsets stepped incrementally (no integer division)
        // (two tiles per iteration, both cursor atomics in flight together, measured slower:
        // emit 0.055 → 0.060 ms at config 2, 0.179 → 0.211 ms at config 5)
        for (int k = 0; __any_sync(kFull, k < cnt); ++k) {
            const int tile = k < cnt ? (ty0 + ky) * ntx + tx0 + kx : -1;
            const int tcx = tx0 + kx, tcy = ty0 + ky;
            if (++kx == ntg) { kx = 0; ++ky; }
            const unsigned peers = __match_any_sync(kFull, tile);
            const int leader = __ffs(peers) - 1;
            uint32_t base = 0;
            if (tile >= 0 && (int)lane == leader) base = atomicAdd(&cursor[tile], (uint32_t)__popc(peers));
            base = __shfl_sync(kFull, base, leader);
            if (tile >= 0) {
                const uint32_t slot = base + __popc(peers & lanemask_lt());
                VTGS_CHECK(slot < tile_start[tile + 1]);   // the counts of k_project_count hold
                keys[slot] = zb;
                vals[slot] = (uint32_t)g;
                pbits[slot] = (uint8_t)subtile_bits(r, tcx * kTile, tcy * kTile);
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// K5: per-tile sort by (z bits, gid).  Stable LSD radix sort on the z bits that vary inside
// the tile (8-bit digits; in-warp stable ranking with 8 ballots per digit; digit-major scan over
// the 8 warps' histograms), then runs of equal z are ordered by gid.  Buffers are shared memory
// for lists ≤ kSortCap, global scratch above that.
// ------------------------------------------------------------------------------------------
template <typename OffT>
__device__ __forceinline__ int block_sort_zgid(uint32_t *K0, uint32_t *V0, uint32_t *K1, uint32_t *V1,
                                               OffT *OFF, uint32_t *HIST, uint32_t *red, int n) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t o = 0, a = 0xffffffffu;
    for (int i = tid; i < n; i += kBlock) {
        const uint32_t k = K0[i];
        o |= k;
        a &= k;
    }
    o = __reduce_or_sync(kFull, o);
    a = __reduce_and_sync(kFull, a);
    if (lane == 0) { red[w] = o; red[8 + w] = a; }
    __syncthreads();
    o = 0; a = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < 8; ++i) { o |= red[i]; a &= red[8 + i]; }
    const uint32_t diff = o ^ a;
    const int lo = diff ? __ffs(diff) - 1 : 0;
    const int hi = diff ? 32 - __clz(diff) : 0;
    const int npass = (hi - lo + 7) >> 3;
    const int S = ((n + 8 * 32 - 1) / (8 * 32)) * 32;  // items per warp segment
    const int seg0 = min(w * S, n), seg1 = min(seg0 + S, n);
    uint32_t *Ks = K0, *Vs = V0, *Kd = K1, *Vd = V1;
    uint32_t *H = HIST + w * 256;
    for (int p = 0; p < npass; ++p) {
        const int shift = lo + 8 * p;
        for (int d = lane; d < 256; d += 32) H[d] = 0;
        __syncwarp();
        for (int base = seg0; base < seg1; base += 32) {
            const int i = base + lane;
            const bool valid = i < seg1;
            const uint32_t d = valid ? (Ks[i] >> shift) & 255u : 0u;
            unsigned m = __ballot_sync(kFull, valid);
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const bool bit = (d >> b) & 1u;
                const unsigned bb = __ballot_sync(kFull, bit);
                m &= bit ? bb : ~bb;
            }
            const uint32_t rank = __popc(m & lanemask_lt());
            const uint32_t cnt0 = valid ? H[d] : 0u;
            __syncwarp();
            if (valid && rank == 0) H[d] = cnt0 + __popc(m);
            __syncwarp();
            if (valid) OFF[i] = (OffT)(cnt0 + rank);
        }
        __syncthreads();
        {   // digit-major exclusive scan over (digit, warp)
            const int d = tid;  // kBlock == 256 digits
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) { c[ww] = HIST[ww * 256 + d]; tot += c[ww]; }
            uint32_t incl = tot;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, off);
                if (lane >= off) incl += y;
            }
            if (lane == 31) red[16 + w] = incl;
            __syncthreads();
            uint32_t wpre = 0;
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) wpre += ww < w ? red[16 + ww] : 0u;
            uint32_t run = wpre + incl - tot;
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) { HIST[ww * 256 + d] = run; run += c[ww]; }
        }
        __syncthreads();
        for (int i = seg0 + lane; i < seg1; i += 32) {
            const uint32_t k = Ks[i];
            const uint32_t dst = H[(k >> shift) & 255u] + (uint32_t)OFF[i];
            Kd[dst] = k;
            Vd[dst] = Vs[i];
        }
        __syncthreads();
        uint32_t *t = Ks; Ks = Kd; Kd = t;
        t = Vs; Vs = Vd; Vd = t;
    }
    // equal z: ascending gid (the tie-break of SPEC.md:171)
    for (int i = tid; i < n; i += kBlock) {
        const uint32_t k = Ks[i];
        if ((i == 0 || Ks[i - 1] != k) && i + 1 < n && Ks[i + 1] == k) {
            int j = i + 1;
            while (j < n && Ks[j] == k) ++j;
            for (int x = i + 1; x < j; ++x) {
                const uint32_t v = Vs[x];
                int y = x - 1;
                while (y >= i && Vs[y] > v) { Vs[y + 1] = Vs[y]; --y; }
                Vs[y + 1] = v;
            }
        }
    }
    __syncthreads();
    return npass & 1;
}

// Sub-lists of the sorted tile list: sub-tile s (4×8 pixels, composite_common.cuh) gets, in
// tile-list order, every entry whose rect touches it.  Stored at out + s·n (capacity n each);
// counts at sub_count[0..7].  Stable block-wide compaction, 256 entries per round.
__device__ __forceinline__ void build_sublists(const uint32_t *V, int n, const uint2 *__restrict__ rect, int tx0,
                                               int ty0, uint32_t *__restrict__ out,
                                               uint32_t *__restrict__ sub_count, uint32_t *sh, uint8_t *bits8) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t *wcnt = sh;        // [8 warps][8 sub-tiles] counts of this round
    uint32_t *woff = sh + 64;   // [8 warps][8 sub-tiles] output offsets of this round
    uint32_t *run = sh + 128;   // [8] running totals
    if (tid < 8) run[tid] = 0;
    // all rect gathers of the tile in flight together, then the ordered compaction rounds
#pragma unroll 4
    for (int i = tid; i < n; i += kBlock) bits8[i] = (uint8_t)subtile_bits(__ldg(rect + V[i]), tx0, ty0);
    __syncthreads();
    for (int r0 = 0; r0 < n; r0 += kBlock) {
        const int i = r0 + tid;
        const uint32_t bits = i < n ? bits8[i] : 0u;
        const uint32_t g = i < n ? V[i] : 0u;
        unsigned b[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) b[s] = __ballot_sync(kFull, (bits >> s) & 1u);
        if (lane < 8) {
            unsigned c = 0;
#pragma unroll
            for (int s = 0; s < 8; ++s) c = lane == s ? __popc(b[s]) : c;
            wcnt[w * 8 + lane] = c;
        }
        __syncthreads();
        if (tid < 64) {   // (warp ww, sub-tile ss): offset = run + counts of the warps before
            const int ww = tid >> 3, ss = tid & 7;
            uint32_t o = run[ss];
            for (int x = 0; x < ww; ++x) o += wcnt[x * 8 + ss];
            woff[tid] = o;
        }
        __syncthreads();
        if (tid < 8) run[tid] = woff[56 + tid] + wcnt[56 + tid];
#pragma unroll
        for (int s = 0; s < 8; ++s)
            if ((bits >> s) & 1u) out[(size_t)s * n + woff[w * 8 + s] + __popc(b[s] & lanemask_lt())] = g;
        __syncthreads();
    }
    if (tid < 8) sub_count[tid] = run[tid];
}

// CAP: longest list sorted in shared memory by this instantiation.  Lists in (LO, CAP] are
// sorted on chip; with GLOBAL = true, lists > CAP use the same code on global scratch.
template <int LO, int CAP, bool GLOBAL>
__global__ void __launch_bounds__(kBlock) k_tile_sort(const uint32_t *__restrict__ tile_count,
                                                      const uint32_t *__restrict__ tile_start,
                                                      uint32_t *keys, uint32_t *vals, uint32_t *keys2,
                                                      uint32_t *vals2, uint32_t *offs,
                                                      const uint2 *__restrict__ rect, int ntx,
                                                      uint32_t *__restrict__ sub_lists,
                                                      uint32_t *__restrict__ sub_count,
                                                      const uint32_t *__restrict__ work_list,
                                                      const DevScalars *__restrict__ dev) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t hist[8 * 256];
    __shared__ uint32_t red[32];
    // without a work list: one CTA per tile, tiles in (LO, CAP]; with one (the bucket-sort path):
    // a small grid walks the list of long / degenerate tiles that k_scan_tiles and
    // k_tile_sort_bucket appended (no wave of empty CTAs over every tile)
    // with a work list: w walks it; without one: a single pass, tile = blockIdx.x
    const int nwork = work_list ? (int)dev->radix_count : (int)blockIdx.x + 1;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int tile = work_list ? (int)work_list[w] : (int)blockIdx.x;
    const int n = (int)tile_count[tile];
    if (!work_list && (n <= LO || (!GLOBAL && n > CAP))) return;
    const uint32_t base = tile_start[tile];
    const int ty = tile / ntx, tx = tile - ty * ntx;
    uint32_t *out = sub_lists + (size_t)8 * base;
    if (n <= CAP) {
        uint32_t *K0 = sm, *V0 = sm + CAP, *K1 = sm + 2 * CAP, *V1 = sm + 3 * CAP;
        uint16_t *OFF = reinterpret_cast<uint16_t *>(sm + 4 * CAP);
        for (int i = threadIdx.x; i < n; i += kBlock) { K0[i] = keys[base + i]; V0[i] = vals[base + i]; }
        __syncthreads();
        bool odd = false;
        if (n > 1) odd = block_sort_zgid<uint16_t>(K0, V0, K1, V1, OFF, hist, red, n);
        const uint32_t *Vr = odd ? V1 : V0;
        uint8_t *bits8 = reinterpret_cast<uint8_t *>(odd ? K0 : K1);  // the idle key buffer
        for (int i = threadIdx.x; i < n; i += kBlock) vals[base + i] = Vr[i];
        build_sublists(Vr, n, rect, tx * kTile, ty * kTile, out, sub_count + 8 * tile, hist, bits8);
    } else if (GLOBAL) {
        const int odd = block_sort_zgid<uint32_t>(keys + base, vals + base, keys2 + base, vals2 + base,
                                                  offs + base, hist, red, n);
        if (odd)
            for (int i = threadIdx.x; i < n; i += kBlock) vals[base + i] = vals2[base + i];
        __syncthreads();
        uint8_t *bits8 = reinterpret_cast<uint8_t *>(odd ? keys + base : keys2 + base);
        build_sublists(vals + base, n, rect, tx * kTile, ty * kTile, out, sub_count + 8 * tile, hist, bits8);
    }
    __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// K5 (main path): per-tile bucket + rank sort by (z bits, gid), lists ≤ CAP on chip.
//   1. keys / gids → shared memory, block min / max of the z bits;
//   2. bucket = (key − kmin) ≫ shift with shift chosen so the key range spans ≤ 4096 buckets
//      (z bits of positive floats are monotone as unsigned integers), counted with shared-memory
//      integer atomics, exclusive scan → contiguous bucket segments;
//   3. scatter into the segments (arbitrary order inside a segment);
//   4. every element's final position = segment start + its rank among the segment's elements
//      by (key, gid) — a direct O(c) count per element, no further passes.
// One global read of the pairs, one write of the sorted gids.  A tile whose largest bucket
// exceeds kMaxBucket (many equal or nearly equal depths) falls back to the radix sort above.
// ------------------------------------------------------------------------------------------
constexpr int kMaxBucket = 256;

// Sub-lists from the sorted gids V and their sub-tile bits B: thread-local runs of E entries,
// one block scan of the 8 per-sub-tile counts packed 4 × 16 bits into two 64-bit words.
// stride = the tile's list length (sub-list capacity); sub_off (chunked tiles, else nullptr) =
// where this part of the tile starts in each of the 8 sub-lists; sub_count is written only for
// whole tiles (sub_off == nullptr).
template <int NT>
__device__ __forceinline__ void sublists_from_bits(const uint32_t *V, const uint8_t *B, int n,
                                                   uint32_t *__restrict__ out, uint32_t *__restrict__ sub_count,
                                                   unsigned long long (*red64)[33], int stride,
                                                   const uint32_t *sub_off) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int E = (n + NT - 1) / NT;
    const int i0 = min(tid * E, n), i1 = min(i0 + E, n);
    unsigned long long c0 = 0, c1 = 0;  // counts of sub-tiles 0-3 / 4-7, 16 bits each
    for (int i = i0; i < i1; ++i) {
        const uint32_t b = B[i];
        c0 += (unsigned long long)(b & 1u) | ((unsigned long long)((b >> 1) & 1u) << 16) |
              ((unsigned long long)((b >> 2) & 1u) << 32) | ((unsigned long long)((b >> 3) & 1u) << 48);
        c1 += (unsigned long long)((b >> 4) & 1u) | ((unsigned long long)((b >> 5) & 1u) << 16) |
              ((unsigned long long)((b >> 6) & 1u) << 32) | ((unsigned long long)((b >> 7) & 1u) << 48);
    }
    unsigned long long s0 = c0, s1 = c1;  // inclusive warp scan (no carries: every total ≤ n < 2^16)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y0 = __shfl_up_sync(kFull, s0, o), y1 = __shfl_up_sync(kFull, s1, o);
        if (lane >= o) { s0 += y0; s1 += y1; }
    }
    if (lane == 31) { red64[0][w] = s0; red64[1][w] = s1; }
    __syncthreads();
    if (w == 0) {   // exclusive scan of the warps' totals (entry NW = the block total)
        unsigned long long a0 = lane < NW ? red64[0][lane] : 0ull, a1 = lane < NW ? red64[1][lane] : 0ull;
        unsigned long long i0s = a0, i1s = a1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y0 = __shfl_up_sync(kFull, i0s, o), y1 = __shfl_up_sync(kFull, i1s, o);
            if (lane >= o) { i0s += y0; i1s += y1; }
        }
        __syncwarp();
        red64[0][lane] = i0s - a0;
        red64[1][lane] = i1s - a1;
        if (lane == 31) { red64[0][NW] = i0s; red64[1][NW] = i1s; }   // NW < 32 (i0s at lane 31 = total)
    }
    __syncthreads();
    const unsigned long long p0 = s0 - c0 + red64[0][w], p1 = s1 - c1 + red64[1][w];
    const unsigned long long t0 = red64[0][NW], t1 = red64[1][NW];
    if (!sub_off && tid < 8) sub_count[tid] = (uint32_t)(((tid < 4 ? t0 : t1) >> (16 * (tid & 3))) & 0xffffu);
    uint32_t off[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        off[q] = (uint32_t)((p0 >> (16 * q)) & 0xffffu);
        off[4 + q] = (uint32_t)((p1 >> (16 * q)) & 0xffffu);
    }
    if (sub_off)
#pragma unroll
        for (int q = 0; q < 8; ++q) off[q] += sub_off[q];
    for (int i = i0; i < i1; ++i) {
        const uint32_t b = B[i], g = V[i];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if ((b >> q) & 1u) out[(size_t)q * stride + off[q]++] = g;
    }
}

// ------------------------------------------------------------------------------------------
// K5 (main path): per-tile bucket + rank sort by (z bits, gid) of lists of ≤ CAP entries on
// chip with NT threads, carrying each pair's sub-tile bits (written by k_emit_pairs).
//   1. keys / gids / bits → shared memory, block min / max of the z bits;
//   2. bucket = (key − kmin) ≫ shift with shift chosen so the key range spans ≤ NB buckets
//      (z bits of positive floats are monotone as unsigned integers), counted with shared-memory
//      integer atomics, exclusive scan → contiguous bucket segments;
//   3. scatter into the segments (arbitrary order inside a segment);
//   4. every element's final position = segment start + its rank among its segment by
//      (key, gid) — a direct O(bucket size) count per element;
//   5. the sorted gids and the 8 sub-lists are written.
// A tile whose largest bucket exceeds kMaxBucket (many equal or nearly equal depths) is flagged
// and left to the radix sort kernel.  Lists in (LO, CAP] are handled; others return at once.
// ------------------------------------------------------------------------------------------
// K5, long lists (> kSortCap entries, configs 4 / 5): instead of one CTA sorting the whole list
// on global scratch, the long tile's CTA of the bucket-sort launch (k_tile_sort_bucket, which
// would otherwise skip it) buckets it by depth — block min / max of the z bits,
// NB buckets over that range (4,096 / 16,384 by length), segment starts s_b — and cuts it into CHUNKS:
// chunk(b) = ⌊s_b / tgt⌋ with tgt = kSortCap − max(largest bucket, kMaxBucket), so a chunk holds
// ≤ kSortCap entries and chunks are depth-ordered.  The pairs are scattered into bucket order (keys2 /
// vals2 / bits2), and per chunk the plan records its offset in the tile, its size and where it
// starts in each of the 8 sub-lists; k_tile_sort_bucket<…, CHUNKED> then sorts every chunk on
// chip (many CTAs per long tile).  A tile with a bucket > kSortCap / 2 (near-equal depths) or
// more than kMaxChunks chunks goes to the radix kernel as before.
// ------------------------------------------------------------------------------------------
// dynamic shared memory of the on-chip bucket sort of lists ≤ cap with nb buckets
__host__ __device__ constexpr size_t bucket_smem(int cap, int nb) { return (4 * (size_t)cap + nb) * sizeof(uint32_t) + 2 * (size_t)cap; }
constexpr int kMaxChunks = 64;
constexpr int kPlanBuckets = 16384;   // fine enough that config 5's densest wall stays ≤ 2048 per bucket
constexpr size_t kPlanSmem = (size_t)kPlanBuckets * (sizeof(uint32_t) + sizeof(uint8_t));

// One long tile's plan with NB depth buckets (NB = 4,096 for lists ≤ 16,384, else 16,384: fine
// enough that config 5's densest wall stays ≤ 2,048 entries per bucket).
template <int NB, int NT>
__device__ __forceinline__ void plan_tile(int tile, int n, uint32_t base, const uint32_t *__restrict__ keys,
                                          const uint32_t *__restrict__ vals, const uint8_t *__restrict__ pbits,
                                          uint32_t *__restrict__ keys2, uint32_t *__restrict__ vals2,
                                          uint32_t *__restrict__ bits2, uint32_t *__restrict__ sub_count,
                                          uint32_t *__restrict__ radix_list, uint32_t *__restrict__ chunk_list,
                                          DevScalars *__restrict__ dev, uint32_t *H, uint8_t *CH,
                                          uint32_t (*csub)[8], uint32_t *ccnt, uint32_t *cbeg, uint32_t (*red)[32]) {
    constexpr int NW = NT / 32;
    constexpr int PT = NB / NT;
    constexpr int kLogNB = NB == 16384 ? 14 : (NB == 8192 ? 13 : (NB == 4096 ? 12 : (NB == 2048 ? 11 : 10)));
    static_assert(PT >= 1 && PT * NT == NB && (1 << kLogNB) == NB, "bucket count");
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int i = tid; i < n; i += NT) {
        const uint32_t k = __ldg(keys + base + i);
        kmin = min(kmin, k);
        kmax = max(kmax, k);
    }
    for (int i = tid; i < NB; i += NT) H[i] = 0u;
    for (int i = tid; i < kMaxChunks * 8; i += NT) (&csub[0][0])[i] = 0u;
    if (tid < kMaxChunks) { ccnt[tid] = 0u; cbeg[tid] = 0xffffffffu; }
    kmin = __reduce_min_sync(kFull, kmin);
    kmax = __reduce_max_sync(kFull, kmax);
    if (lane == 0) { red[0][w] = kmin; red[1][w] = kmax; }
    __syncthreads();
    if (w == 0) {
        const uint32_t a = __reduce_min_sync(kFull, lane < NW ? red[0][lane] : 0xffffffffu);
        const uint32_t b = __reduce_max_sync(kFull, lane < NW ? red[1][lane] : 0u);
        __syncwarp();
        if (lane == 0) { red[0][0] = a; red[1][0] = b; }
    }
    __syncthreads();
    kmin = red[0][0];
    kmax = red[1][0];
    const uint32_t range = kmax - kmin;
    const int nbits = range ? 32 - __clz(range) : 0;
    const int shift = nbits > kLogNB ? nbits - kLogNB : 0;
    for (int i = tid; i < n; i += NT) atomicAdd(&H[(__ldg(keys + base + i) - kmin) >> shift], 1u);
    __syncthreads();
    uint32_t c[PT], tot = 0, cmax = 0;
#pragma unroll
    for (int j = 0; j < PT; ++j) {
        c[j] = H[tid * PT + j];
        tot += c[j];
        cmax = max(cmax, c[j]);
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    cmax = __reduce_max_sync(kFull, cmax);
    if (lane == 31) red[2][w] = incl;
    if (lane == 0) red[3][w] = cmax;
    __syncthreads();
    if (w == 0) {
        const uint32_t a = lane < NW ? red[2][lane] : 0u;
        uint32_t ia = a;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, ia, o);
            if (lane >= o) ia += y;
        }
        const uint32_t m = __reduce_max_sync(kFull, lane < NW ? red[3][lane] : 0u);
        __syncwarp();
        red[2][lane] = ia - a;
        red[3][lane] = m;
    }
    __syncthreads();
    // chunk target: a chunk holds the buckets starting in [c·tgt, (c + 1)·tgt), so it has
    // ≤ tgt + (largest bucket) ≤ kSortCap entries
    const uint32_t bmax = red[3][0];
    const uint32_t tgt = (uint32_t)kSortCap - max(bmax, (uint32_t)kMaxBucket);
    if (bmax > (uint32_t)kSortCap / 2 || (uint32_t)(n - 1) / tgt >= (uint32_t)kMaxChunks) {
        if (tid == 0) radix_list[atomicAdd(&dev->radix_count, 1u)] = (uint32_t)tile;   // degenerate: radix
        return;
    }
    uint32_t run = incl - tot + red[2][w];
#pragma unroll
    for (int j = 0; j < PT; ++j) {   // segment starts; chunk of each bucket; chunk sizes / starts
        const int bkt = tid * PT + j;
        H[bkt] = run;
        const uint32_t ch = run / tgt;
        CH[bkt] = (uint8_t)ch;
        if (c[j]) {
            atomicAdd(&ccnt[ch], c[j]);
            atomicMin(&cbeg[ch], run);
        }
        run += c[j];
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) {   // scatter into bucket order, count sub-tile entries per chunk
        const uint32_t k = __ldg(keys + base + i);
        const uint32_t bkt = (k - kmin) >> shift;
        const uint32_t pos = atomicAdd(&H[bkt], 1u);
        const uint32_t b = __ldg(pbits + base + i);
        keys2[base + pos] = k;
        vals2[base + pos] = __ldg(vals + base + i);
        bits2[base + pos] = b;
        const int ch = CH[bkt];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if ((b >> q) & 1u) atomicAdd(&csub[ch][q], 1u);
    }
    __syncthreads();
    if (tid < 8) {   // sub-list offsets of each chunk (exclusive over chunks), tile totals
        uint32_t r = 0;
        for (int ch = 0; ch < kMaxChunks; ++ch) {
            const uint32_t x = csub[ch][tid];
            csub[ch][tid] = r;
            r += x;
        }
        sub_count[8 * tile + tid] = r;
    }
    __syncthreads();
    if (tid < kMaxChunks && ccnt[tid]) {
        const unsigned x = atomicAdd(&dev->chunk_count, 1u);
        uint32_t *d = chunk_list + (size_t)12 * x;
        d[0] = (uint32_t)tile;
        d[1] = cbeg[tid];
        d[2] = ccnt[tid];
#pragma unroll
        for (int q = 0; q < 8; ++q) d[3 + q] = csub[tid][q];
    }
}

// ------------------------------------------------------------------------------------------
// CHUNKED = false: one CTA per tile, lists in (LO, CAP].  CHUNKED = true: a grid walks the chunk
// work list of the long-tile plans (parts of long tiles, each ≤ CAP entries, already bucketed by depth
// into keys2 / vals2 / bits2) and writes each part at its place in the tile's list and sub-lists.
template <int LO, int CAP, int NB, int NT, bool CHUNKED = false>
__global__ void __launch_bounds__(NT, 2048 / NT) k_tile_sort_bucket(const uint32_t *__restrict__ tile_count,
                                                         const uint32_t *__restrict__ tile_start,
                                                         const uint32_t *__restrict__ keys,
                                                         uint32_t *__restrict__ vals,
                                                         const uint8_t *__restrict__ pbits,
                                                         uint32_t *__restrict__ sub_lists,
                                                         uint32_t *__restrict__ sub_count,
                                                         uint32_t *__restrict__ radix_list,
                                                         DevScalars *__restrict__ dev, int T,
                                                         uint32_t *__restrict__ chunk_list,
                                                         uint32_t *__restrict__ ckeys,
                                                         uint32_t *__restrict__ cvals,
                                                         uint32_t *__restrict__ cbits) {
    constexpr int NW = NT / 32;
    constexpr int PT = NB / NT;
    static_assert(PT >= 1 && PT * NT == NB, "NB must be a multiple of NT");
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t red[4][32];
    __shared__ unsigned long long red64[2][33];
    __shared__ uint32_t s_desc[12];
    __shared__ uint32_t csub[CHUNKED ? 1 : kMaxChunks][8];   // the long-tile plan (plan_tile)
    __shared__ uint32_t ccnt[CHUNKED ? 1 : kMaxChunks], cbeg[CHUNKED ? 1 : kMaxChunks];
    for (int it = 0;; ++it) {
    int tile, n, off = 0, ntile;
    if (CHUNKED) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned w = atomicAdd(&dev->chunk_next, 1u);
            s_desc[0] = w < dev->chunk_count ? 1u : 0u;
            if (w < dev->chunk_count)
                for (int q = 0; q < 11; ++q) s_desc[1 + q] = chunk_list[(size_t)12 * w + q];
        }
        __syncthreads();
        if (!s_desc[0]) return;
        tile = (int)s_desc[1];
        off = (int)s_desc[2];
        n = (int)s_desc[3];
        ntile = (int)tile_count[tile];
    } else {
        if (it > 0) return;
        tile = blockIdx.x;
        n = ntile = (int)tile_count[tile];
        if (n > CAP) {   // a long list: this CTA plans its chunks (k_tile_sort_bucket<…, CHUNKED> sorts them)
            if constexpr (!CHUNKED) {
                static_assert(bucket_smem(CAP, NB) >= kPlanSmem, "the plan reuses the bucket sort's shared memory");
                const uint32_t b0 = tile_start[tile];
                if (n > kMaxChunks * (kSortCap / 2)) {   // beyond the plan's capacity: radix sort
                    if (threadIdx.x == 0) radix_list[atomicAdd(&dev->radix_count, 1u)] = (uint32_t)tile;
                } else if (n <= 16384) {
                    plan_tile<4096, NT>(tile, n, b0, keys, vals, pbits, ckeys, cvals, cbits, sub_count, radix_list,
                                        chunk_list, dev, sm, reinterpret_cast<uint8_t *>(sm + kPlanBuckets), csub,
                                        ccnt, cbeg, red);
                } else {
                    plan_tile<kPlanBuckets, NT>(tile, n, b0, keys, vals, pbits, ckeys, cvals, cbits, sub_count,
                                                radix_list, chunk_list, dev, sm,
                                                reinterpret_cast<uint8_t *>(sm + kPlanBuckets), csub, ccnt, cbeg, red);
                }
            }
            continue;
        }
        if (n <= LO) continue;
    }
    constexpr int kLogNB = NB == 8192 ? 13 : (NB == 4096 ? 12 : (NB == 2048 ? 11 : 10));
    static_assert((1 << kLogNB) == NB, "NB must be 1024 … 8192");
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t base = tile_start[tile];
    // KV2: the bucketed (key, gid) pairs interleaved, so the rank loop compares one 64-bit word
    uint32_t *K = sm, *V = sm + CAP, *H = sm + 4 * CAP;
    unsigned long long *KV2 = reinterpret_cast<unsigned long long *>(sm + 2 * CAP);
    uint8_t *B = reinterpret_cast<uint8_t *>(sm + 4 * CAP + NB), *B2 = B + CAP;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int i = tid; i < n; i += NT) {
        const uint32_t k = CHUNKED ? __ldg(ckeys + base + off + i) : __ldg(keys + base + i);
        K[i] = k;
        V[i] = CHUNKED ? __ldg(cvals + base + off + i) : __ldg(vals + base + i);
        B[i] = CHUNKED ? (uint8_t)__ldg(cbits + base + off + i) : __ldg(pbits + base + i);
        kmin = min(kmin, k);
        kmax = max(kmax, k);
    }
    for (int i = tid; i < NB; i += NT) H[i] = 0u;
    kmin = __reduce_min_sync(kFull, kmin);
    kmax = __reduce_max_sync(kFull, kmax);
    if (lane == 0) { red[0][w] = kmin; red[1][w] = kmax; }
    __syncthreads();
    if (w == 0) {
        const uint32_t a = __reduce_min_sync(kFull, lane < NW ? red[0][lane] : 0xffffffffu);
        const uint32_t b = __reduce_max_sync(kFull, lane < NW ? red[1][lane] : 0u);
        __syncwarp();
        if (lane == 0) { red[0][0] = a; red[1][0] = b; }
    }
    __syncthreads();
    kmin = red[0][0];
    kmax = red[1][0];
    const uint32_t range = kmax - kmin;
    const int nbits = range ? 32 - __clz(range) : 0;
    const int shift = nbits > kLogNB ? nbits - kLogNB : 0;
    for (int i = tid; i < n; i += NT) atomicAdd(&H[(K[i] - kmin) >> shift], 1u);
    __syncthreads();
    uint32_t cmax = 0;
    {   // exclusive scan of the NB counts: PT per thread, then a block scan of the sums
        uint32_t c[PT], tot = 0;
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            c[j] = H[tid * PT + j];
            tot += c[j];
            cmax = max(cmax, c[j]);
        }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        cmax = __reduce_max_sync(kFull, cmax);
        if (lane == 31) red[2][w] = incl;
        if (lane == 0) red[3][w] = cmax;
        __syncthreads();
        if (w == 0) {   // exclusive scan of the warps' sums, max of their largest buckets
            const uint32_t a = lane < NW ? red[2][lane] : 0u;
            uint32_t ia = a;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, ia, o);
                if (lane >= o) ia += y;
            }
            const uint32_t m = __reduce_max_sync(kFull, lane < NW ? red[3][lane] : 0u);
            __syncwarp();
            red[2][lane] = ia - a;
            red[3][lane] = m;
        }
        __syncthreads();
        uint32_t run = incl - tot + red[2][w];
        cmax = red[3][0];
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            H[tid * PT + j] = run;
            run += c[j];
        }
    }
    if (!CHUNKED && cmax > (uint32_t)kMaxBucket) {   // degenerate depth distribution → the radix kernel's list
        if (tid == 0) radix_list[atomicAdd(&dev->radix_count, 1u)] = (uint32_t)tile;
        continue;
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
        const uint32_t k = K[i];
        const uint32_t pos = atomicAdd(&H[(k - kmin) >> shift], 1u);  // H[b] becomes the segment end
        KV2[pos] = ((unsigned long long)k << 32) | V[i];
        B2[pos] = B[i];
    }
    __syncthreads();
    for (int p = tid; p < n; p += NT) {
        const unsigned long long kv = KV2[p];   // (key, gid): the order is that of the 64-bit word
        const uint32_t k = (uint32_t)(kv >> 32), v = (uint32_t)kv;
        const uint32_t b = (k - kmin) >> shift;
        const int s0 = b ? (int)H[b - 1] : 0, s1 = (int)H[b];
        int rank = 0;
        for (int j = s0; j < s1; ++j) rank += KV2[j] < kv ? 1 : 0;
        V[s0 + rank] = v;
        B[s0 + rank] = B2[p];
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) vals[base + off + i] = V[i];
    sublists_from_bits<NT>(V, B, n, sub_lists + (size_t)8 * base, sub_count + 8 * tile, red64, ntile,
                           CHUNKED ? s_desc + 4 : nullptr);
    }
}



// threads per tile CTA and depth buckets of the bucket sort (compile-time A/B: -DVTGS_SORT_NT=…)
#ifndef VTGS_SORT_NT
#define VTGS_SORT_NT 1024
#endif
#ifndef VTGS_SORT_NB
#define VTGS_SORT_NB 4096
#endif
constexpr int kSortNT = VTGS_SORT_NT, kSortNB = VTGS_SORT_NB;
constexpr int kSortCapBig = 8192;
constexpr size_t kSortSmem = 4 * kSortCap * sizeof(uint32_t) + kSortCap * sizeof(uint16_t);
constexpr size_t kSortSmemBig = 4 * kSortCapBig * sizeof(uint32_t) + kSortCapBig * sizeof(uint16_t);

static int sort_variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("VTGS_SORT");
        v = e ? atoi(e) : 1;   // 1: bucket + rank sort; 0: radix sort
    }
    return v;
}

cudaError_t launch_forward(Ctx &c, cudaStream_t s) {
    const int W = c.intr.width, H = c.intr.height;
    const int ntx = (W + kTile - 1) / kTile, nty = (H + kTile - 1) / kTile, T = ntx * nty;
    cudaError_t err;
    if ((err = cudaMemsetAsync(c.tile_count, 0, sizeof(uint32_t) * T, s))) return err;
    if ((err = cudaMemsetAsync(c.dev, 0, sizeof(DevScalars), s))) return err;
    const int64_t N = c.N;
    // projection: a capped grid (its CTAs each derive the view rotation in fp64 first); emit: one
    // Gaussian per thread, many CTAs in flight hiding the load latency
    int64_t gN64 = (N + 255) / 256;
    if (gN64 > (int64_t)1 << 30) gN64 = (int64_t)1 << 30;
    const int gE = (int)gN64;
#ifndef VTGS_PROJ_CTAS_PER_SM
#define VTGS_PROJ_CTAS_PER_SM 16
#endif
    const int64_t gcap = (int64_t)c.num_sms * VTGS_PROJ_CTAS_PER_SM;
    const int gN = (int)(gN64 < gcap ? gN64 : gcap);
    if (N > 0) {
        LaunchScope ls(&c, kProject, s);
        k_project_count<<<gN, 256, 0, s>>>(c.pos_rad, c.col_opa, N, c.view, c.intr, ntx, c.proj, c.rect, c.thr,
                                           c.tile_count);
        if ((err = cudaGetLastError())) return err;
    }
    {
        LaunchScope ls(&c, kScan, s);
        k_scan_tiles<<<1, 1024, 0, s>>>(c.tile_count, c.tile_start, c.tile_cursor, T,
                                         (unsigned long long)c.max_pairs, c.dev, c.view, c.view_copy, c.tile_flag);
    }
    if ((err = cudaGetLastError())) return err;
    if (N > 0) {
        LaunchScope ls(&c, kEmit, s);
        k_emit_pairs<<<gE, 256, 0, s>>>(c.proj, c.rect, N, ntx, c.tile_start, c.tile_cursor, c.keys, c.vals, c.pbits,
                                         c.dev);
        if ((err = cudaGetLastError())) return err;
    }
    {
        LaunchScope ls(&c, kSort, s);
        // every launch exits at once for the tiles it does not own
        if (sort_variant()) {
            // longer lists: chunked (plan_tile); flagged (degenerate) tiles: the radix kernel.
            // One launch for every list ≤ kSortCap (short and long tiles' CTAs interleave; two
            // launches split at 2,048 left each one's tail exposed: 0.143 → 0.136 ms at config 2)
            // (its CTAs of longer lists plan their depth chunks of ≤ kSortCap entries instead)
            k_tile_sort_bucket<-1, kSortCap, kSortNB, kSortNT><<<T, kSortNT, bucket_smem(kSortCap, kSortNB), s>>>(
                c.tile_count, c.tile_start, c.keys, c.vals, c.pbits, c.sub_lists, c.sub_count, c.tile_flag, c.dev, T,
                c.chunk_list, c.keys2, c.vals2, c.offs);
            // the chunks of the long lists, sorted on chip
            k_tile_sort_bucket<0, kSortCap, kSortNB, kSortNT, true><<<2 * c.num_sms, kSortNT, bucket_smem(kSortCap, kSortNB), s>>>(
                c.tile_count, c.tile_start, c.keys, c.vals, c.pbits, c.sub_lists, c.sub_count, c.tile_flag, c.dev, T,
                c.chunk_list, c.keys2, c.vals2, c.offs);
            ++c.launches;
            k_tile_sort<kSortCap, kSortCapBig, true><<<c.num_sms, kBlock, kSortSmemBig, s>>>(
                c.tile_count, c.tile_start, c.keys, c.vals, c.keys2, c.vals2, c.offs, c.rect, ntx, c.sub_lists,
                c.sub_count, c.tile_flag, c.dev);
            ++c.launches;
        } else {
            k_tile_sort<-1, kSortCap, false><<<T, kBlock, kSortSmem, s>>>(
                c.tile_count, c.tile_start, c.keys, c.vals, c.keys2, c.vals2, c.offs, c.rect, ntx, c.sub_lists,
                c.sub_count, nullptr, c.dev);
            k_tile_sort<kSortCap, kSortCapBig, true><<<T, kBlock, kSortSmemBig, s>>>(
                c.tile_count, c.tile_start, c.keys, c.vals, c.keys2, c.vals2, c.offs, c.rect, ntx, c.sub_lists,
                c.sub_count, nullptr, c.dev);
            ++c.launches;
        }
    }
    if ((err = cudaGetLastError())) return err;
    LaunchScope ls(&c, kCompFwd, s);
    return launch_composite_fwd(c, s);
}

cudaError_t forward_set_attributes() {
    cudaError_t e = cudaFuncSetAttribute(k_tile_sort<-1, kSortCap, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSortSmem);

    if (!e)
        e = cudaFuncSetAttribute(k_tile_sort_bucket<-1, kSortCap, kSortNB, kSortNT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bucket_smem(kSortCap, kSortNB));

    if (!e)
        e = cudaFuncSetAttribute(k_tile_sort_bucket<0, kSortCap, kSortNB, kSortNT, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bucket_smem(kSortCap, kSortNB));
    if (!e)
        e = cudaFuncSetAttribute(k_tile_sort<kSortCap, kSortCapBig, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSortSmemBig);
    return e;
}

}  // namespace vtgs
