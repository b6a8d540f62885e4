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
#include "vtgs_internal.cuh"

namespace vtgs {

constexpr unsigned kFull = 0xffffffffu;

struct BwdArgs {
    const float4 *proj;
    const uint2 *rect;
    const float4 *col_opa;
    const float4 *pos_rad;
    const uint32_t *tile_count;
    const uint32_t *tile_start;
    const uint32_t *sorted;
    int W, H, ntx;
    const float *color, *depth, *sil, *T_final;
    const uint32_t *last;
    const float *dC, *dD, *dS;
    const float *tC, *tD;
    const uint8_t *vis;
    float wc, wd;
    int cmode, dmode, normalize;
    const DevScalars *dev;
    const vtgs_pose *view;
    vtgs_intrinsics in;
    int64_t learn_begin, learn_end;
    uint32_t want;
    float4 *d_col_opa;
    float *d_radius;
    double *partials;
};

__device__ __forceinline__ unsigned subtile_mask_b(uint2 r, int sx, int sy) {
    const int x0 = (int)(r.x & 0xffffu) - sx, x1 = (int)(r.x >> 16) - sx;
    const int y0 = (int)(r.y & 0xffffu) - sy, y1 = (int)(r.y >> 16) - sy;
    const int cx0 = max(x0, 0), cx1 = min(x1, 7), cy0 = max(y0, 0), cy1 = min(y1, 3);
    if (cx0 > cx1 || cy0 > cy1) return 0u;
    const unsigned col = (0xffu >> (7 - cx1)) & (0xffu << cx0);
    const unsigned rows = (0xffffffffu >> (8 * (3 - cy1))) & (0xffffffffu << (8 * cy0));
    return (col * 0x01010101u) & rows;
}

__device__ __forceinline__ float sgnf(float r) { return (float)((r > 0.0f) - (r < 0.0f)); }

template <bool ATTR, bool POSE, bool LOSS>
__global__ void __launch_bounds__(kBlock) k_composite_bwd(BwdArgs p) {
    __shared__ float4 sA[kChunk];  // u, v, 9σ², −log2(e)/(2σ²)
    __shared__ float4 sB[kChunk];  // colour, opacity
    __shared__ float4 sX[kChunk];  // X_c (pose) ; .w = ±σ (−: clamped)
    __shared__ float sZ[kChunk];
    __shared__ uint2 sR[kChunk];
    __shared__ uint32_t sGid[kChunk];
    __shared__ float sAcc[ATTR ? 5 * kChunk : 1];
    __shared__ uint16_t sIdx[8][kChunk];
    __shared__ unsigned sMsk[8][kChunk];
    __shared__ PoseR P;
    __shared__ uint32_t sMax[8];
    __shared__ double sRed[8][13];

    const int tile = blockIdx.x;
    const int ty = tile / p.ntx, tx = tile - ty * p.ntx;
    const int tid = threadIdx.x, w = tid >> 5;
    const unsigned lane = lane_id();
    const int sx = tx * kTile + (w & 1) * 8, sy = ty * kTile + (w >> 1) * 4;
    const int px = sx + (lane & 7), py = sy + (lane >> 3);
    const bool inside = px < p.W && py < p.H;
    const float pxf = (float)px, pyf = (float)py;
    const int n = (int)p.tile_count[tile];
    const uint32_t start = p.tile_start[tile];
    if (POSE && tid == 0) pose_rotation(*p.view, P);

    // ---- per-pixel upstream gradient (explicit, or the fused masked-L1 prologue) ----
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, gD = 0.f, gS = 0.f, T = 1.0f;
    float r0 = 0.f, r1 = 0.f, r2 = 0.f, rz = 0.f;
    uint32_t L = 0;
    double lossv = 0.0;
    if (inside) {
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
                const float r0 = p.color[3 * pix] - p.tC[3 * pix];
                const float r1 = p.color[3 * pix + 1] - p.tC[3 * pix + 1];
                const float r2 = p.color[3 * pix + 2] - p.tC[3 * pix + 2];
                const float k = p.wc * sc;
                g0 = k * sgnf(r0); g1 = k * sgnf(r1); g2 = k * sgnf(r2);
                lossv += (double)k * ((double)fabsf(r0) + (double)fabsf(r1) + (double)fabsf(r2));
            }
            if (md) {
                const float r = p.depth[pix] - tDv;
                const float k = p.wd * sd;
                gD = k * sgnf(r);
                lossv += (double)k * (double)fabsf(r);
            }
        } else {
            if (p.dC) { g0 = p.dC[3 * pix]; g1 = p.dC[3 * pix + 1]; g2 = p.dC[3 * pix + 2]; }
            if (p.dD) gD = p.dD[pix];
            if (p.dS) gS = p.dS[pix];
        }
        T = p.T_final[pix];
        L = p.last[pix];
        // reference colour / depth of the pixel (its normalised render): the "behind"
        // accumulators are kept relative to it, so c − c̄ and z − z̄ — differences of nearly
        // equal values when view-tied layers sit on one surface — keep fp32 relative precision
        const float Sv = p.sil[pix];
        if (Sv > 0.0f) {
            const float inv = 1.0f / Sv;
            r0 = p.color[3 * pix] * inv; r1 = p.color[3 * pix + 1] * inv; r2 = p.color[3 * pix + 2] * inv;
            rz = p.depth[pix] * inv;
        }
    }
    const bool on = inside && L > 0 && (g0 != 0.f || g1 != 0.f || g2 != 0.f || gD != 0.f || gS != 0.f);
    if (!on) L = 0;
    const unsigned onmask = __ballot_sync(kFull, on);
    const uint32_t wl = __reduce_max_sync(kFull, L);
    if (lane == 0) sMax[w] = wl;
    __syncthreads();
    uint32_t nmax = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) nmax = max(nmax, sMax[i]);

    // behind-accumulators relative to the references: Xb = Σ_{j behind} w_j (x_j − x_ref) with
    // w_j = α_j T_j / T_{i+1}, and Tb = 1 − Σ w_j = Π (1 − α_j) (so x_i − x̄ = (x_i − x_ref) − Xb +
    // x_ref·Tb and 1 − S̄ = Tb, all without cancellation against x_ref)
    float Cb0 = 0.f, Cb1 = 0.f, Cb2 = 0.f, Db = 0.f, Tb = 1.0f;
    float h0 = 0.f, h1 = 0.f, h2 = 0.f;
    float K00 = 0.f, K01 = 0.f, K02 = 0.f, K10 = 0.f, K11 = 0.f, K12 = 0.f, K20 = 0.f, K21 = 0.f, K22 = 0.f;
    const float fmean = 0.5f * (p.in.fx + p.in.fy);

    for (int cb = nmax > 0 ? (int)((nmax - 1) / kChunk) * kChunk : -kChunk; cb >= 0; cb -= kChunk) {
        const int m = min(kChunk, n - cb);
        if (tid < m) {
            const uint32_t g = p.sorted[start + cb + tid];
            const float4 pr = p.proj[g];
            const float s = fabsf(pr.w);
            const float s2 = __fmul_rn(s, s);
            sA[tid] = make_float4(pr.x, pr.y, __fmul_rn(9.0f, s2), __fdividef(-0.5f * kLog2e, s2));
            sB[tid] = p.col_opa[g];
            sZ[tid] = pr.z;
            sR[tid] = p.rect[g];
            sGid[tid] = g;
            if (POSE) {
                float xc[3];
                view_transform(P.R, P.t, p.pos_rad[g], xc);
                sX[tid] = make_float4(xc[0], xc[1], xc[2], pr.w);
            } else {
                sX[tid] = make_float4(0.f, 0.f, 0.f, pr.w);
            }
            if (ATTR) {
#pragma unroll
                for (int q = 0; q < 5; ++q) sAcc[q * kChunk + tid] = 0.0f;
            }
        }
        __syncthreads();
        if (wl > (uint32_t)cb) {
            int cnt = 0;
            for (int j = 0; j < m; j += 32) {
                const int e = j + (int)lane;
                const unsigned msk = (e < m && (uint32_t)(cb + e) < wl) ? subtile_mask_b(sR[e], sx, sy) & onmask : 0u;
                const unsigned b = __ballot_sync(kFull, msk != 0u);
                if (msk) {
                    const int pos = cnt + __popc(b & lanemask_lt());
                    sIdx[w][pos] = (uint16_t)e;
                    sMsk[w][pos] = msk;
                }
                cnt += __popc(b);
            }
            __syncwarp();
            for (int k = cnt - 1; k >= 0; --k) {
                const int e = sIdx[w][k];
                const unsigned msk = sMsk[w][k];
                bool proc = false;
                float dc0 = 0.f, dc1 = 0.f, dc2 = 0.f, dop = 0.f, dsg = 0.f;
                if (((msk >> lane) & 1u) && (uint32_t)(cb + e) < L) {
                    const float4 A = sA[e];
                    const float dx = __fsub_rn(pxf, A.x), dy = __fsub_rn(pyf, A.y);
                    const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
                    if (d2 <= A.z) {
                        const float4 B = sB[e];
                        const float wgt = fast_exp2(d2 * A.w);
                        const float raw = __fmul_rn(B.w, wgt);
                        const bool aclamp = raw > kAlphaMax;
                        const float a = aclamp ? kAlphaMax : raw;
                        if (a >= 1.0f / 255.0f) {
                            proc = true;
                            const float z = sZ[e];
                            const float Ti = __fdividef(T, 1.0f - a);
                            const float om = a * Ti;
                            dc0 = g0 * om; dc1 = g1 * om; dc2 = g2 * om;
                            const float e0 = B.x - r0, e1 = B.y - r1, e2 = B.z - r2, ez = z - rz;
                            const float fpart = g0 * (e0 - Cb0 + r0 * Tb) + g1 * (e1 - Cb1 + r1 * Tb) +
                                                g2 * (e2 - Cb2 + r2 * Tb) + gD * (ez - Db + rz * Tb) + gS * Tb;
                            const float dA = Ti * fpart;
                            const float oma = 1.0f - a;
                            Cb0 = a * e0 + oma * Cb0;
                            Cb1 = a * e1 + oma * Cb1;
                            Cb2 = a * e2 + oma * Cb2;
                            Db = a * ez + oma * Db;
                            Tb = oma * Tb;
                            T = Ti;
                            float gww = 0.f;
                            if (!aclamp) {
                                dop = dA * wgt;
                                gww = dA * B.w * wgt;  // dL/dw · w
                            }
                            const float4 X = sX[e];
                            const float s = fabsf(X.w);
                            const float inv_s2 = __fdividef(1.0f, s * s);
                            const float du = gww * dx * inv_s2;   // ∂w/∂u = w (x − u) / σ²
                            const float dv = gww * dy * inv_s2;
                            dsg = gww * d2 * inv_s2 / s;          // ∂w/∂σ = w d² / σ³
                            if (POSE) {
                                const float iz = 1.0f / z;
                                float dzt = gD * om - (du * (A.x - p.in.cx) + dv * (A.y - p.in.cy)) * iz;
                                if (X.w > 0.f) dzt -= dsg * s * iz;  // ∂σ/∂z = −σ/z (unclamped)
                                const float gx = du * p.in.fx * iz, gy = dv * p.in.fy * iz, gz = dzt;
                                h0 += gx; h1 += gy; h2 += gz;
                                K00 = fmaf(X.x, gx, K00); K01 = fmaf(X.x, gy, K01); K02 = fmaf(X.x, gz, K02);
                                K10 = fmaf(X.y, gx, K10); K11 = fmaf(X.y, gy, K11); K12 = fmaf(X.y, gz, K12);
                                K20 = fmaf(X.z, gx, K20); K21 = fmaf(X.z, gy, K21); K22 = fmaf(X.z, gz, K22);
                            }
                        }
                    }
                }
                if (ATTR) {
                    const unsigned pm = __ballot_sync(kFull, proc);
                    if (pm) {
                        if (__popc(pm) == 1) {
                            if (proc) {
                                atomicAdd(&sAcc[0 * kChunk + e], dc0);
                                atomicAdd(&sAcc[1 * kChunk + e], dc1);
                                atomicAdd(&sAcc[2 * kChunk + e], dc2);
                                atomicAdd(&sAcc[3 * kChunk + e], dop);
                                atomicAdd(&sAcc[4 * kChunk + e], dsg);
                            }
                        } else {
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) {
                                dc0 += __shfl_xor_sync(kFull, dc0, o);
                                dc1 += __shfl_xor_sync(kFull, dc1, o);
                                dc2 += __shfl_xor_sync(kFull, dc2, o);
                                dop += __shfl_xor_sync(kFull, dop, o);
                                dsg += __shfl_xor_sync(kFull, dsg, o);
                            }
                            if (lane == 0) {
                                atomicAdd(&sAcc[0 * kChunk + e], dc0);
                                atomicAdd(&sAcc[1 * kChunk + e], dc1);
                                atomicAdd(&sAcc[2 * kChunk + e], dc2);
                                atomicAdd(&sAcc[3 * kChunk + e], dop);
                                atomicAdd(&sAcc[4 * kChunk + e], dsg);
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (ATTR && tid < m) {
            const uint32_t g = sGid[tid];
            if ((int64_t)g >= p.learn_begin && (int64_t)g < p.learn_end) {
                const float a0 = sAcc[tid], a1 = sAcc[kChunk + tid], a2 = sAcc[2 * kChunk + tid];
                const float a3 = sAcc[3 * kChunk + tid], a4 = sAcc[4 * kChunk + tid];
                const bool wc = p.want & VTGS_GRAD_COLOR, wo = p.want & VTGS_GRAD_OPACITY;
                if ((wc && (a0 != 0.f || a1 != 0.f || a2 != 0.f)) || (wo && a3 != 0.f))
                    atomicAdd(&p.d_col_opa[g], make_float4(wc ? a0 : 0.f, wc ? a1 : 0.f, wc ? a2 : 0.f, wo ? a3 : 0.f));
                const float4 X = sX[tid];
                if ((p.want & VTGS_GRAD_RADIUS) && X.w > 0.f && a4 != 0.f)
                    atomicAdd(&p.d_radius[g], a4 * fmean / sZ[tid]);  // ∂σ/∂r = f/z
            }
        }
        if (ATTR) __syncthreads();
    }

    if (POSE || LOSS) {
        double v[13] = {h0, h1, h2, K00, K01, K02, K10, K11, K12, K20, K21, K22, lossv};
#pragma unroll
        for (int q = 0; q < 13; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(kFull, v[q], o);
        }
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 13; ++q) sRed[w][q] = v[q];
        __syncthreads();
        if (tid < 13) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) s += sRed[i][tid];
            p.partials[(size_t)tile * 16 + tid] = s;
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
    cc = __reduce_add_sync(kFull, cc);
    cd = __reduce_add_sync(kFull, cd);
    if (lane_id() == 0) {
        atomicAdd(&dev->count_c, cc);
        atomicAdd(&dev->count_d, cd);
    }
}

// Fixed-order sum of the per-tile partials, then the rotation chain (DESIGN.md §3 step 11):
//   dL/dt = −R Σg,  dL/dR = R Σ X_c gᵀ,  dL/dq̂ = Σ_ab (dL/dR)_ab ∂R_ab/∂q̂,
//   dL/dq = (dL/dq̂ − q̂ (q̂·dL/dq̂)) / |q|.
__global__ void __launch_bounds__(256) k_pose_finalize(const double *__restrict__ partials, int T,
                                                       const vtgs_pose *__restrict__ view,
                                                       float *__restrict__ d_pose,
                                                       float *__restrict__ loss_out) {
    __shared__ double red[256][13];
    const int tid = threadIdx.x;
    double acc[13];
#pragma unroll
    for (int q = 0; q < 13; ++q) acc[q] = 0.0;
    for (int t = tid; t < T; t += 256)
#pragma unroll
        for (int q = 0; q < 13; ++q) acc[q] += partials[(size_t)t * 16 + q];
#pragma unroll
    for (int q = 0; q < 13; ++q) red[tid][q] = acc[q];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (tid < s)
#pragma unroll
            for (int q = 0; q < 13; ++q) red[tid][q] += red[tid + s][q];
        __syncthreads();
    }
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

template <bool A, bool P, bool L>
static void launch_bwd_t(const BwdArgs &a, int T, cudaStream_t s) {
    k_composite_bwd<A, P, L><<<T, kBlock, 0, s>>>(a);
}

cudaError_t launch_backward(Ctx &c, const float *dC, const float *dD, const float *dS,
                            const vtgs_l1_loss *loss, uint32_t want, int64_t learn_begin,
                            int64_t learn_end, float4 *d_col_opa, float *d_radius, float *d_pose,
                            float *loss_out, cudaStream_t s) {
    const int W = c.intr.width, H = c.intr.height;
    const int ntx = (W + kTile - 1) / kTile, nty = (H + kTile - 1) / kTile, T = ntx * nty;
    cudaError_t err;
    BwdArgs a{};
    a.proj = c.proj; a.rect = c.rect; a.col_opa = c.col_opa; a.pos_rad = c.pos_rad;
    a.tile_count = c.tile_count; a.tile_start = c.tile_start; a.sorted = c.vals;
    a.W = W; a.H = H; a.ntx = ntx;
    a.color = c.color; a.depth = c.depth; a.sil = c.sil; a.T_final = c.T_final; a.last = c.last;
    a.dC = dC; a.dD = dD; a.dS = dS;
    a.dev = c.dev; a.view = c.view_copy; a.in = c.intr;
    a.learn_begin = learn_begin; a.learn_end = learn_end; a.want = want;
    a.d_col_opa = d_col_opa; a.d_radius = d_radius; a.partials = c.partials;
    const bool L = loss != nullptr;
    if (L) {
        a.tC = loss->target_rgb; a.tD = loss->target_depth; a.vis = loss->vis_mask;
        a.wc = loss->w_color; a.wd = loss->w_depth;
        a.cmode = loss->color_mask_mode; a.dmode = loss->depth_mask_mode; a.normalize = loss->normalize;
        if (a.normalize) {
            if ((err = cudaMemsetAsync(&c.dev->count_c, 0, 2 * sizeof(unsigned int), s))) return err;
            int g = (W * H + 255) / 256;
            if (g > c.num_sms * 8) g = c.num_sms * 8;
            LaunchScope ls(&c, kL1Count, s);
            k_l1_count<<<g, 256, 0, s>>>(c.sil, a.tD, a.vis, W * H, a.cmode, a.dmode, c.dev);
            if ((err = cudaGetLastError())) return err;
        }
    }
    const bool A = (want & (VTGS_GRAD_COLOR | VTGS_GRAD_OPACITY | VTGS_GRAD_RADIUS)) != 0;
    const bool P = (want & VTGS_GRAD_POSE) != 0 && d_pose != nullptr;
    const int sel = (A ? 4 : 0) | (P ? 2 : 0) | (L ? 1 : 0);
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
    if ((err = cudaGetLastError())) return err;
    if (P || (L && loss_out)) {
        LaunchScope ls(&c, kFinalize, s);
        k_pose_finalize<<<1, 256, 0, s>>>(c.partials, T, c.view_copy, P ? d_pose : nullptr, L ? loss_out : nullptr);
        if ((err = cudaGetLastError())) return err;
    }
    return cudaSuccess;
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
