// SSIM term of the mapping objective Eq. 2 — PAPER.md:195-201 ("τ L_S(V_i, V_i') ... L_S is the
// SSIM loss"), τ = 0.2; window / constants per DESIGN.md reading R24 (11×11
// Gaussian, σ = 1.5, C1 = 0.01², C2 = 0.03², per channel, zero padding, L_S = 1 − mean SSIM).
//
// Two separable stencil passes over shared-memory tiles (64×16 output pixels per CTA of 256
// threads, 5-pixel halo), one colour channel per CTA (grid z).  Both passes are register-blocked: in the
// horizontal pass a thread produces 8 consecutive outputs of a row from 18 staged inputs, in the
// vertical pass 4 consecutive outputs of a column from 14 staged row sums.
//   K_ssim_moments: 11-tap sums of x, y, x², y², xy → SSIM_p and the three per-pixel chain
//     factors a = dL/dS·∂S/∂μx, b = dL/dS·∂S/∂E[x²], c = dL/dS·∂S/∂E[xy] (9 floats / pixel to
//     scratch) and a per-CTA partial of Σ SSIM; the last CTA to finish (ticket) sums the partials
//     in a fixed order → loss = τ (1 − Σ S / 3HW) (no separate finalize launch);
//   K_ssim_grad: the adjoint stencil (the window is symmetric, zero padding ⇒ the same filter)
//     dL/dx_q = (G⋆a)_q + 2 x_q (G⋆b)_q + y_q (G⋆c)_q, ACCUMULATED into d_color;
#include "vtgs_internal.cuh"

namespace vtgs {

constexpr int kSsTX = 64, kSsTY = 16, kSsR = 5, kSsThreads = 256;
constexpr int kSsW = kSsTX + 2 * kSsR, kSsH = kSsTY + 2 * kSsR;   // 74 × 26 input tile
constexpr int kSsWp = kSsW + 1;    // staged row stride (odd: the row-per-lane reads spread over banks)
constexpr int kHSeg = 8;                                          // horizontal outputs per thread
constexpr int kVSeg = 4;                                          // vertical outputs per thread
constexpr int kHTasks = kSsH * (kSsTX / kHSeg);                   // 208 (row, segment) tasks
__constant__ float c_ssim_w[11];
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

// Horizontal-pass ownership: lane-consecutive tasks take consecutive ROWS of one 8-column segment
// (row = t mod 26), and the row sums are stored XOR-swizzled (column ^ row): a warp's stores of
// one output column hit 32 distinct banks, and the vertical pass (consecutive columns of one row)
// reads through the same swizzle conflict-free.
__device__ __forceinline__ int hm_col(int r, int q) { return q ^ (r & 31); }

// Stage one channel of NQ planes (tile + halo, zero outside the image) into s[q][r][c].
template <int NQ>
__device__ __forceinline__ void ss_load(float (*s)[kSsH][kSsWp], const float *const *src, int c, size_t stride_q,
                                        bool interleaved, int ox, int oy, int W, int H) {
    // fully unrolled (≤ 8 iterations): every load of the tile is in flight at once (the rolled
    // loop waited on each iteration's loads — long-scoreboard stalls in the adjoint kernel)
#pragma unroll
    for (int i = threadIdx.x; i < kSsH * kSsW; i += kSsThreads) {
        const int r = i / kSsW, q = i - r * kSsW;
        const int gx = ox + q - kSsR, gy = oy + r - kSsR;
        const bool ok = gx >= 0 && gy >= 0 && gx < W && gy < H;
        const size_t p = (size_t)gy * W + gx;
#pragma unroll
        for (int m = 0; m < NQ; ++m)
            s[m][r][q] = ok ? __ldg(src[m] + (interleaved ? p * 3 + c : (size_t)c * stride_q + p)) : 0.f;
    }
}

__global__ void __launch_bounds__(kSsThreads, 4) k_ssim_moments(const float *__restrict__ x,
                                                            const float *__restrict__ y, int W, int H,
                                                            float dLdS, float *__restrict__ abc,
                                                            double *__restrict__ partials, double npx3, float tau,
                                                            float *__restrict__ loss_out,
                                                            unsigned int *__restrict__ ticket) {
    __shared__ float sin[2][kSsH][kSsWp];
    __shared__ float hm[5][kSsH][kSsTX];
    __shared__ double red[kSsThreads / 32];
    __shared__ bool last;
    const int ox = blockIdx.x * kSsTX, oy = blockIdx.y * kSsTY;
    const size_t npx = (size_t)W * H;
    const float *srcs[2] = {x, y};
    // vertical-pass ownership: column vc, rows vr .. vr + kVSeg − 1
    const int vc = threadIdx.x & (kSsTX - 1), vr = (threadIdx.x / kSsTX) * kVSeg;
    const int hr = threadIdx.x % kSsH, hq0 = (threadIdx.x / kSsH) * kHSeg;   // horizontal task
    double ssum = 0.0;
    {   // one channel per CTA (blockIdx.z): 3× the CTAs, a smaller last wave
        const int c = blockIdx.z;
        ss_load<2>(sin, srcs, c, 0, true, ox, oy, W, H);
        __syncthreads();
        if (threadIdx.x < kHTasks) {   // horizontal pass: 8 consecutive outputs of one row
            float a[kHSeg + 10], b[kHSeg + 10];
#pragma unroll
            for (int k = 0; k < kHSeg + 10; ++k) { a[k] = sin[0][hr][hq0 + k]; b[k] = sin[1][hr][hq0 + k]; }
#pragma unroll
            for (int o = 0; o < kHSeg; ++o) {
                float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
                for (int k = 0; k < 11; ++k) {
                    const float w = c_ssim_w[k], u = a[o + k], v = b[o + k];
                    m0 = fmaf(w, u, m0);
                    m1 = fmaf(w, v, m1);
                    m2 = fmaf(w, u * u, m2);
                    m3 = fmaf(w, v * v, m3);
                    m4 = fmaf(w, u * v, m4);
                }
                const int q = hm_col(hr, hq0 + o);
                hm[0][hr][q] = m0; hm[1][hr][q] = m1; hm[2][hr][q] = m2;
                hm[3][hr][q] = m3; hm[4][hr][q] = m4;
            }
        }
        __syncthreads();
        float acc[5][kVSeg];
#pragma unroll
        for (int m = 0; m < 5; ++m) {
            float col[kVSeg + 10];
#pragma unroll
            for (int k = 0; k < kVSeg + 10; ++k) col[k] = hm[m][vr + k][hm_col(vr + k, vc)];
#pragma unroll
            for (int o = 0; o < kVSeg; ++o) {
                float s = 0.f;
#pragma unroll
                for (int k = 0; k < 11; ++k) s = fmaf(c_ssim_w[k], col[o + k], s);
                acc[m][o] = s;
            }
        }
#pragma unroll
        for (int o = 0; o < kVSeg; ++o) {
            const int px = ox + vc, py = oy + vr + o;
            if (px < W && py < H) {
                const float mx = acc[0][o], my = acc[1][o], exx = acc[2][o], eyy = acc[3][o], exy = acc[4][o];
                const float A1 = 2.f * mx * my + kC1, A2 = 2.f * (exy - mx * my) + kC2;
                const float B1 = mx * mx + my * my + kC1, B2 = (exx - mx * mx) + (eyy - my * my) + kC2;
                // one approximate reciprocal per factor instead of seven IEEE divisions per pixel
                const float iA1 = rcp_approx(A1), iA2 = rcp_approx(A2), iB1 = rcp_approx(B1), iB2 = rcp_approx(B2);
                const float S = (A1 * A2) * (iB1 * iB2);
                ssum += (double)S;
                const float k = dLdS * S;
                const size_t p = (size_t)py * W + px;
                abc[(0 * 3 + c) * npx + p] = k * (2.f * my * (iA1 - iA2) + 2.f * mx * (iB2 - iB1));
                abc[(1 * 3 + c) * npx + p] = -k * iB2;
                abc[(2 * 3 + c) * npx + p] = 2.f * k * iA2;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ssum;
    __syncthreads();
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < kSsThreads / 32; ++i) t += red[i];
        partials[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
        last = false;
        if (loss_out) {   // the last CTA to finish sums the partials (no finalize launch)
            __threadfence();
            last = atomicAdd(ticket, 1u) == (unsigned)nblk - 1u;
        }
    }
    __syncthreads();
    if (last) {   // fixed order: strided per-thread sums, then a tree (deterministic)
        __threadfence();
        double *tree = reinterpret_cast<double *>(&hm[0][0][0]);   // the row sums are dead now
        double t = 0.0;
        for (int i = threadIdx.x; i < nblk; i += kSsThreads) t += __ldcg(partials + i);
        tree[threadIdx.x] = t;
        __syncthreads();
        for (int o = kSsThreads / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) tree[threadIdx.x] += tree[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            *loss_out = (float)((double)tau * (1.0 - tree[0] / npx3));
            *ticket = 0u;
        }
    }
}

__global__ void __launch_bounds__(kSsThreads) k_ssim_grad(const float *__restrict__ x, const float *__restrict__ y,
                                                         int W, int H, const float *__restrict__ abc,
                                                         float *__restrict__ d_color) {
    __shared__ float sa[3][kSsH][kSsWp];
    __shared__ float hm[3][kSsH][kSsTX];
    const int ox = blockIdx.x * kSsTX, oy = blockIdx.y * kSsTY;
    const size_t npx = (size_t)W * H;
    const float *srcs[3] = {abc, abc + 3 * npx, abc + 6 * npx};
    const int vc = threadIdx.x & (kSsTX - 1), vr = (threadIdx.x / kSsTX) * kVSeg;
    const int hr = threadIdx.x % kSsH, hq0 = (threadIdx.x / kSsH) * kHSeg;
    {   // one channel per CTA (blockIdx.z): 3× the CTAs, a smaller last wave
        const int c = blockIdx.z;
        ss_load<3>(sa, srcs, c, npx, false, ox, oy, W, H);
        __syncthreads();
        if (threadIdx.x < kHTasks) {
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                float a[kHSeg + 10];
#pragma unroll
                for (int k = 0; k < kHSeg + 10; ++k) a[k] = sa[m][hr][hq0 + k];
#pragma unroll
                for (int o = 0; o < kHSeg; ++o) {
                    float s = 0.f;
#pragma unroll
                    for (int k = 0; k < 11; ++k) s = fmaf(c_ssim_w[k], a[o + k], s);
                    hm[m][hr][hm_col(hr, hq0 + o)] = s;
                }
            }
        }
        __syncthreads();
        float g[3][kVSeg];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            float col[kVSeg + 10];
#pragma unroll
            for (int k = 0; k < kVSeg + 10; ++k) col[k] = hm[m][vr + k][hm_col(vr + k, vc)];
#pragma unroll
            for (int o = 0; o < kVSeg; ++o) {
                float s = 0.f;
#pragma unroll
                for (int k = 0; k < 11; ++k) s = fmaf(c_ssim_w[k], col[o + k], s);
                g[m][o] = s;
            }
        }
#pragma unroll
        for (int o = 0; o < kVSeg; ++o) {
            const int px = ox + vc, py = oy + vr + o;
            if (px < W && py < H) {
                const size_t q = ((size_t)py * W + px) * 3 + c;
                d_color[q] += g[0][o] + 2.f * __ldg(x + q) * g[1][o] + __ldg(y + q) * g[2][o];
            }
        }
        __syncthreads();
    }
}

cudaError_t ssim_set_constants() {
    double g[11], s = 0.0;
    for (int i = 0; i < 11; ++i) {
        g[i] = exp(-((double)(i - 5) * (i - 5)) / (2.0 * 1.5 * 1.5));
        s += g[i];
    }
    float w[11];
    for (int i = 0; i < 11; ++i) w[i] = (float)(g[i] / s);
    return cudaMemcpyToSymbol(c_ssim_w, w, sizeof(w));
}

cudaError_t launch_ssim(Ctx &c, const float *color, const float *target, int W, int H, float tau, float *d_color,
                        float *loss_out, cudaStream_t s) {
    const dim3 grid((W + kSsTX - 1) / kSsTX, (H + kSsTY - 1) / kSsTY, 3);
    const double n3 = 3.0 * (double)W * H;
    const float dLdS = (float)(-(double)tau / n3);
    cudaError_t e;
    {
        LaunchScope ls(&c, kSsim, s);
        k_ssim_moments<<<grid, kSsThreads, 0, s>>>(color, target, W, H, dLdS, c.ssim_abc, c.ssim_partials, n3, tau,
                                                   loss_out, &c.dev->ssim_ticket);
        if ((e = cudaGetLastError())) return e;
    }
    if (d_color) {
        LaunchScope ls(&c, kSsim, s);
        k_ssim_grad<<<grid, kSsThreads, 0, s>>>(color, target, W, H, c.ssim_abc, d_color);
        if ((e = cudaGetLastError())) return e;
    }
    return cudaSuccess;
}

}  // namespace vtgs
