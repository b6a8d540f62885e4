// SSIM term of the mapping objective Eq. 2 — PAPER.md:195-201 ("τ L_S(V_i, V_i') ... L_S is the
// SSIM loss"), τ = 0.2; window / constants per DESIGN.md reading R24 (11×11
// Gaussian, σ = 1.5, C1 = 0.01², C2 = 0.03², per channel, zero padding, L_S = 1 − mean SSIM).
//
// Two separable stencil passes over shared-memory tiles (32×8 output pixels per CTA, 5-pixel
// halo), one thread per output pixel, the 3 channels in turn:
//   K_ssim_moments: horizontal then vertical 11-tap sums of x, y, x², y², xy → SSIM_p and the
//     three per-pixel chain factors a = dL/dS·∂S/∂μx, b = dL/dS·∂S/∂E[x²], c = dL/dS·∂S/∂E[xy]
//     (9 floats / pixel to scratch) and a per-CTA partial of Σ SSIM;
//   K_ssim_grad: the adjoint stencil (the window is symmetric, zero padding ⇒ the same filter)
//     dL/dx_q = (G⋆a)_q + 2 x_q (G⋆b)_q + y_q (G⋆c)_q, ACCUMULATED into d_color;
//   K_ssim_finalize: fixed-order sum of the partials → loss = τ (1 − Σ S / 3HW).
#include "vtgs_internal.cuh"

namespace vtgs {

constexpr int kSsTX = 32, kSsTY = 8, kSsR = 5;
constexpr int kSsW = kSsTX + 2 * kSsR, kSsH = kSsTY + 2 * kSsR;  // 42 × 18 input tile
__constant__ float c_ssim_w[11];
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

__global__ void __launch_bounds__(kSsTX * kSsTY) k_ssim_moments(const float *__restrict__ x,
                                                               const float *__restrict__ y, int W, int H,
                                                               float dLdS, float *__restrict__ abc,
                                                               double *__restrict__ partials) {
    __shared__ float sx[kSsH][kSsW], sy[kSsH][kSsW];
    __shared__ float hm[5][kSsH][kSsTX];
    __shared__ double red[kSsTX * kSsTY / 32];
    const int tx = threadIdx.x & (kSsTX - 1), ty = threadIdx.x / kSsTX;
    const int ox = blockIdx.x * kSsTX, oy = blockIdx.y * kSsTY;
    const int px = ox + tx, py = oy + ty;
    const bool in = px < W && py < H;
    const size_t npx = (size_t)W * H;
    double ssum = 0.0;
    for (int c = 0; c < 3; ++c) {
        for (int i = threadIdx.x; i < kSsH * kSsW; i += kSsTX * kSsTY) {
            const int r = i / kSsW, q = i - r * kSsW;
            const int gx = ox + q - kSsR, gy = oy + r - kSsR;
            const bool ok = gx >= 0 && gy >= 0 && gx < W && gy < H;   // zero padding
            const size_t g = ((size_t)gy * W + gx) * 3 + c;
            sx[r][q] = ok ? __ldg(x + g) : 0.f;
            sy[r][q] = ok ? __ldg(y + g) : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kSsH * kSsTX; i += kSsTX * kSsTY) {   // horizontal pass
            const int r = i / kSsTX, q = i - r * kSsTX;
            float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                const float w = c_ssim_w[k], a = sx[r][q + k], b = sy[r][q + k];
                m0 = fmaf(w, a, m0);
                m1 = fmaf(w, b, m1);
                m2 = fmaf(w, a * a, m2);
                m3 = fmaf(w, b * b, m3);
                m4 = fmaf(w, a * b, m4);
            }
            hm[0][r][q] = m0; hm[1][r][q] = m1; hm[2][r][q] = m2; hm[3][r][q] = m3; hm[4][r][q] = m4;
        }
        __syncthreads();
        float mx = 0.f, my = 0.f, exx = 0.f, eyy = 0.f, exy = 0.f;   // vertical pass
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const float w = c_ssim_w[k];
            mx = fmaf(w, hm[0][ty + k][tx], mx);
            my = fmaf(w, hm[1][ty + k][tx], my);
            exx = fmaf(w, hm[2][ty + k][tx], exx);
            eyy = fmaf(w, hm[3][ty + k][tx], eyy);
            exy = fmaf(w, hm[4][ty + k][tx], exy);
        }
        if (in) {
            const float A1 = 2.f * mx * my + kC1, A2 = 2.f * (exy - mx * my) + kC2;
            const float B1 = mx * mx + my * my + kC1, B2 = (exx - mx * mx) + (eyy - my * my) + kC2;
            const float S = (A1 * A2) / (B1 * B2);
            ssum += (double)S;
            const float k = dLdS * S;
            const size_t p = (size_t)py * W + px;
            abc[(0 * 3 + c) * npx + p] = k * (2.f * my / A1 - 2.f * my / A2 - 2.f * mx / B1 + 2.f * mx / B2);
            abc[(1 * 3 + c) * npx + p] = -k / B2;
            abc[(2 * 3 + c) * npx + p] = 2.f * k / A2;
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ssum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < kSsTX * kSsTY / 32; ++i) t += red[i];
        partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kSsTX * kSsTY) k_ssim_grad(const float *__restrict__ x, const float *__restrict__ y,
                                                            int W, int H, const float *__restrict__ abc,
                                                            float *__restrict__ d_color) {
    __shared__ float sa[3][kSsH][kSsW];
    __shared__ float hm[3][kSsH][kSsTX];
    const int tx = threadIdx.x & (kSsTX - 1), ty = threadIdx.x / kSsTX;
    const int ox = blockIdx.x * kSsTX, oy = blockIdx.y * kSsTY;
    const int px = ox + tx, py = oy + ty;
    const bool in = px < W && py < H;
    const size_t npx = (size_t)W * H;
    for (int c = 0; c < 3; ++c) {
        for (int i = threadIdx.x; i < kSsH * kSsW; i += kSsTX * kSsTY) {
            const int r = i / kSsW, q = i - r * kSsW;
            const int gx = ox + q - kSsR, gy = oy + r - kSsR;
            const bool ok = gx >= 0 && gy >= 0 && gx < W && gy < H;
            const size_t g = (size_t)gy * W + gx;
#pragma unroll
            for (int m = 0; m < 3; ++m) sa[m][r][q] = ok ? __ldg(abc + (m * 3 + c) * npx + g) : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kSsH * kSsTX; i += kSsTX * kSsTY) {
            const int r = i / kSsTX, q = i - r * kSsTX;
            float m0 = 0.f, m1 = 0.f, m2 = 0.f;
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                const float w = c_ssim_w[k];
                m0 = fmaf(w, sa[0][r][q + k], m0);
                m1 = fmaf(w, sa[1][r][q + k], m1);
                m2 = fmaf(w, sa[2][r][q + k], m2);
            }
            hm[0][r][q] = m0; hm[1][r][q] = m1; hm[2][r][q] = m2;
        }
        __syncthreads();
        float ga = 0.f, gb = 0.f, gc = 0.f;
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const float w = c_ssim_w[k];
            ga = fmaf(w, hm[0][ty + k][tx], ga);
            gb = fmaf(w, hm[1][ty + k][tx], gb);
            gc = fmaf(w, hm[2][ty + k][tx], gc);
        }
        if (in) {
            const size_t g = ((size_t)py * W + px) * 3 + c;
            d_color[g] += ga + 2.f * __ldg(x + g) * gb + __ldg(y + g) * gc;
        }
        __syncthreads();
    }
}

__global__ void k_ssim_finalize(const double *__restrict__ partials, int n, double npx3, float tau,
                                float *__restrict__ loss_out) {
    __shared__ double red[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) s += partials[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss_out = (float)((double)tau * (1.0 - red[0] / npx3));
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
    const dim3 grid((W + kSsTX - 1) / kSsTX, (H + kSsTY - 1) / kSsTY);
    const double n3 = 3.0 * (double)W * H;
    const float dLdS = (float)(-(double)tau / n3);
    cudaError_t e;
    {
        LaunchScope ls(&c, kSsim, s);
        k_ssim_moments<<<grid, kSsTX * kSsTY, 0, s>>>(color, target, W, H, dLdS, c.ssim_abc, c.ssim_partials);
        if ((e = cudaGetLastError())) return e;
    }
    if (d_color) {
        LaunchScope ls(&c, kSsim, s);
        k_ssim_grad<<<grid, kSsTX * kSsTY, 0, s>>>(color, target, W, H, c.ssim_abc, d_color);
        if ((e = cudaGetLastError())) return e;
    }
    if (loss_out) {
        LaunchScope ls(&c, kSsim, s);
        k_ssim_finalize<<<1, 256, 0, s>>>(c.ssim_partials, (int)(grid.x * grid.y), n3, tau, loss_out);
        if ((e = cudaGetLastError())) return e;
    }
    return cudaSuccess;
}

}  // namespace vtgs
