// (1) Instantiation of view-tied Gaussians — PAPER.md:110, :119 (§3.1-3.2)
// (Supp. A, r = D_GT / f), SPEC.md:59-67 (back_project), :434-442 (init_gaussians).
//
// One thread per keyframe pixel; HBM-bound (reads 16 B depth+rgb(+4 B opacity), writes 32 B).
// The keyframe rotation is computed once per CTA in fp64 (pose_rotation) and shared.
#include "vtgs_internal.cuh"

namespace vtgs {

__global__ void __launch_bounds__(256) k_instantiate(const float *__restrict__ depth,
                                                     const float *__restrict__ rgb,
                                                     const vtgs_pose *__restrict__ poses, int HW,
                                                     int W, vtgs_intrinsics in,
                                                     const float *__restrict__ opacity,
                                                     float opacity_default,
                                                     float4 *__restrict__ pos_rad,
                                                     float4 *__restrict__ col_opa,
                                                     unsigned long long *__restrict__ n_valid) {
    const int k = blockIdx.y;  // keyframe
    __shared__ PoseR P;
    if (threadIdx.x == 0) pose_rotation(poses[k], P);
    __syncthreads();
    const float fmean = __fmul_rn(0.5f, __fadd_rn(in.fx, in.fy));
    unsigned cnt = 0;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += gridDim.x * blockDim.x) {
        const int64_t g = (int64_t)k * HW + p;
        const float d = depth[g];
        if (!(d > 0.0f) || !isfinite(d)) {
            pos_rad[g] = make_float4(0.f, 0.f, 0.f, 0.f);
            col_opa[g] = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
        ++cnt;
        const int y = p / W, x = p - y * W;
        // X_c = ((x − cx)·d / fx, (y − cy)·d / fy, d)
        const float X0 = __fdiv_rn(__fmul_rn(__fsub_rn((float)x, in.cx), d), in.fx);
        const float X1 = __fdiv_rn(__fmul_rn(__fsub_rn((float)y, in.cy), d), in.fy);
        const float X2 = d;
        float Xw[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
            Xw[a] = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(P.R[3 * a], X0), __fmul_rn(P.R[3 * a + 1], X1)),
                                        __fmul_rn(P.R[3 * a + 2], X2)),
                              P.t[a]);
        pos_rad[g] = make_float4(Xw[0], Xw[1], Xw[2], __fdiv_rn(d, fmean));  // r = D / f
        const float o = opacity ? opacity[g] : opacity_default;
        col_opa[g] = make_float4(rgb[3 * g], rgb[3 * g + 1], rgb[3 * g + 2], o);
    }
    if (n_valid) {   // the valid-slot count: warp sums, one atomic per warp
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_valid, (unsigned long long)cnt);
    }
}

// Densification on a regular frame: a new Gaussian at every
// pixel with valid depth and silhouette < threshold, initialised as above, appended in row-major
// order (deterministic).  Three passes: per-256-pixel counts, one-CTA scan, ranked write.
__device__ __forceinline__ bool densify_sel(const float *depth, const float *sil, float thr, int p) {
    const float d = depth[p];
    return d > 0.0f && isfinite(d) && sil[p] < thr;
}

__global__ void __launch_bounds__(256) k_densify_count(const float *__restrict__ depth, const float *__restrict__ sil,
                                                       float thr, int HW, uint32_t *__restrict__ counts) {
    const int p = blockIdx.x * 256 + threadIdx.x;
    const unsigned b = __ballot_sync(0xffffffffu, p < HW && densify_sel(depth, sil, thr, p));
    __shared__ uint32_t w[8];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = __popc(b);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int i = 0; i < 8; ++i) t += w[i];
        counts[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) k_densify_scan(uint32_t *__restrict__ counts, int nblk,
                                                       int64_t *__restrict__ n_new) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nblk; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nblk ? counts[i] : 0u;
        uint32_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if ((threadIdx.x & 31) >= o) incl += y;
        }
        if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = incl;
        __syncthreads();
        uint32_t pre = carry;
        for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) pre += ws[w];
        if (i < nblk) counts[i] = pre + incl - v;   // exclusive offsets
        __syncthreads();
        if (threadIdx.x == 1023) carry = pre + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_new = (int64_t)carry;
}

__global__ void __launch_bounds__(256) k_densify_write(const float *__restrict__ depth, const float *__restrict__ rgb,
                                                       const vtgs_pose *__restrict__ pose, int HW, int W,
                                                       vtgs_intrinsics in, const float *__restrict__ sil, float thr,
                                                       const float *__restrict__ opacity, float opacity_default,
                                                       const uint32_t *__restrict__ offsets,
                                                       float4 *__restrict__ pos_rad, float4 *__restrict__ col_opa) {
    __shared__ PoseR P;
    __shared__ uint32_t w[8];
    if (threadIdx.x == 0) pose_rotation(*pose, P);
    const int p = blockIdx.x * 256 + threadIdx.x;
    const bool sel = p < HW && densify_sel(depth, sil, thr, p);
    const unsigned b = __ballot_sync(0xffffffffu, sel);
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = __popc(b);
    __syncthreads();
    if (!sel) return;
    uint32_t r = offsets[blockIdx.x] + __popc(b & lanemask_lt());
    for (int i = 0; i < (int)(threadIdx.x >> 5); ++i) r += w[i];
    const float fmean = __fmul_rn(0.5f, __fadd_rn(in.fx, in.fy));
    const float d = depth[p];
    const int y = p / W, x = p - y * W;
    const float X0 = __fdiv_rn(__fmul_rn(__fsub_rn((float)x, in.cx), d), in.fx);
    const float X1 = __fdiv_rn(__fmul_rn(__fsub_rn((float)y, in.cy), d), in.fy);
    float Xw[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        Xw[a] = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(P.R[3 * a], X0), __fmul_rn(P.R[3 * a + 1], X1)),
                                    __fmul_rn(P.R[3 * a + 2], d)),
                          P.t[a]);
    pos_rad[r] = make_float4(Xw[0], Xw[1], Xw[2], __fdiv_rn(d, fmean));
    col_opa[r] = make_float4(rgb[3 * p], rgb[3 * p + 1], rgb[3 * p + 2], opacity ? opacity[p] : opacity_default);
}

cudaError_t launch_densify(Ctx &c, const float *depth, const float *rgb, const vtgs_pose *pose, vtgs_intrinsics intr,
                           const float *sil, float thr, const float *opacity, float opacity_default,
                           float4 *pos_rad, float4 *col_opa, int64_t *n_new, cudaStream_t s) {
    const int HW = intr.width * intr.height;
    const int nblk = (HW + 255) / 256;
    LaunchScope ls(&c, kDensify, s);
    k_densify_count<<<nblk, 256, 0, s>>>(depth, sil, thr, HW, c.offs);
    k_densify_scan<<<1, 1024, 0, s>>>(c.offs, nblk, n_new);
    k_densify_write<<<nblk, 256, 0, s>>>(depth, rgb, pose, HW, intr.width, intr, sil, thr, opacity, opacity_default,
                                         c.offs, pos_rad, col_opa);
    c.launches += 2;
    return cudaGetLastError();
}

// Visibility mask of a frame to a section's reference views ("Visibility Check",
// SPEC.md:313-331): a valid pixel's back-projected point is visible to reference r iff it lies in
// front of it (z > 0.01), projects inside the image, the bilinearly interpolated reference depth
// there is valid (all four neighbours > 0) and |z − d_r| ≤ tol·d_r; the mask is the union over
// the references.  One thread per pixel; decisions in fp32 with the oracle's operation order
// (R25).
constexpr int kMaxVisRefs = 8;

// Back-projection of pixel (x, y) at depth d from the frame's pose (DESIGN.md §3 step 2 order).
__device__ __forceinline__ void vis_world_point(int x, int y, float d, const PoseR &P, const vtgs_intrinsics &in,
                                                float Xw[3]) {
    const float X0 = __fdiv_rn(__fmul_rn(__fsub_rn((float)x, in.cx), d), in.fx);
    const float X1 = __fdiv_rn(__fmul_rn(__fsub_rn((float)y, in.cy), d), in.fy);
#pragma unroll
    for (int a = 0; a < 3; ++a)
        Xw[a] = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(P.R[3 * a], X0), __fmul_rn(P.R[3 * a + 1], X1)),
                                    __fmul_rn(P.R[3 * a + 2], d)),
                          P.t[a]);
}

// The 1 % depth-band test of one world point against one reference view (R25).
__device__ __forceinline__ bool vis_test(const float Xw[3], const PoseR &Pr, const float *__restrict__ D, int W,
                                         int H, const vtgs_intrinsics &in, float tol) {
    float X[3];
    view_transform(Pr.R, Pr.t, make_float4(Xw[0], Xw[1], Xw[2], 0.f), X);
    const float z = X[2];
    if (!(z > kNearClip)) return false;
    const float u = __fadd_rn(__fdiv_rn(__fmul_rn(in.fx, X[0]), z), in.cx);
    const float v = __fadd_rn(__fdiv_rn(__fmul_rn(in.fy, X[1]), z), in.cy);
    if (!(u >= 0.0f && u <= (float)(W - 1) && v >= 0.0f && v <= (float)(H - 1))) return false;
    const int x0 = (int)floorf(u), y0 = (int)floorf(v);
    const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
    const float fa = __fsub_rn(u, (float)x0), fb = __fsub_rn(v, (float)y0);
    const float d00 = D[y0 * W + x0], d10 = D[y0 * W + x1], d01 = D[y1 * W + x0], d11 = D[y1 * W + x1];
    if (!(d00 > 0.0f && d10 > 0.0f && d01 > 0.0f && d11 > 0.0f)) return false;
    const float ia = __fsub_rn(1.0f, fa), ib = __fsub_rn(1.0f, fb);
    const float di = __fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(d00, ia), __fmul_rn(d10, fa)), ib),
                               __fmul_rn(__fadd_rn(__fmul_rn(d01, ia), __fmul_rn(d11, fa)), fb));
    return fabsf(__fsub_rn(z, di)) <= __fmul_rn(tol, di);
}

__global__ void __launch_bounds__(256) k_visibility(const float *__restrict__ depth, const vtgs_pose *__restrict__ pose,
                                                    const float *__restrict__ ref_depth,
                                                    const vtgs_pose *__restrict__ ref_poses, int R, int W, int H,
                                                    vtgs_intrinsics in, float tol, uint8_t *__restrict__ mask,
                                                    unsigned long long *__restrict__ n_vis) {
    __shared__ PoseR P, Pr[kMaxVisRefs];
    if (threadIdx.x == 0) pose_rotation(*pose, P);
    if (threadIdx.x < R) pose_rotation(ref_poses[threadIdx.x], Pr[threadIdx.x]);
    __syncthreads();
    const int HW = W * H;
    unsigned cnt = 0;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += gridDim.x * blockDim.x) {
        uint8_t vis = 0;
        const float d = depth[p];
        if (d > 0.0f && isfinite(d)) {
            const int y = p / W, x = p - y * W;
            float Xw[3];
            vis_world_point(x, y, d, P, in, Xw);
            for (int r = 0; r < R && !vis; ++r)
                if (vis_test(Xw, Pr[r], ref_depth + (size_t)r * HW, W, H, in, tol)) vis = 1;
        }
        mask[p] = vis;
        cnt += vis;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (n_vis && (threadIdx.x & 31) == 0 && cnt) atomicAdd(n_vis, (unsigned long long)cnt);
}

// Per-candidate visible-point counts for the overlapping-section selection ("we
// project the depth D_i from the initialized pose to each one frame in the overlap candidate view
// list. We count the number of visible points to each candidate view"): counts[r] = number of
// valid pixels of the frame visible to candidate r alone (no union); n_valid = valid pixels.
// grid.y = candidate; one thread per pixel; warp sums → one atomic per warp.
__global__ void __launch_bounds__(256) k_visibility_counts(const float *__restrict__ depth,
                                                           const vtgs_pose *__restrict__ pose,
                                                           const float *__restrict__ ref_depth,
                                                           const vtgs_pose *__restrict__ ref_poses, int W, int H,
                                                           vtgs_intrinsics in, float tol,
                                                           unsigned long long *__restrict__ counts,
                                                           unsigned long long *__restrict__ n_valid) {
    __shared__ PoseR P, Pr;
    const int r = blockIdx.y;
    if (threadIdx.x == 0) pose_rotation(*pose, P);
    if (threadIdx.x == 32) pose_rotation(ref_poses[r], Pr);
    __syncthreads();
    const int HW = W * H;
    const float *D = ref_depth + (size_t)r * HW;
    unsigned cnt = 0, nv = 0;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += gridDim.x * blockDim.x) {
        const float d = depth[p];
        if (d > 0.0f && isfinite(d)) {
            ++nv;
            const int y = p / W, x = p - y * W;
            float Xw[3];
            vis_world_point(x, y, d, P, in, Xw);
            cnt += vis_test(Xw, Pr, D, W, H, in, tol) ? 1u : 0u;
        }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    nv = __reduce_add_sync(0xffffffffu, nv);
    if ((threadIdx.x & 31) == 0) {
        if (cnt) atomicAdd(counts + r, (unsigned long long)cnt);
        if (n_valid && r == 0 && nv) atomicAdd(n_valid, (unsigned long long)nv);
    }
}

cudaError_t launch_visibility_counts(Ctx &c, const float *depth, const vtgs_pose *pose, const float *ref_depth,
                                     const vtgs_pose *ref_poses, int R, vtgs_intrinsics intr, float tol,
                                     int64_t *counts, int64_t *n_valid, cudaStream_t s) {
    const int HW = intr.width * intr.height;
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)R, s);
    if (!e && n_valid) e = cudaMemsetAsync(n_valid, 0, sizeof(int64_t), s);
    if (e) return e;
    int gx = (HW + 255) / 256;
    const int cap = (c.num_sms * 8 + R - 1) / R;
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    LaunchScope ls(&c, kVisibility, s);
    k_visibility_counts<<<dim3(gx, R), 256, 0, s>>>(depth, pose, ref_depth, ref_poses, intr.width, intr.height, intr,
                                                     tol, (unsigned long long *)counts, (unsigned long long *)n_valid);
    return cudaGetLastError();
}

cudaError_t launch_visibility(Ctx &c, const float *depth, const vtgs_pose *pose, const float *ref_depth,
                              const vtgs_pose *ref_poses, int R, vtgs_intrinsics intr, float tol, uint8_t *mask,
                              int64_t *n_vis, cudaStream_t s) {
    const int HW = intr.width * intr.height;
    int g = (HW + 255) / 256;
    if (g > c.num_sms * 8) g = c.num_sms * 8;
    cudaError_t e = cudaSuccess;
    if (n_vis && (e = cudaMemsetAsync(n_vis, 0, sizeof(int64_t), s))) return e;
    LaunchScope ls(&c, kVisibility, s);
    k_visibility<<<g, 256, 0, s>>>(depth, pose, ref_depth, ref_poses, R, intr.width, intr.height, intr, tol, mask,
                                   (unsigned long long *)n_vis);
    return cudaGetLastError();
}

cudaError_t launch_instantiate(Ctx &c, const float *depth, const float *rgb, const vtgs_pose *poses, int K,
                               vtgs_intrinsics intr, const float *opacity, float opacity_default,
                               float4 *pos_rad, float4 *col_opa, int64_t *n_valid, cudaStream_t s) {
    const int HW = intr.width * intr.height;
    if (K <= 0 || HW <= 0) return n_valid ? cudaMemsetAsync(n_valid, 0, sizeof(int64_t), s) : cudaSuccess;
    int gx = (HW + 255) / 256;
    if (gx > 4096) gx = 4096;
    dim3 grid(gx, K);
    LaunchScope ls(&c, kInstantiate, s);
    if (n_valid) {
        cudaError_t e = cudaMemsetAsync(n_valid, 0, sizeof(int64_t), s);
        if (e) return e;
    }
    k_instantiate<<<grid, 256, 0, s>>>(depth, rgb, poses, HW, intr.width, intr, opacity, opacity_default,
                                       pos_rad, col_opa, (unsigned long long *)n_valid);
    return cudaGetLastError();
}

// Sensor-format targets (vtgs_step_host_sensor): c = v / 255, z = d · scale, in fp32 (the same
// two IEEE operations a host-side conversion would use).  Four pixels per thread when the pixel
// count allows 16-byte stores (three 4-byte colour words and one 8-byte depth word in, three
// float4 colour and one float4 depth out), else one pixel per thread.
__global__ void __launch_bounds__(256) k_sensor_targets4(const uint32_t *__restrict__ rgb8,
                                                         const uint2 *__restrict__ d16, float scale, int64_t ng,
                                                         float4 *__restrict__ rgb, float4 *__restrict__ depth) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t w[3] = {__ldg(rgb8 + 3 * g), __ldg(rgb8 + 3 * g + 1), __ldg(rgb8 + 3 * g + 2)};
        float c[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) c[i] = __fdiv_rn((float)((w[i >> 2] >> (8 * (i & 3))) & 0xffu), 255.0f);
        rgb[3 * g + 0] = make_float4(c[0], c[1], c[2], c[3]);
        rgb[3 * g + 1] = make_float4(c[4], c[5], c[6], c[7]);
        rgb[3 * g + 2] = make_float4(c[8], c[9], c[10], c[11]);
        const uint2 d = __ldg(d16 + g);
        depth[g] = make_float4(__fmul_rn((float)(d.x & 0xffffu), scale), __fmul_rn((float)(d.x >> 16), scale),
                               __fmul_rn((float)(d.y & 0xffffu), scale), __fmul_rn((float)(d.y >> 16), scale));
    }
}

__global__ void __launch_bounds__(256) k_sensor_targets(const uint8_t *__restrict__ rgb8,
                                                        const uint16_t *__restrict__ d16, float scale, int64_t px,
                                                        float *__restrict__ rgb, float *__restrict__ depth) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < px; i += (int64_t)gridDim.x * blockDim.x) {
        rgb[3 * i + 0] = __fdiv_rn((float)rgb8[3 * i + 0], 255.0f);
        rgb[3 * i + 1] = __fdiv_rn((float)rgb8[3 * i + 1], 255.0f);
        rgb[3 * i + 2] = __fdiv_rn((float)rgb8[3 * i + 2], 255.0f);
        depth[i] = __fmul_rn((float)d16[i], scale);
    }
}

cudaError_t launch_sensor_targets(Ctx &c, const uint8_t *rgb8, const uint16_t *d16, float scale, int64_t px,
                                  float *rgb, float *depth, cudaStream_t s) {
    const bool vec = px % 4 == 0 && ((uintptr_t)rgb8 % 4 == 0) && ((uintptr_t)d16 % 8 == 0) &&
                     ((uintptr_t)rgb % 16 == 0) && ((uintptr_t)depth % 16 == 0);
    const int64_t n = vec ? px / 4 : px;
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)c.num_sms * 8) g = (int64_t)c.num_sms * 8;
    if (g < 1) g = 1;
    if (vec)
        k_sensor_targets4<<<(int)g, 256, 0, s>>>(reinterpret_cast<const uint32_t *>(rgb8),
                                                 reinterpret_cast<const uint2 *>(d16), scale, n,
                                                 reinterpret_cast<float4 *>(rgb), reinterpret_cast<float4 *>(depth));
    else
        k_sensor_targets<<<(int)g, 256, 0, s>>>(rgb8, d16, scale, px, rgb, depth);
    return cudaGetLastError();
}

}  // namespace vtgs
