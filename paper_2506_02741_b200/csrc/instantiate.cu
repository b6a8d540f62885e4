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
                                                     float4 *__restrict__ col_opa) {
    const int k = blockIdx.y;  // keyframe
    __shared__ PoseR P;
    if (threadIdx.x == 0) pose_rotation(poses[k], P);
    __syncthreads();
    const float fmean = __fmul_rn(0.5f, __fadd_rn(in.fx, in.fy));
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += gridDim.x * blockDim.x) {
        const int64_t g = (int64_t)k * HW + p;
        const float d = depth[g];
        if (!(d > 0.0f) || !isfinite(d)) {
            pos_rad[g] = make_float4(0.f, 0.f, 0.f, 0.f);
            col_opa[g] = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
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
}

cudaError_t launch_instantiate(Ctx &c, const float *depth, const float *rgb, const vtgs_pose *poses, int K,
                               vtgs_intrinsics intr, const float *opacity, float opacity_default,
                               float4 *pos_rad, float4 *col_opa, cudaStream_t s) {
    const int HW = intr.width * intr.height;
    if (K <= 0 || HW <= 0) return cudaSuccess;
    int gx = (HW + 255) / 256;
    if (gx > 4096) gx = 4096;
    dim3 grid(gx, K);
    LaunchScope ls(&c, kInstantiate, s);
    k_instantiate<<<grid, 256, 0, s>>>(depth, rgb, poses, HW, intr.width, intr, opacity, opacity_default,
                                       pos_rad, col_opa);
    return cudaGetLastError();
}

}  // namespace vtgs
