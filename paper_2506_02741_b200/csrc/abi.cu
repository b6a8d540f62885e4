// abi.cu — the C ABI of include/vtgs.h: argument validation, context / scratch ownership,
// error capture.  No arithmetic of the method lives here; every step runs in the kernels of
// instantiate.cu, forward.cu and backward.cu.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include "vtgs_internal.cuh"

using vtgs::Ctx;

struct vtgs_ctx {
    Ctx c;
};

namespace {

vtgs_status fail(vtgs_ctx *ctx, vtgs_status s, const char *fmt, ...) __attribute__((format(printf, 3, 4)));

vtgs_status fail(vtgs_ctx *ctx, vtgs_status s, const char *fmt, ...) {
    if (ctx) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(ctx->c.last_error, sizeof(ctx->c.last_error), fmt, ap);
        va_end(ap);
    }
    return s;
}

vtgs_status cuda_fail(vtgs_ctx *ctx, cudaError_t e, const char *where) {
    return fail(ctx, VTGS_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

vtgs_status check_intr(vtgs_ctx *ctx, const vtgs_intrinsics &in) {
    if (in.width <= 0 || in.height <= 0 || in.width > ctx->c.max_w || in.height > ctx->c.max_h)
        return fail(ctx, VTGS_ERR_SHAPE, "image %dx%d outside the context's 1..%dx%d", in.width, in.height,
                    ctx->c.max_w, ctx->c.max_h);
    if (!(in.fx > 0.0f) || !(in.fy > 0.0f) || !(in.cx > 0.0f) || !(in.cx < (float)in.width) ||
        !(in.cy > 0.0f) || !(in.cy < (float)in.height))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "intrinsics need fx, fy > 0, 0 < cx < W, 0 < cy < H (SPEC.md:25)");
    return VTGS_OK;
}

template <typename T>
cudaError_t dalloc(T **p, size_t n) {
    return cudaMalloc((void **)p, sizeof(T) * (n ? n : 1));
}

void free_all(Ctx &c) {
    void *ptrs[] = {c.proj, c.rect, c.thr, c.tile_count, c.tile_start, c.tile_cursor, c.tile_flag, c.keys, c.vals, c.pbits, c.keys2,
                    c.vals2, c.offs, c.sub_lists, c.sub_masks, c.chunk_list, c.sub_count, c.T_final, c.last, c.partials, c.dev, c.host_io, c.sensor_io, c.view_copy, c.ssim_abc, c.ssim_partials, c.det};
    for (void *p : ptrs)
        if (p) cudaFree(p);
}

}  // namespace

extern "C" {

int32_t vtgs_abi_version(void) { return VTGS_ABI_VERSION; }

const char *vtgs_status_string(vtgs_status s) {
    switch (s) {
        case VTGS_OK: return "ok";
        case VTGS_ERR_INVALID_ARG: return "invalid argument";
        case VTGS_ERR_SHAPE: return "shape / size out of range";
        case VTGS_ERR_CAPACITY: return "tile-pair capacity exceeded";
        case VTGS_ERR_CUDA: return "CUDA error";
        case VTGS_ERR_STATE: return "backward without a forward";
        case VTGS_ERR_NO_DEVICE: return "no CUDA device (there is no CPU fallback)";
        default: return "unknown status";
    }
}

const char *vtgs_last_error(const vtgs_ctx *ctx) { return ctx ? ctx->c.last_error : ""; }

vtgs_status vtgs_create(vtgs_ctx **out, int32_t device, int64_t max_gaussians, int32_t max_width,
                        int32_t max_height, int64_t max_pairs) {
    if (!out) return VTGS_ERR_INVALID_ARG;
    *out = nullptr;
    if (max_gaussians < 0 || max_gaussians > 0xffffffffLL || max_width <= 0 || max_height <= 0 ||
        max_width > 65535 || max_height > 65535)
        return VTGS_ERR_SHAPE;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return VTGS_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= ndev) return VTGS_ERR_INVALID_ARG;
    // default: 2 pairs per slot (+256k for small contexts) — the five configs measure P ≤ 1.75 N
    // for one view (config 2: 7.0M of 4.08M slots); a view that needs more reports VTGS_ERR_CAPACITY
    if (max_pairs <= 0) max_pairs = 2 * (max_gaussians > 0 ? max_gaussians : 1) + 262144;
    if (max_pairs > 0xfffffff0LL) max_pairs = 0xfffffff0LL;
    vtgs_ctx *ctx = new (std::nothrow) vtgs_ctx();
    if (!ctx) return VTGS_ERR_CUDA;
    Ctx &c = ctx->c;
    c.device = device;
    c.max_gaussians = max_gaussians;
    c.max_w = max_width;
    c.max_h = max_height;
    c.max_pairs = max_pairs;
    c.max_tiles = ((max_width + 15) / 16) * ((max_height + 15) / 16);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    const size_t px = (size_t)max_width * max_height;
    if (!e) e = cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device);
    if (!e) e = dalloc(&c.proj, (size_t)max_gaussians);
    if (!e) e = dalloc(&c.rect, (size_t)max_gaussians);
    if (!e) e = dalloc(&c.thr, (size_t)max_gaussians);
    if (!e) e = dalloc(&c.tile_count, (size_t)c.max_tiles);
    if (!e) e = dalloc(&c.tile_start, (size_t)c.max_tiles + 1);
    if (!e) e = dalloc(&c.tile_cursor, (size_t)c.max_tiles);
    if (!e) e = dalloc(&c.tile_flag, (size_t)2 * c.max_tiles);
    if (!e) e = dalloc(&c.keys, (size_t)max_pairs);
    if (!e) e = dalloc(&c.vals, (size_t)max_pairs);
    if (!e) e = dalloc(&c.pbits, (size_t)max_pairs);
    if (!e) e = dalloc(&c.keys2, (size_t)max_pairs);
    if (!e) e = dalloc(&c.vals2, (size_t)max_pairs);
    if (!e) e = dalloc(&c.offs, (size_t)max_pairs);
    if (!e) e = dalloc(&c.sub_lists, (size_t)8 * max_pairs);
    if (!e) e = dalloc(&c.sub_masks, (size_t)8 * max_pairs);
    if (!e) e = dalloc(&c.chunk_list, (size_t)12 * ((size_t)max_pairs / 2048 + c.max_tiles + 1));
    if (!e) e = dalloc(&c.sub_count, (size_t)8 * c.max_tiles);
    if (!e) e = dalloc(&c.T_final, px);
    if (!e) e = dalloc(&c.last, px);
    if (!e) e = dalloc(&c.partials, (size_t)c.max_tiles * 8 * 16 + 64 * 16);  // + k_pose_finalize level 2
    if (!e) e = dalloc(&c.dev, 1);
    if (!e) e = dalloc(&c.ssim_abc, 9 * px);
    if (!e) e = dalloc(&c.ssim_partials, ((size_t)(max_width + 31) / 32) * ((max_height + 7) / 8));
    if (!e) e = dalloc(&c.host_io, 4 * px + 64);
    if (!e) e = dalloc(&c.sensor_io, 5 * px + 64);
    if (!e) e = dalloc(&c.view_copy, 1);
    if (!e) e = cudaMemset(c.dev, 0, sizeof(vtgs::DevScalars));
    if (!e) e = cudaMemset(c.tile_count, 0, sizeof(uint32_t) * c.max_tiles);
    if (!e) e = cudaMemset(c.tile_start, 0, sizeof(uint32_t) * (c.max_tiles + 1));
    if (!e) e = vtgs::forward_set_attributes();
    if (!e) e = vtgs::backward_set_attributes();
    if (!e) e = vtgs::ssim_set_constants();
    if (!e) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e) {
        cudaGetLastError();
        free_all(c);
        delete ctx;
        return e == cudaErrorMemoryAllocation ? VTGS_ERR_CAPACITY : VTGS_ERR_CUDA;
    }
    *out = ctx;
    return VTGS_OK;
}

vtgs_status vtgs_destroy(vtgs_ctx *ctx) {
    if (!ctx) return VTGS_OK;
    cudaSetDevice(ctx->c.device);
    cudaDeviceSynchronize();
    for (auto *v : {&ctx->c.prof, &ctx->c.prof_free})
        for (auto &ev : *v) {
            cudaEventDestroy(ev.a);
            cudaEventDestroy(ev.b);
        }
    if (ctx->c.copy_stream) cudaStreamDestroy(ctx->c.copy_stream);
    if (ctx->c.ev_ready) cudaEventDestroy(ctx->c.ev_ready);
    if (ctx->c.ev_copied) cudaEventDestroy(ctx->c.ev_copied);
    if (ctx->c.host_ret) cudaFreeHost(ctx->c.host_ret);
    free_all(ctx->c);
    delete ctx;
    return VTGS_OK;
}

vtgs_status vtgs_instantiate(vtgs_ctx *ctx, const float *depth, const float *rgb,
                             const vtgs_pose *kf_poses, int32_t K, vtgs_intrinsics intr,
                             const float *opacity_init, float opacity_default, float *pos_rad,
                             float *col_opa, int64_t *n_valid, void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    ctx->c.last_error[0] = 0;
    vtgs_status st = check_intr(ctx, intr);
    if (st) return st;
    if (K < 0) return fail(ctx, VTGS_ERR_SHAPE, "K = %d < 0", K);
    const int64_t N = (int64_t)K * intr.width * intr.height;
    if (N > ctx->c.max_gaussians)
        return fail(ctx, VTGS_ERR_CAPACITY, "K·H·W = %lld exceeds max_gaussians %lld", (long long)N,
                    (long long)ctx->c.max_gaussians);
    if (K == 0) {
        if (n_valid) {
            cudaSetDevice(ctx->c.device);
            cudaError_t e = cudaMemsetAsync(n_valid, 0, sizeof(int64_t), (cudaStream_t)stream);
            if (e) return cuda_fail(ctx, e, "vtgs_instantiate");
        }
        return VTGS_OK;
    }
    if (!depth || !rgb || !kf_poses || !pos_rad || !col_opa)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL depth / rgb / kf_poses / pos_rad / col_opa");
    if (!aligned16(pos_rad) || !aligned16(col_opa))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "pos_rad / col_opa must be 16-byte aligned float4 arrays");
    cudaSetDevice(ctx->c.device);
    cudaError_t e = vtgs::launch_instantiate(ctx->c, depth, rgb, kf_poses, K, intr, opacity_init, opacity_default,
                                             (float4 *)pos_rad, (float4 *)col_opa, n_valid, (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_instantiate") : VTGS_OK;
}

vtgs_status vtgs_render_fwd(vtgs_ctx *ctx, const float *pos_rad, const float *col_opa, int64_t N,
                            const vtgs_pose *view, vtgs_intrinsics intr, float *color, float *depth,
                            float *silhouette, void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    c.last_error[0] = 0;
    vtgs_status st = check_intr(ctx, intr);
    if (st) return st;
    if (N < 0) return fail(ctx, VTGS_ERR_SHAPE, "N = %lld < 0", (long long)N);
    if (N > c.max_gaussians)
        return fail(ctx, VTGS_ERR_CAPACITY, "N = %lld exceeds max_gaussians %lld", (long long)N,
                    (long long)c.max_gaussians);
    if ((N > 0 && (!pos_rad || !col_opa)) || !view || !color || !depth || !silhouette)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL state / view / output pointer");
    if (!aligned16(pos_rad) || !aligned16(col_opa))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "pos_rad / col_opa must be 16-byte aligned float4 arrays");
    c.have_fwd = false;
    c.pos_rad = (const float4 *)pos_rad;
    c.col_opa = (const float4 *)col_opa;
    c.N = N;
    c.view = view;
    c.intr = intr;
    c.color = color;
    c.depth = depth;
    c.sil = silhouette;
    cudaSetDevice(c.device);
    cudaError_t e = vtgs::launch_forward(c, (cudaStream_t)stream);
    if (e) return cuda_fail(ctx, e, "vtgs_render_fwd");
    c.have_fwd = true;
    return VTGS_OK;
}

vtgs_status vtgs_render_bwd(vtgs_ctx *ctx, const float *dL_dcolor, const float *dL_ddepth,
                            const float *dL_dsil, const vtgs_l1_loss *loss, uint32_t want,
                            int64_t learn_begin, int64_t learn_end, float *d_col_opa,
                            float *d_radius, float *d_position, float *d_pose, float *loss_out,
                            void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    c.last_error[0] = 0;
    if (!c.have_fwd) return fail(ctx, VTGS_ERR_STATE, "vtgs_render_bwd before any vtgs_render_fwd");
    if (want & ~0x3fu) return fail(ctx, VTGS_ERR_INVALID_ARG, "unknown bits in want = 0x%x", want);
    if (loss && (dL_dcolor || dL_ddepth || dL_dsil))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "pass either upstream gradients or a fused loss, not both");
    if (loss && (!loss->target_rgb || !loss->target_depth))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "fused loss needs target_rgb and target_depth");
    if (loss_out && !loss) return fail(ctx, VTGS_ERR_INVALID_ARG, "loss_out requires a fused loss");
    if ((want & (VTGS_GRAD_COLOR | VTGS_GRAD_OPACITY)) && !d_col_opa)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "colour/opacity gradients wanted but d_col_opa is NULL");
    if ((want & VTGS_GRAD_RADIUS) && !d_radius)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "radius gradient wanted but d_radius is NULL");
    if ((want & VTGS_GRAD_POSE) && !d_pose)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "pose gradient wanted but d_pose is NULL");
    if ((want & VTGS_GRAD_POSITION) && !d_position)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "position gradient wanted but d_position is NULL");
    if (d_position && !aligned16(d_position))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "d_position must be a 16-byte aligned float4 array");
    if (d_col_opa && !aligned16(d_col_opa))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "d_col_opa must be a 16-byte aligned float4 array");
    if (learn_begin < 0) learn_begin = 0;
    if (learn_end > c.N) learn_end = c.N;
    cudaSetDevice(c.device);
    cudaError_t e = vtgs::launch_backward(c, dL_dcolor, dL_ddepth, dL_dsil, loss, want, learn_begin, learn_end,
                                          (float4 *)d_col_opa, d_radius, (float4 *)d_position, d_pose, loss_out,
                                          (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_render_bwd") : VTGS_OK;
}

vtgs_status vtgs_keyframe_pose_grad(vtgs_ctx *ctx, const float *pos_rad, const float *d_position,
                                    const vtgs_pose *kf_poses, int32_t K, int64_t slots_per_kf, float *d_kf_pose,
                                    void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    c.last_error[0] = 0;
    if (!pos_rad || !d_position || !kf_poses || !d_kf_pose)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL pos_rad / d_position / kf_poses / d_kf_pose");
    if (K < 0 || slots_per_kf < 0) return fail(ctx, VTGS_ERR_SHAPE, "K = %d, slots_per_kf = %lld", K,
                                                (long long)slots_per_kf);
    if (!aligned16(pos_rad) || !aligned16(d_position))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "pos_rad / d_position must be 16-byte aligned float4 arrays");
    if (K == 0) return VTGS_OK;
    cudaSetDevice(c.device);
    cudaError_t e = vtgs::launch_keyframe_pose_grad(c, (const float4 *)pos_rad, (const float4 *)d_position, kf_poses,
                                                    K, slots_per_kf, d_kf_pose, (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_keyframe_pose_grad") : VTGS_OK;
}

vtgs_status vtgs_visibility_mask(vtgs_ctx *ctx, const float *depth, const vtgs_pose *pose, const float *ref_depth,
                                 const vtgs_pose *ref_poses, int32_t R, vtgs_intrinsics intr, float tol, uint8_t *mask,
                                 int64_t *n_visible, void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    c.last_error[0] = 0;
    if (!depth || !pose || !ref_depth || !ref_poses || !mask)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL argument to vtgs_visibility_mask");
    if (R < 1 || R > 8) return fail(ctx, VTGS_ERR_SHAPE, "R = %d reference views (1..8)", R);
    vtgs_status st = check_intr(ctx, intr);
    if (st) return st;
    cudaSetDevice(c.device);
    cudaError_t e = vtgs::launch_visibility(c, depth, pose, ref_depth, ref_poses, R, intr, tol, mask, n_visible,
                                            (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_visibility_mask") : VTGS_OK;
}

vtgs_status vtgs_visibility_counts(vtgs_ctx *ctx, const float *depth, const vtgs_pose *pose, const float *ref_depth,
                                   const vtgs_pose *ref_poses, int32_t R, vtgs_intrinsics intr, float tol,
                                   int64_t *counts, int64_t *n_valid, void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    c.last_error[0] = 0;
    if (!depth || !pose || !ref_depth || !ref_poses || !counts)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL argument to vtgs_visibility_counts");
    if (R < 1 || R > 65535) return fail(ctx, VTGS_ERR_SHAPE, "R = %d candidate views (1..65535)", R);
    vtgs_status st = check_intr(ctx, intr);
    if (st) return st;
    cudaSetDevice(c.device);
    cudaError_t e = vtgs::launch_visibility_counts(c, depth, pose, ref_depth, ref_poses, R, intr, tol, counts,
                                                   n_valid, (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_visibility_counts") : VTGS_OK;
}

vtgs_status vtgs_densify(vtgs_ctx *ctx, const float *depth, const float *rgb, const vtgs_pose *pose,
                         vtgs_intrinsics intr, const float *silhouette, float threshold, const float *opacity,
                         float opacity_default, float *pos_rad_out, float *col_opa_out, int64_t *n_new,
                         void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    c.last_error[0] = 0;
    if (!depth || !rgb || !pose || !silhouette || !pos_rad_out || !col_opa_out || !n_new)
        return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL argument to vtgs_densify");
    vtgs_status st = check_intr(ctx, intr);
    if (st) return st;
    if (!aligned16(pos_rad_out) || !aligned16(col_opa_out))
        return fail(ctx, VTGS_ERR_INVALID_ARG, "pos_rad_out / col_opa_out must be 16-byte aligned float4 arrays");
    cudaSetDevice(c.device);
    cudaError_t e = vtgs::launch_densify(c, depth, rgb, pose, intr, silhouette, threshold, opacity, opacity_default,
                                         (float4 *)pos_rad_out, (float4 *)col_opa_out, n_new, (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_densify") : VTGS_OK;
}

vtgs_status vtgs_ssim_loss(vtgs_ctx *ctx, const float *color, const float *target_rgb, int32_t width,
                           int32_t height, float tau, float *d_color, float *loss_out, void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    c.last_error[0] = 0;
    if (!color || !target_rgb) return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL color / target_rgb");
    if (width < 11 || height < 11)
        return fail(ctx, VTGS_ERR_SHAPE, "SSIM needs an image of at least 11×11 (the window), got %d×%d", width,
                    height);
    if (width > c.max_w || height > c.max_h)
        return fail(ctx, VTGS_ERR_CAPACITY, "image %d×%d exceeds the context's %d×%d", width, height, c.max_w,
                    c.max_h);
    cudaSetDevice(c.device);
    cudaError_t e = vtgs::launch_ssim(c, color, target_rgb, width, height, tau, d_color, loss_out, (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_ssim_loss") : VTGS_OK;
}

vtgs_status vtgs_pose_adam_step(vtgs_ctx *ctx, vtgs_pose *pose, const float *d_pose, float *adam_state,
                                float lr_rot, float lr_trans, void *stream) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    ctx->c.last_error[0] = 0;
    if (!pose || !d_pose || !adam_state) return fail(ctx, VTGS_ERR_INVALID_ARG, "NULL pose / d_pose / state");
    cudaSetDevice(ctx->c.device);
    cudaError_t e = vtgs::launch_pose_adam(ctx->c, pose, d_pose, adam_state, lr_rot, lr_trans, (cudaStream_t)stream);
    return e ? cuda_fail(ctx, e, "vtgs_pose_adam_step") : VTGS_OK;
}

vtgs_status vtgs_get_stats(vtgs_ctx *ctx, vtgs_stats *out, void *stream) {
    if (!ctx || !out) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    vtgs::DevScalars d;
    cudaError_t e = cudaMemcpyAsync(&d, c.dev, sizeof(d), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e) return cuda_fail(ctx, e, "vtgs_get_stats");
    out->n_gaussians = c.N;
    out->n_pairs = (int64_t)d.n_pairs;
    out->e_eval = (int64_t)d.e_eval;
    out->e_comp = (int64_t)d.e_comp;
    out->max_tile = d.max_tile;
    out->overflow = d.overflow;
    out->launches = c.launches;
    return d.overflow ? fail(ctx, VTGS_ERR_CAPACITY, "P = %llu pairs > max_pairs %lld", d.n_pairs,
                             (long long)c.max_pairs)
                      : VTGS_OK;
}

vtgs_status vtgs_set_work_counters(vtgs_ctx *ctx, int32_t enable) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    ctx->c.count_work = enable != 0;
    return VTGS_OK;
}

vtgs_status vtgs_set_profiling(vtgs_ctx *ctx, int32_t enable) {
    if (!ctx) return VTGS_ERR_INVALID_ARG;
    ctx->c.profiling = enable != 0;
    return VTGS_OK;
}

vtgs_status vtgs_get_profile(vtgs_ctx *ctx, double *ms, int64_t *counts, void *stream) {
    if (!ctx || !ms) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    cudaSetDevice(c.device);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (!e) e = cudaDeviceSynchronize();
    if (e) return cuda_fail(ctx, e, "vtgs_get_profile");
    int64_t timed[VTGS_NUM_STAGES] = {0};
    for (int i = 0; i < VTGS_NUM_STAGES; ++i) ms[i] = 0.0;
    for (auto &ev : c.prof) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, ev.a, ev.b) == cudaSuccess) {
            ms[ev.stage] += t;
            ++timed[ev.stage];
        }
        c.prof_free.push_back(ev);
    }
    cudaGetLastError();
    c.prof.clear();
    for (int i = 0; i < VTGS_NUM_STAGES; ++i) {
        if (counts) counts[i] = timed[i];
        c.prof_counts[i] = 0;
    }
    return VTGS_OK;
}

vtgs_status vtgs_check(vtgs_ctx *ctx, void *stream) {
    vtgs_stats s;
    return vtgs_get_stats(ctx, &s, stream);
}

vtgs_status vtgs_export_tiles(vtgs_ctx *ctx, int64_t *tile_start, int32_t *sorted_gid, int64_t cap,
                              int64_t *P_out, void *stream) {
    if (!ctx || !tile_start || !P_out) return VTGS_ERR_INVALID_ARG;
    Ctx &c = ctx->c;
    if (!c.have_fwd) return fail(ctx, VTGS_ERR_STATE, "no forward to export");
    const int T = ((c.intr.width + 15) / 16) * ((c.intr.height + 15) / 16);
    cudaSetDevice(c.device);
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *st = new uint32_t[T + 1];
    cudaError_t e = cudaMemcpyAsync(st, c.tile_start, sizeof(uint32_t) * (T + 1), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) {
        delete[] st;
        return cuda_fail(ctx, e, "vtgs_export_tiles");
    }
    for (int i = 0; i <= T; ++i) tile_start[i] = st[i];
    const int64_t P = st[T];
    delete[] st;
    *P_out = P;
    if (sorted_gid && P <= cap && P > 0) {
        e = cudaMemcpyAsync(sorted_gid, c.vals, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
        if (e) return cuda_fail(ctx, e, "vtgs_export_tiles");
    }
    return vtgs_check(ctx, stream);
}

}  // extern "C" (the shared body below is a C++ template)

// Shared body of vtgs_step_host / vtgs_step_host_sensor: `upload` enqueues the target copies (and
// any widening to fp32) on the copy stream after ev_ready; the backward waits for them.
template <typename Upload>
static vtgs_status step_host_core(vtgs_ctx *ctx, const float *pos_rad, const float *col_opa, int64_t N,
                                  const vtgs_pose *view_host, vtgs_intrinsics intr, float w_color, float w_depth,
                                  int32_t color_mask_mode, int32_t depth_mask_mode, int32_t normalize, uint32_t want,
                                  int64_t learn_begin, int64_t learn_end, float *color, float *depth,
                                  float *silhouette, float *d_col_opa, float *d_radius, float *loss_host,
                                  float *d_pose_host, void *stream, Upload upload) {
    Ctx &c = ctx->c;
    const size_t px = (size_t)intr.width * intr.height;
    float *d_rgb = c.host_io;                       // 3·px
    float *d_dep = c.host_io + 3 * px;              // px
    float *d_misc = c.host_io + 4 * px;             // 64 floats: pose(8) | loss(1) | d_pose(7)
    vtgs_pose *d_view = (vtgs_pose *)d_misc;
    float *d_loss = d_misc + 8;
    float *d_dpose = d_misc + 16;
    cudaStream_t s = (cudaStream_t)stream;
    cudaSetDevice(c.device);
    cudaError_t e = cudaSuccess;
    if (!c.copy_stream) {
        e = cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking);
        if (!e) e = cudaEventCreateWithFlags(&c.ev_ready, cudaEventDisableTiming);
        if (!e) e = cudaEventCreateWithFlags(&c.ev_copied, cudaEventDisableTiming);
        // pinned: a device→host copy into pageable memory is staged by the driver after the stream
        // drains, a copy into pinned memory is a DMA the synchronisation below already covers
        if (!e) e = cudaHostAlloc((void **)&c.host_ret, 16 * sizeof(float), cudaHostAllocDefault);
        if (e) return cuda_fail(ctx, e, "vtgs_step_host (copy stream)");
    }
    // the pose goes first on the compute stream; the targets (read only by the backward's loss
    // prologue) upload on a second stream while projection, sort and forward run
    e = cudaMemcpyAsync(d_view, view_host, sizeof(vtgs_pose), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaEventRecord(c.ev_ready, s);   // the previous step's backward is done with the staging
    if (!e) e = cudaStreamWaitEvent(c.copy_stream, c.ev_ready, 0);
    if (!e) e = upload(c.copy_stream, d_rgb, d_dep);
    if (!e) e = cudaEventRecord(c.ev_copied, c.copy_stream);
    if (e) return cuda_fail(ctx, e, "vtgs_step_host (H2D)");
    vtgs_status st = vtgs_render_fwd(ctx, pos_rad, col_opa, N, d_view, intr, color, depth, silhouette, stream);
    if (st) return st;
    if ((e = cudaStreamWaitEvent(s, c.ev_copied, 0))) return cuda_fail(ctx, e, "vtgs_step_host (wait)");
    vtgs_l1_loss L{d_rgb, d_dep, nullptr, w_color, w_depth, color_mask_mode, depth_mask_mode, normalize, nullptr};
    st = vtgs_render_bwd(ctx, nullptr, nullptr, nullptr, &L, want & ~(uint32_t)VTGS_GRAD_POSITION, learn_begin,
                         learn_end, d_col_opa, d_radius, nullptr, (want & VTGS_GRAD_POSE) ? d_dpose : nullptr, d_loss,
                         stream);
    if (st) return st;
    // loss, d_pose and the forward's device-side capacity flag land in the pinned host_ret
    float *hr = c.host_ret;
    const bool want_pose = d_pose_host && (want & VTGS_GRAD_POSE);
    e = cudaMemcpyAsync(hr, d_loss, sizeof(float), cudaMemcpyDeviceToHost, s);
    if (!e && want_pose) e = cudaMemcpyAsync(hr + 8, d_dpose, sizeof(float) * 7, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(hr + 1, &c.dev->overflow, sizeof(unsigned int), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) return cuda_fail(ctx, e, "vtgs_step_host (D2H)");
    *loss_host = hr[0];
    if (want_pose)
        for (int i = 0; i < 7; ++i) d_pose_host[i] = hr[8 + i];
    unsigned int overflow;
    memcpy(&overflow, hr + 1, sizeof(overflow));
    if (overflow)
        return fail(ctx, VTGS_ERR_CAPACITY, "tile pairs exceeded max_pairs %lld (render and gradients empty)",
                    (long long)c.max_pairs);
    return VTGS_OK;
}

extern "C" {

vtgs_status vtgs_step_host(vtgs_ctx *ctx, const float *pos_rad, const float *col_opa, int64_t N,
                           const vtgs_pose *view_host, vtgs_intrinsics intr,
                           const float *target_rgb_host, const float *target_depth_host, float w_color,
                           float w_depth, int32_t color_mask_mode, int32_t depth_mask_mode,
                           int32_t normalize, uint32_t want, int64_t learn_begin, int64_t learn_end,
                           float *color, float *depth, float *silhouette, float *d_col_opa,
                           float *d_radius, float *loss_host, float *d_pose_host, void *stream) {
    if (!ctx || !view_host || !target_rgb_host || !target_depth_host || !loss_host)
        return VTGS_ERR_INVALID_ARG;
    vtgs_status st = check_intr(ctx, intr);
    if (st) return st;
    const size_t px = (size_t)intr.width * intr.height;
    auto upload = [&](cudaStream_t cs, float *d_rgb, float *d_dep) {
        cudaError_t e = cudaMemcpyAsync(d_rgb, target_rgb_host, sizeof(float) * 3 * px, cudaMemcpyHostToDevice, cs);
        if (!e) e = cudaMemcpyAsync(d_dep, target_depth_host, sizeof(float) * px, cudaMemcpyHostToDevice, cs);
        return e;
    };
    return step_host_core(ctx, pos_rad, col_opa, N, view_host, intr, w_color, w_depth, color_mask_mode,
                          depth_mask_mode, normalize, want, learn_begin, learn_end, color, depth, silhouette,
                          d_col_opa, d_radius, loss_host, d_pose_host, stream, upload);
}

vtgs_status vtgs_step_host_sensor(vtgs_ctx *ctx, const float *pos_rad, const float *col_opa, int64_t N,
                                  const vtgs_pose *view_host, vtgs_intrinsics intr,
                                  const uint8_t *rgb8_host, const uint16_t *depth16_host, float depth_scale,
                                  float w_color, float w_depth, int32_t color_mask_mode,
                                  int32_t depth_mask_mode, int32_t normalize, uint32_t want,
                                  int64_t learn_begin, int64_t learn_end, float *color, float *depth,
                                  float *silhouette, float *d_col_opa, float *d_radius,
                                  float *loss_host, float *d_pose_host, void *stream) {
    if (!ctx || !view_host || !rgb8_host || !depth16_host || !loss_host || !(depth_scale > 0.0f))
        return VTGS_ERR_INVALID_ARG;
    vtgs_status st = check_intr(ctx, intr);
    if (st) return st;
    Ctx &c = ctx->c;
    const size_t px = (size_t)intr.width * intr.height;
    uint8_t *s_rgb = c.sensor_io;                                   // 3·px bytes
    uint16_t *s_dep = reinterpret_cast<uint16_t *>(c.sensor_io + ((3 * px + 15) & ~(size_t)15));   // px uint16
    // upload 5 B/px and widen on the copy stream too: both run under projection, sort and forward
    auto upload = [&](cudaStream_t cs, float *d_rgb, float *d_dep) {
        cudaError_t e = cudaMemcpyAsync(s_rgb, rgb8_host, 3 * px, cudaMemcpyHostToDevice, cs);
        if (!e) e = cudaMemcpyAsync(s_dep, depth16_host, sizeof(uint16_t) * px, cudaMemcpyHostToDevice, cs);
        if (!e) e = launch_sensor_targets(c, s_rgb, s_dep, depth_scale, (int64_t)px, d_rgb, d_dep, cs);
        return e;
    };
    return step_host_core(ctx, pos_rad, col_opa, N, view_host, intr, w_color, w_depth, color_mask_mode,
                          depth_mask_mode, normalize, want, learn_begin, learn_end, color, depth, silhouette,
                          d_col_opa, d_radius, loss_host, d_pose_host, stream, upload);
}

}  // extern "C"
