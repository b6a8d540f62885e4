// vtgs_internal.cuh — shared definitions of the sm_100a kernels behind include/vtgs.h.
//
// Decision-exact arithmetic: every quantity that decides something discrete (tile binning,
// sort keys, the 3σ test, the α clamp and floor, the transmittance cut-off) is computed with
// explicit round-to-nearest intrinsics (__fmul_rn / __fadd_rn / __fdiv_rn, fp64 __dmul_rn …)
// so that nvcc never contracts them into FMAs and the operation order is exactly the one
// DESIGN.md §3 fixes.  Value-only arithmetic (colour / depth accumulation, gradients) is free
// to use FMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/vtgs.h"

// Checked build (`python -m paper_2506_02741_b200.build --checked` → libvtgs_checked.so): bounds and
// invariant checks in the kernels that trap on failure — this pool has compute-sanitizer closed,
// so the GPU test suite runs once against this build instead (tests/test_gpu_variants.py).
#ifdef VTGS_CHECKED
#include <cstdio>
#define VTGS_CHECK(cond)                                                                                  \
    do {                                                                                                  \
        if (!(cond)) {                                                                                    \
            printf("VTGS_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);                           \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define VTGS_CHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace vtgs {

constexpr int kTile = 16;                 // 16×16 tiles
constexpr int kBlock = 256;               // threads per tile CTA = pixels per tile
constexpr int kChunk = 256;               // tile-list entries staged in shared memory at once
constexpr int kSortCap = 4096;            // tile lists up to this length are sorted in smem
constexpr float kNearClip = 0.01f;
constexpr float kSigmaMin = 0.3f;
constexpr float kAlphaMax = 0.999f;
constexpr float kTMin = 1e-4f;
constexpr float kLog2e = 1.4426950408889634f;

// Device-resident scalars of one context (written by kernels, read back by sync calls).
struct DevScalars {
    unsigned long long n_pairs;
    unsigned long long e_eval;
    unsigned long long e_comp;
    unsigned int max_tile;
    unsigned int overflow;
    unsigned int count_c;     // fused-L1 mask counts (normalize = 1)
    unsigned int count_d;
    unsigned int fin_ticket;  // k_pose_finalize last-block ticket (self-resetting)
    unsigned int radix_count; // entries in the radix-sort work list (Ctx::tile_flag)
    unsigned int chunk_count; // chunks of long tiles planned by plan_tile (Ctx::chunk_list)
    unsigned int chunk_next;  // their dynamic fetch cursor
    unsigned int ssim_ticket; // k_ssim_moments last-block ticket (self-resetting)
};

enum Stage { kProject = 0, kScan, kEmit, kSort, kCompFwd, kL1Count, kCompBwd, kFinalize, kInstantiate,
             kPoseAdam, kKfPose, kSsim, kDensify, kVisibility, kNumStages };

struct ProfEvent {
    int stage;
    cudaEvent_t a, b;
};

// Host-side context (opaque to ABI users).
struct Ctx {
    int device = 0;
    int num_sms = 148;
    int64_t max_gaussians = 0;
    int32_t max_w = 0, max_h = 0;
    int64_t max_pairs = 0;
    int32_t max_tiles = 0;
    // scratch (device)
    float4 *proj = nullptr;          // (u, v, z, ±σ) per Gaussian, −σ ⇔ σ clamped
    uint2 *rect = nullptr;           // (x0 | x1<<16, y0 | y1<<16)
    float *thr = nullptr;            // packed (D_c, D_clamp): exact α decision thresholds in d² (composite_common.cuh)
    uint32_t *tile_count = nullptr;  // [max_tiles]
    uint32_t *tile_start = nullptr;  // [max_tiles + 1]
    uint32_t *tile_cursor = nullptr; // [max_tiles]
    uint32_t *tile_flag = nullptr;   // [2·max_tiles] work lists: radix sort (> 8192 / degenerate) | 4097..8192
    uint32_t *keys = nullptr;        // bucket: z bits   [max_pairs]
    uint32_t *vals = nullptr;        // bucket: gid      [max_pairs] — sorted in place
    uint8_t *pbits = nullptr;        // bucket: the 8 sub-tiles of its tile the pair's rect touches [max_pairs]
    uint32_t *keys2 = nullptr;       // fallback sort scratch [max_pairs]
    uint32_t *vals2 = nullptr;
    uint32_t *offs = nullptr;        // fallback sort ranks [max_pairs]
    uint32_t *chunk_list = nullptr;  // the long-tile plans' chunk descriptors, 12 u32 each [12·(max_pairs/2048 + max_tiles + 1)]
    uint32_t *sub_masks = nullptr;   // per sub-list entry: the pixels that composited it (forward → backward) [8·max_pairs]
    uint32_t *sub_lists = nullptr;   // per tile 8 sub-lists (4×8 sub-tiles), capacity 8·n_tile [8·max_pairs]
    uint32_t *sub_count = nullptr;   // [8·max_tiles]
    float *T_final = nullptr;        // per pixel
    uint32_t *last = nullptr;        // per pixel: 1 + sub-list position of the last composited entry
    double *partials = nullptr;      // per sub-tile warp: 12 pose accumulators + loss + pad (16)
    float *ssim_abc = nullptr;       // SSIM chain factors a, b, c × 3 channels per pixel [9 · px]
    double *ssim_partials = nullptr; // per-CTA Σ SSIM
    DevScalars *dev = nullptr;
    float *host_io = nullptr;        // step_host device staging (targets + pose)
    uint8_t *sensor_io = nullptr;    // step_host_sensor upload staging (rgb8 | depth16)
    cudaStream_t copy_stream = nullptr;  // step_host: target upload overlapped with the forward
    cudaEvent_t ev_ready = nullptr, ev_copied = nullptr;
    float *host_ret = nullptr;   // step_host: pinned landing buffer of the loss / d_pose / overflow read-back (16 floats)
    vtgs_pose *view_copy = nullptr;  // the forward's view pose, copied on the device for the backward
    unsigned long long *det = nullptr;  // VTGS_GRAD_DETERMINISTIC fixed-point accumulators [det_cap][5]
    int64_t det_cap = 0;
    // remembered forward
    bool have_fwd = false;
    const float4 *pos_rad = nullptr;
    const float4 *col_opa = nullptr;
    int64_t N = 0;
    const vtgs_pose *view = nullptr;
    vtgs_intrinsics intr{};
    float *color = nullptr, *depth = nullptr, *sil = nullptr;
    char last_error[512] = {0};
    // launch accounting / optional per-stage event timing
    int64_t launches = 0;
    bool profiling = false;
    bool count_work = true;           // forward work counters e_eval / e_comp (vtgs_set_work_counters)
    std::vector<ProfEvent> prof;      // recorded since the last vtgs_get_profile
    std::vector<ProfEvent> prof_free; // reusable event pairs
    int64_t prof_counts[kNumStages] = {0};
};

// Bracket one kernel launch: counts it and, when profiling, records events around it.
struct LaunchScope {
    Ctx *c;
    int stage;
    cudaStream_t s;
    ProfEvent ev{};
    LaunchScope(Ctx *c_, int stage_, cudaStream_t s_) : c(c_), stage(stage_), s(s_) {
        if (!c) return;
        ++c->launches;
        ++c->prof_counts[stage];
        if (c->profiling) {
            if (!c->prof_free.empty()) {
                ev = c->prof_free.back();
                c->prof_free.pop_back();
            } else {
                cudaEventCreate(&ev.a);
                cudaEventCreate(&ev.b);
            }
            ev.stage = stage;
            cudaEventRecord(ev.a, s);
        }
    }
    ~LaunchScope() {
        if (c && c->profiling) {
            cudaEventRecord(ev.b, s);
            c->prof.push_back(ev);
        }
    }
};

// ------------------------------------------------------------------------------------------
// Rotation of a camera-to-world pose, computed in fp64 with explicit rounding, rounded once to
// fp32 (DESIGN.md §3 step 1; the oracle's `rotation`).
// ------------------------------------------------------------------------------------------
struct PoseR {
    float R[9];      // row-major, fp32-rounded
    float t[3];
    double qhat[4];  // normalised quaternion (fp64)
    double qnorm;
};

__device__ __forceinline__ void pose_rotation(const vtgs_pose &p, PoseR &o) {
    double w = (double)p.q[0], x = (double)p.q[1], y = (double)p.q[2], z = (double)p.q[3];
    double n2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w, w), __dmul_rn(x, x)), __dmul_rn(y, y)),
                          __dmul_rn(z, z));
    double n = __dsqrt_rn(n2);
    w = __ddiv_rn(w, n); x = __ddiv_rn(x, n); y = __ddiv_rn(y, n); z = __ddiv_rn(z, n);
    const double xx = __dmul_rn(x, x), yy = __dmul_rn(y, y), zz = __dmul_rn(z, z);
    const double xy = __dmul_rn(x, y), xz = __dmul_rn(x, z), yz = __dmul_rn(y, z);
    const double wx = __dmul_rn(w, x), wy = __dmul_rn(w, y), wz = __dmul_rn(w, z);
    double M[9];
    M[0] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(yy, zz)));
    M[1] = __dmul_rn(2.0, __dsub_rn(xy, wz));
    M[2] = __dmul_rn(2.0, __dadd_rn(xz, wy));
    M[3] = __dmul_rn(2.0, __dadd_rn(xy, wz));
    M[4] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(xx, zz)));
    M[5] = __dmul_rn(2.0, __dsub_rn(yz, wx));
    M[6] = __dmul_rn(2.0, __dsub_rn(xz, wy));
    M[7] = __dmul_rn(2.0, __dadd_rn(yz, wx));
    M[8] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(xx, yy)));
#pragma unroll
    for (int i = 0; i < 9; ++i) o.R[i] = __double2float_rn(M[i]);
    o.t[0] = p.t[0]; o.t[1] = p.t[1]; o.t[2] = p.t[2];
    o.qhat[0] = w; o.qhat[1] = x; o.qhat[2] = y; o.qhat[3] = z;
    o.qnorm = n;
}

// Camera-space centre X_c = Rᵀ(X_w − t), Rᵀ applied explicitly (DESIGN.md §3 step 3).
__device__ __forceinline__ void view_transform(const float *R, const float *t, float4 pr, float xc[3]) {
    const float d0 = __fsub_rn(pr.x, t[0]), d1 = __fsub_rn(pr.y, t[1]), d2 = __fsub_rn(pr.z, t[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
        xc[a] = __fadd_rn(__fadd_rn(__fmul_rn(R[a], d0), __fmul_rn(R[3 + a], d1)), __fmul_rn(R[6 + a], d2));
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ unsigned lane_id() {
    unsigned l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ------------------------------------------------------------------------------------------
// kernel launchers (defined in the .cu files)
// ------------------------------------------------------------------------------------------
cudaError_t launch_instantiate(Ctx &c, const float *depth, const float *rgb, const vtgs_pose *poses, int K,
                               vtgs_intrinsics intr, const float *opacity, float opacity_default,
                               float4 *pos_rad, float4 *col_opa, int64_t *n_valid, cudaStream_t s);
cudaError_t launch_forward(Ctx &c, cudaStream_t s);
cudaError_t launch_backward(Ctx &c, const float *dC, const float *dD, const float *dS,
                            const vtgs_l1_loss *loss, uint32_t want, int64_t learn_begin,
                            int64_t learn_end, float4 *d_col_opa, float *d_radius, float4 *d_position,
                            float *d_pose, float *loss_out, cudaStream_t s);
cudaError_t launch_keyframe_pose_grad(Ctx &c, const float4 *pos_rad, const float4 *d_position,
                                      const vtgs_pose *kf_poses, int K, int64_t spk, float *d_kf, cudaStream_t s);
cudaError_t forward_set_attributes();
cudaError_t backward_set_attributes();
cudaError_t launch_composite_fwd(Ctx &c, cudaStream_t s);
cudaError_t ssim_set_constants();
cudaError_t launch_visibility(Ctx &c, const float *depth, const vtgs_pose *pose, const float *ref_depth,
                              const vtgs_pose *ref_poses, int R, vtgs_intrinsics intr, float tol, uint8_t *mask,
                              int64_t *n_vis, cudaStream_t s);
cudaError_t launch_visibility_counts(Ctx &c, const float *depth, const vtgs_pose *pose, const float *ref_depth,
                                     const vtgs_pose *ref_poses, int R, vtgs_intrinsics intr, float tol,
                                     int64_t *counts, int64_t *n_valid, cudaStream_t s);
cudaError_t launch_densify(Ctx &c, const float *depth, const float *rgb, const vtgs_pose *pose, vtgs_intrinsics intr,
                           const float *sil, float thr, const float *opacity, float opacity_default,
                           float4 *pos_rad, float4 *col_opa, int64_t *n_new, cudaStream_t s);
cudaError_t launch_sensor_targets(Ctx &c, const uint8_t *rgb8, const uint16_t *d16, float scale, int64_t px,
                                  float *rgb, float *depth, cudaStream_t s);
cudaError_t launch_ssim(Ctx &c, const float *color, const float *target, int W, int H, float tau, float *d_color,
                        float *loss_out, cudaStream_t s);
cudaError_t launch_pose_adam(Ctx &c, vtgs_pose *pose, const float *d_pose, float *state, float lr_rot,
                             float lr_trans, cudaStream_t s);

}  // namespace vtgs
