// Measurement hook: the FP32 FMA and MUFU ex2 peaks of this GPU, measured.  The
// compositing kernels are bound by plain FP32 / SFU arithmetic; MEASURED_PEAKS.json carries only
// the HBM copy bandwidth and the bf16 tensor rate, so the roofline denominators for the ALU-bound
// kernels come from these two microbenchmarks, run in the same process as the bench.
#include "vtgs_internal.cuh"

namespace vtgs {

constexpr int kPeakChains = 8;      // independent dependency chains per thread (hide the 4-cycle latency)
constexpr int kPeakIters = 4096;

__global__ void __launch_bounds__(256) k_fma_peak(float *out, float a, float b) {
    float x[kPeakChains];
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) x[c] = (float)(threadIdx.x + c);
    for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
        for (int c = 0; c < kPeakChains; ++c) x[c] = fmaf(x[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) s += x[c];
    if (s == 1.2345f) out[0] = s;   // keep the chains alive
}

__global__ void __launch_bounds__(256) k_ex2_peak(float *out, float a) {
    float x[kPeakChains];
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) x[c] = -1e-3f * (float)(threadIdx.x + c);
    for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
        for (int c = 0; c < kPeakChains; ++c) x[c] = fast_exp2(x[c]) * a;   // one MUFU.EX2 + one FMUL
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) s += x[c];
    if (s == 1.2345f) out[0] = s;
}

}  // namespace vtgs

extern "C" VTGS_API vtgs_status vtgs_measure_peaks(int32_t device, double *fp32_tflops, double *ex2_per_s) {
    if (!fp32_tflops || !ex2_per_s) return VTGS_ERR_INVALID_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return VTGS_ERR_NO_DEVICE;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return VTGS_ERR_INVALID_ARG;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float *out = nullptr;
    cudaEvent_t e0, e1;
    cudaError_t e = cudaMalloc(&out, sizeof(float));
    if (!e) e = cudaEventCreate(&e0);
    if (!e) e = cudaEventCreate(&e1);
    const int blocks = sms * 8;   // 8 × 256 threads per SM: 64 warps, every scheduler busy
    double best_f = 0.0, best_x = 0.0;
    for (int rep = 0; rep < 4 && !e; ++rep) {
        vtgs::k_fma_peak<<<blocks, 256>>>(out, 0.999f, 0.001f);
        cudaEventRecord(e0);
        vtgs::k_fma_peak<<<blocks, 256>>>(out, 0.999f, 0.001f);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        float ms = 0.f;
        if (!e) e = cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * blocks * 256.0 * vtgs::kPeakIters * vtgs::kPeakChains;
        if (!e && ms > 0.f) best_f = fmax(best_f, flops / (ms * 1e-3) / 1e12);
        vtgs::k_ex2_peak<<<blocks, 256>>>(out, 0.999f);
        cudaEventRecord(e0);
        vtgs::k_ex2_peak<<<blocks, 256>>>(out, 0.999f);
        cudaEventRecord(e1);
        if (!e) e = cudaEventSynchronize(e1);
        if (!e) e = cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * 256.0 * vtgs::kPeakIters * vtgs::kPeakChains;
        if (!e && ms > 0.f) best_x = fmax(best_x, ops / (ms * 1e-3));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaSetDevice(prev);
    *fp32_tflops = best_f;
    *ex2_per_s = best_x;
    return e ? VTGS_ERR_CUDA : VTGS_OK;
}
