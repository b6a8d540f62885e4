// Microbenchmark: global float4 / float RED throughput on distinct, scattered addresses,
// and shared-memory float atomicAdd (CAS loop) throughput.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>
#include <random>

__global__ void red4(float4* g, float* r, const unsigned* idx, int n, int reps) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned k = idx[i];
    for (int t = 0; t < reps; ++t) {
      atomicAdd(&g[k], make_float4(1.f, 2.f, 3.f, 4.f));
      atomicAdd(&r[k], 1.f);
    }
  }
}
__global__ void red1(float* r, const unsigned* idx, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(&r[idx[i]], 1.f);
}
__global__ void st4(float4* g, const unsigned* idx, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) g[idx[i]] = make_float4(1.f, 2.f, 3.f, 4.f);
}
__global__ void smem_cas(float* out, int iters) {
  __shared__ float s[1280];
  for (int i = threadIdx.x; i < 1280; i += blockDim.x) s[i] = 0;
  __syncthreads();
  for (int t = 0; t < iters; ++t) atomicAdd(&s[(threadIdx.x * 5 + t * 37) % 1280], 1.0f);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
int main() {
  const int N = 4000000, M = 14000000;
  std::vector<unsigned> h(M);
  std::mt19937 rng(1);
  for (int i = 0; i < M; ++i) h[i] = rng() % N;
  unsigned* idx; float4* g; float* r;
  cudaMalloc(&idx, M * 4); cudaMalloc(&g, N * 16); cudaMalloc(&r, N * 4);
  cudaMemcpy(idx, h.data(), M * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a); red4<<<148 * 8, 256>>>(g, r, idx, M, 1); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("red float4+float: %d pairs  %.3f ms  -> %.1f G RED/s\n", M, ms, 2.0 * M / ms / 1e6);
    cudaEventRecord(a); red1<<<148 * 8, 256>>>(r, idx, M); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("red float: %d  %.3f ms  -> %.1f G RED/s\n", M, ms, 1.0 * M / ms / 1e6);
    cudaEventRecord(a); st4<<<148 * 8, 256>>>(g, idx, M); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("scattered st.v4: %d  %.3f ms  -> %.1f G st/s\n", M, ms, 1.0 * M / ms / 1e6);
    float* o; cudaMalloc(&o, 148 * 8 * 4);
    cudaEventRecord(a); smem_cas<<<148 * 8, 256>>>(o, 64); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("smem CAS atomicAdd: %.3f ms -> %.1f G/s chip (%.2f per SM-cycle at 1.9GHz)\n", ms, 148.0 * 8 * 256 * 64 / ms / 1e6,
           148.0 * 8 * 256 * 64 / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
