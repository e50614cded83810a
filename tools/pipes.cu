// pipes.cu — microbenchmark of the pipes that bound the E-step on B200:
// MUFU.EX2, FFMA, FFMA2 (f32x2), FADD, mixed.  Reports lane-ops/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipes tools/pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void k_ex2(float* out, float a) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = a * (threadIdx.x + i) * 1e-6f;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ex2(-v[i]);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, float a, float b) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fmaf_rn(v[i], a, b);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = make_float2(threadIdx.x + i, threadIdx.x - i);
  const float2 aa = make_float2(a, a), bb = make_float2(b, b);
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ffma2_rn(v[i], aa, bb);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i].x + v[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fadd(float* out, float a) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(v[i], a);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 1 ex2 + 7 fp32 ops (pass-1 mix)
__global__ void k_mix(float* out, float a) {
  float v[8], acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[i] = (threadIdx.x + i) * 1e-3f; acc[i] = 0.f; }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float dx = v[i] - a, dy = v[i] - 2 * a, dz = v[i] - 3 * a;
      const float t = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
      acc[i] += ex2(-t);
      v[i] += 1e-7f;
    }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double run(const char* name, F launch, double ops_per_thread_iter, int sms, float* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double threads = double(sms) * 8 * 256;
  const double ops = 5.0 * threads * kIters * ops_per_thread_iter;
  const double per_s = ops / (ms * 1e-3);
  std::printf("%-8s %10.3f ms  %.3e lane-ops/s  %.1f lane-ops/clk/SM @%d MHz(attr)\n", name,
              ms / 5, per_s, per_s / (sms * clk_khz * 1e3), clk_khz / 1000);
  return per_s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  dim3 g(sms * 8), blk(256);
  run("ex2", [&] { k_ex2<<<g, blk>>>(out, 1.0f); }, 8, sms, out);
  run("ffma", [&] { k_ffma<<<g, blk>>>(out, 0.999f, 0.5f); }, 8, sms, out);
  run("ffma2", [&] { k_ffma2<<<g, blk>>>(out, 0.999f, 0.5f); }, 16, sms, out);
  run("fadd", [&] { k_fadd<<<g, blk>>>(out, 0.5f); }, 8, sms, out);
  run("mix1+7", [&] { k_mix<<<g, blk>>>(out, 0.25f); }, 8, sms, out);  // pairs
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
