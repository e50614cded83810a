// fp64_rate_bench.cu — FP64 issue rates on this GPU: DFMA (CUDA cores) and
// DMMA (mma.sync m8n8k4 f64 tensor op), both with independent accumulator
// chains, one launch of 148×k CTAs.  Decides how the top-K Φ·V kernel
// (csrc/topk.cu) should be built.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_rate_bench tools/fp64_rate_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, double a0, double b0) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9 + i;
  double a = a0 + threadIdx.x * 1e-12, b = b0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {128, 256, 512}) {
    for (int per_sm : {1, 2, 4}) {
      const int blocks = sms * per_sm;
      dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * blocks * threads * 16.0 * kIters;
      std::printf("DFMA threads %d ctas/sm %d: %.2f TFLOP/s\n", threads, per_sm, fl / ms * 1e-9);
      dmma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fm = 2.0 * 256.0 * 8.0 * kIters * blocks * (threads / 32);
      std::printf("DMMA threads %d ctas/sm %d: %.2f TFLOP/s\n", threads, per_sm, fm / ms * 1e-9);
    }
  }
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
