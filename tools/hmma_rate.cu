// Legacy warp-level tensor-core throughput on sm_100a (mma.sync, HMMA SASS):
// m16n8k8 tf32 and m16n8k16 bf16, fp32 accumulate, 4 independent
// accumulator chains per warp.  Reports MAC/clk/SM.  Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hmma_rate tools/hmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void tf32_kernel(float* out, long long* cycles) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b0 = a0 * 11u, b1 = a0 * 13u;
  float c[4][4] = {};
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const long long t1 = clock64();
  float s = 0.f;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void bf16_kernel(float* out, long long* cycles) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b0 = a0 * 11u, b1 = a0 * 13u;
  float c[4][4] = {};
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const long long t1 = clock64();
  float s = 0.f;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// Rounding of the fp32 accumulation: C = 1 + p repeated, p a fraction of
// ulp(1) = 2^-23 carried by one nonzero product per MMA.
__global__ void round_kernel(float frac, int reps, float* out) {
  const int lane = threadIdx.x, g = lane >> 2, t4 = lane & 3;
  // A row-major 16×8: a0=(g,t4) a1=(g+8,t4) a2=(g,t4+4) a3=(g+8,t4+4); B col: b0=(t4,g) b1=(t4+4,g)
  const float a0 = (g == 0 && t4 == 0) ? 1.f : 0.f;
  const float b0 = (t4 == 0 && g == 0) ? frac * 0x1p-23f : 0.f;
  float c0 = (g == 0 && t4 == 0) ? 1.f : 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  for (int i = 0; i < reps; ++i)
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c0), "+f"(c1), "+f"(c2), "+f"(c3)
        : "r"(__float_as_uint(a0)), "r"(0u), "r"(0u), "r"(0u), "r"(__float_as_uint(b0)), "r"(0u));
  if (lane == 0) out[0] = c0;
}

int main() {
  {
    float* o;
    cudaMalloc(&o, sizeof(float));
    for (float frac : {0.25f, 0.5f, 0.75f, 1.0f, 1.5f}) {
      round_kernel<<<1, 32>>>(frac, 1000, o);
      float h = 0.f;
      cudaMemcpy(&h, o, sizeof h, cudaMemcpyDeviceToHost);
      std::printf("accumulate 1000 x %.2f ulp onto 1.0: C-1 = %.1f ulp (RN: %s)\n", frac,
                  (h - 1.0f) / 0x1p-23f,
                  frac < 0.5f ? "0" : frac == 0.5f ? "0 (ties-even)" : frac < 1.f ? "1000" : "1000+");
    }
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  cudaMalloc(&cyc, sizeof(long long) * sms * 8);
  for (int warps : {4, 8, 16, 32}) {
    for (int kind = 0; kind < 2; ++kind) {
      const int threads = 32 * warps;
      auto launch = [&] {
        if (kind == 0) tf32_kernel<<<sms, threads>>>(out, cyc);
        else bf16_kernel<<<sms, threads>>>(out, cyc);
      };
      launch();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      long long c0 = 0;
      cudaMemcpy(&c0, cyc, sizeof c0, cudaMemcpyDeviceToHost);
      const double macs_per_mma = kind == 0 ? 16.0 * 8 * 8 : 16.0 * 8 * 16;
      const double mmas_per_sm = double(warps) * kIters * 4;
      std::printf("%s warps/SM=%2d  %.3f ms  %.1f cycles (CTA 0)  %.0f MAC/clk/SM  (%.1f TFLOP/s dense)  %s\n",
                  kind == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16", warps, ms, double(c0),
                  mmas_per_sm * macs_per_mma / double(c0),
                  2.0 * mmas_per_sm * sms * macs_per_mma / (ms * 1e-3) / 1e12,
                  cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
