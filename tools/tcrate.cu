// tcrate.cu — issue-rate of tcgen05.mma.kind::tf32 vs shape (M=128, one CTA
// per SM, one issuing thread): cycles per MMA for SS (A, B in smem) and TS
// (A in TMEM) at several N.  Operands are zero (values do not matter).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tcrate tools/tcrate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

template <int N, bool TS, int KSTEPS>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t base = smem_u32(sm);
    const uint32_t id = idesc_tf32(128, N);
    const uint64_t t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < KSTEPS; ++k) {
        const uint64_t b = sdesc(base + 32768 + k * 1024, 128, 256);
        if (TS) {
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tm),
              "r"(tm + 256 + 8 * k), "l"(b), "r"(id), "r"(1));
        } else {
          const uint64_t a = sdesc(base + k * 4096, 128, 256);
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
              "l"(a), "l"(b), "r"(id), "r"(1));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
    asm volatile(
        "{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(
            smem_u32(&bar)));
    const uint64_t t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, bool TS, int KSTEPS>
void run(const char* name, unsigned long long* d, int sms) {
  auto k = rate<N, TS, KSTEPS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  const int iters = 2000;
  k<<<sms, 128, 120 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = double(h) / (double(iters) * KSTEPS);
  std::printf("%-22s N=%3d  %7.1f cycles/MMA  (%5.1f MAC/clk)  %s\n", name, N, per,
              128.0 * N * 8 / per, cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 8 * sms);
  run<16, true, 4>("TS", d, sms);
  run<32, true, 4>("TS", d, sms);
  run<64, true, 4>("TS", d, sms);
  run<128, true, 4>("TS", d, sms);
  run<256, true, 4>("TS", d, sms);
  run<16, false, 4>("SS", d, sms);
  run<32, false, 4>("SS", d, sms);
  run<64, false, 4>("SS", d, sms);
  run<128, false, 4>("SS", d, sms);
  run<256, false, 4>("SS", d, sms);
  return 0;
}
