// bulk_stream_bench.cu — HBM read rate of a cp.async.bulk + mbarrier ring as
// a function of the bulk-copy piece size, for the M-step basis streams
// (csrc/mstep.cu rowdot_bulk / colsum_bulk read 32 KB stages as 8 pieces of
// 4 KB from 8 rows of Qᵀ).  A 184 × 800 KB matrix (C4's streamed prefix) is
// read once per launch in 32 KB units, each unit `pieces` pieces from
// `pieces` consecutive rows; consumers sum the stage (LDS.128 + FADD).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bulk_stream_bench tools/bulk_stream_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kStage = 32 * 1024;

__device__ __forceinline__ uint32_t s32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(288) stream_kernel(const float* __restrict__ a, int64_t rows,
                                                     int64_t cols, int pieces, int stages,
                                                     int64_t units, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(s32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t u0 = blockIdx.x * units / gridDim.x, u1 = (blockIdx.x + 1) * units / gridDim.x;
  const int64_t piece_cols = kStage / 4 / pieces;       // floats per piece
  const int64_t col_blocks = cols / piece_cols;
  if (tid >= 256) {
    if (tid != 256) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int64_t u = u0; u < u1; ++u) {
      const int64_t ch = u - u0;
      const int s = static_cast<int>(ch % stages);
      const uint32_t ph = static_cast<uint32_t>((ch / stages) & 1);
      asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(s32(&empty[s])), "r"(ph ^ 1) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])), "r"(kStage) : "memory");
      const int64_t rg = u / col_blocks, cb = u - rg * col_blocks;
      for (int p = 0; p < pieces; ++p) {
        const float* src = a + ((rg * pieces + p) % rows) * cols + cb * piece_cols;
        unsigned char* dst = smem + s * kStage + p * (kStage / pieces);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(s32(dst)), "l"(src), "r"(kStage / pieces), "r"(s32(&full[s])), "l"(pol) : "memory");
      }
    }
    return;
  }
  float acc = 0.f;
  for (int64_t u = u0; u < u1; ++u) {
    const int64_t ch = u - u0;
    const int s = static_cast<int>(ch % stages);
    const uint32_t ph = static_cast<uint32_t>((ch / stages) & 1);
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(s32(&full[s])), "r"(ph) : "memory");
    const float4* st = reinterpret_cast<const float4*>(smem + s * kStage);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 q = st[i * 256 + tid];
      acc += q.x + q.y + q.z + q.w;
    }
    __syncwarp();
    if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
  }
  if (acc == 1234.5f) out[tid] = acc;
}

int main() {
  const int64_t rows = 184, cols = 200704;  // 800 KB rows (multiple of 8192 floats)
  float* a;
  float* out;
  cudaMalloc(&a, rows * cols * 4);
  cudaMalloc(&out, 4096);
  cudaMemset(a, 0, rows * cols * 4);
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = static_cast<double>(rows) * cols * 4;
  for (int ctas : {1, 2}) {
    for (int stages : {2, 3, 4, 5, 6}) {
      if (ctas * stages * kStage > 228 * 1024) continue;
      for (int pieces : {8, 4, 2, 1}) {
        const int64_t units = rows / pieces * (cols / (kStage / 4 / pieces));
        const size_t smem = stages * kStage + 2 * stages * 8;
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemsetAsync(flush, rep, 512 << 20);
          cudaEventRecord(e0);
          stream_kernel<<<sms * ctas, 288, smem>>>(a, rows, cols, pieces, stages, units, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        std::printf("ctas/SM %d stages %d pieces/stage %d (%5d B): %7.1f us  %6.0f GB/s\n", ctas,
                    stages, pieces, kStage / pieces, best * 1e3, bytes / best * 1e-6);
      }
    }
  }
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
