// tcprobe.cu — validates the tcgen05 building blocks the tensor-core E-step
// uses (kind::tf32, K-major no-swizzle shared-memory descriptors, A from
// shared memory (SS) and from TMEM (TS), TMEM st/ld, commit → mbarrier)
// against a CPU reference.  One CTA, 128 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tcprobe tools/tcprobe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// K-major, no swizzle: element (r, k) of an R×8 tf32 operand at
// (r/8)*256 + (k/4)*128 + (r%8)*16 + (k%4)*4 bytes → LBO = 128, SBO = 256.
__host__ __device__ __forceinline__ uint32_t kmaj_off(int r, int k) {
  return (r >> 3) * 256 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_u32(p) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version (sm100)
  return d;                              // base offset 0, lbo mode 0, no swizzle
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__global__ void probe(const float* A, const float* B, const float* B2, float* D1, float* D2,
                      float* D3) {
  __shared__ __align__(1024) uint8_t sa[128 * 8 * 4];
  __shared__ __align__(1024) uint8_t sb[32 * 8 * 4];
  __shared__ __align__(1024) uint8_t sb2[16 * 8 * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 128 * 8; i += 128) {
    const int r = i / 8, k = i % 8;
    *reinterpret_cast<float*>(sa + kmaj_off(r, k)) = A[i];
  }
  for (int i = t; i < 32 * 8; i += 128) {
    const int r = i / 8, k = i % 8;
    *reinterpret_cast<float*>(sb + kmaj_off(r, k)) = B[i];
  }
  for (int i = t; i < 16 * 8; i += 128) {
    const int r = i / 8, k = i % 8;
    *reinterpret_cast<float*>(sb2 + kmaj_off(r, k)) = B2[i];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)),
                 "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // generic-proxy smem writes → visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t lane_base = static_cast<uint32_t>(32 * w) << 16;

  // (1) SS: D1[128×32] = A·Bᵀ at TMEM cols [0,32)
  if (t == 0) {
    const uint64_t da = sdesc(sa, 128, 256), db = sdesc(sb, 128, 256);
    const uint32_t id = idesc_tf32(128, 32);
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
        "l"(da), "l"(db), "r"(id), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tm + lane_base));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) D1[t * 32 + j] = __uint_as_float(r[j]);
  }
  // (2) TS: A (row t = A[t][0..7]) stored to TMEM cols [64,72), D2[128×16] = A·B2ᵀ at cols [32,48)
  {
    uint32_t v[8];
    for (int k = 0; k < 8; ++k) v[k] = __float_as_uint(A[t * 8 + k]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tm + lane_base + 64),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                 "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint64_t db = sdesc(sb2, 128, 256);
    const uint32_t id = idesc_tf32(128, 16);
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 32),
        "r"(tm + 64), "l"(db), "r"(id), "r"(0));
    // (3) accumulate: D3 cols [48,64) = A·B2ᵀ + A·B2ᵀ (second MMA with enable-input-d)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 48),
        "r"(tm + 64), "l"(db), "r"(id), "r"(0));
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 48),
        "r"(tm + 64), "l"(db), "r"(id), "r"(1));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  mbar_wait(&bar, 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t r[16], q[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(tm + lane_base + 32));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]),
          "=r"(q[7]), "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]),
          "=r"(q[14]), "=r"(q[15])
        : "r"(tm + lane_base + 48));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) {
      D2[t * 16 + j] = __uint_as_float(r[j]);
      D3[t * 16 + j] = __uint_as_float(q[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(128));
}

static float tf32_exact(float x) {  // keep 10 mantissa bits (inputs exact in tf32)
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

int main() {
  std::vector<float> A(128 * 8), B(32 * 8), B2(16 * 8);
  srand(7);
  for (auto& v : A) v = tf32_exact((rand() % 2001 - 1000) / 256.f);
  for (auto& v : B) v = tf32_exact((rand() % 2001 - 1000) / 128.f);
  for (auto& v : B2) v = tf32_exact((rand() % 2001 - 1000) / 64.f);
  float *dA, *dB, *dB2, *d1, *d2, *d3;
  cudaMalloc(&dA, 4 * A.size());
  cudaMalloc(&dB, 4 * B.size());
  cudaMalloc(&dB2, 4 * B2.size());
  cudaMalloc(&d1, 4 * 128 * 32);
  cudaMalloc(&d2, 4 * 128 * 16);
  cudaMalloc(&d3, 4 * 128 * 16);
  cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB2, B2.data(), 4 * B2.size(), cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dB2, d1, d2, d3);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> h1(128 * 32), h2(128 * 16), h3(128 * 16);
  cudaMemcpy(h1.data(), d1, 4 * h1.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), d2, 4 * h2.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(h3.data(), d3, 4 * h3.size(), cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0, e3 = 0;
  for (int m = 0; m < 128; ++m) {
    for (int n = 0; n < 32; ++n) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += double(A[m * 8 + k]) * B[n * 8 + k];
      e1 = std::fmax(e1, std::fabs(s - h1[m * 32 + n]));
    }
    for (int n = 0; n < 16; ++n) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += double(A[m * 8 + k]) * B2[n * 8 + k];
      e2 = std::fmax(e2, std::fabs(s - h2[m * 16 + n]));
      e3 = std::fmax(e3, std::fabs(2 * s - h3[m * 16 + n]));
    }
  }
  std::printf("SS  max|err| = %.3e  (D1[0][0]=%g)\n", e1, h1[0]);
  std::printf("TS  max|err| = %.3e  (D2[0][0]=%g)\n", e2, h2[0]);
  std::printf("acc max|err| = %.3e  (D3[0][0]=%g)\n", e3, h3[0]);
  const bool ok = e1 < 1e-3 && e2 < 1e-3 && e3 < 2e-3;
  std::printf("%s\n", ok ? "PASS" : "FAIL");
  return ok ? 0 : 2;
}
