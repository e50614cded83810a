// estep_tc.cu — E-step pass 2 with its pair logits on the tensor cores.
//
// Pass 2 needs, per (model row m, scene point n), the logit
//   L_mn = b_n − ‖y'_n − x'_m‖² = log2 P_mn,
// which in the block's centred, scaled frame (u = y' − c, v = x' − c) is a
// dot product of length 5:
//   L_mn = A1_m · B1_n,  A1_m = [2v, 1, −|v|²],  B1_n = [u, b_n − |u|², 1].
// GEMM1 computes L for 256 model rows × 128 scene points per batch on
// tcgen05 (kind::tf32, M = 128 per half, N = 128) into TMEM; the CUDA cores
// then do only what must stay there: w = 2^L on MUFU and the five weighted
// row sums S0, Σw·u, Σw·|u|² (f32x2 FFMA2 with the scene-point operands
// broadcast from shared memory).  The FP32 register-operand traffic that
// bounds the CUDA-core kernel (~28 cycles per 64 pairs per SMSP,
// tools/loopbench.cu) drops to the accumulation (~10), leaving the pass
// MUFU-bound (16).
//
// Exactness: every fp32 component is split into three TF32 pieces
// (x = x0 + x1 + x2 exactly) and the six products with i + j ≤ 2 are packed
// along K (30 of 32 slots, four K=8 steps), smallest first so the fp32
// accumulator rounds once at the scale of L: GEMM1 reproduces the fp32
// centred-form logits (neglected terms ≤ 2^-33 relative).  The centred
// form's own rounding (≈ 4ε·R²) keeps blocks with a large scaled radius R on
// the CUDA-core difference form (the pass-2 list kernel routes each block).
//
// Shape choice: a tf32 tcgen05.mma costs ≥ 44.6 cycles for N ≤ 64 and
// reaches the 2048 MAC/clk rate at N ≥ 128 (tools/tcrate.cu on the B200),
// so the logits go through the tensor core in N = 128 batches and the
// N = 5 weighted sums stay on the CUDA cores.
//
// CTA roles (608 threads, one CTA per SM: all 512 TMEM columns):
//   warps 0–15 compute: warp w serves model rows 32(w%8).. of the 256-row
//              block = TMEM lanes 32(w%4).. of half (w%8)/4; warps w and
//              w+8 take the even / odd 32-point sub-chunks of each batch;
//   warp 16    MMA issue (one thread);
//   warps 17–18 staging: scene tiles → shared memory (double-buffered).
// TMEM holds D1[half][stage] (128 columns each): GEMM1 of batch i+1 runs
// while the compute warps consume batch i.
// Work split: the same persistent stream-K schedule and segment slots as
// the CUDA-core kernel (estep.cu), so the combine is shared.

#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "estep.cuh"

namespace fcpd {

namespace {

constexpr int kTile = kTilePts;
constexpr int kBatch = 128;   // scene points per GEMM1 (N)
constexpr int kSub = 32;      // points per TMEM load (x32)
constexpr int kKPack = 32;    // packed K: 30 split products + 2 zero slots
constexpr int kRowWarps = 8;        // warp w owns rows 32w..32w+31 of the block
constexpr int kComputeWarps = 16;   // two warps per row warp: sub-chunks split even/odd
constexpr int kMmaWarp = kComputeWarps;
constexpr int kStageWarps = 2;
constexpr int kStageThreads = kStageWarps * 32;
constexpr int kThreads = (kComputeWarps + 1 + kStageWarps) * 32;
constexpr float kPadLogit = -1.0e30f;  // padding scene point: 2^L = 0

// shared memory (bytes).  A1 / B1: K-major, no swizzle, K = 32 as 8 chunks
// of 4; element (r, k) at (k/4)·kKChunk + (r/8)·128 + (r%8)·16 + (k%4)·4, so
// LBO (next K chunk) = kKChunk and SBO (next 8 rows) = 128.
constexpr int kKChunk = kTile / 8 * 128;        // 4 KB: one K chunk of 256 rows
constexpr int kA1Bytes = kKPack / 4 * kKChunk;  // 32 KB
constexpr int kB1Bytes = kKPack / 4 * kKChunk;  // 32 KB per buffer
constexpr int kVBytes = kTile / 2 * 32;         // per point pair: 2 float4
constexpr int kOffA1 = 0;
constexpr int kOffB1 = kOffA1 + kA1Bytes;
constexpr int kOffV = kOffB1 + 2 * kB1Bytes;
constexpr int kOffAcc = kOffV + 2 * kVBytes;  // odd sub-group's row sums (fp64)
constexpr int kOffBar = kOffAcc + 5 * kTile * 8;
constexpr int kNumBars = 8;
// > half of the SM's shared memory: exactly one CTA per SM (it owns all
// 512 TMEM columns)
constexpr int kSmemBytes = 120 * 1024;
static_assert(kOffBar + kNumBars * 8 <= kSmemBytes, "shared memory layout");

__device__ __forceinline__ uint32_t col_d1(int h, int s) { return (2 * h + s) * kBatch; }
__device__ __forceinline__ uint32_t kpack_off(int r, int k) {
  return (k >> 2) * kKChunk + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((smem_addr(p) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // sm100 descriptor version; no swizzle
  return d;
}
constexpr uint32_t idesc_tf32(int m, int n) {  // D f32, A/B tf32, both K-major
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void proxy_fence() {  // generic smem writes → tensor core
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                       uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id,
                                       uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_addr(b))
      : "memory");
}

#define FCPD_R32(a) "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), \
    "=r"(a[6]), "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]),  \
    "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]),           \
    "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]),           \
    "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
#define FCPD_W32(a) "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), \
    "r"(a[6]), "r"(a[7]), "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]),   \
    "r"(a[13]), "r"(a[14]), "r"(a[15]), "r"(a[16]), "r"(a[17]), "r"(a[18]),           \
    "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]), "r"(a[24]),           \
    "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31])

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : FCPD_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      FCPD_W32(v)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// TF32 pieces (the tensor core reads the top 19 bits of each operand)
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ void split3(float x, float& a, float& b, float& c) {
  a = tf32_hi(x);
  const float r = __fsub_rn(x, a);  // exact
  b = tf32_hi(r);
  c = tf32_hi(__fsub_rn(r, b));     // exact remainder (≤ 2 bits): x = a + b + c
}
__device__ __forceinline__ void split2(float x, float& a, float& b) {
  a = tf32_hi(x);
  b = tf32_hi(__fsub_rn(x, a));
}

__device__ __forceinline__ float4 scale4(float4 p, float s) {
  return make_float4(__fmul_rn(p.x, s), __fmul_rn(p.y, s), __fmul_rn(p.z, s), p.w);
}

__device__ __forceinline__ int64_t tc_start(int64_t g, int64_t G, int64_t P) { return g * P / G; }

// The tile pieces of a segment [p, pe) of block rb, in schedule order.
struct Piece {
  int64_t base;
  int cnt;
};
__device__ __forceinline__ Piece next_piece(const WorkList& wl, int rb, int64_t& q, int64_t pe,
                                            int64_t n) {
  const int64_t k = q / kTile - wl.off(rb);
  const int a = static_cast<int>(q % kTile);
  const int b = static_cast<int>(min(static_cast<int64_t>(kTile), a + (pe - q)));
  Piece pc;
  pc.base = static_cast<int64_t>(wl.tile(rb, k)) * kTile + a;
  pc.cnt = static_cast<int>(max(int64_t(0), min(static_cast<int64_t>(b - a), n - pc.base)));
  q += b - a;
  return pc;
}

__device__ __forceinline__ int tc_block_of(const WorkList& wl, int64_t u) {
  if (wl.implicit) return static_cast<int>(u / wl.n_other);
  int lo = 0, hi = wl.n_blocks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (wl.offset[mid] <= u) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// The K packing of the split products: slot → (A piece, B piece, component)
// for 5 components; tiny products (i + j = 2) first, then i + j = 1, then
// the main terms, so the accumulator's rounding happens at the scale of L.
__device__ __forceinline__ void kpack(const float (&x)[5][3], bool a_side, float (&out)[kKPack]) {
#pragma unroll
  for (int k = 0; k < kKPack; ++k) out[k] = 0.f;
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    // slots 0–14: (2,0), (1,1), (0,2)
    out[3 * c + 0] = a_side ? x[c][2] : x[c][0];
    out[3 * c + 1] = x[c][1];
    out[3 * c + 2] = a_side ? x[c][0] : x[c][2];
    // slots 16–25: (1,0), (0,1)
    out[16 + 2 * c] = a_side ? x[c][1] : x[c][0];
    out[17 + 2 * c] = a_side ? x[c][0] : x[c][1];
    // slots 26–30: (0,0)
    out[26 + c] = x[c][0];
  }
}

__device__ __forceinline__ void store_kpacked(uint8_t* base, int r, const float (&v)[kKPack]) {
#pragma unroll
  for (int q = 0; q < kKPack / 4; ++q)
    *reinterpret_cast<float4*>(base + kpack_off(r, 4 * q)) =
        make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
    estep_row_tc_kernel(const float4* __restrict__ xt4, int64_t m,
                        const float4* __restrict__ y4b, int64_t n,
                        const IterState* __restrict__ st, WorkList wl,
                        double* __restrict__ seg) {
  if (!st->active) return;
  const int64_t G = gridDim.x, g = blockIdx.x;
  const int64_t P = wl.off(wl.n_blocks) * kTile;
  const int64_t p0 = tc_start(g, G, P), p1 = tc_start(g + 1, G, P);
  if (p0 >= p1) return;  // uniform across the CTA, before any TMEM allocation

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA1 = smem + kOffA1;
  uint8_t* sB1 = smem + kOffB1;
  uint8_t* sV = smem + kOffV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* d1_full = bars + 0;   // [2] commit
  uint64_t* d1_empty = bars + 2;  // [2] 8 compute warps
  uint64_t* s_full = bars + 4;    // [2] staging warps
  uint64_t* s_empty = bars + 6;   // [2] commit (B1) + 8 compute warps (V)
  __shared__ uint32_t tmem_base;
  __shared__ float red[6][kRowWarps];
  __shared__ float3 ctr_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float s = st->sx;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_addr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 2; ++i) {
      bar_init(d1_full + i, 1);
      bar_init(d1_empty + i, kComputeWarps);
      bar_init(s_full + i, kStageWarps);
      bar_init(s_empty + i, 1 + kComputeWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;

  // role-local schedule counters (every role walks the same pieces/batches)
  uint32_t tiles_done = 0, batches_done = 0;
  int rb = tc_block_of(wl, p0 / kTile);
  for (int64_t p = p0; p < p1;) {
    while (wl.off(rb + 1) * kTile <= p) ++rb;
    const int64_t pe = min(p1, wl.off(rb + 1) * kTile);

    // ---- segment setup: own rows, box centre, A1 (K-packed split pieces)
    float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t row = -1;
    if (warp < kRowWarps) {
      row = static_cast<int64_t>(rb) * kTile + 32 * warp + lane;
      float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      if (row < m) {
        xv = scale4(xt4[row], s);
        lo[0] = hi[0] = xv.x;
        lo[1] = hi[1] = xv.y;
        lo[2] = hi[2] = xv.z;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
          hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
      }
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          red[k][warp] = lo[k];
          red[3 + k][warp] = hi[k];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float r[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) r[k] = red[k][0];
      for (int w = 1; w < kRowWarps; ++w) {
#pragma unroll
        for (int k = 0; k < 3; ++k) r[k] = fminf(r[k], red[k][w]);
#pragma unroll
        for (int k = 3; k < 6; ++k) r[k] = fmaxf(r[k], red[k][w]);
      }
      ctr_s = r[0] <= r[3] ? make_float3(0.5f * (r[0] + r[3]), 0.5f * (r[1] + r[4]),
                                         0.5f * (r[2] + r[5]))
                           : make_float3(0.f, 0.f, 0.f);
    }
    __syncthreads();
    const float3 c = ctr_s;
    float vx = 0.f, vy = 0.f, vz = 0.f, vq = 0.f;
    if (warp < kRowWarps) {
      if (row < m) {
        vx = __fsub_rn(xv.x, c.x);
        vy = __fsub_rn(xv.y, c.y);
        vz = __fsub_rn(xv.z, c.z);
        vq = __fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx)));
      }
      const float a[5] = {2.f * vx, 2.f * vy, 2.f * vz, 1.f, -vq};
      float pcs[5][3];
#pragma unroll
      for (int k = 0; k < 5; ++k) split3(a[k], pcs[k][0], pcs[k][1], pcs[k][2]);
      float packed[kKPack];
      kpack(pcs, true, packed);
      store_kpacked(sA1, 32 * warp + lane, packed);  // warp < kRowWarps
      proxy_fence();
    }
    __syncthreads();

    if (warp < kComputeWarps) {
      // ---------------- compute warps: w = 2^L and the five row sums
      const int rw = warp % kRowWarps, sg = warp / kRowWarps;
      const int h = rw >> 2;
      const uint32_t lane_base = static_cast<uint32_t>(32 * (rw & 3)) << 16;
      double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      for (int64_t q = p; q < pe;) {
        const Piece pc = next_piece(wl, rb, q, pe, n);
        if (pc.cnt == 0) continue;
        const int buf = tiles_done & 1;
        const float4* vsrc = reinterpret_cast<const float4*>(sV + buf * kVBytes);
        const int nb = (pc.cnt + kBatch - 1) / kBatch;
        if (nb > 0) bar_wait(s_full + buf, (tiles_done >> 1) & 1);  // V staged
        for (int bi = 0; bi < nb; ++bi, ++batches_done) {
          const int st2 = batches_done & 1;
          bar_wait(d1_full + st2, (batches_done >> 1) & 1);
          tc_fence_after();
          const int left = pc.cnt - bi * kBatch;
          const int nsub = min(kBatch, left + kSub - 1) / kSub;
          float2 f0 = make_float2(0.f, 0.f), fx = f0, fy = f0, fz = f0, fq = f0;
          for (int sc = sg; sc < nsub; sc += 2) {
            uint32_t L[32];
            tmem_ld32(tm + lane_base + col_d1(h, st2) + sc * kSub, L);
            tmem_wait_ld();
            const int pp0 = (bi * kBatch + sc * kSub) >> 1;  // first point pair
#pragma unroll
            for (int j = 0; j < kSub / 2; ++j) {
              const float4 va = vsrc[2 * (pp0 + j)];      // (ux, ux', uy, uy')
              const float4 vb = vsrc[2 * (pp0 + j) + 1];  // (uz, uz', q, q')
              const float2 w = make_float2(ex2_approx(__uint_as_float(L[2 * j])),
                                           ex2_approx(__uint_as_float(L[2 * j + 1])));
              f0 = __fadd2_rn(f0, w);
              fx = __ffma2_rn(w, make_float2(va.x, va.y), fx);
              fy = __ffma2_rn(w, make_float2(va.z, va.w), fy);
              fz = __ffma2_rn(w, make_float2(vb.x, vb.y), fz);
              fq = __ffma2_rn(w, make_float2(vb.z, vb.w), fq);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) bar_arrive(d1_empty + st2);
          acc[0] += static_cast<double>(f0.x) + static_cast<double>(f0.y);
          acc[1] += static_cast<double>(fx.x) + static_cast<double>(fx.y);
          acc[2] += static_cast<double>(fy.x) + static_cast<double>(fy.y);
          acc[3] += static_cast<double>(fz.x) + static_cast<double>(fz.y);
          acc[4] += static_cast<double>(fq.x) + static_cast<double>(fq.y);
        }
        __syncwarp();
        if (lane == 0) bar_arrive(s_empty + buf);  // V of this buffer consumed
        ++tiles_done;
      }
      // the two sub-groups' sums of a row meet in shared memory
      const int li = 32 * rw + lane;
      double* xacc = reinterpret_cast<double*>(smem + kOffAcc);
      if (sg == 1)
#pragma unroll
        for (int k = 0; k < 5; ++k) xacc[k * kTile + li] = acc[k];
      asm volatile("bar.sync 1, %0;" ::"n"(kComputeWarps * 32) : "memory");
      if (sg == 0) {
#pragma unroll
      for (int k = 0; k < 5; ++k) acc[k] += xacc[k * kTile + li];
      // segment out (the CUDA-core kernel's layout): S0, Σw·y', Σw·t
      double* out = seg + (g + rb) * 5 * kTile;
      const double dvx = vx, dvy = vy, dvz = vz, dvq = vq;
      out[li] = acc[0];
      out[kTile + li] = acc[1] + static_cast<double>(c.x) * acc[0];
      out[2 * kTile + li] = acc[2] + static_cast<double>(c.y) * acc[0];
      out[3 * kTile + li] = acc[3] + static_cast<double>(c.z) * acc[0];
      out[4 * kTile + li] =
          acc[4] + dvq * acc[0] - 2.0 * (dvx * acc[1] + dvy * acc[2] + dvz * acc[3]);
      }
    } else if (warp == kMmaWarp) {
      // ---------------- GEMM1 issue (one thread): D1[h][s] = A1_h · B1(batch)ᵀ
      if (lane == 0) {
        constexpr uint32_t id = idesc_tf32(128, kBatch);
        for (int64_t q = p; q < pe;) {
          const Piece pc = next_piece(wl, rb, q, pe, n);
          if (pc.cnt == 0) continue;
          const int buf = tiles_done & 1;
          const int nb = (pc.cnt + kBatch - 1) / kBatch;
          bar_wait(s_full + buf, (tiles_done >> 1) & 1);
          tc_fence_after();
          for (int bi = 0; bi < nb; ++bi, ++batches_done) {
            const int st2 = batches_done & 1;
            if (batches_done >= 2) {
              bar_wait(d1_empty + st2, ((batches_done >> 1) - 1) & 1);
              tc_fence_after();
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
              for (int ks = 0; ks < kKPack / 8; ++ks) {
                const uint64_t a = sdesc(sA1 + 2 * ks * kKChunk + h * (kTile / 2 / 8) * 128,
                                         kKChunk, 128);
                const uint64_t b = sdesc(sB1 + buf * kB1Bytes + 2 * ks * kKChunk +
                                             bi * (kBatch / 8) * 128,
                                         kKChunk, 128);
                mma_ss(tm + col_d1(h, st2), a, b, id, ks > 0 ? 1u : 0u);
              }
            }
            mma_commit(d1_full + st2);
          }
          mma_commit(s_empty + buf);  // B1 of this buffer consumed
          ++tiles_done;
        }
      }
    } else {
      // ---------------- staging warps: B1 (K-packed split pieces), V pairs
      const int sid = threadIdx.x - (kComputeWarps + 1) * 32;
      for (int64_t q = p; q < pe;) {
        const Piece pc = next_piece(wl, rb, q, pe, n);
        if (pc.cnt == 0) continue;
        const int buf = tiles_done & 1;
        if (tiles_done >= 2) bar_wait(s_empty + buf, ((tiles_done >> 1) - 1) & 1);
        uint8_t* b1 = sB1 + buf * kB1Bytes;
        float* vdst = reinterpret_cast<float*>(sV + buf * kVBytes);
        const int npts = (pc.cnt + kBatch - 1) / kBatch * kBatch;
        for (int k = sid; k < npts; k += kStageThreads) {
          float ux = 0.f, uy = 0.f, uz = 0.f, uq = 0.f, B = kPadLogit;
          if (k < pc.cnt) {
            const float4 y = scale4(y4b[pc.base + k], s);
            ux = __fsub_rn(y.x, c.x);
            uy = __fsub_rn(y.y, c.y);
            uz = __fsub_rn(y.z, c.z);
            uq = __fmaf_rn(uz, uz, __fmaf_rn(uy, uy, __fmul_rn(ux, ux)));
            B = __fsub_rn(y.w, uq);  // b − |u|²
          }
          const float bc[5] = {ux, uy, uz, B, 1.f};
          float pcs[5][3];
#pragma unroll
          for (int j = 0; j < 5; ++j) split3(bc[j], pcs[j][0], pcs[j][1], pcs[j][2]);
          float packed[kKPack];
          kpack(pcs, false, packed);
          store_kpacked(b1, k, packed);
          // V pair layout: pair j = points (2j, 2j+1): (ux,ux',uy,uy'), (uz,uz',q,q')
          float* vp = vdst + (k >> 1) * 8 + (k & 1);
          vp[0] = ux;
          vp[2] = uy;
          vp[4] = uz;
          vp[6] = uq;
        }
        proxy_fence();
        __syncwarp();
        if (lane == 0) bar_arrive(s_full + buf);
        ++tiles_done;
      }
    }
    // every role's counters advanced identically; all MMAs of the segment
    // have completed (compute warps consumed every batch)
    __syncthreads();
    p = pe;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

void estep_row_tc_prepare() {
  FCPD_CUDA(cudaFuncSetAttribute(estep_row_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemBytes));
}

void launch_estep_row_tc(const float4* xt4, int64_t m, const float4* y4b, int64_t n,
                         const IterState* st, const WorkList& wl, double* seg, int grid,
                         cudaStream_t stream) {
  estep_row_tc_kernel<<<grid, kThreads, kSmemBytes, stream>>>(xt4, m, y4b, n, st, wl, seg);
  FCPD_LAUNCH_CHECK();
}

}  // namespace fcpd
