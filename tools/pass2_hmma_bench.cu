// pass2_hmma_bench.cu — prototype of E-step pass 2 with the pair logits on
// the legacy tensor path (mma.sync m16n8k8 tf32, 512 MAC/clk/SM measured),
// MUFU ex2, and the five row sums on FFMA2 in the accumulator-fragment
// layout.  Measures cycles per 64 pairs per SMSP (the current FFMA2 loop:
// 26.7, profiles/r1_loopbench.txt) and the logit error against fp64.
//
// Logit of (row m, column n) in the centred frame, with the row's |v|²
// factored out (as estep_row_kernel): L' = 2v·u + (b − |u|²).  K = 16:
//   A[m] = [vxh, vxh, vxl, vyh, vyh, vyl, vzh, vzh, vzl, 1, 1, 0, 0, 0, 0, 0]   (2v split)
//   B[n] = [uxh, uxl, uxh, uyh, uyl, uyh, uzh, uzl, uzh, ch, cl, 0, 0, 0, 0, 0]   (c = b − |u|²)
// so A·B = Σ (hi·hi + hi·lo + lo·hi) + c_hi + c_lo.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pass2_hmma_bench tools/pass2_hmma_bench.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

__device__ __forceinline__ unsigned tf32_of(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0,
                                         unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int kCols = 256;      // staged scene points per CTA (shared memory)
constexpr int kReps = 64;       // passes over the staged points

struct Feat {  // per column: B fragment words by t (k = t, t+4, 8+t, 12+t) and sums features
  unsigned bf[kCols / 8][4][4];  // [tile][t][j]
};

// rows: v (x,y,z) per row; cols: u (x,y,z), c per column
template <int kRowTiles, int kWarps, int kMinBlocks, int kUnroll>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
    pass2_hmma(const float4* __restrict__ rows, const float4* __restrict__ cols, int nrows,
               float* __restrict__ out, long long* cycles, float* __restrict__ logits_out) {
  __shared__ unsigned bfrag[kCols / 8][4][8][4];   // [tile][t][g][j]
  __shared__ float4 feat[kCols / 8][8];            // [tile][col in tile] (ux, uy, uz, |u|²)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // stage columns: B fragments (split) and the accumulation features
  for (int n = tid; n < kCols; n += blockDim.x) {
    const float4 u = cols[n];
    float bv[16] = {};
    float comp[3] = {u.x, u.y, u.z};
    for (int c = 0; c < 3; ++c) {
      const float h = __uint_as_float(tf32_of(comp[c]));
      const float l = __uint_as_float(tf32_of(comp[c] - h));
      bv[3 * c] = h;
      bv[3 * c + 1] = l;
      bv[3 * c + 2] = h;
    }
    const float ch = __uint_as_float(tf32_of(u.w));
    bv[9] = ch;
    bv[10] = __uint_as_float(tf32_of(u.w - ch));
    const int tile = n >> 3, gg = n & 7;
    for (int tt = 0; tt < 4; ++tt)
      for (int j = 0; j < 4; ++j) bfrag[tile][tt][gg][j] = __float_as_uint(bv[tt + 4 * j]);
    feat[tile][gg] = make_float4(u.x, u.y, u.z, u.x * u.x + u.y * u.y + u.z * u.z);
  }
  // A fragments of the warp's row tiles (2 mma: k 0..7, 8..15)
  unsigned a[kRowTiles][2][4];
  for (int rt = 0; rt < kRowTiles; ++rt) {
    float av[2][16];
    for (int h = 0; h < 2; ++h) {
      const int r = (warp * kRowTiles + rt) * 16 + g + 8 * h;
      const float4 v = rows[r % nrows];
      const float comp[3] = {2.f * v.x, 2.f * v.y, 2.f * v.z};
      for (int k = 0; k < 16; ++k) av[h][k] = 0.f;
      for (int c = 0; c < 3; ++c) {
        const float hh = __uint_as_float(tf32_of(comp[c]));
        const float ll = __uint_as_float(tf32_of(comp[c] - hh));
        av[h][3 * c] = hh;
        av[h][3 * c + 1] = hh;
        av[h][3 * c + 2] = ll;
      }
      av[h][9] = 1.f;
      av[h][10] = 1.f;
    }
    for (int mm = 0; mm < 2; ++mm) {
      a[rt][mm][0] = __float_as_uint(av[0][8 * mm + t]);
      a[rt][mm][1] = __float_as_uint(av[1][8 * mm + t]);
      a[rt][mm][2] = __float_as_uint(av[0][8 * mm + t + 4]);
      a[rt][mm][3] = __float_as_uint(av[1][8 * mm + t + 4]);
    }
  }
  __syncthreads();
  // accumulators: per row tile, rows g and g+8, packed over the column pair
  float2 s0[kRowTiles][2], sx[kRowTiles][2], sy[kRowTiles][2], sz[kRowTiles][2], sv[kRowTiles][2];
  for (int rt = 0; rt < kRowTiles; ++rt)
    for (int h = 0; h < 2; ++h)
      s0[rt][h] = sx[rt][h] = sy[rt][h] = sz[rt][h] = sv[rt][h] = make_float2(0.f, 0.f);
  const long long c0 = clock64();
  for (int rep = 0; rep < kReps; ++rep) {
#pragma unroll kUnroll
    for (int tile = 0; tile < kCols / 8; ++tile) {
      const uint4 bb = *reinterpret_cast<const uint4*>(&bfrag[tile][t][g][0]);
      const float4 f0 = feat[tile][2 * t], f1 = feat[tile][2 * t + 1];
      const float2 Ux = make_float2(f0.x, f1.x), Uy = make_float2(f0.y, f1.y);
      const float2 Uz = make_float2(f0.z, f1.z), Uq = make_float2(f0.w, f1.w);
#pragma unroll
      for (int rt = 0; rt < kRowTiles; ++rt) {
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        mma_tf32(d, a[rt][0], bb.x, bb.y);
        mma_tf32(d, a[rt][1], bb.z, bb.w);
        if (logits_out && rep == 0) {
          float* o = logits_out + ((blockIdx.x * kWarps + warp) * kRowTiles + rt) * 16 * kCols;
          o[g * kCols + tile * 8 + 2 * t] = d[0];
          o[g * kCols + tile * 8 + 2 * t + 1] = d[1];
          o[(g + 8) * kCols + tile * 8 + 2 * t] = d[2];
          o[(g + 8) * kCols + tile * 8 + 2 * t + 1] = d[3];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          // (a real kernel subtracts the row's shift; here L' ≤ ~0 by construction)
          const float2 w = make_float2(ex2f(d[2 * h]), ex2f(d[2 * h + 1]));
          s0[rt][h] = __fadd2_rn(s0[rt][h], w);
          sx[rt][h] = __ffma2_rn(w, Ux, sx[rt][h]);
          sy[rt][h] = __ffma2_rn(w, Uy, sy[rt][h]);
          sz[rt][h] = __ffma2_rn(w, Uz, sz[rt][h]);
          sv[rt][h] = __ffma2_rn(w, Uq, sv[rt][h]);
        }
      }
    }
  }
  const long long c1 = clock64();
  float acc = 0.f;
  for (int rt = 0; rt < kRowTiles; ++rt)
    for (int h = 0; h < 2; ++h)
      acc += s0[rt][h].x + s0[rt][h].y + sx[rt][h].x + sy[rt][h].y + sz[rt][h].x + sv[rt][h].y;
  out[blockIdx.x * blockDim.x + tid] = acc;
  if (tid == 0) cycles[blockIdx.x] = c1 - c0;
}

template <int RT, int W, int MB, int UN>
void run(const char* name, int sms, const float4* dr, const float4* dc, int nrows, float* dout,
         long long* dcyc) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass2_hmma<RT, W, MB, UN>, W * 32, 0);
  const int blocks = sms * occ * 4;
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    pass2_hmma<RT, W, MB, UN><<<blocks, W * 32>>>(dr, dc, nrows, dout, dcyc, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double pairs = double(blocks) * W * RT * 128.0 * (kCols / 8) * kReps;
  const double ps = pairs / (best * 1e-3);
  std::printf("%-22s occ=%d warps/SM=%2d  %.3f ms  %.3g pairs/s  %.1f cycles/64 pairs/SMSP @1965  %s\n",
              name, occ, occ * W, best, ps, 64.0 / (ps / (sms * 4.0 * 1.965e9)),
              cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nrows = 8192;
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(-2.f, 2.f), B(-8.f, 0.f);
  std::vector<float4> hr(nrows), hc(kCols);
  for (auto& r : hr) r = make_float4(U(rng), U(rng), U(rng), 0.f);
  // c = b − |u|² chosen so that L' = 2v·u + c ranges over [-40, 0]
  for (auto& c : hc) {
    const float ux = U(rng), uy = U(rng), uz = U(rng);
    c = make_float4(ux, uy, uz, B(rng) - 4.f * (std::fabs(ux) + std::fabs(uy) + std::fabs(uz)));
  }
  float4 *dr, *dc;
  float *dout, *dlog;
  long long* dcyc;
  cudaMalloc(&dr, sizeof(float4) * nrows);
  cudaMalloc(&dc, sizeof(float4) * kCols);
  cudaMemcpy(dr, hr.data(), sizeof(float4) * nrows, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, hc.data(), sizeof(float4) * kCols, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, sizeof(float) * sms * 64 * 1024);
  cudaMalloc(&dcyc, sizeof(long long) * sms * 64);
  constexpr int kWarps = 4, kRowTiles = 4;
  const size_t nlog = static_cast<size_t>(kWarps) * kRowTiles * 16 * kCols;
  cudaMalloc(&dlog, sizeof(float) * nlog);
  // precision run (one block's logits vs fp64)
  pass2_hmma<4, 4, 2, 2><<<1, 4 * 32>>>(dr, dc, nrows, dout, dcyc, dlog);
  cudaDeviceSynchronize();
  std::vector<float> lg(nlog);
  cudaMemcpy(lg.data(), dlog, sizeof(float) * lg.size(), cudaMemcpyDeviceToHost);
  double maxerr = 0.0, maxerr_f32 = 0.0, bias = 0.0;
  for (int r = 0; r < kWarps * kRowTiles * 16; ++r)
    for (int n = 0; n < kCols; ++n) {
      const float4 v = hr[r % nrows], u = hc[n];
      const double ref = 2.0 * (double(v.x) * u.x + double(v.y) * u.y + double(v.z) * u.z) + u.w;
      float f = std::fmaf(2.f * v.x, u.x, u.w);
      f = std::fmaf(2.f * v.y, u.y, f);
      f = std::fmaf(2.f * v.z, u.z, f);
      const double e = lg[static_cast<size_t>(r) * kCols + n] - ref;
      maxerr = std::max(maxerr, std::fabs(e));
      maxerr_f32 = std::max(maxerr_f32, std::fabs(f - ref));
      bias += e;
    }
  std::printf("logit |err| max: hmma %.3g  fp32-ffma %.3g  (log2 units; mean hmma err %.3g)\n",
              maxerr, maxerr_f32, bias / (double(kWarps) * kRowTiles * 16.0 * kCols));
  run<4, 4, 2, 2>("rt4 w4 mb2 un2", sms, dr, dc, nrows, dout, dcyc);
  run<4, 4, 2, 1>("rt4 w4 mb2 un1", sms, dr, dc, nrows, dout, dcyc);
  run<2, 4, 3, 2>("rt2 w4 mb3 un2", sms, dr, dc, nrows, dout, dcyc);
  run<2, 8, 2, 2>("rt2 w8 mb2 un2", sms, dr, dc, nrows, dout, dcyc);
  run<2, 8, 2, 4>("rt2 w8 mb2 un4", sms, dr, dc, nrows, dout, dcyc);
  run<1, 8, 3, 4>("rt1 w8 mb3 un4", sms, dr, dc, nrows, dout, dcyc);
  run<1, 16, 1, 4>("rt1 w16 mb1 un4", sms, dr, dc, nrows, dout, dcyc);
  run<1, 4, 6, 8>("rt1 w4 mb6 un8", sms, dr, dc, nrows, dout, dcyc);
  return 0;
}
