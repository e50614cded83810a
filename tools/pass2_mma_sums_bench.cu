// pass2_mma_sums_bench.cu — prototype of E-step pass 2 with the five row
// sums on the legacy tensor path: logits on FFMA2 (3 per packed pair of
// pairs, as estep_row_kernel's centred form), ex2 on MUFU, and
//   [S0, Σw·ux, Σw·uy, Σw·uz, Σw·|u|²] = W · F
// as mma.sync m16n8k8 tf32 with a hi/lo split (W_hi·F_hi + W_hi·F_lo +
// W_lo·F_hi, fp32 accumulate): the A fragment of m16n8k8 is exactly the
// (rows g, g+8) × (columns t, t+4) quad each thread computes the logits of.
// Per 64 pairs per SMSP: MUFU 16 cycles, FFMA2 6, HMMA 12 (512 MAC/clk/SM).
// Measures cycles per 64 pairs per SMSP (current FFMA2 loop: 26.7) and the
// error of the sums and of the centred-form variance against fp64, beside
// the FFMA2 loop's.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pass2_mma_sums_bench tools/pass2_mma_sums_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ float tf32_hi(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// hi part by truncation on the integer pipe (cvt.rna.tf32 issues on the
// MUFU/XU pipe the ex2 needs: 33 cycles per 64 pairs with it)
__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}
__device__ __forceinline__ float2 ex2x2(float2 x) {
  float2 y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(x.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(x.y));
  return y;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], float a0, float a1, float a2, float a3,
                                         unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(__float_as_uint(a0)), "r"(__float_as_uint(a1)), "r"(__float_as_uint(a2)),
        "r"(__float_as_uint(a3)), "r"(b0), "r"(b1));
}

constexpr int kCols = 256;  // staged scene points
constexpr int kReps = 64;

// rows: (2vx, 2vy, 2vz, |v|²); cols: (ux, uy, uz, c = b − |u|²)
template <int RT, int W, int MB, int RUN>
__global__ void __launch_bounds__(W * 32, MB)
    pass2_mma(const float4* __restrict__ rows, const float4* __restrict__ cols, int nrows,
              double* __restrict__ sums_out, float* __restrict__ out, int reps) {
  __shared__ float4 ua[kCols], ub[kCols];     // (ux,ux,uy,uy), (uz,uz,c,c)
  __shared__ uint4 bfr[kCols / 8][32];         // per tile, per lane: (F_hi[t][g], F_hi[t+4][g], F_lo…)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  for (int n = tid; n < kCols; n += blockDim.x) {
    const float4 u = cols[n];
    ua[n] = make_float4(u.x, u.x, u.y, u.y);
    ub[n] = make_float4(u.z, u.z, u.w, u.w);
  }
  for (int e = tid; e < (kCols / 8) * 32; e += blockDim.x) {
    const int tile = e / 32, ln = e % 32, gg = ln >> 2, tt = ln & 3;
    auto feat = [&](int n) {  // feature gg of column n
      const float4 u = cols[n];
      const float f[8] = {1.f, u.x, u.y, u.z, u.x * u.x + u.y * u.y + u.z * u.z, 0.f, 0.f, 0.f};
      return f[gg];
    };
    const float f0 = feat(tile * 8 + tt), f1 = feat(tile * 8 + tt + 4);
    const float h0 = tf32_hi(f0), h1 = tf32_hi(f1);
    bfr[tile][ln] = make_uint4(__float_as_uint(h0), __float_as_uint(h1),
                               __float_as_uint(f0 - h0), __float_as_uint(f1 - h1));
  }
  // the warp's row tiles: rows g and g+8 packed
  float2 ox[RT], oy[RT], oz[RT];
  for (int rt = 0; rt < RT; ++rt) {
    const int r0 = ((blockIdx.x * W + warp) * RT + rt) * 16 + g;
    const float4 v0 = rows[r0 % nrows], v1 = rows[(r0 + 8) % nrows];
    ox[rt] = make_float2(v0.x, v1.x);
    oy[rt] = make_float2(v0.y, v1.y);
    oz[rt] = make_float2(v0.z, v1.z);
  }
  __syncthreads();
  double acc[RT][4];
  for (int rt = 0; rt < RT; ++rt) acc[rt][0] = acc[rt][1] = acc[rt][2] = acc[rt][3] = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int tile0 = 0; tile0 < kCols / 8; tile0 += RUN) {
      float d[RT][4];
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) d[rt][0] = d[rt][1] = d[rt][2] = d[rt][3] = 0.f;
#pragma unroll
      for (int k = 0; k < RUN; ++k) {
        const int tile = tile0 + k;
        const float4 A0 = ua[tile * 8 + t], B0 = ub[tile * 8 + t];
        const float4 A1 = ua[tile * 8 + t + 4], B1 = ub[tile * 8 + t + 4];
        const uint4 bb = bfr[tile][lane];
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) {
          float2 L0 = __ffma2_rn(make_float2(A0.x, A0.y), ox[rt], make_float2(B0.z, B0.w));
          L0 = __ffma2_rn(make_float2(A0.z, A0.w), oy[rt], L0);
          L0 = __ffma2_rn(make_float2(B0.x, B0.y), oz[rt], L0);
          float2 L1 = __ffma2_rn(make_float2(A1.x, A1.y), ox[rt], make_float2(B1.z, B1.w));
          L1 = __ffma2_rn(make_float2(A1.z, A1.w), oy[rt], L1);
          L1 = __ffma2_rn(make_float2(B1.x, B1.y), oz[rt], L1);
          const float2 w0 = ex2x2(L0), w1 = ex2x2(L1);
          const float2 h0 = make_float2(tf32_trunc(w0.x), tf32_trunc(w0.y));
          const float2 h1 = make_float2(tf32_trunc(w1.x), tf32_trunc(w1.y));
          const float2 l0 = __fadd2_rn(w0, make_float2(-h0.x, -h0.y));
          const float2 l1 = __fadd2_rn(w1, make_float2(-h1.x, -h1.y));
          // A: a0 (g,t) a1 (g+8,t) a2 (g,t+4) a3 (g+8,t+4)
          mma_tf32(d[rt], h0.x, h0.y, h1.x, h1.y, bb.x, bb.y);
          mma_tf32(d[rt], h0.x, h0.y, h1.x, h1.y, bb.z, bb.w);
          mma_tf32(d[rt], l0.x, l0.y, l1.x, l1.y, bb.x, bb.y);
        }
      }
#pragma unroll
      for (int rt = 0; rt < RT; ++rt)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[rt][i] += d[rt][i];
    }
  }
  // C: (g, features 2t, 2t+1), (g+8, 2t, 2t+1)
  for (int rt = 0; rt < RT; ++rt) {
    const int r0 = ((blockIdx.x * W + warp) * RT + rt) * 16 + g;
    if (sums_out) {
      for (int f = 0; f < 2; ++f) {
        if (2 * t + f < 5) {
          sums_out[static_cast<size_t>(r0) * 5 + 2 * t + f] = acc[rt][f];
          sums_out[static_cast<size_t>(r0 + 8) * 5 + 2 * t + f] = acc[rt][2 + f];
        }
      }
    } else if (acc[rt][0] == 1234.5) {
      out[tid] = 1.f;
    }
  }
}

// the production formulation (estep_row_kernel centred loop): FFMA2 sums,
// fp32 runs of RUN·8 points then fp64
template <int RUN>
__global__ void pass2_ffma(const float4* __restrict__ rows, const float4* __restrict__ cols,
                          int nrows, double* __restrict__ sums_out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const float4 v = rows[r];
  double a[5] = {0, 0, 0, 0, 0};
  for (int j0 = 0; j0 < kCols; j0 += 8 * RUN) {
    float f[5] = {0, 0, 0, 0, 0};
    for (int j = j0; j < j0 + 8 * RUN; ++j) {
      const float4 u = cols[j];
      float L = fmaf(u.x, v.x, u.w);
      L = fmaf(u.y, v.y, L);
      L = fmaf(u.z, v.z, L);
      float w;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(L));
      const float q = u.x * u.x + u.y * u.y + u.z * u.z;
      f[0] += w;
      f[1] = fmaf(w, u.x, f[1]);
      f[2] = fmaf(w, u.y, f[2]);
      f[3] = fmaf(w, u.z, f[3]);
      f[4] = fmaf(w, q, f[4]);
    }
    for (int i = 0; i < 5; ++i) a[i] += f[i];
  }
  for (int i = 0; i < 5; ++i) sums_out[static_cast<size_t>(r) * 5 + i] = a[i];
}

template <int RT, int W, int MB, int RUN>
void run(const char* name, int sms, const float4* dr, const float4* dc, int nrows, float* dout) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass2_mma<RT, W, MB, RUN>, W * 32, 0);
  const int blocks = sms * occ * 4;
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    pass2_mma<RT, W, MB, RUN><<<blocks, W * 32>>>(dr, dc, nrows, nullptr, dout, kReps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  const double pairs = double(blocks) * W * RT * 128.0 * (kCols / 8) * kReps;
  const double ps = pairs / (best * 1e-3);
  std::printf("%-24s occ=%d warps/SM=%2d  %.3f ms  %.3g pairs/s  %.1f cycles/64 pairs/SMSP @1965  %s\n",
              name, occ, occ * W, best, ps, 64.0 / (ps / (sms * 4.0 * 1.965e9)),
              cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nrows = 4096;
  std::mt19937 rng(1);
  // centred frame, R² ≤ 16: |u|, |v| ≤ ~2.3 per axis; logits over [-30, 0]
  std::uniform_real_distribution<float> U(-1.3f, 1.3f), B(-20.f, 0.f);
  std::vector<float4> hr(nrows), hc(kCols);
  for (auto& r : hr) {
    const float x = U(rng), y = U(rng), z = U(rng);
    r = make_float4(2.f * x, 2.f * y, 2.f * z, x * x + y * y + z * z);
  }
  for (auto& c : hc) {
    const float ux = U(rng), uy = U(rng), uz = U(rng);
    c = make_float4(ux, uy, uz, B(rng) - 2.f * 1.3f * (std::fabs(ux) + std::fabs(uy) + std::fabs(uz)));
  }
  float4 *dr, *dc;
  float* dout;
  double *ds_mma, *ds_ff;
  cudaMalloc(&dr, sizeof(float4) * nrows);
  cudaMalloc(&dc, sizeof(float4) * kCols);
  cudaMemcpy(dr, hr.data(), sizeof(float4) * nrows, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, hc.data(), sizeof(float4) * kCols, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, sizeof(float) * 1 << 20);
  cudaMalloc(&ds_mma, sizeof(double) * nrows * 5);
  cudaMalloc(&ds_ff, sizeof(double) * nrows * 5);
  // precision: rows 0..nrows-1 once over the 256 columns
  auto check = [&](const char* name, auto launch_mma) {
    launch_mma();
    pass2_ffma<8><<<nrows / 128, 128>>>(dr, dc, nrows, ds_ff);
    cudaDeviceSynchronize();
    std::vector<double> sm(nrows * 5), sf(nrows * 5);
    cudaMemcpy(sm.data(), ds_mma, sizeof(double) * sm.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(sf.data(), ds_ff, sizeof(double) * sf.size(), cudaMemcpyDeviceToHost);
    double em[6] = {}, ef[6] = {}, bias_var = 0.0;
    for (int r = 0; r < nrows; ++r) {
      const float4 v = hr[r];
      double ref[5] = {};
      for (int n = 0; n < kCols; ++n) {
        const float4 u = hc[n];
        const double L = double(u.x) * v.x + double(u.y) * v.y + double(u.z) * v.z + u.w;
        const double w = std::exp2(L);
        const double q = double(u.x) * u.x + double(u.y) * u.y + double(u.z) * u.z;
        ref[0] += w;
        ref[1] += w * u.x;
        ref[2] += w * u.y;
        ref[3] += w * u.z;
        ref[4] += w * q;
      }
      auto var = [&](const double* s) {  // Σw·t = Σw|u|² + |v|²Σw − 2v·Σwu (2v stored)
        return s[4] + double(v.w) * s[0] - (double(v.x) * s[1] + double(v.y) * s[2] + double(v.z) * s[3]);
      };
      for (int i = 0; i < 5; ++i) {
        em[i] = std::max(em[i], std::fabs(sm[r * 5 + i] - ref[i]) / ref[0]);
        ef[i] = std::max(ef[i], std::fabs(sf[r * 5 + i] - ref[i]) / ref[0]);
      }
      const double vr = var(ref);
      em[5] = std::max(em[5], std::fabs(var(&sm[r * 5]) - vr) / vr);
      ef[5] = std::max(ef[5], std::fabs(var(&sf[r * 5]) - vr) / vr);
      bias_var += (var(&sm[r * 5]) - vr) / vr;
    }
    std::printf("%s: max err / S0 (S0, Sx, Sy, Sz, Sq) mma %.2g %.2g %.2g %.2g %.2g  ffma %.2g %.2g %.2g %.2g %.2g\n",
                name, em[0], em[1], em[2], em[3], em[4], ef[0], ef[1], ef[2], ef[3], ef[4]);
    std::printf("%s: variance Σw·t rel err max: mma %.3g (mean %.3g)  ffma %.3g\n", name, em[5],
                bias_var / nrows, ef[5]);
  };
  check("run 1 k-block", [&] { pass2_mma<1, 4, 1, 1><<<nrows / 64, 128>>>(dr, dc, nrows, ds_mma, dout, 1); });
  check("run 8 k-blocks", [&] { pass2_mma<1, 4, 1, 8><<<nrows / 64, 128>>>(dr, dc, nrows, ds_mma, dout, 1); });
  run<2, 4, 4, 1>("rt2 w4 run1", sms, dr, dc, nrows, dout);
  run<2, 4, 4, 8>("rt2 w4 run8", sms, dr, dc, nrows, dout);
  run<4, 4, 2, 8>("rt4 w4 run8", sms, dr, dc, nrows, dout);
  run<4, 4, 3, 8>("rt4 w4 mb3 run8", sms, dr, dc, nrows, dout);
  run<2, 8, 2, 8>("rt2 w8 run8", sms, dr, dc, nrows, dout);
  run<1, 8, 4, 8>("rt1 w8 run8", sms, dr, dc, nrows, dout);
  run<4, 8, 1, 8>("rt4 w8 run8", sms, dr, dc, nrows, dout);
  run<2, 4, 4, 4>("rt2 w4 run4", sms, dr, dc, nrows, dout);
  return 0;
}
