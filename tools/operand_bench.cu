// operand_bench.cu — what bounds the pass-2 inner loop on B200 (sm_100a)?
//
// Part 1: pipe rates (lane-ops per clk per SM) of MUFU.EX2, FFMA, FFMA2 with
// 64-bit operands, FFMA2 with a broadcast (.F32) operand, and mixes.
// Part 2: the pass-2 centred loop (estep_row_kernel) in three operand
// layouts, cycles per 64 pairs per SMSP (MUFU bound: 16):
//   dup  : staged column values duplicated (ux,ux) — the round-2 kernel
//   bc   : staged scalars, FFMA2 broadcast operands (.F32)
//   col  : pairs packed over two columns (one row per lane, row constants
//          broadcast), sums folded at the end
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/operand_bench tools/operand_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kPts = 256;
constexpr int kReps = 64;
constexpr int kIters = 2048;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <bool M>
__device__ __forceinline__ float2 ex2v(float2 v) {
  if (M) return make_float2(ex2f(v.x), ex2f(v.y));
  return make_float2(v.y, v.x);
}

// ---------------- part 1: pipe rates -----------------------------------------
template <int V>
__global__ void __launch_bounds__(128) pipe_kernel(float* out, float a0) {
  float r[8];
  float2 q[8];
  const float2 c = make_float2(a0, a0 * 0.5f), d = make_float2(-a0, 0.25f);
  const float cs = a0 * 0.75f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    r[i] = 1e-6f * (threadIdx.x + i);
    q[i] = make_float2(r[i], -r[i]);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (V == 0) r[i] = ex2f(-r[i]);                           // MUFU.EX2
      if (V == 1) r[i] = __fmaf_rn(r[i], a0, cs);               // FFMA
      if (V == 2) q[i] = __ffma2_rn(q[i], c, d);                // FFMA2, 3×64-bit
      if (V == 3) q[i] = __ffma2_rn(q[i], make_float2(cs, cs), d);  // FFMA2, broadcast B
      if (V == 4) {  // FFMA2 accumulate with per-i varying 64-bit A (like Σw·u)
        q[i] = __ffma2_rn(q[(i + 1) & 7], c, q[i]);
      }
      if (V == 5) {  // 1 MUFU.EX2 per 2 FFMA2 (pass-2 balance: 2 MUFU per 8 FFMA2 lanes... 1:4)
        r[i] = ex2f(-r[i]);
        q[i] = __ffma2_rn(q[i], c, d);
        q[i] = __ffma2_rn(q[i], d, c);
      }
      if (V == 6) {  // 2 MUFU per 8 FFMA2 (exactly the pass-2 ratio per 64 pairs)
        if (i < 2) r[i] = ex2f(-r[i]);
        q[i] = __ffma2_rn(q[i], c, d);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += r[i] + q[i].x + q[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run_pipe(const char* name, int sms, float* out, double lane_ops_per_thread_iter) {
  auto k = pipe_kernel<V>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, 0);
  occ = occ > 8 ? 8 : occ;
  const int grid = sms * occ;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<grid, 128>>>(out, 0.5f);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) k<<<grid, 128>>>(out, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double cycles = (ms / 3) * 1e-3 * clk_khz * 1e3;
  const double ops = double(grid) * 128 * kIters * lane_ops_per_thread_iter;
  std::printf("%-22s occ=%d  %8.3f ms  %7.1f lane-ops/clk/SM  %s\n", name, occ, ms / 3,
              ops / cycles / sms, cudaGetErrorString(cudaGetLastError()));
}

// ---------------- part 2: pass-2 loop layouts --------------------------------
// L = Bn + 2u·v (row constants 2v), w = 2^L, sums S0, Σw·u (3), Σw·|u|².
// V: 0 dup (NP row pairs per thread), 1 bc (NP row pairs), 2 col (NP rows per
// thread, two columns per packed pair)
template <int V, int NP, bool MUFU>
__global__ void __launch_bounds__(128) loop_kernel(float* out, int occ_pad) {
  __shared__ float4 sa[kPts];  // dup: (ux,ux,uy,uy); bc: (ux,uy,uz,Bn); col: (ux0,ux1,uy0,uy1)
  __shared__ float4 sb[kPts];  // dup: (uz,uz,Bn,Bn);  bc: (q, ·);       col: (uz0,uz1,Bn0,Bn1)
  __shared__ float2 sq[kPts];  // dup: (q,q);          col: (q0,q1)
  extern __shared__ char pad[];
  for (int i = threadIdx.x; i < kPts; i += 128) {
    const float f = 1e-3f * (i + 1);
    sa[i] = make_float4(f, f * 0.5f, -f, -2.f * f);
    sb[i] = make_float4(0.5f * f, 0.25f * f, -2.f * f, -f);
    sq[i] = make_float2(f * f, 0.3f * f * f);
  }
  if (occ_pad < 0) pad[threadIdx.x] = 0;
  __syncthreads();
  const float t0 = 1e-4f * threadIdx.x;
  float2 ox[NP], oy[NP], oz[NP];
  float2 f0[NP], fx[NP], fy[NP], fz[NP], fq[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    ox[p] = make_float2(t0 + p, -t0);
    oy[p] = make_float2(0.3f * t0, 0.7f + p);
    oz[p] = make_float2(t0, 0.1f * p);
    f0[p] = fx[p] = fy[p] = fz[p] = fq[p] = make_float2(0.f, 0.f);
  }
  const int steps = (V == 2) ? kPts / 2 : kPts;  // col: two columns per step
  float2 Lp[NP];  // V == 3: the next point's logits
#pragma unroll
  for (int p = 0; p < NP; ++p) Lp[p] = make_float2(-1.f, -2.f);
  for (int r = 0; r < kReps; ++r) {
    for (int j = 0; j < steps; j += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (V == 0) {
          const float4 A = sa[j + u], B = sb[j + u];
          const float2 Q = sq[j + u];
          const float2 Ux = make_float2(A.x, A.y), Uy = make_float2(A.z, A.w);
          const float2 Uz = make_float2(B.x, B.y), Bn = make_float2(B.z, B.w);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            float2 L = __ffma2_rn(Ux, ox[p], Bn);
            L = __ffma2_rn(Uy, oy[p], L);
            L = __ffma2_rn(Uz, oz[p], L);
            const float2 w = ex2v<MUFU>(L);
            f0[p] = __fadd2_rn(f0[p], w);
            fx[p] = __ffma2_rn(w, Ux, fx[p]);
            fy[p] = __ffma2_rn(w, Uy, fy[p]);
            fz[p] = __ffma2_rn(w, Uz, fz[p]);
            fq[p] = __ffma2_rn(w, Q, fq[p]);
          }
        } else if (V == 1) {
          const float4 A = sa[j + u];
          const float q = sq[j + u].x;
          const float2 Ux = make_float2(A.x, A.x), Uy = make_float2(A.y, A.y);
          const float2 Uz = make_float2(A.z, A.z), Bn = make_float2(A.w, A.w);
          const float2 Q = make_float2(q, q);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            float2 L = __ffma2_rn(Ux, ox[p], Bn);
            L = __ffma2_rn(Uy, oy[p], L);
            L = __ffma2_rn(Uz, oz[p], L);
            const float2 w = ex2v<MUFU>(L);
            f0[p] = __fadd2_rn(f0[p], w);
            fx[p] = __ffma2_rn(w, Ux, fx[p]);
            fy[p] = __ffma2_rn(w, Uy, fy[p]);
            fz[p] = __ffma2_rn(w, Uz, fz[p]);
            fq[p] = __ffma2_rn(w, Q, fq[p]);
          }
        } else if (V == 3) {
          // bc with the logits of the next staged point computed before this
          // point's ex2/sums (software-pipelined by one point)
          const int jn = (j + u + 1) & (kPts - 1);
          const float4 An = sa[jn];
          const float4 A = sa[j + u];
          const float q = sq[j + u].x;
          const float2 Q = make_float2(q, q);
          const float2 Ux = make_float2(A.x, A.x), Uy = make_float2(A.y, A.y);
          const float2 Uz = make_float2(A.z, A.z);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const float2 w = ex2v<MUFU>(Lp[p]);
            float2 Ln = __ffma2_rn(make_float2(An.x, An.x), ox[p], make_float2(An.w, An.w));
            Ln = __ffma2_rn(make_float2(An.y, An.y), oy[p], Ln);
            Ln = __ffma2_rn(make_float2(An.z, An.z), oz[p], Ln);
            Lp[p] = Ln;
            f0[p] = __fadd2_rn(f0[p], w);
            fx[p] = __ffma2_rn(w, Ux, fx[p]);
            fy[p] = __ffma2_rn(w, Uy, fy[p]);
            fz[p] = __ffma2_rn(w, Uz, fz[p]);
            fq[p] = __ffma2_rn(w, Q, fq[p]);
          }
        } else {
          const float4 A = sa[j + u], B = sb[j + u];
          const float2 Q = sq[j + u];
          const float2 Ux = make_float2(A.x, A.y), Uy = make_float2(A.z, A.w);
          const float2 Uz = make_float2(B.x, B.y), Bn = make_float2(B.z, B.w);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            // one row per p: constants are scalars (ox[p].x etc.)
            float2 L = __ffma2_rn(Ux, make_float2(ox[p].x, ox[p].x), Bn);
            L = __ffma2_rn(Uy, make_float2(oy[p].x, oy[p].x), L);
            L = __ffma2_rn(Uz, make_float2(oz[p].x, oz[p].x), L);
            const float2 w = ex2v<MUFU>(L);
            f0[p] = __fadd2_rn(f0[p], w);
            fx[p] = __ffma2_rn(w, Ux, fx[p]);
            fy[p] = __ffma2_rn(w, Uy, fy[p]);
            fz[p] = __ffma2_rn(w, Uz, fz[p]);
            fq[p] = __ffma2_rn(w, Q, fq[p]);
          }
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int p = 0; p < NP; ++p)
    s += Lp[p].x + f0[p].x + f0[p].y + fx[p].x + fx[p].y + fy[p].x + fy[p].y + fz[p].x + fz[p].y + fq[p].x +
         fq[p].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V, int NP, bool MUFU>
void run_loop(const char* name, int sms, int ctas_per_sm, float* out) {
  auto k = loop_kernel<V, NP, MUFU>;
  int occ = 0;
  const int pad = 227 * 1024 / ctas_per_sm - 12 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, pad);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  const int grid = sms * occ;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<grid, 128, pad>>>(out, 0);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) k<<<grid, 128, pad>>>(out, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  // pairs per thread per rep: kPts columns × 2·NP rows (every layout)
  const double pairs_per_smsp = double(grid) * 128 * kReps * kPts * 2.0 * NP / (sms * 4.0);
  const double cycles = (ms / 3) * 1e-3 * clk_khz * 1e3;
  std::printf("%-22s occ=%2d CTAs/SM regs=%3d  %8.3f ms  %6.2f cycles/64 pairs/SMSP  %s\n", name,
              occ, fa.numRegs, ms / 3, 64.0 * cycles / pairs_per_smsp,
              cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 32 * 128);
  std::printf("-- pipe rates (lane-ops/clk/SM; FFMA2 counts 2 per lane)\n");
  run_pipe<0>("mufu_ex2", sms, out, 8);
  run_pipe<1>("ffma", sms, out, 8);
  run_pipe<2>("ffma2_64bit", sms, out, 16);
  run_pipe<3>("ffma2_bcast", sms, out, 16);
  run_pipe<4>("ffma2_acc_varA", sms, out, 16);
  run_pipe<5>("ex2+2ffma2 (lanes=ffma)", sms, out, 32);
  run_pipe<6>("2ex2+8ffma2 (lanes=ffma)", sms, out, 16);
  std::printf("-- pass-2 centred loop, cycles per 64 pairs per SMSP (MUFU bound 16)\n");
  for (int occ : {8, 6}) {
    std::printf("   target %d CTAs/SM of 128 threads\n", occ);
    run_loop<0, 1, true>("dup np1", sms, occ, out);
    run_loop<0, 2, true>("dup np2", sms, occ, out);
    run_loop<1, 1, true>("bc np1", sms, occ, out);
    run_loop<1, 2, true>("bc np2", sms, occ, out);
    run_loop<1, 3, true>("bc np3", sms, occ, out);
    run_loop<3, 2, true>("bc np2 pipelined", sms, occ, out);
    run_loop<3, 2, false>("bc np2 pipe nomufu", sms, occ, out);
    run_loop<2, 2, true>("col np2", sms, occ, out);
    run_loop<2, 4, true>("col np4", sms, occ, out);
    run_loop<0, 2, false>("dup np2 nomufu", sms, occ, out);
    run_loop<1, 2, false>("bc np2 nomufu", sms, occ, out);
    run_loop<2, 4, false>("col np4 nomufu", sms, occ, out);
  }
  return 0;
}
