// loopbench.cu — throughput of the E-step inner loops in isolation (B200).
//
// Each variant replays its pass's inner loop over 256 shared-memory points
// R times (no syncs, no global traffic) at the real kernels' occupancy, and
// reports cycles per point-warp (64 pairs): the achievable ceiling the
// full kernels are compared against.
//   row_diff / col_diff : difference form (estep_row_kernel / estep_col_kernel)
//   row_ctr  / col_ctr  : centred form (estep_row_kernel_c / estep_col_kernel_c)
//   *_nomufu            : same FP32 work, ex2 replaced by a register move
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/loopbench tools/loopbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kPts = 256;
constexpr int kReps = 64;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// exp2 on the FMA pipe for x ≤ 0 (f32x2): 2^x = 2^n · p(f), n = round(x),
// f ∈ [−0.5, 0.5], p a degree-5 minimax-style polynomial (rel. err ~1e-7);
// 2^n by adding n to the exponent bits.  x < −126 flushes to 0.
__device__ __forceinline__ float2 ex2_poly(float2 x) {
  x = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5·2^23
  const float2 t = __fadd2_rn(x, magic);
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-n.x, -n.y));
  float2 p = make_float2(1.3333558146e-3f, 1.3333558146e-3f);
  p = __ffma2_rn(p, f, make_float2(9.6181291076e-3f, 9.6181291076e-3f));
  p = __ffma2_rn(p, f, make_float2(5.5504108665e-2f, 5.5504108665e-2f));
  p = __ffma2_rn(p, f, make_float2(2.4022650696e-1f, 2.4022650696e-1f));
  p = __ffma2_rn(p, f, make_float2(6.9314718056e-1f, 6.9314718056e-1f));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  const int ix = __float_as_int(t.x) - 0x4B400000, iy = __float_as_int(t.y) - 0x4B400000;
  float2 r = make_float2(__int_as_float(__float_as_int(p.x) + (ix << 23)),
                         __int_as_float(__float_as_int(p.y) + (iy << 23)));
  if (x.x <= -127.f) r.x = 0.f;
  if (x.y <= -127.f) r.y = 0.f;
  return r;
}

template <bool M>
__device__ __forceinline__ float2 ex2v(float2 v) {
  if (M) return make_float2(ex2(v.x), ex2(v.y));
  return make_float2(v.y, v.x);
}

template <int V, bool MUFU>
__global__ void __launch_bounds__(128) loop_kernel(float* out, int occ_pad) {
  __shared__ float4 sa[kPts];
  __shared__ float4 sb[kPts];
  __shared__ float2 sq[kPts];
  extern __shared__ char pad[];  // occupancy control
  for (int i = threadIdx.x; i < kPts; i += 128) {
    const float f = 1e-3f * (i + 1);
    sa[i] = make_float4(f, f, -f, -f);
    sb[i] = make_float4(0.5f * f, 0.5f * f, -2.f * f, -2.f * f);
    sq[i] = make_float2(f * f, f * f);
  }
  if (occ_pad < 0) pad[threadIdx.x] = 0;
  __syncthreads();
  const float t0 = 1e-4f * threadIdx.x;
  const float2 ax = make_float2(t0, -t0), ay = make_float2(0.3f * t0, 0.7f), az = make_float2(t0, 0.1f);
  const float2 n2 = make_float2(-t0 * t0, -0.5f), minus1 = make_float2(-1.f, -1.f);
  float2 f0 = make_float2(0.f, 0.f), fx = f0, fy = f0, fz = f0, fq = f0;
  float2 g0 = f0, gx = f0, gy = f0, gz = f0, gq = f0;
  for (int r = 0; r < kReps; ++r) {
    for (int j = 0; j < kPts; j += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 a = sa[j + u];
        const float4 b = sb[j + u];
        const float2 A = make_float2(a.x, a.y), B = make_float2(a.z, a.w);
        const float2 C = make_float2(b.x, b.y), D = make_float2(b.z, b.w);
        if (V == 0) {  // row_diff: 3 FADD2 + FMUL2 + 2 FFMA2 + FFMA2 + 2 MUFU + FADD2 + 4 FFMA2
          const float2 dx = __fadd2_rn(A, ax), dy = __fadd2_rn(B, ay), dz = __fadd2_rn(C, az);
          float2 t = __fmul2_rn(dx, dx);
          t = __ffma2_rn(dy, dy, t);
          t = __ffma2_rn(dz, dz, t);
          const float2 L = __ffma2_rn(t, minus1, D);
          const float2 w = ex2v<MUFU>(L);
          f0 = __fadd2_rn(f0, w);
          fx = __ffma2_rn(w, A, fx);
          fy = __ffma2_rn(w, B, fy);
          fz = __ffma2_rn(w, C, fz);
          fq = __ffma2_rn(w, t, fq);
        } else if (V == 1) {  // row_ctr: FADD2 + 3 FFMA2 + 2 MUFU + FADD2 + 4 FFMA2
          const float2 Q = sq[j + u];
          float2 L = __fadd2_rn(D, n2);
          L = __ffma2_rn(A, ax, L);
          L = __ffma2_rn(B, ay, L);
          L = __ffma2_rn(C, az, L);
          const float2 w = ex2v<MUFU>(L);
          f0 = __fadd2_rn(f0, w);
          fx = __ffma2_rn(w, A, fx);
          fy = __ffma2_rn(w, B, fy);
          fz = __ffma2_rn(w, C, fz);
          fq = __ffma2_rn(w, Q, fq);
        } else if (V == 2) {  // col_diff: 3 FADD2 + FMUL2 + 2 FFMA2 + 2 MUFU + FADD2
          const float2 dx = __fadd2_rn(A, ax), dy = __fadd2_rn(B, ay), dz = __fadd2_rn(C, az);
          float2 t = __fmul2_rn(dx, dx);
          t = __ffma2_rn(dy, dy, t);
          t = __ffma2_rn(dz, dz, t);
          f0 = __fadd2_rn(f0, ex2v<MUFU>(make_float2(-t.x, -t.y)));
        } else if (V == 4) {  // row_ctr with two row pairs per thread (operand reuse)
          const float2 Q = sq[j + u];
          float2 L = __fadd2_rn(D, n2);
          float2 L2 = __fadd2_rn(D, ay);
          L = __ffma2_rn(A, ax, L);
          L2 = __ffma2_rn(A, az, L2);
          L = __ffma2_rn(B, ay, L);
          L2 = __ffma2_rn(B, n2, L2);
          L = __ffma2_rn(C, az, L);
          L2 = __ffma2_rn(C, ax, L2);
          const float2 w = ex2v<MUFU>(L);
          const float2 w2 = ex2v<MUFU>(L2);
          f0 = __fadd2_rn(f0, w);
          g0 = __fadd2_rn(g0, w2);
          fx = __ffma2_rn(w, A, fx);
          gx = __ffma2_rn(w2, A, gx);
          fy = __ffma2_rn(w, B, fy);
          gy = __ffma2_rn(w2, B, gy);
          fz = __ffma2_rn(w, C, fz);
          gz = __ffma2_rn(w2, C, gz);
          fq = __ffma2_rn(w, Q, fq);
          gq = __ffma2_rn(w2, Q, gq);
        } else if (V == 5) {  // row_ctr, accumulations as scalar FFMA
          const float2 Q = sq[j + u];
          float2 L = __fadd2_rn(D, n2);
          L = __ffma2_rn(A, ax, L);
          L = __ffma2_rn(B, ay, L);
          L = __ffma2_rn(C, az, L);
          const float2 w = ex2v<MUFU>(L);
          f0.x += w.x; f0.y += w.y;
          fx.x = __fmaf_rn(w.x, A.x, fx.x); fx.y = __fmaf_rn(w.y, A.y, fx.y);
          fy.x = __fmaf_rn(w.x, B.x, fy.x); fy.y = __fmaf_rn(w.y, B.y, fy.y);
          fz.x = __fmaf_rn(w.x, C.x, fz.x); fz.y = __fmaf_rn(w.y, C.y, fz.y);
          fq.x = __fmaf_rn(w.x, Q.x, fq.x); fq.y = __fmaf_rn(w.y, Q.y, fq.y);
        } else if (V == 6) {  // 8 FFMA2 with three distinct varying operands each
          fx = __ffma2_rn(A, B, fx);
          fy = __ffma2_rn(C, D, fy);
          fz = __ffma2_rn(B, C, fz);
          fq = __ffma2_rn(D, A, fq);
          f0 = __ffma2_rn(fx, fy, f0);
          g0 = __ffma2_rn(fz, fq, g0);
          gx = __ffma2_rn(A, C, gx);
          gy = __ffma2_rn(B, D, gy);
        } else if (V == 7) {  // 8 FFMA2, one varying operand + two reusable
          fx = __ffma2_rn(A, ax, fx);
          fy = __ffma2_rn(A, ay, fy);
          fz = __ffma2_rn(A, az, fz);
          fq = __ffma2_rn(A, n2, fq);
          f0 = __ffma2_rn(B, ax, f0);
          g0 = __ffma2_rn(B, ay, g0);
          gx = __ffma2_rn(B, az, gx);
          gy = __ffma2_rn(B, n2, gy);
        } else if (V == 8) {  // tc_acc: L from registers (TMEM stand-in), 2 rows per V load
          const float2 L0 = make_float2(A.x - t0, A.y), L1 = make_float2(B.x + t0, B.y);
          const float2 w = ex2v<MUFU>(L0), w2 = ex2v<MUFU>(L1);
          f0 = __fadd2_rn(f0, w);
          g0 = __fadd2_rn(g0, w2);
          fx = __ffma2_rn(w, A, fx);
          gx = __ffma2_rn(w2, A, gx);
          fy = __ffma2_rn(w, B, fy);
          gy = __ffma2_rn(w2, B, gy);
          fz = __ffma2_rn(w, C, fz);
          gz = __ffma2_rn(w2, C, gz);
          fq = __ffma2_rn(w, D, fq);
          gq = __ffma2_rn(w2, D, gq);
        } else if (V == 9) {  // col_fac: pass 1 with the factored constant (3 FFMA2 + FADD2)
          float2 e = __ffma2_rn(ax, A, D);
          e = __ffma2_rn(ay, B, e);
          e = __ffma2_rn(az, C, e);
          f0 = __fadd2_rn(f0, ex2v<MUFU>(e));
        } else if (V == 10) {  // row_fac: pass 2 with the factored constant (3 + 5 packed)
          const float2 Q = sq[j + u];
          float2 L = __ffma2_rn(A, ax, D);
          L = __ffma2_rn(B, ay, L);
          L = __ffma2_rn(C, az, L);
          const float2 w = ex2v<MUFU>(L);
          f0 = __fadd2_rn(f0, w);
          fx = __ffma2_rn(w, A, fx);
          fy = __ffma2_rn(w, B, fy);
          fz = __ffma2_rn(w, C, fz);
          fq = __ffma2_rn(w, Q, fq);
        } else if (V == 12 || V == 13) {  // col_fac with 1/8 (12) or 2/8 (13) exps on FMA
          float2 e = __ffma2_rn(ax, A, D);
          e = __ffma2_rn(ay, B, e);
          e = __ffma2_rn(az, C, e);
          const bool poly = (V == 12) ? (u == 7) : (u == 3 || u == 7);
          f0 = __fadd2_rn(f0, poly ? ex2_poly(make_float2(-fabsf(e.x), -fabsf(e.y))) : ex2v<MUFU>(e));
        } else if (V == 14) {  // col_fac with two column pairs per thread (staged v shared)
          float2 e = __ffma2_rn(ax, A, D);
          float2 e2 = __ffma2_rn(az, A, D);
          e = __ffma2_rn(ay, B, e);
          e2 = __ffma2_rn(ax, B, e2);
          e = __ffma2_rn(az, C, e);
          e2 = __ffma2_rn(ay, C, e2);
          f0 = __fadd2_rn(f0, ex2v<MUFU>(e));
          g0 = __fadd2_rn(g0, ex2v<MUFU>(e2));
        } else if (V == 11) {  // row_fac with two row pairs per thread (U shared)
          const float2 Q = sq[j + u];
          float2 L = __ffma2_rn(A, ax, D);
          float2 L2 = __ffma2_rn(A, az, D);
          L = __ffma2_rn(B, ay, L);
          L2 = __ffma2_rn(B, n2, L2);
          L = __ffma2_rn(C, az, L);
          L2 = __ffma2_rn(C, ax, L2);
          const float2 w = ex2v<MUFU>(L), w2 = ex2v<MUFU>(L2);
          f0 = __fadd2_rn(f0, w);
          g0 = __fadd2_rn(g0, w2);
          fx = __ffma2_rn(w, A, fx);
          gx = __ffma2_rn(w2, A, gx);
          fy = __ffma2_rn(w, B, fy);
          gy = __ffma2_rn(w2, B, gy);
          fz = __ffma2_rn(w, C, fz);
          gz = __ffma2_rn(w2, C, gz);
          fq = __ffma2_rn(w, Q, fq);
          gq = __ffma2_rn(w2, Q, gq);
        } else {  // col_ctr: FADD2 + 3 FFMA2 + 2 MUFU + FADD2
          float2 e = __fadd2_rn(n2, D);
          e = __ffma2_rn(ax, A, e);
          e = __ffma2_rn(ay, B, e);
          e = __ffma2_rn(az, C, e);
          f0 = __fadd2_rn(f0, ex2v<MUFU>(e));
        }
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] =
      f0.x + f0.y + fx.x + fx.y + fy.x + fy.y + fz.x + fz.y + fq.x + fq.y + g0.x + g0.y + gx.x +
      gx.y + gy.x + gy.y + gz.x + gz.y + gq.x + gq.y;
}

// Pass-2 accumulation on the legacy tensor path (mma.sync m16n8k8 tf32,
// HMMA): logits by FFMA2 in the A-fragment layout (lane g,t4: rows g+16i,
// g+8+16i; columns t4, t4+4 of each 8-column step), w split into tf32 hi/lo,
// B = 8 column quantities (v hi, |v|² hi, v lo, |v|² lo), Σw by FADD2, the
// MMA accumulators flushed into fp32 every 8 steps.  NB row blocks of 16 per
// warp; reports cycles per 64 pairs (point-warp equivalent).
template <int NB, bool MUFU, bool HM = true>
__global__ void __launch_bounds__(128) mma_row_kernel(float* out, int occ_pad) {
  __shared__ float4 sa[kPts];
  __shared__ float4 sd1[kPts], sd2[kPts];  // pre-duplicated (vx,vx,vy,vy), (vz,vz,Bn,Bn)
  __shared__ float sbf[kPts * 8];
  extern __shared__ char pad[];
  for (int i = threadIdx.x; i < kPts; i += 128) {
    const float f = 1e-3f * (i + 1);
    sa[i] = make_float4(f, -f, 0.5f * f, -2.f * f);
    sd1[i] = make_float4(f, f, -f, -f);
    sd2[i] = make_float4(0.5f * f, 0.5f * f, -2.f * f, -2.f * f);
    for (int c = 0; c < 8; ++c) sbf[i * 8 + c] = f * (c + 1);
  }
  if (occ_pad < 0) pad[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  float2 ux[NB], uy[NB], uz[NB], s0[NB];
  float c[NB][4], acc[NB][4];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const float t0 = 1e-4f * (threadIdx.x + i);
    ux[i] = make_float2(t0, -t0);
    uy[i] = make_float2(0.3f * t0, 0.7f);
    uz[i] = make_float2(t0, 0.1f);
    s0[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 4; ++q) c[i][q] = acc[i][q] = 0.f;
  }
  for (int r = 0; r < kReps; ++r) {
    for (int j = 0; j < kPts; j += 64) {
#pragma unroll
      for (int st = 0; st < 8; ++st) {
        const int k0 = j + 8 * st + t4, k1 = k0 + 4;
        const float4 A1 = sd1[k0], A2 = sd2[k0], B1 = sd1[k1], B2 = sd2[k1];
        const unsigned b0 = __float_as_uint(sbf[k0 * 8 + g]), b1 = __float_as_uint(sbf[k1 * 8 + g]);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          float2 L0 = __ffma2_rn(ux[i], make_float2(A1.x, A1.y), make_float2(A2.z, A2.w));
          L0 = __ffma2_rn(uy[i], make_float2(A1.z, A1.w), L0);
          L0 = __ffma2_rn(uz[i], make_float2(A2.x, A2.y), L0);
          float2 L1 = __ffma2_rn(ux[i], make_float2(B1.x, B1.y), make_float2(B2.z, B2.w));
          L1 = __ffma2_rn(uy[i], make_float2(B1.z, B1.w), L1);
          L1 = __ffma2_rn(uz[i], make_float2(B2.x, B2.y), L1);
          const float2 w0 = ex2v<MUFU>(L0), w1 = ex2v<MUFU>(L1);
          s0[i] = __fadd2_rn(s0[i], __fadd2_rn(w0, w1));
          const float2 h0 = make_float2(__uint_as_float(__float_as_uint(w0.x) & 0xffffe000u),
                                        __uint_as_float(__float_as_uint(w0.y) & 0xffffe000u));
          const float2 h1 = make_float2(__uint_as_float(__float_as_uint(w1.x) & 0xffffe000u),
                                        __uint_as_float(__float_as_uint(w1.y) & 0xffffe000u));
          const float2 l0 = __fadd2_rn(w0, make_float2(-h0.x, -h0.y));
          const float2 l1 = __fadd2_rn(w1, make_float2(-h1.x, -h1.y));
          if (!HM) {  // stand-in: the same operands consumed by FP32 adds
            c[i][0] += h0.x + l0.x;
            c[i][1] += h0.y + l0.y;
            c[i][2] += h1.x + __uint_as_float(b0);
            c[i][3] += h1.y + __uint_as_float(b1);
            continue;
          }
          asm volatile(
              "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
              "{%8,%9}, {%0,%1,%2,%3};\n"
              : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
              : "r"(__float_as_uint(h0.x)), "r"(__float_as_uint(h0.y)), "r"(__float_as_uint(h1.x)),
                "r"(__float_as_uint(h1.y)), "r"(b0), "r"(b1));
          asm volatile(
              "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
              "{%8,%9}, {%0,%1,%2,%3};\n"
              : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
              : "r"(__float_as_uint(l0.x)), "r"(__float_as_uint(l0.y)), "r"(__float_as_uint(l1.x)),
                "r"(__float_as_uint(l1.y)), "r"(b0), "r"(b1));
        }
      }
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] += c[i][q], c[i][q] = 0.f;
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < NB; ++i) sum += s0[i].x + s0[i].y + acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
}

template <int NB, bool MUFU, bool HM = true>
void run_mma(const char* name, int sms, int ctas_per_sm, float* out) {
  auto k = mma_row_kernel<NB, MUFU, HM>;
  int occ = 0;
  const int pad = 227 * 1024 / ctas_per_sm - 21 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, pad);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms * occ;
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
  // pairs per warp per rep = kPts columns × 16·NB rows; per SMSP
  const double pairs_per_smsp = double(grid) * 4 * kReps * kPts * 16.0 * NB / (sms * 4.0);
  const double cycles = (ms / 3) * 1e-3 * clk_khz * 1e3;
  cudaError_t e = cudaGetLastError();
  std::printf("%-14s occ=%2d CTAs/SM  %8.3f ms  %6.2f cycles/64 pairs (@%d MHz attr)  %s\n", name,
              occ, ms / 3, 64.0 * cycles / pairs_per_smsp, clk_khz / 1000, cudaGetErrorString(e));
}

template <int V, bool MUFU>
void run(const char* name, int sms, int ctas_per_sm, float* out) {
  auto k = loop_kernel<V, MUFU>;
  int occ = 0;
  // pad dynamic smem so exactly ctas_per_sm CTAs fit (228 KB per SM)
  const int pad = 227 * 1024 / ctas_per_sm - 12 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, pad);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms * occ;
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
  // point-warps per SMSP: (grid·4 warps)·kReps·kPts / (sms·4)
  const double pw_per_smsp = double(grid) * 4 * kReps * kPts / (sms * 4.0);
  const double cycles = (ms / 3) * 1e-3 * clk_khz * 1e3;
  cudaError_t e = cudaGetLastError();
  std::printf("%-14s occ=%2d CTAs/SM  %8.3f ms  %6.2f cycles/point-warp (@%d MHz attr)  %s\n",
              name, occ, ms / 3, cycles / pw_per_smsp, clk_khz / 1000, cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 32 * 128);
  std::printf("-- pass-2 accumulation on HMMA (mma.sync tf32 hi/lo), cycles per 64 pairs\n");
  run<10, true>("row_fac", sms, 8, out);
  run_mma<1, true>("mma_nb1", sms, 8, out);
  run_mma<2, true>("mma_nb2", sms, 8, out);
  run_mma<2, true>("mma_nb2_o4", sms, 4, out);
  run_mma<4, true>("mma_nb4", sms, 4, out);
  run_mma<4, true>("mma_nb4_o6", sms, 6, out);
  run_mma<2, false>("mma_nb2_nm", sms, 8, out);
  run_mma<2, true, false>("mma_nb2_nohmma", sms, 8, out);
  run_mma<2, false, false>("mma_nb2_nm_nohm", sms, 8, out);
  if (std::getenv("LB_MMA_ONLY")) return 0;
  std::printf("-- current kernels' loops at 8 CTAs/SM (tc_acc = 128 pairs per point-warp)\n");
  run<9, true>("col_fac", sms, 8, out);
  run<10, true>("row_fac", sms, 8, out);
  run<14, true>("col_fac_cp2", sms, 8, out);
  run<14, true>("col_fac_cp2_o12", sms, 12, out);
  run<14, false>("col_fac_cp2_nm", sms, 8, out);
  run<12, true>("col_fac_poly1of8", sms, 8, out);
  run<13, true>("col_fac_poly2of8", sms, 8, out);
  run<11, true>("row_fac_rp2", sms, 8, out);
  run<11, true>("row_fac_rp2_o6", sms, 6, out);
  run<8, true>("tc_acc", sms, 8, out);
  run<8, true>("tc_acc_occ4", sms, 4, out);
  run<8, false>("tc_acc_nomufu", sms, 8, out);
  std::printf("-- extra variants at 8 CTAs/SM (row_ctr_rp2 = 128 pairs per point-warp; ffma2_* = 8 FFMA2 per point)\n");
  run<4, true>("row_ctr_rp2", sms, 8, out);
  run<4, false>("row_ctr_rp2_nm", sms, 8, out);
  run<5, true>("row_ctr_sacc", sms, 8, out);
  run<5, false>("row_ctr_sacc_nm", sms, 8, out);
  run<6, false>("ffma2_3var", sms, 8, out);
  run<7, false>("ffma2_1var", sms, 8, out);
  for (int occ : {8}) {
    std::printf("-- target %d CTAs/SM (%d warps/SMSP)\n", occ, occ);
    run<0, true>("row_diff", sms, occ, out);
    run<1, true>("row_ctr", sms, occ, out);
    run<2, true>("col_diff", sms, occ, out);
    run<3, true>("col_ctr", sms, occ, out);
    run<0, false>("row_diff_nomufu", sms, occ, out);
    run<1, false>("row_ctr_nomufu", sms, occ, out);
    run<2, false>("col_diff_nomufu", sms, occ, out);
    run<3, false>("col_ctr_nomufu", sms, occ, out);
  }
  return 0;
}
