// topk.cu — top-K eigenpairs of the Gaussian Gram matrix without forming it.
//
// Configs 2–4 (M = 50k…200k) cannot afford the reference's full dense
// eigensolve (kernel.hpp:54: O(M³) and an M×M fp64 Φ of 20–320 GB).  The
// north star asks for "top-K Lanczos eigenpairs whose G·v products are
// computed on the fly by a custom kernel".  We use the block form of that
// Krylov idea — randomized subspace iteration with Rayleigh–Ritz — because
// it needs only block products G·V (one fp64 GEMM-like kernel that
// regenerates Φ tiles on the fly) and dense b×b algebra:
//
//   V₀ = orth(random M×b),  b = K + p
//   repeat:  W = G V                               (G·V on the fly, fp64)
//            T = Vᵀ W,  T = S Θ Sᵀ,  U = V S[:, :K] (Rayleigh–Ritz)
//            stop if every top-K residual ‖W s_i − θ_i V s_i‖ ≤ 1e-11·θ₁
//            (after ≥ 1 power step) or after q power steps; else V ← orth(W)
//   λ = Θ[:K] (descending),  λ_i < 1e-12·λ_max → 0  (kernel.hpp:68-70)
//
// W s_i = G u_i exactly (in fp64), so the residual check costs two M×b×K
// GEMMs and a b×b eigensolve, not another Φ product.  Large M converges in 2
// power steps (the spectrum has fallen by orders of magnitude between rank K
// and K + p); small M with K/M = 2 % needs all 4.
//
// The Gaussian kernel's spectrum decays super-exponentially (SURVEY App.
// A.4), so the eigenpairs that move x̃ (λ ≳ 1e-10 λ₁) converge in a few
// iterations; eigenpairs below the fp64 noise floor are arbitrary exactly as
// they are in any fp64 dense solver, and the filter λ/(λ+λσ²) ≈ 0 mutes them.
//
// G·V kernel (`gram_dmma_kernel`): the fp64 tensor op (DMMA, mma.sync
// m8n8k4 f64 — 37 TFLOP/s on this B200, the same pipe peak as DFMA but one
// instruction per 256 MACs, so the Φ generation and the loads issue beside
// it).  A CTA owns 64 rows × 64·WC columns (WC = 1…6 column warps × 2 row
// warps; warp tile 32 × 64, 64 fp64 accumulators per thread), i.e. all of
// b ≤ 384 at once, so every Φ entry is generated once per product.  Per
// 16-point reduction chunk, double-buffered: the CTA regenerates the 64×16 Φ
// tile (fp64 exp of the difference form — symmetric, diagonal exactly 1)
// into shared memory while the chunk before it multiplies, and cp.async
// streams the 16 × 64·WC slice of Vᵀ (V transposed to point-major once per
// product).  Bound: FP64 pipe (2·M²·b_pad flops per product).

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "common.cuh"
#include "setup.cuh"

namespace fcpd {

namespace {
constexpr int kGvTileM = 128;
constexpr int kGvTileN = 128;
constexpr int kGvTileK = 32;
// adaptive stop: every top-K Ritz residual ≤ this × θ₁ (100× under the
// 1e-9·λ₁ the parity tests demand of the dense-solver comparison)
constexpr double kTopkResidualTol = 1e-11;

#define FCPD_CUBLAS(call)                                                              \
  do {                                                                                 \
    cublasStatus_t s_ = (call);                                                        \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                   \
      throw ::fcpd::Failure(FCPD_ERR_CUDA, std::string(#call) + ": cublas status " +   \
                                               std::to_string(static_cast<int>(s_)));   \
  } while (0)
#define FCPD_CUSOLVER2(call)                                                           \
  do {                                                                                 \
    cusolverStatus_t s_ = (call);                                                      \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                 \
      throw ::fcpd::Failure(FCPD_ERR_CUDA, std::string(#call) + ": cusolver status " + \
                                               std::to_string(static_cast<int>(s_)));   \
  } while (0)
}  // namespace

// Y (M×b, col-major, ld m) = Φ V,  Φ_ij = exp(−‖x_i − x_j‖² / 2β²), diag 1.
__global__ void __launch_bounds__(256, 1)
    gram_matmul_kernel(const double* __restrict__ x, int64_t m, int d, double inv2b2,
                       const double* __restrict__ v, int64_t b, double* __restrict__ y) {
  extern __shared__ double gv_smem[];
  auto gs = reinterpret_cast<double (*)[kGvTileM]>(gv_smem);                      // Φ tile
  auto vs = reinterpret_cast<double (*)[kGvTileN]>(gv_smem + kGvTileK * kGvTileM);  // V tile
  auto xr = reinterpret_cast<double (*)[kGvTileM]>(gv_smem + kGvTileK * (kGvTileM + kGvTileN));
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kGvTileM;
  const int64_t col0 = static_cast<int64_t>(blockIdx.y) * kGvTileN;
  for (int i = threadIdx.x; i < 3 * kGvTileM; i += 256) {
    const int c = i / kGvTileM, r = i % kGvTileM;
    xr[c][r] = (c < d && row0 + r < m) ? x[c * m + row0 + r] : 0.0;
  }
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

  for (int64_t k0 = 0; k0 < m; k0 += kGvTileK) {
    __syncthreads();
    // Φ tile: 128 rows × 32 columns (k), 16 entries per thread
    for (int e = threadIdx.x; e < kGvTileM * kGvTileK; e += 256) {
      const int r = e % kGvTileM, k = e / kGvTileM;
      const int64_t j = k0 + k;
      double val = 0.0;
      if (j < m && row0 + r < m) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) {
          const double t = xr[c][r] - x[c * m + j];
          s += t * t;
        }
        val = (row0 + r == j) ? 1.0 : exp(-s * inv2b2);
      }
      gs[k][r] = val;
    }
    // V tile: 32 rows (k) × 128 columns
    for (int e = threadIdx.x; e < kGvTileK * kGvTileN; e += 256) {
      const int k = e / kGvTileN, c = e % kGvTileN;
      const int64_t j = k0 + k, col = col0 + c;
      vs[k][c] = (j < m && col < b) ? v[col * m + j] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kGvTileK; ++k) {
      double a[8], bb[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = gs[k][ty * 8 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) bb[j] = vs[k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = row0 + ty * 8 + i;
    if (r >= m) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t c = col0 + tx + 16 * j;
      if (c < b) y[c * m + r] = acc[i][j];
    }
  }
}

// xq[j] = −inv·|x_j|² (0 beyond M), m_pad long.
__global__ void gram_rownorm_kernel(const double* __restrict__ x, int64_t m, int d, double inv2b2,
                                    int64_t m_pad, double* __restrict__ xq) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m_pad) return;
  double q = 0.0;
  if (j < m)
    for (int c = 0; c < d; ++c) q = fma(x[c * m + j], x[c * m + j], q);
  xq[j] = -inv2b2 * q;
}

// V (M×b column-major, ld m) → Vᵀ (m_pad × ldv, point-major, zero padded).
__global__ void transpose_pad_kernel(const double* __restrict__ v, int64_t m, int64_t b,
                                     double* __restrict__ vt, int64_t m_pad, int64_t ldv) {
  __shared__ double tile[32][33];
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t c = c0 + r, j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (c < b && j < m) ? v[c * m + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + r, c = c0 + threadIdx.x;
    if (j < m_pad && c < ldv) vt[j * ldv + c] = tile[threadIdx.x][r];
  }
}

// Wᵀ (point-major, ld ldv) → W (M×b column-major, ld m).
__global__ void untranspose_kernel(const double* __restrict__ wt, int64_t ldv, int64_t m,
                                   int64_t b, double* __restrict__ w) {
  __shared__ double tile[32][33];
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + r, c = c0 + threadIdx.x;
    tile[r][threadIdx.x] = (j < m && c < b) ? wt[j * ldv + c] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t c = c0 + r, j = j0 + threadIdx.x;
    if (c < b && j < m) w[c * m + j] = tile[threadIdx.x][r];
  }
}

namespace {
constexpr int kGdRows = 64;    // CTA rows (2 row warps × 32)
constexpr int kGdChunk = 16;   // reduction points per pipeline stage
constexpr int kGdPhiPitch = kGdChunk + 4;  // ≡ 4 (mod 16) doubles: A fragments in 2 wavefronts
constexpr int kGdCols = 128;   // CTA columns (2 column warps × 64)
constexpr size_t kGdSmem =
    sizeof(double) * (2 * kGdRows * kGdPhiPitch + 2 * kGdChunk * (kGdCols + 8) + 2 * 4 * kGdChunk);

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__constant__ double c_exp2_64[64];  // 2^(i/64), from the host's exp2

// e^a for a ≤ 0: a = (64k + i)·ln2/64 + r, |r| ≤ ln2/128; e^r by its
// degree-5 Taylor polynomial (truncation ≤ 4e-17), times 2^(i/64) from the
// table, times 2^k by exponent arithmetic.  11 FP64 operations against ~18
// in libdevice's exp; ≤ 2 ulp.  a < −707 → 0 (keeps the result normal:
// such entries are < 1e-307 of the diagonal).
__device__ __forceinline__ double exp_nonpos(double a, const double* tab) {
  constexpr double kInvLn2x64 = 92.33248261689366;            // 64/ln2
  constexpr double kLn2by64Hi = 0.010830424695086549;         // ln2/64, 33 bits (n·hi exact)
  constexpr double kLn2by64Lo = 1.162596423439437e-12;        // ln2/64 − hi
  constexpr double kShift = 6755399441055744.0;               // 1.5·2^52
  if (a < -707.0) return 0.0;
  const double kd = fma(a, kInvLn2x64, kShift);
  const int n = __double2loint(kd);                           // round(a·64/ln2)
  const double kf = kd - kShift;
  double r = fma(kf, -kLn2by64Hi, a);
  r = fma(kf, -kLn2by64Lo, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = p * tab[n & 63];
  // v ∈ [0.99, 2): add n >> 6 (≤ 0, ≥ −1020) to the exponent
  return __hiloint2double(__double2hiint(v) + ((n >> 6) << 20), __double2loint(v));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
}  // namespace

// Y (M×b col-major, ld m) = Φ V with V given as Vᵀ (point-major, ld ldv,
// m_pad rows, zero padded).  Grid (⌈M/64⌉, ldv / 128); 128 threads = 2 row
// warps × 2 column warps, warp tile 32 × 64.  Three CTAs per SM keep their
// own barrier phases, so one CTA's Φ generation (FP64 pipe) overlaps the
// others' DMMAs (tensor pipe).
__global__ void __launch_bounds__(128, 3)
    gram_dmma_kernel(const double* __restrict__ x, const double* __restrict__ xq, int64_t m,
                     int d, double inv2b2, const double* __restrict__ vt, int64_t ldv,
                     int64_t m_pad, int64_t b, int64_t row_begin, int64_t row_end,
                     double* __restrict__ y, int point_major) {
  constexpr int kThreads = 128;
  constexpr int kCols = kGdCols;
  constexpr int kVPitch = kCols + 8;         // ≡ 8 (mod 16) doubles: B fragments in 2 wavefronts
  constexpr int kPhiPer = kGdRows * kGdChunk / kThreads;
  extern __shared__ double gd_smem[];
  double* phi = gd_smem;                                   // [2][64][kGdPhiPitch]
  double* vs = phi + 2 * kGdRows * kGdPhiPitch;            // [2][16][kVPitch]
  double* xj = vs + 2 * kGdChunk * kVPitch;                // [2][4][16] chunk points, c_j
  __shared__ double xs[4][kGdRows];                        // the CTA's own rows
  __shared__ double exp2_tab[64];                          // 2^(i/64)
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wr = warp & 1, wc = warp >> 1;
  const int64_t row0 = row_begin + static_cast<int64_t>(blockIdx.x) * kGdRows;
  const int64_t col0 = static_cast<int64_t>(blockIdx.y) * kCols;
  const int64_t nchunks = m_pad / kGdChunk;
  const int64_t rows_end = min(row_end, m);

  // own rows as (2·inv·x_i, −inv·|x_i|²): a_ij = c_i + c_j + x_i'·x_j
  // (absolute error ≈ 1e-16·inv·(|x_i|² + |x_j|²) in a = relative in Φ_ij)
  for (int r = t; r < kGdRows; r += kThreads) {
    double q = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = (c < d && row0 + r < m) ? x[c * m + row0 + r] : 0.0;
      xs[c][r] = 2.0 * inv2b2 * v;
      q = fma(v, v, q);
    }
    xs[3][r] = -inv2b2 * q;
  }
  if (t < 64) exp2_tab[t] = c_exp2_64[t];
  // stage a chunk: its 16 × 128 slice of Vᵀ and its 16 points (cp.async)
  auto load_chunk = [&](int64_t chunk, int buf) {
    constexpr int kPieces = kGdChunk * kCols / 2;  // 16-byte pieces
    const double* src = vt + chunk * kGdChunk * ldv + col0;
    double* dst = vs + buf * kGdChunk * kVPitch;
#pragma unroll
    for (int q = t; q < kPieces; q += kThreads) {
      const int k = q / (kCols / 2), c2 = q % (kCols / 2);
      cp_async16(dst + k * kVPitch + 2 * c2, src + k * ldv + 2 * c2);
    }
    if (t < 4 * kGdChunk) {  // coordinates and c_j = −inv·|x_j|² (xq)
      const int c = t / kGdChunk, k = t % kGdChunk;
      const int64_t j = chunk * kGdChunk + k;
      double* xd = xj + (buf * 4 + c) * kGdChunk + k;
      if (c == 3)
        cp_async8(xd, xq + j);  // xq is m_pad long
      else if (c < d && j < m)
        cp_async8(xd, x + c * m + j);
      else
        *xd = 0.0;
    }
    cp_async_commit();
  };
  // Φ tile of a staged chunk into its shared-memory buffer: entry e =
  // t + i·128 is (row e & 63, chunk point e >> 6)
  auto gen_phi = [&](int64_t chunk, int buf) {
    const double* xjb = xj + buf * 4 * kGdChunk;
#pragma unroll
    for (int i = 0; i < kPhiPer; ++i) {
      const int e = t + i * kThreads;
      const int r = e & 63, k = e >> 6;
      const int64_t j = chunk * kGdChunk + k;
      double val = 0.0;
      if (row0 + r < m && j < m) {
        double a = xs[3][r] + xjb[3 * kGdChunk + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) a = fma(xs[c][r], xjb[c * kGdChunk + k], a);
        val = (row0 + r == j) ? 1.0 : exp_nonpos(fmin(a, 0.0), exp2_tab);
      }
      phi[(buf * kGdRows + r) * kGdPhiPitch + k] = val;
    }
  };

  double acc[4][8][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int n = 0; n < 8; ++n) acc[a][n][0] = acc[a][n][1] = 0.0;

  load_chunk(0, 0);
  cp_async_wait_all();
  __syncthreads();
  if (nchunks > 1) load_chunk(1, 1);
  gen_phi(0, 0);
  __syncthreads();
  const int ar = wr * 32 + (lane >> 2), ak = lane & 3;     // A fragment (row, k)
  const int bk = lane & 3, bc = wc * 64 + (lane >> 2);     // B fragment (k, column)
  // invariant at the top of chunk ch: Φ[ch] and V[ch] ready in buffer ch & 1;
  // V / points of ch + 1 in flight into the other buffer
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    const int buf = static_cast<int>(ch & 1);
    const double* ph = phi + buf * kGdRows * kGdPhiPitch;
    const double* vb = vs + buf * kGdChunk * kVPitch;
#pragma unroll 1
    for (int s4 = 0; s4 < kGdChunk / 4; ++s4) {
      double af[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = ph[(ar + 8 * a) * kGdPhiPitch + 4 * s4 + ak];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const double bf = vb[(4 * s4 + bk) * kVPitch + bc + 8 * n];
#pragma unroll
        for (int a = 0; a < 4; ++a) dmma_8x8x4(acc[a][n][0], acc[a][n][1], af[a], bf);
      }
    }
    if (ch + 1 < nchunks) {
      cp_async_wait_all();
      __syncthreads();  // V / points of ch + 1 visible; buffer `buf` free
      if (ch + 2 < nchunks) load_chunk(ch + 2, buf);
      gen_phi(ch + 1, buf ^ 1);
      __syncthreads();
    }
  }
  // C fragment: row lane >> 2, columns 2·(lane & 3) + {0, 1}; column-major
  // M×b (ld m), or point-major rows [row_begin, row_end) (ld ldv) for the
  // row-sharded product's all-gather
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t r = row0 + wr * 32 + 8 * a + (lane >> 2);
    if (r >= rows_end) continue;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int64_t c = col0 + wc * 64 + 8 * n + 2 * (lane & 3);
      if (point_major) {
        *reinterpret_cast<double2*>(y + (r - row_begin) * ldv + c) =
            make_double2(acc[a][n][0], acc[a][n][1]);
      } else {
        if (c < b) y[c * m + r] = acc[a][n][0];
        if (c + 1 < b) y[(c + 1) * m + r] = acc[a][n][1];
      }
    }
  }
}

// Deterministic Gaussian start block on the device: a counter-based
// generator (splitmix64 of (seed, index)) and Box–Muller — the same numbers
// for a given seed on every run and every GPU, without a host RNG pass over
// M·b values (72 M at C4).
__global__ void gaussian_block_kernel(double* __restrict__ v, int64_t count, uint64_t seed) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  auto mix = [](uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  const uint64_t h1 = mix(seed ^ mix(static_cast<uint64_t>(i) * 2));
  const uint64_t h2 = mix(seed ^ mix(static_cast<uint64_t>(i) * 2 + 1));
  const double u1 = (static_cast<double>(h1 >> 11) + 0.5) * 0x1p-53;  // (0, 1)
  const double u2 = static_cast<double>(h2 >> 11) * 0x1p-53;
  v[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// res[i] = ‖z_i − θ_i u_i‖₂ for the K Ritz pairs (one CTA per column).
__global__ void __launch_bounds__(256) ritz_residual_kernel(const double* __restrict__ z,
                                                            const double* __restrict__ u,
                                                            const double* __restrict__ theta,
                                                            int64_t m, double* __restrict__ res) {
  const int64_t col = blockIdx.x;
  const double th = theta[col];
  const double* zc = z + col * m;
  const double* uc = u + col * m;
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < m; r += 256) {
    const double e = zc[r] - th * uc[r];
    s = fma(e, e, s);
  }
  __shared__ double red[8];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    res[col] = sqrt(t);
  }
}

GramPlan make_gram_plan(int64_t m, int64_t b) {
  GramPlan g;
  g.col_blocks = ceil_div(b, kGdCols);
  g.ldv = g.col_blocks * kGdCols;
  g.m_pad = ceil_div(m, kGdChunk) * kGdChunk;
  return g;
}

static void gram_prepare(const double* x, int64_t m, int d, double inv, const double* v,
                         int64_t b, double* vt, const GramPlan& g, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    double tab[64];
    for (int i = 0; i < 64; ++i) tab[i] = std::exp2(i / 64.0);
    FCPD_CUDA(cudaMemcpyToSymbol(c_exp2_64, tab, sizeof tab));
    FCPD_CUDA(cudaFuncSetAttribute(gram_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kGdSmem)));
    attr = true;
  }
  dim3 tg(static_cast<unsigned>(ceil_div(g.m_pad, 32)), static_cast<unsigned>(ceil_div(g.ldv, 32)));
  transpose_pad_kernel<<<tg, dim3(32, 8), 0, stream>>>(v, m, b, vt, g.m_pad, g.ldv);
  FCPD_LAUNCH_CHECK();
  double* xq = vt + g.m_pad * g.ldv;  // scratch tail of vt (m_pad doubles)
  gram_rownorm_kernel<<<static_cast<unsigned>(ceil_div(g.m_pad, 256)), 256, 0, stream>>>(
      x, m, d, inv, g.m_pad, xq);
  FCPD_LAUNCH_CHECK();
}

static void gram_rows(const double* x, int64_t m, int d, double inv, const double* vt,
                      const GramPlan& g, int64_t b, int64_t r0, int64_t r1, double* y,
                      int point_major, cudaStream_t stream) {
  if (r1 <= r0) return;
  const double* xq = vt + g.m_pad * g.ldv;
  dim3 grid(static_cast<unsigned>(ceil_div(r1 - r0, kGdRows)), static_cast<unsigned>(g.col_blocks));
  gram_dmma_kernel<<<grid, 128, kGdSmem, stream>>>(x, xq, m, d, inv, vt, g.ldv, g.m_pad, b, r0, r1,
                                                   y, point_major);
  FCPD_LAUNCH_CHECK();
}

void gram_matmul(const double* x, int64_t m, int d, double beta, const double* v, int64_t b,
                 double* y, double* vt, const GramPlan& g, cudaStream_t stream) {
  const double inv = 1.0 / (2.0 * beta * beta);
  if (std::getenv("FCPD_GRAM_DFMA")) {  // round-1 DFMA tile kernel, for A/B measurements
    constexpr size_t smem = sizeof(double) * (kGvTileK * (kGvTileM + kGvTileN) + 3 * kGvTileM);
    static bool attr = false;
    if (!attr) {
      FCPD_CUDA(cudaFuncSetAttribute(gram_matmul_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      attr = true;
    }
    dim3 grid(ceil_div(m, kGvTileM), ceil_div(b, kGvTileN));
    gram_matmul_kernel<<<grid, 256, smem, stream>>>(x, m, d, inv, v, b, y);
    FCPD_LAUNCH_CHECK();
    return;
  }
  gram_prepare(x, m, d, inv, v, b, vt, g, stream);
  gram_rows(x, m, d, inv, vt, g, b, 0, m, y, 0, stream);
}

// Row-sharded W = Φ V over a rank group: each local rank q computes its
// block of rows [q·rows, (q+1)·rows) point-major into its slice of wpm,
// an all-gather completes wpm on every rank, and one transpose gives the
// column-major W the orthonormalisation needs.
void gram_matmul_sharded(const double* x, int64_t m, int d, double beta, const double* v,
                         int64_t b, double* y, double* vt, const GramPlan& g, double* wpm,
                         const GramShards& sh, cudaStream_t stream) {
  const double inv = 1.0 / (2.0 * beta * beta);
  const int64_t rows = sh.block_rows(m);
  gram_prepare(x, m, d, inv, v, b, vt, g, stream);
  std::vector<const uint32_t*> send;
  std::vector<uint32_t*> recv;
  for (int q : sh.ranks) {
    double* blk = wpm + static_cast<int64_t>(q) * rows * g.ldv;
    gram_rows(x, m, d, inv, vt, g, b, q * rows, std::min<int64_t>((q + 1) * rows, m), blk, 1,
              stream);
    send.push_back(reinterpret_cast<const uint32_t*>(blk));
    recv.push_back(reinterpret_cast<uint32_t*>(wpm));
  }
  sh.comm->all_gather(send, recv, static_cast<size_t>(rows * g.ldv * 2), stream);
  dim3 tg(static_cast<unsigned>(ceil_div(m, 32)), static_cast<unsigned>(ceil_div(b, 32)));
  untranspose_kernel<<<tg, dim3(32, 8), 0, stream>>>(wpm, g.ldv, m, b, y);
  FCPD_LAUNCH_CHECK();
}

namespace {

// In-place thin QR orthonormalisation of the M×b column-major block.
struct Orth {
  cusolverDnHandle_t h;
  int64_t m, b;
  double* tau = nullptr;
  double* work = nullptr;
  int* info = nullptr;
  int lwork = 0;
  Orth(cusolverDnHandle_t h_, int64_t m_, int64_t b_, double* a) : h(h_), m(m_), b(b_) {
    int l1 = 0, l2 = 0;
    FCPD_CUSOLVER2(cusolverDnDgeqrf_bufferSize(h, static_cast<int>(m), static_cast<int>(b), a,
                                               static_cast<int>(m), &l1));
    FCPD_CUDA(cudaMalloc(&tau, sizeof(double) * b));
    FCPD_CUSOLVER2(cusolverDnDorgqr_bufferSize(h, static_cast<int>(m), static_cast<int>(b),
                                               static_cast<int>(b), a, static_cast<int>(m), tau,
                                               &l2));
    lwork = std::max(l1, l2);
    FCPD_CUDA(cudaMalloc(&work, sizeof(double) * std::max(lwork, 1)));
    FCPD_CUDA(cudaMalloc(&info, sizeof(int)));
  }
  ~Orth() {
    cudaFree(tau);
    cudaFree(work);
    cudaFree(info);
  }
  void run(double* a) {
    FCPD_CUSOLVER2(cusolverDnDgeqrf(h, static_cast<int>(m), static_cast<int>(b), a,
                                    static_cast<int>(m), tau, work, lwork, info));
    FCPD_CUSOLVER2(cusolverDnDorgqr(h, static_cast<int>(m), static_cast<int>(b),
                                    static_cast<int>(b), a, static_cast<int>(m), tau, work, lwork,
                                    info));
  }
};

}  // namespace

void topk_eigensolve(cusolverDnHandle_t solver, cublasHandle_t blas, const double* x_dev,
                     int64_t m, int d, double beta, int64_t rank, int iterations, bool adaptive,
                     uint64_t seed, Basis& b_out, cudaStream_t stream, double* u_host_out,
                     int* products_out, const GramShards* shards,
                     const std::vector<Basis*>* also_out) {
  if (rank < 1 || rank > m) throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: rank out of [1, M]");
  if (!(beta > 0.0)) throw Failure(FCPD_ERR_PARAMETER, "build_gram: beta must be positive");
  const int64_t over = std::max<int64_t>(16, rank / 5);
  const int64_t b = std::min<int64_t>(m, rank + over);
  if (m > INT32_MAX / 2) throw Failure(FCPD_ERR_PARAMETER, "topk: M too large");
  FCPD_CUSOLVER2(cusolverDnSetStream(solver, stream));
  FCPD_CUBLAS(cublasSetStream(blas, stream));

  double *v = nullptr, *w = nullptr, *t = nullptr, *evals = nullptr, *u = nullptr, *z = nullptr,
         *res = nullptr, *dwork = nullptr, *vt = nullptr, *wpm = nullptr;
  int* info = nullptr;
  cusolverDnParams_t params = nullptr;
  auto release = [&] {
    cudaFree(v);
    cudaFree(w);
    cudaFree(t);
    cudaFree(evals);
    cudaFree(u);
    cudaFree(z);
    cudaFree(res);
    cudaFree(dwork);
    cudaFree(vt);
    cudaFree(wpm);
    cudaFree(info);
    if (params) cusolverDnDestroyParams(params);
  };
  try {
    FCPD_CUDA(cudaMalloc(&v, sizeof(double) * m * b));
    FCPD_CUDA(cudaMalloc(&w, sizeof(double) * m * b));
    FCPD_CUDA(cudaMalloc(&t, sizeof(double) * b * b));
    FCPD_CUDA(cudaMalloc(&evals, sizeof(double) * b));
    FCPD_CUDA(cudaMalloc(&u, sizeof(double) * m * rank));
    FCPD_CUDA(cudaMalloc(&info, sizeof(int)));
    const GramPlan gp = make_gram_plan(m, b);
    FCPD_CUDA(cudaMalloc(&vt, sizeof(double) * gp.m_pad * (gp.ldv + 1)));  // + xq
    if (shards && shards->comm && shards->comm->world > 1)
      FCPD_CUDA(cudaMalloc(&wpm, sizeof(double) * shards->block_rows(m) * shards->comm->world *
                                     gp.ldv));
    else
      shards = nullptr;
    // symmetric eigensolver workspace for the b×b Rayleigh quotient
    FCPD_CUSOLVER2(cusolverDnCreateParams(&params));
    size_t dbytes = 0, hbytes = 0;
    FCPD_CUSOLVER2(cusolverDnXsyevd_bufferSize(solver, params, CUSOLVER_EIG_MODE_VECTOR,
                                               CUBLAS_FILL_MODE_LOWER, b, CUDA_R_64F, t, b,
                                               CUDA_R_64F, evals, CUDA_R_64F, &dbytes, &hbytes));
    std::vector<char> hwork(std::max<size_t>(hbytes, 8));
    FCPD_CUDA(cudaMalloc(&dwork, std::max<size_t>(dbytes, 8)));
    // deterministic Gaussian start block (device counter-based RNG)
    gaussian_block_kernel<<<ceil_div(m * b, 256), 256, 0, stream>>>(v, m * b,
                                                                    seed ^ 0x9E3779B97F4A7C15ull);
    FCPD_LAUNCH_CHECK();
    Orth orth(solver, m, b, v);
    orth.run(v);
    const double one = 1.0, zero = 0.0;
    const double* s_top = t + (b - rank) * b;  // eigenvectors of the top `rank` Ritz values
    std::vector<double> hres(rank), hev(b);
    int products = 0;
    for (int step = 0;; ++step) {
      if (shards)  // W = G V
        gram_matmul_sharded(x_dev, m, d, beta, v, b, w, vt, gp, wpm, *shards, stream);
      else
        gram_matmul(x_dev, m, d, beta, v, b, w, vt, gp, stream);
      ++products;
      const bool last = step >= iterations;
      if (!last && !(adaptive && step >= 1)) {
        std::swap(v, w);
        orth.run(v);
        continue;
      }
      // Rayleigh–Ritz: T = Vᵀ W, T = S Θ Sᵀ, U = V S[:, top]
      FCPD_CUBLAS(cublasDgemm(blas, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(b),
                              static_cast<int>(b), static_cast<int>(m), &one, v,
                              static_cast<int>(m), w, static_cast<int>(m), &zero, t,
                              static_cast<int>(b)));
      const cusolverStatus_t st =
          cusolverDnXsyevd(solver, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, b,
                           CUDA_R_64F, t, b, CUDA_R_64F, evals, CUDA_R_64F, dwork, dbytes,
                           hwork.data(), hbytes, info);
      int hinfo = 0;
      FCPD_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, stream));
      FCPD_CUDA(cudaStreamSynchronize(stream));
      if (st != CUSOLVER_STATUS_SUCCESS || hinfo != 0)
        throw Failure(FCPD_ERR_NUMERIC,
                      "eigendecompose: symmetric eigensolver did not converge (info=" +
                          std::to_string(hinfo) + ")");
      FCPD_CUBLAS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(m),
                              static_cast<int>(rank), static_cast<int>(b), &one, v,
                              static_cast<int>(m), s_top, static_cast<int>(b), &zero, u,
                              static_cast<int>(m)));
      if (last) break;
      // residuals ‖G u_i − θ_i u_i‖ with G u_i = W s_i
      if (!z) {
        FCPD_CUDA(cudaMalloc(&z, sizeof(double) * m * rank));
        FCPD_CUDA(cudaMalloc(&res, sizeof(double) * rank));
      }
      FCPD_CUBLAS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(m),
                              static_cast<int>(rank), static_cast<int>(b), &one, w,
                              static_cast<int>(m), s_top, static_cast<int>(b), &zero, z,
                              static_cast<int>(m)));
      ritz_residual_kernel<<<static_cast<unsigned>(rank), 256, 0, stream>>>(z, u, evals + b - rank,
                                                                            m, res);
      FCPD_LAUNCH_CHECK();
      FCPD_CUDA(cudaMemcpyAsync(hres.data(), res, sizeof(double) * rank, cudaMemcpyDeviceToHost,
                                stream));
      FCPD_CUDA(cudaMemcpyAsync(hev.data(), evals, sizeof(double) * b, cudaMemcpyDeviceToHost,
                                stream));
      FCPD_CUDA(cudaStreamSynchronize(stream));
      const double tol = kTopkResidualTol * std::fabs(hev[b - 1]);
      double worst = *std::max_element(hres.begin(), hres.end());
      if (shards) {  // every rank takes the same decision (the collectives stay in step)
        std::vector<std::vector<double>> wv(shards->ranks.size(), std::vector<double>(1, worst));
        shards->comm->host_all_reduce(wv, true, stream);
        worst = wv[0][0];
      }
      if (std::getenv("FCPD_TOPK_LOG"))
        std::fprintf(stderr, "topk: M=%lld K=%lld product %d residual %.3e·θ₁\n",
                     static_cast<long long>(m), static_cast<long long>(rank), products,
                     worst / std::fabs(hev[b - 1]));
      if (worst <= tol) break;
      std::swap(v, w);
      orth.run(v);
    }
    if (products_out) *products_out = products;
    std::vector<double> eh(b);
    FCPD_CUDA(cudaMemcpyAsync(eh.data(), evals, sizeof(double) * b, cudaMemcpyDeviceToHost,
                              stream));
    FCPD_CUDA(cudaStreamSynchronize(stream));
    // pack descending: column i of the basis = Ritz vector of eigenvalue b-1-i,
    // i.e. column rank-1-i of u
    std::vector<double> lam_raw(rank);
    for (int64_t i = 0; i < rank; ++i) lam_raw[i] = eh[b - 1 - i];
    if (u_host_out) {  // descending column order, column-major M×rank
      for (int64_t i = 0; i < rank; ++i)
        FCPD_CUDA(cudaMemcpyAsync(u_host_out + i * m, u + (rank - 1 - i) * m,
                                  sizeof(double) * m, cudaMemcpyDeviceToHost, stream));
      FCPD_CUDA(cudaStreamSynchronize(stream));
    }
    pack_basis_from(b_out, u, m, rank, /*reverse=*/1, lam_raw, stream);
    if (also_out)
      for (Basis* bo : *also_out) pack_basis_from(*bo, u, m, rank, /*reverse=*/1, lam_raw, stream);
  } catch (...) {
    release();
    throw;
  }
  release();
}

}  // namespace fcpd
