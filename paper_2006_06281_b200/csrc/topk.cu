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
//   repeat q times:  V ← orth(G V)                 (G·V on the fly, fp64)
//   W = G V,  T = Vᵀ W,  T = S Θ Sᵀ,  U = V S[:, :K],  λ = Θ[:K] (descending)
//   λ_i < 1e-12·λ_max → 0                           (kernel.hpp:68-70)
//
// The Gaussian kernel's spectrum decays super-exponentially (SURVEY App.
// A.4), so the eigenpairs that move x̃ (λ ≳ 1e-10 λ₁) converge in a few
// iterations; eigenpairs below the fp64 noise floor are arbitrary exactly as
// they are in any fp64 dense solver, and the filter λ/(λ+λσ²) ≈ 0 mutes them.
//
// G·V kernel: 128×128 output tile per CTA, 256 threads × (8×8) fp64
// accumulators; per 32-wide reduction chunk the CTA regenerates the 128×32
// Φ tile (fp64 exp of the difference form — symmetric, diagonal exactly 1)
// into shared memory next to the 32×128 V tile.  Bound: FP64 FMA pipe.

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
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

void gram_matmul(const double* x, int64_t m, int d, double beta, const double* v, int64_t b,
                 double* y, cudaStream_t stream) {
  const double inv = 1.0 / (2.0 * beta * beta);
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
                     int64_t m, int d, double beta, int64_t rank, int iterations, uint64_t seed,
                     Basis& b_out, cudaStream_t stream, double* u_host_out) {
  if (rank < 1 || rank > m) throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: rank out of [1, M]");
  if (!(beta > 0.0)) throw Failure(FCPD_ERR_PARAMETER, "build_gram: beta must be positive");
  const int64_t over = std::max<int64_t>(16, rank / 5);
  const int64_t b = std::min<int64_t>(m, rank + over);
  if (m > INT32_MAX / 2) throw Failure(FCPD_ERR_PARAMETER, "topk: M too large");
  FCPD_CUSOLVER2(cusolverDnSetStream(solver, stream));
  FCPD_CUBLAS(cublasSetStream(blas, stream));

  double *v = nullptr, *w = nullptr, *t = nullptr, *evals = nullptr, *u = nullptr;
  try {
    FCPD_CUDA(cudaMalloc(&v, sizeof(double) * m * b));
    FCPD_CUDA(cudaMalloc(&w, sizeof(double) * m * b));
    FCPD_CUDA(cudaMalloc(&t, sizeof(double) * b * b));
    FCPD_CUDA(cudaMalloc(&evals, sizeof(double) * b));
    // deterministic Gaussian start block (device counter-based RNG)
    gaussian_block_kernel<<<ceil_div(m * b, 256), 256, 0, stream>>>(v, m * b,
                                                                    seed ^ 0x9E3779B97F4A7C15ull);
    FCPD_LAUNCH_CHECK();
    Orth orth(solver, m, b, v);
    orth.run(v);
    for (int it = 0; it < iterations; ++it) {
      gram_matmul(x_dev, m, d, beta, v, b, w, stream);
      std::swap(v, w);
      orth.run(v);
    }
    // Rayleigh–Ritz
    gram_matmul(x_dev, m, d, beta, v, b, w, stream);
    const double one = 1.0, zero = 0.0;
    FCPD_CUBLAS(cublasDgemm(blas, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(b),
                            static_cast<int>(b), static_cast<int>(m), &one, v,
                            static_cast<int>(m), w, static_cast<int>(m), &zero, t,
                            static_cast<int>(b)));
    // symmetric eigensolve of the b×b Rayleigh quotient (lower triangle)
    {
      cusolverDnParams_t params;
      FCPD_CUSOLVER2(cusolverDnCreateParams(&params));
      size_t dbytes = 0, hbytes = 0;
      FCPD_CUSOLVER2(cusolverDnXsyevd_bufferSize(solver, params, CUSOLVER_EIG_MODE_VECTOR,
                                                 CUBLAS_FILL_MODE_LOWER, b, CUDA_R_64F, t, b,
                                                 CUDA_R_64F, evals, CUDA_R_64F, &dbytes,
                                                 &hbytes));
      void* dwork = nullptr;
      int* info = nullptr;
      std::vector<char> hwork(std::max<size_t>(hbytes, 8));
      FCPD_CUDA(cudaMalloc(&dwork, std::max<size_t>(dbytes, 8)));
      FCPD_CUDA(cudaMalloc(&info, sizeof(int)));
      const cusolverStatus_t st =
          cusolverDnXsyevd(solver, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, b,
                           CUDA_R_64F, t, b, CUDA_R_64F, evals, CUDA_R_64F, dwork, dbytes,
                           hwork.data(), hbytes, info);
      int hinfo = 0;
      cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, stream);
      cudaStreamSynchronize(stream);
      cudaFree(dwork);
      cudaFree(info);
      cusolverDnDestroyParams(params);
      if (st != CUSOLVER_STATUS_SUCCESS || hinfo != 0)
        throw Failure(FCPD_ERR_NUMERIC,
                      "eigendecompose: symmetric eigensolver did not converge (info=" +
                          std::to_string(hinfo) + ")");
    }
    // Ritz vectors for the top `rank` (eigenvalues ascending → last columns)
    FCPD_CUDA(cudaMalloc(&u, sizeof(double) * m * rank));
    FCPD_CUBLAS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(m),
                            static_cast<int>(rank), static_cast<int>(b), &one, v,
                            static_cast<int>(m), t + (b - rank) * b, static_cast<int>(b), &zero,
                            u, static_cast<int>(m)));
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
  } catch (...) {
    cudaFree(v);
    cudaFree(w);
    cudaFree(t);
    cudaFree(evals);
    cudaFree(u);
    throw;
  }
  cudaFree(v);
  cudaFree(w);
  cudaFree(t);
  cudaFree(evals);
  cudaFree(u);
}

}  // namespace fcpd
