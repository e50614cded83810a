// setup.cu — one-time spectral setup on the device (kernel.hpp:31-72).
//
// build_gram: Φ_ij = exp(−‖x_i − x_j‖² / 2β²) in fp64, diagonal pinned to 1.
// The difference form makes Φ exactly symmetric, which is what the
// reference's explicit symmetrisation (kernel.hpp:42-45) enforces.
// eigendecompose: cuSOLVER Xsyevd (fp64, divide & conquer) in place of
// Eigen::SelfAdjointEigenSolver; eigenpairs are reordered descending, the
// top `rank` kept, and λ < 1e-12·λ_max clamped to 0 (kernel.hpp:59-70).
// The basis is then packed for the streaming M-step as Q (M×K row-major)
// and Qᵀ (K×M row-major) in fp32 (rounding Q to fp32 moves
// V by ≈ 2e-7‖R‖; λ stays fp64).

#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "setup.cuh"

namespace fcpd {

#define FCPD_CUSOLVER(call)                                                        \
  do {                                                                             \
    cusolverStatus_t s_ = (call);                                                  \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                             \
      throw ::fcpd::Failure(FCPD_ERR_CUDA,                                          \
                            std::string(#call) + ": cusolver status " + std::to_string(s_)); \
  } while (0)

__global__ void gram_kernel(const double* __restrict__ x, int64_t m, int d, double inv2b2,
                            double* __restrict__ phi, int64_t ld) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (i >= m) return;
  double s = 0.0;
  for (int c = 0; c < d; ++c) {
    const double t = x[c * m + i] - x[c * m + j];
    s += t * t;
  }
  phi[j * ld + i] = (i == j) ? 1.0 : exp(-s * inv2b2);
}

// QT[i][r] = V[r + src(i)·ldv]  (row i of Qᵀ = eigenvector src(i))
__global__ void pack_qt_kernel(const double* __restrict__ v, int64_t ldv, int64_t m,
                               int64_t ncols, int reverse, float* __restrict__ qt,
                               int64_t mpad) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  const int64_t src = reverse ? ncols - 1 - i : i;
  if (r < mpad) qt[i * mpad + r] = r < m ? static_cast<float>(v[src * ldv + r]) : 0.f;
}

// Q[r][i] = V[r + src(i)·ldv] via a 32×32 shared-memory transpose.
__global__ void pack_q_kernel(const double* __restrict__ v, int64_t ldv, int64_t m,
                              int64_t ncols, int64_t k, int reverse, float* __restrict__ q,
                              int64_t kpad) {
  __shared__ float tile[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    const int64_t i = i0 + yy, r = r0 + threadIdx.x;
    float val = 0.f;
    if (i < k && r < m) {
      const int64_t src = reverse ? ncols - 1 - i : i;
      val = static_cast<float>(v[src * ldv + r]);
    }
    tile[yy][threadIdx.x] = val;
  }
  __syncthreads();
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    const int64_t r = r0 + yy, i = i0 + threadIdx.x;
    if (r < m && i < kpad) q[r * kpad + i] = tile[threadIdx.x][yy];
  }
}

void Basis::release() {
  if (q) cudaFree(q);
  if (qt) cudaFree(qt);
  if (lam) cudaFree(lam);
  if (u64) cudaFree(u64);
  q = qt = nullptr;
  lam = u64 = nullptr;
  lam_raw_host.clear();
  lam_host.clear();
  m = k = 0;
}

void build_gram_device(const double* x_dev, int64_t m, int d, double beta, double* phi,
                       int64_t ld, cudaStream_t stream) {
  if (!(beta > 0.0)) throw Failure(FCPD_ERR_PARAMETER, "build_gram: beta must be positive");
  const double inv = 1.0 / (2.0 * beta * beta);
  gram_kernel<<<dim3(ceil_div(m, 128), static_cast<unsigned>(m)), 128, 0, stream>>>(x_dev, m, d,
                                                                                     inv, phi, ld);
  FCPD_LAUNCH_CHECK();
}

static void alloc_basis(Basis& b, int64_t m, int64_t k) {
  b.release();
  b.m = m;
  b.k = k;
  b.kpad = (k + 3) / 4 * 4;
  b.mpad = (m + 3) / 4 * 4;
  FCPD_CUDA(cudaMalloc(&b.q, sizeof(float) * m * b.kpad));
  FCPD_CUDA(cudaMalloc(&b.qt, sizeof(float) * k * b.mpad));
  FCPD_CUDA(cudaMalloc(&b.lam, sizeof(double) * 2 * k));
  FCPD_CUDA(cudaMalloc(&b.u64, sizeof(double) * m * k));
}

// u64[:, i] = V[:, src(i)] (fp64 copy kept for the spectral cache)
__global__ void pack_u64_kernel(const double* __restrict__ v, int64_t ldv, int64_t m,
                                int64_t ncols, int reverse, double* __restrict__ u) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  const int64_t src = reverse ? ncols - 1 - i : i;
  if (r < m) u[i * m + r] = v[src * ldv + r];
}

void pack_basis(Basis& b, const double* v, int64_t ldv, int64_t ncols, int reverse,
                cudaStream_t stream) {
  pack_qt_kernel<<<dim3(ceil_div(b.mpad, 256), static_cast<unsigned>(b.k)), 256, 0, stream>>>(
      v, ldv, b.m, ncols, reverse, b.qt, b.mpad);
  FCPD_LAUNCH_CHECK();
  pack_u64_kernel<<<dim3(ceil_div(b.m, 256), static_cast<unsigned>(b.k)), 256, 0, stream>>>(
      v, ldv, b.m, ncols, reverse, b.u64);
  FCPD_LAUNCH_CHECK();
  pack_q_kernel<<<dim3(ceil_div(b.m, 32), ceil_div(b.kpad, 32)), dim3(32, 8), 0, stream>>>(
      v, ldv, b.m, ncols, b.k, reverse, b.q, b.kpad);
  FCPD_LAUNCH_CHECK();
}

void upload_lambda(Basis& b, bool full_rank, cudaStream_t stream) {
  // lam[0..k) = clamped λ (solver diagonal); lam[k..2k) = λ in the transform
  // numerator: raw for full rank (Φ W uses the unclamped Φ), clamped for low
  // rank (apply_transform_lowrank uses basis.lambda).
  std::vector<double> h(2 * b.k);
  for (int64_t i = 0; i < b.k; ++i) {
    h[i] = b.lam_host[i];
    h[b.k + i] = full_rank ? b.lam_raw_host[i] : b.lam_host[i];
  }
  FCPD_CUDA(cudaMemcpyAsync(b.lam, h.data(), sizeof(double) * 2 * b.k, cudaMemcpyHostToDevice,
                            stream));
  FCPD_CUDA(cudaStreamSynchronize(stream));
  b.full_rank = full_rank;
}

void clamp_lambda(Basis& b) {
  b.lam_host = b.lam_raw_host;
  const double floor = 1e-12 * std::max(b.lam_host[0], 0.0);  // kernel.hpp:68-70
  for (auto& v : b.lam_host)
    if (v < floor) v = 0.0;
}

void dense_eigensolve(cusolverDnHandle_t h, double* phi, int64_t m, int64_t rank, Basis& b,
                      double* u_out_host, cudaStream_t stream) {
  if (rank < 1 || rank > m) throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: rank out of [1, M]");
  FCPD_CUSOLVER(cusolverDnSetStream(h, stream));
  cusolverDnParams_t params;
  FCPD_CUSOLVER(cusolverDnCreateParams(&params));
  double* w = nullptr;
  int* info = nullptr;
  void* dwork = nullptr;
  std::vector<char> hwork;
  size_t dbytes = 0, hbytes = 0;
  try {
    FCPD_CUDA(cudaMalloc(&w, sizeof(double) * m));
    FCPD_CUDA(cudaMalloc(&info, sizeof(int)));
    FCPD_CUSOLVER(cusolverDnXsyevd_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR,
                                              CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, phi, m,
                                              CUDA_R_64F, w, CUDA_R_64F, &dbytes, &hbytes));
    FCPD_CUDA(cudaMalloc(&dwork, std::max<size_t>(dbytes, 8)));
    hwork.resize(std::max<size_t>(hbytes, 8));
    FCPD_CUSOLVER(cusolverDnXsyevd(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m,
                                   CUDA_R_64F, phi, m, CUDA_R_64F, w, CUDA_R_64F, dwork, dbytes,
                                   hwork.data(), hbytes, info));
    int hinfo = 0;
    FCPD_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, stream));
    std::vector<double> wh(m);
    FCPD_CUDA(cudaMemcpyAsync(wh.data(), w, sizeof(double) * m, cudaMemcpyDeviceToHost, stream));
    FCPD_CUDA(cudaStreamSynchronize(stream));
    if (hinfo != 0)
      throw Failure(FCPD_ERR_NUMERIC,
                    "eigendecompose: symmetric eigensolver did not converge (info=" +
                        std::to_string(hinfo) + ")");
    alloc_basis(b, m, rank);
    b.lam_raw_host.resize(rank);
    for (int64_t i = 0; i < rank; ++i) b.lam_raw_host[i] = wh[m - 1 - i];
    clamp_lambda(b);
    pack_basis(b, phi, m, m, /*reverse=*/1, stream);
    if (u_out_host) {
      // eigenvector columns in descending order, column-major M×rank
      FCPD_CUDA(cudaMemcpyAsync(u_out_host, phi + (m - rank) * m, sizeof(double) * m * rank,
                                cudaMemcpyDeviceToHost, stream));
      FCPD_CUDA(cudaStreamSynchronize(stream));
      // reverse column order in place on the host
      std::vector<double> tmp(m);
      for (int64_t i = 0; i < rank / 2; ++i) {
        double* a = u_out_host + i * m;
        double* c = u_out_host + (rank - 1 - i) * m;
        std::copy(a, a + m, tmp.begin());
        std::copy(c, c + m, a);
        std::copy(tmp.begin(), tmp.end(), c);
      }
    }
    FCPD_CUDA(cudaStreamSynchronize(stream));
  } catch (...) {
    cudaFree(w);
    cudaFree(info);
    cudaFree(dwork);
    cusolverDnDestroyParams(params);
    throw;
  }
  cudaFree(w);
  cudaFree(info);
  cudaFree(dwork);
  cusolverDnDestroyParams(params);
}

void pack_basis_from(Basis& b, const double* u_dev, int64_t m, int64_t k, int reverse,
                     const std::vector<double>& lam_raw, cudaStream_t stream) {
  alloc_basis(b, m, k);
  pack_basis(b, u_dev, m, k, reverse, stream);
  b.lam_raw_host = lam_raw;
  clamp_lambda(b);
  FCPD_CUDA(cudaStreamSynchronize(stream));
}

void basis_from_host(Basis& b, const double* u_host, const double* lam_host, int64_t m,
                     int64_t k, cudaStream_t stream) {
  double* v = nullptr;
  FCPD_CUDA(cudaMalloc(&v, sizeof(double) * m * k));
  try {
    FCPD_CUDA(cudaMemcpyAsync(v, u_host, sizeof(double) * m * k, cudaMemcpyHostToDevice, stream));
    alloc_basis(b, m, k);
    pack_basis(b, v, m, k, /*reverse=*/0, stream);
    b.lam_raw_host.assign(lam_host, lam_host + k);
    b.lam_host = b.lam_raw_host;
    FCPD_CUDA(cudaStreamSynchronize(stream));
  } catch (...) {
    cudaFree(v);
    throw;
  }
  cudaFree(v);
}

}  // namespace fcpd
