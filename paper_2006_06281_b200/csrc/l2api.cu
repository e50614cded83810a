// l2api.cu — the reference's L2 functions as C-ABI entry points, in fp64 on
// the device (include/fcpd_capi.h "fine-grained entry points").
//
// These are the calls the reference's own unit tests make directly
// (proj/tests/test_correspondence.cpp, test_solvers.cpp, test_kernel.cpp),
// so they keep the reference's fp64 semantics and tolerances: dense P and Φ
// as the caller passes them, products through cuBLAS dgemm (plain library
// GEMMs), reductions in a fixed order.  The EM hot path does NOT go through
// here — register_pointsets runs the fused fp32-pair / fp64-sum kernels of
// estep.cu and the basis streams of mstep*.cu.
//
//   estimated_targets       correspondence.hpp:101-105   P·Y
//   enforce_row_constraint  correspondence.hpp:83-98     row normalise / uniform row
//   update_sigma2           solvers.hpp:160-176          trace form
//   eigendecompose          kernel.hpp:49-72             cuSOLVER syevd of a given Φ
//   solve_fast[_lowrank]    solvers.hpp:61-80            U·diag(1/(λ+λσ²))·Uᵀ·R
//   apply_transform         solvers.hpp:138-144          X + Φ·W
//   apply_transform_lowrank solvers.hpp:147-155          X + U·Λ·Uᵀ·W
//   lowrank_reconstruction_error kernel.hpp:76-83        ‖Φ − UΛUᵀ‖_F

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "setup.cuh"

#define FCPD_CUBLAS_L2(call)                                                             \
  do {                                                                                   \
    cublasStatus_t s_ = (call);                                                          \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                     \
      throw ::fcpd::Failure(FCPD_ERR_CUDA,                                               \
                            std::string(#call) + ": cublas status " + std::to_string(s_)); \
  } while (0)

namespace fcpd {
namespace {

// Device scratch freed at scope exit (these entry points are not on the hot
// path; allocation per call keeps them stateless like the reference's).
template <typename T>
struct Scratch {
  T* p = nullptr;
  explicit Scratch(size_t count) {
    FCPD_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
  }
  ~Scratch() {
    if (p) cudaFree(p);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

template <typename T>
T* upload(Scratch<T>& d, const T* h, size_t count, cudaStream_t s) {
  FCPD_CUDA(cudaMemcpyAsync(d.p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  return d.p;
}

// C (m×n) = alpha·op(A)·op(B) + beta·C, column-major fp64.
void dgemm(cublasHandle_t h, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
           const double* a, int64_t lda, const double* b, int64_t ldb, double beta, double* c,
           int64_t ldc) {
  FCPD_CUBLAS_L2(cublasDgemm(h, ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb ? CUBLAS_OP_T : CUBLAS_OP_N,
                             static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                             &alpha, a, static_cast<int>(lda), b, static_cast<int>(ldb), &beta,
                             c, static_cast<int>(ldc)));
}

// row sums of a column-major M×N matrix: one thread per row, columns in
// increasing order (fixed order; consecutive threads read consecutive words)
__global__ void row_sums_kernel(const double* __restrict__ p, int64_t m, int64_t n,
                                double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int64_t j = 0; j < n; ++j) s += p[j * m + i];
  out[i] = s;
}

// enforce_row_constraint (correspondence.hpp:83-98): rows with sum < 1e-300
// become uniform 1/N (flagged), the others are divided by their sum.
__global__ void row_constrain_kernel(double* __restrict__ p, int64_t m, int64_t n,
                                     const double* __restrict__ sums,
                                     int32_t* __restrict__ degenerate) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double s = sums[i];
  const bool deg = s < 1e-300;
  degenerate[i] = deg ? 1 : 0;
  const double u = 1.0 / static_cast<double>(n);
  for (int64_t j = 0; j < n; ++j) p[j * m + i] = deg ? u : p[j * m + i] / s;
}

// column sums of a column-major M×N matrix: a warp per column (coalesced
// over its contiguous M entries), lanes strided, fixed xor tree
__global__ void col_sums_kernel(const double* __restrict__ p, int64_t m, int64_t n,
                                double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= n) return;
  double s = 0.0;
  for (int64_t i = lane; i < m; i += 32) s += p[j * m + i];
  s = warp_sum(s);
  if (lane == 0) out[j] = s;
}

// the three traces of update_sigma2 (solvers.hpp:166-172) in one block,
// fixed order: Σ_n |y_n|²·(Pᵀ1)_n, Σ Ỹ⊙X̃, ‖X̃‖²_F
__global__ void sigma2_traces_kernel(const double* __restrict__ y, int64_t n,
                                     const double* __restrict__ pt1,
                                     const double* __restrict__ ytilde,
                                     const double* __restrict__ xt, int64_t m, int d,
                                     double* __restrict__ out) {
  __shared__ double red[3][32];
  double a = 0.0, b = 0.0, c = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double q = 0.0;
    for (int k = 0; k < d; ++k) q += y[k * n + j] * y[k * n + j];
    a += q * pt1[j];
  }
  for (int64_t i = threadIdx.x; i < m * d; i += blockDim.x) {
    b += ytilde[i] * xt[i];
    c += xt[i] * xt[i];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  c = warp_sum(c);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = a;
    red[1][w] = b;
    red[2][w] = c;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s[k] += red[k][i];
  out[0] = s[0];
  out[1] = s[1];
  out[2] = s[2];
}

// rows of z (K×D, column-major) scaled by 1/(λ_k + shift) (solve) or by λ_k
// (low-rank transform)
__global__ void scale_rows_kernel(double* __restrict__ z, int64_t k, int d,
                                  const double* __restrict__ lam, double shift, int divide) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const double f = divide ? 1.0 / (lam[i] + shift) : lam[i];
  for (int c = 0; c < d; ++c) z[c * k + i] *= f;
}

// ‖A‖_F² of a column-major matrix (one block, fixed order)
__global__ void frob2_kernel(const double* __restrict__ a, int64_t count,
                             double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += a[i] * a[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
  out[0] = t;
}

void check_d(int32_t d, const char* what) {
  if (d < 1) throw Failure(FCPD_ERR_DIMENSION, std::string(what) + ": dimension mismatch");
}

// U·diag(f)·Uᵀ·V (+ X) in fp64: z = Uᵀ V, z_k *= f_k, out = U z (+ X).
void basis_sandwich(const CtxHandles& h, const double* u, int64_t m, int64_t k,
                    const double* lam, double shift, bool divide, const double* v, int32_t d,
                    const double* x, double* out) {
  cudaStream_t s = h.stream;
  FCPD_CUBLAS_L2(cublasSetStream(h.blas, s));
  Scratch<double> du(static_cast<size_t>(m) * k), dl(k), dv(static_cast<size_t>(m) * d),
      dz(static_cast<size_t>(k) * d), dout(static_cast<size_t>(m) * d);
  upload(du, u, static_cast<size_t>(m) * k, s);
  upload(dl, lam, k, s);
  upload(dv, v, static_cast<size_t>(m) * d, s);
  dgemm(h.blas, true, false, k, d, m, 1.0, du.p, m, dv.p, m, 0.0, dz.p, k);
  scale_rows_kernel<<<ceil_div(k, 256), 256, 0, s>>>(dz.p, k, d, dl.p, shift, divide ? 1 : 0);
  FCPD_LAUNCH_CHECK();
  double beta = 0.0;
  if (x) {
    upload(dout, x, static_cast<size_t>(m) * d, s);
    beta = 1.0;
  }
  dgemm(h.blas, false, false, m, d, k, 1.0, du.p, m, dz.p, k, beta, dout.p, m);
  FCPD_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * m * d, cudaMemcpyDeviceToHost, s));
  FCPD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace
}  // namespace fcpd

using namespace fcpd;

extern "C" {

int fcpd_estimated_targets(fcpd_ctx* ctx, const double* p, int64_t m, int64_t n,
                           const double* y, int64_t ny, int32_t d, double* out) {
  return ctx_guarded(ctx, [&] {
    if (n != ny) throw Failure(FCPD_ERR_PARAMETER, "estimated_targets: shape mismatch");
    check_d(d, "estimated_targets");
    if (m == 0 || d == 0) return;
    const CtxHandles h = ctx_handles(ctx);
    FCPD_CUBLAS_L2(cublasSetStream(h.blas, h.stream));
    Scratch<double> dp(static_cast<size_t>(m) * n), dy(static_cast<size_t>(n) * d),
        dout(static_cast<size_t>(m) * d);
    upload(dp, p, static_cast<size_t>(m) * n, h.stream);
    upload(dy, y, static_cast<size_t>(n) * d, h.stream);
    dgemm(h.blas, false, false, m, d, n, 1.0, dp.p, m, dy.p, n, 0.0, dout.p, m);
    FCPD_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * m * d, cudaMemcpyDeviceToHost,
                              h.stream));
    FCPD_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int fcpd_enforce_row_constraint(fcpd_ctx* ctx, double* p, int64_t m, int64_t n,
                                int32_t* degenerate) {
  return ctx_guarded(ctx, [&] {
    if (m == 0 || n == 0) return;
    const CtxHandles h = ctx_handles(ctx);
    Scratch<double> dp(static_cast<size_t>(m) * n), sums(m);
    Scratch<int32_t> deg(m);
    upload(dp, p, static_cast<size_t>(m) * n, h.stream);
    row_sums_kernel<<<ceil_div(m, 128), 128, 0, h.stream>>>(dp.p, m, n, sums.p);
    FCPD_LAUNCH_CHECK();
    row_constrain_kernel<<<ceil_div(m, 128), 128, 0, h.stream>>>(dp.p, m, n, sums.p, deg.p);
    FCPD_LAUNCH_CHECK();
    FCPD_CUDA(cudaMemcpyAsync(p, dp.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost,
                              h.stream));
    FCPD_CUDA(cudaMemcpyAsync(degenerate, deg.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost,
                              h.stream));
    FCPD_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int fcpd_update_sigma2(fcpd_ctx* ctx, const double* y, int64_t n, const double* p, int64_t m,
                       int64_t np, const double* xt, int64_t mx, int32_t d,
                       int32_t row_constrained, double* out) {
  return ctx_guarded(ctx, [&] {
    if (!row_constrained)
      throw Failure(FCPD_ERR_PARAMETER, "update_sigma2 requires a row-constrained P");
    if (np != n || mx != m) throw Failure(FCPD_ERR_PARAMETER, "update_sigma2: shape mismatch");
    check_d(d, "update_sigma2");
    if (m == 0) throw Failure(FCPD_ERR_PARAMETER, "update_sigma2: empty point set");
    const CtxHandles h = ctx_handles(ctx);
    FCPD_CUBLAS_L2(cublasSetStream(h.blas, h.stream));
    Scratch<double> dp(static_cast<size_t>(m) * n), dy(static_cast<size_t>(n) * d),
        dx(static_cast<size_t>(m) * d), pt1(n), yt(static_cast<size_t>(m) * d), tr(3);
    upload(dp, p, static_cast<size_t>(m) * n, h.stream);
    upload(dy, y, static_cast<size_t>(n) * d, h.stream);
    upload(dx, xt, static_cast<size_t>(m) * d, h.stream);
    col_sums_kernel<<<ceil_div(n, 8), 256, 0, h.stream>>>(dp.p, m, n, pt1.p);
    FCPD_LAUNCH_CHECK();
    dgemm(h.blas, false, false, m, d, n, 1.0, dp.p, m, dy.p, n, 0.0, yt.p, m);
    sigma2_traces_kernel<<<1, 1024, 0, h.stream>>>(dy.p, n, pt1.p, yt.p, dx.p, m, d, tr.p);
    FCPD_LAUNCH_CHECK();
    double t[3];
    FCPD_CUDA(cudaMemcpyAsync(t, tr.p, sizeof t, cudaMemcpyDeviceToHost, h.stream));
    FCPD_CUDA(cudaStreamSynchronize(h.stream));
    const double val =
        (t[0] - 2.0 * t[1] + t[2]) / (static_cast<double>(d) * static_cast<double>(m));
    if (val < -1e-8)
      throw Failure(FCPD_ERR_NUMERIC, "update_sigma2: negative variance " + std::to_string(val));
    *out = std::max(val, kSigma2Floor);
  });
}

int fcpd_eigendecompose(fcpd_ctx* ctx, const double* phi, int64_t m, int64_t rank, double* u,
                        double* lambda, double* lambda_raw) {
  return ctx_guarded(ctx, [&] {
    if (rank < 1 || rank > m)
      throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: rank out of [1, M]");
    if (m > 46000)
      throw Failure(FCPD_ERR_PARAMETER, "eigendecompose: M out of range for the dense path");
    const CtxHandles h = ctx_handles(ctx);
    Scratch<double> dphi(static_cast<size_t>(m) * m);
    upload(dphi, phi, static_cast<size_t>(m) * m, h.stream);
    Basis b;
    dense_eigensolve(h.solver, dphi.p, m, rank, b, u, h.stream);
    if (lambda) std::copy(b.lam_host.begin(), b.lam_host.end(), lambda);
    if (lambda_raw) std::copy(b.lam_raw_host.begin(), b.lam_raw_host.end(), lambda_raw);
    b.release();
  });
}

int fcpd_solve_fast_lowrank(fcpd_ctx* ctx, const double* u, const double* lambda, int64_t m,
                            int64_t k, double lambda_reg, double sigma2, const double* residual,
                            int64_t rm, int32_t d, double* w) {
  return ctx_guarded(ctx, [&] {
    if (rm != m)
      throw Failure(FCPD_ERR_PARAMETER, "solve_fast: residual rows must match basis points");
    if (k < 1 || k > m) throw Failure(FCPD_ERR_PARAMETER, "solve_fast: bad basis shape");
    const double shift = lambda_reg * sigma2;
    double mn = INFINITY;
    for (int64_t i = 0; i < k; ++i) mn = std::min(mn, lambda[i] + shift);
    if (!(mn > 0.0))
      throw Failure(FCPD_ERR_NUMERIC, "solve_fast: lambda_i + lambda*sigma2 not positive");
    if (d == 0) return;
    basis_sandwich(ctx_handles(ctx), u, m, k, lambda, shift, true, residual, d, nullptr, w);
  });
}

int fcpd_apply_transform(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d,
                         const double* phi, int64_t mphi, const double* w, int64_t mw,
                         int32_t dw, double* out) {
  return ctx_guarded(ctx, [&] {
    if (mphi != m || mw != m || dw != d)
      throw Failure(FCPD_ERR_PARAMETER, "apply_transform: shape mismatch");
    if (m == 0 || d == 0) return;
    const CtxHandles h = ctx_handles(ctx);
    FCPD_CUBLAS_L2(cublasSetStream(h.blas, h.stream));
    Scratch<double> dphi(static_cast<size_t>(m) * m), dw_(static_cast<size_t>(m) * d),
        dout(static_cast<size_t>(m) * d);
    upload(dphi, phi, static_cast<size_t>(m) * m, h.stream);
    upload(dw_, w, static_cast<size_t>(m) * d, h.stream);
    upload(dout, x, static_cast<size_t>(m) * d, h.stream);
    dgemm(h.blas, false, false, m, d, m, 1.0, dphi.p, m, dw_.p, m, 1.0, dout.p, m);
    FCPD_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * m * d, cudaMemcpyDeviceToHost,
                              h.stream));
    FCPD_CUDA(cudaStreamSynchronize(h.stream));
  });
}

int fcpd_apply_transform_lowrank(fcpd_ctx* ctx, const double* x, int64_t m, int32_t d,
                                 const double* u, int64_t mu, const double* lambda, int64_t k,
                                 const double* w, int64_t mw, int32_t dw, double* out) {
  return ctx_guarded(ctx, [&] {
    if (mu != m || mw != m || dw != d)
      throw Failure(FCPD_ERR_PARAMETER, "apply_transform_lowrank: shape mismatch");
    if (k < 1 || k > m) throw Failure(FCPD_ERR_PARAMETER, "apply_transform_lowrank: shape mismatch");
    if (d == 0) return;
    basis_sandwich(ctx_handles(ctx), u, m, k, lambda, 0.0, false, w, d, x, out);
  });
}

int fcpd_lowrank_reconstruction_error(fcpd_ctx* ctx, const double* phi, int64_t m,
                                      const double* u, int64_t mu, const double* lambda,
                                      int64_t k, double* out) {
  return ctx_guarded(ctx, [&] {
    if (mu != m)
      throw Failure(FCPD_ERR_PARAMETER, "lowrank_reconstruction_error: size mismatch");
    const CtxHandles h = ctx_handles(ctx);
    FCPD_CUBLAS_L2(cublasSetStream(h.blas, h.stream));
    Scratch<double> dphi(static_cast<size_t>(m) * m), du(static_cast<size_t>(m) * k),
        dul(static_cast<size_t>(m) * k), dl(k), nrm(1);
    upload(dphi, phi, static_cast<size_t>(m) * m, h.stream);
    upload(du, u, static_cast<size_t>(m) * k, h.stream);
    upload(dul, u, static_cast<size_t>(m) * k, h.stream);
    upload(dl, lambda, k, h.stream);
    // UΛ: columns of U scaled by λ (scale_rows on the transposed view = dgmm)
    FCPD_CUBLAS_L2(cublasDdgmm(h.blas, CUBLAS_SIDE_RIGHT, static_cast<int>(m), static_cast<int>(k),
                               du.p, static_cast<int>(m), dl.p, 1, dul.p, static_cast<int>(m)));
    // Φ − (UΛ)Uᵀ in place
    dgemm(h.blas, false, true, m, m, k, -1.0, dul.p, m, du.p, m, 1.0, dphi.p, m);
    frob2_kernel<<<1, 1024, 0, h.stream>>>(dphi.p, m * m, nrm.p);
    FCPD_LAUNCH_CHECK();
    double v = 0.0;
    FCPD_CUDA(cudaMemcpyAsync(&v, nrm.p, sizeof v, cudaMemcpyDeviceToHost, h.stream));
    FCPD_CUDA(cudaStreamSynchronize(h.stream));
    *out = std::sqrt(v);
  });
}

}  // extern "C"
