// setup.cuh — spectral basis setup interface (see setup.cu).
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <stdint.h>

#include <vector>

#include "comm.cuh"

namespace fcpd {

// Device-resident spectral basis, packed for the streaming M-step.
struct Basis {
  int64_t m = 0, k = 0, kpad = 0, mpad = 0;
  float* q = nullptr;    // M×kpad row-major fp32
  float* qt = nullptr;   // K×mpad row-major fp32
  double* lam = nullptr; // [0,k): clamped λ ; [k,2k): transform numerator
  double* u64 = nullptr; // M×K column-major fp64 eigenvectors (descending), for export
  bool full_rank = false;
  std::vector<double> lam_raw_host, lam_host;
  std::vector<int64_t> perm;  // basis row k ↔ original model point perm[k] (empty: identity)
  // cache key
  uint64_t key_hash = 0;
  double key_beta = 0.0;
  int key_variant = -1;
  double t_gram = 0.0, t_eig = 0.0;
  void release();
};

void build_gram_device(const double* x_dev, int64_t m, int d, double beta, double* phi,
                       int64_t ld, cudaStream_t stream);
// In-place eigensolve of phi (M×M col-major, overwritten with eigenvectors);
// packs the top `rank` into b.  Optionally returns U (M×rank) to the host.
void dense_eigensolve(cusolverDnHandle_t h, double* phi, int64_t m, int64_t rank, Basis& b,
                      double* u_out_host, cudaStream_t stream);
void basis_from_host(Basis& b, const double* u_host, const double* lam_host, int64_t m,
                     int64_t k, cudaStream_t stream);
void clamp_lambda(Basis& b);
void upload_lambda(Basis& b, bool full_rank, cudaStream_t stream);
// Pack device eigenvectors u (M×k col-major fp64) + λ_raw (descending) into b.
void pack_basis_from(Basis& b, const double* u_dev, int64_t m, int64_t k, int reverse,
                     const std::vector<double>& lam_raw, cudaStream_t stream);

// topk.cu — on-the-fly Gram products and the randomized block eigensolver.
// A rank group's products are row-sharded: `ranks` are the
// global ranks this process drives (one for NCCL, all for a loopback group).
struct GramShards {
  Comm* comm = nullptr;
  std::vector<int> ranks;
  int64_t block_rows(int64_t m) const {
    return ceil_div(ceil_div(m, static_cast<int64_t>(comm->world)), int64_t(64)) * 64;
  }
};
// Φ·V tile geometry: col_blocks blocks of 128 columns, Vᵀ padded to
// m_pad × ldv
struct GramPlan {
  int64_t col_blocks = 1, ldv = 0, m_pad = 0;
};
GramPlan make_gram_plan(int64_t m, int64_t b);
// Y = Φ V (V, Y: M×b column-major); vt: m_pad × ldv scratch
void gram_matmul(const double* x, int64_t m, int d, double beta, const double* v, int64_t b,
                 double* y, double* vt, const GramPlan& g, cudaStream_t stream);
void topk_eigensolve(cusolverDnHandle_t solver, cublasHandle_t blas, const double* x_dev,
                     int64_t m, int d, double beta, int64_t rank, int iterations, bool adaptive,
                     uint64_t seed, Basis& b_out, cudaStream_t stream,
                     double* u_host_out = nullptr, int* products_out = nullptr,
                     const GramShards* shards = nullptr,
                     const std::vector<Basis*>* also_out = nullptr);
void gram_matmul_sharded(const double* x, int64_t m, int d, double beta, const double* v,
                         int64_t b, double* y, double* vt, const GramPlan& g, double* wpm,
                         const GramShards& sh, cudaStream_t stream);

}  // namespace fcpd
