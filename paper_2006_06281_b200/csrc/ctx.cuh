// ctx.cuh — what the C-ABI translation units outside engine.cu need from a
// context (engine.cu owns struct fcpd_ctx): its device, stream and library
// handles, and the error guard that maps exceptions to FCPD_ERR_* codes.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <functional>

#include "common.cuh"

namespace fcpd {

struct CtxHandles {
  int device;
  cudaStream_t stream;
  cublasHandle_t blas;
  cusolverDnHandle_t solver;
};

CtxHandles ctx_handles(fcpd_ctx* ctx);
// Run f on the context's device; exceptions → FCPD_ERR_* + fcpd_last_error.
int ctx_guarded(fcpd_ctx* ctx, const std::function<void()>& f);

}  // namespace fcpd
