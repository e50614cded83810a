// comm.cuh — collectives of the scene-sharded EM.
//
// Every call covers the ranks this process drives, each with its own device
// buffer (slot i of the pointer vectors = local rank i) and is enqueued on
// one stream (so it is captured into the iteration's CUDA graph):
//  * NcclComm   — one rank per GPU (one per process), NCCL over NVLink;
//  * LoopComm   — G virtual ranks on ONE device in one process: the same
//    sharded data plane with the collectives as device kernels reading every
//    rank's buffer (fixed order).  It exercises the multi-rank code path
//    (shard offsets, padding, the conditional fallback) on a single GPU;
//    no rank ever waits on another (the ranks' work is enqueued in phases
//    between collectives on the one stream).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace fcpd {

constexpr int kMaxLoopRanks = 8;

struct Comm {
  int world = 1;
  virtual ~Comm() = default;
  // recv[r][i] = Σ_q send[q][r·count + i]  (count = per-rank chunk)
  virtual void reduce_scatter_sum(const std::vector<const double*>& send,
                                  const std::vector<double*>& recv, size_t count,
                                  cudaStream_t s) = 0;
  // buf[r][i] = Σ_q buf[q][i], in place
  virtual void all_reduce_sum(const std::vector<double*>& buf, size_t count, cudaStream_t s) = 0;
  // buf[r][i] = max_q buf[q][i], in place
  virtual void all_reduce_max(const std::vector<float*>& buf, size_t count, cudaStream_t s) = 0;
  // recv[r][q·words + i] = send[q][i] (32-bit words; send may alias recv)
  virtual void all_gather(const std::vector<const uint32_t*>& send,
                          const std::vector<uint32_t*>& recv, size_t words, cudaStream_t s) = 0;
  // host values, reduced over the group (sum or max), in place per rank
  virtual void host_all_reduce(std::vector<std::vector<double>>& vals, bool max,
                               cudaStream_t s) = 0;
  // may collectives be captured into a conditional-node body?
  virtual bool conditional_ok() const = 0;
};

struct LoopComm : Comm {
  explicit LoopComm(int w) { world = w; }
  void reduce_scatter_sum(const std::vector<const double*>& send, const std::vector<double*>& recv,
                          size_t count, cudaStream_t s) override;
  void all_reduce_sum(const std::vector<double*>& buf, size_t count, cudaStream_t s) override;
  void all_reduce_max(const std::vector<float*>& buf, size_t count, cudaStream_t s) override;
  void all_gather(const std::vector<const uint32_t*>& send, const std::vector<uint32_t*>& recv,
                  size_t words, cudaStream_t s) override;
  void host_all_reduce(std::vector<std::vector<double>>& vals, bool max, cudaStream_t s) override;
  bool conditional_ok() const override { return true; }
};

}  // namespace fcpd
