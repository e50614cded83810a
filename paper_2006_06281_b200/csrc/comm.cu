// comm.cu — the loopback collectives (see comm.cuh): fixed-order device
// reductions over the G virtual ranks' buffers of one device.
#include <algorithm>

#include "comm.cuh"

namespace fcpd {
namespace {

template <typename T>
struct Ptrs {
  T* p[kMaxLoopRanks];
};

template <typename T, typename V>
Ptrs<T> pack(const std::vector<V*>& v) {
  if (v.size() > static_cast<size_t>(kMaxLoopRanks))
    throw Failure(FCPD_ERR_PARAMETER, "loopback group: at most 8 ranks");
  Ptrs<T> r{};
  for (size_t i = 0; i < v.size(); ++i) r.p[i] = const_cast<T*>(v[i]);
  return r;
}

__global__ void loop_reduce_scatter_kernel(Ptrs<double> send, Ptrs<double> recv, int world,
                                           int64_t count) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= world * count) return;
  const int r = static_cast<int>(j / count);
  const int64_t i = j - r * count;
  double s = 0.0;
  for (int q = 0; q < world; ++q) s += send.p[q][r * count + i];
  recv.p[r][i] = s;
}

template <typename T, bool kMax>
__global__ void loop_all_reduce_kernel(Ptrs<T> buf, int world, int64_t count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  T s = buf.p[0][i];
  for (int q = 1; q < world; ++q) s = kMax ? max(s, buf.p[q][i]) : s + buf.p[q][i];
  for (int q = 0; q < world; ++q) buf.p[q][i] = s;
}

// in place allowed: send[q] = recv[q] + q·words (rank q's own chunk is
// only read; every write goes to another rank's chunk q or is a self-copy)
__global__ void loop_all_gather_kernel(Ptrs<uint32_t> send, Ptrs<uint32_t> recv, int world,
                                       int64_t words) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= static_cast<int64_t>(world) * words) return;
  const int q = static_cast<int>(j / words);
  const int64_t i = j - q * words;
  const uint32_t v = send.p[q][i];
  for (int r = 0; r < world; ++r) recv.p[r][q * words + i] = v;
}

}  // namespace

void LoopComm::reduce_scatter_sum(const std::vector<const double*>& send,
                                  const std::vector<double*>& recv, size_t count, cudaStream_t s) {
  const int64_t tot = static_cast<int64_t>(world) * static_cast<int64_t>(count);
  loop_reduce_scatter_kernel<<<ceil_div(std::max<int64_t>(tot, 1), 256), 256, 0, s>>>(
      pack<double>(send), pack<double>(recv), world, static_cast<int64_t>(count));
  FCPD_LAUNCH_CHECK();
}

void LoopComm::all_reduce_sum(const std::vector<double*>& buf, size_t count, cudaStream_t s) {
  loop_all_reduce_kernel<double, false>
      <<<ceil_div(std::max<int64_t>(static_cast<int64_t>(count), 1), 256), 256, 0, s>>>(
          pack<double>(buf), world, static_cast<int64_t>(count));
  FCPD_LAUNCH_CHECK();
}

void LoopComm::all_reduce_max(const std::vector<float*>& buf, size_t count, cudaStream_t s) {
  loop_all_reduce_kernel<float, true>
      <<<ceil_div(std::max<int64_t>(static_cast<int64_t>(count), 1), 256), 256, 0, s>>>(
          pack<float>(buf), world, static_cast<int64_t>(count));
  FCPD_LAUNCH_CHECK();
}

void LoopComm::all_gather(const std::vector<const uint32_t*>& send,
                          const std::vector<uint32_t*>& recv, size_t words, cudaStream_t s) {
  const int64_t tot = static_cast<int64_t>(world) * static_cast<int64_t>(words);
  loop_all_gather_kernel<<<ceil_div(std::max<int64_t>(tot, 1), 256), 256, 0, s>>>(
      pack<uint32_t>(send), pack<uint32_t>(recv), world, static_cast<int64_t>(words));
  FCPD_LAUNCH_CHECK();
}

void LoopComm::host_all_reduce(std::vector<std::vector<double>>& vals, bool max, cudaStream_t) {
  if (vals.empty()) return;
  std::vector<double> acc = vals[0];
  for (size_t q = 1; q < vals.size(); ++q)
    for (size_t i = 0; i < acc.size(); ++i)
      acc[i] = max ? std::max(acc[i], vals[q][i]) : acc[i] + vals[q][i];
  for (auto& v : vals) v = acc;
}

}  // namespace fcpd
