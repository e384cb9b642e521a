// bcl_fabric.cpp — see bcl_fabric.hpp.
#include "bcl_fabric.hpp"

#include <stdexcept>
#include <string>

#include "bcl_comm.hpp"  // CudaError
#include "bcl_device.cuh"

namespace bcl {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(e, what);
}

std::size_t size_class(std::size_t len) {
  std::size_t c = 256;
  while (c < len) c <<= 1;
  return c;
}

}  // namespace

DeviceFabric::DeviceFabric(const std::vector<int>& devices) : devices_(devices) {
  const int n = static_cast<int>(devices.size());
  if (n < 1) throw std::invalid_argument("rank count must be >= 1");
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  int saved = 0;
  cudaGetDevice(&saved);
  for (int d : devices) {
    if (d < 0 || d >= ndev) throw std::invalid_argument("device id out of range");
    if (!pools_.count(d)) pools_[d] = std::make_unique<Pool>();
  }
  for (const auto& a : pools_) {
    for (const auto& b : pools_) {
      if (a.first == b.first) continue;
      int can = 0;
      ck(cudaDeviceCanAccessPeer(&can, a.first, b.first), "cudaDeviceCanAccessPeer");
      if (!can) throw std::runtime_error("no peer access between devices");
      ck(cudaSetDevice(a.first), "cudaSetDevice");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b.first, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else {
        ck(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }
  for (int r = 0; r < n; ++r) {
    ck(cudaSetDevice(devices[static_cast<std::size_t>(r)]), "cudaSetDevice");
    cudaStream_t s{};
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    streams_.push_back(s);
  }
  for (int i = 0; i < n * n; ++i) pairs_.push_back(std::make_unique<Pair>());
  cudaSetDevice(saved);
}

DeviceFabric::~DeviceFabric() {
  for (std::size_t r = 0; r < streams_.size(); ++r) {
    cudaSetDevice(devices_[r]);
    cudaStreamSynchronize(streams_[r]);
    cudaStreamDestroy(streams_[r]);
  }
  for (auto& kv : pools_) {
    cudaSetDevice(kv.first);
    for (std::uint8_t* p : kv.second->all) cudaFree(p);
  }
}

void DeviceFabric::check_rank(int r) const {
  if (r < 0 || r >= n_ranks()) throw std::invalid_argument("rank out of range");
}

std::uint8_t* DeviceFabric::take(int device, std::size_t len) {
  Pool& p = *pools_.at(device);
  const std::size_t c = size_class(len);
  {
    std::lock_guard<std::mutex> lock(p.mu);
    auto& v = p.free[c];
    if (!v.empty()) {
      std::uint8_t* s = v.back();
      v.pop_back();
      return s;
    }
  }
  std::uint8_t* s = nullptr;
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaMalloc(&s, c), "cudaMalloc(fabric slab)");
  std::lock_guard<std::mutex> lock(p.mu);
  p.all.push_back(s);
  return s;
}

void DeviceFabric::give(int device, std::uint8_t* s, std::size_t len) {
  Pool& p = *pools_.at(device);
  std::lock_guard<std::mutex> lock(p.mu);
  p.free[size_class(len)].push_back(s);
}

void DeviceFabric::send(int src, int dst, std::uint32_t chunk, const std::uint8_t* data, std::size_t len) {
  check_rank(src);
  check_rank(dst);
  const int dev = devices_[static_cast<std::size_t>(src)];
  std::uint8_t* slab = take(dev, len);
  if (len) {
    ck(cudaSetDevice(dev), "cudaSetDevice");
    cudaStream_t s = streams_[static_cast<std::size_t>(src)];
    ck(cudaMemcpyAsync(slab, data, len, cudaMemcpyHostToDevice, s), "H2D (fabric send)");
    ck(cudaStreamSynchronize(s), "synchronize (fabric send)");  // eager: the span may be reused on return
  }
  Pair& p = pair(src, dst);
  {
    std::lock_guard<std::mutex> lock(p.mu);
    p.q.push_back(Msg{chunk, slab, len});
  }
  p.cv.notify_one();
}

std::size_t DeviceFabric::recv_size(int dst, int src, std::uint32_t chunk) {
  check_rank(src);
  check_rank(dst);
  Pair& p = pair(src, dst);
  std::unique_lock<std::mutex> lock(p.mu);
  p.cv.wait(lock, [&] { return !p.q.empty(); });
  const Msg& m = p.q.front();
  if (m.chunk != chunk) {  // transport_inproc.cpp:98-103
    throw std::runtime_error("out-of-order delivery from rank " + std::to_string(src) + " to rank " +
                             std::to_string(dst) + ": expected chunk " + std::to_string(chunk) + ", got " +
                             std::to_string(m.chunk));
  }
  return m.len;
}

void DeviceFabric::recv(int dst, int src, std::uint32_t chunk, std::uint8_t* out, std::size_t len) {
  const std::size_t have = recv_size(dst, src, chunk);
  if (have != len) throw std::invalid_argument("recv buffer length does not match the message");
  Pair& p = pair(src, dst);
  Msg m;
  {
    std::lock_guard<std::mutex> lock(p.mu);
    m = p.q.front();
    p.q.pop_front();
  }
  const int sdev = devices_[static_cast<std::size_t>(src)];
  const int ddev = devices_[static_cast<std::size_t>(dst)];
  if (len) {
    std::uint8_t* slab = take(ddev, len);
    ck(cudaSetDevice(ddev), "cudaSetDevice");
    cudaStream_t s = streams_[static_cast<std::size_t>(dst)];
    ck(static_cast<cudaError_t>(launch_peer_copy(slab, m.dev, len, s)), "launch(peer copy)");  // NVLink pull
    ck(cudaMemcpyAsync(out, slab, len, cudaMemcpyDeviceToHost, s), "D2H (fabric recv)");
    ck(cudaStreamSynchronize(s), "synchronize (fabric recv)");
    give(ddev, slab, len);
  }
  give(sdev, m.dev, m.len);
  std::lock_guard<std::mutex> lock(p.mu);
  p.messages += 1;
  p.bytes += len;
}

void DeviceFabric::stats(int src, int dst, std::uint64_t* messages, std::uint64_t* bytes) const {
  check_rank(src);
  check_rank(dst);
  const Pair& p = pair(src, dst);
  std::lock_guard<std::mutex> lock(p.mu);
  if (messages) *messages = p.messages;
  if (bytes) *bytes = p.bytes;
}

}  // namespace bcl
