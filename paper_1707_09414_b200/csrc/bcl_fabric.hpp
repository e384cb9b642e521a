// bcl_fabric: a GPU-backed stand-in for the reference's message fabric
// (Transport / TransportFabric, proj/include/bcastlab/runtime.hpp:20-39), so
// the reference's own runtime-level callers -- execute_rank, run_bcast and
// the tests built on them -- run with their bytes moving between GPUs.
//
// Same contract as the reference transports (runtime.hpp:20-30,
// transport_inproc.cpp:79-105): delivery is ordered and reliable per
// (src, dst) pair, send is eager (the sender may reuse its span once send
// returns), recv blocks until the matching send arrives and rejects a chunk
// id out of order. The payload path is device-side: send stages the span in
// the sender's GPU (H2D), recv pulls it into the receiver's GPU with the
// library's copy kernel (NVLink P2P loads across GPUs) and hands it back to
// the host (D2H). Ranks are threads of one process, one rank per entry of
// `devices` (several ranks may share a GPU). This is the compatibility path
// for reference-level callers; the hot path is bcl_bcast.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace bcl {

class DeviceFabric {
 public:
  explicit DeviceFabric(const std::vector<int>& devices);
  ~DeviceFabric();
  DeviceFabric(const DeviceFabric&) = delete;
  DeviceFabric& operator=(const DeviceFabric&) = delete;

  int n_ranks() const { return static_cast<int>(devices_.size()); }
  // Called from rank `src`'s thread only (one thread per endpoint).
  void send(int src, int dst, std::uint32_t chunk, const std::uint8_t* data, std::size_t len);
  // Called from rank `dst`'s thread only: waits for the next message from
  // `src`, checks its chunk id and returns its length (the message stays
  // queued); recv then moves it into `out` (len bytes) and dequeues it.
  std::size_t recv_size(int dst, int src, std::uint32_t chunk);
  void recv(int dst, int src, std::uint32_t chunk, std::uint8_t* out, std::size_t len);
  // Messages / payload bytes delivered so far from src to dst.
  void stats(int src, int dst, std::uint64_t* messages, std::uint64_t* bytes) const;

 private:
  struct Msg {
    std::uint32_t chunk;
    std::uint8_t* dev;  // on the sender's GPU
    std::size_t len;
  };
  struct Pair {
    mutable std::mutex mu;
    std::condition_variable cv;
    std::deque<Msg> q;
    std::uint64_t messages{0};
    std::uint64_t bytes{0};
  };
  struct Pool {  // per-GPU slab cache: power-of-two size classes
    std::mutex mu;
    std::map<std::size_t, std::vector<std::uint8_t*>> free;
    std::vector<std::uint8_t*> all;
  };
  Pair& pair(int src, int dst) const { return *pairs_[static_cast<std::size_t>(src * n_ranks() + dst)]; }
  std::uint8_t* take(int device, std::size_t len);
  void give(int device, std::uint8_t* p, std::size_t len);
  void check_rank(int r) const;

  std::vector<int> devices_;
  std::vector<cudaStream_t> streams_;  // one per rank
  std::vector<std::unique_ptr<Pair>> pairs_;
  std::map<int, std::unique_ptr<Pool>> pools_;
};

}  // namespace bcl
