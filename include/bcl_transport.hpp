// bcl_transport.hpp — header-only C++ adapter that plugs the GPU-backed
// device fabric (bcl_fabric_*, include/bcl.h) into the reference's transport
// interface (proj/include/bcastlab/runtime.hpp:20-39):
//
//   class Transport       { virtual void send(int dst, uint32_t chunk, span<const uint8_t>);
//                           virtual vector<uint8_t> recv(int src, uint32_t chunk); };
//   class TransportFabric { virtual int n_ranks() const; virtual Transport& endpoint(int rank); };
//
// The reference's base classes are template parameters, so a reference build
// instantiates
//
//   bcl_b200::DeviceFabricT<bcastlab::Transport, bcastlab::TransportFabric> fabric({0, 1, 2, 3});
//   bcastlab::run_bcast(request, fabric);          // runtime.hpp:140-143, unchanged
//
// and its execute_rank loop (runtime.cpp:32-64) moves every chunk through
// the GPUs (H2D at the sender, a P2P copy kernel into the receiver's GPU,
// D2H). Errors come back as the reference's exception classes:
// std::runtime_error for transport/data errors (out-of-order chunk ids,
// transport_inproc.cpp:98-103), std::invalid_argument for contract errors.
// Without template arguments the classes stand alone (no virtual base).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "bcl.h"

namespace bcl_b200 {

inline void fabric_check(bcl_status_t s) {
  if (s == BCL_OK) return;
  const std::string msg = bcl_last_error();
  if (s == BCL_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct NoBase {};
struct NoFabricBase {};

template <class TransportBase = NoBase, class FabricBase = NoFabricBase>
class DeviceFabricT : public FabricBase {
 public:
  class Endpoint : public TransportBase {
   public:
    Endpoint(bcl_fabric_t f, int rank) : f_(f), rank_(rank) {}
    void send(int dst_rank, std::uint32_t chunk_id, std::span<const std::uint8_t> data) {
      fabric_check(bcl_fabric_send(f_, rank_, dst_rank, chunk_id, data.data(), data.size()));
    }
    std::vector<std::uint8_t> recv(int src_rank, std::uint32_t chunk_id) {
      std::size_t len = 0;
      fabric_check(bcl_fabric_recv_size(f_, rank_, src_rank, chunk_id, &len));
      std::vector<std::uint8_t> out(len);
      fabric_check(bcl_fabric_recv(f_, rank_, src_rank, chunk_id, out.data(), len));
      return out;
    }

   private:
    bcl_fabric_t f_;
    int rank_;
  };

  explicit DeviceFabricT(const std::vector<int>& devices) {
    fabric_check(bcl_fabric_create(static_cast<int>(devices.size()), devices.data(), &f_));
    for (int r = 0; r < static_cast<int>(devices.size()); ++r) ends_.push_back(std::make_unique<Endpoint>(f_, r));
  }
  ~DeviceFabricT() {
    ends_.clear();
    bcl_fabric_destroy(f_);
  }
  DeviceFabricT(const DeviceFabricT&) = delete;
  DeviceFabricT& operator=(const DeviceFabricT&) = delete;

  int n_ranks() const { return static_cast<int>(ends_.size()); }
  Endpoint& endpoint(int rank) {
    if (rank < 0 || rank >= n_ranks()) throw std::invalid_argument("rank out of range");
    return *ends_[static_cast<std::size_t>(rank)];
  }
  // Messages and payload bytes delivered src -> dst so far.
  std::pair<std::uint64_t, std::uint64_t> delivered(int src, int dst) const {
    std::uint64_t m = 0, b = 0;
    fabric_check(bcl_fabric_stats(f_, src, dst, &m, &b));
    return {m, b};
  }

 private:
  bcl_fabric_t f_{};
  std::vector<std::unique_ptr<Endpoint>> ends_;
};

using DeviceFabric = DeviceFabricT<>;

}  // namespace bcl_b200
