// TEST INFRASTRUCTURE — not product code.
//
// The reference's own runtime (run_bcast / execute_rank, compiled unmodified
// from /root/reference/proj/src) driven over the product's GPU-backed device
// fabric (libbcl.so, include/bcl_transport.hpp) instead of its CPU
// transports: the runtime-level cases of proj/tests/test_runtime.cpp
// (:99-272) restated as checks, every byte of every chunk crossing the GPUs.
//
//   ref_device_fabric DEVICES      DEVICES = "0" (every rank on GPU 0) or
//                                  "0,1,..." (rank r on DEVICES[r % count])
// Prints one PASS/FAIL line per case; exit code = number of failures.
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "bcastlab/runtime.hpp"
#include "bcastlab/schedules.hpp"
#include "bcl_transport.hpp"

using namespace bcastlab;
using GpuFabric = bcl_b200::DeviceFabricT<Transport, TransportFabric>;

namespace {

std::vector<int> g_devices;

std::vector<int> devices_for(int n) {
  std::vector<int> d;
  for (int r = 0; r < n; ++r) d.push_back(g_devices[static_cast<std::size_t>(r) % g_devices.size()]);
  return d;
}

std::vector<std::uint8_t> bytes_of(std::size_t size, std::uint64_t seed) {
  std::vector<std::uint8_t> v(size);
  std::mt19937_64 rng(seed ^ 0x5bd1e995ull);
  for (auto& b : v) b = static_cast<std::uint8_t>(rng() >> 17);
  return v;
}

struct Buffers {
  std::vector<std::vector<std::uint8_t>> data;
  std::vector<std::span<std::uint8_t>> views;
  Buffers(int n, const std::vector<std::uint8_t>& payload, int root)
      : data(static_cast<std::size_t>(n), std::vector<std::uint8_t>(payload.size(), 0xEE)) {
    data[static_cast<std::size_t>(root)] = payload;
    for (auto& d : data) views.emplace_back(d);
  }
  bool all(const std::vector<std::uint8_t>& payload) const {
    for (const auto& d : data) {
      if (d != payload) return false;
    }
    return true;
  }
};

// Wraps any fabric and logs each send as (src, dst, chunk) and each rank's
// receive order -- the shape of the reference test's recorder, written here
// against the same public interface.
class Logged final : public TransportFabric {
 public:
  explicit Logged(TransportFabric& inner) : inner_(inner) {
    for (int r = 0; r < inner.n_ranks(); ++r) ends_.emplace_back(new End(*this, r));
  }
  int n_ranks() const override { return inner_.n_ranks(); }
  Transport& endpoint(int rank) override { return *ends_.at(static_cast<std::size_t>(rank)); }
  std::multiset<std::tuple<int, int, std::uint32_t>> sent;
  std::map<int, std::vector<std::uint32_t>> got;

 private:
  struct End final : Transport {
    End(Logged& o, int r) : owner(o), rank(r) {}
    void send(int dst, std::uint32_t chunk, std::span<const std::uint8_t> d) override {
      {
        std::lock_guard<std::mutex> g(owner.mu_);
        owner.sent.insert({rank, dst, chunk});
      }
      owner.inner_.endpoint(rank).send(dst, chunk, d);
    }
    std::vector<std::uint8_t> recv(int src, std::uint32_t chunk) override {
      auto v = owner.inner_.endpoint(rank).recv(src, chunk);
      std::lock_guard<std::mutex> g(owner.mu_);
      owner.got[rank].push_back(chunk);
      return v;
    }
    Logged& owner;
    int rank;
  };
  TransportFabric& inner_;
  std::vector<std::unique_ptr<End>> ends_;
  std::mutex mu_;
};

std::multiset<std::tuple<int, int, std::uint32_t>> schedule_sends(const Schedule& s) {
  std::multiset<std::tuple<int, int, std::uint32_t>> out;
  for (int r = 0; r < s.n_ranks; ++r) {
    for (const Event& e : s.per_rank_ops[static_cast<std::size_t>(r)]) {
      if (e.kind == Event::Kind::Send) out.insert({r, e.peer, e.chunk});
    }
  }
  return out;
}

int failures = 0;

void run_case(const char* name, const std::function<bool()>& body) {
  bool ok = false;
  std::string why;
  try {
    ok = body();
  } catch (const std::exception& e) {
    why = e.what();
  }
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name, why.empty() ? "" : ": ", why.c_str());
  if (!ok) ++failures;
}

}  // namespace

int main(int argc, char** argv) {
  std::stringstream ss(argc > 1 ? argv[1] : "0");
  for (std::string t; std::getline(ss, t, ',');) g_devices.push_back(std::atoi(t.c_str()));

  run_case("pipelined chain n=4 M=64 C=16 fills every buffer (test_runtime.cpp:99-108)", [] {
    const auto p = bytes_of(64, 42);
    Buffers b(4, p, 0);
    GpuFabric f(devices_for(4));
    const auto r = run_bcast(BcastRequest{4, 0, b.views, AlgorithmConfig{Algorithm::ChainPipelined, 0, 16}}, f);
    return b.all(p) && r.wall_s >= 0.0;
  });
  run_case("single rank leaves the buffer untouched (:110-119)", [] {
    const auto p = bytes_of(128, 1);
    Buffers b(1, p, 0);
    GpuFabric f(devices_for(1));
    run_bcast(BcastRequest{1, 0, b.views, AlgorithmConfig{Algorithm::Chain}}, f);
    return b.data[0] == p;
  });
  run_case("scatter-ring-allgather n=8: wire transfers == schedule sends, scatter first (:121-161)", [] {
    const int n = 8;
    const auto p = bytes_of(8192, 7);
    Buffers b(n, p, 0);
    GpuFabric f(devices_for(n));
    Logged log(f);
    run_bcast(BcastRequest{n, 0, b.views, AlgorithmConfig{Algorithm::ScatterRingAllgather}}, log);
    const Schedule s = schedule_scatter_ring_allgather(n, 0, 8192);
    if (!b.all(p) || log.sent != schedule_sends(s)) return false;
    for (int r = 1; r < n; ++r) {  // a rank's first receive is its own partition
      if (log.got[r].empty() || log.got[r][0] != static_cast<std::uint32_t>(r)) return false;
    }
    // the fabric's own delivery counters agree with the schedule per pair
    for (int src = 0; src < n; ++src) {
      for (int dst = 0; dst < n; ++dst) {
        std::uint64_t want = 0;
        for (const auto& t : schedule_sends(s)) want += std::get<0>(t) == src && std::get<1>(t) == dst;
        if (f.delivered(src, dst).first != want) return false;
      }
    }
    return true;
  });
  run_case("zero-byte knomial still runs every event (:163-171)", [] {
    const int n = 6;
    Buffers b(n, {}, 0);
    GpuFabric f(devices_for(n));
    Logged log(f);
    run_bcast(BcastRequest{n, 0, b.views, AlgorithmConfig{Algorithm::Knomial, 2, 0}}, log);
    return log.sent.size() == static_cast<std::size_t>(n - 1);
  });
  run_case("device fabric == inproc fabric on every algorithm, 18 random trials (:173-203)", [] {
    std::mt19937_64 rng(2026);
    for (int trial = 0; trial < 18; ++trial) {
      const auto algo = static_cast<Algorithm>(trial % kAlgorithmCount);
      const int n = (algo == Algorithm::ChainPipelined ? 2 : 1) + static_cast<int>(rng() % 9);
      const int root = static_cast<int>(rng() % static_cast<std::uint64_t>(n));
      const std::uint64_t m = rng() % 40000;
      AlgorithmConfig cfg{algo, 0, 0};
      if (algorithm_uses_radix(algo)) cfg.radix_k = 2 + static_cast<int>(rng() % 3);
      if (algorithm_uses_chunk(algo)) cfg.chunk_bytes = 1 + rng() % (m + 1);
      const auto p = bytes_of(m, rng());
      Buffers a(n, p, root), g(n, p, root);
      auto cpu = make_inproc_fabric(n);
      run_bcast(BcastRequest{n, root, a.views, cfg}, *cpu);
      GpuFabric f(devices_for(n));
      run_bcast(BcastRequest{n, root, g.views, cfg}, f);
      if (!g.all(p) || a.data != g.data) return false;
    }
    return true;
  });
  run_case("sixteen ranks, 1 MiB, C=64 KiB (:224-236)", [] {
    const auto p = bytes_of(1 << 20, 99);
    Buffers b(16, p, 0);
    GpuFabric f(devices_for(16));
    run_bcast(BcastRequest{16, 0, b.views, AlgorithmConfig{Algorithm::ChainPipelined, 0, 65536}}, f);
    return b.all(p);
  });
  run_case("mismatched buffer lengths are a contract error (:238-244)", [] {
    std::vector<std::uint8_t> x(10), y(12);
    GpuFabric f(devices_for(2));
    try {
      run_bcast(BcastRequest{2, 0, {std::span(x), std::span(y)}, AlgorithmConfig{Algorithm::Chain}}, f);
    } catch (const std::invalid_argument&) {
      return true;
    }
    return false;
  });
  run_case("staged knomial from root 5 (:246-254)", [] {
    const auto p = bytes_of(4096, 3);
    Buffers b(8, p, 5);
    GpuFabric f(devices_for(8));
    run_bcast(BcastRequest{8, 5, b.views, AlgorithmConfig{Algorithm::KnomialStaged, 2, 0}}, f);
    return b.all(p);
  });
  run_case("ordered delivery is enforced per pair (:266-272)", [] {
    GpuFabric f(devices_for(2));
    f.endpoint(0).send(1, 0, {});
    f.endpoint(0).send(1, 1, {});
    try {
      f.endpoint(1).recv(0, 1);
    } catch (const std::runtime_error&) {
      return true;
    }
    return false;
  });
  std::printf("%d failure(s)\n", failures);
  return failures;
}
