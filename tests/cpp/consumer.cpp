// A reference-style C++ consumer of libbcl through include/bcl.hpp only
// (no CUDA headers): what a bcastlab maintainer's code looks like when it
// switches to the B200 path. `consumer` runs the host-side checks;
// `consumer gpu` also broadcasts host buffers over 4 ranks on GPU 0.
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "bcl.hpp"

namespace b = bcl_b200;

#define EXPECT(cond)                                              \
  do {                                                            \
    if (!(cond)) {                                                \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                   \
    }                                                             \
  } while (0)

int main(int argc, char** argv) {
  // proj/tests/test_core.cpp:14-20
  const auto ch = b::make_chunks(10, 4);
  EXPECT(ch.size() == 3 && ch[2].offset_bytes == 8 && ch[2].length_bytes == 2);
  // proj/tests/test_schedules.cpp:161-167
  b::Schedule s(b::chain_pipelined(4), 3, 0, 8);
  EXPECT(s.text() == "0 send 1 0\n0 send 1 1\n1 recv 0 0\n1 send 2 0\n1 recv 0 1\n1 send 2 1\n2 recv 1 0\n2 recv 1 1\n");
  s.validate();
  bool threw = false;
  try {
    b::Schedule bad(b::chain_pipelined(4), 1, 0, 8);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  // README.md:101-105 table reproduced by the analytical tuner
  std::vector<std::uint64_t> sizes, chunks;
  for (std::uint64_t x = 1024; x <= 4194304; x *= 2) sizes.push_back(x);
  for (std::uint64_t x = 8192; x <= 4194304; x *= 2) chunks.push_back(x);
  const auto t = b::Table::tune({4}, sizes, {b::knomial(2), b::chain_pipelined(0)}, chunks);
  EXPECT(t.text().find("4,1024,23170,knomial,2,0,1.1741999999999999e-05\n") != std::string::npos);
  EXPECT(t.select(4, 1000000).algorithm == BCL_CHAIN_PIPELINED);
  threw = false;
  try {
    (void)t.select(3, 10);
  } catch (const std::out_of_range&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    (void)b::Table::load_text("n,msg_min_bytes,msg_max_bytes,algorithm,radix,chunk_bytes,predicted_cost_s\n4,1,2,ring,0,0,1\n");
  } catch (const b::TableParseError& e) {
    threw = e.line() == 2;
  }
  EXPECT(threw);
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
    const int n = 4;
    const std::size_t m = (3u << 20) + 5;
    std::vector<std::vector<unsigned char>> host(n, std::vector<unsigned char>(m, 0));
    std::mt19937_64 rng(5);
    for (auto& x : host[2]) x = static_cast<unsigned char>(rng());
    std::vector<void*> ptrs;
    for (auto& h : host) ptrs.push_back(h.data());
    b::LocalGroup g({0, 0, 0, 0}, 10.0);
    const b::Config cfg = b::chain_pipelined(65536);
    const double w = g.run_bcast_host(2, ptrs, m, &cfg);
    EXPECT(w > 0);
    for (int r = 0; r < n; ++r) EXPECT(host[r] == host[2]);
    // tuned path (config = nullptr -> select on the builtin measured table)
    for (int r = 0; r < n; ++r) if (r != 1) std::fill(host[r].begin(), host[r].end(), 0);
    (void)g.run_bcast_host(1, ptrs, m);
    for (int r = 0; r < n; ++r) EXPECT(host[r] == host[1]);
    // every single-GPU transport of the chain: fused (auto), lane executor, LL lines
    for (int proto : {0, 1, 3}) {
      g.set_protocol(proto);
      for (int r = 0; r < n; ++r) if (r != 3) std::fill(host[r].begin(), host[r].end(), 0);
      (void)g.run_bcast_host(3, ptrs, m, &cfg);
      for (int r = 0; r < n; ++r) EXPECT(host[r] == host[3]);
    }
    g.set_protocol(0);
    // one GPU: no NVLS team, and forcing the protocol fails loudly (invalid_argument)
    std::string why;
    EXPECT(!g.nvls(&why) && !why.empty());
    g.set_protocol(5);
    bool threw = false;
    try {
      (void)g.run_bcast_host(0, ptrs, m, &cfg);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    EXPECT(threw);
    g.set_protocol(0);
    std::printf("gpu ok (%.1f us wall)\n", w * 1e6);
  }
  std::printf("consumer ok\n");
  return 0;
}
