// TEST INFRASTRUCTURE — not product code.
//
// A small command-line driver over the *unmodified* reference library
// (bcastlab, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/). It exposes the reference's public API so that
//   * tests/golden/make_golden.py can pin our C restatement (oracle/bcast_oracle.c)
//     and our product library against the reference's own outputs, and
//   * bench.py can time the reference CPU broadcast (the `cpu_baseline` leg and
//     `bench.py --impl reference`), reproducing the osu_bcast method of
//     `bcastlab bench` (proj/tools/bcastlab.cpp:147-206) through the public
//     launch_ranks + execute_rank API (proj/include/bcastlab/runtime.hpp:72-138),
//     because run_bench_size itself is file-local to the CLI.
//
// Subcommands (all output on stdout):
//   schedule ALGO N ROOT M CHUNK RADIX      -> "chunks" lines then to_text()
//   bcast ALGO N ROOT M CHUNK RADIX SEED T  -> FNV-1a of every rank's buffer
//                                              after run_bcast (T = inproc|socket)
//   tune NLIST SIZES_LO SIZES_HI CANDS CHUNKS_LO CHUNKS_HI [ORACLE]
//                                           -> save_table() text
//   select TABLE_PATH N M...                 -> "algo radix chunk" per M
//   bench ALGO N ROOT M CHUNK RADIX WARMUP ITERS T SEED
//                                           -> JSON with min/median/avg/max us
//   models N M CHUNK                         -> Eq.3/4/5 costs at desk params
//   simulate ALGO N ROOT M CHUNK RADIX TS BW OUT.csv
//                                           -> reference simulator trace CSV
//                                              (simengine.hpp:61-70) + completions
#include <algorithm>
#include <barrier>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "bcastlab/models.hpp"
#include "bcastlab/runtime.hpp"
#include "bcastlab/schedules.hpp"
#include "bcastlab/simengine.hpp"
#include "bcastlab/tuner.hpp"

using namespace bcastlab;

namespace {

std::uint64_t fnv1a(const std::uint8_t* p, std::size_t n) {
  std::uint64_t h = 1469598103934665603ull;
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

// Same generator formula as the reference CLI's payload_for
// (proj/tools/bcastlab.cpp:140-145); restated because it is file-local.
std::vector<std::uint8_t> payload(std::uint64_t seed, std::uint64_t size) {
  std::mt19937_64 rng(seed * 0x9e3779b97f4a7c15ULL + size + 1);
  std::vector<std::uint8_t> data(size);
  for (auto& b : data) b = static_cast<std::uint8_t>(rng());
  return data;
}

AlgorithmConfig parse_config(const char* algo, const char* chunk,
                             const char* radix) {
  const auto a = algorithm_from_name(algo);
  if (!a) {
    std::fprintf(stderr, "unknown algorithm %s\n", algo);
    std::exit(2);
  }
  return AlgorithmConfig{*a, std::atoi(radix),
                         std::strtoull(chunk, nullptr, 10)};
}

std::vector<std::uint64_t> pow2(std::uint64_t lo, std::uint64_t hi) {
  std::vector<std::uint64_t> v;
  for (std::uint64_t s = lo; s <= hi; s *= 2) v.push_back(s);
  return v;
}

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string f;
  std::istringstream in(s);
  while (std::getline(in, f, sep)) out.push_back(f);
  return out;
}

std::unique_ptr<TransportFabric> fabric_for(const std::string& t, int n) {
  return t == "socket" ? make_socket_fabric(n) : make_inproc_fabric(n);
}

int cmd_schedule(char** a) {
  const AlgorithmConfig cfg = parse_config(a[0], a[4], a[5]);
  const Schedule s = make_schedule(cfg, std::atoi(a[1]), std::atoi(a[2]),
                                   std::strtoull(a[3], nullptr, 10));
  std::printf("prologue %d\n", static_cast<int>(s.prologue));
  for (const ChunkSpec& c : s.chunks) {
    std::printf("chunk %u %llu %llu\n", c.chunk_id,
                static_cast<unsigned long long>(c.offset_bytes),
                static_cast<unsigned long long>(c.length_bytes));
  }
  for (int r = 0; r < s.n_ranks; ++r) {
    for (const Event& e : s.per_rank_ops[static_cast<std::size_t>(r)]) {
      std::printf("event %d %s %d %u %u\n", r,
                  e.kind == Event::Kind::Send ? "send" : "recv", e.peer,
                  e.chunk, e.group);
    }
  }
  return 0;
}

int cmd_bcast(char** a) {
  const AlgorithmConfig cfg = parse_config(a[0], a[4], a[5]);
  const int n = std::atoi(a[1]);
  const int root = std::atoi(a[2]);
  const std::uint64_t m = std::strtoull(a[3], nullptr, 10);
  const std::uint64_t seed = std::strtoull(a[6], nullptr, 10);
  const auto data = payload(seed, m);
  std::vector<std::vector<std::uint8_t>> bufs(static_cast<std::size_t>(n),
                                              std::vector<std::uint8_t>(m, 0));
  bufs[static_cast<std::size_t>(root)] = data;
  std::vector<std::span<std::uint8_t>> spans(bufs.begin(), bufs.end());
  auto fabric = fabric_for(a[7], n);
  run_bcast(BcastRequest{n, root, spans, cfg}, *fabric);
  std::printf("payload %016llx\n",
              static_cast<unsigned long long>(fnv1a(data.data(), m)));
  for (int r = 0; r < n; ++r) {
    const auto& b = bufs[static_cast<std::size_t>(r)];
    std::printf("rank %d %016llx\n", r,
                static_cast<unsigned long long>(fnv1a(b.data(), b.size())));
  }
  return 0;
}

int cmd_tune(char** a, int argc) {
  std::vector<int> n_list;
  for (const auto& f : split(a[0], ',')) n_list.push_back(std::atoi(f.c_str()));
  const auto sizes = pow2(std::strtoull(a[1], nullptr, 10),
                          std::strtoull(a[2], nullptr, 10));
  std::vector<AlgorithmConfig> cands;
  for (const auto& f : split(a[3], ',')) {
    const auto algo = algorithm_from_name(f);
    AlgorithmConfig c{*algo, 0, 0};
    if (algorithm_uses_radix(*algo)) c.radix_k = 2;
    cands.push_back(c);
  }
  const auto chunks = pow2(std::strtoull(a[4], nullptr, 10),
                           std::strtoull(a[5], nullptr, 10));
  CostOracle oracle = CostOracle::Analytical;
  if (argc > 6) oracle = *oracle_from_name(a[6]);
  NetworkParams p{1e-6, 1e9, 1e10};
  if (argc > 8) {
    p.startup_s = std::strtod(a[7], nullptr);
    p.link_bandwidth_Bps = std::strtod(a[8], nullptr);
  }
  const TuningTable t = tune(n_list, sizes, cands, chunks, p, oracle);
  std::ostringstream out;
  save_table(t, out);
  std::fputs(out.str().c_str(), stdout);
  return 0;
}

int cmd_select(char** a, int argc) {
  TuningTable t;
  try {
    t = load_table(std::filesystem::path(a[0]));
  } catch (const TableParseError& e) {
    std::printf("parse_error %zu %s\n", e.line(), e.what());
    return 0;
  }
  const int n = std::atoi(a[1]);
  for (int i = 2; i < argc; ++i) {
    try {
      const AlgorithmConfig c = select(t, n, std::strtoull(a[i], nullptr, 10));
      std::printf("%s %d %llu\n", std::string(algorithm_name(c.algorithm)).c_str(),
                  c.radix_k, static_cast<unsigned long long>(c.chunk_bytes));
    } catch (const std::out_of_range& e) {
      std::printf("out_of_range\n");
    }
  }
  return 0;
}

int cmd_bench(char** a) {
  const AlgorithmConfig cfg = parse_config(a[0], a[4], a[5]);
  const int n = std::atoi(a[1]);
  const int root = std::atoi(a[2]);
  const std::uint64_t m = std::strtoull(a[3], nullptr, 10);
  const int warmup = std::atoi(a[6]);
  const int iters = std::atoi(a[7]);
  const std::string transport = a[8];
  const std::uint64_t seed = std::strtoull(a[9], nullptr, 10);
  const Schedule schedule = make_schedule(cfg, n, root, m);
  const auto data = payload(seed, m);
  std::vector<std::vector<std::uint8_t>> bufs(static_cast<std::size_t>(n),
                                              std::vector<std::uint8_t>(m));
  bufs[static_cast<std::size_t>(root)] = data;
  auto fabric = fabric_for(transport, n);
  std::barrier sync(n);
  std::vector<double> elapsed(static_cast<std::size_t>(n), 0.0);
  std::vector<double> lat;
  bool ok = true;
  launch_ranks(n, [&](int rank) {
    auto& buf = bufs[static_cast<std::size_t>(rank)];
    for (int it = 0; it < warmup + iters; ++it) {
      if (rank != root) std::fill(buf.begin(), buf.end(), 0);
      sync.arrive_and_wait();
      const auto t0 = std::chrono::steady_clock::now();
      execute_rank(schedule, rank, buf, fabric->endpoint(rank));
      const auto t1 = std::chrono::steady_clock::now();
      if (buf != data) ok = false;
      elapsed[static_cast<std::size_t>(rank)] =
          std::chrono::duration<double, std::micro>(t1 - t0).count();
      sync.arrive_and_wait();
      if (rank == root && it >= warmup) {
        lat.push_back(*std::max_element(elapsed.begin(), elapsed.end()));
      }
      sync.arrive_and_wait();
    }
  });
  std::vector<double> sorted = lat;
  std::sort(sorted.begin(), sorted.end());
  double sum = 0;
  for (double v : lat) sum += v;
  std::printf(
      "{\"ok\": %s, \"n\": %d, \"bytes\": %llu, \"algorithm\": \"%s\", "
      "\"chunk\": %llu, \"transport\": \"%s\", \"iters\": %d, "
      "\"min_us\": %.3f, \"median_us\": %.3f, \"avg_us\": %.3f, "
      "\"max_us\": %.3f}\n",
      ok ? "true" : "false", n, static_cast<unsigned long long>(m), a[0],
      static_cast<unsigned long long>(cfg.chunk_bytes), transport.c_str(),
      iters, sorted.front(), sorted[sorted.size() / 2], sum / lat.size(),
      sorted.back());
  return ok ? 0 : 1;
}

int cmd_models(char** a) {
  const NetworkParams p{1e-6, 1e9, 1e10};
  const int n = std::atoi(a[0]);
  const std::uint64_t m = std::strtoull(a[1], nullptr, 10);
  const std::uint64_t c = std::strtoull(a[2], nullptr, 10);
  std::printf("knomial %.17g\n", cost_knomial(n, 2, m, p).total_s);
  std::printf("scatter_ring_allgather %.17g\n",
              cost_scatter_ring_allgather(n, m, p).total_s);
  std::printf("chain_pipelined %.17g\n",
              cost_chain_pipelined(n, m, c, p).total_s);
  return 0;
}

int cmd_simulate(char** a) {
  const AlgorithmConfig cfg = parse_config(a[0], a[4], a[5]);
  const NetworkParams p{std::strtod(a[6], nullptr), std::strtod(a[7], nullptr), 1e10};
  const Schedule s = make_schedule(cfg, std::atoi(a[1]), std::atoi(a[2]), std::strtoull(a[3], nullptr, 10));
  SimOptions opt;
  opt.record_trace = true;
  const SimResult r = simulate(s, p, opt);
  std::ofstream out(a[8]);
  write_trace_csv(r, out);
  for (std::size_t i = 0; i < r.completion_s.size(); ++i) std::printf("rank %zu %.9g\n", i, r.completion_s[i]);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_harness schedule|bcast|tune|select|bench|models ...\n");
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "schedule" && argc >= 8) return cmd_schedule(argv + 2);
    if (cmd == "bcast" && argc >= 10) return cmd_bcast(argv + 2);
    if (cmd == "tune" && argc >= 8) return cmd_tune(argv + 2, argc - 2);
    if (cmd == "select" && argc >= 5) return cmd_select(argv + 2, argc - 2);
    if (cmd == "bench" && argc >= 12) return cmd_bench(argv + 2);
    if (cmd == "models" && argc >= 5) return cmd_models(argv + 2);
    if (cmd == "simulate" && argc >= 11) return cmd_simulate(argv + 2);
  } catch (const std::exception& e) {
    std::printf("error %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "bad arguments\n");
  return 2;
}
