// bcl_core: broadcast domain types, chunking and the schedule generators.
//
// Host-side C++ mirror of the reference's L1/L2 surface (bcastlab
// core.hpp / schedules.hpp) with identical names, argument meaning and error
// behaviour, so a reference user finds the same vocabulary:
//   Algorithm enum order        = proj/include/bcastlab/core.hpp:27-34 (tie-break order)
//   AlgorithmConfig             = core.hpp:45-53, validate() core.cpp:56-65
//   ChunkSpec / make_chunks     = core.hpp:56-62, core.cpp:67-85
//   Event / Schedule            = core.hpp:71-117
//   schedule_* / make_schedule  = schedules.hpp:17-35, schedules.cpp:115-263
// The schedules are the *contract* the device executor (bcl_kernels.cu) runs:
// every Recv(peer, chunk) event becomes a pull of that chunk from the peer's
// buffer after the peer published it; every Send(peer, chunk) becomes a
// release of the per-lane ready counter in the peer's flag array.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace bcl {

enum class Algorithm : int {
  Direct = 0,
  Chain,
  Knomial,
  ScatterRingAllgather,
  ChainPipelined,
  KnomialStaged,
};
inline constexpr int kAlgorithmCount = 6;

std::string_view algorithm_name(Algorithm a);
std::optional<Algorithm> algorithm_from_name(std::string_view name);
bool algorithm_uses_radix(Algorithm a);
bool algorithm_uses_chunk(Algorithm a);

struct AlgorithmConfig {
  Algorithm algorithm{Algorithm::Chain};
  int radix_k{0};
  std::uint64_t chunk_bytes{0};
  void validate() const;  // std::invalid_argument on a missing parameter
  bool operator==(const AlgorithmConfig&) const = default;
};

struct ChunkSpec {
  std::uint32_t chunk_id{};
  std::uint64_t offset_bytes{};
  std::uint64_t length_bytes{};
  bool operator==(const ChunkSpec&) const = default;
};

struct Event {
  enum class Kind : std::uint8_t { Send, Recv };
  Kind kind{Kind::Send};
  int peer{};
  std::uint32_t chunk{};
  std::uint32_t group{0};
  bool operator==(const Event&) const = default;
};

enum class RootPrologue : std::uint8_t { None, SelfSend, HostStaging };

struct Schedule {
  int n_ranks{};
  int root{};
  std::uint64_t message_bytes{};
  RootPrologue prologue{RootPrologue::None};
  std::vector<ChunkSpec> chunks;
  std::vector<std::vector<Event>> per_rank_ops;
  bool operator==(const Schedule&) const = default;
};

std::vector<ChunkSpec> make_chunks(std::uint64_t message_bytes,
                                   std::uint64_t chunk_bytes);

Schedule schedule_direct(int n, int root, std::uint64_t message_bytes);
Schedule schedule_chain(int n, int root, std::uint64_t message_bytes);
Schedule schedule_knomial(int n, int radix_k, int root,
                          std::uint64_t message_bytes);
Schedule schedule_scatter_ring_allgather(int n, int root,
                                         std::uint64_t message_bytes);
Schedule schedule_chain_pipelined(int n, int root,
                                  std::uint64_t message_bytes,
                                  std::uint64_t chunk_bytes);
Schedule schedule_knomial_staged(int n, int radix_k, int root,
                                 std::uint64_t message_bytes);
Schedule make_schedule(const AlgorithmConfig& config, int n, int root,
                       std::uint64_t message_bytes);

struct ScheduleViolation {
  int rank{-1};
  std::size_t event_index{0};
  std::string description;
};
std::optional<ScheduleViolation> validate_schedule(const Schedule& s);
std::string to_text(const Schedule& s);
int ceil_log(int base, std::int64_t n);

}  // namespace bcl
