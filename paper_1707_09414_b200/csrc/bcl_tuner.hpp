// bcl_tuner: the collective tuning framework (paper §IV-C).
//
// Drop-in for the reference tuner surface (proj/include/bcastlab/tuner.hpp):
//   tune()        tuner.cpp:118-176   brute-force argmin per (n, swept size),
//                                     geometric-mean range bounds, merged ranges
//   select()      tuner.cpp:178-197   exact n else nearest smaller; clamping
//   save/load     tuner.cpp:203-353   7-column CSV, strict parser, TableParseError
//   beats/expand  tuner.cpp:84-116    tie-breaks and chunk fan-out
// plus the closed-form costs it uses as a prior (models.cpp:34-124, Eqs. 1-6).
//
// New on B200: a Measured oracle. Its costs come from a callback that times
// the real device broadcast (see bcl_comm / tools/tune_b200.py); such tables
// carry a "# bcl-oracle: measured ..." comment instead of the reference's
// "# oracle:" pragma so the unmodified reference load_table still accepts
// them (it skips other '#' lines, tuner.cpp:286).
#pragma once

#include <cstdint>
#include <functional>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <vector>

#include "bcl_core.hpp"

namespace bcl {

struct NetworkParams {  // core.hpp:16-25
  double startup_s{1e-6};
  double link_bandwidth_Bps{1e9};
  double staging_bandwidth_Bps{1e10};
  // New on B200: a per-call constant a0 added to every algorithm's cost (the
  // kernel launch, the first flag hand-off and the final acknowledgement).
  // Eq. 5 as the paper states it misses B200 measurements by a median 26-30%;
  // with a0 the fit is within 1-3%. 0 = the reference model.
  double call_overhead_s{0.0};
  void validate() const;
  bool operator==(const NetworkParams&) const = default;
};

struct CostBreakdown {  // models.hpp:15-22
  double startup_term_s{};
  double bandwidth_term_s{};
  double staging_term_s{};
  double total_s{};
};

CostBreakdown cost_for(const AlgorithmConfig& config, int n,
                       std::uint64_t message_bytes, const NetworkParams& p);

enum class CostOracle { Analytical, Simulated, Measured };
std::string_view oracle_name(CostOracle o);

struct TuningEntry {
  int n{};
  std::uint64_t msg_min_bytes{};
  std::uint64_t msg_max_bytes{};
  AlgorithmConfig config{};
  double predicted_cost_s{};
  bool operator==(const TuningEntry&) const = default;
};

struct TuningTable {
  CostOracle oracle{CostOracle::Analytical};
  std::string provenance;  // free text after "# bcl-oracle: measured"
  std::vector<TuningEntry> entries;
  // B200 transport protocol for chain_pipelined: from this many bytes on, at
  // this rank count (nearest smaller tuned n), producers push instead of
  // consumers pulling. Stored as "# bcl-push-from: n=<n> bytes=<b>" lines,
  // which the reference load_table skips as comments.
  std::vector<std::pair<int, std::uint64_t>> push_from;
  // LL128 line protocol for chain_pipelined up to this many bytes at this
  // rank count ("# bcl-ll128-upto: n=<n> bytes=<b>", also a comment to the
  // reference loader); without a rule, up to the group's LL128 cap.
  std::vector<std::pair<int, std::uint64_t>> ll128_upto;
  bool operator==(const TuningTable& o) const {
    return oracle == o.oracle && entries == o.entries;
  }
};

using CostFn = std::function<double(const AlgorithmConfig&, int n, std::uint64_t bytes)>;

bool beats(double lhs_cost, const AlgorithmConfig& lhs, double rhs_cost,
           const AlgorithmConfig& rhs);
std::vector<AlgorithmConfig> expand_candidates(
    const std::vector<AlgorithmConfig>& candidates,
    const std::vector<std::uint64_t>& chunk_candidates,
    std::uint64_t message_bytes);

// Analytical oracle (the reference's default path).
TuningTable tune(const std::vector<int>& n_list,
                 const std::vector<std::uint64_t>& msg_sizes,
                 const std::vector<AlgorithmConfig>& candidates,
                 const std::vector<std::uint64_t>& chunk_candidates,
                 const NetworkParams& params, CostOracle oracle);
// Any oracle given as a cost function (Measured on B200).
TuningTable tune(const std::vector<int>& n_list,
                 const std::vector<std::uint64_t>& msg_sizes,
                 const std::vector<AlgorithmConfig>& candidates,
                 const std::vector<std::uint64_t>& chunk_candidates,
                 const CostFn& cost, CostOracle oracle);

AlgorithmConfig select(const TuningTable& table, int n,
                       std::uint64_t message_bytes);
// Whether a chain_pipelined call of this size should use the push protocol.
bool select_push(const TuningTable& table, int n, std::uint64_t message_bytes);
// Whether a chain_pipelined call of this size may use LL128 lines.
bool select_ll128(const TuningTable& table, int n, std::uint64_t message_bytes);

class TableParseError : public std::runtime_error {
 public:
  TableParseError(std::size_t line, const std::string& what);
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};

void save_table(const TuningTable& table, std::ostream& out);
std::string save_table_text(const TuningTable& table);
void save_table_file(const TuningTable& table, const std::string& path);
TuningTable load_table(std::istream& in);
TuningTable load_table_text(const std::string& text);
TuningTable load_table_file(const std::string& path);

// The B200 default table compiled into the library (measured, see
// tables/b200_measured.csv); used by bcast() when no table was loaded.
const TuningTable& builtin_table();

}  // namespace bcl
