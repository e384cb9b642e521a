// bcl_tuner.cpp — see bcl_tuner.hpp for the reference mapping.
#include "bcl_tuner.hpp"

#include <algorithm>
#include <cstdio>
#include <charconv>
#include <cmath>
#include <fstream>
#include <istream>
#include <map>
#include <ostream>
#include <sstream>

#include "bcl_builtin_table.inc"  // kBuiltinTableCsv

namespace bcl {

namespace {

constexpr std::string_view kColumns =
    "n,msg_min_bytes,msg_max_bytes,algorithm,radix,chunk_bytes,predicted_cost_s";
constexpr std::string_view kPragma = "# oracle:";
constexpr std::string_view kMeasuredPragma = "# bcl-oracle: measured";
constexpr std::string_view kPushPragma = "# bcl-push-from:";
constexpr std::string_view kLL128Pragma = "# bcl-ll128-upto:";

// Rounded geometric mean of two sizes (tuner.cpp:27-31).
std::uint64_t geo_mid(std::uint64_t a, std::uint64_t b) {
  return static_cast<std::uint64_t>(
      std::llround(std::sqrt(static_cast<double>(a) * static_cast<double>(b))));
}

CostBreakdown sum_terms(double startup, double bandwidth, double staging = 0.0) {
  return CostBreakdown{startup, bandwidth, staging, startup + bandwidth + staging};
}

// The per-call constant joins the startup term (0 leaves every reference
// value bit-identical).
CostBreakdown with_call(CostBreakdown c, double call_s) {
  if (call_s == 0.0) return c;
  c.startup_term_s += call_s;
  c.total_s = c.startup_term_s + c.bandwidth_term_s + c.staging_term_s;
  return c;
}

void need_ranks(int n) {
  if (n < 1) throw std::invalid_argument("rank count must be >= 1");
}

}  // namespace

void NetworkParams::validate() const {
  if (startup_s < 0.0) throw std::invalid_argument("startup_s must be >= 0");
  if (!(link_bandwidth_Bps > 0.0)) throw std::invalid_argument("link_bandwidth_Bps must be > 0");
  if (!(staging_bandwidth_Bps > 0.0)) throw std::invalid_argument("staging_bandwidth_Bps must be > 0");
  if (call_overhead_s < 0.0) throw std::invalid_argument("call_overhead_s must be >= 0");
}

// Eqs. 1-6 (models.cpp:34-104); every term is (steps * startup,
// steps * bytes / B) except SRA's 2(n-1)/n bandwidth factor and the staged
// tree's extra M / B_staging.
namespace {
CostBreakdown reference_cost(const AlgorithmConfig& cfg, int n, std::uint64_t m, const NetworkParams& p);
}  // namespace

CostBreakdown cost_for(const AlgorithmConfig& cfg, int n, std::uint64_t m, const NetworkParams& p) {
  return with_call(reference_cost(cfg, n, m, p), p.call_overhead_s);
}

namespace {
CostBreakdown reference_cost(const AlgorithmConfig& cfg, int n, std::uint64_t m,
                             const NetworkParams& p) {
  cfg.validate();
  const double per_msg = static_cast<double>(m) / p.link_bandwidth_Bps;
  switch (cfg.algorithm) {
    case Algorithm::Direct: {
      need_ranks(n); p.validate();
      const double k = static_cast<double>(n);
      return sum_terms(k * p.startup_s, k * per_msg);
    }
    case Algorithm::Chain: {
      need_ranks(n); p.validate();
      const double k = static_cast<double>(n - 1);
      return sum_terms(k * p.startup_s, k * per_msg);
    }
    case Algorithm::Knomial:
    case Algorithm::KnomialStaged: {
      need_ranks(n);
      if (cfg.radix_k < 2) throw std::invalid_argument("radix must be >= 2");
      p.validate();
      const double k = static_cast<double>(ceil_log(cfg.radix_k, n));
      if (cfg.algorithm == Algorithm::Knomial) return sum_terms(k * p.startup_s, k * per_msg);
      return sum_terms(k * p.startup_s, k * per_msg,
                       static_cast<double>(m) / p.staging_bandwidth_Bps);
    }
    case Algorithm::ScatterRingAllgather: {
      need_ranks(n); p.validate();
      const double k = static_cast<double>(ceil_log(2, n) + n - 1);
      const double frac = static_cast<double>(n - 1) / static_cast<double>(n);
      return sum_terms(k * p.startup_s, 2.0 * frac * per_msg);
    }
    case Algorithm::ChainPipelined: {
      if (n < 2) throw std::invalid_argument("pipelined chain needs at least 2 ranks");
      p.validate();
      // Every chunk billed at the (clamped) uniform chunk size.
      const std::uint64_t c = std::min(cfg.chunk_bytes, std::max<std::uint64_t>(m, 0));
      const std::uint64_t count = m == 0 ? 1 : (m + cfg.chunk_bytes - 1) / cfg.chunk_bytes;
      const double k = static_cast<double>(count + static_cast<std::uint64_t>(n) - 2);
      return sum_terms(k * p.startup_s, k * (static_cast<double>(m == 0 ? 0 : c) / p.link_bandwidth_Bps));
    }
  }
  throw std::invalid_argument("unknown algorithm");
}
}  // namespace

std::string_view oracle_name(CostOracle o) {
  switch (o) {
    case CostOracle::Analytical: return "analytical";
    case CostOracle::Simulated: return "simulated";
    case CostOracle::Measured: return "measured";
  }
  return "analytical";
}

bool beats(double lc, const AlgorithmConfig& l, double rc, const AlgorithmConfig& r) {
  if (lc != rc) return lc < rc;
  if (l.algorithm != r.algorithm) return l.algorithm < r.algorithm;
  if (l.chunk_bytes != r.chunk_bytes) return l.chunk_bytes < r.chunk_bytes;
  return l.radix_k < r.radix_k;
}

std::vector<AlgorithmConfig> expand_candidates(
    const std::vector<AlgorithmConfig>& cands,
    const std::vector<std::uint64_t>& chunks, std::uint64_t m) {
  std::vector<AlgorithmConfig> out;
  const auto add = [&out](const AlgorithmConfig& c) {
    if (std::find(out.begin(), out.end(), c) == out.end()) out.push_back(c);
  };
  for (const AlgorithmConfig& c : cands) {
    if (c.algorithm != Algorithm::ChainPipelined) {
      out.push_back(c);  // templates other than the chain are kept verbatim
      continue;
    }
    for (std::uint64_t chunk : chunks) {
      AlgorithmConfig v = c;
      v.chunk_bytes = std::clamp<std::uint64_t>(chunk, 1, std::max<std::uint64_t>(m, 1));
      add(v);
    }
  }
  return out;
}

TuningTable tune(const std::vector<int>& n_list,
                 const std::vector<std::uint64_t>& sizes,
                 const std::vector<AlgorithmConfig>& cands,
                 const std::vector<std::uint64_t>& chunks,
                 const CostFn& cost, CostOracle oracle) {
  if (n_list.empty() || sizes.empty() || cands.empty()) {
    throw std::invalid_argument("tune needs ranks, sizes, and candidates");
  }
  if (!std::is_sorted(sizes.begin(), sizes.end(), std::less_equal<>()) ||
      std::adjacent_find(sizes.begin(), sizes.end()) != sizes.end()) {
    throw std::invalid_argument("message sizes must be strictly increasing");
  }
  if (sizes.front() == 0) throw std::invalid_argument("message sizes must be >= 1");

  // Elementary range i is [edge[i], edge[i+1]) with edges at the geometric
  // means of neighbouring swept sizes; the last range ends at twice the top.
  std::vector<std::uint64_t> edge{sizes.front()};
  for (std::size_t i = 1; i < sizes.size(); ++i) edge.push_back(geo_mid(sizes[i - 1], sizes[i]));
  edge.push_back(sizes.back() * 2);

  TuningTable table;
  table.oracle = oracle;
  for (int n : n_list) {
    std::vector<TuningEntry> row;
    for (std::size_t i = 0; i < sizes.size(); ++i) {
      const auto options = expand_candidates(cands, chunks, sizes[i]);
      if (options.empty()) throw std::invalid_argument("no evaluable candidate");
      AlgorithmConfig best = options.front();
      double best_cost = cost(best, n, sizes[i]);
      for (std::size_t j = 1; j < options.size(); ++j) {
        const double c = cost(options[j], n, sizes[i]);
        if (beats(c, options[j], best_cost, best)) {
          best = options[j];
          best_cost = c;
        }
      }
      if (!row.empty() && row.back().config == best) {
        row.back().msg_max_bytes = edge[i + 1];
      } else {
        row.push_back(TuningEntry{n, edge[i], edge[i + 1], best, 0.0});
      }
    }
    for (TuningEntry& e : row) {
      e.predicted_cost_s = cost(e.config, n, geo_mid(e.msg_min_bytes, e.msg_max_bytes));
    }
    table.entries.insert(table.entries.end(), row.begin(), row.end());
  }
  std::stable_sort(table.entries.begin(), table.entries.end(),
                   [](const TuningEntry& a, const TuningEntry& b) {
                     return a.n != b.n ? a.n < b.n : a.msg_min_bytes < b.msg_min_bytes;
                   });
  return table;
}

TuningTable tune(const std::vector<int>& n_list,
                 const std::vector<std::uint64_t>& sizes,
                 const std::vector<AlgorithmConfig>& cands,
                 const std::vector<std::uint64_t>& chunks,
                 const NetworkParams& params, CostOracle oracle) {
  params.validate();
  if (oracle != CostOracle::Analytical) {
    throw std::invalid_argument(
        "only the analytical oracle is built in; pass a cost function for measured tables");
  }
  return tune(n_list, sizes, cands, chunks,
              [&params](const AlgorithmConfig& c, int n, std::uint64_t m) {
                return cost_for(c, n, m, params).total_s;
              },
              oracle);
}

AlgorithmConfig select(const TuningTable& t, int n, std::uint64_t m) {
  if (t.entries.empty()) throw std::out_of_range("tuning table is empty");
  int best_n = -1;
  for (const TuningEntry& e : t.entries) {
    if (e.n <= n) best_n = std::max(best_n, e.n);
  }
  if (best_n < 0) throw std::out_of_range("no tuned rank count <= " + std::to_string(n));
  const TuningEntry* hit = nullptr;
  for (const TuningEntry& e : t.entries) {
    if (e.n != best_n) continue;
    hit = &e;  // sorted ranges: the last one clamps larger sizes
    if (m < e.msg_max_bytes) break;
  }
  return hit->config;
}

bool select_push(const TuningTable& t, int n, std::uint64_t m) {
  int best_n = -1;
  std::uint64_t from = 0;
  for (const auto& [pn, bytes] : t.push_from) {
    if (pn <= n && pn > best_n) {
      best_n = pn;
      from = bytes;
    }
  }
  return best_n >= 0 && m >= from;
}

bool select_ll128(const TuningTable& t, int n, std::uint64_t m) {
  int best_n = -1;
  std::uint64_t upto = 0;
  for (const auto& [pn, bytes] : t.ll128_upto) {
    if (pn <= n && pn > best_n) {
      best_n = pn;
      upto = bytes;
    }
  }
  return best_n < 0 || m <= upto;  // no rule: up to the group's LL128 cap
}

TableParseError::TableParseError(std::size_t line, const std::string& what)
    : std::runtime_error("line " + std::to_string(line) + ": " + what), line_(line) {}

std::string save_table_text(const TuningTable& t) {
  std::string s;
  if (t.oracle == CostOracle::Measured) {
    s.append(kMeasuredPragma);
    if (!t.provenance.empty()) s.append(" ").append(t.provenance);
  } else {
    s.append(kPragma).append(" ").append(oracle_name(t.oracle));
  }
  s.append("\n");
  for (const auto& [pn, bytes] : t.push_from) {
    s.append(kPushPragma).append(" n=").append(std::to_string(pn)).append(" bytes=").append(std::to_string(bytes));
    s.append("\n");
  }
  for (const auto& [pn, bytes] : t.ll128_upto) {
    s.append(kLL128Pragma).append(" n=").append(std::to_string(pn)).append(" bytes=").append(std::to_string(bytes));
    s.append("\n");
  }
  s.append(kColumns).append("\n");
  char num[64];
  for (const TuningEntry& e : t.entries) {
    const Algorithm a = e.config.algorithm;
    s += std::to_string(e.n) + ',' + std::to_string(e.msg_min_bytes) + ',' +
         std::to_string(e.msg_max_bytes) + ',' + std::string(algorithm_name(a)) + ',' +
         std::to_string(algorithm_uses_radix(a) ? e.config.radix_k : 0) + ',' +
         std::to_string(algorithm_uses_chunk(a) ? e.config.chunk_bytes : 0) + ',';
    const auto r = std::to_chars(num, num + sizeof num, e.predicted_cost_s);
    s.append(num, r.ptr);
    s += '\n';
  }
  return s;
}

void save_table(const TuningTable& t, std::ostream& out) { out << save_table_text(t); }

void save_table_file(const TuningTable& t, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path + " for writing");
  f << save_table_text(t);
  if (!f.flush()) throw std::runtime_error("failed writing " + path);
}

namespace {

template <typename T>
T field_number(const std::string& s, std::size_t line) {
  T v{};
  const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc{} || r.ptr != s.data() + s.size()) {
    if constexpr (std::is_floating_point_v<T>) {
      throw TableParseError(line, "bad cost field '" + s + "'");
    } else {
      throw TableParseError(line, "bad numeric field '" + s + "'");
    }
  }
  return v;
}

std::vector<std::string> csv_fields(const std::string& line) {
  std::vector<std::string> out(1);
  for (char ch : line) {
    if (ch == ',') out.emplace_back();
    else out.back().push_back(ch);
  }
  return out;
}

}  // namespace

TuningTable load_table(std::istream& in) {
  TuningTable t;
  std::string line;
  std::size_t no = 0;
  bool header = false;
  while (std::getline(in, line)) {
    ++no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (line.rfind(kPragma, 0) == 0) {
      std::string name = line.substr(kPragma.size());
      name.erase(0, name.find_first_not_of(' '));
      if (name == "analytical") t.oracle = CostOracle::Analytical;
      else if (name == "simulated") t.oracle = CostOracle::Simulated;
      else throw TableParseError(no, "unknown oracle '" + name + "'");
      continue;
    }
    if (line.rfind(kPushPragma, 0) == 0) {
      int pn = 0;
      unsigned long long bytes = 0;
      if (std::sscanf(line.c_str() + kPushPragma.size(), " n=%d bytes=%llu", &pn, &bytes) != 2 || pn < 1) {
        throw TableParseError(no, "bad push pragma");
      }
      t.push_from.emplace_back(pn, static_cast<std::uint64_t>(bytes));
      continue;
    }
    if (line.rfind(kLL128Pragma, 0) == 0) {
      int pn = 0;
      unsigned long long bytes = 0;
      if (std::sscanf(line.c_str() + kLL128Pragma.size(), " n=%d bytes=%llu", &pn, &bytes) != 2 || pn < 1) {
        throw TableParseError(no, "bad ll128 pragma");
      }
      t.ll128_upto.emplace_back(pn, static_cast<std::uint64_t>(bytes));
      continue;
    }
    if (line.rfind(kMeasuredPragma, 0) == 0) {
      t.oracle = CostOracle::Measured;
      t.provenance = line.size() > kMeasuredPragma.size() + 1 ? line.substr(kMeasuredPragma.size() + 1) : "";
      continue;
    }
    if (line[0] == '#') continue;
    if (!header) {
      if (line != kColumns) throw TableParseError(no, "missing table header");
      header = true;
      continue;
    }
    const auto f = csv_fields(line);
    if (f.size() != 7) {
      throw TableParseError(no, "expected 7 fields, got " + std::to_string(f.size()));
    }
    TuningEntry e;
    e.n = field_number<int>(f[0], no);
    e.msg_min_bytes = field_number<std::uint64_t>(f[1], no);
    e.msg_max_bytes = field_number<std::uint64_t>(f[2], no);
    const auto algo = algorithm_from_name(f[3]);
    if (!algo) throw TableParseError(no, "unknown algorithm '" + f[3] + "'");
    e.config.algorithm = *algo;
    e.config.radix_k = field_number<int>(f[4], no);
    e.config.chunk_bytes = field_number<std::uint64_t>(f[5], no);
    e.predicted_cost_s = field_number<double>(f[6], no);
    if (e.n < 1) throw TableParseError(no, "rank count must be >= 1");
    if (e.msg_min_bytes >= e.msg_max_bytes) throw TableParseError(no, "empty message-size range");
    t.entries.push_back(e);
  }
  if (!header) throw TableParseError(no, "missing table header");
  if (t.entries.empty()) throw TableParseError(no, "table has no entries");
  std::map<int, std::uint64_t> end_of;
  for (const TuningEntry& e : t.entries) {
    const auto it = end_of.find(e.n);
    if (it != end_of.end() && e.msg_min_bytes < it->second) {
      throw TableParseError(no, "overlapping or unsorted ranges for n=" + std::to_string(e.n));
    }
    end_of[e.n] = e.msg_max_bytes;
  }
  return t;
}

TuningTable load_table_text(const std::string& text) {
  std::istringstream in(text);
  return load_table(in);
}

TuningTable load_table_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path);
  return load_table(f);
}

const TuningTable& builtin_table() {
  static const TuningTable t = load_table_text(kBuiltinTableCsv);
  return t;
}

}  // namespace bcl
