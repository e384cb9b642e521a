// bcl_core.cpp — see bcl_core.hpp. Semantics follow the reference
// (proj/src/core.cpp, proj/src/schedules.cpp); the structure is our own:
// every generator describes its transfers as (from, to, chunk, group) pairs in
// *logical* rank space through a Plan, which emits the matching Send/Recv pair
// and relabels logical l -> (l + root) mod n when the schedule is sealed
// (rotate_to_root, schedules.cpp:24-44).
#include "bcl_core.hpp"

#include <algorithm>
#include <array>
#include <map>
#include <sstream>
#include <utility>

namespace bcl {

namespace {

constexpr std::array<std::string_view, kAlgorithmCount> kNames{
    "direct",          "chain",          "knomial", "scatter_ring_allgather",
    "chain_pipelined", "knomial_staged"};

void check_root(int n, int root) {  // schedules.cpp:14-21
  if (n < 1) throw std::invalid_argument("rank count must be >= 1");
  if (root < 0 || root >= n) throw std::invalid_argument("root out of range");
}

// Collects per-logical-rank event lists; seal() rotates to actual ranks.
class Plan {
 public:
  Plan(int n, int root, std::uint64_t message_bytes)
      : n_(n), root_(root), bytes_(message_bytes),
        ops_(static_cast<std::size_t>(n)) {}

  void send(int from, int to, std::uint32_t chunk, std::uint32_t group = 0) {
    ops_[static_cast<std::size_t>(from)].push_back(
        Event{Event::Kind::Send, to, chunk, group});
  }
  void recv(int at, int from, std::uint32_t chunk) {
    ops_[static_cast<std::size_t>(at)].push_back(
        Event{Event::Kind::Recv, from, chunk, 0});
  }
  // A transfer whose send and receive both belong to the same pass.
  void transfer(int from, int to, std::uint32_t chunk, std::uint32_t group = 0) {
    send(from, to, chunk, group);
    recv(to, from, chunk);
  }

  Schedule seal(std::vector<ChunkSpec> chunks,
                RootPrologue prologue = RootPrologue::None) {
    Schedule s;
    s.n_ranks = n_;
    s.root = root_;
    s.message_bytes = bytes_;
    s.prologue = prologue;
    s.chunks = std::move(chunks);
    s.per_rank_ops.resize(static_cast<std::size_t>(n_));
    const auto actual = [this](int logical) { return (logical + root_) % n_; };
    for (int l = 0; l < n_; ++l) {
      auto& list = ops_[static_cast<std::size_t>(l)];
      for (Event& e : list) e.peer = actual(e.peer);
      s.per_rank_ops[static_cast<std::size_t>(actual(l))] = std::move(list);
    }
    return s;
  }

 private:
  int n_, root_;
  std::uint64_t bytes_;
  std::vector<std::vector<Event>> ops_;
};

std::vector<ChunkSpec> single_chunk(std::uint64_t m) {
  return make_chunks(m, std::max<std::uint64_t>(m, 1));
}

// Near-equal partitions, the first (M mod n) one byte longer
// (partition_chunks, schedules.cpp:53-66).
std::vector<ChunkSpec> near_equal_partitions(int n, std::uint64_t m) {
  const std::uint64_t parts = static_cast<std::uint64_t>(n);
  std::vector<ChunkSpec> v(parts);
  std::uint64_t at = 0;
  for (std::uint64_t i = 0; i < parts; ++i) {
    const std::uint64_t len = m / parts + (i < m % parts ? 1 : 0);
    v[i] = ChunkSpec{static_cast<std::uint32_t>(i), at, len};
    at += len;
  }
  return v;
}

std::int64_t ipow(int base, int e) {
  std::int64_t v = 1;
  while (e-- > 0) v *= base;
  return v;
}

// k-nomial tree over logical ranks (knomial_logical_ops, schedules.cpp:73-111):
// a rank's lowest nonzero base-k digit names its parent (digit cleared) and
// bounds the digit positions it fans out over, highest position first; a
// multi-child fan-out shares one group id.
void knomial_tree(Plan& plan, int n, int k) {
  const int depth = ceil_log(k, n);
  std::vector<std::uint32_t> group(static_cast<std::size_t>(n), 1);
  std::vector<std::vector<Event>> unused;
  for (int r = 0; r < n; ++r) {
    int fan_positions = depth;
    if (r != 0) {
      int pos = 0;
      while (r % ipow(k, pos + 1) == 0) ++pos;
      const std::int64_t unit = ipow(k, pos);
      const int parent = r - static_cast<int>(((r / unit) % k) * unit);
      plan.recv(r, parent, 0);
      fan_positions = pos;
    }
    for (int pos = fan_positions - 1; pos >= 0; --pos) {
      const std::int64_t unit = ipow(k, pos);
      std::vector<int> kids;
      for (int d = 1; d < k; ++d) {
        if (r + d * unit < n) kids.push_back(static_cast<int>(r + d * unit));
      }
      if (kids.empty()) continue;
      const std::uint32_t g =
          kids.size() > 1 ? group[static_cast<std::size_t>(r)]++ : 0;
      for (int kid : kids) plan.send(r, kid, 0, g);
    }
  }
}

}  // namespace

std::string_view algorithm_name(Algorithm a) {
  return kNames.at(static_cast<std::size_t>(a));
}

std::optional<Algorithm> algorithm_from_name(std::string_view name) {
  const auto it = std::find(kNames.begin(), kNames.end(), name);
  if (it == kNames.end()) return std::nullopt;
  return static_cast<Algorithm>(it - kNames.begin());
}

bool algorithm_uses_radix(Algorithm a) {
  return a == Algorithm::Knomial || a == Algorithm::KnomialStaged;
}
bool algorithm_uses_chunk(Algorithm a) { return a == Algorithm::ChainPipelined; }

void AlgorithmConfig::validate() const {
  const std::string name(algorithm_name(algorithm));
  if (algorithm_uses_radix(algorithm) && radix_k < 2) {
    throw std::invalid_argument("radix_k must be >= 2 for " + name);
  }
  if (algorithm_uses_chunk(algorithm) && chunk_bytes == 0) {
    throw std::invalid_argument("chunk_bytes must be >= 1 for " + name);
  }
}

std::vector<ChunkSpec> make_chunks(std::uint64_t m, std::uint64_t c) {
  if (c == 0) throw std::invalid_argument("chunk_bytes must be >= 1");
  if (m == 0) return {ChunkSpec{0, 0, 0}};
  std::vector<ChunkSpec> v((m + c - 1) / c);
  for (std::size_t i = 0; i < v.size(); ++i) {
    const std::uint64_t at = static_cast<std::uint64_t>(i) * c;
    v[i] = ChunkSpec{static_cast<std::uint32_t>(i), at, std::min(c, m - at)};
  }
  return v;
}

int ceil_log(int base, std::int64_t n) {
  if (base < 2) throw std::invalid_argument("ceil_log base must be >= 2");
  if (n < 1) throw std::invalid_argument("ceil_log argument must be >= 1");
  int levels = 0;
  for (std::int64_t span = 1; span < n; span *= base) ++levels;
  return levels;
}

Schedule schedule_direct(int n, int root, std::uint64_t m) {
  check_root(n, root);
  Plan plan(n, root, m);
  for (int r = 1; r < n; ++r) plan.transfer(0, r, 0);
  return plan.seal(single_chunk(m), RootPrologue::SelfSend);
}

Schedule schedule_chain(int n, int root, std::uint64_t m) {
  check_root(n, root);
  Plan plan(n, root, m);
  for (int r = 1; r < n; ++r) plan.transfer(r - 1, r, 0);
  return plan.seal(single_chunk(m));
}

Schedule schedule_knomial(int n, int radix_k, int root, std::uint64_t m) {
  check_root(n, root);
  if (radix_k < 2) throw std::invalid_argument("radix must be >= 2");
  Plan plan(n, root, m);
  knomial_tree(plan, n, radix_k);
  return plan.seal(single_chunk(m));
}

Schedule schedule_knomial_staged(int n, int radix_k, int root,
                                 std::uint64_t m) {
  Schedule s = schedule_knomial(n, radix_k, root, m);
  s.prologue = RootPrologue::HostStaging;
  return s;
}

Schedule schedule_chain_pipelined(int n, int root, std::uint64_t m,
                                  std::uint64_t chunk_bytes) {
  check_root(n, root);
  if (n < 2) throw std::invalid_argument("pipelined chain needs at least 2 ranks");
  std::vector<ChunkSpec> chunks = make_chunks(m, chunk_bytes);
  const auto count = static_cast<std::uint32_t>(chunks.size());
  Plan plan(n, root, m);
  // Head streams every chunk; each interior rank forwards chunk c right after
  // receiving it (store-and-forward); the tail only receives.
  for (std::uint32_t c = 0; c < count; ++c) plan.send(0, 1, c);
  for (int r = 1; r < n; ++r) {
    for (std::uint32_t c = 0; c < count; ++c) {
      plan.recv(r, r - 1, c);
      if (r + 1 < n) plan.send(r, r + 1, c);
    }
  }
  return plan.seal(std::move(chunks));
}

Schedule schedule_scatter_ring_allgather(int n, int root, std::uint64_t m) {
  check_root(n, root);
  Plan plan(n, root, m);
  // held[r][p]: logical rank r obtains partition p during the scatter.
  std::vector<std::vector<char>> held(static_cast<std::size_t>(n),
                                      std::vector<char>(static_cast<std::size_t>(n), 0));
  std::fill(held[0].begin(), held[0].end(), 1);
  std::vector<std::uint32_t> group(static_cast<std::size_t>(n), 1);
  // Range-halving scatter, breadth-first over the pending ranges: the owner
  // of [lo, hi) hands [mid, hi) to mid and keeps halving its own part.
  std::vector<std::pair<int, int>> pending{{0, n}};
  for (std::size_t head = 0; head < pending.size(); ++head) {
    int lo = pending[head].first;
    int hi = pending[head].second;
    while (hi - lo > 1) {
      const int mid = lo + (hi - lo + 1) / 2;
      const std::uint32_t g = hi - mid > 1 ? group[static_cast<std::size_t>(lo)]++ : 0;
      for (int p = mid; p < hi; ++p) {
        plan.transfer(lo, mid, static_cast<std::uint32_t>(p), g);
        held[static_cast<std::size_t>(mid)][static_cast<std::size_t>(p)] = 1;
      }
      pending.emplace_back(mid, hi);
      hi = mid;
    }
  }
  // Ring allgather: at step s rank r forwards partition (r - s + 1) mod n to
  // r + 1, except into the root or where the scatter already delivered it.
  for (int step = 1; step < n; ++step) {
    for (int r = 0; r < n; ++r) {
      const int to = (r + 1) % n;
      const int part = ((r - step + 1) % n + n) % n;
      if (to == 0 || held[static_cast<std::size_t>(to)][static_cast<std::size_t>(part)]) continue;
      plan.transfer(r, to, static_cast<std::uint32_t>(part));
    }
  }
  return plan.seal(near_equal_partitions(n, m));
}

Schedule make_schedule(const AlgorithmConfig& cfg, int n, int root,
                       std::uint64_t m) {
  cfg.validate();
  switch (cfg.algorithm) {
    case Algorithm::Direct: return schedule_direct(n, root, m);
    case Algorithm::Chain: return schedule_chain(n, root, m);
    case Algorithm::Knomial: return schedule_knomial(n, cfg.radix_k, root, m);
    case Algorithm::ScatterRingAllgather: return schedule_scatter_ring_allgather(n, root, m);
    case Algorithm::ChainPipelined: return schedule_chain_pipelined(n, root, m, cfg.chunk_bytes);
    case Algorithm::KnomialStaged: return schedule_knomial_staged(n, cfg.radix_k, root, m);
  }
  throw std::invalid_argument("unknown algorithm");
}

// Invariants of core.hpp:99-107 (checked like core.cpp:96-230, same
// messages): chunk layout, structural event checks, exactly-once receipt,
// store-and-forward ownership, and one-to-one send/recv pairing.
std::optional<ScheduleViolation> validate_schedule(const Schedule& s) {
  const auto bad = [](int rank, std::size_t i, std::string what) {
    return std::optional<ScheduleViolation>(ScheduleViolation{rank, i, std::move(what)});
  };
  if (s.n_ranks < 1) return bad(-1, 0, "n_ranks must be >= 1");
  if (s.root < 0 || s.root >= s.n_ranks) return bad(-1, 0, "root out of range");
  if (s.per_rank_ops.size() != static_cast<std::size_t>(s.n_ranks)) {
    return bad(-1, 0, "per_rank_ops size does not match n_ranks");
  }
  if (s.chunks.empty()) return bad(-1, 0, "schedule has no chunks");
  const std::uint64_t first_len = s.chunks.front().length_bytes;
  std::uint64_t covered = 0;
  for (std::size_t i = 0; i < s.chunks.size(); ++i) {
    const ChunkSpec& c = s.chunks[i];
    if (c.chunk_id != i) return bad(-1, 0, "chunk ids must be dense and ordered");
    if (c.offset_bytes != covered) return bad(-1, 0, "chunks must be contiguous from offset 0");
    const bool interior = i + 1 < s.chunks.size();
    if (interior && c.length_bytes != first_len && c.length_bytes + 1 != first_len) {
      return bad(-1, 0, "interior chunks must have equal length");
    }
    covered += c.length_bytes;
  }
  if (covered != s.message_bytes) return bad(-1, 0, "chunk lengths do not cover the message");
  const std::size_t nc = s.chunks.size();
  for (int r = 0; r < s.n_ranks; ++r) {
    const auto& ops = s.per_rank_ops[static_cast<std::size_t>(r)];
    for (std::size_t i = 0; i < ops.size(); ++i) {
      const Event& e = ops[i];
      if (e.peer < 0 || e.peer >= s.n_ranks) return bad(r, i, "peer out of range");
      if (e.peer == r) return bad(r, i, "rank communicates with itself");
      if (e.chunk >= nc) return bad(r, i, "chunk id out of range");
      if (r == s.root && e.kind == Event::Kind::Recv) return bad(r, i, "root must not receive");
    }
  }
  for (int r = 0; r < s.n_ranks; ++r) {
    if (r == s.root) continue;
    const auto& ops = s.per_rank_ops[static_cast<std::size_t>(r)];
    std::vector<std::uint32_t> got(nc, 0);
    for (std::size_t i = 0; i < ops.size(); ++i) {
      if (ops[i].kind == Event::Kind::Recv && ++got[ops[i].chunk] > 1) {
        return bad(r, i, "chunk received more than once");
      }
    }
    for (std::size_t c = 0; c < nc; ++c) {
      if (got[c] != 1) return bad(r, ops.size(), "chunk " + std::to_string(c) + " never received");
    }
  }
  for (int r = 0; r < s.n_ranks; ++r) {
    std::vector<char> own(nc, r == s.root ? 1 : 0);
    const auto& ops = s.per_rank_ops[static_cast<std::size_t>(r)];
    for (std::size_t i = 0; i < ops.size(); ++i) {
      if (ops[i].kind == Event::Kind::Recv) {
        own[ops[i].chunk] = 1;
      } else if (!own[ops[i].chunk]) {
        return bad(r, i, "chunk sent before it is owned");
      }
    }
  }
  // Net count per (src, dst, chunk): +1 per send, -1 per receive.
  std::map<std::tuple<int, int, std::uint32_t>, long> net;
  for (int r = 0; r < s.n_ranks; ++r) {
    for (const Event& e : s.per_rank_ops[static_cast<std::size_t>(r)]) {
      if (e.kind == Event::Kind::Send) ++net[{r, e.peer, e.chunk}];
      else --net[{e.peer, r, e.chunk}];
    }
  }
  for (int r = 0; r < s.n_ranks; ++r) {
    const auto& ops = s.per_rank_ops[static_cast<std::size_t>(r)];
    for (std::size_t i = 0; i < ops.size(); ++i) {
      const Event& e = ops[i];
      const bool snd = e.kind == Event::Kind::Send;
      const long v = net[snd ? std::make_tuple(r, e.peer, e.chunk) : std::make_tuple(e.peer, r, e.chunk)];
      if (v != 0) return bad(r, i, v > 0 ? "send without matching receive" : "receive without matching send");
    }
  }
  return std::nullopt;
}

std::string to_text(const Schedule& s) {
  std::ostringstream out;
  for (int r = 0; r < s.n_ranks; ++r) {
    for (const Event& e : s.per_rank_ops[static_cast<std::size_t>(r)]) {
      out << r << (e.kind == Event::Kind::Send ? " send " : " recv ") << e.peer
          << ' ' << e.chunk << '\n';
    }
  }
  return out.str();
}

}  // namespace bcl
