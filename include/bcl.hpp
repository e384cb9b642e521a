// bcl.hpp — header-only C++ veneer over the bcl C-ABI (include/bcl.h).
//
// For hosts written against the reference's C++ API (bcastlab): the same
// vocabulary (make_chunks, make_schedule, select, load_table, save_table,
// tune, run_bcast) and the same exception classes, rethrown from the C
// status codes, so reference-style tests keep their CHECK_THROWS_AS
// semantics (std::invalid_argument, std::out_of_range, TableParseError with
// line(), AggregateRankError). Only the C-ABI crosses the library boundary.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bcl.h"

namespace bcl_b200 {

class TableParseError : public std::runtime_error {  // tuner.hpp:76-83
 public:
  TableParseError(std::size_t line, const std::string& what) : std::runtime_error(what), line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};
class CudaError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class DeviceTimeout : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class AggregateRankError : public std::runtime_error {  // runtime.hpp:56-63
  using std::runtime_error::runtime_error;
};

inline void check(bcl_status_t s) {
  if (s == BCL_OK) return;
  const std::string msg = bcl_last_error();
  switch (s) {
    case BCL_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case BCL_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case BCL_ERR_TABLE_PARSE: throw TableParseError(bcl_last_error_line(), msg);
    case BCL_ERR_CUDA: throw CudaError(msg);
    case BCL_ERR_TIMEOUT: throw DeviceTimeout(msg);
    case BCL_ERR_RANKS: throw AggregateRankError(msg);
    default: throw std::runtime_error(msg);
  }
}

using Config = bcl_config_t;
inline Config chain_pipelined(std::uint64_t chunk) { return Config{BCL_CHAIN_PIPELINED, 0, chunk}; }
inline Config knomial(int radix) { return Config{BCL_KNOMIAL, radix, 0}; }
inline Config scatter_ring_allgather() { return Config{BCL_SCATTER_RING_ALLGATHER, 0, 0}; }
inline Config chain() { return Config{BCL_CHAIN, 0, 0}; }
inline Config direct() { return Config{BCL_DIRECT, 0, 0}; }

inline std::vector<bcl_chunk_t> make_chunks(std::uint64_t message_bytes, std::uint64_t chunk_bytes) {
  std::size_t n = 0;
  check(bcl_make_chunks(message_bytes, chunk_bytes, nullptr, 0, &n));
  std::vector<bcl_chunk_t> v(n);
  check(bcl_make_chunks(message_bytes, chunk_bytes, v.data(), n, &n));
  return v;
}

class Schedule {
 public:
  Schedule(const Config& c, int n, int root, std::uint64_t message_bytes) {
    bcl_schedule_t s = nullptr;
    check(bcl_schedule_create(&c, n, root, message_bytes, &s));
    h_.reset(s);
  }
  std::vector<bcl_chunk_t> chunks() const {
    std::size_t k = 0;
    check(bcl_schedule_info(h_.get(), nullptr, nullptr, nullptr, nullptr, &k));
    std::vector<bcl_chunk_t> v(k);
    check(bcl_schedule_chunks(h_.get(), v.data(), k));
    return v;
  }
  std::vector<bcl_event_t> rank_events(int rank) const {
    std::size_t k = 0;
    check(bcl_schedule_rank_events(h_.get(), rank, nullptr, 0, &k));
    std::vector<bcl_event_t> v(k);
    check(bcl_schedule_rank_events(h_.get(), rank, v.data(), k, &k));
    return v;
  }
  std::string text() const {
    std::size_t len = 0;
    check(bcl_schedule_text(h_.get(), nullptr, 0, &len));
    std::string s(len, '\0');
    check(bcl_schedule_text(h_.get(), s.data(), len, &len));
    s.resize(len ? len - 1 : 0);
    return s;
  }
  void validate() const { check(bcl_schedule_validate(h_.get())); }

 private:
  struct Del {
    void operator()(bcl_schedule_t s) const { bcl_schedule_destroy(s); }
  };
  std::unique_ptr<bcl_schedule_s, Del> h_;
};

class Table {
 public:
  explicit Table(bcl_table_t t) : h_(t) {}
  static Table load(const std::string& path) {
    bcl_table_t t = nullptr;
    check(bcl_table_load(path.c_str(), &t));
    return Table(t);
  }
  static Table load_text(const std::string& text) {
    bcl_table_t t = nullptr;
    check(bcl_table_load_text(text.c_str(), &t));
    return Table(t);
  }
  static Table builtin() {
    bcl_table_t t = nullptr;
    check(bcl_table_builtin(&t));
    return Table(t);
  }
  static Table tune(const std::vector<int>& n_list, const std::vector<std::uint64_t>& sizes,
                    const std::vector<Config>& candidates, const std::vector<std::uint64_t>& chunks,
                    double startup_s = 1e-6, double link_Bps = 1e9, double staging_Bps = 1e10) {
    bcl_table_t t = nullptr;
    check(bcl_tune_analytical(n_list.data(), n_list.size(), sizes.data(), sizes.size(), candidates.data(),
                              candidates.size(), chunks.data(), chunks.size(), startup_s, link_Bps, staging_Bps,
                              &t));
    return Table(t);
  }
  Config select(int n, std::uint64_t message_bytes) const {
    Config c{};
    check(bcl_table_select(h_.get(), n, message_bytes, &c));
    return c;
  }
  std::string text() const {
    std::size_t len = 0;
    check(bcl_table_save_text(h_.get(), nullptr, 0, &len));
    std::string s(len, '\0');
    check(bcl_table_save_text(h_.get(), s.data(), len, &len));
    s.resize(len ? len - 1 : 0);
    return s;
  }
  void save(const std::string& path) const { check(bcl_table_save(h_.get(), path.c_str())); }
  bcl_table_t get() const { return h_.get(); }

 private:
  struct Del {
    void operator()(bcl_table_t t) const { bcl_table_destroy(t); }
  };
  std::unique_ptr<bcl_table_s, Del> h_;
};

// One process drives every rank (the reference's launch_ranks shape).
class LocalGroup {
 public:
  explicit LocalGroup(const std::vector<int>& devices, double timeout_s = 0) : comms_(devices.size()) {
    check(bcl_comm_init_all(static_cast<int>(devices.size()), devices.data(), timeout_s, comms_.data()));
  }
  ~LocalGroup() {
    for (bcl_comm_t c : comms_) bcl_comm_destroy(c);
  }
  LocalGroup(const LocalGroup&) = delete;
  LocalGroup& operator=(const LocalGroup&) = delete;
  int size() const { return static_cast<int>(comms_.size()); }
  bcl_comm_t rank(int r) const { return comms_.at(static_cast<std::size_t>(r)); }
  void set_table(const Table& t) {
    for (bcl_comm_t c : comms_) check(bcl_comm_set_table(c, t.get()));
  }
  // Transport (B200 only): 0 auto, 1 pull, 2 push, 3 LL, 4 LL128, 5 NVLS multicast.
  void set_protocol(int protocol) {
    for (bcl_comm_t c : comms_) check(bcl_comm_set_protocol(c, protocol));
  }
  // Whether the group has an NVLS multicast team (ranks on >= 2 GPUs with
  // multicast support); `why` receives the reason when it has none.
  bool nvls(std::string* why = nullptr) const {
    int ok = 0;
    std::size_t len = 0;
    check(bcl_comm_nvls(comms_.front(), &ok, nullptr, 0, &len));
    if (why != nullptr) {
      std::string s(len, '\0');
      check(bcl_comm_nvls(comms_.front(), &ok, s.data(), len, &len));
      s.resize(len ? len - 1 : 0);
      *why = s;
    }
    return ok != 0;
  }
  // run_bcast (runtime.hpp:140-143) over device buffers; wall seconds.
  double run_bcast(int root, const std::vector<void*>& device_bufs, std::uint64_t bytes,
                   const Config* config = nullptr) {
    double w = 0;
    check(bcl_run_bcast(size(), root, device_bufs.data(), bytes, config, comms_.data(), &w));
    return w;
  }
  // run_bcast over host buffers (the reference's spans live in host memory).
  double run_bcast_host(int root, const std::vector<void*>& host_bufs, std::uint64_t bytes,
                        const Config* config = nullptr) {
    double w = 0;
    check(bcl_run_bcast_host(size(), root, host_bufs.data(), bytes, config, comms_.data(), &w));
    return w;
  }

 private:
  std::vector<bcl_comm_t> comms_;
};

// Group fusion (bcl_group_start/end): broadcasts issued while a Group object
// lives are deferred and fused when the outermost one ends (end() reports
// errors; the destructor ends an un-ended group and swallows them).
class Group {
 public:
  Group() { check(bcl_group_start()); }
  ~Group() {
    if (open_) bcl_group_end();
  }
  Group(const Group&) = delete;
  Group& operator=(const Group&) = delete;
  void end() {
    open_ = false;
    check(bcl_group_end());
  }

 private:
  bool open_{true};
};

// MPI_Bcast-shaped per-rank call: bcast(buf, count, dtype, root, comm).
inline void bcast(void* buf, std::size_t count, bcl_dtype_t dtype, int root, bcl_comm_t comm,
                  const Config* config = nullptr, void* stream = nullptr) {
  check(bcl_bcast(buf, count, dtype, root, comm, config, stream));
}

}  // namespace bcl_b200
