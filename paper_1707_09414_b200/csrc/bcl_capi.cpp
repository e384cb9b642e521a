// bcl_capi.cpp — the extern "C" veneer (include/bcl.h) over bcl_core,
// bcl_tuner and bcl_comm. Exceptions never cross the boundary: each entry
// point maps them onto a status code and a thread-local message.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <system_error>

#include "../../include/bcl.h"
#include "bcl_comm.hpp"
#include "bcl_fabric.hpp"
#include "bcl_core.hpp"
#include "bcl_tuner.hpp"

struct bcl_schedule_s {
  bcl::Schedule s;
};
struct bcl_table_s {
  bcl::TuningTable t;
};
struct bcl_fabric_s {
  std::unique_ptr<bcl::DeviceFabric> f;
};
struct bcl_comm_s {
  std::shared_ptr<bcl::Group> g;
  int local{0};
};

namespace {

thread_local std::string g_error;
thread_local std::size_t g_error_line = 0;

template <typename F>
bcl_status_t guard(F&& f) {
  g_error.clear();
  g_error_line = 0;
  try {
    f();
    return BCL_OK;
  } catch (const bcl::TableParseError& e) {
    g_error = e.what();
    g_error_line = e.line();
    return BCL_ERR_TABLE_PARSE;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return BCL_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return BCL_ERR_OUT_OF_RANGE;
  } catch (const bcl::CudaError& e) {
    g_error = e.what();
    return BCL_ERR_CUDA;
  } catch (const bcl::DeviceTimeout& e) {
    g_error = e.what();
    return BCL_ERR_TIMEOUT;
  } catch (const bcl::AggregateRankError& e) {
    g_error = e.what();
    return BCL_ERR_RANKS;
  } catch (const std::system_error& e) {
    g_error = e.what();
    return BCL_ERR_SYSTEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return BCL_ERR_RUNTIME;
  } catch (...) {
    g_error = "unknown error";
    return BCL_ERR_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (p == nullptr) throw std::invalid_argument(std::string(what) + " must not be NULL");
}

bcl::AlgorithmConfig to_cfg(const bcl_config_t* c) {
  if (c->algorithm < 0 || c->algorithm >= bcl::kAlgorithmCount) {
    throw std::invalid_argument("unknown algorithm id");
  }
  return bcl::AlgorithmConfig{static_cast<bcl::Algorithm>(c->algorithm), c->radix_k, c->chunk_bytes};
}

bcl_config_t from_cfg(const bcl::AlgorithmConfig& c) {
  return bcl_config_t{static_cast<int32_t>(c.algorithm), c.radix_k, c.chunk_bytes};
}

std::vector<bcl::AlgorithmConfig> cands_of(const bcl_config_t* c, std::size_t n) {
  std::vector<bcl::AlgorithmConfig> v;
  for (std::size_t i = 0; i < n; ++i) {
    bcl::AlgorithmConfig a = to_cfg(&c[i]);
    if (a.algorithm == bcl::Algorithm::ChainPipelined) a.chunk_bytes = 0;
    v.push_back(a);
  }
  return v;
}

std::uint64_t message_bytes(std::size_t count, bcl_dtype_t dtype) {
  const std::size_t sz = bcl::dtype_size(static_cast<bcl::DataType>(dtype));
  if (count > UINT64_MAX / sz) throw std::invalid_argument("message too large");
  return static_cast<std::uint64_t>(count) * sz;
}

void copy_text(const std::string& s, char* out, std::size_t cap, std::size_t* len) {
  if (len) *len = s.size() + 1;
  if (out && cap > 0) {
    const std::size_t k = std::min(cap - 1, s.size());
    std::memcpy(out, s.data(), k);
    out[k] = '\0';
  }
}

}  // namespace

namespace {

// Orders per-rank pointers of an init_all group by local index.
std::shared_ptr<bcl::Group> group_of(const bcl_comm_t* comms, int n) {
  need(comms, "comms");
  if (n < 1) throw std::invalid_argument("rank count must be >= 1");
  for (int i = 0; i < n; ++i) need(comms[i], "comm");
  auto g = comms[0]->g;
  for (int i = 0; i < n; ++i) {
    if (comms[i]->g != g) throw std::invalid_argument("communicators belong to different groups");
  }
  if (g->local_count() != n) throw std::invalid_argument("one communicator per rank required");
  return g;
}

template <typename T>
std::vector<T> by_local(const bcl_comm_t* comms, int n, T const* vals) {
  std::vector<T> v(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) v[static_cast<std::size_t>(comms[i]->local)] = vals[i];
  return v;
}

}  // namespace

extern "C" {

const char* bcl_last_error(void) { return g_error.c_str(); }
size_t bcl_last_error_line(void) { return g_error_line; }
const char* bcl_version(void) { return "bcl 0.1 (sm_100a)"; }

bcl_status_t bcl_make_chunks(uint64_t m, uint64_t c, bcl_chunk_t* out, size_t cap, size_t* count) {
  return guard([&] {
    const auto v = bcl::make_chunks(m, c);
    if (count) *count = v.size();
    for (std::size_t i = 0; i < v.size() && i < cap && out; ++i) {
      out[i] = bcl_chunk_t{v[i].chunk_id, v[i].offset_bytes, v[i].length_bytes};
    }
  });
}

bcl_status_t bcl_schedule_create(const bcl_config_t* cfg, int n, int root, uint64_t m,
                                 bcl_schedule_t* out) {
  return guard([&] {
    need(cfg, "config");
    need(out, "out");
    auto s = std::make_unique<bcl_schedule_s>();
    s->s = bcl::make_schedule(to_cfg(cfg), n, root, m);
    *out = s.release();
  });
}

bcl_status_t bcl_schedule_destroy(bcl_schedule_t s) {
  delete s;
  return BCL_OK;
}

bcl_status_t bcl_schedule_info(bcl_schedule_t s, int* n, int* root, uint64_t* m, int* prologue,
                               size_t* n_chunks) {
  return guard([&] {
    need(s, "schedule");
    if (n) *n = s->s.n_ranks;
    if (root) *root = s->s.root;
    if (m) *m = s->s.message_bytes;
    if (prologue) *prologue = static_cast<int>(s->s.prologue);
    if (n_chunks) *n_chunks = s->s.chunks.size();
  });
}

bcl_status_t bcl_schedule_chunks(bcl_schedule_t s, bcl_chunk_t* out, size_t cap) {
  return guard([&] {
    need(s, "schedule");
    for (std::size_t i = 0; i < s->s.chunks.size() && i < cap; ++i) {
      const auto& c = s->s.chunks[i];
      out[i] = bcl_chunk_t{c.chunk_id, c.offset_bytes, c.length_bytes};
    }
  });
}

bcl_status_t bcl_schedule_rank_events(bcl_schedule_t s, int rank, bcl_event_t* out, size_t cap,
                                      size_t* count) {
  return guard([&] {
    need(s, "schedule");
    if (rank < 0 || rank >= s->s.n_ranks) throw std::invalid_argument("rank out of range");
    const auto& ops = s->s.per_rank_ops[static_cast<std::size_t>(rank)];
    if (count) *count = ops.size();
    for (std::size_t i = 0; i < ops.size() && i < cap && out; ++i) {
      out[i] = bcl_event_t{ops[i].kind == bcl::Event::Kind::Send ? 0 : 1, ops[i].peer, ops[i].chunk,
                           ops[i].group};
    }
  });
}

bcl_status_t bcl_schedule_validate(bcl_schedule_t s) {
  return guard([&] {
    need(s, "schedule");
    if (const auto v = bcl::validate_schedule(s->s)) {
      throw std::invalid_argument("rank " + std::to_string(v->rank) + " event " +
                                  std::to_string(v->event_index) + ": " + v->description);
    }
  });
}

bcl_status_t bcl_schedule_text(bcl_schedule_t s, char* out, size_t cap, size_t* len) {
  return guard([&] {
    need(s, "schedule");
    copy_text(bcl::to_text(s->s), out, cap, len);
  });
}

bcl_status_t bcl_model_cost(const bcl_config_t* cfg, int n, uint64_t m, double ts, double bw,
                            double st, double* total) {
  return guard([&] {
    need(cfg, "config");
    need(total, "total_s");
    *total = bcl::cost_for(to_cfg(cfg), n, m, bcl::NetworkParams{ts, bw, st}).total_s;
  });
}

bcl_status_t bcl_tune_analytical(const int* n_list, size_t n_count, const uint64_t* sizes,
                                 size_t n_sizes, const bcl_config_t* cands, size_t n_cands,
                                 const uint64_t* chunks, size_t n_chunks, double ts, double bw,
                                 double st, bcl_table_t* out) {
  return guard([&] {
    need(out, "out");
    auto t = std::make_unique<bcl_table_s>();
    t->t = bcl::tune(std::vector<int>(n_list, n_list + n_count),
                     std::vector<std::uint64_t>(sizes, sizes + n_sizes), cands_of(cands, n_cands),
                     std::vector<std::uint64_t>(chunks, chunks + n_chunks),
                     bcl::NetworkParams{ts, bw, st}, bcl::CostOracle::Analytical);
    *out = t.release();
  });
}

bcl_status_t bcl_model_cost_ex(const bcl_config_t* cfg, int n, uint64_t m, const bcl_network_params_t* p,
                               double* total) {
  return guard([&] {
    need(cfg, "config");
    need(p, "params");
    need(total, "total_s");
    *total = bcl::cost_for(to_cfg(cfg), n, m,
                           bcl::NetworkParams{p->startup_s, p->link_Bps, p->staging_Bps, p->call_overhead_s})
                 .total_s;
  });
}

bcl_status_t bcl_tune_analytical_ex(const int* n_list, size_t n_count, const uint64_t* sizes, size_t n_sizes,
                                    const bcl_config_t* cands, size_t n_cands, const uint64_t* chunks,
                                    size_t n_chunks, const bcl_network_params_t* p, bcl_table_t* out) {
  return guard([&] {
    need(out, "out");
    need(p, "params");
    auto t = std::make_unique<bcl_table_s>();
    t->t = bcl::tune(std::vector<int>(n_list, n_list + n_count),
                     std::vector<std::uint64_t>(sizes, sizes + n_sizes), cands_of(cands, n_cands),
                     std::vector<std::uint64_t>(chunks, chunks + n_chunks),
                     bcl::NetworkParams{p->startup_s, p->link_Bps, p->staging_Bps, p->call_overhead_s},
                     bcl::CostOracle::Analytical);
    *out = t.release();
  });
}

bcl_status_t bcl_tune_measured(const int* n_list, size_t n_count, const uint64_t* sizes,
                               size_t n_sizes, const bcl_config_t* cands, size_t n_cands,
                               const uint64_t* chunks, size_t n_chunks, bcl_cost_fn cost,
                               void* user, const char* provenance, bcl_table_t* out) {
  return guard([&] {
    need(out, "out");
    need(reinterpret_cast<const void*>(cost), "cost");
    auto t = std::make_unique<bcl_table_s>();
    t->t = bcl::tune(
        std::vector<int>(n_list, n_list + n_count), std::vector<std::uint64_t>(sizes, sizes + n_sizes),
        cands_of(cands, n_cands), std::vector<std::uint64_t>(chunks, chunks + n_chunks),
        [&](const bcl::AlgorithmConfig& c, int n, std::uint64_t m) {
          const bcl_config_t cc = from_cfg(c);
          const double v = cost(&cc, n, m, user);
          if (std::isnan(v)) throw std::runtime_error("cost function failed");
          return v;
        },
        bcl::CostOracle::Measured);
    if (provenance) t->t.provenance = provenance;
    *out = t.release();
  });
}

bcl_status_t bcl_table_load(const char* path, bcl_table_t* out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    auto t = std::make_unique<bcl_table_s>();
    t->t = bcl::load_table_file(path);
    *out = t.release();
  });
}

bcl_status_t bcl_table_load_text(const char* text, bcl_table_t* out) {
  return guard([&] {
    need(text, "text");
    need(out, "out");
    auto t = std::make_unique<bcl_table_s>();
    t->t = bcl::load_table_text(text);
    *out = t.release();
  });
}

bcl_status_t bcl_table_save(bcl_table_t t, const char* path) {
  return guard([&] {
    need(t, "table");
    need(path, "path");
    bcl::save_table_file(t->t, path);
  });
}

bcl_status_t bcl_table_save_text(bcl_table_t t, char* out, size_t cap, size_t* len) {
  return guard([&] {
    need(t, "table");
    copy_text(bcl::save_table_text(t->t), out, cap, len);
  });
}

bcl_status_t bcl_table_builtin(bcl_table_t* out) {
  return guard([&] {
    need(out, "out");
    auto t = std::make_unique<bcl_table_s>();
    t->t = bcl::builtin_table();
    *out = t.release();
  });
}

bcl_status_t bcl_table_destroy(bcl_table_t t) {
  delete t;
  return BCL_OK;
}

bcl_status_t bcl_table_info(bcl_table_t t, int* oracle, size_t* n) {
  return guard([&] {
    need(t, "table");
    if (oracle) *oracle = static_cast<int>(t->t.oracle);
    if (n) *n = t->t.entries.size();
  });
}

bcl_status_t bcl_table_entries(bcl_table_t t, bcl_table_entry_t* out, size_t cap) {
  return guard([&] {
    need(t, "table");
    for (std::size_t i = 0; i < t->t.entries.size() && i < cap; ++i) {
      const auto& e = t->t.entries[i];
      out[i] = bcl_table_entry_t{e.n, e.msg_min_bytes, e.msg_max_bytes, from_cfg(e.config),
                                 e.predicted_cost_s};
    }
  });
}

bcl_status_t bcl_table_select(bcl_table_t t, int n, uint64_t m, bcl_config_t* out) {
  return guard([&] {
    need(t, "table");
    need(out, "out");
    *out = from_cfg(bcl::select(t->t, n, m));
  });
}

bcl_status_t bcl_comm_init_all(int n, const int* devices, double timeout_s, bcl_comm_t* out) {
  return guard([&] {
    need(devices, "devices");
    need(out, "out");
    if (n < 1) throw std::invalid_argument("rank count must be >= 1");
    bcl::GroupOptions opt = bcl::GroupOptions::from_env();
    if (timeout_s > 0) opt.timeout_ns = static_cast<std::uint64_t>(timeout_s * 1e9);
    auto g = bcl::Group::create_local(std::vector<int>(devices, devices + n), opt);
    for (int r = 0; r < n; ++r) out[r] = new bcl_comm_s{g, r};
  });
}

bcl_status_t bcl_comm_init_rank(int n, int rank, int device, size_t heap_bytes, double timeout_s,
                                bcl_comm_t* out) {
  return guard([&] {
    need(out, "out");
    bcl::GroupOptions opt = bcl::GroupOptions::from_env();
    if (timeout_s > 0) opt.timeout_ns = static_cast<std::uint64_t>(timeout_s * 1e9);
    *out = new bcl_comm_s{bcl::Group::create_rank(n, rank, device, heap_bytes, opt), 0};
  });
}

bcl_status_t bcl_comm_init_all_opts(int n, const int* devices, const char* options, bcl_comm_t* out) {
  return guard([&] {
    need(devices, "devices");
    need(out, "out");
    if (n < 1) throw std::invalid_argument("rank count must be >= 1");
    bcl::GroupOptions opt = bcl::GroupOptions::from_env();
    if (options) opt.apply(options);
    auto g = bcl::Group::create_local(std::vector<int>(devices, devices + n), opt);
    for (int r = 0; r < n; ++r) out[r] = new bcl_comm_s{g, r};
  });
}

bcl_status_t bcl_comm_init_rank_opts(int n, int rank, int device, size_t heap_bytes, const char* options,
                                     bcl_comm_t* out) {
  return guard([&] {
    need(out, "out");
    bcl::GroupOptions opt = bcl::GroupOptions::from_env();
    if (options) opt.apply(options);
    *out = new bcl_comm_s{bcl::Group::create_rank(n, rank, device, heap_bytes, opt), 0};
  });
}

bcl_status_t bcl_comm_export(bcl_comm_t c, void* blob, size_t cap, size_t* len) {
  return guard([&] {
    need(c, "comm");
    const auto v = c->g->export_info();
    if (len) *len = v.size();
    if (blob && cap >= v.size()) std::memcpy(blob, v.data(), v.size());
  });
}

bcl_status_t bcl_comm_connect(bcl_comm_t c, const void* blobs, size_t blob_len) {
  return guard([&] {
    need(c, "comm");
    need(blobs, "blobs");
    std::vector<std::vector<std::uint8_t>> v;
    const auto* p = static_cast<const std::uint8_t*>(blobs);
    for (int r = 0; r < c->g->n_ranks(); ++r) v.emplace_back(p + r * blob_len, p + (r + 1) * blob_len);
    c->g->connect(v);
  });
}

bcl_status_t bcl_comm_register_export(bcl_comm_t c, void* ptr, size_t bytes, void* blob, size_t cap,
                                      size_t* len) {
  return guard([&] {
    need(c, "comm");
    const std::size_t need_bytes = c->g->register_blob_bytes();
    if (len) *len = need_bytes;
    if (blob == nullptr || need_bytes == 0) return;  // size query (no registration happens)
    if (cap < need_bytes) throw std::invalid_argument("blob buffer too small");
    const auto v = c->g->register_export(ptr, bytes);
    std::memcpy(blob, v.data(), v.size());
  });
}

bcl_status_t bcl_comm_register_connect(bcl_comm_t c, const void* blobs, size_t blob_len) {
  return guard([&] {
    need(c, "comm");
    if (!c->g->ipc()) return;
    need(blobs, "blobs");
    std::vector<std::vector<std::uint8_t>> v;
    const auto* p = static_cast<const std::uint8_t*>(blobs);
    for (int r = 0; r < c->g->n_ranks(); ++r) v.emplace_back(p + r * blob_len, p + (r + 1) * blob_len);
    c->g->register_connect(v);
  });
}

bcl_status_t bcl_comm_destroy(bcl_comm_t c) {
  delete c;
  return BCL_OK;
}

bcl_status_t bcl_comm_info(bcl_comm_t c, int* n, int* rank, int* device, int* lanes) {
  return guard([&] {
    need(c, "comm");
    if (n) *n = c->g->n_ranks();
    if (rank) *rank = c->g->local(c->local).rank;
    if (device) *device = c->g->local(c->local).device;
    if (lanes) *lanes = c->g->lanes();
  });
}

bcl_status_t bcl_comm_protocol_caps(bcl_comm_t c, uint64_t* ll_direct_max, uint64_t* ll_chain_max,
                                    uint64_t* ll128_max) {
  return guard([&] {
    need(c, "comm");
    if (ll_direct_max) *ll_direct_max = c->g->ll_direct_max();
    if (ll_chain_max) *ll_chain_max = c->g->ll_chain_max();
    if (ll128_max) *ll128_max = c->g->ll128_max();
  });
}

bcl_status_t bcl_comm_set_table(bcl_comm_t c, bcl_table_t t) {
  return guard([&] {
    need(c, "comm");
    need(t, "table");
    c->g->set_table(t->t);
  });
}

bcl_status_t bcl_comm_plan(bcl_comm_t c, const bcl_config_t* config, int root, uint64_t bytes, int* slices,
                           uint64_t* slice_bytes, uint32_t* n_chunks, int* ctas) {
  return guard([&] {
    need(c, "comm");
    need(config, "config");
    const bcl::CallPlan p = c->g->plan(to_cfg(config), root, bytes);
    if (slices) *slices = p.slices;
    if (slice_bytes) *slice_bytes = p.slice_bytes;
    if (n_chunks) *n_chunks = p.n_chunks;
    if (ctas) *ctas = p.ctas;
  });
}

bcl_status_t bcl_comm_path(bcl_comm_t c, const bcl_config_t* config, int root, uint64_t bytes, char* out,
                           size_t cap, size_t* len) {
  return guard([&] {
    need(c, "comm");
    const bcl::AlgorithmConfig cc = config ? to_cfg(config) : bcl::AlgorithmConfig{};
    copy_text(c->g->path(config ? &cc : nullptr, root, bytes), out, cap, len);
  });
}

bcl_status_t bcl_group_start(void) {
  return guard([&] { bcl::Group::group_start(); });
}

bcl_status_t bcl_group_end(void) {
  return guard([&] { bcl::Group::group_end(); });
}

bcl_status_t bcl_comm_nvls(bcl_comm_t c, int* available, char* reason, size_t cap, size_t* len) {
  return guard([&] {
    need(c, "comm");
    if (available) *available = c->g->nvls_available() ? 1 : 0;
    copy_text(c->g->nvls_reason(), reason, cap, len);
  });
}

bcl_status_t bcl_comm_set_protocol(bcl_comm_t c, int protocol) {
  return guard([&] {
    need(c, "comm");
    c->g->set_protocol(protocol);
  });
}

bcl_status_t bcl_comm_choose(bcl_comm_t c, uint64_t m, bcl_config_t* out) {
  return guard([&] {
    need(c, "comm");
    need(out, "out");
    *out = from_cfg(c->g->choose(m, nullptr));
  });
}

bcl_status_t bcl_mem_alloc(bcl_comm_t c, size_t bytes, void** ptr) {
  return guard([&] {
    need(c, "comm");
    need(ptr, "ptr");
    *ptr = c->g->mem_alloc(c->local, bytes);
  });
}

bcl_status_t bcl_mem_reset(bcl_comm_t c) {
  return guard([&] {
    need(c, "comm");
    c->g->mem_reset(c->local);
  });
}

bcl_status_t bcl_bcast(void* buf, size_t count, bcl_dtype_t dtype, int root, bcl_comm_t comm,
                       const bcl_config_t* config, void* stream) {
  return guard([&] {
    need(comm, "comm");
    const bcl::AlgorithmConfig c = config ? to_cfg(config) : bcl::AlgorithmConfig{};
    comm->g->bcast(comm->local, buf, message_bytes(count, dtype), root, config ? &c : nullptr,
                   static_cast<cudaStream_t>(stream));
  });
}

bcl_status_t bcl_bcast_host(void* host_buf, size_t count, bcl_dtype_t dtype, int root,
                            bcl_comm_t comm, const bcl_config_t* config, void* stream) {
  return guard([&] {
    need(comm, "comm");
    const bcl::AlgorithmConfig c = config ? to_cfg(config) : bcl::AlgorithmConfig{};
    comm->g->bcast_host(comm->local, host_buf, message_bytes(count, dtype), root,
                        config ? &c : nullptr, static_cast<cudaStream_t>(stream));
  });
}


bcl_status_t bcl_bcast_all(void* const* bufs, size_t count, bcl_dtype_t dtype, int root,
                           const bcl_comm_t* comms, int n, const bcl_config_t* config,
                           void* const* streams) {
  return guard([&] {
    auto g = group_of(comms, n);
    need(bufs, "bufs");
    const bcl::AlgorithmConfig c = config ? to_cfg(config) : bcl::AlgorithmConfig{};
    std::vector<cudaStream_t> ss;
    if (streams) {
      for (auto s : by_local(comms, n, streams)) ss.push_back(static_cast<cudaStream_t>(s));
    }
    g->bcast_all(by_local(comms, n, bufs), message_bytes(count, dtype), root, config ? &c : nullptr, ss);
  });
}

bcl_status_t bcl_run_bcast(int n, int root, void* const* bufs, uint64_t bytes,
                           const bcl_config_t* config, const bcl_comm_t* comms, double* wall_s) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("rank count must be >= 1");
    auto g = group_of(comms, n);
    need(bufs, "buffers");
    if (g->n_ranks() < n) throw std::invalid_argument("fabric has too few ranks");
    const bcl::AlgorithmConfig c = config ? to_cfg(config) : bcl::AlgorithmConfig{};
    const double w = g->run_bcast(by_local(comms, n, bufs), bytes, root, config ? &c : nullptr);
    if (wall_s) *wall_s = w;
  });
}

bcl_status_t bcl_run_bcast_host(int n, int root, void* const* bufs, uint64_t bytes,
                                const bcl_config_t* config, const bcl_comm_t* comms, double* wall_s) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("rank count must be >= 1");
    auto g = group_of(comms, n);
    need(bufs, "buffers");
    const bcl::AlgorithmConfig c = config ? to_cfg(config) : bcl::AlgorithmConfig{};
    const double w = g->run_bcast_host(by_local(comms, n, bufs), bytes, root, config ? &c : nullptr);
    if (wall_s) *wall_s = w;
  });
}

bcl_status_t bcl_barrier(bcl_comm_t comm, void* stream) {
  return guard([&] {
    need(comm, "comm");
    comm->g->barrier(comm->local, static_cast<cudaStream_t>(stream));
  });
}

bcl_status_t bcl_barrier_all(const bcl_comm_t* comms, int n, void* const* streams) {
  return guard([&] {
    auto g = group_of(comms, n);
    std::vector<cudaStream_t> ss;
    if (streams) {
      for (auto s : by_local(comms, n, streams)) ss.push_back(static_cast<cudaStream_t>(s));
    }
    g->barrier_all(ss);
  });
}

bcl_status_t bcl_comm_check(bcl_comm_t comm, void* stream) {
  return guard([&] {
    need(comm, "comm");
    comm->g->check(comm->local, static_cast<cudaStream_t>(stream));
  });
}

bcl_status_t bcl_comm_set_provenance(bcl_comm_t comm, unsigned long long* counters) {
  return guard([&] {
    need(comm, "comm");
    comm->g->set_provenance(comm->local, counters);
  });
}

bcl_status_t bcl_comm_set_trace(bcl_comm_t comm, unsigned long long* records, uint32_t per_lane) {
  return guard([&] {
    need(comm, "comm");
    comm->g->set_trace(comm->local, records, per_lane);
  });
}

bcl_status_t bcl_comm_launches(bcl_comm_t comm, uint64_t* launches) {
  return guard([&] {
    need(comm, "comm");
    need(launches, "launches");
    *launches = comm->g->launches(comm->local);
  });
}

bcl_status_t bcl_fabric_create(int n, const int* devices, bcl_fabric_t* out) {
  return guard([&] {
    need(devices, "devices");
    need(out, "out");
    if (n < 1) throw std::invalid_argument("rank count must be >= 1");
    auto f = std::make_unique<bcl_fabric_s>();
    f->f = std::make_unique<bcl::DeviceFabric>(std::vector<int>(devices, devices + n));
    *out = f.release();
  });
}

bcl_status_t bcl_fabric_destroy(bcl_fabric_t f) {
  delete f;
  return BCL_OK;
}

bcl_status_t bcl_fabric_n_ranks(bcl_fabric_t f, int* n) {
  return guard([&] {
    need(f, "fabric");
    need(n, "n");
    *n = f->f->n_ranks();
  });
}

bcl_status_t bcl_fabric_send(bcl_fabric_t f, int src, int dst, uint32_t chunk, const void* data, size_t len) {
  return guard([&] {
    need(f, "fabric");
    if (len) need(data, "data");
    f->f->send(src, dst, chunk, static_cast<const std::uint8_t*>(data), len);
  });
}

bcl_status_t bcl_fabric_recv_size(bcl_fabric_t f, int dst, int src, uint32_t chunk, size_t* len) {
  return guard([&] {
    need(f, "fabric");
    need(len, "len");
    *len = f->f->recv_size(dst, src, chunk);
  });
}

bcl_status_t bcl_fabric_recv(bcl_fabric_t f, int dst, int src, uint32_t chunk, void* out, size_t len) {
  return guard([&] {
    need(f, "fabric");
    if (len) need(out, "out");
    f->f->recv(dst, src, chunk, static_cast<std::uint8_t*>(out), len);
  });
}

bcl_status_t bcl_fabric_stats(bcl_fabric_t f, int src, int dst, uint64_t* messages, uint64_t* bytes) {
  return guard([&] {
    need(f, "fabric");
    f->f->stats(src, dst, messages, bytes);
  });
}

}  // extern "C"
