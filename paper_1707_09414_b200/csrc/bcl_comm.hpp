// bcl_comm: the B200 replacement of the reference's TransportFabric /
// run_bcast / execute_rank boundary (proj/include/bcastlab/runtime.hpp:20-143).
//
//   Group         owns the device state of the ranks this process drives:
//                 per-rank flag/ack/mailbox region (with the device-side call
//                 state: epochs advance on the device, so captured CUDA graphs
//                 replay correctly), the peer table and host-mapped error
//                 records. Two ways to build one:
//                 * create_local(devices): one process drives every rank, one
//                   rank per entry of `devices` (UVA + peer access; several
//                   ranks may share a GPU — they then run in one launch);
//                 * create_rank(n, rank, device, heap): one process per GPU;
//                   export_info()/connect() swap CUDA IPC handles (the caller
//                   moves the bytes, e.g. with torch.distributed).
//   bcast()       per-rank MPI_Bcast-shaped call, enqueued on a stream.
//   bcast_all()   every local rank, one launch per GPU (required when ranks
//                 share a GPU: waiting kernels must be co-resident).
//   run_bcast()   synchronous all-ranks call with wall time, the mirror of
//                 run_bcast (runtime.cpp:66-103); run_bcast_host() takes host
//                 buffers (H2D at the root, D2H at the others).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "bcl_core.hpp"
#include "bcl_device.cuh"
#include "bcl_nvls.hpp"
#include "bcl_tuner.hpp"

namespace bcl {

enum class DataType : int {
  Int8 = 0, Uint8, Int32, Uint32, Int64, Uint64, Float16, Float32, Float64, Bfloat16,
};
std::size_t dtype_size(DataType t);

class CudaError : public std::runtime_error {
 public:
  CudaError(cudaError_t e, const std::string& where);
  cudaError_t code() const { return code_; }

 private:
  cudaError_t code_;
};

class DeviceTimeout : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct RankFailure {
  int rank{};
  std::string message;
};

// Mirrors AggregateRankError (runtime.hpp:51-63).
class AggregateRankError : public std::runtime_error {
 public:
  explicit AggregateRankError(std::vector<RankFailure> failures);
  const std::vector<RankFailure>& failures() const { return failures_; }

 private:
  std::vector<RankFailure> failures_;
};

struct GroupOptions {
  std::uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;  // device spin bound
  std::uint64_t window_bytes = 0;                           // bytes in flight per rank (chunks x slices);
                                                            // 0 = auto (4 MiB across GPUs, 32 MiB on one GPU)
  std::uint64_t min_slice = 2048;                           // smallest per-lane slice of a chunk
  int max_ctas_per_rank = 0;                                // 0 = SM count
  std::uint32_t poll_ns = 64;                               // back-off between flag polls (ns)
  bool strict_sys = true;                                   // the publisher releases every flag batch with a
                                                            // system-scope fence (the PTX-model release; free at
                                                            // n = 2, where no rank forwards; and LL128, the n >= 3
                                                            // default, needs no fence). 0: the copy warps' gpu-scope
                                                            // writer fence instead (a hardware property, ~1.5x
                                                            // faster for pull at n = 4)
  int sys_scope = -1;                                       // flag polls/fences at system scope: -1 auto (ranks
                                                            // span GPUs), 1 always (runs the cross-GPU code on one GPU)
  bool eager_post = true;                                   // bulk chain: forward a chunk once its store is done
  int writer_fence = 1;                                     // copy warps fence their own data before the hand-off:
                                                            // 0 no (the publisher fences), 1 gpu scope, 2 the call's
                                                            // scope (system across GPUs; 2.6x slower at n = 4, the
                                                            // fence waits for the warp's in-flight TMA pulls)
  int ll128_ctas = 0;                                       // LL128 CTAs per rank cap (0 = 3 per SM; identical on
                                                            // every rank)
  bool ll128_coop = true;                                   // LL128 with one rank per GPU: cooperative launch
  int ll128 = -1;                                           // LL128 chain lines: -1 auto (every rank on its own
                                                            // GPU), 0 off, 1 also for ranks sharing a GPU
  bool local_fused = true;                                  // single-GPU groups: fused flag-free chain kernel
  int local_ctas = 0;                                       // its grid (0 = all resident CTAs)
  std::uint64_t local_item = 0;                             // its per-warp item bytes (0 = auto)
  int local_claim = 1;                                      // its items: 1 claimed dynamically (46.3 vs 49.6 us,
                                                            // config 1), 0 static round robin
  bool ll = true;                                           // LL push protocol for small `direct` calls
  std::uint64_t ll128_direct_min = 128ull << 10;            // `direct` calls from this size up to the LL threshold
                                                            // travel as 128-byte LL128 lines (every rank on its own
                                                            // GPU; 0 = never, no landing areas for them either):
                                                            // n = 4, 8 back to back, 1 MiB: 11.4 vs 15.4 us
  int ll128_direct_ctas = 0;                                // its CTAs per rank cap (0 = one per SM: n = 2, 1 MiB,
                                                            // 8 back to back 7.9 vs 8.4 us with 64)
  int protocol = 0;                                         // chain: 0 auto (table), 1 pull, 2 push
  std::uint64_t ll_max_bytes = 0;                           // LL threshold (0 = 2 MiB, lowered for many ranks)
  std::int64_t ll_chain_max_bytes = -1;                     // LL pipelined chain up to this size (-1 = default)
  std::int64_t ll128_max_bytes = -1;                        // LL128 pipelined chain up to this size (-1 = no limit
                                                            // beyond the table's rule; 0 = off)
  std::uint64_t host_piece = 16ull << 20;                   // host-buffer calls: H2D/bcast/D2H pipeline piece
                                                            // (config 1 e2e: 4.78 ms vs 5.25 ms with 4 MiB)
  std::int64_t stage_bytes = -1;                            // bulk-copy stage per warp: 0 = vector loads,
                                                            // -1 = auto (8 KiB across GPUs, 0 on one GPU)
  std::uint32_t stages = 2;                                 // bulk-copy stages per copy warp
  int nvls = -1;                                            // NVLS multicast: -1 auto (ranks on >= 2 GPUs with
                                                            // multicast support), 0 off, 1 required
  bool nvls_strict = false;                                 // system-scope fence before every NVLS counter bump
  std::uint32_t nvls_slot = 0;                              // NVLS ring slot bytes (0 = 256 KiB; power of two,
                                                            // 16 KiB .. 8 MiB; identical on every rank)
  int nvls_ctas = 0;                                        // NVLS pieces per wave / CTAs per rank (0 = 148)
  std::uint64_t nvls_ll_max = 2ull << 20;                   // NVLS messages up to this size travel as multicast
                                                            // LL lines (0 = never; at most 2 MiB)
  static GroupOptions from_env();                           // BCL_* overrides (tuning runs)
  // "key=value,key=value" with the BCL_* names in lower case (e.g.
  // "stage_bytes=8192,sys_scope=1,protocol=2"); applied over *this.
  void apply(const std::string& options);
};

// What one call does on the device, derived identically on every rank.
struct CallPlan {
  AlgorithmConfig config;
  std::uint32_t chunk_mode{};
  std::uint32_t n_chunks{};
  std::uint64_t chunk_bytes{};
  int slices{};                 // Q
  std::uint64_t slice_bytes{};
  int ctas{};                   // CTAs per rank actually launched
  bool implicit_chain{};
  std::vector<std::vector<std::uint64_t>> events;  // [rank] packed (explicit only)
};

struct LocalRank {
  int rank{-1};
  int device{-1};
  std::uint64_t* region{};      // flags | acks | mbox | bar
  std::size_t region_bytes{};
  dev::PeerTable* d_peers{};
  dev::PeerTable h_peers{};
  dev::ErrorRecord* err_host{};
  dev::ErrorRecord* err_dev{};
  std::uint64_t epoch{0};        // host call count (local-rank lockstep check; kernels use the device CallState)
  std::uint8_t* heap{};
  std::size_t heap_bytes{};
  std::size_t heap_used{};
  std::uint8_t* scratch{};      // device staging for host-buffer calls
  std::size_t scratch_bytes{};
  cudaStream_t stream{};        // internal stream for run_bcast
  cudaStream_t copy_in{};       // host-buffer calls: H2D stream
  cudaStream_t copy_out{};      // host-buffer calls: D2H stream
  cudaStream_t host_mid{};      // run_bcast_host: broadcast stream (non-blocking)
  std::vector<cudaEvent_t> events;
  unsigned long long* prov{};   // optional provenance counters
  unsigned long long* trace{};  // optional per-lane event timestamps
  std::uint32_t trace_cap{0};
  std::uint64_t launches{0};
  std::vector<void*> opened;    // IPC mappings to close
  // Per-process mode: allocations registered for zero-copy broadcasts
  // (bcl_comm_register_*), id = index; peers' bases as mapped here.
  struct Registration {
    std::uint8_t* base{};
    std::size_t size{};
  };
  std::vector<Registration> regs;
  std::vector<std::uint64_t> h_regs;  // [peer][kMaxRegs]
  std::uint64_t* d_regs{};
};

class Group {
 public:
  static std::shared_ptr<Group> create_local(const std::vector<int>& devices,
                                             const GroupOptions& opt = {});
  static std::shared_ptr<Group> create_rank(int n, int rank, int device,
                                            std::size_t heap_bytes,
                                            const GroupOptions& opt = {});
  ~Group();

  // Multi-process wiring (create_rank only).
  std::vector<std::uint8_t> export_info() const;
  void connect(const std::vector<std::vector<std::uint8_t>>& infos);
  // Buffer registration (per-process ranks; collective, same order on every
  // rank): the device allocation holding [ptr, ptr + bytes) is exported with
  // CUDA IPC; after register_connect with every rank's blob, broadcasts on
  // buffers inside it read and write peers' memory directly (zero copy).
  // One-process groups need no registration (UVA): export returns an empty
  // blob and connect is a no-op.
  std::vector<std::uint8_t> register_export(void* ptr, std::size_t bytes);
  void register_connect(const std::vector<std::vector<std::uint8_t>>& blobs);
  std::size_t register_blob_bytes() const;  // 0 for one-process groups

  int n_ranks() const { return n_; }
  int lanes() const { return lanes_; }
  // Line-protocol landing-area caps (bytes) and whether LL128 is available.
  std::uint64_t ll_direct_max() const { return opt_.ll ? ll_max_ : 0; }
  std::uint64_t ll_chain_max() const { return opt_.ll ? ll_chain_max_ : 0; }
  std::uint64_t ll128_max() const { return opt_.ll && ll128_ok_ ? ll128_max_ : 0; }
  bool ipc() const { return ipc_; }
  int local_count() const { return static_cast<int>(local_.size()); }
  LocalRank& local(int i) { return local_.at(static_cast<std::size_t>(i)); }
  int local_index_of(int rank) const;

  void set_table(const TuningTable& t);
  void set_protocol(int protocol);  // 0 auto (LL128/LL chain, then the table's push-from rule), 1 pull, 2 push, 3 LL,
                                    // 4 LL128, 5 NVLS multicast (any schedule)
  // NVLS multicast availability (agreed by every rank) and, if unavailable, why.
  bool nvls_available() const { return nvls_ != nullptr; }
  const std::string& nvls_reason() const { return nvls_why_; }
  void clear_table();
  const TuningTable& table() const;
  AlgorithmConfig choose(std::uint64_t bytes, const AlgorithmConfig* cfg) const;
  CallPlan plan(const AlgorithmConfig& cfg, int root, std::uint64_t bytes) { return *plan_ptr(cfg, root, bytes); }
  // The cached plan itself (shared: a call neither copies its event lists nor
  // outlives it if connect() clears the cache).
  std::shared_ptr<const CallPlan> plan_ptr(const AlgorithmConfig& cfg, int root, std::uint64_t bytes);
  // Name of the device path (kernel/protocol) a call of this shape runs.
  std::string path(const AlgorithmConfig* cfg, int root, std::uint64_t bytes);

  void* mem_alloc(int local_index, std::size_t bytes);
  void mem_reset(int local_index);

  void bcast(int local_index, void* buf, std::uint64_t bytes, int root,
             const AlgorithmConfig* cfg, cudaStream_t stream);
  void bcast_all(const std::vector<void*>& bufs, std::uint64_t bytes, int root,
                 const AlgorithmConfig* cfg, const std::vector<cudaStream_t>& streams);
  void bcast_host(int local_index, void* host_buf, std::uint64_t bytes, int root,
                  const AlgorithmConfig* cfg, cudaStream_t stream);
  double run_bcast(const std::vector<void*>& bufs, std::uint64_t bytes, int root,
                   const AlgorithmConfig* cfg);
  double run_bcast_host(const std::vector<void*>& host_bufs, std::uint64_t bytes,
                        int root, const AlgorithmConfig* cfg);
  void barrier(int local_index, cudaStream_t stream);
  void barrier_all(const std::vector<cudaStream_t>& streams);
  // Synchronizes `stream` (or the device) and raises the first device error.
  void check(int local_index, cudaStream_t stream);
  // Group fusion (bcl_group_start / bcl_group_end, per thread, nestable):
  // broadcasts issued in between are deferred and fused at the end.
  static void group_start();
  static void group_end();
  static bool in_group();

  void set_provenance(int local_index, unsigned long long* counters);
  void set_trace(int local_index, unsigned long long* records, std::uint32_t per_lane);
  std::uint64_t launches(int local_index) const;

 private:
  Group() = default;
  struct Deferred {
    bool all;                           // bcast_all (every local rank) or bcast (rank li)
    int li;
    std::vector<void*> bufs;            // bcast_all: one per local rank
    std::uint64_t bytes;
    int root;
    std::shared_ptr<const CallPlan> plan;
    std::vector<cudaStream_t> streams;  // bcast_all: one per device (by_device_ order)
    int protocol;                       // set_protocol in effect at the call
  };
  bool defer(Deferred d);
  int fuse_kind(const Deferred& d);
  static int mode_of_kind(int kind) { return kind == 1 ? 0 : kind == 2 ? 3 : kind == 3 ? 1 : 2; }
  void flush_deferred();
  std::vector<Deferred> deferred_;
  void alloc_rank(LocalRank& r, std::size_t heap_bytes);
  void upload_peers(LocalRank& r);
  void cache_device_limits(int device);
  void fill_rank_work(dev::RankWork& w, LocalRank& r, const CallPlan& p, void* buf, std::uint64_t bytes);
  std::uint64_t ipc_mailbox_value(const LocalRank& r, const std::uint8_t* b, std::uint64_t bytes) const;
  void launch_group(const std::vector<int>& locals, const std::vector<void*>& bufs,
                    std::uint64_t bytes, int root, const CallPlan& p, cudaStream_t stream);
  bool use_push(const CallPlan& p, std::uint64_t bytes) const;
  bool use_nvls(const CallPlan& p, std::uint64_t bytes) const;
  void launch_nvls_group(const std::vector<int>& locals, const std::vector<void*>& bufs, std::uint64_t bytes, int root,
                         cudaStream_t stream);
  void setup_nvls_ipc(const std::vector<std::vector<std::uint8_t>>& infos, const std::vector<std::uint64_t*>& regions,
                      const std::vector<std::uint64_t>& region_bytes);
  cudaEvent_t event(LocalRank& r, std::size_t i);
  void ensure_scratch(int local_index, std::uint64_t bytes);
  void launch_ll(const std::vector<int>& locals, const std::vector<void*>& bufs, std::uint64_t bytes, int root,
                 cudaStream_t stream, int mode);
  void launch_ll_segs(const std::vector<int>& locals, const std::vector<std::vector<void*>>& seg_bufs,
                      const std::vector<std::uint64_t>& seg_bytes, int root, cudaStream_t stream, int mode);
  static std::uint64_t ll_lines_of(std::uint64_t bytes, int mode);
  void raise_errors(const std::vector<int>& locals);
  int ll_chain_mode(const CallPlan& p, std::uint64_t bytes, const std::vector<int>& locals) const;
  bool use_local_chain(const CallPlan& p, const std::vector<int>& locals) const;
  void launch_local_chain(const std::vector<int>& locals, const std::vector<void*>& bufs, std::uint64_t bytes,
                          int root, const CallPlan& p, cudaStream_t stream);
  std::size_t region_stride() const { return static_cast<std::size_t>(n_) * lanes_; }
  // The rank's device-side call state (after its LL areas; local use only).
  dev::CallState* state_of(LocalRank& r) const {
    return reinterpret_cast<dev::CallState*>(r.region + ll_offset(lanes_alloc_) + ll_words());
  }
  // Offset (in 8-byte words) of the LL landing area for a flag stride of L lanes.
  std::size_t ll_offset(int lanes) const {
    const std::size_t w = 4 * static_cast<std::size_t>(n_) * lanes + 3 * static_cast<std::size_t>(n_) + 2 +
                          3 * static_cast<std::size_t>(dev::kLL128WarpsMax);  // wcredit | wseq | rseq
    return (w + 31) / 32 * 32;  // 256-byte aligned: warp stores of LL lines cover whole 128-byte lines
  }
  std::uint64_t ll_max_{dev::kLLMaxBytes};  // LL protocol threshold (bytes), direct schedule
  std::uint64_t ll_chain_max_{0};           // LL pipelined chain up to this size (0 = off)
  std::uint64_t ll128_max_{0};              // LL128 pipelined chain up to this size (0 = off; the ring is bounded)
  bool ll128_ok_{false};                    // every rank on its own GPU (LL128 needs NVLink hops)
  std::uint64_t d128_min_{0};               // LL128 direct from this size (0 = off)
  bool use_ll128_direct(const CallPlan& p, std::uint64_t bytes) const;
  std::uint32_t ll128_lines() const { return ll128_max_ > 0 ? dev::kLL128RingLines : 0; }
  // LL128 area offset from the LL base (16-byte units), 128-byte aligned given
  // a 256-byte aligned region.
  std::uint32_t ll128_area() const {
    const std::size_t units = static_cast<std::size_t>(n_) * 2 * (ll_max_ / 8) + 2 * (ll_chain_max_ / 8);
    const std::size_t base_bytes = ll_offset(lanes_) * 8 + units * 16;
    return static_cast<std::uint32_t>(units + ((128 - base_bytes % 128) % 128) / 16);
  }
  // LL128 direct landing areas [n sources][2 halves][d128_lines()] 128-byte
  // lines, behind the LL128 ring (128-byte aligned like it).
  std::uint32_t d128_lines() const {
    return d128_min_ > 0 && ll128_lines() > 0 ? static_cast<std::uint32_t>((ll_max_ + 119) / 120) : 0;
  }
  std::uint32_t d128_area() const { return ll128_area() + ll128_lines() * 8; }
  std::size_t ll_words() const {            // 8-byte words of LL landing areas per rank (+ alignment pad)
    return (static_cast<std::size_t>(n_) * 2 * (ll_max_ / 8) + 2 * (ll_chain_max_ / 8)) * 2 +
           static_cast<std::size_t>(ll128_lines()) * 16 + static_cast<std::size_t>(n_) * 2 * d128_lines() * 16 + 16;
  }

  int n_{0};
  int lanes_{0};
  int lanes_alloc_{0};
  bool ipc_{false};
  bool single_device_{false};  // every rank on one GPU: gpu-scope ordering suffices
  bool sys_{false};            // system-scope flags (ranks span GPUs, or the sys_scope=1 option)
  bool connected_{false};
  bool broken_{false};
  GroupOptions opt_;
  std::vector<LocalRank> local_;
  std::map<int, std::vector<int>> by_device_;
  TuningTable table_;
  bool have_table_{false};
  int sms_{0};                  // SM count of the first device
  int local_chain_occ_{0};      // resident local_chain_kernel CTAs per SM
  int ll128_occ_{0};            // resident ll128_kernel CTAs per SM
  int ll128_occ_shared_{0};     // the same for the kernel serving ranks that share a GPU
  int nvls_occ_{0};             // resident nvls_kernel CTAs per SM
  int nvls_ll_occ_{0};          // resident nvls_ll_kernel CTAs per SM
  unsigned long long* lc_claim_{nullptr};  // local_chain_kernel item counters [64] (device; zero between uses)
  std::uint64_t lc_launches_{0};
  std::unique_ptr<NvlsTeam> nvls_;  // multicast team (null: NVLS unavailable on this group)
  std::string nvls_why_{"not set up"};
  std::mutex plan_mu_;
  std::map<std::tuple<int, int, std::uint64_t, int, std::uint64_t>, std::shared_ptr<CallPlan>> plans_;
};

}  // namespace bcl
