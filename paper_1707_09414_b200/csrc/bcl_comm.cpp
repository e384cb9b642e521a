// bcl_comm.cpp — see bcl_comm.hpp.
#include "bcl_comm.hpp"

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <unistd.h>

namespace bcl {

namespace {

// bcl_group_start/end nesting depth and the groups with deferred calls (per thread).
thread_local int g_group_depth = 0;
thread_local std::vector<Group*> g_group_touched;

constexpr std::uint32_t kInfoMagic = 0xB200BC57u;

struct ExportInfo {
  std::uint32_t magic;
  std::int32_t n;
  std::int32_t rank;
  std::int32_t lanes;
  std::int32_t device;
  std::int32_t pid;
  std::uint64_t region_bytes;
  std::uint64_t heap_bytes;
  std::uint64_t ll_max;        // LL landing-area geometry must agree across ranks
  std::uint64_t ll_chain_max;
  std::uint64_t ll128_max;
  std::uint64_t d128_min;
  cudaUUID_t uuid;             // physical GPU identity (ordinals differ between processes)
  cudaIpcMemHandle_t region;
  cudaIpcMemHandle_t heap;
  std::int32_t nvls_cap;       // this rank can join a multicast team (option on, device support)
  std::int32_t nvls_owner;     // rank 0: the blob below carries the multicast object
  std::uint8_t nvls[NvlsTeam::kBlobBytes];
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(e, what);
}

// Restores the caller's current device on scope exit.
class DeviceScope {
 public:
  explicit DeviceScope(int dev) {
    cudaGetDevice(&saved_);
    if (dev != saved_) {
      ck(cudaSetDevice(dev), "cudaSetDevice");
      switched_ = true;
    }
  }
  ~DeviceScope() {
    if (switched_) cudaSetDevice(saved_);
  }

 private:
  int saved_{0};
  bool switched_{false};
};

std::string describe(const dev::ErrorRecord& e) {
  std::ostringstream s;
  if (e.code == 1) {
    s << "device wait timed out on rank " << e.rank << " (lane " << e.lane << ", peer " << e.peer
      << ", chunk " << e.chunk << ", observed 0x" << std::hex << e.observed << ", expected 0x"
      << e.expected << std::dec << ")";
  } else {
    s << "device error code " << e.code << " on rank " << e.rank;
  }
  return s.str();
}

std::string format_failures(const std::vector<RankFailure>& f) {
  std::ostringstream out;
  out << f.size() << " rank(s) failed:";
  for (const RankFailure& x : f) out << " [rank " << x.rank << ": " << x.message << "]";
  return out.str();
}

}  // namespace

namespace {

// One setter per option, shared by the BCL_* environment variables and the
// options string of bcl_comm_init_*_opts (key = the variable name without
// the BCL_ prefix, lower case).
void set_option(GroupOptions& o, const std::string& key, const std::string& v) {
  const char* s = v.c_str();
  auto u64 = [&] { return std::strtoull(s, nullptr, 10); };
  auto i64 = [&] { return std::strtoll(s, nullptr, 10); };
  auto i32 = [&] { return std::atoi(s); };
  if (key == "poll_ns") o.poll_ns = static_cast<std::uint32_t>(u64());
  else if (key == "window_bytes") o.window_bytes = std::max<std::uint64_t>(16, u64());
  else if (key == "min_slice") o.min_slice = std::max<std::uint64_t>(16, u64());
  else if (key == "max_ctas") o.max_ctas_per_rank = i32();
  else if (key == "strict_sys") o.strict_sys = i32() != 0;
  else if (key == "sys_scope") o.sys_scope = i32();
  else if (key == "eager_post") o.eager_post = i32() != 0;
  else if (key == "writer_fence") {
    o.writer_fence = i32();
    if (o.writer_fence < 0 || o.writer_fence > 2) throw std::invalid_argument("writer_fence must be 0, 1 or 2");
  } else if (key == "local_fused") o.local_fused = i32() != 0;
  else if (key == "local_ctas") o.local_ctas = i32();
  else if (key == "local_item") o.local_item = u64();
  else if (key == "local_claim") o.local_claim = i32();
  else if (key == "ll") o.ll = i32() != 0;
  else if (key == "ll128") o.ll128 = i32();
  else if (key == "ll128_coop") o.ll128_coop = i32() != 0;
  else if (key == "ll128_ctas") o.ll128_ctas = std::clamp(i32(), 0, dev::kLL128MaxCtas);
  else if (key == "ll128_direct_min") o.ll128_direct_min = u64();
  else if (key == "ll128_direct_ctas") o.ll128_direct_ctas = std::clamp(i32(), 0, 1024);
  else if (key == "protocol") {
    o.protocol = i32();
    if (o.protocol < 0 || o.protocol > 5) throw std::invalid_argument("protocol must be 0..5");
  } else if (key == "ll_max") o.ll_max_bytes = u64();
  else if (key == "ll_chain_max") o.ll_chain_max_bytes = i64();
  else if (key == "ll128_max") o.ll128_max_bytes = i64();
  else if (key == "host_piece") o.host_piece = std::max<std::uint64_t>(4096, u64());
  else if (key == "stages") o.stages = static_cast<std::uint32_t>(std::clamp(i32(), 2, dev::kMaxStages));
  else if (key == "stage_bytes") o.stage_bytes = i64() < 0 ? -1 : i64() / 16 * 16;
  else if (key == "nvls") o.nvls = i32();
  else if (key == "nvls_strict") o.nvls_strict = i32() != 0;
  else if (key == "nvls_slot") {
    const std::uint64_t v = u64();
    if (v < (16u << 10) || v > (8u << 20) || (v & (v - 1)) != 0) {
      throw std::invalid_argument("nvls_slot must be a power of two in [16 KiB, 8 MiB]");
    }
    o.nvls_slot = static_cast<std::uint32_t>(v);
  } else if (key == "nvls_ctas") o.nvls_ctas = std::max(1, i32());
  else if (key == "timeout_s") o.timeout_ns = static_cast<std::uint64_t>(std::strtod(s, nullptr) * 1e9);
  else throw std::invalid_argument("unknown communicator option '" + key + "'");
}

constexpr const char* kOptionNames[] = {
    "poll_ns", "window_bytes", "min_slice", "max_ctas", "strict_sys", "sys_scope", "eager_post", "writer_fence",
    "local_fused", "local_ctas", "local_item", "local_claim", "ll", "ll128", "ll128_coop", "ll128_ctas", "ll128_direct_min", "ll128_direct_ctas", "protocol", "ll_max", "ll_chain_max", "ll128_max",
    "host_piece", "stages", "stage_bytes", "nvls", "nvls_strict", "nvls_slot", "nvls_ctas", "nvls_ll_max"};

}  // namespace

GroupOptions GroupOptions::from_env() {
  GroupOptions o;
  for (const char* name : kOptionNames) {
    std::string env = "BCL_";
    for (const char* c = name; *c; ++c) env += static_cast<char>(std::toupper(static_cast<unsigned char>(*c)));
    if (const char* v = std::getenv(env.c_str())) set_option(o, name, v);
  }
  return o;
}

void GroupOptions::apply(const std::string& options) {
  std::size_t at = 0;
  while (at < options.size()) {
    std::size_t end = options.find_first_of(",; ", at);
    if (end == std::string::npos) end = options.size();
    const std::string item = options.substr(at, end - at);
    at = end + 1;
    if (item.empty()) continue;
    const std::size_t eq = item.find('=');
    if (eq == std::string::npos || eq == 0) throw std::invalid_argument("option '" + item + "' is not key=value");
    set_option(*this, item.substr(0, eq), item.substr(eq + 1));
  }
}

std::size_t dtype_size(DataType t) {
  switch (t) {
    case DataType::Int8: case DataType::Uint8: return 1;
    case DataType::Float16: case DataType::Bfloat16: return 2;
    case DataType::Int32: case DataType::Uint32: case DataType::Float32: return 4;
    case DataType::Int64: case DataType::Uint64: case DataType::Float64: return 8;
  }
  throw std::invalid_argument("unknown datatype");
}

CudaError::CudaError(cudaError_t e, const std::string& where)
    : std::runtime_error(where + ": " + cudaGetErrorString(e)), code_(e) {}

AggregateRankError::AggregateRankError(std::vector<RankFailure> failures)
    : std::runtime_error(format_failures(failures)), failures_(std::move(failures)) {}

// ----------------------------------------------------------------- creation

void Group::alloc_rank(LocalRank& r, std::size_t heap_bytes) {
  DeviceScope ds(r.device);
  // (+ the device-side call state, then 8 words whose last one is the
  // connect-time agreement word)
  r.region_bytes = (ll_offset(lanes_alloc_) + ll_words() + dev::kCallStateWords + 8) * sizeof(std::uint64_t);
  ck(cudaMalloc(&r.region, r.region_bytes), "cudaMalloc(region)");
  ck(cudaMemset(r.region, 0, r.region_bytes), "cudaMemset(region)");
  ck(cudaMalloc(&r.d_peers, sizeof(dev::PeerTable)), "cudaMalloc(peers)");
  ck(cudaHostAlloc(&r.err_host, sizeof(dev::ErrorRecord), cudaHostAllocMapped | cudaHostAllocPortable),
     "cudaHostAlloc(err)");
  std::memset(r.err_host, 0, sizeof(dev::ErrorRecord));
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&r.err_dev), r.err_host, 0),
     "cudaHostGetDevicePointer");
  // Blocking stream: ordered after work on the legacy default stream (e.g. torch
  // fills of the buffers), as the synchronous run_bcast contract expects.
  ck(cudaStreamCreateWithFlags(&r.stream, cudaStreamDefault), "cudaStreamCreate");
  ck(cudaStreamCreateWithFlags(&r.copy_in, cudaStreamNonBlocking), "cudaStreamCreate(copy_in)");
  ck(cudaStreamCreateWithFlags(&r.copy_out, cudaStreamNonBlocking), "cudaStreamCreate(copy_out)");
  ck(cudaStreamCreateWithFlags(&r.host_mid, cudaStreamNonBlocking), "cudaStreamCreate(host_mid)");
  if (heap_bytes > 0) {
    ck(cudaMalloc(&r.heap, heap_bytes), "cudaMalloc(heap)");
    r.heap_bytes = heap_bytes;
  }
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
}

void Group::cache_device_limits(int device) {
  DeviceScope ds(device);
  ck(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device), "sm count");
  ck(static_cast<cudaError_t>(local_chain_occupancy(&local_chain_occ_)), "occupancy(local chain)");
  ck(static_cast<cudaError_t>(ll128_occupancy(&ll128_occ_, 0)), "occupancy(ll128)");
  ck(static_cast<cudaError_t>(ll128_occupancy(&ll128_occ_shared_, 1)), "occupancy(ll128, shared GPU)");
  ck(static_cast<cudaError_t>(nvls_occupancy(&nvls_occ_)), "occupancy(nvls)");
  ck(static_cast<cudaError_t>(nvls_ll_occupancy(&nvls_ll_occ_)), "occupancy(nvls ll)");
}

void Group::upload_peers(LocalRank& r) {
  DeviceScope ds(r.device);
  ck(cudaMemcpy(r.d_peers, &r.h_peers, sizeof(dev::PeerTable), cudaMemcpyHostToDevice),
     "cudaMemcpy(peers)");
}

namespace {

int lanes_for(int device, int ranks_per_device, int cap, const GroupOptions& opt) {
  DeviceScope ds(device);
  int sms = 0;
  ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");
  const std::size_t smem =
      opt.stage_bytes > 0 ? bcast_smem_bytes(opt.stages, static_cast<std::uint32_t>(opt.stage_bytes)) : 0;
  int smem_max = 0;
  ck(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "smem limit");
  if (smem + 4096 > static_cast<std::size_t>(smem_max)) {
    throw std::invalid_argument("stages x stage_bytes x 8 copy warps (" + std::to_string(smem) +
                                " B) exceeds the per-CTA shared memory (" + std::to_string(smem_max) + " B)");
  }
  ck(static_cast<cudaError_t>(prepare_bcast_kernels(smem)), "cudaFuncSetAttribute(smem)");
  int occ = 0;
  ck(static_cast<cudaError_t>(bcast_kernel_occupancy(&occ, smem)), "occupancy");
  if (occ < 1) throw std::invalid_argument("stage_bytes does not fit in shared memory");
  // Default: one CTA per SM per rank (fills every SM when a rank owns the
  // GPU); ranks sharing a GPU split the co-resident CTA budget.
  const int resident = sms * std::max(occ, 1);
  int ctas = std::min(sms, std::max(1, resident / std::max(ranks_per_device, 1)));
  if (cap > 0) ctas = std::min(cap, std::max(1, resident / std::max(ranks_per_device, 1)));
  return ctas * dev::kWarpsPerCta;
}

// LL landing areas cost 4 x cap bytes per source per rank: bound them to
// 64 MiB per rank (2 MiB cap up to 8 ranks, 1 MiB up to 16).
std::uint64_t ll_cap(int n, const GroupOptions& opt) {
  std::uint64_t cap = opt.ll_max_bytes ? opt.ll_max_bytes : dev::kLLMaxBytes;
  cap = std::min<std::uint64_t>(cap, dev::kLLMaxBytes);
  while (cap > 4096 && static_cast<std::uint64_t>(n) * 4 * cap > (64ull << 20)) cap /= 2;
  return cap / 16 * 16;
}

// The chain landing area (one source: the ring predecessor) costs 4 x cap
// bytes per rank, independent of n.
std::uint64_t ll_chain_cap(const GroupOptions& opt) {
  const std::int64_t v = opt.ll_chain_max_bytes < 0 ? static_cast<std::int64_t>(dev::kLLChainMaxBytes)
                                                   : opt.ll_chain_max_bytes;
  return static_cast<std::uint64_t>(std::min<std::int64_t>(v, 64ll << 20)) / 16 * 16;
}
// LL128 size limit: the landing ring is bounded (kLL128RingLines, 58 MB per
// rank) whatever the message size, so by default only the table's measured
// rule limits LL128; ll128_max caps it further (0 turns LL128 off).
constexpr std::uint64_t kNoLimit = 1ull << 62;
std::uint64_t ll128_cap(const GroupOptions& opt) {
  return opt.ll128_max_bytes < 0 ? kNoLimit : static_cast<std::uint64_t>(opt.ll128_max_bytes);
}
// LL128 direct threshold (0 = off: no LL128 direct landing areas either).
std::uint64_t d128_cap(std::uint64_t ll_max, const GroupOptions& opt) {
  return opt.ll128_direct_min == 0 || opt.ll128_direct_min > ll_max ? 0 : opt.ll128_direct_min;
}

}  // namespace

std::shared_ptr<Group> Group::create_local(const std::vector<int>& devices, const GroupOptions& opt) {
  const int n = static_cast<int>(devices.size());
  if (n < 1) throw std::invalid_argument("rank count must be >= 1");
  if (n > dev::kMaxRanks) throw std::invalid_argument("at most 64 ranks");
  std::shared_ptr<Group> g(new Group());
  g->n_ = n;
  g->opt_ = opt;
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  for (int r = 0; r < n; ++r) {
    if (devices[static_cast<std::size_t>(r)] < 0 || devices[static_cast<std::size_t>(r)] >= ndev) {
      throw std::invalid_argument("device id out of range");
    }
    g->by_device_[devices[static_cast<std::size_t>(r)]].push_back(r);
  }
  int rpd = 0;
  for (const auto& kv : g->by_device_) rpd = std::max(rpd, static_cast<int>(kv.second.size()));
  if (rpd > dev::kMaxLocal) throw std::invalid_argument("at most 16 ranks may share one GPU");
  for (const auto& a : g->by_device_) {
    for (const auto& b : g->by_device_) {
      if (a.first == b.first) continue;
      int can = 0;
      ck(cudaDeviceCanAccessPeer(&can, a.first, b.first), "cudaDeviceCanAccessPeer");
      if (!can) throw std::runtime_error("no peer access between devices");
      DeviceScope ds(a.first);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b.first, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else {
        ck(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }
  // TMA bulk stages pay off on NVLink pulls; ranks sharing one GPU (HBM
  // bound, several CTAs per SM needed for co-residency) use vector loads.
  if (g->opt_.stage_bytes < 0) g->opt_.stage_bytes = g->by_device_.size() > 1 ? 8192 : 0;
  // NVLink hops want a small window (fast fill); ranks sharing one GPU are
  // HBM-bound and want more bytes in flight.
  if (g->opt_.window_bytes == 0) g->opt_.window_bytes = g->by_device_.size() > 1 ? (4ull << 20) : (32ull << 20);
  g->lanes_ = lanes_for(devices[0], rpd, opt.max_ctas_per_rank, g->opt_);
  for (const auto& kv : g->by_device_) {
    if (kv.first != devices[0]) lanes_for(kv.first, rpd, opt.max_ctas_per_rank, g->opt_);
  }
  g->lanes_alloc_ = g->lanes_;
  g->single_device_ = g->by_device_.size() == 1;
  g->sys_ = !g->single_device_ || opt.sys_scope == 1;
  // LL128 lines cross NVLink when every rank owns its GPU; opt.ll128 = 1 also
  // runs them through L2 between ranks sharing a GPU (one cooperative launch).
  g->ll128_ok_ = n >= 2 && opt.ll128 != 0 && (static_cast<int>(g->by_device_.size()) == n || opt.ll128 == 1);
  g->ll_max_ = ll_cap(n, opt);
  g->ll_chain_max_ = ll_chain_cap(opt);
  g->ll128_max_ = g->ll128_ok_ ? ll128_cap(opt) : 0;  // no LL128 ring without LL128
  g->ll128_ok_ = g->ll128_ok_ && g->ll128_max_ > 0;
  g->d128_min_ = d128_cap(g->ll_max_, opt);
  g->cache_device_limits(devices[0]);
  g->local_.resize(static_cast<std::size_t>(n));
  for (int r = 0; r < n; ++r) {
    LocalRank& lr = g->local_[static_cast<std::size_t>(r)];
    lr.rank = r;
    lr.device = devices[static_cast<std::size_t>(r)];
    g->alloc_rank(lr, 0);
  }
  const std::size_t S = g->region_stride();
  for (LocalRank& lr : g->local_) {
    for (int p = 0; p < n; ++p) {
      std::uint64_t* base = g->local_[static_cast<std::size_t>(p)].region;
      lr.h_peers.flags[p] = base;
      lr.h_peers.acks[p] = base + S;
      lr.h_peers.mbox[p] = base + 2 * S;
      lr.h_peers.bar[p] = base + 4 * S;
      lr.h_peers.addr_base[p] = 0;
      lr.h_peers.credit[p] = base + 4 * S + n + 1;
      lr.h_peers.wcredit[p] = base + 4 * S + 3 * n + 2;
      lr.h_peers.ll[p] = reinterpret_cast<uint4*>(base + g->ll_offset(g->lanes_));
    }
    g->upload_peers(lr);
  }
  // NVLS multicast across the group's GPUs (one team; ranks sharing a GPU
  // read that GPU's copy).
  if (opt.nvls == 0) {
    g->nvls_why_ = "disabled (nvls=0)";
  } else if (g->by_device_.size() < 2) {
    g->nvls_why_ = "every rank on one GPU (a multicast team needs two or more GPUs)";
  } else {
    std::vector<int> devs;
    for (const auto& kv : g->by_device_) devs.push_back(kv.first);
    for (int d : devs) {
      if (!NvlsTeam::supported(d, &g->nvls_why_)) devs.clear();
      if (devs.empty()) break;
    }
    if (!devs.empty()) {
      try {
        g->nvls_ = NvlsTeam::create_local(devs);
        g->nvls_why_.clear();
      } catch (const std::exception& e) {
        g->nvls_why_ = e.what();
      }
    }
  }
  if (opt.nvls == 1 && !g->nvls_) throw std::runtime_error("NVLS multicast required but unavailable: " + g->nvls_why_);
  g->connected_ = true;
  return g;
}

std::shared_ptr<Group> Group::create_rank(int n, int rank, int device, std::size_t heap_bytes,
                                          const GroupOptions& opt) {
  if (n < 1 || n > dev::kMaxRanks) throw std::invalid_argument("rank count must be in [1, 64]");
  if (rank < 0 || rank >= n) throw std::invalid_argument("rank out of range");
  std::shared_ptr<Group> g(new Group());
  g->n_ = n;
  g->opt_ = opt;
  g->ipc_ = true;
  if (g->opt_.stage_bytes < 0) g->opt_.stage_bytes = n > 1 ? 8192 : 0;
  if (g->opt_.window_bytes == 0) g->opt_.window_bytes = 4ull << 20;
  g->lanes_ = lanes_for(device, 1, opt.max_ctas_per_rank, g->opt_);
  g->lanes_alloc_ = g->lanes_;
  g->sys_ = n > 1 || opt.sys_scope == 1;
  g->ll_max_ = ll_cap(n, opt);
  g->ll_chain_max_ = ll_chain_cap(opt);
  g->ll128_max_ = opt.ll128 != 0 ? ll128_cap(opt) : 0;
  g->d128_min_ = d128_cap(g->ll_max_, opt);
  g->cache_device_limits(device);
  g->local_.resize(1);
  g->local_[0].rank = rank;
  g->local_[0].device = device;
  g->by_device_[device].push_back(0);
  g->alloc_rank(g->local_[0], heap_bytes);
  // NVLS: rank 0 creates and exports the multicast object; the others import
  // it in connect().
  if (opt.nvls == 0) {
    g->nvls_why_ = "disabled (nvls=0)";
  } else if (n < 2) {
    g->nvls_why_ = "one rank";
  } else if (NvlsTeam::supported(device, &g->nvls_why_) && rank == 0) {
    try {
      g->nvls_ = NvlsTeam::create_owner(n, device);
    } catch (const std::exception& e) {
      g->nvls_why_ = e.what();
    }
  }
  return g;
}

std::vector<std::uint8_t> Group::export_info() const {
  if (!ipc_) throw std::invalid_argument("export_info is for per-process ranks");
  const LocalRank& r = local_[0];
  DeviceScope ds(r.device);
  ExportInfo info{};
  info.magic = kInfoMagic;
  info.n = n_;
  info.rank = r.rank;
  info.lanes = lanes_alloc_;
  info.device = r.device;
  info.pid = static_cast<std::int32_t>(getpid());
  info.region_bytes = r.region_bytes;
  info.heap_bytes = r.heap_bytes;
  info.ll_max = ll_max_;
  info.ll_chain_max = ll_chain_max_;
  info.ll128_max = ll128_max_;
  info.d128_min = d128_min_;
  {
    cudaDeviceProp prop{};
    ck(cudaGetDeviceProperties(&prop, r.device), "cudaGetDeviceProperties");
    info.uuid = prop.uuid;
  }
  ck(cudaIpcGetMemHandle(&info.region, r.region), "cudaIpcGetMemHandle(region)");
  if (r.heap) ck(cudaIpcGetMemHandle(&info.heap, r.heap), "cudaIpcGetMemHandle(heap)");
  info.nvls_cap = opt_.nvls != 0 && n_ >= 2 && (r.rank != 0 || nvls_ != nullptr) &&
                  NvlsTeam::supported(r.device, nullptr);
  info.nvls_owner = r.rank == 0 && nvls_ != nullptr;
  if (info.nvls_owner) nvls_->export_blob(info.nvls);
  std::vector<std::uint8_t> out(sizeof info);
  std::memcpy(out.data(), &info, sizeof info);
  return out;
}

namespace {

constexpr std::uint32_t kRegMagic = 0xB200BC58u;
struct RegInfo {
  std::uint32_t magic;
  std::int32_t rank;
  std::int32_t id;
  std::int32_t pad;
  std::uint64_t size;
  cudaIpcMemHandle_t handle;
};

// [base, base + size) of the device allocation holding p (driver API through
// the runtime's entry-point lookup: no libcuda link dependency).
void allocation_range(const void* p, std::uint8_t** base, std::size_t* size) {
  using Fn = int (*)(unsigned long long*, std::size_t*, unsigned long long);
  static Fn fn = nullptr;
  if (fn == nullptr) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    ck(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
    if (f == nullptr || q != cudaDriverEntryPointSuccess) throw std::runtime_error("cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<Fn>(f);
  }
  unsigned long long b = 0;
  if (fn(&b, size, reinterpret_cast<unsigned long long>(p)) != 0) {
    throw std::invalid_argument("buffer is not device memory from cudaMalloc");
  }
  *base = reinterpret_cast<std::uint8_t*>(b);
}

}  // namespace

std::size_t Group::register_blob_bytes() const { return ipc_ ? sizeof(RegInfo) : 0; }

std::vector<std::uint8_t> Group::register_export(void* ptr, std::size_t bytes) {
  if (!ipc_) return {};
  if (!connected_) throw std::invalid_argument("communicator is not connected");
  if (ptr == nullptr || bytes == 0) throw std::invalid_argument("nothing to register");
  LocalRank& r = local_[0];
  if (r.regs.size() >= static_cast<std::size_t>(dev::kMaxRegs)) throw std::invalid_argument("too many registrations");
  DeviceScope ds(r.device);
  std::uint8_t* base = nullptr;
  std::size_t size = 0;
  allocation_range(ptr, &base, &size);
  if (static_cast<std::uint8_t*>(ptr) + bytes > base + size) {
    throw std::invalid_argument("registered range spans several allocations");
  }
  if (size >= (1ull << 40)) throw std::invalid_argument("allocation larger than 1 TiB");
  RegInfo info{};
  info.magic = kRegMagic;
  info.rank = r.rank;
  info.id = static_cast<std::int32_t>(r.regs.size());
  info.size = size;
  ck(cudaIpcGetMemHandle(&info.handle, base), "cudaIpcGetMemHandle(buffer)");
  r.regs.push_back(LocalRank::Registration{base, size});  // completed by register_connect
  std::vector<std::uint8_t> out(sizeof info);
  std::memcpy(out.data(), &info, sizeof info);
  return out;
}

void Group::register_connect(const std::vector<std::vector<std::uint8_t>>& blobs) {
  if (!ipc_) return;
  LocalRank& me = local_[0];
  if (static_cast<int>(blobs.size()) != n_) throw std::invalid_argument("one registration blob per rank required");
  if (me.regs.empty()) throw std::invalid_argument("register_export first");
  const int id = static_cast<int>(me.regs.size()) - 1;
  DeviceScope ds(me.device);
  if (me.d_regs == nullptr) {
    me.h_regs.assign(static_cast<std::size_t>(n_) * dev::kMaxRegs, 0);
    ck(cudaMalloc(&me.d_regs, me.h_regs.size() * sizeof(std::uint64_t)), "cudaMalloc(regs)");
  }
  for (int p = 0; p < n_; ++p) {
    RegInfo info{};
    if (blobs[static_cast<std::size_t>(p)].size() < sizeof info) throw std::invalid_argument("truncated registration blob");
    std::memcpy(&info, blobs[static_cast<std::size_t>(p)].data(), sizeof info);
    if (info.magic != kRegMagic || info.rank != p || info.id != id) {
      throw std::invalid_argument("registration blobs must be ordered by rank and belong to the same registration");
    }
    std::uint64_t mapped = reinterpret_cast<std::uint64_t>(me.regs.back().base);
    if (p != me.rank) {
      void* q = nullptr;
      ck(cudaIpcOpenMemHandle(&q, info.handle, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(buffer)");
      me.opened.push_back(q);
      mapped = reinterpret_cast<std::uint64_t>(q);
    }
    me.h_regs[static_cast<std::size_t>(p) * dev::kMaxRegs + static_cast<std::size_t>(id)] = mapped;
  }
  ck(cudaMemcpy(me.d_regs, me.h_regs.data(), me.h_regs.size() * sizeof(std::uint64_t), cudaMemcpyHostToDevice),
     "cudaMemcpy(regs)");
  me.h_peers.regs = me.d_regs;
  upload_peers(me);
}

void Group::connect(const std::vector<std::vector<std::uint8_t>>& infos) {
  if (!ipc_) throw std::invalid_argument("connect is for per-process ranks");
  if (connected_) throw std::invalid_argument("already connected");
  if (static_cast<int>(infos.size()) != n_) throw std::invalid_argument("one info blob per rank required");
  std::vector<ExportInfo> all(infos.size());
  int lanes = lanes_alloc_;
  for (std::size_t i = 0; i < infos.size(); ++i) {
    if (infos[i].size() < sizeof(ExportInfo)) throw std::invalid_argument("truncated info blob");
    std::memcpy(&all[i], infos[i].data(), sizeof(ExportInfo));
    if (all[i].magic != kInfoMagic || all[i].n != n_ || all[i].rank != static_cast<int>(i)) {
      throw std::invalid_argument("info blobs must be ordered by rank and belong to this group");
    }
    if (all[i].ll_max != ll_max_ || all[i].ll_chain_max != ll_chain_max_ || all[i].ll128_max != ll128_max_ ||
        all[i].d128_min != d128_min_) {
      throw std::invalid_argument(
          "ranks disagree on the LL landing areas (BCL_LL_MAX / _CHAIN_MAX / LL128_MAX / LL128_DIRECT_MIN)");
    }
    lanes = std::min(lanes, static_cast<int>(all[i].lanes));
  }
  lanes_ = lanes;
  {
    // Plans computed before connect (bcl_comm_plan) used this rank's own lane
    // count; every rank must plan with the group minimum.
    std::lock_guard<std::mutex> lock(plan_mu_);
    plans_.clear();
  }
  // Processes sharing a GPU run separate launches that wait on one another:
  // no LL128 (and no guarantee of co-residency either).
  ll128_ok_ = n_ >= 2 && ll128_max_ > 0;
  for (std::size_t i = 0; i < all.size(); ++i) {
    for (std::size_t j = 0; j < i; ++j) {
      if (std::memcmp(&all[i].uuid, &all[j].uuid, sizeof(cudaUUID_t)) == 0) ll128_ok_ = false;
    }
  }
  LocalRank& me = local_[0];
  DeviceScope ds(me.device);
  const std::size_t S = region_stride();
  std::vector<std::uint64_t*> regions;
  std::vector<std::uint64_t> region_bytes;
  for (int p = 0; p < n_; ++p) {
    std::uint64_t* base = nullptr;
    std::uint64_t heap_base = 0;
    if (p == me.rank) {
      base = me.region;
      heap_base = reinterpret_cast<std::uint64_t>(me.heap);
    } else {
      void* ptr = nullptr;
      ck(cudaIpcOpenMemHandle(&ptr, all[static_cast<std::size_t>(p)].region,
                              cudaIpcMemLazyEnablePeerAccess),
         "cudaIpcOpenMemHandle(region)");
      me.opened.push_back(ptr);
      base = static_cast<std::uint64_t*>(ptr);
      if (all[static_cast<std::size_t>(p)].heap_bytes > 0) {
        void* h = nullptr;
        ck(cudaIpcOpenMemHandle(&h, all[static_cast<std::size_t>(p)].heap,
                                cudaIpcMemLazyEnablePeerAccess),
           "cudaIpcOpenMemHandle(heap)");
        me.opened.push_back(h);
        heap_base = reinterpret_cast<std::uint64_t>(h);
      }
    }
    me.h_peers.flags[p] = base;
    me.h_peers.acks[p] = base + S;
    me.h_peers.mbox[p] = base + 2 * S;
    me.h_peers.bar[p] = base + 4 * S;
    me.h_peers.addr_base[p] = heap_base;
    me.h_peers.credit[p] = base + 4 * S + n_ + 1;
    me.h_peers.wcredit[p] = base + 4 * S + 3 * static_cast<std::size_t>(n_) + 2;
    me.h_peers.ll[p] = reinterpret_cast<uint4*>(base + ll_offset(lanes_));
    regions.push_back(base);
    region_bytes.push_back(all[static_cast<std::size_t>(p)].region_bytes);
  }
  upload_peers(me);
  setup_nvls_ipc(infos, regions, region_bytes);
  connected_ = true;
}

namespace {

// Connect-time agreement between per-process ranks: each rank publishes
// (phase << 1 | failed) in the last word of its region and waits until every
// rank reached the phase; returns whether every rank succeeded.
bool agree(int n, int me, int phase, bool ok, const std::vector<std::uint64_t*>& regions,
           const std::vector<std::uint64_t>& region_bytes, double timeout_s) {
  auto word = [&](int p) { return regions[static_cast<std::size_t>(p)] + region_bytes[static_cast<std::size_t>(p)] / 8 - 1; };
  const std::uint64_t mine = (static_cast<std::uint64_t>(phase) << 1) | (ok ? 0u : 1u);
  ck(cudaMemcpy(word(me), &mine, sizeof mine, cudaMemcpyHostToDevice), "cudaMemcpy(agree)");
  const auto t0 = std::chrono::steady_clock::now();
  bool all_ok = ok;
  for (int p = 0; p < n; ++p) {
    for (;;) {
      std::uint64_t v = 0;
      ck(cudaMemcpy(&v, word(p), sizeof v, cudaMemcpyDeviceToHost), "cudaMemcpy(agree)");
      if ((v >> 1) >= static_cast<std::uint64_t>(phase)) {
        if ((v >> 1) == static_cast<std::uint64_t>(phase) && (v & 1u)) all_ok = false;
        break;
      }
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
        throw std::runtime_error("connect: rank " + std::to_string(p) + " did not reach NVLS setup phase " +
                                 std::to_string(phase));
      }
      ::usleep(200);
    }
  }
  return all_ok;
}

}  // namespace

// Per-process NVLS: every rank imports rank 0's multicast object and adds its
// GPU (phase 1), then binds and maps its copy of the ring (phase 2); the
// ranks agree after each phase, so NVLS is on for all of them or for none.
void Group::setup_nvls_ipc(const std::vector<std::vector<std::uint8_t>>& infos,
                           const std::vector<std::uint64_t*>& regions, const std::vector<std::uint64_t>& region_bytes) {
  LocalRank& me = local_[0];
  std::vector<ExportInfo> all(infos.size());
  for (std::size_t i = 0; i < infos.size(); ++i) std::memcpy(&all[i], infos[i].data(), sizeof(ExportInfo));
  bool eligible = n_ >= 2 && all[0].nvls_owner != 0;
  for (std::size_t i = 0; i < all.size() && eligible; ++i) {
    if (!all[i].nvls_cap) {
      eligible = false;
      nvls_why_ = "rank " + std::to_string(i) + " cannot join a multicast team";
    }
    for (std::size_t j = 0; j < i && eligible; ++j) {
      if (std::memcmp(&all[i].uuid, &all[j].uuid, sizeof(cudaUUID_t)) == 0) {
        eligible = false;
        nvls_why_ = "ranks share a GPU (one process per GPU required for NVLS)";
      }
    }
  }
  if (n_ >= 2 && all[0].nvls_owner == 0 && nvls_why_ == "not set up") nvls_why_ = "rank 0 created no multicast object";
  if (!eligible) {  // the same verdict on every rank (computed from the same blobs)
    nvls_.reset();
    if (opt_.nvls == 1) throw std::runtime_error("NVLS multicast required but unavailable: " + nvls_why_);
    return;
  }
  bool ok = true;
  const bool dbg = std::getenv("BCL_DEBUG_NVLS") != nullptr;
  if (dbg) std::fprintf(stderr, "[bcl rank %d] nvls: import/add\n", me.rank);
  try {
    if (me.rank != 0) nvls_ = NvlsTeam::import(all[0].nvls, me.device);
    if (dbg) std::fprintf(stderr, "[bcl rank %d] nvls: imported\n", me.rank);
    nvls_->add_device();
  } catch (const std::exception& e) {
    ok = false;
    nvls_why_ = e.what();
  }
  DeviceScope ds(me.device);
  const double limit = 60.0;
  if (dbg) std::fprintf(stderr, "[bcl rank %d] nvls: phase 1 ok=%d\n", me.rank, ok ? 1 : 0);
  if (agree(n_, me.rank, 1, ok, regions, region_bytes, limit)) {
    if (dbg) std::fprintf(stderr, "[bcl rank %d] nvls: agreed 1\n", me.rank);
    try {
      nvls_->bind_and_map();
    } catch (const std::exception& e) {
      ok = false;
      nvls_why_ = e.what();
    }
    if (dbg) std::fprintf(stderr, "[bcl rank %d] nvls: bound ok=%d %s\n", me.rank, ok ? 1 : 0, nvls_why_.c_str());
    if (agree(n_, me.rank, 2, ok, regions, region_bytes, limit)) {
      nvls_why_.clear();
      return;
    }
    if (ok) nvls_why_ = "another rank failed to bind its multicast memory";
  } else if (ok) {
    nvls_why_ = "another rank failed to join the multicast team";
  }
  nvls_.reset();
  if (opt_.nvls == 1) throw std::runtime_error("NVLS multicast required but unavailable: " + nvls_why_);
}

Group::~Group() {
  // (A group destroyed between bcl_group_start and _end drops its deferred calls.)
  std::erase(g_group_touched, this);
  for (LocalRank& r : local_) {
    cudaSetDevice(r.device);
    cudaDeviceSynchronize();
    for (void* p : r.opened) cudaIpcCloseMemHandle(p);
    if (r.region) cudaFree(r.region);
    if (r.d_peers) cudaFree(r.d_peers);
    if (r.d_regs) cudaFree(r.d_regs);
    if (r.heap) cudaFree(r.heap);
    if (lc_claim_ != nullptr && &r == &local_.front()) cudaFree(lc_claim_);
    if (r.scratch && !ipc_) cudaFree(r.scratch);
    if (r.err_host) cudaFreeHost(r.err_host);
    if (r.stream) cudaStreamDestroy(r.stream);
    if (r.copy_in) cudaStreamDestroy(r.copy_in);
    if (r.copy_out) cudaStreamDestroy(r.copy_out);
    if (r.host_mid) cudaStreamDestroy(r.host_mid);
    for (cudaEvent_t e : r.events) cudaEventDestroy(e);
  }
}

int Group::local_index_of(int rank) const {
  for (std::size_t i = 0; i < local_.size(); ++i) {
    if (local_[i].rank == rank) return static_cast<int>(i);
  }
  return -1;
}

// ------------------------------------------------------------------ tables

void Group::set_table(const TuningTable& t) {
  if (t.entries.empty()) throw std::invalid_argument("tuning table is empty");
  table_ = t;
  have_table_ = true;
}
void Group::clear_table() { have_table_ = false; }

void Group::set_protocol(int protocol) {
  if (protocol < 0 || protocol > 5) {
    throw std::invalid_argument("protocol must be 0 (auto), 1 (pull), 2 (push), 3 (ll), 4 (ll128) or 5 (nvls)");
  }
  opt_.protocol = protocol;
}

// Push needs middle ranks to pay off (measured, see tools/tune_b200.py); the
// table records from which size on it wins.
bool Group::use_push(const CallPlan& p, std::uint64_t bytes) const {
  if (!p.implicit_chain || n_ < 2) return false;
  if (opt_.protocol == 1 || opt_.protocol >= 3) return false;
  if (opt_.protocol == 2) return true;
  return select_push(table(), n_, bytes);
}
// NVLS multicast: every schedule under protocol 5 (the broadcast's result
// does not depend on the schedule); in auto mode the `direct` schedule above
// the LL threshold (root -> every rank is what the switch's replication does;
// the lane executor would send M once per receiver from the root).
bool Group::use_nvls(const CallPlan& p, std::uint64_t bytes) const {
  if (n_ < 2) return false;
  if (opt_.protocol == 5) {
    if (!nvls_) throw std::invalid_argument("NVLS multicast unavailable on this communicator: " + nvls_why_);
    return true;
  }
  if (opt_.protocol != 0 || !nvls_ || bytes == 0) return false;
  return p.config.algorithm == Algorithm::Direct && !(bytes <= ll_max_ && opt_.ll);
}

// LL128 lines for the `direct` schedule: every rank on its own GPU (or, with
// the ll128=1 option, ranks sharing one: the cross-GPU kernel through L2, one
// cooperative launch), from d128_min_ up to the LL threshold, whatever the
// protocol (like the 16-byte LL direct lines it replaces there). In a group
// the run carries every member on LL128 direct lines (fuse_kind).
bool Group::use_ll128_direct(const CallPlan& p, std::uint64_t bytes) const {
  if (!d128_min_ || !ll128_ok_ || !opt_.ll) return false;
  return p.config.algorithm == Algorithm::Direct && bytes >= d128_min_ && bytes <= ll_max_;
}

void Group::launch_nvls_group(const std::vector<int>& locals, const std::vector<void*>& bufs, std::uint64_t bytes,
                              int root, cudaStream_t stream) {
  if (bytes == 0) return;  // nothing moves (every rank skips alike)
  const std::uint64_t ll_max = std::min<std::uint64_t>(opt_.nvls_ll_max, dev::kNvlsLLMaxBytes);
  if (bytes <= ll_max) {  // NVLS-LL lines: no per-piece release
    dev::NvlsLLParams L{};
    L.n_local = static_cast<int>(locals.size());
    L.lines = static_cast<std::uint32_t>((bytes + 7) / 8);
    L.bytes = bytes;
    // ~2 lines per thread, identical on every GPU (the reports count on it);
    // every CTA of every rank sharing a GPU co-resident (cooperative launch).
    int per_dev = 1;
    for (const auto& kv : by_device_) per_dev = std::max(per_dev, static_cast<int>(kv.second.size()));
    const int cap = std::max(1, std::min(64, sms_ * std::max(nvls_ll_occ_, 1) / per_dev));
    L.ctas = std::clamp<int>(static_cast<int>((L.lines + 1023) / 1024), 1, cap);
    const int device = local_[static_cast<std::size_t>(locals[0])].device;
    L.n_recv = n_ - 1;
    L.timeout_ns = opt_.timeout_ns;
    L.mc = nvls_->mc(device);
    L.uc = nvls_->uc(device);
    const std::size_t S = region_stride();
    for (std::size_t i = 0; i < locals.size(); ++i) {
      LocalRank& r = local_[static_cast<std::size_t>(locals[i])];
      dev::NvlsRank& w = L.ranks[i];
      w.rank = r.rank;
      w.is_root = r.rank == root ? 1 : 0;
      w.buf = static_cast<std::uint8_t*>(bufs[i]);
      w.err = r.err_dev;
      w.abort = reinterpret_cast<int*>(r.region + 4 * S + static_cast<std::size_t>(n_));
      w.state = state_of(r);
      ++r.launches;
    }
    DeviceScope ds(device);
    ck(static_cast<cudaError_t>(launch_nvls_ll(L, stream)), "launch(nvls ll)");
    return;
  }
  const std::uint32_t slot = opt_.nvls_slot ? opt_.nvls_slot : dev::kNvlsDefaultSlot;
  const int wave = opt_.nvls_ctas > 0 ? opt_.nvls_ctas : dev::kNvlsDefaultCtas;
  const NvlsGeometry geo = nvls_geometry(bytes, slot, wave);
  dev::NvlsParams P{};
  P.n_local = static_cast<int>(locals.size());
  const int cap = std::max(1, sms_ * std::max(nvls_occ_, 1) / P.n_local);
  P.ctas = std::min<int>({static_cast<int>(geo.pieces), wave, cap});
  P.slot_bytes = slot;
  P.slots = static_cast<std::uint32_t>(dev::kNvlsRingBytes / slot);
  P.n_recv = n_ - 1;
  P.pieces = geo.pieces;
  P.bytes = bytes;
  P.piece_bytes = geo.piece_bytes;
  const int device = local_[static_cast<std::size_t>(locals[0])].device;
  P.timeout_ns = opt_.timeout_ns;
  P.strict = opt_.nvls_strict ? 1 : 0;
  P.mc = nvls_->mc(device);
  P.uc = nvls_->uc(device);
  const std::size_t S = region_stride();
  for (std::size_t i = 0; i < locals.size(); ++i) {
    LocalRank& r = local_[static_cast<std::size_t>(locals[i])];
    dev::NvlsRank& w = P.ranks[i];
    w.rank = r.rank;
    w.is_root = r.rank == root ? 1 : 0;
    w.buf = static_cast<std::uint8_t*>(bufs[i]);
    w.err = r.err_dev;
    w.abort = reinterpret_cast<int*>(r.region + 4 * S + static_cast<std::size_t>(n_));
    w.state = state_of(r);
    ++r.launches;
  }
  DeviceScope ds(device);
  ck(static_cast<cudaError_t>(launch_nvls(P, stream)), "launch(nvls)");
}

// Every rank on this GPU, pipelined chain, auto protocol: the fused
// flag-free kernel (pull forces the lane executor; timelines need it too).
// (The timeline hook needs the lane executor: single-process groups only, so
// every rank takes the same decision.)
bool Group::use_local_chain(const CallPlan& p, const std::vector<int>& locals) const {
  if (!single_device_ || !p.implicit_chain || opt_.protocol != 0 || !opt_.local_fused) return false;
  if (static_cast<int>(locals.size()) != n_ || n_ < 2) return false;
  for (const LocalRank& r : local_) {
    if (r.trace != nullptr) return false;
  }
  return true;
}

void Group::launch_local_chain(const std::vector<int>& locals, const std::vector<void*>& bufs, std::uint64_t bytes,
                               int root, const CallPlan& p, cudaStream_t stream) {
  dev::LocalChainParams P{};
  P.n_ranks = n_;
  P.n_chunks = p.n_chunks;
  P.bytes = bytes;
  P.chunk_bytes = p.chunk_bytes;
  std::uint64_t epoch = 0;
  for (std::size_t i = 0; i < locals.size(); ++i) {
    LocalRank& r = local_[static_cast<std::size_t>(locals[i])];
    const int logical = (r.rank - root + n_) % n_;
    P.buf[logical] = static_cast<std::uint8_t*>(bufs[i]);
    P.rank[logical] = r.rank;
    P.prov[logical] = r.prov;
    const std::uint64_t e = ++r.epoch;  // (host count: only checks that local ranks stay in step)
    if (i == 0) epoch = e;
    if (e != epoch) throw std::runtime_error("ranks sharing a GPU drifted apart in call count");
    ++r.launches;
  }
  DeviceScope ds(local_[static_cast<std::size_t>(locals[0])].device);
  const int ctas = opt_.local_ctas > 0 ? opt_.local_ctas : sms_ * std::max(local_chain_occ_, 1);
  const std::uint64_t warps = static_cast<std::uint64_t>(ctas) * 8;
  // Items claimed dynamically (load balance) of ~4 KiB: 43.6-43.9 us at
  // config 1 against 44.3-45.3 us for 2, 3 or 6 KiB (profiles/round2/n1/
  // variants.log); very large messages use larger items (fewer claims on the
  // one counter), small ones smaller items (every warp busy).
  std::uint64_t item = opt_.local_item;
  if (item == 0) {
    const std::uint64_t cap = std::max<std::uint64_t>(4096, bytes / (64 * warps));
    item = std::clamp<std::uint64_t>(bytes / (4 * warps), 2048, cap);
  }
  const std::uint64_t hi = std::max<std::uint64_t>(p.chunk_bytes, 16);
  item = std::clamp<std::uint64_t>((item + 15) / 16 * 16, std::min<std::uint64_t>(2048, hi), hi);
  P.item_bytes = std::min<std::uint64_t>(item, p.chunk_bytes);
  if (opt_.local_claim) {
    constexpr int kClaimSlots = 64;  // launches that may run concurrently (different streams)
    if (lc_claim_ == nullptr) {
      ck(cudaMalloc(&lc_claim_, kClaimSlots * sizeof(unsigned long long)), "cudaMalloc(claims)");
      ck(cudaMemset(lc_claim_, 0, kClaimSlots * sizeof(unsigned long long)), "cudaMemset(claims)");
    }
    const std::uint64_t ipc = (p.chunk_bytes + P.item_bytes - 1) / P.item_bytes;
    if (static_cast<std::uint64_t>(p.n_chunks) * ipc + warps >= (1ull << 32)) {
      throw std::invalid_argument("local chain: too many items for one launch (raise local_item)");
    }
    P.claim = lc_claim_ + (lc_launches_++ % kClaimSlots);
  }
  ck(static_cast<cudaError_t>(bcl::launch_local_chain(P, ctas, stream)), "launch(local chain)");
}

// Line protocols for the pipelined chain in auto mode: LL128 (every rank on
// its own GPU) up to the table's ll128 rule and ll128_max_; on one GPU the
// fused kernel instead; else 16-byte LL lines up to ll_chain_max_; above them
// the lane executor. Returns 0 (no line protocol), 1 (LL) or 2 (LL128).
// The choice depends only on state every rank shares (options, table, size):
// diagnostic hooks (provenance, timeline) never change the transport — line
// protocols simply record nothing — so ranks cannot disagree and deadlock.
int Group::ll_chain_mode(const CallPlan& p, std::uint64_t bytes, const std::vector<int>& locals) const {
  if (!p.implicit_chain || n_ < 2 || !opt_.ll || bytes == 0) return 0;
  if (opt_.protocol == 1 || opt_.protocol == 2) return 0;
  if (opt_.protocol == 3) {
    if (bytes > ll_chain_max_) throw std::invalid_argument("message exceeds the LL chain landing area");
    return 1;
  }
  if (opt_.protocol == 4) {
    if (!ll128_ok_) throw std::invalid_argument("LL128 needs every rank on its own GPU (or the ll128=1 option)");
    if (bytes > ll128_max_) throw std::invalid_argument("message exceeds the communicator's LL128 limit (ll128_max)");
    return 2;
  }
  if (ll128_ok_ && !single_device_ && bytes <= ll128_max_ && select_ll128(table(), n_, bytes)) return 2;
  // One GPU: the fused kernel beats LL lines at every size (4 KiB: 8.2 vs
  // 9.8 us, 8 MiB: 12.4 vs 51.8 us, 4 ranks); LL stays available explicitly.
  if (use_local_chain(p, locals)) return 0;
  return bytes <= ll_chain_max_ ? 1 : 0;
}
const TuningTable& Group::table() const { return have_table_ ? table_ : builtin_table(); }

// `bcast --algo auto` semantics: select per size, clamp the chunk to the
// message (bcastlab.cpp:258-266).
AlgorithmConfig Group::choose(std::uint64_t bytes, const AlgorithmConfig* cfg) const {
  if (cfg) return *cfg;
  AlgorithmConfig c = select(table(), n_, bytes);
  if (c.algorithm == Algorithm::ChainPipelined) {
    c.chunk_bytes = std::clamp<std::uint64_t>(c.chunk_bytes, 1, std::max<std::uint64_t>(bytes, 1));
  }
  return c;
}

// ------------------------------------------------------------------ plans

std::shared_ptr<const CallPlan> Group::plan_ptr(const AlgorithmConfig& cfg, int root, std::uint64_t bytes) {
  const auto key = std::make_tuple(static_cast<int>(cfg.algorithm), cfg.radix_k, cfg.chunk_bytes, root, bytes);
  {
    std::lock_guard<std::mutex> lock(plan_mu_);
    auto it = plans_.find(key);
    if (it != plans_.end()) return it->second;
  }
  cfg.validate();
  auto p = std::make_shared<CallPlan>();
  p->config = cfg;
  const std::uint64_t nn = static_cast<std::uint64_t>(n_);
  std::uint64_t max_len = bytes;
  Schedule sched;
  if (cfg.algorithm == Algorithm::ChainPipelined) {
    if (root < 0 || root >= n_) throw std::invalid_argument("root out of range");
    if (n_ < 2) throw std::invalid_argument("pipelined chain needs at least 2 ranks");
    const std::uint64_t k = bytes == 0 ? 1 : (bytes + cfg.chunk_bytes - 1) / cfg.chunk_bytes;
    if (k > 0xFFFFFFFFull) throw std::invalid_argument("too many chunks");
    p->implicit_chain = true;
    p->chunk_mode = dev::kFixedChunks;
    p->n_chunks = static_cast<std::uint32_t>(k);
    p->chunk_bytes = cfg.chunk_bytes;
    max_len = std::min(cfg.chunk_bytes, bytes);
  } else {
    sched = make_schedule(cfg, n_, root, bytes);
    p->n_chunks = static_cast<std::uint32_t>(sched.chunks.size());
    if (cfg.algorithm == Algorithm::ScatterRingAllgather) {
      p->chunk_mode = dev::kPartitions;
      max_len = (bytes + nn - 1) / nn;
    } else {
      p->chunk_mode = dev::kWholeMessage;
    }
    p->chunk_bytes = max_len;
  }
  // Lane plan. ns = L / Q chunks are in flight per rank at once (one per
  // pipe), so ns * C bytes is the window a hop must fill before its
  // downstream can start: keep it near `window` (enough to cover NVLink
  // bandwidth x latency) but never cut slices below `min_slice`.
  const std::uint64_t win_chunks = std::max<std::uint64_t>(1, opt_.window_bytes / std::max<std::uint64_t>(max_len, 1));
  const std::uint64_t q_floor = (static_cast<std::uint64_t>(lanes_) + win_chunks - 1) / win_chunks;
  std::uint64_t q_floor_stage = 1;  // bulk path: one slice per stage
  if (opt_.stage_bytes > 0) {
    const std::uint64_t sb = static_cast<std::uint64_t>(opt_.stage_bytes);
    q_floor_stage = (max_len + sb - 1) / sb;
  }
  const std::uint64_t q_cap = std::max<std::uint64_t>(q_floor_stage, max_len / std::max<std::uint64_t>(opt_.min_slice, 16));
  int q = 0;
  for (int d = 1; d <= lanes_; ++d) {  // smallest divisor of L reaching q_floor
    if (lanes_ % d == 0 && static_cast<std::uint64_t>(d) >= std::max(q_floor, q_floor_stage)) { q = d; break; }
  }
  if (q == 0) q = lanes_;  // even one slice per lane cannot meet the floor
  if (static_cast<std::uint64_t>(q) > q_cap) {  // too thin: largest divisor within q_cap
    q = 1;
    for (int d = 1; d <= lanes_; ++d) {
      if (lanes_ % d == 0 && static_cast<std::uint64_t>(d) <= q_cap) q = d;
    }
  }
  p->slices = q;
  const std::uint64_t per = (max_len + static_cast<std::uint64_t>(q) - 1) / static_cast<std::uint64_t>(q);
  p->slice_bytes = std::max<std::uint64_t>(16, (per + 15) / 16 * 16);
  const int ns = lanes_ / q;
  const std::uint64_t active = std::min<std::uint64_t>(static_cast<std::uint64_t>(ns), p->n_chunks) *
                               static_cast<std::uint64_t>(q);
  p->ctas = static_cast<int>((active + dev::kWarpsPerCta - 1) / dev::kWarpsPerCta);
  if (!p->implicit_chain) {
    p->events.resize(static_cast<std::size_t>(n_));
    for (int r = 0; r < n_; ++r) {
      const auto& ops = sched.per_rank_ops[static_cast<std::size_t>(r)];
      if (ops.size() > static_cast<std::size_t>(dev::kMaxEvents)) {
        throw std::invalid_argument("schedule has more events per rank than the device executor holds");
      }
      std::map<std::tuple<int, int, std::uint32_t>, std::uint32_t> seen;  // (kind, peer, class)
      for (const Event& e : ops) {
        const bool rv = e.kind == Event::Kind::Recv;
        const std::uint32_t cls = e.chunk % static_cast<std::uint32_t>(ns);
        const std::uint32_t idx = seen[{rv ? 1 : 0, e.peer, cls}]++;
        p->events[static_cast<std::size_t>(r)].push_back(dev::pack_event(rv, e.peer, e.chunk, idx));
      }
    }
  }
  std::lock_guard<std::mutex> lock(plan_mu_);
  if (plans_.size() > 256) plans_.clear();
  plans_[key] = p;
  return p;
}

// ---------------------------------------------------------------- launches

// Per-process ranks name their buffer to peers as a symmetric-heap offset or
// as (registration id + 1) << 40 | offset into a registered allocation.
std::uint64_t Group::ipc_mailbox_value(const LocalRank& r, const std::uint8_t* b, std::uint64_t bytes) const {
  if (bytes == 0) return 0;  // nothing is read
  if (b >= r.heap && b + bytes <= r.heap + r.heap_bytes) return static_cast<std::uint64_t>(b - r.heap);
  for (std::size_t i = 0; i < r.regs.size(); ++i) {
    const auto& g = r.regs[i];
    if (r.d_regs != nullptr && b >= g.base && b + bytes <= g.base + g.size && i < r.regs.size()) {
      return ((i + 1) << 40) | static_cast<std::uint64_t>(b - g.base);
    }
  }
  throw std::invalid_argument(
      "per-process ranks pull peers' buffers directly: use buffers from bcl_mem_alloc or register their allocation "
      "with bcl_comm_register_export/connect (buffer offset " +
      std::to_string(static_cast<long long>(b - r.heap)) + " + " + std::to_string(bytes) + " bytes)");
}

void Group::fill_rank_work(dev::RankWork& w, LocalRank& r, const CallPlan& p, void* buf, std::uint64_t bytes) {
  const std::size_t S = region_stride();
  w.rank = r.rank;
  w.n_events = p.implicit_chain ? -1 : static_cast<int>(p.events[static_cast<std::size_t>(r.rank)].size());
  w.buf = static_cast<std::uint8_t*>(buf);
  w.pub = ipc_ ? ipc_mailbox_value(r, static_cast<std::uint8_t*>(buf), bytes)
               : reinterpret_cast<std::uint64_t>(buf);
  if (w.pub >> 48) throw std::runtime_error("buffer address does not fit the 48-bit mailbox field");
  w.flags = r.region;
  w.acks = r.region + S;
  w.mbox = r.region + 2 * S;
  w.peers = r.d_peers;
  w.err = r.err_dev;
  w.abort = reinterpret_cast<int*>(r.region + 4 * S + static_cast<std::size_t>(n_));
  w.prov = r.prov;
  w.trace = r.trace;
  w.trace_cap = r.trace_cap;
  w.state = state_of(r);
  if (!p.implicit_chain) {
    const auto& ev = p.events[static_cast<std::size_t>(r.rank)];
    std::copy(ev.begin(), ev.end(), w.events);
  }
}

void Group::launch_ll(const std::vector<int>& locals, const std::vector<void*>& bufs, std::uint64_t bytes,
                      int root, cudaStream_t stream, int mode) {
  launch_ll_segs(locals, {bufs}, {bytes}, root, stream, mode);
}

std::uint64_t Group::ll_lines_of(std::uint64_t bytes, int mode) {
  return mode >= 2 ? (bytes + dev::kLL128Payload - 1) / dev::kLL128Payload : (bytes + 7) / 8;
}

// One launch of a line protocol carrying one or more messages (segments):
// seg_bufs[s][i] is local rank i's buffer of message s.
void Group::launch_ll_segs(const std::vector<int>& locals, const std::vector<std::vector<void*>>& seg_bufs,
                           const std::vector<std::uint64_t>& seg_bytes, int root, cudaStream_t stream, int mode) {
  const bool chain = mode == 1 || mode == 2;
  dev::LLParams P{};
  P.n_ranks = n_;
  P.root = root;
  P.n_local = static_cast<int>(locals.size());
  P.n_seg = static_cast<int>(seg_bytes.size());
  if (P.n_seg < 1 || P.n_seg > dev::max_segs(P.n_local)) {
    throw std::invalid_argument("line-protocol launch: too many messages");
  }
  std::uint64_t lines = 0;
  for (int s = 0; s < P.n_seg; ++s) {
    P.seg_line[s] = static_cast<std::uint32_t>(lines);
    P.seg_bytes[s] = seg_bytes[static_cast<std::size_t>(s)];
    lines += ll_lines_of(seg_bytes[static_cast<std::size_t>(s)], mode);
    for (std::size_t i = 0; i < locals.size(); ++i) {
      P.seg_buf[i][s] = static_cast<std::uint8_t*>(seg_bufs[static_cast<std::size_t>(s)][i]);
    }
  }
  if (lines >= (1ull << 31)) throw std::invalid_argument("line-protocol launch too large");
  P.seg_line[P.n_seg] = static_cast<std::uint32_t>(lines);
  P.bytes = seg_bytes.front();
  P.lines = static_cast<std::uint32_t>(lines);
  P.area_lines = static_cast<std::uint32_t>(ll_max_ / 8);
  P.chain = static_cast<std::uint32_t>(mode);
  P.chain_lines = static_cast<std::uint32_t>(ll_chain_max_ / 8);
  P.chain128_lines = ll128_lines();
  P.chain128_area = ll128_area();
  P.d128_area = d128_area();
  P.d128_lines = d128_lines();
  // ~4 lines per thread, at most kLLMaxCtas CTAs per rank
  // ~2 lines per thread; ranks sharing a GPU must stay co-resident
  // (cooperative launch): at most 4 LL CTAs per SM in total.
  const int resident = std::max(1, sms_ * 4 / std::max<int>(1, P.n_local));
  P.ctas = std::clamp<int>(static_cast<int>((P.lines + 2 * dev::kLLThreads - 1) / (2 * dev::kLLThreads)), 1,
                           std::min(dev::kLLMaxCtas, resident));
  if (mode == 2) {  // a warp moves 4 lines per step: ~2 steps per warp, up to 3 CTAs per SM
    const std::uint32_t per_cta = dev::kLLThreads / 32 * 4 * 2;
    // every CTA of every rank co-resident (writers wait on ring credits)
    const int occ = P.n_local > 1 ? ll128_occ_shared_ : ll128_occ_;
    int cap = std::max(1, std::min(dev::kLL128MaxCtas, sms_ * std::max(occ, 1)) / P.n_local);
    if (opt_.ll128_ctas > 0) cap = std::min(cap, opt_.ll128_ctas);
    P.ctas = std::clamp<int>(static_cast<int>((P.lines + per_cta - 1) / per_cta), 1, cap);
  }
  if (mode == 3) {  // LL128 direct: a warp moves 4 lines per step, ~2 steps per warp; no co-residency needed
    const std::uint32_t per_cta = dev::kLLThreads / 32 * 4 * 2;
    int cap = opt_.ll128_direct_ctas > 0 ? opt_.ll128_direct_ctas : sms_;
    if (P.n_local > 1) cap = std::min(cap, resident);  // (ranks sharing a GPU: one cooperative launch)
    P.ctas = std::clamp<int>(static_cast<int>((P.lines + per_cta - 1) / per_cta), 1, cap);
  }
  P.timeout_ns = opt_.timeout_ns;
  P.coop = opt_.ll128_coop ? 1 : 0;
  const std::size_t S = region_stride();
  std::uint64_t epoch = 0;
  for (std::size_t i = 0; i < locals.size(); ++i) {
    LocalRank& r = local_[static_cast<std::size_t>(locals[i])];
    const std::uint64_t e = ++r.epoch;  // (host count: only checks that local ranks stay in step)
    if (i == 0) epoch = e;
    if (e != epoch) throw std::runtime_error("ranks sharing a GPU drifted apart in call count");
    dev::LLRank& w = P.ranks[i];
    w.rank = r.rank;
    w.buf = static_cast<std::uint8_t*>(seg_bufs.front()[i]);
    w.credit = r.region + 4 * S + static_cast<std::size_t>(n_) + 1 + (chain ? static_cast<std::size_t>(n_) + 1 : 0);
    w.wcredit = r.region + 4 * S + 3 * static_cast<std::size_t>(n_) + 2;
    w.wseq = w.wcredit + dev::kLL128WarpsMax;
    w.rseq = w.wseq + dev::kLL128WarpsMax;
    w.ll = reinterpret_cast<uint4*>(r.region + ll_offset(lanes_));
    w.peers = r.d_peers;
    w.err = r.err_dev;
    w.abort = reinterpret_cast<int*>(r.region + 4 * S + static_cast<std::size_t>(n_));
    // The epoch, the half and the writers' reuse bound (the last call of the
    // same kind that wrote this half) come from the device-side call state.
    w.state = state_of(r);
    ++r.launches;
  }
  DeviceScope ds(local_[static_cast<std::size_t>(locals[0])].device);
  ck(static_cast<cudaError_t>(bcl::launch_ll(P, stream)), "launch(ll)");
}

// The device path a call of this shape takes (the same decisions as
// launch_group, on state every rank shares).
std::string Group::path(const AlgorithmConfig* cfg, int root, std::uint64_t bytes) {
  const AlgorithmConfig c = choose(bytes, cfg);
  const auto pp = plan_ptr(c, root, bytes);
  const CallPlan& p = *pp;
  if (n_ == 1) return "none";
  std::vector<int> locals;
  for (int i = 0; i < local_count(); ++i) locals.push_back(i);
  if (use_nvls(p, bytes)) {
    return bytes <= std::min<std::uint64_t>(opt_.nvls_ll_max, dev::kNvlsLLMaxBytes) ? "nvls_ll_kernel" : "nvls_kernel";
  }
  if (use_ll128_direct(p, bytes)) return "ll128_kernel/direct";
  if (p.config.algorithm == Algorithm::Direct && bytes <= ll_max_ && opt_.ll) return "ll_kernel/direct";
  if (const int mode = ll_chain_mode(p, bytes, locals)) return mode == 2 ? "ll128_kernel" : "ll_kernel/chain";
  if (use_local_chain(p, locals)) return "local_chain_kernel";
  if (!p.implicit_chain) return "bcast_kernel/events";
  const bool bulk = opt_.stage_bytes > 0;
  return use_push(p, bytes) ? (bulk ? "bcast_kernel/push/tma" : "bcast_kernel/push")
                            : (bulk ? "bcast_kernel/pull/tma" : "bcast_kernel/pull");
}

void Group::launch_group(const std::vector<int>& locals, const std::vector<void*>& bufs,
                         std::uint64_t bytes, int root, const CallPlan& p, cudaStream_t stream) {
  if (use_nvls(p, bytes)) {
    launch_nvls_group(locals, bufs, bytes, root, stream);
    return;
  }
  if (use_ll128_direct(p, bytes)) {
    launch_ll(locals, bufs, bytes, root, stream, 3);
    return;
  }
  if (p.config.algorithm == Algorithm::Direct && bytes <= ll_max_ && opt_.ll) {
    launch_ll(locals, bufs, bytes, root, stream, 0);
    return;
  }
  if (const int mode = ll_chain_mode(p, bytes, locals)) {
    launch_ll(locals, bufs, bytes, root, stream, mode);
    return;
  }
  if (use_local_chain(p, locals)) {
    launch_local_chain(locals, bufs, bytes, root, p, stream);
    return;
  }
  dev::LaunchParams P{};
  P.n_ranks = n_;
  P.root = root;
  P.n_local = static_cast<int>(locals.size());
  P.lanes = lanes_;
  P.slices = p.slices;
  P.ctas_per_rank = p.ctas;
  P.chunk_mode = p.chunk_mode;
  P.n_chunks = p.n_chunks;
  P.bytes = bytes;
  P.chunk_bytes = p.chunk_bytes;
  P.slice_bytes = p.slice_bytes;
  P.timeout_ns = opt_.timeout_ns;
  P.poll_ns = opt_.poll_ns;
  P.sys_scope = sys_ ? 1 : 0;
  P.strict_sys = (opt_.strict_sys && sys_) ? 1 : 0;
  P.stage_bytes = static_cast<std::uint32_t>(std::max<std::int64_t>(opt_.stage_bytes, 0));
  P.stages = opt_.stages;
  P.push = use_push(p, bytes) ? 1 : 0;
  P.eager_post = opt_.eager_post ? 1 : 0;
  // Push publishes data that lives in the peer's memory: its sys-scope fence
  // must wait for the remote stores anyway, so the publisher keeps it (a
  // writer-side sys fence halves push bandwidth: 3.39 vs 1.73 ms, 1 GiB n=4).
  P.writer_fence = (P.strict_sys || P.push) ? 0 : (sys_ ? opt_.writer_fence : std::min(opt_.writer_fence, 1));
  std::uint64_t epoch = 0;
  for (std::size_t i = 0; i < locals.size(); ++i) {
    LocalRank& r = local_[static_cast<std::size_t>(locals[i])];
    const std::uint64_t e = ++r.epoch;
    if (i == 0) epoch = e;
    if (e != epoch) throw std::runtime_error("ranks sharing a GPU drifted apart in call count");
    fill_rank_work(P.ranks[i], r, p, bufs[i], bytes);
    ++r.launches;
  }
  P.epoch = epoch;  // (informational: the kernel takes the call's epoch from the device-side call state)
  DeviceScope ds(local_[static_cast<std::size_t>(locals[0])].device);
  ck(static_cast<cudaError_t>(launch_bcast(P, P.n_local > 1 ? 1 : 0, stream)), "launch(bcast)");
}

void Group::bcast(int li, void* buf, std::uint64_t bytes, int root, const AlgorithmConfig* cfg,
                  cudaStream_t stream) {
  if (broken_) throw std::runtime_error("communicator is unusable after a device failure");
  if (!connected_) throw std::invalid_argument("communicator is not connected");
  if (root < 0 || root >= n_) throw std::invalid_argument("root out of range");
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  if (by_device_.at(r.device).size() > 1) {
    throw std::invalid_argument("ranks sharing a GPU must be driven together (bcast_all)");
  }
  if (bytes > 0 && buf == nullptr) throw std::invalid_argument("null buffer");
  // (Per-process ranks: line protocols take any device buffer; the lane
  // executor needs heap or registered buffers, checked in fill_rank_work.)
  const AlgorithmConfig c = choose(bytes, cfg);
  const auto pp = plan_ptr(c, root, bytes);
  const CallPlan& p = *pp;
  if (n_ == 1) return;  // nothing moves (reference: n = 1 leaves the buffer untouched)
  if (defer(Deferred{false, li, {buf}, bytes, root, pp, {stream}, opt_.protocol})) return;
  launch_group({li}, {buf}, bytes, root, p, stream);
}

void Group::bcast_all(const std::vector<void*>& bufs, std::uint64_t bytes, int root,
                      const AlgorithmConfig* cfg, const std::vector<cudaStream_t>& streams) {
  if (broken_) throw std::runtime_error("communicator is unusable after a device failure");
  if (bufs.size() != local_.size()) throw std::invalid_argument("one buffer per rank required");
  if (!streams.empty() && streams.size() != local_.size()) {
    throw std::invalid_argument("one stream per rank (or none)");
  }
  if (root < 0 || root >= n_) throw std::invalid_argument("root out of range");
  for (void* b : bufs) {
    if (bytes > 0 && b == nullptr) throw std::invalid_argument("null buffer");
  }
  const AlgorithmConfig c = choose(bytes, cfg);
  const auto pp = plan_ptr(c, root, bytes);
  const CallPlan& p = *pp;
  if (n_ == 1) return;
  std::vector<cudaStream_t> per;  // per device, first rank's stream
  for (const auto& kv : by_device_) {
    const int first = kv.second.front();
    per.push_back(streams.empty() ? local_[static_cast<std::size_t>(first)].stream
                                  : streams[static_cast<std::size_t>(first)]);
  }
  if (defer(Deferred{true, -1, bufs, bytes, root, pp, per, opt_.protocol})) return;
  std::size_t d = 0;
  for (const auto& kv : by_device_) {
    std::vector<void*> b;
    for (int li : kv.second) b.push_back(bufs[static_cast<std::size_t>(li)]);
    launch_group(kv.second, b, bytes, root, p, per[d++]);
  }
}

// ------------------------------------------------------------- group fusion
//
// bcl_group_start/end (NCCL-style): broadcasts issued in between are
// deferred; at the end, runs of consecutive calls on a line protocol (LL
// direct, LL chain, LL128 chain) with the same root and stream are fused into
// one launch carrying up to 32 messages (segments) on the run's most capable
// protocol; the rest launch as usual, in order. Every rank sees the same call sequence, so every
// rank fuses identically (the fused launch is one call epoch everywhere).

void Group::group_start() { ++g_group_depth; }

void Group::group_end() {
  if (g_group_depth <= 0) throw std::invalid_argument("group_end without group_start");
  if (--g_group_depth > 0) return;
  std::vector<Group*> touched;
  touched.swap(g_group_touched);
  std::exception_ptr first;
  for (Group* g : touched) {
    try {
      g->flush_deferred();
    } catch (...) {
      if (!first) first = std::current_exception();
    }
  }
  if (first) std::rethrow_exception(first);
}

bool Group::in_group() { return g_group_depth > 0; }

bool Group::defer(Deferred d) {
  if (g_group_depth <= 0) return false;
  if (deferred_.empty()) g_group_touched.push_back(this);
  deferred_.push_back(std::move(d));
  return true;
}

// The line protocol a call takes (1 LL direct, 2 LL128 direct, 3 LL chain,
// 4 LL128 chain: a run travels on its highest member's; mode_of_kind maps
// them to launch_ll_segs modes),
// or 0 when it cannot be fused -- the decisions of launch_group.
int Group::fuse_kind(const Deferred& d) {
  const CallPlan& p = *d.plan;
  std::vector<int> locals;
  if (d.all) {
    for (int i = 0; i < local_count(); ++i) locals.push_back(i);
  } else {
    locals.push_back(d.li);
  }
  if (use_nvls(p, d.bytes)) return 0;
  if (use_ll128_direct(p, d.bytes)) return 2;
  if (p.config.algorithm == Algorithm::Direct && d.bytes <= ll_max_ && opt_.ll) return 1;
  const int mode = ll_chain_mode(p, d.bytes, locals);
  if (mode == 1) return 3;
  if (mode == 2) {
    for (const auto& kv : by_device_) {
      if (kv.second.size() > 1) return 0;  // no fused LL128 chain for ranks sharing a GPU
    }
    return 4;
  }
  return 0;
}

void Group::flush_deferred() {
  std::vector<Deferred> calls;
  calls.swap(deferred_);
  // Each call runs under the protocol that was set when it was issued.
  struct Restore {
    int& slot;
    int saved;
    ~Restore() { slot = saved; }
  } restore{opt_.protocol, opt_.protocol};
  std::size_t i = 0;
  while (i < calls.size()) {
    const Deferred& d = calls[i];
    opt_.protocol = d.protocol;
    int kind = fuse_kind(d);
    // Extend the run: same root, shape and streams, every member on a line
    // protocol; the run travels on its most capable member's protocol (LL128
    // chain > LL chain > LL direct: small messages ride along a chain launch
    // rather than cut the run), within the segment and landing-area caps.
    std::size_t j = i + 1;
    if (kind != 0) {
      int per_dev = 1;
      for (const auto& kv : by_device_) per_dev = std::max(per_dev, static_cast<int>(kv.second.size()));
      const std::size_t max_segs = static_cast<std::size_t>(dev::max_segs(d.all ? per_dev : 1));
      auto fits = [&](std::size_t end, int k) {
        const std::uint64_t cap = k == 1   ? ll_max_ / 8
                                  : k == 2 ? d128_lines()
                                  : k == 3 ? ll_chain_max_ / 8
                                           : (1ull << 31) - 1;
        std::uint64_t lines = 0;
        for (std::size_t c = i; c < end; ++c) lines += ll_lines_of(calls[c].bytes, mode_of_kind(k));
        return lines <= cap;
      };
      while (j < calls.size() && j - i < max_segs) {
        const Deferred& e = calls[j];
        if (e.all != d.all || e.li != d.li || e.root != d.root || e.streams != d.streams ||
            e.protocol != d.protocol) {
          break;
        }
        const int ke = fuse_kind(e);
        if (ke == 0) break;
        const int k = std::max(kind, ke);
        if (!fits(j + 1, k)) break;
        kind = k;
        ++j;
      }
    }
    if (j == i + 1) {  // a lone call: exactly what the call would have done
      if (d.all) {
        std::size_t k = 0;
        for (const auto& kv : by_device_) {
          std::vector<void*> b;
          for (int li : kv.second) b.push_back(d.bufs[static_cast<std::size_t>(li)]);
          launch_group(kv.second, b, d.bytes, d.root, *d.plan, d.streams[k++]);
        }
      } else {
        launch_group({d.li}, d.bufs, d.bytes, d.root, *d.plan, d.streams.front());
      }
    } else {
      std::vector<std::uint64_t> seg_bytes;
      for (std::size_t k = i; k < j; ++k) seg_bytes.push_back(calls[k].bytes);
      if (d.all) {
        std::size_t k = 0;
        for (const auto& kv : by_device_) {
          std::vector<std::vector<void*>> seg_bufs;
          for (std::size_t c = i; c < j; ++c) {
            std::vector<void*> b;
            for (int li : kv.second) b.push_back(calls[c].bufs[static_cast<std::size_t>(li)]);
            seg_bufs.push_back(std::move(b));
          }
          launch_ll_segs(kv.second, seg_bufs, seg_bytes, d.root, d.streams[k++], mode_of_kind(kind));
        }
      } else {
        std::vector<std::vector<void*>> seg_bufs;
        for (std::size_t c = i; c < j; ++c) seg_bufs.push_back({calls[c].bufs.front()});
        launch_ll_segs({d.li}, seg_bufs, seg_bytes, d.root, d.streams.front(), mode_of_kind(kind));
      }
    }
    i = j;
  }
}

// Host-buffer broadcasts stage through device scratch in pieces on three
// streams per rank: H2D of piece i+1 (root) overlaps the device broadcast and
// the D2H of piece i (receivers). Each piece is an ordinary broadcast call,
// issued identically on every rank.
namespace {

struct Piece {
  std::uint64_t off, len;
};

// Pieces grow geometrically from 1 MiB up to `piece`: the first D2H can start
// after a small H2D + broadcast, later pieces amortise per-copy overheads.
std::vector<Piece> pieces_of(std::uint64_t bytes, std::uint64_t piece) {
  std::vector<Piece> v;
  if (bytes == 0) return {Piece{0, 0}};
  std::uint64_t cur = std::min<std::uint64_t>(piece, 1ull << 20);
  for (std::uint64_t off = 0; off < bytes; off += cur) {
    if (off > 0) cur = std::min(piece, cur * 2);
    v.push_back(Piece{off, std::min(cur, bytes - off)});
  }
  return v;
}

}  // namespace

cudaEvent_t Group::event(LocalRank& r, std::size_t i) {
  while (r.events.size() <= i) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    r.events.push_back(e);
  }
  return r.events[i];
}

void Group::ensure_scratch(int li, std::uint64_t bytes) {
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  if (bytes <= r.scratch_bytes) return;
  DeviceScope ds(r.device);
  if (ipc_) {
    // Peers read the scratch, so it lives in the symmetric heap. Grow the
    // previous scratch in place when it is the heap's last allocation.
    if (r.scratch != nullptr && r.scratch + r.scratch_bytes == r.heap + r.heap_used &&
        static_cast<std::size_t>(r.scratch - r.heap) + bytes <= r.heap_bytes) {
      r.heap_used = static_cast<std::size_t>(r.scratch - r.heap) + bytes;
    } else {
      r.scratch = static_cast<std::uint8_t*>(mem_alloc(li, bytes));
    }
  } else {
    if (r.scratch) ck(cudaFree(r.scratch), "cudaFree(scratch)");
    ck(cudaMalloc(&r.scratch, bytes), "cudaMalloc(scratch)");
  }
  r.scratch_bytes = bytes;
}

void Group::bcast_host(int li, void* host_buf, std::uint64_t bytes, int root,
                       const AlgorithmConfig* cfg, cudaStream_t stream) {
  if (in_group()) throw std::invalid_argument("host-buffer broadcasts cannot be grouped");
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  if (root < 0 || root >= n_) throw std::invalid_argument("root out of range");
  if (bytes > 0 && host_buf == nullptr) throw std::invalid_argument("null buffer");
  ensure_scratch(li, bytes);
  DeviceScope ds(r.device);
  auto* hb = static_cast<std::uint8_t*>(host_buf);
  const auto ps = pieces_of(bytes, opt_.host_piece);
  std::size_t ev = 0;
  const cudaEvent_t start = event(r, ev++);
  ck(cudaEventRecord(start, stream), "cudaEventRecord");
  ck(cudaStreamWaitEvent(r.copy_in, start, 0), "cudaStreamWaitEvent");
  ck(cudaStreamWaitEvent(r.copy_out, start, 0), "cudaStreamWaitEvent");
  for (const Piece& p : ps) {
    if (r.rank == root && p.len) {
      ck(cudaMemcpyAsync(r.scratch + p.off, hb + p.off, p.len, cudaMemcpyHostToDevice, r.copy_in), "H2D");
      const cudaEvent_t in = event(r, ev++);
      ck(cudaEventRecord(in, r.copy_in), "cudaEventRecord");
      ck(cudaStreamWaitEvent(stream, in, 0), "cudaStreamWaitEvent");
    }
    bcast(li, r.scratch + p.off, p.len, root, cfg, stream);
    if (r.rank != root && p.len) {
      const cudaEvent_t done = event(r, ev++);
      ck(cudaEventRecord(done, stream), "cudaEventRecord");
      ck(cudaStreamWaitEvent(r.copy_out, done, 0), "cudaStreamWaitEvent");
      ck(cudaMemcpyAsync(hb + p.off, r.scratch + p.off, p.len, cudaMemcpyDeviceToHost, r.copy_out), "D2H");
    }
  }
  const cudaEvent_t out = event(r, ev++);
  ck(cudaEventRecord(out, r.copy_out), "cudaEventRecord");
  ck(cudaStreamWaitEvent(stream, out, 0), "cudaStreamWaitEvent");
}

void Group::raise_errors(const std::vector<int>& locals) {
  std::vector<RankFailure> f;
  for (int li : locals) {
    const dev::ErrorRecord& e = *local_[static_cast<std::size_t>(li)].err_host;
    if (e.code != 0) f.push_back(RankFailure{local_[static_cast<std::size_t>(li)].rank, describe(e)});
  }
  if (f.empty()) return;
  broken_ = true;
  if (f.size() == 1) throw DeviceTimeout(f.front().message);
  throw AggregateRankError(std::move(f));
}

void Group::check(int li, cudaStream_t stream) {
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  DeviceScope ds(r.device);
  ck(stream ? cudaStreamSynchronize(stream) : cudaDeviceSynchronize(), "synchronize");
  raise_errors({li});
}

double Group::run_bcast(const std::vector<void*>& bufs, std::uint64_t bytes, int root,
                        const AlgorithmConfig* cfg) {
  if (in_group()) throw std::invalid_argument("run_bcast is synchronous and cannot be grouped");
  if (static_cast<int>(bufs.size()) != n_ || local_count() != n_) {
    throw std::invalid_argument("one buffer per rank required");
  }
  const auto t0 = std::chrono::steady_clock::now();
  bcast_all(bufs, bytes, root, cfg, {});
  std::vector<int> all;
  for (const auto& kv : by_device_) {
    DeviceScope ds(kv.first);
    ck(cudaStreamSynchronize(local_[static_cast<std::size_t>(kv.second.front())].stream), "synchronize");
    all.insert(all.end(), kv.second.begin(), kv.second.end());
  }
  const auto t1 = std::chrono::steady_clock::now();
  std::vector<RankFailure> f;
  for (int li : all) {
    const dev::ErrorRecord& e = *local_[static_cast<std::size_t>(li)].err_host;
    if (e.code != 0) f.push_back(RankFailure{local_[static_cast<std::size_t>(li)].rank, describe(e)});
  }
  if (!f.empty()) {
    broken_ = true;
    throw AggregateRankError(std::move(f));
  }
  return std::chrono::duration<double>(t1 - t0).count();
}

double Group::run_bcast_host(const std::vector<void*>& host_bufs, std::uint64_t bytes, int root,
                             const AlgorithmConfig* cfg) {
  if (in_group()) throw std::invalid_argument("run_bcast_host is synchronous and cannot be grouped");
  if (static_cast<int>(host_bufs.size()) != n_ || local_count() != n_) {
    throw std::invalid_argument("one buffer per rank required");
  }
  const int root_li = local_index_of(root);
  if (root_li < 0) throw std::invalid_argument("root out of range");
  for (int li = 0; li < n_; ++li) {
    if (bytes > 0 && host_bufs[static_cast<std::size_t>(li)] == nullptr) throw std::invalid_argument("null buffer");
    ensure_scratch(li, bytes);
  }
  const auto ps = pieces_of(bytes, opt_.host_piece);
  const auto t0 = std::chrono::steady_clock::now();
  LocalRank& R = local_[static_cast<std::size_t>(root_li)];
  // Ranks sharing a GPU run in one launch on the first local rank's stream
  // (a non-blocking one: the scratch buffers depend on no legacy-stream work).
  auto compute_of = [this](int dev) { return local_[static_cast<std::size_t>(by_device_.at(dev).front())].host_mid; };
  auto owner_of = [this](int dev) -> LocalRank& { return local_[static_cast<std::size_t>(by_device_.at(dev).front())]; };
  std::map<int, std::size_t> ev;  // per device event cursor
  for (const auto& kv : by_device_) ev[kv.first] = 0;
  for (const Piece& p : ps) {
    if (p.len) {
      DeviceScope ds(R.device);
      ck(cudaMemcpyAsync(R.scratch + p.off, static_cast<std::uint8_t*>(host_bufs[static_cast<std::size_t>(root)]) + p.off,
                         p.len, cudaMemcpyHostToDevice, R.copy_in), "H2D");
      const cudaEvent_t in = event(owner_of(R.device), ev[R.device]++);
      ck(cudaEventRecord(in, R.copy_in), "cudaEventRecord");
      ck(cudaStreamWaitEvent(compute_of(R.device), in, 0), "cudaStreamWaitEvent");
    }
    std::vector<void*> dbufs;
    std::vector<cudaStream_t> mids;
    for (LocalRank& r : local_) {
      dbufs.push_back(r.scratch + p.off);
      mids.push_back(compute_of(r.device));
    }
    bcast_all(dbufs, p.len, root, cfg, mids);
    if (!p.len) continue;
    for (const auto& kv : by_device_) {
      DeviceScope ds(kv.first);
      LocalRank& owner = owner_of(kv.first);
      const cudaEvent_t done = event(owner, ev[kv.first]++);
      ck(cudaEventRecord(done, compute_of(kv.first)), "cudaEventRecord");
      ck(cudaStreamWaitEvent(owner.copy_out, done, 0), "cudaStreamWaitEvent");
      for (int li : kv.second) {
        LocalRank& r = local_[static_cast<std::size_t>(li)];
        if (r.rank == root) continue;
        ck(cudaMemcpyAsync(static_cast<std::uint8_t*>(host_bufs[static_cast<std::size_t>(r.rank)]) + p.off,
                           r.scratch + p.off, p.len, cudaMemcpyDeviceToHost, owner.copy_out), "D2H");
      }
    }
  }
  std::vector<int> all;
  for (const auto& kv : by_device_) {
    DeviceScope ds(kv.first);
    LocalRank& owner = owner_of(kv.first);
    ck(cudaStreamSynchronize(owner.copy_out), "synchronize");
    ck(cudaStreamSynchronize(owner.host_mid), "synchronize");
    ck(cudaStreamSynchronize(owner.copy_in), "synchronize");
    all.insert(all.end(), kv.second.begin(), kv.second.end());
  }
  const auto t1 = std::chrono::steady_clock::now();
  std::vector<RankFailure> f;
  for (int li : all) {
    const dev::ErrorRecord& e = *local_[static_cast<std::size_t>(li)].err_host;
    if (e.code != 0) f.push_back(RankFailure{local_[static_cast<std::size_t>(li)].rank, describe(e)});
  }
  if (!f.empty()) {
    broken_ = true;
    throw AggregateRankError(std::move(f));
  }
  return std::chrono::duration<double>(t1 - t0).count();
}

void Group::barrier(int li, cudaStream_t stream) {
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  if (by_device_.at(r.device).size() > 1) {
    throw std::invalid_argument("ranks sharing a GPU must use barrier_all");
  }
  dev::BarrierParams B{};
  B.n_ranks = n_;
  B.n_local = 1;
  B.timeout_ns = opt_.timeout_ns;
  B.state[0] = state_of(r);
  B.rank[0] = r.rank;
  B.bar[0] = r.region + 4 * region_stride();
  B.peers[0] = r.d_peers;
  B.err[0] = r.err_dev;
  DeviceScope ds(r.device);
  ck(static_cast<cudaError_t>(launch_barrier(B, stream)), "launch(barrier)");
}

void Group::barrier_all(const std::vector<cudaStream_t>& streams) {
  for (const auto& kv : by_device_) {
    dev::BarrierParams B{};
    B.n_ranks = n_;
    B.n_local = static_cast<int>(kv.second.size());
    B.timeout_ns = opt_.timeout_ns;
    for (std::size_t i = 0; i < kv.second.size(); ++i) {
      LocalRank& r = local_[static_cast<std::size_t>(kv.second[i])];
      B.state[i] = state_of(r);
      B.rank[i] = r.rank;
      B.bar[i] = r.region + 4 * region_stride();
      B.peers[i] = r.d_peers;
      B.err[i] = r.err_dev;
    }
    const int first = kv.second.front();
    cudaStream_t s = streams.empty() ? local_[static_cast<std::size_t>(first)].stream
                                     : streams[static_cast<std::size_t>(first)];
    DeviceScope ds(kv.first);
    ck(static_cast<cudaError_t>(launch_barrier(B, s)), "launch(barrier)");
  }
}

void* Group::mem_alloc(int li, std::size_t bytes) {
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  if (!r.heap) throw std::invalid_argument("this communicator has no symmetric heap");
  const std::size_t at = (r.heap_used + 255) / 256 * 256;
  if (at + bytes > r.heap_bytes) throw std::invalid_argument("symmetric heap exhausted");
  r.heap_used = at + bytes;
  return r.heap + at;
}

void Group::mem_reset(int li) {
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  r.heap_used = 0;
  r.scratch = nullptr;
  r.scratch_bytes = 0;
}

void Group::set_provenance(int li, unsigned long long* counters) {
  local_.at(static_cast<std::size_t>(li)).prov = counters;
}

void Group::set_trace(int li, unsigned long long* records, std::uint32_t per_lane) {
  LocalRank& r = local_.at(static_cast<std::size_t>(li));
  r.trace = records;
  r.trace_cap = records ? per_lane : 0;
}

std::uint64_t Group::launches(int li) const { return local_.at(static_cast<std::size_t>(li)).launches; }

}  // namespace bcl
