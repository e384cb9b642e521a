// bcl_device.cuh — the host/device contract of the broadcast executor.
//
// The per-rank copy/forward loop of the reference (execute_rank,
// proj/src/runtime.cpp:32-64) runs on the GPU as a set of independent
// *lanes* (one warp each). A chunk is cut into Q slices; lane l serves slice
// (l % Q) of every chunk c with c % (L/Q) == l / Q, walking the rank's event
// list in order. A Recv(peer, c) waits for the peer's per-lane ready counter
// to reach this pull's index, then copies the slice straight out of the
// peer's buffer (NVLink P2P load, or a local load when ranks share a GPU); a
// Send(peer, c) release-stores this lane's counter into the peer's flag
// array. Because sender and receiver filter the same per-pair ordered event
// sequence with the same lane predicate, the i-th send of lane l to d is the
// i-th receive of lane l at d from the sender: one monotone 64-bit counter per
// (src, lane) suffices, tagged with the call epoch in its upper 32 bits so
// flags never need resetting. Consumers ack after their last pull so the
// producer's kernel cannot finish (and its buffer cannot be reused) while a
// downstream lane still reads it.
#pragma once

#include <cstddef>
#include <cstdint>

namespace bcl {
namespace dev {

constexpr int kMaxLocal = 16;    // ranks served by one launch (ranks sharing a GPU)
constexpr int kMaxEvents = 64;   // explicit per-rank event list (trees, SRA)
constexpr int kMaxRanks = 64;    // communicator size limit
constexpr int kMaxRegs = 255;    // registered allocations per rank (per-process mode; 8-bit id in the mailbox)
constexpr int kWarpsPerCta = 8;  // lanes per CTA
constexpr int kThreads = (kWarpsPerCta + 1) * 32;  // + one publisher warp
constexpr int kMaxStages = 4;    // bulk-copy stages per copy warp
constexpr std::uint32_t kLLMaxBytes = 2048 * 1024;      // largest LL message (per-group cap may be lower)
constexpr std::uint32_t kLLChainMaxBytes = 8u << 20;     // default LL pipelined-chain cap
constexpr std::uint32_t kLL128Payload = 120;             // payload bytes per 128-byte LL128 line
constexpr int kLL128MaxCtas = 444;  // 3 per SM: +4% at 64 MiB n=4 over one per SM (measured)
constexpr int kLLThreads = 512;
// LL128 landing ring: every warp of the (identical) grid on each rank owns a
// private sub-ring of kLL128Depth groups of 4 lines; the reader returns
// per-warp credits every kLL128Depth / 2 groups. Bounded memory for any
// message size: 7104 warps x 16 x 4 lines x 128 B = 58 MB per rank.
constexpr int kLL128Depth = 16;
constexpr int kLL128WarpsMax = kLL128MaxCtas * (kLLThreads / 32);
constexpr std::uint32_t kLL128RingLines = static_cast<std::uint32_t>(kLL128WarpsMax) * kLL128Depth * 4;
constexpr int kLLMaxCtas = 64;                          // CTAs per rank for one LL call

// Explicit event word: chunk (bits 0-23) | peer (24-30) | recv (31) |
// pair index within the lane class (32-55).
__host__ __device__ inline std::uint64_t pack_event(bool recv, int peer, std::uint32_t chunk,
                                                    std::uint32_t pidx) {
  return static_cast<std::uint64_t>(chunk & 0xFFFFFFu) |
         (static_cast<std::uint64_t>(peer & 0x7F) << 24) |
         (static_cast<std::uint64_t>(recv ? 1u : 0u) << 31) |
         (static_cast<std::uint64_t>(pidx & 0xFFFFFFu) << 32);
}

enum ChunkMode : std::uint32_t {
  kWholeMessage = 0,  // one chunk = the message (direct, chain, knomial)
  kFixedChunks = 1,   // make_chunks(M, C) (chain_pipelined)
  kPartitions = 2,    // partition_chunks(n, M) (scatter_ring_allgather)
};

// Addresses of every peer's state as mapped in *this* rank's address space.
// Region layout of a rank (8-byte words): flags[n][L] | acks[n][L] | mbox[n][L][2]
// | bar[n] | abort | credit[n] | ll_done | chain_credit[n] | wcredit[kLL128WarpsMax]
// | wseq[kLL128WarpsMax] | rseq[kLL128WarpsMax] | pad to 256 B
// | ll[n][2][ll_lines] (16-byte lines, ll_lines = the group's LL cap / 8) | chain LL [2][chain_lines]
// | LL128 ring [kLL128RingLines] (128-byte lines).
struct PeerTable {
  std::uint64_t* flags[kMaxRanks];  // peer's flags array (index [my_rank][lane])
  std::uint64_t* acks[kMaxRanks];   // peer's acks array  (index [my_rank][lane])
  std::uint64_t* mbox[kMaxRanks];   // peer's mailbox     (16-byte slots, index [my_rank][lane])
  std::uint64_t* bar[kMaxRanks];    // peer's barrier slots (index [my_rank])
  std::uint64_t addr_base[kMaxRanks];  // added to a mailbox value from that peer
  std::uint64_t* credit[kMaxRanks];    // peer's LL credit array (index [my_rank])
  uint4* ll[kMaxRanks];                // peer's LL landing area (index [my_rank][half][line])
  std::uint64_t* wcredit[kMaxRanks];   // peer's LL128 per-warp ring credits (written by its successor)
  const std::uint64_t* regs;           // per-process mode: [peer][kMaxRegs] registered allocation bases as mapped
                                       // here (device array), else null
};

// Per-rank call state, in the rank's own region (device memory). Every
// kernel reads it when it starts and the last CTA of the rank to finish
// advances it, so epochs and the line protocols' reuse bookkeeping live on
// the device: a CUDA graph that replays a captured broadcast sees fresh
// values on every replay (kernel parameters hold only the call's shape).
struct CallState {
  unsigned long long epoch;              // last call epoch (lane executor, LL, LL128)
  unsigned long long bar_epoch;          // last device barrier
  unsigned long long ll_last_direct[2];  // LL direct: last epoch this rank wrote each half as the root
  unsigned long long ll_last_chain[2];   // LL chain: last epoch this rank wrote each half to its successor
  unsigned long long ll_last_ring;       // LL128: last epoch this rank wrote into its successor's ring
  unsigned long long finished;           // CTAs of this rank's running launch that finished
  unsigned long long nvls_seq;           // NVLS ring sequence (identical on every rank)
  unsigned long long nvls_ll_calls;      // NVLS-LL calls
  unsigned long long nvls_ll_reports[2]; // NVLS-LL receiver-CTA reports expected per half so far
  unsigned long long pad[4];
};
constexpr int kCallStateWords = sizeof(CallState) / 8;

struct ErrorRecord {  // host-mapped, written by the first failing lane
  int code;           // 0 ok, 1 timeout, 2 aborted
  int rank;
  int peer;
  int lane;
  unsigned long long chunk;
  unsigned long long observed;
  unsigned long long expected;
};

struct RankWork {
  int rank;                      // global rank id
  int n_events;                  // explicit list length; -1 = implicit pipelined chain
  std::uint8_t* buf;             // this rank's buffer (device)
  std::uint64_t pub;             // mailbox value naming buf to consumers
  std::uint64_t* flags;          // local flags[n][L]
  std::uint64_t* acks;           // local acks[n][L]
  std::uint64_t* mbox;           // local mbox[n][L] (16-byte slots)
  const PeerTable* peers;        // device-resident
  ErrorRecord* err;              // host-mapped error record of this rank (written once, on failure)
  int* abort;                    // device-memory abort word polled by waiting lanes
  unsigned long long* prov;      // optional provenance: bytes pulled per [src][chunk]
  unsigned long long* trace;     // optional timeline: [lane][trace_cap][4] globaltimer stamps
  std::uint32_t trace_cap;
  CallState* state;              // this rank's call state (epoch read at start, advanced at the end)
  std::uint64_t events[kMaxEvents];
};

// Launch parameters for a launch serving NL ranks. NL = 1 (one rank per GPU,
// the production shape) keeps the parameter block small for launch latency;
// NL = kMaxLocal serves ranks that share a GPU (emulation, tests).
template <int NL>
struct LaunchParamsT {
  int n_ranks;
  int root;
  int n_local;
  int lanes;          // L: lanes per rank (identical on every rank of the comm)
  int slices;         // Q: slices per chunk, divides L
  int ctas_per_rank;  // CTAs launched per local rank (active lanes only)
  std::uint32_t chunk_mode;
  std::uint32_t n_chunks;
  std::uint64_t bytes;
  std::uint64_t chunk_bytes;
  std::uint64_t slice_bytes;  // multiple of 16
  std::uint64_t epoch;        // the call's epoch: filled in on the device from CallState (kernel-side copy)
  std::uint64_t timeout_ns;
  std::uint32_t poll_ns;      // __nanosleep between polls (0 = spin)
  std::uint32_t sys_scope;    // 1: peers on other GPUs; 0: every rank on this GPU
  std::uint32_t strict_sys;   // 1: system-scope fence before every flag (see run_publisher)
  std::uint32_t stage_bytes;  // bytes per bulk-copy stage; 0 = vector loads only
  std::uint32_t stages;       // bulk-copy stages per copy warp (2..kMaxStages)
  std::uint32_t push;         // chain: producers store into the consumer's buffer
  std::uint32_t eager_post;   // bulk chain: publish each chunk as soon as its store completes
  std::uint32_t writer_fence; // 1: each copy warp fences its own data before the hand-off; 0: the publisher does
  RankWork ranks[NL];
};
using LaunchParams = LaunchParamsT<kMaxLocal>;

// LL (low-latency) protocol for small messages on the `direct` schedule: the
// root writes 16-byte lines {4 B payload, epoch, 4 B payload, epoch} into
// every receiver's landing area for that source; receivers poll the lines
// (8-byte halves are single-copy atomic) and copy the payload out. No fence,
// no pull round trip, no ack wait; epoch-parity double buffering plus lazily
// written credits (receiver -> root, "done with epoch e") guard reuse.
struct LLRank {
  int rank;
  std::uint8_t* buf;
  uint4* ll;                  // local landing area base
  std::uint64_t* credit;      // local credit array [n] of this call's kind (direct, or chain: LL and LL128)
  std::uint64_t* wcredit;     // local LL128 per-warp ring credits [kLL128WarpsMax] (written by the successor)
  std::uint64_t* wseq;        // local: groups each warp has written into the successor's ring, all calls
  std::uint64_t* rseq;        // local: groups each warp has read from this rank's ring, all calls
  const PeerTable* peers;
  ErrorRecord* err;
  int* abort;
  CallState* state;           // epoch, the half-reuse bookkeeping and the finished-CTA count
};

struct LLHeader {
  int n_ranks;
  int root;
  int n_local;
  int ctas;                   // CTAs per rank
  std::uint32_t lines;        // lines of the launch (every segment's)
  std::uint64_t bytes;        // one segment: its bytes
  std::uint32_t area_lines;   // lines per (source, half) landing area of the direct schedule
  std::uint32_t chain;        // 0 direct, 1 pipelined chain on 16-byte LL lines, 2 chain on 128-byte LL128 lines,
                              // 3 direct on 128-byte LL128 lines (in the LL128 direct areas)
  std::uint32_t chain_lines;  // lines per half of the chain landing area (after the direct areas)
  std::uint32_t chain128_lines;  // 128-byte lines of the LL128 ring (kLL128RingLines)
  std::uint32_t chain128_area;   // its offset from the LL base in 16-byte units (128-byte aligned)
  std::uint32_t d128_area;       // LL128 direct areas [n][2][d128_lines]: offset from the LL base, 16-byte units
  std::uint32_t d128_lines;      // 128-byte lines per (source, half)
  std::uint64_t timeout_ns;
  std::uint32_t coop;            // LL128, one rank per GPU: cooperative launch (co-residency guaranteed)
  int n_seg;                     // messages fused into this launch (bcl_group_*); 1 = an ordinary call
};

// A launch of the line protocols may carry up to NS messages ("segments",
// fused by bcl_group_start/end): segment s owns lines [seg_line[s],
// seg_line[s + 1]) and its own buffer on every rank. NS = 1 is an ordinary
// call (the segment is R.buf / bytes; the tables stay unused).
constexpr int kMaxSegs = 32;        // one rank per launch
constexpr int kMaxSegsShared = 8;   // ranks sharing a GPU (a 16-rank parameter block; no spills)
constexpr int max_segs(int n_local) { return n_local > 1 ? kMaxSegsShared : kMaxSegs; }
template <int NL, int NS = 1>
struct LLParamsT : LLHeader {
  std::uint32_t seg_line[NS + 1];
  std::uint64_t seg_bytes[NS];
  LLRank ranks[NL];
  std::uint8_t* seg_buf[NL][NS];
};
using LLParams = LLParamsT<kMaxLocal, kMaxSegs>;  // host-side superset; launchers copy into the smallest fit

// Every rank of the group on this GPU (one process): the pipelined chain's
// hops run as one flag-free kernel. Each warp takes byte ranges ("items") of
// the message and performs every hop for its item in chain order: logical
// rank h copies the item from logical rank h - 1's buffer into its own, the
// next hop reading what the previous one just wrote (an L2 hit). Same bytes
// read and written per hop as the chain across GPUs; no flags, no waits, no
// pipeline fill.
struct LocalChainParams {
  int n_ranks;
  std::uint32_t n_chunks;
  std::uint64_t bytes;
  std::uint64_t chunk_bytes;
  std::uint64_t item_bytes;                  // per warp work unit, multiple of 16, <= chunk
  std::uint8_t* buf[kMaxLocal];              // by logical rank (root first)
  int rank[kMaxLocal];                       // global rank of each logical rank
  unsigned long long* prov[kMaxLocal];       // optional provenance of each logical rank
  unsigned long long* claim;                 // dynamic item claims: a zeroed counter this launch owns
                                             // (the last claimer re-zeroes it), or null: static
};

struct BarrierParams {
  int n_ranks;
  int n_local;
  std::uint64_t timeout_ns;
  CallState* state[kMaxLocal];          // bar_epoch read and advanced on the device
  int rank[kMaxLocal];
  std::uint64_t* bar[kMaxLocal];        // local barrier slots
  const PeerTable* peers[kMaxLocal];
  ErrorRecord* err[kMaxLocal];
};

}  // namespace dev

// Launchers (bcl_kernels.cu). Return cudaError_t as int.
// Fills attr[] (room for 2) for a launch: cooperative, or programmatic stream
// serialization; returns the count. (cudaLaunchAttribute from cuda_runtime.h.)
int fill_launch_attrs(struct cudaLaunchAttribute_st* attr, int cooperative);
int launch_bcast(const dev::LaunchParams& p, int cooperative, void* stream);
int launch_barrier(const dev::BarrierParams& p, void* stream);
int launch_ll(const dev::LLParams& p, void* stream);
int launch_peer_copy(std::uint8_t* dst, const std::uint8_t* src, std::uint64_t len, void* stream);
int launch_local_chain(const dev::LocalChainParams& p, int ctas, void* stream);
int local_chain_occupancy(int* blocks_per_sm);
int ll128_occupancy(int* blocks_per_sm, int shared);  // shared: the kernel for ranks sharing a GPU
int bcast_kernel_occupancy(int* blocks_per_sm, std::size_t smem);
std::size_t bcast_smem_bytes(std::uint32_t stages, std::uint32_t stage_bytes);
int prepare_bcast_kernels(std::size_t smem);

}  // namespace bcl
