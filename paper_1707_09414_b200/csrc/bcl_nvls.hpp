// bcl_nvls — NVLS multicast broadcast (no reference
// counterpart: the reference is CPU-only).
//
// One multicast object per communicator, bound to a staging ring on every GPU
// of the group. The root streams the message through the multicast address
// (multimem.st: the NVSwitch replicates every store to every GPU's copy, so
// the root's NVLink egress carries M once and receivers only ingest); every
// receiver copies its GPU's copy of each piece into its own buffer. All
// signalling lives in the multicast-bound memory too: the root bumps a
// per-slot `ready` counter and every receiver a per-slot `done` counter with
// multimem.red (each GPU polls its local copy), so the path needs no peer
// pointers at all.
//
// Ring geometry: a 64 MiB ring of `slots` slots (slot size: the nvls_slot
// option); the message is cut into pieces (<= one slot) identically on every
// rank; piece k of a call occupies global sequence number seq_base + k,
// slot = seq % slots, round = seq / slots. The sequence lives in each rank's
// device-side call state (CallState::nvls_seq), advanced by the rank's last
// CTA, identical on every rank.
// Writers wait for done[slot] >= n_recv * round, readers for
// ready[slot] >= round + 1 (monotone counters: never reset).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "bcl_device.cuh"

namespace bcl {

namespace dev {

constexpr std::uint64_t kNvlsRingBytes = 64ull << 20;  // staging ring per GPU
constexpr std::uint32_t kNvlsMaxSlots = 4096;            // ring / slot bytes (slot >= 16 KiB)
constexpr std::uint32_t kNvlsCtlBytes = 128u << 10;     // ready[kNvlsMaxSlots] | done[kNvlsMaxSlots] | ll_done[2],
                                                         // then the ring, then the LL area
constexpr std::uint32_t kNvlsLLDone = 2 * kNvlsMaxSlots;  // word index of ll_done[2]
constexpr std::uint64_t kNvlsLLMaxBytes = 2ull << 20;     // NVLS-LL: largest message (8-byte payload per 16-byte line)
constexpr std::uint64_t kNvlsLLLines = kNvlsLLMaxBytes / 8;  // lines per half of the LL area
constexpr std::uint32_t kNvlsDefaultSlot = 256u << 10;  // 1 GiB at n = 4: 2007 us vs 2350 us with 128 KiB (profiles/round2/nvls)
constexpr int kNvlsThreads = 512;
constexpr int kNvlsDefaultCtas = 148;                    // pieces per wave (identical on every rank)
constexpr std::uint64_t kNvlsMinPiece = 16u << 10;

struct NvlsRank {
  int rank;
  int is_root;
  std::uint8_t* buf;
  ErrorRecord* err;
  int* abort;
  CallState* state;         // nvls_seq / nvls_ll_* read at start, advanced by the rank's last CTA
};

template <int NL>
struct NvlsParamsT {
  int n_local;
  int ctas;                 // CTAs per local rank
  int n_recv;               // receivers of every piece (n - 1)
  std::uint32_t pieces;
  std::uint64_t bytes;
  std::uint64_t piece_bytes;
  std::uint32_t slots;      // ring slots (kNvlsRingBytes / slot_bytes)
  std::uint32_t slot_bytes;
  std::uint64_t timeout_ns;
  std::uint32_t strict;     // fence.acq_rel.sys before every counter bump
  std::uint8_t* mc;         // multicast mapping of the bound range (this GPU)
  std::uint8_t* uc;         // this GPU's own copy
  NvlsRank ranks[NL];
};
using NvlsParams = NvlsParamsT<kMaxLocal>;

// NVLS-LL: small messages as 16-byte LL lines {4 B payload, flag, 4 B
// payload, flag} written once through the multicast address into every
// GPU's LL area (half = epoch & 1); receivers poll their own copy, no fence
// and no per-piece release. ll_done[half] counts receiver CTAs that finished
// reading that half (multimem.red), so the root reuses it safely.
template <int NL>
struct NvlsLLParamsT {
  int n_local;
  int ctas;                  // CTAs per local rank (identical on every GPU)
  int n_recv;                // receiving ranks (each reports `ctas` CTAs per call)
  std::uint32_t lines;
  std::uint64_t bytes;
  std::uint64_t timeout_ns;
  std::uint8_t* mc;
  std::uint8_t* uc;
  NvlsRank ranks[NL];
};
using NvlsLLParams = NvlsLLParamsT<kMaxLocal>;

}  // namespace dev

int launch_nvls(const dev::NvlsParams& p, void* stream);
int launch_nvls_ll(const dev::NvlsLLParams& p, void* stream);
int nvls_occupancy(int* blocks_per_sm);
int nvls_ll_occupancy(int* blocks_per_sm);

// Piece geometry of an M-byte call (identical on every rank, given the same
// slot size and wave width): about `wave` pieces per wave, each <= one slot.
struct NvlsGeometry {
  std::uint64_t piece_bytes{};
  std::uint32_t pieces{};
};
NvlsGeometry nvls_geometry(std::uint64_t bytes, std::uint32_t slot_bytes, int wave);

// The multicast object and its per-device bindings owned by one process.
class NvlsTeam {
 public:
  ~NvlsTeam();
  // Whether the device (and driver) support multicast objects; `why` says
  // why not.
  static bool supported(int device, std::string* why);
  // One process drives every GPU of the team.
  static std::unique_ptr<NvlsTeam> create_local(const std::vector<int>& devices);

  // One process per GPU. The owner (rank 0) creates the object for n GPUs and
  // exports it: a fabric handle when the driver allows, else a POSIX fd served
  // over an abstract Unix socket to the n - 1 importers.
  static std::unique_ptr<NvlsTeam> create_owner(int n_devices, int device);
  static constexpr std::size_t kBlobBytes = 128;
  void export_blob(std::uint8_t out[kBlobBytes]) const;
  static std::unique_ptr<NvlsTeam> import(const std::uint8_t blob[kBlobBytes], int device);
  // Per-process steps after every rank imported: add this GPU, then bind and
  // map (after every rank added its GPU; the caller agrees between steps).
  void add_device();
  void bind_and_map();

  std::uint8_t* mc(int device) const;
  std::uint8_t* uc(int device) const;
  std::uint64_t size() const { return size_; }

  const std::string& handle_kind() const { return kind_; }

 private:
  NvlsTeam() = default;
  struct Binding {
    int device{-1};
    unsigned long long mem{};  // CUmemGenericAllocationHandle
    unsigned long long uc{};   // CUdeviceptr
    unsigned long long mc{};
    bool bound{false};
  };
  void bind_device(Binding& b);
  unsigned long long handle_{};  // CUmemGenericAllocationHandle of the multicast object
  std::uint64_t size_{};
  std::uint64_t gran_{};
  std::vector<Binding> bindings_;
  std::string kind_;             // "local", "fabric" or "fd"
  std::uint8_t fabric_[64]{};
  std::string socket_name_;
  int fd_{-1};
  int listen_fd_{-1};
  std::thread server_;
  int n_devices_{0};
};

}  // namespace bcl
