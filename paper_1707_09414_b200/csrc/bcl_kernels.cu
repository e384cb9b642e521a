// bcl_kernels.cu — sm_100a broadcast executors (see bcl_device.cuh).
//
// bcast_kernel — the lane executor. One launch per GPU serves every rank that
// GPU hosts (normally one). A CTA holds kWarpsPerCta *copy warps* (the lanes)
// and one *publisher warp*:
//  * a copy warp owns slice q = lane % Q of the chunks c with
//    c % (L/Q) == lane / Q and walks its rank's schedule: it waits for the
//    upstream peer's per-lane counter, pulls the slice straight out of the
//    peer's buffer (TMA bulk copies through shared-memory stages across
//    GPUs, 16-byte vector loads otherwise), fences its own completed stores
//    (gpu scope) and hands "store value v to flag f" to the publisher through
//    a shared-memory ring (CTA-scope release);
//  * the publisher drains the rings of its CTA and issues the remote flag
//    stores. It never fences (a fence would wait for its previous remote flag
//    stores, ~16 us under NVLink load) except in push / strict modes.
// ll_kernel / ll128_kernel — line protocols (flag travels with the data):
//   the direct schedule's LL push and the pipelined chain forwarded line by
//   line (16-byte LL lines, 128-byte LL128 lines across GPUs).
// local_chain_kernel — every rank on this GPU: the chain's hops fused per item.
// barrier_kernel — device barrier across ranks.
//
// Data never leaves HBM / NVLink: no staging buffers, no cudaMemcpy, no NCCL.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <algorithm>

#include "bcl_device.cuh"

// 16-byte loads a lane issues before its stores (bytes in flight per warp =
// 512 x BCL_LDG_UNROLL), and the co-resident CTAs per SM the shared-GPU
// kernel is compiled for (register budget).
#ifndef BCL_LDG_UNROLL
#define BCL_LDG_UNROLL 8
#endif
#ifndef BCL_SHARED_MIN_BLOCKS
#define BCL_SHARED_MIN_BLOCKS 2
#endif

namespace bcl {
namespace dev {
namespace {

constexpr int kRing = 16;  // pending publishes per copy warp

// Programmatic dependent launch: with the stream-serialization attribute a
// kernel may be scheduled before the previous kernel of its stream has
// finished; everything it reads (the call state, user buffers) may be that
// kernel's output, so it waits here first (a no-op without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Whether this CTA is the last of its rank's `ctas` to finish (a single-CTA
// launch is, without the round trip of the counter).
__device__ __forceinline__ bool last_cta(CallState* st, int ctas) {
  if (ctas == 1) return true;
  if (atomicAdd(&st->finished, 1ull) + 1 != static_cast<unsigned long long>(ctas)) return false;
  st->finished = 0;
  return true;
}

__device__ __forceinline__ std::uint64_t ld_relaxed_sys(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ std::uint64_t ld_acquire_sys(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ std::uint64_t ld_relaxed_gpu(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ std::uint64_t ld_acquire_gpu(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(std::uint64_t* p, std::uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ std::uint32_t ld_acquire_cta(const std::uint32_t* p) {
  std::uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
               : "=r"(v)
               : "r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(p)))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(std::uint32_t* p, std::uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(
                   static_cast<std::uint32_t>(__cvta_generic_to_shared(p))),
               "r"(v)
               : "memory");
}
__device__ __forceinline__ std::uint64_t globaltimer() {
  std::uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ std::uint8_t ld_u8(const std::uint8_t* p) {
  unsigned short v;
  asm volatile("ld.global.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<std::uint8_t>(v);
}
__device__ __forceinline__ uint4 ld_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}


__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\nBCL_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra BCL_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(std::uint64_t* bar, std::uint32_t parity) {  // non-blocking
  std::uint32_t ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// TMA-engine bulk copies (SASS UBLKCP): global -> shared completing on an
// mbarrier, and shared -> global tracked by bulk async-groups.
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gsrc, std::uint32_t bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem, std::uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Shared-memory hand-off from the copy warps to the publisher warp.
struct Publication {
  std::uint64_t* addr;
  std::uint64_t value;
};
struct CtaShared {
  Publication ring[kWarpsPerCta][kRing];
  std::uint64_t full[kWarpsPerCta][kMaxStages];  // bulk-copy mbarriers (one per stage)
  std::uint32_t tail[kWarpsPerCta];  // written by copy warp w (release)
  std::uint32_t head[kWarpsPerCta];  // written by the publisher (release)
  std::uint32_t done;                // copy warps finished enqueueing
};

struct Ctx {
  const LaunchParamsT<1>* P;
  const RankWork* W;
  CtaShared* sh;
  int lane_id;         // 0..31
  int warp;            // copy warp index within the CTA
  int ell;             // lane (copy warp) index within the rank
  std::uint32_t tail;  // private copy of sh->tail[warp] (lane 0)
  std::uint8_t* stage; // 2 x stage_bytes of dynamic shared memory (bulk path), or null
  std::uint64_t epoch; // this call's epoch (from the rank's device-side call state)
};

// Record the first failure of this rank; every waiting lane then drains out.
__device__ void fail(const Ctx& c, int code, int peer, std::uint64_t chunk, std::uint64_t seen,
                     std::uint64_t want) {
  atomicExch(c.W->abort, 1);
  ErrorRecord* e = c.W->err;
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->rank = c.W->rank;
    e->peer = peer;
    e->lane = c.ell;
    e->chunk = chunk;
    e->observed = seen;
    e->expected = want;
    __threadfence_system();
  }
}

// Warp-wide wait until *p >= target. Lane 0 polls (relaxed, with back-off);
// then every thread performs its own system-scope acquire so its later loads
// observe the producer's data. Returns false on timeout / abort.
__device__ bool wait_geq(const Ctx& c, const std::uint64_t* p, std::uint64_t target, int peer,
                         std::uint64_t chunk) {
  int ok = 1;
  // Every rank on one GPU: gpu-scope polling/acquire is the complete ordering.
  const bool sys = c.P->sys_scope != 0;
  if (c.lane_id == 0) {
    std::uint64_t v = sys ? ld_relaxed_sys(p) : ld_relaxed_gpu(p);
    if (v < target) {
      const std::uint64_t t0 = globaltimer();
      unsigned spins = 0;
      while ((v = sys ? ld_relaxed_sys(p) : ld_relaxed_gpu(p)) < target) {
        if (c.P->poll_ns) __nanosleep(c.P->poll_ns);
        if ((++spins & 255u) == 0) {
          if (*(volatile int*)c.W->abort != 0) {
            ok = 0;
            break;
          }
          if (globaltimer() - t0 > c.P->timeout_ns) {
            fail(c, 1, peer, chunk, v, target);
            ok = 0;
            break;
          }
        }
      }
    }
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  if (ok) (void)(sys ? ld_acquire_sys(p) : ld_acquire_gpu(p));
  __syncwarp();
  return ok != 0;
}

// Writer-side fence (writer_fence = 1): the copy warp that produced the data
// fences it before handing the flag to the publisher. A fence waits for the
// issuing warp's outstanding writes; in the publisher that meant the previous
// batch's remote flag stores, whose acknowledgements queue behind loaded
// NVLink traffic (measured ~16 us per batch at n = 4, 64 MiB); the copy warp
// has only its own, already completed, data writes outstanding.
// writer_fence = 1 (default): gpu scope. The flag names data in this GPU's
// own HBM, which NVLink readers reach through this GPU's L2 (its point of
// coherence), so data performed at gpu scope is what a peer reads once it
// sees the flag -- a hardware property, not a PTX-model guarantee (DESIGN.md
// §5 "Memory ordering"; stress-tested across GPUs). writer_fence = 2 fences
// at system scope, the textbook release: in a middle rank of the chain that
// fence also waits for the warp's in-flight TMA pulls from its upstream
// (64 MiB at n = 4: 376 us against 126-145 us), so it is an option.
__device__ __forceinline__ void writer_fence(const LaunchParamsT<1>& P) {
  if (P.writer_fence == 2) {
    fence_acq_rel_sys();
  } else if (P.writer_fence == 1) {
    fence_acq_rel_gpu();
  }
}

// Queue "*addr = value" behind this warp's preceding stores. The warp
// barrier orders every lane's stores before lane 0's fence and CTA-scope
// release; the flag store follows in the publisher.
__device__ void publish(Ctx& c, std::uint64_t* addr, std::uint64_t value) {
  __syncwarp();
  if (c.lane_id == 0) {
    writer_fence(*c.P);
    while (c.tail - ld_acquire_cta(&c.sh->head[c.warp]) >= static_cast<std::uint32_t>(kRing)) {
      __nanosleep(32);
    }
    c.sh->ring[c.warp][c.tail % kRing] = Publication{addr, value};
    c.tail += 1;
    st_release_cta(&c.sh->tail[c.warp], c.tail);
  }
  __syncwarp();
}

// Mailboxes are 16-byte slots {epoch16 << 48 | value, epoch}: both halves
// carry the call's epoch, so a consumer can validate the slot itself and the
// producer needs no system-scope fence between its mailbox store and its
// first flag (that fence cost ~4-6 us at lane start, profiles/round1/mbox).
__device__ __forceinline__ void st_mbox(std::uint64_t* slot, std::uint64_t value, std::uint64_t epoch) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1,%2};" ::"l"(slot),
               "l"(value | ((epoch & 0xFFFFull) << 48)), "l"(epoch)
               : "memory");
}
// Warp-collective: lane 0 polls the mailbox until it carries this call's
// epoch in both halves; every lane gets the value.
__device__ std::uint64_t read_mbox(const Ctx& c, const std::uint64_t* slot, int peer) {
  unsigned long long value = 0;
  if (c.lane_id == 0) {
    const std::uint64_t epoch = c.epoch;
    const std::uint64_t hi = (epoch & 0xFFFFull) << 48;
    const std::uint64_t t0 = globaltimer();
    unsigned spins = 0;
    for (;;) {
      std::uint64_t a, b;
      asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(slot) : "memory");
      if (b == epoch && (a & 0xFFFF000000000000ull) == hi) {
        value = a & 0x0000FFFFFFFFFFFFull;
        break;
      }
      if ((++spins & 255u) == 0) {
        if (*(volatile int*)c.W->abort != 0) break;
        if (globaltimer() - t0 > c.P->timeout_ns) {
          fail(c, 1, peer, 0, b, epoch);
          break;
        }
      }
    }
  }
  return __shfl_sync(0xffffffffu, value, 0);
}

// A peer buffer address from its mailbox value: a raw pointer (one process,
// UVA), a symmetric-heap offset (per-process ranks), or, with the registration
// id in bits 40-47, an offset into a registered allocation of that peer as
// mapped here (bcl_comm_register_*).
__device__ __forceinline__ std::uint64_t peer_addr(const RankWork& W, int peer, std::uint64_t v) {
  const std::uint64_t id = v >> 40;
  if (W.peers->regs != nullptr && id != 0) {
    return W.peers->regs[static_cast<std::size_t>(peer) * kMaxRegs + id - 1] + (v & ((1ull << 40) - 1));
  }
  return W.peers->addr_base[peer] + v;
}

// A remote store straight from the copy warp, for hand-offs that need no
// fence: the head's "every chunk ready" (its data was written by earlier
// stream work) and a consumer's final ack (its reads have completed). Safe to
// issue here because the lane issues no fence afterwards, which would wait for
// this store's acknowledgement; skips the publisher hop (~1-2 us).
__device__ __forceinline__ void publish_direct(const Ctx& c, std::uint64_t* addr, std::uint64_t value) {
  __syncwarp();
  if (c.lane_id == 0) st_relaxed_sys(addr, value);
  __syncwarp();
}

// The publisher warp (lane 0): drain every ring, one fence per batch.
__device__ void run_publisher(const LaunchParamsT<1>& P, CtaShared* sh, const RankWork& W, int cta) {
  if ((threadIdx.x & 31) != 0) return;
  std::uint32_t head[kWarpsPerCta] = {};
  std::uint32_t stamped = 0;  // timeline: lanes whose first hand-off has been stamped
  for (;;) {
    const std::uint32_t done = ld_acquire_cta(&sh->done);
    std::uint32_t tail[kWarpsPerCta];
    bool any = false;
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; ++w) {
      tail[w] = ld_acquire_cta(&sh->tail[w]);
      any |= tail[w] != head[w];
    }
    if (!any) {
      if (done == static_cast<std::uint32_t>(kWarpsPerCta)) return;
      __nanosleep(20);
      continue;
    }
    // Every flag published here names data in this GPU's own memory, which
    // peers read through this GPU's L2 (its point of coherence): once the
    // stores are performed at gpu scope they are visible to NVLink readers.
    // strict_sys keeps the textbook system-scope release instead.
    const std::uint64_t t_seen = W.trace ? globaltimer() : 0;
    if (!P.writer_fence) {
      if (P.strict_sys || P.push) {  // push mode: the published data is in the peer's memory
        fence_acq_rel_sys();
      } else {
        fence_acq_rel_gpu();
      }
    }
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; ++w) {
      for (std::uint32_t i = head[w]; i != tail[w]; ++i) {
        const Publication e = sh->ring[w][i % kRing];
        st_relaxed_sys(e.addr, e.value);
      }
      if (W.trace && head[w] != tail[w] && !((stamped >> w) & 1u) && W.trace_cap > 0) {
        stamped |= 1u << w;  // lifecycle record fields 1/2: first batch seen / stored
        unsigned long long* rec =
            W.trace + (static_cast<std::size_t>(cta * kWarpsPerCta + w) * W.trace_cap + W.trace_cap - 1) * 4;
        rec[1] = t_seen;
        rec[2] = globaltimer();
      }
      if (head[w] != tail[w]) {
        head[w] = tail[w];
        st_release_cta(&sh->head[w], head[w]);
      }
    }
  }
}

// Warp copy of bytes [lo, hi) from src to dst (same offsets in both buffers).
// Every 16-byte load of a batch is issued before the batch's stores, so a
// batch costs one load round trip however short the slice is.
__device__ void warp_copy(const Ctx& c, const std::uint8_t* src, std::uint8_t* dst, std::uint64_t lo,
                          std::uint64_t hi) {
  if (hi <= lo) return;
  const int t = c.lane_id;
  const std::uintptr_t s0 = reinterpret_cast<std::uintptr_t>(src + lo);
  const std::uintptr_t d0 = reinterpret_cast<std::uintptr_t>(dst + lo);
  if (((s0 ^ d0) & 15u) != 0) {  // relative misalignment: byte path
    for (std::uint64_t i = lo + t; i < hi; i += 32) dst[i] = ld_u8(src + i);
    return;
  }
  const std::uint64_t head = (16u - (d0 & 15u)) & 15u;
  const std::uint64_t body_lo = lo + (head < hi - lo ? head : hi - lo);
  if (t < static_cast<int>(body_lo - lo)) dst[lo + t] = ld_u8(src + lo + t);
  const std::uint64_t nvec = (hi - body_lo) / 16;
  const uint4* vs = reinterpret_cast<const uint4*>(src + body_lo);
  uint4* vd = reinterpret_cast<uint4*>(dst + body_lo);
  constexpr int U = BCL_LDG_UNROLL;
  for (std::uint64_t base = 0; base < nvec; base += U * 32) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const std::uint64_t i = base + t + u * 32;
      if (i < nvec) r[u] = ld_v4(vs + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const std::uint64_t i = base + t + u * 32;
      if (i < nvec) st_v4(vd + i, r[u]);
    }
  }
  const std::uint64_t tail_lo = body_lo + nvec * 16;
  if (tail_lo + t < hi) dst[tail_lo + t] = ld_u8(src + tail_lo + t);
}

__device__ __forceinline__ void chunk_range(const LaunchParamsT<1>& P, std::uint32_t ch, std::uint64_t* off,
                                            std::uint64_t* len) {
  if (P.chunk_mode == kFixedChunks) {
    *off = static_cast<std::uint64_t>(ch) * P.chunk_bytes;
    *len = P.bytes - *off < P.chunk_bytes ? P.bytes - *off : P.chunk_bytes;
  } else if (P.chunk_mode == kPartitions) {
    const std::uint64_t n = static_cast<std::uint64_t>(P.n_ranks);
    const std::uint64_t base = P.bytes / n, rem = P.bytes % n;
    *off = ch * base + (ch < rem ? ch : rem);
    *len = base + (ch < rem ? 1 : 0);
  } else {
    *off = 0;
    *len = P.bytes;
  }
}

__device__ __forceinline__ void pull_slice(const Ctx& c, std::uint32_t ch, int q, const std::uint8_t* src,
                                           int src_rank) {
  std::uint64_t off, len;
  chunk_range(*c.P, ch, &off, &len);
  const std::uint64_t lo = static_cast<std::uint64_t>(q) * c.P->slice_bytes;
  if (lo >= len) return;
  const std::uint64_t hi = lo + c.P->slice_bytes < len ? lo + c.P->slice_bytes : len;
  warp_copy(c, src, c.W->buf, off + lo, off + hi);
  if (c.W->prov != nullptr && c.lane_id == 0) {
    atomicAdd(&c.W->prov[static_cast<std::uint64_t>(src_rank) * c.P->n_chunks + ch],
              static_cast<unsigned long long>(hi - lo));
  }
}

__device__ __forceinline__ void trace_pull(const Ctx& c, std::uint32_t k, std::uint64_t t_wait,
                                           std::uint64_t t_ready) {
  const RankWork& W = *c.W;
  if (W.trace && c.lane_id == 0 && k + 1 < W.trace_cap) {
    unsigned long long* rec = W.trace + (static_cast<std::size_t>(c.ell) * W.trace_cap + k) * 4;
    rec[0] = t_wait;
    rec[1] = t_ready;
    rec[2] = globaltimer();
  }
}


__device__ __forceinline__ void bulk_wait_read_n(int n) {
  switch (n) {
    case 0: bulk_wait_read<0>(); break;
    case 1: bulk_wait_read<1>(); break;
    case 2: bulk_wait_read<2>(); break;
    default: bulk_wait_read<3>(); break;
  }
}

// Bulk-copy variant of the chain's middle/tail loop, driven by lane 0 alone.
// Slices of the lane's chunks stream through a ring of S shared-memory
// stages: a TMA load (global -> smem, mbarrier completion) is issued for
// every chunk the upstream has already published while a stage is free, the
// oldest landed slice is written back with a TMA store, and chunks are
// published as soon as their stores have completed (async-group
// accounting). When nothing is in flight the lane finishes and publishes
// what it holds before blocking on the upstream, so downstream progress
// never waits for this rank's upstream. Requires 16-byte aligned slices; the
// ragged end of the message goes byte-wise.
__device__ bool chain_pull_bulk(Ctx& c, int pipe, int q, int ns, std::uint32_t mine, const std::uint64_t* ready,
                                const std::uint8_t* src, std::uint8_t* dst, int prev, bool has_next,
                                std::uint64_t* next_flag, std::uint64_t tag) {
  const LaunchParamsT<1>& P = *c.P;
  const RankWork& W = *c.W;
  std::uint64_t* bars = c.sh->full[c.warp];
  const std::uint32_t sb = P.stage_bytes;
  const std::uint32_t S = P.stages;
  std::uint32_t parity = 0;
  int ok = 1;
  // Slice geometry of the lane's k-th chunk: [gofs, gofs + len), body = 16 B multiple.
  auto geom = [&](std::uint32_t k, std::uint64_t* gofs, std::uint32_t* body, std::uint32_t* len) {
    std::uint64_t off, clen;
    chunk_range(P, pipe + k * ns, &off, &clen);
    const std::uint64_t lo = static_cast<std::uint64_t>(q) * P.slice_bytes;
    const std::uint64_t hi = lo < clen ? (lo + P.slice_bytes < clen ? lo + P.slice_bytes : clen) : lo;
    *gofs = off + lo;
    *len = static_cast<std::uint32_t>(hi - lo);
    *body = *len & ~15u;
  };
  auto stamp = [&](std::uint32_t k, int field) {
    if (W.trace && k + 1 < W.trace_cap) {
      W.trace[(static_cast<std::size_t>(c.ell) * W.trace_cap + k) * 4 + field] = globaltimer();
    }
  };
  std::uint32_t issued = 0, landed = 0, posted = 0;
  auto issue = [&]() {  // load the lane's chunk `issued` into stage issued % S
    if (issued >= S) bulk_wait_read_n(static_cast<int>(landed + S - 1 - issued));  // stage's last store read it
    std::uint64_t g;
    std::uint32_t body, len;
    geom(issued, &g, &body, &len);
    const std::uint32_t st = issued % S;
    fence_proxy_async();  // generic-proxy acquire of the flag before async-proxy reads
    mbar_expect_tx(&bars[st], body);
    if (body) bulk_g2s(c.stage + static_cast<std::size_t>(st) * sb, src + g, body, &bars[st]);
    stamp(issued, 0);
    ++issued;
  };
  auto post = [&](std::uint32_t count) {  // "chunks 0..count-1 forwarded"
    if (count <= posted) return;
    posted = count;
    stamp(count - 1, 3);
    if (!has_next) return;
    fence_proxy_async();  // completed TMA writes ordered before the generic-proxy hand-off
    writer_fence(P);
    while (c.tail - ld_acquire_cta(&c.sh->head[c.warp]) >= static_cast<std::uint32_t>(kRing)) __nanosleep(32);
    c.sh->ring[c.warp][c.tail % kRing] = Publication{next_flag, tag | count};
    c.tail += 1;
    st_release_cta(&c.sh->tail[c.warp], c.tail);
  };
  auto ready_now = [&](std::uint32_t j) {  // chunk j available (a null `ready` means always)
    return ready == nullptr || ld_relaxed_sys(ready) >= (tag | (j + 1));
  };
  auto block_for = [&](std::uint32_t j) -> bool {  // wait until the lane's chunk j is ready upstream
    if (ready == nullptr) return true;
    const std::uint64_t want = tag | (j + 1);
    std::uint64_t v = ld_relaxed_sys(ready);
    if (v < want) {
      const std::uint64_t t0 = globaltimer();
      unsigned spins = 0;
      while ((v = ld_relaxed_sys(ready)) < want) {
        if (P.poll_ns) __nanosleep(P.poll_ns);
        if ((++spins & 255u) == 0) {
          if (*(volatile int*)W.abort != 0) return false;
          if (globaltimer() - t0 > P.timeout_ns) {
            fail(c, 1, prev, pipe + static_cast<std::uint64_t>(j) * ns, v, want);
            return false;
          }
        }
      }
    }
    (void)ld_acquire_sys(ready);
    return true;
  };
  if (c.lane_id == 0) {
    issue();  // chunk 0 was acquired by the caller
    while (landed < mine) {
      // Prefetch every chunk the upstream has already published, up to S in flight.
      while (issued < mine && issued - landed < S && ready_now(issued)) {
        if (ready != nullptr) (void)ld_acquire_sys(ready);
        issue();
      }
      if (issued == landed) {  // nothing in flight: publish what we hold, then block
        bulk_wait<0>();
        post(landed);
        if (!block_for(issued)) {
          ok = 0;
          break;
        }
        issue();
        continue;
      }
      const std::uint32_t st = landed % S;
      if (issued < mine && issued - landed < S) {
        // A stage is free: watch the oldest load and the upstream flag of the
        // next chunk together, so a chunk published while this lane waits
        // goes out at once instead of after the landing.
        bool got;
        while (!(got = mbar_test(&bars[st], (parity >> st) & 1u)) && !ready_now(issued)) {
        }
        if (!got) continue;
      } else {
        mbar_wait(&bars[st], (parity >> st) & 1u);
      }
      parity ^= 1u << st;
      stamp(landed, 1);
      std::uint64_t g;
      std::uint32_t body, len;
      geom(landed, &g, &body, &len);
      if (body) bulk_s2g(dst + g, c.stage + static_cast<std::size_t>(st) * sb, body);
      bulk_commit();
      stamp(landed, 2);
      for (std::uint32_t i = body; i < len; ++i) dst[g + i] = ld_u8(src + g + i);  // ragged end
      if (W.prov != nullptr && len && dst == W.buf) {
        atomicAdd(&W.prov[static_cast<std::uint64_t>(prev) * P.n_chunks + pipe + landed * ns],
                  static_cast<unsigned long long>(len));
      }
      ++landed;
      if (has_next && P.eager_post && !P.push) {
        // Forward now: a local store completes in about a microsecond, while
        // waiting for the next slice to land (the lazy rule below) would hold
        // every chunk back one loaded NVLink round trip per hop.
        bulk_wait<0>();
        post(landed);
      } else if (issued > landed) {
        bulk_wait<1>();  // every store but the newest is complete
        post(landed - 1);
      } else {
        bulk_wait<0>();
        post(landed);
      }
    }
    bulk_wait<0>();
    if (ok) post(mine);
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  __syncwarp();
  return ok != 0;
}


// Push-mode chain: logical rank l writes its chunks straight into l+1's
// buffer (NVLink stores instead of loads). Each consumer lane first tells its
// producer where to write and that its buffer is free (mailbox + "ready" in
// the producer's ack slot); a producer lane forwards chunk k once it has
// landed locally (or immediately at the head) and publishes it with a
// system-scope release (the data now lives in the peer's memory).
__device__ void run_chain_push(Ctx& c, int pipe, int q, int ns) {
  const LaunchParamsT<1>& P = *c.P;
  const RankWork& W = *c.W;
  const int n = P.n_ranks;
  const int L = P.lanes;
  const int me = W.rank;
  const int logical = (me - P.root + n) % n;
  const int prev = (me + n - 1) % n;
  const int next = (me + 1) % n;
  const bool has_prev = logical > 0;
  const bool has_next = logical + 1 < n;
  const std::uint32_t K = P.n_chunks;
  if (static_cast<std::uint32_t>(pipe) >= K) return;
  const std::uint32_t mine = (K - 1 - pipe) / ns + 1;
  const std::uint64_t tag = c.epoch << 32;
  const std::size_t slot = static_cast<std::size_t>(me) * L + c.ell;
  const std::uint64_t* arrived = has_prev ? W.flags + static_cast<std::size_t>(prev) * L + c.ell : nullptr;
  if (has_prev) {  // consumer: announce the destination, then "ready"
    if (c.lane_id == 0) st_mbox(W.peers->mbox[prev] + 2 * slot, W.pub, c.epoch);
    publish(c, W.peers->acks[prev] + slot, c.epoch);
  }
  if (!has_next) {  // tail: wait until every chunk of this lane has landed
    (void)wait_geq(c, arrived, tag | mine, prev, K);
    return;
  }
  if (!wait_geq(c, W.acks + static_cast<std::size_t>(next) * L + c.ell, c.epoch, next, 0)) return;
  auto* dst = reinterpret_cast<std::uint8_t*>(
      peer_addr(W, next, read_mbox(c, W.mbox + 2 * (static_cast<std::size_t>(next) * L + c.ell), next)));
  std::uint64_t* next_flag = W.peers->flags[next] + slot;
  const bool aligned = c.stage != nullptr &&
                       ((reinterpret_cast<std::uintptr_t>(dst) | reinterpret_cast<std::uintptr_t>(W.buf)) & 15u) == 0 &&
                       (P.chunk_bytes & 15u) == 0 && (P.slice_bytes & 15u) == 0 && P.slice_bytes <= P.stage_bytes;
  if (aligned) {
    if (has_prev && !wait_geq(c, arrived, tag | 1, prev, pipe)) return;
    (void)chain_pull_bulk(c, pipe, q, ns, mine, arrived, W.buf, dst, prev, true, next_flag, tag);
    return;
  }
  for (std::uint32_t k = 0; k < mine; ++k) {
    if (has_prev && !wait_geq(c, arrived, tag | (k + 1), prev, pipe + static_cast<std::uint64_t>(k) * ns)) return;
    std::uint64_t off, len;
    chunk_range(P, pipe + k * ns, &off, &len);
    const std::uint64_t lo = static_cast<std::uint64_t>(q) * P.slice_bytes;
    if (lo < len) {
      const std::uint64_t hi = lo + P.slice_bytes < len ? lo + P.slice_bytes : len;
      warp_copy(c, W.buf, dst, off + lo, off + hi);
    }
    publish(c, next_flag, tag | (k + 1));
  }
}

// Implicit pipelined chain (schedule_chain_pipelined, schedules.cpp:161-187):
// logical rank l pulls from l-1 and serves l+1.
__device__ void run_chain(Ctx& c, int pipe, int q, int ns) {
  const LaunchParamsT<1>& P = *c.P;
  const RankWork& W = *c.W;
  const int n = P.n_ranks;
  const int L = P.lanes;
  const int me = W.rank;
  const int logical = (me - P.root + n) % n;
  const int prev = (me + n - 1) % n;
  const int next = (me + 1) % n;
  const bool has_prev = logical > 0;
  const bool has_next = logical + 1 < n;
  const std::uint32_t K = P.n_chunks;
  if (static_cast<std::uint32_t>(pipe) >= K) return;
  const std::uint32_t mine = (K - 1 - pipe) / ns + 1;
  const std::uint64_t tag = c.epoch << 32;
  const std::size_t slot = static_cast<std::size_t>(me) * L + c.ell;

  if (has_next && c.lane_id == 0) st_mbox(W.peers->mbox[next] + 2 * slot, W.pub, c.epoch);
  if (!has_prev) {
    publish_direct(c, W.peers->flags[next] + slot, tag | mine);  // the head owns every chunk
  } else {
    const std::uint64_t* ready = W.flags + static_cast<std::size_t>(prev) * L + c.ell;
    const std::uint8_t* src = nullptr;
    if (c.stage != nullptr) {
      if (!wait_geq(c, ready, tag | 1, prev, pipe)) return;
      src = reinterpret_cast<const std::uint8_t*>(
          peer_addr(W, prev, read_mbox(c, W.mbox + 2 * (static_cast<std::size_t>(prev) * L + c.ell), prev)));
      const bool aligned = ((reinterpret_cast<std::uintptr_t>(src) | reinterpret_cast<std::uintptr_t>(W.buf)) & 15u) == 0 &&
                           (P.chunk_bytes & 15u) == 0 && (P.slice_bytes & 15u) == 0 &&
                           P.slice_bytes <= P.stage_bytes;
      if (aligned) {
        if (!chain_pull_bulk(c, pipe, q, ns, mine, ready, src, W.buf, prev, has_next, W.peers->flags[next] + slot,
                             tag)) {
          return;
        }
        publish_direct(c, W.peers->acks[prev] + slot, c.epoch);
        if (has_next) (void)wait_geq(c, W.acks + static_cast<std::size_t>(next) * L + c.ell, c.epoch, next, K);
        return;
      }
    }
    for (std::uint32_t k = 0; k < mine; ++k) {
      const std::uint64_t t_wait = W.trace ? globaltimer() : 0;
      if (!wait_geq(c, ready, tag | (k + 1), prev, pipe + static_cast<std::uint64_t>(k) * ns)) return;
      const std::uint64_t t_ready = W.trace ? globaltimer() : 0;
      if (k == 0) {
        src = reinterpret_cast<const std::uint8_t*>(
            peer_addr(W, prev, read_mbox(c, W.mbox + 2 * (static_cast<std::size_t>(prev) * L + c.ell), prev)));
      }
      pull_slice(c, pipe + k * ns, q, src, prev);
      if (has_next) publish(c, W.peers->flags[next] + slot, tag | (k + 1));  // forward chunk k
      trace_pull(c, k, t_wait, t_ready);
    }
    publish_direct(c, W.peers->acks[prev] + slot, c.epoch);  // done reading prev's buffer
  }
  if (has_next) {
    (void)wait_geq(c, W.acks + static_cast<std::size_t>(next) * L + c.ell, c.epoch, next, K);
  }
}

// Explicit schedule (direct, chain, knomial, scatter_ring_allgather): walk
// the rank's event list, keeping the events of this lane's chunk class.
__device__ void run_events(Ctx& c, int pipe, int q, int ns) {
  const LaunchParamsT<1>& P = *c.P;
  const RankWork& W = *c.W;
  const int L = P.lanes;
  const std::size_t slot = static_cast<std::size_t>(W.rank) * L + c.ell;
  const std::uint64_t tag = c.epoch << 32;
  std::uint64_t sent_mask = 0, recv_mask = 0;
  // Announce our buffer to every peer this lane will serve.
  for (int i = 0; i < W.n_events; ++i) {
    const std::uint64_t ev = W.events[i];
    const std::uint32_t ch = static_cast<std::uint32_t>(ev & 0xFFFFFFu);
    if ((ev >> 31) & 1u) continue;
    if (static_cast<int>(ch % ns) != pipe) continue;
    const int peer = static_cast<int>((ev >> 24) & 0x7F);
    if (!((sent_mask >> peer) & 1u)) {
      sent_mask |= 1ull << peer;
      if (c.lane_id == 0) st_mbox(W.peers->mbox[peer] + 2 * slot, W.pub, c.epoch);
    }
  }
  const std::uint8_t* src_of[kMaxRanks];
  std::uint32_t k = 0;
  for (int i = 0; i < W.n_events; ++i) {
    const std::uint64_t ev = W.events[i];
    const std::uint32_t ch = static_cast<std::uint32_t>(ev & 0xFFFFFFu);
    if (static_cast<int>(ch % ns) != pipe) continue;
    const int peer = static_cast<int>((ev >> 24) & 0x7F);
    const bool is_recv = (ev >> 31) & 1u;
    const std::uint64_t idx = ((ev >> 32) & 0xFFFFFFu) + 1;
    if (is_recv) {
      const std::uint64_t* ready = W.flags + static_cast<std::size_t>(peer) * L + c.ell;
      const std::uint64_t t_wait = W.trace ? globaltimer() : 0;
      if (!wait_geq(c, ready, tag | idx, peer, ch)) return;
      const std::uint64_t t_ready = W.trace ? globaltimer() : 0;
      if (!((recv_mask >> peer) & 1u)) {
        recv_mask |= 1ull << peer;
        src_of[peer] = reinterpret_cast<const std::uint8_t*>(
            peer_addr(W, peer, read_mbox(c, W.mbox + 2 * (static_cast<std::size_t>(peer) * L + c.ell), peer)));
      }
      pull_slice(c, ch, q, src_of[peer], peer);
      trace_pull(c, k++, t_wait, t_ready);
    } else {
      publish(c, W.peers->flags[peer] + slot, tag | idx);
    }
  }
  for (std::uint64_t m = recv_mask; m; m &= m - 1) {
    publish_direct(c, W.peers->acks[__ffsll(static_cast<long long>(m)) - 1] + slot, c.epoch);
  }
  for (std::uint64_t m = sent_mask; m; m &= m - 1) {
    const int peer = __ffsll(static_cast<long long>(m)) - 1;
    if (!wait_geq(c, W.acks + static_cast<std::size_t>(peer) * L + c.ell, c.epoch, peer, 0)) return;
  }
}

// NL = 1: one rank per GPU (full register budget). NL = kMaxLocal: ranks
// sharing a GPU need several co-resident CTAs per SM: 2 per SM (112 registers,
// no spills; the 3-CTA bound spilled 224 bytes).
template <int NL>
__global__ void __launch_bounds__(kThreads, NL == 1 ? 1 : BCL_SHARED_MIN_BLOCKS) bcast_kernel(const __grid_constant__ LaunchParamsT<NL> P) {
  pdl_wait();
  __shared__ CtaShared sh;
  const int local = NL == 1 ? 0 : static_cast<int>(blockIdx.x) / P.ctas_per_rank;
  const int cta = NL == 1 ? static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x) % P.ctas_per_rank;
  const int warp = static_cast<int>(threadIdx.x >> 5);
  if (threadIdx.x < kWarpsPerCta) {
    sh.tail[threadIdx.x] = 0;
    sh.head[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) sh.done = 0;
  extern __shared__ __align__(128) std::uint8_t dyn_smem[];
  if (P.stage_bytes && warp < kWarpsPerCta && (threadIdx.x & 31) == 0) {
    for (std::uint32_t i = 0; i < P.stages; ++i) mbar_init(&sh.full[warp][i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // The call's epoch comes from the rank's device-side call state (so a
  // replayed CUDA graph gets a fresh one); every helper takes it from Ctx.
  __shared__ unsigned long long epoch_sh;
  __shared__ CallState* state_sh;
  if (threadIdx.x == 0) {
    state_sh = P.ranks[local].state;
    epoch_sh = state_sh->epoch + 1;
  }
  __syncthreads();
  const auto* hdr = reinterpret_cast<const LaunchParamsT<1>*>(&P);
  if (warp == kWarpsPerCta) {
    run_publisher(*hdr, &sh, P.ranks[local], cta);
    // The publisher leaves last (after every copy warp of the CTA): the last
    // CTA of the rank to finish advances the rank's epoch.
    if ((threadIdx.x & 31) == 0) {
      CallState* st = state_sh;
      if (last_cta(st, P.ctas_per_rank)) st->epoch = epoch_sh;
    }
    return;
  }
  Ctx c;
  c.P = hdr;
  c.W = &P.ranks[local];
  c.sh = &sh;
  c.lane_id = static_cast<int>(threadIdx.x & 31);
  c.warp = warp;
  c.ell = cta * kWarpsPerCta + warp;
  c.epoch = epoch_sh;
  c.tail = 0;
  c.stage = P.stage_bytes ? dyn_smem + static_cast<std::size_t>(warp) * P.stages * P.stage_bytes : nullptr;
  if (c.ell < P.lanes) {
    const std::uint64_t t_enter = c.W->trace ? globaltimer() : 0;
    const int ns = P.lanes / P.slices;
    const int pipe = c.ell / P.slices;
    const int q = c.ell % P.slices;
    if (c.W->n_events < 0) {
      if (P.push) {
        run_chain_push(c, pipe, q, ns);
      } else {
        run_chain(c, pipe, q, ns);
      }
    } else {
      run_events(c, pipe, q, ns);
    }
    if (c.W->trace && c.lane_id == 0 && c.W->trace_cap > 0) {
      unsigned long long* rec =
          c.W->trace + (static_cast<std::size_t>(c.ell) * c.W->trace_cap + c.W->trace_cap - 1) * 4;
      rec[0] = t_enter;
      rec[3] = globaltimer();
    }
  }
  __syncwarp();
  if (c.lane_id == 0) {
    __threadfence_block();  // the last tail release is ordered before the count
    atomicAdd_block(&sh.done, 1u);
  }
}


// Single-GPU groups: the chain's hops fused per item (LocalChainParams).
#ifndef BCL_LC_MINB
#define BCL_LC_MINB 3  // 80 registers, no spills: 43.7 us at config 1 vs 47.5 us at 4 CTAs/SM (64 registers,
                       // spilling once items are claimed dynamically; profiles/round2/n1/variants.log)
#endif
__global__ void __launch_bounds__(256, BCL_LC_MINB) local_chain_kernel(const __grid_constant__ LocalChainParams P) {
  const int lane = static_cast<int>(threadIdx.x & 31);
  const std::uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const std::uint32_t G = (gridDim.x * blockDim.x) >> 5;
  const std::uint32_t ipc = static_cast<std::uint32_t>((P.chunk_bytes + P.item_bytes - 1) / P.item_bytes);
  const std::uint32_t items = P.n_chunks * ipc;  // < 2^32 (host-checked)
  Ctx c{};
  c.lane_id = lane;
  // Items are claimed statically (i = g, g + G, ...) or, with a claim
  // counter, dynamically: each warp takes the next unclaimed item, so warps
  // whose items ran slower do not leave the others idle at the end. Every
  // warp claims once past the last item, so the claim that returns
  // items + G - 1 is the launch's last: it re-zeroes the counter for the
  // launch that reuses it (stream order; the host rotates 64 counters).
  const bool dyn = P.claim != nullptr;
  auto claim = [&]() -> std::uint32_t {
    unsigned long long v = 0;
    if (lane == 0) {
      v = atomicAdd(P.claim, 1ull);
      if (v == static_cast<unsigned long long>(items) + G - 1) *P.claim = 0;
    }
    return static_cast<std::uint32_t>(__shfl_sync(0xffffffffu, v, 0));
  };
  std::uint32_t i = dyn ? claim() : g;
  while (i < items) {
    const std::uint32_t ch = i / ipc;
    const std::uint64_t off = static_cast<std::uint64_t>(ch) * P.chunk_bytes;
    const std::uint64_t end = P.bytes - off < P.chunk_bytes ? P.bytes : off + P.chunk_bytes;
    const std::uint64_t lo = off + static_cast<std::uint64_t>(i - ch * ipc) * P.item_bytes;
    if (lo < end) {
      const std::uint64_t hi = lo + P.item_bytes < end ? lo + P.item_bytes : end;
      for (int h = 1; h < P.n_ranks; ++h) {
        warp_copy(c, P.buf[h - 1], P.buf[h], lo, hi);
        __syncwarp();  // hop h's stores are visible to hop h + 1's loads (same warp)
        if (P.prov[h] != nullptr && lane == 0) {
          atomicAdd(&P.prov[h][static_cast<std::uint64_t>(P.rank[h - 1]) * P.n_chunks + ch],
                    static_cast<unsigned long long>(hi - lo));
        }
      }
    }
    i = dyn ? claim() : i + G;
  }
}

// ---------------------------------------------------------------- LL path
__device__ __forceinline__ void st_volatile_v4(uint4* p, std::uint32_t a, std::uint32_t b, std::uint32_t c,
                                               std::uint32_t d) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

__device__ void ll_fail(const LLRank& R, int peer, std::uint64_t line, std::uint64_t seen, std::uint64_t want) {
  atomicExch(R.abort, 1);
  if (atomicCAS(&R.err->code, 0, 1) == 0) {
    R.err->rank = R.rank;
    R.err->peer = peer;
    R.err->lane = -2;  // LL protocol
    R.err->chunk = line;
    R.err->observed = seen;
    R.err->expected = want;
    __threadfence_system();
  }
}

// LL kernel. direct: the root writes every line into each receiver's
// landing area for that source. chain (pipelined chain, schedules.cpp:161-187
// at line granularity): logical rank l polls its chain landing area, copies
// each line's payload out and forwards the very same line to l + 1, so the
// hops overlap line by line with no fence and no flag round trip. Writers
// first wait for their targets' credits for the half they are about to reuse.
// The message ("segment") a line belongs to: its first line, this rank's
// buffer and its bytes. One segment for an ordinary call; a binary search of
// the launch's segment table for a fused group (bcl_group_start/end).
struct LineSeg {
  std::uint32_t line0;
  std::uint8_t* buf;
  std::uint64_t bytes;
};
template <int NL, int NS>
__device__ __forceinline__ LineSeg seg_of(const LLParamsT<NL, NS>& P, int li, std::uint32_t line) {
  if constexpr (NS == 1) {
    return LineSeg{0, P.ranks[li].buf, P.bytes};
  } else {
    int lo = 0, hi = P.n_seg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.seg_line[mid] <= line) lo = mid; else hi = mid - 1;
    }
    return LineSeg{P.seg_line[lo], P.seg_buf[li][lo], P.seg_bytes[lo]};
  }
}

template <int NL, int NS>
__global__ void __launch_bounds__(kLLThreads) ll_kernel(const __grid_constant__ LLParamsT<NL, NS> P) {
  pdl_wait();
  const int li = NL == 1 ? 0 : static_cast<int>(blockIdx.x) / P.ctas;
  const LLRank& R = P.ranks[li];
  const std::uint32_t cta = NL == 1 ? blockIdx.x : blockIdx.x % P.ctas;
  const std::uint32_t first = cta * blockDim.x + threadIdx.x;
  const std::uint32_t stride = static_cast<std::uint32_t>(P.ctas) * blockDim.x;
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) s_epoch = R.state->epoch + 1;  // the call's epoch (device-side call state)
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const std::uint32_t half = static_cast<std::uint32_t>(epoch & 1u);
  const std::uint32_t flag = static_cast<std::uint32_t>(epoch);
  const int n = P.n_ranks;
  const int logical = (R.rank - P.root + n) % n;
  const int next = (R.rank + 1) % n;
  const bool chain = P.chain != 0;
  const bool writer = chain ? logical + 1 < n : logical == 0;
  const std::size_t area =
      chain ? static_cast<std::size_t>(n) * 2 * P.area_lines + static_cast<std::size_t>(half) * P.chain_lines
            : (static_cast<std::size_t>(P.root) * 2 + half) * P.area_lines;
  if (writer) {
    // The half we are about to overwrite was last written (same kind) in
    // epoch need: wait until the targets have read it (normally long ago).
    const std::uint64_t need = chain ? R.state->ll_last_chain[half] : R.state->ll_last_direct[half];
    const int t = static_cast<int>(threadIdx.x);
    if (need > 0 && (chain ? t == next : (t < n && t != P.root))) {
      const std::uint64_t* cr = R.credit + t;
      const std::uint64_t t0 = globaltimer();
      std::uint64_t v;
      while ((v = ld_relaxed_sys(cr)) < need) {
        if (globaltimer() - t0 > P.timeout_ns) {
          ll_fail(R, t, 0, v, need);
          break;
        }
      }
    }
    __syncthreads();
  }
  if (logical == 0) {
    for (std::uint32_t i = first; i < P.lines; i += stride) {
      const LineSeg sg = seg_of(P, li, i);
      const bool aligned = (reinterpret_cast<std::uintptr_t>(sg.buf) & 7u) == 0;
      const std::uint64_t off = static_cast<std::uint64_t>(i - sg.line0) * 8;
      std::uint32_t lo = 0, hi = 0;
      if (aligned && off + 8 <= sg.bytes) {
        const uint2 v = *reinterpret_cast<const uint2*>(sg.buf + off);
        lo = v.x;
        hi = v.y;
      } else {
        for (std::uint32_t b = 0; b < 8 && off + b < sg.bytes; ++b) {
          const std::uint32_t byte = sg.buf[off + b];
          if (b < 4) lo |= byte << (8 * b); else hi |= byte << (8 * (b - 4));
        }
      }
      if (chain) {
        st_volatile_v4(R.peers->ll[next] + area + i, lo, flag, hi, flag);
      } else {
        for (int d = 0; d < n; ++d) {
          if (d == P.root) continue;
          st_volatile_v4(R.peers->ll[d] + area + i, lo, flag, hi, flag);
        }
      }
    }
  }
  // Receiver: poll our landing lines, forward (chain, not the tail), copy out.
  const uint4* src = R.ll + area;
  uint4* fwd = chain && writer ? R.peers->ll[next] + area : nullptr;
  const int source = chain ? (R.rank + n - 1) % n : P.root;
  bool ok = true;
  for (std::uint32_t i = logical == 0 ? P.lines : first; i < P.lines && ok; i += stride) {
    uint4 v = ld_volatile_v4(src + i);
    if (v.y != flag || v.w != flag) {
      const std::uint64_t t0 = globaltimer();
      unsigned spins = 0;
      while (true) {
        v = ld_volatile_v4(src + i);
        if (v.y == flag && v.w == flag) break;
        if ((++spins & 1023u) == 0) {
          if (*(volatile int*)R.abort != 0 || globaltimer() - t0 > P.timeout_ns) {
            if (*(volatile int*)R.abort == 0) ll_fail(R, source, i, v.y, flag);
            ok = false;
            break;
          }
        }
      }
      if (!ok) break;
    }
    if (fwd != nullptr) st_volatile_v4(fwd + i, v.x, v.y, v.z, v.w);
    const LineSeg sg = seg_of(P, li, i);
    const bool aligned = (reinterpret_cast<std::uintptr_t>(sg.buf) & 7u) == 0;
    const std::uint64_t off = static_cast<std::uint64_t>(i - sg.line0) * 8;
    if (aligned && off + 8 <= sg.bytes) {
      *reinterpret_cast<uint2*>(sg.buf + off) = make_uint2(v.x, v.z);
    } else {
      for (std::uint32_t b = 0; b < 8 && off + b < sg.bytes; ++b) {
        sg.buf[off + b] = static_cast<std::uint8_t>((b < 4 ? v.x >> (8 * b) : v.z >> (8 * (b - 4))) & 0xFFu);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // The rank's last CTA to finish advances its call state and, as a
    // receiver, tells the source every line of this epoch has been read, so
    // the source may reuse the half.
    CallState* st = R.state;
    if (last_cta(st, P.ctas)) {
      st->epoch = epoch;
      if (writer) (chain ? st->ll_last_chain : st->ll_last_direct)[half] = epoch;
      if (logical != 0 && *(volatile int*)R.abort == 0) {
        st_relaxed_sys(R.peers->credit[source] + (chain ? n + 1 : 0) + R.rank, epoch);
      }
    }
  }
}

// Payload bytes thread `part` (0-7) of an LL128 line carries: line `line`
// of a message of `bytes` bytes holds [line * 120, line * 120 + 120); the
// thread moves [off, off + len0) as word 0 and [off + 8, off + 8 + len1) as
// word 1 (part 7's word 1 is the flag).
__device__ __forceinline__ void ll128_piece(int part, std::uint32_t line, std::uint64_t bytes, std::uint64_t* off,
                                            std::uint32_t* len0, std::uint32_t* len1) {
  *off = static_cast<std::uint64_t>(line) * kLL128Payload + static_cast<std::uint64_t>(part) * 16;
  const std::uint64_t end = static_cast<std::uint64_t>(line) * kLL128Payload + kLL128Payload;
  const std::uint64_t lim = end < bytes ? end : bytes;
  auto clip = [&](std::uint64_t a) -> std::uint32_t {
    return a >= lim ? 0u : static_cast<std::uint32_t>(lim - a < 8 ? lim - a : 8);
  };
  *len0 = clip(*off);
  *len1 = part == 7 ? 0u : clip(*off + 8);
}

// LL128 pipelined chain. A 128-byte line carries 120 payload bytes and a flag
// in its last 8 bytes; eight threads own one line (16 bytes each) and a warp
// moves four lines (a "group") per instruction. Like NCCL's LL128 this relies
// on a 128-byte warp-coalesced store arriving as one unit (over NVLink, and
// through L2 between ranks sharing a GPU): a reader that sees a line's flag
// sees the whole line. Readers vote per warp and reload until all four flags
// match. Lines land in a bounded ring: warp w's k-th group goes to slot
// (w * D + k % D) of its successor's ring with flag (epoch << 20 | k / D); a
// writer reuses a slot once the successor's warp w has returned a credit
// for the group D earlier (credits every D / 2 groups, per warp).
__device__ __forceinline__ void st_volatile_v2u64(ulonglong2* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const std::uint64_t* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ ulonglong2 ld_volatile_v2u64(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
// Bytes [off, off + len) of buf (len <= 8) as a little-endian word; the fast
// path needs 8-byte alignment of buf + off.
__device__ __forceinline__ unsigned long long ll128_get(const std::uint8_t* buf, std::uint64_t off, std::uint32_t len,
                                                        bool aligned) {
  if (len == 8 && aligned) return *reinterpret_cast<const unsigned long long*>(buf + off);
  unsigned long long v = 0;
  for (std::uint32_t b = 0; b < len; ++b) v |= static_cast<unsigned long long>(buf[off + b]) << (8 * b);
  return v;
}
__device__ __forceinline__ void ll128_put(std::uint8_t* buf, std::uint64_t off, std::uint32_t len, bool aligned,
                                          unsigned long long v) {
  if (len == 8 && aligned) {
    *reinterpret_cast<unsigned long long*>(buf + off) = v;
    return;
  }
  for (std::uint32_t b = 0; b < len; ++b) buf[off + b] = static_cast<std::uint8_t>(v >> (8 * b));
}

// NL > 1: ranks sharing one GPU (cooperative launch, P.ctas CTAs per rank).
// (3 CTAs per SM for one rank per GPU; the 16-rank block, for ranks sharing a
// GPU, is compiled for 2 so it does not spill at 42 registers.)
template <int NL, int NS>
__global__ void __launch_bounds__(kLLThreads, NL == 1 ? 3 : 2) ll128_kernel(const __grid_constant__ LLParamsT<NL, NS> P) {
  pdl_wait();
  const int li = NL == 1 ? 0 : static_cast<int>(blockIdx.x) / P.ctas;
  const LLRank& R = P.ranks[li];
  const std::uint32_t cta = NL == 1 ? blockIdx.x : blockIdx.x % P.ctas;
  const int lane = static_cast<int>(threadIdx.x & 31);
  const int part = lane & 7;  // 16-byte piece of the line
  const int sub = lane >> 3;  // line within the warp's group of four
  const std::uint32_t warp = (cta * blockDim.x + threadIdx.x) >> 5;
  const std::uint32_t warps = (static_cast<std::uint32_t>(P.ctas) * blockDim.x) >> 5;
  const int n = P.n_ranks;
  const int logical = (R.rank - P.root + n) % n;
  const int next = (R.rank + 1) % n;
  const int source = (R.rank + n - 1) % n;
  const bool writer = logical + 1 < n;
  // Ring positions continue across calls: warp w's groups into its
  // successor's ring are numbered by wseq[w] (this rank's count of groups it
  // wrote there, over every call) and read back by the successor's warp w by
  // its rseq[w] (the same count). A call therefore never waits for the
  // previous call to drain: only each slot's own credit gates its reuse.
  // (32-bit positions, compared modulo 2^32: the registers LL128 can spare.
  // Loaded before the call-state barrier so the loads overlap.)
  const std::uint32_t wbase = writer ? static_cast<std::uint32_t>(R.wseq[warp]) : 0u;
  const std::uint32_t rbase = logical > 0 ? static_cast<std::uint32_t>(R.rseq[warp]) : 0u;
  // (LL128 needs no call epoch while it runs: its lines carry ring laps; the
  // rank's last CTA just advances the epoch at the end.)
  // `line` counts from its segment's first line; `bytes` = the segment's.
  auto piece = [&](std::uint32_t line, std::uint64_t bytes, std::uint64_t* off, std::uint32_t* len0,
                   std::uint32_t* len1) { ll128_piece(part, line, bytes, off, len0, len1); };
  const ulonglong2* ring_self = reinterpret_cast<const ulonglong2*>(R.ll + P.chain128_area);
  ulonglong2* ring_next = writer ? reinterpret_cast<ulonglong2*>(R.peers->ll[next] + P.chain128_area) : nullptr;
  const std::uint64_t* my_credit = R.wcredit + warp;  // our successor's consumption of our groups
  std::uint64_t* prev_credit = logical > 0 ? R.peers->wcredit[source] + warp : nullptr;
  // This thread's 16-byte word of the slot of ring position q, and the flag
  // a line at position q carries (its lap + 1: a slot's previous content is
  // one lap older, a zeroed ring matches nothing).
  auto at = [&](std::uint32_t q) -> std::size_t {
    return ((static_cast<std::size_t>(warp) * kLL128Depth + q % kLL128Depth) * 4 + sub) * 8 + part;
  };
  auto flag_of = [&](std::uint32_t q) -> unsigned long long { return q / kLL128Depth + 1u; };
  // Warp-collective: the successor has consumed our position q - D (its slot
  // is free); credits count positions consumed, over every call. The last
  // credit seen is cached (warp-uniform), so the local credit word is polled
  // about once per D / 2 groups. Like NCCL's LL128 credits the overwrite is
  // ordered after the poll by its control dependency (no acquire: an acquire
  // invalidates L1 on every call, ~6% at 64 MiB, n = 4).
  // Lane 0 caches the last credit it saw; the first value is loaded when the
  // kernel starts, so its latency overlaps the first payload loads / polls.
  std::uint32_t seen = 0;
  if (writer && lane == 0) seen = static_cast<std::uint32_t>(ld_volatile_u64(my_credit));
  auto room = [&](std::uint32_t q) -> bool {
    const std::uint32_t want = q - kLL128Depth + 1;  // consumed positions needed (modulo 2^32)
    int ok = 1;
    if (lane == 0 && static_cast<std::int32_t>(seen - want) < 0) {
      const std::uint64_t t0 = globaltimer();
      unsigned spins = 0;
      while (static_cast<std::int32_t>((seen = static_cast<std::uint32_t>(ld_volatile_u64(my_credit))) - want) < 0) {
        if ((++spins & 1023u) == 0) {
          if (*(volatile int*)R.abort != 0) { ok = 0; break; }
          if (globaltimer() - t0 > P.timeout_ns) {
            ll_fail(R, next, q, seen, want);
            ok = 0;
            break;
          }
        }
      }
    }
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
  };
  std::uint32_t k = 0;  // groups this warp moved in this call
  if (logical == 0) {
    for (std::uint32_t g = warp; g * 4 < P.lines; g += warps, ++k) {
      const std::uint32_t line = g * 4 + sub;
      const bool active = line < P.lines;
      unsigned long long a = 0, b = 0;
      if (active) {  // payload first: its load overlaps the credit check
        const LineSeg sg = seg_of(P, li, line);
        const bool aligned = (reinterpret_cast<std::uintptr_t>(sg.buf) & 7u) == 0;
        std::uint64_t off;
        std::uint32_t l0, l1;
        piece(line - sg.line0, sg.bytes, &off, &l0, &l1);
        a = ll128_get(sg.buf, off, l0, aligned);
        b = part == 7 ? flag_of(wbase + k) : ll128_get(sg.buf, off + 8, l1, aligned);
      }
      if (!room(wbase + k)) break;
      if (active) st_volatile_v2u64(ring_next + at(wbase + k), a, b);
    }
  }
  bool ok = true;
  for (std::uint32_t g = logical == 0 ? P.lines : warp; g * 4 < P.lines && ok; g += warps, ++k) {
    const std::uint32_t line = g * 4 + sub;
    const bool active = line < P.lines;
    const unsigned long long flag = flag_of(rbase + k);
    ulonglong2 v = make_ulonglong2(0, 0);
    const std::uint64_t t0 = globaltimer();
    unsigned spins = 0;
    while (true) {
      if (active) v = ld_volatile_v2u64(ring_self + at(rbase + k));
      const bool stale = active && part == 7 && v.y != flag;
      if (!__any_sync(0xffffffffu, stale)) break;
      if ((++spins & 1023u) == 0) {
        const int give_up = (*(volatile int*)R.abort != 0 || globaltimer() - t0 > P.timeout_ns) ? 1 : 0;
        if (__any_sync(0xffffffffu, give_up)) {
          if (lane == 0 && *(volatile int*)R.abort == 0) ll_fail(R, source, line, 0, flag);
          ok = false;
          break;
        }
      }
    }
    if (!ok) break;
    if (writer) {  // forward the same line into the successor's ring (at our position, with its flag)
      if (!room(wbase + k)) {
        ok = false;
        break;
      }
      if (active) st_volatile_v2u64(ring_next + at(wbase + k), v.x, part == 7 ? flag_of(wbase + k) : v.y);
    }
    if (active) {
      const LineSeg sg = seg_of(P, li, line);
      const bool aligned = (reinterpret_cast<std::uintptr_t>(sg.buf) & 7u) == 0;
      std::uint64_t off;
      std::uint32_t l0, l1;
      piece(line - sg.line0, sg.bytes, &off, &l0, &l1);
      ll128_put(sg.buf, off, l0, aligned, v.x);
      if (part != 7) ll128_put(sg.buf, off + 8, l1, aligned, v.y);
    }
    if ((rbase + k + 1) % (kLL128Depth / 2) == 0) {
      // Every lane's loads of these groups have returned (their values were
      // stored above), so the predecessor may overwrite the slots.
      __syncwarp();
      if (lane == 0) st_relaxed_sys(prev_credit, rbase + k + 1);
    }
  }
  // The warp's ring positions after this call (warp-private counters).
  if (lane == 0 && ok) {
    if (writer) R.wseq[warp] = wbase + k;
    if (logical > 0) R.rseq[warp] = rbase + k;
  }
  __syncthreads();
  if (threadIdx.x == 0 && last_cta(R.state, P.ctas)) R.state->epoch += 1;  // the rank's last CTA
}

// LL128 lines for the `direct` schedule (chain == 3): the root writes each
// 128-byte line (120 payload bytes, flag = the call's epoch in the last 8)
// into every receiver's LL128 direct landing area for that source and half,
// and receivers poll their own copy line by line: half the root's egress of
// 16-byte LL lines. The halves, the credits and the reuse rule are the LL
// direct ones (a half is reused once its receivers credited the last call of
// either format that wrote it). One launch's lines -- one call, or a group's
// run of messages as segments -- fit the area: no ring, no co-residency needed.
template <int NL, int NS>
__global__ void __launch_bounds__(kLLThreads) ll128_direct_kernel(const __grid_constant__ LLParamsT<NL, NS> P) {
  pdl_wait();
  const int li = NL == 1 ? 0 : static_cast<int>(blockIdx.x) / P.ctas;
  const LLRank& R = P.ranks[li];
  const std::uint32_t cta = NL == 1 ? blockIdx.x : blockIdx.x % P.ctas;
  const int lane = static_cast<int>(threadIdx.x & 31);
  const int part = lane & 7;
  const int sub = lane >> 3;
  const std::uint32_t warp = (cta * blockDim.x + threadIdx.x) >> 5;
  const std::uint32_t warps = (static_cast<std::uint32_t>(P.ctas) * blockDim.x) >> 5;
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) s_epoch = R.state->epoch + 1;
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const std::uint32_t half = static_cast<std::uint32_t>(epoch & 1u);
  const int n = P.n_ranks;
  const bool root = R.rank == P.root;
  const std::size_t area = P.d128_area + (static_cast<std::size_t>(P.root) * 2 + half) * P.d128_lines * 8;
  // (a group's messages are segments: a line belongs to one, its payload
  // offset counts from the segment's first line)
  auto piece = [&](std::uint32_t line, std::uint64_t bytes, std::uint64_t* off, std::uint32_t* len0,
                   std::uint32_t* len1) { ll128_piece(part, line, bytes, off, len0, len1); };
  if (root) {
    // The half was last written (LL or LL128 direct) in epoch need: its
    // receivers must have read it.
    const std::uint64_t need = R.state->ll_last_direct[half];
    const int t = static_cast<int>(threadIdx.x);
    if (need > 0 && t < n && t != P.root) {
      const std::uint64_t t0 = globaltimer();
      std::uint64_t v;
      while ((v = ld_relaxed_sys(R.credit + t)) < need) {
        if (globaltimer() - t0 > P.timeout_ns) {
          ll_fail(R, t, 0, v, need);
          break;
        }
      }
    }
    __syncthreads();
    for (std::uint32_t g = warp; g * 4 < P.lines; g += warps) {
      const std::uint32_t line = g * 4 + sub;
      if (line >= P.lines) continue;
      const LineSeg sg = seg_of(P, li, line);
      const bool aligned = (reinterpret_cast<std::uintptr_t>(sg.buf) & 7u) == 0;
      std::uint64_t off;
      std::uint32_t l0, l1;
      piece(line - sg.line0, sg.bytes, &off, &l0, &l1);
      const unsigned long long a = ll128_get(sg.buf, off, l0, aligned);
      const unsigned long long b = part == 7 ? epoch : ll128_get(sg.buf, off + 8, l1, aligned);
      const std::size_t at = area + static_cast<std::size_t>(line) * 8 + part;
      for (int d = 0; d < n; ++d) {
        if (d != P.root) st_volatile_v2u64(reinterpret_cast<ulonglong2*>(R.peers->ll[d] + at), a, b);
      }
    }
  } else {
    bool ok = true;
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(R.ll + area);
    for (std::uint32_t g = warp; g * 4 < P.lines && ok; g += warps) {
      const std::uint32_t line = g * 4 + sub;
      const bool active = line < P.lines;
      ulonglong2 v = make_ulonglong2(0, 0);
      const std::uint64_t t0 = globaltimer();
      unsigned spins = 0;
      while (true) {
        if (active) v = ld_volatile_v2u64(src + static_cast<std::size_t>(line) * 8 + part);
        const bool stale = active && part == 7 && v.y != epoch;
        if (!__any_sync(0xffffffffu, stale)) break;
        if ((++spins & 1023u) == 0) {
          const int give_up = (*(volatile int*)R.abort != 0 || globaltimer() - t0 > P.timeout_ns) ? 1 : 0;
          if (__any_sync(0xffffffffu, give_up)) {
            if (lane == 0 && *(volatile int*)R.abort == 0) ll_fail(R, P.root, line, 0, epoch);
            ok = false;
            break;
          }
        }
      }
      if (!ok) break;
      if (active) {
        const LineSeg sg = seg_of(P, li, line);
        const bool aligned = (reinterpret_cast<std::uintptr_t>(sg.buf) & 7u) == 0;
        std::uint64_t off;
        std::uint32_t l0, l1;
        piece(line - sg.line0, sg.bytes, &off, &l0, &l1);
        ll128_put(sg.buf, off, l0, aligned, v.x);
        if (part != 7) ll128_put(sg.buf, off + 8, l1, aligned, v.y);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    CallState* st = R.state;
    if (last_cta(st, P.ctas)) {
      st->epoch = epoch;
      if (root) st->ll_last_direct[half] = epoch;
      else if (*(volatile int*)R.abort == 0) st_relaxed_sys(R.peers->credit[P.root] + R.rank, epoch);
    }
  }
}

// All-ranks barrier: rank r bumps slot [r] in every peer, then waits for
// every peer's bump in its own slots.
__global__ void barrier_kernel(const __grid_constant__ BarrierParams B) {
  pdl_wait();
  const int local = blockIdx.x;
  const int t = threadIdx.x;
  const int me = B.rank[local];
  const PeerTable* peers = B.peers[local];
  __shared__ unsigned long long s_epoch;
  if (t == 0) s_epoch = B.state[local]->bar_epoch + 1;  // one CTA per rank: read, then advanced below
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  if (t < B.n_ranks && t != me) {
    fence_acq_rel_sys();
    st_relaxed_sys(peers->bar[t] + me, epoch);
  }
  __syncthreads();
  if (t < B.n_ranks && t != me) {
    const std::uint64_t* slot = B.bar[local] + t;
    const std::uint64_t t0 = globaltimer();
    while (ld_relaxed_sys(slot) < epoch) {
      if (globaltimer() - t0 > B.timeout_ns) {
        ErrorRecord* e = B.err[local];
        if (atomicCAS(&e->code, 0, 1) == 0) {
          e->rank = me;
          e->peer = t;
          e->lane = -1;
          e->expected = epoch;
          __threadfence_system();
        }
        break;
      }
    }
    (void)ld_acquire_sys(slot);
  }
  __syncthreads();
  if (t == 0) B.state[local]->bar_epoch = epoch;
}

// Plain copy of one message slab (the DeviceFabric transport, bcl_fabric.cpp):
// 16-byte loads from the source GPU's slab (NVLink across GPUs), 4 in flight
// per thread; both slabs are 256-byte aligned allocations.
__global__ void __launch_bounds__(512) peer_copy_kernel(std::uint8_t* __restrict__ dst,
                                                          const std::uint8_t* __restrict__ src, std::uint64_t len) {
  const std::uint64_t nvec = len / 16;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  const uint4* vs = reinterpret_cast<const uint4*>(src);
  uint4* vd = reinterpret_cast<uint4*>(dst);
  std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    uint4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = ld_v4(vs + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) st_v4(vd + i + u * stride, r[u]);
  }
  for (; i < nvec; i += stride) st_v4(vd + i, ld_v4(vs + i));
  const std::uint64_t t = nvec * 16 + static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < len) dst[t] = ld_u8(src + t);
}

}  // namespace
}  // namespace dev

// Launch attributes shared by the launchers: cooperative when asked, else
// programmatic stream serialization, so a broadcast kernel is scheduled while
// the previous kernel of its stream drains and starts the moment it is done
// (back to back, N = 2: 5.2 -> 3.2 us per small broadcast;
// profiles/round2/pdl/). BCL_PDL=0 turns it off.
int fill_launch_attrs(cudaLaunchAttribute_st* attr, int cooperative) {
  static const bool pdl = [] {
    const char* v = std::getenv("BCL_PDL");
    return v == nullptr || std::atoi(v) != 0;
  }();
  int k = 0;
  attr[k].id = cudaLaunchAttributeCooperative;
  attr[k].val.cooperative = cooperative ? 1 : 0;
  ++k;
  if (!cooperative && pdl) {
    attr[k].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[k].val.programmaticStreamSerializationAllowed = 1;
    ++k;
  }
  return k;
}

int launch_peer_copy(std::uint8_t* dst, const std::uint8_t* src, std::uint64_t len, void* stream) {
  const std::uint64_t nvec = (len + 15) / 16;
  const unsigned blocks = static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(296, (nvec + 511) / 512)));
  dev::peer_copy_kernel<<<blocks, 512, 0, static_cast<cudaStream_t>(stream)>>>(dst, src, len);
  return static_cast<int>(cudaGetLastError());
}

std::size_t bcast_smem_bytes(std::uint32_t stages, std::uint32_t stage_bytes) {
  return static_cast<std::size_t>(dev::kWarpsPerCta) * stages * stage_bytes;
}

// The dynamic shared-memory limit is a per-function, per-device attribute:
// raise it to the largest stage budget any group on the device asked for
// (a later group with fewer stages must not lower it under an earlier one).
int prepare_bcast_kernels(std::size_t smem) {
  static std::mutex mu;
  static std::map<int, std::size_t> raised;  // device -> attribute value set
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  if (e != cudaSuccess) return static_cast<int>(e);
  std::lock_guard<std::mutex> lock(mu);
  std::size_t& cur = raised[device];
  if (smem <= cur && cur != 0) return 0;
  cur = std::max(cur, smem);
  const int v = static_cast<int>(cur);
  e = cudaFuncSetAttribute(dev::bcast_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaFuncSetAttribute(dev::bcast_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(
      cudaFuncSetAttribute(dev::bcast_kernel<dev::kMaxLocal>, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
}

template <int NL>
int launch_narrow(cudaLaunchConfig_t& cfg, const dev::LaunchParams& p) {
  dev::LaunchParamsT<NL> q;
  std::memcpy(&q, &p, offsetof(dev::LaunchParams, ranks));
  for (int i = 0; i < p.n_local; ++i) q.ranks[i] = p.ranks[i];
  return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::bcast_kernel<NL>, q));
}

int launch_bcast(const dev::LaunchParams& p, int cooperative, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.n_local * p.ctas_per_rank));
  cfg.blockDim = dim3(dev::kThreads);
  cfg.dynamicSmemBytes = p.stage_bytes ? bcast_smem_bytes(p.stages, p.stage_bytes) : 0;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = static_cast<unsigned>(fill_launch_attrs(attr, cooperative));
  // Same header layout: copy the header and the ranks into the smallest
  // parameter block that holds them (a 10 KB block for 16 ranks costs launch
  // latency; 4 ranks sharing a GPU is the emulated bench shape).
  if (p.n_local == 1) return launch_narrow<1>(cfg, p);
  if (p.n_local <= 4) return launch_narrow<4>(cfg, p);
  return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::bcast_kernel<dev::kMaxLocal>, p));
}

int local_chain_occupancy(int* blocks_per_sm) {
  return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, dev::local_chain_kernel, 256, 0));
}

int ll128_occupancy(int* blocks_per_sm, int shared) {
  if (shared) {
    return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        blocks_per_sm, dev::ll128_kernel<dev::kMaxLocal, 1>, dev::kLLThreads, 0));
  }
  return static_cast<int>(
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, dev::ll128_kernel<1, 1>, dev::kLLThreads, 0));
}

int launch_local_chain(const dev::LocalChainParams& p, int ctas, void* stream) {
  dev::local_chain_kernel<<<static_cast<unsigned>(ctas), 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return static_cast<int>(cudaGetLastError());
}

int launch_barrier(const dev::BarrierParams& p, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.n_local));
  cfg.blockDim = dim3(dev::kMaxRanks);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = static_cast<unsigned>(fill_launch_attrs(attr, p.n_local > 1 ? 1 : 0));
  return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::barrier_kernel, p));
}

namespace {

// Copy the host-side superset into the smallest parameter block that holds
// the launch (NL local ranks, NS segments).
template <int NL, int NS>
int launch_ll_as(cudaLaunchConfig_t& cfg, const dev::LLParams& p) {
  dev::LLParamsT<NL, NS> q;
  static_cast<dev::LLHeader&>(q) = p;
  for (int s = 0; s <= NS && s <= p.n_seg; ++s) q.seg_line[s] = p.seg_line[s];
  for (int s = 0; s < NS && s < p.n_seg; ++s) q.seg_bytes[s] = p.seg_bytes[s];
  for (int i = 0; i < p.n_local; ++i) {
    q.ranks[i] = p.ranks[i];
    for (int s = 0; s < NS && s < p.n_seg; ++s) q.seg_buf[i][s] = p.seg_buf[i][s];
  }
  if (p.chain == 3) return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::ll128_direct_kernel<NL, NS>, q));
  if (p.chain == 2) {
    // (LL128 groups are not fused for ranks sharing a GPU: the 16-rank fused
    // block would spill at LL128's 42-register budget; the host never asks.)
    if constexpr (NL > 1 && NS > 1) return static_cast<int>(cudaErrorInvalidValue);
    else return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::ll128_kernel<NL, NS>, q));
  }
  return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::ll_kernel<NL, NS>, q));
}

}  // namespace

int launch_ll(const dev::LLParams& p, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.n_local * p.ctas));
  cfg.blockDim = dim3(dev::kLLThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  // LL128 writers wait on ring credits from the successor's CTAs: co-residency
  // is required even for one rank per GPU (the successor's warp w may be any CTA).
  cfg.numAttrs = static_cast<unsigned>(fill_launch_attrs(attr, (p.n_local > 1 || (p.chain == 2 && p.coop)) ? 1 : 0));
  if (p.n_seg < 1 || p.n_seg > dev::max_segs(p.n_local)) return static_cast<int>(cudaErrorInvalidValue);
  const bool fused = p.n_seg > 1;
  if (p.n_local == 1) return fused ? launch_ll_as<1, dev::kMaxSegs>(cfg, p) : launch_ll_as<1, 1>(cfg, p);
  return fused ? launch_ll_as<dev::kMaxLocal, dev::kMaxSegsShared>(cfg, p) : launch_ll_as<dev::kMaxLocal, 1>(cfg, p);
}

int bcast_kernel_occupancy(int* blocks_per_sm, std::size_t smem) {
  return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      blocks_per_sm, dev::bcast_kernel<dev::kMaxLocal>, dev::kThreads, smem));
}

}  // namespace bcl
