// bcl_nvls.cu — NVLS multicast broadcast: the kernel and the multicast
// object's lifetime (see bcl_nvls.hpp, DESIGN.md §5 "nvls_kernel").
//
// Driver entry points come through the runtime's cudaGetDriverEntryPoint, so
// libbcl.so keeps no link-time dependency on libcuda.
#include "bcl_nvls.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <random>
#include <stdexcept>

namespace bcl {
namespace dev {
namespace {

__device__ __forceinline__ std::uint64_t nv_ld_acquire_sys(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ std::uint64_t nv_ld_relaxed_sys(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ std::uint64_t nv_timer() {
  std::uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Multicast store: the NVSwitch writes the 16 bytes into every GPU's copy.
// (.f32 lanes are moved, not computed on: the bits arrive unchanged.)
__device__ __forceinline__ void mc_st_v4(void* p, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
// Multicast add with release: the counter on every GPU is bumped after this
// thread's earlier memory operations (and, through the preceding CTA barrier,
// the CTA's) are visible system-wide.
__device__ __forceinline__ void mc_add_release(std::uint64_t* p, std::uint64_t v) {
  asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint4 ld_v4_na(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// Thread 0 waits until *p >= target; the CTA learns the outcome. Returns
// false on timeout (recorded) or abort.
__device__ bool cta_wait_geq(const NvlsRank& R, const std::uint64_t* p, std::uint64_t target, std::uint64_t timeout_ns,
                             std::uint64_t piece, int* ok_sh) {
  if (threadIdx.x == 0) {
    int ok = 1;
    std::uint64_t v = nv_ld_relaxed_sys(p);
    if (v < target) {
      const std::uint64_t t0 = nv_timer();
      unsigned spins = 0;
      while ((v = nv_ld_relaxed_sys(p)) < target) {
        if ((++spins & 127u) == 0) {
          if (*(volatile int*)R.abort != 0) {
            ok = 0;
            break;
          }
          if (nv_timer() - t0 > timeout_ns) {
            atomicExch(R.abort, 1);
            if (atomicCAS(&R.err->code, 0, 1) == 0) {
              R.err->rank = R.rank;
              R.err->peer = -1;
              R.err->lane = static_cast<int>(blockIdx.x);
              R.err->chunk = piece;
              R.err->observed = v;
              R.err->expected = target;
              __threadfence_system();
            }
            ok = 0;
            break;
          }
        }
      }
    }
    if (ok) (void)nv_ld_acquire_sys(p);
    *ok_sh = ok;
  }
  __syncthreads();
  const bool ok = *ok_sh != 0;
  // Readers of the unicast copy order their loads after a counter bumped
  // through the multicast alias of the same memory.
  asm volatile("fence.proxy.alias;" ::: "memory");
  return ok;
}

__device__ __forceinline__ uint4 gather16(const std::uint8_t* s, std::uint32_t n) {
  std::uint8_t b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) b[i] = i < static_cast<int>(n) ? s[i] : 0;
  uint4 v;
  std::memcpy(&v, b, 16);
  return v;
}

// The rank's last CTA to finish: advance its call state (`advance` runs once).
template <class F>
__device__ void nvls_finish(const NvlsRank& R, int ctas, F advance) {
  __syncthreads();
  if (threadIdx.x == 0 &&
      (ctas == 1 || atomicAdd(&R.state->finished, 1ull) + 1 == static_cast<unsigned long long>(ctas))) {
    R.state->finished = 0;
    advance(R.state);
  }
}

template <int NL>
__global__ void __launch_bounds__(kNvlsThreads) nvls_kernel(const __grid_constant__ NvlsParamsT<NL> P) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (programmatic dependent launch: see bcl_kernels.cu)
  __shared__ int ok_sh;
  __shared__ unsigned long long seq_sh;
  const int li = static_cast<int>(blockIdx.x) / P.ctas;
  const int j = static_cast<int>(blockIdx.x) % P.ctas;
  if (li >= P.n_local) return;
  const NvlsRank& R = P.ranks[li];
  if (threadIdx.x == 0) seq_sh = R.state->nvls_seq;  // this call's first ring sequence number
  __syncthreads();
  const unsigned long long seq_base = seq_sh;
  std::uint64_t* mc_ready = reinterpret_cast<std::uint64_t*>(P.mc);
  std::uint64_t* mc_done = mc_ready + kNvlsMaxSlots;
  const std::uint64_t* uc_ready = reinterpret_cast<const std::uint64_t*>(P.uc);
  const std::uint64_t* uc_done = uc_ready + kNvlsMaxSlots;
  const unsigned T = blockDim.x;
  const unsigned tid = threadIdx.x;
  for (std::uint32_t k = static_cast<std::uint32_t>(j); k < P.pieces; k += static_cast<std::uint32_t>(P.ctas)) {
    const std::uint64_t seq = seq_base + k;
    const std::uint32_t slot = static_cast<std::uint32_t>(seq % P.slots);
    const std::uint64_t round = seq / P.slots;
    const std::uint64_t off = static_cast<std::uint64_t>(k) * P.piece_bytes;
    const std::uint32_t len = static_cast<std::uint32_t>(min(P.piece_bytes, P.bytes - off));
    const std::uint32_t n16 = len / 16;
    const std::uint32_t tail = len % 16;
    const std::size_t data_off = kNvlsCtlBytes + static_cast<std::size_t>(slot) * P.slot_bytes;
    if (R.is_root) {
      // The slot's previous occupant must be consumed by every receiver.
      if (round > 0 && !cta_wait_geq(R, uc_done + slot, static_cast<std::uint64_t>(P.n_recv) * round, P.timeout_ns, k,
                                     &ok_sh)) {
        break;
      }
      const std::uint8_t* src = R.buf + off;
      uint4* dst = reinterpret_cast<uint4*>(P.mc + data_off);
      if ((reinterpret_cast<std::uintptr_t>(src) & 15u) == 0) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        unsigned i = tid;
        for (; i + 3 * T < n16; i += 4 * T) {
          const uint4 a = ld_v4_na(s4 + i), b = ld_v4_na(s4 + i + T), c = ld_v4_na(s4 + i + 2 * T),
                      d = ld_v4_na(s4 + i + 3 * T);
          mc_st_v4(dst + i, a);
          mc_st_v4(dst + i + T, b);
          mc_st_v4(dst + i + 2 * T, c);
          mc_st_v4(dst + i + 3 * T, d);
        }
        for (; i < n16; i += T) mc_st_v4(dst + i, ld_v4_na(s4 + i));
      } else {
        for (unsigned i = tid; i < n16; i += T) mc_st_v4(dst + i, gather16(src + 16 * static_cast<std::size_t>(i), 16));
      }
      if (tail && tid == 0) mc_st_v4(dst + n16, gather16(src + 16 * static_cast<std::size_t>(n16), tail));
      __syncthreads();
      if (tid == 0) {
        if (P.strict) asm volatile("fence.acq_rel.sys;" ::: "memory");
        mc_add_release(mc_ready + slot, 1);
      }
    } else {
      if (!cta_wait_geq(R, uc_ready + slot, round + 1, P.timeout_ns, k, &ok_sh)) break;
      const uint4* src = reinterpret_cast<const uint4*>(P.uc + data_off);
      std::uint8_t* dst = R.buf + off;
      if ((reinterpret_cast<std::uintptr_t>(dst) & 15u) == 0) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        unsigned i = tid;
        for (; i + 3 * T < n16; i += 4 * T) {
          const uint4 a = ld_v4_na(src + i), b = ld_v4_na(src + i + T), c = ld_v4_na(src + i + 2 * T),
                      d = ld_v4_na(src + i + 3 * T);
          d4[i] = a;
          d4[i + T] = b;
          d4[i + 2 * T] = c;
          d4[i + 3 * T] = d;
        }
        for (; i < n16; i += T) d4[i] = ld_v4_na(src + i);
      } else {
        for (unsigned i = tid; i < n16; i += T) {
          const uint4 v = ld_v4_na(src + i);
          std::uint8_t b[16];
          std::memcpy(b, &v, 16);
#pragma unroll
          for (int x = 0; x < 16; ++x) dst[16 * static_cast<std::size_t>(i) + x] = b[x];
        }
      }
      if (tail && tid == 0) {
        const uint4 v = ld_v4_na(src + n16);
        std::uint8_t b[16];
        std::memcpy(b, &v, 16);
        for (std::uint32_t x = 0; x < tail; ++x) dst[16 * static_cast<std::size_t>(n16) + x] = b[x];
      }
      __syncthreads();
      if (tid == 0) {
        if (P.strict) asm volatile("fence.acq_rel.sys;" ::: "memory");
        mc_add_release(mc_done + slot, 1);
      }
    }
  }
  const std::uint32_t pieces = P.pieces;
  nvls_finish(R, P.ctas, [&](CallState* st) { st->nvls_seq = seq_base + pieces; });
}

__device__ __forceinline__ void mc_st_u4(void* p, std::uint32_t a, std::uint32_t b, std::uint32_t c,
                                         std::uint32_t d) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

template <int NL>
__global__ void __launch_bounds__(512) nvls_ll_kernel(const __grid_constant__ NvlsLLParamsT<NL> P) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ int ok_sh;
  const int li = static_cast<int>(blockIdx.x) / P.ctas;
  const int j = static_cast<int>(blockIdx.x) % P.ctas;
  if (li >= P.n_local) return;
  const NvlsRank& R = P.ranks[li];
  __shared__ unsigned long long epoch_sh, need_sh;
  if (threadIdx.x == 0) {  // the call's epoch and its half's reuse bound (device-side call state)
    epoch_sh = R.state->nvls_ll_calls + 1;
    need_sh = R.state->nvls_ll_reports[epoch_sh & 1u];
  }
  __syncthreads();
  const unsigned long long epoch = epoch_sh;
  const std::uint32_t half = static_cast<std::uint32_t>(epoch & 1u);
  const std::uint32_t flag = static_cast<std::uint32_t>(epoch);
  const std::size_t area = (static_cast<std::size_t>(kNvlsCtlBytes) + kNvlsRingBytes) +
                           static_cast<std::size_t>(half) * kNvlsLLLines * 16;
  const std::uint32_t first = static_cast<std::uint32_t>(j) * blockDim.x + threadIdx.x;
  const std::uint32_t stride = static_cast<std::uint32_t>(P.ctas) * blockDim.x;
  const bool aligned = (reinterpret_cast<std::uintptr_t>(R.buf) & 7u) == 0;
  std::uint64_t* mc_done = reinterpret_cast<std::uint64_t*>(P.mc) + kNvlsLLDone + half;
  const std::uint64_t* uc_done = reinterpret_cast<const std::uint64_t*>(P.uc) + kNvlsLLDone + half;
  const unsigned long long reports = static_cast<unsigned long long>(P.n_recv) * static_cast<unsigned long long>(P.ctas);
  auto advance = [&](CallState* st) {
    st->nvls_ll_calls = epoch;
    st->nvls_ll_reports[half] += reports;
  };
  if (R.is_root) {
    // The half was last read two calls ago: every receiver CTA has reported.
    if (need_sh > 0 && !cta_wait_geq(R, uc_done, need_sh, P.timeout_ns, 0, &ok_sh)) {
      nvls_finish(R, P.ctas, advance);
      return;
    }
    uint4* dst = reinterpret_cast<uint4*>(P.mc + area);
    for (std::uint32_t i = first; i < P.lines; i += stride) {
      const std::uint64_t off = static_cast<std::uint64_t>(i) * 8;
      std::uint32_t lo = 0, hi = 0;
      if (aligned && off + 8 <= P.bytes) {
        const uint2 v = *reinterpret_cast<const uint2*>(R.buf + off);
        lo = v.x;
        hi = v.y;
      } else {
        for (std::uint32_t b = 0; b < 8 && off + b < P.bytes; ++b) {
          const std::uint32_t byte = R.buf[off + b];
          if (b < 4) lo |= byte << (8 * b); else hi |= byte << (8 * (b - 4));
        }
      }
      mc_st_u4(dst + i, lo, flag, hi, flag);
    }
    nvls_finish(R, P.ctas, advance);
    return;
  }
  const uint4* src = reinterpret_cast<const uint4*>(P.uc + area);
  bool ok = true;
  for (std::uint32_t i = first; i < P.lines && ok; i += stride) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i)
                 : "memory");
    if (v.y != flag || v.w != flag) {
      const std::uint64_t t0 = nv_timer();
      unsigned spins = 0;
      for (;;) {
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(src + i)
                     : "memory");
        if (v.y == flag && v.w == flag) break;
        if ((++spins & 1023u) == 0) {
          if (*(volatile int*)R.abort != 0) {
            ok = false;
            break;
          }
          if (nv_timer() - t0 > P.timeout_ns) {
            atomicExch(R.abort, 1);
            if (atomicCAS(&R.err->code, 0, 1) == 0) {
              R.err->rank = R.rank;
              R.err->peer = -1;
              R.err->lane = static_cast<int>(blockIdx.x);
              R.err->chunk = i;
              R.err->observed = v.y;
              R.err->expected = flag;
              __threadfence_system();
            }
            ok = false;
            break;
          }
        }
      }
      if (!ok) break;
    }
    const std::uint64_t off = static_cast<std::uint64_t>(i) * 8;
    if (aligned && off + 8 <= P.bytes) {
      *reinterpret_cast<uint2*>(R.buf + off) = make_uint2(v.x, v.z);
    } else {
      for (std::uint32_t b = 0; b < 8 && off + b < P.bytes; ++b) {
        R.buf[off + b] = static_cast<std::uint8_t>((b < 4 ? v.x >> (8 * b) : v.z >> (8 * (b - 4))) & 0xFFu);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && ok) mc_add_release(mc_done, 1);  // this CTA's lines of the half are read
  nvls_finish(R, P.ctas, advance);
}

}  // namespace
}  // namespace dev

NvlsGeometry nvls_geometry(std::uint64_t bytes, std::uint32_t slot_bytes, int wave) {
  NvlsGeometry g;
  if (bytes == 0) return g;
  const std::uint64_t w = static_cast<std::uint64_t>(std::max(wave, 1));
  const std::uint64_t per_wave = w * slot_bytes;
  const std::uint64_t waves = (bytes + per_wave - 1) / per_wave;
  std::uint64_t piece = (bytes + w * waves - 1) / (w * waves);
  piece = std::clamp<std::uint64_t>((piece + 15) / 16 * 16, std::min<std::uint64_t>(dev::kNvlsMinPiece, slot_bytes),
                                    slot_bytes);
  g.piece_bytes = piece;
  g.pieces = static_cast<std::uint32_t>((bytes + piece - 1) / piece);
  return g;
}

int nvls_occupancy(int* blocks_per_sm) {
  return static_cast<int>(
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, dev::nvls_kernel<1>, dev::kNvlsThreads, 0));
}

int nvls_ll_occupancy(int* blocks_per_sm) {
  return static_cast<int>(
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, dev::nvls_ll_kernel<1>, 512, 0));
}

int launch_nvls_ll(const dev::NvlsLLParams& p, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.n_local * p.ctas));
  cfg.blockDim = dim3(512);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = static_cast<unsigned>(fill_launch_attrs(attr, p.n_local > 1 ? 1 : 0));
  if (p.n_local == 1) {
    dev::NvlsLLParamsT<1> one;
    std::memcpy(&one, &p, offsetof(dev::NvlsLLParams, ranks));
    one.ranks[0] = p.ranks[0];
    return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::nvls_ll_kernel<1>, one));
  }
  return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::nvls_ll_kernel<dev::kMaxLocal>, p));
}

int launch_nvls(const dev::NvlsParams& p, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.n_local * p.ctas));
  cfg.blockDim = dim3(dev::kNvlsThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  // The root and the receivers sharing its GPU wait on one another.
  cfg.numAttrs = static_cast<unsigned>(fill_launch_attrs(attr, p.n_local > 1 ? 1 : 0));
  if (p.n_local == 1) {
    dev::NvlsParamsT<1> one;
    std::memcpy(&one, &p, offsetof(dev::NvlsParams, ranks));
    one.ranks[0] = p.ranks[0];
    return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::nvls_kernel<1>, one));
  }
  return static_cast<int>(cudaLaunchKernelEx(&cfg, dev::nvls_kernel<dev::kMaxLocal>, p));
}

// ------------------------------------------------------------ driver API

namespace {

struct Driver {
  CUresult (*GetErrorString)(CUresult, const char**){};
  CUresult (*DeviceGet)(CUdevice*, int){};
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice){};
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*){};
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice){};
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long){};
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t){};
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags){};
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long){};
  CUresult (*MemRelease)(CUmemGenericAllocationHandle){};
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long){};
  CUresult (*MemAddressFree)(CUdeviceptr, size_t){};
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long){};
  CUresult (*MemUnmap)(CUdeviceptr, size_t){};
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t){};
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags){};
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long){};
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType){};
  std::string error;
};

template <class F>
void load(F& f, const char* name, std::string& err) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || p == nullptr ||
      q != cudaDriverEntryPointSuccess) {
    if (err.empty()) err = std::string("driver entry point ") + name + " unavailable";
    cudaGetLastError();
    return;
  }
  f = reinterpret_cast<F>(p);
}

const Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    load(d.GetErrorString, "cuGetErrorString", d.error);
    load(d.DeviceGet, "cuDeviceGet", d.error);
    load(d.DeviceGetAttribute, "cuDeviceGetAttribute", d.error);
    load(d.MulticastCreate, "cuMulticastCreate", d.error);
    load(d.MulticastAddDevice, "cuMulticastAddDevice", d.error);
    load(d.MulticastBindMem, "cuMulticastBindMem", d.error);
    load(d.MulticastUnbind, "cuMulticastUnbind", d.error);
    load(d.MulticastGetGranularity, "cuMulticastGetGranularity", d.error);
    load(d.MemCreate, "cuMemCreate", d.error);
    load(d.MemRelease, "cuMemRelease", d.error);
    load(d.MemAddressReserve, "cuMemAddressReserve", d.error);
    load(d.MemAddressFree, "cuMemAddressFree", d.error);
    load(d.MemMap, "cuMemMap", d.error);
    load(d.MemUnmap, "cuMemUnmap", d.error);
    load(d.MemSetAccess, "cuMemSetAccess", d.error);
    load(d.MemGetAllocationGranularity, "cuMemGetAllocationGranularity", d.error);
    load(d.MemExportToShareableHandle, "cuMemExportToShareableHandle", d.error);
    load(d.MemImportFromShareableHandle, "cuMemImportFromShareableHandle", d.error);
  });
  if (!d.error.empty()) throw std::runtime_error("NVLS: " + d.error);
  return d;
}

void cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  throw std::runtime_error(std::string("NVLS: ") + what + ": " + (s ? s : "unknown driver error"));
}

void rt(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("NVLS: ") + what + ": " + cudaGetErrorString(e));
}

std::uint64_t ll_area_offset() { return static_cast<std::uint64_t>(dev::kNvlsCtlBytes) + dev::kNvlsRingBytes; }
std::uint64_t bound_bytes() { return ll_area_offset() + 2 * dev::kNvlsLLLines * 16; }

CUmulticastObjectProp mc_prop(int n_devices, std::uint64_t size, unsigned long long handle_types) {
  CUmulticastObjectProp prop = {};
  prop.numDevices = static_cast<unsigned>(n_devices);
  prop.size = size;
  prop.handleTypes = handle_types;
  return prop;
}

constexpr std::uint32_t kBlobMagic = 0xB200BC59u;
struct Blob {
  std::uint32_t magic;
  std::int32_t kind;  // 1 fabric, 2 fd over a Unix socket
  std::int32_t n_devices;
  std::int32_t pad;
  std::uint64_t size;
  std::uint8_t fabric[64];
  char socket[32];
};
static_assert(sizeof(Blob) <= NvlsTeam::kBlobBytes, "NVLS blob too large");

// Sends `fd` once per accepted connection, `count` times, or until the
// listening socket is shut down (the owner's destructor).
void serve_fd(int listen_fd, int fd, int count) {
  for (int served = 0; served < count;) {
    pollfd p{listen_fd, POLLIN, 0};
    const int r = ::poll(&p, 1, 200);
    if (r < 0 || (p.revents & (POLLERR | POLLHUP | POLLNVAL))) return;
    if (r == 0) continue;
    const int c = ::accept(listen_fd, nullptr, nullptr);
    if (c < 0) return;
    char byte = 'n';
    iovec iov{&byte, 1};
    alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))];
    msghdr m{};
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = ctl;
    m.msg_controllen = sizeof ctl;
    cmsghdr* h = CMSG_FIRSTHDR(&m);
    h->cmsg_level = SOL_SOCKET;
    h->cmsg_type = SCM_RIGHTS;
    h->cmsg_len = CMSG_LEN(sizeof(int));
    std::memcpy(CMSG_DATA(h), &fd, sizeof(int));
    if (::sendmsg(c, &m, 0) == 1) ++served;
    ::close(c);
  }
}

sockaddr_un abstract_addr(const std::string& name, socklen_t* len) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  a.sun_path[0] = '\0';
  std::memcpy(a.sun_path + 1, name.data(), std::min(name.size(), sizeof(a.sun_path) - 2));
  *len = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + name.size());
  return a;
}

int receive_fd(const std::string& name, double timeout_s) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const int s = ::socket(AF_UNIX, SOCK_STREAM, 0);
    if (s < 0) throw std::runtime_error("NVLS: socket() failed");
    socklen_t len = 0;
    sockaddr_un a = abstract_addr(name, &len);
    if (::connect(s, reinterpret_cast<sockaddr*>(&a), len) == 0) {
      char byte = 0;
      iovec iov{&byte, 1};
      alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))];
      msghdr m{};
      m.msg_iov = &iov;
      m.msg_iovlen = 1;
      m.msg_control = ctl;
      m.msg_controllen = sizeof ctl;
      const ssize_t r = ::recvmsg(s, &m, 0);
      ::close(s);
      cmsghdr* h = CMSG_FIRSTHDR(&m);
      if (r == 1 && h != nullptr && h->cmsg_type == SCM_RIGHTS) {
        int fd = -1;
        std::memcpy(&fd, CMSG_DATA(h), sizeof(int));
        return fd;
      }
      throw std::runtime_error("NVLS: no descriptor received from the multicast owner");
    }
    ::close(s);
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      throw std::runtime_error("NVLS: cannot reach the multicast owner's socket");
    }
    ::usleep(2000);
  }
}

}  // namespace

bool NvlsTeam::supported(int device, std::string* why) {
  try {
    const Driver& d = drv();
    CUdevice dv{};
    cu(d.DeviceGet(&dv, device), "cuDeviceGet");
    int mc = 0;
    cu(d.DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dv), "cuDeviceGetAttribute");
    if (!mc) {
      if (why) *why = "device reports no multicast support";
      return false;
    }
    return true;
  } catch (const std::exception& e) {
    if (why) *why = e.what();
    return false;
  }
}

NvlsTeam::~NvlsTeam() {
  if (listen_fd_ >= 0) ::shutdown(listen_fd_, SHUT_RDWR);
  if (server_.joinable()) server_.join();
  if (listen_fd_ >= 0) ::close(listen_fd_);
  if (fd_ >= 0) ::close(fd_);
  if (handle_ == 0) return;
  const Driver& d = drv();
  for (Binding& b : bindings_) {
    int saved = 0;
    cudaGetDevice(&saved);
    cudaSetDevice(b.device);
    cudaDeviceSynchronize();
    if (b.mc) {
      d.MemUnmap(b.mc, size_);
      d.MemAddressFree(b.mc, size_);
    }
    if (b.uc) {
      d.MemUnmap(b.uc, size_);
      d.MemAddressFree(b.uc, size_);
    }
    if (b.bound) {
      CUdevice dv{};
      d.DeviceGet(&dv, b.device);
      d.MulticastUnbind(handle_, dv, 0, size_);
    }
    if (b.mem) d.MemRelease(b.mem);
    cudaSetDevice(saved);
  }
  d.MemRelease(handle_);
}

void NvlsTeam::bind_device(Binding& b) {
  const Driver& d = drv();
  int saved = 0;
  rt(cudaGetDevice(&saved), "cudaGetDevice");
  rt(cudaSetDevice(b.device), "cudaSetDevice");
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = b.device;
  std::size_t mgran = 0;
  cu(d.MemGetAllocationGranularity(&mgran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity");
  // The bound memory carries the object's handle type (one process per GPU:
  // POSIX descriptors), as the driver requires for binding.
  if (kind_ == "fd") ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  cu(d.MemCreate(&b.mem, size_, &ap, 0), "cuMemCreate");
  // Every GPU of the team has been added by now (one process: above; one
  // process per GPU: the caller agreed on it), so binding does not wait.
  cu(d.MulticastBindMem(handle_, 0, b.mem, 0, size_, 0), "cuMulticastBindMem");
  b.bound = true;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = b.device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu(d.MemAddressReserve(&b.uc, size_, std::max<std::size_t>(mgran, gran_), 0, 0), "cuMemAddressReserve");
  cu(d.MemMap(b.uc, size_, 0, b.mem, 0), "cuMemMap(unicast)");
  cu(d.MemSetAccess(b.uc, size_, &acc, 1), "cuMemSetAccess(unicast)");
  cu(d.MemAddressReserve(&b.mc, size_, gran_, 0, 0), "cuMemAddressReserve");
  cu(d.MemMap(b.mc, size_, 0, handle_, 0), "cuMemMap(multicast)");
  cu(d.MemSetAccess(b.mc, size_, &acc, 1), "cuMemSetAccess(multicast)");
  // Counters start at zero (monotone afterwards), so do the LL lines' flags
  // (call epochs start at 1); the data ring needs no init.
  rt(cudaMemset(reinterpret_cast<void*>(b.uc), 0, dev::kNvlsCtlBytes), "cudaMemset(counters)");
  rt(cudaMemset(reinterpret_cast<void*>(b.uc + ll_area_offset()), 0, 2 * dev::kNvlsLLLines * 16),
     "cudaMemset(ll area)");
  rt(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  rt(cudaSetDevice(saved), "cudaSetDevice");
}

std::unique_ptr<NvlsTeam> NvlsTeam::create_local(const std::vector<int>& devices) {
  const Driver& d = drv();
  if (devices.size() < 2) throw std::runtime_error("NVLS: a multicast team needs at least two GPUs");
  std::unique_ptr<NvlsTeam> t(new NvlsTeam());
  t->kind_ = "local";
  t->n_devices_ = static_cast<int>(devices.size());
  CUmulticastObjectProp prop = mc_prop(t->n_devices_, bound_bytes(), 0);
  std::size_t gran = 0;
  cu(d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  t->gran_ = gran;
  t->size_ = (bound_bytes() + gran - 1) / gran * gran;
  prop.size = t->size_;
  cu(d.MulticastCreate(&t->handle_, &prop), "cuMulticastCreate");
  for (int dv : devices) {
    CUdevice cdev{};
    cu(d.DeviceGet(&cdev, dv), "cuDeviceGet");
    cu(d.MulticastAddDevice(t->handle_, cdev), "cuMulticastAddDevice");
    t->bindings_.push_back(Binding{dv, 0, 0, 0, false});
  }
  for (Binding& b : t->bindings_) t->bind_device(b);
  return t;
}

std::unique_ptr<NvlsTeam> NvlsTeam::create_owner(int n_devices, int device) {
  const Driver& d = drv();
  std::unique_ptr<NvlsTeam> t(new NvlsTeam());
  t->n_devices_ = n_devices;
  t->bindings_.push_back(Binding{device, 0, 0, 0, false});
  // The POSIX descriptor of the object is handed to each importer over an
  // abstract Unix socket (SCM_RIGHTS). (Fabric handles would travel as bytes
  // but need an IMEX channel; exporting one without it fails with an unknown
  // error that poisons later CUDA IPC calls on this box, so they are not tried.)
  CUmulticastObjectProp prop = mc_prop(n_devices, bound_bytes(), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  std::size_t gran = 0;
  cu(d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  t->gran_ = gran;
  t->size_ = (bound_bytes() + gran - 1) / gran * gran;
  prop.size = t->size_;
  cu(d.MulticastCreate(&t->handle_, &prop), "cuMulticastCreate(posix fd)");
  int fd = -1;
  cu(d.MemExportToShareableHandle(&fd, t->handle_, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
     "cuMemExportToShareableHandle(posix fd)");
  t->fd_ = fd;
  t->kind_ = "fd";
  std::random_device rd;
  char name[32];
  std::snprintf(name, sizeof name, "bcl-nvls-%d-%08x", static_cast<int>(::getpid()), rd());
  t->socket_name_ = name;
  t->listen_fd_ = ::socket(AF_UNIX, SOCK_STREAM, 0);
  socklen_t len = 0;
  sockaddr_un a = abstract_addr(t->socket_name_, &len);
  if (t->listen_fd_ < 0 || ::bind(t->listen_fd_, reinterpret_cast<sockaddr*>(&a), len) != 0 ||
      ::listen(t->listen_fd_, 64) != 0) {
    throw std::runtime_error("NVLS: cannot open the descriptor socket");
  }
  t->server_ = std::thread(serve_fd, t->listen_fd_, t->fd_, n_devices - 1);
  return t;
}

void NvlsTeam::export_blob(std::uint8_t out[kBlobBytes]) const {
  Blob b{};
  b.magic = kBlobMagic;
  b.kind = kind_ == "fabric" ? 1 : 2;
  b.n_devices = n_devices_;
  b.size = size_;
  std::memcpy(b.fabric, fabric_, sizeof b.fabric);
  std::snprintf(b.socket, sizeof b.socket, "%s", socket_name_.c_str());
  std::memset(out, 0, kBlobBytes);
  std::memcpy(out, &b, sizeof b);
}

std::unique_ptr<NvlsTeam> NvlsTeam::import(const std::uint8_t blob[kBlobBytes], int device) {
  const Driver& d = drv();
  Blob b{};
  std::memcpy(&b, blob, sizeof b);
  if (b.magic != kBlobMagic) throw std::runtime_error("NVLS: malformed multicast blob");
  std::unique_ptr<NvlsTeam> t(new NvlsTeam());
  t->n_devices_ = b.n_devices;
  t->size_ = b.size;
  t->bindings_.push_back(Binding{device, 0, 0, 0, false});
  CUmulticastObjectProp prop = mc_prop(b.n_devices, b.size, 0);
  std::size_t gran = 0;
  cu(d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  t->gran_ = gran;
  if (b.kind == 1) {
    CUmemFabricHandle fh{};
    std::memcpy(&fh, b.fabric, sizeof b.fabric);
    cu(d.MemImportFromShareableHandle(&t->handle_, &fh, CU_MEM_HANDLE_TYPE_FABRIC), "import(fabric)");
    t->kind_ = "fabric";
  } else {
    t->fd_ = receive_fd(std::string(b.socket, strnlen(b.socket, sizeof b.socket)), 30.0);
    cu(d.MemImportFromShareableHandle(&t->handle_, reinterpret_cast<void*>(static_cast<std::uintptr_t>(t->fd_)),
                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
       "import(fd)");
    t->kind_ = "fd";
  }
  return t;
}

void NvlsTeam::add_device() {
  const Driver& d = drv();
  CUdevice cdev{};
  cu(d.DeviceGet(&cdev, bindings_.front().device), "cuDeviceGet");
  cu(d.MulticastAddDevice(handle_, cdev), "cuMulticastAddDevice");
}

void NvlsTeam::bind_and_map() { bind_device(bindings_.front()); }

std::uint8_t* NvlsTeam::mc(int device) const {
  for (const Binding& b : bindings_) {
    if (b.device == device) return reinterpret_cast<std::uint8_t*>(b.mc);
  }
  throw std::invalid_argument("NVLS: device not in the multicast team");
}

std::uint8_t* NvlsTeam::uc(int device) const {
  for (const Binding& b : bindings_) {
    if (b.device == device) return reinterpret_cast<std::uint8_t*>(b.uc);
  }
  throw std::invalid_argument("NVLS: device not in the multicast team");
}

}  // namespace bcl
