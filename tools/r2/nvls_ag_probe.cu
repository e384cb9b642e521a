// NVLS probe 3 (round 2): can several sources multicasting at once beat the
// single-source multicast ceiling (~572 GB/s) and the chain's bidirectional
// ceiling (653 GB/s)? One process, D GPUs.
//
//   mode 1  single source: GPU 0 writes all M bytes through the multicast
//           address (the probe-2 baseline).
//   mode 2  all sources: GPU d writes bytes [d*M/D, (d+1)*M/D) through the
//           multicast address (an NVLS all-gather of M bytes); every GPU
//           waits until every source's flag arrived (multimem.red on a
//           counter replicated on every GPU).
//   mode 3  direct-pull all-gather: GPU d reads the D-1 foreign pieces from
//           the peers' unicast copies (P2P loads) into its own copy.
// Also reports: multicast support, handle types (fabric / POSIX fd), and
// whether a one-device multicast object can be created and written.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/r2/nvls_ag_probe tools/r2/nvls_ag_probe.cu -lcuda
//   tools/r2/nvls_ag_probe [devices] [bytes...]
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CU(x)                                                                   \
  do {                                                                          \
    CUresult r = (x);                                                           \
    if (r != CUDA_SUCCESS) {                                                    \
      const char* s = nullptr;                                                  \
      cuGetErrorString(r, &s);                                                  \
      std::printf("CU error %s at %s:%d\n", s ? s : "?", __FILE__, __LINE__); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)
#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e = (x);                                                                       \
    if (e != cudaSuccess) {                                                                    \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                            \
    }                                                                                          \
  } while (0)

__device__ __forceinline__ void mc_st(void* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_add(unsigned long long* mc, unsigned long long v) {
  asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Writes n16 16-byte words of src through the multicast address, then adds 1
// to the replicated counter once per CTA; then waits until the counter
// reaches target (every CTA of every source).
__global__ void mc_kernel(const uint4* __restrict__ src, uint4* mc, unsigned long long* mc_cnt,
                          const unsigned long long* cnt, size_t n16, unsigned long long target) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 r0 = __ldg(src + i), r1 = __ldg(src + i + stride), r2 = __ldg(src + i + 2 * stride),
          r3 = __ldg(src + i + 3 * stride);
    mc_st(mc + i, r0);
    mc_st(mc + i + stride, r1);
    mc_st(mc + i + 2 * stride, r2);
    mc_st(mc + i + 3 * stride, r3);
  }
  for (; i < n16; i += stride) mc_st(mc + i, src[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (n16 > 0) {
      asm volatile("fence.proxy.alias;" ::: "memory");
      mc_add(mc_cnt, 1);
    }
    while (ld_acq(cnt) < target) {
    }
  }
  __syncthreads();
}

// Direct-pull all-gather: this GPU reads every foreign piece from its owner.
struct Pieces {
  const uint4* src[8];
};
__global__ void pull_kernel(Pieces p, uint4* dst, int D, int me, size_t piece16) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t total = piece16 * static_cast<size_t>(D - 1);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total; i += 4 * stride) {
    uint4 r[4];
    size_t at[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t j = i + u * stride;
      at[u] = ~size_t(0);
      if (j < total) {
        int k = static_cast<int>(j / piece16);
        const int owner = k >= me ? k + 1 : k;
        at[u] = static_cast<size_t>(owner) * piece16 + j % piece16;
        r[u] = p.src[owner][at[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (at[u] != ~size_t(0)) dst[at[u]] = r[u];
  }
}

int main(int argc, char** argv) {
  CU(cuInit(0));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int D = argc > 1 ? std::atoi(argv[1]) : ndev;
  std::vector<size_t> sizes;
  for (int i = 2; i < argc; ++i) sizes.push_back(std::strtoull(argv[i], nullptr, 10));
  if (sizes.empty()) sizes = {1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20};
  size_t maxb = 0;
  for (size_t s : sizes) maxb = s > maxb ? s : maxb;
  int mc_ok = 0, fab = 0, fd = 0;
  CUdevice d0;
  CU(cuDeviceGet(&d0, 0));
  CU(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d0));
  CU(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d0));
  CU(cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, d0));
  std::printf("devices %d (visible %d) multicast_supported %d fabric_handles %d posix_fd_handles %d\n", D, ndev,
              mc_ok, fab, fd);
  if (!mc_ok) return 0;

  // One-device multicast object with a shareable handle: does it create,
  // export and take multimem stores?
  for (int ht = 0; ht < 3; ++ht) {
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    prop.handleTypes = ht == 0 ? 0 : ht == 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_FABRIC;
    size_t gran = 0;
    prop.size = 2 << 20;
    CUresult r = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    prop.size = gran > 0 ? (2 << 20) / gran * gran + ((2 << 20) % gran ? gran : 0) : (2 << 20);
    CUmemGenericAllocationHandle mc{};
    CUresult r2 = r == CUDA_SUCCESS ? cuMulticastCreate(&mc, &prop) : r;
    CUresult r3 = CUDA_ERROR_UNKNOWN;
    if (r2 == CUDA_SUCCESS && ht == 1) {
      int f = -1;
      r3 = cuMemExportToShareableHandle(&f, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    } else if (r2 == CUDA_SUCCESS && ht == 2) {
      CUmemFabricHandle fh;
      r3 = cuMemExportToShareableHandle(&fh, mc, CU_MEM_HANDLE_TYPE_FABRIC, 0);
    }
    std::printf("one-device multicast handle_type=%s: granularity %zu (%d) create %d export %d\n",
                ht == 0 ? "none" : ht == 1 ? "posix_fd" : "fabric", gran, r, r2, ht == 0 ? 0 : (int)r3);
    if (r2 == CUDA_SUCCESS) {
      CU(cuMulticastAddDevice(mc, d0));
      CUmemAllocationProp ap = {};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ap.location.id = 0;
      ap.requestedHandleTypes = static_cast<CUmemAllocationHandleType>(prop.handleTypes);
      CUmemGenericAllocationHandle mem;
      CU(cuMemCreate(&mem, prop.size, &ap, 0));
      CU(cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0));
      CUdeviceptr uc, mv;
      CUmemAccessDesc acc = {};
      acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc.location.id = 0;
      acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      CU(cuMemAddressReserve(&uc, prop.size, gran, 0, 0));
      CU(cuMemMap(uc, prop.size, 0, mem, 0));
      CU(cuMemSetAccess(uc, prop.size, &acc, 1));
      CU(cuMemAddressReserve(&mv, prop.size, gran, 0, 0));
      CU(cuMemMap(mv, prop.size, 0, mc, 0));
      CU(cuMemSetAccess(mv, prop.size, &acc, 1));
      CK(cudaSetDevice(0));
      char* src;
      CK(cudaMalloc(&src, 1 << 20));
      CK(cudaMemset(src, 0x5a, 1 << 20));
      CK(cudaMemset(reinterpret_cast<void*>(uc), 0, prop.size));
      unsigned long long* cnt = reinterpret_cast<unsigned long long*>(uc + (1 << 20));
      mc_kernel<<<4, 256>>>(reinterpret_cast<uint4*>(src), reinterpret_cast<uint4*>(mv),
                            reinterpret_cast<unsigned long long*>(mv + (1 << 20)), cnt, (1 << 20) / 16, 4);
      CK(cudaDeviceSynchronize());
      std::vector<unsigned char> h(1 << 20);
      CK(cudaMemcpy(h.data(), reinterpret_cast<void*>(uc), 1 << 20, cudaMemcpyDeviceToHost));
      bool ok = true;
      for (unsigned char c : h) ok = ok && c == 0x5a;
      std::printf("  one-device multimem.st + red: %s\n", ok ? "landed" : "MISMATCH");
      CK(cudaFree(src));
      CU(cuMemUnmap(uc, prop.size));
      CU(cuMemUnmap(mv, prop.size));
      CU(cuMemAddressFree(uc, prop.size));
      CU(cuMemAddressFree(mv, prop.size));
      CU(cuMulticastUnbind(mc, d0, 0, prop.size));
      CU(cuMemRelease(mem));
      CU(cuMemRelease(mc));
    }
  }
  if (D < 2) return 0;

  CUmulticastObjectProp prop = {};
  prop.numDevices = static_cast<unsigned>(D);
  prop.handleTypes = 0;
  size_t gran = 0;
  prop.size = maxb + (2 << 20);
  CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t total = (maxb + (2 << 20) + gran - 1) / gran * gran;
  prop.size = total;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &prop));
  for (int d = 0; d < D; ++d) {
    CUdevice dv;
    CU(cuDeviceGet(&dv, d));
    CU(cuMulticastAddDevice(mc, dv));
  }
  std::vector<CUdeviceptr> uc(D), mv(D);
  std::vector<CUmemGenericAllocationHandle> mem(D);
  std::vector<char*> src(D);
  std::vector<cudaStream_t> st(D);
  for (int d = 0; d < D; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < D; ++e)
      if (e != d) cudaDeviceEnablePeerAccess(e, 0);
    cudaGetLastError();
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    CU(cuMemCreate(&mem[d], total, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, mem[d], 0, total, 0));
    CUmemAccessDesc acc[8] = {};
    for (int e = 0; e < D; ++e) {
      acc[e].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc[e].location.id = e;
      acc[e].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CU(cuMemAddressReserve(&uc[d], total, gran, 0, 0));
    CU(cuMemMap(uc[d], total, 0, mem[d], 0));
    CU(cuMemSetAccess(uc[d], total, acc, D));  // peers may read it (mode 3)
    CU(cuMemAddressReserve(&mv[d], total, gran, 0, 0));
    CU(cuMemMap(mv[d], total, 0, mc, 0));
    CU(cuMemSetAccess(mv[d], total, &acc[d], 1));
    CK(cudaMemset(reinterpret_cast<void*>(uc[d]), 0, total));
    CK(cudaMalloc(&src[d], maxb));
    std::vector<unsigned char> h(maxb);
    unsigned long long x = 88172645463325252ull ^ (d + 1) * 0x9e3779b97f4a7c15ull;
    for (auto& c : h) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      c = static_cast<unsigned char>(x);
    }
    CK(cudaMemcpy(src[d], h.data(), maxb, cudaMemcpyHostToDevice));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaDeviceSynchronize());
  }
  unsigned long long count = 0;  // replicated counter value after each round
  const int grids[] = {148, 296};
  for (int mode = 1; mode <= 3; ++mode) {
    for (int grid : grids) {
      for (size_t bytes : sizes) {
        const size_t piece = bytes / D / 16 * 16;
        const int K = bytes >= (256u << 20) ? 10 : 40;
        auto one = [&]() {
          if (mode == 1) count += grid;
          if (mode == 2) count += static_cast<unsigned long long>(grid) * D;
          for (int d = 0; d < D; ++d) {
            CK(cudaSetDevice(d));
            auto* cnt_uc = reinterpret_cast<unsigned long long*>(uc[d] + maxb);
            auto* cnt_mc = reinterpret_cast<unsigned long long*>(mv[d] + maxb);
            if (mode == 1) {
              mc_kernel<<<grid, 512, 0, st[d]>>>(reinterpret_cast<uint4*>(src[0]), reinterpret_cast<uint4*>(mv[d]),
                                                  cnt_mc, cnt_uc, d == 0 ? bytes / 16 : 0, count);
            } else if (mode == 2) {
              mc_kernel<<<grid, 512, 0, st[d]>>>(reinterpret_cast<uint4*>(src[d] + d * piece),
                                                  reinterpret_cast<uint4*>(mv[d] + d * piece), cnt_mc, cnt_uc,
                                                  piece / 16, count);
            } else {
              Pieces p{};
              for (int e = 0; e < D; ++e) p.src[e] = reinterpret_cast<const uint4*>(uc[e]);
              pull_kernel<<<grid, 512, 0, st[d]>>>(p, reinterpret_cast<uint4*>(src[d]), D, d, piece / 16);
            }
          }
        };
        // mode 1/2 kernels of non-sources also wait on the counter: they launch too
        for (int w = 0; w < 3; ++w) one();
        for (int d = 0; d < D; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        const auto t0 = std::chrono::steady_clock::now();
        for (int k = 0; k < K; ++k) one();
        for (int d = 0; d < D; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / K;
        const double moved = mode == 1 ? bytes : static_cast<double>(piece) * D;
        // check mode 2: every GPU's copy holds every source's piece
        const char* verdict = "";
        if (mode == 2) {
          bool ok = true;
          std::vector<unsigned char> a(piece), b(piece);
          for (int s = 0; s < D && ok; ++s) {
            CK(cudaSetDevice(s));
            CK(cudaMemcpy(a.data(), src[s] + s * piece, piece, cudaMemcpyDeviceToHost));
            for (int d = 0; d < D; ++d) {
              CK(cudaSetDevice(d));
              CK(cudaMemcpy(b.data(), reinterpret_cast<char*>(uc[d]) + s * piece, piece, cudaMemcpyDeviceToHost));
              ok = ok && a == b;
            }
          }
          verdict = ok ? "bit-exact" : "MISMATCH";
        }
        std::printf("mode %d (%s) D=%d grid=%d bytes=%zu  %.2f us  %.1f GB/s per receiver ingress %s\n", mode,
                    mode == 1 ? "one source" : mode == 2 ? "all sources" : "pull all-gather", D, grid, bytes,
                    sec * 1e6, moved * (mode == 1 ? 1.0 : (D - 1.0) / D) / sec / 1e9, verdict);
      }
    }
  }
  return 0;
}
