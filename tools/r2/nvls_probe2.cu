// NVLS multicast broadcast probe v2 (round 2): root kernel variants (grid, block, loads in flight).
//
// One process, D GPUs. A multicast object of M bytes is bound to memory on
// every GPU; the root writes the payload ONCE through the multicast address
// (multimem.st, replicated by the NVSwitch), then publishes an epoch flag the
// same way; receivers poll their local copy of the flag and (optionally) copy
// the landed payload into a separate user buffer. Reported: steady-state time
// per broadcast over K back-to-back broadcasts (wall clock / K after a full
// device sync), bit-exact check of every GPU.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
//   tools/nvls_probe [devices] [bytes...]
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

__device__ __forceinline__ void mc_store_v4(void* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_store_u64(void* mc, unsigned long long v) {
  asm volatile("multimem.st.release.sys.global.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}

// Root: stream the payload into the multicast range, then the flag. Each
// thread keeps U 16-byte loads in flight before its multimem stores.
template <int U>
__global__ void root_kernel(const uint4* __restrict__ src, uint4* mc_data, unsigned long long* mc_flag,
                            unsigned int* done, size_t n16, unsigned long long epoch) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldg(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) mc_store_v4(mc_data + i + u * stride, r[u]);
  }
  for (; i < n16; i += stride) mc_store_v4(mc_data + i, src[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(done, 1u) + 1 == gridDim.x * epoch) mc_store_u64(mc_flag, epoch);
  }
}

// Receiver: wait for the flag on the local copy; optionally copy out.
__global__ void recv_kernel(const unsigned long long* flag, const uint4* landed, uint4* user, size_t n16,
                            unsigned long long epoch, int copy_out) {
  if (threadIdx.x == 0) {
    unsigned long long v;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    } while (v < epoch);
  }
  __syncthreads();
  if (!copy_out) return;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride) {
    user[i] = landed[i];
  }
}

int main(int argc, char** argv) {
  CU(cuInit(0));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int D = argc > 1 ? std::atoi(argv[1]) : ndev;
  std::vector<size_t> sizes;
  for (int i = 2; i < argc; ++i) sizes.push_back(std::strtoull(argv[i], nullptr, 10));
  if (sizes.empty()) sizes = {1 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30};
  size_t maxb = 0;
  for (size_t s : sizes) maxb = s > maxb ? s : maxb;
  int mc_ok = 0;
  CU(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0));
  std::printf("devices %d multicast_supported %d\n", D, mc_ok);
  if (!mc_ok || D < 2) return 0;

  CUmulticastObjectProp prop = {};
  prop.numDevices = static_cast<unsigned>(D);
  prop.handleTypes = 0;
  size_t gran = 0;
  prop.size = maxb + (2 << 20);
  CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t bytes_total = (maxb + (2 << 20) + gran - 1) / gran * gran;  // data + flag page
  prop.size = bytes_total;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &prop));
  std::vector<CUdevice> devs(D);
  for (int d = 0; d < D; ++d) {
    CU(cuDeviceGet(&devs[d], d));
    CU(cuMulticastAddDevice(mc, devs[d]));
  }
  std::vector<CUdeviceptr> uc(D), mcva(D);
  std::vector<CUmemGenericAllocationHandle> mem(D);
  std::vector<char*> src(D), user(D);
  std::vector<unsigned int*> done(D);
  std::vector<cudaStream_t> st(D);
  for (int d = 0; d < D; ++d) {
    CK(cudaSetDevice(d));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    size_t mgran = 0;
    CU(cuMemGetAllocationGranularity(&mgran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CU(cuMemCreate(&mem[d], bytes_total, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, mem[d], 0, bytes_total, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemAddressReserve(&uc[d], bytes_total, mgran, 0, 0));
    CU(cuMemMap(uc[d], bytes_total, 0, mem[d], 0));
    CU(cuMemSetAccess(uc[d], bytes_total, &acc, 1));
    CU(cuMemAddressReserve(&mcva[d], bytes_total, gran, 0, 0));
    CU(cuMemMap(mcva[d], bytes_total, 0, mc, 0));
    CU(cuMemSetAccess(mcva[d], bytes_total, &acc, 1));
    CK(cudaMemset(reinterpret_cast<void*>(uc[d]), 0, bytes_total));
    CK(cudaMalloc(&src[d], maxb));
    CK(cudaMalloc(&user[d], maxb));
    CK(cudaMalloc(&done[d], sizeof(unsigned int)));
    CK(cudaMemset(done[d], 0, sizeof(unsigned int)));
    CK(cudaStreamCreate(&st[d]));
  }
  // payload on the root
  {
    std::vector<unsigned char> h(maxb);
    unsigned long long x = 88172645463325252ull;
    for (auto& c : h) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      c = static_cast<unsigned char>(x);
    }
    CK(cudaSetDevice(0));
    CK(cudaMemcpy(src[0], h.data(), maxb, cudaMemcpyHostToDevice));
  }
  for (int d = 0; d < D; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
  unsigned long long epoch = 0;
  struct Cfg { int grid, block, unroll; };
  const Cfg cfgs[] = {{148, 512, 1}, {148, 512, 4}, {148, 512, 8}, {296, 512, 4}, {296, 1024, 4}, {592, 512, 8},
                      {148, 1024, 8}};
  for (const Cfg& cf : cfgs) {
  const int grid = cf.grid, block = cf.block;
  for (auto& dd : done) { CK(cudaSetDevice(0)); }
  for (int copy_out = 0; copy_out < 1; ++copy_out) {
    for (size_t bytes : sizes) {
      const size_t n16 = bytes / 16;
      const int K = bytes >= (256u << 20) ? 10 : 50;
      auto one = [&]() {
        ++epoch;
        for (int d = 1; d < D; ++d) {
          CK(cudaSetDevice(d));
          recv_kernel<<<grid, block, 0, st[d]>>>(reinterpret_cast<unsigned long long*>(uc[d] + maxb),
                                                reinterpret_cast<uint4*>(uc[d]), reinterpret_cast<uint4*>(user[d]),
                                                n16, epoch, copy_out);
        }
        CK(cudaSetDevice(0));
        auto* sp = reinterpret_cast<uint4*>(src[0]);
        auto* mp = reinterpret_cast<uint4*>(mcva[0]);
        auto* fp = reinterpret_cast<unsigned long long*>(mcva[0] + maxb);
        if (cf.unroll == 1) root_kernel<1><<<grid, block, 0, st[0]>>>(sp, mp, fp, done[0], n16, epoch);
        else if (cf.unroll == 4) root_kernel<4><<<grid, block, 0, st[0]>>>(sp, mp, fp, done[0], n16, epoch);
        else root_kernel<8><<<grid, block, 0, st[0]>>>(sp, mp, fp, done[0], n16, epoch);
      };
      // reset the root counter so epoch accounting (grid * epoch) holds
      for (int w = 0; w < 3; ++w) one();
      for (int d = 0; d < D; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      const auto t0 = std::chrono::steady_clock::now();
      for (int k = 0; k < K; ++k) one();
      for (int d = 0; d < D; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / K;
      // verify
      bool ok = true;
      std::vector<unsigned char> a(bytes), b(bytes);
      CK(cudaSetDevice(0));
      CK(cudaMemcpy(a.data(), src[0], bytes, cudaMemcpyDeviceToHost));
      for (int d = 1; d < D; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMemcpy(b.data(), copy_out ? user[d] : reinterpret_cast<void*>(uc[d]), bytes, cudaMemcpyDeviceToHost));
        ok = ok && a == b;
      }
      std::printf("nvls D=%d grid=%d block=%d unroll=%d bytes=%zu  %.2f us/bcast  %.1f GB/s  %s\n", D, grid, block,
                  cf.unroll, bytes, sec * 1e6, bytes / sec / 1e9, ok ? "bit-exact" : "MISMATCH");
    }
  }
  // the root's done counter counts grid * epoch arrivals: restart it per config
  CK(cudaSetDevice(0));
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(done[0], 0, sizeof(unsigned int)));
  epoch = 0;
  for (int d = 1; d < D; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMemset(reinterpret_cast<void*>(uc[d] + maxb), 0, 64));
  }
  for (int d = 0; d < D; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
  }
  return 0;
}
