// NVLink P2P probe (dev tool, not product): pull bandwidth (LDG.128 and
// cp.async.bulk staged through shared memory), cross-GPU flag ping-pong
// latency, and cudaMemcpyPeerAsync bandwidth between device 0 and 1.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void pull_ldg(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = 8;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One elected thread per CTA streams [lo,hi) of the message through a ring of
// shared-memory stages: bulk load from (peer) global, bulk store to local.
__global__ void pull_bulk(const char* src, char* dst, size_t bytes, size_t piece) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[8];
  const int S = 8;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  size_t per_cta = (bytes + gridDim.x - 1) / gridDim.x;
  per_cta = (per_cta + 15) & ~size_t(15);
  size_t lo = blockIdx.x * per_cta, hi = lo + per_cta < bytes ? lo + per_cta : bytes;
  uint32_t phase[8] = {0};
  const size_t L = 4;
  size_t npieces = hi > lo ? (hi - lo + piece - 1) / piece : 0;
  for (size_t p = 0; p < npieces + L; ++p) {
    if (p < npieces) {
      int s = p % S;
      if (p >= (size_t)S) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
      size_t off = lo + p * piece;
      uint32_t len = (uint32_t)((hi - off) < piece ? (hi - off) : piece);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&full[s])), "r"(len) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(smem + s * piece)), "l"(src + off), "r"(len), "r"(smem_u32(&full[s])) : "memory");
    }
    if (p >= L) {
      size_t q = p - L;
      int sq = q % S;
      uint32_t ph = phase[sq];
      asm volatile("{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}" :: "r"(smem_u32(&full[sq])), "r"(ph) : "memory");
      phase[sq] ^= 1;
      size_t qoff = lo + q * piece;
      uint32_t qlen = (uint32_t)((hi - qoff) < piece ? (hi - qoff) : piece);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + qoff), "r"(smem_u32(smem + sq * piece)), "r"(qlen) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void pingpong(volatile uint64_t* my_flag, uint64_t* peer_flag, int iters, int role, unsigned long long* out_ns) {
  uint64_t t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (role == 0) {
      asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((uint64_t)i) : "memory");
      uint64_t v; do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory"); } while (v < (uint64_t)i);
    } else {
      uint64_t v; do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory"); } while (v < (uint64_t)i);
      asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(peer_flag), "l"((uint64_t)i) : "memory");
    }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (role == 0) *out_ns = t1 - t0;
}

int main() {
  int ndev = 0; CK(cudaGetDeviceCount(&ndev));
  printf("devices %d\n", ndev);
  for (int d = 0; d < ndev; ++d) {
    int mc = 0; cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    printf("dev %d sms %d multicast %d\n", d, sms, mc);
  }
  if (ndev < 2) return 0;
  int can = 0; CK(cudaDeviceCanAccessPeer(&can, 1, 0)); printf("can access peer 1->0: %d\n", can);
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));
  const size_t bytes = 256ull << 20;
  char *a, *b; CK(cudaSetDevice(0)); CK(cudaMalloc(&a, bytes)); CK(cudaMemset(a, 1, bytes));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&b, bytes)); CK(cudaMemset(b, 0, bytes));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  int grids[] = {148, 296, 592, 1184};
  for (int g : grids) for (int t : {256, 512}) {
    for (int w = 0; w < 2; ++w) pull_ldg<<<g, t>>>((const int4*)a, (int4*)b, bytes / 16);
    CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) pull_ldg<<<g, t>>>((const int4*)a, (int4*)b, bytes / 16);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("pull_ldg grid %d thr %d: %.1f GB/s\n", g, t, 5.0 * bytes / (ms * 1e6));
  }
  for (int g : {148, 296}) for (size_t piece : {4096ul, 8192ul, 16384ul, 24576ul}) {
    size_t sm = piece * 8;
    if (sm > 200 * 1024) continue;
    CK(cudaFuncSetAttribute(pull_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (int w = 0; w < 2; ++w) pull_bulk<<<g, 32, sm>>>(a, b, bytes, piece);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) pull_bulk<<<g, 32, sm>>>(a, b, bytes, piece);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("pull_bulk grid %d piece %zu: %.1f GB/s\n", g, piece, 5.0 * bytes / (ms * 1e6));
  }
  // verify last copy
  {
    char h[64]; CK(cudaMemcpy(h, b + bytes - 64, 64, cudaMemcpyDeviceToHost));
    printf("verify tail byte %d\n", (int)h[63]);
  }
  // local copy for reference
  {
    char* c; CK(cudaMalloc(&c, bytes));
    for (int w = 0; w < 2; ++w) pull_ldg<<<592, 512>>>((const int4*)b, (int4*)c, bytes / 16);
    CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) pull_ldg<<<592, 512>>>((const int4*)b, (int4*)c, bytes / 16);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("local copy (r+w counted once): %.1f GB/s\n", 5.0 * bytes / (ms * 1e6));
    CK(cudaFree(c));
  }
  // memcpy peer
  CK(cudaMemcpyPeerAsync(b, 1, a, 0, bytes));
  CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) CK(cudaMemcpyPeerAsync(b, 1, a, 0, bytes));
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("memcpyPeer: %.1f GB/s\n", 5.0 * bytes / (ms * 1e6));
  // ping-pong latency
  uint64_t *f0, *f1; unsigned long long* out;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&f0, 64)); CK(cudaMemset(f0, 0, 64)); CK(cudaMallocManaged(&out, 8));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&f1, 64)); CK(cudaMemset(f1, 0, 64));
  CK(cudaDeviceSynchronize());
  const int iters = 10000;
  CK(cudaSetDevice(1)); pingpong<<<1, 1>>>(f1, f0, iters, 1, out);
  CK(cudaSetDevice(0)); pingpong<<<1, 1>>>(f0, f1, iters, 0, out);
  CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
  printf("pingpong round trip: %.3f us\n", (double)*out / iters / 1000.0);
  return 0;
}
