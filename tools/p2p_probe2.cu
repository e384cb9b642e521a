// Dev probe: NVLink throughput of pull (peer loads) vs push (peer stores),
// one direction, both directions at once, and a 3/4-GPU "chain" where every
// GPU moves data from its upstream at the same time (no synchronisation).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void copy_k(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
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

int main() {
  int nd = 0; CK(cudaGetDeviceCount(&nd));
  const size_t bytes = 512ull << 20;
  std::vector<char*> a(nd), b(nd);
  std::vector<cudaStream_t> st(nd);
  std::vector<cudaEvent_t> e0(nd), e1(nd);
  for (int d = 0; d < nd; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < nd; ++p) if (p != d) cudaDeviceEnablePeerAccess(p, 0);
    cudaGetLastError();
    CK(cudaMalloc(&a[d], bytes)); CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], d + 1, bytes)); CK(cudaMemset(b[d], 0, bytes));
    CK(cudaStreamCreate(&st[d])); CK(cudaEventCreate(&e0[d])); CK(cudaEventCreate(&e1[d]));
  }
  for (int d = 0; d < nd; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
  // A transfer = (executing device, src ptr, dst ptr)
  struct T { int dev; const char* src; char* dst; };
  auto run = [&](const char* name, std::vector<T> ts) -> int {
    for (int rep = 0; rep < 4; ++rep) {
      for (auto& t : ts) { CK(cudaSetDevice(t.dev)); CK(cudaEventRecord(e0[t.dev], st[t.dev]));
        copy_k<<<296, 512, 0, st[t.dev]>>>((const int4*)t.src, (int4*)t.dst, bytes / 16);
        CK(cudaEventRecord(e1[t.dev], st[t.dev])); }
      float worst = 0;
      for (auto& t : ts) { CK(cudaSetDevice(t.dev)); CK(cudaEventSynchronize(e1[t.dev])); float ms; CK(cudaEventElapsedTime(&ms, e0[t.dev], e1[t.dev])); if (ms > worst) worst = ms; }
      if (rep == 3) printf("%-44s per-transfer %.1f GB/s (slowest of %zu)\n", name, bytes / (worst * 1e6), ts.size());
    }
    return 0;
  };
  if (nd < 2) return 0;
  run("pull 1<-0 (dev1 loads peer)", {{1, a[0], b[1]}});
  run("push 0->1 (dev0 stores peer)", {{0, a[0], b[1]}});
  run("pull both ways 1<-0, 0<-1", {{1, a[0], b[1]}, {0, a[1], b[0]}});
  run("push both ways 0->1, 1->0", {{0, a[0], b[1]}, {1, a[1], b[0]}});
  if (nd >= 3) {
    run("pull chain 1<-0, 2<-1", {{1, a[0], b[1]}, {2, a[1], b[2]}});
    run("push chain 0->1, 1->2", {{0, a[0], b[1]}, {1, a[1], b[2]}});
  }
  if (nd >= 4) {
    run("pull chain 1<-0, 2<-1, 3<-2", {{1, a[0], b[1]}, {2, a[1], b[2]}, {3, a[2], b[3]}});
    run("push chain 0->1, 1->2, 2->3", {{0, a[0], b[1]}, {1, a[1], b[2]}, {2, a[2], b[3]}});
    run("pull ring 4 GPUs", {{1, a[0], b[1]}, {2, a[1], b[2]}, {3, a[2], b[3]}, {0, a[3], b[0]}});
    run("push fan-out 0->1,2,3 (root egress)", {{0, a[0], b[1]}, {0, a[0], b[2]}});
  }
  // local copy on a middle GPU while it is read by a peer
  if (nd >= 3) run("dev1 local copy while 2 pulls from 1", {{1, a[1], b[1]}, {2, a[1], b[2]}});
  return 0;
}
