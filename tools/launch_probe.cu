// Dev probe: event-timed cost of launching an (almost) empty kernel of the
// broadcast kernel's shape -- 148 CTAs x 288 threads, with/without 128 KiB of
// dynamic shared memory, cooperative or not -- against a one-CTA launch.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>
__global__ void k_empty(int* p) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0 && p[0] == 12345) sm[0] = 1, p[1] = sm[0];
}
__global__ void k_gate(long long ns) {
  long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); if (t - t0 > ns) break; }
}
__global__ void k_big_static(int* p) {  // a barrier-shaped predecessor
  if (threadIdx.x == 0 && p[0] == 12345) p[1] = 1;
}
int main() {
  int* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct Cfg { const char* name; int grid, block, smem, coop, pre; };
  Cfg cfgs[] = {{"1x32", 1, 32, 0, 0, 0}, {"148x288", 148, 288, 0, 0, 0}, {"148x288 smem128K", 148, 288, 128 << 10, 0, 0},
                {"148x288 smem128K after barrier-kernel", 148, 288, 128 << 10, 0, 1},
                {"148x288 smem128K coop", 148, 288, 128 << 10, 1, 0}, {"64x512", 64, 512, 0, 0, 0},
                {"148x288 smem64K", 148, 288, 64 << 10, 0, 0}, {"148x288 smem16K", 148, 288, 16 << 10, 0, 0}};
  for (int gate = 0; gate < 2; ++gate)
  for (auto& c : cfgs) {
    std::vector<float> t;
    for (int i = 0; i < 200; ++i) {
      if (gate) k_gate<<<1, 1, 0, s>>>(100000);
      if (c.pre) k_big_static<<<1, 64, 0, s>>>(d);
      cudaEventRecord(a, s);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c.grid); cfg.blockDim = dim3(c.block); cfg.dynamicSmemBytes = c.smem; cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = c.coop;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_empty, d);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    std::printf("%s %-40s median %.2f us  p10 %.2f  p90 %.2f\n", gate ? "gated  " : "ungated", c.name, t[100], t[20], t[180]);
  }
  std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
