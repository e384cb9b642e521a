// Traffic-mix ceiling of the N=1 workload (config 1): what HBM delivers for
// "read 64 MiB once, write it 3 times" without any chain dependency, against
// a plain 1:1 copy of the same bytes. Grid-stride 16-byte loads, 4 in flight
// per thread, 3 stores each; a 256 MiB read sweep evicts L2 before every timed
// launch; CUDA events, median of 20.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/r2/mix_probe tools/r2/mix_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void fanout(const uint4* __restrict__ s, uint4* a, uint4* b, uint4* c, size_t n, int outs) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = s[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[i + u * stride] = v[u];
      if (outs > 1) b[i + u * stride] = v[u];
      if (outs > 2) c[i + u * stride] = v[u];
    }
  }
  for (; i < n; i += stride) {
    const uint4 v = s[i];
    a[i] = v;
    if (outs > 1) b[i] = v;
    if (outs > 2) c[i] = v;
  }
}

__global__ void sweep(const int4* f, size_t n, int* sink) {
  int acc = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    acc ^= f[i].x;
  if (acc == 0x12345678) *sink = acc;
}

int main() {
  const size_t M = 64ull << 20, n = M / 16;
  uint4 *s, *a, *b, *c;
  int4* fl;
  int* sink;
  cudaMalloc(&s, M);
  cudaMalloc(&a, M);
  cudaMalloc(&b, M);
  cudaMalloc(&c, M);
  cudaMalloc(&fl, 256ull << 20);
  cudaMalloc(&sink, 4);
  cudaMemset(s, 1, M);
  cudaMemset(fl, 0, 256ull << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int outs = 1; outs <= 3; ++outs) {
    for (int per_sm : {2, 4, 8}) {
      std::vector<float> ts;
      for (int it = 0; it < 25; ++it) {
        sweep<<<sms * 8, 512>>>(fl, (256ull << 20) / 16, sink);
        cudaEventRecord(e0);
        fanout<<<sms * per_sm, 256>>>(s, a, b, c, n, outs);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 5) ts.push_back(ms * 1000.f);
      }
      std::sort(ts.begin(), ts.end());
      const double us = ts[ts.size() / 2];
      const double bytes = static_cast<double>(M) * (1 + outs);
      std::printf("read 64 MiB, write x%d, %d CTAs/SM: %.1f us  %.0f GB/s of (1+%d)M\n", outs, per_sm, us,
                  bytes / us / 1e3, outs);
    }
  }
  std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
