// Host cost per call (dev probe, 2 GPUs, one process): bcl_bcast of 8 bytes
// (`direct` on LL lines) issued for rank 0 then rank 1, against bare
// cudaLaunchKernelEx of an empty kernel with and without the PDL attribute.
// Host time only (the device drains after each batch).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/r2/host_cost.cu \
//        -Lpaper_1707_09414_b200 -lbcl -Xlinker -rpath=$PWD/paper_1707_09414_b200 -o tools/r2/host_cost
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

#include "bcl.h"

__global__ void empty_kernel(int) {}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  int devs[2] = {0, 1};
  bcl_comm_t comms[2];
  if (bcl_comm_init_all(2, devs, 10.0, comms) != 0) {
    std::printf("init failed: %s\n", bcl_last_error());
    return 1;
  }
  void* buf[2];
  cudaStream_t st[2];
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(r);
    cudaMalloc(&buf[r], 1 << 20);
    cudaStreamCreateWithFlags(&st[r], cudaStreamNonBlocking);
  }
  bcl_config_t cfg{BCL_DIRECT, 0, 0};
  const int kCalls = 400;
  for (int rep = 0; rep < 4; ++rep) {
    double t = 0;
    for (int i = 0; i < kCalls; ++i) {
      for (int r = 0; r < 2; ++r) {
        const double t0 = now_us();
        const int s = bcl_bcast(buf[r], 8, BCL_UINT8, 0, comms[r], &cfg, st[r]);
        t += now_us() - t0;
        if (s) {
          std::printf("bcast failed: %s\n", bcl_last_error());
          return 1;
        }
      }
      if (i % 64 == 63) {  // keep the launch queues short
        for (int r = 0; r < 2; ++r) cudaStreamSynchronize(st[r]);
      }
    }
    for (int r = 0; r < 2; ++r) cudaStreamSynchronize(st[r]);
    std::printf("bcl_bcast (C-ABI, per rank call): %.2f us host per call\n", t / (2.0 * kCalls));
  }
  cudaSetDevice(0);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(1);
    c.blockDim = dim3(512);
    c.stream = st[0];
    c.attrs = attr;
    c.numAttrs = pdl;
    double t = 0;
    for (int i = 0; i < kCalls; ++i) {
      const double t0 = now_us();
      cudaLaunchKernelEx(&c, empty_kernel, i);
      t += now_us() - t0;
      if (i % 64 == 63) cudaStreamSynchronize(st[0]);
    }
    cudaStreamSynchronize(st[0]);
    std::printf("cudaLaunchKernelEx empty kernel%s: %.2f us host per call\n", pdl ? " + PDL attribute" : "", t / kCalls);
  }
  for (int r = 0; r < 2; ++r) bcl_comm_destroy(comms[r]);
  return 0;
}
