// Launch + completion latency of a small kernel, four ways: cudaStreamSynchronize;
// spinning on a mapped host flag the kernel's last CTA writes (st.release.sys);
// a 1-thread flag kernel queued behind it; cuStreamWriteValue32 queued behind it.
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__global__ void k_work(unsigned *ctr, volatile uint32_t *flag, uint32_t val) {
  __syncthreads();
  if (flag && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr, 1) == gridDim.x - 1) {
      *ctr = 0;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(val) : "memory");
    }
  }
}
__global__ void k_flag(volatile uint32_t *flag, uint32_t val) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(val) : "memory");
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  uint32_t *h, *d;
  cudaHostAlloc(&h, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&d, h, 0);
  unsigned *ctr;
  cudaMalloc(&ctr, 4);
  cudaMemset(ctr, 0, 4);
  *h = 0;
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q);
  auto write_value = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fn);
  const char *names[] = {"stream sync", "kernel flag", "flag kernel", "write value"};
  uint32_t val = 0;
  for (int w = 0; w < 20000; ++w) { k_work<<<16, 64, 0, st>>>(ctr, nullptr, 0); cudaStreamSynchronize(st); } // clocks up
  for (int pass = 0; pass < 2; ++pass)
  for (int grid : {1, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      if (mode == 3 && !write_value) continue;
      std::vector<double> ts;
      for (int i = 0; i < 3000; ++i) {
        ++val;
        auto t0 = std::chrono::steady_clock::now();
        k_work<<<grid, 64, 0, st>>>(ctr, mode == 1 ? d : nullptr, val);
        if (mode == 2) k_flag<<<1, 1, 0, st>>>(d, val);
        if (mode == 3) write_value(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(d), val, 0);
        if (mode == 0) cudaStreamSynchronize(st);
        else while (*reinterpret_cast<volatile uint32_t *>(h) != val) {}
        auto t1 = std::chrono::steady_clock::now();
        if (i >= 300) ts.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      }
      cudaStreamSynchronize(st);
      std::sort(ts.begin(), ts.end());
      printf("grid %2d %-12s p50 %.2f us  p99 %.2f us\n", grid, names[mode], ts[ts.size() / 2], ts[ts.size() * 99 / 100]);
    }
  }
  return 0;
}
