// Host cost of the pointer queries on the small-batch path: p50 of
// cudaPointerGetAttributes on pinned (cudaHostAlloc mapped), pageable and
// device pointers, next to pc_crypt_pages_host on one pinned page.
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/diag/ptrattr_probe.cu \
//        -Lpaper_2004_09252_b200 -lpagecrypt -Xlinker -rpath,$PWD/paper_2004_09252_b200 -o tools/diag/ptrattr_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pagecrypt.h"

template <class F>
static double p50_ns(F f, int reps) {
  std::vector<double> t(reps);
  for (int i = 0; i < reps; ++i) {
    auto a = std::chrono::steady_clock::now();
    f();
    t[i] = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - a).count();
  }
  std::sort(t.begin(), t.end());
  return t[reps / 2];
}

int main() {
  cudaSetDevice(0);
  void *pinned = nullptr, *dev = nullptr, *pinned_out = nullptr;
  cudaHostAlloc(&pinned, 4096, cudaHostAllocMapped);
  cudaHostAlloc(&pinned_out, 4096, cudaHostAllocMapped);
  cudaMalloc(&dev, 4096);
  void *pageable = std::malloc(4096);
  cudaPointerAttributes a;
  const char *names[3] = {"pinned", "pageable", "device"};
  void *ptrs[3] = {pinned, pageable, dev};
  for (int k = 0; k < 3; ++k) {
    double ns = p50_ns([&] { cudaPointerGetAttributes(&a, ptrs[k]); cudaGetLastError(); }, 20000);
    std::printf("cudaPointerGetAttributes(%s): p50 %.0f ns\n", names[k], ns);
  }
  pc_engine *e = nullptr;
  pc_key *key = nullptr;
  uint8_t ent[32];
  for (int i = 0; i < 32; ++i) ent[i] = static_cast<uint8_t>(i * 7 + 1);
  if (pc_engine_create(0, 4, 0, &e) != 0 || pc_key_generate(0, ent, &key) != 0) {
    std::printf("engine/key: %s\n", pc_last_error());
    return 1;
  }
  for (int i = 0; i < 3000; ++i) pc_crypt_pages_host(e, key, nullptr, nullptr, nullptr, 1ull << 32, 1, pinned, pinned_out, 1, 20);
  double us = p50_ns([&] { pc_crypt_pages_host(e, key, nullptr, nullptr, nullptr, 1ull << 32, 1, pinned, pinned_out, 1, 20); },
                     5000) / 1e3;
  std::printf("pc_crypt_pages_host 1 pinned page: p50 %.2f us\n", us);
  pc_key_destroy(key);
  pc_engine_destroy(e);
  return 0;
}
