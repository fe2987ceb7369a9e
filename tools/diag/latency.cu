// Where does the small-batch (fault-path) latency go?  Native loop, no
// Python: p50/p99 of
//   * an empty kernel launch + cudaStreamSynchronize (the launch floor),
//   * the same with cudaDeviceScheduleSpin / BlockingSync not changed (default),
//   * pc_crypt_pages_host on 1..64 pinned pages (the library's zero-copy path),
//   * pc_service_crypt of one page (the persistent worker service).
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/diag/latency.cu \
//        -Lpaper_2004_09252_b200 -lpagecrypt -Xlinker -rpath,$PWD/paper_2004_09252_b200 -o tools/diag/latency
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pagecrypt.h"

#define CK(x)                                                           \
  do {                                                                  \
    int rc_ = (x);                                                      \
    if (rc_) {                                                          \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, pc_last_error()); \
      std::exit(1);                                                     \
    }                                                                   \
  } while (0)

__global__ void empty_kernel() {}

template <class F>
static void measure(const char *what, int pages, F fn, int reps = 3000) {
  for (int i = 0; i < 200; ++i) fn();
  std::vector<double> ts(reps);
  for (int i = 0; i < reps; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    fn();
    ts[i] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  }
  std::sort(ts.begin(), ts.end());
  printf("{\"what\": \"%s\", \"pages\": %d, \"p50_us\": %.2f, \"p99_us\": %.2f, \"min_us\": %.2f}\n", what, pages,
         ts[reps / 2], ts[reps * 99 / 100], ts[0]);
  fflush(stdout);
}

int main(int argc, char **argv) {
  const int svc_workers = argc > 1 ? std::atoi(argv[1]) : 8;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  measure("empty launch + stream sync", 0, [&] {
    empty_kernel<<<1, 32, 0, st>>>();
    cudaStreamSynchronize(st);
  });
  measure("empty launch 148x256 + stream sync", 0, [&] {
    empty_kernel<<<148, 256, 0, st>>>();
    cudaStreamSynchronize(st);
  });
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  measure("empty launch + event spin", 0, [&] {
    empty_kernel<<<1, 32, 0, st>>>();
    cudaEventRecord(ev, st);
    while (cudaEventQuery(ev) == cudaErrorNotReady) {
    }
  });
  uint8_t entropy[32] = {1, 2, 3};
  pc_key *key = nullptr;
  CK(pc_key_generate(0, entropy, &key));
  pc_engine *eng = nullptr;
  CK(pc_engine_create(0, 4, 8192, &eng));
  void *in = nullptr, *out = nullptr;
  CK(pc_host_alloc(64 * 4096, &in));
  CK(pc_host_alloc(64 * 4096, &out));
  for (int n : {1, 4, 16, 64})
    measure("pc_crypt_pages_host (pinned)", n, [&] {
      CK(pc_crypt_pages_host(eng, key, nullptr, nullptr, nullptr, 0x100000000ull, 1, in, out, n, 20));
    });
  std::vector<uint8_t> pin_in(4096), pin_out(4096);
  measure("pc_crypt_pages_host (pageable)", 1, [&] {
    CK(pc_crypt_pages_host(eng, key, nullptr, nullptr, nullptr, 0x100000000ull, 1, pin_in.data(), pin_out.data(), 1,
                           20));
  });
  pc_service *svc = nullptr;
  CK(pc_service_start(key, svc_workers, 64, 20, &svc));
  measure("pc_service_crypt", 1, [&] { CK(pc_service_crypt(svc, 0, 0x100000000ull, 1, in, out, -1)); });
  CK(pc_service_stop(svc));
  CK(pc_engine_destroy(eng));
  CK(pc_key_destroy(key));
  return 0;
}
