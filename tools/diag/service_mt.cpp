// Native capacity of the persistent crypto-worker service (pc_service_*),
// without Python in the loop: T producer threads, each bound to its own
// worker (or all to worker 0), each keeping `depth` requests in flight
// (submit depth, then wait the oldest / submit a new one).  One JSON line
// per (workers, producers, depth, shared) point: pages/s and GB/s.
//
//   g++ -O2 -std=c++17 -Iinclude tools/diag/service_mt.cpp \
//       -Lpaper_2004_09252_b200 -lpagecrypt -Wl,-rpath,$PWD/paper_2004_09252_b200 -lpthread
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "pagecrypt.h"

#define CK(x)                                                               \
  do {                                                                      \
    int rc_ = (x);                                                          \
    if (rc_) {                                                              \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, pc_last_error());     \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)

static double run(pc_service *svc, int n_workers, int producers, int depth, bool shared, double secs) {
  std::atomic<bool> go{false}, stop{false};
  std::atomic<uint64_t> total{0};
  std::vector<std::thread> th;
  for (int p = 0; p < producers; ++p) {
    th.emplace_back([&, p] {
      const int w = shared ? 0 : p % n_workers;
      std::vector<uint8_t> page(4096 * static_cast<size_t>(depth), static_cast<uint8_t>(p));
      std::vector<uint64_t> tk(depth);
      while (!go.load()) std::this_thread::yield();
      uint64_t n = 0, i = 0;
      for (int d = 0; d < depth; ++d)
        CK(pc_service_submit(svc, w, 4096ull * d, 1000 + p, &page[4096 * d], &page[4096 * d], &tk[d]));
      while (!stop.load(std::memory_order_relaxed)) {
        const int d = static_cast<int>(i % depth);
        CK(pc_service_wait(svc, w, tk[d], 10000000));
        ++n;
        CK(pc_service_submit(svc, w, 4096ull * i, 1000 + p, &page[4096 * d], &page[4096 * d], &tk[d]));
        ++i;
      }
      for (int d = 0; d < depth; ++d) CK(pc_service_wait(svc, w, tk[(i + d) % depth], 10000000));
      total += n;
    });
  }
  const auto t0 = std::chrono::steady_clock::now();
  go = true;
  std::this_thread::sleep_for(std::chrono::duration<double>(secs));
  stop = true;
  const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (auto &t : th) t.join();
  return total.load() / el;
}

int main(int argc, char **argv) {
  const int n_workers = argc > 1 ? std::atoi(argv[1]) : 148;
  const double secs = argc > 2 ? std::atof(argv[2]) : 0.5;
  uint8_t entropy[32];
  for (int i = 0; i < 32; ++i) entropy[i] = static_cast<uint8_t>(rand());
  pc_key *key = nullptr;
  CK(pc_key_generate(0, entropy, &key));
  pc_service *svc = nullptr;
  CK(pc_service_start(key, n_workers, 64, 20, &svc));
  CK(pc_key_destroy(key));
  run(svc, n_workers, 1, 1, false, 0.2); // warm-up
  const int producers[] = {1, 2, 4, 8, 16, 32};
  const int depths[] = {1, 4, 16};
  for (int depth : depths)
    for (int p : producers) {
      const double r = run(svc, n_workers, p, depth, false, secs);
      printf("{\"what\": \"service native\", \"workers\": %d, \"producers\": %d, \"depth\": %d, "
             "\"shared_worker\": false, \"pages_per_s\": %.0f, \"gbs\": %.3f}\n",
             n_workers, p, depth, r, r * 4096 / 1e9);
      fflush(stdout);
    }
  for (int p : {1, 4, 16}) {
    const double r = run(svc, n_workers, p, 16, true, secs);
    printf("{\"what\": \"service native\", \"workers\": %d, \"producers\": %d, \"depth\": 16, "
           "\"shared_worker\": true, \"pages_per_s\": %.0f, \"gbs\": %.3f}\n",
           n_workers, p, r, r * 4096 / 1e9);
    fflush(stdout);
  }
  CK(pc_service_stop(svc));
  return 0;
}
