// PCIe request/response floor for the fault path (host thread <-> resident
// GPU thread block over mapped pinned memory), to bound what the persistent
// worker service can reach.  p50/p99 in microseconds of:
//   flag      host writes a ticket, the GPU polls it (1 thread) and writes an
//             ack to host memory; host spins on the ack            (1 RTT)
//   flag+page as flag, then the block reads the 4 KiB page from host
//             memory and writes it back before the ack             (2 RTT + write)
//   ll-page   the page is sent in LL form (every 8-byte word = 4 data bytes +
//             the ticket), the block polls the whole 8 KiB until all flags
//             carry the ticket, XORs, writes the 4 KiB back, acks  (1 RTT + write)
//   ll-first  as ll-page but only lane 0 polls the first LL line; the rest of
//             the page is read once the first line is valid       (2 RTT, L1-free)
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/diag/pingpong.cu -o tools/diag/pingpong
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CU(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                 \
      return 1;                                                                \
    }                                                                          \
  } while (0)

struct alignas(64) Ctl {
  volatile uint64_t ticket; // host -> GPU
  uint64_t pad[7];
  volatile uint64_t ack;    // GPU -> host
  uint64_t pad2[7];
  volatile uint32_t stop;
};

__device__ __forceinline__ uint64_t ld_vol64(const volatile uint64_t *p) { return *p; }
__device__ __forceinline__ uint2 ld_vol_v2(const void *p) {
  uint2 r;
  asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ uint4 ld_vol_v4(const void *p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p) : "memory");
  return r;
}

template <int MODE>
__global__ void server(Ctl *c, uint4 *page, uint2 *ll, uint4 *out) {
  __shared__ uint64_t want_s;
  const uint32_t tid = threadIdx.x; // 256 threads
  for (uint64_t t = 1;; ++t) {
    if (MODE == 0 || MODE == 1 || MODE == 3) {
      if (tid == 0) {
        if (MODE == 3) {
          // poll the first LL word of the page
          for (;;) {
            uint2 w = ld_vol_v2(ll);
            if (w.y == static_cast<uint32_t>(t)) break;
            if (c->stop) { want_s = 0; break; }
          }
        } else {
          for (;;) {
            if (ld_vol64(&c->ticket) == t) break;
            if (c->stop) { want_s = 0; break; }
          }
        }
        if (!c->stop) want_s = t;
      }
      __syncthreads();
      if (want_s == 0) return;
    }
    if (MODE == 1) {
      uint4 v = ld_vol_v4(page + tid);
      v.x ^= 0x5a5a5a5au;
      out[tid] = v;
      __syncthreads();
    } else if (MODE == 2 || MODE == 3) {
      // 4 KiB in LL form = 1024 uint2 words, 4 per thread
      uint2 w[4];
      for (;;) {
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          w[k] = ld_vol_v2(ll + tid + 256 * k);
          ok &= w[k].y == static_cast<uint32_t>(t);
        }
        if (__syncthreads_and(ok)) break;
        if (__syncthreads_or(c->stop != 0)) return;
      }
      uint4 v = make_uint4(w[0].x ^ 0x5a5a5a5au, w[1].x, w[2].x, w[3].x);
      out[tid] = v;
      __syncthreads();
    }
    if (tid == 0) {
      __threadfence_system();
      c->ack = t;
    }
  }
}

int main(int argc, char **argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 20000;
  Ctl *c = nullptr;
  uint4 *page = nullptr, *out = nullptr;
  uint2 *ll = nullptr;
  CU(cudaHostAlloc(&c, sizeof(Ctl), cudaHostAllocMapped));
  CU(cudaHostAlloc(&page, 4096, cudaHostAllocMapped));
  CU(cudaHostAlloc(&out, 4096, cudaHostAllocMapped));
  CU(cudaHostAlloc(&ll, 8192, cudaHostAllocMapped));
  std::vector<uint8_t> src(4096, 7), dst(4096);
  const char *names[] = {"flag", "flag+page", "ll-page", "ll-first"};
  for (int mode = 0; mode < 4; ++mode) {
    memset(c, 0, sizeof(Ctl));
    memset(ll, 0, 8192);
    cudaStream_t st;
    CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    switch (mode) {
      case 0: server<0><<<1, 256, 0, st>>>(c, page, ll, out); break;
      case 1: server<1><<<1, 256, 0, st>>>(c, page, ll, out); break;
      case 2: server<2><<<1, 256, 0, st>>>(c, page, ll, out); break;
      default: server<3><<<1, 256, 0, st>>>(c, page, ll, out); break;
    }
    CU(cudaGetLastError());
    std::vector<double> us;
    for (int i = 1; i <= reps; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      if (mode == 2 || mode == 3) {
        // pack the page: word j = (4 data bytes, ticket)
        const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src.data());
        uint64_t *l64 = reinterpret_cast<uint64_t *>(ll);
        for (int j = 1023; j >= 0; --j) // first word last: ll-first sees a complete page
          l64[j] = static_cast<uint64_t>(s32[j]) | (static_cast<uint64_t>(static_cast<uint32_t>(i)) << 32);
      } else {
        memcpy(page, src.data(), 4096);
        std::atomic_thread_fence(std::memory_order_release);
        c->ticket = static_cast<uint64_t>(i);
      }
      while (c->ack != static_cast<uint64_t>(i)) {
      }
      memcpy(dst.data(), out, 4096);
      const auto t1 = std::chrono::steady_clock::now();
      if (i > 100) us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    c->stop = 1;
    // release pollers waiting on LL words too
    CU(cudaStreamSynchronize(st));
    CU(cudaStreamDestroy(st));
    std::sort(us.begin(), us.end());
    printf("{\"what\": \"%s\", \"p50_us\": %.2f, \"p99_us\": %.2f, \"min_us\": %.2f}\n", names[mode],
           us[us.size() / 2], us[us.size() * 99 / 100], us[0]);
    fflush(stdout);
  }
  return 0;
}
