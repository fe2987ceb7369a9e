// Which CUDA runtime calls block while a persistent kernel runs on a
// non-blocking stream?  Each probe runs on its own thread with a deadline.
#include <cuda_runtime.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <functional>
#include <string>
#include <unistd.h>
#include <thread>

__global__ void spin(volatile unsigned *stop) {
  while (*stop == 0) __nanosleep(1000);
}
__global__ void tiny(int *p) { p[threadIdx.x] = threadIdx.x; }

static bool probe(const char *name, std::function<void()> fn, int ms = 3000) {
  std::atomic<bool> done{false};
  std::thread t([&] { fn(); done = true; });
  auto t0 = std::chrono::steady_clock::now();
  while (!done && std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(ms))
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  printf("%-40s %s\n", name, done ? "ok" : "BLOCKS");
  fflush(stdout);
  if (!done) t.detach(); else t.join();
  return done;
}

int main(int argc, char **argv) {
  const char *which = argc > 1 ? argv[1] : "";
  unsigned *h_stop;
  cudaHostAlloc(&h_stop, 64, cudaHostAllocMapped);
  *h_stop = 0;
  unsigned *d_stop;
  cudaHostGetDevicePointer((void **)&d_stop, h_stop, 0);
  int *d = nullptr;
  cudaMalloc(&d, 1 << 20);
  void *pre_h = nullptr;
  cudaHostAlloc(&pre_h, 1 << 20, 0);
  int *pre_d = nullptr;
  cudaMalloc(&pre_d, 4096);
  void *pre_reg = malloc(1 << 20);
  cudaHostRegister(pre_reg, 1 << 20, 0);
  cudaStream_t pre_s;
  cudaStreamCreateWithFlags(&pre_s, cudaStreamNonBlocking);
  cudaEvent_t pre_e;
  cudaEventCreateWithFlags(&pre_e, cudaEventDisableTiming);
  tiny<<<1, 32>>>(d); // load tiny before the spin kernel starts
  cudaDeviceSynchronize();
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  spin<<<2, 32, 0, s>>>(d_stop);
  std::this_thread::sleep_for(std::chrono::milliseconds(100));
  std::string w(which);
  bool ok = true;
  if (w == "malloc") ok = probe("cudaMalloc", [&] { int *q; cudaMalloc(&q, 1 << 20); });
  else if (w == "free") ok = probe("cudaFree", [&] { cudaFree(pre_d); });
  else if (w == "hostalloc") ok = probe("cudaHostAlloc", [&] { void *h; cudaHostAlloc(&h, 1 << 20, 0); });
  else if (w == "freehost") ok = probe("cudaFreeHost", [&] { cudaFreeHost(pre_h); });
  else if (w == "hostregister") ok = probe("cudaHostRegister", [&] { void *m = malloc(1 << 20); cudaHostRegister(m, 1 << 20, 0); });
  else if (w == "hostunregister") ok = probe("cudaHostUnregister", [&] { cudaHostUnregister(pre_reg); });
  else if (w == "streamcreate") ok = probe("cudaStreamCreateWithFlags(NonBlocking)", [&] { cudaStream_t x; cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking); });
  else if (w == "streamdestroy") ok = probe("cudaStreamDestroy", [&] { cudaStreamDestroy(pre_s); });
  else if (w == "eventcreate") ok = probe("cudaEventCreate", [&] { cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); });
  else if (w == "eventdestroy") ok = probe("cudaEventDestroy", [&] { cudaEventDestroy(pre_e); });
  else if (w == "mallocasync") ok = probe("cudaMallocAsync+FreeAsync", [&] { void *a; cudaMallocAsync(&a, 1 << 20, pre_s); cudaFreeAsync(a, pre_s); cudaStreamSynchronize(pre_s); });
  else if (w == "legacykernel") ok = probe("loaded kernel on legacy stream + sync(0)", [&] { tiny<<<1, 32>>>(d); cudaStreamSynchronize(0); });
  else if (w == "nbkernel") ok = probe("loaded kernel on nonblocking + sync", [&] { tiny<<<1, 32, 0, pre_s>>>(d); cudaStreamSynchronize(pre_s); });
  else if (w == "memcpyasync") ok = probe("cudaMemcpyAsync pinned D2H + sync", [&] { cudaMemcpyAsync(pre_h, d, 4096, cudaMemcpyDeviceToHost, pre_s); cudaStreamSynchronize(pre_s); });
  else if (w == "memcpypageable") ok = probe("cudaMemcpyAsync pageable H2D + sync", [&] { static char b[4096]; cudaMemcpyAsync(d, b, 4096, cudaMemcpyHostToDevice, pre_s); cudaStreamSynchronize(pre_s); });
  else if (w == "memset") ok = probe("cudaMemsetAsync + sync", [&] { cudaMemsetAsync(d, 0, 4096, pre_s); cudaStreamSynchronize(pre_s); });
  else if (w == "pointerattr") ok = probe("cudaPointerGetAttributes", [&] { cudaPointerAttributes a; cudaPointerGetAttributes(&a, pre_h); });
  else if (w == "funcattr") ok = probe("cudaFuncGetAttributes(spin)", [&] { cudaFuncAttributes a; cudaFuncGetAttributes(&a, spin); });
  else if (w == "occupancy") ok = probe("cudaOccupancyMaxActiveBlocks", [&] { int o; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tiny, 32, 0); });
  if (!ok) _exit(3);
  *h_stop = 1;
  cudaStreamSynchronize(s);
  return 0;
}
