// Host-memory read round trip per SM: one CTA per SM, run one at a time (a
// device-memory turn counter), thread 0 times 256 dependent ld.volatile of a
// mapped pinned word with %globaltimer.  Prints "smid rtt_ns" per CTA.
// Question: do the two B200 dies see different PCIe latency (the service's
// workers pay 3 host round trips per request)?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void rtt(const volatile uint32_t *host, unsigned *turn, uint32_t *out_sm, uint64_t *out_ns, int reps) {
  if (threadIdx.x) return;
  while (atomicAdd(turn, 0) != blockIdx.x) __nanosleep(100);
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) acc += host[acc & 0];  // warm
  uint64_t t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < reps; ++i) acc += host[acc & 0]; // each load depends on the last
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out_sm[blockIdx.x] = smid + (acc & 0) ;
  out_ns[blockIdx.x] = (t1 - t0) / reps;
  __threadfence();
  atomicAdd(turn, 1);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *h, *d;
  cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
  h[0] = 0;
  cudaHostGetDevicePointer(&d, h, 0);
  unsigned *turn; uint32_t *sm; uint64_t *ns;
  cudaMalloc(&turn, 4); cudaMemset(turn, 0, 4);
  cudaMallocManaged(&sm, nsm * 4); cudaMallocManaged(&ns, nsm * 8);
  rtt<<<nsm, 32>>>(d, turn, sm, ns, 256);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<std::pair<uint32_t, uint64_t>> v;
  for (int i = 0; i < nsm; ++i) v.push_back({sm[i], ns[i]});
  std::sort(v.begin(), v.end());
  for (auto &p : v) printf("%u %llu\n", p.first, (unsigned long long)p.second);
  return 0;
}
