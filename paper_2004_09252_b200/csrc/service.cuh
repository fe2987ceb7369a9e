// service.cuh -- persistent GPU crypto-worker service (the paper's design).
//
// MemShield runs "a GPU kernel [that] consists of several CUDA blocks; each
// block acts as a worker whose job is to extract pages from a queue and
// process them using 32 CUDA threads (one warp). Each CUDA thread generates
// two ChaCha20 keystream blocks (128 bytes)" and keeps the key in registers
// for the kernel's lifetime, fed through "a circular buffer implementing a
// multiple-producer, single-consumer queue" in mapped host memory
// (/root/reference/PAPER.md:615-632).  The reference emulates it with
// WorkerPool / WorkerRing / Completion (pkg/src/pagecrypt/workers.py:28-254).
//
// Here: one 32-thread CTA per worker plus one dispatcher CTA.  Each worker
// owns a ring of C slots in mapped pinned host memory: a 64-byte header
// (vaddr, pid, done_seq) and a 4 KiB page.  Request t of a worker lives in
// slot t % C.  Producers publish tickets in order per worker by advancing
// doorbell[w] (mapped host memory).  Only the dispatcher polls the doorbells
// over PCIe -- one coalesced read for all workers per poll -- and forwards
// them into device memory, where the idle workers poll cheaply (L2).  A worker
// that sees bell > head reads the slot header and the page in one PCIe round
// trip, XORs the page in place and stores done_seq = t+1.  The key is loaded
// into registers once at start (the device copy can then be destroyed); the
// cipher state never leaves registers (ptxas: 0 bytes stack/spill).
#pragma once
#include <cstdint>

#include "chacha.cuh"

namespace pc {

struct alignas(64) SvcSlot {
  uint64_t vaddr;
  uint32_t pid;
  uint32_t pad0;
  uint64_t done_seq;  // device -> host: ticket + 1 once the page holds the result
  uint64_t t_ns[4];   // %globaltimer when the worker saw the bell / had the page /
                      // had the keystream / had written the page (diagnostics)
  uint64_t pad1;
};
static_assert(sizeof(SvcSlot) == 64, "slot header is one 64-byte line");

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t *p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4 *p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_volatile_v4(uint4 *p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_volatile_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16-byte chunk q of a page -> its slot in a 128-byte-row XOR-swizzled tile
// (conflict-free for both the coalesced and the per-lane 128-byte patterns).
__device__ __forceinline__ uint32_t svc_swz(uint32_t q) { return (q & ~7u) | ((q ^ (q >> 3)) & 7u); }

// Device-side control block (device memory).
struct SvcDev {
  uint64_t bell[4096]; // forwarded doorbells, one per worker
  uint32_t stop;
};

__device__ __forceinline__ void named_bar(uint32_t count) {
  asm volatile("bar.sync 1, %0;" ::"r"(count) : "memory");
}

// Block n_workers: the dispatcher (warp 0 only).  Blocks 0..n_workers-1: the
// workers (64 threads each).
template <int ROUNDS>
__global__ void __launch_bounds__(64, 1)
k_service(const uint32_t *__restrict__ key, SvcSlot *slots, uint4 *pages, uint32_t ring, uint32_t n_workers,
          const uint64_t *host_bell, const uint32_t *host_stop, uint32_t *started, SvcDev *dev) {
  __shared__ uint4 tile[256]; // one 4 KiB page
  const uint32_t lane = threadIdx.x;
  if (blockIdx.x == n_workers) {
    if (threadIdx.x >= 32) return;
    // ---- dispatcher: host doorbells -> device memory ---------------------
    // all doorbells are read in parallel (relaxed), then one acquire fence
    // orders the page reads the workers will do after seeing the new bells
    constexpr uint32_t kMaxPerLane = 4096 / 32;
    uint32_t idle = 0;
    for (;;) {
      uint64_t b[4];
      bool moved = false;
      for (uint32_t w0 = 0; w0 < n_workers; w0 += 128) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = w0 + u * 32 + lane;
          b[u] = w < n_workers ? ld_relaxed_sys(host_bell + w) : 0;
        }
        asm volatile("fence.acq_rel.sys;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = w0 + u * 32 + lane;
          if (w < n_workers && b[u] != dev->bell[w]) {
            st_release_gpu(&dev->bell[w], b[u]);
            moved = true;
          }
        }
      }
      (void)kMaxPerLane;
      const bool stop = ld_volatile_u32(host_stop) != 0u;
      if (__any_sync(0xffffffffu, stop)) {
        if (lane == 0) atomicExch(&dev->stop, 1u);
        break;
      }
      // poll back to back while busy; back off only after ~1 ms idle
      idle = __any_sync(0xffffffffu, moved) ? 0 : idle + 1;
      if (idle > 1000) __nanosleep(2000);
    }
    return;
  }
  // ---- worker: 64 threads, thread t = block t -------------------------------
  if (threadIdx.x >= 64) return;
  constexpr RotMul rm{};
  const uint32_t worker = blockIdx.x;
  const uint32_t tid = threadIdx.x;
  uint32_t k[8];
  {
    const uint4 a = reinterpret_cast<const uint4 *>(key)[0];
    const uint4 b = reinterpret_cast<const uint4 *>(key)[1];
    k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
    k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
  }
  named_bar(64);
  if (tid == 0) {
    __threadfence_system();
    st_volatile_u32(started + worker, 1u); // key now lives in registers
  }
  SvcSlot *myring = slots + static_cast<uint64_t>(worker) * ring;
  uint4 *mypages = pages + static_cast<uint64_t>(worker) * ring * 256;
  uint64_t bell = 0;

  for (uint64_t head = 0;; ++head) {
    // wait until ticket `head` is published (device-memory poll)
    while (bell <= head) {
      bell = ld_acquire_gpu(&dev->bell[worker]);
      if (bell > head) break;
      if (*reinterpret_cast<volatile uint32_t *>(&dev->stop)) return;
      __nanosleep(32);
    }
    uint64_t t0, t1, t2, t3;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    SvcSlot *sl = myring + (head % ring);
    uint4 *page = mypages + (head % ring) * 256;
    // header and page in one PCIe round trip (published before the doorbell):
    // 64 threads x 4 coalesced 16-byte loads (1 KiB per instruction)
    uint4 d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j] = ld_volatile_v4(page + 64 * j + tid);
    const uint64_t vaddr = *reinterpret_cast<volatile uint64_t *>(&sl->vaddr);
    const uint32_t pid = *reinterpret_cast<volatile uint32_t *>(&sl->pid);
#pragma unroll
    for (int j = 0; j < 4; ++j) tile[svc_swz(64 * j + tid)] = d[j];
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1) : : "memory");
    uint32_t x[16];
    const uint32_t sd[4] = {static_cast<uint32_t>(vaddr), static_cast<uint32_t>(vaddr >> 32), pid, tid};
    chacha_block<ROUNDS, 0>(x, k, sd, rm);
    named_bar(64);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2) : : "memory");
    // thread owns chunks 4*tid .. 4*tid+3 (its 64-byte block)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint4 v = tile[svc_swz(4 * tid + c)];
      v.x ^= x[4 * c]; v.y ^= x[4 * c + 1]; v.z ^= x[4 * c + 2]; v.w ^= x[4 * c + 3];
      tile[svc_swz(4 * tid + c)] = v;
    }
    named_bar(64);
#pragma unroll
    for (int j = 0; j < 4; ++j) st_volatile_v4(page + 64 * j + tid, tile[svc_swz(64 * j + tid)]);
    __threadfence_system(); // each warp's page stores reach host memory ...
    named_bar(64);          // ... before thread 0 raises the flag
    if (tid == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3) : : "memory");
      sl->t_ns[0] = t0; sl->t_ns[1] = t1; sl->t_ns[2] = t2; sl->t_ns[3] = t3;
      st_release_sys(&sl->done_seq, head + 1);
    }
  }
}

} // namespace pc
