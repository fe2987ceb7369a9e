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
// Here: one 32-thread CTA per worker.  Each worker owns a ring of C slots in
// mapped pinned host memory: a 64-byte header (ready_seq written by host
// producers, done_seq written by the worker) and a 4 KiB page.  Request t of a
// worker lives in slot t % C; the host publishes it by storing ready_seq =
// t+1, the worker XORs the page in place and stores done_seq = t+1.  The key
// is loaded into registers once at start (the device copy can then be
// destroyed); the state never leaves registers (ptxas: 0 bytes stack/spill).
#pragma once
#include <cstdint>

#include "chacha.cuh"

namespace pc {

struct alignas(64) SvcSlot {
  uint64_t ready_seq; // host -> device: ticket + 1 once vaddr/pid/page are written
  uint64_t vaddr;
  uint32_t pid;
  uint32_t pad0;
  uint64_t done_seq;  // device -> host: ticket + 1 once the page holds the result
  uint64_t pad1[4];
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

template <int ROUNDS>
__global__ void __launch_bounds__(32, 1)
k_service(const uint32_t *__restrict__ key, SvcSlot *slots, uint4 *pages, uint32_t ring,
          const uint32_t *ctrl_stop, uint32_t *started) {
  __shared__ uint4 tile[256]; // one 4 KiB page
  constexpr RotMul rm{};
  const uint32_t worker = blockIdx.x, lane = threadIdx.x;
  uint32_t k[8];
  {
    const uint4 a = reinterpret_cast<const uint4 *>(key)[0];
    const uint4 b = reinterpret_cast<const uint4 *>(key)[1];
    k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
    k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence_system();
    st_volatile_u32(started + worker, 1u); // key now lives in registers
  }
  SvcSlot *myring = slots + static_cast<uint64_t>(worker) * ring;
  uint4 *mypages = pages + static_cast<uint64_t>(worker) * ring * 256;
  const uint32_t ia = 2 * lane, ib = 2 * lane + 1; // the paper's 128-byte lane unit

  for (uint64_t head = 0;; ++head) {
    SvcSlot *sl = myring + (head % ring);
    // wait for request `head` (all lanes read the same word: one request per poll)
    uint32_t backoff = 32;
    bool stop = false;
    for (;;) {
      const uint64_t r = ld_acquire_sys(&sl->ready_seq);
      if (__all_sync(0xffffffffu, r == head + 1)) break;
      if (__any_sync(0xffffffffu, ld_volatile_u32(ctrl_stop) != 0u)) {
        stop = true;
        break;
      }
      __nanosleep(backoff);
      if (backoff < 1024) backoff <<= 1;
    }
    if (stop) break;
    const uint64_t vaddr = *reinterpret_cast<volatile uint64_t *>(&sl->vaddr);
    const uint32_t pid = *reinterpret_cast<volatile uint32_t *>(&sl->pid);
    uint4 *page = mypages + (head % ring) * 256;
    // coalesced 512-byte reads of the page into the tile
#pragma unroll
    for (int j = 0; j < 8; ++j) tile[svc_swz(32 * j + lane)] = ld_volatile_v4(page + 32 * j + lane);
    // two keystream blocks per lane, interleaved for ILP
    uint32_t xa[16], xb[16];
    const uint32_t sa[4] = {static_cast<uint32_t>(vaddr), static_cast<uint32_t>(vaddr >> 32), pid, ia};
    const uint32_t sb[4] = {static_cast<uint32_t>(vaddr), static_cast<uint32_t>(vaddr >> 32), pid, ib};
    chacha_block<ROUNDS, 0>(xa, k, sa, rm);
    chacha_block<ROUNDS, 0>(xb, k, sb, rm);
    __syncwarp();
    // lane owns chunks 8*lane .. 8*lane+7 = blocks ia (first 4) and ib (last 4)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint4 v = tile[svc_swz(8 * lane + c)];
      v.x ^= xa[4 * c]; v.y ^= xa[4 * c + 1]; v.z ^= xa[4 * c + 2]; v.w ^= xa[4 * c + 3];
      tile[svc_swz(8 * lane + c)] = v;
      uint4 w = tile[svc_swz(8 * lane + 4 + c)];
      w.x ^= xb[4 * c]; w.y ^= xb[4 * c + 1]; w.z ^= xb[4 * c + 2]; w.w ^= xb[4 * c + 3];
      tile[svc_swz(8 * lane + 4 + c)] = w;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) st_volatile_v4(page + 32 * j + lane, tile[svc_swz(32 * j + lane)]);
    __threadfence_system(); // page bytes reach host memory before the flag
    __syncwarp();
    if (lane == 0) st_release_sys(&sl->done_seq, head + 1);
  }
  // registers (and with them the key) die with the kernel; scrub the tile
#pragma unroll
  for (int j = 0; j < 8; ++j) tile[32 * j + lane] = make_uint4(0, 0, 0, 0);
}

} // namespace pc
