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
// Here: one 64-thread CTA per worker (thread t makes block t of the page,
// so a page is one pass) plus one dispatcher warp.  Each worker
// owns a ring of C slots in mapped pinned host memory: a 64-byte header
// (vaddr, pid, done_seq) and a 4 KiB page.  Request t of a worker lives in
// slot t % C.  Producers publish tickets in order per worker by storing
// doorbell[w] = {count, pid, vaddr of the newest ticket} with one 16-byte
// store (mapped host memory).  Only the dispatcher polls the doorbells over
// PCIe -- one coalesced read for all workers per poll -- and forwards them
// into device memory, where the idle workers poll cheaply (L2).  A worker
// whose next ticket is the newest one gets its header with the bell and
// computes the keystream while the page bytes cross PCIe; otherwise it reads
// the slot header.  It XORs the page in place and stores done_seq = t+1.  The key is loaded
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
// LDG.128.STRONG.SYS + CCTL.IVALL: an acquire without the MEMBAR.SYS of a
// fence (which waits for this SM's outstanding posted writes to host memory:
// 1.9 us per request measured, profiles/r02_service_direct.txt)
__device__ __forceinline__ uint4 ld_acquire_sys_v4(const uint4 *p) {
  uint4 r;
  asm volatile("ld.acquire.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
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

// A page-store operation riding a service ticket: the pager's single fault
// (refault out of the HBM slab and the eviction its window admission forces,
// /root/reference/pkg/src/pagecrypt/orchestrator.py:175-240) served by a
// resident worker instead of a kernel launch (pc_store_service).  The
// ticket's vaddr carries the op flags in its low 12 bits (vaddrs are page
// aligned); the rest lives in the slot's SvcOp line (mapped host memory).
struct alignas(64) SvcOp {
  uint64_t slab;        // device address of the store's slab (4 KiB slots)
  uint64_t evict_vaddr; // kOpPut: vaddr the ring page's plaintext is evicted to
  uint32_t get_slot;    // kOpGet: slab slot decrypted into the ring page, then zeroed
  uint32_t put_slot;    // kOpPut: slab slot the ring page is encrypted into
  uint32_t pad[10];
};
static_assert(sizeof(SvcOp) == 64, "one 64-byte line per ring slot");
constexpr uint32_t kOpStore = 1, kOpGet = 2, kOpPut = 4;
// The newest store ticket's slots also ride in the doorbell's line (the
// 16 bytes after the bell: evict_vaddr | tag, get_slot, put_slot), so a
// worker of a store's own service knows every address at the poll and starts
// the HBM slab read and both keystreams while the page crosses PCIe.  tag =
// ticket % 4095 + 1 (never 0: a crypt ticket zeroes the chunk); a chunk whose
// tag is not the ticket's is stale and the worker reads the SvcOp line.
__host__ __device__ constexpr uint32_t op_tag(uint64_t ticket) { return static_cast<uint32_t>(ticket % 4095) + 1; }

// Device-side control block (device memory).
// Host doorbell of one worker (mapped pinned memory, 16 bytes, written by
// the producer that publishes ticket t: vaddr and pid of t first, then
// count = t + 1), so one 16-byte read gives the dispatcher the count AND the
// header of the latest ticket.
struct alignas(16) SvcBell {
  uint32_t count; // tickets published, mod 2^32
  uint32_t pid;   // of the latest published ticket
  uint64_t vaddr;
};
static_assert(sizeof(SvcBell) == 16, "one 16-byte read per doorbell");
// Doorbells sit kBellStride x 16 bytes apart in host memory: one 64-byte
// line each, so a producer's store never shares a line other workers poll
// (16 workers: 1-page p50 9.2 -> 8.4 us, p99 12.0 -> 9.3, profiles/r02_ab_bell.txt).
#ifndef PC_BELL_STRIDE
#define PC_BELL_STRIDE 4
#endif
constexpr uint32_t kBellStride = PC_BELL_STRIDE;

// Device-memory mirror of the doorbells.  bell[w] is the 64-bit count of
// published tickets.  When the dispatcher forwards a new count it also files
// the header of the newest ticket T under hdr[w * ring + T % ring] =
// {vaddr_lo, vaddr_hi, pid, tag = T} BEFORE releasing the count, so the
// entry for a ticket is never rewritten while that ticket is pending (the
// ring's back-pressure), and a worker that finds tag == its ticket uses it;
// any other tag means the header was never forwarded -> read the slot.
struct SvcDev {
  uint64_t bell[4096];
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
          const SvcBell *host_bell, const uint32_t *host_stop, uint32_t *started, SvcDev *dev,
          uint4 *hdr, uint32_t direct, const SvcOp *ops, uint4 *store_slab) {
  __shared__ uint4 tile[256]; // one 4 KiB page
  __shared__ uint4 bell_s;    // direct mode: the doorbell thread 0 saw (count, pid, vaddr)
  __shared__ uint4 op_s;      // ... and the store-op chunk of its line
  const uint32_t lane = threadIdx.x;
  if (blockIdx.x == n_workers) {
    if (threadIdx.x >= 32) return;
    // ---- dispatcher: host doorbells -> device memory ---------------------
    // all doorbells (and the stop flag) are read in parallel: one PCIe round
    // trip per poll for up to 256 workers.  The low 32 bits of every
    // forwarded count are cached in this CTA's (otherwise unused) shared
    // tile, so a poll does not read L2; the acquire fence orders the page
    // reads the workers will do after a bell moved.
    uint32_t *seen = reinterpret_cast<uint32_t *>(tile); // 1024 workers
    const bool cache = n_workers <= 1024;
    if (cache)
      for (uint32_t w = lane; w < n_workers; w += 32) seen[w] = 0;
    __syncwarp();
    uint32_t idle = 0;
    for (;;) {
      uint4 b[8];
      bool moved = false;
      bool stop = false;
      for (uint32_t w0 = 0; w0 < n_workers; w0 += 256) {
        bool changed = false;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t w = w0 + u * 32 + lane;
          b[u] = w < n_workers ? ld_volatile_v4(reinterpret_cast<const uint4 *>(host_bell + w * kBellStride))
                               : make_uint4(0, 0, 0, 0);
        }
        if (w0 == 0) stop = ld_volatile_u32(host_stop) != 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t w = w0 + u * 32 + lane;
          if (w < n_workers)
            changed |= b[u].x != (cache ? seen[w] : static_cast<uint32_t>(dev->bell[w]));
        }
        // the fence runs on every poll: measured, it also paces the polls
        // (8 workers: 8.6 us per request vs 10.1 without it; 148 workers:
        // 9.9 vs 10.6 us; profiles/r01_service_dispatch_ab.txt)
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        if (!__any_sync(0xffffffffu, changed)) continue;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t w = w0 + u * 32 + lane;
          if (w >= n_workers) continue;
          const uint32_t low = cache ? seen[w] : static_cast<uint32_t>(dev->bell[w]);
          const uint32_t delta = b[u].x - low;
          if (delta != 0) {
            const uint64_t cnt = dev->bell[w] + delta;
            const uint64_t newest = cnt - 1;
            st_volatile_v4(&hdr[static_cast<uint64_t>(w) * ring + newest % ring],
                           make_uint4(b[u].z, b[u].w, b[u].y, static_cast<uint32_t>(newest)));
            __threadfence();                 // header filed before the count
            st_release_gpu(&dev->bell[w], cnt);
            if (cache) seen[w] = b[u].x;
            moved = true;
          }
        }
      }
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
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    st_volatile_u32(started + worker, smid + 1); // key now lives in registers; nonzero = started
  }
  SvcSlot *myring = slots + static_cast<uint64_t>(worker) * ring;
  uint4 *mypages = pages + static_cast<uint64_t>(worker) * ring * 256;
  uint4 seen_bell = make_uint4(0, 0, 0, 0); // direct mode: last doorbell read (count, pid, vaddr)
  uint4 seen_op = make_uint4(0, 0, 0, 0);   // direct mode: the op chunk read with it
  for (uint64_t head = 0;; ++head) {
    uint4 hd;
    if (direct) {
      // direct mode: the worker polls its own doorbell in host memory (one
      // PCIe read per poll, no dispatcher hop); the newest ticket's header
      // rides in the doorbell
      if (seen_bell.x == static_cast<uint32_t>(head)) { // nothing published beyond head yet
        if (tid == 0) {
          uint4 b, o = make_uint4(0, 0, 0, 0);
          for (uint32_t polls = 1;; ++polls) {
            // the op chunk is read beside the doorbell (not ordered after it:
            // its tag says whether it belongs to the newest ticket)
            // (a store's own service only: other services poll the doorbell alone --
            // a second load per poll took 16 workers from 8.0 to 20.6 us per request)
            if (store_slab) o = ld_volatile_v4(reinterpret_cast<const uint4 *>(host_bell + worker * kBellStride + 1));
            // acquire: the page reads below are ordered after the doorbell
            b = ld_acquire_sys_v4(reinterpret_cast<const uint4 *>(host_bell + worker * kBellStride));
            if (b.x != static_cast<uint32_t>(head)) break;
            if ((polls & 255) == 0 && ld_volatile_u32(host_stop) != 0u) {
              b.x = static_cast<uint32_t>(head); // stop marker: count unchanged
              b.y = 0xffffffffu; b.z = b.w = 0xffffffffu;
              break;
            }
          }
          bell_s = b;
          op_s = o;
        }
        named_bar(64);
        seen_bell = bell_s;
        seen_op = op_s;
        named_bar(64); // bell_s may be rewritten by the next request
        if (seen_bell.x == static_cast<uint32_t>(head)) return; // stop
      }
      const uint32_t newest = seen_bell.x - 1;
      hd = make_uint4(seen_bell.z, seen_bell.w, seen_bell.y, newest);
    } else {
      // wait until ticket `head` is published (device-memory poll)
      for (;;) {
        const uint64_t bell = ld_acquire_gpu(&dev->bell[worker]);
        if (bell > head) break;
        if (*reinterpret_cast<volatile uint32_t *>(&dev->stop)) return;
        __nanosleep(32);
      }
    }
    uint64_t t0, t1, t2, t3;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    SvcSlot *sl = myring + (head % ring);
    uint4 *page = mypages + (head % ring) * 256;
    // page loads go out first; when `head` is the latest published ticket its
    // header came with the bell, so the keystream is computed while the page
    // bytes cross PCIe; otherwise the header comes from the slot
    uint4 d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j] = ld_volatile_v4(page + 64 * j + tid);
    uint64_t vaddr;
    uint32_t pid;
    if (!direct) hd = ld_volatile_v4(&hdr[static_cast<uint64_t>(worker) * ring + head % ring]);
    if (hd.w == static_cast<uint32_t>(head)) { // header forwarded with the bell
      vaddr = static_cast<uint64_t>(hd.x) | (static_cast<uint64_t>(hd.y) << 32);
      pid = hd.z;
    } else {
      vaddr = *reinterpret_cast<volatile uint64_t *>(&sl->vaddr);
      pid = *reinterpret_cast<volatile uint32_t *>(&sl->pid);
    }
    const uint32_t op = static_cast<uint32_t>(vaddr) & 4095u;
    vaddr &= ~uint64_t(4095);
    uint32_t x[16];
    if (op & kOpStore) {
      // ---- store op: refault (slab -> ring page) and/or evict (ring page -> slab)
      uint4 h0, h1; // {slab lo, slab hi, evict lo, evict hi}, {get_slot, put_slot, -, -}
      const bool in_bell = store_slab && direct && hd.w == static_cast<uint32_t>(head) &&
                           (seen_op.x & 4095u) == op_tag(head);
      if (in_bell) { // every address came with the doorbell: no op-line round trip
        const uint64_t sp = reinterpret_cast<uint64_t>(store_slab);
        h0 = make_uint4(static_cast<uint32_t>(sp), static_cast<uint32_t>(sp >> 32), seen_op.x & ~4095u, seen_op.y);
        h1 = make_uint4(seen_op.z, seen_op.w, 0, 0);
      } else {
        const uint4 *oh = reinterpret_cast<const uint4 *>(ops + static_cast<uint64_t>(worker) * ring + head % ring);
        h0 = ld_volatile_v4(oh); // one PCIe read per warp
        h1 = ld_volatile_v4(oh + 1);
      }
      uint4 *slab = reinterpret_cast<uint4 *>(static_cast<uint64_t>(h0.x) | (static_cast<uint64_t>(h0.y) << 32));
      uint4 *gblk = slab + static_cast<uint64_t>(h1.x) * 256 + 4 * tid; // this thread's 64-byte block
      uint4 *pblk = slab + static_cast<uint64_t>(h1.y) * 256 + 4 * tid;
      uint4 c[4];
      if (in_bell && (op & kOpGet)) { // the HBM slab read goes out before the keystream, too
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = gblk[j];
      }
      if (op & kOpGet) { // the refault keystream is computed while the loads are in flight
        const uint32_t sd[4] = {static_cast<uint32_t>(vaddr), static_cast<uint32_t>(vaddr >> 32), pid, tid};
        chacha_block<ROUNDS, 0>(x, k, sd, rm);
      }
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1) : : "memory");
      if (!in_bell && (op & kOpGet)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = gblk[j];
      }
      if (op & kOpPut) {
        uint32_t y[16];
        const uint64_t ev = static_cast<uint64_t>(h0.z) | (static_cast<uint64_t>(h0.w) << 32);
        const uint32_t se[4] = {static_cast<uint32_t>(ev), static_cast<uint32_t>(ev >> 32), pid, tid};
        chacha_block<ROUNDS, 0>(y, k, se, rm);
#pragma unroll
        for (int j = 0; j < 4; ++j) tile[svc_swz(64 * j + tid)] = d[j];
        named_bar(64);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 v = tile[svc_swz(4 * tid + q)];
          v.x ^= y[4 * q]; v.y ^= y[4 * q + 1]; v.z ^= y[4 * q + 2]; v.w ^= y[4 * q + 3];
          pblk[q] = v;
        }
        named_bar(64); // tile free again
      }
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2) : : "memory");
      if (op & kOpGet) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 v = c[q];
          v.x ^= x[4 * q]; v.y ^= x[4 * q + 1]; v.z ^= x[4 * q + 2]; v.w ^= x[4 * q + 3];
          tile[svc_swz(4 * tid + q)] = v;
          if (!(op & kOpPut) || h1.x != h1.y) gblk[q] = make_uint4(0, 0, 0, 0); // refaulted slot wiped
        }
        named_bar(64);
#pragma unroll
        for (int j = 0; j < 4; ++j) st_volatile_v4(page + 64 * j + tid, tile[svc_swz(64 * j + tid)]);
      }
      named_bar(64); // every thread's stores before thread 0's release
      if (tid == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3) : : "memory");
        sl->t_ns[0] = t0; sl->t_ns[1] = t1; sl->t_ns[2] = t2; sl->t_ns[3] = t3;
        st_release_sys(&sl->done_seq, head + 1);
      }
      continue;
    }
    const uint32_t sd[4] = {static_cast<uint32_t>(vaddr), static_cast<uint32_t>(vaddr >> 32), pid, tid};
    chacha_block<ROUNDS, 0>(x, k, sd, rm);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1) : : "memory");
#pragma unroll
    for (int j = 0; j < 4; ++j) tile[svc_swz(64 * j + tid)] = d[j];
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
    // the CTA barrier orders every thread's page stores before thread 0's
    // system-scope release of done_seq (release is cumulative over what the
    // barrier made visible to thread 0), so one fence per page, not 64
    named_bar(64);
    if (tid == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3) : : "memory");
      sl->t_ns[0] = t0; sl->t_ns[1] = t1; sl->t_ns[2] = t2; sl->t_ns[3] = t3;
      st_release_sys(&sl->done_seq, head + 1);
    }
  }
}

} // namespace pc
