// kernels.cuh -- sm_100a kernels of the page-cipher engine.
//
// Data layout in HBM: a batch is n pages of 4096 bytes, page-major and
// contiguous (uint8[n][4096]); page p's descriptors are vaddrs[p] (u64) and
// pids[p] (u32) or the contiguous/scalar forms (PageDesc).  Block b of page p
// is bytes [64b, 64b+64) of the page (pkg/src/pagecrypt/cipher.py:197-217).
#pragma once
#include <cstdint>

#include "chacha.cuh"
#include "tma.cuh"

namespace pc {

struct PageDesc {
  const uint64_t *vaddrs; // device (or mapped host) array, or nullptr
  const uint32_t *pids;   // device (or mapped host) array, or nullptr
  uint64_t vaddr0;        // used when vaddrs == nullptr: vaddr0 + 4096*p
  uint32_t pid0;          // used when pids == nullptr
};

__device__ __forceinline__ uint4 ld_nc(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// Plain coherent load: used when the input may alias the output (in place).
__device__ __forceinline__ uint4 ld_v4(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(uint4 *p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// 32 bytes with one 256-bit store (STG.E.ENL2.256, new on sm_100): v5 writes
// a thread's 64-byte block with two of them at ChaCha8/12 -- half the store
// instructions on the MIO queue the page stream shares with its cp.async
// copies and shared-memory reads (R=12 with pid + vaddr arrays 2620 -> 2675
// GB/s; contiguous unchanged; profiles/r02_ab_st256.txt).  ChaCha20 keeps
// four STG.128.
__device__ __forceinline__ void st_v8(uint4 *p, uint4 a, uint4 b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w),
               "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

__device__ __forceinline__ void load_key(const uint32_t *__restrict__ key, uint32_t (&k)[8]) {
  const uint4 a = __ldg(reinterpret_cast<const uint4 *>(key));
  const uint4 b = __ldg(reinterpret_cast<const uint4 *>(key) + 1);
  k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
  k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
}

// A page's descriptor (vaddr, pid): loaded one page ahead by the persistent
// kernels so the global-load latency hides under the current page's rounds.
__device__ __forceinline__ void desc_fetch(const PageDesc &d, uint64_t page, uint64_t &va, uint32_t &pid) {
  va = d.vaddrs ? __ldg(d.vaddrs + page) : d.vaddr0 + (page << 12);
  pid = d.pids ? __ldg(d.pids + page) : d.pid0;
}

__device__ __forceinline__ void page_seed(const PageDesc &d, uint64_t page, uint32_t (&s)[4]) {
  const uint64_t va = d.vaddrs ? __ldg(d.vaddrs + page) : d.vaddr0 + (page << 12);
  s[0] = static_cast<uint32_t>(va);        // word 12 = vaddr lo
  s[1] = static_cast<uint32_t>(va >> 32);  // word 13 = vaddr hi
  s[2] = d.pids ? __ldg(d.pids + page) : d.pid0; // word 14 = pid
}

// ---------------------------------------------------------------------------
// v1: one thread = one 64-byte block.  The thread XORs its keystream into the
// page bytes with four 16-byte loads/stores; a warp covers 2 KiB (half a page)
// contiguously, sectors shared between the 4 loads of a thread hit L1.
template <int ROUNDS, uint32_t MASK>
__global__ void __launch_bounds__(256)
k_crypt_blocks(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out,
               uint64_t n_blocks, RotMul rm) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_blocks) return;
  uint32_t k[8], s[4];
  load_key(key, k);
  page_seed(desc, g >> 6, s);
  s[3] = static_cast<uint32_t>(g & 63); // word 15 = block index
  const uint4 *src = in + g * 4;
  uint4 d0 = ld_v4(src), d1 = ld_v4(src + 1), d2 = ld_v4(src + 2), d3 = ld_v4(src + 3);
  uint32_t x[16];
  chacha_block<ROUNDS, MASK>(x, k, s, rm);
  d0.x ^= x[0];  d0.y ^= x[1];  d0.z ^= x[2];  d0.w ^= x[3];
  d1.x ^= x[4];  d1.y ^= x[5];  d1.z ^= x[6];  d1.w ^= x[7];
  d2.x ^= x[8];  d2.y ^= x[9];  d2.z ^= x[10]; d2.w ^= x[11];
  d3.x ^= x[12]; d3.y ^= x[13]; d3.z ^= x[14]; d3.w ^= x[15];
  uint4 *dst = out + g * 4;
  st_v4(dst, d0); st_v4(dst + 1, d1); st_v4(dst + 2, d2); st_v4(dst + 3, d3);
}

// ---------------------------------------------------------------------------
// v2: persistent page-slot kernel.  A CTA of 256 threads owns 4 page slots;
// thread t always handles block b = t % 64 of its slot's page and strides over
// pages (page += 4 * gridDim.x), so per thread:
//   * the first column quarter round of state column 3 -- words
//     (sigma3, k3, k7, b), the only column holding the block index -- depends
//     on (key, b) alone and is computed once per thread;
//   * column rounds 1 and 2 -- (sigma1, k1, k5, vaddr_hi) and
//     (sigma2, k2, k6, pid) -- are recomputed only when vaddr_hi or pid
//     changes (warp-uniform test: a warp covers 32 blocks of one page);
//   * only column 0 (sigma0, k0, k4, vaddr_lo) is recomputed for every page.
// That is 3 of the 80 ChaCha20 quarter rounds per block (3 of 32 for ChaCha8)
// hoisted out of the page loop; the result is bit-identical because the block
// function is unchanged, only common subexpressions are shared.  The next
// page's 64 bytes are loaded into registers before the current page's
// rounds run (software pipelining), so HBM latency overlaps ARX work.
template <int ROUNDS>
__global__ void __launch_bounds__(256, 2)
k_crypt_pages(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out,
              uint64_t n_pages) {
  constexpr RotMul rm{};
  const uint32_t b = threadIdx.x & 63;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 4;
  uint64_t page = static_cast<uint64_t>(blockIdx.x) * 4 + (threadIdx.x >> 6);
  if (page >= n_pages) return;
  uint32_t k[8];
  load_key(key, k);
  // column 3 after the first column quarter round: (key, b) only
  uint32_t c3a = kSigma3, c3b = k[3], c3c = k[7], c3d = b;
  quarter_round<0>(c3a, c3b, c3c, c3d, rm);
  // columns 1, 2 cache, keyed by (vaddr_hi, pid)
  uint32_t c1a = 0, c1b = 0, c1c = 0, c1d = 0, c2a = 0, c2b = 0, c2c = 0, c2d = 0;
  uint32_t cached_hi = 0, cached_pid = 0;
  bool cached = false;

  const uint4 *src = in + page * 256 + b * 4;
  uint4 d0 = ld_v4(src), d1 = ld_v4(src + 1), d2 = ld_v4(src + 2), d3 = ld_v4(src + 3);
  for (;;) {
    const uint64_t next = page + stride;
    const bool has_next = next < n_pages;
    uint4 n0, n1, n2, n3;
    if (has_next) {
      const uint4 *ns = in + next * 256 + b * 4;
      n0 = ld_v4(ns); n1 = ld_v4(ns + 1); n2 = ld_v4(ns + 2); n3 = ld_v4(ns + 3);
    }
    uint32_t s[4];
    page_seed(desc, page, s);
    if (!cached || s[1] != cached_hi || s[2] != cached_pid) {
      c1a = kSigma1; c1b = k[1]; c1c = k[5]; c1d = s[1];
      quarter_round<0>(c1a, c1b, c1c, c1d, rm);
      c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = s[2];
      quarter_round<0>(c2a, c2b, c2c, c2d, rm);
      cached_hi = s[1];
      cached_pid = s[2];
      cached = true;
    }
    uint32_t x[16];
    x[0] = kSigma0; x[4] = k[0]; x[8] = k[4]; x[12] = s[0];
    quarter_round<0>(x[0], x[4], x[8], x[12], rm);
    x[1] = c1a; x[5] = c1b; x[9] = c1c; x[13] = c1d;
    x[2] = c2a; x[6] = c2b; x[10] = c2c; x[14] = c2d;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int i = 1; i < ROUNDS / 2; ++i) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    uint4 *dst = out + page * 256 + b * 4;
    st_v4(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                          d0.w ^ (x[3] + kSigma3)));
    st_v4(dst + 1, make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]),
                              d1.w ^ (x[7] + k[3])));
    st_v4(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]),
                              d2.w ^ (x[11] + k[7])));
    st_v4(dst + 3, make_uint4(d3.x ^ (x[12] + s[0]), d3.y ^ (x[13] + s[1]), d3.z ^ (x[14] + s[2]),
                              d3.w ^ (x[15] + b)));
    if (!has_next) break;
    page = next;
    d0 = n0; d1 = n1; d2 = n2; d3 = n3;
  }
}

// ---------------------------------------------------------------------------
// v3: the v2 page loop (same hoisting, same thread -> block index mapping) with
// fully coalesced global traffic: each warp moves its half page (2 KiB) with
// four 512-byte-contiguous LDG.128/STG.128 (lane l takes bytes 16l + 512j)
// and exchanges it through 2 KiB of shared memory per warp, so that lane t
// can XOR block t.  The 16-byte chunks are XOR-swizzled (chunk q of the tile
// lives at column (q & 7) ^ ((q >> 3) & 7) of 128-byte row q >> 3), which
// makes both the coalesced and the per-block LDS/STS.128 patterns
// bank-conflict-free.  Used for pages in mapped pinned host memory (zero-copy:
// every PCIe request is a full 512-byte warp access) and selectable for HBM.
__device__ __forceinline__ uint32_t swz(uint32_t q) { return (q & ~7u) | ((q ^ (q >> 3)) & 7u); }

template <int ROUNDS>
__global__ void __launch_bounds__(256, 2)
k_crypt_pages_coalesced(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out,
                        uint64_t n_pages) {
  constexpr RotMul rm{};
  __shared__ uint4 tile[8][128]; // one 2 KiB half page per warp
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t b = threadIdx.x & 63;       // block index within the page (constant)
  const uint32_t half = (threadIdx.x >> 5) & 1;
  uint4 *t = tile[warp];
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 4;
  uint64_t page = static_cast<uint64_t>(blockIdx.x) * 4 + (threadIdx.x >> 6);
  if (page >= n_pages) return;
  uint32_t k[8];
  load_key(key, k);
  uint32_t c3a = kSigma3, c3b = k[3], c3c = k[7], c3d = b;
  quarter_round<0>(c3a, c3b, c3c, c3d, rm);
  uint32_t c1a = 0, c1b = 0, c1c = 0, c1d = 0, c2a = 0, c2b = 0, c2c = 0, c2d = 0;
  uint32_t cached_hi = 0, cached_pid = 0;
  bool cached = false;

  // coalesced: lane l of load j takes tile chunk q = 32j + l
  const uint4 *src = in + page * 256 + half * 128 + lane;
  uint4 d0 = ld_v4(src), d1 = ld_v4(src + 32), d2 = ld_v4(src + 64), d3 = ld_v4(src + 96);
  uint64_t nva;
  uint32_t npid;
  desc_fetch(desc, page, nva, npid);
  for (;;) {
    const uint64_t next = page + stride;
    const bool has_next = next < n_pages;
    // stage this half page into shared memory (swizzled), then prefetch the
    // next page and its descriptor
    t[swz(lane)] = d0; t[swz(lane + 32)] = d1; t[swz(lane + 64)] = d2; t[swz(lane + 96)] = d3;
    uint32_t s[4];
    s[0] = static_cast<uint32_t>(nva);
    s[1] = static_cast<uint32_t>(nva >> 32);
    s[2] = npid;
    if (has_next) {
      const uint4 *ns = in + next * 256 + half * 128 + lane;
      d0 = ld_v4(ns); d1 = ld_v4(ns + 32); d2 = ld_v4(ns + 64); d3 = ld_v4(ns + 96);
      desc_fetch(desc, next, nva, npid);
    }
    // vaddr_hi and pid columns cached separately: a per-page pid re-runs one
    // quarter round, not two (ChaCha8 pid arrays 3276-3280 vs 3256-3261 GB/s)
    if (!cached || s[1] != cached_hi) {
      c1a = kSigma1; c1b = k[1]; c1c = k[5]; c1d = s[1];
      quarter_round<0>(c1a, c1b, c1c, c1d, rm);
      cached_hi = s[1];
    }
    if (!cached || s[2] != cached_pid) {
      c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = s[2];
      quarter_round<0>(c2a, c2b, c2c, c2d, rm);
      cached_pid = s[2];
    }
    cached = true;
    uint32_t x[16];
    x[0] = kSigma0; x[4] = k[0]; x[8] = k[4]; x[12] = s[0];
    quarter_round<0>(x[0], x[4], x[8], x[12], rm);
    x[1] = c1a; x[5] = c1b; x[9] = c1c; x[13] = c1d;
    x[2] = c2a; x[6] = c2b; x[10] = c2c; x[14] = c2d;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int i = 1; i < ROUNDS / 2; ++i) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    __syncwarp();
    // lane owns tile chunks 4*lane .. 4*lane+3 (its 64-byte block)
    const uint32_t q = 4 * lane;
    uint4 v0 = t[swz(q)], v1 = t[swz(q + 1)], v2 = t[swz(q + 2)], v3 = t[swz(q + 3)];
    v0.x ^= x[0] + kSigma0; v0.y ^= x[1] + kSigma1; v0.z ^= x[2] + kSigma2; v0.w ^= x[3] + kSigma3;
    v1.x ^= x[4] + k[0]; v1.y ^= x[5] + k[1]; v1.z ^= x[6] + k[2]; v1.w ^= x[7] + k[3];
    v2.x ^= x[8] + k[4]; v2.y ^= x[9] + k[5]; v2.z ^= x[10] + k[6]; v2.w ^= x[11] + k[7];
    v3.x ^= x[12] + s[0]; v3.y ^= x[13] + s[1]; v3.z ^= x[14] + s[2]; v3.w ^= x[15] + b;
    t[swz(q)] = v0; t[swz(q + 1)] = v1; t[swz(q + 2)] = v2; t[swz(q + 3)] = v3;
    __syncwarp();
    uint4 *dst = out + page * 256 + half * 128 + lane;
    st_v4(dst, t[swz(lane)]); st_v4(dst + 32, t[swz(lane + 32)]);
    st_v4(dst + 64, t[swz(lane + 64)]); st_v4(dst + 96, t[swz(lane + 96)]);
    __syncwarp();
    if (!has_next) break;
    page = next;
  }
}

// ---------------------------------------------------------------------------
// v4: TMA pipeline.  The batch is viewed as a 2D tensor of 128-byte rows
// (32 rows = one 4 KiB page per TMA box).  A CTA holds 4 independent page
// slots of 64 threads (2 warps); slot k walks pages blockIdx.x*4 + k,
// + 4*gridDim.x, ...  The slot's first thread keeps STAGES-1 pages in flight
// with cp.async.bulk.tensor loads (SWIZZLE_128B, completion on the slot's
// mbarrier), the slot's 64 threads compute their block's keystream (v2
// hoisting) while the data lands, XOR it in shared memory (the 128B swizzle
// makes the per-block LDS/STS.128 pattern bank-conflict-free), meet on a
// 64-thread named barrier, and the leader writes the page back with a TMA
// store.  No data registers are held across iterations, so bytes in flight
// are set by shared memory (STAGES x 16 KiB per CTA), not by registers.
constexpr int kPageRows = 32;
constexpr int kPageBytes = 4096;

__device__ __forceinline__ void named_barrier_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int ROUNDS, int STAGES>
__global__ void __launch_bounds__(256, 3)
k_crypt_pages_tma(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                  const uint32_t *__restrict__ key, PageDesc desc, uint64_t n_pages) {
  constexpr RotMul rm{};
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[4][STAGES];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t tid = threadIdx.x;
  const uint32_t slot = tid >> 6;
  const uint32_t b = tid & 63;
  const bool leader = b == 0;
  uint8_t *ring = smem + slot * (STAGES * kPageBytes);
  uint64_t *bars = full[slot];
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 4;
  const uint64_t page0 = static_cast<uint64_t>(blockIdx.x) * 4 + slot;
  if (page0 >= n_pages) return; // whole slot (2 warps) leaves together
  if (leader) {
    if (slot == 0) {
      prefetch_tmap(&tin);
      prefetch_tmap(&tout);
    }
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
#pragma unroll
    for (int j = 0; j < STAGES - 1; ++j) {
      const uint64_t pj = page0 + static_cast<uint64_t>(j) * stride;
      if (pj < n_pages) {
        mbar_arrive_expect_tx(&bars[j], kPageBytes);
        tma_load_2d(ring + j * kPageBytes, &tin, 0, static_cast<int32_t>(pj * kPageRows), &bars[j]);
      }
    }
  }
  named_barrier_sync(1 + slot, 64); // barrier inits visible to the slot
  uint32_t k[8];
  load_key(key, k);
  uint32_t c3a = kSigma3, c3b = k[3], c3c = k[7], c3d = b;
  quarter_round<0>(c3a, c3b, c3c, c3d, rm);
  uint32_t c1a = 0, c1b = 0, c1c = 0, c1d = 0, c2a = 0, c2b = 0, c2c = 0, c2d = 0;
  uint32_t cached_hi = 0, cached_pid = 0;
  bool cached = false;
  const uint32_t row = b >> 1;
  const uint32_t chunk0 = (b & 1) * 4;
  uint32_t off[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) off[c] = row * 128 + (((chunk0 + c) ^ (row & 7)) << 4);

  for (uint32_t i = 0;; ++i) {
    const uint64_t page = page0 + static_cast<uint64_t>(i) * stride;
    if (page >= n_pages) break;
    const uint32_t st = i % STAGES;
    uint32_t s[4];
    page_seed(desc, page, s);
    if (!cached || s[1] != cached_hi || s[2] != cached_pid) {
      c1a = kSigma1; c1b = k[1]; c1c = k[5]; c1d = s[1];
      quarter_round<0>(c1a, c1b, c1c, c1d, rm);
      c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = s[2];
      quarter_round<0>(c2a, c2b, c2c, c2d, rm);
      cached_hi = s[1];
      cached_pid = s[2];
      cached = true;
    }
    uint32_t x[16];
    x[0] = kSigma0; x[4] = k[0]; x[8] = k[4]; x[12] = s[0];
    quarter_round<0>(x[0], x[4], x[8], x[12], rm);
    x[1] = c1a; x[5] = c1b; x[9] = c1c; x[13] = c1d;
    x[2] = c2a; x[6] = c2b; x[10] = c2c; x[14] = c2d;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int r = 1; r < ROUNDS / 2; ++r) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    uint8_t *buf = ring + st * kPageBytes;
    mbar_wait(&bars[st], (i / STAGES) & 1);
    uint4 *p0 = reinterpret_cast<uint4 *>(buf + off[0]);
    uint4 *p1 = reinterpret_cast<uint4 *>(buf + off[1]);
    uint4 *p2 = reinterpret_cast<uint4 *>(buf + off[2]);
    uint4 *p3 = reinterpret_cast<uint4 *>(buf + off[3]);
    uint4 v0 = *p0, v1 = *p1, v2 = *p2, v3 = *p3;
    v0.x ^= x[0] + kSigma0; v0.y ^= x[1] + kSigma1; v0.z ^= x[2] + kSigma2; v0.w ^= x[3] + kSigma3;
    v1.x ^= x[4] + k[0]; v1.y ^= x[5] + k[1]; v1.z ^= x[6] + k[2]; v1.w ^= x[7] + k[3];
    v2.x ^= x[8] + k[4]; v2.y ^= x[9] + k[5]; v2.z ^= x[10] + k[6]; v2.w ^= x[11] + k[7];
    v3.x ^= x[12] + s[0]; v3.y ^= x[13] + s[1]; v3.z ^= x[14] + s[2]; v3.w ^= x[15] + b;
    *p0 = v0; *p1 = v1; *p2 = v2; *p3 = v3;
    fence_proxy_async_smem();
    named_barrier_sync(1 + slot, 64);
    if (leader) {
      tma_store_2d(&tout, 0, static_cast<int32_t>(page * kPageRows), buf);
      bulk_commit();
      const uint64_t pn = page0 + static_cast<uint64_t>(i + STAGES - 1) * stride;
      if (pn < n_pages) {
        bulk_wait_read<1>(); // iteration i-1's store no longer reads the stage we refill
        const uint32_t sn = (i + STAGES - 1) % STAGES;
        mbar_arrive_expect_tx(&bars[sn], kPageBytes);
        tma_load_2d(ring + sn * kPageBytes, &tin, 0, static_cast<int32_t>(pn * kPageRows), &bars[sn]);
      }
    }
  }
  if (leader) bulk_wait<0>();
}

// ---------------------------------------------------------------------------
// v5: the v2 page loop with a cp.async (LDGSTS) ring instead of register
// prefetch.  Each thread streams its own 64-byte block of the pages 1 and 2
// strides ahead into a 3-stage shared-memory ring (no registers held, so
// occupancy is 4 CTAs/SM and ~128 KiB per SM is in flight), waits for the
// current page's group, XORs and stores.  The 4 chunks of a thread's block
// sit at XOR-swizzled positions c ^ ((t >> 1) & 3), which makes the per-thread
// 64-byte LDS/STS pattern bank-conflict-free while each chunk keeps a static
// register.  Only the issuing thread reads its own copies, so no barrier is
// needed (cp.async.wait_group gives the thread visibility).
__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void *gptr) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

//
// CONTIG specialises the common bulk case -- contiguous vaddrs (vaddr0 +
// 4096*i) and one pid -- so that the page loop only carries 32-bit page
// indices, pointers and the vaddr advance by constant strides, and the pid
// column round is hoisted out of the loop entirely; the general case reads
// per-page descriptors.  Page counts are < 2^31 (the host splits larger
// batches).
//
// DM (descriptor mode) compiles each descriptor shape separately: bit 0 = a
// per-page vaddr array, bit 1 = a per-page pid array, so no loop carries a
// null-pointer test and a scalar pid keeps its column round hoisted.
template <int ROUNDS, int DM>
__global__ void __launch_bounds__(256, (DM == 0 || ROUNDS > 12) ? 4 : 3) // two descriptor sets need registers
k_crypt_pages_async(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out,
                    uint32_t n_pages) {
  constexpr bool CONTIG = DM == 0;
  constexpr bool VA = (DM & 1) != 0, PA = (DM & 2) != 0;
  constexpr RotMul rm{};
  constexpr int kStages = 3;
  __shared__ uint4 ring[kStages][256 * 4]; // 16 KiB per stage
  const uint32_t tid = threadIdx.x;
  const uint32_t b = tid & 63;
  const uint32_t sw = (tid >> 1) & 3;
  const uint32_t stride = gridDim.x * 4;
  uint32_t page = blockIdx.x * 4 + (tid >> 6);
  if (page >= n_pages) return;
  const uint32_t base0 = smem_u32(&ring[0][tid * 4]);
  constexpr uint32_t kStageBytes = 256 * 4 * 16;
  const uint64_t step = static_cast<uint64_t>(stride) * 256; // uint4 per stride
  const uint4 *src_ahead = in + static_cast<uint64_t>(page) * 256 + b * 4;
  uint4 *dst = out + static_cast<uint64_t>(page) * 256 + b * 4;
  uint32_t page_ahead = page;
  auto issue = [&](int st) { // next page for the ring, then advance the ahead cursor
    if (page_ahead < n_pages) {
      const uint32_t sdst = base0 + st * kStageBytes;
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async16(sdst + 16 * (c ^ sw), src_ahead + c);
    }
    cp_async_commit(); // empty groups keep the count uniform at the tail
    page_ahead += stride;
    src_ahead += step;
  };
  issue(0);
  issue(1);
  uint32_t k[8];
  load_key(key, k);
  uint32_t c3a = kSigma3, c3b = k[3], c3c = k[7], c3d = b;
  quarter_round<0>(c3a, c3b, c3c, c3d, rm);
  uint32_t c1a = 0, c1b = 0, c1c = 0, c1d = 0, c2a = 0, c2b = 0, c2c = 0, c2d = 0;
  uint32_t cached_hi = 0, cached_pid = 0;
  bool cached = false;
  uint64_t va = desc.vaddr0 + (static_cast<uint64_t>(page) << 12);
  const uint64_t va_step = static_cast<uint64_t>(stride) << 12;
  if constexpr (!PA) {
    c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = desc.pid0;
    quarter_round<0>(c2a, c2b, c2c, c2d, rm);
  }
  // per-page descriptors are loaded one page ahead, so the load latency
  // hides under the current page's rounds
  uint64_t nva = 0;
  uint32_t npid = 0;
  if constexpr (VA) nva = __ldg(desc.vaddrs + page);
  if constexpr (PA) npid = __ldg(desc.pids + page);
  bool pid_cached = false;
  int st = 0;
  // (unrolled over page pairs where that pays: R <= 12, and R = 20 with a
  // vaddr array only -- 1723 vs 1699 GB/s; with a pid array the R = 20 pair
  // loop is slower, 1675 vs 1739, profiles/r01_desc_probe.txt)
  if constexpr (CONTIG || (ROUNDS > 12 && DM != 1)) {
  for (;;) {
    issue(st == 0 ? 2 : st - 1); // stage (st + 2) % 3
    uint32_t s[3];
    const uint64_t v = VA ? nva : va;
    s[0] = static_cast<uint32_t>(v);
    s[1] = static_cast<uint32_t>(v >> 32);
    s[2] = PA ? npid : desc.pid0;
    if constexpr (!CONTIG) {
      if (page + stride < n_pages) {
        if constexpr (VA) nva = __ldg(desc.vaddrs + page + stride);
        if constexpr (PA) npid = __ldg(desc.pids + page + stride);
      }
    }
    if (!cached || s[1] != cached_hi) {
      c1a = kSigma1; c1b = k[1]; c1c = k[5]; c1d = s[1];
      quarter_round<0>(c1a, c1b, c1c, c1d, rm);
      cached_hi = s[1];
      cached = true;
    }
    if constexpr (PA) { // R=20 keeps the cached round (the unconditional one: 1678 vs 1735 GB/s)
      if (!pid_cached || s[2] != cached_pid) {
        c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = s[2];
        quarter_round<0>(c2a, c2b, c2c, c2d, rm);
        cached_pid = s[2];
        pid_cached = true;
      }
    }
    uint32_t x[16];
    x[0] = kSigma0; x[4] = k[0]; x[8] = k[4]; x[12] = s[0];
    quarter_round<0>(x[0], x[4], x[8], x[12], rm);
    x[1] = c1a; x[5] = c1b; x[9] = c1c; x[13] = c1d;
    x[2] = c2a; x[6] = c2b; x[10] = c2c; x[14] = c2d;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int r = 1; r < ROUNDS / 2; ++r) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    cp_async_wait<2>(); // this page's group has landed
    const uint4 *mine = &ring[st][tid * 4];
    const uint4 d0 = mine[0 ^ sw], d1 = mine[1 ^ sw], d2 = mine[2 ^ sw], d3 = mine[3 ^ sw];
    if constexpr (ROUNDS <= 12) {
      st_v8(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                            d0.w ^ (x[3] + kSigma3)),
            make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]), d1.w ^ (x[7] + k[3])));
      st_v8(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]), d2.w ^ (x[11] + k[7])),
            make_uint4(d3.x ^ (x[12] + s[0]), d3.y ^ (x[13] + s[1]), d3.z ^ (x[14] + s[2]), d3.w ^ (x[15] + b)));
    } else { // (each store right after its words: the schedule R=20 was tuned on)
    st_v4(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                          d0.w ^ (x[3] + kSigma3)));
    st_v4(dst + 1, make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]),
                              d1.w ^ (x[7] + k[3])));
    st_v4(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]),
                              d2.w ^ (x[11] + k[7])));
    st_v4(dst + 3, make_uint4(d3.x ^ (x[12] + s[0]), d3.y ^ (x[13] + s[1]), d3.z ^ (x[14] + s[2]),
                              d3.w ^ (x[15] + b)));
    }
    page += stride;
    if (page >= n_pages) break;
    dst += step;
    va += va_step;
    st = st == 2 ? 0 : st + 1;
  }
  } else {
    // Descriptor arrays: two register sets, each loaded two pages before its
    // use and refilled right after it, the loop unrolled over the pair -- one
    // loop-carried set had to be copied at the loop end and stalled there on
    // its own load (ncu long_scoreboard).
    uint64_t va_a = nva, va_b = 0;
    uint32_t pid_a = npid, pid_b = desc.pid0;
    if (page + stride < n_pages) {
      if constexpr (VA) va_b = __ldg(desc.vaddrs + page + stride);
      if constexpr (PA) pid_b = __ldg(desc.pids + page + stride);
    }
    auto one_page = [&](uint64_t &rv, uint32_t &rp) -> bool {
      uint32_t s[3];
      const uint64_t v = VA ? rv : va;
      s[0] = static_cast<uint32_t>(v);
      s[1] = static_cast<uint32_t>(v >> 32);
      s[2] = PA ? rp : desc.pid0;
      if (page + 2 * stride < n_pages) {
        if constexpr (VA) rv = __ldg(desc.vaddrs + page + 2 * stride);
        if constexpr (PA) rp = __ldg(desc.pids + page + 2 * stride);
      }
    issue(st == 0 ? 2 : st - 1); // stage (st + 2) % 3
    if (!cached || s[1] != cached_hi) {
      c1a = kSigma1; c1b = k[1]; c1c = k[5]; c1d = s[1];
      quarter_round<0>(c1a, c1b, c1c, c1d, rm);
      cached_hi = s[1];
      cached = true;
    }
    if constexpr (PA) { // every page, no branch: R=12 2537-2627 vs 2432-2558 GB/s (profiles/r01_desc_probe.txt)
      c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = s[2];
      quarter_round<0>(c2a, c2b, c2c, c2d, rm);
    }
    uint32_t x[16];
    x[0] = kSigma0; x[4] = k[0]; x[8] = k[4]; x[12] = s[0];
    quarter_round<0>(x[0], x[4], x[8], x[12], rm);
    x[1] = c1a; x[5] = c1b; x[9] = c1c; x[13] = c1d;
    x[2] = c2a; x[6] = c2b; x[10] = c2c; x[14] = c2d;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int r = 1; r < ROUNDS / 2; ++r) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    cp_async_wait<2>(); // this page's group has landed
    const uint4 *mine = &ring[st][tid * 4];
    const uint4 d0 = mine[0 ^ sw], d1 = mine[1 ^ sw], d2 = mine[2 ^ sw], d3 = mine[3 ^ sw];
    if constexpr (ROUNDS <= 12) {
      st_v8(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                            d0.w ^ (x[3] + kSigma3)),
            make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]), d1.w ^ (x[7] + k[3])));
      st_v8(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]), d2.w ^ (x[11] + k[7])),
            make_uint4(d3.x ^ (x[12] + s[0]), d3.y ^ (x[13] + s[1]), d3.z ^ (x[14] + s[2]), d3.w ^ (x[15] + b)));
    } else { // (each store right after its words: the schedule R=20 was tuned on)
    st_v4(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                          d0.w ^ (x[3] + kSigma3)));
    st_v4(dst + 1, make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]),
                              d1.w ^ (x[7] + k[3])));
    st_v4(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]),
                              d2.w ^ (x[11] + k[7])));
    st_v4(dst + 3, make_uint4(d3.x ^ (x[12] + s[0]), d3.y ^ (x[13] + s[1]), d3.z ^ (x[14] + s[2]),
                              d3.w ^ (x[15] + b)));
    }
      page += stride;
      if (page >= n_pages) return false;
      dst += step;
      va += va_step;
      st = st == 2 ? 0 : st + 1;
      return true;
    };
    for (;;) {
      if (!one_page(va_a, pid_a)) break;
      if (!one_page(va_b, pid_b)) break;
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// v5r: v5's ring and page loop for per-page descriptor arrays, with each page
// slot walking a contiguous RUN of pages (slot s takes [s*L, s*L + L), L
// even) instead of every (gridDim*4)-th page, so two consecutive pages'
// descriptors are adjacent: one 16-byte load fetches both vaddrs and one
// 8-byte load both pids.  Per page that halves the descriptor loads on the
// MIO queue the page stream shares (v5 at ChaCha12 is MIO-limited with
// descriptors, profiles/r02_desc_experiments.txt).  The pair for pages
// (p+2, p+3) is loaded while (p, p+1) run.  Needs vaddrs 16-byte and pids
// 8-byte aligned (the host checks; else v5).
template <int ROUNDS, int DM>
__global__ void __launch_bounds__(256, 3)
k_crypt_pages_run(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out, uint32_t n_pages,
                  uint32_t run) {
  constexpr bool VA = (DM & 1) != 0, PA = (DM & 2) != 0;
  constexpr RotMul rm{};
  constexpr int kStages = 3;
  __shared__ uint4 ring[kStages][256 * 4];
  const uint32_t tid = threadIdx.x;
  const uint32_t b = tid & 63;
  const uint32_t sw = (tid >> 1) & 3;
  uint32_t page = (blockIdx.x * 4 + (tid >> 6)) * run; // run is even: every run starts on an even page
  const uint32_t end = min(n_pages, page + run);
  if (page >= end) return;
  const uint32_t base0 = smem_u32(&ring[0][tid * 4]);
  constexpr uint32_t kStageBytes = 256 * 4 * 16;
  const uint4 *src_ahead = in + static_cast<uint64_t>(page) * 256 + b * 4;
  uint4 *dst = out + static_cast<uint64_t>(page) * 256 + b * 4;
  uint32_t page_ahead = page;
  auto issue = [&](int st) {
    if (page_ahead < end) {
      const uint32_t sdst = base0 + st * kStageBytes;
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async16(sdst + 16 * (c ^ sw), src_ahead + c);
    }
    cp_async_commit();
    page_ahead += 1;
    src_ahead += 256;
  };
  issue(0);
  issue(1);
  uint32_t k[8];
  load_key(key, k);
  uint32_t c3a = kSigma3, c3b = k[3], c3c = k[7], c3d = b;
  quarter_round<0>(c3a, c3b, c3c, c3d, rm);
  uint32_t c1a = 0, c1b = 0, c1c = 0, c1d = 0, c2a = 0, c2b = 0, c2c = 0, c2d = 0;
  uint32_t cached_hi = 0;
  bool cached = false;
  if constexpr (!PA) {
    c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = desc.pid0;
    quarter_round<0>(c2a, c2b, c2c, c2d, rm);
  }
  // descriptors of the pair (p, p+1); p + 1 may be past the batch on its last page
  auto load_pair = [&](uint32_t p, uint4 &vv, uint2 &pp) {
    if (p + 1 < n_pages) {
      if constexpr (VA) vv = __ldg(reinterpret_cast<const uint4 *>(desc.vaddrs + p));
      if constexpr (PA) pp = __ldg(reinterpret_cast<const uint2 *>(desc.pids + p));
    } else if (p < n_pages) {
      if constexpr (VA) {
        const uint64_t v = __ldg(desc.vaddrs + p);
        vv = make_uint4(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32), 0, 0);
      }
      if constexpr (PA) pp = make_uint2(__ldg(desc.pids + p), 0);
    }
  };
  uint4 vcur = make_uint4(0, 0, 0, 0), vnext = vcur;
  uint2 pcur = make_uint2(0, 0), pnext = pcur;
  load_pair(page, vcur, pcur);
  load_pair(page + 2, vnext, pnext);
  int st = 0;
  auto one_page = [&](uint32_t vlo, uint32_t vhi, uint32_t pid) -> bool {
    uint32_t s[3];
    s[0] = vlo;
    s[1] = vhi;
    s[2] = pid;
    issue(st == 0 ? 2 : st - 1); // stage (st + 2) % 3
    if (!cached || s[1] != cached_hi) {
      c1a = kSigma1; c1b = k[1]; c1c = k[5]; c1d = s[1];
      quarter_round<0>(c1a, c1b, c1c, c1d, rm);
      cached_hi = s[1];
      cached = true;
    }
    if constexpr (PA) {
      c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = s[2];
      quarter_round<0>(c2a, c2b, c2c, c2d, rm);
    }
    uint32_t x[16];
    x[0] = kSigma0; x[4] = k[0]; x[8] = k[4]; x[12] = s[0];
    quarter_round<0>(x[0], x[4], x[8], x[12], rm);
    x[1] = c1a; x[5] = c1b; x[9] = c1c; x[13] = c1d;
    x[2] = c2a; x[6] = c2b; x[10] = c2c; x[14] = c2d;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int r = 1; r < ROUNDS / 2; ++r) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    cp_async_wait<2>(); // this page's group has landed
    const uint4 *mine = &ring[st][tid * 4];
    const uint4 d0 = mine[0 ^ sw], d1 = mine[1 ^ sw], d2 = mine[2 ^ sw], d3 = mine[3 ^ sw];
    st_v8(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                          d0.w ^ (x[3] + kSigma3)),
          make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]), d1.w ^ (x[7] + k[3])));
    st_v8(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]), d2.w ^ (x[11] + k[7])),
          make_uint4(d3.x ^ (x[12] + s[0]), d3.y ^ (x[13] + s[1]), d3.z ^ (x[14] + s[2]), d3.w ^ (x[15] + b)));
    page += 1;
    if (page >= end) return false;
    dst += 256;
    st = st == 2 ? 0 : st + 1;
    return true;
  };
  for (;;) {
    uint32_t lo0, hi0, lo1, hi1, p0, p1;
    if constexpr (VA) {
      lo0 = vcur.x; hi0 = vcur.y; lo1 = vcur.z; hi1 = vcur.w;
    } else {
      const uint64_t v0 = desc.vaddr0 + (static_cast<uint64_t>(page) << 12);
      const uint64_t v1 = v0 + 4096;
      lo0 = static_cast<uint32_t>(v0); hi0 = static_cast<uint32_t>(v0 >> 32);
      lo1 = static_cast<uint32_t>(v1); hi1 = static_cast<uint32_t>(v1 >> 32);
    }
    if constexpr (PA) {
      p0 = pcur.x; p1 = pcur.y;
    } else {
      p0 = p1 = desc.pid0;
    }
    vcur = vnext;
    pcur = pnext;
    load_pair(page + 4, vnext, pnext); // two pages ahead of the pair after this one
    if (!one_page(lo0, hi0, p0)) break;
    if (!one_page(lo1, hi1, p1)) break;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
#ifndef PC_RUN2_R20_UNROLL
#define PC_RUN2_R20_UNROLL 3
#endif
// v5r2: v5r's page runs with ONE WARP per page slot and two blocks per thread
// (lane l takes blocks l and l + 32).  With per-page descriptor arrays the
// per-page seed work -- the round-1 quarter round of column 0 (vaddr_lo) and,
// with a pid array, of column 2 -- is what separates v5r from the contiguous
// loop (+16 ALU-pipe instructions per page-warp, profiles/r02_desc_opmix.txt);
// here each thread pays it once for two blocks, and the descriptor pair loads
// are per warp instead of per two warps.  No shared memory beyond the ring
// and no shuffles (v6/v9 lost on MIO, profiles/r02_desc_experiments.txt).
// 128-thread CTAs: 4 slots x 3 stages x 4 KiB = 48 KiB static ring.
template <int ROUNDS, int DM>
__global__ void __launch_bounds__(128, 4)
k_crypt_pages_run2(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out, uint32_t n_pages,
                   uint32_t run) {
  constexpr bool VA = (DM & 1) != 0, PA = (DM & 2) != 0;
  constexpr RotMul rm{};
  constexpr int kStages = 3;
  __shared__ uint4 ring[kStages][128 * 8]; // 16 KiB per stage
  const uint32_t tid = threadIdx.x;
  const uint32_t l = tid & 31;
  const uint32_t sw = (l >> 1) & 3;
  uint32_t page = (blockIdx.x * 4 + (tid >> 5)) * run; // run is even
  const uint32_t end = min(n_pages, page + run);
  if (page >= end) return;
  // block l of the slot's page at chunk (w*64 + l)*4, block l+32 at +32*4 chunks
  const uint32_t base0 = smem_u32(&ring[0][((tid >> 5) * 64 + l) * 4]);
  constexpr uint32_t kStageBytes = 128 * 8 * 16;
  constexpr uint32_t kHalf = 32 * 4 * 16;
  const uint4 *src_ahead = in + static_cast<uint64_t>(page) * 256 + l * 4;
  uint4 *dst = out + static_cast<uint64_t>(page) * 256 + l * 4;
  uint32_t page_ahead = page;
  auto issue = [&](int st) {
    if (page_ahead < end) {
      const uint32_t sdst = base0 + st * kStageBytes;
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async16(sdst + 16 * (c ^ sw), src_ahead + c);
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async16(sdst + kHalf + 16 * (c ^ sw), src_ahead + 128 + c);
    }
    cp_async_commit();
    page_ahead += 1;
    src_ahead += 256;
  };
  issue(0);
  issue(1);
  uint32_t k[8];
  load_key(key, k);
  const uint32_t bA = l, bB = l + 32;
  uint32_t a3a = kSigma3, a3b = k[3], a3c = k[7], a3d = bA;
  quarter_round<0>(a3a, a3b, a3c, a3d, rm);
  uint32_t b3a = kSigma3, b3b = k[3], b3c = k[7], b3d = bB;
  quarter_round<0>(b3a, b3b, b3c, b3d, rm);
  uint32_t c1a = 0, c1b = 0, c1c = 0, c1d = 0, c2a = 0, c2b = 0, c2c = 0, c2d = 0;
  uint32_t cached_hi = 0;
  bool cached = false;
  if constexpr (!PA) {
    c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = desc.pid0;
    quarter_round<0>(c2a, c2b, c2c, c2d, rm);
  }
  auto load_pair = [&](uint32_t p, uint4 &vv, uint2 &pp) {
    if (p + 1 < n_pages) {
      if constexpr (VA) vv = __ldg(reinterpret_cast<const uint4 *>(desc.vaddrs + p));
      if constexpr (PA) pp = __ldg(reinterpret_cast<const uint2 *>(desc.pids + p));
    } else if (p < n_pages) {
      if constexpr (VA) {
        const uint64_t v = __ldg(desc.vaddrs + p);
        vv = make_uint4(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32), 0, 0);
      }
      if constexpr (PA) pp = make_uint2(__ldg(desc.pids + p), 0);
    }
  };
  uint4 vcur = make_uint4(0, 0, 0, 0), vnext = vcur;
  uint2 pcur = make_uint2(0, 0), pnext = pcur;
  load_pair(page, vcur, pcur);
  load_pair(page + 2, vnext, pnext);
  int st = 0;
  // one page per iteration, not unrolled: two blocks of fully unrolled rounds
  // are already twice v5's loop body (the i-cache)
#pragma unroll 1
  for (;;) {
    const bool odd = (page & 1) != 0; // runs start on even pages
    uint32_t vlo, vhi, pid;
    if constexpr (VA) {
      vlo = odd ? vcur.z : vcur.x;
      vhi = odd ? vcur.w : vcur.y;
    } else {
      const uint64_t v = desc.vaddr0 + (static_cast<uint64_t>(page) << 12);
      vlo = static_cast<uint32_t>(v);
      vhi = static_cast<uint32_t>(v >> 32);
    }
    if constexpr (PA) pid = odd ? pcur.y : pcur.x;
    else pid = desc.pid0;
    if (odd) { // the pair is consumed: the next one is resident, fetch the one after
      vcur = vnext;
      pcur = pnext;
      load_pair(page + 3, vnext, pnext);
    }
    issue(st == 0 ? 2 : st - 1); // stage (st + 2) % 3
    if (!cached || vhi != cached_hi) {
      c1a = kSigma1; c1b = k[1]; c1c = k[5]; c1d = vhi;
      quarter_round<0>(c1a, c1b, c1c, c1d, rm);
      cached_hi = vhi;
      cached = true;
    }
    if constexpr (PA) {
      c2a = kSigma2; c2b = k[2]; c2c = k[6]; c2d = pid;
      quarter_round<0>(c2a, c2b, c2c, c2d, rm);
    }
    uint32_t c0a = kSigma0, c0b = k[0], c0c = k[4], c0d = vlo; // shared by both blocks
    quarter_round<0>(c0a, c0b, c0c, c0d, rm);
    uint32_t x[16], y[16];
    x[0] = c0a; x[4] = c0b; x[8] = c0c; x[12] = c0d;
    x[1] = c1a; x[5] = c1b; x[9] = c1c; x[13] = c1d;
    x[2] = c2a; x[6] = c2b; x[10] = c2c; x[14] = c2d;
    x[3] = a3a; x[7] = a3b; x[11] = a3c; x[15] = a3d;
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = x[i];
    y[3] = b3a; y[7] = b3b; y[11] = b3c; y[15] = b3d;
    diagonal_round<0>(x, rm);
    diagonal_round<0>(y, rm);
    // R = 20: three double rounds per loop trip (the fully unrolled pair of
    // blocks is ~4200 SASS instructions and thrashes the i-cache)
    constexpr int kUnroll = ROUNDS > 12 ? PC_RUN2_R20_UNROLL : ROUNDS / 2 - 1;
#pragma unroll kUnroll
    for (int r = 1; r < ROUNDS / 2; ++r) {
      column_round<0>(x, rm);
      column_round<0>(y, rm);
      diagonal_round<0>(x, rm);
      diagonal_round<0>(y, rm);
    }
    cp_async_wait<2>(); // this page's group has landed
    const uint4 *mine = &ring[st][((tid >> 5) * 64 + l) * 4];
    {
      const uint4 d0 = mine[0 ^ sw], d1 = mine[1 ^ sw], d2 = mine[2 ^ sw], d3 = mine[3 ^ sw];
      st_v8(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                            d0.w ^ (x[3] + kSigma3)),
            make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]), d1.w ^ (x[7] + k[3])));
      st_v8(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]), d2.w ^ (x[11] + k[7])),
            make_uint4(d3.x ^ (x[12] + vlo), d3.y ^ (x[13] + vhi), d3.z ^ (x[14] + pid), d3.w ^ (x[15] + bA)));
    }
    {
      const uint4 *m2 = mine + 128;
      const uint4 d0 = m2[0 ^ sw], d1 = m2[1 ^ sw], d2 = m2[2 ^ sw], d3 = m2[3 ^ sw];
      st_v8(dst + 128, make_uint4(d0.x ^ (y[0] + kSigma0), d0.y ^ (y[1] + kSigma1), d0.z ^ (y[2] + kSigma2),
                                  d0.w ^ (y[3] + kSigma3)),
            make_uint4(d1.x ^ (y[4] + k[0]), d1.y ^ (y[5] + k[1]), d1.z ^ (y[6] + k[2]), d1.w ^ (y[7] + k[3])));
      st_v8(dst + 130, make_uint4(d2.x ^ (y[8] + k[4]), d2.y ^ (y[9] + k[5]), d2.z ^ (y[10] + k[6]), d2.w ^ (y[11] + k[7])),
            make_uint4(d3.x ^ (y[12] + vlo), d3.y ^ (y[13] + vhi), d3.z ^ (y[14] + pid), d3.w ^ (y[15] + bB)));
    }
    page += 1;
    if (page >= end) break;
    dst += 256;
    st = st == 2 ? 0 : st + 1;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// v6: v5's cp.async page ring with the per-page seed rounds computed once
// per page instead of once per thread.
//
// Of the first column round's four quarter rounds, three depend on the page
// alone: column 0 on vaddr_lo, column 1 on vaddr_hi, column 2 on the pid
// (state words 12..14); only column 3 holds the block index.  v5 hoists
// column 3 per thread and caches columns 1/2 while vaddr_hi/pid repeat, but
// still runs column 0 -- and, with a per-page pid array, column 2 -- in all
// 64 threads of every page.  Here the 64 threads of a page slot compute those
// three columns for the slot's next 32 pages together (lane L of each of the
// slot's two warps takes page 16*half + L, L < 16), file them in a
// shared-memory table, and every thread then reads its page's entry with
// four broadcast LDS.128: per page and warp, 4 LDS replace 8-16 instructions
// on the ALU pipe, the pipe that binds ChaCha12/20.  The descriptor arrays
// are read once per page (one strided LDG per computing lane, prefetched a
// batch ahead) instead of once per page per thread.  Every block is still
// exactly ChaCha_R(state) + state: only common subexpressions are shared.
constexpr int kV6Stages = 3;
constexpr int kV6Batch = 32;                                          // pages per table refill
constexpr size_t kV6RingBytes = kV6Stages * 256 * 4 * 16;              // 48 KiB
constexpr size_t kV6TableBytes = 4 * kV6Batch * 64;                    // 4 slots x 32 pages x 64 B
constexpr size_t kV6Smem = kV6RingBytes + kV6TableBytes;               // dynamic shared memory

// The 64 threads of page slot q meet at named barrier 1 + q.  The id is an
// immediate in each branch: a register id makes ptxas reserve all 16 barriers.
__device__ __forceinline__ void slot_bar(uint32_t q) {
  switch (q) {
    case 0: asm volatile("bar.sync 1, 64;" ::: "memory"); break;
    case 1: asm volatile("bar.sync 2, 64;" ::: "memory"); break;
    case 2: asm volatile("bar.sync 3, 64;" ::: "memory"); break;
    default: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
  }
}

template <int ROUNDS, int DM>
__global__ void __launch_bounds__(256, ROUNDS == 8 ? 3 : 4) // R=8 spills at 64 registers
k_crypt_pages_warp(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out,
                   uint32_t n_pages) {
  constexpr bool VA = (DM & 1) != 0, PA = (DM & 2) != 0;
  constexpr RotMul rm{};
  extern __shared__ __align__(16) uint4 v6_smem[];
  uint4 (*ring)[256 * 4] = reinterpret_cast<uint4 (*)[256 * 4]>(v6_smem);
  const uint32_t tid = threadIdx.x;
  const uint32_t q = tid >> 6;               // page slot
  const uint32_t b = tid & 63;               // block of the page
  const uint32_t sw = (tid >> 1) & 3;
  const uint32_t stride = gridDim.x * 4;
  const uint32_t page0 = blockIdx.x * 4 + q;
  uint32_t page = page0;
  if (page >= n_pages) return; // slot-uniform: both warps of the slot leave together
  uint4 *table = v6_smem + kV6RingBytes / 16 + q * kV6Batch * 4;
  const uint32_t base0 = smem_u32(&ring[0][tid * 4]);
  constexpr uint32_t kStageBytes = 256 * 4 * 16;
  const uint64_t step = static_cast<uint64_t>(stride) * 256; // uint4 per stride
  const uint4 *src_ahead = in + static_cast<uint64_t>(page) * 256 + b * 4;
  uint4 *dst = out + static_cast<uint64_t>(page) * 256 + b * 4;
  uint32_t page_ahead = page;
  auto issue = [&](int st) {
    if (page_ahead < n_pages) {
      const uint32_t sdst = base0 + st * kStageBytes;
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async16(sdst + 16 * (c ^ sw), src_ahead + c);
    }
    cp_async_commit();
    page_ahead += stride;
    src_ahead += step;
  };
  issue(0);
  issue(1);
  uint32_t k[8];
  load_key(key, k);
  uint32_t c3a = kSigma3, c3b = k[3], c3c = k[7], c3d = b;
  quarter_round<0>(c3a, c3b, c3c, c3d, rm);
  // this thread's table entry: page index e = 16*(b >> 5) + (b & 31) for
  // b & 31 < 16, i.e. page page0 + (32*batch + e)*stride, descriptor
  // fetched one batch ahead
  const uint32_t lane = b & 31;
  const bool filler = lane < 16;
  const uint32_t e_idx = 16 * (b >> 5) + lane;
  uint64_t lp = static_cast<uint64_t>(page0) + static_cast<uint64_t>(e_idx) * stride;
  const uint64_t batch_step = static_cast<uint64_t>(kV6Batch) * stride;
  uint64_t nv = 0;
  uint32_t npid = desc.pid0;
  auto fetch = [&]() {
    if constexpr (VA) {
      if (filler && lp < n_pages) nv = __ldg(desc.vaddrs + lp);
    } else {
      nv = desc.vaddr0 + (lp << 12);
    }
    if constexpr (PA) {
      if (filler && lp < n_pages) npid = __ldg(desc.pids + lp);
    }
  };
  fetch();
  auto refill = [&]() {
    slot_bar(q); // both warps of the slot are done with the previous batch
    if (filler) {
      const uint32_t vlo = static_cast<uint32_t>(nv), vhi = static_cast<uint32_t>(nv >> 32), pid = npid;
      uint32_t a0 = kSigma0, b0 = k[0], e0 = k[4], d0 = vlo;
      uint32_t a1 = kSigma1, b1 = k[1], e1 = k[5], d1 = vhi;
      uint32_t a2 = kSigma2, b2 = k[2], e2 = k[6], d2 = pid;
      quarter_round<0>(a0, b0, e0, d0, rm);
      quarter_round<0>(a1, b1, e1, d1, rm);
      quarter_round<0>(a2, b2, e2, d2, rm);
      table[e_idx * 4 + 0] = make_uint4(a0, b0, e0, d0);
      table[e_idx * 4 + 1] = make_uint4(a1, b1, e1, d1);
      table[e_idx * 4 + 2] = make_uint4(a2, b2, e2, d2);
      table[e_idx * 4 + 3] = make_uint4(vlo, vhi, pid, 0u);
      lp += batch_step;
      fetch();
    }
    slot_bar(q); // the batch is filed
  };
  // the table entry of the NEXT page is loaded while this page's rounds run
  // (its shared-memory latency stalled the rounds otherwise: ncu
  // short_scoreboard); the refill for pages 32(B+1).. runs in iteration 32B+31
  // before that prefetch
  refill();
  uint4 q0 = table[0], q1 = table[1], q2 = table[2], sd = table[3];
  int st = 0;
  for (uint32_t j = 0;; ++j) {
    issue(st == 0 ? 2 : st - 1); // stage (st + 2) % 3
    uint32_t x[16];
    x[0] = q0.x; x[4] = q0.y; x[8] = q0.z; x[12] = q0.w;
    x[1] = q1.x; x[5] = q1.y; x[9] = q1.z; x[13] = q1.w;
    x[2] = q2.x; x[6] = q2.y; x[10] = q2.z; x[14] = q2.w;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    const uint32_t s0 = sd.x, s1 = sd.y, s2 = sd.z;
    if (((j + 1) & (kV6Batch - 1)) == 0) refill();
    {
      const uint4 *ent = table + ((j + 1) & (kV6Batch - 1)) * 4;
      q0 = ent[0]; q1 = ent[1]; q2 = ent[2]; sd = ent[3];
    }
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int r = 1; r < ROUNDS / 2; ++r) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    cp_async_wait<2>(); // this page's group has landed
    const uint4 *mine = &ring[st][tid * 4];
    const uint4 d0 = mine[0 ^ sw], d1 = mine[1 ^ sw], d2 = mine[2 ^ sw], d3 = mine[3 ^ sw];
    st_v4(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                          d0.w ^ (x[3] + kSigma3)));
    st_v4(dst + 1, make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]),
                              d1.w ^ (x[7] + k[3])));
    st_v4(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]),
                              d2.w ^ (x[11] + k[7])));
    st_v4(dst + 3, make_uint4(d3.x ^ (x[12] + s0), d3.y ^ (x[13] + s1), d3.z ^ (x[14] + s2),
                              d3.w ^ (x[15] + b)));
    page += stride;
    if (page >= n_pages) break;
    dst += step;
    st = st == 2 ? 0 : st + 1;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// v9: v5's cp.async page ring fed by a per-page seed table.  A pre-pass
// (k_page_seed_table, one thread per page) computes the three page-only
// quarter rounds of round 1 -- columns 0, 1, 2 start from (sigma_c, k_c,
// k_c+4, word 12+c), i.e. vaddr_lo, vaddr_hi and the pid -- and files them
// with state words 12..14 as one 64-byte record per page.  The page loop
// streams each page's record into its ring stage next to the page bytes
// (lanes 0-3 of each warp, one 16-byte cp.async each) and reads it back with
// four broadcast LDS.128, so it runs no seed round and loads no descriptor:
// only column 3 (the block index) is per thread, and it is hoisted.  Every
// descriptor shape (contiguous, vaddr array, pid array) is the same loop.
// Every block is still exactly ChaCha_R(state) + state.
constexpr int kV9Stages = 4;
constexpr size_t kV9Smem = kV9Stages * (256 * 4 * 16 + 8 * 64); // ring + one record per warp per stage

__global__ void __launch_bounds__(256)
k_page_seed_table(const uint32_t *__restrict__ key, PageDesc desc, uint4 *__restrict__ rec, uint32_t n_pages) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pages) return;
  constexpr RotMul rm{};
  uint32_t k[8];
  load_key(key, k);
  uint64_t va;
  uint32_t pid;
  desc_fetch(desc, p, va, pid);
  const uint32_t lo = static_cast<uint32_t>(va), hi = static_cast<uint32_t>(va >> 32);
  uint32_t a0 = kSigma0, b0 = k[0], c0 = k[4], d0 = lo;
  uint32_t a1 = kSigma1, b1 = k[1], c1 = k[5], d1 = hi;
  uint32_t a2 = kSigma2, b2 = k[2], c2 = k[6], d2 = pid;
  quarter_round<0>(a0, b0, c0, d0, rm);
  quarter_round<0>(a1, b1, c1, d1, rm);
  quarter_round<0>(a2, b2, c2, d2, rm);
  uint4 *r = rec + static_cast<uint64_t>(p) * 4;
  r[0] = make_uint4(a0, b0, c0, d0);
  r[1] = make_uint4(a1, b1, c1, d1);
  r[2] = make_uint4(a2, b2, c2, d2);
  r[3] = make_uint4(lo, hi, pid, 0);
}

// The record of page i+1 is read from shared memory at the end of page i
// (after the wait that page i's bytes need anyway), so the next page's rounds
// start from registers: no shared-memory latency at the top of the loop.
template <int ROUNDS>
__global__ void __launch_bounds__(256, 3)
k_crypt_pages_seeded(const uint32_t *__restrict__ key, const uint4 *__restrict__ rec, const uint4 *in, uint4 *out,
                     uint32_t n_pages) {
  constexpr RotMul rm{};
  constexpr int S = kV9Stages;
  extern __shared__ __align__(128) uint4 v9_smem[];
  uint4 *ring = v9_smem;                    // [stage][256 threads x 4 chunks]
  uint4 *recs = v9_smem + S * 256 * 4;      // [stage][8 warps x 4 chunks]
  const uint32_t tid = threadIdx.x;
  const uint32_t b = tid & 63, lane = tid & 31, warp = tid >> 5;
  const uint32_t sw = (tid >> 1) & 3;
  const uint32_t stride = gridDim.x * 4;
  uint32_t page = blockIdx.x * 4 + (tid >> 6);
  if (page >= n_pages) return;
  constexpr uint32_t kStageBytes = 256 * 4 * 16, kRecStage = 8 * 64;
  const uint32_t base0 = smem_u32(ring + tid * 4);
  const uint32_t rbase0 = smem_u32(recs + warp * 4 + (lane & 3));
  const uint64_t step = static_cast<uint64_t>(stride) * 256;
  const uint4 *src_ahead = in + static_cast<uint64_t>(page) * 256 + b * 4;
  const uint4 *rec_ahead = rec + static_cast<uint64_t>(page) * 4 + (lane & 3);
  uint4 *dst = out + static_cast<uint64_t>(page) * 256 + b * 4;
  uint32_t page_ahead = page;
  auto issue = [&](int st) { // next page (bytes + record) for the ring, then advance
    if (page_ahead < n_pages) {
      const uint32_t sdst = base0 + st * kStageBytes;
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async16(sdst + 16 * (c ^ sw), src_ahead + c);
      if (lane < 4) cp_async16(rbase0 + st * kRecStage, rec_ahead);
    }
    cp_async_commit();
    page_ahead += stride;
    src_ahead += step;
    rec_ahead += static_cast<uint64_t>(stride) * 4;
  };
#pragma unroll
  for (int i = 0; i < S - 1; ++i) issue(i);
  uint32_t k[8];
  load_key(key, k);
  uint32_t c3a = kSigma3, c3b = k[3], c3c = k[7], c3d = b;
  quarter_round<0>(c3a, c3b, c3c, c3d, rm);
  cp_async_wait<S - 2>(); // page 0's group
  __syncwarp();
  uint4 r0 = recs[warp * 4], r1 = recs[warp * 4 + 1], r2 = recs[warp * 4 + 2], r3 = recs[warp * 4 + 3];
  int st = 0;
  for (;;) {
    __syncwarp(); // every lane is past its reads of the stage the next issue overwrites
    issue(st == 0 ? S - 1 : st - 1); // stage (st + S - 1) % S
    uint32_t x[16];
    x[0] = r0.x; x[4] = r0.y; x[8] = r0.z; x[12] = r0.w;
    x[1] = r1.x; x[5] = r1.y; x[9] = r1.z; x[13] = r1.w;
    x[2] = r2.x; x[6] = r2.y; x[10] = r2.z; x[14] = r2.w;
    x[3] = c3a; x[7] = c3b; x[11] = c3c; x[15] = c3d;
    const uint32_t s0 = r3.x, s1 = r3.y, s2 = r3.z;
    diagonal_round<0>(x, rm);
#pragma unroll
    for (int i = 1; i < ROUNDS / 2; ++i) {
      column_round<0>(x, rm);
      diagonal_round<0>(x, rm);
    }
    cp_async_wait<S - 2>(); // the next page's group has landed (and this page's)
    __syncwarp();           // lanes 0-3's record copies are visible to the warp
    const int nst = st == S - 1 ? 0 : st + 1;
    const uint4 *rn = recs + nst * 32 + warp * 4;
    r0 = rn[0]; r1 = rn[1]; r2 = rn[2]; r3 = rn[3];
    const uint4 *mine = ring + st * 1024 + tid * 4;
    const uint4 d0 = mine[0 ^ sw], d1 = mine[1 ^ sw], d2 = mine[2 ^ sw], d3 = mine[3 ^ sw];
    st_v4(dst, make_uint4(d0.x ^ (x[0] + kSigma0), d0.y ^ (x[1] + kSigma1), d0.z ^ (x[2] + kSigma2),
                          d0.w ^ (x[3] + kSigma3)));
    st_v4(dst + 1, make_uint4(d1.x ^ (x[4] + k[0]), d1.y ^ (x[5] + k[1]), d1.z ^ (x[6] + k[2]),
                              d1.w ^ (x[7] + k[3])));
    st_v4(dst + 2, make_uint4(d2.x ^ (x[8] + k[4]), d2.y ^ (x[9] + k[5]), d2.z ^ (x[10] + k[6]),
                              d2.w ^ (x[11] + k[7])));
    st_v4(dst + 3, make_uint4(d3.x ^ (x[12] + s0), d3.y ^ (x[13] + s1), d3.z ^ (x[14] + s2),
                              d3.w ^ (x[15] + b)));
    page += stride;
    if (page >= n_pages) break;
    dst += step;
    st = nst;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Slab moves for the HBM page store: page i of a staging batch <-> slot
// slots[i] of a device slab, optionally through the cipher (key != nullptr).
// DIR 0: staging -> slab (evict/insert), DIR 1: slab -> staging (refault/lookup).
// One thread per 64-byte block, like v1; these moves are PCIe-bound.
template <int ROUNDS, int DIR>
__global__ void __launch_bounds__(256)
k_slab_move(const uint32_t *__restrict__ key, PageDesc desc, const uint32_t *__restrict__ slots,
            uint4 *slab, uint4 *staging, uint64_t n_blocks, bool wipe_src) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_blocks) return;
  const uint64_t page = g >> 6;
  const uint32_t blk = static_cast<uint32_t>(g & 63);
  uint4 *sp = slab + static_cast<uint64_t>(__ldg(slots + page)) * 256 + blk * 4;
  uint4 *tp = staging + g * 4;
  const uint4 *src = DIR == 0 ? tp : sp;
  uint4 *dst = DIR == 0 ? sp : tp;
  uint4 d0 = ld_v4(src), d1 = ld_v4(src + 1), d2 = ld_v4(src + 2), d3 = ld_v4(src + 3);
  if (DIR == 1 && wipe_src) { // refault: the slot is freed, zero it on the way out
    const uint4 z = make_uint4(0, 0, 0, 0);
    st_v4(sp, z); st_v4(sp + 1, z); st_v4(sp + 2, z); st_v4(sp + 3, z);
  }
  if (key) {
    uint32_t k[8], s[4], x[16];
    load_key(key, k);
    page_seed(desc, page, s);
    s[3] = blk;
    chacha_block<ROUNDS, 0>(x, k, s, RotMul{});
    d0.x ^= x[0];  d0.y ^= x[1];  d0.z ^= x[2];  d0.w ^= x[3];
    d1.x ^= x[4];  d1.y ^= x[5];  d1.z ^= x[6];  d1.w ^= x[7];
    d2.x ^= x[8];  d2.y ^= x[9];  d2.z ^= x[10]; d2.w ^= x[11];
    d3.x ^= x[12]; d3.y ^= x[13]; d3.z ^= x[14]; d3.w ^= x[15];
  }
  st_v4(dst, d0); st_v4(dst + 1, d1); st_v4(dst + 2, d2); st_v4(dst + 3, d3);
}

// Fused refault + evict for one fault (pc_store_swap): pages [0, n_get) of
// the batch move slab -> staging through the cipher and their slots are
// zeroed (a refault, orchestrator.py:190-198); pages [n_get, n) move
// staging -> slab through the cipher (an eviction, orchestrator.py:230-238).
// The two slot sets are disjoint (the store pops the eviction slots before
// it frees the refault slots), so one launch does both.
template <int ROUNDS>
__global__ void __launch_bounds__(256)
k_slab_swap(const uint32_t *__restrict__ key, PageDesc desc, const uint32_t *__restrict__ slots,
            uint4 *slab, uint4 *staging, uint32_t n_get, uint64_t n_blocks) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_blocks) return;
  const uint64_t page = g >> 6;
  const uint32_t blk = static_cast<uint32_t>(g & 63);
  const bool get = page < n_get;
  uint4 *sp = slab + static_cast<uint64_t>(__ldg(slots + page)) * 256 + blk * 4;
  uint4 *tp = staging + g * 4;
  const uint4 *src = get ? sp : tp;
  uint4 *dst = get ? tp : sp;
  uint4 d0 = ld_v4(src), d1 = ld_v4(src + 1), d2 = ld_v4(src + 2), d3 = ld_v4(src + 3);
  if (get) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    st_v4(sp, z); st_v4(sp + 1, z); st_v4(sp + 2, z); st_v4(sp + 3, z);
  }
  uint32_t k[8], s[4], x[16];
  load_key(key, k);
  page_seed(desc, page, s);
  s[3] = blk;
  chacha_block<ROUNDS, 0>(x, k, s, RotMul{});
  d0.x ^= x[0];  d0.y ^= x[1];  d0.z ^= x[2];  d0.w ^= x[3];
  d1.x ^= x[4];  d1.y ^= x[5];  d1.z ^= x[6];  d1.w ^= x[7];
  d2.x ^= x[8];  d2.y ^= x[9];  d2.z ^= x[10]; d2.w ^= x[11];
  d3.x ^= x[12]; d3.y ^= x[13]; d3.z ^= x[14]; d3.w ^= x[15];
  st_v4(dst, d0); st_v4(dst + 1, d1); st_v4(dst + 2, d2); st_v4(dst + 3, d3);
}

// Descriptor validation on the device (crypt_pages' checks): flags bit 0 =
// some vaddr is not page-aligned, bit 1 = some 64-bit pid is outside u32;
// 64-bit pids are narrowed into pids32.  A library kernel (preloaded), so the
// checks never launch a foreign kernel beside the persistent worker service.
__global__ void __launch_bounds__(256)
k_desc_check(const uint64_t *__restrict__ vaddrs, const int64_t *__restrict__ pids64, uint32_t *pids32, uint64_t n,
             uint32_t *flags) {
  uint32_t f = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (vaddrs && (__ldg(vaddrs + i) & 4095u)) f |= 1u;
    if (pids64) {
      const int64_t p = __ldg(pids64 + i);
      if (p < 0 || p > 0xFFFFFFFFll) f |= 2u;
      pids32[i] = static_cast<uint32_t>(p);
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

// Zero the given slab slots (freed store entries are wiped, store.py:86-92).
__global__ void __launch_bounds__(256)
k_slab_wipe(const uint32_t *__restrict__ slots, uint4 *slab, uint64_t n_chunks) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_chunks) return;
  slab[static_cast<uint64_t>(__ldg(slots + (g >> 8))) * 256 + (g & 255)] = make_uint4(0, 0, 0, 0);
}

// ---------------------------------------------------------------------------
// Keystream only, arbitrary seeds: seeds[4*i .. 4*i+3] are state words 12..15
// of block i; out[16*i ..] its 16 keystream words (block-major, like
// _chacha_numba.keystream_words, _chacha_numba.py:45-50).
template <int ROUNDS>
__global__ void __launch_bounds__(128)
k_keystream_seeds(const uint32_t *__restrict__ key, const uint32_t *__restrict__ seeds,
                  uint64_t n, uint32_t *__restrict__ out) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t k[8], s[4], x[16];
  load_key(key, k);
  const uint4 sv = __ldg(reinterpret_cast<const uint4 *>(seeds) + i);
  s[0] = sv.x; s[1] = sv.y; s[2] = sv.z; s[3] = sv.w;
  chacha_block<ROUNDS, 0>(x, k, s, RotMul{});
  uint4 *o = reinterpret_cast<uint4 *>(out) + i * 4;
  o[0] = make_uint4(x[0], x[1], x[2], x[3]);
  o[1] = make_uint4(x[4], x[5], x[6], x[7]);
  o[2] = make_uint4(x[8], x[9], x[10], x[11]);
  o[3] = make_uint4(x[12], x[13], x[14], x[15]);
}

// ---------------------------------------------------------------------------
// Device-side key derivation: key = first 8 words of ChaCha20(entropy,
// device timer/clock/SM words).  The caller's entropy alone does not determine
// the key, and the derived key only ever exists in device memory.
__global__ void k_keygen(const uint32_t *__restrict__ entropy, uint32_t *__restrict__ key_out) {
  uint32_t k[8], s[4], x[16];
  load_key(entropy, k);
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const uint64_t c = clock64();
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  s[0] = static_cast<uint32_t>(t); s[1] = static_cast<uint32_t>(t >> 32);
  s[2] = static_cast<uint32_t>(c) ^ (smid << 24); s[3] = static_cast<uint32_t>(c >> 32);
  chacha_block<20, 0>(x, k, s, RotMul{});
#pragma unroll
  for (int i = 0; i < 8; ++i) key_out[i] = x[i];
}

// ---------------------------------------------------------------------------
// Integer-pipe microbenchmarks (roofline denominators, pc_intpeak).  Eight
// independent chains per thread so issue, not latency, bounds them.
//   0 LOP3   1 IADD (ptxas fuses pairs into IADD3)   2 IMAD   3 SHF rotate
//   4 ChaCha quarter rounds as ptxas schedules them (adds on IMAD)
//   5 quarter rounds with the rotate by 7 on the FMA pipe (ROTMASK nibble 8)
//   6 IMAD.HI   7 IMAD.WIDE
template <int KIND>
__global__ void __launch_bounds__(256)
k_intpeak(uint32_t seed, RotMul rm, int iters, uint32_t *sink) {
  uint32_t v[8], w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { v[j] = seed ^ (threadIdx.x * 0x9e3779b9u + j); w[j] = v[j] * 3u + j; }
  for (int it = 0; it < iters; ++it) {
    if constexpr (KIND <= 3 || KIND >= 6) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if constexpr (KIND == 0) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[j]) : "r"(w[j]), "r"(v[(j + 1) & 7]));
          } else if constexpr (KIND == 1) {
            asm volatile("add.u32 %0, %0, %1;" : "+r"(v[j]) : "r"(w[j]));
          } else if constexpr (KIND == 2) {
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[j]) : "r"(rm.m16), "r"(w[j]));
          } else if constexpr (KIND == 3) {
            asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(v[j]));
          } else if constexpr (KIND == 6) {
            asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[j]) : "r"(rm.m12), "r"(w[j]));
          } else {
            uint64_t p;
            asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(v[j]), "r"(rm.m12));
            v[j] = static_cast<uint32_t>(p) ^ static_cast<uint32_t>(p >> 32);
          }
        }
      }
    } else {
      // two independent ChaCha states per thread (v, w), 16 quarter rounds
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        constexpr uint32_t N = KIND == 4 ? 0u : 8u;
        quarter_round<N>(v[0], v[1], v[2], v[3], rm);
        quarter_round<N>(v[4], v[5], v[6], v[7], rm);
        quarter_round<N>(w[0], w[1], w[2], w[3], rm);
        quarter_round<N>(w[4], w[5], w[6], w[7], rm);
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc ^= v[j] ^ w[j];
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
}

} // namespace pc
