// kernels.cuh -- sm_100a kernels of the page-cipher engine.
//
// Data layout in HBM: a batch is n pages of 4096 bytes, page-major and
// contiguous (uint8[n][4096]); page p's descriptors are vaddrs[p] (u64) and
// pids[p] (u32) or the contiguous/scalar forms (PageDesc).  Block b of page p
// is bytes [64b, 64b+64) of the page (pkg/src/pagecrypt/cipher.py:197-217).
#pragma once
#include <cstdint>

#include "chacha.cuh"

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

__device__ __forceinline__ void load_key(const uint32_t *__restrict__ key, uint32_t (&k)[8]) {
  const uint4 a = __ldg(reinterpret_cast<const uint4 *>(key));
  const uint4 b = __ldg(reinterpret_cast<const uint4 *>(key) + 1);
  k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
  k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
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
template <int ROUNDS, int AM>
__global__ void __launch_bounds__(256)
k_crypt_blocks(const uint32_t *__restrict__ key, PageDesc desc, const uint4 *in, uint4 *out,
               uint64_t n_blocks, uint32_t one) {
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_blocks) return;
  uint32_t k[8], s[4];
  load_key(key, k);
  page_seed(desc, g >> 6, s);
  s[3] = static_cast<uint32_t>(g & 63); // word 15 = block index
  const uint4 *src = in + g * 4;
  uint4 d0 = ld_v4(src), d1 = ld_v4(src + 1), d2 = ld_v4(src + 2), d3 = ld_v4(src + 3);
  uint32_t x[16];
  chacha_block<ROUNDS, AM>(x, k, s, one);
  d0.x ^= x[0];  d0.y ^= x[1];  d0.z ^= x[2];  d0.w ^= x[3];
  d1.x ^= x[4];  d1.y ^= x[5];  d1.z ^= x[6];  d1.w ^= x[7];
  d2.x ^= x[8];  d2.y ^= x[9];  d2.z ^= x[10]; d2.w ^= x[11];
  d3.x ^= x[12]; d3.y ^= x[13]; d3.z ^= x[14]; d3.w ^= x[15];
  uint4 *dst = out + g * 4;
  st_v4(dst, d0); st_v4(dst + 1, d1); st_v4(dst + 2, d2); st_v4(dst + 3, d3);
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
  chacha_block<ROUNDS, kAddAlu>(x, k, s, 1u);
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
  chacha_block<20, kAddAlu>(x, k, s, 1u);
#pragma unroll
  for (int i = 0; i < 8; ++i) key_out[i] = x[i];
}

// ---------------------------------------------------------------------------
// Integer-pipe microbenchmarks (roofline denominators, pc_intpeak).  Eight
// independent chains per thread so issue, not latency, bounds them.
template <int KIND>
__global__ void __launch_bounds__(256)
k_intpeak(uint32_t seed, uint32_t one, int iters, uint32_t *sink) {
  uint32_t v[8], w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { v[j] = seed ^ (threadIdx.x * 0x9e3779b9u + j); w[j] = v[j] * 3u + j; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (KIND == 0) { // LOP3
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[j]) : "r"(w[j]), "r"(v[(j + 1) & 7]));
        } else if constexpr (KIND == 1) { // IADD
          asm volatile("add.u32 %0, %0, %1;" : "+r"(v[j]) : "r"(w[j]));
        } else if constexpr (KIND == 2) { // IMAD
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[j]) : "r"(one), "r"(w[j]));
        } else if constexpr (KIND == 3) { // SHF rotate
          asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(v[j]));
        }
      }
    }
    if constexpr (KIND == 4 || KIND == 5) {
      // ChaCha ARX: two independent quarter-round states per thread.
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        quarter_round<KIND == 4 ? kAddAlu : kAddSplitA>(v[0], v[1], v[2], v[3], one);
        quarter_round<KIND == 4 ? kAddAlu : kAddSplitA>(v[4], v[5], v[6], v[7], one);
        quarter_round<KIND == 4 ? kAddAlu : kAddSplitA>(w[0], w[1], w[2], w[3], one);
        quarter_round<KIND == 4 ? kAddAlu : kAddSplitA>(w[4], w[5], w[6], w[7], one);
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc ^= v[j] ^ w[j];
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
}

} // namespace pc
