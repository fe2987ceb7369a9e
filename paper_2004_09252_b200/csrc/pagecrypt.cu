// pagecrypt.cu -- host side of libpagecrypt.so: the C ABI in include/pagecrypt.h.
//
// Replaces the reference's two in-process seams:
//   kernel seam  pkg/src/pagecrypt/_chacha_numba.py:44-93  -> pc_keystream_words
//   API seam     pkg/src/pagecrypt/cipher.py:188-249       -> pc_crypt_pages_{dev,host}
// and the host side of the crypto worker service
// (pkg/src/pagecrypt/workers.py: key slots :168,174-202,240-254; routing
// :204-206 -> the page-range partitioner pc_crypt_pages_multi).
#include <cuda_runtime.h>
#include <immintrin.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <memory>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <shared_mutex>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pagecrypt.h"
#include "kernels.cuh"
#include "service.cuh"
#include "hostpool.hpp"

namespace {

thread_local std::string g_err = "";

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(e_ == cudaErrorMemoryAllocation ? PC_ENOMEM : PC_ECUDA, "%s: %s (%s:%d)",  \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                        \
  } while (0)

// Volatile wipe the compiler cannot elide (key material in host memory).
void wipe(void *p, size_t n) {
  volatile uint8_t *v = static_cast<volatile uint8_t *>(p);
  for (size_t i = 0; i < n; ++i) v[i] = 0;
}

struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) {
      err = cudaSetDevice(dev);
      changed = (err == cudaSuccess);
    }
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

bool valid_rounds(int r) { return r == 8 || r == 12 || r == 20; }

int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

#ifndef PC_RUN_MAX_R
#define PC_RUN_MAX_R 12
#endif
// Tuning knobs (env defaults at first use, pc_tune() at run time).
struct Tuning {
  std::atomic<uint32_t> rot_mask{0};   // ROTMASK of the crypt kernel (one of kRotMasks)
  std::atomic<int> small_mode{1};      // 0 = staged copies, 1 = zero-copy on mapped pinned memory
  std::atomic<size_t> small_max{64};   // host batches up to this many pages take the small path
  std::atomic<int> run_desc{1};
  std::atomic<int> svc_bell_ops{1};    // a store's service: its tickets' slots ride in the doorbell line
                                       // (0 = the workers read every op line: tests the fallback)        // v5 with descriptor arrays at R <= 12: contiguous runs per slot
  std::atomic<int64_t> svc_pages{0};   // host batches up to this many pages go to the key's resident
                                       // workers when it has them (pc_key_service); 0 = 1 per worker, <= 6
  std::atomic<int> kernel{0};          // HBM kernel: 0 = auto (per rounds, below), 1 = k_crypt_blocks,
                                       // 2 = k_crypt_pages, 3 = k_crypt_pages_coalesced,
                                       // 4 = k_crypt_pages_tma, 5 = k_crypt_pages_async,
                                       // 6 = k_crypt_pages_warp
  std::atomic<int> host_mode{2};       // large host batches: 0 = round-robin streams, 1 = zero-copy kernel
                                       // (pinned I/O only), 2 = dedicated H2D/compute/D2H streams,
                                       // 3 = as 2 but the kernel writes pinned output directly
  std::atomic<int> ctas_per_sm{0};     // k_crypt_pages residency; 0 = occupancy calculator
  std::atomic<int> dev_direct{1};      // device pages on the engine's own GPU: 1 = one in-place launch,
                                       // 0 = stage through the engine's slots (tests the peer path on 1 GPU)
  std::atomic<int> svc_direct{2};      // worker service: 1 = each worker polls its own doorbell in host
                                       // memory, 0 = one dispatcher CTA forwards doorbells to device
                                       // memory, 2 = auto (direct up to 32 workers)
  std::atomic<int> peer_direct{1};     // device pages on a peer GPU: 1 = kernel works on them in place over
                                       // NVLink when peer access is available, 0 = peer copies via staging
  Tuning() {
    kernel = env_int("PAGECRYPT_KERNEL", 0);
    host_mode = env_int("PAGECRYPT_HOST_MODE", 2);
    ctas_per_sm = env_int("PAGECRYPT_CTAS_PER_SM", 0);
    run_desc = env_int("PAGECRYPT_RUN_DESC", 1);
    svc_bell_ops = env_int("PAGECRYPT_SVC_BELL_OPS", 1);
    if (const char *v = std::getenv("PAGECRYPT_ROTMASK")) rot_mask = static_cast<uint32_t>(std::strtoul(v, nullptr, 0));
    small_mode = env_int("PAGECRYPT_SMALL_MODE", 1);
    small_max = static_cast<size_t>(env_int("PAGECRYPT_SMALL_MAX", 64));
    svc_direct = env_int("PAGECRYPT_SVC_DIRECT", 2);
  }
};
// Kernel launches issued by this library (all kernels, all devices), read
// through pc_tune_get("launches"): bench.py reports the launches inside its
// timed regions from it.
std::atomic<uint64_t> g_launches{0};
inline void counted(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Helper threads for pageable <-> pinned bounce copies (the caller's thread
// works too): PAGECRYPT_HOST_THREADS, default min(7, cores/2).
unsigned host_pool_threads() {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int env = env_int("PAGECRYPT_HOST_THREADS", -1);
  if (env >= 0) return static_cast<unsigned>(std::min(env, 256));
  return std::min(7u, hw > 1 ? hw / 2 : 0u);
}

Tuning &tuning() {
  static Tuning t;
  return t;
}

// Compiled ROTMASK variants of k_crypt_blocks (chacha.cuh): FMA-pipe rotates
// per double round.  Measured on B200 (profiles/r01_rotmask_sweep.txt): no
// variant beats 0 -- IMAD.HI is half rate and adds dispatch stalls -- so 0 is
// the default and the others stay for the record.
constexpr uint32_t kRotMasks[] = {0x00000000u, 0x88888888u, 0x888888AAu, 0x88888AAAu,
                                  0xAAAA8888u, 0xAAAAAAAAu};

constexpr pc::RotMul kRotMul{1u << 16, 1u << 12, 1u << 8, 1u << 7};

template <int R, uint32_t M>
void launch_crypt_rm(const uint32_t *key, const pc::PageDesc &d, const void *in, void *out,
                     uint64_t n_blocks, cudaStream_t st) {
  const dim3 block(256);
  const dim3 grid(static_cast<unsigned>((n_blocks + 255) / 256));
  pc::k_crypt_blocks<R, M><<<grid, block, 0, st>>>(key, d, static_cast<const uint4 *>(in),
                                                   static_cast<uint4 *>(out), n_blocks, kRotMul);
  counted();
}

template <int R>
void launch_crypt_r(uint32_t mask, const uint32_t *key, const pc::PageDesc &d, const void *in,
                    void *out, uint64_t n_blocks, cudaStream_t st) {
  switch (mask) {
    case 0x88888888u: launch_crypt_rm<R, 0x88888888u>(key, d, in, out, n_blocks, st); break;
    case 0x888888AAu: launch_crypt_rm<R, 0x888888AAu>(key, d, in, out, n_blocks, st); break;
    case 0x88888AAAu: launch_crypt_rm<R, 0x88888AAAu>(key, d, in, out, n_blocks, st); break;
    case 0xAAAA8888u: launch_crypt_rm<R, 0xAAAA8888u>(key, d, in, out, n_blocks, st); break;
    case 0xAAAAAAAAu: launch_crypt_rm<R, 0xAAAAAAAAu>(key, d, in, out, n_blocks, st); break;
    default: launch_crypt_rm<R, 0u>(key, d, in, out, n_blocks, st); break;
  }
}

// Per-device launch geometry, computed once and published as ONE atomic word
// (SM count << 16 | resident CTAs per SM): a concurrent first caller once read
// the SM count set and the occupancy still 0 -> grid 0 -> "invalid
// configuration argument" (found by tools/soak.py).  Racing first callers
// compute the same value; the hot path is one acquire load.
template <typename Init> // Init(int &n_sm, int &occ) -> cudaError_t
cudaError_t cached_geometry(std::atomic<uint32_t> (&cache)[64], int dev, int &n_sm, int &occ, Init init) {
  uint32_t g = cache[dev & 63].load(std::memory_order_acquire);
  if (!g) {
    int s = 0, o = 0;
    const cudaError_t e = init(s, o);
    if (e != cudaSuccess) return e;
    g = (static_cast<uint32_t>(s) << 16) | static_cast<uint32_t>(o > 0 ? o : 1);
    cache[dev & 63].store(g, std::memory_order_release);
  }
  n_sm = static_cast<int>(g >> 16);
  occ = static_cast<int>(g & 0xFFFF);
  return cudaSuccess;
}

// Persistent grid for k_crypt_pages: SMs x resident CTAs (occupancy), capped
// by the number of 4-page slots.
// v6 needs more than the 48 KiB static limit of dynamic shared memory: opt
// each instantiation in once per device.
template <int R, int DM>
cudaError_t v6_opt_in() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(pc::k_crypt_pages_warp<R, DM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(pc::kV6Smem));
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <int R>
cudaError_t v9_opt_in() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(pc::k_crypt_pages_seeded<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(pc::kV9Smem));
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// Stream-ordered scratch for v9's per-page seed records (64 B per page): a
// private memory pool per device that keeps its memory (release threshold
// max), so a launch's allocation is a pool hit, not a cudaMalloc.
cudaMemPool_t seed_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t p = nullptr;
  if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
  pools[dev] = p;
  return p;
}

template <int R, int Variant> // 0 = v2, 1 = v3 coalesced, 2 = v5 cp.async, 3 = v6 warp-shared seeds, 4 = v9 seeded,
                              // 5 = v5r2 (128-thread CTAs: the grid is in CTAs of 4 warp slots)
unsigned pages_grid(size_t n_pages) {
  static std::atomic<uint32_t> geo[64] = {};
  int dev = 0, n_sm = 0, occ = 0;
  cudaGetDevice(&dev);
  if (cached_geometry(geo, dev, n_sm, occ, [dev](int &s, int &o) {
        cudaError_t e = cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        if constexpr (Variant == 1)
          return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pc::k_crypt_pages_coalesced<R>, 256, 0);
        else if constexpr (Variant == 2)
          return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pc::k_crypt_pages_async<R, 0>, 256, 0);
        else if constexpr (Variant == 3) {
          cudaError_t e2 = v6_opt_in<R, 0>();
          if (e2 != cudaSuccess) return e2;
          return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pc::k_crypt_pages_warp<R, 0>, 256, pc::kV6Smem);
        }
        else if constexpr (Variant == 5)
          return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pc::k_crypt_pages_run2<R, 3>, 128, 0);
        else if constexpr (Variant == 4) {
          cudaError_t e2 = v9_opt_in<R>();
          if (e2 != cudaSuccess) return e2;
          return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pc::k_crypt_pages_seeded<R>, 256, pc::kV9Smem);
        }
        else
          return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pc::k_crypt_pages<R>, 256, 0);
      }) != cudaSuccess)
    return 0; // the launch then fails loudly ("invalid configuration")
  // v5 at ChaCha12 runs best below its 4 resident CTAs per SM: round 1, 2
  // CTAs: 2835 vs 2774 GB/s (profiles/r01_ctas_ab.txt) -- fewer concurrent
  // page streams, same ALU feed (ILP 4 per thread); with the 256-bit stores
  // (round 2) 3 CTAs: 2853 vs 2845 contiguous, 2747-2751 vs 2692-2746 with
  // descriptor arrays (profiles/r02_ctas_r12.txt)
  const int dflt = ((Variant == 2 || Variant == 3 || Variant == 4) && R == 12) ? std::min(occ, 3) : occ;
  const int per_sm = tuning().ctas_per_sm.load() > 0 ? tuning().ctas_per_sm.load() : dflt;
  const uint64_t want = static_cast<uint64_t>(n_sm) * per_sm;
  const uint64_t slots = (n_pages + 3) / 4;
  return static_cast<unsigned>(std::min<uint64_t>(want, slots));
}

template <int R>
void launch_pages_r(int kern, const uint32_t *key, const pc::PageDesc &d, const void *in,
                    void *out, size_t n_pages, cudaStream_t st) {
  auto i4 = static_cast<const uint4 *>(in);
  auto o4 = static_cast<uint4 *>(out);
  if (kern == 3) {
    pc::k_crypt_pages_coalesced<R><<<pages_grid<R, 1>(n_pages), 256, 0, st>>>(key, d, i4, o4, n_pages);
    counted();
  } else if (kern == 5) {
    // 32-bit page loop: split batches at 2^30 pages (4 TiB)
    constexpr size_t kMax = size_t(1) << 30;
    for (size_t p0 = 0; p0 < n_pages; p0 += kMax) {
      const uint32_t m = static_cast<uint32_t>(std::min(kMax, n_pages - p0));
      pc::PageDesc dd{d.vaddrs ? d.vaddrs + p0 : nullptr, d.pids ? d.pids + p0 : nullptr,
                      d.vaddr0 + 4096ull * p0, d.pid0};
      const unsigned grid = pages_grid<R, 2>(m);
      const auto a = i4 + p0 * 256;
      const auto b = o4 + p0 * 256;
      const int dm = (dd.vaddrs ? 1 : 0) | (dd.pids ? 2 : 0);
      const int rd = tuning().run_desc.load();
      if (dm && rd == 2 &&
          (reinterpret_cast<uintptr_t>(dd.vaddrs) & 15) == 0 && (reinterpret_cast<uintptr_t>(dd.pids) & 7) == 0) {
        // one warp per page slot, two blocks per thread
        const unsigned g2 = pages_grid<R, 5>(m);
        if (g2) {
          const uint64_t slots = uint64_t(g2) * 4;
          const uint32_t run = static_cast<uint32_t>((((m + slots - 1) / slots) + 1) & ~uint64_t(1));
          const unsigned g = static_cast<unsigned>((m + uint64_t(run) * 4 - 1) / (uint64_t(run) * 4));
          switch (dm) {
            case 1: pc::k_crypt_pages_run2<R, 1><<<g, 128, 0, st>>>(key, dd, a, b, m, run); break;
            case 2: pc::k_crypt_pages_run2<R, 2><<<g, 128, 0, st>>>(key, dd, a, b, m, run); break;
            default: pc::k_crypt_pages_run2<R, 3><<<g, 128, 0, st>>>(key, dd, a, b, m, run); break;
          }
          counted();
          continue;
        }
      }
      if constexpr (R <= PC_RUN_MAX_R) {
        // descriptor arrays at ChaCha8/12: contiguous page runs per slot, so a
        // page pair's descriptors are one 16-byte and one 8-byte load
        if (dm && rd && grid &&
            (reinterpret_cast<uintptr_t>(dd.vaddrs) & 15) == 0 && (reinterpret_cast<uintptr_t>(dd.pids) & 7) == 0) {
          const uint64_t slots = uint64_t(grid) * 4;
          const uint32_t run = static_cast<uint32_t>((((m + slots - 1) / slots) + 1) & ~uint64_t(1));
          const unsigned g = static_cast<unsigned>((m + uint64_t(run) * 4 - 1) / (uint64_t(run) * 4));
          switch (dm) {
            case 1: pc::k_crypt_pages_run<R, 1><<<g, 256, 0, st>>>(key, dd, a, b, m, run); break;
            case 2: pc::k_crypt_pages_run<R, 2><<<g, 256, 0, st>>>(key, dd, a, b, m, run); break;
            default: pc::k_crypt_pages_run<R, 3><<<g, 256, 0, st>>>(key, dd, a, b, m, run); break;
          }
          counted();
          continue;
        }
      }
      switch (dm) {
        case 0: pc::k_crypt_pages_async<R, 0><<<grid, 256, 0, st>>>(key, dd, a, b, m); break;
        case 1: pc::k_crypt_pages_async<R, 1><<<grid, 256, 0, st>>>(key, dd, a, b, m); break;
        case 2: pc::k_crypt_pages_async<R, 2><<<grid, 256, 0, st>>>(key, dd, a, b, m); break;
        default: pc::k_crypt_pages_async<R, 3><<<grid, 256, 0, st>>>(key, dd, a, b, m); break;
      }
      counted();
    }
  }
  else if (kern == 9) {
    constexpr size_t kMax = size_t(1) << 30;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = seed_pool(dev);
    v9_opt_in<R>();
    for (size_t p0 = 0; p0 < n_pages; p0 += kMax) {
      const uint32_t m = static_cast<uint32_t>(std::min(kMax, n_pages - p0));
      pc::PageDesc dd{d.vaddrs ? d.vaddrs + p0 : nullptr, d.pids ? d.pids + p0 : nullptr,
                      d.vaddr0 + 4096ull * p0, d.pid0};
      uint4 *rec = nullptr;
      if (!pool || cudaMallocFromPoolAsync(reinterpret_cast<void **>(&rec), size_t(m) * 64, pool, st) != cudaSuccess)
        return; // the caller's cudaGetLastError reports it
      pc::k_page_seed_table<<<(m + 255) / 256, 256, 0, st>>>(key, dd, rec, m);
      counted();
      pc::k_crypt_pages_seeded<R><<<pages_grid<R, 4>(m), 256, pc::kV9Smem, st>>>(key, rec, i4 + p0 * 256,
                                                                                  o4 + p0 * 256, m);
      counted();
      cudaFreeAsync(rec, st);
    }
  }
  else if (kern == 6) {
    constexpr size_t kMax = size_t(1) << 30;
    for (size_t p0 = 0; p0 < n_pages; p0 += kMax) {
      const uint32_t m = static_cast<uint32_t>(std::min(kMax, n_pages - p0));
      pc::PageDesc dd{d.vaddrs ? d.vaddrs + p0 : nullptr, d.pids ? d.pids + p0 : nullptr,
                      d.vaddr0 + 4096ull * p0, d.pid0};
      const unsigned grid = pages_grid<R, 3>(m);
      const auto a = i4 + p0 * 256;
      const auto b = o4 + p0 * 256;
      constexpr size_t sm = pc::kV6Smem;
      switch ((dd.vaddrs ? 1 : 0) | (dd.pids ? 2 : 0)) {
        case 0: v6_opt_in<R, 0>(); pc::k_crypt_pages_warp<R, 0><<<grid, 256, sm, st>>>(key, dd, a, b, m); break;
        case 1: v6_opt_in<R, 1>(); pc::k_crypt_pages_warp<R, 1><<<grid, 256, sm, st>>>(key, dd, a, b, m); break;
        case 2: v6_opt_in<R, 2>(); pc::k_crypt_pages_warp<R, 2><<<grid, 256, sm, st>>>(key, dd, a, b, m); break;
        default: v6_opt_in<R, 3>(); pc::k_crypt_pages_warp<R, 3><<<grid, 256, sm, st>>>(key, dd, a, b, m); break;
      }
      counted();
    }
  }
  else {
    pc::k_crypt_pages<R><<<pages_grid<R, 0>(n_pages), 256, 0, st>>>(key, d, i4, o4, n_pages);
    counted();
  }
}

// ---- v4: TMA pipeline --------------------------------------------------------
constexpr int kTmaStages = 4;
constexpr size_t kTmaSmem = 4 * kTmaStages * pc::kPageBytes + 1024; // 4 slots + 1 KiB alignment slack

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 2D view of n_pages pages: 128-byte rows, 32 per page; 128x128-byte boxes.
int page_tensor_map(CUtensorMap *m, const void *base, uint64_t n_pages) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(PC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {128, n_pages * 32};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, static_cast<cuuint32_t>(pc::kPageRows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return PC_OK;
}

template <int R>
int launch_tma_r(const uint32_t *key, const pc::PageDesc &d, const void *in, void *out, size_t n_pages,
                 cudaStream_t st) {
  static std::atomic<uint32_t> geo[64] = {};
  int dev = 0, n_sm = 0, occ = 0;
  CU(cudaGetDevice(&dev));
  auto kfn = pc::k_crypt_pages_tma<R, kTmaStages>;
  CU(cached_geometry(geo, dev, n_sm, occ, [dev, kfn](int &s, int &o) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTmaSmem));
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kfn, 256, kTmaSmem);
    return e;
  }));
  // TMA row coordinates are int32: split batches above 2^25 pages
  constexpr size_t kMaxPages = size_t(1) << 25;
  for (size_t p0 = 0; p0 < n_pages; p0 += kMaxPages) {
    const size_t m = std::min(kMaxPages, n_pages - p0);
    CUtensorMap tin, tout;
    int rc = page_tensor_map(&tin, static_cast<const uint8_t *>(in) + p0 * PC_PAGE_SIZE, m);
    if (rc == PC_OK) rc = page_tensor_map(&tout, static_cast<uint8_t *>(out) + p0 * PC_PAGE_SIZE, m);
    if (rc != PC_OK) return rc;
    pc::PageDesc dd{d.vaddrs ? d.vaddrs + p0 : nullptr, d.pids ? d.pids + p0 : nullptr,
                    d.vaddr0 + 4096ull * p0, d.pid0};
    const int per_sm = tuning().ctas_per_sm.load() > 0 ? tuning().ctas_per_sm.load() : occ;
    const uint64_t slots = (m + 3) / 4;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(static_cast<uint64_t>(n_sm) * per_sm, slots));
    kfn<<<grid, 256, kTmaSmem, st>>>(tin, tout, key, dd, m);
    counted();
    CU(cudaGetLastError());
  }
  return PC_OK;
}

// Default kernel per round count, from the B200 sweeps in profiles/
// (r01_kernel_sweep_*.txt, r01_clock_power_sweep.txt): ChaCha8 is HBM-bound
// and wants the fully coalesced v3; ChaCha12/20 are ALU-bound and v5 (cp.async
// ring, 4 CTAs/SM) is at least as fast as v2 there.
int auto_kernel(int rounds) { return rounds == 8 ? 3 : 5; }

// kernel_override: 0 = the "kernel" knob, else force 1..5 (the zero-copy
// host path forces 3).
int launch_crypt(const uint32_t *key, const pc::PageDesc &d, const void *in, void *out,
                 size_t n_pages, int rounds, cudaStream_t st, int kernel_override = 0) {
  if (n_pages == 0) return PC_OK;
  int kern = kernel_override ? kernel_override : tuning().kernel.load();
  if (kern == 0) kern = auto_kernel(rounds);
  if (kern == 4) {
    switch (rounds) {
      case 8: return launch_tma_r<8>(key, d, in, out, n_pages, st);
      case 12: return launch_tma_r<12>(key, d, in, out, n_pages, st);
      default: return launch_tma_r<20>(key, d, in, out, n_pages, st);
    }
  }
  if (kern == 2 || kern == 3 || kern == 5 || kern == 6 || kern == 9) {
    switch (rounds) {
      case 8: launch_pages_r<8>(kern, key, d, in, out, n_pages, st); break;
      case 12: launch_pages_r<12>(kern, key, d, in, out, n_pages, st); break;
      default: launch_pages_r<20>(kern, key, d, in, out, n_pages, st); break;
    }
    CU(cudaGetLastError());
    return PC_OK;
  }
  const uint64_t n_blocks = static_cast<uint64_t>(n_pages) * PC_BLOCKS_PER_PAGE;
  const uint32_t mask = tuning().rot_mask.load(std::memory_order_relaxed);
  switch (rounds) {
    case 8: launch_crypt_r<8>(mask, key, d, in, out, n_blocks, st); break;
    case 12: launch_crypt_r<12>(mask, key, d, in, out, n_blocks, st); break;
    default: launch_crypt_r<20>(mask, key, d, in, out, n_blocks, st); break;
  }
  CU(cudaGetLastError());
  return PC_OK;
}

int launch_keystream(const uint32_t *key, const uint32_t *seeds, size_t k, uint32_t *out, int rounds,
                     cudaStream_t st) {
  const dim3 block(128);
  const dim3 grid(static_cast<unsigned>((k + 127) / 128));
  switch (rounds) {
    case 8: pc::k_keystream_seeds<8><<<grid, block, 0, st>>>(key, seeds, k, out); break;
    case 12: pc::k_keystream_seeds<12><<<grid, block, 0, st>>>(key, seeds, k, out); break;
    default: pc::k_keystream_seeds<20><<<grid, block, 0, st>>>(key, seeds, k, out); break;
  }
  counted();
  CU(cudaGetLastError());
  return PC_OK;
}

// Is p host memory the device can address (pinned / registered)?  Returns the
// device-visible alias in *dev (nullptr when not pinned).
bool pinned_alias(const void *p, void **dev) {
  *dev = nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type != cudaMemoryTypeHost || a.devicePointer == nullptr) return false;
  *dev = a.devicePointer;
  return true;
}

// Both answers from ONE cudaPointerGetAttributes (the fault-sized path asks
// for each of its two buffers; every query is a driver call).
struct PtrInfo {
  bool dev = false;        // device (or managed) memory of GPU `device`
  int device = -1;
  void *host_dev = nullptr; // pinned host memory: its device-visible alias
};
PtrInfo ptr_info(const void *p) {
  PtrInfo r;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return r;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    r.dev = true;
    r.device = a.device;
  } else if (a.type == cudaMemoryTypeHost) {
    r.host_dev = a.devicePointer;
  }
  return r;
}

// Is p device memory (of any GPU; managed memory counts)?  *device = its GPU.
bool device_memory(const void *p, int *device) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return false;
  *device = a.device;
  return true;
}

// Persistent services running per device (pc_service_start/stop).
std::atomic<int> g_services_on[64];
bool service_running(int d) { return d >= 0 && d < 64 && g_services_on[d].load() > 0; }

// Can kernels on `dev` load/store `peer`'s memory?  Enables peer access once
// per (dev, peer) pair and caches the answer (NVSwitch: every pair can).
// Enabling is never attempted while a persistent service runs on either
// device (the enable may wait for that device to idle): the answer is then
// "no" for now, and callers take their staged-copy paths.  pc_service_start
// enables the pairs it can see before it launches, so this is the rare case.
bool peer_access(int dev, int peer) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, bool> known;
  std::lock_guard<std::mutex> lk(mu);
  auto it = known.find({dev, peer});
  if (it != known.end()) return it->second;
  if (service_running(dev) || service_running(peer)) return false; // not cached: retried later
  int can = 0;
  bool ok = cudaDeviceCanAccessPeer(&can, dev, peer) == cudaSuccess && can;
  if (ok) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
    ok = e == cudaSuccess;
    cudaGetLastError(); // clear a sticky-free error from the enable call
    cudaSetDevice(cur);
  } else {
    cudaGetLastError();
  }
  known[{dev, peer}] = ok;
  return ok;
}

// Process-wide recycler of pinned host buffers.  cudaFreeHost (like cudaFree
// and cudaHostUnregister) synchronises the whole device, which never returns
// while a persistent service kernel runs (tools/diag/persistent_probe), so the
// library never frees pinned memory it allocated: released buffers are kept
// by size and handed out again.  All are mapped + portable.
struct PinnedPool {
  std::mutex mu;
  std::unordered_map<size_t, std::vector<void *>> free;
};
PinnedPool &pinned_pool() {
  static PinnedPool *p = new PinnedPool(); // intentionally never destroyed
  return *p;
}
cudaError_t pinned_get(void **out, size_t bytes) {
  {
    PinnedPool &pp = pinned_pool();
    std::lock_guard<std::mutex> lk(pp.mu);
    auto it = pp.free.find(bytes);
    if (it != pp.free.end() && !it->second.empty()) {
      *out = it->second.back();
      it->second.pop_back();
      return cudaSuccess;
    }
  }
  return cudaHostAlloc(out, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
}
void pinned_put(void *p, size_t bytes) {
  if (!p) return;
  PinnedPool &pp = pinned_pool();
  std::lock_guard<std::mutex> lk(pp.mu);
  pp.free[bytes].push_back(p);
}

// Per-device scratch for the synchronous seams and key staging (guarded): a
// device buffer (stream-ordered allocation, so no call here ever forces a
// device-wide synchronisation -- a persistent service kernel may be running)
// and a pinned host buffer, so key material never passes through the
// driver's own pageable-copy staging and is wiped right after each use.
struct Scratch {
  std::mutex mu;
  void *d = nullptr;
  size_t cap = 0;
  uint8_t *h = nullptr; // pinned, same capacity
  cudaStream_t st = nullptr;
};
Scratch &scratch(int dev) {
  static Scratch s[64];
  return s[dev & 63];
}

// Caller holds sc.mu and the device is current.
int scratch_reserve(Scratch &sc, size_t need) {
  if (!sc.st) CU(cudaStreamCreateWithFlags(&sc.st, cudaStreamNonBlocking));
  if (sc.cap >= need) return PC_OK;
  if (sc.d) {
    CU(cudaFreeAsync(sc.d, sc.st));
    CU(cudaStreamSynchronize(sc.st));
  }
  if (sc.h) {
    wipe(sc.h, sc.cap);
    pinned_put(sc.h, sc.cap);
  }
  sc.d = nullptr;
  sc.h = nullptr;
  sc.cap = 0;
  const size_t cap = std::max<size_t>(need, 64 * 1024);
  CU(cudaMallocAsync(&sc.d, cap, sc.st));
  CU(cudaStreamSynchronize(sc.st));
  CU(pinned_get(reinterpret_cast<void **>(&sc.h), cap));
  sc.cap = cap;
  return PC_OK;
}

int keystream_sync(const uint32_t kw[8], const uint32_t *seeds, size_t k, uint32_t *out, int rounds) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  Scratch &sc = scratch(dev);
  std::lock_guard<std::mutex> lk(sc.mu);
  const size_t out_off = 256 + 16 * k;
  const size_t need = out_off + 64 * k;
  int rc = scratch_reserve(sc, need);
  if (rc != PC_OK) return rc;
  // pinned staging: key at [0,32), seeds at [256, 256+16k), keystream after
  std::memcpy(sc.h, kw, 32);
  std::memcpy(sc.h + 256, seeds, 16 * k);
  if (k <= 4096) {
    // seam-sized calls (a page is 64 blocks): one zero-copy launch on the
    // mapped staging -- the kernel reads key and seeds and writes the
    // keystream across PCIe, no DMA round trips
    uint8_t *hd = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&hd), sc.h, 0);
    if (e == cudaSuccess) {
      rc = launch_keystream(reinterpret_cast<uint32_t *>(hd), reinterpret_cast<uint32_t *>(hd + 256), k,
                            reinterpret_cast<uint32_t *>(hd + out_off), rounds, sc.st);
      e = cudaStreamSynchronize(sc.st);
      if (rc == PC_OK && e == cudaSuccess) std::memcpy(out, sc.h + out_off, 64 * k);
    }
    wipe(sc.h, need);
    if (rc != PC_OK) return rc;
    CU(e);
    return PC_OK;
  }
  uint8_t *d = static_cast<uint8_t *>(sc.d);
  cudaError_t e = cudaMemcpyAsync(d, sc.h, out_off, cudaMemcpyHostToDevice, sc.st);
  if (e == cudaSuccess) {
    rc = launch_keystream(reinterpret_cast<uint32_t *>(d), reinterpret_cast<uint32_t *>(d + 256), k,
                          reinterpret_cast<uint32_t *>(d + out_off), rounds, sc.st);
    if (rc == PC_OK) e = cudaMemcpyAsync(sc.h + out_off, d + out_off, 64 * k, cudaMemcpyDeviceToHost, sc.st);
  }
  cudaError_t e2 = cudaMemsetAsync(d, 0, need, sc.st); // wipe key + keystream on the device
  cudaError_t e3 = cudaStreamSynchronize(sc.st);
  if (rc == PC_OK && e == cudaSuccess && e3 == cudaSuccess) std::memcpy(out, sc.h + out_off, 64 * k);
  wipe(sc.h, need);
  if (rc != PC_OK) return rc;
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = e3;
  CU(e);
  return PC_OK;
}

constexpr uint32_t kKeyMagic = 0x6b657931u;    // "key1"
constexpr uint32_t kEngineMagic = 0x656e6731u; // "eng1"

} // namespace

struct pc_key {
  uint32_t magic;
  int device;
  uint32_t *d_words;     // 256-byte device allocation, key in the first 32 bytes
  cudaStream_t kst;      // key's private stream: depends on every device-path use
  cudaEvent_t ev;
  std::mutex mu;
  std::atomic<int> refs{0}; // stores holding this key; destroy refuses while > 0
  void *ipc_buf = nullptr;  // live CUDA-IPC export of the key (pc_key_export), or NULL
  uint64_t serial = 0;      // process-unique identity (a service started from this key records it)
  pc_service *svc = nullptr; // resident workers for fault-sized host batches (pc_key_service)
  int svc_rounds = 0;
  int svc_workers = 0;
  std::shared_mutex svc_mu;  // shared: a call using svc; exclusive: starting / stopping it
};

namespace {
// Make the key's private stream depend on the work just enqueued on `st`, so
// pc_key_destroy can wait for every use without a device-wide synchronise.
int note_key_use(pc_key *key, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(key->mu);
  CU(cudaEventRecord(key->ev, st));
  CU(cudaStreamWaitEvent(key->kst, key->ev, 0));
  return PC_OK;
}

// Free a key object's device slot (zeroed first), stream and event.
void key_free(pc_key *k) {
  if (k->d_words) {
    cudaMemsetAsync(k->d_words, 0, 256, k->kst);
    cudaFreeAsync(k->d_words, k->kst);
    cudaStreamSynchronize(k->kst);
  }
  if (k->ev) cudaEventDestroy(k->ev);
  if (k->kst) cudaStreamDestroy(k->kst);
  k->magic = 0;
  delete k;
}

// An empty key object on `device` (current device must be `device`): its
// private stream and event and a zeroed 256-byte stream-ordered slot.
int key_new(int device, pc_key **out) {
  *out = nullptr;
  static std::atomic<uint64_t> next_serial{1};
  auto *k = new pc_key();
  k->magic = kKeyMagic;
  k->serial = next_serial.fetch_add(1);
  k->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&k->kst, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&k->ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void **>(&k->d_words), 256, k->kst);
  if (e == cudaSuccess) e = cudaMemsetAsync(k->d_words, 0, 256, k->kst);
  if (e != cudaSuccess) {
    key_free(k);
    return fail(e == cudaErrorMemoryAllocation ? PC_ENOMEM : PC_ECUDA, "key slot: %s", cudaGetErrorString(e));
  }
  *out = k;
  return PC_OK;
}

// Allocate a key object on `device` and fill its 32 bytes from `src` through
// the pinned scratch (wiped afterwards).  If `derive`, src is entropy and the
// key is derived on the device by k_keygen.
int key_create(int device, const uint8_t *src, bool derive, pc_key **out) {
  *out = nullptr;
  DeviceGuard g(device);
  CU(g.err);
  pc_key *k = nullptr;
  int rc = key_new(device, &k);
  if (rc != PC_OK) return rc;
  cudaError_t e;
  {
    Scratch &sc = scratch(device);
    std::lock_guard<std::mutex> lk(sc.mu);
    rc = scratch_reserve(sc, 256);
    if (rc != PC_OK) {
      key_free(k);
      return rc;
    }
    std::memcpy(sc.h, src, 32);
    // key (or entropy) lands at d_words[0..7] / d_words[8..15]
    uint32_t *dst = derive ? k->d_words + 8 : k->d_words;
    e = cudaMemcpyAsync(dst, sc.h, 32, cudaMemcpyHostToDevice, k->kst);
    if (e == cudaSuccess && derive) {
      pc::k_keygen<<<1, 1, 0, k->kst>>>(k->d_words + 8, k->d_words);
      counted();
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaMemsetAsync(k->d_words + 8, 0, 32, k->kst);
    }
    cudaError_t e2 = cudaStreamSynchronize(k->kst);
    wipe(sc.h, 32);
    if (e == cudaSuccess) e = e2;
  }
  if (e != cudaSuccess) {
    key_free(k);
    return fail(PC_ECUDA, "key install: %s", cudaGetErrorString(e));
  }
  *out = k;
  return PC_OK;
}

// CUDA-IPC export buffers (cudaMalloc'd: IPC handles cannot name
// stream-ordered pool memory).  cudaFree synchronises the device, which never
// returns while a persistent service runs, so closed exports are zeroed and
// recycled here instead of freed.
struct ExportPool {
  std::mutex mu;
  std::map<int, std::vector<void *>> free; // device -> zeroed 256-byte buffers
};
ExportPool &export_pool() {
  static ExportPool *p = new ExportPool(); // intentionally never destroyed
  return *p;
}
} // namespace

struct pc_engine {
  uint32_t magic = kEngineMagic;
  int device = 0;
  int n_streams = 0;
  size_t chunk_pages = 0;
  std::mutex mu;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> done;    // slot's D2H complete
  std::vector<cudaEvent_t> ev_h2d;  // slot's H2D complete (host_mode 2)
  std::vector<cudaEvent_t> ev_k;    // slot's kernel complete (host_mode 2)
  std::vector<uint8_t *> d_pages;   // per-stream device staging, chunk_pages*4096
  std::vector<uint64_t *> d_vaddrs; // per-stream descriptor staging
  std::vector<uint32_t *> d_pids;
  std::vector<uint8_t *> h_bounce;  // pinned bounce for pageable I/O (lazy)
  std::vector<uint8_t *> h_desc;    // pinned descriptor staging (chunk*16 bytes)
  uint8_t *h_key = nullptr;         // pinned 256-B raw-key staging
  uint32_t *d_rawkey = nullptr;     // caller-key device slot (wiped after use)
  // small-batch path: one pinned+mapped region and its device mirror
  uint8_t *h_small = nullptr;
  uint8_t *hd_small = nullptr;      // device alias of h_small (zero-copy)
  uint8_t *d_small = nullptr;
  size_t small_bytes = 0;
  std::unique_ptr<pc::HostPool> pool; // pageable <-> pinned bounce copies (lazy)
  std::unique_ptr<pc::Runner> runner; // this engine's thread for multi-device calls (lazy)
  std::mutex runner_mu;
  pc::DevicePlacement place;          // GPU-local CPUs / NUMA node for threads and pinned staging
};

// ===========================================================================
extern "C" {

int pc_abi_version(void) { return PC_ABI_VERSION; }

const char *pc_last_error(void) { return g_err.c_str(); }

int pc_device_count(int *count) {
  if (!count) return fail(PC_EINVAL, "count is NULL");
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(PC_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  return PC_OK;
}

int pc_device_info(int device, int *sm_count, int *cc_major, int *cc_minor) {
  if (!sm_count || !cc_major || !cc_minor) return fail(PC_EINVAL, "NULL output");
  CU(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  CU(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  CU(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return PC_OK;
}

// ---- (i) kernel seam -------------------------------------------------------
int pc_keystream_words(const uint32_t kw[8], uint64_t vaddr, uint32_t pid, const int64_t *idx,
                       size_t k, uint32_t *out, int rounds) {
  if (!kw) return fail(PC_EINVAL, "key words are NULL");
  if (!valid_rounds(rounds)) return fail(PC_EINVAL, "rounds must be 8, 12 or 20, got %d", rounds);
  if (k == 0) return PC_OK;
  if (!idx || !out) return fail(PC_EINVAL, "indices/out are NULL");
  std::vector<uint32_t> seeds(4 * k);
  for (size_t i = 0; i < k; ++i) {
    seeds[4 * i + 0] = static_cast<uint32_t>(vaddr);
    seeds[4 * i + 1] = static_cast<uint32_t>(vaddr >> 32);
    seeds[4 * i + 2] = pid;
    seeds[4 * i + 3] = static_cast<uint32_t>(static_cast<uint64_t>(idx[i]));
  }
  return keystream_sync(kw, seeds.data(), k, out, rounds);
}

// ---- (ii) raw seeds --------------------------------------------------------
int pc_keystream_raw(const uint8_t key[32], const uint8_t *seeds16, size_t k, int rounds, uint8_t *out) {
  if (!key) return fail(PC_EINVAL, "key is NULL");
  if (!valid_rounds(rounds)) return fail(PC_EINVAL, "rounds must be 8, 12 or 20, got %d", rounds);
  if (k == 0) return PC_OK;
  if (!seeds16 || !out) return fail(PC_EINVAL, "seeds/out are NULL");
  uint32_t kw[8];
  std::memcpy(kw, key, 32);
  std::vector<uint32_t> seeds(4 * k);
  std::memcpy(seeds.data(), seeds16, 16 * k);
  std::vector<uint32_t> words(16 * k);
  int rc = keystream_sync(kw, seeds.data(), k, words.data(), rounds);
  wipe(kw, sizeof kw);
  if (rc == PC_OK) std::memcpy(out, words.data(), 64 * k);
  wipe(words.data(), 64 * k);
  return rc;
}

// ---- (iii) key residency ---------------------------------------------------
int pc_key_install(int device, const uint8_t key[32], pc_key **out) {
  if (!key || !out) return fail(PC_EINVAL, "key/out is NULL");
  return key_create(device, key, false, out);
}

int pc_key_generate(int device, const uint8_t entropy[32], pc_key **out) {
  if (!entropy || !out) return fail(PC_EINVAL, "entropy/out is NULL");
  return key_create(device, entropy, true, out);
}

int pc_key_destroy(pc_key *key) {
  if (!key) return PC_OK;
  if (key->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  if (const int r = key->refs.load())
    return fail(PC_ESTATE, "key is still held by %d page store(s); destroy them first", r);
  if (key->svc) {
    int rc = pc_key_service(key, 0, 0);
    if (rc != PC_OK) return rc;
  }
  DeviceGuard g(key->device);
  CU(g.err);
  if (key->ipc_buf) {
    int rc = pc_key_export_close(key);
    if (rc != PC_OK) return rc;
  }
  {
    std::lock_guard<std::mutex> lk(key->mu);
    // kst already waits for every device-path use of the key (note_key_use)
    CU(cudaMemsetAsync(key->d_words, 0, 256, key->kst));
    CU(cudaFreeAsync(key->d_words, key->kst));
    CU(cudaStreamSynchronize(key->kst));
    cudaEventDestroy(key->ev);
    cudaStreamDestroy(key->kst);
    key->magic = 0;
    key->d_words = nullptr;
  }
  delete key;
  return PC_OK;
}

int pc_key_device(const pc_key *key, int *device) {
  if (!key || key->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  if (!device) return fail(PC_EINVAL, "device is NULL");
  *device = key->device;
  return PC_OK;
}


// ---- key replication (the key replicated into each device) -----
int pc_key_replicate(const pc_key *src, int device, pc_key **out) {
  if (!out) return fail(PC_EINVAL, "out is NULL");
  *out = nullptr;
  if (!src || src->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(PC_EINVAL, "device %d outside 0..%d", device, ndev - 1);
  // a cross-device copy without peer access would be staged by the driver
  // through host memory: refuse rather than let the key touch host RAM
  if (device != src->device && !peer_access(device, src->device))
    return fail(PC_ESTATE, "no peer access from device %d to device %d: the key cannot be copied "
                "device-to-device", device, src->device);
  DeviceGuard g(device);
  CU(g.err);
  pc_key *k = nullptr;
  int rc = key_new(device, &k);
  if (rc != PC_OK) return rc;
  cudaError_t e = cudaMemcpyPeerAsync(k->d_words, device, src->d_words, src->device, 32, k->kst);
  if (e == cudaSuccess) e = cudaStreamSynchronize(k->kst);
  if (e != cudaSuccess) {
    key_free(k);
    return fail(PC_ECUDA, "key replicate: %s", cudaGetErrorString(e));
  }
  *out = k;
  return PC_OK;
}

int pc_key_export(pc_key *key, uint8_t handle[PC_KEY_HANDLE_SIZE]) {
  if (!key || key->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  if (!handle) return fail(PC_EINVAL, "handle is NULL");
  static_assert(sizeof(cudaIpcMemHandle_t) == PC_KEY_HANDLE_SIZE, "IPC handle size");
  DeviceGuard g(key->device);
  CU(g.err);
  std::lock_guard<std::mutex> lk(key->mu);
  if (!key->ipc_buf) {
    void *buf = nullptr;
    {
      ExportPool &xp = export_pool();
      std::lock_guard<std::mutex> l2(xp.mu);
      auto &v = xp.free[key->device];
      if (!v.empty()) {
        buf = v.back();
        v.pop_back();
      }
    }
    if (!buf) {
      cudaError_t e = cudaMalloc(&buf, 256);
      if (e != cudaSuccess) return fail(PC_ENOMEM, "export buffer: %s", cudaGetErrorString(e));
    }
    cudaError_t e = cudaMemcpyAsync(buf, key->d_words, 32, cudaMemcpyDeviceToDevice, key->kst);
    if (e == cudaSuccess) e = cudaStreamSynchronize(key->kst);
    if (e != cudaSuccess) {
      std::lock_guard<std::mutex> l2(export_pool().mu);
      export_pool().free[key->device].push_back(buf);
      return fail(PC_ECUDA, "key export: %s", cudaGetErrorString(e));
    }
    key->ipc_buf = buf;
  }
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, key->ipc_buf));
  std::memcpy(handle, &h, sizeof h);
  return PC_OK;
}

int pc_key_export_close(pc_key *key) {
  if (!key || key->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  DeviceGuard g(key->device);
  CU(g.err);
  std::lock_guard<std::mutex> lk(key->mu);
  if (!key->ipc_buf) return PC_OK;
  cudaError_t e = cudaMemsetAsync(key->ipc_buf, 0, 256, key->kst);
  if (e == cudaSuccess) e = cudaStreamSynchronize(key->kst);
  CU(e);
  {
    std::lock_guard<std::mutex> l2(export_pool().mu);
    export_pool().free[key->device].push_back(key->ipc_buf);
  }
  key->ipc_buf = nullptr;
  return PC_OK;
}

int pc_key_import(int device, const uint8_t handle[PC_KEY_HANDLE_SIZE], pc_key **out) {
  if (!out) return fail(PC_EINVAL, "out is NULL");
  *out = nullptr;
  if (!handle) return fail(PC_EINVAL, "handle is NULL");
  DeviceGuard g(device);
  CU(g.err);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void *peer = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&peer, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(PC_ECUDA, "cudaIpcOpenMemHandle: %s (the exporting process must be alive, its export "
                "open, and this device able to reach the exporter's device)", cudaGetErrorString(e));
  }
  pc_key *k = nullptr;
  int rc = key_new(device, &k);
  if (rc == PC_OK) {
    // device-to-device (same GPU, or NVLink peer read of the exporter's GPU)
    e = cudaMemcpyAsync(k->d_words, peer, 32, cudaMemcpyDeviceToDevice, k->kst);
    if (e == cudaSuccess) e = cudaStreamSynchronize(k->kst);
    if (e != cudaSuccess) {
      key_free(k);
      k = nullptr;
      rc = fail(PC_ECUDA, "key import: %s", cudaGetErrorString(e));
    }
  }
  cudaIpcCloseMemHandle(peer);
  *out = k;
  return rc;
}

int pc_engine_placement(const pc_engine *e, int *numa_node, int *n_cpus) {
  if (!e || e->magic != kEngineMagic) return fail(PC_ESTATE, "not a live pc_engine");
  if (!numa_node || !n_cpus) return fail(PC_EINVAL, "NULL output");
  *numa_node = e->place.node;
  *n_cpus = e->place.has_cpus ? CPU_COUNT(&e->place.cpus) : 0;
  return PC_OK;
}

// ---- (iv) device-resident batch -------------------------------------------
int pc_crypt_pages_dev(const pc_key *key, const uint64_t *vaddrs, const uint32_t *pids,
                       uint64_t vaddr0, uint32_t pid0, const void *in, void *out, size_t n,
                       int rounds, void *stream) {
  if (!key || key->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  if (!valid_rounds(rounds)) return fail(PC_EINVAL, "rounds must be 8, 12 or 20, got %d", rounds);
  if (n == 0) return PC_OK;
  if (!in || !out) return fail(PC_EINVAL, "in/out is NULL");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(PC_EINVAL, "page buffers must be 16-byte aligned");
  if (!vaddrs && (vaddr0 & 4095)) return fail(PC_EINVAL, "vaddr0 %#llx not page-aligned", (unsigned long long)vaddr0);
  if (!vaddrs && n > 1 && vaddr0 + 4096ull * (n - 1) < vaddr0)
    return fail(PC_EINVAL, "contiguous vaddr range overflows u64");
  DeviceGuard g(key->device);
  CU(g.err);
  const pc::PageDesc d{vaddrs, pids, vaddr0, pid0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = launch_crypt(key->d_words, d, in, out, n, rounds, st);
  if (rc != PC_OK) return rc;
  return note_key_use(const_cast<pc_key *>(key), st);
}

// ---- (v) host-resident batch ---------------------------------------------
int pc_engine_create(int device, int n_streams, size_t chunk_pages, pc_engine **out) {
  if (!out) return fail(PC_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_streams <= 0) n_streams = 4;
  if (n_streams > 16) n_streams = 16;
  if (chunk_pages == 0) chunk_pages = 8192; // 32 MiB per stage
  DeviceGuard g(device);
  CU(g.err);
  auto *e = new pc_engine();
  e->device = device;
  e->n_streams = n_streams;
  e->chunk_pages = chunk_pages;
  e->place = pc::device_placement(device);
  pc::NodeScope near_gpu(e->place); // pinned staging below is first touched on the GPU's node
  auto cleanup = [&](int rc) {
    pc_engine_destroy(e);
    return rc;
  };
#define CUE(call)                                                                           \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return cleanup(fail(e_ == cudaErrorMemoryAllocation ? PC_ENOMEM : PC_ECUDA, "%s: %s", \
                          #call, cudaGetErrorString(e_)));                                  \
  } while (0)
  e->streams.assign(n_streams, nullptr);
  e->done.assign(n_streams, nullptr);
  e->ev_h2d.assign(n_streams, nullptr);
  e->ev_k.assign(n_streams, nullptr);
  e->d_pages.assign(n_streams, nullptr);
  e->d_vaddrs.assign(n_streams, nullptr);
  e->d_pids.assign(n_streams, nullptr);
  e->h_bounce.assign(n_streams, nullptr);
  e->h_desc.assign(n_streams, nullptr);
  for (int s = 0; s < n_streams; ++s) {
    CUE(cudaStreamCreateWithFlags(&e->streams[s], cudaStreamNonBlocking));
    CUE(cudaEventCreateWithFlags(&e->done[s], cudaEventDisableTiming));
    CUE(cudaEventCreateWithFlags(&e->ev_h2d[s], cudaEventDisableTiming));
    CUE(cudaEventCreateWithFlags(&e->ev_k[s], cudaEventDisableTiming));
    CUE(cudaMallocAsync(reinterpret_cast<void **>(&e->d_pages[s]), chunk_pages * PC_PAGE_SIZE, e->streams[0]));
    CUE(cudaMallocAsync(reinterpret_cast<void **>(&e->d_vaddrs[s]), chunk_pages * 8, e->streams[0]));
    // d_pids: pids at [0, C), slab slots at [C, 2C); h_desc: vaddrs, pids, slots
    CUE(cudaMallocAsync(reinterpret_cast<void **>(&e->d_pids[s]), chunk_pages * 8, e->streams[0]));
    CUE(pinned_get(reinterpret_cast<void **>(&e->h_desc[s]), chunk_pages * 16));
  }
  CUE(pinned_get(reinterpret_cast<void **>(&e->h_key), 256));
  CUE(cudaMallocAsync(reinterpret_cast<void **>(&e->d_rawkey), 256, e->streams[0]));
  const size_t sm = tuning().small_max.load();
  e->small_bytes = 256 + sm * 16 + sm * PC_PAGE_SIZE;
  CUE(pinned_get(reinterpret_cast<void **>(&e->h_small), e->small_bytes));
  CUE(cudaHostGetDevicePointer(reinterpret_cast<void **>(&e->hd_small), e->h_small, 0));
  CUE(cudaMallocAsync(reinterpret_cast<void **>(&e->d_small), e->small_bytes, e->streams[0]));
  CUE(cudaStreamSynchronize(e->streams[0]));
#undef CUE
  *out = e;
  return PC_OK;
}

int pc_engine_destroy(pc_engine *e) {
  if (!e) return PC_OK;
  if (e->magic != kEngineMagic) return fail(PC_ESTATE, "not a live pc_engine");
  DeviceGuard g(e->device);
  for (auto s : e->streams)
    if (s) cudaStreamSynchronize(s);
  // stream-ordered frees on stream 0: no device-wide synchronisation
  cudaStream_t s0 = e->streams.empty() ? nullptr : e->streams[0];
  if (s0) {
    if (e->d_rawkey) { cudaMemsetAsync(e->d_rawkey, 0, 256, s0); cudaFreeAsync(e->d_rawkey, s0); }
    if (e->d_small) { cudaMemsetAsync(e->d_small, 0, 256, s0); cudaFreeAsync(e->d_small, s0); }
    for (size_t s = 0; s < e->streams.size(); ++s) {
      if (e->d_pages[s]) cudaFreeAsync(e->d_pages[s], s0);
      if (e->d_vaddrs[s]) cudaFreeAsync(e->d_vaddrs[s], s0);
      if (e->d_pids[s]) cudaFreeAsync(e->d_pids[s], s0);
    }
    cudaStreamSynchronize(s0);
  }
  if (e->h_key) { wipe(e->h_key, 256); pinned_put(e->h_key, 256); }
  if (e->h_small) { wipe(e->h_small, e->small_bytes); pinned_put(e->h_small, e->small_bytes); }
  for (size_t s = 0; s < e->streams.size(); ++s) {
    if (e->h_bounce[s]) pinned_put(e->h_bounce[s], e->chunk_pages * PC_PAGE_SIZE);
    if (e->h_desc[s]) pinned_put(e->h_desc[s], e->chunk_pages * 16);
    if (e->done[s]) cudaEventDestroy(e->done[s]);
    if (e->ev_h2d[s]) cudaEventDestroy(e->ev_h2d[s]);
    if (e->ev_k[s]) cudaEventDestroy(e->ev_k[s]);
    if (e->streams[s]) cudaStreamDestroy(e->streams[s]);
  }
  cudaGetLastError();
  e->magic = 0;
  delete e;
  return PC_OK;
}

namespace {

// Small batches: one staging region [key | vaddrs | pids | pages] in pinned,
// mapped memory.  Zero-copy mode runs the kernel directly on it (one launch,
// no copies); copy mode does one H2D, the kernel and one D2H.
int crypt_small(pc_engine *e, const uint32_t *dkey, const uint8_t *raw_key, const uint64_t *vaddrs,
                const uint32_t *pids, uint64_t vaddr0, uint32_t pid0, const void *in, void *out,
                size_t n, int rounds, void *in_dev, void *out_dev) {
  const size_t off_v = 256, off_p = off_v + ((n * 8 + 255) & ~size_t(255));
  const size_t off_pg = off_p + ((n * 4 + 255) & ~size_t(255));
  const size_t used = off_pg + n * PC_PAGE_SIZE;
  uint8_t *h = e->h_small;
  cudaStream_t st = e->streams[0];
  const bool zc = tuning().small_mode == 1;
  // zero-copy straight on the caller's pages when they are pinned already
  // (in_dev/out_dev: their device aliases, from the caller's pointer query)
  const bool direct = zc && in_dev && out_dev;
  if (raw_key) std::memcpy(h, raw_key, 32);
  if (vaddrs) std::memcpy(h + off_v, vaddrs, n * 8);
  if (pids) std::memcpy(h + off_p, pids, n * 4);
  if (!direct) std::memcpy(h + off_pg, in, n * PC_PAGE_SIZE);
  uint8_t *base = zc ? e->hd_small : e->d_small;
  const pc::PageDesc d{vaddrs ? reinterpret_cast<const uint64_t *>(base + off_v) : nullptr,
                       pids ? reinterpret_cast<const uint32_t *>(base + off_p) : nullptr, vaddr0, pid0};
  const uint32_t *key = raw_key ? reinterpret_cast<const uint32_t *>(base) : dkey;
  int rc = PC_OK;
  cudaError_t err = cudaSuccess;
  if (!zc) err = cudaMemcpyAsync(e->d_small, h, used, cudaMemcpyHostToDevice, st);
  if (err == cudaSuccess) {
    if (direct)
      rc = launch_crypt(key, d, in_dev, out_dev, n, rounds, st, 3);
    else
      rc = launch_crypt(key, d, base + off_pg, base + off_pg, n, rounds, st, zc ? 3 : 0);
  }
  if (err == cudaSuccess && rc == PC_OK && !zc)
    err = cudaMemcpyAsync(h + off_pg, e->d_small + off_pg, n * PC_PAGE_SIZE, cudaMemcpyDeviceToHost, st);
  if (!zc && raw_key) {
    cudaError_t e2 = cudaMemsetAsync(e->d_small, 0, 256, st);
    if (err == cudaSuccess) err = e2;
  }
  cudaError_t e3 = cudaStreamSynchronize(st);
  if (raw_key) wipe(h, 32);
  if (rc != PC_OK) return rc;
  if (err == cudaSuccess) err = e3;
  CU(err);
  if (!direct) std::memcpy(out, h + off_pg, n * PC_PAGE_SIZE);
  return PC_OK;
}

int crypt_large(pc_engine *e, const uint32_t *key, const uint64_t *vaddrs, const uint32_t *pids,
                uint64_t vaddr0, uint32_t pid0, const void *in, void *out, size_t n, int rounds) {
  void *in_dev = nullptr, *out_dev = nullptr;
  int gin = -1, gout = -1;
  // device memory (this GPU or a peer) is an endpoint like pinned memory:
  // no bounce buffer, copies by UVA (peer copies over NVLink), but the
  // zero-copy modes below only apply to mapped host memory
  const bool pin_in = pinned_alias(in, &in_dev) || device_memory(in, &gin);
  const bool pin_out = pinned_alias(out, &out_dev) || device_memory(out, &gout);
  const bool has_desc = vaddrs || pids;
  if (tuning().host_mode.load() == 1 && in_dev && out_dev) {
    // zero-copy: one coalesced kernel streams the pages over PCIe itself
    // (GPU-initiated reads and posted writes, both directions at once)
    void *v_dev = nullptr, *p_dev = nullptr;
    const bool desc_ok = (!vaddrs || pinned_alias(vaddrs, &v_dev)) && (!pids || pinned_alias(pids, &p_dev));
    if (desc_ok) {
      const pc::PageDesc d{static_cast<const uint64_t *>(v_dev), static_cast<const uint32_t *>(p_dev),
                           vaddr0, pid0};
      int rc = launch_crypt(key, d, in_dev, out_dev, n, rounds, e->streams[0], 3);
      if (rc != PC_OK) return rc;
      CU(cudaStreamSynchronize(e->streams[0]));
      return PC_OK;
    }
  }
  // Staged pipeline over S device slots.  host_mode 2 (default): one H2D
  // stream, one compute stream and one D2H stream chained by events, so each
  // copy engine sees its transfers back to back; host_mode 0: chunk c runs
  // H2D -> kernel -> D2H in order on stream c % S.
  const int S = e->n_streams;
  const size_t C = e->chunk_pages;
  const int hm = tuning().host_mode.load();
  const bool dedicated = (hm == 2 || hm == 3) && S >= 3;
  // host_mode 3: the kernel stores each chunk's result straight into the
  // caller's pinned output over PCIe (posted writes), so no D2H copy runs
  const bool direct_out = hm == 3 && out_dev && dedicated;
  if (!pin_in || !pin_out) {
    pc::NodeScope near_gpu(e->place);
    for (int s = 0; s < S; ++s)
      if (!e->h_bounce[s]) CU(pinned_get(reinterpret_cast<void **>(&e->h_bounce[s]), C * PC_PAGE_SIZE));
    if (!e->pool) e->pool.reset(new pc::HostPool(host_pool_threads(), e->place));
  }
  // Chunk schedule: ramp up C/8, C/4, C/2 at the start and down at the end
  // (when the batch is large enough) so the pipeline fills and drains with
  // small transfers while the steady state uses full C-page chunks.
  std::vector<size_t> starts;
  {
    std::vector<size_t> sizes;
    size_t left = n;
    // ramp: powers of two from 1024 pages (4 MiB) up to C/2, so the first
    // transfer is small whatever the steady-state chunk is
    std::vector<size_t> ramp;
    for (size_t r = std::max<size_t>(1, std::min<size_t>(1024, C / 8)); r < C; r *= 2) ramp.push_back(r);
    size_t ramp_sum = 0;
    for (size_t r : ramp) ramp_sum += r;
    const bool do_ramp = C >= 64 && n >= 2 * ramp_sum + 2 * C;
    std::vector<size_t> tail;
    if (do_ramp) {
      for (size_t r : ramp) { sizes.push_back(r); left -= r; }
      for (size_t r : ramp) { tail.push_back(r); left -= r; }
    }
    while (left > 0) {
      const size_t m = std::min(C, left);
      sizes.push_back(m);
      left -= m;
    }
    for (auto it = tail.rbegin(); it != tail.rend(); ++it) sizes.push_back(*it);
    size_t p = 0;
    for (size_t m : sizes) { starts.push_back(p); p += m; }
    starts.push_back(p);
  }
  const size_t n_chunks = starts.size() - 1;
  auto *src_b = static_cast<const uint8_t *>(in);
  auto *dst_b = static_cast<uint8_t *>(out);
  auto finish = [&](size_t c) -> int { // chunk c's slot is about to be reused / drained
    const int s = static_cast<int>(c % S);
    CU(cudaEventSynchronize(e->done[s]));
    if (!pin_out) {
      const size_t p0 = starts[c], m = starts[c + 1] - p0;
      e->pool->memcpy(dst_b + p0 * PC_PAGE_SIZE, e->h_bounce[s], m * PC_PAGE_SIZE);
    }
    return PC_OK;
  };
  for (size_t c = 0; c < n_chunks; ++c) {
    const int s = static_cast<int>(c % S);
    cudaStream_t sh = dedicated ? e->streams[0] : e->streams[s];
    cudaStream_t sk = dedicated ? e->streams[1] : e->streams[s];
    cudaStream_t sd = dedicated ? e->streams[2] : e->streams[s];
    const size_t p0 = starts[c], m = starts[c + 1] - p0;
    if (c >= static_cast<size_t>(S)) {
      if (!pin_in || !pin_out || has_desc) {
        int rc = finish(c - S); // host reuses this slot's bounce / descriptor staging
        if (rc != PC_OK) return rc;
      } else if (dedicated) {
        CU(cudaStreamWaitEvent(sh, e->done[s], 0)); // device slot free once its D2H is done
      }
    }
    const uint8_t *src = src_b + p0 * PC_PAGE_SIZE;
    if (!pin_in) {
      e->pool->memcpy(e->h_bounce[s], src, m * PC_PAGE_SIZE);
      src = e->h_bounce[s];
    }
    CU(cudaMemcpyAsync(e->d_pages[s], src, m * PC_PAGE_SIZE, cudaMemcpyDefault, sh));
    pc::PageDesc d{nullptr, nullptr, vaddr0 + 4096ull * p0, pid0};
    if (vaddrs) {
      std::memcpy(e->h_desc[s], vaddrs + p0, m * 8);
      CU(cudaMemcpyAsync(e->d_vaddrs[s], e->h_desc[s], m * 8, cudaMemcpyHostToDevice, sh));
      d.vaddrs = e->d_vaddrs[s];
    }
    if (pids) {
      std::memcpy(e->h_desc[s] + C * 8, pids + p0, m * 4);
      CU(cudaMemcpyAsync(e->d_pids[s], e->h_desc[s] + C * 8, m * 4, cudaMemcpyHostToDevice, sh));
      d.pids = e->d_pids[s];
    }
    if (dedicated) {
      CU(cudaEventRecord(e->ev_h2d[s], sh));
      CU(cudaStreamWaitEvent(sk, e->ev_h2d[s], 0));
    }
    if (direct_out) {
      int rc = launch_crypt(key, d, e->d_pages[s], static_cast<uint8_t *>(out_dev) + p0 * PC_PAGE_SIZE, m,
                            rounds, sk, 3);
      if (rc != PC_OK) return rc;
      CU(cudaEventRecord(e->done[s], sk));
      continue;
    }
    int rc = launch_crypt(key, d, e->d_pages[s], e->d_pages[s], m, rounds, sk);
    if (rc != PC_OK) return rc;
    if (dedicated) {
      CU(cudaEventRecord(e->ev_k[s], sk));
      CU(cudaStreamWaitEvent(sd, e->ev_k[s], 0));
    }
    uint8_t *dst = pin_out ? dst_b + p0 * PC_PAGE_SIZE : e->h_bounce[s];
    CU(cudaMemcpyAsync(dst, e->d_pages[s], m * PC_PAGE_SIZE, cudaMemcpyDefault, sd));
    CU(cudaEventRecord(e->done[s], sd));
  }
  const size_t first_pending = n_chunks > static_cast<size_t>(S) ? n_chunks - S : 0;
  for (size_t c = first_pending; c < n_chunks; ++c) {
    int rc = finish(c);
    if (rc != PC_OK) return rc;
  }
  return PC_OK;
}

} // namespace

namespace {
int svc_submit(pc_service *s, int worker, uint64_t vaddr, uint32_t pid, const void *src, void *dst,
               const pc::SvcOp *op, uint64_t *ticket);
constexpr size_t kSvcMaxPages = 64; // largest host batch crypt_on_service takes (its ticket array)
int crypt_on_service(const pc_key *key, const uint64_t *vaddrs, const uint32_t *pids, uint64_t vaddr0,
                     uint32_t pid0, const void *in, void *out, size_t n) {
  uint64_t tickets[kSvcMaxPages];
  const int W = key->svc_workers;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t va = vaddrs ? vaddrs[i] : vaddr0 + 4096ull * i;
    const uint32_t pid = pids ? pids[i] : pid0;
    int rc = svc_submit(key->svc, static_cast<int>(i % W), va, pid, static_cast<const uint8_t *>(in) + i * PC_PAGE_SIZE,
                        static_cast<uint8_t *>(out) + i * PC_PAGE_SIZE, nullptr, &tickets[i]);
    if (rc != PC_OK) {
      for (size_t j = 0; j < i; ++j) pc_service_wait(key->svc, static_cast<int>(j % W), tickets[j], -1);
      return rc;
    }
  }
  int rc = PC_OK;
  for (size_t i = 0; i < n; ++i) {
    const int r = pc_service_wait(key->svc, static_cast<int>(i % W), tickets[i], -1);
    if (rc == PC_OK) rc = r;
  }
  return rc;
}
} // namespace

int pc_crypt_pages_host(pc_engine *e, const pc_key *key, const uint8_t *raw_key, const uint64_t *vaddrs,
                        const uint32_t *pids, uint64_t vaddr0, uint32_t pid0, const void *in, void *out,
                        size_t n, int rounds) {
  if (!e || e->magic != kEngineMagic) return fail(PC_ESTATE, "not a live pc_engine");
  if (!raw_key && (!key || key->magic != kKeyMagic)) return fail(PC_ESTATE, "not a live pc_key");
  if (!raw_key && key->device != e->device)
    return fail(PC_EINVAL, "key lives on device %d, engine on device %d", key->device, e->device);
  if (!valid_rounds(rounds)) return fail(PC_EINVAL, "rounds must be 8, 12 or 20, got %d", rounds);
  if (n == 0) return PC_OK;
  if (!in || !out) return fail(PC_EINVAL, "in/out is NULL");
  if (!vaddrs && (vaddr0 & 4095)) return fail(PC_EINVAL, "vaddr0 %#llx not page-aligned", (unsigned long long)vaddr0);
  if (!vaddrs && n > 1 && vaddr0 + 4096ull * (n - 1) < vaddr0)
    return fail(PC_EINVAL, "contiguous vaddr range overflows u64");
  if (vaddrs)
    for (size_t i = 0; i < n; ++i)
      if (vaddrs[i] & 4095) return fail(PC_EINVAL, "vaddr %#llx not page-aligned", (unsigned long long)vaddrs[i]);
  if (!raw_key) {
    // fault-sized host batches on the key's resident workers: one ticket
    // per page, spread over the workers, no launch (the shared lock keeps a
    // concurrent pc_key_service stop from freeing them under us)
    std::shared_lock<std::shared_mutex> sl(const_cast<pc_key *>(key)->svc_mu);
    const int64_t lim = tuning().svc_pages.load();
    // auto: one page per worker, at most 6 -- each ticket costs the host
    // ~1.2 us of copies and doorbell work, and a worker's second ticket waits
    // for its first, so beyond that one launch is faster
    // (profiles/r02_key_service_sweep.json)
    const size_t max_pages = std::min<size_t>(
        kSvcMaxPages, lim > 0 ? static_cast<size_t>(lim) : std::min<size_t>(6, static_cast<size_t>(key->svc_workers)));
    if (key->svc && key->svc_rounds == rounds && n <= max_pages) {
      const PtrInfo a = ptr_info(in), b = ptr_info(out);
      if (!a.dev && !b.dev) return crypt_on_service(key, vaddrs, pids, vaddr0, pid0, in, out, n);
    }
  }
  std::lock_guard<std::mutex> lk(e->mu);
  DeviceGuard g(e->device);
  CU(g.err);
  const PtrInfo pin = ptr_info(in), pout = ptr_info(out);
  const bool din = pin.dev, dout = pout.dev;
  const int gin = pin.device, gout = pout.device;
  if (n <= tuning().small_max && !din && !dout)
    return crypt_small(e, raw_key ? nullptr : key->d_words, raw_key, vaddrs, pids, vaddr0, pid0, in, out, n, rounds,
                       pin.host_dev, pout.host_dev);
  if (din && dout && gin == e->device && gout == e->device && !vaddrs && !pids && !raw_key &&
      tuning().dev_direct.load()) {
    // pages already in this GPU's memory: one in-place launch, no staging
    const pc::PageDesc d{nullptr, nullptr, vaddr0, pid0};
    int rc = launch_crypt(key->d_words, d, in, out, n, rounds, e->streams[0]);
    if (rc != PC_OK) return rc;
    CU(cudaStreamSynchronize(e->streams[0]));
    return PC_OK;
  }
  if (din && dout && gin == gout && gin != e->device && !vaddrs && !pids && !raw_key &&
      tuning().peer_direct.load() && peer_access(e->device, gin)) {
    // pages in a peer GPU's memory (NVLink/NVSwitch): this GPU's kernel reads
    // and writes them in place over the fabric -- the scatter, the cipher and
    // the gather are one kernel, with no staging copies.  The coalesced
    // variant keeps every warp access a 512-byte contiguous run.
    const pc::PageDesc d{nullptr, nullptr, vaddr0, pid0};
    int rc = launch_crypt(key->d_words, d, in, out, n, rounds, e->streams[0], 3);
    if (rc != PC_OK) return rc;
    CU(cudaStreamSynchronize(e->streams[0]));
    return PC_OK;
  }
  const uint32_t *dkey = nullptr;
  if (raw_key) {
    std::memcpy(e->h_key, raw_key, 32);
    cudaError_t err = cudaMemcpyAsync(e->d_rawkey, e->h_key, 32, cudaMemcpyHostToDevice, e->streams[0]);
    if (err == cudaSuccess) err = cudaStreamSynchronize(e->streams[0]);
    wipe(e->h_key, 32);
    CU(err);
    dkey = e->d_rawkey;
  } else {
    dkey = key->d_words;
  }
  int rc = crypt_large(e, dkey, vaddrs, pids, vaddr0, pid0, in, out, n, rounds);
  if (raw_key) {
    // drain every stream that may read the slot, then zero it
    for (auto s : e->streams) cudaStreamSynchronize(s);
    cudaError_t err = cudaMemsetAsync(e->d_rawkey, 0, 256, e->streams[0]);
    if (err == cudaSuccess) err = cudaStreamSynchronize(e->streams[0]);
    if (rc == PC_OK) CU(err);
  }
  return rc;
}

} // extern "C"

// ---- (viii) HBM page store: slab moves ------------------------------------------
namespace {
template <int R>
void launch_slab_r(int dir, const uint32_t *key, const pc::PageDesc &d, const uint32_t *slots, void *slab,
                   void *staging, size_t n, bool wipe_src, cudaStream_t st) {
  const uint64_t nb = static_cast<uint64_t>(n) * 64;
  const dim3 grid(static_cast<unsigned>((nb + 255) / 256));
  auto sl = static_cast<uint4 *>(slab);
  auto sg = static_cast<uint4 *>(staging);
  if (dir == 0) pc::k_slab_move<R, 0><<<grid, 256, 0, st>>>(key, d, slots, sl, sg, nb, false);
  else pc::k_slab_move<R, 1><<<grid, 256, 0, st>>>(key, d, slots, sl, sg, nb, wipe_src);
  counted();
}
} // namespace

extern "C" int pc_slab_transfer(pc_engine *e, const pc_key *key, void *slab, size_t slab_pages,
                                const uint32_t *slots, const uint64_t *vaddrs, const uint32_t *pids,
                                uint64_t vaddr0, uint32_t pid0, void *host, size_t n, int dir, int rounds,
                                int flags) {
  if (!e || e->magic != kEngineMagic) return fail(PC_ESTATE, "not a live pc_engine");
  const bool wipe_src = (flags & PC_SLAB_WIPE_SRC) != 0;
  if (key && (key->magic != kKeyMagic || key->device != e->device))
    return fail(PC_ESTATE, "key is not live or not on the engine's device");
  if (dir != 0 && dir != 1) return fail(PC_EINVAL, "dir must be 0 (host->slab) or 1 (slab->host)");
  if (!valid_rounds(rounds)) return fail(PC_EINVAL, "rounds must be 8, 12 or 20, got %d", rounds);
  if (n == 0) return PC_OK;
  if (!slab || !slots || !host) return fail(PC_EINVAL, "slab/slots/host is NULL");
  if (reinterpret_cast<uintptr_t>(slab) & 15) return fail(PC_EINVAL, "slab must be 16-byte aligned");
  for (size_t i = 0; i < n; ++i)
    if (slots[i] >= slab_pages) return fail(PC_EINVAL, "slot %u outside the %zu-page slab", slots[i], slab_pages);
  if (key && !vaddrs && (vaddr0 & 4095)) return fail(PC_EINVAL, "vaddr0 not page-aligned");
  if (key && vaddrs)
    for (size_t i = 0; i < n; ++i)
      if (vaddrs[i] & 4095) return fail(PC_EINVAL, "vaddr %#llx not page-aligned", (unsigned long long)vaddrs[i]);
  std::lock_guard<std::mutex> lk(e->mu);
  DeviceGuard g(e->device);
  CU(g.err);
  if (n <= std::min<size_t>(64, tuning().small_max.load())) {
    // small batch (a fault's refault/evict): one zero-copy launch over the
    // engine's mapped staging -- slots, vaddrs and pages read/written by the
    // kernel across PCIe, no DMA round trips
    uint8_t *h = e->h_small;
    uint8_t *hd = e->hd_small;
    std::memcpy(h, slots, n * 4);
    // staging layout: slots [0,256) | vaddrs [256,768) | pids [768,1024) | pages
    if (key && vaddrs) std::memcpy(h + 256, vaddrs, n * 8);
    if (key && pids) std::memcpy(h + 768, pids, n * 4);
    if (dir == 0) std::memcpy(h + 1024, host, n * PC_PAGE_SIZE);
    const pc::PageDesc d{key && vaddrs ? reinterpret_cast<const uint64_t *>(hd + 256) : nullptr,
                         key && pids ? reinterpret_cast<const uint32_t *>(hd + 768) : nullptr, vaddr0, pid0};
    const uint32_t *k = key ? key->d_words : nullptr;
    cudaStream_t st = e->streams[0];
    switch (rounds) {
      case 8: launch_slab_r<8>(dir, k, d, reinterpret_cast<const uint32_t *>(hd), slab, hd + 1024, n, wipe_src, st); break;
      case 12: launch_slab_r<12>(dir, k, d, reinterpret_cast<const uint32_t *>(hd), slab, hd + 1024, n, wipe_src, st); break;
      default: launch_slab_r<20>(dir, k, d, reinterpret_cast<const uint32_t *>(hd), slab, hd + 1024, n, wipe_src, st); break;
    }
    cudaError_t err = cudaGetLastError();
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (err == cudaSuccess) err = e2;
    if (err == cudaSuccess && dir == 1) std::memcpy(host, h + 1024, n * PC_PAGE_SIZE);
    wipe(h + 1024, n * PC_PAGE_SIZE); // plaintext passed through the staging
    CU(err);
    return PC_OK;
  }
  void *host_dev = nullptr;
  const bool pinned = pinned_alias(host, &host_dev);
  const int S = e->n_streams;
  const size_t C = e->chunk_pages;
  if (!pinned) {
    pc::NodeScope near_gpu(e->place);
    for (int s = 0; s < S; ++s)
      if (!e->h_bounce[s]) CU(pinned_get(reinterpret_cast<void **>(&e->h_bounce[s]), C * PC_PAGE_SIZE));
    if (!e->pool) e->pool.reset(new pc::HostPool(host_pool_threads(), e->place));
  }
  auto *hb = static_cast<uint8_t *>(host);
  const size_t n_chunks = (n + C - 1) / C;
  auto finish = [&](size_t c) -> int { // wait for chunk c; deliver bounce -> host for gets
    const int s = static_cast<int>(c % S);
    CU(cudaEventSynchronize(e->done[s]));
    if (dir == 1 && !pinned) {
      const size_t p0 = c * C, m = std::min(C, n - p0);
      e->pool->memcpy(hb + p0 * PC_PAGE_SIZE, e->h_bounce[s], m * PC_PAGE_SIZE);
      wipe(e->h_bounce[s], m * PC_PAGE_SIZE); // plaintext left the pipeline
    }
    return PC_OK;
  };
  for (size_t c = 0; c < n_chunks; ++c) {
    const int s = static_cast<int>(c % S);
    cudaStream_t st = e->streams[s];
    const size_t p0 = c * C, m = std::min(C, n - p0);
    if (c >= static_cast<size_t>(S)) {
      int rc = finish(c - S);
      if (rc != PC_OK) return rc;
    }
    uint8_t *hd = e->h_desc[s];
    std::memcpy(hd + C * 12, slots + p0, m * 4);
    uint32_t *d_slots = e->d_pids[s] + C;
    CU(cudaMemcpyAsync(d_slots, hd + C * 12, m * 4, cudaMemcpyHostToDevice, st));
    pc::PageDesc d{nullptr, nullptr, vaddr0 + 4096ull * p0, pid0};
    if (key && vaddrs) {
      std::memcpy(hd, vaddrs + p0, m * 8);
      CU(cudaMemcpyAsync(e->d_vaddrs[s], hd, m * 8, cudaMemcpyHostToDevice, st));
      d.vaddrs = e->d_vaddrs[s];
    }
    if (key && pids) {
      std::memcpy(hd + C * 8, pids + p0, m * 4);
      CU(cudaMemcpyAsync(e->d_pids[s], hd + C * 8, m * 4, cudaMemcpyHostToDevice, st));
      d.pids = e->d_pids[s];
    }
    uint8_t *staging = e->d_pages[s];
    if (dir == 0) {
      const uint8_t *src = hb + p0 * PC_PAGE_SIZE;
      if (!pinned) {
        e->pool->memcpy(e->h_bounce[s], src, m * PC_PAGE_SIZE);
        src = e->h_bounce[s];
      }
      CU(cudaMemcpyAsync(staging, src, m * PC_PAGE_SIZE, cudaMemcpyHostToDevice, st));
    }
    const uint32_t *k = key ? key->d_words : nullptr;
    switch (rounds) {
      case 8: launch_slab_r<8>(dir, k, d, d_slots, slab, staging, m, wipe_src, st); break;
      case 12: launch_slab_r<12>(dir, k, d, d_slots, slab, staging, m, wipe_src, st); break;
      default: launch_slab_r<20>(dir, k, d, d_slots, slab, staging, m, wipe_src, st); break;
    }
    CU(cudaGetLastError());
    if (dir == 1) {
      uint8_t *dst = pinned ? hb + p0 * PC_PAGE_SIZE : e->h_bounce[s];
      CU(cudaMemcpyAsync(dst, staging, m * PC_PAGE_SIZE, cudaMemcpyDeviceToHost, st));
    }
    // the staging slot held plaintext (evict input / refault output): zero it
    CU(cudaMemsetAsync(staging, 0, m * PC_PAGE_SIZE, st));
    CU(cudaEventRecord(e->done[s], st));
  }
  const size_t first = n_chunks > static_cast<size_t>(S) ? n_chunks - S : 0;
  for (size_t c = first; c < n_chunks; ++c) {
    int rc = finish(c);
    if (rc != PC_OK) return rc;
  }
  if (dir == 0 && !pinned)
    for (int s = 0; s < S; ++s) wipe(e->h_bounce[s], std::min(C, n) * PC_PAGE_SIZE);
  return PC_OK;
}

extern "C" int pc_slab_wipe(pc_engine *e, void *slab, size_t slab_pages, const uint32_t *slots, size_t n) {
  if (!e || e->magic != kEngineMagic) return fail(PC_ESTATE, "not a live pc_engine");
  if (n == 0) return PC_OK;
  if (!slab || !slots) return fail(PC_EINVAL, "slab/slots is NULL");
  for (size_t i = 0; i < n; ++i)
    if (slots[i] >= slab_pages) return fail(PC_EINVAL, "slot %u outside the %zu-page slab", slots[i], slab_pages);
  std::lock_guard<std::mutex> lk(e->mu);
  DeviceGuard g(e->device);
  CU(g.err);
  cudaStream_t st = e->streams[0];
  const size_t C = e->chunk_pages;
  for (size_t p0 = 0; p0 < n; p0 += C) {
    const size_t m = std::min(C, n - p0);
    std::memcpy(e->h_desc[0] + C * 12, slots + p0, m * 4);
    uint32_t *d_slots = e->d_pids[0] + C;
    CU(cudaMemcpyAsync(d_slots, e->h_desc[0] + C * 12, m * 4, cudaMemcpyHostToDevice, st));
    const uint64_t chunks = static_cast<uint64_t>(m) * 256;
    pc::k_slab_wipe<<<static_cast<unsigned>((chunks + 255) / 256), 256, 0, st>>>(d_slots, static_cast<uint4 *>(slab), chunks);
    counted();
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st)); // h_desc[0] is reused by the next piece
  }
  return PC_OK;
}

extern "C" {
// ---- (vi) multi-device partition --------------------------------------------
int pc_desc_check(const uint64_t *vaddrs, const int64_t *pids64, uint32_t *pids32, size_t n, void *stream,
                  uint32_t *flags) {
  if (!flags) return fail(PC_EINVAL, "flags is NULL");
  *flags = 0;
  if (n == 0 || (!vaddrs && !pids64)) return PC_OK;
  if (pids64 && !pids32) return fail(PC_EINVAL, "pids32 is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0;
  // the launch must run on the stream's own device, whatever is current
  CU(st ? cudaStreamGetDevice(st, &dev) : cudaGetDevice(&dev));
  DeviceGuard g(dev);
  CU(g.err);
  Scratch &sc = scratch(dev);
  std::lock_guard<std::mutex> lk(sc.mu);
  int rc = scratch_reserve(sc, 256);
  if (rc != PC_OK) return rc;
  uint32_t *d_flag = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void **>(&d_flag), 4, st)); // stream-ordered: safe beside the service
  cudaError_t e = cudaMemsetAsync(d_flag, 0, 4, st);
  if (e == cudaSuccess) {
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096));
    pc::k_desc_check<<<grid, 256, 0, st>>>(vaddrs, pids64, pids32, n, d_flag);
    counted();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(sc.h, d_flag, 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e2 = cudaFreeAsync(d_flag, st);
  cudaError_t e3 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e2 != cudaSuccess ? e2 : e3;
  CU(e);
  std::memcpy(flags, sc.h, 4);
  return PC_OK;
}

int pc_crypt_pages_multi(pc_engine *const *engines, const pc_key *const *keys, int n_dev,
                         const uint64_t *vaddrs, const uint32_t *pids, uint64_t vaddr0, uint32_t pid0,
                         const void *in, void *out, size_t n, int rounds) {
  if (!engines || !keys || n_dev <= 0) return fail(PC_EINVAL, "need >= 1 engine and key");
  for (int g = 0; g < n_dev; ++g)
    if (!engines[g] || engines[g]->magic != kEngineMagic) return fail(PC_ESTATE, "engine %d is not live", g);
  std::vector<int> rcs(n_dev, PC_OK);
  std::vector<std::string> errs(n_dev);
  auto job = [&](int g) {
    const size_t lo = n * g / n_dev, hi = n * (g + 1) / n_dev;
    if (hi == lo) return;
    rcs[g] = pc_crypt_pages_host(engines[g], keys[g], nullptr, vaddrs ? vaddrs + lo : nullptr,
                                 pids ? pids + lo : nullptr, vaddr0 + 4096ull * lo, pid0,
                                 static_cast<const uint8_t *>(in) + lo * PC_PAGE_SIZE,
                                 static_cast<uint8_t *>(out) + lo * PC_PAGE_SIZE, hi - lo, rounds);
    if (rcs[g] != PC_OK) errs[g] = pc_last_error();
  };
  // engines 1..G-1 run on their persistent runner threads, engine 0 here
  std::vector<std::function<void()>> waits;
  for (int g = 1; g < n_dev; ++g) {
    pc_engine *e = engines[g];
    {
      std::lock_guard<std::mutex> lk(e->runner_mu);
      if (!e->runner) e->runner.reset(new pc::Runner(e->place));
    }
    waits.push_back(e->runner->submit([&job, g] { job(g); }));
  }
  job(0);
  for (auto &w : waits) w();
  for (int g = 0; g < n_dev; ++g)
    if (rcs[g] != PC_OK) return fail(rcs[g], "device slot %d: %s", g, errs[g].c_str());
  return PC_OK;
}

} // extern "C"

// ---- module preloading ------------------------------------------------------------
// With CUDA's default lazy module loading, the first launch of a kernel loads
// it into the context, and that load waits for the context to go idle -- it
// deadlocks behind a persistent kernel (measured: tools/diag/persistent_probe).
// pc_preload loads every kernel of this library up front; pc_service_start
// calls it before launching the service.
namespace {
template <typename F>
cudaError_t touch(F *fn) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, fn);
}

template <int R>
cudaError_t touch_rounds() {
  cudaError_t e = cudaSuccess;
  auto acc = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  for (uint32_t m : kRotMasks) (void)m;
  acc(touch(pc::k_crypt_blocks<R, 0x00000000u>));
  acc(touch(pc::k_crypt_blocks<R, 0x88888888u>));
  acc(touch(pc::k_crypt_blocks<R, 0x888888AAu>));
  acc(touch(pc::k_crypt_blocks<R, 0x88888AAAu>));
  acc(touch(pc::k_crypt_blocks<R, 0xAAAA8888u>));
  acc(touch(pc::k_crypt_blocks<R, 0xAAAAAAAAu>));
  acc(touch(pc::k_crypt_pages<R>));
  acc(touch(pc::k_crypt_pages_coalesced<R>));
  acc(touch(pc::k_crypt_pages_tma<R, kTmaStages>));
  acc(touch(pc::k_crypt_pages_async<R, 0>));
  acc(touch(pc::k_crypt_pages_async<R, 1>));
  acc(touch(pc::k_crypt_pages_async<R, 2>));
  acc(touch(pc::k_crypt_pages_async<R, 3>));
  if constexpr (R <= PC_RUN_MAX_R) {
    acc(touch(pc::k_crypt_pages_run<R, 1>));
    acc(touch(pc::k_crypt_pages_run<R, 2>));
    acc(touch(pc::k_crypt_pages_run<R, 3>));
  }
  acc(touch(pc::k_crypt_pages_run2<R, 1>));
  acc(touch(pc::k_crypt_pages_run2<R, 2>));
  acc(touch(pc::k_crypt_pages_run2<R, 3>));
  acc(v6_opt_in<R, 0>()); // loads the module and sets the shared-memory opt-in
  acc(v6_opt_in<R, 1>());
  acc(v6_opt_in<R, 2>());
  acc(v6_opt_in<R, 3>());
  acc(v9_opt_in<R>());
  acc(touch(pc::k_keystream_seeds<R>));
  acc(touch(pc::k_service<R>));
  acc(touch(pc::k_slab_move<R, 0>));
  acc(touch(pc::k_slab_move<R, 1>));
  acc(touch(pc::k_slab_swap<R>));
  return e;
}
} // namespace

extern "C" int pc_preload(int device) {
  DeviceGuard g(device);
  CU(g.err);
  CU(touch_rounds<8>());
  CU(touch_rounds<12>());
  CU(touch_rounds<20>());
  CU(touch(pc::k_keygen));
  CU(touch(pc::k_page_seed_table));
  if (!seed_pool(device)) return fail(PC_ECUDA, "seed pool");
  CU(touch(pc::k_slab_wipe));
  CU(touch(pc::k_desc_check));
  CU(touch(pc::k_intpeak<0>));
  CU(touch(pc::k_intpeak<1>));
  CU(touch(pc::k_intpeak<2>));
  CU(touch(pc::k_intpeak<3>));
  CU(touch(pc::k_intpeak<4>));
  CU(touch(pc::k_intpeak<5>));
  CU(touch(pc::k_intpeak<6>));
  CU(touch(pc::k_intpeak<7>));
  return PC_OK;
}

// ---- (vii) persistent crypto-worker service -------------------------------------
namespace {
constexpr uint32_t kServiceMagic = 0x73766331u; // "svc1"

int service_launch(int rounds, int workers, cudaStream_t st, const uint32_t *key, pc::SvcSlot *slots,
                   uint4 *pages, uint32_t ring, const pc::SvcBell *bell, const uint32_t *stop, uint32_t *started,
                   pc::SvcDev *dev, uint4 *hdr, const pc::SvcOp *ops, uint4 *store_slab) {
  // direct: every worker polls its own doorbell; else one extra CTA is the dispatcher
  // auto (2): direct polling while few workers poll -- 8.6 vs 10.0 us per
  // 1-page request at 16 workers, but 148 pollers congest PCIe (11.2 us)
  const int sd = tuning().svc_direct.load();
  const uint32_t direct = (sd == 1 || (sd == 2 && workers <= 32)) ? 1u : 0u;
  const unsigned grid = static_cast<unsigned>(workers) + (direct ? 0 : 1);
  const uint32_t nw = static_cast<uint32_t>(workers);
  switch (rounds) {
    case 8: pc::k_service<8><<<grid, 64, 0, st>>>(key, slots, pages, ring, nw, bell, stop, started, dev, hdr, direct, ops, store_slab); break;
    case 12: pc::k_service<12><<<grid, 64, 0, st>>>(key, slots, pages, ring, nw, bell, stop, started, dev, hdr, direct, ops, store_slab); break;
    default: pc::k_service<20><<<grid, 64, 0, st>>>(key, slots, pages, ring, nw, bell, stop, started, dev, hdr, direct, ops, store_slab); break;
  }
  counted();
  CU(cudaGetLastError());
  return PC_OK;
}

// Enable peer access both ways between `dev` and every GPU this process
// already has a context on (a device with no context is left alone: creating
// contexts on every GPU of the node from every rank would cost HBM on each).
void enable_peers_of(int dev) {
  using GetState = int (*)(int, unsigned *, int *);
  static GetState get_state = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuDevicePrimaryCtxGetState", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<GetState>(f);
  }();
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || !get_state) {
    cudaGetLastError();
    return;
  }
  for (int p = 0; p < n; ++p) {
    if (p == dev) continue;
    unsigned flags = 0;
    int active = 0;
    if (get_state(p, &flags, &active) != 0 || !active) continue; // CUdevice == ordinal
    peer_access(dev, p);
    peer_access(p, dev);
  }
}

inline void cpu_relax() {
#if defined(__x86_64__)
  __builtin_ia32_pause();
#endif
}
} // namespace

struct pc_service {
  uint32_t magic = kServiceMagic;
  int device = 0;
  int n_workers = 0;
  uint32_t ring = 0;
  int rounds = 20;
  cudaStream_t st = nullptr;
  pc::SvcSlot *h_slots = nullptr, *d_slots = nullptr; // mapped pinned
  uint8_t *h_pages = nullptr, *d_pages = nullptr;     // mapped pinned
  uint32_t *h_ctrl = nullptr, *d_ctrl = nullptr;      // [0] stop, [64..] started[w]
  pc::SvcBell *h_bell = nullptr, *d_bell = nullptr;   // per worker: tickets published (in order) + header
  pc::SvcDev *dev = nullptr;                          // device-memory doorbell mirror
  pc::SvcOp *h_ops = nullptr, *d_ops = nullptr;       // mapped pinned: per slot, a store op's line
  uint64_t key_serial = 0;                            // the key the workers hold (pc_key::serial)
  uint4 *store_slab = nullptr;                        // a store's own service: its slab (pc_store_service)
  uint4 *hdr = nullptr;                               // forwarded headers, n_workers x ring
  // Host-side slot protocol.  Slot j of a worker carries tickets j, j+R, ...
  //   next[j]  = the ticket whose result is the next to be delivered in slot j
  //   claim[j] = ticket a finisher may claim (CAS t -> t+R) to deliver it
  //   dst[j]   = where the result of the slot's current ticket goes
  // Any thread may deliver a finished result (a waiter, a poller, or a
  // producer that needs the slot), so a full ring never deadlocks.
  std::unique_ptr<std::atomic<uint64_t>[]> tail;  // per worker: next ticket
  std::unique_ptr<std::atomic<uint64_t>[]> next;  // per slot
  std::unique_ptr<std::atomic<uint64_t>[]> claim; // per slot
  std::unique_ptr<std::atomic<void *>[]> dst;     // per slot
  std::atomic<uint64_t> in_flight{0};
  bool stopped = false;
};

extern "C" {

int pc_service_max_workers(int device, int *n) {
  if (!n) return fail(PC_EINVAL, "n is NULL");
  DeviceGuard g(device);
  CU(g.err);
  int sms = 0, occ = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pc::k_service<20>, 64, 0));
  *n = std::min(sms * std::max(occ, 1) - 1, 4096); // one CTA is the dispatcher
  return PC_OK;
}

} // extern "C"
int service_start(const pc_key *key, int n_workers, int ring_slots, int rounds, void *store_slab,
                  pc_service **out);
extern "C" {
int pc_service_start(const pc_key *key, int n_workers, int ring_slots, int rounds, pc_service **out) {
  return service_start(key, n_workers, ring_slots, rounds, nullptr, out);
}
} // extern "C"

// store_slab: the slab of the store that owns this service (its workers then
// take a store ticket's slots from the doorbell line), or NULL
int service_start(const pc_key *key, int n_workers, int ring_slots, int rounds, void *store_slab,
                  pc_service **out) {
  if (!out) return fail(PC_EINVAL, "out is NULL");
  *out = nullptr;
  if (!key || key->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  if (!valid_rounds(rounds)) return fail(PC_EINVAL, "rounds must be 8, 12 or 20, got %d", rounds);
  if (ring_slots < 1 || ring_slots > 4096 || (ring_slots & (ring_slots - 1)))
    return fail(PC_EINVAL, "ring capacity %d not a power of two in 1..4096", ring_slots);
  int maxw = 0;
  int rc = pc_service_max_workers(key->device, &maxw);
  if (rc != PC_OK) return rc;
  if (n_workers < 1 || n_workers > maxw)
    return fail(PC_EINVAL, "n_workers must be 1..%d (all workers must be co-resident), got %d", maxw, n_workers);
  DeviceGuard g(key->device);
  CU(g.err);
  rc = pc_preload(key->device); // nothing of ours may lazy-load behind the service
  if (rc != PC_OK) return rc;
  enable_peers_of(key->device); // no peer-access enable has to happen beside the kernel
  auto *s = new pc_service();
  s->device = key->device;
  s->n_workers = n_workers;
  s->ring = static_cast<uint32_t>(ring_slots);
  s->rounds = rounds;
  const size_t nslots = static_cast<size_t>(n_workers) * ring_slots;
  s->tail.reset(new std::atomic<uint64_t>[n_workers]);
  s->next.reset(new std::atomic<uint64_t>[nslots]);
  s->claim.reset(new std::atomic<uint64_t>[nslots]);
  s->dst.reset(new std::atomic<void *>[nslots]);
  for (int w = 0; w < n_workers; ++w) s->tail[w] = 0;
  for (size_t i = 0; i < nslots; ++i) {
    s->next[i] = i % ring_slots;
    s->claim[i] = i % ring_slots;
    s->dst[i] = nullptr;
  }
  auto bail = [&](int code) {
    if (s->dev) cudaFreeAsync(s->dev, s->st);
    if (s->hdr) cudaFreeAsync(s->hdr, s->st);
    if (s->dev || s->hdr) cudaStreamSynchronize(s->st);
    const size_t ns = static_cast<size_t>(s->n_workers) * s->ring;
    pinned_put(s->h_slots, ns * sizeof(pc::SvcSlot));
    pinned_put(s->h_pages, ns * PC_PAGE_SIZE);
    pinned_put(s->h_ctrl, (64 + static_cast<size_t>(s->n_workers)) * 4);
    pinned_put(s->h_bell, s->n_workers * pc::kBellStride * sizeof(pc::SvcBell));
    pinned_put(s->h_ops, ns * sizeof(pc::SvcOp));
    if (s->st) cudaStreamDestroy(s->st);
    delete s;
    return code;
  };
#define CUS(call)                                                                       \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) return bail(fail(PC_ECUDA, "%s: %s", #call, cudaGetErrorString(e_))); \
  } while (0)
  CUS(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
  CUS(pinned_get(reinterpret_cast<void **>(&s->h_slots), nslots * sizeof(pc::SvcSlot)));
  CUS(pinned_get(reinterpret_cast<void **>(&s->h_pages), nslots * PC_PAGE_SIZE));
  const size_t ctrl_bytes = (64 + static_cast<size_t>(n_workers)) * 4;
  CUS(pinned_get(reinterpret_cast<void **>(&s->h_ctrl), ctrl_bytes));
  std::memset(s->h_slots, 0, nslots * sizeof(pc::SvcSlot));
  std::memset(s->h_pages, 0, nslots * PC_PAGE_SIZE);
  std::memset(s->h_ctrl, 0, ctrl_bytes);
  CUS(cudaHostGetDevicePointer(reinterpret_cast<void **>(&s->d_slots), s->h_slots, 0));
  CUS(cudaHostGetDevicePointer(reinterpret_cast<void **>(&s->d_pages), s->h_pages, 0));
  CUS(cudaHostGetDevicePointer(reinterpret_cast<void **>(&s->d_ctrl), s->h_ctrl, 0));
  CUS(pinned_get(reinterpret_cast<void **>(&s->h_bell), n_workers * pc::kBellStride * sizeof(pc::SvcBell)));
  std::memset(s->h_bell, 0, n_workers * pc::kBellStride * sizeof(pc::SvcBell));
  CUS(cudaHostGetDevicePointer(reinterpret_cast<void **>(&s->d_bell), s->h_bell, 0));
  CUS(pinned_get(reinterpret_cast<void **>(&s->h_ops), nslots * sizeof(pc::SvcOp)));
  std::memset(s->h_ops, 0, nslots * sizeof(pc::SvcOp));
  CUS(cudaHostGetDevicePointer(reinterpret_cast<void **>(&s->d_ops), s->h_ops, 0));
  CUS(cudaMallocAsync(reinterpret_cast<void **>(&s->dev), sizeof(pc::SvcDev), s->st));
  CUS(cudaMemsetAsync(s->dev, 0, sizeof(pc::SvcDev), s->st));
  CUS(cudaMallocAsync(reinterpret_cast<void **>(&s->hdr), nslots * sizeof(uint4), s->st));
  CUS(cudaMemsetAsync(s->hdr, 0xff, nslots * sizeof(uint4), s->st)); // tags match no ticket
  CUS(cudaStreamSynchronize(s->st));
#undef CUS
  // the kernel reads the key once; it must be resident before we report success
  rc = service_launch(rounds, n_workers, s->st, key->d_words, s->d_slots, reinterpret_cast<uint4 *>(s->d_pages),
                      s->ring, s->d_bell, s->d_ctrl, s->d_ctrl + 64, s->dev, s->hdr, s->d_ops,
                      static_cast<uint4 *>(store_slab));
  if (rc != PC_OK) return bail(rc);
  const auto t0 = std::chrono::steady_clock::now();
  volatile uint32_t *started = s->h_ctrl + 64;
  for (int w = 0; w < n_workers; ++w) {
    while (started[w] == 0) {
      if (cudaStreamQuery(s->st) != cudaErrorNotReady) {
        cudaError_t e = cudaStreamSynchronize(s->st);
        return bail(fail(PC_ECUDA, "service kernel exited during start: %s", cudaGetErrorString(e)));
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20)) {
        s->h_ctrl[0] = 1; // ask the resident workers to leave
        cudaStreamSynchronize(s->st);
        return bail(fail(PC_ETIMEOUT, "service workers did not start (%d of %d)", w, n_workers));
      }
      std::this_thread::yield();
    }
  }
  s->key_serial = key->serial;
  s->store_slab = static_cast<uint4 *>(store_slab);
  g_services_on[s->device].fetch_add(1);
  *out = s;
  return PC_OK;
}
extern "C" {

} // extern "C"

namespace {
inline size_t svc_slot(const pc_service *s, int worker, uint64_t t) {
  return static_cast<size_t>(worker) * s->ring + (t % s->ring);
}

// Deliver ticket t's result if the GPU has finished it and nobody else is
// delivering it.  Returns true when t is delivered (by us or someone else).
bool svc_try_finish(pc_service *s, int worker, uint64_t t) {
  const size_t slot = svc_slot(s, worker, t);
  if (s->next[slot].load(std::memory_order_acquire) > t) return true;
  const uint64_t d = *reinterpret_cast<volatile uint64_t *>(&s->h_slots[slot].done_seq);
  if (d != t + 1) return false;
  uint64_t expect = t;
  if (!s->claim[slot].compare_exchange_strong(expect, t + s->ring, std::memory_order_acq_rel))
    return false; // another thread is delivering it
  std::atomic_thread_fence(std::memory_order_acquire);
  uint8_t *page = s->h_pages + slot * PC_PAGE_SIZE;
  void *dst = s->dst[slot].load(std::memory_order_acquire);
  if (dst) std::memcpy(dst, page, PC_PAGE_SIZE);
  wipe(page, PC_PAGE_SIZE); // the ring page held a plaintext or ciphertext copy
  s->dst[slot].store(nullptr, std::memory_order_relaxed);
  s->in_flight.fetch_sub(1, std::memory_order_relaxed);
  s->next[slot].store(t + s->ring, std::memory_order_release);
  return true;
}

int svc_check(pc_service *s, int worker) {
  if (!s || s->magic != kServiceMagic) return fail(PC_ESTATE, "not a live pc_service");
  if (worker < 0 || worker >= s->n_workers) return fail(PC_EINVAL, "worker %d out of range", worker);
  return PC_OK;
}
} // namespace

extern "C" {

} // extern "C"

namespace {
// Publish one ticket: the page (src, or nothing when src is NULL: the ring
// page was wiped when its last result was delivered), the header, the op
// line of a store op (op != NULL; its flags ride in vaddr's low 12 bits),
// then the doorbell, in ticket order.
int svc_submit(pc_service *s, int worker, uint64_t vaddr, uint32_t pid, const void *src, void *dst,
               const pc::SvcOp *op, uint64_t *ticket) {
  const uint64_t t = s->tail[worker].fetch_add(1, std::memory_order_relaxed);
  const size_t slot = svc_slot(s, worker, t);
  // back-pressure (WorkerRing.push blocks while full): the slot's previous
  // ticket must be delivered; help deliver it if the GPU is done with it
  uint32_t spins = 0;
  while (s->next[slot].load(std::memory_order_acquire) != t) {
    if (t >= s->ring) svc_try_finish(s, worker, t - s->ring);
    if (++spins > 64) std::this_thread::yield();
    else cpu_relax();
  }
  s->in_flight.fetch_add(1, std::memory_order_relaxed);
  pc::SvcSlot *sl = s->h_slots + slot;
  if (src) std::memcpy(s->h_pages + slot * PC_PAGE_SIZE, src, PC_PAGE_SIZE);
  if (op) s->h_ops[slot] = *op;
  s->dst[slot].store(dst, std::memory_order_relaxed);
  sl->vaddr = vaddr;
  sl->pid = pid;
  std::atomic_thread_fence(std::memory_order_release);
  // publish in ticket order: the doorbell counts consecutive published
  // tickets; the header of the newest one rides along (dispatcher fast path)
  pc::SvcBell *hb = s->h_bell + static_cast<size_t>(worker) * pc::kBellStride;
  auto *count = reinterpret_cast<std::atomic<uint32_t> *>(&hb->count);
  uint32_t bspins = 0;
  while (count->load(std::memory_order_acquire) != static_cast<uint32_t>(t)) {
    if (++bspins > 64) std::this_thread::yield();
    else cpu_relax();
  }
  // a store's own service: the newest ticket's slots ride in the doorbell
  // line (tagged with the ticket), written before the doorbell
  if (s->store_slab) {
    const __m128i o = op && tuning().svc_bell_ops.load() ? _mm_set_epi32(static_cast<int>(op->put_slot), static_cast<int>(op->get_slot),
                                         static_cast<int>(op->evict_vaddr >> 32),
                                         static_cast<int>((op->evict_vaddr & ~uint64_t(4095)) | pc::op_tag(t)))
                         : _mm_setzero_si128();
    _mm_store_si128(reinterpret_cast<__m128i *>(hb + 1), o);
  }
  // count, pid and vaddr in ONE aligned 16-byte store (atomic on x86-64
  // CPUs with AVX), so the dispatcher's 16-byte read never sees a count
  // paired with another ticket's header
  std::atomic_thread_fence(std::memory_order_release);
  const __m128i v = _mm_set_epi64x(static_cast<long long>(vaddr),
                                   static_cast<long long>((static_cast<uint64_t>(pid) << 32) |
                                                          static_cast<uint32_t>(t + 1)));
  _mm_store_si128(reinterpret_cast<__m128i *>(hb), v);
  *ticket = t;
  return PC_OK;
}
} // namespace

extern "C" {

int pc_service_submit(pc_service *s, int worker, uint64_t vaddr, uint32_t pid, const void *src, void *dst,
                      uint64_t *ticket) {
  int rc = svc_check(s, worker);
  if (rc != PC_OK) return rc;
  if (s->stopped) return fail(PC_ESTATE, "service is not running");
  if (!src || !ticket) return fail(PC_EINVAL, "src/ticket is NULL");
  if (vaddr & 4095) return fail(PC_EINVAL, "vaddr %#llx not page-aligned", (unsigned long long)vaddr);
  return svc_submit(s, worker, vaddr, pid, src, dst, nullptr, ticket);
}

int pc_service_poll(pc_service *s, int worker, uint64_t t, int *done) {
  int rc = svc_check(s, worker);
  if (rc != PC_OK) return rc;
  if (!done) return fail(PC_EINVAL, "done is NULL");
  if (t >= s->tail[worker].load(std::memory_order_relaxed)) return fail(PC_EINVAL, "ticket %llu not issued", (unsigned long long)t);
  *done = svc_try_finish(s, worker, t) ? 1 : 0;
  return PC_OK;
}

int pc_service_wait(pc_service *s, int worker, uint64_t t, int64_t timeout_us) {
  int rc = svc_check(s, worker);
  if (rc != PC_OK) return rc;
  if (t >= s->tail[worker].load(std::memory_order_relaxed)) return fail(PC_EINVAL, "ticket %llu not issued", (unsigned long long)t);
  const auto t0 = std::chrono::steady_clock::now();
  uint32_t spins = 0;
  while (!svc_try_finish(s, worker, t)) {
    if (++spins < 4096) {
      cpu_relax();
      continue;
    }
    spins = 0;
    if (timeout_us >= 0 && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(timeout_us))
      return fail(PC_ETIMEOUT, "timed out waiting for crypto completion");
    if (cudaStreamQuery(s->st) != cudaErrorNotReady) return fail(PC_ECUDA, "service kernel is no longer running");
    std::this_thread::yield();
  }
  return PC_OK;
}

int pc_service_crypt(pc_service *s, int worker, uint64_t vaddr, uint32_t pid, const void *src, void *dst,
                     int64_t timeout_us) {
  uint64_t t = 0;
  int rc = pc_service_submit(s, worker, vaddr, pid, src, dst, &t);
  if (rc != PC_OK) return rc;
  return pc_service_wait(s, worker, t, timeout_us);
}

int pc_service_timing(pc_service *s, int worker, uint64_t t, uint64_t out_ns[4]) {
  int rc = svc_check(s, worker);
  if (rc != PC_OK) return rc;
  if (!out_ns) return fail(PC_EINVAL, "out is NULL");
  const pc::SvcSlot *sl = s->h_slots + svc_slot(s, worker, t);
  for (int i = 0; i < 4; ++i) out_ns[i] = reinterpret_cast<const volatile uint64_t *>(sl->t_ns)[i];
  return PC_OK;
}

// Diagnostic: the SM a worker runs on (recorded when it started).
int pc_service_worker_sm(pc_service *s, int worker, int *smid) {
  int rc = svc_check(s, worker);
  if (rc != PC_OK) return rc;
  if (!smid) return fail(PC_EINVAL, "smid is NULL");
  *smid = static_cast<int>(reinterpret_cast<volatile uint32_t *>(s->h_ctrl + 64)[worker]) - 1;
  return PC_OK;
}

int pc_service_in_flight(pc_service *s, uint64_t *n) {
  if (!s || s->magic != kServiceMagic) return fail(PC_ESTATE, "not a live pc_service");
  if (!n) return fail(PC_EINVAL, "n is NULL");
  *n = s->in_flight.load();
  return PC_OK;
}

// Resident workers for one key (section vii kernel, started from this key):
// while they run, pc_crypt_pages_host batches of up to svc_pages host pages
// under this key and round count are service tickets instead of launches.
int pc_key_service(pc_key *key, int n_workers, int rounds) {
  if (!key || key->magic != kKeyMagic) return fail(PC_ESTATE, "not a live pc_key");
  if (n_workers < 0) return fail(PC_EINVAL, "n_workers must be >= 0, got %d", n_workers);
  std::unique_lock<std::shared_mutex> xl(key->svc_mu);
  if (n_workers == 0) {
    if (!key->svc) return PC_OK;
    int rc = pc_service_stop(key->svc);
    if (rc != PC_OK) return rc;
    key->svc = nullptr;
    key->svc_workers = 0;
    key->svc_rounds = 0;
    return PC_OK;
  }
  if (key->svc) return fail(PC_ESTATE, "key already has resident workers");
  if (!valid_rounds(rounds)) return fail(PC_EINVAL, "rounds must be 8, 12 or 20, got %d", rounds);
  pc_service *s = nullptr;
  int rc = pc_service_start(key, n_workers, 64, rounds, &s);
  if (rc != PC_OK) return rc;
  key->svc_rounds = rounds;
  key->svc_workers = n_workers;
  key->svc = s;
  return PC_OK;
}

int pc_service_stop(pc_service *s) {
  if (!s || s->magic != kServiceMagic) return fail(PC_ESTATE, "not a live pc_service");
  const uint64_t n = s->in_flight.load();
  if (n) return fail(PC_ESTATE, "%llu requests in flight", (unsigned long long)n);
  DeviceGuard g(s->device);
  CU(g.err);
  s->stopped = true;
  *reinterpret_cast<volatile uint32_t *>(s->h_ctrl) = 1;
  cudaError_t e = cudaStreamSynchronize(s->st);
  g_services_on[s->device].fetch_sub(1);
  const size_t nslots = static_cast<size_t>(s->n_workers) * s->ring;
  wipe(s->h_pages, nslots * PC_PAGE_SIZE);
  cudaFreeAsync(s->dev, s->st);
  cudaFreeAsync(s->hdr, s->st);
  cudaStreamSynchronize(s->st);
  pinned_put(s->h_slots, nslots * sizeof(pc::SvcSlot));
  pinned_put(s->h_pages, nslots * PC_PAGE_SIZE);
  pinned_put(s->h_ctrl, (64 + static_cast<size_t>(s->n_workers)) * 4);
  pinned_put(s->h_bell, s->n_workers * pc::kBellStride * sizeof(pc::SvcBell));
  pinned_put(s->h_ops, nslots * sizeof(pc::SvcOp));
  cudaStreamDestroy(s->st);
  s->magic = 0;
  delete s;
  CU(e);
  return PC_OK;
}

} // extern "C"

extern "C" {
// ---- pinned memory ---------------------------------------------------------
int pc_host_alloc(size_t bytes, void **out) {
  if (!out) return fail(PC_EINVAL, "out is NULL");
  *out = nullptr;
  CU(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped));
  return PC_OK;
}
int pc_host_free(void *p) {
  if (p) CU(cudaFreeHost(p));
  return PC_OK;
}
int pc_host_register(void *p, size_t bytes) {
  if (!p || !bytes) return fail(PC_EINVAL, "null/empty range");
  CU(cudaHostRegister(p, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  return PC_OK;
}
int pc_host_unregister(void *p) {
  if (!p) return fail(PC_EINVAL, "null pointer");
  CU(cudaHostUnregister(p));
  return PC_OK;
}

// ---- measurement -------------------------------------------------------------
int pc_intpeak(int device, int kind, double *ops_per_s) {
  if (!ops_per_s) return fail(PC_EINVAL, "ops_per_s is NULL");
  if (kind < 0 || kind > 7) return fail(PC_EINVAL, "kind must be 0..7");
  DeviceGuard g(device);
  CU(g.err);
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  uint32_t *sink = nullptr;
  cudaStream_t st = nullptr;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CU(cudaMallocAsync(reinterpret_cast<void **>(&sink), 1024 * 4, st));
  const dim3 grid(sms * 8), block(256);
  const bool arx = kind == 4 || kind == 5;
  const int iters = arx ? 1000 : 1500;
  auto run = [&](int it) {
    switch (kind) {
      case 0: pc::k_intpeak<0><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
      case 1: pc::k_intpeak<1><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
      case 2: pc::k_intpeak<2><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
      case 3: pc::k_intpeak<3><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
      case 4: pc::k_intpeak<4><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
      case 5: pc::k_intpeak<5><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
      case 6: pc::k_intpeak<6><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
      default: pc::k_intpeak<7><<<grid, block, 0, st>>>(1u, kRotMul, it, sink); break;
    }
    counted();
  };
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  run(iters / 10); // warm-up
  float best_ms = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CU(cudaEventRecord(a, st));
    run(iters);
    CU(cudaEventRecord(b, st));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, a, b));
    best_ms = std::min(best_ms, ms);
  }
  CU(cudaGetLastError());
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFreeAsync(sink, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  // ops per iteration: ARX = 16 quarter rounds x 12 ops (op-count convention,
  // independent of how many instructions implement them); others 16 x 8 chains
  // (kind 7 counts IMAD.WIDE + its LOP3 as 2 ops).
  const double ops_per_iter = arx ? 16.0 * 12.0 : (kind == 7 ? 16.0 * 8.0 * 2.0 : 16.0 * 8.0);
  *ops_per_s = static_cast<double>(grid.x) * block.x * iters * ops_per_iter / (best_ms * 1e-3);
  return PC_OK;
}

int pc_tune(const char *knob, int64_t value) {
  if (!knob) return fail(PC_EINVAL, "knob is NULL");
  Tuning &t = tuning();
  if (!std::strcmp(knob, "rotmask")) {
    for (uint32_t m : kRotMasks)
      if (static_cast<int64_t>(m) == value) {
        t.rot_mask = m;
        return PC_OK;
      }
    return fail(PC_EINVAL, "rotmask %#llx is not a compiled variant", (unsigned long long)value);
  }
  if (!std::strcmp(knob, "svc_bell_ops")) {
    if (value != 0 && value != 1) return fail(PC_EINVAL, "svc_bell_ops must be 0 or 1");
    t.svc_bell_ops = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "run_desc")) {
    if (value < 0 || value > 2) return fail(PC_EINVAL, "run_desc must be 0, 1 or 2");
    t.run_desc = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "svc_pages")) {
    if (value < 0 || value > 64) return fail(PC_EINVAL, "svc_pages must be 0..64");
    t.svc_pages = value;
    return PC_OK;
  }
  if (!std::strcmp(knob, "small_mode")) {
    if (value != 0 && value != 1) return fail(PC_EINVAL, "small_mode must be 0 or 1");
    t.small_mode = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "kernel")) {
    if (value < 0 || (value > 6 && value != 9)) return fail(PC_EINVAL, "kernel must be 0 (auto), 1..6 or 9");
    t.kernel = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "svc_direct")) {
    if (value < 0 || value > 2) return fail(PC_EINVAL, "svc_direct must be 0, 1 or 2 (auto)");
    t.svc_direct = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "peer_direct")) {
    if (value < 0 || value > 1) return fail(PC_EINVAL, "peer_direct must be 0 or 1");
    t.peer_direct = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "dev_direct")) {
    if (value < 0 || value > 1) return fail(PC_EINVAL, "dev_direct must be 0 or 1");
    t.dev_direct = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "host_mode")) {
    if (value < 0 || value > 3) return fail(PC_EINVAL, "host_mode must be 0, 1, 2 or 3");
    t.host_mode = static_cast<int>(value);
    return PC_OK;
  }
  if (!std::strcmp(knob, "ctas_per_sm")) {
    if (value < 0 || value > 32) return fail(PC_EINVAL, "ctas_per_sm must be 0..32");
    t.ctas_per_sm = static_cast<int>(value);
    return PC_OK;
  }
  return fail(PC_EINVAL, "unknown knob '%s'", knob);
}

int pc_tune_get(const char *knob, int64_t *value) {
  if (!knob || !value) return fail(PC_EINVAL, "NULL argument");
  Tuning &t = tuning();
  if (!std::strcmp(knob, "rotmask")) *value = t.rot_mask;
  else if (!std::strcmp(knob, "small_mode")) *value = t.small_mode;
  else if (!std::strcmp(knob, "svc_pages")) *value = t.svc_pages.load();
  else if (!std::strcmp(knob, "run_desc")) *value = t.run_desc.load();
  else if (!std::strcmp(knob, "svc_bell_ops")) *value = t.svc_bell_ops.load();
  else if (!std::strcmp(knob, "small_max")) *value = static_cast<int64_t>(t.small_max.load());
  else if (!std::strcmp(knob, "kernel")) *value = t.kernel;
  else if (!std::strcmp(knob, "host_mode")) *value = t.host_mode;
  else if (!std::strcmp(knob, "launches")) *value = static_cast<int64_t>(g_launches.load());
  else if (!std::strcmp(knob, "dev_direct")) *value = t.dev_direct;
  else if (!std::strcmp(knob, "peer_direct")) *value = t.peer_direct;
  else if (!std::strcmp(knob, "svc_direct")) *value = t.svc_direct;
  else if (!std::strcmp(knob, "ctas_per_sm")) *value = t.ctas_per_sm;
  else return fail(PC_EINVAL, "unknown knob '%s'", knob);
  return PC_OK;
}

} // extern "C"

#include "store.inc"
