/*
 * pagecrypt.h -- C ABI of the B200 page-cipher engine (libpagecrypt.so).
 *
 * Drop-in boundary for MemShield's page-cipher hot path.  The reference
 * (/root/reference/pkg) is a Python package with two in-process seams
 * (SURVEY.md §8b); every entry point below names the reference interface it
 * replaces.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - Every function returns int: PC_OK (0) on success, else a PC_E* code;
 *     pc_last_error() returns a thread-local message for the last failure.
 *     The Python wrapper maps PC_EINVAL to pagecrypt's ContractViolation
 *     (pkg/src/pagecrypt/errors.py:8-10) and everything else to
 *     PageCryptError (errors.py:4).
 *   - The caller owns every buffer; the library retains none after the call
 *     (or, for *_dev entry points, after the stream reaches the call).
 *   - rounds is 8, 12 or 20 (ChaCha8/12/20).  The reference has 20 only
 *     (pkg/src/pagecrypt/cipher.py:158, _chacha_numba.py:68).
 *   - Block i of page (vaddr, pid) uses the RFC 8439 state
 *     "expand 32-byte k" || key[8] || vaddr_lo, vaddr_hi, pid, i
 *     (pkg/src/pagecrypt/cipher.py:3-11,133-141).  Pages are 4096 bytes,
 *     64 blocks each.  Page descriptors: per-page arrays vaddrs[n] / pids[n],
 *     or, when an array pointer is NULL, vaddr0 + 4096*i and the scalar pid0.
 *   - Entry points are thread-safe; a pc_engine serialises its own use.
 */
#ifndef PAGECRYPT_H
#define PAGECRYPT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PC_OK 0
#define PC_EINVAL 1 /* contract violation (bad size/alignment/rounds/handle) */
#define PC_ECUDA 2  /* CUDA runtime/launch failure (message has the detail) */
#define PC_ENOMEM 3 /* device or pinned allocation failed */
#define PC_ESTATE 4 /* object used after destroy, wrong device, ... */
#define PC_ETIMEOUT 5 /* a service request did not complete in time */
#define PC_EFULL 6    /* the HBM page store has no free slot for the batch */

#define PC_PAGE_SIZE 4096
#define PC_BLOCK_SIZE 64
#define PC_BLOCKS_PER_PAGE 64
#define PC_KEY_SIZE 32

typedef struct pc_key pc_key;       /* device-resident 256-bit master key   */
typedef struct pc_engine pc_engine; /* per-device streams + staging buffers */

/* ---- library ---------------------------------------------------------- */
int pc_abi_version(void);          /* PC_ABI_VERSION below                 */
const char *pc_last_error(void);   /* thread-local, never NULL             */
int pc_device_count(int *count);
int pc_device_info(int device, int *sm_count, int *cc_major, int *cc_minor);
#define PC_ABI_VERSION 1

/* ---- (i) kernel seam ---------------------------------------------------
 * Replaces pagecrypt._chacha_numba.keystream_words(kw, vaddr, pid, indices,
 * out) (pkg/src/pagecrypt/_chacha_numba.py:44-93), consumed at
 * pkg/src/pagecrypt/cipher.py:176-182.  Host memory in and out: kw[8] LE key
 * words, idx[k] block indices (any int64, truncated to u32 like the
 * reference's uint64 & 0xffffffff), out[16*k] words, block-major.
 * Runs on the calling thread's current device; synchronous. */
int pc_keystream_words(const uint32_t kw[8], uint64_t vaddr, uint32_t pid,
                       const int64_t *idx, size_t k, uint32_t *out, int rounds);

/* ---- (ii) raw-seed blocks ----------------------------------------------
 * The 16-byte state tail as raw bytes (counter||nonce), one seed per block:
 * RFC 8439 vectors that BlockSeed (cipher.py:79-104) cannot express.
 * Mirrors pkg/tests/reference_chacha.py:28 chacha20_block_ref(key, seed16).
 * Host memory; out = 64*k bytes. */
int pc_keystream_raw(const uint8_t key[32], const uint8_t *seeds16, size_t k,
                     int rounds, uint8_t *out);

/* ---- (iii) key residency -----------------------------------------------
 * Replaces WorkerPool.install_key / key slots / shutdown wipe
 * (pkg/src/pagecrypt/workers.py:168,174-202,240-254).  The key is copied
 * into device memory of `device`; the library keeps no host copy.
 * pc_key_generate derives the key ON the device from 32 bytes of caller
 * entropy mixed with device-only entropy, so the final key never exists in
 * host RAM.  pc_key_destroy zeroes the device copy before freeing it. */
int pc_key_install(int device, const uint8_t key[32], pc_key **out);
int pc_key_generate(int device, const uint8_t entropy[32], pc_key **out);
int pc_key_destroy(pc_key *key);  /* PC_ESTATE while a page store holds the key */
int pc_key_device(const pc_key *key, int *device);

/* Key replication across GPUs: the analog of copying the staged key into
 * every worker's private slot (pkg/src/pagecrypt/workers.py:193-194), with
 * the copy never passing through host RAM.
 *   pc_key_replicate: same process, device-to-device (cudaMemcpyPeer over
 *     NVLink; PC_ESTATE when `device` has no peer access to the source, since
 *     the driver would otherwise stage the copy through host memory).
 *   pc_key_export / pc_key_import: one process per GPU (torchrun).  export
 *     copies the key into a device buffer and returns its 64-byte CUDA-IPC
 *     handle (an opaque name of device memory, not key material); import, in
 *     another process, maps that buffer and copies the 32 bytes device-to-
 *     device into a new key on `device`.  The exporter keeps the export open
 *     until every importer has returned, then pc_key_export_close zeroes it
 *     (destroy closes it too). */
#define PC_KEY_HANDLE_SIZE 64
int pc_key_replicate(const pc_key *src, int device, pc_key **out);
int pc_key_export(pc_key *key, uint8_t handle[PC_KEY_HANDLE_SIZE]);
int pc_key_export_close(pc_key *key);
int pc_key_import(int device, const uint8_t handle[PC_KEY_HANDLE_SIZE], pc_key **out);

/* ---- (iv) device-resident batch ----------------------------------------
 * The batched form of cipher.crypt_page (pkg/src/pagecrypt/cipher.py:205-217)
 * for the worker call site (pkg/src/pagecrypt/workers.py:136-138).
 * in/out: device pointers to n*4096 bytes (16-byte aligned; in == out
 * allowed).  vaddrs/pids: device pointers or NULL (see conventions).
 * Asynchronous on `stream` (a cudaStream_t; NULL = legacy default). */
int pc_crypt_pages_dev(const pc_key *key, const uint64_t *vaddrs, const uint32_t *pids,
                       uint64_t vaddr0, uint32_t pid0, const void *in, void *out,
                       size_t n, int rounds, void *stream);
/* Device-side validation of descriptor arrays for (iv), stream-ordered and
 * synchronous: *flags bit 0 = a vaddr is not page-aligned, bit 1 = a 64-bit
 * pid (pids64, may be NULL) is outside u32; 64-bit pids are narrowed into
 * pids32.  One library kernel -- never a foreign one, so it is safe beside
 * the persistent worker service. */
int pc_desc_check(const uint64_t *vaddrs, const int64_t *pids64, uint32_t *pids32, size_t n, void *stream,
                  uint32_t *flags);

/* ---- (v) host-resident batch -------------------------------------------
 * Same result over host buffers.  Pinned buffers (pc_host_alloc /
 * pc_host_register / torch pin_memory) stream through the engine's staging
 * ring on several CUDA streams so H2D, cipher and D2H overlap; small
 * batches take a single-launch path.  in/out may also be device memory of
 * any GPU: pages on the engine's own GPU (contiguous vaddrs, scalar pid,
 * DeviceKey) run as one in-place launch; pages on another GPU are ciphered in
 * place by this GPU's kernel over NVLink when peer access is available (same
 * conditions; knob "peer_direct"), else stream through the engine's ring by
 * peer copies.  vaddrs/pids: host arrays or NULL.
 * Synchronous: returns when out holds the result.  `key` may be NULL when
 * raw_key is given (caller-key mode: the engine copies raw_key into a device
 * slot for this call and zeroes it before returning). */
int pc_engine_create(int device, int n_streams, size_t chunk_pages, pc_engine **out);
int pc_engine_destroy(pc_engine *eng);
/* Host placement chosen for the engine: the NUMA node of the
 * GPU's PCIe root (-1 = not reported) and how many GPU-local CPUs its runner
 * and bounce threads are bound to (0 = unbound).  Pinned staging is
 * allocated on that node. */
int pc_engine_placement(const pc_engine *eng, int *numa_node, int *n_cpus);
int pc_crypt_pages_host(pc_engine *eng, const pc_key *key, const uint8_t *raw_key,
                        const uint64_t *vaddrs, const uint32_t *pids, uint64_t vaddr0,
                        uint32_t pid0, const void *in, void *out, size_t n, int rounds);

/* ---- (vi) multi-device partition ---------------------------------------
 * Contiguous page range [g*n/G, (g+1)*n/G) per engine g, each with its own
 * device key (keys[g] must live on engines[g]'s device); no collective.
 * Host buffers, or device memory of one GPU (the other GPUs' ranges cross
 * NVLink peer-to-peer); one host thread per device; synchronous. */
int pc_crypt_pages_multi(pc_engine *const *engines, const pc_key *const *keys, int n_dev,
                         const uint64_t *vaddrs, const uint32_t *pids, uint64_t vaddr0,
                         uint32_t pid0, const void *in, void *out, size_t n, int rounds);

/* ---- (vii) persistent crypto-worker service -----------------------------
 * The paper's GPU design and the B200 replacement of the
 * reference's WorkerPool / WorkerRing / Completion
 * (pkg/src/pagecrypt/workers.py:28-254): one persistent kernel whose
 * n_workers 64-thread CTAs each serve a multiple-producer ring of ring_slots
 * (power of two) requests in mapped pinned host memory.  The key is read
 * into the workers' registers once; after pc_service_start returns the
 * pc_key may be destroyed and the key then exists only in registers.
 * submit copies one 4 KiB page into the worker's ring, registers `dst` (may
 * equal src; may be NULL to discard) as the destination of the result and
 * returns a ticket; it blocks while the ring is full (back-pressure, like
 * WorkerRing.push), delivering finished results to free a slot.  The result
 * reaches dst when any thread delivers it: wait/poll do, and so does a
 * producer that needs the slot.  dst must stay valid until wait/poll report
 * the ticket done.  stop refuses with PC_ESTATE while requests are in flight
 * (WorkerPool.shutdown, workers.py:240-254). */
typedef struct pc_service pc_service;
/* Load every kernel of the library into the context now.  Under CUDA's
 * default lazy module loading the first launch of any kernel waits for the
 * context to go idle, i.e. forever while a persistent kernel runs; the
 * service start calls this itself.  Other libraries' kernels (torch, ...)
 * must be warmed before pc_service_start, or run with
 * CUDA_MODULE_LOADING=EAGER, if they are first launched while the service
 * is up. */
int pc_preload(int device);
int pc_service_start(const pc_key *key, int n_workers, int ring_slots, int rounds, pc_service **out);
int pc_service_submit(pc_service *svc, int worker, uint64_t vaddr, uint32_t pid, const void *src,
                      void *dst, uint64_t *ticket);
int pc_service_poll(pc_service *svc, int worker, uint64_t ticket, int *done);
int pc_service_wait(pc_service *svc, int worker, uint64_t ticket, int64_t timeout_us);
int pc_service_crypt(pc_service *svc, int worker, uint64_t vaddr, uint32_t pid, const void *src,
                     void *dst, int64_t timeout_us);
int pc_service_in_flight(pc_service *svc, uint64_t *n);
/* Diagnostics: device %globaltimer stamps of the slot's last request (bell
 * seen, page loaded, keystream done, page written back). */
int pc_service_timing(pc_service *svc, int worker, uint64_t ticket, uint64_t out_ns[4]);
/* diagnostic: the SM (%smid) worker `worker` runs on */
int pc_service_worker_sm(pc_service *svc, int worker, int *smid);
int pc_service_max_workers(int device, int *n);
int pc_service_stop(pc_service *svc);
/* key service: start (n_workers > 0) or stop (0) resident workers holding
 * `key` (this section's kernel).  While they run, pc_crypt_pages_host calls
 * under `key` with `rounds` on at most svc_pages host pages (pc_tune knob;
 * 0 = one per worker, at most 6) are one service ticket per page instead of a launch --
 * the fault handler's 1-2 page calls (orchestrator.py:197-198,234-235) skip
 * the launch and stream sync.  pc_key_destroy stops them. */
int pc_key_service(pc_key *key, int n_workers, int rounds);

/* ---- (viii) HBM page store (device-resident ciphertext) -----
 * The B200 side of EncryptedPageStore (pkg/src/pagecrypt/store.py:41-105)
 * with the ciphertext pages resident in a device slab of slab_pages pages.
 * pc_slab_transfer moves n pages between host memory and slab slots
 * slots[i]; dir 0 = host -> slab (evict / insert), 1 = slab -> host
 * (refault / lookup).  With a key the page passes through the cipher on the
 * way (encrypt on evict, decrypt on refault; vaddrs/pids or vaddr0/pid0 as
 * in pc_crypt_pages_host), so plaintext never rests in HBM and ciphertext
 * never crosses PCIe; with key == NULL the bytes are copied verbatim.
 * Synchronous.  flags PC_SLAB_WIPE_SRC (dir 1): zero each slot as it is
 * read (a refault frees it).  pc_slab_wipe zeroes freed slots
 * (store.py:86-92). */
#define PC_SLAB_WIPE_SRC 1
int pc_slab_transfer(pc_engine *eng, const pc_key *key, void *slab, size_t slab_pages,
                     const uint32_t *slots, const uint64_t *vaddrs, const uint32_t *pids,
                     uint64_t vaddr0, uint32_t pid0, void *host, size_t n, int dir, int rounds,
                     int flags);
int pc_slab_wipe(pc_engine *eng, void *slab, size_t slab_pages, const uint32_t *slots, size_t n);

/* The store itself: an HBM slab plus a native index client -> vaddr -> slot
 * (the reference store's client -> SortedDict, store.py:41-51).  `client`
 * is any 64-bit id (the Python layer uses pid << 32 | epoch); `pid` is what
 * enters the cipher seed (workers.py:137).  put: evict (encrypt = 1) or
 * insert verbatim ciphertext (0); duplicates or a full slab reject the whole
 * batch (PC_EINVAL / PC_EFULL).  get: refault (decrypt = 1, remove = 1: slots
 * zeroed as read and freed) or lookup (0, 0); missing entries -> PC_EINVAL.
 * remove / drop_client wipe the freed slots.  list returns sorted vaddrs. */
typedef struct pc_store pc_store;
int pc_store_create(pc_engine *eng, const pc_key *key, size_t capacity_pages, int rounds, pc_store **out);
int pc_store_destroy(pc_store *store);
int pc_store_put(pc_store *store, uint64_t client, uint32_t pid, const uint64_t *vaddrs, size_t n,
                 const void *host, int encrypt);
int pc_store_get(pc_store *store, uint64_t client, uint32_t pid, const uint64_t *vaddrs, size_t n,
                 void *host, int decrypt, int remove);
int pc_store_remove(pc_store *store, uint64_t client, const uint64_t *vaddrs, size_t n);
int pc_store_drop_client(pc_store *store, uint64_t client);
int pc_store_contains(pc_store *store, uint64_t client, uint64_t vaddr, int *found);
int pc_store_contains_many(pc_store *store, uint64_t client, const uint64_t *vaddrs, size_t n, uint8_t *found);
int pc_store_list(pc_store *store, uint64_t client, uint64_t *vaddrs, size_t cap, size_t *n);
int pc_store_free_slots(pc_store *store, size_t *n);
/* swap: one fault of the orchestrator (handle_fault + evict_page,
 * pkg/src/pagecrypt/orchestrator.py:175-240) in one GPU round trip --
 * refault get_vaddrs into get_out (decrypt, remove, slots zeroed) and evict
 * put_in to put_vaddrs (encrypt, insert).  Same result as get(1, 1) then
 * put(1).  Up to 128 pages in total are one zero-copy launch and
 * all-or-nothing; larger batches (or a slab too full to take the evictions
 * before the refault frees its slots) run as get then put. */
int pc_store_swap(pc_store *store, uint64_t client, uint32_t pid, const uint64_t *get_vaddrs, size_t n_get,
                  void *get_out, const uint64_t *put_vaddrs, size_t n_put, const void *put_in);
/* fault: one orchestrator fault in one call -- vaddr is refaulted into out if
 * stored (*refaulted = 1), else out is untouched (first touch, *refaulted =
 * 0); evict_in (or NULL) is evicted to evict_vaddr; together one launch. */
int pc_store_fault(pc_store *store, uint64_t client, uint32_t pid, uint64_t vaddr, void *out,
                   uint64_t evict_vaddr, const void *evict_in, int *refaulted);
/* service: start (n_workers > 0) or stop (0) a resident worker service
 * (section vii) started from the store's own key.  While it runs,
 * pc_store_fault is one service ticket served by worker 0 (the slab read,
 * both keystreams, the eviction's write into HBM and the refault's write to
 * the host in one pass) instead of a launch + stream sync; batched calls keep
 * their launches.  The store's requests are serialised by its lock, so one
 * worker is enough.  pc_store_destroy stops it.  Replaces the launch in the
 * worker thread's call of crypt_page on the fault path
 * (pkg/src/pagecrypt/workers.py:130-142 <- orchestrator.py:197-198,234-235). */
int pc_store_service(pc_store *store, int n_workers);

/* ---- pinned host memory helpers ---------------------------------------
 * Note: freeing pinned memory (pc_host_free = cudaFreeHost) and
 * pc_host_unregister synchronise the whole device and therefore block while
 * a pc_service is running; the library itself recycles its own pinned
 * buffers instead of freeing them and allocates device memory
 * stream-ordered, so none of its entry points has that hazard. */
int pc_host_alloc(size_t bytes, void **out);
int pc_host_free(void *p);
int pc_host_register(void *p, size_t bytes);
int pc_host_unregister(void *p);

/* ---- measurement and tuning ------------------------------------------- */
/* Integer-pipe microbenchmark used for the roofline denominator: runs `kind`
 * on `device` and returns measured int32 lane-ops/s.  0 = LOP3, 1 = IADD,
 * 2 = IMAD, 3 = SHF rotate, 4 = ChaCha quarter rounds (12 ops each) as ptxas
 * schedules them, 5 = quarter rounds with one rotate on the FMA pipe,
 * 6 = IMAD.HI, 7 = IMAD.WIDE(+LOP3). */
int pc_intpeak(int device, int kind, double *ops_per_s);
/* Process-wide knobs: "rotmask" (compiled FMA-pipe rotate pattern of the
 * crypt kernel, see chacha.cuh), "small_mode" (0 staged copies / 1 zero-copy
 * for small host batches), "small_max", "kernel" (0 auto, 1..6 or 9 page-kernel
 * variant), "host_mode" (0..3 host pipeline), "ctas_per_sm", "dev_direct",
 * "peer_direct" (device-memory endpoints, see (v)), "svc_direct" (0/1/2 auto:
 * worker service doorbell polling), "run_desc" (1: descriptor arrays at
 * ChaCha8/12 walk contiguous page runs per slot; 2: the same runs with one
 * warp per page and two blocks per thread, any round count), "svc_pages" (key service
 * batch limit, 0 auto), "svc_bell_ops" (1: a store service's ticket slots
 * ride in the doorbell line); pc_tune_get also reads "launches", the number
 * of kernels this library has launched. */
int pc_tune(const char *knob, int64_t value);
int pc_tune_get(const char *knob, int64_t *value);

#ifdef __cplusplus
}
#endif
#endif /* PAGECRYPT_H */
