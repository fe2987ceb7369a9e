/*
 * CPU oracle for the page cipher -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library (oracle/liboracle.so).  The
 * product library (paper_2004_09252_b200/csrc) never links it and the product
 * Python package never loads it.
 *
 * Scalar C restatement of the reference page cipher, one page per call like
 * the reference (pkg/src/pagecrypt/cipher.py:205-217), with the round count as
 * a parameter (the reference fixes 20: _chacha_numba.py:68):
 *   quarter round         pkg/src/pagecrypt/_chacha_numba.py:27-41
 *   state setup / rounds  pkg/src/pagecrypt/_chacha_numba.py:51-76
 *   feed-forward / store  pkg/src/pagecrypt/_chacha_numba.py:77-93
 *   seed <QII packing     pkg/src/pagecrypt/cipher.py:41,95-97
 *   page XOR              pkg/src/pagecrypt/cipher.py:211-215
 * The multi-threaded driver splits a batch into contiguous page ranges, the
 * same partition the reference's WorkerPool parity test shows is
 * order-independent (pkg/tests/test_workers.py:136-148).
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define ROTL(x, n) (((x) << (n)) | ((x) >> (32 - (n))))
#define QR(a, b, c, d)                 \
    a += b; d ^= a; d = ROTL(d, 16);   \
    c += d; b ^= c; b = ROTL(b, 12);   \
    a += b; d ^= a; d = ROTL(d, 8);    \
    c += d; b ^= c; b = ROTL(b, 7);

static inline uint32_t ld32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
static inline void st32(uint8_t *p, uint32_t v) {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}

/* 16 output words of one block for the 16-word input state `in`. */
static void block_words(const uint32_t in[16], int rounds, uint32_t out[16]) {
    uint32_t x0 = in[0], x1 = in[1], x2 = in[2], x3 = in[3];
    uint32_t x4 = in[4], x5 = in[5], x6 = in[6], x7 = in[7];
    uint32_t x8 = in[8], x9 = in[9], x10 = in[10], x11 = in[11];
    uint32_t x12 = in[12], x13 = in[13], x14 = in[14], x15 = in[15];
    for (int r = 0; r < rounds; r += 2) {
        QR(x0, x4, x8, x12) QR(x1, x5, x9, x13) QR(x2, x6, x10, x14) QR(x3, x7, x11, x15)
        QR(x0, x5, x10, x15) QR(x1, x6, x11, x12) QR(x2, x7, x8, x13) QR(x3, x4, x9, x14)
    }
    out[0] = x0 + in[0]; out[1] = x1 + in[1]; out[2] = x2 + in[2]; out[3] = x3 + in[3];
    out[4] = x4 + in[4]; out[5] = x5 + in[5]; out[6] = x6 + in[6]; out[7] = x7 + in[7];
    out[8] = x8 + in[8]; out[9] = x9 + in[9]; out[10] = x10 + in[10]; out[11] = x11 + in[11];
    out[12] = x12 + in[12]; out[13] = x13 + in[13]; out[14] = x14 + in[14]; out[15] = x15 + in[15];
}

static void init_state(uint32_t st[16], const uint8_t key[32], const uint8_t seed[16]) {
    st[0] = 0x61707865u; st[1] = 0x3320646eu; st[2] = 0x79622d32u; st[3] = 0x6b206574u;
    for (int i = 0; i < 8; i++) st[4 + i] = ld32(key + 4 * i);
    for (int i = 0; i < 4; i++) st[12 + i] = ld32(seed + 4 * i);
}

/* reference_chacha.py:28-45 with a raw 16-byte seed (counter || nonce). */
void oracle_block_raw(const uint8_t key[32], const uint8_t seed[16], int rounds, uint8_t out[64]) {
    uint32_t st[16], w[16];
    init_state(st, key, seed);
    block_words(st, rounds, w);
    for (int i = 0; i < 16; i++) st32(out + 4 * i, w[i]);
    memset(st, 0, sizeof st);
    memset(w, 0, sizeof w);
}

/* cipher.py:205-217 for one page; in == out allowed. */
void oracle_crypt_page(const uint8_t key[32], uint64_t vaddr, uint32_t pid,
                       const uint8_t *in, uint8_t *out, int rounds) {
    uint32_t st[16], w[16];
    st[0] = 0x61707865u; st[1] = 0x3320646eu; st[2] = 0x79622d32u; st[3] = 0x6b206574u;
    for (int i = 0; i < 8; i++) st[4 + i] = ld32(key + 4 * i);
    st[12] = (uint32_t)vaddr;
    st[13] = (uint32_t)(vaddr >> 32);
    st[14] = pid;
    for (uint32_t b = 0; b < 64; b++) {
        st[15] = b;
        block_words(st, rounds, w);
        const uint8_t *src = in + 64 * b;
        uint8_t *dst = out + 64 * b;
        for (int i = 0; i < 16; i++) st32(dst + 4 * i, ld32(src + 4 * i) ^ w[i]);
    }
    memset(st, 0, sizeof st);
    memset(w, 0, sizeof w);
}

typedef struct {
    const uint8_t *key;
    const uint64_t *vaddrs;
    const uint32_t *pids;
    uint64_t vaddr0;
    uint32_t pid0;
    const uint8_t *in;
    uint8_t *out;
    size_t lo, hi;
    int rounds;
} job_t;

static void *run_job(void *arg) {
    job_t *j = (job_t *)arg;
    for (size_t p = j->lo; p < j->hi; p++) {
        uint64_t va = j->vaddrs ? j->vaddrs[p] : j->vaddr0 + 4096ull * p;
        uint32_t pid = j->pids ? j->pids[p] : j->pid0;
        oracle_crypt_page(j->key, va, pid, j->in + 4096 * p, j->out + 4096 * p, j->rounds);
    }
    return NULL;
}

/* Batched driver: per-page vaddrs/pids, or (when NULL) vaddr0 + 4096*i and a
 * scalar pid0.  Contiguous page ranges per thread; nthreads <= 0 means 1. */
void oracle_crypt_pages(const uint8_t key[32], const uint64_t *vaddrs, const uint32_t *pids,
                        uint64_t vaddr0, uint32_t pid0, const uint8_t *in, uint8_t *out,
                        size_t n, int rounds, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((size_t)nthreads > n) nthreads = n ? (int)n : 1;
    job_t jobs[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (job_t){key, vaddrs, pids, vaddr0, pid0, in, out,
                          n * (size_t)t / nthreads, n * (size_t)(t + 1) / nthreads, rounds};
    }
    for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, run_job, &jobs[t]);
    run_job(&jobs[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
}
