"""The reference's own CPU path, timed on this host's cores (TEST / BASELINE
INFRASTRUCTURE ONLY: bench.py's ``--impl reference`` arm and cpu_baseline
leg; the product never imports this).

Runs the UNMODIFIED reference package snapshotted in oracle/_ref/src
(oracle/fetch_ref.py) through its public API, with its numba kernel
(pkg/src/pagecrypt/_chacha_numba.py) JIT-compiled here -- SURVEY §8(d):

  (i)   cipher.crypt_page, one page per call, one thread
        (pkg/src/pagecrypt/cipher.py:205-217);
  (ii)  cipher.crypt_page on one forked process per host core, each on a
        contiguous slice of one shared-memory page buffer (the reference
        holds the GIL in its kernel, so processes are its only parallelism);
  (iii) WorkerPool(n_workers=cores): submit()/wait() of one request per page
        from clients pid 1..64 (routed over the workers,
        pkg/src/pagecrypt/workers.py:204-229), the reference's fault-path API.

Workload: the bench's pages (uniform random, contiguous vaddrs from
0x100000000, pid 1; key = np.random.default_rng(0).bytes(32)).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from multiprocessing import shared_memory

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.path.join(HERE, "_ref", "src")
PAGE = 4096
BASE_VADDR = 0x1_0000_0000

_ref = None


def load():
    """Import the snapshotted reference with numba; None when unavailable
    (no snapshot, or numba missing so the reference would silently use its
    numpy fallback -- not the path the reference ships as its fast path)."""
    global _ref
    if _ref is not None:
        return _ref
    if not os.path.isdir(os.path.join(REF_SRC, "pagecrypt")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "pc_numba_cache"))
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    try:
        import pagecrypt
        import pagecrypt.cipher as cipher
    except Exception:
        return None
    if getattr(cipher, "_chacha_numba", None) is None:
        return None
    if not pagecrypt.__file__.startswith(REF_SRC):
        return None
    _ref = pagecrypt
    return _ref


def _key():
    return np.random.default_rng(0).bytes(32)


def _pages(n, seed=1):
    return np.random.default_rng(seed).integers(0, 256, size=(n, PAGE), dtype=np.uint8)


def warm(pc) -> None:
    """JIT-compile the reference kernel (both kw specialisations) before timing."""
    key, page = _key(), bytes(PAGE)
    pc.crypt_page(key, BASE_VADDR, 1, page)
    pc.crypt_page(pc.MasterKey(key), BASE_VADDR, 1, page)


def single_thread(pc, seconds: float = 3.0, n: int = 256) -> dict:
    """(i) crypt_page, one thread, until `seconds` have elapsed."""
    key, pages = _key(), _pages(n)
    warm(pc)
    done, t0 = 0, time.perf_counter()
    while True:
        for i in range(n):
            pc.crypt_page(key, BASE_VADDR + PAGE * (done + i), 1, pages[i])
        done += n
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": done * PAGE / el / 1e9, "unit": "GB/s", "cores": 1, "pages": done, "seconds": el,
            "us_per_page": 1e6 * el / done}


# ---- (ii) one process per core ------------------------------------------------

def _proc_main(conn, inp, out):
    # forked: inp/out are the parent's MAP_SHARED shared-memory views
    pc = load()
    key = _key()
    crypt = pc.crypt_page
    while True:
        msg = conn.recv()
        if msg is None:
            break
        lo, hi, vaddr0 = msg
        for i in range(lo, hi):
            out[i] = np.frombuffer(crypt(key, vaddr0 + PAGE * i, 1, inp[i]), np.uint8)
        conn.send(hi - lo)
    conn.close()


class ProcessPool:
    """`cores` forked processes, each running crypt_page over its contiguous
    slice of one shared page buffer per step."""

    def __init__(self, cores: int, n_pages: int):
        pc = load()
        warm(pc)  # compiled before the fork: children inherit the JIT'd kernel
        self.n, self.cores = n_pages, cores
        self.shm_in = shared_memory.SharedMemory(create=True, size=n_pages * PAGE)
        self.shm_out = shared_memory.SharedMemory(create=True, size=n_pages * PAGE)
        self.inp = np.ndarray((n_pages, PAGE), np.uint8, buffer=self.shm_in.buf)
        self.out = np.ndarray((n_pages, PAGE), np.uint8, buffer=self.shm_out.buf)
        self.inp[:] = _pages(n_pages)
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        for _ in range(cores):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_proc_main, args=(b, self.inp, self.out), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)

    def step(self, vaddr0: int = BASE_VADDR) -> float:
        """One pass over the buffer; returns seconds."""
        t0 = time.perf_counter()
        for c, conn in enumerate(self.conns):
            conn.send((self.n * c // self.cores, self.n * (c + 1) // self.cores, vaddr0))
        done = sum(conn.recv() for conn in self.conns)
        el = time.perf_counter() - t0
        assert done == self.n
        return el

    def close(self):
        for conn in self.conns:
            try:
                conn.send(None)
            except OSError:
                pass
        for p in self.procs:
            p.join(timeout=10)
        del self.inp, self.out
        for s in (self.shm_in, self.shm_out):
            s.close()
            s.unlink()


# ---- (iii) WorkerPool ---------------------------------------------------------

def worker_pool(pc, cores: int, seconds: float = 3.0, batch: int = 512) -> dict:
    """(iii) WorkerPool(n_workers=cores): batches of submit() (clients pid
    1..64, so requests spread over the workers by route()) then wait()."""
    from pagecrypt.ram import TaggedRam
    from pagecrypt.workers import WorkerPool
    from pagecrypt.store import ClientId

    key = _key()
    ram = TaggedRam()
    pool = WorkerPool(n_workers=cores, keysource=lambda n: key, ram=ram)
    try:
        clients = [ClientId(1 + i % 64, 0) for i in range(batch)]
        bufs = [ram.alloc("server_misc", PAGE) for _ in range(batch)]
        src = _pages(batch)
        for b, p in zip(bufs, src):
            b.data[:] = p.tobytes()
        for c in clients[:64]:  # warm-up: every worker has run once
            pool.crypt(c, BASE_VADDR, "encrypt", bufs[0])
        done, t0 = 0, time.perf_counter()
        while True:
            comps = [pool.submit(clients[i], BASE_VADDR + PAGE * i, "encrypt", bufs[i]) for i in range(batch)]
            for c in comps:
                c.wait()
            done += batch
            el = time.perf_counter() - t0
            if el >= seconds:
                break
        # the 1-page synchronous fault-path call, for latency
        lat = []
        for i in range(200):
            t = time.perf_counter_ns()
            pool.crypt(clients[0], BASE_VADDR, "encrypt", bufs[0])
            lat.append(time.perf_counter_ns() - t)
        lat.sort()
        for b in bufs:
            ram.free(b)
    finally:
        pool.shutdown()
    return {"value": done * PAGE / el / 1e9, "unit": "GB/s", "cores": cores, "pages": done, "seconds": el,
            "crypt_1page_p50_us": lat[len(lat) // 2] / 1e3, "crypt_1page_p99_us": lat[int(len(lat) * .99)] / 1e3}


def crypt_page_latency(pc, reps: int = 2000) -> dict:
    """Same-run reference latency for BASELINE configs[3]: one crypt_page call
    (1 page) and a 64-page loop, p50/p99 in microseconds."""
    key, pages = _key(), _pages(64)
    warm(pc)
    res = {}
    for n in (1, 64):
        ts = []
        for r in range(max(50, reps // n)):
            t = time.perf_counter_ns()
            for i in range(n):
                pc.crypt_page(key, BASE_VADDR + PAGE * i, 1, pages[i])
            ts.append(time.perf_counter_ns() - t)
        ts.sort()
        res[str(n)] = {"p50_us": round(ts[len(ts) // 2] / 1e3, 2), "p99_us": round(ts[int(len(ts) * .99)] / 1e3, 2)}
    return res


def check_sample(pc, out: np.ndarray, inp: np.ndarray, vaddr0: int, k: int = 4) -> bool:
    """Spot-check k pages of a multi-process pass against a direct call."""
    key = _key()
    idx = np.linspace(0, len(inp) - 1, k).astype(int)
    return all(pc.crypt_page(key, vaddr0 + PAGE * int(i), 1, inp[i]) == out[i].tobytes() for i in idx)
