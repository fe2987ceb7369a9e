"""1-page service latency (bare ctypes pc_service_crypt, p50) against the
worker count (1, 8, 16, 148) and the worker a client routes to
(profiles/r01_service_workers_probe.txt)."""
import os, sys, time, ctypes
sys.path.insert(0, os.getcwd())
import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import _native
from paper_2004_09252_b200.workers import ClientId, WorkerPool
for nw in (1, 8, 16, 148):
    pool = WorkerPool(n_workers=nw, keysource=os.urandom)
    lib = _native.load(); buf = (ctypes.c_char * 4096)()
    for w in (0, pool.route(ClientId(1, 0))):
        for _ in range(200): lib.pc_service_crypt(pool._svc, w, 0x100000000, 1, buf, buf, -1)
        ts = []
        for _ in range(2000):
            t0 = time.perf_counter_ns(); lib.pc_service_crypt(pool._svc, w, 0x100000000, 1, buf, buf, -1); ts.append(time.perf_counter_ns() - t0)
        ts.sort(); print("python ctypes workers", nw, "worker", w, "p50", ts[1000] / 1e3, flush=True)
    pool.shutdown()
