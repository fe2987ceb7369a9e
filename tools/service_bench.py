"""Latency/throughput of the persistent crypto-worker service (config 4:
1-page requests on the fault path) vs the launch-per-call host path."""

import ctypes
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402
from paper_2004_09252_b200.workers import ClientId, WorkerPool  # noqa: E402


def pct(ts):
    ts = sorted(ts)
    return ts[len(ts) // 2] / 1e3, ts[int(len(ts) * 0.99)] / 1e3


def main():
    reps = 3000
    for workers in (1, 148):
        pool = WorkerPool(n_workers=workers, keysource=os.urandom)
        page = bytearray(4096)
        c = ClientId(1, 0)
        for _ in range(100):
            pool.crypt(c, 0x1000, "encrypt", page)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter_ns()
            pool.crypt(c, 0x1000, "encrypt", page)
            ts.append(time.perf_counter_ns() - t0)
        p50, p99 = pct(ts)
        print(json.dumps({"what": "WorkerPool.crypt 1 page (python)", "workers": workers, "p50_us": p50,
                          "p99_us": p99}), flush=True)
        # raw C ABI call (no Python object overhead)
        lib = _native.load()
        buf = (ctypes.c_char * 4096)()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter_ns()
            lib.pc_service_crypt(pool._svc, 0, 0x1000, 1, buf, buf, -1)
            ts.append(time.perf_counter_ns() - t0)
        p50, p99 = pct(ts)
        print(json.dumps({"what": "pc_service_crypt 1 page (ctypes)", "workers": workers, "p50_us": p50,
                          "p99_us": p99}), flush=True)
        # device-side breakdown of single requests (submit/wait split by hand)
        tk = ctypes.c_uint64()
        stamps = (ctypes.c_uint64 * 4)()
        parts = []
        for _ in range(500):
            t0 = time.perf_counter_ns()
            lib.pc_service_submit(pool._svc, 0, 0x1000, 1, buf, buf, ctypes.byref(tk))
            t1 = time.perf_counter_ns()
            lib.pc_service_wait(pool._svc, 0, tk.value, -1)
            t2 = time.perf_counter_ns()
            lib.pc_service_timing(pool._svc, 0, tk.value, stamps)
            parts.append((t1 - t0, stamps[1] - stamps[0], stamps[2] - stamps[1], stamps[3] - stamps[2], t2 - t0))
        med = [sorted(p[i] for p in parts)[len(parts) // 2] / 1e3 for i in range(5)]
        print(json.dumps({"what": "service breakdown us (median)", "workers": workers, "submit": med[0],
                          "load_page_pcie": med[1], "keystream_xor": med[2], "store_fence": med[3],
                          "total": med[4], "unaccounted_poll_and_notify": round(med[4] - sum(med[:4]), 2)}),
              flush=True)
        # throughput: T producer threads, each its own client
        for T in (1, 4, 8, 16):
            n_each = 2000
            done = []

            def prod(i):
                pg = bytearray(4096)
                cl = ClientId(1000 + i, 0)
                for j in range(n_each):
                    pool.crypt(cl, 4096 * j, "encrypt", pg)
                done.append(1)

            th = [threading.Thread(target=prod, args=(i,)) for i in range(T)]
            t0 = time.perf_counter()
            for t in th:
                t.start()
            for t in th:
                t.join()
            el = time.perf_counter() - t0
            print(json.dumps({"what": "WorkerPool.crypt throughput", "workers": workers, "producers": T,
                              "pages_per_s": round(T * n_each / el), "gbs": round(T * n_each * 4096 / el / 1e9, 3)}),
                  flush=True)
        pool.shutdown()
    # the launch-per-call path for comparison (pc.crypt_page, raw key bytes)
    key = os.urandom(32)
    page = bytes(4096)
    for _ in range(100):
        pc.crypt_page(key, 0x1000, 1, page)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        pc.crypt_page(key, 0x1000, 1, page)
        ts.append(time.perf_counter_ns() - t0)
    p50, p99 = pct(ts)
    print(json.dumps({"what": "crypt_page (launch per call)", "p50_us": p50, "p99_us": p99}), flush=True)


if __name__ == "__main__":
    main()
