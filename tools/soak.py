"""Soak test: every public path at once, for --seconds, every result checked.

Six host threads loop over random work until the deadline:
  * device batches (random size, contiguous or descriptor arrays, 8/12/20 rounds),
  * host batches through the shared default engine (pinned and pageable),
  * the reference single-page API and the keystream seam,
  * WorkerPool requests (crypt, and submit + poll),
  * HBM store evict / refault / swap / fault on per-thread clients.
Each result is compared with the C oracle; the first mismatch or exception
stops the run.  Prints one JSON line: operations per kind and the verdict.
"""

import argparse
import json
import os
import random
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _chacha_cuda  # noqa: E402
from paper_2004_09252_b200 import partition  # noqa: E402
from paper_2004_09252_b200.pager import WindowPager  # noqa: E402
from paper_2004_09252_b200.store import DevicePageStore  # noqa: E402
from paper_2004_09252_b200.workers import ClientId, WorkerPool  # noqa: E402
from oracle import coracle as C  # noqa: E402

KEY = bytes(range(60, 92))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120)
    ap.add_argument("--threads", type=int, default=6)
    ap.add_argument("--no-service", action="store_true", help="leave the persistent worker service out")
    a = ap.parse_args()
    import faulthandler

    faulthandler.dump_traceback_later(a.seconds + 90, exit=True)  # a hang prints every thread's stack
    # Everything torch needs is created and warmed BEFORE the persistent
    # service starts (a lazily loaded kernel or a device-wide
    # synchronisation never returns while a persistent kernel runs; run with
    # CUDA_MODULE_LOADING=EAGER for the same reason).
    np.random.default_rng(0)
    streams = [torch.cuda.Stream() for _ in range(a.threads)]
    warm = torch.from_numpy(np.zeros((2, 4096), np.uint8))
    warm.pin_memory()
    warm.cuda().cpu()
    if os.environ.get("SOAK_WARM_TORCH_OPS"):  # the ops crypt_pages' own checks launch
        wv = torch.zeros(4, dtype=torch.int64, device="cuda")
        bool(((wv & 4095) != 0).any())
    torch.cuda.synchronize()
    dkey = pc.DeviceKey.install(KEY, 0)
    engines = [pc.Engine(0, n_streams=3, chunk_pages=512) for _ in range(2)]
    pool = None if a.no_service else WorkerPool(n_workers=8, keysource=lambda n: KEY)
    store = DevicePageStore(1 << 15, dkey)
    if not a.no_service:
        # round 2: single faults on the store's resident worker, 1-2 page host
        # calls on the key's resident workers -- beside all the launches
        store.start_service()
        dkey.start_service(n_workers=2)
    counts = {}
    errors = []
    lock = threading.Lock()
    deadline = time.time() + a.seconds
    last_op = {}

    def bump(k):
        with lock:
            counts[k] = counts.get(k, 0) + 1

    def worker(t):
        rng = random.Random(t)
        nrng = np.random.default_rng(t)
        stream = streams[t]
        client = ClientId(1000 + t, 0)
        stored = {}
        spare = [0]
        pclient = ClientId(5000 + t, 0)
        pmem, pseen = {}, {}
        pager = WindowPager(store, lambda c, vs: np.stack([np.frombuffer(pmem.pop(v), np.uint8) for v in vs]), 4)
        pager.register(pclient)
        try:
            while time.time() < deadline and not errors:
                op = rng.randrange(9) if rng.random() > 0.01 else 9
                if op == 3 and pool is None:
                    continue
                with lock:
                    last_op[t] = op
                if op == 0:  # device batch
                    n = rng.choice([1, 3, 64, 1000, 4097])
                    r = rng.choice([8, 12, 20])
                    pages = nrng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
                    if rng.random() < 0.5:
                        v0 = 4096 * rng.randrange(1 << 40)
                        want = C.crypt_pages(KEY, None, None, pages, rounds=r, vaddr0=v0, pid0=t, nthreads=2)
                        with torch.cuda.stream(stream):
                            got = pc.crypt_pages(dkey, v0, t, torch.from_numpy(pages).cuda(), rounds=r, stream=stream)
                    else:
                        va = (4096 * nrng.integers(0, 1 << 40, size=n)).astype(np.uint64)
                        pid = nrng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
                        want = C.crypt_pages(KEY, va, pid, pages, rounds=r, nthreads=2)
                        with torch.cuda.stream(stream):
                            got = pc.crypt_pages(dkey, torch.from_numpy(va.view(np.int64)).cuda(),
                                                 torch.from_numpy(pid.view(np.int32)).cuda(),
                                                 torch.from_numpy(pages).cuda(), rounds=r, stream=stream)
                    stream.synchronize()
                    assert np.array_equal(got.cpu().numpy(), want), "device batch"
                    bump("device_batch")
                elif op == 1:  # host batch (1-2 pages: the key's resident workers when they run)
                    n = rng.choice([1, 2, 64, 65, 5000])
                    pages = nrng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
                    v0 = 4096 * rng.randrange(1 << 30)
                    want = C.crypt_pages(KEY, None, None, pages, vaddr0=v0, pid0=t, nthreads=2)
                    src = torch.from_numpy(pages).pin_memory() if rng.random() < 0.5 else pages
                    got = pc.crypt_pages(dkey, v0, t, src)
                    got = got.numpy() if hasattr(got, "numpy") else got
                    assert np.array_equal(got, want), "host batch"
                    bump("host_batch")
                elif op == 2:  # reference API + kernel seam
                    page = nrng.integers(0, 256, 4096, dtype=np.uint8).tobytes()
                    v = 4096 * rng.randrange(1 << 30)
                    want = C.crypt_pages(KEY, [v], t, np.frombuffer(page, np.uint8).reshape(1, 4096))[0]
                    assert pc.crypt_page(KEY, v, t, page) == want.tobytes(), "crypt_page"
                    out = np.empty(1024, np.uint32)
                    _chacha_cuda.keystream_words(np.frombuffer(KEY, "<u4"), np.uint64(v), np.uint32(t),
                                                 np.arange(64, dtype=np.int64), out)
                    assert out.tobytes() == (want ^ np.frombuffer(page, np.uint8)).tobytes(), "seam"
                    bump("api_and_seam")
                elif op == 3:  # worker service
                    plain = nrng.integers(0, 256, 4096, dtype=np.uint8).tobytes()
                    v = 4096 * rng.randrange(1 << 20)
                    want = C.crypt_pages(KEY, [v], client.pid, np.frombuffer(plain, np.uint8).reshape(1, 4096))[0]
                    buf = bytearray(plain)
                    if rng.random() < 0.5:
                        pool.crypt(client, v, "encrypt", buf)
                    else:
                        c = pool.submit(client, v, "encrypt", buf)
                        while not c.done:
                            pass
                        c.wait()
                    assert bytes(buf) == want.tobytes(), "service"
                    bump("service")
                elif op == 6:  # key lifecycle: a fresh key, a batch with it, destroyed
                    kb = bytes(nrng.integers(0, 256, 32, dtype=np.uint8))
                    pages = nrng.integers(0, 256, size=(rng.choice([1, 70, 600]), 4096), dtype=np.uint8)
                    with pc.DeviceKey.install(kb, 0) as k2:
                        with torch.cuda.stream(stream):
                            got = pc.crypt_pages(k2, 0x5000, t, torch.from_numpy(pages).cuda(), stream=stream)
                        stream.synchronize()
                        assert np.array_equal(got.cpu().numpy(), C.crypt_pages(kb, None, None, pages, vaddr0=0x5000,
                                                                              pid0=t, nthreads=2)), "fresh key"
                    bump("key_lifecycle")
                elif op == 7:  # pager faults on this thread's client (window 4), client memory as the model
                    v = 0x3_0000_0000 + 4096 * rng.randrange(12)
                    if v in pmem:
                        continue
                    got = pager.fault(pclient, v)
                    want = pseen.get(v, bytes(4096))
                    assert got == want, "pager fault"
                    data = bytearray(got)
                    data[rng.randrange(4096)] ^= 0x5A
                    pmem[v] = bytes(data)
                    pseen[v] = bytes(data)
                    bump("pager_fault")
                elif op == 8:  # device-resident partition over two engines
                    n = rng.choice([5, 300, 3000])
                    pages = nrng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
                    with torch.cuda.stream(stream):
                        dpages = torch.from_numpy(pages).cuda()
                    got = partition.crypt_pages_multi([dkey, dkey], engines, 0x9000, t, dpages)
                    assert np.array_equal(got.cpu().numpy(), C.crypt_pages(KEY, None, None, pages, vaddr0=0x9000,
                                                                          pid0=t, nthreads=2)), "multi"
                    bump("partition")
                elif op == 9:  # a second, short-lived worker service beside the first
                    kb = bytes(nrng.integers(0, 256, 32, dtype=np.uint8))
                    p2 = WorkerPool(n_workers=2, keysource=lambda n: kb)
                    try:
                        for i in range(8):
                            plain = nrng.integers(0, 256, 4096, dtype=np.uint8).tobytes()
                            buf = bytearray(plain)
                            p2.crypt(ClientId(9000 + t, 0), 4096 * i, "encrypt", buf)
                            want = C.crypt_pages(kb, [4096 * i], 9000 + t, np.frombuffer(plain, np.uint8).reshape(1, 4096))[0]
                            assert bytes(buf) == want.tobytes(), "second service"
                    finally:
                        p2.shutdown()
                    bump("service_lifecycle")
                else:  # store
                    v = 0x1_0000_0000 + 4096 * rng.randrange(256)
                    page = nrng.integers(0, 256, 4096, dtype=np.uint8)
                    if v in stored:
                        if rng.random() < 0.5:
                            assert np.array_equal(np.frombuffer(store.refault(client, v), np.uint8), stored.pop(v)), "refault"
                        else:
                            out = np.empty(4096, np.uint8)
                            # evict a page of the same 256-page range that is not stored
                            free = [x for x in (0x1_0000_0000 + 4096 * rng.randrange(256) for _ in range(8))
                                    if x not in stored and x != v]
                            if not free:
                                continue
                            e = free[0]
                            assert store.fault(client, v, out, e, page) is True, "fault: not refaulted"
                            assert np.array_equal(out, stored.pop(v)), "fault"
                            stored[e] = page
                    else:
                        store.evict(client, v, page)
                        stored[v] = page
                    bump("store")
            for v, p in list(stored.items()):
                assert np.array_equal(np.frombuffer(store.refault(client, v), np.uint8), p), "drain"
        except BaseException as exc:  # noqa: BLE001
            errors.append(f"thread {t}: {exc!r}")

    th = [threading.Thread(target=worker, args=(t,)) for t in range(a.threads)]
    t0 = time.time()
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=a.seconds + 60)
    if any(x.is_alive() for x in th):
        print(json.dumps({"hung_threads": [i for i, x in enumerate(th) if x.is_alive()], "last_op": last_op,
                          "ops": counts}), flush=True)
        faulthandler.dump_traceback(all_threads=True)
        os._exit(2)
    if pool is not None:
        pool.shutdown()
    store.close()
    dkey.destroy()
    print(json.dumps({"seconds": round(time.time() - t0, 1), "threads": a.threads, "ops": counts,
                      "ok": not errors, "errors": errors[:3]}))
    sys.exit(0 if not errors else 1)


if __name__ == "__main__":
    main()
