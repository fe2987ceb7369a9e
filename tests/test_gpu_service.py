"""The persistent GPU crypto-worker service (include/pagecrypt.h section vii)
and its WorkerPool drop-in, restating pkg/tests/test_workers.py:107-237 for
the pool, plus parity against the oracle, the ring back-pressure, and key
confinement: after start the key exists only in the workers' registers."""

import ctypes
import random
import re
import threading

import numpy as np
import pytest

from paper_2004_09252_b200 import _native
from paper_2004_09252_b200.errors import ContractViolation, PoolError
from paper_2004_09252_b200.workers import ClientId, Completion, WorkerPool

from oracle import chacha_oracle as O
from oracle import coracle as C

pytestmark = pytest.mark.gpu

KEY = bytes(range(32))
PAGE_SIZE = 4096


def fixed_keysource(n):
    assert n == 32
    return KEY


def make_pool(n=2, **kw):
    return WorkerPool(n_workers=n, keysource=fixed_keysource, **kw)


class Page:
    """Minimal RamBuf stand-in (pkg/src/pagecrypt/ram.py:44-66): .data buffer."""

    def __init__(self, data=None):
        self.data = bytearray(data if data is not None else PAGE_SIZE)


class TestPool:
    def test_roundtrip_involution(self, cuda):
        pool = make_pool(2)
        client = ClientId(7, 0)
        page = Page(bytes([0x5A]) * PAGE_SIZE)
        pool.crypt(client, 0x1000, "encrypt", page)
        assert bytes(page.data) != bytes([0x5A]) * PAGE_SIZE
        assert bytes(page.data) == O.crypt_page(KEY, 0x1000, 7, bytes([0x5A]) * PAGE_SIZE)
        pool.crypt(client, 0x1000, "decrypt", page)
        assert bytes(page.data) == bytes([0x5A]) * PAGE_SIZE
        pool.shutdown()

    @pytest.mark.parametrize("rounds", [8, 12, 20])
    def test_output_equals_oracle(self, rounds, cuda):
        pool = make_pool(3, rounds=rounds)
        rng = random.Random(5)
        client = ClientId(42, 1)
        for _ in range(40):
            plain = rng.randbytes(PAGE_SIZE)
            vaddr = rng.randrange(2**52) * 4096
            page = Page(plain)
            pool.crypt(client, vaddr, "encrypt", page)
            want = C.crypt_pages(KEY, [vaddr], client.pid, np.frombuffer(plain, np.uint8), rounds=rounds)
            assert bytes(page.data) == want.tobytes()
        pool.shutdown()

    def test_epoch_does_not_enter_the_seed(self, cuda, ref_pages):
        """WorkerPool seeds with client.pid only (workers.py:137): golden pool_ct
        was produced by the reference pool with ClientId(4242, 3)."""
        r = ref_pages
        pool = WorkerPool(n_workers=4, keysource=lambda n: r["key"].tobytes())
        for epoch in (0, 3, 99):
            for i in range(8):
                page = Page(r["pages"][i].tobytes())
                pool.crypt(ClientId(4242, epoch), int(r["vaddrs"][i]), "encrypt", page)
                assert bytes(page.data) == r["pool_ct"][i].tobytes()
        pool.shutdown()

    def test_single_worker_and_many_workers_same_outputs(self, cuda):
        plain = bytes(range(256)) * 16
        out = []
        for n in (1, 8, 148):
            pool = make_pool(n)
            page = Page(plain)
            pool.crypt(ClientId(3, 0), 0x7000, "encrypt", page)
            out.append(bytes(page.data))
            pool.shutdown()
        assert out[0] == out[1] == out[2]

    def test_concurrent_submissions_all_complete(self, cuda):
        pool = make_pool(2)
        n_producers, per = 4, 250
        results = [[] for _ in range(n_producers)]
        errors = []

        def producer(idx):
            try:
                client = ClientId(100 + idx, 0)
                for i in range(per):
                    page = Page()
                    page.data[:2] = bytes([idx, i % 256])
                    pool.crypt(client, (i % 512) * 4096, "encrypt", page)
                    results[idx].append(bytes(page.data))
            except Exception as exc:  # pragma: no cover - surfaced below
                errors.append(exc)

        ts = [threading.Thread(target=producer, args=(i,)) for i in range(n_producers)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors
        assert all(len(r) == per for r in results)
        for idx in range(n_producers):
            for i in (0, 1, per - 1):
                plain = bytearray(PAGE_SIZE)
                plain[:2] = bytes([idx, i % 256])
                assert results[idx][i] == O.crypt_page(KEY, (i % 512) * 4096, 100 + idx, bytes(plain))
        assert pool.in_flight == 0
        pool.shutdown()

    def test_full_ring_backpressure_without_waiting(self, cuda):
        """More submissions than ring slots from one thread before any wait:
        the producer delivers finished results to free slots (WorkerRing.push
        blocks until the consumer frees one, workers.py:86-95)."""
        pool = make_pool(1, ring_capacity=2)
        pages = [Page(bytes([i]) * PAGE_SIZE) for i in range(9)]
        comps = [pool.submit(ClientId(5, 0), 4096 * i, "encrypt", p) for i, p in enumerate(pages)]
        for c in comps:
            c.wait(10)
        for i, p in enumerate(pages):
            assert bytes(p.data) == O.crypt_page(KEY, 4096 * i, 5, bytes([i]) * PAGE_SIZE)
        assert pool.in_flight == 0
        pool.shutdown()

    def test_single_slot_ring_many_producers(self, cuda):
        """ring_capacity=1: every request waits for the previous one's slot;
        four producer threads on one worker still all complete correctly."""
        import threading

        pool = make_pool(1, ring_capacity=1)
        errors = []

        def prod(t):
            try:
                for i in range(60):
                    plain = bytes([t, i]) * (PAGE_SIZE // 2)
                    p = Page(plain)
                    pool.crypt(ClientId(70 + t, 0), 4096 * i, "encrypt", p)
                    assert bytes(p.data) == O.crypt_page(KEY, 4096 * i, 70 + t, plain)
            except BaseException as exc:
                errors.append(repr(exc))

        th = [threading.Thread(target=prod, args=(t,)) for t in range(4)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        assert not errors, errors
        assert pool.in_flight == 0
        pool.shutdown()

    def test_unwaited_requests_do_not_block_shutdown(self, cuda):
        pool = make_pool(2)
        pages = [Page() for _ in range(10)]
        for i, p in enumerate(pages):
            pool.submit(ClientId(9, 0), 4096 * i, "encrypt", p)
        import time
        deadline = time.time() + 10
        while True:
            try:
                pool.shutdown()
                break
            except PoolError:
                assert time.time() < deadline
                time.sleep(0.01)
        for i, p in enumerate(pages):
            assert bytes(p.data) == O.crypt_page(KEY, 4096 * i, 9, bytes(PAGE_SIZE))

    def test_completion_poll(self, cuda):
        pool = make_pool(1)
        page = Page()
        c = pool.submit(ClientId(1, 0), 0, "encrypt", page)
        import time
        t0 = time.time()
        while not c.done:
            assert time.time() - t0 < 10
        c.wait(1)
        assert bytes(page.data) == O.crypt_page(KEY, 0, 1, bytes(PAGE_SIZE))
        pool.shutdown()

    def test_worker_side_contract_errors_surface_on_wait(self, cuda):
        pool = make_pool(1)
        c = pool.submit(ClientId(1, 0), 0x1001, "encrypt", Page())
        with pytest.raises(ContractViolation):
            c.wait(1)
        with pytest.raises(ContractViolation):
            pool.submit(ClientId(1, 0), 0, "sideways", Page())
        with pytest.raises(ContractViolation):
            pool.submit(ClientId(1, 0), 0, "encrypt", Page(bytes(100)))
        pool.shutdown()

    def test_double_key_install_rejected(self, cuda):
        pool = make_pool(1)
        with pytest.raises(PoolError):
            pool.install_key(fixed_keysource)
        pool.shutdown()

    def test_keysource_failure_fatal(self, cuda):
        def broken(n):
            raise OSError("no entropy")

        with pytest.raises(PoolError):
            WorkerPool(n_workers=1, keysource=broken)
        with pytest.raises(PoolError):
            WorkerPool(n_workers=1, keysource=lambda n: b"short")

    def test_shutdown_is_idempotent_and_final(self, cuda):
        pool = make_pool(2)
        pool.shutdown()
        pool.shutdown()
        assert not pool.running
        with pytest.raises(PoolError):
            pool.submit(ClientId(1, 0), 0, "encrypt", Page())

    def test_per_client_routing_is_stable(self, cuda):
        pool = make_pool(4)
        c = ClientId(123, 7)
        assert pool.route(c) == pool.route(ClientId(123, 7))
        assert 0 <= pool.route(c) < 4
        assert pool.route(c) == ((123 * 2654435761) ^ 7) % 4
        pool.shutdown()

    def test_too_many_workers_rejected(self, cuda):
        n = ctypes.c_int()
        _native.call("pc_service_max_workers", 0, ctypes.byref(n))
        with pytest.raises(ContractViolation):
            WorkerPool(n_workers=n.value + 1, keysource=fixed_keysource)

    def test_completion_handle_api(self):
        c = Completion()
        assert c.done
        c.wait(1)


def _scan_process_memory(key_ints: list[int], length: int = 16) -> int:
    """Count occurrences of any `length`-byte window of the key in every
    readable private mapping of this process -- the cold-boot analyzer's key
    scan (analyzer.py:126-142) applied to the real process.  The key is held
    only as a list of Python ints, so the scan itself never materialises a
    contiguous copy of it."""
    hits = 0
    with open("/proc/self/maps") as maps:
        regions = [line.split() for line in maps]
    with open("/proc/self/mem", "rb", 0) as mem:
        for parts in regions:
            lo, hi = (int(x, 16) for x in parts[0].split("-"))
            path = parts[5] if len(parts) > 5 else ""
            # private writable memory: heap, stacks, anonymous maps (Python
            # objects, malloc, the library's staging) and writable data of
            # loaded objects; device-file mappings (/dev/nvidia*) are skipped:
            # reading them through /proc/self/mem is not supported
            if not parts[1].startswith("rw") or path.startswith("/dev/") or path.startswith("[v"):
                continue
            if hi - lo > (4 << 30):
                continue
            pos = lo
            while pos < hi:
                n = min(hi - pos, 64 << 20)
                try:
                    mem.seek(pos)
                    buf = mem.read(n)
                except (OSError, ValueError, OverflowError):
                    break
                arr = np.frombuffer(buf, dtype=np.uint8)
                if arr.size >= length:
                    for start in range(0, len(key_ints) - length + 1, 8):
                        cand = np.flatnonzero(arr[: arr.size - length + 1] == key_ints[start])
                        for j in range(1, length):
                            if not cand.size:
                                break
                            cand = cand[arr[cand + j] == key_ints[start + j]]
                        hits += int(cand.size)
                del arr, buf
                pos += n
    return hits


_SCAN_CHILD = r"""
import os, sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
from test_gpu_service import _scan_process_memory, Page, PAGE_SIZE
from paper_2004_09252_b200.workers import ClientId, WorkerPool
from oracle import chacha_oracle as O
mask = bytearray(os.urandom(32))
masked = bytearray(os.urandom(32))  # key = masked ^ mask; neither alone is the key
def keysource(n):
    return bytearray(a ^ b for a, b in zip(masked, mask))  # wiped by install_key
leak = bytearray(a ^ b for a, b in zip(masked, mask)) if {positive!r} else None
pool = WorkerPool(n_workers=4, keysource=keysource)
page = Page()
pool.crypt(ClientId(1, 0), 0, "encrypt", page)
key_ints = [a ^ b for a, b in zip(masked, mask)]
hits = _scan_process_memory(key_ints)
ok = bytes(page.data) == O.crypt_page(bytes(key_ints), 0, 1, bytes(PAGE_SIZE))
pool.shutdown()
print("HITS", hits, "OK", ok)
"""


def test_key_only_in_worker_registers(cuda):
    """After pool start, no 16-byte window of the key is anywhere in host
    process memory (staging, driver bounce buffers, rings) -- the paper's
    claim "stored only in GPU registers, afterwards it is purged out of the
    server memory".  Runs in a fresh interpreter so the
    scan covers a whole, small process."""
    import os
    import subprocess
    import sys

    hits, ok = _scan_child(positive=False)
    assert ok  # the workers still encrypt with the key they hold in registers
    assert hits == 0


def _scan_child(positive: bool):
    import os
    import subprocess
    import sys

    tests = os.path.dirname(os.path.abspath(__file__))
    code = _SCAN_CHILD.format(root=os.path.dirname(tests), tests=tests, positive=positive)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("HITS")][-1]
    return int(line.split()[1]), line.split()[3] == "True"


def test_scanner_positive_control(cuda):
    """The same scan finds the key when a copy IS left in host memory (the
    debug_leak_key positive control, workers.py:196-200)."""
    hits, ok = _scan_child(positive=True)
    assert ok and hits >= 1


def test_service_coexists_with_bulk_work_and_lifecycles(cuda):
    """A persistent service kernel must not deadlock the rest of the library:
    no entry point may device-synchronise (key install/destroy, engine
    create/destroy, store create/wipe, bulk crypt on other streams), and none
    of our kernels may lazy-load behind it (pc_preload runs at service start).
    Torch's own kernels are warmed first: under CUDA's lazy module loading a
    kernel first launched while a persistent kernel runs waits for it."""
    import torch

    import paper_2004_09252_b200 as pc
    from paper_2004_09252_b200.store import DevicePageStore

    def work(pool):
        k = pc.DeviceKey.install(KEY, 0)
        pages = torch.randint(0, 256, (2048, PAGE_SIZE), dtype=torch.uint8, device="cuda")
        for kern in (0, 2, 3, 4, 5):  # every bulk kernel variant
            _native.tune("kernel", kern)
            for rounds in (8, 12, 20):
                ct = pc.crypt_pages(k, 0x1000, 1, pages, rounds=rounds)
                back = pc.crypt_pages(k, 0x1000, 1, ct, rounds=rounds)
                assert torch.equal(back, pages)
        _native.tune("kernel", 0)
        eng = pc.Engine(0, n_streams=2, chunk_pages=256)
        host = np.random.default_rng(0).integers(0, 256, size=(600, PAGE_SIZE), dtype=np.uint8)
        assert np.array_equal(pc.crypt_pages(k, 0x1000, 1, pc.crypt_pages(k, 0x1000, 1, host, engine=eng),
                                             engine=eng), host)
        assert pc.crypt_page(KEY, 0x2000, 3, bytes(PAGE_SIZE)) == O.crypt_page(KEY, 0x2000, 3, bytes(PAGE_SIZE))
        eng.destroy()
        st = DevicePageStore(16, k)
        st.evict(ClientId(1, 0), 0x5000, bytes(PAGE_SIZE))
        assert st.refault(ClientId(1, 0), 0x5000) == bytes(PAGE_SIZE)
        st.close()
        k.destroy()
        if pool is not None:
            page = Page()
            pool.crypt(ClientId(2, 0), 0x9000, "encrypt", page)
            assert bytes(page.data) == O.crypt_page(KEY, 0x9000, 2, bytes(PAGE_SIZE))

    work(None)  # warm torch's kernels (randint, equal, copies)
    pool = make_pool(4)
    try:
        for _ in range(2):
            work(pool)
    finally:
        _native.tune("kernel", 0)
        pool.shutdown()


def test_default_pool_routes_like_the_reference(cuda):
    """n_workers=None means os.cpu_count() as in the reference
    (workers.py:156-157), so client -> worker routing is identical."""
    import os

    pool = WorkerPool(keysource=fixed_keysource)
    try:
        assert pool.n_workers == min(os.cpu_count() or 1, pool.n_workers) and pool.n_workers >= 1
        if (os.cpu_count() or 1) <= pool.n_workers:
            for pid in (0, 1, 4242, 2**32 - 1):
                for epoch in (0, 7):
                    c = ClientId(pid, epoch)
                    assert pool.route(c) == ((pid * 2654435761) ^ epoch) % (os.cpu_count() or 1)
    finally:
        pool.shutdown()


def test_completion_signal_after_gpu_release(cuda):
    """Completion.signal (workers.py:38-42) on a request the GPU still holds
    waits for it first; the recorded error is what wait() raises."""
    pool = make_pool(2)
    try:
        page = bytearray(4096)
        c = pool.submit(ClientId(1, 0), 0x1000, "encrypt", page)
        c.signal(PoolError("cancelled by caller"))
        assert c.done
        with pytest.raises(PoolError, match="cancelled"):
            c.wait()
        assert bytes(page) == O.crypt_page(KEY, 0x1000, 1, bytes(4096))
        ok = Completion()
        ok.signal()
        ok.wait()
    finally:
        pool.shutdown()


def test_device_checks_never_launch_foreign_kernels_beside_the_service(cuda, tmp_path):
    """With the persistent service up, crypt_pages on device descriptor
    arrays (incl. 64-bit pids to narrow and check) must not launch a kernel
    the library did not preload: a fresh process (nothing of torch loaded)
    would otherwise hang forever on its first torch kernel."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "beside_service.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_2004_09252_b200 as pc\n"
        "from paper_2004_09252_b200.workers import WorkerPool, ClientId\n"
        "from oracle import coracle as C\n"
        "KEY = bytes(range(32))\n"
        "pool = WorkerPool(n_workers=4, keysource=lambda n: KEY)\n"
        "k = pc.DeviceKey.install(KEY, 0)\n"
        "n = 300\n"
        "pages = np.random.default_rng(1).integers(0, 256, size=(n, 4096), dtype=np.uint8)\n"
        "va = (0x100000000 + 4096 * np.arange(n)).astype(np.uint64)\n"
        "pid = (7 + np.arange(n) % 5).astype(np.int64)\n"
        "got = pc.crypt_pages(k, torch.from_numpy(va.view(np.int64)).cuda(), torch.from_numpy(pid).cuda(),\n"
        "                     torch.from_numpy(pages).cuda())\n"
        "torch.cuda.current_stream().synchronize()\n"
        "assert np.array_equal(got.cpu().numpy(), C.crypt_pages(KEY, va, pid.astype(np.uint32), pages))\n"
        "try:\n"
        "    pc.crypt_pages(k, torch.from_numpy((va + 1).view(np.int64)).cuda(), 1, torch.from_numpy(pages).cuda())\n"
        "    raise SystemExit('unaligned vaddr accepted')\n"
        "except pc.ContractViolation:\n"
        "    pass\n"
        "k.destroy(); pool.shutdown(); print('ok')\n")
    env = dict(os.environ)
    env.pop("CUDA_MODULE_LOADING", None)  # the default lazy loading, where the hazard lives
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=180, env=env,
                       cwd=root)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (r.returncode, r.stdout[-500:], r.stderr[-1500:])


@pytest.mark.parametrize("rounds", [8, 12, 20])
def test_key_service_small_host_batches_match_oracle(cuda, rounds):
    """DeviceKey.start_service: fault-sized host batches (contiguous, per-page
    vaddr/pid arrays, in place) run as service tickets and equal the oracle;
    larger batches and other round counts keep the launch path; the knob
    svc_pages moves the boundary; destroy() stops the workers."""
    import paper_2004_09252_b200 as pc

    key = bytes(range(40, 72))
    rng = np.random.default_rng(rounds)
    dk = pc.DeviceKey.install(key, 0)
    dk.start_service(n_workers=4, rounds=rounds)
    with pytest.raises(Exception):
        dk.start_service()  # already running
    before = _native.tune_get("launches")
    for n in (1, 2, 3, 4):
        pages = rng.integers(0, 256, (n, 4096), dtype=np.uint8)
        va = (0x7F00_0000_0000 + 4096 * rng.permutation(64)[:n]).astype(np.uint64)
        pids = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        want = C.crypt_pages(key, va, pids, pages, rounds=rounds)
        assert np.array_equal(pc.crypt_pages(dk, va, pids, pages, rounds=rounds), want)
        want1 = C.crypt_pages(key, va[0] + 4096 * np.arange(n, dtype=np.uint64),
                              np.full(n, 9, np.uint32), pages, rounds=rounds)
        buf = pages.copy()
        pc.crypt_pages(dk, int(va[0]), 9, buf, out=buf, rounds=rounds)  # in place, contiguous
        assert np.array_equal(buf, want1)
    assert _native.tune_get("launches") == before  # every batch above was <= 4 pages on 4 workers
    pages = rng.integers(0, 256, (5, 4096), dtype=np.uint8)
    want = C.crypt_pages(key, 0x1000 + 4096 * np.arange(5, dtype=np.uint64), np.full(5, 3, np.uint32), pages,
                         rounds=rounds)
    assert np.array_equal(pc.crypt_pages(dk, 0x1000, 3, pages, rounds=rounds), want)
    assert _native.tune_get("launches") > before  # 5 pages > 4 workers: the launch path
    other = 20 if rounds != 20 else 8
    before = _native.tune_get("launches")
    pc.crypt_pages(dk, 0x1000, 3, pages[:1], rounds=other)
    assert _native.tune_get("launches") > before  # the workers hold `rounds` only
    _native.tune("svc_pages", 5)
    try:
        before = _native.tune_get("launches")
        assert np.array_equal(pc.crypt_pages(dk, 0x1000, 3, pages, rounds=rounds), want)
        assert _native.tune_get("launches") == before
    finally:
        _native.tune("svc_pages", 0)
    dk.destroy()  # stops the workers first
    assert dk.destroyed


def test_key_service_start_stop_beside_concurrent_calls(cuda):
    """Four threads run 1-2 page crypt_pages calls under a key while a fifth
    starts and stops the key's resident workers over and over: every result
    equals the oracle (service or launch path, whichever was up) and no call
    uses a stopped service."""
    import paper_2004_09252_b200 as pc

    key = bytes(range(90, 122))
    dk = pc.DeviceKey.install(key, 0)
    stop = threading.Event()
    errors = []

    def worker(seed):
        rng = np.random.default_rng(seed)
        try:
            while not stop.is_set():
                n = int(rng.integers(1, 3))
                pages = rng.integers(0, 256, (n, 4096), dtype=np.uint8)
                va = 0x5000_0000 + 4096 * int(rng.integers(0, 1 << 20))
                want = C.crypt_pages(key, None, None, pages, vaddr0=va, pid0=seed)
                got = pc.crypt_pages(dk, va, seed, pages)
                if not np.array_equal(got, want):
                    errors.append(f"mismatch seed {seed}")
                    return
        except Exception as exc:  # surfaced below
            errors.append(repr(exc))

    threads = [threading.Thread(target=worker, args=(s,)) for s in range(4)]
    for t in threads:
        t.start()
    try:
        for _ in range(15):
            dk.start_service(n_workers=1)
            stop.wait(0.02)
            dk.stop_service()
    finally:
        stop.set()
        for t in threads:
            t.join()
    dk.destroy()
    assert not errors, errors[:3]


def test_key_service_many_workers_batch_limit(cuda):
    """With 40 resident workers (past the direct-polling limit: the
    dispatcher forwards the doorbells) the service takes host batches up to
    6 pages by default (each ticket costs the host ~1.2 us, so from ~8 pages
    one launch is faster) and up to the knob svc_pages (<= 64, its ticket
    array) when set; larger batches launch; all equal the oracle."""
    import paper_2004_09252_b200 as pc

    key = bytes(range(130, 162))
    rng = np.random.default_rng(5)
    with pc.DeviceKey.install(key, 0) as dk:
        dk.start_service(n_workers=40)
        cases = [(None, 6, False), (None, 7, True), (64, 64, False), (64, 70, True)]
        saved = _native.tune_get("svc_pages")
        try:
            for knob, n, launches in cases:
                _native.tune("svc_pages", 0 if knob is None else knob)
                pages = rng.integers(0, 256, (n, 4096), dtype=np.uint8)
                before = _native.tune_get("launches")
                got = pc.crypt_pages(dk, 0x8000_0000, 17, pages)
                assert (_native.tune_get("launches") > before) == launches, (knob, n)
                assert np.array_equal(got, C.crypt_pages(key, None, None, pages, vaddr0=0x8000_0000, pid0=17))
        finally:
            _native.tune("svc_pages", saved)
