"""HBM-resident encrypted page store: the reference store
semantics (pkg/tests/test_store.py restated) plus the fused evict/refault
paths, byte-exact against the oracle."""

import random

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200.errors import ContractViolation, PageCryptError
from paper_2004_09252_b200.store import DevicePageStore, StoreFull
from paper_2004_09252_b200.workers import ClientId

from oracle import coracle as C

pytestmark = pytest.mark.gpu

C1 = ClientId(100, 0)
C2 = ClientId(200, 0)
KEY = bytes(range(32))


def page(fill):
    return bytes([fill]) * 4096


@pytest.fixture
def store(cuda):
    return DevicePageStore(64)


@pytest.fixture(scope="module")
def dkey(cuda):
    k = pc.DeviceKey.install(KEY, 0)
    yield k
    k.destroy()


def test_insert_then_lookup_identical(store):
    store.insert(C1, 0x1000, page(0xAB))
    assert store.lookup(C1, 0x1000) == page(0xAB)


def test_traversal_sorted_by_vaddr(store):
    for v in (0x3000, 0x1000, 0x2000):
        store.insert(C1, v, page(v >> 12))
    assert [(v, d) for v, d in store.pages(C1)] == [(v, page(v >> 12)) for v in (0x1000, 0x2000, 0x3000)]


def test_duplicate_insert_rejected(store):
    store.insert(C1, 0x1000, page(1))
    with pytest.raises(ContractViolation):
        store.insert(C1, 0x1000, page(2))


def test_lookup_empty_and_after_remove(store):
    assert store.lookup(C1, 0x1000) is None
    store.insert(C1, 0x1000, page(1))
    store.remove(C1, 0x1000)
    assert store.lookup(C1, 0x1000) is None
    with pytest.raises(ContractViolation):
        store.remove(C1, 0x1000)


def test_remove_then_reinsert(store):
    store.insert(C1, 0x1000, page(1))
    store.remove(C1, 0x1000)
    store.insert(C1, 0x1000, page(2))
    assert store.lookup(C1, 0x1000) == page(2)


def test_freed_slots_are_wiped(cuda):
    """Remove/refault/drop_client zero the HBM slot: a 1-slot store reused
    through the raw path shows zeros in between (store.py:86-92)."""
    s = DevicePageStore(1)
    s.insert(C1, 0x1000, page(0xEE))
    s.remove(C1, 0x1000)
    s.insert(C1, 0x1000, page(0x11))
    assert s.lookup(C1, 0x1000) == page(0x11)
    s.drop_client(C1)
    assert s.free_slots == 1


def test_epoch_separates_clients(cuda):
    s = DevicePageStore(4)
    s.insert(ClientId(5, 0), 0x1000, page(1))
    assert s.lookup(ClientId(5, 1), 0x1000) is None


def test_drop_client_and_isolation(store):
    for v in (0x1000, 0x2000):
        store.insert(C1, v, page(1))
    store.insert(C2, 0x1000, page(2))
    assert store.lookup(C2, 0x2000) is None
    store.drop_client(C1)
    store.drop_client(ClientId(999, 0))
    assert store.lookup(C1, 0x1000) is None and store.page_count(C1) == 0
    assert store.lookup(C2, 0x1000) == page(2)
    assert store.free_slots == 63


def test_validation(store):
    with pytest.raises(ContractViolation):
        store.insert(C1, 0x1234, page(1))
    with pytest.raises(ContractViolation):
        store.insert(C1, 0x1000, b"short")


def test_capacity(cuda):
    s = DevicePageStore(2)
    s.insert(C1, 0x1000, page(1))
    s.insert(C1, 0x2000, page(2))
    with pytest.raises(StoreFull):
        s.insert(C1, 0x3000, page(3))
    s.remove(C1, 0x1000)
    s.insert(C1, 0x3000, page(3))


def test_matches_sorted_assoc_list_on_random_ops(cuda):
    rng = random.Random(42)
    s = DevicePageStore(300)
    model = {}
    vaddrs = [v * 4096 for v in range(1, 257)]
    for step in range(3000):
        v = rng.choice(vaddrs)
        op = rng.random()
        if op < 0.5:
            if v not in model:
                data = bytes([step % 256]) * 4096
                s.insert(C1, v, data)
                model[v] = data
        elif op < 0.8:
            assert s.lookup(C1, v) == model.get(v)
        elif v in model:
            s.remove(C1, v)
            del model[v]
    assert [(v, d) for v, d in s.pages(C1)] == sorted(model.items())


@pytest.mark.parametrize("rounds", [8, 20])
def test_evict_refault_roundtrip_matches_oracle(dkey, rounds):
    s = DevicePageStore(5000, dkey, rounds=rounds)
    rng = np.random.default_rng(rounds)
    n = 3000
    plains = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
    vaddrs = (rng.permutation(100000)[:n].astype(np.uint64) * np.uint64(4096) + np.uint64(0x1_0000_0000))
    c = ClientId(4242, 7)
    s.evict_many(c, vaddrs, plains)
    # the stored bytes are the reference ciphertext (only pid in the seed)
    want = C.crypt_pages(KEY, vaddrs, 4242, plains, rounds=rounds, nthreads=8)
    for i in (0, 1, n - 1):
        assert s.lookup(c, int(vaddrs[i])) == want[i].tobytes()
    got = dict(s.pages(c))
    assert all(got[int(v)] == want[i].tobytes() for i, v in enumerate(vaddrs[:50]))
    # refault in a different order returns the plaintexts and frees the slots
    order = rng.permutation(n)
    back = s.refault_many(c, vaddrs[order])
    assert np.array_equal(back, plains[order])
    assert s.page_count(c) == 0 and s.free_slots == 5000


def test_single_page_fused_paths(dkey):
    s = DevicePageStore(8, dkey)
    plain = bytes(range(256)) * 16
    s.evict(C1, 0x7000, plain)
    assert s.lookup(C1, 0x7000) == pc.crypt_page(KEY, 0x7000, C1.pid, plain)
    assert s.refault(C1, 0x7000) == plain
    assert not s.contains(C1, 0x7000)
    with pytest.raises(ContractViolation):
        s.refault(C1, 0x7000)
    # batches are all-or-nothing
    s.evict(C1, 0x1000, plain)
    with pytest.raises(ContractViolation):
        s.evict_many(C1, [0x2000, 0x1000], np.zeros((2, 4096), np.uint8))
    assert not s.contains(C1, 0x2000)
    with pytest.raises(ContractViolation):
        s.refault_many(C1, [0x1000, 0x3000])
    assert s.contains(C1, 0x1000)
    with pytest.raises(StoreFull):
        s.evict_many(C1, [0x10000 * i for i in range(1, 9)], np.zeros((8, 4096), np.uint8))


# ---- pc_store_swap: one fault (refault + eviction) in one GPU round trip ----


@pytest.mark.parametrize("rounds", [8, 12, 20])
def test_swap_matches_refault_then_evict(dkey, rounds):
    """swap == refault_many followed by evict_many: same plaintexts out, same
    ciphertext stored (the oracle's), same slot accounting."""
    rng = np.random.default_rng(rounds)
    s = DevicePageStore(512, dkey, rounds=rounds)
    c = ClientId(77, 3)
    va = [0x1_0000_0000 + 4096 * i for i in range(300)]
    plains = rng.integers(0, 256, size=(300, 4096), dtype=np.uint8)
    s.evict_many(c, va[:20], plains[:20])
    for n_get, n_put in ((1, 1), (0, 3), (5, 0), (7, 9), (20, 20), (20, 108), (64, 64), (100, 100)):
        # fused up to 128 pages in total, refault-then-evict above
        get = [v for v in va if s.contains(c, v)][:n_get]
        put = [v for v in va if not s.contains(c, v)][:n_put]
        want_out = np.stack([plains[va.index(v)] for v in get]) if get else np.empty((0, 4096), np.uint8)
        put_pl = np.stack([plains[va.index(v)] for v in put]) if put else np.empty((0, 4096), np.uint8)
        free0 = s.free_slots
        got = s.swap(c, get, put, put_pl)
        assert np.array_equal(got, want_out)
        assert s.free_slots == free0 + len(get) - len(put)
        assert not any(s.contains(c, v) for v in get)
        if put:
            want_ct = C.crypt_pages(KEY, np.array(put, np.uint64), c.pid, put_pl, rounds=rounds)
            for v, ct in zip(put, want_ct):
                assert s.lookup(c, v) == ct.tobytes()


def test_swap_same_vaddr_out_and_back_in(dkey):
    s = DevicePageStore(4, dkey)
    p1, p2 = page(1), page(2)
    s.evict(C1, 0x5000, p1)
    got = s.swap(C1, [0x5000], [0x5000], np.frombuffer(p2, np.uint8).reshape(1, 4096))
    assert got[0].tobytes() == p1
    assert s.refault(C1, 0x5000) == p2
    assert s.free_slots == 4


def test_swap_full_slab_falls_back_and_zeroes_freed_slots(dkey):
    s = DevicePageStore(2, dkey)
    s.evict(C1, 0x1000, page(1))
    s.evict(C1, 0x2000, page(2))
    # no free slot before the refault frees one: runs as refault then evict
    got = s.swap(C1, [0x1000], [0x3000], np.frombuffer(page(3), np.uint8).reshape(1, 4096))
    assert got[0].tobytes() == page(1)
    assert s.refault(C1, 0x3000) == page(3)
    assert s.refault(C1, 0x2000) == page(2)
    assert s.free_slots == 2


def test_swap_is_all_or_nothing(dkey):
    s = DevicePageStore(16, dkey)
    s.evict(C1, 0x1000, page(1))
    s.evict(C1, 0x2000, page(2))
    one = np.frombuffer(page(9), np.uint8).reshape(1, 4096)
    with pytest.raises(ContractViolation):  # refault of a missing page
        s.swap(C1, [0x1000, 0x9000], [0x3000], one)
    with pytest.raises(ContractViolation):  # eviction onto a stored page
        s.swap(C1, [0x1000], [0x2000], one)
    with pytest.raises(ContractViolation):  # unaligned eviction vaddr
        s.swap(C1, [0x1000], [0x3001], one)
    with pytest.raises(ContractViolation):  # duplicate refault
        s.swap(C1, [0x1000, 0x1000], [], np.empty((0, 4096), np.uint8))
    assert s.contains(C1, 0x1000) and s.contains(C1, 0x2000) and not s.contains(C1, 0x3000)
    assert s.free_slots == 14
    assert s.refault(C1, 0x1000) == page(1)


def test_batch_naming_a_page_twice_is_rejected_whole(dkey):
    """remove / refault batches that name a page twice fail without freeing
    any slot (a double free would hand one slot to two pages later)."""
    import ctypes

    from paper_2004_09252_b200 import _native
    from paper_2004_09252_b200.store import _cid

    s = DevicePageStore(8, dkey)
    s.evict_many(C1, [0x1000, 0x2000], np.stack([np.frombuffer(page(1), np.uint8), np.frombuffer(page(2), np.uint8)]))
    lib = _native.load()
    va = np.array([0x1000, 0x2000, 0x1000], dtype=np.uint64)
    assert lib.pc_store_remove(s._h, _cid(C1), va.ctypes.data, 3) == _native.PC_EINVAL
    assert b"duplicate" in lib.pc_last_error()
    assert s.free_slots == 6 and s.contains(C1, 0x1000) and s.contains(C1, 0x2000)
    with pytest.raises(ContractViolation):
        s.refault_many(C1, [0x2000, 0x1000, 0x2000])
    assert s.free_slots == 6
    assert s.refault(C1, 0x1000) == page(1) and s.refault(C1, 0x2000) == page(2)
    assert s.free_slots == 8
    # duplicate lookups (no remove) are fine
    s.evict(C1, 0x3000, page(3))
    assert s.lookup(C1, 0x3000) == s.lookup(C1, 0x3000)


def test_stored_ciphertext_histogram(dkey):
    """The reference's ciphertext smoke test (analyzer.ciphertext_histogram_ok,
    pkg/tests/test_analyzer.py:200-215): 260 low-entropy pages (each one
    repeated byte) evicted into the HBM store, >= 1 MiB of ciphertext, and no
    byte value more frequent than 3x uniform -- here also a chi-square bound."""
    s = DevicePageStore(512, dkey)
    pages = np.stack([np.full(4096, i % 256, np.uint8) for i in range(260)])
    va = [0x1_0000_0000 + 4096 * i for i in range(260)]
    s.evict_many(ClientId(5, 0), va, pages)
    blob = np.concatenate([np.frombuffer(ct, np.uint8) for _, ct in s.pages(ClientId(5, 0))])
    assert blob.size >= 1 << 20
    counts = np.bincount(blob, minlength=256)
    expect = blob.size / 256
    assert counts.max() <= 3.0 * expect
    chi2 = float(((counts - expect) ** 2 / expect).sum())
    assert chi2 < 400  # 255 dof: mean 255, sd ~22.6
    s.close()


@pytest.mark.parametrize("service", [False, True], ids=["launch", "service"])
def test_native_fault_entry(dkey, service):
    """DevicePageStore.fault (pc_store_fault): one orchestrator fault --
    lookup, refault and the forced eviction -- in one call (one launch, or
    one ticket of the store's resident worker)."""
    s = DevicePageStore(8, dkey)
    if service:
        s.start_service()
    out = np.full(4096, 7, np.uint8)
    assert s.fault(C1, 0x1000, out) is False and (out == 7).all()  # first touch: untouched
    assert s.fault(C1, 0x2000, out, 0x1000, np.frombuffer(page(1), np.uint8)) is False
    assert s.lookup(C1, 0x1000) == pc.crypt_page(KEY, 0x1000, C1.pid, page(1))
    # refault 0x1000 while evicting 0x2000: one launch
    assert s.fault(C1, 0x1000, out, 0x2000, np.frombuffer(page(2), np.uint8)) is True
    assert out.tobytes() == page(1)
    assert not s.contains(C1, 0x1000) and s.refault(C1, 0x2000) == page(2)
    assert s.free_slots == 8
    with pytest.raises(ContractViolation):
        s.fault(C1, 0x1001, out)
    with pytest.raises(ContractViolation):
        s.fault(C1, 0x1000, out, 0x3000, np.zeros(100, np.uint8))


def test_out_of_range_vaddrs_never_alias_stored_pages(dkey):
    """contains/lookup of a vaddr the store can never hold (negative,
    >= 2**64, unaligned) answer False/None like the reference's dict lookups
    (store.py:67-86) -- in particular -4096 must not wrap onto
    0xffff_ffff_ffff_f000 -- and insert/remove of one raise."""
    s = DevicePageStore(8, dkey)
    top = 2**64 - 4096
    s.evict(C1, top, bytes(4096))
    assert s.contains(C1, top)
    for bad in (-4096, 2**64 + top, top + 1):
        assert not s.contains(C1, bad)
        assert s.lookup(C1, bad) is None
        with pytest.raises(ContractViolation):
            s.remove(C1, bad)
        with pytest.raises(ContractViolation):
            s.insert(C1, bad, bytes(4096))
    assert s.refault(C1, top) == bytes(4096)
    s.close()


@pytest.fixture
def bell_ops():
    """Set the svc_bell_ops knob for one test (1: a store ticket's slots ride
    in the doorbell line; 0: the workers read the op line, the fallback)."""
    from paper_2004_09252_b200 import _native

    saved = _native.tune_get("svc_bell_ops")
    yield lambda v: _native.tune("svc_bell_ops", v)
    _native.tune("svc_bell_ops", saved)


@pytest.mark.parametrize("in_bell", [1, 0], ids=["slots_in_doorbell", "op_line"])
@pytest.mark.parametrize("rounds", [8, 12, 20])
def test_service_faults_match_launch_faults(dkey, rounds, in_bell, bell_ops):
    """A random fault stream (refault + eviction, refault only, eviction only,
    first touch) through the resident worker gives the same outputs, the
    same stored ciphertext (== the oracle's) and the same free-slot count as
    the same stream through pc_store_swap launches."""
    bell_ops(in_bell)
    rng = np.random.default_rng(rounds)
    stores = [DevicePageStore(40, dkey, rounds=rounds) for _ in range(2)]
    stores[1].start_service()
    assert stores[1].service_running and not stores[0].service_running
    held = {}  # vaddr -> plaintext the client holds (evictable)
    stored = set()
    for step in range(300):
        v = 0x7000_0000 + 4096 * int(rng.integers(0, 64))
        if v in held:
            continue
        ev = None
        if held and (rng.random() < 0.7 or len(stored) >= 38):
            ev = list(held)[int(rng.integers(0, len(held)))]
        if ev is None and len(stored) >= 38:
            continue
        outs = []
        for s in stores:
            out = np.full(4096, 0xEE, np.uint8)
            plain = None if ev is None else np.frombuffer(held[ev], np.uint8).copy()
            hit = s.fault(C1, v, out, ev, plain)
            outs.append((hit, out.tobytes()))
        assert outs[0] == outs[1], step
        hit, got = outs[0]
        assert hit == (v in stored)
        if ev is not None:
            stored.add(ev)
            del held[ev]
        if hit:
            stored.discard(v)
        held[v] = (got if hit else bytes(4096))[:7] + rng.bytes(4096 - 7)
    for s in stores:
        assert s.free_slots == 40 - len(stored)
        for v in stored:
            assert s.lookup(C1, v) == stores[0].lookup(C1, v)
    for v in list(stored)[:5]:
        plain = stores[1].refault(C1, v)
        want = C.crypt_pages(KEY, np.array([v], np.uint64), np.array([C1.pid], np.uint32),
                             np.frombuffer(plain, np.uint8).reshape(1, 4096), rounds=rounds)
        assert stores[0].lookup(C1, v) == want.tobytes()
    stores[1].stop_service()
    assert not stores[1].service_running
    for s in stores:
        s.close()


def test_service_fault_errors_leave_store_unchanged(dkey):
    """Errors on the service path are the launch path's: a duplicate insert,
    a full store, bad arguments -- and nothing changes."""
    s = DevicePageStore(1, dkey)
    s.start_service()
    out = np.zeros(4096, np.uint8)
    assert s.fault(C1, 0x2000, out, 0x1000, np.frombuffer(page(1), np.uint8)) is False
    with pytest.raises(StoreFull):  # first touch + eviction into a full slab
        s.fault(C1, 0x3000, out, 0x4000, np.frombuffer(page(2), np.uint8))
    with pytest.raises(ContractViolation):  # 0x1000 is stored and not refaulted by this fault
        s.fault(C1, 0x5000, out, 0x1000, np.frombuffer(page(3), np.uint8))
    with pytest.raises(ContractViolation):
        s.fault(C1, 0x1001, out)
    assert s.free_slots == 0 and s.lookup(C1, 0x1000) == pc.crypt_page(KEY, 0x1000, C1.pid, page(1))
    # refault + evict the same vaddr back in (the freed slot is reused)
    assert s.fault(C1, 0x1000, out, 0x1000, np.frombuffer(page(4), np.uint8)) is True
    assert out.tobytes() == page(1) and s.refault(C1, 0x1000) == page(4)
    with pytest.raises(ContractViolation):
        s.start_service(0)
    with pytest.raises(PageCryptError):
        s.start_service()  # already running
    s.close()  # stops the worker
    keyless = DevicePageStore(2)
    with pytest.raises(PageCryptError):
        keyless.start_service()
    keyless.close()


def test_store_service_start_stop_beside_concurrent_faults(dkey):
    """Three threads fault their own clients' pages through one store while a
    fourth starts and stops the store's resident worker over and over: every
    refault returns what was evicted (oracle-checked ciphertext in between),
    whichever path -- ticket or launch -- served it."""
    import threading

    s = DevicePageStore(256, dkey)
    stop = threading.Event()
    errors = []

    def worker(t):
        rng = np.random.default_rng(t)
        c = ClientId(500 + t, 0)
        held = {}  # vaddr -> plaintext the client holds
        stored = {}  # vaddr -> plaintext evicted into the store
        try:
            while not stop.is_set():
                v = 0x4000_0000 + 4096 * int(rng.integers(0, 24))
                if v in held:
                    continue
                out = np.zeros(4096, np.uint8)
                ev = next(iter(held)) if len(held) >= 4 else None
                plain = None if ev is None else np.frombuffer(held[ev], np.uint8).copy()
                hit = s.fault(c, v, out, ev, plain)
                if hit != (v in stored) or (hit and out.tobytes() != stored.pop(v)):
                    errors.append(f"thread {t}: wrong refault of {v:#x}")
                    return
                if ev is not None:
                    stored[ev] = held.pop(ev)
                held[v] = rng.bytes(4096)
        except Exception as exc:
            errors.append(f"thread {t}: {exc!r}")

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(3)]
    for th in threads:
        th.start()
    try:
        for _ in range(12):
            s.start_service()
            stop.wait(0.03)
            s.stop_service()
            stop.wait(0.01)
    finally:
        stop.set()
        for th in threads:
            th.join()
    s.close()
    assert not errors, errors[:3]
