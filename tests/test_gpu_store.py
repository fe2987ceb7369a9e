"""HBM-resident encrypted page store: the reference store
semantics (pkg/tests/test_store.py restated) plus the fused evict/refault
paths, byte-exact against the oracle."""

import random

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200.errors import ContractViolation
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
