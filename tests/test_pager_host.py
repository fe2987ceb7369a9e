"""CPU tests of WindowPager's host logic (no GPU): the pager runs over an
in-memory stand-in for DevicePageStore whose cipher is the oracle, and is
checked against a pure-Python model of the reference orchestrator's fault /
eviction semantics (pkg/src/pagecrypt/orchestrator.py:175-240), including
which store calls it makes (one fused swap per refaulting fault) and that a
failed fault leaves the window untouched."""

import random

import numpy as np
import pytest

from oracle import chacha_oracle as O
from paper_2004_09252_b200.errors import ContractViolation
from paper_2004_09252_b200.pager import SlidingWindow, WindowPager
from paper_2004_09252_b200.workers import ClientId

KEY = bytes(range(3, 35))
C = ClientId(99, 1)


class FakeStore:
    """DevicePageStore's pager-facing API over a dict, oracle cipher."""

    def __init__(self):
        self.key = object()
        self.ct = {}
        self.calls = []
        self.fail_next = None

    def _maybe_fail(self, name):
        if self.fail_next == name:
            self.fail_next = None
            raise RuntimeError(f"{name} failed")

    def contains(self, client, v):
        return (client, v) in self.ct

    def refault_many(self, client, vaddrs):
        self.calls.append(("refault_many", len(vaddrs)))
        self._maybe_fail("refault_many")
        out = np.stack([np.frombuffer(O.crypt_page(KEY, v, client.pid, self.ct[(client, v)]), np.uint8)
                        for v in vaddrs])
        for v in vaddrs:
            del self.ct[(client, v)]
        return out

    def evict_many(self, client, vaddrs, plains):
        self.calls.append(("evict_many", len(vaddrs)))
        self._maybe_fail("evict_many")
        for v, p in zip(vaddrs, plains):
            assert (client, v) not in self.ct
            self.ct[(client, v)] = O.crypt_page(KEY, v, client.pid, p.tobytes())

    def swap(self, client, get, put, plains):
        self.calls.append(("swap", len(get), len(put)))
        self._maybe_fail("swap")
        out = np.stack([np.frombuffer(O.crypt_page(KEY, v, client.pid, self.ct.pop((client, v))), np.uint8)
                        for v in get])
        for v, p in zip(put, plains):
            self.ct[(client, v)] = O.crypt_page(KEY, v, client.pid, p.tobytes())
        return out

    def drop_client(self, client):
        for k in [k for k in self.ct if k[0] == client]:
            del self.ct[k]


def scribble(v, plain: bytes) -> bytes:
    b = bytearray(plain)
    b[(v >> 12) % 4096] ^= 0xA5
    return bytes(b)


class Model:
    def __init__(self, W):
        self.win = SlidingWindow(W)
        self.store = {}
        self.client = {}

    def batch(self, vs):
        outs, fresh = [], {}
        for v in vs:
            ct = self.store.pop(v, None)
            plain = bytes(4096) if ct is None else O.crypt_page(KEY, v, C.pid, ct)
            ev = self.win.admit(v)
            if ev is not None:
                ev_plain = fresh.pop(ev) if ev in fresh else self.client.pop(ev)
                self.store[ev] = O.crypt_page(KEY, ev, C.pid, ev_plain)
            fresh[v] = plain
            outs.append(plain)
        for v, plain in fresh.items():
            self.client[v] = scribble(v, plain)
        return outs


def make(W):
    store = FakeStore()
    mem = {}

    def fetch(client, vaddrs):
        return np.stack([np.frombuffer(mem.pop(v), np.uint8) for v in vaddrs])

    pager = WindowPager(store, fetch, window_capacity=W)
    pager.register(C)
    return pager, store, mem


@pytest.mark.parametrize("batch", [1, 2, 5, 12])
def test_random_traces_match_reference_semantics(batch):
    W = 5
    rng = random.Random(batch)
    pager, store, mem = make(W)
    model = Model(W)
    pages = [0x40000 + 4096 * i for i in range(24)]
    for _ in range(30):
        resident = set(pager.window(C))
        vs = rng.sample([p for p in pages if p not in resident], batch)
        got = pager.fault_batch(C, vs)
        assert [g.tobytes() for g in got] == model.batch(vs)
        for v in pager.window(C):
            if v in vs:
                mem[v] = scribble(v, got[vs.index(v)].tobytes())
        assert pager.window(C) == model.win.members()
    assert {v: ct for (c, v), ct in store.ct.items()} == model.store
    m = pager.metrics[C]
    assert m.faults == 30 * batch and m.first_touch_faults + m.decrypt_ops == m.faults
    # batch <= W: the evictions were all resident before the batch (and a
    # refault implies a full window), so every refaulting batch is ONE swap
    if batch <= W:
        assert not any(c[0] == "refault_many" for c in store.calls)
        assert any(c[0] == "swap" for c in store.calls)
    else:
        assert not any(c[0] == "swap" for c in store.calls)


def test_single_faults_use_one_swap_when_refaulting():
    pager, store, mem = make(2)
    for v in (0x1000, 0x2000):
        pager.fault(C, v)
        mem[v] = bytes([v >> 12]) * 4096
    assert store.calls == []  # first touches with room in the window: no GPU work
    pager.fault(C, 0x3000)  # first touch, evicts 0x1000
    assert store.calls == [("evict_many", 1)]
    mem[0x3000] = b"\x03" * 4096
    store.calls.clear()
    assert pager.fault(C, 0x1000) == b"\x01" * 4096  # refault + evict 0x2000
    assert store.calls == [("swap", 1, 1)]
    assert pager.metrics[C].gpu_batches == 2


def test_batch_larger_than_window_does_not_fuse():
    pager, store, mem = make(2)
    pager.fault_batch(C, [0x1000, 0x2000, 0x3000, 0x4000])  # 0x1000, 0x2000 evicted by the batch itself
    assert store.calls == [("evict_many", 2)]
    store.calls.clear()
    mem[0x3000], mem[0x4000] = b"\x03" * 4096, b"\x04" * 4096
    got = pager.fault_batch(C, [0x1000, 0x2000, 0x5000])  # refaults; 0x1000 is evicted again by 0x5000
    assert [g.tobytes() for g in got] == [bytes(4096)] * 3
    assert store.calls == [("refault_many", 2), ("evict_many", 3)]


@pytest.mark.parametrize("where", ["fetch", "swap", "refault_many", "evict_many"])
def test_failed_fault_restores_the_window(where):
    pager, store, mem = make(2)
    for v in (0x1000, 0x2000, 0x3000):
        pager.fault(C, v)
        mem[v] = bytes([v >> 12]) * 4096
    before = pager.window(C)
    if where == "fetch":
        pager.fetch_evicted = lambda c, vs: (_ for _ in ()).throw(RuntimeError("client gone"))
        vs = [0x1000]
    elif where == "swap":
        store.fail_next = "swap"
        vs = [0x1000]
    else:  # the unfused path: a batch bigger than the window
        store.fail_next = where
        vs = [0x1000, 0x4000, 0x5000]
    with pytest.raises(RuntimeError):
        pager.fault_batch(C, vs)
    assert pager.window(C) == before


def test_contract_errors_on_cpu():
    pager, store, mem = make(2)
    with pytest.raises(ContractViolation):
        pager.fault(ClientId(1, 1), 0x1000)
    with pytest.raises(ContractViolation):
        pager.fault_batch(C, [0x1000, 0x1000])
    with pytest.raises(ContractViolation):
        pager.fault(C, 0x1001)
    pager.fault(C, 0x1000)
    with pytest.raises(ContractViolation):
        pager.fault(C, 0x1000)


def test_clients_are_isolated():
    """Several clients interleave faults through one pager and one store:
    each sees exactly its own single-client history (test_bench.py:143-156
    counter isolation; the pid enters every ciphertext)."""
    W = 3
    store = FakeStore()
    mems = {}

    def fetch(client, vaddrs):
        return np.stack([np.frombuffer(mems[client].pop(v), np.uint8) for v in vaddrs])

    pager = WindowPager(store, fetch, window_capacity=W)
    clients = [ClientId(10 + i, i) for i in range(3)]
    solo = {}
    for cl in clients:
        pager.register(cl)
        mems[cl] = {}
        # the same client alone, for reference
        s_store = FakeStore()
        s_mem = {}
        s_pager = WindowPager(s_store, lambda c, vs, m=s_mem: np.stack([np.frombuffer(m.pop(v), np.uint8) for v in vs]), W)
        s_pager.register(cl)
        solo[cl] = (s_pager, s_store, s_mem)
    rng = random.Random(5)
    pages = [0x70000 + 4096 * i for i in range(8)]
    for _ in range(150):
        cl = rng.choice(clients)
        v = rng.choice([p for p in pages if p not in pager.window(cl)])
        got = pager.fault(cl, v)
        s_pager, s_store, s_mem = solo[cl]
        want = s_pager.fault(cl, v)
        assert got == want
        data = scribble(v ^ cl.pid, got)
        mems[cl][v] = data
        s_mem[v] = data
    for cl in clients:
        s_pager, s_store, _ = solo[cl]
        assert pager.window(cl) == s_pager.window(cl)
        assert {k: c for k, c in store.ct.items() if k[0] == cl} == s_store.ct
        a, b = pager.metrics[cl], s_pager.metrics[cl]
        assert (a.faults, a.evictions, a.decrypt_ops, a.encrypt_ops) == (b.faults, b.evictions, b.decrypt_ops, b.encrypt_ops)


class NativeFakeStore(FakeStore):
    """FakeStore plus DevicePageStore.fault (pc_store_fault's contract): the
    pager then resolves a single fault as one native call."""

    def fault(self, client, vaddr, out, evict_vaddr=None, evict_plain=None):
        self.calls.append(("fault", evict_plain is not None))
        self._maybe_fail("fault")
        assert out.dtype == np.uint8 and out.size == 4096
        if evict_plain is not None:
            assert isinstance(evict_plain, np.ndarray) and evict_plain.dtype == np.uint8
            assert evict_plain.size == 4096 and evict_plain.flags.c_contiguous
            if (client, evict_vaddr) in self.ct and evict_vaddr != vaddr:
                raise ContractViolation("duplicate store insert")
        hit = (client, vaddr) in self.ct
        if hit:
            out[:] = np.frombuffer(O.crypt_page(KEY, vaddr, client.pid, self.ct.pop((client, vaddr))), np.uint8)
        if evict_plain is not None:
            self.ct[(client, evict_vaddr)] = O.crypt_page(KEY, evict_vaddr, client.pid, evict_plain.tobytes())
        return hit


@pytest.mark.parametrize("W", [1, 4])
def test_native_single_faults_match_reference_semantics(W):
    """Single faults through the store's one-call fault (the resident-worker
    path on a GPU) give the reference orchestrator's results; the client's
    page handed to the eviction is not modified (the library copies it)."""
    store = NativeFakeStore()
    mem = {}
    handed = []

    def fetch(client, vaddrs):
        page = np.frombuffer(mem.pop(vaddrs[0]), np.uint8).copy()
        handed.append((page, page.copy()))
        return page  # one page as is (the bench's client)

    pager = WindowPager(store, fetch, window_capacity=W)
    pager.register(C)
    model = Model(W)
    rng = random.Random(W)
    pages = [0x20000 + 4096 * i for i in range(12)]
    for _ in range(200):
        resident = set(pager.window(C))
        v = rng.choice([p for p in pages if p not in resident])
        got = pager.fault(C, v)
        assert [got] == model.batch([v])
        mem[v] = scribble(v, got)
    assert all(np.array_equal(a, b) for a, b in handed)
    assert {k[1]: c for k, c in store.ct.items()} == model.store
    assert all(c[0] == "fault" for c in store.calls)


def test_native_fault_converts_and_checks_the_evicted_page():
    """fetch_evicted may hand back any array-like of the page's 4096 byte
    values (a private uint8 copy is made, and wiped); a wrong size is a
    ContractViolation and the window is left as it was."""
    store = NativeFakeStore()
    mem = {}
    pager = WindowPager(store, lambda c, vs: mem.pop(vs[0]), window_capacity=1)
    pager.register(C)
    pager.fault(C, 0x1000)
    mem[0x1000] = np.arange(4096, dtype=np.int64) % 256  # int64 values, not uint8 bytes
    pager.fault(C, 0x2000)  # evicts 0x1000
    assert store.ct[(C, 0x1000)] == O.crypt_page(KEY, 0x1000, C.pid, (np.arange(4096) % 256).astype(np.uint8).tobytes())
    mem[0x2000] = np.zeros(100, np.uint8)
    with pytest.raises(ContractViolation):
        pager.fault(C, 0x3000)
    assert pager.window(C) == [0x2000]
