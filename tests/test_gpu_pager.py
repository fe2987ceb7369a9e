"""Batched fault/eviction resolution: WindowPager over the
HBM store against a pure-Python model of the reference orchestrator's
semantics (orchestrator.py:175-240: zero page on first touch, decrypt +
remove on refault, FIFO window admission, encrypt + insert of the client's
page on eviction), with the cipher from the oracle.  The client writes into
its pages after each batch; a page faulted in and evicted by the same batch
is stored as it was resolved."""

import random

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200.errors import ContractViolation
from paper_2004_09252_b200.pager import SlidingWindow, WindowPager
from paper_2004_09252_b200.store import DevicePageStore
from paper_2004_09252_b200.workers import ClientId

from oracle import chacha_oracle as O

pytestmark = pytest.mark.gpu

KEY = bytes(range(7, 39))
C = ClientId(321, 5)


def scribble(v, plain: bytes) -> bytes:
    """The client's write into a resident page (deterministic)."""
    b = bytearray(plain)
    b[(v >> 12) % 4096] ^= 0x5A
    b[0] = (b[0] + 1) % 256
    return bytes(b)


class Model:
    def __init__(self, W):
        self.win = SlidingWindow(W)
        self.store = {}  # vaddr -> ciphertext
        self.client = {}  # resident vaddr -> bytes the client holds

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
        for v, plain in fresh.items():  # client installs, then writes
            self.client[v] = scribble(v, plain)
        return outs


@pytest.fixture(scope="module")
def dkey(cuda):
    k = pc.DeviceKey.install(KEY, 0)
    yield k
    k.destroy()


@pytest.mark.parametrize("service", [False, True], ids=["launch", "service"])
@pytest.mark.parametrize("batch", [1, 3, 8, 20])
def test_trace_matches_reference_semantics(dkey, batch, service):
    W = 8
    rng = random.Random(batch)
    store = DevicePageStore(512, dkey)
    if service:  # single faults through the resident worker, batches still launch
        store.start_service()
    client_mem = {}

    def fetch(client, vaddrs):
        return np.stack([np.frombuffer(client_mem.pop(v), np.uint8) for v in vaddrs])

    pager = WindowPager(store, fetch, window_capacity=W)
    pager.register(C)
    model = Model(W)
    pages = [0x10000 + 4096 * i for i in range(48)]
    for _ in range(40):
        resident = set(pager.window(C))
        vs = rng.sample([p for p in pages if p not in resident], batch)
        got = pager.fault_batch(C, vs)
        want = model.batch(vs)
        assert [g.tobytes() for g in got] == want
        for v in pager.window(C):  # the client installs and writes its resident pages
            if v in vs:
                client_mem[v] = scribble(v, got[vs.index(v)].tobytes())
        assert pager.window(C) == model.win.members()
    # HBM ciphertext == the reference ciphertext of what was evicted
    for v, ct in model.store.items():
        assert store.lookup(C, v) == ct
    assert sorted(v for v, _ in store.pages(C)) == sorted(model.store)
    m = pager.metrics[C]
    assert m.faults == 40 * batch
    assert m.first_touch_faults + m.decrypt_ops == m.faults
    assert m.evictions == m.decrypt_ops + len(model.store)  # every refault consumed one eviction
    pager.unregister(C)
    assert store.page_count(C) == 0


@pytest.mark.parametrize("service", [False, True], ids=["launch", "service"])
def test_single_fault_matches_orchestrator_flow(dkey, service):
    """W=1: every fault evicts the previous page (test_orchestrator.py:212-229 style)."""
    store = DevicePageStore(16, dkey)
    if service:
        store.start_service()
    mem = {}
    pager = WindowPager(store, lambda c, vs: np.stack([np.frombuffer(mem.pop(v), np.uint8) for v in vs]), 1)
    pager.register(C)
    assert pager.fault(C, 0x1000) == bytes(4096)  # first touch
    mem[0x1000] = b"\x11" * 4096
    assert pager.fault(C, 0x2000) == bytes(4096)  # evicts 0x1000
    assert store.lookup(C, 0x1000) == O.crypt_page(KEY, 0x1000, C.pid, b"\x11" * 4096)
    mem[0x2000] = b"\x22" * 4096
    assert pager.fault(C, 0x1000) == b"\x11" * 4096  # refault decrypts, evicts 0x2000
    assert not store.contains(C, 0x1000)
    assert store.lookup(C, 0x2000) == O.crypt_page(KEY, 0x2000, C.pid, b"\x22" * 4096)
    m = pager.metrics[C]
    assert (m.faults, m.first_touch_faults, m.decrypt_ops, m.evictions) == (3, 2, 1, 2)
    assert m.gpu_batches == 2  # the refaulting fault is ONE pc_store_swap round trip


def test_failed_fault_leaves_window_and_store_unchanged(dkey):
    store = DevicePageStore(16, dkey)
    mem = {}
    fail = [False]

    def fetch(c, vs):
        if fail[0]:
            raise RuntimeError("client unreachable")
        return np.stack([np.frombuffer(mem.pop(v), np.uint8) for v in vs])

    pager = WindowPager(store, fetch, 2)
    pager.register(C)
    for v in (0x1000, 0x2000, 0x3000):  # 0x1000 evicted by the third fault
        pager.fault(C, v)
        mem[v] = bytes([v >> 12]) * 4096
    mem.pop(0x1000, None)
    fail[0] = True
    with pytest.raises(RuntimeError):
        pager.fault(C, 0x1000)  # would refault 0x1000 and evict 0x2000
    assert pager.window(C) == [0x2000, 0x3000]
    assert store.contains(C, 0x1000) and not store.contains(C, 0x2000)
    fail[0] = False
    assert pager.fault(C, 0x1000) == b"\x01" * 4096
    assert pager.window(C) == [0x3000, 0x1000]
    assert store.lookup(C, 0x2000) == O.crypt_page(KEY, 0x2000, C.pid, b"\x02" * 4096)


def test_contract_errors(dkey):
    st = DevicePageStore(8, dkey)
    p = WindowPager(st, lambda c, v: np.zeros((len(v), 4096), np.uint8), 2)
    with pytest.raises(ContractViolation):
        p.fault(C, 0x1000)  # unknown client
    p.register(C)
    p.fault(C, 0x1000)
    with pytest.raises(ContractViolation):
        p.fault(C, 0x1000)  # already resident
    with pytest.raises(ContractViolation):
        p.fault_batch(C, [0x2000, 0x2000])
    with pytest.raises(ContractViolation):
        p.fault(C, 0x2001)
    with pytest.raises(ContractViolation):
        WindowPager(DevicePageStore(8), lambda c, v: None, 2)  # no key
    with pytest.raises(ContractViolation):
        SlidingWindow(0)
