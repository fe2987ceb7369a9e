"""WindowPager against the REFERENCE orchestrator's own traces.

``tests/golden/make_orchestrator_golden.py`` drove the unmodified reference
stack (``Orchestrator`` + ``ClientSpace`` + real-crypto ``WorkerPool``,
pkg/src/pagecrypt/orchestrator.py:171-240) through seeded read/write
sequences at window capacities 1, 4 and 8 and recorded every read, the
client's stored ciphertexts, the FIFO window and the counters.  Here the same
accesses replay through ``WindowPager`` -- over an oracle-cipher store on the
CPU, and over the HBM ``DevicePageStore`` on the GPU -- and must reproduce all
of it byte for byte.
"""

import os

import numpy as np
import pytest

from oracle import chacha_oracle as O
from paper_2004_09252_b200.pager import WindowPager
from paper_2004_09252_b200.workers import ClientId

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "orchestrator_traces.npz")


@pytest.fixture(scope="module")
def traces():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


class OracleStore:
    """The pager-facing store API over a dict, ciphered by the oracle."""

    def __init__(self, key: bytes):
        self.key = key
        self.ct = {}

    def contains(self, client, v):
        return (client, v) in self.ct

    def _crypt(self, client, v, page):
        return np.frombuffer(O.crypt_page(self.key, v, client.pid, bytes(page)), np.uint8)

    def refault_many(self, client, vaddrs):
        return np.stack([self._crypt(client, v, self.ct.pop((client, v))) for v in vaddrs])

    def evict_many(self, client, vaddrs, plains):
        for v, p in zip(vaddrs, plains):
            assert (client, v) not in self.ct
            self.ct[(client, v)] = self._crypt(client, v, p).tobytes()

    def swap(self, client, get, put, plains):
        out = self.refault_many(client, get)
        self.evict_many(client, put, plains)
        return out

    def pages(self, client):
        return sorted((v, c) for (cl, v), c in self.ct.items() if cl == client)

    def drop_client(self, client):
        pass


def replay(z, i, store):
    """The reference client's accesses, demand-paged through WindowPager."""
    pid, base = int(z["pid"]), int(z["base"])
    client = ClientId(pid, 0)
    mem = {}

    def fetch(c, vaddrs):  # the client hands evicted pages back (client.py:251-265)
        return np.stack([np.frombuffer(bytes(mem.pop(v)), np.uint8) for v in vaddrs])

    pager = WindowPager(store, fetch, window_capacity=int(z[f"t{i}_window"]))
    pager.register(client)
    reads = []
    for w, off, n, data in zip(z[f"t{i}_is_write"], z[f"t{i}_offset"], z[f"t{i}_length"], z[f"t{i}_data"]):
        off, n = int(off), int(n)
        v = base + (off // 4096) * 4096
        if v not in mem:
            mem[v] = bytearray(pager.fault(client, v))
        o = off % 4096
        if w:
            mem[v][o:o + n] = bytes(data[:n])
        else:
            reads.append(bytes(mem[v][o:o + n]).ljust(8, b"\0"))
    return pager, client, reads


def check(z, i, pager, client, reads, stored):
    assert np.array_equal(np.frombuffer(b"".join(reads), np.uint8).reshape(-1, 8), z[f"t{i}_reads"])
    assert [v for v, _ in stored] == [int(v) for v in z[f"t{i}_store_vaddrs"]]
    for (v, ct), want in zip(stored, z[f"t{i}_store_cts"]):
        assert bytes(ct) == want.tobytes(), hex(v)
    assert pager.window(client) == [int(v) for v in z[f"t{i}_window_fifo"]]
    m = pager.metrics[client]
    assert [m.faults, m.first_touch_faults, m.evictions, m.encrypt_ops, m.decrypt_ops] == \
        [int(x) for x in z[f"t{i}_metrics"]]


@pytest.mark.parametrize("i", [0, 1, 2])
def test_pager_reproduces_reference_orchestrator_on_cpu(traces, i):
    store = OracleStore(traces["key"].tobytes())
    pager, client, reads = replay(traces, i, store)
    check(traces, i, pager, client, reads, store.pages(client))


@pytest.mark.gpu
@pytest.mark.parametrize("service", [False, True], ids=["launch", "service"])
@pytest.mark.parametrize("i", [0, 1, 2])
def test_pager_over_hbm_store_reproduces_reference_orchestrator(traces, i, cuda, service):
    import paper_2004_09252_b200 as pc
    from paper_2004_09252_b200.store import DevicePageStore

    key = pc.DeviceKey.install(traces["key"].tobytes(), 0)
    try:
        store = DevicePageStore(64, key)
        if service:  # every single fault through the store's resident worker
            store.start_service()
        pager, client, reads = replay(traces, i, store)
        check(traces, i, pager, client, reads, list(store.pages(client)))
        store.close()
    finally:
        key.destroy()
