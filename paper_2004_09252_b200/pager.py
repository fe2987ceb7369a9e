"""Batched fault/eviction resolution over the HBM page store.

The reference resolves one fault at a time (``Orchestrator.handle_fault`` /
``evict_page``, ``pkg/src/pagecrypt/orchestrator.py:175-240``): look the page
up in the store, decrypt it (or hand out a zero page on first touch), admit
it into the client's FIFO sliding window (``window.py:31-45``) and, when the
window overflows, pull the oldest resident page back from the client,
encrypt it and store it -- two synchronous single-page crypto calls per
fault.  ``WindowPager`` keeps those semantics and adds ``fault_batch``: all
faults of a batch are resolved with ONE ``refault_many`` (decrypt out of
HBM) and ONE ``evict_many`` (encrypt into HBM), so the GPU sees real batches.
When the evicted pages were all resident before the batch (always, for a
single fault with a full window), refault and eviction are independent and
run as ONE ``DevicePageStore.swap`` -- one GPU round trip per fault.

A batch is equivalent to faulting its pages one by one in order (checked in
``tests/test_gpu_pager.py``): a page evicted by a later fault of the same
batch is stored with the plaintext it was just resolved to, which is what
the client would hand back.

The transport to the client (``transport.py``, ``client.py``) is out of
scope; the caller supplies ``fetch_evicted(client, vaddrs) -> uint8[m, 4096]``,
the data-port pull of ``client.py:251-265``.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

from .errors import ContractViolation
from .store import DevicePageStore

PAGE_SIZE = 4096
_U8 = np.dtype(np.uint8)
FUSED_MAX = 128  # pages per pc_store_swap launch (refaults + evictions)


class SlidingWindow:
    """Bounded FIFO of plaintext-resident vaddrs (window.py:15-67)."""

    MAX_CAPACITY = 4096

    def __init__(self, capacity: int = 16):
        if not 1 <= capacity <= self.MAX_CAPACITY:
            raise ContractViolation(f"window capacity {capacity} outside 1..{self.MAX_CAPACITY}")
        self.capacity = capacity
        self._queue: deque[int] = deque()
        self._members: set[int] = set()

    def admit(self, vaddr: int):
        if vaddr in self._members:
            raise ContractViolation(f"page {vaddr:#x} already in window")
        evicted = None
        if len(self._queue) == self.capacity:
            evicted = self._queue.popleft()
            self._members.discard(evicted)
        self._queue.append(vaddr)
        self._members.add(vaddr)
        return evicted

    def undo_admits(self, admitted: list[int], evicted: list) -> None:
        """Roll back admit() calls, newest first: admitted[i] evicted
        evicted[i] (or None)."""
        for v, e in zip(reversed(admitted), reversed(evicted)):
            self._queue.pop()
            self._members.discard(v)
            if e is not None:
                self._queue.appendleft(e)
                self._members.add(e)

    def remove(self, vaddr: int) -> bool:
        if vaddr not in self._members:
            return False
        self._members.discard(vaddr)
        self._queue.remove(vaddr)
        return True

    def resident(self, vaddr: int) -> bool:
        return vaddr in self._members

    def clear(self) -> None:
        self._queue.clear()
        self._members.clear()

    def __len__(self) -> int:
        return len(self._queue)

    def __iter__(self):
        return iter(list(self._queue))

    def members(self) -> list[int]:
        return list(self._queue)


@dataclass(slots=True)
class PagerMetrics:
    """Per-client counters (orchestrator.py:41-63)."""

    faults: int = 0
    first_touch_faults: int = 0
    evictions: int = 0
    encrypt_ops: int = 0
    decrypt_ops: int = 0
    gpu_batches: int = 0


class WindowPager:
    def __init__(self, store: DevicePageStore, fetch_evicted, window_capacity: int = 16):
        if store.key is None:
            raise ContractViolation("the pager needs a store with a DeviceKey")
        SlidingWindow(window_capacity)  # validate range up front
        self.store = store
        self._native_fault = getattr(store, "fault", None)  # DevicePageStore.fault: one call per fault
        self.fetch_evicted = fetch_evicted
        self.window_capacity = window_capacity
        self._windows: dict[object, SlidingWindow] = {}
        self.metrics: dict[object, PagerMetrics] = {}
        self._state: dict[object, tuple] = {}  # client -> (window, metrics): one lookup per fault

    def register(self, client) -> None:
        if client in self._windows:
            raise ContractViolation(f"client {client} already registered")
        self._windows[client] = SlidingWindow(self.window_capacity)
        self.metrics[client] = PagerMetrics()
        self._state[client] = (self._windows[client], self.metrics[client])

    def unregister(self, client) -> None:
        """Drop all server-side state of a client; its ciphertext is wiped."""
        self._state.pop(client, None)
        if self._windows.pop(client, None) is not None:
            self.store.drop_client(client)

    def window(self, client) -> list[int]:
        return self._window(client).members()

    def _window(self, client) -> SlidingWindow:
        w = self._windows.get(client)
        if w is None:
            raise ContractViolation(f"unknown client {client}")
        return w

    def fault(self, client, vaddr: int) -> bytes:
        """Resolve one fault (handle_fault, orchestrator.py:175-211)."""
        return self._fault_one(client, vaddr)[0].tobytes()

    def fault_batch(self, client, vaddrs) -> np.ndarray:
        """Resolve faults on distinct, non-resident pages, in order; returns
        their plaintexts as uint8[k, 4096]."""
        if len(vaddrs) == 1:
            return self._fault_one(client, vaddrs[0])
        win = self._window(client)
        m = self.metrics[client]
        vlist = [int(v) for v in vaddrs]
        if len(set(vlist)) != len(vlist):
            raise ContractViolation("a batch faults each page once")
        for v in vlist:
            if v % PAGE_SIZE:
                raise ContractViolation(f"vaddr {v:#x} not page-aligned")
            if win.resident(v):
                raise ContractViolation(f"fault on resident page {v:#x}")
        k = len(vlist)
        out = np.zeros((k, PAGE_SIZE), dtype=np.uint8)  # first touch: zero pages
        if not k:
            return out
        many = getattr(self.store, "contains_many", None)
        if many is not None:  # one native lookup for the whole batch
            refault_idx = np.flatnonzero(many(client, vlist)).tolist()
        else:
            refault_idx = [i for i, v in enumerate(vlist) if self.store.contains(client, v)]
        batch_pos = {v: i for i, v in enumerate(vlist)}
        # window admission in fault order (host state only); collect evictions
        # and keep an undo log (admission i evicted undo[i] or None)
        undo: list = []
        evicted: list[int] = []
        for v in vlist:
            e = win.admit(v)
            undo.append(e)
            if e is not None:
                evicted.append(e)
        try:
            if (refault_idx and evicted and len(refault_idx) + len(evicted) <= FUSED_MAX
                    and not any(e in batch_pos for e in evicted)):
                # the common single fault: the evicted pages were resident
                # before the batch, so refault and eviction are independent
                # -> one GPU round trip (pc_store_swap)
                plain_ev = self._from_client(client, evicted)
                out[refault_idx] = self.store.swap(client, [vlist[i] for i in refault_idx], evicted, plain_ev)
                plain_ev.fill(0)  # scratch_evict.wipe(), orchestrator.py:239
                m.gpu_batches += 1
            else:
                # 1. refaults: one decrypt-out-of-HBM batch (entries are removed)
                if refault_idx:
                    out[refault_idx] = self.store.refault_many(client, [vlist[i] for i in refault_idx])
                    m.gpu_batches += 1
                # 2. evictions: pages resident before the batch come back from
                #    the client; pages faulted in by this batch carry their
                #    resolved bytes
                if evicted:
                    from_client = [e for e in evicted if e not in batch_pos]
                    got = self._from_client(client, from_client)
                    row = {e: j for j, e in enumerate(from_client)}
                    plain_ev = np.empty((len(evicted), PAGE_SIZE), dtype=np.uint8)
                    for j, e in enumerate(evicted):
                        plain_ev[j] = out[batch_pos[e]] if e in batch_pos else got[row[e]]
                    self.store.evict_many(client, evicted, plain_ev)
                    plain_ev.fill(0)
                    got.fill(0)
                    m.gpu_batches += 1
        except BaseException:
            win.undo_admits(vlist, undo)
            raise
        m.decrypt_ops += len(refault_idx)
        m.first_touch_faults += k - len(refault_idx)
        m.faults += k
        m.evictions += len(evicted)
        m.encrypt_ops += len(evicted)
        return out

    def _fault_one(self, client, vaddr) -> np.ndarray:
        """fault_batch for one page (the reference's flow): the same steps
        without the batch bookkeeping.  The page it evicts (if any) was
        resident before, so a refault and its eviction are one swap."""
        st = self._state.get(client)
        if st is None:
            raise ContractViolation(f"unknown client {client}")
        win, m = st
        v = int(vaddr)
        if v % PAGE_SIZE:
            raise ContractViolation(f"vaddr {v:#x} not page-aligned")
        if win.resident(v):
            raise ContractViolation(f"fault on resident page {v:#x}")
        if self._native_fault is not None:
            return self._fault_one_native(client, win, m, v, self._native_fault)
        refault = self.store.contains(client, v)
        e = win.admit(v)
        try:
            if refault and e is not None:
                plain_ev = self._from_client(client, [e])
                out = self.store.swap(client, [v], [e], plain_ev)
                plain_ev.fill(0)  # scratch_evict.wipe(), orchestrator.py:239
                m.gpu_batches += 1
            else:
                if refault:
                    out = self.store.refault_many(client, [v])
                    m.gpu_batches += 1
                else:
                    out = np.zeros((1, PAGE_SIZE), dtype=np.uint8)  # first touch
                if e is not None:
                    plain_ev = self._from_client(client, [e])
                    self.store.evict_many(client, [e], plain_ev)
                    plain_ev.fill(0)
                    m.gpu_batches += 1
        except BaseException:
            win.undo_admits([v], [e])
            raise
        m.faults += 1
        if refault:
            m.decrypt_ops += 1
        else:
            m.first_touch_faults += 1
        if e is not None:
            m.evictions += 1
            m.encrypt_ops += 1
        return out

    def _fault_one_native(self, client, win, m, v, native) -> np.ndarray:
        """The single fault as one store call (``DevicePageStore.fault``):
        lookup, refault and the forced eviction in one native call and one
        GPU round trip."""
        e = win.admit(v)
        out = np.empty((1, PAGE_SIZE), dtype=np.uint8)  # filled by a refault, zeroed on a first touch
        try:
            if e is None:
                refault = native(client, v, out, None, None)
            else:
                # no private copy here: the library copies the page into its
                # own staging (the server's scratch_evict) and wipes it there
                # (orchestrator.py:230-239); the client's buffer is only read
                got = self.fetch_evicted(client, [e])
                plain_ev = got if type(got) is np.ndarray else np.asarray(got)
                if plain_ev.dtype is not _U8 or plain_ev.size != PAGE_SIZE or not plain_ev.flags.c_contiguous:
                    plain_ev = np.array(plain_ev, dtype=np.uint8, copy=True, order="C")
                    if plain_ev.size != PAGE_SIZE:
                        raise ContractViolation(f"fetch_evicted returned {plain_ev.size} bytes for one page")
                    try:
                        refault = native(client, v, out, e, plain_ev)
                    finally:
                        plain_ev.fill(0)  # our private copy: scratch_evict.wipe()
                else:
                    refault = native(client, v, out, e, plain_ev)
        except BaseException:
            win.undo_admits([v], [e])
            raise
        if not refault:
            out.fill(0)  # a first touch reads as a zero page (orchestrator.py:178,192)
        if refault or e is not None:
            m.gpu_batches += 1
        m.faults += 1
        if refault:
            m.decrypt_ops += 1
        else:
            m.first_touch_faults += 1
        if e is not None:
            m.evictions += 1
            m.encrypt_ops += 1
        return out

    def _from_client(self, client, vaddrs: list[int]) -> np.ndarray:
        """Pull evicted pages back from the client (client.py:251-265)."""
        if not vaddrs:
            return np.empty((0, PAGE_SIZE), dtype=np.uint8)
        # a private copy (the server's scratch_evict, orchestrator.py:230-239):
        # it is wiped after use, the caller's buffer is not touched
        got = np.array(self.fetch_evicted(client, vaddrs), dtype=np.uint8, copy=True, order="C")
        return got.reshape(len(vaddrs), PAGE_SIZE)
