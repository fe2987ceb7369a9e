"""HBM-resident encrypted page store.

``pagecrypt.store.EncryptedPageStore`` (``pkg/src/pagecrypt/store.py:41-105``)
keeps one ciphertext copy per (client, vaddr) in host RAM.  Here the pages
live in a device slab (``capacity_pages`` x 4 KiB of HBM; 180 GB holds ~44M
pages) and only the index (client -> vaddr -> slot) is on the host.

Same API and errors as the reference store (``insert``/``lookup``/``remove``/
``contains``/``drop_client``/``pages``/``page_count``; ContractViolation for
unaligned vaddrs, wrong sizes, duplicate inserts and missing entries; freed
slots are wiped), plus the fused paths the B200 makes possible:

* ``evict(client, vaddr, plain)``: the plaintext page crosses PCIe once and
  is encrypted on the way into its HBM slot (the orchestrator's
  encrypt-then-insert, ``orchestrator.py:234-238``, in one step);
* ``refault(client, vaddr)``: the ciphertext is decrypted on the way out of
  HBM and the entry removed (``orchestrator.py:190-198``);
* ``evict_many`` / ``refault_many``: the same for whole batches, one
  pipelined transfer per batch.

Only ``client.pid`` enters the cipher seed, as in the reference worker
(``workers.py:137``).
"""

from __future__ import annotations

from collections import deque

import numpy as np

from . import _native
from .engine import DeviceKey, Engine, _check_vaddr_int, _host_vaddrs, default_engine
from .errors import ContractViolation, PageCryptError

PAGE_SIZE = 4096


class StoreFull(PageCryptError):
    """No free slot left in the device slab."""


class DevicePageStore:
    def __init__(self, capacity_pages: int, key: DeviceKey | None = None, *, device: int = 0,
                 rounds: int = 20, engine: Engine | None = None):
        import torch

        if capacity_pages < 1 or capacity_pages >= 2**32:
            raise ContractViolation("capacity_pages must be in 1..2^32-1")
        if key is not None and key.device != device:
            raise ContractViolation(f"key on device {key.device}, store on {device}")
        self.device = device
        self.key = key
        self.rounds = rounds
        self.capacity = capacity_pages
        self._engine = engine or default_engine(device)
        self._slab = torch.zeros((capacity_pages, PAGE_SIZE), dtype=torch.uint8, device=f"cuda:{device}")
        torch.cuda.synchronize(device)
        # free-slot stack: _free_arr[:_nfree] are free (top = lowest slots first)
        self._free_arr = np.arange(capacity_pages - 1, -1, -1, dtype=np.uint32)
        self._nfree = capacity_pages
        self._clients: dict[object, dict[int, int]] = {}

    # -- bookkeeping -------------------------------------------------------

    @property
    def free_slots(self) -> int:
        return self._nfree

    def _take(self, n: int) -> np.ndarray:
        if n > self._nfree:
            raise StoreFull(f"need {n} slots, {self._nfree} free of {self.capacity}")
        self._nfree -= n
        return self._free_arr[self._nfree:self._nfree + n][::-1].copy()

    def _release(self, slots) -> None:
        sl = np.asarray(slots, dtype=np.uint32)
        self._free_arr[self._nfree:self._nfree + sl.size] = sl
        self._nfree += sl.size

    def _move(self, slots, host: np.ndarray, direction: int, vaddrs=None, pid: int = 0, cipher: bool = False,
              wipe_src: bool = False):
        sl = np.ascontiguousarray(slots, dtype=np.uint32)
        va = None
        if cipher:
            if self.key is None:
                raise PageCryptError("this store has no DeviceKey: use insert/lookup for ciphertext")
            va, _ = _host_vaddrs(np.asarray(vaddrs, dtype=np.uint64), sl.size)
        _native.call("pc_slab_transfer", self._engine.handle, self.key.handle if cipher else None,
                     self._slab.data_ptr(), self.capacity, sl.ctypes.data,
                     None if va is None else va.ctypes.data, None, 0, pid & 0xFFFFFFFF,
                     host.ctypes.data, sl.size, direction, self.rounds, 1 if wipe_src else 0)

    def _wipe(self, slots) -> None:
        sl = np.ascontiguousarray(slots, dtype=np.uint32)
        _native.call("pc_slab_wipe", self._engine.handle, self._slab.data_ptr(), self.capacity,
                     sl.ctypes.data, sl.size)

    @staticmethod
    def _page(buf) -> np.ndarray:
        arr = np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf.reshape(-1)
        if arr.size != PAGE_SIZE:
            raise ContractViolation(f"page must be {PAGE_SIZE} bytes")
        return np.ascontiguousarray(arr, dtype=np.uint8)

    # -- reference API (store.py:53-105) --------------------------------------

    def insert(self, client, vaddr: int, cipher) -> None:
        """Store a private copy of a ciphertext page.  Double insert is a bug."""
        if vaddr % PAGE_SIZE:
            raise ContractViolation(f"vaddr {vaddr:#x} not page-aligned")
        arr = self._page(cipher)
        sub = self._clients.setdefault(client, {})
        if vaddr in sub:
            raise ContractViolation(f"duplicate store insert for {client} {vaddr:#x}")
        slot = self._take(1)
        try:
            self._move(slot, arr, 0)
        except Exception:
            self._release(slot)
            raise
        sub[vaddr] = int(slot[0])

    def lookup(self, client, vaddr: int):
        """Ciphertext bytes if present, else None (a first touch)."""
        slot = self._clients.get(client, {}).get(vaddr)
        if slot is None:
            return None
        out = np.empty(PAGE_SIZE, dtype=np.uint8)
        self._move([slot], out, 1)
        return out.tobytes()

    def remove(self, client, vaddr: int) -> None:
        """Delete an entry; the released slot is wiped before reuse."""
        sub = self._clients.get(client)
        if sub is None or vaddr not in sub:
            raise ContractViolation(f"no store entry for {client} {vaddr:#x}")
        slot = sub.pop(vaddr)
        self._wipe([slot])
        self._release([slot])

    def contains(self, client, vaddr: int) -> bool:
        return vaddr in self._clients.get(client, {})

    def drop_client(self, client) -> None:
        """Remove and wipe every entry of a client.  Unknown client: no-op."""
        sub = self._clients.pop(client, None)
        if not sub:
            return
        slots = np.fromiter(sub.values(), dtype=np.uint32, count=len(sub))
        self._wipe(slots)
        self._release(slots)

    def pages(self, client):
        """(vaddr, ciphertext) in strictly increasing vaddr order."""
        sub = self._clients.get(client)
        if not sub:
            return
        vaddrs = sorted(sub)
        out = np.empty((len(vaddrs), PAGE_SIZE), dtype=np.uint8)
        self._move([sub[v] for v in vaddrs], out, 1)
        for v, row in zip(vaddrs, out):
            yield v, row.tobytes()

    def page_count(self, client) -> int:
        return len(self._clients.get(client, {}))

    # -- fused cipher paths ----------------------------------------------------

    def evict(self, client, vaddr: int, plain) -> None:
        """Encrypt a plaintext page into a new HBM entry."""
        self.evict_many(client, [vaddr], self._page(plain).reshape(1, PAGE_SIZE))

    def refault(self, client, vaddr: int) -> bytes:
        """Decrypt an entry out of HBM and remove it (a refault)."""
        return self.refault_many(client, [vaddr])[0].tobytes()

    def evict_many(self, client, vaddrs, plains) -> None:
        va, _ = _host_vaddrs(np.asarray(vaddrs) if not isinstance(vaddrs, (list, tuple)) else vaddrs,
                             len(vaddrs))
        arr = np.ascontiguousarray(plains, dtype=np.uint8).reshape(-1, PAGE_SIZE)
        if arr.shape[0] != va.size:
            raise ContractViolation(f"{va.size} vaddrs for {arr.shape[0]} pages")
        vlist = va.tolist()
        vset = set(vlist)
        sub = self._clients.setdefault(client, {})
        if len(vset) != len(vlist) or not vset.isdisjoint(sub.keys()):
            raise ContractViolation("duplicate store insert")
        slots = self._take(len(vlist))
        try:
            self._move(slots, arr, 0, vaddrs=va, pid=client.pid, cipher=True)
        except Exception:
            self._release(slots)
            raise
        sub.update(zip(vlist, slots.tolist()))

    def refault_many(self, client, vaddrs, out: np.ndarray | None = None) -> np.ndarray:
        va, _ = _host_vaddrs(np.asarray(vaddrs) if not isinstance(vaddrs, (list, tuple)) else vaddrs,
                             len(vaddrs))
        vlist = va.tolist()
        sub = self._clients.get(client, {})
        if len(set(vlist)) != len(vlist):
            raise ContractViolation("duplicate vaddr in refault batch")
        try:
            slots = np.fromiter(map(sub.__getitem__, vlist), dtype=np.uint32, count=len(vlist))
        except KeyError as exc:
            raise ContractViolation(f"no store entry for {client} {exc.args[0]:#x}") from None
        if out is None:
            out = np.empty((len(vlist), PAGE_SIZE), dtype=np.uint8)
        elif out.nbytes != len(vlist) * PAGE_SIZE or not out.flags.c_contiguous:
            raise ContractViolation("out must be a C-contiguous uint8[n, 4096] buffer")
        # decrypt on the way out and zero each slot as it is read (freed)
        self._move(slots, out, 1, vaddrs=va, pid=client.pid, cipher=True, wipe_src=True)
        deque(map(sub.pop, vlist), maxlen=0)
        self._release(slots)
        return out
