"""HBM-resident encrypted page store.

``pagecrypt.store.EncryptedPageStore`` (``pkg/src/pagecrypt/store.py:41-105``)
keeps one ciphertext copy per (client, vaddr) in host RAM under a
client -> SortedDict index.  Here the pages live in a device slab
(``capacity_pages`` x 4 KiB of HBM; 180 GB holds ~44M pages) and the index
is native (``pc_store_*``, ``csrc/store.inc``), so batched calls spend their
time on PCIe, not on per-page bookkeeping.

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
  pipelined transfer per batch;
* ``swap(client, refault_vaddrs, evict_vaddrs, evict_plains)``: a whole
  fault (refault + eviction) in one GPU round trip (``pc_store_swap``).

Only ``client.pid`` enters the cipher seed, as in the reference worker
(``workers.py:137``); the index is keyed by (pid, epoch).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .engine import DeviceKey, Engine, _addr, _fastmod, _host_vaddrs, default_engine
from .errors import ContractViolation, PageCryptError

PAGE_SIZE = 4096


class StoreFull(PageCryptError):
    """No free slot left in the device slab."""


def _p(arr: np.ndarray):
    """Address of an array for the C ABI (None when empty)."""
    return _addr(arr) if arr.size else None


def _cid(client) -> int:
    return ((int(client.pid) & 0xFFFFFFFF) << 32) | (int(getattr(client, "epoch", 0)) & 0xFFFFFFFF)


class DevicePageStore:
    def __init__(self, capacity_pages: int, key: DeviceKey | None = None, *, device: int = 0,
                 rounds: int = 20, engine: Engine | None = None):
        if key is not None and key.device != device:
            raise ContractViolation(f"key on device {key.device}, store on {device}")
        self.device = device
        self.key = key
        self.rounds = rounds
        self.capacity = capacity_pages
        self._engine = engine or default_engine(device)
        self._lib = _native.load()
        h = ctypes.c_void_p()
        _native.call("pc_store_create", self._engine.handle, None if key is None else key.handle,
                     capacity_pages, rounds, ctypes.byref(h))
        self._h = h.value
        self._clients = {}  # cid -> client object (for iteration helpers)

    def _call(self, name, *args):
        rc = getattr(self._lib, name)(*args)
        if rc:
            self._raise(rc)

    def _raise(self, rc: int):
        if rc == _native.PC_EFULL:
            raise StoreFull(self._lib.pc_last_error().decode())
        _native.check(rc)

    def start_service(self, n_workers: int = 1) -> None:
        """Serve single faults (``fault``) from a resident GPU worker started
        with the store's key (``pc_store_service``): one service ticket per
        fault instead of a kernel launch and a stream sync.  Batched calls
        keep their launches.  ``close`` stops it."""
        if n_workers < 1:
            raise ContractViolation(f"n_workers must be >= 1, got {n_workers}")
        self._need_key()
        _native.call("pc_store_service", self._h, n_workers)
        self._service = True

    def stop_service(self) -> None:
        if self._h is not None and getattr(self, "_service", False):
            _native.call("pc_store_service", self._h, 0)
        self._service = False

    @property
    def service_running(self) -> bool:
        return getattr(self, "_service", False)

    def close(self) -> None:
        """Wipe the slab and free it."""
        self._service = False  # pc_store_destroy stops it
        if self._h is not None:
            h, self._h = self._h, None
            _native.call("pc_store_destroy", h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def free_slots(self) -> int:
        n = ctypes.c_size_t()
        _native.call("pc_store_free_slots", self._h, ctypes.byref(n))
        return n.value

    @staticmethod
    def _page(buf) -> np.ndarray:
        arr = np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf.reshape(-1)
        if arr.size != PAGE_SIZE:
            raise ContractViolation(f"page must be {PAGE_SIZE} bytes")
        return np.ascontiguousarray(arr, dtype=np.uint8)

    @staticmethod
    def _vaddrs(vaddrs) -> np.ndarray:
        v = vaddrs if isinstance(vaddrs, (list, tuple)) else np.asarray(vaddrs)
        arr, _ = _host_vaddrs(v, len(v))
        return arr

    # -- reference API (store.py:53-105) --------------------------------------

    def insert(self, client, vaddr: int, cipher) -> None:
        """Store a private copy of a ciphertext page.  Double insert is a bug."""
        va = self._vaddrs([vaddr])
        arr = self._page(cipher)
        self._call("pc_store_put", self._h, _cid(client), client.pid, _p(va), 1, _p(arr), 0)

    def lookup(self, client, vaddr: int):
        """Ciphertext bytes if present, else None (a first touch)."""
        if not self.contains(client, vaddr):
            return None
        out = np.empty(PAGE_SIZE, dtype=np.uint8)
        va = self._vaddrs([vaddr])
        self._call("pc_store_get", self._h, _cid(client), client.pid, _p(va), 1, _p(out), 0, 0)
        return out.tobytes()

    def remove(self, client, vaddr: int) -> None:
        """Delete an entry; the released slot is wiped before reuse."""
        va = self._vaddrs([vaddr])
        self._call("pc_store_remove", self._h, _cid(client), _p(va), 1)

    def contains(self, client, vaddr: int) -> bool:
        v = int(vaddr)
        if not 0 <= v < 2**64 or v % PAGE_SIZE:
            return False  # never stored (insert rejects it); a negative vaddr must not wrap onto a stored one
        f = ctypes.c_int()
        _native.call("pc_store_contains", self._h, _cid(client), v, ctypes.byref(f))
        return bool(f.value)

    def contains_many(self, client, vaddrs) -> np.ndarray:
        """contains() for a batch, in one native call: bool[n]."""
        va = self._vaddrs(vaddrs)
        found = np.zeros(va.size, dtype=np.uint8)
        if va.size:
            _native.call("pc_store_contains_many", self._h, _cid(client), _p(va), va.size, _p(found))
        return found.astype(bool)

    def drop_client(self, client) -> None:
        """Remove and wipe every entry of a client.  Unknown client: no-op."""
        _native.call("pc_store_drop_client", self._h, _cid(client))

    def _list(self, client) -> np.ndarray:
        n = ctypes.c_size_t()
        _native.call("pc_store_list", self._h, _cid(client), None, 0, ctypes.byref(n))
        out = np.empty(n.value, dtype=np.uint64)
        if n.value:
            _native.call("pc_store_list", self._h, _cid(client), _p(out), out.size, ctypes.byref(n))
        return out

    def pages(self, client):
        """(vaddr, ciphertext) in strictly increasing vaddr order."""
        va = self._list(client)
        if not va.size:
            return
        out = np.empty((va.size, PAGE_SIZE), dtype=np.uint8)
        self._call("pc_store_get", self._h, _cid(client), client.pid, _p(va), va.size,
                   _p(out), 0, 0)
        for v, row in zip(va.tolist(), out):
            yield v, row.tobytes()

    def page_count(self, client) -> int:
        n = ctypes.c_size_t()
        _native.call("pc_store_list", self._h, _cid(client), None, 0, ctypes.byref(n))
        return n.value

    # -- fused cipher paths ----------------------------------------------------

    def _need_key(self):
        if self.key is None:
            raise PageCryptError("this store has no DeviceKey: use insert/lookup for ciphertext")

    def evict(self, client, vaddr: int, plain) -> None:
        """Encrypt a plaintext page into a new HBM entry."""
        self.evict_many(client, [vaddr], self._page(plain).reshape(1, PAGE_SIZE))

    def refault(self, client, vaddr: int) -> bytes:
        """Decrypt an entry out of HBM and remove it (a refault)."""
        return self.refault_many(client, [vaddr])[0].tobytes()

    def evict_many(self, client, vaddrs, plains) -> None:
        self._need_key()
        va = self._vaddrs(vaddrs)
        arr = plains if isinstance(plains, np.ndarray) else np.asarray(plains)
        arr = np.ascontiguousarray(arr, dtype=np.uint8).reshape(-1, PAGE_SIZE)
        if arr.shape[0] != va.size:
            raise ContractViolation(f"{va.size} vaddrs for {arr.shape[0]} pages")
        self._call("pc_store_put", self._h, _cid(client), client.pid, _p(va), va.size,
                   _p(arr), 1)

    def refault_many(self, client, vaddrs, out: np.ndarray | None = None) -> np.ndarray:
        self._need_key()
        va = self._vaddrs(vaddrs)
        if out is None:
            out = np.empty((va.size, PAGE_SIZE), dtype=np.uint8)
        elif out.nbytes != va.size * PAGE_SIZE or not out.flags.c_contiguous or not out.flags.writeable:
            raise ContractViolation("out must be a writable C-contiguous uint8[n, 4096] buffer")
        self._call("pc_store_get", self._h, _cid(client), client.pid, _p(va), va.size,
                   _p(out), 1, 1)
        return out

    def swap(self, client, refault_vaddrs, evict_vaddrs, evict_plains, out: np.ndarray | None = None) -> np.ndarray:
        """Refault ``refault_vaddrs`` (decrypt out of HBM, remove) and evict
        ``evict_plains`` to ``evict_vaddrs`` (encrypt into HBM) -- one fault of
        the orchestrator (``orchestrator.py:175-240``) -- in one GPU round trip
        for up to 128 pages in total.  Same result as ``refault_many`` then
        ``evict_many``.  Returns the refaulted plaintexts."""
        self._need_key()
        gv = self._vaddrs(refault_vaddrs)
        pv = self._vaddrs(evict_vaddrs)
        arr = evict_plains if isinstance(evict_plains, np.ndarray) else np.asarray(evict_plains)
        arr = np.ascontiguousarray(arr, dtype=np.uint8).reshape(-1, PAGE_SIZE)
        if arr.shape[0] != pv.size:
            raise ContractViolation(f"{pv.size} vaddrs for {arr.shape[0]} pages")
        if out is None:
            out = np.empty((gv.size, PAGE_SIZE), dtype=np.uint8)
        elif out.nbytes != gv.size * PAGE_SIZE or not out.flags.c_contiguous or not out.flags.writeable:
            raise ContractViolation("out must be a writable C-contiguous uint8[n, 4096] buffer")
        self._call("pc_store_swap", self._h, _cid(client), client.pid, _p(gv), gv.size,
                   _p(out), _p(pv), pv.size, _p(arr))
        return out

    def fault(self, client, vaddr: int, out: np.ndarray, evict_vaddr: int | None = None, evict_plain=None) -> bool:
        """One orchestrator fault (``orchestrator.py:175-240``) in one call:
        refault ``vaddr`` into ``out`` (uint8[4096]) if it is stored and return
        True, else leave ``out`` untouched (a first touch) and return False;
        evict ``evict_plain`` to ``evict_vaddr`` if given.  Refault and
        eviction share one GPU round trip."""
        self._need_key()
        if vaddr % PAGE_SIZE or not 0 <= vaddr < 2**64:
            raise ContractViolation(f"vaddr {vaddr:#x} not a page-aligned u64")
        fm = _fastmod()
        if fm and self._h is not None:
            # METH_FASTCALL into pc_store_fault (csrc/fastpath.c): the buffer
            # checks run in C; anything unusual comes back as None and takes
            # the general path below, which reports it
            r = fm.store_fault_buf(self._h, _cid(client), client.pid, vaddr, out,
                                   0 if evict_plain is None else evict_vaddr, evict_plain)
            if r is not None:
                if r[0]:
                    self._raise(r[0])
                return bool(r[1])
        if out.nbytes != PAGE_SIZE or not out.flags.c_contiguous or not out.flags.writeable:
            raise ContractViolation("out must be a writable C-contiguous 4096-byte array")
        ev = None
        if evict_plain is not None:
            if evict_vaddr is None or evict_vaddr % PAGE_SIZE or not 0 <= evict_vaddr < 2**64:
                raise ContractViolation("evict_vaddr must be a page-aligned u64")
            ev = evict_plain if isinstance(evict_plain, np.ndarray) else np.frombuffer(evict_plain, np.uint8)
            if ev.nbytes != PAGE_SIZE or not ev.flags.c_contiguous:
                raise ContractViolation("evict_plain must be 4096 contiguous bytes")
        flag = ctypes.c_int()
        self._call("pc_store_fault", self._h, _cid(client), client.pid, vaddr, _addr(out),
                   evict_vaddr or 0, None if ev is None else ev.ctypes.data, ctypes.byref(flag))
        return bool(flag.value)
