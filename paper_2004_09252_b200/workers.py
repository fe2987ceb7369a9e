"""GPU crypto-worker service: drop-in for ``pagecrypt.workers.WorkerPool``.

The reference emulates MemShield's GPU service with Python threads
(``pkg/src/pagecrypt/workers.py:28-254``): N workers, each with a bounded
MPSC ring (``WorkerRing``), a private 32-byte key slot, client-affine routing
and a ``Completion`` per request.  This is the real thing on the B200
(``include/pagecrypt.h`` section vii, ``csrc/service.cuh``): one persistent
kernel whose 64-thread CTAs are the workers, rings in mapped pinned host
memory, and the key held only in the workers' registers -- the device copy
used to start the kernel is destroyed as soon as every worker has loaded it
(PAPER.md:592-594,624-637).

Same constructor, methods, routing and errors as the reference
(``PoolError`` for lifecycle misuse, ``ContractViolation`` for bad
arguments, worker-side cipher errors re-raised by ``Completion.wait``).  The
page (``page.data`` of a RamBuf, or any writable buffer) is transformed in
place, as the reference worker does (``workers.py:136-138``); the result is
delivered by whichever host thread first observes the GPU's completion (a
waiter, a poller, or a producer that needs the ring slot), so a full ring
never deadlocks and un-waited requests still complete.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .engine import DeviceKey, _check_pid_int, _check_vaddr_int, _fastmod
from .errors import ContractViolation, PageCryptError, PoolError

PAGE_SIZE = 4096
KEY_SIZE = 32
DEFAULT_RING_SLOTS = 64  # workers.py:25
_Page = ctypes.c_char * PAGE_SIZE


@dataclass(frozen=True)
class ClientId:
    """Client identity (pid, epoch), as ``pagecrypt.store.ClientId``
    (pkg/src/pagecrypt/store.py:19-38).  Any object with ``pid``/``epoch``
    works with the pool; only ``pid`` enters the cipher seed
    (workers.py:137)."""

    pid: int
    epoch: int

    def __post_init__(self):
        if not 0 <= self.pid < 2**32:
            raise ContractViolation(f"pid {self.pid} not a u32")
        if not 0 <= self.epoch < 2**32:
            raise ContractViolation(f"epoch {self.epoch} not a u32")
        # the fault path looks clients up in dicts on every fault: hash once
        object.__setattr__(self, "_hash", hash((self.pid, self.epoch)))

    def __hash__(self):
        return self._hash


def _page_view(page) -> np.ndarray:
    data = getattr(page, "data", page)  # RamBuf-like (ram.py:44-66) or a raw buffer
    arr = np.frombuffer(data, dtype=np.uint8)
    return arr


class Completion:
    """Signaling slot for one request (workers.py:28-52)."""

    __slots__ = ("_pool", "_worker", "_ticket", "error", "_done")

    def __init__(self, pool=None, worker=0, ticket=0, error=None):
        self._pool, self._worker, self._ticket = pool, worker, ticket
        self.error = error
        self._done = pool is None

    def signal(self, error=None) -> None:
        """Mark the request finished, optionally with an error that ``wait``
        re-raises (workers.py:38-42).  The GPU service completes requests by
        itself; signalling a request it still holds first waits for the GPU to
        let go of the page, so no result can land in a released buffer."""
        if not self._done:
            rc = self._pool._lib.pc_service_wait(self._pool._svc, self._worker, self._ticket, -1)
            _native.check(rc)
            self._done = True
            self._pool._pending.pop((self._worker, self._ticket), None)
        self.error = error

    def wait(self, timeout: float | None = None) -> None:
        if not self._done:
            us = -1 if timeout is None else int(timeout * 1e6)
            rc = self._pool._lib.pc_service_wait(self._pool._svc, self._worker, self._ticket, us)
            if rc == _native.PC_ETIMEOUT:
                raise PoolError("timed out waiting for crypto completion")
            _native.check(rc)
            self._done = True
            self._pool._pending.pop((self._worker, self._ticket), None)
        if self.error is not None:
            raise self.error

    @property
    def done(self) -> bool:
        if not self._done:
            flag = ctypes.c_int(0)
            _native.check(self._pool._lib.pc_service_poll(self._pool._svc, self._worker, self._ticket,
                                                          ctypes.byref(flag)))
            if flag.value:
                self._done = True
                self._pool._pending.pop((self._worker, self._ticket), None)
        return self._done


class WorkerPool:
    """N GPU service workers with client-affine routing (workers.py:145-254)."""

    def __init__(self, n_workers: int | None = None, keysource=os.urandom, ram=None,
                 ring_capacity: int = DEFAULT_RING_SLOTS, debug_leak_key: bool = False,
                 *, device: int = 0, rounds: int = 20):
        self._lib = _native.load()
        if n_workers is None:
            # the reference's default (workers.py:156-157), so route() assigns
            # clients exactly as it does; capped by the co-resident CTAs.  Fewer
            # workers also poll fewer doorbells: 8.7 us per 1-page request at 8
            # workers vs 9.8 at 148 (profiles/r01_service_dispatch_ab.txt)
            n = ctypes.c_int()
            _native.call("pc_service_max_workers", device, ctypes.byref(n))
            n_workers = max(1, min(os.cpu_count() or 1, n.value))
        if n_workers < 1:
            raise ContractViolation(f"n_workers must be >= 1, got {n_workers}")
        if ring_capacity < 1 or ring_capacity & (ring_capacity - 1):
            raise ContractViolation(f"ring capacity {ring_capacity} not a power of two")
        self.ram = ram
        self.n_workers = n_workers
        self.device = device
        self.rounds = rounds
        self.ring_capacity = ring_capacity
        self._svc = None
        self._pending = {}  # (worker, ticket) -> page array, alive until delivered
        self._keyed = False
        self._shut_down = False
        self.install_key(keysource, debug_leak_key=debug_leak_key)

    def install_key(self, keysource, debug_leak_key: bool = False) -> None:
        """Stage the master key, start the workers with it, wipe every copy
        outside the workers' registers (workers.py:174-202)."""
        if self._keyed:
            raise PoolError("pool already initialized with a key")
        if self._shut_down:
            raise PoolError("pool is shut down")
        try:
            material = keysource(KEY_SIZE)
        except Exception as exc:
            raise PoolError(f"keysource failed: {exc}") from exc
        if len(material) != KEY_SIZE:
            raise PoolError(f"keysource yielded {len(material)} bytes, need {KEY_SIZE}")
        staging = bytearray(material)
        if isinstance(material, bytearray):
            material[:] = bytes(KEY_SIZE)  # a writable keysource buffer is purged too
        if debug_leak_key and self.ram is not None:
            # positive control for the cold-boot key scanner (workers.py:196-200)
            from_ram = getattr(self.ram, "alloc", None)
            if from_ram is not None:
                leak = self.ram.alloc("server_misc", KEY_SIZE)  # TAG_SERVER_MISC (ram.py:29)
                leak.data[:] = staging
        dkey = DeviceKey.install(staging, self.device)
        staging[:] = bytes(KEY_SIZE)
        try:
            h = ctypes.c_void_p()
            _native.call("pc_service_start", dkey.handle, self.n_workers, self.ring_capacity,
                         self.rounds, ctypes.byref(h))
            self._svc = h.value
        finally:
            dkey.destroy()  # the key now lives only in the workers' registers
        self._keyed = True

    def route(self, client) -> int:
        """Stable client -> worker assignment (workers.py:204-206)."""
        return ((client.pid * 2654435761) ^ client.epoch) % self.n_workers

    def submit(self, client, vaddr: int, direction: str, page) -> Completion:
        if self._shut_down:
            raise PoolError("submit on a shut-down pool")
        if direction not in ("encrypt", "decrypt"):
            raise ContractViolation(f"bad direction {direction!r}")
        arr = _page_view(page)
        if arr.size != PAGE_SIZE:
            raise ContractViolation("crypto requests operate on whole pages")
        try:  # the reference worker raises these from crypt_page (cipher.py:205-210)
            _check_vaddr_int(vaddr)
            _check_pid_int(client.pid)
        except ContractViolation as exc:
            return Completion(error=exc)
        if not arr.flags.writeable:
            raise ContractViolation("page buffer must be writable (it is transformed in place)")
        w = self.route(client)
        t = ctypes.c_uint64()
        _native.call("pc_service_submit", self._svc, w, vaddr, client.pid, arr.ctypes.data,
                     arr.ctypes.data, ctypes.byref(t))
        self._pending[(w, t.value)] = arr
        if len(self._pending) > 4 * self.ring_capacity * self.n_workers:
            self._prune()
        return Completion(self, w, t.value)

    def _prune(self) -> None:
        """Drop buffers of delivered requests nobody waited for."""
        flag = ctypes.c_int(0)
        for (w, t) in list(self._pending):
            _native.check(self._lib.pc_service_poll(self._svc, w, t, ctypes.byref(flag)))
            if flag.value:
                self._pending.pop((w, t), None)

    def crypt(self, client, vaddr: int, direction: str, page) -> None:
        """Submit and wait: the synchronous fault-path helper (workers.py:227-229).
        Same checks and errors as ``submit(...).wait()``, in ONE native call
        (pc_service_crypt) with no per-request bookkeeping: the page is
        transformed in place before this returns."""
        if self._shut_down:
            raise PoolError("submit on a shut-down pool")
        if direction not in ("encrypt", "decrypt"):
            raise ContractViolation(f"bad direction {direction!r}")
        data = getattr(page, "data", page)
        fm = _fastmod()
        if fm and 0 <= vaddr < 2**64 and not vaddr & 4095 and 0 <= client.pid < 2**32:
            rc = fm.service_crypt_buf(self._svc, self.route(client), vaddr, client.pid, data, -1)
            if rc == 0:
                return
            if rc > 0:
                if rc == _native.PC_ETIMEOUT:
                    raise PoolError("timed out waiting for crypto completion")
                _native.check(rc)
            # rc < 0: not a writable 4 KiB buffer -- the general path below reports it
        if type(data) is bytearray and len(data) == PAGE_SIZE:
            arr = _Page.from_buffer(data)  # cheapest way to its address (~1 us)
            ptr = arr
        else:
            arr = _page_view(page)
            if arr.size != PAGE_SIZE:
                raise ContractViolation("crypto requests operate on whole pages")
            if not arr.flags.writeable:
                raise ContractViolation("page buffer must be writable (it is transformed in place)")
            ptr = arr.ctypes.data
        _check_vaddr_int(vaddr)
        _check_pid_int(client.pid)
        rc = self._lib.pc_service_crypt(self._svc, self.route(client), vaddr, client.pid, ptr, ptr, -1)
        if rc != _native.PC_OK:
            if rc == _native.PC_ETIMEOUT:
                raise PoolError("timed out waiting for crypto completion")
            _native.check(rc)

    @property
    def in_flight(self) -> int:
        if self._svc is None:
            return 0
        n = ctypes.c_uint64()
        _native.call("pc_service_in_flight", self._svc, ctypes.byref(n))
        return n.value

    @property
    def running(self) -> bool:
        return self._keyed and not self._shut_down

    def shutdown(self) -> None:
        """Stop the workers (their registers, and the key, die with the
        kernel).  Idempotent; errors if requests are still in flight."""
        if self._shut_down:
            return
        if self._pending:
            self._prune()  # deliver finished results nobody waited for
        if self.in_flight:
            raise PoolError(f"{self.in_flight} requests in flight")
        self._shut_down = True
        if self._svc is not None:
            svc, self._svc = self._svc, None
            rc = self._lib.pc_service_stop(svc)
            if rc != _native.PC_OK:
                raise PageCryptError(self._lib.pc_last_error().decode())

    def __del__(self):
        try:
            if not self._shut_down and self._svc is not None and not self.in_flight:
                self.shutdown()
        except Exception:
            pass
