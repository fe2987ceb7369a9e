"""Device keys, per-device engines and the batched page-cipher entry point.

This is the B200 replacement for the host side of the reference's crypto
worker service (``pkg/src/pagecrypt/workers.py``):

* :class:`DeviceKey` -- the key slot.  The reference keeps one private 32-byte
  copy per worker thread, installed through a staging buffer that is wiped
  (``workers.py:167-169,174-202``) and wiped again on shutdown
  (``workers.py:252-254``).  Here the key lives only in device memory
  (``pc_key_install`` / ``pc_key_generate``) and ``destroy`` zeroes it there.
* :class:`Engine` -- one per device: CUDA streams, device staging and pinned
  bounce buffers so host-resident page batches stream H2D -> cipher -> D2H
  with the three stages of consecutive chunks overlapped.
* :func:`crypt_pages` -- the batched form of ``cipher.crypt_page``
  (``pkg/src/pagecrypt/cipher.py:205-217``) over ``uint8[n, 4096]`` pages that
  are either device-resident (torch CUDA tensors; asynchronous on the current
  stream) or host-resident (numpy / torch CPU / any buffer; synchronous).
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Any

import numpy as np

from . import _native
from .errors import ContractViolation, PageCryptError

PAGE_SIZE = 4096
KEY_SIZE = 32
ROUNDS = (8, 12, 20)


def _check_rounds(rounds: int) -> None:
    if rounds not in ROUNDS:
        raise ContractViolation(f"rounds must be one of {ROUNDS}, got {rounds}")


def key_bytes(key) -> memoryview:
    """32 raw key bytes from MasterKey / bytes / bytearray / memoryview
    (``cipher._key_words``, pkg/src/pagecrypt/cipher.py:119-124)."""
    view = getattr(key, "view", None)
    if callable(view) and not isinstance(key, (bytes, bytearray, memoryview, np.ndarray)):
        key = view()
    mv = memoryview(key).cast("B")
    if len(mv) != KEY_SIZE:
        raise ContractViolation(f"key must be {KEY_SIZE} bytes, got {len(mv)}")
    return mv


def _addr_of_readonly(buf) -> tuple[int, Any]:
    """(address, keepalive) of any C-contiguous buffer, read-only allowed."""
    arr = np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf
    return arr.ctypes.data, arr


_Key = ctypes.c_char * KEY_SIZE


def _ptr(buf, ctype):
    """(argument, keepalive): something ctypes passes as a c_void_p to buf's
    bytes, without copying them (a copy of key material could not be wiped).
    bytes and bytearray take the cheap paths; anything else goes through numpy."""
    if type(buf) is bytes:
        return buf, buf
    if type(buf) is bytearray:
        return ctype.from_buffer(buf), buf
    arr = np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf
    if not arr.flags.c_contiguous:
        raise ContractViolation("buffer must be C-contiguous")
    return arr.ctypes.data, arr


def _addr(arr: np.ndarray) -> int:
    """Address of a non-empty C-contiguous array (``arr.ctypes.data`` costs
    ~2 us; a ctypes view of a writable buffer ~0.8 us)."""
    if arr.flags.writeable:
        return ctypes.addressof(ctypes.c_char.from_buffer(arr))
    return arr.ctypes.data


def raw_key_arg(key):
    """(argument, keepalive) for the raw-key (caller-key) mode of the C ABI:
    32 key bytes from MasterKey / bytes / bytearray / memoryview, validated,
    passed by address without a copy."""
    kv = key_bytes(key)
    obj = kv.obj
    return _ptr(obj if type(obj) in (bytes, bytearray) and len(obj) == KEY_SIZE else kv, _Key)


class DeviceKey:
    """A 256-bit master key resident in one GPU's memory (the key slot)."""

    __slots__ = ("_handle", "_device", "__weakref__")

    def __init__(self, handle: int, device: int):
        self._handle = handle
        self._device = device

    @classmethod
    def install(cls, key, device: int = 0) -> "DeviceKey":
        """Copy caller key bytes into device memory (parity / caller-key mode)."""
        kb = key_bytes(key)
        addr, keep = _addr_of_readonly(kb)
        h = ctypes.c_void_p()
        _native.call("pc_key_install", device, addr, ctypes.byref(h))
        del keep
        return cls(h.value, device)

    @classmethod
    def generate(cls, device: int = 0) -> "DeviceKey":
        """Fresh key derived on the device from OS entropy mixed with
        device-only entropy; the key itself never exists in host RAM
        (reference: ``MasterKey.generate`` = os.urandom, cipher.py:59-62)."""
        ent = bytearray(os.urandom(KEY_SIZE))
        buf = (ctypes.c_char * KEY_SIZE).from_buffer(ent)
        h = ctypes.c_void_p()
        try:
            _native.call("pc_key_generate", device, ctypes.addressof(buf), ctypes.byref(h))
        finally:
            ctypes.memset(ctypes.addressof(buf), 0, KEY_SIZE)
            del buf
        return cls(h.value, device)

    def replicate(self, device: int) -> "DeviceKey":
        """The same key on another GPU, copied device-to-device (NVLink peer
        copy; refused rather than staged through host RAM when the GPUs have
        no peer access).  The analog of the per-worker key slots filled from
        one staged key (workers.py:193-194)."""
        h = ctypes.c_void_p()
        _native.call("pc_key_replicate", self.handle, int(device), ctypes.byref(h))
        return DeviceKey(h.value, int(device))

    def export_handle(self) -> bytes:
        """64-byte CUDA-IPC handle of a device copy of the key, for
        :meth:`import_handle` in another process (one process per GPU).  The
        handle names device memory; it is not key material.  Keep the export
        open until every importer has returned, then :meth:`close_export`."""
        buf = (ctypes.c_uint8 * 64)()
        _native.call("pc_key_export", self.handle, buf)
        return bytes(buf)

    def close_export(self) -> None:
        """Zero the exported copy (importers already hold their own keys)."""
        _native.call("pc_key_export_close", self.handle)

    @classmethod
    def import_handle(cls, handle: bytes, device: int = 0) -> "DeviceKey":
        """A key on ``device`` copied device-to-device from another process's
        :meth:`export_handle` (the exporter must keep its export open)."""
        if len(handle) != 64:
            raise ContractViolation("key handle must be 64 bytes")
        buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
        h = ctypes.c_void_p()
        _native.call("pc_key_import", int(device), buf, ctypes.byref(h))
        return cls(h.value, int(device))

    @property
    def device(self) -> int:
        return self._device

    @property
    def destroyed(self) -> bool:
        return self._handle is None

    @property
    def handle(self) -> int:
        if self._handle is None:
            raise PageCryptError("device key already destroyed")
        return self._handle

    def start_service(self, n_workers: int = 1, rounds: int = 20) -> None:
        """Start resident GPU workers holding this key (``pc_key_service``):
        host batches of up to one page per worker (at most 6) under this key and round
        count then run as service tickets instead of launches -- the fault
        handler's 1-2 page calls skip the launch and the stream sync.
        ``stop_service``/``destroy`` stop them."""
        if n_workers < 1:
            raise ContractViolation(f"n_workers must be >= 1, got {n_workers}")
        if rounds not in (8, 12, 20):
            raise ContractViolation(f"rounds must be 8, 12 or 20, got {rounds}")
        _native.call("pc_key_service", self.handle, n_workers, rounds)

    def stop_service(self) -> None:
        if self._handle is not None:
            _native.call("pc_key_service", self._handle, 0, 0)

    def destroy(self) -> None:
        """Zero the device copy and free it (workers.py:252-254).  Idempotent."""
        if self._handle is not None:
            # a key still held by a page store is refused (PC_ESTATE) and stays live
            _native.call("pc_key_destroy", self._handle)
            self._handle = None

    def __enter__(self) -> "DeviceKey":
        return self

    def __exit__(self, *exc) -> None:
        self.destroy()

    def __del__(self):  # best effort; explicit destroy() is the contract
        try:
            self.destroy()
        except Exception:
            pass


class Engine:
    """Per-device streams + staging for host-resident batches."""

    def __init__(self, device: int = 0, n_streams: int = 4, chunk_pages: int = 8192):
        h = ctypes.c_void_p()
        _native.call("pc_engine_create", device, n_streams, chunk_pages, ctypes.byref(h))
        self._handle = h.value
        self.device = device
        self.n_streams = n_streams
        self.chunk_pages = chunk_pages

    @property
    def handle(self) -> int:
        if self._handle is None:
            raise PageCryptError("engine destroyed")
        return self._handle

    def destroy(self) -> None:
        if self._handle is not None:
            h, self._handle = self._handle, None
            _native.call("pc_engine_destroy", h)

    @property
    def placement(self) -> dict:
        """Host placement of the engine's threads and pinned staging: the
        GPU's NUMA node (-1 = not reported) and the GPU-local CPUs bound."""
        node, ncpu = ctypes.c_int(), ctypes.c_int()
        _native.call("pc_engine_placement", self.handle, ctypes.byref(node), ctypes.byref(ncpu))
        return {"numa_node": node.value, "bound_cpus": ncpu.value}

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def crypt_host(self, key, vaddrs, pids, src_addr: int, dst_addr: int, n: int, rounds: int) -> None:
        """Raw-pointer host path.  ``key`` is a DeviceKey or raw key bytes."""
        _check_rounds(rounds)
        v_arr, vaddr0 = _host_vaddrs(vaddrs, n)
        p_arr, pid0 = _host_pids(pids, n)
        if isinstance(key, DeviceKey):
            if key.device != self.device:
                raise ContractViolation(f"key on device {key.device}, engine on {self.device}")
            kh, raw = key.handle, (None, None)
        else:
            kh, raw = None, raw_key_arg(key)
        rc = _native.load().pc_crypt_pages_host(
            self.handle, kh, raw[0],
            None if v_arr is None else v_arr.ctypes.data,
            None if p_arr is None else p_arr.ctypes.data,
            vaddr0, pid0, src_addr, dst_addr, n, rounds,
        )
        if rc:
            _native.check(rc)


_engines: dict[int, Engine] = {}
_engines_lock = threading.Lock()


_default_device: int | None = None


def default_engine(device: int | None = None) -> Engine:
    global _default_device
    if device is None:
        if _default_device is None:
            _default_device = int(os.environ.get("PAGECRYPT_DEVICE", "0"))
        device = _default_device
    eng = _engines.get(device)
    if eng is None:
        with _engines_lock:
            eng = _engines.get(device)
            if eng is None:
                eng = _engines[device] = Engine(device)
    return eng


# ---------------------------------------------------------------------------
# page descriptors


def _check_vaddr_int(v: int) -> None:
    if not 0 <= v < 2**64:
        raise ContractViolation(f"vaddr {v:#x} not a u64")
    if v % PAGE_SIZE:
        raise ContractViolation(f"vaddr {v:#x} not page-aligned")


def _check_pid_int(p: int) -> None:
    if not 0 <= p < 2**32:
        raise ContractViolation(f"pid {p} not a u32")


def _host_vaddrs(vaddrs, n: int):
    """(array or None, vaddr0).  An int is the first page of a contiguous run."""
    if isinstance(vaddrs, (int, np.integer)):
        v0 = int(vaddrs)
        _check_vaddr_int(v0)
        if n and v0 + PAGE_SIZE * (n - 1) >= 2**64:
            raise ContractViolation("contiguous vaddr range overflows u64")
        return None, v0
    if isinstance(vaddrs, (list, tuple, range)):
        ints = [int(v) for v in vaddrs]
        for v in ints:
            _check_vaddr_int(v)  # range and alignment: the array needs no more checks
        if len(ints) != n:
            raise ContractViolation(f"{len(ints)} vaddrs for {n} pages")
        return np.array(ints, dtype=np.uint64), 0
    arr = np.asarray(vaddrs)
    if arr.dtype.kind not in "iu":
        raise ContractViolation(f"vaddrs must be integers, got {arr.dtype}")
    if arr.dtype.kind == "i" and (arr < 0).any():
        raise ContractViolation("vaddr not a u64 (negative)")
    arr = np.ascontiguousarray(arr.astype(np.uint64, copy=False)).reshape(-1)
    if arr.size != n:
        raise ContractViolation(f"{arr.size} vaddrs for {n} pages")
    if (arr & np.uint64(PAGE_SIZE - 1)).any():
        bad = int(arr[(arr & np.uint64(PAGE_SIZE - 1)) != 0][0])
        raise ContractViolation(f"vaddr {bad:#x} not page-aligned")
    return arr, 0


def _host_pids(pids, n: int):
    if isinstance(pids, (int, np.integer)):
        _check_pid_int(int(pids))
        return None, int(pids)
    if isinstance(pids, (list, tuple, range)):
        for p in pids:
            _check_pid_int(int(p))
        pids = np.array([int(p) for p in pids], dtype=np.uint32)
    arr = np.asarray(pids)
    if arr.dtype.kind not in "iu":
        raise ContractViolation(f"pids must be integers, got {arr.dtype}")
    if arr.size and (int(arr.min()) < 0 or int(arr.max()) >= 2**32):
        raise ContractViolation("pid not a u32")
    arr = np.ascontiguousarray(arr.astype(np.uint32, copy=False)).reshape(-1)
    if arr.size != n:
        raise ContractViolation(f"{arr.size} pids for {n} pages")
    return arr, 0


# ---------------------------------------------------------------------------
# batched entry point


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def crypt_pages(key, vaddrs, pids, pages, *, rounds: int = 20, out=None, stream=None,
                engine: Engine | None = None, check: bool = True):
    """XOR ``n`` 4 KiB pages with their keystreams (encrypt == decrypt).

    key     DeviceKey (production: the key never leaves device memory) or
            32 raw key bytes / MasterKey (caller-key parity mode).
    vaddrs  int (page i gets vaddrs + 4096*i) or n per-page addresses.
    pids    int or n per-page pids.  Only the pid enters the seed, as in the
            reference worker (pkg/src/pagecrypt/workers.py:137).
    pages   uint8[n, 4096]: a CUDA tensor (device path, asynchronous on
            ``stream`` or torch's current stream) or host memory (numpy /
            torch CPU tensor / buffer; synchronous, via the engine's pipeline).
    out     destination of the same kind; defaults to a new buffer.  ``out``
            may be ``pages`` (in place).
    check   device path with a CUDA vaddr tensor: validate page alignment
            on the device first (ContractViolation at call time, as the
            reference raises).  The check synchronises ``stream``; pass
            False to keep the call fully asynchronous when the descriptors
            are known good.  (An int64 pid tensor is always narrowed to
            u32 by the same library kernel, which also synchronises; its
            range check raises only when ``check`` is True.)
    Returns ``out``.
    """
    if (type(key) is DeviceKey and type(vaddrs) is int and type(pids) is int and out is not None
            and engine is None and (rounds == 20 or rounds == 12 or rounds == 8)):
        done = _fast_host(key, vaddrs, pids, pages, out, rounds)
        if done is not None:
            return done
    _check_rounds(rounds)
    if _is_torch(pages) and pages.is_cuda:
        return _crypt_pages_device(key, vaddrs, pids, pages, rounds, out, stream, check)
    return _crypt_pages_host(key, vaddrs, pids, pages, rounds, out, engine)


_fast = None  # the _pcfast extension (csrc/fastpath.c), loaded on first use


def _fastmod():
    global _fast
    if _fast is None:
        _native.load()
        try:
            from . import _pcfast
        except ImportError:  # not built: the ctypes path below serves every call
            _pcfast = False
        _fast = _pcfast
    return _fast


def _fast_host(key, vaddr0, pid0, pages, out, rounds):
    """The fault handler's call shape -- a DeviceKey, a contiguous vaddr run
    and one pid, host pages with a host ``out`` -- in one METH_FASTCALL call
    (csrc/fastpath.c: ~0.1 us instead of ~5 us of checks and ctypes
    conversions).  Returns ``out``, or None to hand anything unusual
    (including every error case, so the messages stay the general path's) to
    the general path."""
    fm = _fastmod()
    if not fm:
        return None
    tp = type(pages)
    if tp is np.ndarray or tp is bytearray or tp is bytes or tp is memoryview:
        if vaddr0 < 0 or vaddr0 & 4095 or not 0 <= pid0 < 2**32 or vaddr0 >= 2**64:
            return None  # (a contiguous run past 2^64 is refused by the library itself)
        h = key._handle
        if h is None:
            return None
        eng = _engines.get(key._device) or default_engine(key._device)
        rc = fm.crypt_host_buf(eng._handle, h, vaddr0, pid0, pages, out, rounds)
        if rc < 0:
            return None  # not contiguous / writable / whole pages: the general path says why
        if rc:
            _native.check(rc)
        return out
    if tp.__module__ == "torch" and type(out) is tp:
        if pages.is_cuda or out.is_cuda or not pages.is_contiguous() or not out.is_contiguous():
            return None
        nb = pages.nbytes
        if out.nbytes != nb:
            return None
        src, dst = pages.data_ptr(), out.data_ptr()
    else:
        return None
    if nb == 0 or nb & 4095 or vaddr0 < 0 or vaddr0 & 4095 or not 0 <= pid0 < 2**32:
        return None
    n = nb >> 12
    if vaddr0 + PAGE_SIZE * (n - 1) >= 2**64:
        return None
    h = key._handle
    if h is None:
        return None
    eng = _engines.get(key._device) or default_engine(key._device)
    rc = fm.crypt_host(eng._handle, h, vaddr0, pid0, src, dst, n, rounds)
    if rc:
        _native.check(rc)
    return out


def _page_count(nbytes: int) -> int:
    if nbytes % PAGE_SIZE:
        raise ContractViolation(f"page buffer of {nbytes} bytes is not a whole number of pages")
    return nbytes // PAGE_SIZE


def _crypt_pages_host(key, vaddrs, pids, pages, rounds, out, engine):
    if _is_torch(pages):
        if not pages.is_contiguous():
            raise ContractViolation("pages must be contiguous")
        n = _page_count(pages.numel() * pages.element_size())
        src = pages.data_ptr()
        if out is None:
            import torch
            out = torch.empty_like(pages, pin_memory=pages.is_pinned())
        dst = out.data_ptr()
        if out.numel() * out.element_size() != n * PAGE_SIZE:
            raise ContractViolation("out has the wrong size")
        keep = (pages, out)
    else:
        arr = pages if isinstance(pages, np.ndarray) else np.frombuffer(pages, dtype=np.uint8)
        if not arr.flags.c_contiguous:
            raise ContractViolation("pages must be C-contiguous")
        n = _page_count(arr.nbytes)
        if out is None:
            out = np.empty((n, PAGE_SIZE), dtype=np.uint8)
        oarr = out if isinstance(out, np.ndarray) else np.frombuffer(out, dtype=np.uint8)
        if oarr.nbytes != n * PAGE_SIZE or not oarr.flags.writeable:
            raise ContractViolation("out must be a writable buffer of the same size")
        if n == 0:
            return out
        src, dst = _addr(arr), _addr(oarr)
        keep = (arr, oarr)
    if n == 0:
        return out
    eng = engine or default_engine(key.device if isinstance(key, DeviceKey) else None)
    eng.crypt_host(key, vaddrs, pids, src, dst, n, rounds)
    del keep
    return out


def _desc_flags(vaddrs_ptr, pids64_ptr, pids32_ptr, n: int, stream_handle) -> int:
    flags = ctypes.c_uint32()
    _native.call("pc_desc_check", vaddrs_ptr, pids64_ptr, pids32_ptr, n, stream_handle, ctypes.byref(flags))
    return flags.value


def _crypt_pages_device(key, vaddrs, pids, pages, rounds, out, stream, check):
    import torch

    if pages.dtype != torch.uint8 or not pages.is_contiguous():
        raise ContractViolation("device pages must be a contiguous uint8 tensor")
    n = _page_count(pages.numel())
    dev = pages.device.index if pages.device.index is not None else torch.cuda.current_device()
    if out is None:
        out = torch.empty_like(pages)
    elif not (out.is_cuda and out.dtype == torch.uint8 and out.is_contiguous() and out.numel() == pages.numel()):
        raise ContractViolation("out must be a contiguous uint8 CUDA tensor like pages")
    if n == 0:
        return out
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    # page descriptors: scalar/contiguous forms, or device arrays
    v_ptr = p_ptr = None
    vaddr0 = pid0 = 0
    keep = []
    if isinstance(vaddrs, (int, np.integer)):
        vaddr0 = int(vaddrs)
        _check_vaddr_int(vaddr0)
        if vaddr0 + PAGE_SIZE * (n - 1) >= 2**64:
            raise ContractViolation("contiguous vaddr range overflows u64")
    else:
        if not _is_torch(vaddrs):
            host, _ = _host_vaddrs(vaddrs, n)
            vaddrs = torch.from_numpy(host.view(np.int64)).to(pages.device, non_blocking=False)
        elif vaddrs.numel() != n or vaddrs.element_size() != 8 or vaddrs.dtype.is_floating_point:
            raise ContractViolation("vaddrs must be n 64-bit integers")
        else:
            vaddrs = vaddrs.to(pages.device).contiguous()
            if check and _desc_flags(vaddrs.data_ptr(), None, None, n, sh) & 1:
                raise ContractViolation("vaddr not page-aligned")
        keep.append(vaddrs)
        v_ptr = vaddrs.data_ptr()
    if isinstance(pids, (int, np.integer)):
        pid0 = int(pids)
        _check_pid_int(pid0)
    else:
        if not _is_torch(pids):
            host, _ = _host_pids(pids, n)
            pids = torch.from_numpy(host.view(np.int32)).to(pages.device)
        elif pids.numel() != n:
            raise ContractViolation("need n pids")
        else:
            pids = pids.to(pages.device).contiguous()
            if pids.dtype.is_floating_point or pids.dtype.is_complex or pids.dtype == torch.bool:
                raise ContractViolation("pids must be 32- or 64-bit integers")
            if pids.element_size() != 4:
                if pids.element_size() != 8:
                    raise ContractViolation("pids must be 32- or 64-bit integers")
                # narrowed (and range-checked) by a library kernel: no torch
                # kernel launches here, so this is safe beside the worker service
                p32 = torch.empty(n, dtype=torch.int32, device=pages.device)
                if _desc_flags(None, pids.data_ptr(), p32.data_ptr(), n, sh) & 2 and check:
                    raise ContractViolation("pid not a u32")
                pids = p32
        keep.append(pids)
        p_ptr = pids.data_ptr()

    if isinstance(key, DeviceKey):
        if key.device != dev:
            raise ContractViolation(f"key on device {key.device}, pages on {dev}")
        _native.call("pc_crypt_pages_dev", key.handle, v_ptr, p_ptr, vaddr0, pid0,
                     pages.data_ptr(), out.data_ptr(), n, rounds, sh)
    else:
        # caller-key mode: a temporary device key slot, destroyed (zeroed) after
        # the stream has consumed it
        tmp = DeviceKey.install(key, dev)
        try:
            _native.call("pc_crypt_pages_dev", tmp.handle, v_ptr, p_ptr, vaddr0, pid0,
                         pages.data_ptr(), out.data_ptr(), n, rounds, sh)
        finally:
            tmp.destroy()  # zeroed on the key's stream after the batch's use of it
    if keep:
        # keep descriptor tensors alive until the stream has used them
        for t in keep:
            t.record_stream(stream if hasattr(stream, "cuda_stream") else torch.cuda.current_stream(dev))
    return out
