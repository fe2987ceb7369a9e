"""ctypes binding of libpagecrypt.so (the C ABI in include/pagecrypt.h).

ctypes releases the GIL around every foreign call, so concurrent Python
callers (e.g. the reference's worker threads, pkg/src/pagecrypt/workers.py:
130-142) run the engine in parallel instead of serialising on the GIL the way
the reference numba kernel does (_chacha_numba.py:44 has no ``nogil``).

Status codes map to the reference's exception convention
(pkg/src/pagecrypt/errors.py:4-10): PC_EINVAL -> ContractViolation,
everything else -> PageCryptError.  If the library is missing the import of
the product API fails loudly; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ContractViolation, NativeLibraryMissing, PageCryptError

LIB_NAME = "libpagecrypt.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

PC_OK, PC_EINVAL, PC_ECUDA, PC_ENOMEM, PC_ESTATE, PC_ETIMEOUT, PC_EFULL = 0, 1, 2, 3, 4, 5, 6

c_void_p, c_size_t, c_int = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
c_u32, c_u64 = ctypes.c_uint32, ctypes.c_uint64
P = ctypes.POINTER

# name -> (restype, argtypes); the exact set of functions include/pagecrypt.h declares
SIGNATURES = {
    "pc_abi_version": (c_int, []),
    "pc_last_error": (ctypes.c_char_p, []),
    "pc_device_count": (c_int, [P(c_int)]),
    "pc_device_info": (c_int, [c_int, P(c_int), P(c_int), P(c_int)]),
    "pc_keystream_words": (c_int, [c_void_p, c_u64, c_u32, c_void_p, c_size_t, c_void_p, c_int]),
    "pc_keystream_raw": (c_int, [c_void_p, c_void_p, c_size_t, c_int, c_void_p]),
    "pc_key_install": (c_int, [c_int, c_void_p, P(c_void_p)]),
    "pc_key_generate": (c_int, [c_int, c_void_p, P(c_void_p)]),
    "pc_key_destroy": (c_int, [c_void_p]),
    "pc_key_device": (c_int, [c_void_p, P(c_int)]),
    "pc_key_replicate": (c_int, [c_void_p, c_int, P(c_void_p)]),
    "pc_key_export": (c_int, [c_void_p, c_void_p]),
    "pc_key_export_close": (c_int, [c_void_p]),
    "pc_key_import": (c_int, [c_int, c_void_p, P(c_void_p)]),
    "pc_crypt_pages_dev": (c_int, [c_void_p, c_void_p, c_void_p, c_u64, c_u32, c_void_p, c_void_p,
                                   c_size_t, c_int, c_void_p]),
    "pc_desc_check": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, P(c_u32)]),
    "pc_engine_create": (c_int, [c_int, c_int, c_size_t, P(c_void_p)]),
    "pc_engine_destroy": (c_int, [c_void_p]),
    "pc_engine_placement": (c_int, [c_void_p, P(c_int), P(c_int)]),
    "pc_crypt_pages_host": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_u64, c_u32,
                                    c_void_p, c_void_p, c_size_t, c_int]),
    "pc_crypt_pages_multi": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_u64, c_u32,
                                     c_void_p, c_void_p, c_size_t, c_int]),
    "pc_preload": (c_int, [c_int]),
    "pc_service_start": (c_int, [c_void_p, c_int, c_int, c_int, P(c_void_p)]),
    "pc_service_submit": (c_int, [c_void_p, c_int, c_u64, c_u32, c_void_p, c_void_p, P(c_u64)]),
    "pc_service_poll": (c_int, [c_void_p, c_int, c_u64, P(c_int)]),
    "pc_service_wait": (c_int, [c_void_p, c_int, c_u64, ctypes.c_int64]),
    "pc_service_crypt": (c_int, [c_void_p, c_int, c_u64, c_u32, c_void_p, c_void_p, ctypes.c_int64]),
    "pc_service_in_flight": (c_int, [c_void_p, P(c_u64)]),
    "pc_service_timing": (c_int, [c_void_p, c_int, c_u64, P(c_u64)]),
    "pc_service_max_workers": (c_int, [c_int, P(c_int)]),
    "pc_service_stop": (c_int, [c_void_p]),
    "pc_slab_transfer": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p, c_void_p,
                                 c_u64, c_u32, c_void_p, c_size_t, c_int, c_int, c_int]),
    "pc_slab_wipe": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t]),
    "pc_store_create": (c_int, [c_void_p, c_void_p, c_size_t, c_int, P(c_void_p)]),
    "pc_store_destroy": (c_int, [c_void_p]),
    "pc_store_put": (c_int, [c_void_p, c_u64, c_u32, c_void_p, c_size_t, c_void_p, c_int]),
    "pc_store_get": (c_int, [c_void_p, c_u64, c_u32, c_void_p, c_size_t, c_void_p, c_int, c_int]),
    "pc_store_remove": (c_int, [c_void_p, c_u64, c_void_p, c_size_t]),
    "pc_store_drop_client": (c_int, [c_void_p, c_u64]),
    "pc_store_contains": (c_int, [c_void_p, c_u64, c_u64, P(c_int)]),
    "pc_store_list": (c_int, [c_void_p, c_u64, c_void_p, c_size_t, P(c_size_t)]),
    "pc_store_free_slots": (c_int, [c_void_p, P(c_size_t)]),
    "pc_store_swap": (c_int, [c_void_p, c_u64, c_u32, c_void_p, c_size_t, c_void_p, c_void_p, c_size_t,
                              c_void_p]),
    "pc_store_contains_many": (c_int, [c_void_p, c_u64, c_void_p, c_size_t, c_void_p]),
    "pc_store_fault": (c_int, [c_void_p, c_u64, c_u32, c_u64, c_void_p, c_u64, c_void_p, P(c_int)]),
    "pc_store_service": (c_int, [c_void_p, c_int]),
    "pc_key_service": (c_int, [c_void_p, c_int, c_int]),
    "pc_service_worker_sm": (c_int, [c_void_p, c_int, P(c_int)]),
    "pc_host_alloc": (c_int, [c_size_t, P(c_void_p)]),
    "pc_host_free": (c_int, [c_void_p]),
    "pc_host_register": (c_int, [c_void_p, c_size_t]),
    "pc_host_unregister": (c_int, [c_void_p]),
    "pc_intpeak": (c_int, [c_int, c_int, P(ctypes.c_double)]),
    "pc_tune": (c_int, [ctypes.c_char_p, ctypes.c_int64]),
    "pc_tune_get": (c_int, [ctypes.c_char_p, P(ctypes.c_int64)]),
}

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load (once) and type the native library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            try:
                lib = ctypes.CDLL(LIB_PATH)
            except OSError as exc:  # pragma: no cover - broken build
                raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    """Raise the reference-style exception for a non-zero status."""
    if rc == PC_OK:
        return
    msg = load().pc_last_error().decode(errors="replace")
    if rc == PC_EINVAL:
        raise ContractViolation(msg)
    raise PageCryptError(f"libpagecrypt error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def tune(knob: str, value: int) -> None:
    call("pc_tune", knob.encode(), int(value))


def tune_get(knob: str) -> int:
    v = ctypes.c_int64()
    call("pc_tune_get", knob.encode(), ctypes.byref(v))
    return v.value


def device_info(device: int = 0) -> dict:
    sms, ma, mi = c_int(), c_int(), c_int()
    call("pc_device_info", device, ctypes.byref(sms), ctypes.byref(ma), ctypes.byref(mi))
    return {"sm_count": sms.value, "cc": (ma.value, mi.value)}


def device_count() -> int:
    n = c_int(0)
    rc = load().pc_device_count(ctypes.byref(n))
    return n.value if rc == PC_OK else 0
