"""ctypes binding of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Used by tests/ (parity at sizes the pure-Python oracle cannot reach), by
__graft_entry__.smoke() and by bench.py's CPU-baseline legs.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "chacha_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_block_raw.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p]
        L.oracle_block_raw.restype = None
        L.oracle_crypt_pages.argtypes = [
            ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
        ]
        L.oracle_crypt_pages.restype = None
        _lib = L
    return _lib


def block_raw(key: bytes, seed16: bytes, rounds: int = 20) -> bytes:
    out = ctypes.create_string_buffer(64)
    lib().oracle_block_raw(bytes(key), bytes(seed16), rounds, out)
    return out.raw


def crypt_pages(key: bytes, vaddrs, pids, pages: np.ndarray, rounds: int = 20,
                nthreads: int = 1, out: np.ndarray | None = None,
                vaddr0: int = 0, pid0: int = 0) -> np.ndarray:
    """uint8[n,4096] -> uint8[n,4096].  vaddrs/pids None => vaddr0 + 4096*i / pid0."""
    pages = np.ascontiguousarray(pages, dtype=np.uint8).reshape(-1, 4096)
    n = pages.shape[0]
    if out is None:
        out = np.empty_like(pages)
    va = None if vaddrs is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(vaddrs, dtype=np.uint64), (n,)))
    pi = None if pids is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(pids, dtype=np.uint32), (n,)))
    lib().oracle_crypt_pages(
        bytes(key),
        None if va is None else va.ctypes.data,
        None if pi is None else pi.ctypes.data,
        vaddr0, pid0, pages.ctypes.data, out.ctypes.data, n, rounds, nthreads,
    )
    return out
