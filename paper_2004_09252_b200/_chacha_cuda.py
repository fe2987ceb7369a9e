"""Kernel-seam shim: a drop-in for ``pagecrypt._chacha_numba``.

The reference cipher imports its kernel optionally
(``pkg/src/pagecrypt/cipher.py:28-31``) and calls exactly one function,
``keystream_words(kw, vaddr, pid, indices, out)``
(``pkg/src/pagecrypt/_chacha_numba.py:44-93``, consumed at
``cipher.py:178-181``).  Binding this module in its place
(``pagecrypt.cipher._chacha_numba = paper_2004_09252_b200._chacha_cuda``) runs
the reference package's keystream on the B200 with identical results; see
INTEGRATION.md.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .engine import _addr


def keystream_words(kw, vaddr, pid, indices, out) -> None:
    """Write the keystream blocks for ``indices`` into ``out``.

    kw:      uint32[8] little-endian key words (may be read-only)
    vaddr:   u64 page address, pid: u32
    indices: int64[k] block indices
    out:     uint32[16 * k], block-major, C-contiguous, writable
    Same contract as the numba kernel: no validation beyond buffer shapes.
    """
    kw = np.ascontiguousarray(kw, dtype=np.uint32)
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    if kw.size != 8:
        raise ValueError("kw must hold 8 words")
    if out.dtype != np.uint32 or not out.flags.c_contiguous or out.size != 16 * idx.size:
        raise ValueError("out must be a C-contiguous uint32[16*k] array")
    if idx.size == 0:
        return
    _native.call("pc_keystream_words", _addr(kw), int(vaddr) & (2**64 - 1),
                 int(pid) & 0xFFFFFFFF, _addr(idx), idx.size, _addr(out), 20)
