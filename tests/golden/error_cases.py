"""Edge-case / bad-input calls of the cipher API seam, evaluated identically
against the reference ``pagecrypt.cipher`` (make_error_golden.py) and the
B200 ``paper_2004_09252_b200.cipher`` (tests/test_error_golden.py)."""

from __future__ import annotations

import numpy as np

K = bytes(range(32))
P = bytes(4096)


def _cases(c):
    return {
        # keys
        "key_31_bytes": lambda: c.crypt_page(K[:31], 0x1000, 1, P),
        "key_33_bytes": lambda: c.crypt_page(K + b"\0", 0x1000, 1, P),
        "key_bytearray": lambda: c.crypt_page(bytearray(K), 0x1000, 1, P),
        "key_memoryview": lambda: c.crypt_page(memoryview(K), 0x1000, 1, P),
        "key_masterkey": lambda: c.crypt_page(c.MasterKey(K), 0x1000, 1, P),
        "masterkey_short": lambda: c.MasterKey(K[:16]),
        "masterkey_destroyed_view": lambda: (lambda m: (m.destroy(), m.view()))(c.MasterKey(K)),
        # vaddr / pid
        "vaddr_unaligned": lambda: c.crypt_page(K, 0x1001, 1, P),
        "vaddr_negative": lambda: c.crypt_page(K, -4096, 1, P),
        "vaddr_2_64": lambda: c.crypt_page(K, 2**64, 1, P),
        "vaddr_max_page": lambda: c.crypt_page(K, 2**64 - 4096, 1, P),
        "vaddr_zero": lambda: c.crypt_page(K, 0, 1, P),
        "pid_negative": lambda: c.crypt_page(K, 0x1000, -1, P),
        "pid_2_32": lambda: c.crypt_page(K, 0x1000, 2**32, P),
        "pid_max": lambda: c.crypt_page(K, 0x1000, 2**32 - 1, P),
        # pages
        "page_4095": lambda: c.crypt_page(K, 0x1000, 1, P[:-1]),
        "page_4097": lambda: c.crypt_page(K, 0x1000, 1, P + b"\0"),
        "page_empty": lambda: c.crypt_page(K, 0x1000, 1, b""),
        "page_bytearray": lambda: c.crypt_page(K, 0x1000, 1, bytearray(P)),
        "page_memoryview": lambda: c.crypt_page(K, 0x1000, 1, memoryview(P)),
        "page_ndarray_u8": lambda: c.crypt_page(K, 0x1000, 1, np.zeros(4096, np.uint8)),
        "page_ndarray_2d": lambda: c.crypt_page(K, 0x1000, 1, np.zeros((1, 4096), np.uint8)),
        # lanes
        "lanes_zero": lambda: c.parallel_crypt_page(K, 0x1000, 1, P, 0),
        "lanes_negative": lambda: c.parallel_crypt_page(K, 0x1000, 1, P, -3),
        "lanes_one": lambda: c.parallel_crypt_page(K, 0x1000, 1, P, 1),
        "lanes_1000": lambda: c.parallel_crypt_page(K, 0x1000, 1, P, 1000),
        "lanes_bad_page": lambda: c.parallel_crypt_page(K, 0x1000, 1, P[:100], 4),
        # block seeds
        "seed_idx_64": lambda: c.BlockSeed(0x1000, 1, 64),
        "seed_idx_negative": lambda: c.BlockSeed(0x1000, 1, -1),
        "seed_unaligned": lambda: c.BlockSeed(0x1001, 1, 0),
        "seed_pid_2_32": lambda: c.BlockSeed(0x1000, 2**32, 0),
        "seed_from_bytes_15": lambda: c.BlockSeed.from_bytes(bytes(15)),
        "seed_from_bytes_idx_64": lambda: c.BlockSeed.from_bytes(
            (0x1000).to_bytes(8, "little") + (1).to_bytes(4, "little") + (64).to_bytes(4, "little")),
        "block_ok": lambda: c.chacha20_block(K, c.BlockSeed(0x1000, 1, 63)),
        "block_bad_key": lambda: c.chacha20_block(K[:8], c.BlockSeed(0x1000, 1, 0)),
        "keystream_unaligned": lambda: c.page_keystream(K, 0x10, 1),
        "keystream_bad_pid": lambda: c.page_keystream(K, 0x1000, 2**40),
    }


CASES = sorted(_cases(type("Null", (), {})).keys())


def run_case(cipher_module, name: str) -> str:
    """'ok' or the name of the exception the call raised."""
    try:
        _cases(cipher_module)[name]()
        return "ok"
    except Exception as exc:  # noqa: BLE001 - the class is the result
        return type(exc).__name__
