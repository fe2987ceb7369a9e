"""B200 page-cipher engine for MemShield's hot path (arXiv 2004.09252).

Drop-in for the reference ``pagecrypt`` cipher API
(``/root/reference/pkg/src/pagecrypt/__init__.py:10-18``) backed by sm_100a
CUDA kernels in ``libpagecrypt.so`` (C ABI: ``include/pagecrypt.h``), plus
batched device/host entry points, device-resident keys and a multi-GPU
page-range partitioner.
"""

from .cipher import (
    BLOCK_SIZE,
    BLOCKS_PER_PAGE,
    KEY_SIZE,
    PAGE_SIZE,
    BlockSeed,
    MasterKey,
    chacha20_block,
    crypt_page,
    keystream_raw,
    page_keystream,
    parallel_crypt_page,
)
from .engine import DeviceKey, Engine, crypt_pages, default_engine
from .errors import ContractViolation, NativeLibraryMissing, PageCryptError, PoolError

__version__ = "0.1.0"

__all__ = [
    "BLOCK_SIZE", "BLOCKS_PER_PAGE", "BlockSeed", "ContractViolation", "DeviceKey", "Engine",
    "KEY_SIZE", "MasterKey", "NativeLibraryMissing", "PAGE_SIZE", "PageCryptError", "PoolError",
    "chacha20_block", "crypt_page", "crypt_pages", "default_engine", "keystream_raw",
    "page_keystream", "parallel_crypt_page",
]
