"""Exception types, mirroring the reference hierarchy.

``pkg/src/pagecrypt/errors.py:4-27``: every cipher precondition raises
``ContractViolation`` (a ``PageCryptError``); worker-pool lifecycle errors are
``PoolError``.  CUDA failures surface as plain ``PageCryptError`` carrying the
native library's message.
"""


class PageCryptError(Exception):
    """Base class for all framework errors (errors.py:4)."""


class ContractViolation(PageCryptError):
    """A caller broke a documented precondition (errors.py:8-10)."""


class PoolError(PageCryptError):
    """Worker pool lifecycle error (errors.py:25-27)."""


class NativeLibraryMissing(PageCryptError):
    """libpagecrypt.so is not built or cannot be loaded.  There is no CPU
    fallback: the product path fails loudly instead."""
