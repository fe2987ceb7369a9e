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


def adopt_host_errors(host) -> None:
    """Drop-in integration: make this package raise the HOST package's
    exception classes (e.g. ``pagecrypt.errors``), so callers written against
    the reference -- ``except pagecrypt.PoolError`` / ``pytest.raises`` --
    see the same types when the B200 engine is bound into them
    (INTEGRATION.md).  ``host`` is a module (or object) with attributes
    PageCryptError, ContractViolation and PoolError; every module of this
    package that imported our class under that name is rebound."""
    import sys

    ours = {"PageCryptError": PageCryptError, "ContractViolation": ContractViolation, "PoolError": PoolError}
    theirs = {name: getattr(host, name) for name in ours}
    for name, cls in theirs.items():
        if not (isinstance(cls, type) and issubclass(cls, BaseException)):
            raise TypeError(f"host {name} is not an exception class")
    prefix = __name__.rsplit(".", 1)[0]
    for modname, mod in list(sys.modules.items()):
        if mod is None or not (modname == prefix or modname.startswith(prefix + ".")):
            continue
        for name, cls in ours.items():
            if getattr(mod, name, None) is cls:
                setattr(mod, name, theirs[name])
