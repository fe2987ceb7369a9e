"""Record the REFERENCE's public surface on the hot path, for the drop-in check.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_api_surface.py

Writes ``api_surface.json``: for ``pagecrypt.cipher`` (the API seam,
SURVEY §8b), ``pagecrypt.workers.WorkerPool`` / ``Completion`` and
``pagecrypt.store.EncryptedPageStore`` every public callable with its
parameters (name, kind, whether it has a default) and the cipher constants'
values.  ``tests/test_api_surface.py`` checks the B200 package against it.
"""

from __future__ import annotations

import inspect
import json
import os
import sys
from pathlib import Path

REF = Path(os.environ.get("PAGECRYPT_REF", "/root/reference/pkg"))
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from pagecrypt import cipher, store, workers  # noqa: E402


def params(fn) -> list:
    return [[p.name, p.kind.name, p.default is not inspect.Parameter.empty]
            for p in inspect.signature(fn).parameters.values()]


def members(cls) -> dict:
    out = {}
    for name, obj in vars(cls).items():
        if name.startswith("_") and name != "__init__":
            continue
        if isinstance(obj, property):
            out[name] = "property"
        elif isinstance(obj, (staticmethod, classmethod)):
            out[name] = params(obj.__func__)
        elif callable(obj):
            out[name] = params(obj)
    return out


def main() -> None:
    surface = {
        "cipher_functions": {n: params(getattr(cipher, n)) for n in
                             ("chacha20_block", "page_keystream", "crypt_page", "parallel_crypt_page")},
        "cipher_classes": {n: members(getattr(cipher, n)) for n in ("MasterKey", "BlockSeed")},
        "cipher_constants": {n: getattr(cipher, n) for n in
                             ("PAGE_SIZE", "BLOCK_SIZE", "BLOCKS_PER_PAGE", "LANE_UNIT_BLOCKS", "LANE_UNITS",
                              "KEY_SIZE")},
        "workers": {"WorkerPool": members(workers.WorkerPool), "Completion": members(workers.Completion)},
        "store": {"EncryptedPageStore": members(store.EncryptedPageStore)},
    }
    (OUT / "api_surface.json").write_text(json.dumps(surface, indent=1, sort_keys=True) + "\n")
    print("wrote", OUT / "api_surface.json")


if __name__ == "__main__":
    main()
