"""Record how the REFERENCE cipher API reacts to edge-case and bad inputs.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_error_golden.py

Each case in ``CASES`` (shared with ``tests/test_error_golden.py`` through
``error_cases.py``) is evaluated against the reference ``pagecrypt.cipher``
and its outcome -- "ok" or the exception class name -- is written to
``error_golden.json``.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

REF = Path(os.environ.get("PAGECRYPT_REF", "/root/reference/pkg"))
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(OUT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from pagecrypt import cipher  # noqa: E402

from error_cases import CASES, run_case  # noqa: E402


def main() -> None:
    out = {}
    for name in CASES:
        out[name] = run_case(cipher, name)
    (OUT / "error_golden.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("wrote", len(out), "cases to", OUT / "error_golden.json")


if __name__ == "__main__":
    main()
