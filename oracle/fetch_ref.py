"""Copy the reference package and its test suite into oracle/_ref/ (TEST
INFRASTRUCTURE ONLY -- never imported by the product).

The reference (arxiv/paper_2004_09252, /root/reference) is a pure-Python
package ``pagecrypt`` whose only native code is a numba kernel
(pkg/src/pagecrypt/_chacha_numba.py).  It cannot be pip-built into
baseline/_ref here usefully and /root/reference does not exist on the GPU
box, so this script snapshots the UNMODIFIED sources

    /root/reference/pkg/src/pagecrypt  ->  oracle/_ref/src/pagecrypt
    /root/reference/pkg/tests          ->  oracle/_ref/tests

so they travel with the repo (oracle/_ref/ is git-ignored, not
gpurun-ignored).  Two consumers:

* bench.py --impl reference times the reference's own CPU path
  (cipher.crypt_page on 1 thread and on one process per core, and
  WorkerPool(cores)) on the GPU box's host cores;
* tests/test_gpu_ref_suite.py runs the reference's own test files unmodified
  with pagecrypt.cipher._chacha_numba bound to the B200 kernel seam.

Files are copied byte-for-byte; a MANIFEST with their sha256 is written so a
stale or edited snapshot is detected (``check()``).
"""

from __future__ import annotations

import hashlib
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")
SRC_ROOT = os.environ.get("PAGECRYPT_REFERENCE", "/root/reference")
TREES = (("pkg/src/pagecrypt", "src/pagecrypt"), ("pkg/tests", "tests"))


def _files(root):
    for d, dirs, fs in os.walk(root):
        dirs[:] = sorted(x for x in dirs if x != "__pycache__")
        for f in sorted(fs):
            if not f.endswith(".pyc"):
                yield os.path.join(d, f)


def _manifest_lines():
    out = []
    for _, dst in TREES:
        base = os.path.join(DEST, dst)
        for p in _files(base):
            with open(p, "rb") as fh:
                out.append(f"{hashlib.sha256(fh.read()).hexdigest()}  {os.path.relpath(p, DEST)}")
    return out


def fetch(src_root: str = SRC_ROOT) -> bool:
    """Snapshot the reference; returns False (and leaves _ref alone) when the
    reference tree is absent (the GPU box)."""
    if not os.path.isdir(os.path.join(src_root, "pkg", "src", "pagecrypt")):
        return False
    for src, dst in TREES:
        d = os.path.join(DEST, dst)
        if os.path.isdir(d):
            shutil.rmtree(d)
        shutil.copytree(os.path.join(src_root, src), d,
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache"))
    with open(os.path.join(DEST, "MANIFEST"), "w") as fh:
        fh.write("\n".join(_manifest_lines()) + "\n")
    return True


def check() -> bool:
    """True when oracle/_ref exists and matches its MANIFEST."""
    m = os.path.join(DEST, "MANIFEST")
    if not os.path.isfile(m):
        return False
    with open(m) as fh:
        want = fh.read().split("\n")
    return [x for x in want if x] == _manifest_lines()


def src_path() -> str:
    return os.path.join(DEST, "src")


if __name__ == "__main__":
    ok = fetch(sys.argv[1] if len(sys.argv) > 1 else SRC_ROOT)
    print("fetched" if ok else "reference absent: oracle/_ref left as is", "| manifest ok:", check())
