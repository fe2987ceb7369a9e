"""Golden fault/eviction traces from the REFERENCE orchestrator itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_orchestrator_golden.py

For each window capacity W it drives the unmodified reference stack --
``Orchestrator(ram, pool=WorkerPool(...), window_capacity=W)`` with a
``ClientSpace`` (pkg/src/pagecrypt/orchestrator.py:79-240,
pkg/src/pagecrypt/client.py) and real ChaCha20 through the reference worker
pool -- through a seeded random sequence of reads and writes over a
12-page region, and records:

* the access sequence (page, offset, written bytes or read length);
* the reference's resulting HBM-store equivalent: every stored
  (vaddr, ciphertext) of the client (``orch.store.pages``);
* the window in FIFO order and the fault/eviction/crypto counters;
* every read's result.

``tests/test_orchestrator_golden.py`` replays the same accesses through
``WindowPager`` (oracle cipher on CPU; the HBM store on the GPU) and must
reproduce all of it byte for byte.  Only ``orchestrator_traces.npz`` travels.
"""

from __future__ import annotations

import os
import random
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("PAGECRYPT_REF", "/root/reference/pkg"))
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from pagecrypt.client import BASE_VADDR, ClientSpace  # noqa: E402
from pagecrypt.orchestrator import Orchestrator  # noqa: E402
from pagecrypt.ram import TaggedRam  # noqa: E402
from pagecrypt.workers import WorkerPool  # noqa: E402

KEY = bytes(range(200, 232))
PID = 4242
PAGES = 12
OPS = 400


def run(window: int, seed: int) -> dict:
    rng = random.Random(seed)
    ram = TaggedRam()
    pool = WorkerPool(n_workers=2, keysource=lambda n: KEY, ram=ram)
    orch = Orchestrator(ram, pool=pool, window_capacity=window)
    space = ClientSpace(orch, ram, pid=PID)
    region = space.alloc(PAGES * 4096)
    assert region.base == BASE_VADDR
    ops = []  # (is_write, offset, length, data[8])
    reads = []
    for _ in range(OPS):
        off = rng.randrange(PAGES) * 4096 + rng.randrange(4096 - 8)
        n = rng.randrange(1, 9)
        if rng.random() < 0.6:
            data = bytes(rng.randrange(256) for _ in range(n))
            space.write_region(region, off, data)
            ops.append((1, off, n, data.ljust(8, b"\0")))
        else:
            got = space.read_region(region, off, n)
            reads.append(got.ljust(8, b"\0"))
            ops.append((0, off, n, bytes(8)))
    cid = space.client_id
    stored = sorted(orch.store.pages(cid))
    st = orch._state(cid)
    m = orch.metrics(cid)
    out = {
        "window": window,
        "is_write": np.array([o[0] for o in ops], np.uint8),
        "offset": np.array([o[1] for o in ops], np.int64),
        "length": np.array([o[2] for o in ops], np.int64),
        "data": np.frombuffer(b"".join(o[3] for o in ops), np.uint8).reshape(-1, 8),
        "reads": np.frombuffer(b"".join(reads), np.uint8).reshape(-1, 8),
        "store_vaddrs": np.array([v for v, _ in stored], np.uint64),
        "store_cts": np.stack([np.frombuffer(bytes(c), np.uint8) for _, c in stored]),
        "window_fifo": np.array(list(st.window), np.uint64),
        "metrics": np.array([m.faults, m.first_touch_faults, m.evictions, m.encrypt_ops, m.decrypt_ops], np.int64),
    }
    space.close()
    pool.shutdown()
    return out


def main() -> None:
    arrays = {"key": np.frombuffer(KEY, np.uint8), "pid": np.array(PID), "base": np.array(BASE_VADDR, np.uint64),
              "pages": np.array(PAGES)}
    for i, (w, seed) in enumerate(((1, 11), (4, 12), (8, 13))):
        for k, v in run(w, seed).items():
            arrays[f"t{i}_{k}"] = np.asarray(v)
    np.savez_compressed(OUT / "orchestrator_traces.npz", **arrays)
    print("wrote", OUT / "orchestrator_traces.npz")


if __name__ == "__main__":
    main()
