"""Pageable (non-pinned) host batches through crypt_pages: GB/s for the
bounce-copy pool sizes given on the command line (PAGECRYPT_HOST_THREADS is
read when an engine first needs its pool, so each size runs in a fresh
process: python tools/pageable_probe.py 7 -> one JSON line)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402

mib = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
n = (mib << 20) // 4096
src = np.random.default_rng(0).integers(0, 256, size=(n, 4096), dtype=np.uint8)
dst = np.empty_like(src)
key = pc.DeviceKey.generate(0)
eng = pc.Engine(0)
pc.crypt_pages(key, 0x100000000, 1, src, out=dst, engine=eng)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    pc.crypt_pages(key, 0x100000000, 1, src, out=dst, engine=eng)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"what": "crypt_pages pageable", "host_threads": os.environ.get("PAGECRYPT_HOST_THREADS", "default"),
                  "mib": mib, "gbs_mean": round(n * 4096 / (sum(ts) / len(ts)) / 1e9, 2),
                  "gbs_best": round(n * 4096 / min(ts) / 1e9, 2)}))
key.destroy()
