"""Latency of the reference-facing keystream seams (one page = 64 blocks):
_chacha_cuda.keystream_words (the numba kernel's drop-in), chacha20_block and
page_keystream, p50/p99 over 3000 calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _chacha_cuda  # noqa: E402

kw = np.frombuffer(bytes(range(32)), dtype="<u4").copy()
idx = np.arange(64, dtype=np.int64)
out = np.empty(1024, np.uint32)
seed = pc.BlockSeed(0x1000, 7, 3)
cases = {
    "keystream_words (64 blocks)": lambda: _chacha_cuda.keystream_words(kw, np.uint64(0x1000), np.uint32(7), idx, out),
    "chacha20_block": lambda: pc.chacha20_block(bytes(range(32)), seed),
    "page_keystream": lambda: pc.page_keystream(bytes(range(32)), 0x1000, 7),
}
for name, f in cases.items():
    for _ in range(300):
        f()
    ts = []
    for _ in range(3000):
        t0 = time.perf_counter_ns()
        f()
        ts.append(time.perf_counter_ns() - t0)
    ts.sort()
    print(f"{name}: p50 {ts[1500] / 1e3:.2f} us, p99 {ts[2970] / 1e3:.2f} us")
