"""1-page host-resident latency: crypt_pages (Python API, torch pinned
tensors) against the same pc_crypt_pages_host call made directly through
ctypes, p50/p99 over 3000 calls each, interleaved."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402

key = pc.DeviceKey.generate(0)
eng = pc.default_engine(0)
lib = _native.load()
for n in (1, 64):
    src = torch.randint(0, 256, (n, 4096), dtype=torch.uint8).pin_memory()
    dst = torch.empty_like(src).pin_memory()
    a, b = src.data_ptr(), dst.data_ptr()
    fns = {"crypt_pages": lambda: pc.crypt_pages(key, 0x100000000, 1, src, out=dst),
           "ctypes pc_crypt_pages_host": lambda: lib.pc_crypt_pages_host(eng.handle, key.handle, None, None, None,
                                                                         0x100000000, 1, a, b, n, 20)}
    ts = {k: [] for k in fns}
    for _ in range(300):
        for f in fns.values():
            f()
    for _ in range(3000):
        for k, f in fns.items():
            t0 = time.perf_counter_ns()
            f()
            ts[k].append(time.perf_counter_ns() - t0)
    for k, v in ts.items():
        v.sort()
        print(f"{n} page(s) {k}: p50 {v[1500] / 1e3:.2f} us p99 {v[2970] / 1e3:.2f} us")
key.destroy()
