"""Minimal launcher for ncu captures: runs the crypt kernel (or an intpeak
microbenchmark) a few times on a device-resident batch.

    ncu ... python tools/profile_driver.py --rounds 20 --rotmask 0 --pages 262144 --launches 3
    ncu ... python tools/profile_driver.py --intpeak 4
"""

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--rotmask", type=lambda s: int(s, 0), default=None)
    ap.add_argument("--pages", type=int, default=262144)
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--intpeak", type=int, default=None)
    ap.add_argument("--desc", action="store_true",
                    help="per-page descriptor arrays: permuted vaddrs, pid = 1 + i % 64 (bench extras.desc)")
    a = ap.parse_args()
    if a.intpeak is not None:
        v = ctypes.c_double()
        _native.call("pc_intpeak", 0, a.intpeak, ctypes.byref(v))
        print(f"intpeak {a.intpeak}: {v.value / 1e12:.3f} Tops")
        return
    if a.rotmask is not None:
        _native.tune("rotmask", a.rotmask)
    pages = torch.randint(0, 256, (a.pages, 4096), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(pages)
    with pc.DeviceKey.install(bytes(range(32)), 0) as k:
        va, pid = 0x1_0000_0000, 1
        if a.desc:
            import numpy as np
            n = a.pages
            perm = np.random.default_rng(0).permutation(n).astype(np.uint64)
            va = torch.from_numpy((0x1_0000_0000 + 4096 * perm).view(np.int64)).cuda()
            pid = torch.from_numpy((1 + np.arange(n) % 64).astype(np.int32)).cuda()
        for _ in range(a.launches):
            pc.crypt_pages(k, va, pid, pages, out=out, rounds=a.rounds, check=False)
        torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
