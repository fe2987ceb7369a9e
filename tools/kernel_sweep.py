"""Sweep the crypt kernel's compiled variants on one GPU (CUDA-event timed,
1 GiB device-resident batch) and print one JSON line per (rounds, rotmask).
Used to pick the default ROTMASK; results are committed under profiles/."""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402
from oracle import coracle  # noqa: E402

MASKS = [0x00000000, 0x88888888, 0x888888AA, 0x88888AAA, 0xAAAA8888, 0xAAAAAAAA]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pages", type=int, default=262144)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--rounds", default="8,12,20")
    ap.add_argument("--masks", default=",".join(hex(m) for m in MASKS))
    ap.add_argument("--configs", default="k1:0,k2:0,k3:0",
                    help="kernel:ctas_per_sm list (k1 sweeps --masks)")
    ap.add_argument("--no-intpeak", action="store_true")
    ap.add_argument("--trials", type=int, default=5)
    a = ap.parse_args()
    for kind in ([] if a.no_intpeak else range(8)):
        v = ctypes.c_double()
        _native.call("pc_intpeak", 0, kind, ctypes.byref(v))
        print(json.dumps({"intpeak_kind": kind, "tops": round(v.value / 1e12, 3)}), flush=True)
    n = a.pages
    key = bytes(range(32))
    g = torch.Generator(device="cuda").manual_seed(1)
    pages = torch.randint(0, 256, (n, 4096), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.empty_like(pages)
    sample = np.arange(0, n, 4099)
    host_sample = pages[sample].cpu().numpy()
    runs = []
    for cfg in a.configs.split(","):
        kern, ctas = cfg.split(":")
        if kern == "k1":
            runs += [(1, 0, m) for m in [int(x, 0) for x in a.masks.split(",")]]
        else:
            runs.append((int(kern[1:]), int(ctas), 0))
    results = {}
    with pc.DeviceKey.install(key, 0) as dk:
        # ~1 s of untimed work first so SM clocks leave their idle state
        t_end = time.time() + 1.0
        while time.time() < t_end:
            pc.crypt_pages(dk, 0x1_0000_0000, 1, pages, out=out, rounds=20, check=False)
            torch.cuda.synchronize()
        for r in [int(x) for x in a.rounds.split(",")]:
            want = coracle.crypt_pages(key, 0x1_0000_0000 + 4096 * sample.astype(np.uint64), 1,
                                       host_sample, rounds=r, nthreads=8)
            for trial in range(a.trials):  # interleave configs to spread clock drift
                for kern, ctas, m in runs:
                    _native.tune("kernel", kern)
                    _native.tune("ctas_per_sm", ctas)
                    _native.tune("rotmask", m)
                    for _ in range(3):
                        pc.crypt_pages(dk, 0x1_0000_0000, 1, pages, out=out, rounds=r, check=False)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.iters):
                        pc.crypt_pages(dk, 0x1_0000_0000, 1, pages, out=out, rounds=r, check=False)
                    e1.record()
                    e1.synchronize()
                    ms = e0.elapsed_time(e1) / a.iters
                    ok = np.array_equal(out[sample].cpu().numpy(), want)
                    results.setdefault((r, kern, ctas, m), []).append((ms, ok))
            for (rr, kern, ctas, m), v in results.items():
                if rr != r:
                    continue
                mss = sorted(x[0] for x in v)
                med = mss[len(mss) // 2]
                print(json.dumps({"rounds": r, "kernel": kern, "ctas_per_sm": ctas, "rotmask": hex(m),
                                  "ms_median": round(med, 4), "ms_min": round(mss[0], 4),
                                  "gbs_median": round(n * 4096 / med / 1e6, 1),
                                  "parity": all(x[1] for x in v), "trials": len(v)}), flush=True)


if __name__ == "__main__":
    main()
