"""Host-resident path measurements: raw PCIe copy rates (H2D, D2H, both at
once) and pc_crypt_pages_host over engine (streams, chunk) configurations,
plus the small-batch latency path in both modes.  One JSON line per result."""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--configs", default="2:1024,3:1024,4:2048,4:4096,6:2048,8:1024,8:4096,4:8192")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    nbytes = a.mib << 20
    n = nbytes // 4096
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_in.random_()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=a.reps):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    t = timed(lambda: d.copy_(h_in, non_blocking=True))
    print(json.dumps({"what": "h2d_pinned", "gbs": round(nbytes / t / 1e9, 2)}), flush=True)
    t = timed(lambda: h_out.copy_(d, non_blocking=True))
    print(json.dumps({"what": "d2h_pinned", "gbs": round(nbytes / t / 1e9, 2)}), flush=True)

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d2, non_blocking=True)
    t = timed(both)
    print(json.dumps({"what": "h2d+d2h_concurrent", "gbs_each_dir": round(nbytes / t / 1e9, 2)}), flush=True)

    key = pc.DeviceKey.generate(0)
    for hm in (1, 0, 2):
        _native.tune("host_mode", hm)
        for cfg in (a.configs.split(",") if hm != 1 else ["4:2048"]):
            ns, chunk = (int(x) for x in cfg.split(":"))
            eng = pc.Engine(0, n_streams=ns, chunk_pages=chunk)
            for rounds in ((20, 8) if hm == 1 else (20,)):
                t = timed(lambda: pc.crypt_pages(key, 0x1_0000_0000, 1, h_in, out=h_out, engine=eng,
                                                 rounds=rounds))
                print(json.dumps({"what": "crypt_pages_host_pinned", "host_mode": hm, "streams": ns,
                                  "chunk_pages": chunk, "rounds": rounds,
                                  "gbs": round(nbytes / t / 1e9, 2)}), flush=True)
            eng.destroy()
    _native.tune("host_mode", 2)
    # pageable source/destination (bounce buffers)
    import numpy as np
    p_in = np.random.default_rng(0).integers(0, 256, size=(n // 4, 4096), dtype=np.uint8)
    p_out = np.empty_like(p_in)
    eng = pc.Engine(0, n_streams=4, chunk_pages=2048)
    t = timed(lambda: pc.crypt_pages(key, 0x1_0000_0000, 1, p_in, out=p_out, engine=eng))
    print(json.dumps({"what": "crypt_pages_host_pageable", "mib": a.mib // 4,
                      "gbs": round(p_in.nbytes / t / 1e9, 2)}), flush=True)
    eng.destroy()
    # small batches, both modes
    for mode in (0, 1):
        _native.tune("small_mode", mode)
        for npg in (1, 4, 16, 64):
            src = torch.randint(0, 256, (npg, 4096), dtype=torch.uint8).pin_memory()
            dst = torch.empty_like(src).pin_memory()
            for _ in range(50):
                pc.crypt_pages(key, 0x1_0000_0000, 1, src, out=dst)
            ts = []
            for _ in range(2000):
                t0 = time.perf_counter_ns()
                pc.crypt_pages(key, 0x1_0000_0000, 1, src, out=dst)
                ts.append(time.perf_counter_ns() - t0)
            ts.sort()
            print(json.dumps({"what": "small_batch", "small_mode": mode, "pages": npg,
                              "p50_us": ts[len(ts) // 2] / 1e3, "p99_us": ts[int(len(ts) * .99)] / 1e3}),
                  flush=True)
        # the raw-key crypt_page API (reference signature), pageable bytes
        page = bytes(4096)
        kb = bytes(range(32))
        for _ in range(50):
            pc.crypt_page(kb, 0x1000, 1, page)
        ts = []
        for _ in range(2000):
            t0 = time.perf_counter_ns()
            pc.crypt_page(kb, 0x1000, 1, page)
            ts.append(time.perf_counter_ns() - t0)
        ts.sort()
        print(json.dumps({"what": "crypt_page_rawkey_bytes", "small_mode": mode,
                          "p50_us": ts[len(ts) // 2] / 1e3, "p99_us": ts[int(len(ts) * .99)] / 1e3}), flush=True)
    key.destroy()


if __name__ == "__main__":
    main()
