"""BASELINE configs[4] on the GPUs available: 64 GiB of pages split by page
range over the local GPUs (here: in-process, one engine per device), device-
resident in place, plus a host-resident pass when enough pinned host memory
is available.  Prints one JSON line."""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200.partition import page_ranges  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=64.0)
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--host-gib", type=float, default=0.0, help="host-resident pass size (0 = skip)")
    a = ap.parse_args()
    ngpu = torch.cuda.device_count()
    n = int(a.gib * 2**30) // 4096
    ranges = page_ranges(n, ngpu)
    keys = [pc.DeviceKey.generate(d) for d in range(ngpu)]
    bufs = []
    for d, (lo, hi) in enumerate(ranges):
        t = torch.empty((hi - lo, 4096), dtype=torch.uint8, device=f"cuda:{d}")
        t.view(torch.int64).random_()
        bufs.append(t)
    for d in range(ngpu):
        torch.cuda.synchronize(d)
    res = {"config": f"{a.gib:g} GiB device-resident in place, ChaCha{a.rounds}, {ngpu} GPU(s)", "pages": n}
    # warm-up + timed pass (events per device, max over devices)
    for _ in range(2):
        evs = []
        for d, t in enumerate(bufs):
            with torch.cuda.device(d):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                lo, _ = ranges[d]
                pc.crypt_pages(keys[d], 0x1_0000_0000 + 4096 * lo, 1, t, out=t, rounds=a.rounds, check=False)
                e1.record()
                evs.append((e0, e1))
        ms = max(e0.elapsed_time(e1) for e0, e1 in (ev for ev in evs if not ev[1].synchronize()))
    res["device_ms"] = round(ms, 2)
    res["device_gbs"] = round(n * 4096 / ms / 1e6, 1)
    # property check: crypt again restores a sample
    first = bufs[0][:4].clone()
    with torch.cuda.device(0):
        pc.crypt_pages(keys[0], 0x1_0000_0000, 1, bufs[0][:4], out=bufs[0][:4], rounds=a.rounds)
        pc.crypt_pages(keys[0], 0x1_0000_0000, 1, bufs[0][:4], out=bufs[0][:4], rounds=a.rounds)
        torch.cuda.synchronize()
    res["involution_ok"] = bool(torch.equal(first, bufs[0][:4]))
    del bufs
    torch.cuda.empty_cache()
    if a.host_gib > 0:
        m = int(a.host_gib * 2**30) // 4096
        host = torch.empty((m, 4096), dtype=torch.uint8).pin_memory()
        engines = [pc.Engine(d) for d in range(ngpu)]
        from paper_2004_09252_b200.partition import crypt_pages_multi
        crypt_pages_multi(keys, engines, 0x1_0000_0000, 1, host.numpy()[:8192], host.numpy()[:8192])
        t0 = time.perf_counter()
        crypt_pages_multi(keys, engines, 0x1_0000_0000, 1, host.numpy(), host.numpy(), rounds=a.rounds)
        el = time.perf_counter() - t0
        res["host_gib"] = a.host_gib
        res["host_gbs"] = round(m * 4096 / el / 1e9, 2)
        for e in engines:
            e.destroy()
    for k in keys:
        k.destroy()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
