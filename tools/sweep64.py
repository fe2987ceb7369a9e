"""BASELINE configs[4] on the GPUs available: 64 GiB of pages split by page
range over the local GPUs (here: in-process, one engine per device), device-
resident in place, plus a host-resident pass when enough pinned host memory
is available.  Prints one JSON line."""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200.partition import page_ranges  # noqa: E402

_KEY = bytes(range(100, 132))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=64.0)
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--host-gib", type=float, default=0.0, help="host-resident pass size (0 = skip)")
    ap.add_argument("--verify", action="store_true",
                    help="fill from per-GiB seeded host data and check EVERY byte of the device pass "
                         "against the C oracle (all host cores), one GiB at a time")
    a = ap.parse_args()
    ngpu = torch.cuda.device_count()
    n = int(a.gib * 2**30) // 4096
    ranges = page_ranges(n, ngpu)
    # --verify needs the key on the host for the oracle; the timing pass uses
    # the production device-generated key otherwise
    keys = [pc.DeviceKey.install(_KEY, d) if a.verify else pc.DeviceKey.generate(d) for d in range(ngpu)]
    G1 = 262144  # pages per GiB
    bufs = []

    def chunk_data(c, m):  # deterministic content of global GiB chunk c (writable for torch)
        return np.frombuffer(bytearray(np.random.default_rng(1000 + c).bytes(m * 4096)), np.uint8).reshape(m, 4096)

    for d, (lo, hi) in enumerate(ranges):
        t = torch.empty((hi - lo, 4096), dtype=torch.uint8, device=f"cuda:{d}")
        if a.verify:
            for p0 in range(lo, hi, G1):
                m = min(G1, hi - p0)
                t[p0 - lo:p0 - lo + m].copy_(torch.from_numpy(chunk_data(p0 // G1, m)))
        else:
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
    if a.verify:
        # two passes ran (warm-up + timed): even count -> plaintext; run one more for ciphertext
        for d, t in enumerate(bufs):
            with torch.cuda.device(d):
                lo, _ = ranges[d]
                pc.crypt_pages(keys[d], 0x1_0000_0000 + 4096 * lo, 1, t, out=t, rounds=a.rounds, check=False)
                torch.cuda.synchronize(d)
        from oracle import coracle  # checker only
        from paper_2004_09252_b200.engine import DeviceKey  # noqa: F401
        threads = len(os.sched_getaffinity(0))
        key_bytes = _KEY
        bad = 0
        t0 = time.perf_counter()
        for d, (lo, hi) in enumerate(ranges):
            for p0 in range(lo, hi, G1):
                m = min(G1, hi - p0)
                want = coracle.crypt_pages(key_bytes, None, None, chunk_data(p0 // G1, m), rounds=a.rounds,
                                           vaddr0=0x1_0000_0000 + 4096 * p0, pid0=1, nthreads=threads)
                got = bufs[d][p0 - lo:p0 - lo + m].cpu().numpy()
                bad += int(not np.array_equal(got, want))
        res["verified_gib"] = round(n / G1, 2)
        res["verified_chunks_mismatched"] = bad
        res["verify_s"] = round(time.perf_counter() - t0, 1)
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
