"""Diagnostic: host-resident pinned batches of 1/4/16 GiB, out of place vs in
place, through crypt_pages and crypt_pages_multi (one engine)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2004_09252_b200 as pc
from paper_2004_09252_b200.partition import crypt_pages_multi
key = pc.DeviceKey.generate(0)
eng = pc.Engine(0)
for gib in (1, 4, 16):
    n = gib * 262144
    a = torch.empty((n, 4096), dtype=torch.uint8).pin_memory()
    b = torch.empty_like(a).pin_memory()
    for label, src, dst in (("out-of-place", a, b), ("in-place", a, a)):
        pc.crypt_pages(key, 0x1000, 1, src[:8192], out=dst[:8192], engine=eng)
        t0 = time.perf_counter(); pc.crypt_pages(key, 0x1000, 1, src, out=dst, engine=eng); el = time.perf_counter() - t0
        print(json.dumps({"gib": gib, "mode": label, "api": "crypt_pages", "gbs": round(n * 4096 / el / 1e9, 2)}), flush=True)
    t0 = time.perf_counter(); crypt_pages_multi([key], [eng], 0x1000, 1, a.numpy(), a.numpy()); el = time.perf_counter() - t0
    print(json.dumps({"gib": gib, "mode": "in-place", "api": "crypt_pages_multi", "gbs": round(n * 4096 / el / 1e9, 2)}), flush=True)
    del a, b
