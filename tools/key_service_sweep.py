import sys, time, json, os
sys.path.insert(0, os.getcwd())
import torch, paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import _native
dk = pc.DeviceKey.generate(0)
res = {}
for W in (0, 8, 16, 32):
    if W:
        dk.start_service(n_workers=W)
        _native.tune("svc_pages", 64)
    row = {}
    for n in (1, 2, 4, 8, 16, 32, 64):
        src = torch.randint(0, 256, (n, 4096), dtype=torch.uint8).pin_memory()
        dst = torch.empty_like(src).pin_memory()
        for _ in range(200):
            pc.crypt_pages(dk, 0x1000, 1, src, out=dst)
        ts = []
        for _ in range(1000):
            t0 = time.perf_counter_ns(); pc.crypt_pages(dk, 0x1000, 1, src, out=dst); ts.append(time.perf_counter_ns() - t0)
        ts.sort()
        row[n] = round(ts[500] / 1e3, 2)
    res[W] = row
    if W:
        dk.stop_service()
print(json.dumps(res))
