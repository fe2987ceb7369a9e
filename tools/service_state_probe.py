"""Diagnostic: 1-page service latency (bare ctypes pc_service_crypt, p50)
before and after other library/torch state is created in the process."""
import os, sys, time, ctypes
sys.path.insert(0, os.getcwd())
import torch
import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import _native
from paper_2004_09252_b200.workers import ClientId, WorkerPool
def lat(tag):
    pool = WorkerPool(keysource=os.urandom)
    lib = _native.load(); buf = (ctypes.c_char * 4096)(); w = pool.route(ClientId(1, 0))
    for _ in range(200): lib.pc_service_crypt(pool._svc, w, 0x100000000, 1, buf, buf, -1)
    ts = []
    for _ in range(2000):
        t0 = time.perf_counter_ns(); lib.pc_service_crypt(pool._svc, w, 0x100000000, 1, buf, buf, -1); ts.append(time.perf_counter_ns() - t0)
    ts.sort(); print(tag, "p50", ts[1000] / 1e3, "us", "workers", pool.n_workers, flush=True)
    pool.shutdown()
lat("fresh")
key = pc.DeviceKey.generate(0)
pages = torch.randint(0, 256, (262144, 4096), dtype=torch.uint8, device="cuda"); out = torch.empty_like(pages)
for _ in range(40): pc.crypt_pages(key, 0x100000000, 1, pages, out=out, check=False)
torch.cuda.synchronize()
lat("after 1 GiB device loop")
h = torch.empty((262144, 4096), dtype=torch.uint8).pin_memory(); h2 = torch.empty_like(h).pin_memory()
for _ in range(3): pc.crypt_pages(key, 0x100000000, 1, h, out=h2)
lat("after e2e, pinned 2 GiB alive")
del h, h2
lat("after freeing pinned")
time.sleep(2)
lat("after 2 s idle")
