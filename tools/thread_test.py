"""Diagnostic: pc_crypt_pages_host on 1 GiB pinned from the main thread, from a
fresh Python thread and through pc_crypt_pages_multi (the per-engine runner
thread) -- the first-CUDA-call-per-thread cost noted in DESIGN.md §6."""
import sys, os, time, json, threading, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import _native
key = pc.DeviceKey.generate(0)
eng = pc.Engine(0)
n = 262144
a = torch.empty((n, 4096), dtype=torch.uint8).pin_memory()
lib = _native.load()
def run():
    t0 = time.perf_counter()
    rc = lib.pc_crypt_pages_host(eng.handle, key.handle, None, None, None, 0x1000, 1, a.data_ptr(), a.data_ptr(), n, 20)
    return rc, time.perf_counter() - t0
print("main", run(), run())
res = []
th = threading.Thread(target=lambda: res.append((run(), run())))
th.start(); th.join()
print("thread", res)
# multi with one engine
eh = (ctypes.c_void_p * 1)(eng.handle); kh = (ctypes.c_void_p * 1)(key.handle)
for _ in range(2):
    t0 = time.perf_counter()
    rc = lib.pc_crypt_pages_multi(eh, kh, 1, None, None, 0x1000, 1, a.data_ptr(), a.data_ptr(), n, 20)
    print("multi", rc, time.perf_counter() - t0)
