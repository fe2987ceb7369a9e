"""p50/p99 latency of the reference-API crypt_page for each key/page type
(bytes, MasterKey + bytearray, ndarray, DeviceKey)."""
import time, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2004_09252_b200 as pc
key = bytes(range(32)); page = bytes(4096)
mk = pc.MasterKey(key); ba = bytearray(page); arr = np.zeros(4096, np.uint8)
dk = pc.DeviceKey.install(key, 0)
for name, k, p in (("bytes key, bytes page", key, page), ("MasterKey, bytearray", mk, ba), ("bytes, ndarray", key, arr), ("DeviceKey, bytes", dk, page)):
    for _ in range(200): pc.crypt_page(k, 0x1000, 1, p)
    ts = []
    for _ in range(3000):
        t0 = time.perf_counter_ns(); pc.crypt_page(k, 0x1000, 1, p); ts.append(time.perf_counter_ns() - t0)
    ts.sort(); print(name, "p50 %.2f us p99 %.2f us" % (ts[1500]/1e3, ts[2970]/1e3))
assert pc.crypt_page(mk, 0x1000, 7, page) == pc.crypt_page(dk, 0x1000, 7, ba) == pc.crypt_page(key, 0x1000, 7, arr)
dk.destroy()
