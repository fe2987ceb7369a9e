"""Where does batched evict/refault time go?  pc_store_put/get (index +
transfer) against pc_slab_transfer alone (the same pages and slots, no
index), 65536 pinned pages each way, best of 5."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402
from paper_2004_09252_b200.store import DevicePageStore  # noqa: E402
from paper_2004_09252_b200.workers import ClientId  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
key = pc.DeviceKey.generate(0)
st = DevicePageStore(n, key)
src = torch.randint(0, 256, (n, 4096), dtype=torch.uint8).pin_memory()
dst = torch.empty_like(src).pin_memory()
va = (np.arange(n, dtype=np.uint64) * np.uint64(4096) + np.uint64(0x100000000))
c = ClientId(1, 0)


def best(f, reps=5):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return n * 4096 / min(ts) / 1e9


def evict_refault():
    st.evict_many(c, va, src.numpy())
    st.refault_many(c, va, out=dst.numpy())


ev = best(lambda: (st.evict_many(c, va, src.numpy()), st.refault_many(c, va, out=dst.numpy())))
t_e, t_r = [], []
for _ in range(5):
    t0 = time.perf_counter(); st.evict_many(c, va, src.numpy()); t1 = time.perf_counter()
    st.refault_many(c, va, out=dst.numpy()); t2 = time.perf_counter()
    t_e.append(t1 - t0); t_r.append(t2 - t1)
lib = _native.load()
slab = ctypes.c_void_p()
slots = np.arange(n, dtype=np.uint32)
eng = pc.default_engine(0)
buf = torch.empty((n, 4096), dtype=torch.uint8, device="cuda")


def xfer(direction):
    _native.call("pc_slab_transfer", eng.handle, key.handle, ctypes.c_void_p(buf.data_ptr()), n,
                 slots.ctypes.data, va.ctypes.data, None, 0, 1,
                 (src if direction == 0 else dst).data_ptr(), n, direction, 20, 1 if direction else 0)


te, tr = [], []
for _ in range(5):
    t0 = time.perf_counter(); xfer(0); t1 = time.perf_counter(); xfer(1); t2 = time.perf_counter()
    te.append(t1 - t0); tr.append(t2 - t1)
print(json.dumps({"pages": n, "store_evict_gbs": round(n * 4096 / min(t_e) / 1e9, 2),
                  "store_refault_gbs": round(n * 4096 / min(t_r) / 1e9, 2),
                  "slab_transfer_in_gbs": round(n * 4096 / min(te) / 1e9, 2),
                  "slab_transfer_out_gbs": round(n * 4096 / min(tr) / 1e9, 2)}))
st.close()
key.destroy()
