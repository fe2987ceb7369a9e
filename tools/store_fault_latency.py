"""Single-fault latency of DevicePageStore.fault (pc_store_fault), launch
path (k_slab_swap + stream sync) against the store's resident worker
(pc_store_service), for the three shapes a fault takes: refault + eviction
(window full), refault only, eviction only (first touch, window full).
Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200.store import DevicePageStore  # noqa: E402
from paper_2004_09252_b200.workers import ClientId  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000


def pct(ts):
    ts.sort()
    return {"p50_us": round(ts[len(ts) // 2] / 1e3, 2), "p99_us": round(ts[int(len(ts) * .99)] / 1e3, 2)}


key = pc.DeviceKey.generate(0)
c = ClientId(7, 0)
plain = np.random.default_rng(0).integers(0, 256, 4096, dtype=np.uint8)
res = {}
for service in (False, True):
    st = DevicePageStore(64, key)
    if service:
        st.start_service()
    out = np.zeros(4096, np.uint8)
    r = {}
    # refault a, evict b (then the other way round)
    a, b = 0x10000, 0x20000
    st.evict(c, a, plain)
    ts = []
    for i in range(reps + 200):
        t0 = time.perf_counter_ns()
        st.fault(c, a, out, b, plain)
        t1 = time.perf_counter_ns()
        a, b = b, a
        if i >= 200:
            ts.append(t1 - t0)
    assert (out == plain).all()
    r["refault+evict"] = pct(ts)
    st.refault(c, a)
    # eviction only (a first touch), then refault only, alternating
    te, tr = [], []
    for i in range(reps + 200):
        t0 = time.perf_counter_ns()
        st.fault(c, 0x30000, out, 0x40000, plain)  # first touch of 0x30000, evict 0x40000
        t1 = time.perf_counter_ns()
        st.fault(c, 0x40000, out)                  # refault 0x40000, nothing evicted
        t2 = time.perf_counter_ns()
        if i >= 200:
            te.append(t1 - t0)
            tr.append(t2 - t1)
    assert (out == plain).all()
    r["evict_only"] = pct(te)
    r["refault_only"] = pct(tr)
    res["service" if service else "launch"] = r
    st.close()
key.destroy()
print(json.dumps({"store_fault": res, "reps": reps}))
