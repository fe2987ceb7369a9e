"""Single-fault latency of DevicePageStore.fault (pc_store_fault): refault
one page and evict another, launch path (k_slab_swap + stream sync) against
the store's resident worker (pc_store_service), plus the WindowPager
single-fault rate on both.  Prints one JSON line."""
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
key = pc.DeviceKey.generate(0)
c = ClientId(7, 0)
res = {}
for service in (False, True):
    st = DevicePageStore(64, key)
    if service:
        st.start_service()
    out = np.zeros(4096, np.uint8)
    plain = np.random.default_rng(0).integers(0, 256, 4096, dtype=np.uint8)
    a, b = 0x10000, 0x20000
    st.evict(c, a, plain)
    ts = []
    for i in range(reps + 200):
        t0 = time.perf_counter_ns()
        st.fault(c, a, out, b, plain)  # refault a, evict b
        t1 = time.perf_counter_ns()
        a, b = b, a
        if i >= 200:
            ts.append(t1 - t0)
    assert (out == plain).all()
    ts.sort()
    res["service" if service else "launch"] = {"p50_us": round(ts[len(ts) // 2] / 1e3, 2),
                                               "p99_us": round(ts[int(len(ts) * .99)] / 1e3, 2)}
    st.close()
key.destroy()
print(json.dumps({"store_fault_refault_plus_evict": res, "reps": reps}))
