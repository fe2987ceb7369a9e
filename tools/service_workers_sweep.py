"""1-page WorkerPool.crypt latency (p50/p99) against the number of resident
workers: every idle worker polls its own doorbell over PCIe, so more
workers load the link the request's own poll crosses."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_09252_b200.workers import ClientId, WorkerPool  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
for w in [int(x) for x in os.environ.get("SWEEP_WORKERS", "1,2,4,8,16,32").split(",")]:
    pool = WorkerPool(n_workers=w, keysource=os.urandom)
    page = bytearray(4096)
    c = ClientId(1, 0)
    for _ in range(200):
        pool.crypt(c, 0x1000, "encrypt", page)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        pool.crypt(c, 0x1000, "encrypt", page)
        ts.append(time.perf_counter_ns() - t0)
    ts.sort()
    print(json.dumps({"workers": w, "p50_us": round(ts[len(ts) // 2] / 1e3, 2),
                      "p99_us": round(ts[int(len(ts) * .99)] / 1e3, 2)}), flush=True)
    pool.shutdown()
