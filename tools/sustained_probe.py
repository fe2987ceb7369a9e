"""Sustained (power-capped) throughput of one round count: back-to-back
1 GiB launches for --seconds, CUDA events over the last half, NVML SM clock
and power sampled.  For A/B of kernels under the 1000 W cap:
    PAGECRYPT_KERNEL=3 python tools/sustained_probe.py --rounds 8"""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    n = 262144
    pages = torch.randint(0, 256, (n, 4096), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(pages)
    key = pc.DeviceKey.generate(0)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
            time.sleep(0.01)

    th = threading.Thread(target=sample)
    th.start()
    t_end = time.time() + a.seconds / 2
    while time.time() < t_end:  # reach the power-capped steady state
        for _ in range(20):
            pc.crypt_pages(key, 0x1000, 1, pages, out=out, rounds=a.rounds, check=False)
        torch.cuda.synchronize()
    samples.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    e0.record()
    t_end = time.time() + a.seconds / 2
    while time.time() < t_end:
        for _ in range(20):
            pc.crypt_pages(key, 0x1000, 1, pages, out=out, rounds=a.rounds, check=False)
        launches += 20
    e1.record()
    e1.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1)
    clk = sorted(s[0] for s in samples)
    pw = sorted(s[1] for s in samples)
    print(json.dumps({"kernel": os.environ.get("PAGECRYPT_KERNEL", "auto"), "rounds": a.rounds,
                      "gbs": round(launches * n * 4096 / (ms / 1e3) / 1e9, 1),
                      "sm_mhz_median": clk[len(clk) // 2], "power_w_median": round(pw[len(pw) // 2], 1)}))
    key.destroy()


if __name__ == "__main__":
    main()
