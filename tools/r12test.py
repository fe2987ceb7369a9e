"""Diagnostic: ChaCha12 kernel time vs SM/memory clocks, power and clock-event
reasons (NVML) over back-to-back launches -- the power-cap study behind
profiles/r01_clock_power_sweep.txt."""
import sys, os, time, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2004_09252_b200 as pc
import pynvml
pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)
def clk():
    return (pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_MEM),
            hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(H)), pynvml.nvmlDeviceGetPowerUsage(H) // 1000,
            pynvml.nvmlDeviceGetTemperature(H, 0))
from paper_2004_09252_b200 import _native
n = 262144
pages = torch.randint(0, 256, (n, 4096), dtype=torch.uint8, device="cuda")
out = torch.empty_like(pages)
key = pc.DeviceKey.generate(0)
def run(r, iters, kern=2):
    _native.tune("kernel", kern)
    for _ in range(3): pc.crypt_pages(key, 0x100000000, 1, pages, out=out, rounds=r, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): pc.crypt_pages(key, 0x100000000, 1, pages, out=out, rounds=r, check=False)
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / iters
t_end = time.time() + 1
while time.time() < t_end: run(20, 5)
for trial in range(3):
    for r in (20, 12, 8):
        for iters in (10, 200):
            for kern in (2, 3, 5):
                ms = run(r, iters, kern)
                print(json.dumps({"r": r, "iters": iters, "kern": kern, "ms": round(ms, 4), "gbs": round(n*4096/ms/1e6), "clk": clk()}))
