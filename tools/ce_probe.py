"""Copy-engine probe: do more concurrent H2D / D2H streams raise PCIe throughput
(alone and bidirectional)?  1 GiB each way, mean/best of 8."""
import torch, time
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
def timed(fn, reps=8):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        t0=time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    return n/(sum(ts)/len(ts))/1e9, n/min(ts)/1e9
for k in (1, 2, 4):
    hs = [torch.cuda.Stream() for _ in range(k)]; ds = [torch.cuda.Stream() for _ in range(k)]
    def both():
        part = n // k
        for i in range(k):
            with torch.cuda.stream(hs[i]): d[i*part:(i+1)*part].copy_(h_in[i*part:(i+1)*part], non_blocking=True)
            with torch.cuda.stream(ds[i]): h_out[i*part:(i+1)*part].copy_(d2[i*part:(i+1)*part], non_blocking=True)
    m, b = timed(both)
    print(f"{k} H2D + {k} D2H streams, 1 GiB each way: mean {m:.2f} best {b:.2f} GB/s per direction")
    def h2d():
        part = n // k
        for i in range(k):
            with torch.cuda.stream(hs[i]): d[i*part:(i+1)*part].copy_(h_in[i*part:(i+1)*part], non_blocking=True)
    m, b = timed(h2d)
    print(f"{k} H2D streams alone: mean {m:.2f} best {b:.2f}")
