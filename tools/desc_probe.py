"""Device-resident 1 GiB: contiguous vaddrs + one pid (the bench) against
per-page descriptor arrays (SURVEY §8d's pid = 1 + i % 64 variant, permuted
vaddrs), 20 back-to-back launches each, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402

n = 262144
pages = torch.randint(0, 256, (n, 4096), dtype=torch.uint8, device="cuda")
out = torch.empty_like(pages)
key = pc.DeviceKey.generate(0)
va_seq = torch.from_numpy((0x100000000 + 4096 * np.arange(n, dtype=np.uint64)).view(np.int64)).cuda()
va_perm = torch.from_numpy((0x100000000 + 4096 * np.random.default_rng(0).permutation(n).astype(np.uint64)).view(np.int64)).cuda()
pids = torch.from_numpy((1 + np.arange(n) % 64).astype(np.int32)).cuda()
pids1 = torch.ones(n, dtype=torch.int32, device="cuda")
cases = {"contiguous, pid 1": (0x100000000, 1), "vaddr array (sequential), pid 1": (va_seq, 1),
         "vaddr array (sequential), pid array of 1s": (va_seq, pids1),
         "vaddr array (sequential), pid = 1 + i % 64": (va_seq, pids),
         "vaddr array (permuted), pid = 1 + i % 64": (va_perm, pids)}
rounds = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else (20, 12, 8)
for r in rounds:
    for name, (v, p) in cases.items():
        for _ in range(3):
            pc.crypt_pages(key, v, p, pages, out=out, rounds=r, check=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            pc.crypt_pages(key, v, p, pages, out=out, rounds=r, check=False)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"ChaCha{r} {name}: {n * 4096 / ms / 1e6:.0f} GB/s")
key.destroy()
