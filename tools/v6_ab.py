"""A/B of the page kernels (knob "kernel") on the 1 GiB batch: contiguous
descriptors and per-page arrays (permuted vaddrs, pid = 1 + i % 64), CUDA
events over 10 launches after warm-up and a 0.5 s cool-down, alternating the variants 3 times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402

n = 262144
kernels = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "5,6").split(",")]
ctas = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
pages = torch.randint(0, 256, (n, 4096), dtype=torch.uint8, device="cuda")
out = torch.empty_like(pages)
key = pc.DeviceKey.generate(0)
va = torch.from_numpy((0x100000000 + 4096 * np.random.default_rng(0).permutation(n).astype(np.uint64)).view(np.int64)).cuda()
pids = torch.from_numpy((1 + np.arange(n) % 64).astype(np.int32)).cuda()
cases = {"contig": (0x100000000, 1), "desc": (va, pids)}
res = {}
for rep in range(3):
    for r in (20, 12):
        for cname, (v, p) in cases.items():
            for kern in kernels:
                for c in ctas:
                    _native.tune("kernel", kern)
                    _native.tune("ctas_per_sm", c)
                    for _ in range(3):
                        pc.crypt_pages(key, v, p, pages, out=out, rounds=r, check=False)
                    torch.cuda.synchronize()
                    time.sleep(0.5)  # cool down: short bursts stay below the power cap
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(10):
                        pc.crypt_pages(key, v, p, pages, out=out, rounds=r, check=False)
                    e1.record()
                    e1.synchronize()
                    ms = e0.elapsed_time(e1) / 10
                    res.setdefault((r, cname, kern, c), []).append(n * 4096 / ms / 1e6)
for (r, cname, kern, c), v in sorted(res.items()):
    print(f"ChaCha{r} {cname:6s} kernel {kern} ctas/SM {c or 'auto'}: " + " ".join(f"{x:.0f}" for x in v) + f"  best {max(v):.0f} GB/s")
key.destroy()
