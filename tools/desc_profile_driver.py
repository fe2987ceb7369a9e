"""ncu launcher: the 1 GiB device-resident batch with per-page descriptor
arrays (permuted vaddrs, pid = 1 + i % 64), a few launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n = 262144
pages = torch.randint(0, 256, (n, 4096), dtype=torch.uint8, device="cuda")
out = torch.empty_like(pages)
va = torch.from_numpy((0x100000000 + 4096 * np.random.default_rng(0).permutation(n).astype(np.uint64)).view(np.int64)).cuda()
pids = torch.from_numpy((1 + np.arange(n) % 64).astype(np.int32)).cuda()
with pc.DeviceKey.install(bytes(range(32)), 0) as k:
    for _ in range(3):
        pc.crypt_pages(k, va, pids, pages, out=out, rounds=rounds, check=False)
    torch.cuda.synchronize()
