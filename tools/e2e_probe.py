"""Host-resident end-to-end probe (BASELINE configs[1] through the host API):
where does the gap between the pipeline and the concurrent-copy PCIe rate go?

Prints one JSON line per measurement: raw copies (whole and chunked, one or
both directions), then pc_crypt_pages_host in host_mode 2 (H2D / kernel /
D2H on dedicated streams) and host_mode 3 (the kernel writes the pinned
output itself) over (streams, chunk) configurations.  Mean and best of
--reps host-timed steps, like bench.py's e2e leg."""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--configs", default="4:8192,3:8192,4:16384,6:8192,8:4096,4:32768,6:16384")
    ap.add_argument("--modes", default="2,3")
    a = ap.parse_args()
    nbytes = a.mib << 20
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_in.random_()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return nbytes / (sum(ts) / len(ts)) / 1e9, nbytes / min(ts) / 1e9

    def emit(**kw):
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in kw.items()}), flush=True)

    m, b = timed(lambda: d.copy_(h_in, non_blocking=True))
    emit(what="h2d", mean_gbs=m, best_gbs=b)
    m, b = timed(lambda: h_out.copy_(d, non_blocking=True))
    emit(what="d2h", mean_gbs=m, best_gbs=b)

    def both(chunk):
        def run():
            cb = chunk * 4096
            for off in range(0, nbytes, cb):
                with torch.cuda.stream(s1):
                    d[off:off + cb].copy_(h_in[off:off + cb], non_blocking=True)
                with torch.cuda.stream(s2):
                    h_out[off:off + cb].copy_(d2[off:off + cb], non_blocking=True)
        return run

    for chunk in (nbytes // 4096, 32768, 8192, 2048):
        m, b = timed(both(chunk))
        emit(what="h2d+d2h concurrent", chunk_pages=chunk, mean_gbs_each=m, best_gbs_each=b)

    key = pc.DeviceKey.generate(0)
    ref = None
    for hm in (int(x) for x in a.modes.split(",")):
        _native.tune("host_mode", hm)
        for cfg in a.configs.split(","):
            ns, chunk = (int(x) for x in cfg.split(":"))
            eng = pc.Engine(0, n_streams=ns, chunk_pages=chunk)
            m, b = timed(lambda: pc.crypt_pages(key, 0x1_0000_0000, 1, h_in, out=h_out, engine=eng))
            if ref is None:
                ref = h_out.clone()
                same = True
            else:
                same = bool(torch.equal(ref, h_out))
            emit(what="crypt_pages_host", host_mode=hm, streams=ns, chunk_pages=chunk, mean_gbs=m,
                 best_gbs=b, identical=same)
            eng.destroy()
    _native.tune("host_mode", 2)
    key.destroy()


if __name__ == "__main__":
    main()
