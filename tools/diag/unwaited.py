import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2004_09252_b200.workers import WorkerPool, ClientId
from paper_2004_09252_b200.errors import PoolError
from oracle import chacha_oracle as O
KEY = bytes(range(32))
class Page:
    def __init__(self): self.data = bytearray(4096)
for trial in range(3):
    pool = WorkerPool(n_workers=2, keysource=lambda n: KEY)
    pages = [Page() for _ in range(10)]
    comps = [pool.submit(ClientId(9, 0), 4096 * i, "encrypt", p) for i, p in enumerate(pages)]
    while True:
        try:
            pool.shutdown(); break
        except PoolError:
            time.sleep(0.01)
    for i, p in enumerate(pages):
        want = O.crypt_page(KEY, 4096 * i, 9, bytes(4096))
        got = bytes(p.data)
        if got != want:
            bad = [b for b in range(64) if got[64*b:64*b+64] != want[64*b:64*b+64]]
            # which ticket's keystream is it?
            who = [j for j in range(10) if got[:64] == O.crypt_page(KEY, 4096 * j, 9, bytes(4096))[:64]]
            print(f"trial {trial} page {i}: bad blocks {bad[:8]}{'...' if len(bad)>8 else ''} ({len(bad)}) block0 matches ticket {who}; zero? {got[:16] == bytes(16)}")
    print("trial", trial, "done")
