"""Regenerate the golden fixtures from the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the unmodified reference ``pagecrypt`` (numba kernel path,
``/root/reference/pkg/src/pagecrypt/cipher.py``) and its independent test
oracle (``/root/reference/pkg/tests/reference_chacha.py``) and writes:

* ``chacha_blocks.txt`` -- the reference's 31 frozen block vectors
  (``pkg/tests/vectors/chacha_blocks.txt``), each line re-derived through the
  reference ``chacha20_block`` and asserted equal before it is written;
* ``rfc8439.json`` -- RFC 8439 §2.3.2 and A.1 #1-#5 blocks (raw 16-byte
  counter||nonce seeds, which ``BlockSeed`` cannot express), computed with the
  reference's ``chacha20_block_ref`` and checked against the RFC's published
  bytes; plus the published ChaCha8/ChaCha12 zero-key/zero-IV blocks (the
  reference has no round knob, so these pin only our rounds parameter);
* ``ref_pages.npz`` -- config 1 of BASELINE.json: 64 random 4 KiB pages and
  their ciphertexts from the reference ``crypt_page``; the page keystreams and
  ``parallel_crypt_page`` outputs for lanes {1, 7, 32, 64}; 1000 random
  (key, vaddr, pid, idx) blocks from ``chacha20_block`` (SPEC.md:577 asks for
  1000); a WorkerPool round (``pkg/src/pagecrypt/workers.py:227``) for
  8 pages.

Nothing on the GPU box reads /root/reference; only these files travel.
"""

from __future__ import annotations

import json
import os
import random
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("PAGECRYPT_REF", "/root/reference/pkg"))
OUT = Path(__file__).resolve().parent

sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from pagecrypt import cipher  # noqa: E402  (the reference package)
from pagecrypt.ram import TaggedRam, TAG_SERVER_MISC  # noqa: E402
from pagecrypt.store import ClientId  # noqa: E402
from pagecrypt.workers import WorkerPool  # noqa: E402
from reference_chacha import chacha20_block_ref  # noqa: E402

assert cipher._chacha_numba is not None, "reference numba kernel not importable"


def seed(counter: int, nonce_hex: str) -> bytes:
    return counter.to_bytes(4, "little") + bytes.fromhex(nonce_hex)


# RFC 8439 (published bytes).  Full blocks where the RFC text is reproduced in
# full here, otherwise the first 16 bytes (the survey's check).
RFC = [
    ("rfc8439_2.3.2", bytes(range(32)), seed(1, "000000090000004a00000000"), 20,
     "10f1e7e4d13b5915500fdd1fa32071c4c7d1f4c733c068030422aa9ac3d46c4e"
     "d2826446079faa0914c2d705d98b02a2b5129cd1de164eb9cbd083e8a2503c4e"),
    ("rfc8439_A.1.1", bytes(32), seed(0, "00" * 12), 20,
     "76b8e0ada0f13d90405d6ae55386bd28bdd219b8a08ded1aa836efcc8b770dc7"
     "da41597c5157488d7724e03fb8d84a376a43b8f41518a11cc387b669b2ee6586"),
    ("rfc8439_A.1.2", bytes(32), seed(1, "00" * 12), 20, "9f07e7be5551387a98ba977c732d080d"),
    ("rfc8439_A.1.3", bytes(31) + b"\x01", seed(1, "00" * 12), 20, "3aeb5224ecf849929b9d828db1ced4dd"),
    ("rfc8439_A.1.4", b"\x00\xff" + bytes(30), seed(2, "00" * 12), 20, "72d54dfbf12ec44b362692df94137f32"),
    ("rfc8439_A.1.5", bytes(32), seed(0, "00" * 11 + "02"), 20, "c2c64d378cd536374ae204b9ef933fcd"),
]
# Published reduced-round zero-key / zero-IV blocks (first keystream block).
REDUCED = [
    ("chacha8_zero", 8,
     "3e00ef2f895f40d67f5bb8e81f09a5a12c840ec3ce9a7f3b181be188ef711a1e"
     "984ce172b9216f419f445367456d5619314a42a3da86b001387bfdb80e0cfe42"),
    ("chacha12_zero", 12,
     "9bf49a6a0755f953811fce125f2683d50429c3bb49e074147e0089a52eae155f"
     "0564f879d27ae3c02ce82834acfa8c793a629f2ca0de6919610be82f411326be"),
]


def main() -> None:
    # 1. frozen block vectors, re-derived through the reference API
    lines = (REF / "tests" / "vectors" / "chacha_blocks.txt").read_text().splitlines()
    for line in lines:
        key_hex, vaddr_hex, pid, idx, expect = line.split()
        got = cipher.chacha20_block(bytes.fromhex(key_hex),
                                    cipher.BlockSeed(int(vaddr_hex, 16), int(pid), int(idx)))
        assert got.hex() == expect, line
    (OUT / "chacha_blocks.txt").write_text("\n".join(lines) + "\n")

    # 2. RFC 8439 raw-seed blocks via the reference's own oracle
    rfc = []
    for name, key, s16, rounds, published in RFC:
        full = chacha20_block_ref(key, s16).hex()
        assert full.startswith(published), (name, full)
        rfc.append({"name": name, "key": key.hex(), "seed16": s16.hex(), "rounds": rounds,
                    "block": full})
    for name, rounds, published in REDUCED:
        rfc.append({"name": name, "key": "00" * 32, "seed16": "00" * 16, "rounds": rounds,
                    "block": published})
    (OUT / "rfc8439.json").write_text(json.dumps(rfc, indent=1) + "\n")

    # 3. config 1: 64 random pages, reference crypt_page
    rng = np.random.default_rng(2004_09252)
    key = rng.bytes(32)
    n = 64
    pages = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
    vaddrs = (rng.integers(0, 2**52, size=n, dtype=np.uint64) * np.uint64(4096)).astype(np.uint64)
    vaddrs[0] = 0x1_0000_0000  # BASE_VADDR, pkg/src/pagecrypt/client.py:42
    vaddrs[1] = 0xFFFF_FFFF_FFFF_F000  # max page-aligned u64
    vaddrs[2] = 0
    pids = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    pids[0] = 4242
    pids[1] = 0xFFFFFFFF
    pids[2] = 0
    ct = np.stack([np.frombuffer(cipher.crypt_page(key, int(v), int(p), pg.tobytes()), np.uint8)
                   for v, p, pg in zip(vaddrs, pids, pages)])
    ks = np.stack([np.frombuffer(cipher.page_keystream(key, int(v), int(p)), np.uint8)
                   for v, p in zip(vaddrs[:8], pids[:8])])
    par = {}
    for lanes in (1, 7, 32, 64):
        par[lanes] = np.stack([
            np.frombuffer(cipher.parallel_crypt_page(key, int(v), int(p), pg.tobytes(), lanes), np.uint8)
            for v, p, pg in zip(vaddrs[:10], pids[:10], pages[:10])])
        assert np.array_equal(par[lanes], ct[:10])

    # 4. 1000 random blocks through chacha20_block
    r = random.Random(577)
    bkeys, bv, bp, bi, bout = [], [], [], [], []
    for _ in range(1000):
        k = bytes(r.randrange(256) for _ in range(32))
        v = r.randrange(2**52) * 4096
        p = r.randrange(2**32)
        i = r.randrange(64)
        bkeys.append(np.frombuffer(k, np.uint8))
        bv.append(v); bp.append(p); bi.append(i)
        bout.append(np.frombuffer(cipher.chacha20_block(k, cipher.BlockSeed(v, p, i)), np.uint8))

    # 5. WorkerPool (the fault-path API) over 8 pages, client pid 4242 epoch 3
    ram = TaggedRam()
    pool = WorkerPool(n_workers=2, keysource=lambda m: key, ram=ram)
    client = ClientId(4242, 3)
    pool_ct = []
    for v, pg in zip(vaddrs[:8], pages[:8]):
        buf = ram.alloc(TAG_SERVER_MISC, 4096)
        buf.data[:] = pg.tobytes()
        pool.crypt(client, int(v), "encrypt", buf)
        pool_ct.append(np.frombuffer(bytes(buf.data), np.uint8))
        ram.free(buf)
    pool.shutdown()

    np.savez(
        OUT / "ref_pages.npz",
        key=np.frombuffer(key, np.uint8), pages=pages, vaddrs=vaddrs, pids=pids, ct=ct,
        ks=ks, par1=par[1], par7=par[7], par32=par[32], par64=par[64],
        blk_keys=np.stack(bkeys), blk_vaddrs=np.array(bv, np.uint64),
        blk_pids=np.array(bp, np.uint32), blk_idx=np.array(bi, np.uint32),
        blk_out=np.stack(bout), pool_ct=np.stack(pool_ct),
    )
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
