"""Pin the CPU oracle (pure-Python, numpy and C restatements) against the
reference's golden vectors before trusting it as the GPU checker.

Sources (tests/golden/make_golden.py regenerates them from the reference):
  chacha_blocks.txt  = /root/reference/pkg/tests/vectors/chacha_blocks.txt
                       (consumed by pkg/tests/test_cipher.py:32-37)
  rfc8439.json       = RFC 8439 §2.3.2 / A.1 blocks via reference_chacha.py:28,
                       plus published ChaCha8/12 zero-key blocks
  ref_pages.npz      = outputs of the reference crypt_page / page_keystream /
                       parallel_crypt_page / chacha20_block / WorkerPool
"""

import json
import os

import numpy as np
import pytest

from oracle import chacha_oracle as O
from oracle import coracle as C


def _vectors(golden_dir):
    for line in open(os.path.join(golden_dir, "chacha_blocks.txt")).read().splitlines():
        key_hex, vaddr_hex, pid, idx, expect = line.split()
        yield bytes.fromhex(key_hex), int(vaddr_hex, 16), int(pid), int(idx), bytes.fromhex(expect)


def test_frozen_vectors_python(golden_dir):
    n = 0
    for key, vaddr, pid, idx, want in _vectors(golden_dir):
        assert O.block(key, vaddr, pid, idx) == want
        n += 1
    assert n == 31


def test_frozen_vectors_c(golden_dir):
    for key, vaddr, pid, idx, want in _vectors(golden_dir):
        assert C.block_raw(key, O.seed_bytes(vaddr, pid, idx)) == want


def test_frozen_vectors_numpy(golden_dir):
    vs = list(_vectors(golden_dir))
    for key, vaddr, pid, idx, want in vs:
        w = O.keystream_words_np(key, [vaddr], [pid], [idx])
        assert w.astype("<u4").tobytes() == want


@pytest.mark.parametrize("impl", ["python", "c"])
def test_rfc8439_and_reduced_rounds(golden_dir, impl):
    vecs = json.load(open(os.path.join(golden_dir, "rfc8439.json")))
    assert {v["rounds"] for v in vecs} == {8, 12, 20}
    for v in vecs:
        key, seed = bytes.fromhex(v["key"]), bytes.fromhex(v["seed16"])
        f = O.block_raw if impl == "python" else C.block_raw
        assert f(key, seed, v["rounds"]).hex() == v["block"], v["name"]


def test_reference_pages_c(ref_pages):
    r = ref_pages
    key = r["key"].tobytes()
    got = C.crypt_pages(key, r["vaddrs"], r["pids"], r["pages"])
    assert np.array_equal(got, r["ct"])
    # involution back to the plaintext
    assert np.array_equal(C.crypt_pages(key, r["vaddrs"], r["pids"], got), r["pages"])
    # multi-threaded partition gives the same bytes
    assert np.array_equal(C.crypt_pages(key, r["vaddrs"], r["pids"], r["pages"], nthreads=5), r["ct"])


def test_reference_pages_numpy(ref_pages):
    r = ref_pages
    got = O.crypt_pages_np(r["key"].tobytes(), r["vaddrs"], r["pids"], r["pages"])
    assert np.array_equal(got, r["ct"])


def test_reference_pages_python_subset(ref_pages):
    r = ref_pages
    key = r["key"].tobytes()
    for i in range(3):  # includes BASE_VADDR/4242, max vaddr/max pid, zero
        got = O.crypt_page(key, int(r["vaddrs"][i]), int(r["pids"][i]), r["pages"][i].tobytes())
        assert got == r["ct"][i].tobytes()


def test_reference_keystream_and_lanes(ref_pages):
    r = ref_pages
    key = r["key"].tobytes()
    for i in range(r["ks"].shape[0]):
        want = r["ks"][i].tobytes()
        zero = np.zeros((1, 4096), np.uint8)
        assert C.crypt_pages(key, r["vaddrs"][i:i + 1], r["pids"][i:i + 1], zero)[0].tobytes() == want
    for lanes in (1, 7, 32, 64):
        assert np.array_equal(r[f"par{lanes}"], r["ct"][:10])
    # lane partition covers every block exactly once (cipher.py:232-242)
    for lanes in (1, 7, 32, 64):
        blocks = sorted(b for lane in range(min(lanes, 32)) for b in O.lane_blocks(lane, lanes))
        assert blocks == list(range(64))


def test_reference_random_blocks(ref_pages):
    r = ref_pages
    for j in range(0, 1000, 7):
        got = O.block(r["blk_keys"][j].tobytes(), int(r["blk_vaddrs"][j]), int(r["blk_pids"][j]),
                      int(r["blk_idx"][j]))
        assert got == r["blk_out"][j].tobytes()
    # all 1000 through the C oracle
    for j in range(1000):
        seed = O.seed_bytes(int(r["blk_vaddrs"][j]), int(r["blk_pids"][j]), int(r["blk_idx"][j]))
        assert C.block_raw(r["blk_keys"][j].tobytes(), seed) == r["blk_out"][j].tobytes()


def test_reference_worker_pool(ref_pages):
    """WorkerPool.crypt seeds with client.pid only (workers.py:137), not epoch."""
    r = ref_pages
    key = r["key"].tobytes()
    got = C.crypt_pages(key, r["vaddrs"][:8], 4242, r["pages"][:8])
    assert np.array_equal(got, r["pool_ct"])


def test_c_oracle_contiguous_and_scalar_forms(ref_pages):
    r = ref_pages
    key = r["key"].tobytes()
    pages = r["pages"][:16]
    va = np.uint64(0x1_0000_0000) + np.arange(16, dtype=np.uint64) * np.uint64(4096)
    a = C.crypt_pages(key, va, 7, pages)
    b = C.crypt_pages(key, None, None, pages, vaddr0=0x1_0000_0000, pid0=7)
    assert np.array_equal(a, b)
    c = O.crypt_pages_np(key, va, 7, pages)
    assert np.array_equal(a, c)
