"""GPU parity of the drop-in cipher API against the reference's golden
vectors and the oracle.  Restates pkg/tests/test_cipher.py test by test (the
reference's own cipher suite), with the SPEC.md:577-578 counts (1000 random
blocks, 1000 involution pages, 100 pages per lane count) where the reference
tests used fewer."""

import json
import os
import random

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import _chacha_cuda, cipher
from paper_2004_09252_b200.errors import ContractViolation

from oracle import chacha_oracle as O
from oracle import coracle as C

pytestmark = pytest.mark.gpu


def rand_key(rng):
    return bytes(rng.randrange(256) for _ in range(32))


def rand_page(rng):
    return rng.randbytes(4096)


class TestBlock:
    def test_frozen_vectors(self, golden_dir, cuda):
        lines = open(os.path.join(golden_dir, "chacha_blocks.txt")).read().splitlines()
        assert len(lines) == 31
        for line in lines:
            key_hex, vaddr_hex, pid, idx, expect = line.split()
            got = pc.chacha20_block(bytes.fromhex(key_hex), pc.BlockSeed(int(vaddr_hex, 16), int(pid), int(idx)))
            assert got.hex() == expect

    def test_rfc8439_raw_seeds(self, golden_dir, cuda):
        for v in json.load(open(os.path.join(golden_dir, "rfc8439.json"))):
            got = pc.keystream_raw(bytes.fromhex(v["key"]), bytes.fromhex(v["seed16"]), rounds=v["rounds"])
            assert got.hex() == v["block"], v["name"]

    def test_raw_seed_batch(self, cuda):
        rng = random.Random(11)
        key = rand_key(rng)
        seeds = b"".join(rng.randbytes(16) for _ in range(300))
        got = pc.keystream_raw(key, seeds, rounds=12)
        want = b"".join(O.block_raw(key, seeds[16 * i:16 * i + 16], 12) for i in range(300))
        assert got == want

    def test_zero_input_block_matches_oracle(self, cuda):
        got = pc.chacha20_block(b"\x00" * 32, pc.BlockSeed(0, 0, 0))
        assert got == O.block(b"\x00" * 32, 0, 0, 0)

    def test_against_reference_random_1000(self, ref_pages, cuda):
        r = ref_pages
        for j in range(1000):
            seed = pc.BlockSeed(int(r["blk_vaddrs"][j]), int(r["blk_pids"][j]), int(r["blk_idx"][j]))
            assert pc.chacha20_block(r["blk_keys"][j].tobytes(), seed) == r["blk_out"][j].tobytes()

    def test_deterministic_and_index_sensitive(self, cuda):
        seed = pc.BlockSeed(0x7000, 9, 3)
        assert pc.chacha20_block(b"\x42" * 32, seed) == pc.chacha20_block(b"\x42" * 32, seed)
        a = pc.chacha20_block(b"\x00" * 32, pc.BlockSeed(0, 0, 0))
        b = pc.chacha20_block(b"\x00" * 32, pc.BlockSeed(0, 0, 1))
        assert a != b

    @pytest.mark.parametrize("rounds", [8, 12, 20])
    def test_rounds_vs_oracle(self, rounds, cuda):
        rng = random.Random(rounds)
        for _ in range(50):
            key, v, p, i = rand_key(rng), rng.randrange(2**52) * 4096, rng.randrange(2**32), rng.randrange(64)
            assert pc.chacha20_block(key, pc.BlockSeed(v, p, i), rounds=rounds) == O.block(key, v, p, i, rounds)


class TestPageKeystream:
    def test_first_block_is_block_zero(self, cuda):
        key = b"\x05" * 32
        assert pc.page_keystream(key, 0x4000, 11)[:64] == pc.chacha20_block(key, pc.BlockSeed(0x4000, 11, 0))

    def test_lane_units_are_consecutive_block_pairs(self, cuda):
        key = b"\x06" * 32
        ks = pc.page_keystream(key, 0x8000, 3)
        for i in (0, 7, 31):
            unit = ks[128 * i: 128 * (i + 1)]
            assert unit[:64] == pc.chacha20_block(key, pc.BlockSeed(0x8000, 3, 2 * i))
            assert unit[64:] == pc.chacha20_block(key, pc.BlockSeed(0x8000, 3, 2 * i + 1))

    def test_distinct_vaddrs_distinct_streams(self, cuda):
        k = b"\x01" * 32
        assert pc.page_keystream(k, 0x1000, 42) != pc.page_keystream(k, 0x2000, 42)

    def test_matches_reference(self, ref_pages, cuda):
        r = ref_pages
        key = r["key"].tobytes()
        for i in range(r["ks"].shape[0]):
            assert pc.page_keystream(key, int(r["vaddrs"][i]), int(r["pids"][i])) == r["ks"][i].tobytes()


class TestCryptPage:
    def test_matches_reference_64_pages(self, ref_pages, cuda):
        """BASELINE config 1: 64 random pages, ciphertext from the reference."""
        r = ref_pages
        key = r["key"].tobytes()
        for i in range(64):
            ct = pc.crypt_page(key, int(r["vaddrs"][i]), int(r["pids"][i]), r["pages"][i].tobytes())
            assert ct == r["ct"][i].tobytes(), i
            assert pc.crypt_page(key, int(r["vaddrs"][i]), int(r["pids"][i]), ct) == r["pages"][i].tobytes()

    def test_involution_random_pages_1000(self, cuda):
        rng = random.Random(3)
        for _ in range(1000):
            key, page = rand_key(rng), rand_page(rng)
            vaddr, pid = rng.randrange(2**40) * 4096, rng.randrange(2**32)
            assert pc.crypt_page(key, vaddr, pid, pc.crypt_page(key, vaddr, pid, page)) == page

    def test_zero_page_gives_keystream(self, cuda):
        key = b"\x09" * 32
        assert pc.crypt_page(key, 0x5000, 8, bytes(4096)) == pc.page_keystream(key, 0x5000, 8)

    def test_pid_separates_ciphertexts(self, cuda):
        rng = random.Random(4)
        key, page = rand_key(rng), rand_page(rng)
        assert pc.crypt_page(key, 0x1000, 1, page) != pc.crypt_page(key, 0x1000, 2, page)

    def test_accepts_every_buffer_kind_and_does_not_mutate(self, cuda):
        rng = random.Random(5)
        key, page = rand_key(rng), rand_page(rng)
        want = O.crypt_page(key, 0x6000, 123, page)
        ba = bytearray(page)
        for buf in (page, ba, memoryview(ba), np.frombuffer(page, np.uint8)):
            assert pc.crypt_page(key, 0x6000, 123, buf) == want
        assert bytes(ba) == page
        assert pc.crypt_page(pc.MasterKey(key), 0x6000, 123, page) == want

    def test_wrong_page_size_rejected(self, cuda):
        with pytest.raises(ContractViolation):
            pc.crypt_page(b"\x00" * 32, 0, 0, b"short")

    def test_boundary_seeds(self, cuda):
        key = b"\xff" * 32
        page = bytes(range(256)) * 16
        for vaddr, pid in ((0, 0), (2**64 - 4096, 2**32 - 1), (0x1_0000_0000, 4242)):
            assert pc.crypt_page(key, vaddr, pid, page) == O.crypt_page(key, vaddr, pid, page)


class TestParallelCryptPage:
    @pytest.mark.parametrize("lanes", [1, 7, 32, 64])
    def test_equals_reference_and_sequential(self, lanes, ref_pages, cuda):
        r = ref_pages
        key = r["key"].tobytes()
        for i in range(10):
            got = pc.parallel_crypt_page(key, int(r["vaddrs"][i]), int(r["pids"][i]), r["pages"][i].tobytes(), lanes)
            assert got == r[f"par{lanes}"][i].tobytes()
        rng = random.Random(100 + lanes)
        for _ in range(100):
            key, page = rand_key(rng), rand_page(rng)
            vaddr, pid = rng.randrange(2**30) * 4096, rng.randrange(2**32)
            assert pc.parallel_crypt_page(key, vaddr, pid, page, lanes) == pc.crypt_page(key, vaddr, pid, page)

    def test_zero_lanes_rejected(self, cuda):
        with pytest.raises(ContractViolation):
            pc.parallel_crypt_page(b"\x00" * 32, 0, 0, bytes(4096), 0)


class TestProperties:
    def test_keystream_injectivity_in_practice(self, cuda):
        rng = random.Random(6)
        key = rand_key(rng)
        triples = set()
        while len(triples) < 10_000:
            triples.add((rng.randrange(2**40) * 4096, rng.randrange(2**32), rng.randrange(64)))
        seeds = b"".join(O.seed_bytes(*t) for t in triples)
        blocks = pc.keystream_raw(key, seeds)
        assert len({blocks[64 * i: 64 * i + 64] for i in range(len(triples))}) == len(triples)

    def test_keystream_words_seam_matches_numba_contract(self, cuda):
        """_chacha_cuda.keystream_words is a drop-in for _chacha_numba's
        (cipher.py:178-181): block-major uint32 words, read-only kw allowed."""
        rng = random.Random(7)
        for _ in range(20):
            key = rand_key(rng)
            kw = np.frombuffer(key, dtype="<u4")  # read-only, like cipher._key_words
            vaddr, pid = rng.randrange(2**45) * 4096, rng.randrange(2**32)
            idx = np.arange(64, dtype=np.int64)
            out = np.empty(16 * 64, dtype=np.uint32)
            _chacha_cuda.keystream_words(kw, np.uint64(vaddr), np.uint32(pid), idx, out)
            want = O.keystream_words_np(key, vaddr, pid, idx).reshape(-1)
            assert np.array_equal(out, want)
        # arbitrary index lists (parallel_crypt_page lanes, chacha20_block)
        idx = np.array([63, 0, 17, 17], dtype=np.int64)
        out = np.empty(64, dtype=np.uint32)
        _chacha_cuda.keystream_words(np.frombuffer(key, "<u4"), np.uint64(0x1000), np.uint32(5), idx, out)
        assert np.array_equal(out, O.keystream_words_np(key, 0x1000, 5, idx).reshape(-1))

    def test_private_keystream_words(self, cuda):
        key = bytes(range(32))
        w = cipher._keystream_words(key, 0x2000, 9, np.array([3], dtype=np.int64))
        assert w.astype("<u4").tobytes() == O.block(key, 0x2000, 9, 3)
