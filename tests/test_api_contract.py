"""Host-side contract of the drop-in API (no GPU needed): the preconditions
and error types of pkg/src/pagecrypt/cipher.py (ContractViolation,
errors.py:8-10), exercised before any device work starts.  Mirrors the
rejection tests of pkg/tests/test_cipher.py:62-70,128-130,145-147,150-164."""

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import cipher
from paper_2004_09252_b200.engine import _host_pids, _host_vaddrs
from paper_2004_09252_b200.errors import ContractViolation, PageCryptError
from paper_2004_09252_b200.partition import page_ranges, shard


def test_constants_match_reference():
    assert (cipher.PAGE_SIZE, cipher.BLOCK_SIZE, cipher.BLOCKS_PER_PAGE) == (4096, 64, 64)
    assert (cipher.LANE_UNIT_BLOCKS, cipher.LANE_UNITS, cipher.KEY_SIZE) == (2, 32, 32)
    assert issubclass(ContractViolation, PageCryptError)


class TestBlockSeed:
    def test_bad_block_index_rejected(self):
        with pytest.raises(ContractViolation):
            pc.BlockSeed(0, 0, 64)
        with pytest.raises(ContractViolation):
            pc.BlockSeed(0, 0, -1)

    def test_unaligned_vaddr_rejected(self):
        with pytest.raises(ContractViolation):
            pc.BlockSeed(0x1001, 0, 0)

    def test_out_of_range_fields_rejected(self):
        with pytest.raises(ContractViolation):
            pc.BlockSeed(2**64, 0, 0)
        with pytest.raises(ContractViolation):
            pc.BlockSeed(0, 2**32, 0)
        with pytest.raises(ContractViolation):
            pc.BlockSeed(-4096, 0, 0)

    def test_seed_serializes_to_16_bytes(self):
        s = pc.BlockSeed(0x2000, 77, 5)
        raw = s.to_bytes()
        assert raw == (0x2000).to_bytes(8, "little") + (77).to_bytes(4, "little") + (5).to_bytes(4, "little")
        assert pc.BlockSeed.from_bytes(raw) == s
        with pytest.raises(ContractViolation):
            pc.BlockSeed.from_bytes(b"short")


class TestMasterKey:
    def test_generate_is_32_bytes_and_random(self):
        a, b = pc.MasterKey.generate(), pc.MasterKey.generate()
        assert len(a) == 32 and bytes(a.view()) != bytes(b.view())

    def test_destroy_zeroizes(self):
        k = pc.MasterKey(b"\xAA" * 32)
        k.destroy()
        assert bytes(k.view()) == bytes(32) and k.destroyed

    def test_wrong_size_rejected(self):
        with pytest.raises(ContractViolation):
            pc.MasterKey(b"\x00" * 16)


class TestRejectionsBeforeDevice:
    def test_wrong_page_size(self):
        with pytest.raises(ContractViolation):
            pc.crypt_page(b"\x00" * 32, 0, 0, b"short")
        with pytest.raises(ContractViolation):
            pc.parallel_crypt_page(b"\x00" * 32, 0, 0, b"short", 4)

    def test_zero_lanes(self):
        with pytest.raises(ContractViolation):
            pc.parallel_crypt_page(b"\x00" * 32, 0, 0, bytes(4096), 0)

    def test_bad_key(self):
        with pytest.raises(ContractViolation):
            pc.crypt_page(b"\x00" * 31, 0, 0, bytes(4096))

    def test_bad_vaddr_pid(self):
        with pytest.raises(ContractViolation):
            pc.crypt_page(bytes(32), 0x1001, 0, bytes(4096))
        with pytest.raises(ContractViolation):
            pc.crypt_page(bytes(32), 0, 2**32, bytes(4096))
        with pytest.raises(ContractViolation):
            pc.page_keystream(bytes(32), 2**64, 0)

    def test_bad_rounds(self):
        with pytest.raises(ContractViolation):
            pc.crypt_page(bytes(32), 0, 0, bytes(4096), rounds=10)
        with pytest.raises(ContractViolation):
            pc.crypt_pages(bytes(32), 0, 0, np.zeros((1, 4096), np.uint8), rounds=7)

    def test_ragged_batch(self):
        with pytest.raises(ContractViolation):
            pc.crypt_pages(bytes(32), 0, 0, np.zeros(4097, np.uint8))


class TestDescriptors:
    def test_contiguous_vaddr(self):
        assert _host_vaddrs(0x1000, 4) == (None, 0x1000)
        with pytest.raises(ContractViolation):
            _host_vaddrs(2**64 - 4096, 2)  # overflows u64
        with pytest.raises(ContractViolation):
            _host_vaddrs(0x1008, 1)

    def test_vaddr_arrays(self):
        arr, v0 = _host_vaddrs([0, 4096, 2**64 - 4096], 3)
        assert arr.dtype == np.uint64 and v0 == 0 and int(arr[2]) == 2**64 - 4096
        with pytest.raises(ContractViolation):
            _host_vaddrs([0, 4097], 2)
        with pytest.raises(ContractViolation):
            _host_vaddrs([0, -4096], 2)
        with pytest.raises(ContractViolation):
            _host_vaddrs([0], 2)

    def test_pid_arrays(self):
        arr, _ = _host_pids([0, 2**32 - 1], 2)
        assert arr.dtype == np.uint32 and int(arr[1]) == 2**32 - 1
        with pytest.raises(ContractViolation):
            _host_pids([2**32], 1)
        with pytest.raises(ContractViolation):
            _host_pids(-1, 1)


class TestPartition:
    @pytest.mark.parametrize("n,parts", [(0, 1), (1, 8), (7, 3), (262144, 8), (1000003, 7)])
    def test_ranges_cover_disjoint_balanced(self, n, parts):
        rs = page_ranges(n, parts)
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        sizes = [hi - lo for lo, hi in rs]
        assert max(sizes) - min(sizes) <= 1

    def test_shard_bounds(self):
        assert shard(10, 1, 2) == (5, 10)
        with pytest.raises(ContractViolation):
            shard(10, 2, 2)
        with pytest.raises(ContractViolation):
            page_ranges(10, 0)
