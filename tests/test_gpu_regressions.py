"""Regression tests for the round-1 advisor findings, each
checked against the oracle where bytes are produced."""

import ctypes

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import _native, partition
from paper_2004_09252_b200.errors import ContractViolation, PageCryptError
from paper_2004_09252_b200.store import DevicePageStore

from oracle import coracle as C

pytestmark = pytest.mark.gpu

KEY = bytes(range(32))
BASE = 0x1_0000_0000


def rand_pages(n, seed=7):
    return np.random.default_rng(seed).integers(0, 256, size=(n, 4096), dtype=np.uint8)


@pytest.mark.parametrize("chunk", [1, 4, 7])
def test_tiny_chunk_engine_finishes(cuda, chunk):
    """chunk_pages 1..7 used to spin forever building the ramp schedule."""
    eng = pc.Engine(0, n_streams=3, chunk_pages=chunk)
    try:
        pages = rand_pages(130)
        with pc.DeviceKey.install(KEY, 0) as dk:
            got = pc.crypt_pages(dk, BASE, 1, pages, engine=eng)
        assert np.array_equal(got, C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=1))
    finally:
        eng.destroy()


def test_key_destroy_refused_while_store_holds_it(cuda):
    dk = pc.DeviceKey.install(KEY, 0)
    st = DevicePageStore(8, dk, device=0)
    with pytest.raises(PageCryptError):
        dk.destroy()
    assert not dk.destroyed  # still live and usable
    pages = rand_pages(2)
    from paper_2004_09252_b200.workers import ClientId

    c = ClientId(5, 0)
    vs = np.array([BASE, BASE + 4096], dtype=np.uint64)
    st.evict_many(c, vs, pages)
    out = np.empty_like(pages)
    st.refault_many(c, vs, out=out)
    assert np.array_equal(out, pages)
    st.close()
    dk.destroy()
    assert dk.destroyed


@pytest.mark.parametrize("n", [1, 5, 64, 65, 200])
def test_slab_transfer_honours_per_page_pids(cuda, n):
    """The n <= 64 zero-copy path used to ignore a per-page pids array."""
    import torch

    lib = _native.load()
    eng = pc.Engine(0)
    slab = torch.zeros((n + 3, 4096), dtype=torch.uint8, device="cuda:0")
    pages = rand_pages(n, seed=n)
    slots = np.arange(n, dtype=np.uint32)[::-1].copy()
    vaddrs = (np.arange(n, dtype=np.uint64) * np.uint64(8192) + np.uint64(BASE))
    pids = (1 + np.arange(n) % 64).astype(np.uint32) * np.uint32(977)
    try:
        with pc.DeviceKey.install(KEY, 0) as dk:
            _native.check(lib.pc_slab_transfer(
                ctypes.c_void_p(eng.handle), ctypes.c_void_p(dk.handle), ctypes.c_void_p(slab.data_ptr()),
                ctypes.c_size_t(n + 3), slots.ctypes.data, vaddrs.ctypes.data, pids.ctypes.data,
                ctypes.c_uint64(0), ctypes.c_uint32(0), pages.ctypes.data, ctypes.c_size_t(n), 0, 20, 0))
            torch.cuda.synchronize()
        want = C.crypt_pages(KEY, vaddrs, pids, pages)
        got = slab.cpu().numpy()[slots]
        assert np.array_equal(got, want)
    finally:
        eng.destroy()


def test_desc_check_on_side_stream(cuda):
    """pc_desc_check launches on the stream's own device (cudaStreamGetDevice)."""
    import torch

    n = 33
    pages = rand_pages(n)
    vaddrs = np.arange(n, dtype=np.uint64) * np.uint64(4096) * np.uint64(3) + np.uint64(BASE)
    pids = (1 + np.arange(n) % 64).astype(np.int64)
    s = torch.cuda.Stream(device="cuda:0")
    with pc.DeviceKey.install(KEY, 0) as dk:
        got = pc.crypt_pages(dk, torch.from_numpy(vaddrs.view(np.int64)).cuda(), torch.from_numpy(pids).cuda(),
                             torch.from_numpy(pages).cuda(), stream=s)
        s.synchronize()
    assert np.array_equal(got.cpu().numpy(), C.crypt_pages(KEY, vaddrs, pids.astype(np.uint32), pages))


@pytest.mark.parametrize("bad", ["short", "readonly", "dtype", "strided"])
def test_multi_host_out_validated(cuda, bad):
    pages = rand_pages(16)
    good = np.empty_like(pages)
    out = {"short": np.empty((15, 4096), np.uint8), "readonly": good.copy(),
           "dtype": np.empty((16, 1024), np.uint32), "strided": np.empty((16, 8192), np.uint8)[:, ::2]}[bad]
    if bad == "readonly":
        out.flags.writeable = False
    eng = pc.Engine(0)
    try:
        with pc.DeviceKey.install(KEY, 0) as dk:
            with pytest.raises(ContractViolation):
                partition.crypt_pages_multi([dk], [eng], BASE, 1, pages, out=out)
            partition.crypt_pages_multi([dk], [eng], BASE, 1, pages, out=good)
        assert np.array_equal(good, C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=1))
    finally:
        eng.destroy()
