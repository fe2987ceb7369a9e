"""GPU parity of the batched engine: device-resident and host-resident
paths, descriptor forms, rounds, in-place, edge sizes, the key lifecycle and
the multi-device partition -- byte-exact against the C oracle at sizes it
finishes in seconds, and at BASELINE's 1 GiB size through size-independent
properties (involution, keystream linearity, chunk/partition independence)."""

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import partition
from paper_2004_09252_b200.errors import ContractViolation, PageCryptError

from oracle import coracle as C

pytestmark = pytest.mark.gpu

KEY = bytes.fromhex("8b034a0ee06db6c134b1c8fc867c39bae599f01835025a7acf4b57268dc7853c")
BASE = 0x1_0000_0000


def rand_pages(n, seed=1):
    return np.random.default_rng(seed).integers(0, 256, size=(n, 4096), dtype=np.uint8)


@pytest.fixture(scope="module")
def dkey(cuda):
    k = pc.DeviceKey.install(KEY, 0)
    yield k
    k.destroy()


def t(x, device="cuda"):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(device)


@pytest.fixture
def knob():
    """Set engine knobs for one test and restore them afterwards."""
    from paper_2004_09252_b200 import _native

    saved = {}

    def set_(name, value):
        saved.setdefault(name, _native.tune_get(name))
        _native.tune(name, value)

    yield set_
    for name, value in saved.items():
        _native.tune(name, value)


class TestDevicePath:
    @pytest.mark.parametrize("kernel", [1, 2, 3, 4, 5, 6, 9])
    @pytest.mark.parametrize("rounds", [8, 12, 20])
    @pytest.mark.parametrize("n", [1, 3, 64, 4097])
    def test_contiguous_scalar_pid(self, dkey, n, rounds, kernel, knob):
        import torch

        knob("kernel", kernel)
        pages = rand_pages(n, seed=n)
        got = pc.crypt_pages(dkey, BASE, 1, t(pages), rounds=rounds)
        torch.cuda.synchronize()
        want = C.crypt_pages(KEY, None, None, pages, rounds=rounds, vaddr0=BASE, pid0=1, nthreads=8)
        assert np.array_equal(got.cpu().numpy(), want)

    @pytest.mark.parametrize("kernel", [1, 2, 3, 4, 5, 6, 9])
    def test_per_page_descriptors(self, dkey, ref_pages, kernel, knob):
        import torch

        knob("kernel", kernel)
        r = ref_pages
        with pc.DeviceKey.install(r["key"].tobytes(), 0) as k:
            got = pc.crypt_pages(k, t(r["vaddrs"].view(np.int64)), t(r["pids"].view(np.int32)), t(r["pages"]))
            torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), r["ct"])

    def test_numpy_descriptors_and_uint64(self, ref_pages):
        import torch

        r = ref_pages
        got = pc.crypt_pages(r["key"].tobytes(), r["vaddrs"], r["pids"], t(r["pages"]))
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), r["ct"])

    @pytest.mark.parametrize("shape", ["vaddr_array", "pid_array", "both"])
    @pytest.mark.parametrize("rounds", [8, 12, 20])
    @pytest.mark.parametrize("n", [1, 2, 3, 5, 1183, 2369, 4097])
    @pytest.mark.parametrize("kernel", [0, 5, 6, 9])
    @pytest.mark.parametrize("run_desc", [0, 1, 2])
    def test_every_descriptor_shape_ragged(self, dkey, shape, rounds, n, kernel, run_desc, knob):
        """Each descriptor shape compiles to its own loop (DM = vaddr array |
        pid array; page-pair loops for R <= 12 and for R = 20 with a vaddr
        array alone): ragged counts around the grid stride (296 or 444 CTAs
        x 4 pages), random vaddrs whose high word changes page to page,
        vaddrs crossing 4 GiB, random u32 pids."""
        import torch

        rng = np.random.default_rng(n * 31 + rounds)
        pages = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
        va = (rng.integers(0, 2**52, size=n, dtype=np.uint64) << np.uint64(12))
        va[: n // 2] = 0xFFFF_F000 + 4096 * np.arange(n // 2, dtype=np.uint64)  # crosses 4 GiB
        pi = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        if run_desc == 0 and kernel not in (0, 5):
            pytest.skip("run_desc only changes v5")
        knob("kernel", kernel)
        knob("run_desc", run_desc)  # v5 at R <= 12: contiguous page runs per slot (pair descriptor loads)
        v_arg = t(va.view(np.int64)) if shape != "pid_array" else BASE
        p_arg = t(pi.view(np.int32)) if shape != "vaddr_array" else 77
        v_ref = va if shape != "pid_array" else BASE + 4096 * np.arange(n, dtype=np.uint64)
        p_ref = pi if shape != "vaddr_array" else np.full(n, 77, np.uint32)
        got = pc.crypt_pages(dkey, v_arg, p_arg, t(pages), rounds=rounds)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), C.crypt_pages(KEY, v_ref, p_ref, pages, rounds=rounds, nthreads=8))

    @pytest.mark.parametrize("rounds", [8, 12, 20])
    @pytest.mark.parametrize("run_desc", [0, 1, 2])
    @pytest.mark.parametrize("n", [1, 2, 3, 593, 1186])
    def test_descriptor_loops_stay_inside_the_batch(self, dkey, rounds, run_desc, n, knob):
        """The batch is a window of a larger buffer with guard pages on both
        sides and its descriptor arrays are windows of longer arrays: every
        descriptor loop (v5 strided, page runs, two blocks per thread) writes
        exactly the window and leaves the guards and the input untouched
        (compute-sanitizer is not available on this pool; this is the write
        side of its memcheck)."""
        import torch

        knob("kernel", 5)
        knob("run_desc", run_desc)
        g = 3  # guard pages each side
        rng = np.random.default_rng(n * 7 + rounds + run_desc)
        pages = rng.integers(0, 256, size=(n + 2 * g, 4096), dtype=np.uint8)
        va = rng.integers(0, 2**52, size=n + 2 * g, dtype=np.uint64) << np.uint64(12)
        pi = rng.integers(0, 2**32, size=n + 2 * g, dtype=np.uint64).astype(np.uint32)
        src = t(pages)
        dst = torch.full_like(src, 0xA5)
        v_t = t(va.view(np.int64))[g:g + n]  # offset g = 3: 8-byte aligned only (v5 fallback) ...
        p_t = t(pi.view(np.int32))[g:g + n]
        for vv, pp, lo in ((v_t, p_t, g), (t(va[g:g + n].copy().view(np.int64)), t(pi[g:g + n].copy().view(np.int32)), g)):
            dst.fill_(0xA5)  # ... and fresh, aligned copies (the run loops)
            pc.crypt_pages(dkey, vv, pp, src[lo:lo + n], out=dst[lo:lo + n], rounds=rounds)
            torch.cuda.synchronize()
            got = dst.cpu().numpy()
            assert (got[:lo] == 0xA5).all() and (got[lo + n:] == 0xA5).all()
            want = C.crypt_pages(KEY, va[g:g + n], pi[g:g + n], pages[g:g + n], rounds=rounds)
            assert np.array_equal(got[lo:lo + n], want)
        assert np.array_equal(src.cpu().numpy(), pages)

    @pytest.mark.parametrize("rounds", [8, 12])
    @pytest.mark.parametrize("offset", [0, 1])
    @pytest.mark.parametrize("run_desc", [1, 2])
    def test_run_desc_alignment_fallback(self, dkey, rounds, offset, run_desc, knob):
        """v5's page-run loop loads a page pair's descriptors as one 16-byte
        vaddr and one 8-byte pid load; arrays that start off that alignment
        (a tensor view one element in) take the per-page loop.  Both equal
        the oracle, with odd and even page counts."""
        import torch

        knob("kernel", 5)
        knob("run_desc", run_desc)  # 2: one warp per page slot, two blocks per thread
        for n in (1, 2, 7, 1184, 2371):
            rng = np.random.default_rng(n + offset)
            pages = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
            va = rng.integers(0, 2**52, size=n + 1, dtype=np.uint64) << np.uint64(12)
            pi = rng.integers(0, 2**32, size=n + 1, dtype=np.uint64).astype(np.uint32)
            v_t = t(va.view(np.int64))[offset:offset + n]
            p_t = t(pi.view(np.int32))[offset:offset + n]
            got = pc.crypt_pages(dkey, v_t, p_t, t(pages), rounds=rounds)
            torch.cuda.synchronize()
            want = C.crypt_pages(KEY, va[offset:offset + n], pi[offset:offset + n], pages, rounds=rounds)
            assert np.array_equal(got.cpu().numpy(), want), n

    @pytest.mark.parametrize("kernel", [6, 9])
    @pytest.mark.parametrize("shape", ["contig", "vaddr_array", "pid_array", "both"])
    @pytest.mark.parametrize("rounds", [12, 20])
    @pytest.mark.parametrize("n", [75_777, 151_553])
    def test_v6_many_table_refills(self, dkey, shape, rounds, n, kernel, knob):
        """k_crypt_pages_warp refills its per-slot seed table every 32 pages of
        a thread: batches long enough for several refills (n > 32 x the grid
        stride of 296/592 CTAs x 4 pages), ragged tails, every descriptor
        shape, random vaddrs whose high word changes."""
        import torch

        knob("kernel", kernel)
        rng = np.random.default_rng(n + rounds)
        pages = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
        va = (rng.integers(0, 2**52, size=n, dtype=np.uint64) << np.uint64(12))
        pi = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        v_arg = t(va.view(np.int64)) if shape in ("vaddr_array", "both") else BASE
        p_arg = t(pi.view(np.int32)) if shape in ("pid_array", "both") else 77
        v_ref = va if shape in ("vaddr_array", "both") else BASE + 4096 * np.arange(n, dtype=np.uint64)
        p_ref = pi if shape in ("pid_array", "both") else np.full(n, 77, np.uint32)
        buf = t(pages)
        got = pc.crypt_pages(dkey, v_arg, p_arg, buf, out=buf if kernel == 9 else None, rounds=rounds)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), C.crypt_pages(KEY, v_ref, p_ref, pages, rounds=rounds, nthreads=16))

    @pytest.mark.parametrize("kernel", [1, 2, 3, 4, 5, 6, 9])
    def test_pid_per_page_variant(self, dkey, kernel, knob):
        """pid = 1 + (i % 64); also vaddr_hi changing mid-batch
        (the v2/v3 kernels cache the vaddr_hi/pid column rounds)."""
        import torch

        knob("kernel", kernel)
        n = 3000
        pages = rand_pages(n, 31)
        v0 = 0x1_0000_0000 - 1500 * 4096  # crosses the 4 GiB boundary half way
        got = pc.crypt_pages(dkey, v0, 9, t(pages))
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(),
                              C.crypt_pages(KEY, None, None, pages, vaddr0=v0, pid0=9, nthreads=8))

        n = 2048
        pages = rand_pages(n, 3)
        pids = (1 + np.arange(n) % 64).astype(np.uint32)
        got = pc.crypt_pages(dkey, BASE, t(pids.view(np.int32)), t(pages))
        torch.cuda.synchronize()
        want = C.crypt_pages(KEY, None, pids, pages, vaddr0=BASE, nthreads=8)
        assert np.array_equal(got.cpu().numpy(), want)

    def test_in_place(self, dkey):
        import torch

        pages = rand_pages(513, 4)
        d = t(pages)
        out = pc.crypt_pages(dkey, BASE, 7, d, out=d)
        torch.cuda.synchronize()
        assert out.data_ptr() == d.data_ptr()
        assert np.array_equal(d.cpu().numpy(), C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=7, nthreads=8))

    def test_empty_batch(self, dkey):
        import torch

        d = torch.empty((0, 4096), dtype=torch.uint8, device="cuda")
        assert pc.crypt_pages(dkey, BASE, 1, d).numel() == 0

    def test_side_stream(self, dkey):
        import torch

        pages = rand_pages(300, 5)
        s = torch.cuda.Stream()
        d = t(pages)
        torch.cuda.current_stream().synchronize()
        with torch.cuda.stream(s):
            got = pc.crypt_pages(dkey, BASE, 2, d)
        s.synchronize()
        assert np.array_equal(got.cpu().numpy(), C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=2))

    def test_unaligned_device_vaddrs_rejected(self, dkey):
        v = t(np.array([4096, 4097], dtype=np.int64))
        with pytest.raises(ContractViolation):
            pc.crypt_pages(dkey, v, 1, t(rand_pages(2)))

    def test_float_device_descriptors_rejected(self, dkey):
        """Descriptor tensors must hold integers: a float64 vaddr tensor has
        the right element size but not the meaning."""
        import torch

        pages = t(rand_pages(2))
        with pytest.raises(ContractViolation):
            pc.crypt_pages(dkey, torch.tensor([4096.0, 8192.0], dtype=torch.float64, device="cuda"), 1, pages)
        with pytest.raises(ContractViolation):
            pc.crypt_pages(dkey, BASE, torch.tensor([1.0, 2.0], dtype=torch.float32, device="cuda"), pages)
        with pytest.raises(ContractViolation):
            pc.crypt_pages(dkey, BASE, torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda"), pages)

    def test_max_vaddr_and_pid(self, dkey):
        import torch

        pages = rand_pages(4, 6)
        v0 = 2**64 - 4 * 4096
        got = pc.crypt_pages(dkey, v0, 2**32 - 1, t(pages))
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), C.crypt_pages(KEY, None, None, pages, vaddr0=v0, pid0=2**32 - 1))
        with pytest.raises(ContractViolation):
            pc.crypt_pages(dkey, 2**64 - 2 * 4096, 1, t(pages))  # range overflows u64


class TestFullSize:
    """BASELINE config 2/3 size (1 GiB) through size-independent properties."""

    @pytest.mark.parametrize("rounds", [8, 12, 20])
    def test_1gib_roundtrip_and_samples(self, dkey, rounds):
        import torch

        n = 262_144
        g = torch.Generator(device="cuda").manual_seed(1)
        pages = torch.randint(0, 256, (n, 4096), dtype=torch.uint8, device="cuda", generator=g)
        ct = pc.crypt_pages(dkey, BASE, 1, pages, rounds=rounds)
        back = pc.crypt_pages(dkey, BASE, 1, ct, rounds=rounds)
        assert torch.equal(back, pages)
        # keystream linearity: ct ^ pt is the keystream, = crypt(zero page)
        idx = torch.tensor([0, 1, 4095, 131072, n - 1], device="cuda")
        ks = (ct[idx] ^ pages[idx]).cpu().numpy()
        for j, p in enumerate(idx.tolist()):
            want = C.crypt_pages(KEY, None, None, np.zeros((1, 4096), np.uint8), rounds=rounds,
                                 vaddr0=BASE + 4096 * p, pid0=1)
            assert np.array_equal(ks[j], want[0])
        # a strided sample byte-exact against the oracle
        sl = slice(0, n, 997)
        sample_idx = np.arange(0, n, 997)
        pv = BASE + 4096 * sample_idx.astype(np.uint64)
        want = C.crypt_pages(KEY, pv, 1, pages[sl].cpu().numpy(), rounds=rounds, nthreads=8)
        assert np.array_equal(ct[sl].cpu().numpy(), want)
        del pages, ct, back
        torch.cuda.empty_cache()

    @pytest.mark.parametrize("rounds", [8, 12, 20])
    def test_1gib_every_byte_against_the_oracle(self, dkey, rounds):
        """The whole BASELINE configs[1]/[2] batch (1 GiB, the bench's
        workload: contiguous vaddrs from BASE, pid 1) byte-exact against the
        C oracle on all host cores, per-page descriptors included."""
        import os

        import torch

        n = 262_144
        host = np.random.default_rng(rounds).integers(0, 256, size=(n, 4096), dtype=np.uint8)
        pages = torch.from_numpy(host).cuda()
        threads = max(1, len(os.sched_getaffinity(0)))
        got = pc.crypt_pages(dkey, BASE, 1, pages, rounds=rounds).cpu().numpy()
        want = C.crypt_pages(KEY, None, None, host, rounds=rounds, vaddr0=BASE, pid0=1, nthreads=threads)
        assert np.array_equal(got, want)
        # per-page descriptors: a permutation of vaddrs, 64 pids
        va = BASE + 4096 * np.random.default_rng(7).permutation(n).astype(np.uint64)
        pid = (1 + np.arange(n) % 64).astype(np.uint32)
        got = pc.crypt_pages(dkey, torch.from_numpy(va.view(np.int64)).cuda(),
                             torch.from_numpy(pid.view(np.int32)).cuda(), pages, rounds=rounds).cpu().numpy()
        want = C.crypt_pages(KEY, va, pid, host, rounds=rounds, nthreads=threads)
        assert np.array_equal(got, want)
        del pages
        torch.cuda.empty_cache()

    def test_1gib_host_resident_every_byte(self, dkey):
        """The bench's e2e leg (1 GiB pinned host pages through the ramped
        H2D / cipher / D2H pipeline, out of place and in place) byte-exact."""
        import os

        import torch

        n = 262_144
        host = np.random.default_rng(5).integers(0, 256, size=(n, 4096), dtype=np.uint8)
        threads = max(1, len(os.sched_getaffinity(0)))
        want = C.crypt_pages(KEY, None, None, host, vaddr0=BASE, pid0=1, nthreads=threads)
        src = torch.from_numpy(host).pin_memory()
        dst = torch.empty_like(src).pin_memory()
        pc.crypt_pages(dkey, BASE, 1, src, out=dst)
        assert np.array_equal(dst.numpy(), want)
        pc.crypt_pages(dkey, BASE, 1, src, out=src)
        assert np.array_equal(src.numpy(), want)


class TestHostPath:
    @pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 2048, 2049, 10_000])
    def test_pageable_numpy(self, dkey, n):
        pages = rand_pages(n, 10 + n)
        got = pc.crypt_pages(dkey, BASE, 3, pages)
        assert np.array_equal(got, C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=3, nthreads=8))

    @pytest.mark.parametrize("host_mode", [0, 1, 2, 3])
    @pytest.mark.parametrize("n", [1, 64, 65, 9000])
    def test_pinned_torch(self, dkey, n, host_mode, knob):
        import torch

        knob("host_mode", host_mode)
        pages = rand_pages(n, 20 + n)
        src = torch.from_numpy(pages).pin_memory()
        dst = torch.empty_like(src).pin_memory()
        pc.crypt_pages(dkey, BASE, 4, src, out=dst)
        assert np.array_equal(dst.numpy(), C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=4, nthreads=8))

    @pytest.mark.parametrize("host_mode", [0, 1, 2, 3])
    def test_raw_key_host_with_descriptors(self, ref_pages, host_mode, knob):
        knob("host_mode", host_mode)
        r = ref_pages
        got = pc.crypt_pages(r["key"].tobytes(), r["vaddrs"], r["pids"], r["pages"])
        assert np.array_equal(got, r["ct"])
        big = np.concatenate([r["pages"]] * 40)  # 2560 pages -> large path with descriptors
        va = np.concatenate([r["vaddrs"]] * 40)
        pi = np.concatenate([r["pids"]] * 40)
        got = pc.crypt_pages(r["key"].tobytes(), va, pi, big)
        assert np.array_equal(got, np.concatenate([r["ct"]] * 40))

    def test_in_place_host(self, dkey):
        pages = rand_pages(3000, 7)
        buf = pages.copy()
        pc.crypt_pages(dkey, BASE, 5, buf, out=buf)
        assert np.array_equal(buf, C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=5, nthreads=8))

    @pytest.mark.parametrize("host_mode", [0, 1, 2, 3])
    def test_in_place_pinned_with_pinned_descriptors(self, dkey, host_mode, knob):
        import torch

        knob("host_mode", host_mode)
        n = 1000
        pages = rand_pages(n, 17)
        buf = torch.from_numpy(pages.copy()).pin_memory()
        va = torch.from_numpy((BASE + 4096 * np.arange(n, dtype=np.uint64)[::-1].copy()).view(np.int64)).pin_memory()
        pi = torch.from_numpy((np.arange(n) % 7).astype(np.int32)).pin_memory()
        pc.crypt_pages(dkey, va.numpy().view(np.uint64), pi.numpy().view(np.uint32), buf, out=buf)
        want = C.crypt_pages(KEY, va.numpy().view(np.uint64), pi.numpy().view(np.uint32), pages, nthreads=8)
        assert np.array_equal(buf.numpy(), want)

    def test_engine_stream_configs_agree(self, dkey):
        pages = rand_pages(5000, 8)
        want = C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=6, nthreads=8)
        for ns, chunk in ((1, 512), (3, 777), (8, 4096)):
            eng = pc.Engine(0, n_streams=ns, chunk_pages=chunk)
            try:
                got = pc.crypt_pages(dkey, BASE, 6, pages, engine=eng)
                assert np.array_equal(got, want), (ns, chunk)
            finally:
                eng.destroy()


class TestKeys:
    def test_generate_distinct_and_roundtrip(self, cuda):
        import torch

        pages = rand_pages(16, 9)
        a, b = pc.DeviceKey.generate(0), pc.DeviceKey.generate(0)
        try:
            ca = pc.crypt_pages(a, BASE, 1, t(pages))
            cb = pc.crypt_pages(b, BASE, 1, t(pages))
            assert not torch.equal(ca, cb)
            assert np.array_equal(pc.crypt_pages(a, BASE, 1, ca).cpu().numpy(), pages)
            assert pc.crypt_page(a, BASE, 1, pages[0].tobytes()) == ca[0].cpu().numpy().tobytes()
        finally:
            a.destroy()
            b.destroy()

    def test_destroy_is_idempotent_and_final(self, cuda):
        k = pc.DeviceKey.install(KEY, 0)
        k.destroy()
        k.destroy()
        assert k.destroyed
        with pytest.raises(PageCryptError):
            pc.crypt_pages(k, BASE, 1, rand_pages(1))

    def test_device_key_matches_raw_key(self, dkey):
        page = rand_pages(1, 12)[0].tobytes()
        assert pc.crypt_page(dkey, BASE, 9, page) == pc.crypt_page(KEY, BASE, 9, page)


class TestMultiDevice:
    def test_partition_over_engines_is_identical(self, cuda):
        import torch

        ndev = torch.cuda.device_count()
        devs = [d % ndev for d in range(max(2, ndev))]  # >= 2 slots even on one GPU
        engines = [pc.Engine(d, n_streams=2, chunk_pages=1024) for d in devs]
        keys = [pc.DeviceKey.install(KEY, d) for d in devs]
        try:
            pages = rand_pages(7001, 13)
            got = partition.crypt_pages_multi(keys, engines, BASE, 11, pages)
            assert np.array_equal(got, C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=11, nthreads=8))
            va = BASE + 4096 * np.random.default_rng(0).permutation(7001).astype(np.uint64)
            got = partition.crypt_pages_multi(keys, engines, va, 11, pages)
            assert np.array_equal(got, C.crypt_pages(KEY, va, 11, pages, nthreads=8))
        finally:
            for k in keys:
                k.destroy()
            for e in engines:
                e.destroy()

    @pytest.mark.parametrize("dev_direct", [1, 0])
    def test_device_resident_partition(self, cuda, dev_direct, knob):
        """Pages resident on one GPU, split over engines: the
        owning GPU runs in place, the others pull their range peer-to-peer.
        With one GPU, dev_direct=0 forces every range through the engines'
        staging ring (the peer path, as same-device copies)."""
        import torch

        knob("dev_direct", dev_direct)
        ndev = torch.cuda.device_count()
        devs = [d % ndev for d in range(max(3, ndev))]
        engines = [pc.Engine(d, n_streams=3, chunk_pages=512) for d in devs]
        keys = [pc.DeviceKey.install(KEY, d) for d in devs]
        try:
            host = rand_pages(5003, 17)
            pages = torch.from_numpy(host).to("cuda:0")
            want = C.crypt_pages(KEY, None, None, host, vaddr0=BASE, pid0=5, nthreads=8)
            got = partition.crypt_pages_multi(keys, engines, BASE, 5, pages)
            assert got.is_cuda and np.array_equal(got.cpu().numpy(), want)
            # in place, per-page descriptors (staged path), then back
            va = BASE + 4096 * np.random.default_rng(1).permutation(5003).astype(np.uint64)
            partition.crypt_pages_multi(keys, engines, va, 5, pages, out=pages)
            assert np.array_equal(pages.cpu().numpy(), C.crypt_pages(KEY, va, 5, host, nthreads=8))
            partition.crypt_pages_multi(keys, engines, va, 5, pages, out=pages)
            assert np.array_equal(pages.cpu().numpy(), host)
            # through the C ABI directly: device in, host out
            out = np.empty_like(host)
            engines[0].crypt_host(keys[0], BASE, 5, pages.data_ptr(), out.ctypes.data, 5003, 20)
            assert np.array_equal(out, want)
        finally:
            for k in keys:
                k.destroy()
            for e in engines:
                e.destroy()


class TestConcurrentCallers:
    """The reference cipher is 'pure and safe for concurrent callers'
    (SPEC.md:101-102).  Eight host threads share the default engine, one
    HBM store and the keystream seams, each checking every result against
    the oracle."""

    def test_threads_share_engine_store_and_seams(self, dkey, cuda):
        import threading

        import torch

        from paper_2004_09252_b200 import _chacha_cuda
        from paper_2004_09252_b200.store import DevicePageStore
        from paper_2004_09252_b200.workers import ClientId

        store = DevicePageStore(4096, dkey)
        errors = []

        def worker(t):
            try:
                rng = np.random.default_rng(100 + t)
                cl = ClientId(500 + t, 0)
                stream = torch.cuda.Stream()
                for it in range(6):
                    n = int(rng.integers(1, 3000))
                    pages = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
                    v0 = BASE + 4096 * int(rng.integers(0, 1 << 20))
                    want = C.crypt_pages(KEY, None, None, pages, vaddr0=v0, pid0=cl.pid, nthreads=2)
                    # host batch through the shared default engine (pageable and pinned)
                    got = pc.crypt_pages(dkey, v0, cl.pid, pages)
                    assert np.array_equal(got, want)
                    src = torch.from_numpy(pages).pin_memory()
                    dst = pc.crypt_pages(dkey, v0, cl.pid, src)
                    assert np.array_equal(dst.numpy(), want)
                    # device batch on this thread's own stream
                    with torch.cuda.stream(stream):
                        d = pc.crypt_pages(dkey, v0, cl.pid, torch.from_numpy(pages).cuda(), stream=stream)
                    stream.synchronize()
                    assert np.array_equal(d.cpu().numpy(), want)
                    # reference single-page API with raw key bytes, and the kernel seam
                    assert pc.crypt_page(KEY, v0, cl.pid, pages[0].tobytes()) == want[0].tobytes()
                    out = np.empty(1024, np.uint32)
                    _chacha_cuda.keystream_words(np.frombuffer(KEY, "<u4"), np.uint64(v0), np.uint32(cl.pid),
                                                 np.arange(64, dtype=np.int64), out)
                    assert out.tobytes() == (want[0] ^ pages[0]).tobytes()
                    # the shared HBM store: evict then refault this thread's pages
                    m = min(n, 200)
                    va = [v0 + 4096 * i for i in range(m)]
                    store.evict_many(cl, va, pages[:m])
                    assert store.lookup(cl, va[0]) == want[0].tobytes()
                    assert np.array_equal(store.refault_many(cl, va), pages[:m])
            except BaseException as exc:  # surfaced below
                errors.append((t, repr(exc)))

        threads = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        assert not errors, errors
        assert store.free_slots == 4096
        store.close()


class TestEdgeShapes:
    def test_fewer_pages_than_engines(self, dkey, cuda):
        """Engines whose range is empty do nothing; the rest still match."""
        devs = [0, 0, 0, 0]
        engines = [pc.Engine(d, n_streams=3, chunk_pages=64) for d in devs]
        keys = [pc.DeviceKey.install(KEY, d) for d in devs]
        try:
            for n in (1, 2, 3):
                pages = rand_pages(n, 40 + n)
                got = partition.crypt_pages_multi(keys, engines, BASE, 2, pages)
                assert np.array_equal(got, C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=2))
        finally:
            for k in keys:
                k.destroy()
            for e in engines:
                e.destroy()

    @pytest.mark.parametrize("n", [0, 1, 5])
    def test_tiny_and_empty_device_batches_every_kernel(self, dkey, n, knob):
        import torch

        for kernel in (1, 2, 3, 4, 5, 6, 9):
            knob("kernel", kernel)
            pages = rand_pages(n, 50 + n) if n else np.empty((0, 4096), np.uint8)
            got = pc.crypt_pages(dkey, BASE, 3, torch.from_numpy(pages).cuda())
            torch.cuda.synchronize()
            want = C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=3) if n else pages
            assert np.array_equal(got.cpu().numpy(), want), kernel


_FIRST_USE_CHILD = r"""
import sys, threading
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2004_09252_b200 as pc
from oracle import coracle as C
KEY = bytes(range(32))
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
dkey = pc.DeviceKey.install(KEY, 0)
n_threads = 24
bar = threading.Barrier(n_threads)
bad = []
def run(t):
    rng = np.random.default_rng(t)
    r = (8, 12, 20)[t % 3]
    n = (1, 64, 700)[(t // 3) % 3]
    pages = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
    s = torch.cuda.Stream()
    d = torch.from_numpy(pages).cuda()
    torch.cuda.synchronize()
    try:
        bar.wait()
        if t % 2:
            with torch.cuda.stream(s):
                got = pc.crypt_pages(dkey, 0x10000, t, d, rounds=r, stream=s)
            s.synchronize()
            got = got.cpu().numpy()
        else:
            got = np.asarray(pc.crypt_pages(dkey, 0x10000, t, pages, rounds=r))
        if not np.array_equal(got, C.crypt_pages(KEY, None, None, pages, rounds=r, vaddr0=0x10000, pid0=t)):
            bad.append((t, "mismatch"))
    except Exception as e:
        bad.append((t, repr(e)))
th = [threading.Thread(target=run, args=(t,)) for t in range(n_threads)]
[x.start() for x in th]; [x.join() for x in th]
print("BAD", bad)
"""


@pytest.mark.parametrize("attempt", range(3))
def test_concurrent_first_use_in_fresh_process(cuda, attempt):
    """24 threads make their FIRST library call at the same instant (a
    barrier), across round counts and host/device buffers, in a fresh
    interpreter.  Regression for the lazily cached launch geometry
    (pagecrypt.cu pages_grid): a racing thread once read the SM count set
    but the occupancy still 0 and launched a grid of 0 CTAs."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _FIRST_USE_CHILD.format(root=root)], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "BAD []", out.stdout[-2000:]
