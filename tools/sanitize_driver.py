"""Small invocations of every kernel for compute-sanitizer (memcheck,
racecheck, synccheck): each page-kernel variant x rounds on ragged batches,
in place and with per-page descriptors, the host paths, the keystream seams,
the worker service, the HBM store and its resident worker, and the key's
resident workers.  Checks results against the oracle
too, so a sanitizer run is also a parity run."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_09252_b200 as pc  # noqa: E402
from paper_2004_09252_b200 import _native  # noqa: E402
from paper_2004_09252_b200.store import DevicePageStore  # noqa: E402
from paper_2004_09252_b200.workers import ClientId, WorkerPool  # noqa: E402
from oracle import coracle as C  # noqa: E402

KEY = bytes(range(32))
# page-kernel variants to run (argv[1], comma-separated; default all)
KERNELS = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (1, 2, 3, 4, 5, 6, 9)


def main():
    rng = np.random.default_rng(0)
    n = 37
    pages = rng.integers(0, 256, size=(n, 4096), dtype=np.uint8)
    va = (np.arange(n, dtype=np.uint64)[::-1] * np.uint64(4096) + np.uint64(0xFFFF_F000_0000)).copy()
    pi = (np.arange(n) % 5).astype(np.uint32)
    with pc.DeviceKey.install(KEY, 0) as k:
        for kern in KERNELS:
            print("kernel", kern, flush=True)
            _native.tune("kernel", kern)
            for r in (8, 12, 20):
                d = torch.from_numpy(pages).cuda()
                pc.crypt_pages(k, 0x1_0000_0000, 3, d, out=d, rounds=r)
                want = C.crypt_pages(KEY, None, None, pages, rounds=r, vaddr0=0x1_0000_0000, pid0=3)
                assert np.array_equal(d.cpu().numpy(), want), (kern, r)
                # every descriptor shape (vaddr array and/or pid array)
                dva = torch.from_numpy(va.view(np.int64)).cuda()
                dpi = torch.from_numpy(pi.view(np.int32)).cuda()
                # v5's descriptor loops: strided (run_desc 0), page runs (1), runs with two blocks per thread (2)
                for rd in ((0, 1, 2) if kern == 5 else (1,)):
                    _native.tune("run_desc", rd)
                    for v_arg, p_arg, v_ref, p_ref in ((dva, dpi, va, pi), (dva, 7, va, np.full(n, 7, np.uint32)),
                                                       (0x5000, dpi, 0x5000 + 4096 * np.arange(n, dtype=np.uint64), pi)):
                        got = pc.crypt_pages(k, v_arg, p_arg, torch.from_numpy(pages).cuda(), rounds=r)
                        want = C.crypt_pages(KEY, v_ref, p_ref, pages, rounds=r)
                        assert np.array_equal(got.cpu().numpy(), want), (kern, r, rd)
                _native.tune("run_desc", 1)
        _native.tune("kernel", 0)
        print("host paths", flush=True)
        for hm in (0, 1, 2, 3):
            _native.tune("host_mode", hm)
            src = torch.from_numpy(np.concatenate([pages] * 3)).pin_memory()
            out = torch.empty_like(src).pin_memory()
            eng = pc.Engine(0, n_streams=3, chunk_pages=16)
            pc.crypt_pages(k, 0x2000, 1, src, out=out, engine=eng)
            eng.destroy()
            assert np.array_equal(out.numpy(), C.crypt_pages(KEY, None, None, src.numpy(), vaddr0=0x2000, pid0=1))
        _native.tune("host_mode", 2)
        assert pc.crypt_page(KEY, 0x3000, 9, pages[0].tobytes()) == C.crypt_pages(KEY, [0x3000], 9, pages[:1])[0].tobytes()
        assert pc.page_keystream(KEY, 0x3000, 9)[:64] == C.crypt_pages(KEY, [0x3000], 9, np.zeros((1, 4096), np.uint8))[0, :64].tobytes()
        print("store", flush=True)
        st = DevicePageStore(64, k)
        st.evict_many(ClientId(5, 0), va[:20], pages[:20])
        back = st.refault_many(ClientId(5, 0), va[:20])
        assert np.array_equal(back, pages[:20])
        # one fused fault (refault + eviction in one launch, pc_store_swap)
        st.evict_many(ClientId(5, 0), va[:3], pages[:3])
        got = st.swap(ClientId(5, 0), va[:3], va[3:7], pages[3:7])
        assert np.array_equal(got, pages[:3])
        assert np.array_equal(st.refault_many(ClientId(5, 0), va[3:7]), pages[3:7])
        # single faults as tickets of the store's resident worker (pc_store_service):
        # first touch + eviction, refault + eviction, refault only, full-slab slot reuse
        print("store service", flush=True)
        st2 = DevicePageStore(2, k)
        st2.start_service()
        c5, out1 = ClientId(5, 0), np.zeros(4096, np.uint8)
        assert not st2.fault(c5, 0x9000, out1, 0xA000, pages[0])
        assert not st2.fault(c5, 0xB000, out1, 0xC000, pages[1])
        assert st2.fault(c5, 0xA000, out1, 0xD000, pages[2]) and np.array_equal(out1, pages[0])
        assert st2.fault(c5, 0xC000, out1) and np.array_equal(out1, pages[1])
        # (a sanitizer serialises kernels: no launch may run beside a resident worker)
        st2.stop_service()
        assert st2.lookup(c5, 0xD000) == C.crypt_pages(KEY, [0xD000], 5, pages[2:3])[0].tobytes()
        st2.close()
        st.close()
        # 1-2 page host calls on the key's resident workers (pc_key_service)
        print("key service", flush=True)
        k.start_service(n_workers=4)
        for m in (1, 2, 4):  # <= 1 page per worker: every call is service tickets, no launch
            got = pc.crypt_pages(k, 0x4000, 6, pages[:m])
            assert np.array_equal(got, C.crypt_pages(KEY, None, None, pages[:m], vaddr0=0x4000, pid0=6))
        k.stop_service()
    print("worker pool", flush=True)
    pool = WorkerPool(n_workers=3, keysource=lambda m: KEY)
    for i in range(12):
        buf = bytearray(pages[i].tobytes())
        pool.crypt(ClientId(7, 0), 4096 * i, "encrypt", type("P", (), {"data": buf})())
        assert bytes(buf) == C.crypt_pages(KEY, [4096 * i], 7, pages[i:i + 1])[0].tobytes()
    pool.shutdown()
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
