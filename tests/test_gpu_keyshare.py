"""One key across GPUs and processes (SURVEY §8e "the key is replicated into
each device's memory"; reference: the staged key copied into every worker
slot, pkg/src/pagecrypt/workers.py:193-194).  A production key
(DeviceKey.generate) never exists in host RAM, so the only way to check a
replica is through ciphertext: the replica must produce exactly the
source key's pages, and a split batch must equal the single-GPU batch
(pkg/tests/test_workers.py:136-148).  Cross-device copies cannot run on the
one-GPU test box; same-device replication and cross-PROCESS export/import
(CUDA IPC between two processes on cuda:0) exercise the same entry points."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import partition
from paper_2004_09252_b200.errors import ContractViolation, PageCryptError

from oracle import coracle as C

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEY = bytes(range(32))
BASE = 0x1_0000_0000


def rand_pages(n, seed=3):
    return np.random.default_rng(seed).integers(0, 256, size=(n, 4096), dtype=np.uint8)


def test_replicate_same_device_matches_source(cuda):
    pages = rand_pages(100)
    with pc.DeviceKey.generate(0) as k:
        r = k.replicate(0)
        try:
            a = pc.crypt_pages(k, BASE, 7, pages)
            b = pc.crypt_pages(r, BASE, 7, pages)
            assert np.array_equal(a, b) and not np.array_equal(a, pages)
        finally:
            r.destroy()
        # the source still works after the replica is gone
        assert np.array_equal(pc.crypt_pages(k, BASE, 7, pages), a)


def test_replicate_installed_key_against_oracle(cuda):
    pages = rand_pages(65)
    with pc.DeviceKey.install(KEY, 0) as k, k.replicate(0) as r:
        assert np.array_equal(pc.crypt_pages(r, BASE, 1, pages),
                              C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=1))


def test_replicate_bad_device(cuda):
    import torch

    with pc.DeviceKey.install(KEY, 0) as k:
        with pytest.raises(ContractViolation):
            k.replicate(torch.cuda.device_count())
        with pytest.raises(ContractViolation):
            k.replicate(-1)


def test_split_with_replicated_keys_equals_single(cuda):
    """crypt_pages_multi over engines with replicated keys == one call."""
    pages = rand_pages(301)
    engines = [pc.Engine(0), pc.Engine(0, n_streams=3)]
    with pc.DeviceKey.generate(0) as k:
        keys = partition.replicated_keys(k, [e.device for e in engines])
        assert keys[0] is k and keys[1] is k  # same device: the key itself
        whole = pc.crypt_pages(k, BASE, 2, pages)
        split = partition.crypt_pages_multi(keys, engines, BASE, 2, pages)
        assert np.array_equal(whole, split)
    for e in engines:
        e.destroy()


_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2004_09252_b200 as pc
h = bytes.fromhex(sys.argv[2])
pages = np.random.default_rng(3).integers(0, 256, size=(77, 4096), dtype=np.uint8)
if sys.argv[3] == "expect_fail":
    try:
        pc.DeviceKey.import_handle(h, 0)
    except pc.PageCryptError:
        print("import refused"); sys.exit(0)
    print("import unexpectedly succeeded"); sys.exit(1)
with pc.DeviceKey.import_handle(h, 0) as k:
    out = pc.crypt_pages(k, 0x100000000, 9, pages)
np.save(sys.argv[3], out)
print("child ok")
"""


def _child(handle, arg):
    return subprocess.run([sys.executable, "-c", _CHILD, ROOT, handle.hex(), arg], capture_output=True, text=True,
                          timeout=300)


def test_export_import_across_processes(cuda, tmp_path):
    pages = rand_pages(77)
    with pc.DeviceKey.generate(0) as k:
        h = k.export_handle()
        assert len(h) == 64 and k.export_handle() == h  # idempotent while open
        r = _child(h, str(tmp_path / "ct.npy"))
        assert r.returncode == 0, r.stdout + r.stderr
        k.close_export()
        want = pc.crypt_pages(k, BASE, 9, pages)
    got = np.load(tmp_path / "ct.npy")
    assert np.array_equal(got, want)


def test_closed_export_is_zeroed(cuda, tmp_path):
    """After close the exported buffer holds zeros (it is recycled, never
    freed, because cudaFree would wait on a running service): a stale handle
    yields the all-zero key, never the real one."""
    with pc.DeviceKey.install(KEY, 0) as k:
        h = k.export_handle()
        k.close_export()
        k.close_export()  # idempotent
        r = _child(h, str(tmp_path / "stale.npy"))
        assert r.returncode == 0, r.stdout + r.stderr
    pages = rand_pages(77)
    got = np.load(tmp_path / "stale.npy")
    assert np.array_equal(got, C.crypt_pages(bytes(32), None, None, pages, vaddr0=BASE, pid0=9))
    assert not np.array_equal(got, C.crypt_pages(KEY, None, None, pages, vaddr0=BASE, pid0=9))


def test_destroy_closes_a_live_export(cuda, tmp_path):
    k = pc.DeviceKey.install(KEY, 0)
    h = k.export_handle()
    k.destroy()
    r = _child(h, str(tmp_path / "after.npy"))
    assert r.returncode == 0, r.stdout + r.stderr
    got = np.load(tmp_path / "after.npy")
    assert np.array_equal(got, C.crypt_pages(bytes(32), None, None, rand_pages(77), vaddr0=BASE, pid0=9))


def test_import_garbage_handle_fails(cuda):
    with pytest.raises(PageCryptError):
        pc.DeviceKey.import_handle(bytes(64), 0)
    with pytest.raises(ContractViolation):
        pc.DeviceKey.import_handle(b"x", 0)


def test_engine_placement_reported(cuda):
    e = pc.Engine(0)
    try:
        p = e.placement
        assert set(p) == {"numa_node", "bound_cpus"}
        assert p["numa_node"] >= -1 and p["bound_cpus"] >= 0
        if p["numa_node"] < 0:
            assert p["bound_cpus"] == 0
    finally:
        e.destroy()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


_RANK = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import partition
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
torch.cuda.set_device(0)
key = partition.shared_key(0)
pages = np.random.default_rng(5).integers(0, 256, size=(96, 4096), dtype=np.uint8)
lo, hi = partition.shard(96, rank, world)
mine = torch.from_numpy(pc.crypt_pages(key, 0x100000000 + 4096 * lo, 1, pages[lo:hi]))
parts = [torch.empty_like(mine) for _ in range(world)]
dist.all_gather(parts, mine)
if rank == 0:
    whole = pc.crypt_pages(key, 0x100000000, 1, pages)
    print("SPLIT_EQUAL", bool(np.array_equal(torch.cat(parts).numpy(), whole)))
key.destroy()
dist.destroy_process_group()
"""


def test_shared_key_two_ranks_split_equals_whole(cuda, tmp_path):
    """partition.shared_key over two gloo ranks on cuda:0: rank 0 generates,
    rank 1 imports over CUDA IPC; the gathered shards equal rank 0's
    single-call ciphertext of the whole batch."""
    script = tmp_path / "rank.py"
    script.write_text(_RANK)
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(script), ROOT],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SPLIT_EQUAL True" in r.stdout, r.stdout
