"""The N>1 path on CPU: two gloo ranks run the bench's weak-scaling plan
(partition.rank_pages), each crypts its own page range (with the C oracle
standing in for the GPU, test-side only), and the gathered shards must equal
the single-process result; max_over_ranks must return the slowest rank's time.
No page data crosses ranks in the product path -- the all_gather here is the
test's checker."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEY = bytes(range(32))
BASE = 0x1_0000_0000
PER_RANK = 96


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, rounds, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import coracle
    from paper_2004_09252_b200.partition import max_over_ranks, rank_pages

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi, vaddr0 = rank_pages(PER_RANK, rank, world, BASE)
        rng = np.random.default_rng(123)
        job = rng.integers(0, 256, size=(PER_RANK * world, 4096), dtype=np.uint8)
        mine = coracle.crypt_pages(KEY, None, None, job[lo:hi], rounds=rounds, vaddr0=vaddr0, pid0=1)
        parts = [torch.empty((hi - lo, 4096), dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        t = max_over_ranks(1.0 + rank)
        if rank == 0:
            whole = coracle.crypt_pages(KEY, None, None, job, rounds=rounds, vaddr0=BASE, pid0=1)
            q.put((bool(np.array_equal(torch.cat(parts).numpy(), whole)), t, (lo, hi, vaddr0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rounds", [8, 20])
def test_two_rank_partition_matches_single_process(rounds):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rounds, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    equal, tmax, plan0 = q.get(timeout=5)
    assert equal
    assert tmax == 2.0
    assert plan0 == (0, PER_RANK, BASE)


def test_rank_pages_plan():
    from paper_2004_09252_b200.partition import rank_pages

    assert rank_pages(10, 0, 1, BASE) == (0, 10, BASE)
    assert rank_pages(10, 3, 4, BASE) == (30, 40, BASE + 30 * 4096)
    from paper_2004_09252_b200.errors import ContractViolation

    with pytest.raises(ContractViolation):
        rank_pages(10, 1, 2, 2**64 - 4096 * 5)
