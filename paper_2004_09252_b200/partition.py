"""Multi-GPU page-range partitioner (no collective on the data path).

Each block's keystream depends only on (key, vaddr, pid, block index)
(pkg/src/pagecrypt/cipher.py:133-141), so any partition of a batch is
bit-identical to processing it in one piece -- the same property the
reference shows for 1 vs 8 workers (pkg/tests/test_workers.py:136-148).  The
reference routes whole clients to workers (``WorkerPool.route``,
pkg/src/pagecrypt/workers.py:204-206); for page batches the B200 analog is a
contiguous page range per GPU, each GPU holding its own copy of the key (the
per-worker key slots, workers.py:167-169,193-195).

Two launch shapes:

* one process per GPU (torchrun): :func:`shard` gives rank r its range; the
  only cross-rank traffic is the benchmark's barrier and max-over-ranks time
  (:func:`max_over_ranks`), never page data;
* one process, several GPUs: :func:`crypt_pages_multi` drives
  ``pc_crypt_pages_multi`` (one host thread per device) over host-resident
  pages, or over pages resident on one GPU whose ranges the other GPUs pull
  over NVLink peer-to-peer and return the same way.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .engine import DeviceKey, Engine, _host_pids, _host_vaddrs, PAGE_SIZE
from .errors import ContractViolation


def page_ranges(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) ranges, sizes differing by at most one page."""
    if parts < 1:
        raise ContractViolation(f"parts must be >= 1, got {parts}")
    if n < 0:
        raise ContractViolation("negative page count")
    return [(n * g // parts, n * (g + 1) // parts) for g in range(parts)]


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    if not 0 <= rank < world:
        raise ContractViolation(f"rank {rank} outside world of {world}")
    return page_ranges(n, world)[rank]


def rank_pages(pages_per_rank: int, rank: int, world: int, base_vaddr: int) -> tuple[int, int, int]:
    """Weak-scaling plan of the multi-GPU bench: the job is world *
    pages_per_rank pages at contiguous vaddrs from base_vaddr, rank r owns
    global pages [lo, hi) and therefore vaddrs from base_vaddr + 4096*lo.
    Returns (lo, hi, vaddr0)."""
    lo, hi = shard(pages_per_rank * world, rank, world)
    vaddr0 = base_vaddr + PAGE_SIZE * lo
    if vaddr0 % PAGE_SIZE or vaddr0 + PAGE_SIZE * max(hi - lo - 1, 0) >= 2**64:
        raise ContractViolation("rank's vaddr range is not a valid u64 page range")
    return lo, hi, vaddr0


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (the bench's
    timing reduction); identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def crypt_pages_multi(keys: list[DeviceKey], engines: list[Engine], vaddrs, pids,
                      pages, out=None, *, rounds: int = 20):
    """A batch split by contiguous page range over len(engines) devices
    (keys[g] must live on engines[g]'s device), no collective.

    ``pages`` is host memory (numpy / buffer: PCIe to every GPU), or a CUDA
    tensor resident on one GPU: that GPU ciphers its own range in place and
    every other range crosses NVLink peer-to-peer to its GPU and back
    (SURVEY §8e).  vaddrs/pids: int or host arrays.  Synchronous."""
    if len(keys) != len(engines) or not engines:
        raise ContractViolation("need one key per engine")
    for k, e in zip(keys, engines):
        if k.device != e.device:
            raise ContractViolation(f"key on device {k.device}, engine on {e.device}")
    if type(pages).__module__.startswith("torch") and pages.is_cuda:
        import torch

        if pages.dtype != torch.uint8 or not pages.is_contiguous() or pages.numel() % PAGE_SIZE:
            raise ContractViolation("device pages must be a contiguous uint8 tensor of whole pages")
        n = pages.numel() // PAGE_SIZE
        if out is None:
            out = torch.empty_like(pages)
        elif not (out.is_cuda and out.dtype == torch.uint8 and out.is_contiguous() and out.numel() == pages.numel()):
            raise ContractViolation("out must be a contiguous uint8 CUDA tensor like pages")
        # the library's streams must see the producer's writes
        torch.cuda.current_stream(pages.device).synchronize()
        if out.device != pages.device:
            torch.cuda.current_stream(out.device).synchronize()
        src, dst = pages.data_ptr(), out.data_ptr()
    else:
        arr = np.ascontiguousarray(pages, dtype=np.uint8).reshape(-1, PAGE_SIZE)
        n = arr.shape[0]
        if out is None:
            out = np.empty_like(arr)
        elif not (isinstance(out, np.ndarray) and out.dtype == np.uint8 and out.flags.c_contiguous
                  and out.flags.writeable and out.nbytes == n * PAGE_SIZE):
            raise ContractViolation("out must be a writable C-contiguous uint8 array of n*4096 bytes")
        src, dst = arr.ctypes.data, out.ctypes.data
    v_arr, vaddr0 = _host_vaddrs(vaddrs, n)
    p_arr, pid0 = _host_pids(pids, n)
    G = len(engines)
    eh = (ctypes.c_void_p * G)(*[e.handle for e in engines])
    kh = (ctypes.c_void_p * G)(*[k.handle for k in keys])
    _native.call("pc_crypt_pages_multi", eh, kh, G,
                 None if v_arr is None else v_arr.ctypes.data,
                 None if p_arr is None else p_arr.ctypes.data,
                 vaddr0, pid0, src, dst, n, rounds)
    return out


def replicated_keys(key: DeviceKey, devices: list[int]) -> list[DeviceKey]:
    """One key per device for :func:`crypt_pages_multi`: ``key`` itself on
    its own device, device-to-device replicas elsewhere (never via host RAM;
    workers.py:193-194 fills every worker slot from one staged key)."""
    return [key if d == key.device else key.replicate(d) for d in devices]


def shared_key(device: int, *, group=None, src: int = 0) -> DeviceKey:
    """One production key shared by every rank of the default process group
    (one process per GPU).  Rank ``src`` derives it on its GPU
    (DeviceKey.generate: never in host RAM) and exports a CUDA-IPC handle of a
    device copy; the handle (an opaque name of device memory, not key
    material) is broadcast, every other rank copies the key device-to-device
    onto ``device``, and after a barrier the exporter zeroes its export.
    Collective: every rank must call it.  Without an initialised process
    group it is DeviceKey.generate(device)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return DeviceKey.generate(device)
    rank = dist.get_rank(group)
    key = DeviceKey.generate(device) if rank == src else None
    box = [key.export_handle() if key is not None else None]
    dist.broadcast_object_list(box, src=src, group=group)
    err = None
    if key is None:
        try:
            key = DeviceKey.import_handle(box[0], device)
        except Exception as exc:  # keep the collective schedule; raise after the barrier
            err = exc
    dist.barrier(group=group)
    if rank == src:
        key.close_export()
    if err is not None:
        raise err
    return key
