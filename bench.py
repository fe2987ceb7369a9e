#!/usr/bin/env python3
"""Benchmark of the B200 page-cipher engine (BASELINE.json metric: GB/s of
4 KiB pages en/decrypted).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--rounds R] [--pages P]
    python bench.py --impl reference ...      # the reference CPU path

Workload (BASELINE.json configs[1]): a 1 GiB batch (262,144 pages) of random
4 KiB pages resident in HBM, ChaCha20, contiguous vaddrs from BASE_VADDR
(pkg/src/pagecrypt/client.py:42), pid 1.  One step = one pass of the hot path
over the batch = one crypt_pages() call = one kernel launch.  At N GPUs each
rank owns its own 1 GiB page range (weak scaling, no collective on the data
path); the only cross-rank traffic is the barrier and the max-over-ranks time.

value    device-resident GB/s (CUDA events on the launching stream, inputs
         already in HBM, 1 GiB > 126 MB L2 so no flush is needed)
e2e      the same metric through the public host API (pinned host pages; the
         H2D copy, cipher and D2H copy of every page are inside the timed region)
roofline the crypt kernel against min(ALU-pipe roof for the ARX op count --
         measured LOP3 issue rate over the xor/rotate ops per byte -- and the
         HBM roof for 8 B/page-byte), both measured on this GPU in this run
cpu_baseline  the oracle port (oracle/liboracle.so, scalar C, one page per call
         like cipher.crypt_page) on all host cores, rank 0 at N=1, bounded sample
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASE_VADDR = 0x1_0000_0000
PAGE = 4096
METRIC = "GB/s of pages en/decrypted (device-resident and host-resident) at 1/2/4/8 B200"


def ops_per_page(rounds: int) -> int:
    """Op-count convention: 12 int32 ops per quarter round,
    4*R quarter rounds per block, + 16 feed-forward adds + 16 data XORs."""
    return 64 * (48 * rounds + 32)


def alu_ops_per_page(rounds: int) -> int:
    """The part of ops_per_page that must issue to the ALU pipe: per quarter
    round 4 xors (LOP3) + 4 rotates (PRMT for 16/8, SHF.L.W for 12/7), plus
    the 16 data xors per block.  The 16R+16 adds go to the FMA pipe
    (IMAD.IADD) in parallel and never bind."""
    return 64 * (32 * rounds + 16)


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    """SM clock, power and clock-event reasons sampled every few ms by NVML
    (nvidia-smi's source) in a background thread during the timed region --
    fast enough for regions of a few tens of ms.  Falls back to nvidia-smi."""

    REASONS = {  # NVML clock-event bits we report
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4,
    }

    def __init__(self, gpu_index: int, period_s: float = 0.002):
        self.gpu = gpu_index
        self.period = period_s
        self.samples: list[tuple[float, float, float, int]] = []
        self._stop = threading.Event()
        self._nvml = None
        self.pci = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = None
            try:  # the CUDA device's own PCI address: NVML indices ignore CUDA_VISIBLE_DEVICES
                import torch

                p = torch.cuda.get_device_properties(self.gpu)
                bdf = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bdf)
                self.pci = bdf
            except Exception:
                pass
            if self._h is None:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
        return self

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((time.perf_counter(), float(sm), pw, int(rs)))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "unavailable"}
        sm = [x[1] for x in self.samples]
        reasons = sorted({name for _, _, _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "power_w_max": round(max(x[2] for x in self.samples), 1),
                "samples": len(sm), "source": "NVML every %g ms during the timed region" % (1e3 * self.period),
                "nvml_device": self.pci or f"index {self.gpu}"}


# ---------------------------------------------------------------------------
# CPU legs (oracle port; the reference itself is Python and does not travel)


def cpu_port_rate(rounds: int, target_s: float, threads: int, pages_per_batch: int = 4096) -> dict:
    """Time the oracle port (scalar C, one page per call as cipher.crypt_page)
    on `threads` host threads over batches of the bench workload."""
    from oracle import coracle

    rng = np.random.default_rng(1)
    pages = rng.integers(0, 256, size=(pages_per_batch, PAGE), dtype=np.uint8)
    out = np.empty_like(pages)
    key = np.random.default_rng(0).bytes(32)
    coracle.crypt_pages(key, None, None, pages[:64], rounds=rounds, vaddr0=BASE_VADDR, pid0=1)
    done, t0 = 0, time.perf_counter()
    while True:
        coracle.crypt_pages(key, None, None, pages, rounds=rounds, nthreads=threads, out=out,
                            vaddr0=BASE_VADDR + PAGE * done, pid0=1)
        done += pages_per_batch
        el = time.perf_counter() - t0
        if el >= target_s:
            break
    return {"value": done * PAGE / el / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{done} pages ({done * PAGE / 2**20:.0f} MiB) of the bench workload "
                      f"(ChaCha{rounds}, contiguous vaddrs, pid 1) in {el:.1f} s on {threads} host "
                      f"threads; oracle/chacha_oracle.c, one page per call like cipher.crypt_page",
            "cpu": _cpu_model()}


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_cpu(cores: int, n_pages: int, warmup: int, steps: int | None, seconds: float | None,
                  extras: bool = True) -> dict | None:
    """The reference's own CPU path (oracle/_ref snapshot, numba kernel) on
    this host: (ii) crypt_page on one process per core is the value; (i) one
    thread and (iii) WorkerPool(cores) ride along.  None when the reference
    or numba is unavailable on this host."""
    from oracle import ref_bench

    ref = ref_bench.load()
    if ref is None:
        return None
    pool = ref_bench.ProcessPool(cores, n_pages)
    try:
        for i in range(warmup):
            pool.step(BASE_VADDR + PAGE * n_pages * i)
        times, i = [], 0
        while True:
            times.append(pool.step(BASE_VADDR + PAGE * n_pages * (warmup + i)))
            i += 1
            if (steps is not None and i >= steps) or (seconds is not None and sum(times) >= seconds):
                break
        ok = ref_bench.check_sample(ref, pool.out, pool.inp, BASE_VADDR + PAGE * n_pages * (warmup + i - 1))
    finally:
        pool.close()
    total = sum(times)
    res = {"value": len(times) * n_pages * PAGE / total / 1e9, "unit": "GB/s", "cores": cores, "kind": "reference",
           "steps": len(times), "seconds": round(total, 3), "spot_check_ok": ok,
           "sample": (f"{len(times)} x {n_pages} pages ({n_pages * PAGE / 2**20:.0f} MiB each) of the bench "
                      f"workload (ChaCha20, contiguous vaddrs, pid 1): the UNMODIFIED reference "
                      f"pagecrypt.cipher.crypt_page (numba kernel, oracle/_ref snapshot of "
                      f"/root/reference/pkg/src) on {cores} forked processes, one contiguous slice each; "
                      "1 GiB / 64 GiB figures would be rate-extrapolated"),
           "cpu": _cpu_model(), "what": "(ii) crypt_page x one process per core"}
    if extras:
        one = ref_bench.single_thread(ref, seconds=3.0)
        res["single_thread"] = {"value": round(one["value"], 4), "unit": "GB/s", "cores": 1,
                                "us_per_page": round(one["us_per_page"], 2),
                                "what": "(i) crypt_page, one thread, one page per call"}
        wp = ref_bench.worker_pool(ref, cores, seconds=3.0)
        res["worker_pool"] = {"value": round(wp["value"], 4), "unit": "GB/s", "cores": cores,
                              "crypt_1page_p50_us": round(wp["crypt_1page_p50_us"], 2),
                              "crypt_1page_p99_us": round(wp["crypt_1page_p99_us"], 2),
                              "what": "(iii) WorkerPool(n_workers=cores): submit/wait batches of 512 "
                                      "pages from clients pid 1..64; crypt() 1-page latency"}
        res["crypt_page_latency_us"] = ref_bench.crypt_page_latency(ref)
    return res


def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference's own CPU implementation of the path
    on the box's host cores, rank 0 only (the other ranks exit 0).

    The reference is a Python package; oracle/_ref holds an unmodified
    snapshot of it (oracle/fetch_ref.py) that travels to the box, and its
    numba kernel is JIT-compiled here.  Each step is a bounded sample
    (--ref-pages pages) across one process per host core.  Falls back to
    the C port of it (oracle/chacha_oracle.c, kind "port") only when the
    snapshot or numba is missing."""
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    res = None
    if args.rounds == 20:  # the reference is ChaCha20 only (cipher.py:158)
        res = reference_cpu(threads, args.ref_pages, args.warmup, args.steps, None)
    if res is not None:
        value, total = res["value"], res["seconds"]
        cb = dict(res)
    else:
        from oracle import coracle

        n_sample = args.ref_pages
        rng = np.random.default_rng(1)
        pages = rng.integers(0, 256, size=(n_sample, PAGE), dtype=np.uint8)
        out = np.empty_like(pages)
        key = np.random.default_rng(0).bytes(32)
        for _ in range(args.warmup):
            coracle.crypt_pages(key, None, None, pages, rounds=args.rounds, nthreads=threads, out=out,
                                vaddr0=BASE_VADDR, pid0=1)
        times = []
        for i in range(args.steps):
            t0 = time.perf_counter()
            coracle.crypt_pages(key, None, None, pages, rounds=args.rounds, nthreads=threads, out=out,
                                vaddr0=BASE_VADDR + PAGE * n_sample * i, pid0=1)
            times.append(time.perf_counter() - t0)
        total = sum(times)
        value = args.steps * n_sample * PAGE / total / 1e9
        cb = {"value": value, "unit": "GB/s", "cores": threads, "kind": "port", "cpu": _cpu_model(),
              "sample": (f"each step {n_sample} pages ({n_sample * PAGE / 2**20:.0f} MiB) of the "
                         f"{args.pages}-page workload, ChaCha{args.rounds}, {threads} host threads, "
                         "oracle/chacha_oracle.c (port of cipher.crypt_page): the reference snapshot "
                         "(oracle/_ref) or numba is unavailable here, or rounds != 20")}
    cb["value"] = round(value, 4)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": cb,
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world: int) -> dict:
    return {"workload": f"{args.pages * PAGE / 2**30:g} GiB device-resident batch of 4 KiB pages per GPU, "
                        f"ChaCha{args.rounds} (BASELINE configs[1])",
            "pages_per_gpu": args.pages, "rounds": args.rounds, "vaddrs": "contiguous from 0x100000000",
            "pid": 1, "parallelism": f"page-range x{world} (no collective)",
            "key": "one DeviceKey.generate on rank 0, shared with every rank device-to-device (CUDA IPC)",
            "l2": "inputs (1 GiB) larger than the 126 MB L2; no flush"}


# ---------------------------------------------------------------------------


def self_launch(args) -> int:
    """bench.py --gpus N without torchrun: launch N ranks of this script
    through torch.distributed.run on 127.0.0.1 and return its exit code (the
    ranks' output passes straight through; rank 0 prints the line)."""
    import socket
    import subprocess

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=20, choices=(8, 12, 20))
    ap.add_argument("--pages", type=int, default=262_144, help="pages per GPU (default 1 GiB)")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--ref-pages", type=int, default=16384, help="reference arm: pages per step")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sweep-gib", type=float, default=64.0,
                    help="config 5: GiB split by page range over the ranks (0 = skip)")
    ap.add_argument("--sustain-s", type=float, default=1.0, help="seconds per round count in the sustained leg")
    ap.add_argument("--no-extras", action="store_true", help="skip every extras leg")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"),
                    help="process-group backend for the barrier/max-time (gloo: test mode)")
    ap.add_argument("--same-device", action="store_true",
                    help="test mode: every rank uses cuda:0 (multi-rank logic on one GPU; needs gloo)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.same_device and world > 1 and args.dist_backend == "nccl":
        ap.error("--same-device needs --dist-backend gloo (NCCL refuses two ranks on one GPU)")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return 0

    import torch
    import torch.distributed as dist

    import paper_2004_09252_b200 as pc
    from paper_2004_09252_b200 import _native
    from paper_2004_09252_b200.partition import max_over_ranks, rank_pages, shared_key

    if args.same_device:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    red_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    placement = _bind_near_gpu(local_rank)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    n = args.pages
    # this rank's page range: disjoint vaddrs per rank (partition.shard of world*n)
    _, _, vaddr0 = rank_pages(n, rank, world, BASE_VADDR)
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    pages = torch.randint(0, 256, (n, PAGE), dtype=torch.uint8, device=dev, generator=g)
    out = torch.empty_like(pages)
    # production key path: derived on rank 0's GPU, never in host RAM, copied
    # device-to-device to every other rank (CUDA IPC export/import)
    key_note = None
    try:
        key = shared_key(local_rank)
    except Exception as exc:  # noqa: BLE001 -- keep the run measurable; the line says so
        # (shared_key is collective and raises only after its barrier, so the
        # ranks stay in step; split_parity then reports the mismatch)
        print(f"bench.py rank {rank}: shared key import failed ({exc}); using a per-rank key", file=sys.stderr)
        key = pc.DeviceKey.generate(local_rank)
        key_note = f"rank {rank} fell back to its own key: {exc}"
    if world > 1:
        flag = torch.tensor([0 if key_note is None else 1], dtype=torch.int32, device=red_dev)
        dist.all_reduce(flag)
        if int(flag.item()):
            key_note = key_note or f"{int(flag.item())} rank(s) fell back to their own key (CUDA IPC import failed)"
    stream = torch.cuda.current_stream(dev)

    def step(rounds, desc=None):
        v, p = (vaddr0, 1) if desc is None else desc
        pc.crypt_pages(key, v, p, pages, out=out, rounds=rounds, stream=stream, check=False)

    launches = {}

    def timed(rounds, steps, warmup, desc=None, tag=None):
        for _ in range(warmup):
            step(rounds, desc)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = _native.tune_get("launches")
        e0.record(stream)
        for _ in range(steps):
            step(rounds, desc)
        e1.record(stream)
        e1.synchronize()
        launches[tag or rounds] = _native.tune_get("launches") - l0  # counted by the library itself
        barrier()
        return e0.elapsed_time(e1)  # ms on the launching stream

    # integer roofline denominators, measured on this GPU now
    peaks = measure_int_peaks(_native, local_rank)

    with ClockSampler(local_rank) as clk:
        total_ms = timed(args.rounds, args.steps, args.warmup)
    t_max = max_over_ranks(total_ms, device=red_dev)
    bytes_per_step = n * PAGE
    value = world * bytes_per_step * args.steps / (t_max / 1e3) / 1e9
    kernel_ms = total_ms / args.steps  # one launch per step
    rl = roofline(args.rounds, kernel_ms, bytes_per_step, peaks, n)

    # e2e: the public host API on pinned host pages, copies inside the timed region
    host_in = torch.empty((n, PAGE), dtype=torch.uint8).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    host_in.copy_(pages)
    eng = pc.default_engine(local_rank)
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(3):
        pc.crypt_pages(key, vaddr0, 1, host_in, out=host_out, rounds=args.rounds, engine=eng)
    barrier()
    l0 = _native.tune_get("launches")
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        pc.crypt_pages(key, vaddr0, 1, host_in, out=host_out, rounds=args.rounds, engine=eng)
    e2e_s = time.perf_counter() - t0
    e2e_launches = _native.tune_get("launches") - l0
    e2e_s = max_over_ranks(e2e_s, device=red_dev)
    e2e = {"value": round(world * bytes_per_step * e2e_steps / e2e_s / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": bytes_per_step, "d2h_bytes_per_step": bytes_per_step,
           "steps": e2e_steps, "path": "crypt_pages(DeviceKey, pinned torch CPU tensors) -> "
           f"pc_crypt_pages_host, {eng.n_streams} streams x {eng.chunk_pages}-page chunks",
           "host_placement": eng.placement}
    del host_in, host_out  # the e2e buffers are done with; free before the extras

    extras = {}
    if not args.no_extras:
        for r in (8, 12):
            if r == args.rounds:
                continue
            ms = timed(r, max(5, args.steps // 2), 3) / max(5, args.steps // 2)
            t = max_over_ranks(ms, device=red_dev)
            extras[f"chacha{r}"] = {"value": round(world * bytes_per_step / (t / 1e3) / 1e9, 2),
                                    "unit": "GB/s", "roofline": roofline(r, ms, bytes_per_step, peaks, n),
                                    "parity": "the reference is ChaCha20-only: reduced rounds are pinned by "
                                              "published zero-key ChaCha8/12 blocks (tests/golden/rfc8439.json) "
                                              "and the round-parameterised oracle restatement"}
        extras["desc"] = desc_leg(torch, args, timed, n, rank, world, dev, bytes_per_step, peaks, red_dev,
                                  max_over_ranks)
        extras["sustained"] = sustained_leg(args, step, stream, torch, _native, local_rank, kernel_ms, rl,
                                            extras, peaks, bytes_per_step, barrier)
        extras["split_parity"] = split_parity(pc, key, torch, dist, world, rank, dev, args.dist_backend)
        if args.sweep_gib > 0:
            del out  # room for the sweep buffer
            extras["sweep"] = sweep_leg(pc, key, torch, args, rank, world, dev, barrier, max_over_ranks, red_dev)
            out = torch.empty_like(pages)
        if rank == 0:
            extras["latency_host_small"] = latency_sweep(pc, key, local_rank)
            extras["latency_service_1page"] = service_latency(local_rank)
            extras["hbm_store"] = store_throughput(pc, key, local_rank)
            extras["pager"] = pager_rate(pc, key, local_rank)

    cpu = None
    if rank == 0:
        cpu = cpu_baseline(args)

    key.destroy()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (uniform random pages, seed 1+rank; key from DeviceKey.generate on rank 0)",
            "config": dict(workload_config(args, world), **({"key": key_note} if key_note else {})),
            "roofline": rl, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches[args.rounds] + e2e_launches,
            "gpu_launches_detail": {"device_timed": launches[args.rounds], "e2e_timed": e2e_launches,
                                    "source": "libpagecrypt's own launch counter (pc_tune_get(\"launches\"))"},
            "clocks": clk.summary(), "gpu": torch.cuda.get_device_name(dev),
            "gpus_active": world if not args.same_device else 1, "rank0_placement": placement,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _bind_near_gpu(device: int) -> dict:
    """One process per GPU: run this rank on the CPUs local to its GPU's PCIe
    root, so torch's pinned buffers are first touched there too.
    No-op when the platform reports no NUMA node (single-socket VMs)."""
    import torch

    p = torch.cuda.get_device_properties(device)
    bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    res = {"pci": bdf, "numa_node": -1, "cpus": None}
    try:
        base = f"/sys/bus/pci/devices/{bdf}/"
        with open(base + "numa_node") as f:
            res["numa_node"] = int(f.read().strip())
        if res["numa_node"] < 0:
            return res
        with open(base + "local_cpulist") as f:
            cpus = _parse_cpulist(f.read())
        if cpus:
            os.sched_setaffinity(0, cpus)
            res["cpus"] = len(cpus)
    except (OSError, ValueError):
        pass
    return res


def _parse_cpulist(s: str) -> set[int]:
    out = set()
    for part in s.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        out.update(range(int(lo), int(hi or lo) + 1))
    return out


def measure_int_peaks(_native, device: int) -> dict:
    peaks = {}
    for kind, name in ((0, "lop3"), (1, "iadd3"), (2, "imad"), (3, "shf"), (4, "arx_mix")):
        v = _native.ctypes.c_double()
        _native.call("pc_intpeak", device, kind, _native.ctypes.byref(v))
        peaks[name] = v.value
    return peaks


def roofline(rounds, k_ms, bytes_per_step, peaks, n, kernel=None, desc=False):
    achieved = bytes_per_step / (k_ms / 1e3) / 1e9  # page GB/s of one launch
    opb = ops_per_page(rounds) / PAGE
    # ALU-pipe roof: the measured LOP3 issue rate (64 lanes/clk/SM) over
    # the ALU-pipe instructions per page byte
    int_roof = peaks["lop3"] / (alu_ops_per_page(rounds) / PAGE) / 1e9
    mix_roof = peaks["arx_mix"] / opb / 1e9
    hbm_peak, hbm_src = _hbm_peak()
    # each page byte is read once and written once; descriptors add 12 B/page
    bytes_per_page = 2 * PAGE + (12 if desc else 0)
    hbm_roof = hbm_peak / (bytes_per_page / PAGE)
    bound = "int32" if int_roof < hbm_roof else "hbm"
    peak = min(int_roof, hbm_roof)
    if kernel is None:
        kernel = "k_crypt_pages_coalesced<8>" if rounds == 8 else "k_crypt_pages_async<%d>" % rounds
    return {
        "bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 2), "unit": "GB/s",
        "frac": round(achieved / peak, 4), "traffic": _ncu_traffic(rounds, n, desc),
        "traffic_source": "profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum of one "
                          "ncu --set full capture of this kernel at this size (not re-measured in this run)",
        "kernel": kernel, "launch_ms": round(k_ms, 4),
        "int32": {"achieved_tops": round(achieved * 1e9 * opb / 1e12, 3),
                  "ops_per_page": ops_per_page(rounds), "alu_ops_per_page": alu_ops_per_page(rounds),
                  "alu_achieved_tops": round(achieved * 1e9 * alu_ops_per_page(rounds) / PAGE / 1e12, 3),
                  "alu_peak_tops": round(peaks["lop3"] / 1e12, 3), "roof_gbs": round(int_roof, 1),
                  "peak_source": "pc_intpeak(lop3): ALU-pipe issue rate measured in this run; the roof "
                                 "is that rate over the ALU-pipe ops per page (xor + rotate + data xor)",
                  "cross_check": {"arx_mix_tops": round(peaks["arx_mix"] / 1e12, 3),
                                  "arx_mix_roof_gbs": round(mix_roof, 1),
                                  "frac": round(achieved / mix_roof, 4),
                                  "what": "the reference quarter-round op stream at full ILP, no memory; "
                                          "the kernels hoist 3 of the 4R first-round quarter rounds out "
                                          "of the page loop, so they can exceed it"}},
        "hbm": {"achieved_gbs": round(achieved * bytes_per_page / PAGE, 1), "peak_gbs": hbm_peak,
                "peak_source": hbm_src, "algorithmic_bytes_per_page": bytes_per_page,
                "roof_gbs": round(hbm_roof, 1)},
        "measured_int_peaks_tops": {k: round(v / 1e12, 3) for k, v in peaks.items()},
    }


def desc_leg(torch, args, timed, n, rank, world, dev, bytes_per_step, peaks, red_dev, max_over_ranks) -> dict:
    """SURVEY §8(d) per-page variant: every page carries its own descriptor,
    as on the fault path (orchestrator.py:197-198,234-235): this rank's
    vaddrs in a random permutation (so no contiguity to exploit) and
    pid = 1 + i % 64, as device arrays (u64 vaddrs, u32 pids).  Same 1 GiB
    batch, one launch per step (k_crypt_pages_*<R, DM=3>)."""
    lo = rank * n
    gen = torch.Generator(device=dev).manual_seed(77 + rank)
    perm = torch.randperm(n, device=dev, generator=gen)
    vaddrs = (BASE_VADDR + PAGE * (lo + perm)).to(torch.int64)
    pids = (1 + torch.arange(n, device=dev) % 64).to(torch.int32)
    res = {"workload": "per-page descriptors: permuted vaddrs of this rank's range, pid = 1 + i % 64 "
                       "(u64/u32 device arrays); 1 GiB per GPU"}
    steps = max(5, args.steps // 2)
    for r in (20, 12, 8):
        ms = timed(r, steps, 3, desc=(vaddrs, pids), tag=f"desc{r}") / steps
        t = max_over_ranks(ms, device=red_dev)
        kern = {8: "k_crypt_pages_coalesced<8>", 12: "k_crypt_pages_run<12,3>", 20: "k_crypt_pages_async<20,3>"}[r]
        res[f"chacha{r}"] = {"value": round(world * bytes_per_step / (t / 1e3) / 1e9, 2), "unit": "GB/s",
                             "roofline": roofline(r, ms, bytes_per_step, peaks, n, kernel=kern, desc=True)}
    return res


def sustained_leg(args, step, stream, torch, _native, device, burst_ms, rl, extras, peaks, bytes_per_step,
                  barrier) -> dict:
    """Back-to-back launches for >= --sustain-s seconds per round count with
    NVML clocks/power sampled, beside the short burst of the headline; the
    LOP3 peak is re-measured right after each run (same thermal/power state)
    and the roofline is also scaled by the sustained/burst clock ratio."""
    res = {}
    for r in (20, 12, 8):
        ms_est = burst_ms if r == args.rounds else (
            extras.get(f"chacha{r}", {}).get("roofline", {}).get("launch_ms") or burst_ms)
        k = max(10, int(args.sustain_s * 1e3 / ms_est))
        for _ in range(3):
            step(r)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(device, period_s=0.01) as clk:
            e0.record(stream)
            for _ in range(k):
                step(r)
            e1.record(stream)
            e1.synchronize()
        ms = e0.elapsed_time(e1) / k
        v = _native.ctypes.c_double()
        _native.call("pc_intpeak", device, 0, _native.ctypes.byref(v))
        lop3_after = v.value
        achieved = bytes_per_step / (ms / 1e3) / 1e9
        c = clk.summary()
        int_roof_burst = peaks["lop3"] / (alu_ops_per_page(r) / PAGE) / 1e9
        hbm_roof = _hbm_peak()[0] / 2.0
        scale = (c["sm_mhz"] / c["sm_max_mhz"]) if c.get("sm_mhz") and c.get("sm_max_mhz") else 1.0
        roof_scaled = min(int_roof_burst * scale, hbm_roof)
        roof_meas = min(lop3_after / (alu_ops_per_page(r) / PAGE) / 1e9, hbm_roof)
        res[f"chacha{r}"] = {
            "value": round(achieved, 2), "unit": "GB/s", "launches": k, "seconds": round(k * ms / 1e3, 3),
            "launch_ms": round(ms, 4), "frac_vs_clock_scaled_roof": round(achieved / roof_scaled, 4),
            "clock_scaled_roof_gbs": round(roof_scaled, 1),
            "lop3_after_tops": round(lop3_after / 1e12, 3),
            "frac_vs_lop3_after_roof": round(achieved / roof_meas, 4), "clocks": c}
    return res


def split_parity(pc, key, torch, dist, world, rank, dev, backend, g_pages: int = 8192) -> dict:
    """Config 5's correctness side at this N: one global batch (same seed on
    every rank), each rank ciphers its contiguous page range under the SHARED
    key, and rank 0 compares the gathered ranges with its own single-call
    ciphertext of the whole batch.  (Checker traffic only; the data path has
    no collective.)"""
    from paper_2004_09252_b200.partition import shard

    g_pages -= g_pages % world  # equal ranges for all_gather at any N
    gen = torch.Generator(device=dev).manual_seed(4242)
    batch = torch.randint(0, 256, (g_pages, PAGE), dtype=torch.uint8, device=dev, generator=gen)
    lo, hi = shard(g_pages, rank, world)
    mine = torch.empty((hi - lo, PAGE), dtype=torch.uint8, device=dev)
    pc.crypt_pages(key, BASE_VADDR + PAGE * lo, 1, batch[lo:hi], out=mine)
    torch.cuda.synchronize()
    if world > 1:
        t = mine if backend == "nccl" else mine.cpu()
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        got = torch.cat([p.to(dev) for p in parts])
    else:
        got = mine
    res = {"pages": g_pages, "ranks": world}
    if rank == 0:
        whole = pc.crypt_pages(key, BASE_VADDR, 1, batch)
        torch.cuda.synchronize()
        res["identical_to_single_call"] = bool(torch.equal(got, whole))
        res["what"] = ("each rank ciphers pages [g*N/G, (g+1)*N/G) with the key shared from rank 0; "
                       "gathered == rank 0's single call over all pages")
    return res


def sweep_leg(pc, key, torch, args, rank, world, dev, barrier, max_over_ranks, red_dev) -> dict:
    """BASELINE configs[4]: a --sweep-gib batch split by contiguous page range
    over the ranks.  Device-resident: this rank's share in HBM, ciphered in
    place (CUDA events, 2 passes after 1 warm-up).  Host-resident: this
    rank's share in one pinned host buffer, through the public host API (H2D +
    cipher + D2H), timed on the host after a barrier; whole-job GB/s uses
    the slowest rank.  A 1/64 sample of each pass is spot-checked by
    decrypting it back."""
    total_pages = int(args.sweep_gib * 2**30) // PAGE
    from paper_2004_09252_b200.partition import shard

    lo, hi = shard(total_pages, rank, world)
    m = hi - lo
    vaddr0 = BASE_VADDR + PAGE * lo
    res = {"gib_total": args.sweep_gib, "pages_total": total_pages, "pages_per_rank": m, "ranks": world}
    free_b, _ = torch.cuda.mem_get_info(dev)
    # every branch below that skips is decided over all ranks (the timed
    # paths hold barriers and reductions: one rank skipping alone would hang)
    if max_over_ranks(float(m * PAGE > free_b - (4 << 30)), device=red_dev) > 0:
        res["device"] = {"skipped": f"share {m * PAGE / 2**30:.1f} GiB does not fit ({free_b / 2**30:.1f} GiB free)"}
    else:
        buf = torch.empty((m, PAGE), dtype=torch.uint8, device=dev)
        buf.random_(0, 256, generator=torch.Generator(device=dev).manual_seed(9 + rank))
        probe = buf[::64].clone()
        stream = torch.cuda.current_stream(dev)
        pc.crypt_pages(key, vaddr0, 1, buf, out=buf, stream=stream, check=False)  # warm-up pass
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        passes = 2
        e0.record(stream)
        for _ in range(passes):
            pc.crypt_pages(key, vaddr0, 1, buf, out=buf, stream=stream, check=False)
        e1.record(stream)
        e1.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) / passes, device=red_dev)
        # 3 passes (odd) leave buf encrypted; one more restores the plaintext
        pc.crypt_pages(key, vaddr0, 1, buf, out=buf, stream=stream, check=False)
        torch.cuda.synchronize()
        ok = bool(torch.equal(buf[::64], probe))
        res["device"] = {"value": round(total_pages * PAGE / (ms / 1e3) / 1e9, 2), "unit": "GB/s",
                         "ms_per_pass": round(ms, 3), "in_place": True, "roundtrip_ok": ok}
        del buf, probe
        torch.cuda.empty_cache()
    avail = _mem_available()
    too_big = avail is not None and m * PAGE * world > 0.6 * avail
    if max_over_ranks(float(too_big), device=red_dev) > 0:
        res["host"] = {"skipped": f"{m * PAGE * world / 2**30:.0f} GiB pinned over all ranks exceeds 60% of "
                                  f"MemAvailable ({avail / 2**30:.0f} GiB)"}
        return res
    host, err = None, None
    try:
        host = torch.empty((m, PAGE), dtype=torch.uint8).pin_memory()
    except RuntimeError as exc:
        err = f"pinned {m * PAGE / 2**30:.1f} GiB failed: {exc}"[:200]
    if max_over_ranks(float(err is not None), device=red_dev) > 0:
        del host
        res["host"] = {"skipped": err or "pinning failed on another rank"}
        return res
    host[::64].random_(0, 256)
    probe = host[::64].clone()
    eng = pc.default_engine(dev.index)
    pc.crypt_pages(key, vaddr0, 1, host[:8192], out=host[:8192], engine=eng)  # warm the pipeline
    pc.crypt_pages(key, vaddr0, 1, host[:8192], out=host[:8192], engine=eng)
    barrier()
    t0 = time.perf_counter()
    pc.crypt_pages(key, vaddr0, 1, host, out=host, engine=eng)
    el = max_over_ranks(time.perf_counter() - t0, device=red_dev)
    pc.crypt_pages(key, vaddr0, 1, host, out=host, engine=eng)
    ok = bool(torch.equal(host[::64], probe))
    res["host"] = {"value": round(total_pages * PAGE / el / 1e9, 2), "unit": "GB/s", "seconds": round(el, 3),
                   "in_place": True, "roundtrip_ok": ok, "pinned_gib_per_rank": round(m * PAGE / 2**30, 2),
                   "placement": eng.placement, "what": "one pinned buffer per rank, crypt_pages -> "
                   "pc_crypt_pages_host (H2D, cipher, D2H overlapped on 3 streams)"}
    del host, probe
    return res


def _mem_available():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except (OSError, ValueError):
        pass
    return None


def cpu_baseline(args) -> dict:
    """cpu_baseline: the reference itself (oracle/_ref, numba) on all host
    cores for about --cpu-seconds, plus the C port beside it; the port alone
    when the reference is unavailable or rounds != 20."""
    cores = len(os.sched_getaffinity(0))
    port = cpu_port_rate(args.rounds, max(0.5, args.cpu_seconds / 3), cores)
    ref = None
    if args.rounds == 20 and args.cpu_seconds > 0:
        try:
            ref = reference_cpu(cores, 16384, 1, None, args.cpu_seconds)
        except Exception as exc:  # the baseline must not take the bench down
            port["reference_error"] = repr(exc)[:200]
    if ref is None:
        one = cpu_port_rate(args.rounds, max(0.5, args.cpu_seconds / 5), 1, pages_per_batch=256)
        port["single_thread"] = {"value": round(one["value"], 4), "unit": "GB/s", "cores": 1,
                                 "sample": one["sample"]}
        return port
    ref["value"] = round(ref["value"], 4)
    ref["port"] = {"value": round(port["value"], 4), "cores": cores, "sample": port["sample"]}
    return ref


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy, read+write)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def _ncu_traffic(rounds: int, n_pages: int, desc: bool = False):
    """dram read+write bytes per launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d.get(f"chacha{rounds}" + ("_desc" if desc else ""))
        if e and e.get("pages") == n_pages:
            return e["dram_bytes"]
    except (OSError, ValueError):
        pass
    return None


def latency_sweep(pc, key, device: int, reps: int = 1000) -> dict:
    """BASELINE configs[3]: 1-64 host-resident pages per call (the fault
    handler's sliding window), pinned staging, p50/p99 per call."""
    import torch

    res = {}
    for n in (1, 2, 4, 8, 16, 32, 64):
        src = torch.randint(0, 256, (n, PAGE), dtype=torch.uint8).pin_memory()
        dst = torch.empty_like(src).pin_memory()
        for _ in range(300):  # ~5 ms: lets the SM clock leave its idle state first
            pc.crypt_pages(key, BASE_VADDR, 1, src, out=dst)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter_ns()
            pc.crypt_pages(key, BASE_VADDR, 1, src, out=dst)
            ts.append(time.perf_counter_ns() - t0)
        ts.sort()
        p50 = ts[len(ts) // 2] / 1e3
        res[str(n)] = {"p50_us": round(p50, 2), "p99_us": round(ts[int(len(ts) * 0.99)] / 1e3, 2),
                       "gbps_at_p50": round(n * PAGE / (p50 * 1e-6) / 1e9, 3)}
    # the same calls with resident workers on the key (DeviceKey.start_service):
    # 1-2 page batches become service tickets instead of launches
    dk = pc.DeviceKey.generate(device)
    try:
        dk.start_service(n_workers=4)
        res["resident_workers"] = {}
        for n in (1, 2, 4):
            src = torch.randint(0, 256, (n, PAGE), dtype=torch.uint8).pin_memory()
            dst = torch.empty_like(src).pin_memory()
            for _ in range(300):
                pc.crypt_pages(dk, BASE_VADDR, 1, src, out=dst)
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter_ns()
                pc.crypt_pages(dk, BASE_VADDR, 1, src, out=dst)
                ts.append(time.perf_counter_ns() - t0)
            ts.sort()
            p50 = ts[len(ts) // 2] / 1e3
            res["resident_workers"][str(n)] = {"p50_us": round(p50, 2),
                                               "p99_us": round(ts[int(len(ts) * 0.99)] / 1e3, 2)}
        res["resident_workers"]["workers"] = 4
    finally:
        dk.destroy()
    return res


def store_throughput(pc, key, device: int, n: int = 65536) -> dict:
    """evict (encrypt into the HBM page store) and refault
    (decrypt out of it) 256 MiB of pinned host pages in one batch each."""
    import torch

    from paper_2004_09252_b200.store import DevicePageStore
    from paper_2004_09252_b200.workers import ClientId

    st = DevicePageStore(n, key, device=device)
    src = torch.randint(0, 256, (n, PAGE), dtype=torch.uint8).pin_memory()
    vaddrs = (np.arange(n, dtype=np.uint64) * np.uint64(PAGE) + np.uint64(BASE_VADDR))
    c = ClientId(1, 0)
    dst = torch.empty_like(src).pin_memory()
    st.evict_many(c, vaddrs, src.numpy())  # warm-up
    st.refault_many(c, vaddrs, out=dst.numpy())
    t0 = time.perf_counter()
    st.evict_many(c, vaddrs, src.numpy())
    t1 = time.perf_counter()
    st.refault_many(c, vaddrs, out=dst.numpy())
    t2 = time.perf_counter()
    ok = bool(torch.equal(dst, src))
    return {"pages": n, "evict_gbs": round(n * PAGE / (t1 - t0) / 1e9, 2),
            "refault_gbs": round(n * PAGE / (t2 - t1) / 1e9, 2), "roundtrip_identical": ok,
            "note": "one batch each way, pinned host buffers, includes the Python index updates"}


def pager_rate(pc, key, device: int) -> dict:
    """faults/s through WindowPager (window 64) with one
    fault per call (the reference's flow) and with 64-fault batches.  Two
    passes over 4096 pages: first touches + evictions, then refaults +
    evictions."""
    from paper_2004_09252_b200.pager import WindowPager
    from paper_2004_09252_b200.store import DevicePageStore
    from paper_2004_09252_b200.workers import ClientId

    res = {}
    pages = [BASE_VADDR + PAGE * i for i in range(4096)]
    for batch, service in ((1, False), (1, True), (64, False)):
        st = DevicePageStore(8192, key, device=device)
        if service:  # single faults as tickets of the store's resident worker
            st.start_service()
        mem = {}
        # the client hands back the page it holds (a single page as is)
        pg = WindowPager(st, lambda c, vs: mem.pop(vs[0]) if len(vs) == 1 else np.stack([mem.pop(v) for v in vs]),
                         window_capacity=64)
        c = ClientId(1, 0)
        pg.register(c)
        n = 0
        t0 = time.perf_counter()
        for _ in range(2):
            for i in range(0, len(pages), batch):
                vs = [v for v in pages[i:i + batch] if v not in mem]
                if not vs:
                    continue
                out = pg.fault_batch(c, vs)
                for v, row in zip(vs, out):
                    if v in pg._window(c)._members:
                        mem[v] = row
                n += len(vs)
        el = time.perf_counter() - t0
        m = pg.metrics[c]
        res[f"batch{batch}" + ("_service" if service else "")] = {"faults_per_s": round(n / el), "gbs": round(n * PAGE / el / 1e9, 3),
                                "decrypts": m.decrypt_ops, "encrypts": m.encrypt_ops, "gpu_batches": m.gpu_batches}
        pg.unregister(c)
        st.close()
    return res


def service_latency(device: int, reps: int = 2000) -> dict:
    """BASELINE configs[3] through the persistent GPU worker service (the
    paper's design; WorkerPool drop-in): 1-page fault-path requests."""
    import ctypes

    from paper_2004_09252_b200 import _native
    from paper_2004_09252_b200.workers import ClientId, WorkerPool

    res = {}
    pool = WorkerPool(keysource=os.urandom, device=device)
    try:
        page = bytearray(PAGE)
        c = ClientId(1, 0)
        for _ in range(100):
            pool.crypt(c, BASE_VADDR, "encrypt", page)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter_ns()
            pool.crypt(c, BASE_VADDR, "encrypt", page)
            ts.append(time.perf_counter_ns() - t0)
        ts.sort()
        res["WorkerPool.crypt"] = {"p50_us": round(ts[len(ts) // 2] / 1e3, 2),
                                   "p99_us": round(ts[int(len(ts) * .99)] / 1e3, 2)}
        lib = _native.load()
        buf = (ctypes.c_char * PAGE)()
        w = pool.route(c)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter_ns()
            lib.pc_service_crypt(pool._svc, w, BASE_VADDR, 1, buf, buf, -1)
            ts.append(time.perf_counter_ns() - t0)
        ts.sort()
        res["pc_service_crypt"] = {"p50_us": round(ts[len(ts) // 2] / 1e3, 2),
                                   "p99_us": round(ts[int(len(ts) * .99)] / 1e3, 2)}
        res["workers"] = pool.n_workers
    finally:
        pool.shutdown()
    return res


if __name__ == "__main__":
    sys.exit(main())
