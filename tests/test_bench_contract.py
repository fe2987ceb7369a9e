"""The driver's bench contract, checked where it can be without a GPU: the
reference arm (``bench.py --impl reference``) runs on host cores only and
must print one JSON line with the agreed keys; under a multi-rank launch
only rank 0 prints."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=e, cwd=ROOT)


def test_reference_arm_line():
    r = run_bench("--impl", "reference", "--steps", "3", "--warmup", "3", "--ref-pages", "1024")
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("GB/s of pages") and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    # the unmodified reference (oracle/_ref snapshot, numba) whenever it is here
    assert cb["kind"] == ("reference" if _reference_available() else "port")
    if cb["kind"] == "reference":
        assert cb["spot_check_ok"] is True
        assert {"single_thread", "worker_pool", "crypt_page_latency_us"} <= set(cb)
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["rounds"] == 20 and d["config"]["pages_per_gpu"] == 262144


def _reference_available():
    sys.path.insert(0, ROOT)
    from oracle import ref_bench

    return ref_bench.load() is not None


def test_self_launch_two_ranks_without_torchrun():
    """--gpus 2 with no WORLD_SIZE: bench.py starts its own two ranks
    (torch.distributed.run on 127.0.0.1) and rank 0's line says n_gpus 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--ref-pages", "256", "--dist-backend", "gloo"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


def test_gpus_must_match_world_size():
    r = run_bench("--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "3", "--ref-pages", "64",
                  env={"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


def test_reference_arm_other_ranks_are_silent():
    r = run_bench("--impl", "reference", "--steps", "3", "--warmup", "3", "--ref-pages", "64",
                  env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 2  # --gpus defaults to 1: a mismatched world is refused
    r = run_bench("--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "3", "--ref-pages", "64",
                  env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_warmup_below_three_is_refused():
    r = run_bench("--impl", "reference", "--steps", "3", "--warmup", "2")
    assert r.returncode != 0


import pytest  # noqa: E402


@pytest.mark.gpu
def test_own_arm_line_has_every_contract_key(cuda):
    r = run_bench("--steps", "3", "--warmup", "3", "--pages", "8192", "--no-extras", "--cpu-seconds", "0.2")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["scaling"] == "weak" and d["vs_baseline"] is None and d["higher_is_better"] is True
    assert "workload" in d["config"] and "model" not in d["config"]
    rl = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rl)
    assert rl["unit"] == "GB/s" and abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-3
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 8192 * 4096 and e["value"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_share_the_key_and_split_the_pages(cuda):
    """The N>1 path on the one B200 here (test mode: both ranks on cuda:0,
    gloo): bench.py --gpus 2 self-launches two ranks, rank 0 generates the key
    on the device and rank 1 imports it over CUDA IPC, each rank ciphers its
    page range, and the gathered ranges equal rank 0's single call."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--same-device",
                        "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--pages", "16384",
                        "--sweep-gib", "0.25", "--sustain-s", "0.1", "--cpu-seconds", "0.2"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_active"] == 1
    assert "CUDA IPC" in d["config"]["key"]
    sp = d["extras"]["split_parity"]
    assert sp["ranks"] == 2 and sp["identical_to_single_call"] is True
    sw = d["extras"]["sweep"]
    assert sw["ranks"] == 2 and sw["device"]["roundtrip_ok"] and sw["host"]["roundtrip_ok"]
