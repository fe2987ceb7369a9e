"""The reference's OWN test files, unmodified, run against the B200 engine
(SURVEY §7.2).

oracle/_ref/ holds a byte-for-byte snapshot of /root/reference/pkg
(oracle/fetch_ref.py, checked against its MANIFEST).  Each test runs pytest in
a subprocess on the reference test files with tests/ref_seam_plugin.py
binding our engine in:

* kernel seam: pagecrypt.cipher._chacha_numba -> paper_2004_09252_b200._chacha_cuda
  (cipher.py:28-31, consumed at cipher.py:176-182).  test_cipher.py,
  test_workers.py and test_orchestrator.py must pass in full, and the seam
  must have been called (every keystream from the GPU).
* pool seam: additionally pagecrypt.workers.WorkerPool -> the persistent GPU
  worker service.  Two reference tests inspect the reference's host-RAM key
  slots themselves (``ram.private_bytes() == 32 * n_workers``,
  ``pool._workers[i].key_slot``); the GPU service deliberately has no host
  key slot (the key lives in the workers' registers), so those two are
  deselected, by name, and nothing else.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu

FILES = ["test_cipher.py", "test_workers.py", "test_orchestrator.py"]
# host-RAM key-slot internals of the reference pool (see module docstring)
POOL_DESELECT = [
    "test_workers.py::TestPool::test_key_confined_outside_dumpable_ram",
    "test_workers.py::TestPool::test_shutdown_wipes_keys_and_is_idempotent",
]


def _snapshot_ok():
    import fetch_ref

    return fetch_ref.check()


def _run(seam, tmp_path, extra=()):
    if not os.path.isdir(REF):
        pytest.skip("oracle/_ref absent (run oracle/fetch_ref.py where /root/reference exists)")
    assert _snapshot_ok(), "oracle/_ref differs from its MANIFEST: not the unmodified reference"
    report = tmp_path / f"seam_{seam}.json"
    env = dict(os.environ)
    env.update(PC_SEAM=seam, PC_SEAM_REPORT=str(report), NUMBA_CACHE_DIR=str(tmp_path / "numba"),
               PYTHONPATH=os.pathsep.join([os.path.join(REF, "src"), os.path.join(REF, "tests"),
                                           os.path.join(ROOT, "tests"), ROOT]))
    args = [sys.executable, "-m", "pytest", "-p", "ref_seam_plugin", "-p", "no:cacheprovider", "-q",
            "--rootdir", os.path.join(REF, "tests"), *[os.path.join(REF, "tests", f) for f in FILES], *extra]
    r = subprocess.run(args, capture_output=True, text=True, timeout=900, env=env, cwd=os.path.join(REF, "tests"))
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    with open(report) as fh:
        rep = json.load(fh)
    return r.stdout, rep


def test_reference_suite_through_kernel_seam(cuda, tmp_path):
    out, rep = _run("kernel", tmp_path)
    assert rep["keystream_calls"] > 1000, rep  # the reference's keystreams all came from the B200
    assert rep["library_launches"] > 0, rep
    assert " passed" in out and "failed" not in out


def test_reference_suite_through_gpu_worker_pool(cuda, tmp_path):
    extra = []
    for d in POOL_DESELECT:
        extra += ["--deselect", d]  # node ids are relative to --rootdir
    out, rep = _run("pool", tmp_path, extra)
    assert rep["library_launches"] > 0, rep
    assert " passed" in out and "failed" not in out
