"""pytest plugin (test infrastructure) that binds the B200 engine into the
UNMODIFIED reference package before the reference's own test files are
collected.  Used by tests/test_gpu_ref_suite.py as

    python -m pytest -p ref_seam_plugin oracle/_ref/tests/test_cipher.py ...

PC_SEAM=kernel  pagecrypt.cipher._chacha_numba = paper_2004_09252_b200._chacha_cuda
                (the kernel seam, pkg/src/pagecrypt/cipher.py:28-31, consumed at
                cipher.py:176-182): every keystream the reference computes
                comes from the B200 through pc_keystream_words.
PC_SEAM=pool    additionally pagecrypt.workers.WorkerPool (and the names the
                orchestrator and package re-export) = the persistent GPU
                worker service (paper_2004_09252_b200.workers.WorkerPool),
                raising the reference's own exception classes
                (errors.adopt_host_errors, as INTEGRATION.md binds it).

At session end the number of seam calls and the library's launch counter are
written to $PC_SEAM_REPORT so the caller can prove the GPU path ran.
"""

from __future__ import annotations

import json
import os

_calls = {"keystream_words": 0}


def pytest_configure(config):
    import pagecrypt
    import pagecrypt.cipher as cipher

    from paper_2004_09252_b200 import _chacha_cuda, _native

    _native.load()  # fail loudly if the CUDA extension is missing
    real = _chacha_cuda.keystream_words

    class _CountingSeam:
        @staticmethod
        def keystream_words(kw, vaddr, pid, indices, out):
            _calls["keystream_words"] += 1
            return real(kw, vaddr, pid, indices, out)

    cipher._chacha_numba = _CountingSeam
    if os.environ.get("PC_SEAM") == "pool":
        import pagecrypt.errors

        import paper_2004_09252_b200.engine  # noqa: F401  (every module that raises is loaded first)
        import paper_2004_09252_b200.workers  # noqa: F401
        from paper_2004_09252_b200.errors import adopt_host_errors

        adopt_host_errors(pagecrypt.errors)  # the drop-in raises the host's exception types
        import pagecrypt.orchestrator as orch
        import pagecrypt.workers as rw

        from paper_2004_09252_b200.workers import WorkerPool

        rw.WorkerPool = WorkerPool
        orch.WorkerPool = WorkerPool
        pagecrypt.WorkerPool = WorkerPool
        for name in ("pagecrypt.bench",):
            mod = __import__(name, fromlist=["WorkerPool"])
            mod.WorkerPool = WorkerPool


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PC_SEAM_REPORT")
    if not path:
        return
    from paper_2004_09252_b200 import _native

    with open(path, "w") as fh:
        json.dump({"seam": os.environ.get("PC_SEAM", "kernel"), "keystream_calls": _calls["keystream_words"],
                   "library_launches": _native.tune_get("launches"), "exitstatus": int(exitstatus)}, fh)
