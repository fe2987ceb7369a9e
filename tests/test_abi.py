"""CPU checks of the C ABI: the library loads, exports exactly what
include/pagecrypt.h declares, and refuses to compute without a GPU (no CPU
fallback)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2004_09252_b200 import _native
from paper_2004_09252_b200.errors import ContractViolation, PageCryptError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pagecrypt.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(pc_\w+)\s*\(", text, flags=re.M))


def test_header_matches_binding_table():
    assert header_functions() == set(_native.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pc_\w+)", out))
    assert header_functions() <= exported


def test_abi_version():
    assert _native.load().pc_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_rejected_before_device_use():
    lib = _native.load()
    # rounds validated first: EINVAL even without a GPU
    out = (ctypes.c_uint32 * 16)()
    kw = (ctypes.c_uint32 * 8)()
    idx = (ctypes.c_int64 * 1)(0)
    rc = lib.pc_keystream_words(kw, 0, 0, idx, 1, out, 7)
    assert rc == _native.PC_EINVAL
    assert b"rounds" in lib.pc_last_error()
    with pytest.raises(ContractViolation):
        _native.check(rc)
    # NULL handles are state errors
    assert lib.pc_crypt_pages_dev(None, None, None, 0, 0, None, None, 1, 20, None) == _native.PC_ESTATE
    assert lib.pc_key_destroy(None) == _native.PC_OK


@pytest.mark.skipif(_native.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    import paper_2004_09252_b200 as pc

    with pytest.raises(PageCryptError):
        pc.crypt_page(bytes(32), 0, 0, bytes(4096))
    with pytest.raises(PageCryptError):
        pc.page_keystream(bytes(32), 0, 0)
    with pytest.raises(PageCryptError):
        pc.DeviceKey.install(bytes(32), 0)


def test_no_kernel_uses_local_memory():
    """Key and cipher state stay in registers in every kernel (PAPER.md:634-637:
    "the current implementation of the GPU kernel never does register
    spilling")."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    fns = re.findall(r"Function (\S+):\n\s+REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", out)
    assert len(fns) >= 20
    names = " ".join(f[0] for f in fns)
    for k in ("k_crypt_pages", "k_crypt_pages_tma", "k_service", "k_keystream_seeds", "k_keygen"):
        assert k in names
    bad = [(f, st, lo) for f, _, st, lo in fns if st != "0" or lo != "0"]
    assert not bad


def test_header_is_plain_c_and_links(tmp_path):
    """include/pagecrypt.h is a C ABI: a C99 program (-pedantic -Werror)
    includes it, links libpagecrypt.so and calls it -- no C++ or torch types
    anywhere on the boundary."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    _native.load()  # builds must exist
    src = tmp_path / "abi.c"
    src.write_text(
        '#include "pagecrypt.h"\n#include <stdio.h>\n'
        "int main(void) {\n"
        "  int n = -1;\n"
        "  if (pc_abi_version() != PC_ABI_VERSION) return 2;\n"
        "  (void)pc_device_count(&n);\n"
        "  if (pc_keystream_words(0, 0, 0, 0, 1, 0, 20) != PC_EINVAL) return 3;\n"
        '  printf("%s\\n", pc_last_error());\n'
        "  return 0;\n}\n")
    exe = tmp_path / "abi"
    libdir = os.path.dirname(_native.LIB_PATH)
    subprocess.run([gcc, "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-L", libdir, "-lpagecrypt", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "NULL" in r.stdout


@pytest.mark.parametrize("knob,good,bad", [
    ("run_desc", [0, 1, 2], [-1, 3]),
    ("kernel", [0, 1, 2, 3, 4, 5, 6, 9], [-1, 7, 8, 10]),
    ("svc_pages", [0, 1, 64], [-1, 65]),
    ("small_mode", [0, 1], [2]),
])
def test_tuning_knobs_validate_without_a_gpu(knob, good, bad):
    """pc_tune range-checks every knob value (no device is touched); a bad
    value leaves the knob as it was."""
    before = _native.tune_get(knob)
    try:
        for v in good:
            _native.tune(knob, v)
            assert _native.tune_get(knob) == v
        _native.tune(knob, good[0])
        for v in bad:
            with pytest.raises(ContractViolation):
                _native.tune(knob, v)
            assert _native.tune_get(knob) == good[0]
    finally:
        _native.tune(knob, before)
    with pytest.raises(ContractViolation):
        _native.tune("no_such_knob", 1)
