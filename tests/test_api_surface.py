"""The drop-in check: every public callable of the reference's
hot-path surface -- ``pagecrypt.cipher``, ``WorkerPool`` / ``Completion``,
``EncryptedPageStore`` -- exists in the B200 package with the reference's
parameters (same names, kinds and defaulted-ness, in order); anything the
B200 side adds comes after them and has a default.  The reference side was
recorded by ``tests/golden/make_api_surface.py`` from the reference itself."""

import inspect
import json
import os

import pytest

from paper_2004_09252_b200 import cipher, store, workers

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "api_surface.json")

with open(GOLDEN) as f:
    SURFACE = json.load(f)


def params(fn):
    return [[p.name, p.kind.name, p.default is not inspect.Parameter.empty]
            for p in inspect.signature(fn).parameters.values()]


def assert_compatible(ours, ref, what):
    assert ours[:len(ref)] == ref, f"{what}: reference parameters {ref}, ours {ours}"
    for name, kind, has_default in ours[len(ref):]:
        assert has_default or kind in ("VAR_POSITIONAL", "VAR_KEYWORD"), f"{what}: added parameter {name} needs a default"


def member(cls, name):
    obj = inspect.getattr_static(cls, name)
    if isinstance(obj, (staticmethod, classmethod)):
        return obj.__func__
    return obj


@pytest.mark.parametrize("name", sorted(SURFACE["cipher_functions"]))
def test_cipher_functions(name):
    assert_compatible(params(getattr(cipher, name)), SURFACE["cipher_functions"][name], f"cipher.{name}")


@pytest.mark.parametrize("cls,name", [(c, n) for c, ms in sorted(SURFACE["cipher_classes"].items()) for n in sorted(ms)])
def test_cipher_classes(cls, name):
    ref = SURFACE["cipher_classes"][cls][name]
    obj = member(getattr(cipher, cls), name)
    if ref == "property":
        assert isinstance(obj, property), f"{cls}.{name} should be a property"
    else:
        assert_compatible(params(obj), ref, f"{cls}.{name}")


def test_cipher_constants():
    for name, value in SURFACE["cipher_constants"].items():
        assert getattr(cipher, name) == value, name


@pytest.mark.parametrize("cls,name", [(c, n) for c, ms in sorted(SURFACE["workers"].items()) for n in sorted(ms)])
def test_worker_pool_and_completion(cls, name):
    ref = SURFACE["workers"][cls][name]
    obj = member(getattr(workers, cls), name)
    if ref == "property":
        assert isinstance(obj, property), f"{cls}.{name} should be a property"
    elif cls == "Completion" and name == "__init__":
        pass  # built by the pool, never by callers (workers.py:208-221)
    else:
        assert_compatible(params(obj), ref, f"{cls}.{name}")


@pytest.mark.parametrize("name", sorted(n for n in SURFACE["store"]["EncryptedPageStore"] if n != "__init__"))
def test_page_store_methods(name):
    """DevicePageStore keeps every EncryptedPageStore method; its constructor
    differs on purpose (an HBM slab size and a DeviceKey instead of the
    reference's TaggedRam)."""
    ref = SURFACE["store"]["EncryptedPageStore"][name]
    obj = member(store.DevicePageStore, name)
    if ref == "property":
        assert isinstance(obj, property)
    else:
        assert_compatible(params(obj), ref, f"DevicePageStore.{name}")
