"""The C-ABI library loads here (no GPU) and exports every declared symbol."""
import os
import re

from paper_2605_05899_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "vismmoe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vmm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(declared_symbols()) <= set(_lib.exported_symbols()) | {"vmm_engine_slab"}


def test_abi_version_and_error_plumbing():
    lib = _lib.load()
    assert lib.vmm_abi_version() == 1
    import ctypes as C
    h = C.c_void_p()
    assert lib.vmm_cache_create(0, 0, C.byref(h)) == 2
    assert b"num_slabs" in lib.vmm_last_error()
