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


def _header_params(name):
    src = open(os.path.join(ROOT, "include", "vismmoe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    m = re.search(r"\bint\s+" + name + r"\s*\((.*?)\)\s*;", src, flags=re.S)
    assert m, name
    return [p.strip() for p in m.group(1).split(",")]


def test_ctypes_signatures_match_the_header():
    """Every binding in _lib._SIGS passes as many arguments as the header declares."""
    for name, (_, args) in _lib._SIGS.items():
        src = open(os.path.join(ROOT, "include", "vismmoe.h")).read()
        if not re.search(r"\b" + name + r"\s*\(", re.sub(r"/\*.*?\*/", "", src, flags=re.S)):
            continue
        params = _header_params(name) if re.search(r"\bint\s+" + name + r"\s*\(", src) else None
        if params is None:
            continue
        n = 0 if params == ["void"] else len(params)
        assert len(args) == n, (name, len(args), n)


def test_integration_prune_stub_matches_the_header():
    """INTEGRATION.md §8's ctypes stub for vmm_prune declares the header's argument list."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"lib\.vmm_prune\.argtypes = (.*)", doc)
    assert m
    import ctypes as C  # noqa: F401  (the stub's expression refers to C)

    argtypes = eval(m.group(1), {"C": C})
    params = _header_params("vmm_prune")
    assert len(argtypes) == len(params)
    for t, p in zip(argtypes, params):
        want = C.c_void_p if "*" in p else (C.c_double if p.startswith("double") else C.c_int)
        assert t is want, (t, p)
