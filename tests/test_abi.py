"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads, and exports every
entry point include/solid.h declares; the product package never touches the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "solid.h")).read()
    return sorted(set(re.findall(r"^\s*(?:solid_status|uint32_t|const char\*)\s+(solid_\w+)\(",
                                 src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_10726_b200.build import build
    return ctypes.CDLL(build())


def test_header_declares_the_boundary():
    names = _declared()
    for must in ["solid_init", "solid_destroy", "solid_lookup_batch", "solid_insert_batch",
                 "solid_stats"]:      # SURVEY §8(b), north star
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    lib.solid_abi_version.restype = ctypes.c_uint32
    assert lib.solid_abi_version() == 7


def test_binding_symbols_match_header():
    import paper_2603_10726_b200 as P
    assert sorted(P.ABI_SYMBOLS) == _declared()


def test_library_is_sm100a_and_uses_128bit_cas(lib):
    from paper_2603_10726_b200.build import LIB
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True,
                                       text=True).stdout
    assert "ATOMG.E.CAS.128" in sass          # index insert (north star kernel 3)
    assert "VOTE.ANY" in sass or "VOTE.ALL" in sass   # warp ballot first-miss (kernel 4)


def test_init_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2603_10726_b200 as P
    with pytest.raises(P.SolidError):
        P.Index()


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2603_10726_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ["import oracle", "from oracle", "liboracle", "solid_oracle"]:
                    assert bad not in txt, (f, bad)
