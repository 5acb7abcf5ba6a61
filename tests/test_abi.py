"""CPU checks of the boundary: libwn loads, exports every symbol include/wn.h declares, host-only logic,
and the product path has no CPU fallback (no compute calls here — there is no GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wn.h")
LIB = os.path.join(ROOT, "paper_2405_16634_b200", "libwn.so")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|wn_status|uint64_t)\s+(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2405_16634_b200 import build

        build.build()
    import paper_2405_16634_b200.wn as wn

    return wn


def test_header_declares_the_north_star_calls():
    names = _declared()
    for required in ("wn_build_tree", "wn_eval", "wn_eval_grad", "wn_eval_adjoint", "wnnc_iterate"):
        assert required in names
    assert len(names) >= 19


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert set(lib.EXPORTED) == set(_declared())


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_shard_range_partitions(lib):
    for n in (1, 255, 256, 1000, 500000, 4000000):
        for world in (1, 2, 3, 4, 8):
            ranges = [lib.wn_shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            for b, e in ranges:
                assert b % 256 == 0 and b <= e
    with pytest.raises(lib.WnError):
        lib.wn_shard_range(10, 2, 2)


def test_no_cpu_fallback(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    # compute entry points refuse to run without a device instead of falling back
    with pytest.raises(ValueError):
        lib.wn_build_tree(torch.zeros(10, 3))
    import ctypes as C

    h = C.c_void_p()
    st = lib._L.wn_build_tree(None, 10, 15, None, C.byref(h))
    assert st == lib.WN_ERR_ARG
    st = lib._L.wn_build_tree(C.c_void_p(1), 10, 15, None, C.byref(h))
    assert st == lib.WN_ERR_CUDA
    assert "device" in lib._L.wn_last_error().decode()
    assert lib._L.wn_build_tree(C.c_void_p(1), 0, 15, None, C.byref(h)) == lib.WN_ERR_EMPTY
    assert lib._L.wn_build_tree(C.c_void_p(1), 10, 22, None, C.byref(h)) == lib.WN_ERR_ARG


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2405_16634_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "wn_oracle" not in txt, f
