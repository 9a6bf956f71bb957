"""libhrb200.so builds for sm_100a, loads without a GPU, and exports every
entry point declared in include/hrb200.h."""

import os
import re
import subprocess

import pytest

from paper_1211_3056_b200 import _native
from paper_1211_3056_b200.build import LIB, ROOT, build


def declared_symbols() -> list[str]:
    text = open(os.path.join(ROOT, "include", "hrb200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(hrb_\w+)\s*\(", text, re.M)))


def test_header_lists_expected_entry_points():
    assert set(declared_symbols()) == set(_native.EXPORTS)


def test_library_builds_and_exports_all_symbols():
    build()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (hrb_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing


def test_library_loads_without_gpu_and_reports_version():
    lib = _native.load()
    assert lib.hrb_version() == 100
    for name in declared_symbols():
        assert hasattr(lib, name)


def test_sass_is_sm100a():
    build()
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_errors_do_not_need_a_gpu():
    lib = _native.load()
    # bad algorithm code is rejected before any device work
    rc = lib.hrb_search_batch(9, 0, 64, 0, None, None, None, None, None, None, None, None, None, None)
    assert rc == _native.HRB_ERR_CONFIG
    assert b"algorithm" in lib.hrb_last_error()


def host_declared_symbols() -> list[str]:
    text = open(os.path.join(ROOT, "include", "hrb_host.h")).read()
    return sorted(set(re.findall(r"^int\s+(hrbh_\w+)\s*\(", text, re.M)))


def test_host_library_exports_all_symbols():
    """libhrbhost.so (native host generation + confirmation) exports every
    entry point of include/hrb_host.h and loads without a GPU."""
    from paper_1211_3056_b200 import hostgen
    from paper_1211_3056_b200.build import HOST_LIB, build_host

    build_host()
    out = subprocess.run(["nm", "-D", "--defined-only", HOST_LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (hrbh_\w+)", out))
    want = set(host_declared_symbols())
    assert want and not (want - exported), want - exported
    assert hostgen.load().hrbh_version() == 100


def test_wide_config_errors_do_not_need_a_gpu():
    import ctypes as C

    lib = _native.load()
    bad = _native.HrbWSlice(n_super=1, n_total=1, max_dom_n=8, degree=2, frac_limbs=4, word_bits=64)
    out = _native.HrbRunOut()
    assert lib.hrb_wrun_slice(C.byref(bad), 2, 8, C.byref(out), None) == _native.HRB_ERR_CONFIG
    assert b"degree" in lib.hrb_last_error()
