"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares (no compute calls without a GPU)."""

import os
import re

from paper_2409_18749_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tsb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsb_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_lib.exported_symbols())


def test_library_loads_and_exports_all_symbols():
    L = _lib.load()
    for name in header_functions():
        assert hasattr(L, name), name
    assert L.tsb_version() == 1
    # host-only entry points work without a GPU
    assert L.tsb_mix64(1) == 0x5692161D100B05E5
    assert L.tsb_derive_key(0, 0, 0x53485546) == 0x239A8DD44B4BA285


def test_host_permutation_matches_golden(golden):
    from paper_2409_18749_b200 import dataplane as dp
    import zlib

    for case in golden["permutation"]:
        p = dp.permutation(case["n"], case["key"])
        assert zlib.crc32(p.astype("<i8").tobytes()) == case["crc_i64"]
    for case in golden["epoch_order"]:
        o = dp.epoch_order(case["n"], case["shuffle_seed"], case["epoch"], case["reshuffle"])
        assert zlib.crc32(o.astype("<i8").tobytes()) == case["crc_i64"]


def test_missing_library_fails_loudly(tmp_path):
    import pytest

    from paper_2409_18749_b200.errors import LibraryMissing

    saved = _lib._lib
    try:
        _lib._lib = None
        with pytest.raises(LibraryMissing):
            _lib.load(str(tmp_path / "nope.so"))
    finally:
        _lib._lib = saved


def test_sm100a_cubin_in_library():
    import shutil
    import subprocess

    import pytest

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_the_oracle():
    """The oracle is test infrastructure: no module of the product package may
    import, load or execute anything under oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2409_18749_b200")
    offenders = []
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                if re.search(r"^\s*(from|import)\s+oracle\b|ts_oracle|libts_oracle|"
                             r"import_module\(\s*['\"]oracle", src, flags=re.M):
                    offenders.append(f)
    assert not offenders, offenders
