"""The ctypes mirror of tsb_produce_args (paper_2409_18749_b200/_lib.py)
matches the C header's layout: field order, every offset and the size, as
gcc sees include/tsb200.h (CPU only: compiles a probe, launches nothing)."""
import os
import re
import shutil
import subprocess

import pytest

from paper_2409_18749_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "tsb200.h")


def header_fields():
    src = open(HDR).read()
    body = src[:src.index("} tsb_produce_args;")]
    body = body[body.rindex("typedef struct {") + len("typedef struct {"):]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        for part in decl.split(","):
            m = re.search(r"\**\s*(\w+)\s*(\[\d+\])?\s*$", part.strip())
            names.append(m.group(1))
    return names


def test_field_order_matches_header():
    assert [f[0] for f in _lib.ProduceArgs._fields_] == header_fields()


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no gcc")
def test_offsets_and_size_match_gcc(tmp_path):
    names = header_fields()
    prog = tmp_path / "probe.c"
    prog.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"tsb200.h\"\nint main(void){\n"
                    + "".join(f'printf("%zu\\n", offsetof(tsb_produce_args, {n}));\n' for n in names)
                    + 'printf("%zu\\n", sizeof(tsb_produce_args));\nreturn 0;}\n')
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)],
                   check=True, capture_output=True)
    got = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True,
                                          text=True).stdout.split()]
    import ctypes

    want = [getattr(_lib.ProduceArgs, n).offset for n in names] + [ctypes.sizeof(_lib.ProduceArgs)]
    assert got == want
