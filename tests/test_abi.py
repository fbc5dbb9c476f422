"""Host-side checks of the C ABI (no GPU): the library loads, exports every
symbol include/pic.h declares, and the ctypes struct matches the C layout."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2507_20719_b200 import build_lib, pic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pic.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"PIC_API\s+[\w\s\*]+?\b(pic_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    build_lib.build()
    return pic.load_library()


def test_header_declares_entry_points():
    names = declared()
    for need in ("pic_init", "pic_mover", "pic_moments", "pic_exchange"):
        assert need in names
    assert set(names) == set(pic.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", build_lib.LIB]).decode()
    exported = set(re.findall(r" T (pic_\w+)", out))
    missing = set(declared()) - exported
    assert not missing, missing
    for name in declared():
        assert hasattr(lib, name)


def test_abi_version(lib):
    assert lib.pic_abi_version() == 6


def test_struct_layout_matches_header():
    """sizeof / offsetof of pic_config from a C program against pic.h equal ctypes'."""
    fields = [f for f, _ in pic.pic_config._fields_]
    prog = "#include <stdio.h>\n#include <stddef.h>\n#include \"pic.h\"\nint main(){\n"
    prog += 'printf("%zu\\n", sizeof(pic_config));\n'
    for f in fields:
        prog += f'printf("%zu\\n", offsetof(pic_config, {f}));\n'
    prog += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        vals = [int(v) for v in subprocess.check_output([exe]).split()]
    assert vals[0] == C.sizeof(pic.pic_config)
    for f, off in zip(fields, vals[1:]):
        assert getattr(pic.pic_config, f).offset == off, f


def test_workspace_query_rejects_bad_config(lib):
    cfg = pic.pic_config()
    out = C.c_int64()
    assert lib.pic_workspace_bytes(C.byref(cfg), C.byref(out)) == pic.PIC_EINVAL


def test_null_context_is_einval(lib):
    assert lib.pic_mover(None, 0) == pic.PIC_EINVAL
    assert lib.pic_exchange(None) == pic.PIC_EINVAL
    assert lib.pic_last_error(None) == b"null context"
