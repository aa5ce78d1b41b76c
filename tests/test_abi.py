"""CPU-side checks of the C-ABI boundary: libcls.so builds for sm_100a, loads without a
GPU, exports every symbol include/cls.h declares, and validates arguments before
touching the device.  No compute call is made here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def native():
    from paper_2506_21117_b200 import build
    build.build()
    from paper_2506_21117_b200 import _native
    return _native


def _declared():
    src = open(os.path.join(ROOT, "include", "cls.h")).read()
    return sorted(set(re.findall(r"^\s*(?:cls_status|const char \*|int64_t)\s*\**\s*(cls_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("cls_create", "cls_destroy", "cls_render_fwd", "cls_active", "cls_render_bwd", "cls_adam_masked"):
        assert n in names


def test_library_exports_every_declared_symbol(native):
    lib = ctypes.CDLL(native.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(native.EXPORTS)


def test_flag_constants_match_header(native):
    src = open(os.path.join(ROOT, "include", "cls.h")).read()
    flags = {k: int(v) for k, v in re.findall(r"#define (CLS_FLAG_\w+) (\d+)u", src)}
    assert flags == {"CLS_FLAG_ALL_TILES": native.CLS_FLAG_ALL_TILES, "CLS_FLAG_TARGETS_U8": native.CLS_FLAG_TARGETS_U8,
                     "CLS_FLAG_STATIC_CACHE": native.CLS_FLAG_STATIC_CACHE}
    assert len(set(flags.values())) == len(flags) and all(v & (v - 1) == 0 for v in flags.values())


def test_struct_layouts_match_header(native):
    """The ctypes mirrors of the ABI structs have the header's sizes (C layout, x86-64)."""
    import ctypes as C
    assert C.sizeof(native.cls_gaussians) == 8 + 8 + 4 * 8 + 8          # n, degree (+pad), 4 pointers, generation
    src = open(os.path.join(ROOT, "include", "cls.h")).read()
    assert int(re.search(r"#define CLS_PROF_GROUPS (\d+)", src).group(1)) == native.CLS_PROF_GROUPS
    end = src.index("} cls_stats_t;")
    block = src[src.rindex("typedef struct {", 0, end):end]
    block = re.sub(r"/\*.*?\*/", "", block, flags=re.S)
    names = re.findall(r"\b(\w+)(?:\[\w+\])?;", block)
    assert names == [f[0] for f in native.cls_stats_t._fields_]


def test_status_strings(native):
    for code, name in native.STATUS.items():
        assert native.lib.cls_status_string(code).decode() == name


def test_create_validates_limits_without_device(native):
    h = ctypes.c_void_p()
    lim = native.cls_limits()           # all zero -> invalid
    assert native.lib.cls_create(ctypes.byref(h), 0, ctypes.byref(lim)) == 1
    assert native.lib.cls_create(None, 0, None) == 1
    assert native.lib.cls_destroy(None) == 1
    assert native.lib.cls_last_error(None).decode() == "null ctx"


def test_sm100a_code_in_library(native):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2506_21117_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "cls_oracle" not in txt, f
