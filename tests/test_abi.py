"""C ABI checks that need no GPU: libfgs.so loads and exports every entry point include/fgs.h
declares; struct layouts in the ctypes binding match the header's field order."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "fgs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fgs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libfgs():
    from paper_2409_04751_b200 import build, _lib

    build()
    return _lib.load()


def test_header_declares_entry_points():
    names = declared_functions()
    for n in ("fgs_create", "fgs_destroy", "fgs_forward", "fgs_backward", "fgs_render_host", "fgs_backward_host"):
        assert n in names


def test_library_exports_every_declared_symbol(libfgs):
    from paper_2409_04751_b200 import _lib

    exported = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", exported), name
        getattr(libfgs, name)
    assert set(_lib.EXPORTS) <= set(declared_functions())


def test_sm100a_cubin_embedded(libfgs):
    from paper_2409_04751_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_checked_library_matches_and_checks():
    """libfgs_checked.so (tests/test_checked_gpu.py) exports the same C ABI, and its kernels carry
    the device checks: more trap sites in the SASS than the product library's."""
    from paper_2409_04751_b200 import _lib

    assert os.path.exists(_lib.CHECKED_LIB_PATH), "build libfgs_checked.so"
    exported = subprocess.run(["nm", "-D", "--defined-only", _lib.CHECKED_LIB_PATH], capture_output=True,
                              text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", exported), name

    def traps(path):
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        return len(re.findall(r"\bBPT\.TRAP\b", sass))

    assert traps(_lib.CHECKED_LIB_PATH) > traps(_lib.LIB_PATH) + 20


def test_struct_layouts_match_header():
    import ctypes as C

    from paper_2409_04751_b200 import _lib

    assert C.sizeof(_lib.fgs_camera) == 4 * (3 + 4 + 9 + 3 + 1)
    assert C.sizeof(_lib.fgs_gaussians) == 8 * 6
    assert C.sizeof(_lib.fgs_gradients) == 8 * 5
    assert C.sizeof(_lib.fgs_backward_options) == 4 * 6
    hdr = open(os.path.join(ROOT, "include", "fgs.h")).read()
    body = hdr[hdr.index("typedef struct fgs_camera"):hdr.index("} fgs_camera;")]
    fields = re.findall(r"\b(model|width|height|fx|fy|cx|cy|rotation_wc|translation_wc|fov_max)\b", body)
    assert [f for f, *_ in _lib.fgs_camera._fields_] == ["model", "width", "height", "fx", "fy", "cx", "cy",
                                                          "rotation_wc", "translation_wc", "fov_max"]
    assert fields[:3] == ["model", "width", "height"]


def test_missing_library_fails_loudly(tmp_path):
    from paper_2409_04751_b200 import _lib

    saved = _lib._lib
    _lib._lib = None
    try:
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            _lib.load(str(tmp_path / "absent.so"))
    finally:
        _lib._lib = saved
